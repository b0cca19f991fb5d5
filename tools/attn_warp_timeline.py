#!/usr/bin/env python
"""Per-warp timeline of consecutive decode-attention launches (asv_attn_args.warp_timestamps):
for each launch, the spread of warp START times (relative to the launch's first warp) and of warp
END times (relative to its last warp), and the idle share each causes — separates the start skew of
a PDL-chained launch (its CTAs enter as the previous launch's leave) from the tail of the item
schedule.  Shapes: C4 (13B GQA-8, b32, 1K-8K) and C2 (7B MHA, b4, 1K-16K); deferred merge as the
engine's attention-only step runs it."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_23389_b200 import PagedDecodeAttention, _lib  # noqa: E402


def run(name, n_q, n_kv, L, seq, launches=12):
    dev = torch.device("cuda", 0)
    att = PagedDecodeAttention(n_q, n_kv, L, device=0)
    npages = [(s + 16) // 16 for s in seq]
    P = sum(npages)
    usable = int(_lib.lib().asv_pool_usable_pages(C.byref(att.shape), P + 8))
    pool = torch.empty((P + 8) * att.page_bytes // 2, dtype=torch.bfloat16, device=dev)
    pool.uniform_(-1, 1)
    perm = np.random.default_rng(0).permutation(usable)[:P].astype(np.int32)
    indptr = np.concatenate([[0], np.cumsum(npages)]).astype(np.int32)
    b = len(seq)
    q = torch.randn(b, n_q, 128, device=dev, dtype=torch.bfloat16)
    outs = [torch.empty_like(q) for _ in range(2)]
    plan = att.plan(seq, indptr, perm)
    W = plan.desc.num_workers
    ts = [torch.zeros(W, 2, dtype=torch.int64, device=dev) for _ in range(launches)]
    for rep in range(2):
        for i in range(launches):
            last = i == launches - 1
            att.run(q, pool, i % L, plan, outs[i % 2], defer_merge=not last,
                    prev_out=outs[(i - 1) % 2] if i > 0 else None, warp_ts=ts[i] if rep == 1 else None)
        torch.cuda.synchronize()
    print(f"{name}: {W} warps, {plan.desc.num_items} items, {plan.total_splits} splits")
    for i in range(2, launches - 1):
        t = ts[i].cpu().numpy().astype(np.float64)
        st, en = t[:, 0], t[:, 1]
        span = en.max() - st.min()
        start_idle = (st - st.min()).sum() / (W * span)
        end_idle = (en.max() - en).sum() / (W * span)
        print(f"  launch {i}: span {span / 1e3:6.1f} us | start spread p50/p90/max "
              f"{np.percentile(st - st.min(), 50) / 1e3:5.1f}/{np.percentile(st - st.min(), 90) / 1e3:5.1f}/"
              f"{(st.max() - st.min()) / 1e3:5.1f} us ({100 * start_idle:4.1f}% idle) | end spread p50/p90/max "
              f"{np.percentile(en.max() - en, 50) / 1e3:5.1f}/{np.percentile(en.max() - en, 90) / 1e3:5.1f}/"
              f"{(en.max() - en.min()) / 1e3:5.1f} us ({100 * end_idle:4.1f}% idle)")


def main():
    rng = np.random.default_rng(1)
    run("C4 13B GQA-8 b32", 40, 8, 40, rng.integers(1024, 8193, 32).tolist())
    run("C2 7B MHA b4", 32, 32, 32, rng.integers(1024, 16385, 4).tolist())


if __name__ == "__main__":
    main()
