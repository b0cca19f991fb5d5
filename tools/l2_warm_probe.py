#!/usr/bin/env python
"""Experiment: fill the decode-linear kernel boundaries' idle HBM time with the NEXT attention
launch's first-wave KV pages (L2 prefetch on a side stream, asv.h l2_warm_items).

Per iteration on the main stream: the 7B linear stack of one layer (O, gate/up, down, QKV; PDL chain,
weights rotated over 8 layers) then one C2-like decode-attention launch (batch 4, ~55K tokens,
~0.9 GB of KV; layers alternate over the pool so L2 never carries a layer over).  With warming, a
side stream prefetches the first `pages` pages of the first `items` work items of that attention
launch when the linear stack starts.  Reports us per iteration (CUDA events on the main stream) and,
separately, the attention launch alone after a completed warm (L2 benefit bound) and the linear stack
with a concurrent warm (interference)."""
import ctypes as C
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_23389_b200 import PagedDecodeAttention, _lib  # noqa: E402
from paper_2605_23389_b200 import linear as L  # noqa: E402

D, INTER, NQ = 4096, 11008, 32


def main():
    dev = torch.device("cuda", 0)
    torch.manual_seed(0)
    nl = 8
    batch = 4
    rows = 16

    def w(n, k):
        return ((torch.rand(n, k, device=dev) * 2 - 1) / math.sqrt(k)).to(torch.bfloat16)

    layers = [dict(o=w(D, D), gu=w(2 * INTER, D), down=w(D, INTER), qkv=w(3 * D, D)) for _ in range(nl)]
    attn_x = (torch.rand(rows, D, device=dev) * 2 - 1).to(torch.bfloat16)
    h = (torch.rand(rows, D, device=dev) * 2 - 1).to(torch.bfloat16)
    act = torch.zeros(rows, INTER, dtype=torch.bfloat16, device=dev)
    ss_a = torch.zeros(2 * D // 128, rows, dtype=torch.float32, device=dev)
    ss_b = torch.zeros(2 * D // 128, rows, dtype=torch.float32, device=dev)
    pos = torch.arange(batch, dtype=torch.int32, device=dev) + 1000
    qb = torch.zeros(batch, NQ, 128, dtype=torch.bfloat16, device=dev)
    kk = torch.zeros(batch, NQ, 128, dtype=torch.bfloat16, device=dev)
    vv = torch.zeros(batch, NQ, 128, dtype=torch.bfloat16, device=dev)

    def lin_stack(l):
        ly = layers[l % nl]
        L.linear(attn_x, ly["o"], batch, h, L.RESIDUAL, ss_out=ss_b, pdl=True)
        L.linear(h, ly["gu"], batch, act, L.SILU_MUL, ss_in=ss_b, pdl=True)
        L.linear(act, ly["down"], batch, h, L.RESIDUAL, ss_out=ss_a, pdl=True)
        L.linear(h, ly["qkv"], batch, None, L.QKV_ROPE, positions=pos, q=qb, k_out=kk, v_out=vv,
                 n_q_heads=NQ, n_kv_heads=NQ, ss_in=ss_a, pdl=True)

    # attention: 2-layer pool, C2-like batch
    AL = 2
    att = PagedDecodeAttention(NQ, NQ, AL, device=0)
    seq = [16000, 14000, 12500, 13000]
    npages = [(s + 16) // 16 for s in seq]
    P = sum(npages)
    pool_pages = P + 8
    usable = int(_lib.lib().asv_pool_usable_pages(C.byref(att.shape), pool_pages))
    pool = torch.empty(pool_pages * att.page_bytes // 2, dtype=torch.bfloat16, device=dev)
    pool.uniform_(-1, 1)
    perm = np.random.default_rng(0).permutation(usable)[:P].astype(np.int32)
    indptr = np.concatenate([[0], np.cumsum(npages)]).astype(np.int32)
    q = torch.randn(batch, NQ, 128, device=dev, dtype=torch.bfloat16)
    out = torch.empty_like(q)
    plan = att.plan(seq, indptr, perm)
    kv_mb = sum(seq) * 2 * NQ * 256 / 1e6
    workers = plan.desc.num_workers
    side = torch.cuda.Stream(device=dev)
    main_s = torch.cuda.current_stream()

    def iteration(i, items, pages):
        if items > 0:
            ev = torch.cuda.Event()
            ev.record(main_s)
            side.wait_event(ev)
            att.l2_warm(q, pool, i % AL, plan, out, items, pages, stream=side)
        lin_stack(i)
        att.run(q, pool, i % AL, plan, out)

    def timed(fn, n=24):
        for i in range(4):
            fn(i)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main_s)
        for i in range(n):
            fn(i)
        b.record(main_s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e3 / n

    res = {"kv_mb_per_launch": round(kv_mb, 1), "workers": workers, "items": plan.desc.num_items}
    res["lin_only_us"] = round(timed(lambda i: lin_stack(i)), 2)
    res["attn_only_us"] = round(timed(lambda i: att.run(q, pool, i % AL, plan, out)), 2)
    res["base_us"] = round(timed(lambda i: iteration(i, 0, 0)), 2)
    for items_f, pages in [(1, 2), (1, 4), (1, 8), (2, 4), (1, 16)]:
        items = workers * items_f
        mb = items * pages * 8192 / 1e6
        key = f"warm_{items}x{pages}_{mb:.0f}MB"
        res[key] = round(timed(lambda i: iteration(i, items, pages)), 2)

        def warmed_attn(i):  # warm completes first, then attention alone: the L2 benefit bound
            att.l2_warm(q, pool, i % AL, plan, out, items, pages)
            att.run(q, pool, i % AL, plan, out)
        res[key + "_attn_after_warm_us"] = round(timed(warmed_attn) - 0.0, 2)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
