#!/usr/bin/env python
"""The bench's first timed decode iteration as a standalone, profileable launch sequence.

Takes the batch (prefix lengths, running order) of iteration S+W of the C2 trace from the
engine's decision log, lays it out on a resident 32-layer pool (pages in random order), plans it
once and runs the 32 layer launches three times (PDL chained, KV append on).  Under
`ncu --set full -k regex:decode_attn --launch-skip 32 --launch-count 1` the profiled launch is one
layer of that iteration; its ALGORITHMIC bytes (the bench's per-launch formula: K+V of every
attended token + q + out + appended rows + plan) are written to gpurun_out/ncu_launch_alg.json so
tools/ncu_summarize.py can put the launch's DRAM traffic beside its own algorithmic bytes.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_23389_b200 import PagedDecodeAttention, engine  # noqa: E402

ITER = int(os.environ.get("ITER", 305))  # bench.py STEADY_START + warmup (first timed iteration)


def main():
    cfg = engine.load_config(os.path.join(ROOT, "configs", "c2_7b_1024req.json"))
    log = engine.run_config_jsonl(cfg)
    its = [json.loads(l) for l in log.splitlines()[1:] if '"type":"iteration"' in l]
    lens = [int(x) for x in its[ITER]["prefix_lengths"]]
    n_q = n_kv = 32
    L = 32
    att = PagedDecodeAttention(n_q, n_kv, L, device=0)
    npages = [(s + 16) // 16 for s in lens]
    P = sum(npages)
    dev = torch.device("cuda", 0)
    pool = torch.empty((P + 8) * att.page_bytes // 2, dtype=torch.bfloat16, device=dev)
    pool.uniform_(-1, 1)
    perm = np.random.default_rng(0).permutation(P).astype(np.int32)
    indptr = np.concatenate([[0], np.cumsum(npages)]).astype(np.int32)
    b = len(lens)
    q = torch.randn(b, n_q, 128, device=dev, dtype=torch.bfloat16)
    kn = torch.randn(b, n_kv, 128, device=dev, dtype=torch.bfloat16)
    vn = torch.randn(b, n_kv, 128, device=dev, dtype=torch.bfloat16)
    out = torch.empty_like(q)
    plan = att.plan(lens, indptr, perm)
    for _ in range(3):
        for l in range(L):
            att.run(q, pool, l, plan, out, k_new=kn, v_new=vn)
    torch.cuda.synchronize()
    tok = sum(lens)
    alg = tok * 2 * n_kv * 256 + b * n_q * 512 + b * 2 * n_kv * 256 + plan.desc.total_int32 * 4 / L
    rec = {"iteration": ITER, "batch": b, "tokens": tok, "alg_bytes_per_launch": alg,
           "plan_int32": plan.desc.total_int32, "splits": plan.total_splits}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "ncu_launch_alg.json"), "w") as f:
        json.dump(rec, f)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
