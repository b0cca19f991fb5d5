"""Decode-attention kernel microbenchmark (per-layer launches over an L-layer pool).

Reports algorithmic HBM GB/s = (K+V bytes of every attended token + q + out + page
indices) / kernel time, timed with CUDA events on the launching stream.
"""
import argparse
import json
import math
import time

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_23389_b200 import PagedDecodeAttention


def run(n_q, n_kv, L, seq_lens, iters=20, warmup=3, num_workers=None, seed=0, dtype=torch.bfloat16):
    dev = torch.device("cuda", 0)
    att = PagedDecodeAttention(n_q, n_kv, L, device=0, dtype=dtype)
    npages = [(s + 16) // 16 for s in seq_lens]
    P = sum(npages)
    # grouped layer-major pool: page ids must stay below asv_pool_usable_pages (include/asv.h)
    import ctypes as C
    from paper_2605_23389_b200 import _lib
    pool_pages = P + 8
    usable = int(_lib.lib().asv_pool_usable_pages(C.byref(att.shape), pool_pages))
    assert usable >= P
    pool = torch.empty(pool_pages * att.page_bytes // 2, dtype=dtype, device=dev)
    pool.uniform_(-1, 1)
    rng = np.random.default_rng(seed)
    perm = rng.permutation(usable)[:P].astype(np.int32)
    indptr = np.concatenate([[0], np.cumsum(npages)]).astype(np.int32)
    b = len(seq_lens)
    q = torch.randn(b, n_q, 128, device=dev, dtype=dtype)
    out = torch.empty_like(q)
    lse = torch.empty(b, n_q, device=dev)
    plan = att.plan(seq_lens, indptr, perm, num_workers=num_workers)
    st = torch.cuda.current_stream()
    for i in range(warmup):
        for l in range(L):
            att.run(q, pool, l, plan, out, lse)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(iters):
        for l in range(L):
            att.run(q, pool, l, plan, out, lse)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (iters * L)
    tok = sum(seq_lens)
    kv_bytes = tok * 2 * n_kv * 128 * 2
    alg = kv_bytes + b * n_q * 128 * 2 * 2 + 4 * P + b * n_q * 4
    return {"n_q": n_q, "n_kv": n_kv, "b": b, "tokens": tok, "splits": plan.total_splits,
            "items": plan.desc.num_items, "workers": plan.desc.num_workers,
            "us_per_layer": ms * 1e3, "GBps": alg / (ms * 1e-3) / 1e9, "alg_bytes": alg}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--case", default=None)
    ap.add_argument("--fp16", action="store_true", help="fp16 KV / q / out instead of bf16")
    a = ap.parse_args()
    rng = np.random.default_rng(1)
    cases = {
        "C1_b16_256-2048": (32, 32, 32, rng.integers(256, 2049, 16).tolist()),
        "C2_aligned_b13_8k": (32, 32, 32, (8000 + rng.integers(0, 500, 13)).tolist()),
        "C2_b64_1k-16k": (32, 32, 8, rng.integers(1024, 16385, 64).tolist()),
        "C4_13b_gqa8_b32": (40, 8, 40, rng.integers(1024, 8192, 32).tolist()),
        "gqa_7b_b64": (32, 8, 32, rng.integers(1024, 4096, 64).tolist()),
        "mha_b1_128k": (32, 32, 4, [131072]),
        "C2_step_b4_1k-16k": (32, 32, 32, rng.integers(1024, 16385, 4).tolist()),
        # same launches with one layer per page: page stride 64 KiB / 256 KiB instead of
        # 2.5 MiB / 8 MiB (probes address-stride / TLB effects of the all-layers page)
        "C4_13b_gqa8_b32_L1": (40, 8, 1, None),
        "C2_aligned_b13_8k_L1": (32, 32, 1, None),
    }
    cases["C4_13b_gqa8_b32_L1"] = (40, 8, 1, cases["C4_13b_gqa8_b32"][3])
    # same KV bytes and work items as C4 with one query head per kv head (FHFMA path):
    # isolates the GQA tensor-core path's cost from the memory system's
    cases["C4_shape_mha8_b32"] = (8, 8, 40, cases["C4_13b_gqa8_b32"][3])
    cases["C2_aligned_b13_8k_L1"] = (32, 32, 1, cases["C2_aligned_b13_8k"][3])
    for name, (nq, nkv, L, seq) in cases.items():
        if a.case and a.case != name:
            continue
        r = run(nq, nkv, L, seq, iters=a.iters, warmup=a.warmup,
                dtype=torch.float16 if a.fp16 else torch.bfloat16)
        r["case"] = name
        r["dtype"] = "fp16" if a.fp16 else "bf16"
        print(json.dumps(r), flush=True)
