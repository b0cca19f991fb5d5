#!/usr/bin/env python
"""Library comparison (tools only, never on the product path): FlashInfer's paged decode
attention (BatchDecodeWithPagedKVCacheWrapper, installed in this image) on the same shapes
as tools/attn_microbench.py — bf16 KV, 16-token pages, one layer per launch over a pool
whose pages are in random order — timed the same way (CUDA events, per layer) and reported
with the same algorithmic bytes, beside this repo's kernel.

usage: python tools/flashinfer_compare.py [--iters 10]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def flashinfer_case(n_q, n_kv, L, seq_lens, iters):
    import flashinfer
    dev = torch.device("cuda", 0)
    npages = [(s + 15) // 16 for s in seq_lens]
    P = sum(npages)
    # one pool per layer ([pages][2][n_kv][16][128], HND), L layers rotated so reads come from HBM
    pools = [torch.empty(P + 8, 2, n_kv, 16, 128, dtype=torch.bfloat16, device=dev).uniform_(-1, 1) for _ in range(L)]
    rng = np.random.default_rng(0)
    perm = torch.from_numpy(rng.permutation(P + 8)[:P].astype(np.int32)).to(dev)
    indptr = torch.from_numpy(np.concatenate([[0], np.cumsum(npages)]).astype(np.int32)).to(dev)
    last = torch.tensor([(s - 1) % 16 + 1 for s in seq_lens], dtype=torch.int32, device=dev)
    b = len(seq_lens)
    q = torch.randn(b, n_q, 128, device=dev, dtype=torch.bfloat16)
    ws = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "HND", use_tensor_cores=(n_q != n_kv))
    w.plan(indptr, perm, last, n_q, n_kv, 128, 16, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
    for l in range(L):
        w.run(q, pools[l])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        for l in range(L):
            w.run(q, pools[l])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (iters * L)
    tok = sum(seq_lens)
    alg = tok * 2 * n_kv * 128 * 2 + b * n_q * 128 * 2 * 2 + 4 * P + b * n_q * 4
    return {"us_per_layer": ms * 1e3, "GBps": alg / (ms * 1e-3) / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    import attn_microbench as M
    rng = np.random.default_rng(1)
    cases = {  # the same draws as tools/attn_microbench.py
        "C1_b16_256-2048": (32, 32, 32, rng.integers(256, 2049, 16).tolist()),
        "C2_aligned_b13_8k": (32, 32, 32, (8000 + rng.integers(0, 500, 13)).tolist()),
        "C2_b64_1k-16k": (32, 32, 8, rng.integers(1024, 16385, 64).tolist()),
        "C4_13b_gqa8_b32": (40, 8, 40, rng.integers(1024, 8192, 32).tolist()),
        "gqa_7b_b64": (32, 8, 32, rng.integers(1024, 4096, 64).tolist()),
        "mha_b1_128k": (32, 32, 4, [131072]),
        "C2_step_b4_1k-16k": (32, 32, 32, rng.integers(1024, 16385, 4).tolist()),
    }
    for name, (nq, nkv, L, seq) in cases.items():
        ours = M.run(nq, nkv, L, seq, iters=a.iters)
        try:
            fi = flashinfer_case(nq, nkv, L, seq, a.iters)
        except Exception as exc:  # JIT / API unavailable on this box
            fi = {"error": str(exc)[:200]}
        print(json.dumps({"case": name, "ours_GBps": round(ours["GBps"]), "ours_us": round(ours["us_per_layer"], 1),
                          "flashinfer_GBps": round(fi["GBps"]) if "GBps" in fi else None,
                          "flashinfer_us": round(fi["us_per_layer"], 1) if "us_per_layer" in fi else None,
                          **({"flashinfer_error": fi["error"]} if "error" in fi else {})}), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
