#!/usr/bin/env python
"""Decode-step linear layers (asv_linear, tcgen05) microbenchmark: Llama-2-7B / 13B
projection shapes at decode batch sizes.  Reports time per call (CUDA events on
the launching stream, weights rotated across calls so each launch streams its
weights from HBM, not L2) and the weight-streaming rate (algorithmic bytes =
weights + activations in + outputs) vs the measured HBM peak."""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_23389_b200 import linear as L  # noqa: E402

SHAPES = {  # name: (n_out, k, epilogue)
    "7b.qkv": (3 * 4096, 4096, L.QKV_ROPE),
    "7b.o": (4096, 4096, L.RESIDUAL),
    "7b.gate_up": (2 * 11008, 4096, L.SILU_MUL),
    "7b.down": (4096, 11008, L.RESIDUAL),
}


def bench(name, n_out, k, epi, batch, copies=8, iters=20):
    dev = torch.device("cuda", 0)
    ws = [((torch.rand(n_out, k, device=dev) * 2 - 1) / math.sqrt(k)).to(torch.bfloat16) for _ in range(copies)]
    rows = (batch + 15) // 16 * 16
    x = (torch.rand(rows, k, device=dev) * 2 - 1).to(torch.bfloat16)
    out_n = n_out // 2 if epi == L.SILU_MUL else n_out
    y = torch.zeros(batch, out_n, dtype=torch.bfloat16, device=dev)
    kw = {}
    if epi == L.QKV_ROPE:
        kw = dict(positions=torch.arange(batch, dtype=torch.int32, device=dev) + 1000,
                  q=torch.empty(batch, 32, 128, dtype=torch.bfloat16, device=dev),
                  k_out=torch.empty(batch, 32, 128, dtype=torch.bfloat16, device=dev),
                  v_out=torch.empty(batch, 32, 128, dtype=torch.bfloat16, device=dev), n_q_heads=32, n_kv_heads=32)
    kw["pdl"] = os.environ.get("PDL", "1") == "1"
    for i in range(3):
        L.linear(x, ws[i % copies], batch, y if epi != L.QKV_ROPE else None, epi, **kw)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(iters):
        L.linear(x, ws[i % copies], batch, y if epi != L.QKV_ROPE else None, epi, **kw)
    b.record()
    b.synchronize()
    us = a.elapsed_time(b) * 1e3 / iters
    alg = n_out * k * 2 + batch * k * 2 + batch * out_n * 2 * (2 if epi == L.RESIDUAL else 1)
    return {"shape": name, "batch": batch, "us": round(us, 2), "GBps": round(alg / (us * 1e-6) / 1e9, 1),
            "tflops": round(2 * n_out * k * batch / (us * 1e-6) / 1e12, 2)}


def main():
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs", 6450.0)
    out = []
    for batch in [int(b) for b in os.environ.get("BATCHES", "4,16,64,128").split(",")]:
        for name, (n, k, epi) in SHAPES.items():
            r = bench(name, n, k, epi, batch)
            r["frac_hbm"] = round(r["GBps"] / peak, 3)
            out.append(r)
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
