#!/usr/bin/env python
"""Library comparison (tools only): the decode linear layers (asv_linear, tcgen05 swap-AB) vs
cuBLAS through torch.matmul on the Llama-2-7B projection shapes at decode batch sizes; plain
STORE epilogue for both, weights rotated over 8 copies so every call streams them from HBM."""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_23389_b200 import linear as L  # noqa: E402

SHAPES = {"7b.qkv": (3 * 4096, 4096), "7b.o": (4096, 4096), "7b.gate_up": (2 * 11008, 4096), "7b.down": (4096, 11008)}


def timed(fn, iters=20):
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(iters):
        fn(i)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / iters


def main():
    dev = torch.device("cuda", 0)
    for batch in (1, 4, 16, 64):
        for name, (n, k) in SHAPES.items():
            ws = [((torch.rand(n, k, device=dev) * 2 - 1) / math.sqrt(k)).to(torch.bfloat16) for _ in range(8)]
            rows = (batch + 15) // 16 * 16
            x = (torch.rand(rows, k, device=dev) * 2 - 1).to(torch.bfloat16)
            y = torch.empty(batch, n, dtype=torch.bfloat16, device=dev)
            ours = timed(lambda i: L.linear(x, ws[i % 8], batch, y, L.STORE, pdl=True))
            xb = x[:batch]
            lib = timed(lambda i: torch.matmul(xb, ws[i % 8].t(), out=y))
            gb = n * k * 2 / 1e9
            print(json.dumps({"shape": name, "batch": batch, "ours_us": round(ours, 2), "cublas_us": round(lib, 2),
                              "ours_GBps": round(gb / (ours * 1e-6)), "cublas_GBps": round(gb / (lib * 1e-6)),
                              "speedup": round(lib / ours, 2)}), flush=True)
            del ws


if __name__ == "__main__":
    main()
