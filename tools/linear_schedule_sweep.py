#!/usr/bin/env python
"""Sweep of the decode-linear schedule (asv_linear_set_schedule: K splits = cluster size, ring stages)
on the Llama-2-7B projections at decode batches: time per call in a PDL chain of the same GEMM
(weights rotated past L2, as tools/linear_microbench.py), every valid (splits, stages).  Prints one
JSON line per shape/batch with the automatic schedule's time and the best forced one.
Env: BATCHES (default 4,16,64), SHAPES (default all 7B)."""
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from paper_2605_23389_b200 import _lib  # noqa: E402
import linear_microbench as M  # noqa: E402


def smem_for(bn, st):
    ring = st * (16384 + bn * 128)
    return max(ring, bn * 512) + 1024 + 17 * 8 + 16 + 1024 + 16 + 2048


def main():
    h = _lib.lib()
    shapes = os.environ.get("SHAPES", ",".join(M.SHAPES)).split(",")
    for batch in [int(b) for b in os.environ.get("BATCHES", "4,16,64").split(",")]:
        bn = (batch + 15) // 16 * 16
        for name in shapes:
            n, k, epi = M.SHAPES[name]
            kbs = k // 64
            _lib.check(h.asv_linear_set_schedule(0, 0))
            auto = M.bench(name, n, k, epi, batch, iters=30)["us"]
            res = []
            for sp in range(1, 9):
                per = -(-kbs // sp)
                if (sp > 1 and per < 2) or -(-kbs // per) != sp:
                    continue
                for st in range(2, 9):
                    if smem_for(bn, st) > 227 * 1024:
                        break
                    _lib.check(h.asv_linear_set_schedule(sp, st))
                    us = M.bench(name, n, k, epi, batch, iters=30)["us"]
                    per_sm = 233472 // (smem_for(bn, st) + 1024)
                    res.append({"splits": sp, "stages": st, "us": us, "ctas": n // 128 * sp, "per_sm": per_sm})
            _lib.check(h.asv_linear_set_schedule(0, 0))
            res.sort(key=lambda r: r["us"])
            print(json.dumps({"shape": name, "batch": batch, "auto_us": auto, "best": res[:4],
                              "all": sorted(res, key=lambda r: (r["splits"], r["stages"]))}), flush=True)


if __name__ == "__main__":
    main()
