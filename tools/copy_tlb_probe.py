#!/usr/bin/env python
"""Copy-engine throughput vs destination address span (measurement tool).

The layer-major device pool puts the 32 layer slices of one 8 MiB KV page
pool_pages * 256 KiB apart; a 2-D H2D copy of a page then writes 32 rows
scattered over the whole pool.  This probe measures, over pools of growing
size (random page positions):
  2d_h2d    : one 2-D copy per page (32 x 256 KiB rows, pitch = layer slab)
  1d_h2d_rows: 32 separate 1-D 256 KiB copies per page
  1d_h2d_page: one 1-D 8 MiB copy per page (page-major layout)
  stage_d2d : 1-D H2D into a staging buffer + one 2-D D2D scatter copy per page
  d2d_2d    : the 2-D D2D scatter alone (copy-engine, HBM -> HBM)
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np
import torch

rt = C.CDLL("libcudart.so.12")
rt.cudaMemcpy2DAsync.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t,
                                 C.c_int, C.c_void_p]
rt.cudaMemcpyAsync.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]
H2D, D2D = 1, 3


def main():
    L, slice_ = 32, 256 << 10
    pb = L * slice_
    dev = torch.device("cuda", 0)
    host_pages = 256
    host = torch.empty(host_pages * pb, dtype=torch.uint8, pin_memory=True)
    host.fill_(1)
    stage = torch.empty(64 * pb, dtype=torch.uint8, device=dev)
    st = torch.cuda.Stream(dev)
    sp = st.cuda_stream
    rng = np.random.default_rng(0)
    out = []
    for pool_pages in [int(x) for x in os.environ.get("POOLS", "512,2048,4096,8192,16384").split(",")]:
        pool = torch.empty(pool_pages * pb, dtype=torch.uint8, device=dev)
        base = pool.data_ptr()
        pitch = pool_pages * slice_
        n = 96
        pages = rng.permutation(pool_pages)[:n]
        row = {"pool_pages": pool_pages, "pool_GiB": pool_pages * pb / 2**30}

        def timed(fn, nbytes):
            fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            b.synchronize()
            return round(nbytes / (a.elapsed_time(b) * 1e-3) / 1e9, 2)

        def c2d():
            for j, p in enumerate(pages):
                rt.cudaMemcpy2DAsync(base + int(p) * slice_, pitch, host.data_ptr() + (j % host_pages) * pb, slice_,
                                     slice_, L, H2D, sp)

        def rows1d():
            for j, p in enumerate(pages):
                for l in range(L):
                    rt.cudaMemcpyAsync(base + l * pitch + int(p) * slice_,
                                       host.data_ptr() + (j % host_pages) * pb + l * slice_, slice_, H2D, sp)

        def page1d():
            for j, p in enumerate(pages):
                rt.cudaMemcpyAsync(base + int(p) * pb, host.data_ptr() + (j % host_pages) * pb, pb, H2D, sp)

        def staged():
            for j, p in enumerate(pages):
                s = stage.data_ptr() + (j % 64) * pb
                rt.cudaMemcpyAsync(s, host.data_ptr() + (j % host_pages) * pb, pb, H2D, sp)
                rt.cudaMemcpy2DAsync(base + int(p) * slice_, pitch, s, slice_, slice_, L, D2D, sp)

        def d2d():
            for j, p in enumerate(pages):
                s = stage.data_ptr() + (j % 64) * pb
                rt.cudaMemcpy2DAsync(base + int(p) * slice_, pitch, s, slice_, slice_, L, D2D, sp)

        nb = n * pb
        row["2d_h2d"] = timed(c2d, nb)
        row["1d_h2d_rows"] = timed(rows1d, nb)
        row["1d_h2d_page"] = timed(page1d, nb)
        row["stage_d2d"] = timed(staged, nb)
        row["d2d_2d"] = timed(d2d, nb)
        out.append(row)
        print(json.dumps(row), flush=True)
        del pool
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
