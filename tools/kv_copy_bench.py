#!/usr/bin/env python
"""Microbenchmark of the KV page moves (asv_kv_copy_h2d / d2h) against plain
1-D pinned copies of the same bytes (measurement tool, not product code).

Moves `n` requests of random lengths (7B MHA shape, 32 layers: 8 MiB pages)
from a pinned page-major host arena into the layer-major device pool and
reports GB/s for: whole pages only, valid-rows-only partial pages, and mixed
requests, next to one 1-D copy per 8 MiB page.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_23389_b200 import _lib  # noqa: E402


def main():
    h = _lib.lib()
    n_kv, L = int(os.environ.get("NKV", 32)), int(os.environ.get("LAYERS", 32))
    shape = _lib.AttnShape(n_kv, n_kv, 128, 16, L)
    pb = L * 2 * n_kv * 4096
    dev = torch.device("cuda", 0)
    host_pages = 512
    host = torch.empty(host_pages * pb, dtype=torch.uint8, pin_memory=True)
    host.fill_(3)
    pool_pages = int(os.environ.get("POOL_PAGES", 1024))  # device pitch of a layer = pool_pages * slice
    pool = torch.empty(pool_pages * pb, dtype=torch.uint8, device=dev)
    st = torch.cuda.Stream(dev)
    rng = np.random.default_rng(0)
    res = {"page_bytes": pb, "pool_pages": pool_pages, "layer_pitch_bytes": pool_pages * pb // L}

    def run(lens, direction):
        fn = h.asv_kv_copy_h2d if direction == "h2d" else h.asv_kv_copy_d2h
        total = 0
        beg, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        beg.record(st)
        k = 0
        import time
        t_issue = 0.0
        for s in lens:
            npg = (s + 15) // 16
            pages = rng.permutation(pool_pages)[:npg].astype(np.int32)
            ptrs = (C.c_void_p * npg)(*[host.data_ptr() + ((k + j) % host_pages) * pb for j in range(npg)])
            k += npg
            moved = C.c_int64(0)
            pp = pages.ctypes.data_as(C.POINTER(C.c_int32))
            t0 = time.perf_counter()
            _lib.check(fn(C.byref(shape), pool.data_ptr(), pool_pages, pp, s, ptrs, st.cuda_stream, C.byref(moved)))
            t_issue += time.perf_counter() - t0
            total += moved.value
        end.record(st)
        end.synchronize()
        ms = beg.elapsed_time(end)
        npages = sum((x + 15) // 16 for x in lens)
        return total / (ms * 1e-3) / 1e9, ms, t_issue * 1e6 / npages

    def plain(npages):
        beg, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            beg.record(st)
            for j in range(npages):
                pool[(j % pool_pages) * pb:(j % pool_pages + 1) * pb].copy_(
                    host[(j % host_pages) * pb:(j % host_pages + 1) * pb], non_blocking=True)
            end.record(st)
        end.synchronize()
        return npages * pb / (beg.elapsed_time(end) * 1e-3) / 1e9

    def d2d(lens):
        """device -> device request moves between two pools (the pair's admit path, one device)"""
        pool2 = torch.empty(pool_pages * pb, dtype=torch.uint8, device=dev)
        total = 0
        beg, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        beg.record(st)
        for s in lens:
            npg = (s + 15) // 16
            sp = rng.permutation(pool_pages)[:npg].astype(np.int32)
            dp = rng.permutation(pool_pages)[:npg].astype(np.int32)
            moved = C.c_int64(0)
            _lib.check(h.asv_kv_copy_d2d(C.byref(shape), pool2.data_ptr(), pool_pages, 0,
                                         dp.ctypes.data_as(C.POINTER(C.c_int32)), pool.data_ptr(), pool_pages, 0,
                                         sp.ctypes.data_as(C.POINTER(C.c_int32)), s, st.cuda_stream, C.byref(moved)))
            total += moved.value
        end.record(st)
        end.synchronize()
        del pool2
        return round(total / (beg.elapsed_time(end) * 1e-3) / 1e9, 1)

    if os.environ.get("D2D"):
        d2d([16 * 8] * 4)
        res["d2d_full_pages_16x256tok"] = d2d([16 * 16] * 16)
        res["d2d_mixed_1k_8k"] = d2d(rng.integers(1024, 8192, 16).tolist())
        res["d2d_partial_rows"] = d2d([7] * 64)
        print(json.dumps(res))
        return
    plain(8)
    res["plain_1d_8MiB_pages_h2d"] = round(plain(256), 2)
    if os.environ.get("QUICK"):
        run([16 * 8] * 4, "h2d")
        res["h2d_full_pages"] = [round(x, 2) for x in run([16 * 16] * 16, "h2d")]
        print(json.dumps(res))
        return
    for direction in ("h2d", "d2h"):
        run([16 * 8] * 4, direction)
        res[f"{direction}_full_pages"] = [round(x, 2) for x in run([16 * 16] * 16, direction)]
        res[f"{direction}_partial_only_8rows"] = [round(x, 2) for x in run([8] * 256, direction)]
        res[f"{direction}_partial_only_1row"] = [round(x, 2) for x in run([1] * 256, direction)]
        lens = rng.integers(1024, 4096, 64).tolist()
        res[f"{direction}_mixed_1k_4k"] = [round(x, 2) for x in run(lens, direction)]
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
