#!/usr/bin/env python
"""Streaming-read HBM ceiling on this B200 (tools only; see tools/probe/hbm_read_probe.cu):
LDG.128 grid-stride reads and the decode kernel's producer pattern (per-warp rings of 4 KiB
cp.async.bulk loads), over an 8 GiB buffer (>> L2), timed with CUDA events."""
import ctypes as C
import json
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    so = os.path.join(ROOT, "tools", "probe", "_hbm_read_probe.so")
    h = C.CDLL(so)
    dev = torch.device("cuda", 0)
    nbytes = int(os.environ.get("PROBE_MIB", 8192)) << 20
    buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    buf.fill_(1)
    out = torch.zeros(1, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream()
    sms = torch.cuda.get_device_properties(0).multi_processor_count

    def timed(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(reps):
            a.record(st)
            fn()
            b.record(st)
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        return round(nbytes / (best * 1e-3) / 1e9, 1)

    h.probe_bulk.restype = C.c_int
    h.probe_ldg.restype = C.c_int

    res = {}
    only_bulk = os.environ.get("ONLY_BULK")
    for k in (() if only_bulk else (4, 8, 16)):
        res[f"ldg_{k}ctas_per_sm"] = timed(lambda: h.probe_ldg(C.c_void_p(buf.data_ptr()), C.c_int64(nbytes),
                                                                 C.c_void_p(out.data_ptr()), sms * k,
                                                                 C.c_void_p(st.cuda_stream)))
    for cps, stages in ((2, 3 if False else 4), (2, 6), (2, 12), (3, 4), (4, 4), (4, 8), (2, 2)):
        res[f"bulk4k_{cps}cta_{stages}st"] = timed(
            lambda: h.probe_bulk(C.c_void_p(buf.data_ptr()), C.c_int64(nbytes), C.c_void_p(out.data_ptr()), cps,
                                 stages, C.c_void_p(st.cuda_stream)))
    # torch copy (the driver's MEASURED_PEAKS method: read + write bytes)
    half = nbytes // 2
    src, dst = buf[:half], buf[half:]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dst.copy_(src)
    best = 1e9
    for _ in range(10):
        a.record(st)
        dst.copy_(src)
        b.record(st)
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    res["torch_copy_read_plus_write"] = round(2 * half / (best * 1e-3) / 1e9, 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
