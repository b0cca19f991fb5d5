#!/usr/bin/env python
"""B200 calibration of the reference's cost model (the virtual clock's input format).

The reference fits its iteration-latency model (cost_model.hpp calibrate(), the
`calibration` key of a config) to measured anchors — batches of prefix lengths with
a measured decode-iteration time; its built-in anchors are H100 numbers from the
paper (reference_mixed_batch_anchors: 64 requests, 0/1/2/4 of them 4696 tokens
long, the rest 632).  This tool measures those anchors, and a wider set, as real
B200 decode iterations — the whole Llama-2-7B decoder stack per step (RMSNorm,
QKV + RoPE, paged attention + KV append, O + residual, RMSNorm, gate/up SiLU, down
+ residual; 32 layers, synthetic weights streamed from HBM) through the C ABI —
writes them in the reference's anchors format and fits them with the reference's
own `calibrate` (prefixsim_gpu calibrate).  The fitted constants drop into any
config's `calibration` key, so the reference's simulator prices B200 iterations.

usage: python tools/calibrate_b200.py [--out-dir gpurun_out/calib] [--reps 10]
"""
import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_23389_b200 import PagedDecodeAttention, _lib  # noqa: E402
from paper_2605_23389_b200 import linear as LIN  # noqa: E402

D, INTER, NH, L = 4096, 11008, 32, 32


def anchors():
    out = []
    for longs in (0, 1, 2, 4):  # the reference's own anchor batches (reference_mixed_batch_anchors)
        out.append([632] * (64 - longs) + [4696] * longs)
    for b, s in ((16, 1024), (16, 4096), (32, 2048), (64, 1024), (8, 8192), (128, 512)):
        out.append([s] * b)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out-dir", default=os.path.join(ROOT, "gpurun_out", "calib"))
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    os.makedirs(a.out_dir, exist_ok=True)
    dev = torch.device("cuda", 0)
    torch.manual_seed(0)

    def rnd(shape, scale):
        return ((torch.rand(shape, device=dev) * 2 - 1) * scale).to(torch.bfloat16)

    layers = [dict(wqkv=rnd((3 * D, D), 1 / math.sqrt(D)), wo=rnd((D, D), 1 / math.sqrt(D)),
                   wgu=rnd((2 * INTER, D), 1 / math.sqrt(D)), wd=rnd((D, INTER), 1 / math.sqrt(INTER)),
                   g1=(1 + rnd((D,), 0.1)), g2=(1 + rnd((D,), 0.1))) for _ in range(L)]
    att = PagedDecodeAttention(NH, NH, L, device=0)
    results = []
    for lens in anchors():
        b = len(lens)
        rows = (b + 15) // 16 * 16
        npg = [(s + 16) // 16 for s in lens]
        pool_pages = sum(npg) + 8
        usable = int(_lib.lib().asv_pool_usable_pages(C.byref(att.shape), pool_pages))
        pool = torch.empty(pool_pages * att.page_bytes // 2, dtype=torch.bfloat16, device=dev)
        pool.uniform_(-1, 1)
        perm = np.random.default_rng(b).permutation(usable)[:sum(npg)].astype(np.int32)
        indptr = np.concatenate([[0], np.cumsum(npg)]).astype(np.int32)
        plan = att.plan(lens, indptr, perm)
        h = rnd((rows, D), 1.0)
        x = torch.zeros(rows, D, dtype=torch.bfloat16, device=dev)
        act = torch.zeros(rows, INTER, dtype=torch.bfloat16, device=dev)
        q = torch.empty(rows, NH, 128, dtype=torch.bfloat16, device=dev)
        kn, vn = torch.empty_like(q), torch.empty_like(q)
        out = torch.zeros(rows, NH, 128, dtype=torch.bfloat16, device=dev)
        pos = torch.tensor(lens, dtype=torch.int32, device=dev)

        def step():
            for li, w in enumerate(layers):
                LIN.rmsnorm(h, w["g1"], x, b, 1e-5, pdl=True)
                LIN.linear(x, w["wqkv"], b, None, LIN.QKV_ROPE, positions=pos, q=q, k_out=kn, v_out=vn,
                           n_q_heads=NH, n_kv_heads=NH, pdl=True)
                att.run(q, pool, li, plan, out, k_new=kn, v_new=vn)
                LIN.linear(out.view(rows, D), w["wo"], b, h, LIN.RESIDUAL, pdl=True)
                LIN.rmsnorm(h, w["g2"], x, b, 1e-5, pdl=True)
                LIN.linear(x, w["wgu"], b, act, LIN.SILU_MUL, pdl=True)
                LIN.linear(act, w["wd"], b, h, LIN.RESIDUAL, pdl=True)

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        # one decode step = one CUDA graph (224 launches with their PDL edges): replaying it takes
        # the host's launch rate out of the measured iteration time
        run, mode = step, "eager"
        try:
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    step()
            torch.cuda.current_stream().wait_stream(s)
            g.replay()
            torch.cuda.synchronize()
            run, mode = g.replay, "graph"
        except Exception as exc:  # capture unsupported: fall back to eager launches
            print(json.dumps({"graph_capture_failed": str(exc)[:200]}), flush=True)
            torch.cuda.synchronize()
        times = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = float(np.median(times))
        kv_gb = sum(lens) * L * 2 * NH * 256 / 1e9
        results.append({"prefix_lengths": lens, "measured_ms": ms})
        print(json.dumps({"batch": b, "tokens": sum(lens), "ms": round(ms, 3), "mode": mode, "kv_gb": round(kv_gb, 2),
                          "hbm_gbps": round((kv_gb + 12.95) / (ms * 1e-3), 0)}), flush=True)
        del pool
        torch.cuda.empty_cache()
    anchors_path = os.path.join(a.out_dir, "b200_anchors.json")
    json.dump(results, open(anchors_path, "w"), indent=1)
    model_path = os.path.join(a.out_dir, "llama2_7b.json")
    json.dump({"hidden_dim": D, "num_layers": L, "bytes_per_element": 2}, open(model_path, "w"))
    cli = os.path.join(ROOT, "paper_2605_23389_b200", "prefixsim_gpu")
    r = subprocess.run([cli, "calibrate", "--anchors", anchors_path, "--model", model_path, "--out",
                        os.path.join(a.out_dir, "b200_calibration.json")], capture_output=True, text=True)
    print(r.stdout)
    if r.returncode != 0:
        print(r.stderr)
        sys.exit(r.returncode)


if __name__ == "__main__":
    main()
