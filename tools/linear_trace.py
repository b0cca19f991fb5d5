#!/usr/bin/env python
"""Timeline of the per-GEMM decode linear stack (asv_linear, decode_gemm.cu): 4 layers x (O+res,
gate/up+SiLU, down+res, next QKV+RoPE), PDL-chained as the engine runs them; for each launch of the
last two layers, the spread over CTAs of the %globaltimer stamps (entry, dependency satisfied, last
weight load issued, first stage landed, accumulator complete, reduce entered, exit) relative to the
first layer's first entry, plus the HBM-idle estimate at each boundary (next launch's first landed
stage - this launch's last accumulator).  Env: BATCH (default 4)."""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_23389_b200 import linear as L  # noqa: E402

D, INTER, NQ = 4096, 11008, 32
NAMES = ["entry", "dep_ok", "issued", "landed", "acc_done", "reduce", "exit"]


def main():
    dev = torch.device("cuda", 0)
    batch = int(os.environ.get("BATCH", "4"))
    nl = 8
    rows = (batch + 15) // 16 * 16

    def w(n, k, seed):
        g = torch.Generator(device=dev).manual_seed(seed)
        return ((torch.rand(n, k, device=dev, generator=g) * 2 - 1) / math.sqrt(k)).to(torch.bfloat16)

    layers = [dict(o=w(D, D, 10 * l), gu=w(2 * INTER, D, 10 * l + 1), down=w(D, INTER, 10 * l + 2),
                   qkv=w(128 * 3 * NQ, D, 10 * l + 3)) for l in range(nl)]
    attn = (torch.rand(rows, D, device=dev) * 2 - 1).to(torch.bfloat16)
    h = (torch.rand(rows, D, device=dev) * 2 - 1).to(torch.bfloat16)
    act = torch.zeros(rows, INTER, dtype=torch.bfloat16, device=dev)
    ss_a = torch.zeros(2 * D // 128, rows, dtype=torch.float32, device=dev)
    ss_b = torch.zeros(2 * D // 128, rows, dtype=torch.float32, device=dev)
    pos = torch.arange(batch, dtype=torch.int32, device=dev) + 1000
    q = torch.zeros(batch, NQ, 128, dtype=torch.bfloat16, device=dev)
    kk = torch.zeros(batch, NQ, 128, dtype=torch.bfloat16, device=dev)
    v = torch.zeros(batch, NQ, 128, dtype=torch.bfloat16, device=dev)

    def phases(l):
        ly = layers[l % nl]
        return [dict(x=attn, w=ly["o"], batch=batch, y=h, epilogue=L.RESIDUAL, ss_out=ss_b, pdl=True),
                dict(x=h, w=ly["gu"], batch=batch, y=act, epilogue=L.SILU_MUL, ss_in=ss_b, pdl=True),
                dict(x=act, w=ly["down"], batch=batch, y=h, epilogue=L.RESIDUAL, ss_out=ss_a, pdl=True),
                dict(x=h, w=ly["qkv"], batch=batch, epilogue=L.QKV_ROPE, positions=pos, q=q, k_out=kk, v_out=v,
                     n_q_heads=NQ, n_kv_heads=NQ, ss_in=ss_a, pdl=True)]

    for l in range(nl):  # warm
        for p in phases(l):
            L.linear(**p)
    torch.cuda.synchronize()
    for rep in range(2):
        L.linear_trace(True)
        h.uniform_(-1, 1)
        for l in range(nl):
            for p in phases(l):
                L.linear(**p)
        torch.cuda.synchronize()
    tr = L.linear_trace().astype(np.float64)  # [launches][512][8]
    L.linear_trace(False)
    names = ["O+res", "gate/up", "down+res", "QKV+rope"]
    ent = tr[:, :, 0]
    valid = ent > 0
    t0 = ent[valid].min()
    grids = valid.sum(axis=1)
    print(f"batch {batch}; us since the first launch's first CTA entry (min / median / max over CTAs)")
    prev_acc = None
    gaps = []
    for li in range(tr.shape[0]):
        g = int(grids[li])
        rel = (tr[li, :g, :7] - t0) / 1e3
        rel[tr[li, :g, :7] == 0] = np.nan
        parts = []
        for k, nm in enumerate(NAMES):
            col = rel[:, k]
            col = col[~np.isnan(col)]
            if col.size:
                parts.append(f"{nm} {col.min():6.1f}/{np.median(col):6.1f}/{col.max():6.1f}")
        landed_min = np.nanmin(rel[:, 3]) if g else np.nan
        if prev_acc is not None:
            gaps.append(landed_min - prev_acc)
        prev_acc = np.nanmax(rel[:, 4])
        if li >= tr.shape[0] - 8:
            sms = np.unique(tr[li, :g, 7]).size
            print(f"  L{li // 4} {names[li % 4]:9s} grid {g:3d} on {sms:3d} SMs | " + " | ".join(parts))
    per_layer = ((np.nanmax(tr[-1, :, 6]) - np.nanmin(np.where(tr[-8, :, 0] > 0, tr[-8, :, 0], np.nan))) / 1e3) / 2
    print(f"per layer (last two layers, entry to exit): {per_layer:.1f} us")
    print("boundary: next launch's first landed stage - this launch's last accumulator (us): "
          + " ".join(f"{x:.1f}" for x in gaps[-8:]))


if __name__ == "__main__":
    main()
