#!/usr/bin/env python
"""Timeline of one persistent GEMM-chain launch (asv_linear_chain, decode_chain.cu): per phase, the
spread over CTAs of the %globaltimer stamps (dependency satisfied, last unit issued, first / last
segment accumulated, contributors complete, phase finished), relative to the launch's first stamp.
Env: BATCH (default 4)."""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_23389_b200 import linear as L  # noqa: E402

D, INTER, NQ = 4096, 11008, 32
NAMES = ["dep_ok", "issued", "seg_first", "seg_last", "contrib", "finished"]
# cluster split-K chain (default kernel) slots: producer dependency satisfied, first tile accumulated,
# a later tile accumulated, last tile written, phase signalled
NAMES2 = ["dep_ok", "tile1_acc", "tileN_acc", "last_done", "signaled", "-"]
if os.environ.get("ASV_CHAIN_KIND") != "streamk":
    NAMES = NAMES2


def main():
    dev = torch.device("cuda", 0)
    batch = int(os.environ.get("BATCH", "4"))
    rows = (batch + 15) // 16 * 16

    def w(n, k, seed):
        g = torch.Generator(device=dev).manual_seed(seed)
        return ((torch.rand(n, k, device=dev, generator=g) * 2 - 1) / math.sqrt(k)).to(torch.bfloat16)

    layers = [dict(o=w(D, D, 10 * l), gu=w(2 * INTER, D, 10 * l + 1), down=w(D, INTER, 10 * l + 2),
                   qkv=w(128 * 3 * NQ, D, 10 * l + 3)) for l in range(4)]
    attn = (torch.rand(rows, D, device=dev) * 2 - 1).to(torch.bfloat16)
    h = (torch.rand(rows, D, device=dev) * 2 - 1).to(torch.bfloat16)
    act = torch.zeros(rows, INTER, dtype=torch.bfloat16, device=dev)
    ss_a = torch.zeros(2 * D // 128, rows, dtype=torch.float32, device=dev)
    ss_b = torch.zeros(2 * D // 128, rows, dtype=torch.float32, device=dev)
    pos = torch.arange(batch, dtype=torch.int32, device=dev) + 1000
    q = torch.zeros(batch, NQ, 128, dtype=torch.bfloat16, device=dev)
    kk = torch.zeros(batch, NQ, 128, dtype=torch.bfloat16, device=dev)
    v = torch.zeros(batch, NQ, 128, dtype=torch.bfloat16, device=dev)
    ws = L.ChainWorkspace(0)
    ws.trace(True)

    def phases(l):
        ly = layers[l % 4]
        return [dict(x=attn, w=ly["o"], batch=batch, y=h, epilogue=L.RESIDUAL, ss_out=ss_b, pdl=True),
                dict(x=h, w=ly["gu"], batch=batch, y=act, epilogue=L.SILU_MUL, ss_in=ss_b, pdl=True),
                dict(x=act, w=ly["down"], batch=batch, y=h, epilogue=L.RESIDUAL, ss_out=ss_a, pdl=True),
                dict(x=h, w=ly["qkv"], batch=batch, epilogue=L.QKV_ROPE, positions=pos, q=q, k_out=kk, v_out=v,
                     n_q_heads=NQ, n_kv_heads=NQ, ss_in=ss_a, pdl=True)]

    for l in range(6):
        L.linear_chain(phases(l), ws)
    torch.cuda.synchronize()
    tr = ws.trace().astype(np.float64)  # [grid][4][6]
    valid = tr > 0
    t0 = tr[valid].min()
    rel = np.where(valid, (tr - t0) / 1e3, np.nan)  # us
    print(f"batch {batch}, grid {tr.shape[0]} CTAs; us since the launch's first stamp (min / median / max over CTAs)")
    for qi, name in enumerate(["O+res", "gate/up", "down+res", "QKV+rope"]):
        parts = []
        for k, nm in enumerate(NAMES):
            col = rel[:, qi, k]
            col = col[~np.isnan(col)]
            if col.size:
                parts.append(f"{nm} {col.min():6.1f}/{np.median(col):6.1f}/{col.max():6.1f}")
        print(f"  {name:9s} " + " | ".join(parts))


if __name__ == "__main__":
    main()
