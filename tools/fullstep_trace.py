#!/usr/bin/env python
"""Timeline of the full decode step's linear launches inside the engine (C2, KV resident): the
asv_linear timeline probe records 64 consecutive linear launches (16 layers x QKV, O, gate/up, down)
from the middle of a timed step; per layer it reports the gaps between the linear launches and the
QKV(l) exit -> O(l) dependency span that holds the layer's attention + split merge.
Env: CONFIG (default c2_7b_1024req), ASV_LINEAR_TRACE_SKIP (set here: 2 steps + 8 layers)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("ASV_LINEAR_TRACE_SKIP", str(2 * 128 + 32 + 1))
from paper_2605_23389_b200 import engine as E  # noqa: E402
from paper_2605_23389_b200 import linear as L  # noqa: E402


def main():
    cfg = E.load_config(os.path.join(ROOT, "configs", os.environ.get("CONFIG", "c2_7b_1024req") + ".json"))
    a = cfg["b200"]
    L.linear_trace(True)
    st = E.engine_run(cfg, device=0, num_q_heads=a["num_q_heads"], num_kv_heads=a["num_kv_heads"],
                      num_layers=a["num_layers"], execute_transfers=False, exec_begin=300, timed_begin=300,
                      exec_end=305, full_step=True)
    tr = L.linear_trace().astype(np.float64)
    L.linear_trace(False)
    print(json.dumps({"tok_s": st["tokens_timed"] / (st["window_ms"] * 1e-3), "launches_recorded": int(tr.shape[0])}))
    ent = tr[:, :, 0]
    t0 = ent[ent > 0].min()
    rows = []
    for li in range(tr.shape[0]):
        g = int((ent[li] > 0).sum())
        x = tr[li, :g, :7]
        x = np.where(x > 0, (x - t0) / 1e3, np.nan)
        rows.append(dict(grid=g, entry=np.nanmedian(x[:, 0]), entry_min=np.nanmin(x[:, 0]), dep=np.nanmedian(x[:, 1]),
                         landed=np.nanmin(x[:, 3]), acc_last=np.nanmax(x[:, 4]), exit_max=np.nanmax(x[:, 6])))
    # identify launch kinds by grid: QKV 192, O / down 256, gate/up 172 (7B, batch <= 256)
    names = {192: "QKV", 172: "gate/up"}
    prev = None
    for i, r in enumerate(rows):
        nm = names.get(r["grid"], "O/down")
        if nm == "O/down":
            nm = "O" if prev is not None and prev == "QKV" else "down"
        line = (f"{i:2d} {nm:7s} grid {r['grid']:3d} entry {r['entry']:8.1f} dep {r['dep']:8.1f} "
                f"landed {r['landed']:8.1f} acc_last {r['acc_last']:8.1f} exit {r['exit_max']:8.1f}")
        if i > 0:
            line += f" | gap(prev acc_last -> landed) {r['landed'] - rows[i - 1]['acc_last']:6.1f}"
        print(line)
        prev = nm


if __name__ == "__main__":
    main()
