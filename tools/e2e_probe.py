#!/usr/bin/env python
"""Where does the end-to-end decode step go?  (measurement tool, not product code)

Runs the C2 window of bench.py through asv_engine_run with KV moves executed,
for several host run-ahead depths, and prints per-step: GPU window, attention
time, PCIe link busy (union of copy intervals), host time blocked on the GPU,
and copy-stream hazard waits — next to the KV-resident run of the same window.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_23389_b200 import engine as E  # noqa: E402


def main():
    cfg_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "configs", "c2_7b_1024req.json")
    steps = int(os.environ.get("STEPS", 500))
    S, W = 300, 5
    cfg = E.load_config(cfg_path)
    a = cfg["b200"]
    kw = dict(device=0, num_q_heads=a["num_q_heads"], num_kv_heads=a["num_kv_heads"], num_layers=a["num_layers"],
              exec_begin=S, timed_begin=S + W, exec_end=S + W + steps, host_pool_bytes=4 << 30)
    out = []
    res = E.engine_run(cfg, execute_transfers=False, **kw)
    n = max(1, res["iterations_timed"])
    out.append({"mode": "resident", "tok_s": res["tokens_timed"] / res["window_ms"] * 1e3,
                "ms_step": res["window_ms"] / n, "attn_ms_step": res["attn_ms"] / n,
                "host_wait_ms": res["host_wait_ms"], "host_decide_ms": res["host_decide_ms"]})
    for ra in [int(x) for x in os.environ.get("RUN_AHEAD", "16,64").split(",")]:
        r = E.engine_run(cfg, execute_transfers=True, copy_begin=max(0, S - 400), run_ahead=ra, **kw)
        n = max(1, r["iterations_timed"])
        out.append({"mode": f"e2e run_ahead={ra}", "tok_s": r["tokens_timed"] / r["window_ms"] * 1e3,
                    "ms_step": r["window_ms"] / n, "attn_ms_step": r["attn_ms"] / n,
                    "pcie_union_ms_step": r["pcie_union_ms"] / n,
                    "pcie_busy_sum_ms_step": r["h2d_busy_ms"] / n,
                    "h2d_MB_step": r["h2d_bytes_window"] / n / 1e6, "d2h_MB_step": r["d2h_bytes_window"] / n / 1e6,
                    "link_gbps_union": ((r["h2d_bytes_window"] + r["d2h_bytes_window"]) /
                                        max(1e-9, r["pcie_union_ms"] * 1e-3) / 1e9),
                    "host_wait_ms": r["host_wait_ms"], "host_decide_ms": r["host_decide_ms"],
                    "hazard_waits": r["hazard_waits"], "tokens": r["tokens_timed"]})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
