#!/usr/bin/env python
"""Run a few full decode steps (C2 workload, KV resident) through asv_engine_run —
a short target for ncu launch lists / captures of the whole decoder layer stack."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_23389_b200 import engine as E  # noqa: E402


def main():
    cfg = E.load_config(os.path.join(ROOT, "configs", os.environ.get("CONFIG", "c2_7b_1024req") + ".json"))
    a = cfg["b200"]
    steps = int(os.environ.get("STEPS", 3))
    st = E.engine_run(cfg, device=0, num_q_heads=a["num_q_heads"], num_kv_heads=a["num_kv_heads"],
                      num_layers=a["num_layers"], execute_transfers=False, exec_begin=300, timed_begin=300,
                      exec_end=300 + steps, full_step=os.environ.get("FULL", "1") == "1")
    out = {k: st[k] for k in ("iterations_timed", "tokens_timed", "window_ms", "kernel_launches_timed",
                              "weight_bytes", "attn_bytes")}
    out["tok_s"] = st["tokens_timed"] / (st["window_ms"] * 1e-3) if st["window_ms"] > 0 else 0.0
    out["hbm_gbps"] = (st["weight_bytes"] + st["attn_bytes"]) / (st["window_ms"] * 1e-3) / 1e9 if st["window_ms"] > 0 else 0.0
    print(json.dumps(out))


if __name__ == "__main__":
    main()
