"""Run every BASELINE config (C1-C5) through the GPU engine on one B200 and
record decode tok/s, attention GB/s and measured vs virtual bubbles.

C3/C4 are multi-GPU configs; on one GPU they run with pair_mode (candidate
buffers in a separate pool: admits/evicts become device copies) so the pair
code path executes.  C5 runs aligned and FCFS (prefix-aware vs FCFS batching).
usage: python tools/run_configs.py [--steps 40] [--out profiles/configs_rXX.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

RUNS = [
    ("c1_7b_b16", None, 200, False),
    ("c2_7b_1024req", None, 300, False),
    ("c3_pair_32k", None, 200, True),
    ("c4_13b_gqa8", None, 200, False),
    ("c5_zipf_128k", None, 300, False),
    ("c5_zipf_128k", "fcfs", 300, False),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--e2e", action="store_true")
    ap.add_argument("--full", action="store_true", help="also run the full decoder-layer step (tcgen05 GEMMs)")
    ap.add_argument("--bubble", action="store_true",
                    help="also run the attention-only step with the per-warp %%globaltimer probe on every launch "
                         "(measured intra-iteration bubble per iteration: p50 / p90 / p99 / max)")
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default=None, help="comma-separated config names (default: all)")
    a = ap.parse_args()
    from paper_2605_23389_b200 import engine as E
    results = []
    for name, pol, start, pair in RUNS:
        if a.only and name not in a.only.split(","):
            continue
        cfg = E.load_config(os.path.join(ROOT, "configs", name + ".json"))
        at = cfg["b200"]
        row = {"config": name, "policy": pol or "aligned", "start": start, "pair_mode": pair}
        modes = ["value"] + (["e2e"] if a.e2e else []) + (["full_step"] if a.full else []) + \
            (["bubble"] if a.bubble else [])
        for mode in modes:
            try:
                    st = E.engine_run(cfg, policy=pol, device=0, num_q_heads=at["num_q_heads"],
                                  num_kv_heads=at["num_kv_heads"], num_layers=at["num_layers"],
                                  execute_transfers=(mode == "e2e"), exec_begin=start, timed_begin=start + a.warmup,
                                  exec_end=start + a.warmup + a.steps, copy_begin=max(0, start - 400),
                                  host_pool_bytes=2 << 30, pair_mode=pair, full_step=(mode == "full_step"),
                                  probe_bubble=(mode == "bubble"))
            except ValueError as exc:  # e.g. full_step weights next to a pool sized for KV alone
                row[mode] = {"skipped": str(exc)}
                continue
            it = max(1, st["iterations_timed"])
            row[mode] = {"tok_s": st["tokens_timed"] / (st["window_ms"] / 1e3) if st["window_ms"] > 0 else 0,
                         "ms_per_step": st["window_ms"] / it, "mean_batch": st["tokens_timed"] / it,
                         "attn_gbps": st["attn_bytes"] / (st["attn_ms"] * 1e-3) / 1e9 if st["attn_ms"] > 0 else 0,
                         "measured_idle_frac": st["measured_idle_frac"],
                         "measured_bubble_ms_per_step": st["measured_bubble_ms"] / it,
                         "virtual_bubble_ms_per_step": st["bubble_ms_timed"] / it,
                         "virtual_tok_s_whole_run": st["virtual_decode_tok_s"],
                         "h2d_gb": st["h2d_bytes_window"] / 1e9, "p2p_gb": st["p2p_bytes_window"] / 1e9,
                         "p2p_gbps": (st["p2p_bytes_window"] / (st["p2p_busy_ms"] * 1e-3) / 1e9
                                      if st["p2p_busy_ms"] > 0 else None)}
            if mode == "bubble":
                row[mode].update({"bubble_p50_ms": st["bubble_p50_ms"], "bubble_p90_ms": st["bubble_p90_ms"],
                                  "bubble_p99_ms": st["bubble_p99_ms"], "bubble_max_ms": st["bubble_max_ms"],
                                  "bubble_per_iteration_ms": st.get("bubble_per_iteration_ms", []),
                                  "virtual_bubble_per_iteration": "reference cost model, same iterations"})
            if mode == "full_step":
                row[mode]["hbm_gbps"] = ((st["attn_bytes"] + st["weight_bytes"]) / (st["window_ms"] * 1e-3) / 1e9
                                         if st["window_ms"] > 0 else 0)
                row[mode]["weight_gb_per_step"] = st["weight_bytes"] / it / 1e9
        print(json.dumps(row), flush=True)
        results.append(row)
    if a.out:
        json.dump(results, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
