"""Regenerate tests/golden/golden.json from the UNMODIFIED reference (TEST INFRASTRUCTURE).

Sources, all produced by the reference itself compiled from /root/reference
(oracle/_ref/libprefixsim_ref.so, see oracle/Makefile):
  * schema-1 log sha256 + per-kind transfer bytes for the reference's own configs
    (proj/configs/smoke.json, short95.json under the three policies) and for the
    repo's BASELINE configs C1, C2, C3, C5 (aligned and fcfs);
  * density_first_search member ids (composition AND order = page-table order)
    on 300 random pool snapshots drawn like tests/test_batch_gen.cpp:141-188
    (splitmix64 seed 31), from both the reference's QuadTree search and its
    independent flat-list oracle (proj/tests/reference_dfs.hpp).
The reference's two config files are embedded verbatim as fixtures so the
parity tests run where /root/reference is absent (the GPU box).

Run:  python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import _util as U  # noqa: E402
from make_traces import Rng  # noqa: E402

REF_CONFIGS = "/root/reference/proj/configs"


def log_digest(text):
    kinds = {}
    its = 0
    for line in text.splitlines()[1:]:
        rec = json.loads(line)
        if rec["type"] == "transfer":
            k = kinds.setdefault(rec["kind"], [0, 0])
            k[0] += rec["bytes"]
            k[1] += 1
        elif rec["type"] == "iteration":
            its += 1
    return {"sha256": hashlib.sha256(text.encode()).hexdigest(), "iterations": its,
            "transfer_bytes": {k: v[0] for k, v in sorted(kinds.items())},
            "transfer_count": {k: v[1] for k, v in sorted(kinds.items())}}


def dfs_cases(ref, n_cases=300, seed=31):
    rng = Rng(seed)
    cases = []
    for _ in range(n_cases):
        n = rng.uniform_int(1, 64)
        b_max = rng.uniform_int(40, 2000)
        k_min = rng.uniform_int(1, 24)
        clustered = rng.next_double() < 0.5
        center = rng.uniform_int(1, 60000)
        res = []
        for i in range(n):
            if clustered:
                p = max(1, center + rng.uniform_int(0, 600) - 300)
            else:
                p = rng.uniform_int(1, 70000)
            blocks = min((min(p, 65536) + 15) // 16, b_max)
            res.append([i, p, blocks])
        ids, tot = ref.dfs(res, b_max, k_min)
        ids2, tot2 = ref.dfs(res, b_max, k_min, flat_oracle=True)
        assert ids == ids2 and tot == tot2, "reference search disagrees with its own oracle"
        cases.append({"residents": res, "b_max": b_max, "k_min": k_min, "ids": ids, "total_blocks": tot})
    return cases


def main():
    ref = U.RefEngine()
    out = {"configs": {}, "logs": {}, "dfs": None}
    for name in ("smoke", "short95"):
        cfg = json.load(open(os.path.join(REF_CONFIGS, name + ".json")))
        out["configs"][name] = cfg
        for pol in (None, "fcfs", "disagg-fcfs"):
            text, _, _ = ref.run_config_jsonl(cfg, pol)
            out["logs"][f"{name}:{pol or 'aligned'}"] = log_digest(text)
    from paper_2605_23389_b200 import engine
    for c in ("c1_7b_b16", "c2_7b_1024req", "c3_pair_32k", "c5_zipf_128k"):
        cfg = engine.load_config(os.path.join(ROOT, "configs", c + ".json"))
        for pol in (None, "fcfs"):
            text, _, _ = ref.run_config_jsonl(cfg, pol)
            out["logs"][f"{c}:{pol or 'aligned'}"] = log_digest(text)
    out["dfs"] = dfs_cases(ref)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", os.path.join(HERE, "golden.json"), len(out["logs"]), "logs,", len(out["dfs"]), "dfs cases")


if __name__ == "__main__":
    main()
