"""CPU: the B200 engine's decision path is bit-exact with the reference.

Batch composition and order (= GPU page-table order), every transfer's bytes and
the whole schema-1 log must match the reference exactly on the same trace:
  * against golden digests made by the UNMODIFIED reference (tests/golden,
    tests/golden/make_golden.py) — always;
  * against the live reference library (oracle/_ref) when it is present.
"""
import hashlib
import json
import os

import pytest

import _util as U

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
POL = {"aligned": None, "fcfs": "fcfs", "disagg-fcfs": "disagg-fcfs"}


def digest(text):
    kinds = {}
    for line in text.splitlines()[1:]:
        rec = json.loads(line)
        if rec["type"] == "transfer":
            kinds[rec["kind"]] = kinds.get(rec["kind"], 0) + rec["bytes"]
    return hashlib.sha256(text.encode()).hexdigest(), kinds


def config_for(name):
    from paper_2605_23389_b200 import engine
    if name in GOLDEN["configs"]:
        return GOLDEN["configs"][name]
    return engine.load_config(os.path.join(ROOT, "configs", name + ".json"))


@pytest.mark.parametrize("key", sorted(GOLDEN["logs"]))
def test_log_matches_reference_golden(key):
    from paper_2605_23389_b200 import engine
    name, pol = key.split(":")
    text = engine.run_config_jsonl(config_for(name), POL[pol])
    sha, kinds = digest(text)
    g = GOLDEN["logs"][key]
    assert kinds == g["transfer_bytes"], "KV bytes moved differ from the reference"
    assert sha == g["sha256"], "log differs from the reference"


def test_survey_appendix_b_golden_hashes():
    """The two sha256 values SURVEY.md Appendix B recorded from the reference."""
    assert GOLDEN["logs"]["smoke:aligned"]["sha256"].startswith("f5f5c9d42128fe1a")
    assert GOLDEN["logs"]["short95:aligned"]["sha256"].startswith("b36e0678169c6e91")


@pytest.mark.skipif(not os.path.exists(U.REF_SO), reason="reference library not built")
@pytest.mark.parametrize("seed", [2, 3, 5])
@pytest.mark.parametrize("policy", [None, "fcfs", "disagg-fcfs"])
def test_randomised_configs_match_live_reference(seed, policy):
    from paper_2605_23389_b200 import engine
    cfg = json.loads(json.dumps(GOLDEN["configs"]["short95"]))
    cfg["seed"] = seed
    cfg["workload"]["seed"] = seed
    cfg["workload"]["count"] = 400
    cfg["cluster"]["nvlink_available"] = seed != 3
    cfg["constraints"]["k_min"] = 8 + 4 * seed
    ref_text, _, _ = U.RefEngine().run_config_jsonl(cfg, policy)
    assert engine.run_config_jsonl(cfg, policy) == ref_text


@pytest.mark.parametrize("case", range(0, 300, 1))
def test_dfs_batch_order_matches_reference(case):
    from paper_2605_23389_b200 import engine
    c = GOLDEN["dfs"][case]
    ids, tot = engine.dfs_batch(c["residents"], c["b_max"], c["k_min"])
    assert ids == c["ids"] and tot == c["total_blocks"]


def test_iteration_prefix_lengths_are_running_order():
    """IterationRecord.prefix_lengths is the page-table order the executor uploads."""
    from paper_2605_23389_b200 import engine
    text = engine.run_config_jsonl(GOLDEN["configs"]["smoke"])
    its = [json.loads(l) for l in text.splitlines()[1:] if '"type":"iteration"' in l]
    assert its and all(len(i["prefix_lengths"]) >= 1 for i in its)
