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


def _stress_config(i):
    """Seeded stress variant of short95: tight decode HBM (evictions, spills), a small host pool
    (prefill back-pressure), narrow / wide similarity windows, small candidate buffers, both
    link settings, random FCFS victims — the corners of the orchestrator (cluster_sim.hpp)."""
    import random
    rnd = random.Random(1000 + i)
    cfg = json.loads(json.dumps(GOLDEN["configs"]["short95"]))
    cfg["seed"] = cfg["workload"]["seed"] = 50 + i
    cfg["workload"]["count"] = rnd.choice([120, 200, 300])
    cfg["workload"]["arrival"]["rate_per_s"] = rnd.choice([50, 400, 2000])
    cfg["workload"]["short_ratio"] = rnd.choice([0.5, 0.8, 0.95])
    c = cfg["cluster"]
    c["decode_hbm_blocks"] = rnd.choice([2600, 4000, 6000, 10240])
    c["prefill_hbm_blocks"] = c["decode_hbm_blocks"] + rnd.choice([0, 1000, 4000])
    c["nvlink_available"] = rnd.random() < 0.7
    c["kv_pool_bytes"] = rnd.choice([800_000_000_000, 800_000_000_000, 150_000_000_000, 25_000_000_000])
    k = cfg["constraints"]
    k["k_min"] = rnd.choice([4, 8, 16, 36])
    k["b_max_fraction"] = rnd.choice([0.4, 0.85, 0.92])
    cfg["workload"]["output_len"]["hi"] = rnd.choice([68, 300])
    k["starvation_threshold_ms"] = rnd.choice([200, 2000, 6000])
    k["similarity_delta"] = rnd.choice([8, 32, 128])
    k["candidate_buffer_fraction"] = rnd.choice([0.05, 0.2, 0.3])
    k["fcfs_max_batch"] = rnd.choice([32, 256])
    return cfg


@pytest.mark.skipif(not os.path.exists(U.REF_SO), reason="reference library not built")
@pytest.mark.parametrize("policy", [None, "fcfs", "disagg-fcfs"])
@pytest.mark.parametrize("i", range(16))
def test_stress_configs_match_live_reference(i, policy):
    """The orchestrator's decisions under memory pressure equal the reference's byte for byte —
    or both refuse the config.  (A prefill held by host-pool back-pressure is retried only when a
    prefill offload lands, as in the reference; when nothing is in flight it never completes.  The
    reference reports that as a census mismatch — it counts the held request twice — this
    orchestrator as the request that did not complete.)"""
    from paper_2605_23389_b200 import engine
    cfg = _stress_config(i)
    try:
        ref_text, _, _ = U.RefEngine().run_config_jsonl(cfg, policy)
    except RuntimeError as exc:
        with pytest.raises(Exception) as got:
            engine.run_config_jsonl(cfg, policy)
        assert ("census mismatch" in str(exc) and "did not complete" in str(got.value)) or \
            str(exc).split(":")[-1].strip() in str(got.value), (str(exc), str(got.value))
        return
    assert engine.run_config_jsonl(cfg, policy) == ref_text


def test_stress_configs_exercise_pressure_paths():
    """The stress set really reaches evictions, spills, flushes and prefill back-pressure."""
    from paper_2605_23389_b200 import engine
    seen = {}
    for i in range(16):
        try:
            text = engine.run_config_jsonl(_stress_config(i))
        except Exception:
            continue
        for line in text.splitlines()[1:]:
            r = json.loads(line)
            if r.get("type") == "transfer":
                seen[r["kind"]] = seen.get(r["kind"], 0) + 1
    for kind in ("evict", "spill", "flush", "stray_prefetch", "admit"):
        assert seen.get(kind, 0) > 0, (kind, seen)
