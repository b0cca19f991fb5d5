"""GPU: runs executed on the B200 emit the reference's own artefacts.

* asv_engine_run_ex: the decision log of a run whose every iteration and KV move
  was executed on the GPU is byte-identical (sha256) to the log the UNMODIFIED
  reference produced for the same config (tests/golden, reference
  tools/prefixsim_main.cpp cmd_run -> log_to_jsonl).
* prefixsim_gpu run: the reference CLI's `run` subcommand (prefixsim_main.cpp:66-111)
  over the C ABI — same flags, same artefact files, the same log bytes.
"""
import hashlib
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
CLI = os.path.join(ROOT, "paper_2605_23389_b200", "prefixsim_gpu")


def _sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


@pytest.mark.parametrize("policy", ["aligned", "fcfs", "disagg-fcfs"])
def test_executed_run_log_is_the_references(policy):
    from paper_2605_23389_b200 import engine
    st, log = engine.engine_run(GOLDEN["configs"]["smoke"], policy=policy, device=0, num_q_heads=32,
                                num_kv_heads=32, num_layers=32, execute_transfers=True, exec_begin=0,
                                exec_end=-1, timed_begin=0, copy_begin=0, host_pool_bytes=1 << 30,
                                prefill_offload=True, return_log=True)
    want = GOLDEN["logs"][f"smoke:{policy}"]
    assert st["iterations_timed"] == want["iterations"]
    assert _sha(log) == want["sha256"]


def test_cli_run_writes_the_reference_artefacts(tmp_path):
    cfg = tmp_path / "smoke.json"
    cfg.write_text(json.dumps(GOLDEN["configs"]["smoke"]))
    out = tmp_path / "run_out"
    r = subprocess.run([CLI, "run", "--config", str(cfg), "--out", str(out)], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr
    assert "policy aligned:" in r.stdout and "B200:" in r.stdout
    for f in ("config_used.json", "log.jsonl", "summary.json", "ttft_cdf.csv", "sched_cdf.csv", "gpu_stats.json"):
        assert (out / f).exists(), f
    assert _sha((out / "log.jsonl").read_text()) == GOLDEN["logs"]["smoke:aligned"]["sha256"]
    gs = json.loads((out / "gpu_stats.json").read_text())
    assert gs["iterations_timed"] == GOLDEN["logs"]["smoke:aligned"]["iterations"]
    assert gs["h2d_bytes"] == gs["logical_bytes"]["batch_prefetch"] + gs["logical_bytes"]["stray_prefetch"]
    assert gs["decode_tokens_per_s_measured"] > 0
    summ = json.loads((out / "summary.json").read_text())
    assert summ["completed_requests"] == 40


def test_cli_run_policy_and_nvlink_flags(tmp_path):
    """--policy / --no-nvlink change the run exactly as the reference's flags do (config_used.json)."""
    cfg = tmp_path / "smoke.json"
    cfg.write_text(json.dumps(GOLDEN["configs"]["smoke"]))
    out = tmp_path / "fcfs"
    r = subprocess.run([CLI, "run", "--config", str(cfg), "--out", str(out), "--policy", "fcfs", "--resident"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert _sha((out / "log.jsonl").read_text()) == GOLDEN["logs"]["smoke:fcfs"]["sha256"]
    assert json.loads((out / "config_used.json").read_text())["policy"] == "fcfs"
    out2 = tmp_path / "nonv"
    r = subprocess.run([CLI, "run", "--config", str(cfg), "--out", str(out2), "--no-nvlink", "--resident"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert json.loads((out2 / "config_used.json").read_text())["cluster"]["nvlink_available"] is False


def test_cli_whole_c1_trace_on_the_gpu(tmp_path):
    """BASELINE C1 end to end: all 2 146 iterations (32-layer attention each) and every KV move
    (0.62 TB host -> GPU) executed on the B200; the decision log equals the reference's byte for byte."""
    out = tmp_path / "c1"
    r = subprocess.run([CLI, "run", "--config", os.path.join(ROOT, "configs", "c1_7b_b16.json"), "--out", str(out),
                        "--host-pool-mib", "2048"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    assert _sha((out / "log.jsonl").read_text()) == GOLDEN["logs"]["c1_7b_b16:aligned"]["sha256"]
    gs = json.loads((out / "gpu_stats.json").read_text())
    assert gs["iterations_timed"] == GOLDEN["logs"]["c1_7b_b16:aligned"]["iterations"]
    lb = gs["logical_bytes"]
    assert gs["h2d_bytes"] == lb["batch_prefetch"] + lb["stray_prefetch"] > 0


def test_cli_compare_with_gpu_measurements(tmp_path):
    """`compare --gpu`: the reference's policy sweep (virtual clock) plus each policy executed on the B200."""
    cfg = tmp_path / "smoke.json"
    cfg.write_text(json.dumps(GOLDEN["configs"]["smoke"]))
    out = tmp_path / "cmp"
    r = subprocess.run([CLI, "compare", "--config", str(cfg), "--seeds", "1", "--policies", "aligned,fcfs", "--gpu",
                        "--resident", "--out", str(out)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr
    m = json.loads((out / "gpu_measured.json").read_text())
    assert set(m) == {"aligned", "fcfs_continuous"}
    assert all(v["decode_tokens_per_s_measured"] > 0 for v in m.values())
    assert (out / "compare.csv").exists() and (out / "ratios.json").exists()
