"""CPU: the prefixsim_gpu CLI's host-only subcommands behave like the reference CLI
(tools/prefixsim_main.cpp: trace-gen :258-284, compare :113-160, calibrate :51-64)."""
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2605_23389_b200", "prefixsim_gpu")
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


def test_cli_is_built():
    assert os.access(CLI, os.X_OK)
    r = subprocess.run([CLI, "--help"], capture_output=True, text=True)
    assert r.returncode == 0 and "run --config" in r.stderr


def test_trace_gen_is_deterministic(tmp_path):
    def gen(seed, name):
        out = tmp_path / name
        r = subprocess.run([CLI, "trace-gen", "--count", "50", "--seed", str(seed), "--out", str(out)],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        assert "wrote 50 requests" in r.stdout
        return out.read_text()
    a, b, c = gen(3, "a.jsonl"), gen(3, "b.jsonl"), gen(4, "c.jsonl")
    assert a == b and a != c
    lines = a.splitlines()
    assert len(lines) == 50
    assert set(json.loads(lines[0])) == {"arrival_ms", "prompt_tokens", "output_tokens"}


def test_compare_virtual_clock(tmp_path):
    cfg = tmp_path / "smoke.json"
    cfg.write_text(json.dumps(GOLDEN["configs"]["smoke"]))
    r = subprocess.run([CLI, "compare", "--config", str(cfg), "--seeds", "1", "--out", str(tmp_path / "c")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    csv = (tmp_path / "c" / "compare.csv").read_text().splitlines()
    assert csv[0].startswith("policy,throughput_mean") and len(csv) == 4
    ratios = json.loads((tmp_path / "c" / "ratios.json").read_text())
    assert set(ratios) == {"aligned_over_fcfs_continuous", "aligned_over_disagg_fcfs"}


def test_bad_arguments_fail_like_the_reference():
    r = subprocess.run([CLI, "run"], capture_output=True, text=True)
    assert r.returncode != 0 and "--config" in r.stderr
    r = subprocess.run([CLI, "run", "--config", "/nonexistent.json"], capture_output=True, text=True)
    assert r.returncode != 0 and "cannot" in r.stderr.lower()
