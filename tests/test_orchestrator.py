"""CPU: the per-pair orchestrator's typed data-plane orders (cluster_sim.hpp DataPlane / KvMove) equal
the decision log one for one, and wall-clock mode drives the clock with measured step times
(tests/cpp/orchestrator_test.cpp, compiled against the product headers)."""
import hashlib
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


def _binary():
    src = os.path.join(ROOT, "tests", "cpp", "orchestrator_test.cpp")
    h = hashlib.sha256(open(src, "rb").read())
    for d in ("paper_2605_23389_b200/include/prefixsim",):
        for fn in sorted(os.listdir(os.path.join(ROOT, d))):
            h.update(open(os.path.join(ROOT, d, fn), "rb").read())
    out = f"/tmp/asv_orchestrator_test_{h.hexdigest()[:16]}"
    if not os.path.exists(out):
        subprocess.run(["g++", "-std=c++20", "-O1", "-ffp-contract=off",
                        "-I" + os.path.join(ROOT, "paper_2605_23389_b200", "include"),
                        "-I" + os.path.join(ROOT, "third_party", "nlohmann"), src, "-o", out],
                       check=True, capture_output=True, text=True)
    return out


@pytest.mark.parametrize("policy", ["aligned", "fcfs", "disagg-fcfs"])
@pytest.mark.parametrize("config", ["smoke", "short95"])
def test_orders_match_log_and_wall_clock(tmp_path, config, policy):
    cfg = json.loads(json.dumps(GOLDEN["configs"][config]))
    if config == "short95":
        cfg["workload"]["count"] = 600
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps(cfg))
    r = subprocess.run([_binary(), str(p), policy], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stderr
    assert "PASS" in r.stdout
