"""GPU: the multi-rank bench paths (torchrun, 2 ranks) on the one GPU this build has.

ASV_BENCH_DEVICE=0 puts both ranks on cuda:0 (gloo for the bench's own barrier and
reductions), so the code a 2-GPU run executes is exercised end to end:
  * dp:    each rank decodes its shard (request i -> rank i % 2);
  * pairs: rank 0's engine runs the (decode, prefetch) pair — candidate buffers in
           a separate pool, admits/evicts as device copies, prefill offloads on the
           prefetch side — rank 1 only joins the barriers.
C1 is used (its 32 GiB decode pool fits twice on one B200; C2's does not).
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bench(extra, port=None):
    port = port or _free_port()
    env = dict(os.environ, ASV_BENCH_DEVICE="0", ASV_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "5", "--warmup", "3", "--config", os.path.join(ROOT, "configs", "c1_7b_b16.json"),
           "--attention-only", "--no-cpu-baseline"] + list(extra)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_dp_two_ranks():
    line = _bench(["--no-pairs"])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "dp2"
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0


def test_pairs_two_ranks():
    line = _bench([])
    pairs = line["pairs"]
    assert pairs["parallelism"] == "pairs1"
    assert pairs["value"] > 0 and pairs["window_steps"] > 0
    assert pairs["p2p_bytes_per_step"] > 0            # admits moved buffer -> decode pool
    assert pairs["h2d_bytes_per_step"] > 0
    assert "colocated_prefill_offload" not in line["e2e"]
