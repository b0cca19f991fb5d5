"""CPU, world_size 2 over gloo: the data-parallel sharding of the decode path.

Each rank runs the decision path of its shard (request i -> rank i % N), exactly
what every rank of `torchrun bench.py --gpus N` does before driving its GPU.
Checked: shards partition the trace (disjoint, complete), the token count adds up
to the trace's output tokens, there is no cross-shard dependency (a shard's log
is the same whether computed alone or beside the other), and each shard's log is
bit-exact with the reference engine run on that shard's sub-trace.
"""
import json
import os
import socket
import tempfile

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import _util as U

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_23389_b200 import engine
    log = engine.run_config_jsonl_shard(cfg, rank, world)
    recs = [json.loads(l) for l in log.splitlines()[1:]]
    tokens = sum(len(r["prefix_lengths"]) for r in recs if r["type"] == "iteration")
    n_req = sum(1 for r in recs if r["type"] == "request")
    t = [tokens, n_req]
    gathered = [None] * world
    dist.all_gather_object(gathered, t)
    with open(os.path.join(out_dir, f"rank{rank}.jsonl"), "w") as f:
        f.write(log)
    if rank == 0:
        with open(os.path.join(out_dir, "gathered.json"), "w") as f:
            json.dump(gathered, f)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_over_gloo():
    from paper_2605_23389_b200 import engine
    cfg = engine.load_config(os.path.join(ROOT, "configs", "c1_7b_b16.json"))
    trace = [json.loads(l) for l in open(cfg["workload"]["path"])]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), cfg, d), nprocs=2, join=True)
        gathered = json.load(open(os.path.join(d, "gathered.json")))
        assert sum(g[1] for g in gathered) == len(trace)
        assert sum(g[0] for g in gathered) == sum(r["output_tokens"] for r in trace)
        for rank in range(2):
            log = open(os.path.join(d, f"rank{rank}.jsonl")).read()
            assert log == engine.run_config_jsonl_shard(cfg, rank, 2)  # no cross-shard state
            # the shard is an ordinary trace for the reference engine
            sub = trace[rank::2]
            tp = os.path.join(d, f"shard{rank}.jsonl")
            with open(tp, "w") as f:
                for r in sub:
                    f.write(json.dumps(r) + "\n")
            c2 = json.loads(json.dumps(cfg))
            c2["workload"]["path"] = tp
            assert log == engine.run_config_jsonl(c2)
            if os.path.exists(U.REF_SO):
                assert log == U.RefEngine().run_config_jsonl(c2)[0]


def test_bad_shard_arguments_raise():
    from paper_2605_23389_b200 import engine
    cfg = engine.load_config(os.path.join(ROOT, "configs", "c1_7b_b16.json"))
    with pytest.raises(ValueError, match="bad shard"):
        engine.run_config_jsonl_shard(cfg, 2, 2)
