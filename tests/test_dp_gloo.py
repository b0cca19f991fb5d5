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


def _pair_worker(rank, world, port, cfg, out_dir):
    """bench.py's pair topology: ranks 2p / 2p+1 = (decode, prefetch) GPUs of pair p; the global trace
    is P = world/2 copies of the config's trace; the decode rank's orchestrator drives its pair
    (shard p of P), the prefetch rank only joins the collectives."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    import bench
    from paper_2605_23389_b200 import engine
    P = world // 2
    gcfg = bench.replicated_config(cfg, P, f"gloo_pair{rank}")
    log, tokens = "", 0
    if rank % 2 == 0:
        log = engine.run_config_jsonl_shard(gcfg, rank // 2, P)
        tokens = sum(len(json.loads(l)["prefix_lengths"]) for l in log.splitlines()[1:] if '"type":"iteration"' in l)
    if gcfg is not cfg:
        os.unlink(gcfg["workload"]["path"])
    gathered = [None] * world
    dist.all_gather_object(gathered, [rank, tokens])
    with open(os.path.join(out_dir, f"pair_rank{rank}.jsonl"), "w") as f:
        f.write(log)
    if rank == 0:
        with open(os.path.join(out_dir, "pair_gathered.json"), "w") as f:
            json.dump(gathered, f)
    dist.barrier()
    dist.destroy_process_group()


def test_four_rank_pair_topology_over_gloo():
    """2 pairs on 4 ranks: every pair decodes a full copy of the trace (weak scaling), its log is
    bit-exact with the reference's run of that trace, and prefetch ranks decode nothing."""
    from paper_2605_23389_b200 import engine
    cfg = engine.load_config(os.path.join(ROOT, "configs", "c1_7b_b16.json"))
    trace = [json.loads(l) for l in open(cfg["workload"]["path"])]
    ref = U.RefEngine().run_config_jsonl(cfg)[0] if os.path.exists(U.REF_SO) else engine.run_config_jsonl(cfg)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_pair_worker, args=(4, _free_port(), cfg, d), nprocs=4, join=True)
        gathered = json.load(open(os.path.join(d, "pair_gathered.json")))
        out_tokens = sum(r["output_tokens"] for r in trace)
        assert [g[1] for g in sorted(gathered)] == [out_tokens, 0, out_tokens, 0]
        for rank in (0, 2):
            assert open(os.path.join(d, f"pair_rank{rank}.jsonl")).read() == ref
        for rank in (1, 3):
            assert open(os.path.join(d, f"pair_rank{rank}.jsonl")).read() == ""
