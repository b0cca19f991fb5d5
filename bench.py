#!/usr/bin/env python
"""Benchmark of the B200-native AlignedServe decode-iteration hot path.

Metric (BASELINE.json): decode tokens/sec at 1/2/4/8 B200, with decode-attention
HBM GB/s and KV-prefetch GB/s beside it.  Workload at N=1: BASELINE configs[1]
("Llama-2-7B-shape synthetic trace, 1024 in-flight requests in host memory, KV
lengths 1K-16K, bf16 KV, 1 B200") = configs/c2_7b_1024req.json.

A step is one decode iteration of the engine: the reference-API scheduler's
boundary decisions (virtual clock, bit-exact with the reference), the page-table
build + upload, and the whole Llama-2-7B-shape decoder stack over 32 layers
(RMSNorm, QKV GEMM + RoPE, paged split-KV attention + KV append, O GEMM +
residual, RMSNorm, gate/up GEMM + SiLU, down GEMM + residual; GEMMs on tcgen05,
synthetic weights).  Iterations [S, S+W) are warm-up, [S+W, S+W+K) are timed with
CUDA events on the compute stream; S is a steady-state point of the trace
(earlier iterations run decisions only).

  value : full decoder step, KV resident in HBM when the window starts
  e2e   : the same step through the C-ABI engine (asv_engine_run) with every
          boundary KV move executed from/to the pinned host pool (H2D prefetch,
          D2H spill/flush; P2P with a partner GPU) and every step's result read
          back to pinned host memory, inside the timed region; >= 500 steps
          because prefetch traffic is bursty
  attention_only / roofline : the attention-only step (the dominant kernel) of
          the same window: decode-attention HBM GB/s vs the measured peak

N > 1: `--gpus N` without WORLD_SIZE relaunches itself under torch.distributed.run.
Weak scaling: the global trace is N copies of the C2 request set (N x 1024
requests, copy p of request j has global index j*N + p), sharded data-parallel
(request i -> rank i % N), so every rank decodes a full C2 workload and its
decisions are bit-exact with the reference run of C2; no data-path collective.
Beside it the north-star pair topology is measured in the same run (`pairs`):
ranks 2p / 2p+1 form a (decode, prefetch) pair, the global trace has N/2 copies,
the decode rank's engine drives both GPUs (candidate buffers, host->GPU
prefetches and prefill offloads on the prefetch GPU, admits / evicts as NVLink
peer moves).  `--impl reference` times the reference's CPU path (the compiled
reference decision engine + the fp32 CPU decoder-step oracle) on the host cores
over the same window and prints the same config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = os.path.join(ROOT, "configs", "c2_7b_1024req.json")
WORKLOAD_NAME = ("C2: Llama-2-7B shape (32 q/kv heads, d=128, 32 layers, bf16 KV, 16-token pages), "
                 "1024 requests in the host pool per rank, KV 1K-16K, aligned policy")
STEADY_START = 300          # first executed iteration of the trace (per shard)
COPY_LEAD = 400             # KV moves are executed from this many iterations before the span
E2E_MIN_STEPS = 500         # e2e window: prefetch traffic is bursty (batch switches), so the
                            # end-to-end rate is taken over >= this many steps
HOST_POOL_BYTES = 4 << 30   # pinned host arena (request KV pages alias into it)
METRIC = "decode tokens/sec"
STEP = ("full decoder step: decisions + page table + 32 x (RMSNorm, QKV+RoPE GEMM, paged attention + KV "
        "append, O GEMM + residual, RMSNorm, gate/up GEMM + SiLU, down GEMM + residual)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=WORKLOAD)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pairs", action="store_true", help="N > 1: skip the pair-topology measurement")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-s", type=float, default=20.0)
    ap.add_argument("--attention-only", action="store_true",
                    help="headline step = attention only (no decoder GEMMs); for kernel A/B runs")
    return ap.parse_args()


def load_config(path: str) -> dict:
    """Config JSON with its trace path resolved against the repo root (no product import: the
    reference arm must not load the product library)."""
    with open(path) as f:
        cfg = json.load(f)
    wl = cfg.get("workload", {})
    if wl.get("kind") == "trace" and not os.path.isabs(wl.get("path", "")):
        wl["path"] = os.path.join(ROOT, wl["path"])
    return cfg


def replicated_config(cfg: dict, copies: int, tag: str) -> dict:
    """The weak-scaling global trace: `copies` copies of the config's request set, interleaved so
    that shard p of `copies` (request i -> shard i % copies) is exactly the original trace."""
    if copies <= 1:
        return cfg
    wl = cfg["workload"]
    if wl.get("kind") != "trace" or wl.get("format", "jsonl") != "jsonl":
        raise SystemExit("weak-scaling replication needs a JSONL trace workload")
    lines = [l for l in open(wl["path"]) if l.strip()]
    fd, path = tempfile.mkstemp(prefix=f"asv_trace_{tag}_", suffix=".jsonl")
    with os.fdopen(fd, "w") as f:
        for l in lines:
            f.write((l.rstrip("\n") + "\n") * copies)
    out = json.loads(json.dumps(cfg))
    out["workload"]["path"] = path
    return out


def bench_config(world: int, S: int, W: int, K: int, headline_step: str) -> dict:
    """`config` of the JSON line — identical in both arms (driver checks same_config)."""
    return {"workload": WORKLOAD_NAME, "step": headline_step, "window_iterations": [S + W, S + W + K],
            "parallelism": f"dp{world}", "scaling_rule": "weak: every rank decodes a full C2 request set "
            "(global trace = N copies, request i -> rank i % N)",
            "seq_len": "1K-16K (+ up to 68 generated)",
            "l2": "inputs larger than L2: every step reads ~10-60 GB of KV + 13 GB of weights (L2 is 126 MB)"}


# --------------------------------------------------------------- distributed
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        # testing only: several ranks on one GPU (ASV_BENCH_DEVICE=0 ASV_BENCH_BACKEND=gloo)
        if os.environ.get("ASV_BENCH_DEVICE"):
            self.local = int(os.environ["ASV_BENCH_DEVICE"])
        self.pg = None
        self.backend = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            backend = os.environ.get("ASV_BENCH_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
            if backend == "nccl":
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend)
            self.pg = dist
            self.backend = backend

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def reduce(self, values, op):
        if not self.pg:
            return values
        import torch
        dev = f"cuda:{self.local}" if self.backend == "nccl" else "cpu"
        t = torch.tensor(values, dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=getattr(self.pg.ReduceOp, op))
        return t.cpu().tolist()

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


def relaunch_distributed(args) -> None:
    """`bench.py --gpus N` (N > 1) without a torchrun environment: become torchrun with N ranks."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


# -------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        loaded = [c for c, _, _ in rows if c > 600] or [c for c, _, _ in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(m for _, m, _ in rows),
                "reasons": reasons, "samples": len(rows)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, read+write copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def read_ceiling():
    """Streaming-read ceiling of the decode kernel's own access pattern (per-warp rings of 4 KiB
    bulk loads, no compute), measured by tools/hbm_read_probe.py on a B200 (committed profile)."""
    p = os.path.join(ROOT, "profiles", "hbm_read_probe_r01f.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    v = [x for k, x in d.items() if k.startswith("bulk4k_")]
    return max(v) if v else None


def ncu_traffic():
    """DRAM bytes of ONE profiled decode-attention launch (ncu --set full, committed under
    profiles/) beside that same launch's algorithmic bytes: the traffic ratio is per launch."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        k = json.load(open(p)).get("bench_kernel", {})
    except (OSError, ValueError):
        return None
    dram, alg = k.get("dram_bytes_per_launch"), k.get("alg_bytes_per_launch")
    if not dram or not alg:
        return None
    return {"dram_bytes": dram, "alg_bytes": alg, "ratio": dram / alg, "source": k.get("source")}


def link_probe(dev: int, peer: int | None):
    """Startup measurement of the link rooflines the KV moves run on: pinned host ->
    device over PCIe on this rank's GPU, and device -> device over NVLink to the pair partner."""
    import torch
    out = {}
    n = 1 << 30
    try:
        h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        dbuf = torch.empty(n, dtype=torch.uint8, device=f"cuda:{dev}")
        st = torch.cuda.Stream(device=dev)
        with torch.cuda.device(dev), torch.cuda.stream(st):
            dbuf.copy_(h, non_blocking=True)
            st.synchronize()
            best = 0.0
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                dbuf.copy_(h, non_blocking=True)
                b.record(st)
                b.synchronize()
                best = max(best, n / (a.elapsed_time(b) * 1e-3) / 1e9)
        out["pcie_h2d_gbps"] = best
        if peer is not None and peer != dev and torch.cuda.device_count() > peer:
            pbuf = torch.empty(n, dtype=torch.uint8, device=f"cuda:{peer}")
            with torch.cuda.device(dev), torch.cuda.stream(st):
                dbuf.copy_(pbuf, non_blocking=True)
                st.synchronize()
                best = 0.0
                for _ in range(3):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(st)
                    dbuf.copy_(pbuf, non_blocking=True)
                    b.record(st)
                    b.synchronize()
                    best = max(best, n / (a.elapsed_time(b) * 1e-3) / 1e9)
            out["nvlink_p2p_gbps"] = best
            del pbuf
        del h, dbuf
        torch.cuda.empty_cache()
    except Exception as exc:  # a probe failure must not hide the bench line
        out["error"] = str(exc)
    return out


# ------------------------------------------------------------- CPU reference
def cpu_reference(cfg, window_begin: int, window_end: int, sample_budget_s: float, full_step: bool):
    """The reference's CPU path on this host, over the bench window [window_begin, window_end) of
    the trace: the compiled reference decision engine (oracle/_ref, unmodified headers) for the
    decisions, and per sampled iteration the fp32 CPU oracle of the step — paged attention
    (oracle/attn_oracle.c, all host cores) and, for the full decoder step, the layer's GEMMs,
    RMSNorms, RoPE and SiLU in fp32 numpy (oracle/decoder_oracle.py).  One layer is computed per
    sampled iteration and scaled by the layer count (every layer is identical work).  Iterations are
    taken in window order until the sample budget is spent."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import _util as U  # test-infrastructure loader of the oracles
    import decoder_oracle as D

    attn = cfg["b200"]
    n_q, n_kv, L = attn["num_q_heads"], attn["num_kv_heads"], attn["num_layers"]
    ref = U.RefEngine()
    log, decide_s, iters = ref.run_config_timed(cfg)
    decide_ms = decide_s * 1e3 / max(1, iters)
    its = [json.loads(l) for l in log.splitlines()[1:] if l.startswith('{"attn_ms"')]
    threads = os.cpu_count() or 1
    layer = D.CpuDecoderLayer(n_q, n_kv, 128, threads=threads, full_step=full_step)
    window = its[window_begin:window_end]
    layer.step([int(x) for x in window[0]["prefix_lengths"]])  # untimed: page in weights, thread pools
    tokens, elapsed, done = 0, 0.0, 0
    t_begin = time.time()
    for it in window:
        lens = [int(x) for x in it["prefix_lengths"]]
        layer_s = layer.step(lens)
        elapsed += layer_s * L + decide_ms / 1e3
        tokens += len(lens)
        done += 1
        if time.time() - t_begin > sample_budget_s:
            break
    what = "full decoder step" if full_step else "attention-only step"
    return {"value": tokens / elapsed if elapsed > 0 else 0.0, "unit": "tokens/s", "cores": threads,
            "kind": "reference",
            "sample": (f"the first {done} of the {len(window)} window iterations [{window_begin}, {window_end}) of "
                       f"{os.path.basename(cfg.get('_path', 'C2'))}: decisions by the compiled reference engine "
                       f"({decide_ms * 1e3:.2f} us/iteration), {what} of one layer per iteration by the fp32 CPU "
                       f"oracle on {threads} threads (attention: oracle/attn_oracle.c; GEMMs: numpy/BLAS), "
                       f"x{L} layers"),
            "iterations": done, "seconds_measured": elapsed}


# ------------------------------------------------------------------- main
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_distributed(args)
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if world_env != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}")
    W, K, S = max(3, args.warmup), args.steps, STEADY_START
    full_headline = not args.attention_only
    headline_step = STEP if full_headline else "attention-only step (decisions + page table + 32 attention layers)"
    d = Dist()
    cfg = load_config(args.config)
    cfg["_path"] = args.config
    global WORKLOAD_NAME
    if os.path.abspath(args.config) != os.path.abspath(WORKLOAD):
        WORKLOAD_NAME = f"{os.path.basename(args.config)} (not the headline workload)"
    conf = bench_config(d.world, S, W, K, headline_step)

    if args.impl == "reference":
        # the reference arm never imports the product package (libasv.so stays unloaded)
        if d.rank == 0:
            cpu = cpu_reference(cfg, S + W, S + W + K, args.cpu_sample_s, full_headline)
            line = {"metric": METRIC, "value": cpu["value"], "unit": "tokens/s", "n_gpus": d.world,
                    "steps": K, "warmup": W, "higher_is_better": True, "scaling": "weak",
                    "vs_baseline": None, "dtype": "fp32 (bf16 inputs)", "data": "synthetic",
                    "impl": "reference", "config": conf, "cpu_baseline": dict(cpu),
                    "e2e": {"value": cpu["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                            "d2h_bytes_per_step": 0}}
            print(json.dumps(line), flush=True)
        d.close()
        return

    from paper_2605_23389_b200 import _lib
    from paper_2605_23389_b200 import engine as E

    attn = cfg["b200"]
    dev = d.local
    dp_cfg = replicated_config(cfg, d.world, f"dp{d.rank}")
    base_kw = dict(device=dev, num_q_heads=attn["num_q_heads"], num_kv_heads=attn["num_kv_heads"],
                   num_layers=attn["num_layers"], exec_begin=S, timed_begin=S + W, exec_end=S + W + K,
                   shard_index=d.rank, shard_count=d.world, host_pool_bytes=HOST_POOL_BYTES)
    links = link_probe(dev, dev + 1 if d.world > 1 and d.rank % 2 == 0 else None)
    d.barrier()
    with ClockSampler(dev) as clk:
        res = E.engine_run(dp_cfg, execute_transfers=False, full_step=full_headline, **base_kw)
    clocks = clk.summary()
    d.barrier()
    # the attention-only step over the same window: the dominant kernel's roofline
    att = res if not full_headline else E.engine_run(dp_cfg, execute_transfers=False, **base_kw)
    d.barrier()
    # the same attention-only window with the per-warp %globaltimer probe on every launch:
    # a separate run, so the probe's stores never touch the roofline numbers above
    probe = E.engine_run(dp_cfg, execute_transfers=False, probe_bubble=True, **base_kw)
    d.barrier()

    e2e = e2e_res = e2e_att = e2e_pair1 = e2e_colo = None
    ek = max(K, E2E_MIN_STEPS)
    e2e_kw = dict(base_kw, exec_end=S + W + ek)
    lead = max(0, S - COPY_LEAD)
    if not args.no_e2e:
        e2e = E.engine_run(dp_cfg, execute_transfers=True, copy_begin=lead, full_step=full_headline, **e2e_kw)
        d.barrier()
        # the same (longer) window with the KV resident: what the e2e run would reach without the link
        e2e_res = E.engine_run(dp_cfg, execute_transfers=False, full_step=full_headline, **e2e_kw)
        d.barrier()
        if full_headline:  # attention-only end to end: the link vs the attention kernel alone
            e2e_att = E.engine_run(dp_cfg, execute_transfers=True, copy_begin=lead, **e2e_kw)
            d.barrier()
        if d.world == 1:
            # the pair data path on this one device: candidate buffers in their own pool, every admit /
            # evict a real device move on the pair's P2P lane (the NVLink push of a 2-GPU pair)
            e2e_pair1 = E.engine_run(dp_cfg, execute_transfers=True, copy_begin=lead, pair_mode=True,
                                     full_step=full_headline, **e2e_kw)
            # the prefill instance colocated on this GPU: every prefill_offload is a real D2H copy
            # sharing this GPU's PCIe link with the prefetches
            e2e_colo = E.engine_run(dp_cfg, execute_transfers=True, copy_begin=lead, prefill_offload=True,
                                    full_step=full_headline, **e2e_kw)

    # ---- north-star pair topology (N even): (decode, prefetch) pairs, requests sharded over pairs
    pairs = None
    if d.world > 1 and d.world % 2 == 0 and not args.no_pairs and not args.no_e2e:
        P = d.world // 2
        pr_cfg = replicated_config(cfg, P, f"pair{d.rank}")
        pkw = dict(e2e_kw, shard_index=d.rank // 2, shard_count=P)
        if os.environ.get("ASV_BENCH_DEVICE"):  # testing: the pair on one device (separate pools)
            pkw.update(pair_mode=True)
        else:
            pkw.update(prefetch_device=dev + 1)
        d.barrier()
        pair_err = None
        if d.rank % 2 == 0:
            try:  # never measured on two physical GPUs before the driver's run: an error is reported, not fatal
                pr = E.engine_run(pr_cfg, execute_transfers=True, copy_begin=lead, full_step=full_headline, **pkw)
            except Exception as ex:  # noqa: BLE001
                pair_err = f"{type(ex).__name__}: {ex}"
                pr = _lib.EngineStats().as_dict()
        else:  # the prefetch rank's GPU is driven by its decode partner's engine
            pr = _lib.EngineStats().as_dict()
        d.barrier()
        pw = d.reduce([pr["window_ms"]], "MAX")[0]
        ptok = d.reduce([float(pr["tokens_timed"])], "SUM")[0]
        psteps = max(1, pr["iterations_timed"])
        if pr_cfg is not cfg:
            os.unlink(pr_cfg["workload"]["path"])
        pairs = {"value": ptok / (pw / 1e3) if pw > 0 else 0.0, "unit": "tokens/s", "parallelism": f"pairs{P}",
                 "e2e": True, "ms_per_step": pw / psteps, "window_steps": int(pr["iterations_timed"]),
                 "p2p_bytes_per_step": int(pr["p2p_bytes_window"] / psteps),
                 "h2d_bytes_per_step": int(pr["h2d_bytes_window"] / psteps),
                 "p2p_gbps": (pr["p2p_bytes_window"] / (pr["p2p_busy_ms"] * 1e-3) / 1e9
                              if pr["p2p_busy_ms"] > 0 else None),
                 "what": "end to end, north-star topology: ranks 2p / 2p+1 = (decode, prefetch) GPU pair; "
                         "global trace = N/2 copies of C2 sharded over the pairs; prefetch GPU pulls KV from "
                         "pinned host memory (PCIe) and carries the prefill offloads, admits / evicts are SM "
                         "page moves over NVLink peer pointers into / out of the decode GPU"}
        n_err = int(d.reduce([1.0 if pair_err else 0.0], "SUM")[0])
        if n_err:
            pairs["error"] = {"failed_pairs": n_err, "rank0": pair_err}

    # ---- reductions (max window over ranks, summed tokens)
    def rate(st):
        w = d.reduce([st["window_ms"]], "MAX")[0]
        t = d.reduce([float(st["tokens_timed"])], "SUM")[0]
        return (t / (w / 1e3) if w > 0 else 0.0), w

    value, win = rate(res)
    att_value, att_win = rate(att)
    peak, peak_src = measured_peaks()
    achieved = att["attn_bytes"] / (att["attn_ms"] * 1e-3) / 1e9 if att["attn_ms"] > 0 else 0.0
    launches = max(1, att["attn_launches"])
    tr = ncu_traffic()
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": tr["dram_bytes"] if tr else None,
                "traffic_launch_alg_bytes": tr["alg_bytes"] if tr else None,
                "traffic_ratio": tr["ratio"] if tr else None,
                "traffic_source": tr["source"] if tr else None, "peak_source": peak_src,
                "kernel": "decode_attn_kernel (split-KV, PDL-chained; the previous layer's split merge folded into each launch, the last layer's by merge_splits_kernel), per layer",
                "alg_bytes_per_launch": att["attn_bytes"] / launches,
                "avg_launch_us": att["attn_ms"] * 1e3 / launches,
                "frac_of_8TBps": achieved / 8000.0}
    rc = read_ceiling()
    if rc:
        roofline.update({"read_ceiling_gbps": rc, "frac_of_read_ceiling": achieved / rc,
                         "read_ceiling_source": "profiles/hbm_read_probe_r01f.json (4 KiB bulk-load rings, "
                                                "no compute; MEASURED_PEAKS is a read+write copy)"})

    def e2e_block(st, st_res):
        w = d.reduce([st["window_ms"]], "MAX")[0]
        t = d.reduce([float(st["tokens_timed"])], "SUM")[0]
        n = max(1, st["iterations_timed"])
        link = st["pcie_union_ms"]
        busy = st["attn_ms"]  # GPU decode time of the window (att_beg..att_end of every step)
        overlap = max(0.0, link + busy - st["window_ms"])
        blk = {"value": t / (w / 1e3) if w > 0 else 0.0, "unit": "tokens/s",
               "h2d_bytes_per_step": int(st["h2d_bytes_window"] / n),
               "d2h_bytes_per_step": int((st["d2h_bytes_window"] + st["offload_bytes_window"] +
                                          st["result_d2h_bytes_window"]) / n),
               "prefill_offload_d2h_bytes_per_step": int(st["offload_bytes_window"] / n),
               "p2p_bytes_per_step": int(st["p2p_bytes_window"] / n),
               "ms_per_step": w / n, "window_steps": int(st["iterations_timed"]),
               "decode_ms_per_step": busy / n, "pcie_busy_ms_per_step": link / n,
               "pcie_utilisation": link / max(1e-9, st["window_ms"]),
               "prefetch_hidden_fraction": overlap / link if link > 0 else None,
               "prefetch_hidden_fraction_def": "time the PCIe link and decode were both busy / PCIe busy time",
               "h2d_gbps": ((st["h2d_bytes_window"] + st["d2h_bytes_window"]) / (link * 1e-3) / 1e9
                            if link > 0 else None),
               "bound": "pcie" if link >= busy else "hbm"}
        if st_res is not None:
            rv, _ = rate(st_res)
            blk["resident_value_same_window"] = rv
        return blk

    e2e_obj = None
    if e2e is not None:
        e2e_obj = e2e_block(e2e, e2e_res)
        e2e_obj["path"] = ("asv_engine_run (C ABI): KV moves from/to the pinned host pool + per-step result "
                           "read-back to pinned host memory, inside the timed region")
        if e2e_pair1 is not None:
            b = e2e_block(e2e_pair1, None)
            b["p2p_copy_gbps"] = (e2e_pair1["p2p_bytes_window"] / (e2e_pair1["p2p_busy_ms"] * 1e-3) / 1e9
                                  if e2e_pair1["p2p_busy_ms"] > 0 else None)
            b["what"] = ("same window with the (prefetch, decode) pair's data path on this one GPU: admits / "
                         "evicts are SM page moves between the candidate-buffer pool and the decode pool on the "
                         "P2P lane (HBM to HBM here; NVLink peer pulls with two GPUs)")
            e2e_obj["pair_path_one_device"] = b
        if e2e_colo is not None:
            b = e2e_block(e2e_colo, None)
            b["what"] = ("same window, plus every prefill_offload (reference cluster_sim.hpp:285-299) executed as a "
                         "D2H copy into the host pool over this GPU's own PCIe link (prefill instance colocated); "
                         "the headline e2e leaves it to the prefill instance's link, as the reference's "
                         "disaggregated model does")
            e2e_obj["colocated_prefill_offload"] = b

    att_obj = {"value": att_value, "unit": "tokens/s", "ms_per_step": att_win / max(1, att["iterations_timed"]),
               "decode_attn_hbm_gbps": achieved,
               "what": "same window, attention only (32 x paged split-KV attention + KV append per step, "
                       "no decoder GEMMs)"}
    if e2e_att is not None:
        att_obj["e2e"] = e2e_block(e2e_att, None)

    full_obj = None
    if full_headline:
        f_steps = max(1, res["iterations_timed"])
        f_bytes = res["attn_bytes"] + res["weight_bytes"]
        full_obj = {"weight_gb_per_step": res["weight_bytes"] / f_steps / 1e9,
                    "kv_gb_per_step": res["attn_bytes"] / f_steps / 1e9,
                    "hbm_gbps": f_bytes / (res["window_ms"] * 1e-3) / 1e9 if res["window_ms"] > 0 else None,
                    "frac_of_hbm_peak": (f_bytes / (res["window_ms"] * 1e-3) / 1e9 / peak
                                         if res["window_ms"] > 0 else None)}

    cpu = None
    if d.rank == 0 and d.world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference(cfg, S + W, S + W + K, args.cpu_sample_s, full_headline)
        except Exception as exc:  # baseline is reported, never required
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if d.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": d.world, "steps": K,
            "warmup": W, "ms_per_step": win / max(1, res["iterations_timed"]), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": (f"synthetic: deterministic splitmix64 trace {os.path.basename(cfg['workload'].get('path', '?'))}"
                     f" (x{d.world} for N ranks), random bf16 KV / activations / weights"),
            "config": conf,
            "mean_batch": res["tokens_timed"] / max(1, res["iterations_timed"]),
            "e2e": e2e_obj, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks,
            "gpu_launches": int(res["kernel_launches_timed"]),
            "decode_attn_hbm_gbps": achieved, "attention_only": att_obj, "full_decode_step": full_obj,
            "links": links, "pairs": pairs,
            "virtual_clock_tok_s": res["virtual_decode_tok_s"],
            "bubble_ms_per_step_virtual": res["bubble_ms_timed"] / max(1, res["iterations_timed"]),
            "bubble_measured": {"idle_frac": probe["measured_idle_frac"],
                                "ms_per_step": probe["measured_bubble_ms"] / max(1, probe["iterations_timed"]),
                                "per_iteration_ms": {"p50": probe["bubble_p50_ms"], "p90": probe["bubble_p90_ms"],
                                                     "p99": probe["bubble_p99_ms"], "max": probe["bubble_max_ms"],
                                                     "iterations": probe["bubble_iterations"]},
                                "probe": "per-warp %globaltimer start/end of every attention launch (all 32 layers) "
                                         "of every timed step; bubble of a launch = sum over warps of (launch span - "
                                         "warp busy) / warps; per iteration = sum over its launches (attention-only "
                                         "run with the probe, separate from the roofline run)"},
            "host_decide_ms": res["host_decide_ms"],
            "logical_bytes_moved": res["logical_bytes"],
        }
        print(json.dumps(line), flush=True)
    for c in (dp_cfg,):
        if c is not cfg:
            try:
                os.unlink(c["workload"]["path"])
            except OSError:
                pass
    d.close()


if __name__ == "__main__":
    main()
