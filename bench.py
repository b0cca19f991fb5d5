#!/usr/bin/env python
"""Benchmark of the B200-native AlignedServe decode-iteration hot path.

Metric (BASELINE.json): decode tokens/sec at 1/2/4/8 B200, with decode-attention
HBM GB/s and KV-prefetch GB/s beside it.  Workload at N=1: BASELINE configs[1]
("Llama-2-7B-shape synthetic trace, 1024 in-flight requests in host memory, KV
lengths 1K-16K, bf16 KV, 1 B200") = configs/c2_7b_1024req.json.

A step is one decode iteration of the engine: the reference-API scheduler's
boundary decisions (virtual clock, bit-exact with the reference), the page-table
build + upload, and attention over all 32 layers (one persistent sm_100a decode
kernel per layer plus a PDL-chained split-merge kernel).  Iterations [S, S+W)
are warm-up, [S+W, S+W+K) are timed with CUDA events on the compute stream; S is
a steady-state point of the trace (earlier iterations run decisions only).

  value : KV resident in HBM when the window starts (no KV moves executed)
  e2e   : the same window through the C-ABI engine (asv_engine_run) with every
          boundary KV move executed from/to the pinned host pool (H2D prefetch,
          D2H spill/flush; P2P with a partner GPU) and every step's result
          (attention output) read back to pinned host memory, inside the timed
          region; >= 500 steps because prefetch traffic is bursty

N > 1 (torchrun): requests are sharded data-parallel (request i -> rank i % N),
every rank runs its shard's engine on its GPU, no data-path collective; the
window is the max over ranks.  `--topology pairs`: ranks 2p (decode) and 2p+1
(prefetch) form a pair; the decode rank's engine drives both GPUs (candidate
buffers, host->GPU prefetches and prefill offloads on the prefetch GPU, admits /
evicts as NVLink peer copies), requests are sharded over the N/2 pairs, and the
prefetch rank only joins the barriers and reductions.  `--impl reference` times the reference's CPU
path (the compiled reference decision engine + the fp32 CPU attention oracle)
on the host cores instead.
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
                 "1024 requests in the host pool, KV 1K-16K, aligned policy, 1 B200 per shard")
STEADY_START = 300          # first executed iteration of the trace (per shard)
COPY_LEAD = 400             # KV moves are executed from this many iterations before the span
E2E_MIN_STEPS = 500         # e2e window: prefetch traffic is bursty (batch switches), so the
                            # end-to-end rate is taken over >= this many steps
HOST_POOL_BYTES = 4 << 30   # pinned host arena (request KV pages alias into it)
METRIC = "decode tokens/sec"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=WORKLOAD)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-full-step", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-s", type=float, default=12.0)
    ap.add_argument("--topology", default="dp", choices=["dp", "pairs"],
                    help="dp: every GPU decodes its own shard over its own PCIe link (default); pairs: "
                         "GPUs 2p / 2p+1 form a (decode, prefetch) pair, the prefetch GPU pulls KV from host "
                         "memory and pushes it to its decode partner over NVLink (SURVEY §8(e))")
    return ap.parse_args()


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
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
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
    """dram bytes per launch of the decode kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            return d.get("bench_kernel", {}).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            return None
    return None


# ------------------------------------------------------------- CPU reference
def cpu_reference(cfg, steps: int, start: int, sample_budget_s: float):
    """The reference's CPU path on this host: the compiled reference decision
    engine (oracle/_ref, unmodified headers) for the decisions, and the fp32 CPU
    attention oracle (all host cores) for the attention of each sampled
    iteration.  One layer is computed per sampled iteration and scaled by the
    layer count (layers are identical work)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import _util as U  # test-infrastructure loader of the oracles

    attn = cfg["b200"]
    n_q, n_kv, L = attn["num_q_heads"], attn["num_kv_heads"], attn["num_layers"]
    ref = U.RefEngine()
    log, secs, iters = ref.run_config_jsonl(cfg)
    decide_ms = secs * 1e3 / max(1, iters)
    its = [json.loads(l) for l in log.splitlines()[1:] if l.startswith('{"attn_ms"')]
    oracle = U.Oracle()
    threads = os.cpu_count() or 1
    # one-layer paged pool, aliased (KV content does not change the work)
    pool_pages = 1024
    pb = U.page_bytes(n_kv, 1)
    pool = U.random_bf16(5, pool_pages * pb // 2).view(np.uint8)
    rng = np.random.default_rng(0)
    tokens = 0
    elapsed = 0.0
    done = 0
    t_begin = time.time()
    for it in its[start:start + steps]:
        lens = [int(x) for x in it["prefix_lengths"]]
        indptr = np.zeros(len(lens) + 1, np.int32)
        indptr[1:] = np.cumsum([(s + 15) // 16 for s in lens])
        indices = rng.integers(0, pool_pages, int(indptr[-1])).astype(np.int32)
        q = U.random_bf16(7, len(lens) * n_q * 128)
        t0 = time.perf_counter()
        oracle.attention(n_q, n_kv, 1, 0, q, pool, lens, indptr, indices, 0.08838834764831845, threads)
        layer_s = time.perf_counter() - t0
        elapsed += layer_s * L + decide_ms / 1e3
        tokens += len(lens)
        done += 1
        if time.time() - t_begin > sample_budget_s:
            break
    return {"value": tokens / elapsed if elapsed > 0 else 0.0, "unit": "tokens/s", "cores": threads,
            "kind": "reference",
            "sample": (f"{done} decode iterations of {os.path.basename(cfg.get('_path', 'C2'))} from iteration "
                       f"{start}: decisions by the compiled reference engine ({decide_ms*1e3:.1f} us/iteration), "
                       f"attention of one layer per iteration by the fp32 CPU oracle on {threads} threads, "
                       f"x{L} layers"),
            "iterations": done, "seconds_measured": elapsed}


# ------------------------------------------------------------------- main
def main():
    args = parse()
    if args.warmup < 3:
        args.warmup = 3
    d = Dist()
    from paper_2605_23389_b200 import engine as E

    cfg = E.load_config(args.config)
    cfg["_path"] = args.config
    global WORKLOAD_NAME
    if os.path.abspath(args.config) != os.path.abspath(WORKLOAD):
        WORKLOAD_NAME = f"{os.path.basename(args.config)} (not the headline workload)"
    attn = cfg["b200"]
    S, W, K = STEADY_START, args.warmup, args.steps

    if args.impl == "reference":
        if d.rank == 0:
            cpu = cpu_reference(cfg, W + K, S, sample_budget_s=max(30.0, args.cpu_sample_s))
            line = {"metric": METRIC, "value": cpu["value"], "unit": "tokens/s", "n_gpus": d.world,
                    "steps": K, "warmup": W, "higher_is_better": True, "scaling": "weak",
                    "vs_baseline": None, "dtype": "fp32 (bf16 inputs)", "data": "synthetic",
                    "impl": "reference",
                    "config": {"workload": WORKLOAD_NAME, "parallelism": "host cores"},
                    "cpu_baseline": dict(cpu),
                    "e2e": {"value": cpu["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                            "d2h_bytes_per_step": 0}}
            print(json.dumps(line), flush=True)
        d.close()
        return

    dev = d.local
    pairs = args.topology == "pairs" and d.world > 1
    if pairs and d.world % 2:
        raise SystemExit("--topology pairs needs an even number of GPUs")
    run_kw = dict(device=dev, num_q_heads=attn["num_q_heads"], num_kv_heads=attn["num_kv_heads"],
                  num_layers=attn["num_layers"], exec_begin=S, timed_begin=S + W, exec_end=S + W + K,
                  shard_index=d.rank, shard_count=d.world, host_pool_bytes=HOST_POOL_BYTES)
    idle = False  # a pair's prefetch rank: its GPU is driven by the decode rank's engine
    if pairs:
        run_kw.update(shard_index=d.rank // 2, shard_count=d.world // 2)
        if os.environ.get("ASV_BENCH_DEVICE"):  # testing: the pair on one device (separate pools)
            run_kw.update(pair_mode=True)
        else:
            run_kw.update(prefetch_device=dev + 1)
        idle = d.rank % 2 == 1

    def run_engine(cfg_, **kw):
        """asv_engine_run on this rank's GPU(s); a pair's prefetch rank runs nothing (zero stats)."""
        if idle:
            from paper_2605_23389_b200 import _lib
            return _lib.EngineStats().as_dict()
        return E.engine_run(cfg_, **kw)
    d.barrier()
    with ClockSampler(dev) as clk:
        res = run_engine(cfg, execute_transfers=False, **run_kw)
    clocks = clk.summary()
    d.barrier()
    # the whole decoder layer stack per step (RMSNorm, QKV+RoPE / O / gate-up / down GEMMs on
    # tcgen05 with synthetic weights, attention), KV resident: SURVEY §8(f) rank 1
    full = None
    if not args.no_full_step:
        full = run_engine(cfg, execute_transfers=False, full_step=True, **run_kw)
        d.barrier()
    e2e = None
    if not args.no_e2e:
        ek = max(K, E2E_MIN_STEPS)
        kw = dict(run_kw, exec_end=S + W + ek)
        e2e = run_engine(cfg, execute_transfers=True, copy_begin=max(0, S - COPY_LEAD), **kw)
        d.barrier()
        # the same (longer) window with the KV resident: what the e2e run would reach without the link
        e2e_res = run_engine(cfg, execute_transfers=False, **kw)
        d.barrier()
        # end to end with the whole decoder layer stack per step: decode work long enough to hide the
        # KV prefetch behind it
        e2e_full = None
        if not args.no_full_step:
            e2e_full = run_engine(cfg, execute_transfers=True, copy_begin=max(0, S - COPY_LEAD), full_step=True,
                                    **kw)
            d.barrier()
        # the same window with the prefill instance colocated on this GPU: every prefill_offload
        # (prefill GPU -> host pool) is a real D2H copy sharing this GPU's PCIe link with the prefetches
        # the pair data path on this one device: candidate buffers in their own pool, every admit /
        # evict a real device copy on the pair's P2P lane (the NVLink push of a 2-GPU pair)
        e2e_pair1 = None
        if not pairs and d.world == 1:
            e2e_pair1 = run_engine(cfg, execute_transfers=True, copy_begin=max(0, S - COPY_LEAD), pair_mode=True,
                                   **kw)
            d.barrier()
        e2e_colo = None
        if not pairs:  # a pair already runs its prefill offloads on the prefetch GPU's link
            e2e_colo = run_engine(cfg, execute_transfers=True, copy_begin=max(0, S - COPY_LEAD),
                                    prefill_offload=True, **kw)
            d.barrier()

    win, tok = d.reduce([res["window_ms"], float(res["tokens_timed"])], "MAX")[0], \
        d.reduce([float(res["tokens_timed"])], "SUM")[0]
    value = tok / (win / 1e3) if win > 0 else 0.0
    e2e_obj = None
    if e2e is not None:
        ewin = d.reduce([e2e["window_ms"]], "MAX")[0]
        etok = d.reduce([float(e2e["tokens_timed"])], "SUM")[0]
        e2e_obj = {"value": etok / (ewin / 1e3) if ewin > 0 else 0.0, "unit": "tokens/s",
                   "h2d_bytes_per_step": int(e2e["h2d_bytes_window"] / max(1, e2e["iterations_timed"])),
                   "d2h_bytes_per_step": int((e2e["d2h_bytes_window"] + e2e["offload_bytes_window"] +
                                              e2e["result_d2h_bytes_window"]) / max(1, e2e["iterations_timed"])),
                   "prefill_offload_d2h_bytes_per_step": int(e2e["offload_bytes_window"] /
                                                             max(1, e2e["iterations_timed"])),
                   "p2p_bytes_per_step": int(e2e["p2p_bytes_window"] / max(1, e2e["iterations_timed"])),
                   "ms_per_step": ewin / max(1, e2e["iterations_timed"]),
                   "window_steps": int(e2e["iterations_timed"]),
                   "resident_value_same_window": (d.reduce([float(e2e_res["tokens_timed"])], "SUM")[0] /
                                                  (d.reduce([e2e_res["window_ms"]], "MAX")[0] / 1e3)),
                   "path": "asv_engine_run (C ABI): KV moves from/to the pinned host pool (incl. prefill offloads prefill GPU -> host pool) + per-step result "
                           "read-back to pinned host memory"}
        if e2e_full is not None:
            fw = d.reduce([e2e_full["window_ms"]], "MAX")[0]
            fsteps = max(1, e2e_full["iterations_timed"])
            link = e2e_full["pcie_union_ms"]
            e2e_obj["full_step"] = {
                "value": d.reduce([float(e2e_full["tokens_timed"])], "SUM")[0] / (fw / 1e3) if fw > 0 else 0.0,
                "unit": "tokens/s", "ms_per_step": fw / fsteps,
                "decode_ms_per_step": e2e_full["attn_ms"] / fsteps,
                "pcie_busy_ms_per_step": link / fsteps,
                "prefetch_hidden_fraction": (max(0.0, link + e2e_full["attn_ms"] - e2e_full["window_ms"]) / link
                                             if link > 0 else None),
                "what": "same window and KV moves, every step runs the full decoder layer stack (see full_decode_step)"}

    if e2e is not None and e2e_colo is not None:
        cw = d.reduce([e2e_colo["window_ms"]], "MAX")[0]
        c_steps = max(1, e2e_colo["iterations_timed"])
        c_link = e2e_colo["pcie_union_ms"]
        e2e_obj["colocated_prefill_offload"] = {
            "value": d.reduce([float(e2e_colo["tokens_timed"])], "SUM")[0] / (cw / 1e3) if cw > 0 else 0.0,
            "unit": "tokens/s", "ms_per_step": cw / c_steps,
            "h2d_bytes_per_step": int(e2e_colo["h2d_bytes_window"] / c_steps),
            "d2h_bytes_per_step": int((e2e_colo["d2h_bytes_window"] + e2e_colo["offload_bytes_window"] +
                                       e2e_colo["result_d2h_bytes_window"]) / c_steps),
            "pcie_gbps_both_directions": ((e2e_colo["h2d_bytes_window"] + e2e_colo["d2h_bytes_window"] +
                                           e2e_colo["offload_bytes_window"]) / (c_link * 1e-3) / 1e9
                                          if c_link > 0 else None),
            "what": "same window, plus every prefill_offload (reference cluster_sim.hpp:285-299) executed as a D2H "
                    "copy into the host pool over this GPU's own PCIe link (prefill instance colocated); the "
                    "headline e2e leaves it to the prefill instance's link, as the reference's disaggregated "
                    "model does"}

    if e2e is not None and e2e_pair1 is not None:
        pw = e2e_pair1["window_ms"]
        ps = max(1, e2e_pair1["iterations_timed"])
        e2e_obj["pair_path_one_device"] = {
            "value": e2e_pair1["tokens_timed"] / (pw / 1e3) if pw > 0 else 0.0, "unit": "tokens/s",
            "p2p_bytes_per_step": int(e2e_pair1["p2p_bytes_window"] / ps),
            "p2p_copy_gbps": (e2e_pair1["p2p_bytes_window"] / (e2e_pair1["p2p_busy_ms"] * 1e-3) / 1e9
                              if e2e_pair1["p2p_busy_ms"] > 0 else None),
            "what": "same window with the (prefetch, decode) pair's data path on this one GPU: admits / evicts "
                    "are device copies between the candidate-buffer pool and the decode pool on the P2P lane "
                    "(HBM to HBM here; NVLink peer copies with two GPUs, roofline 770 GB/s)"}

    peak, peak_src = measured_peaks()
    achieved = res["attn_bytes"] / (res["attn_ms"] * 1e-3) / 1e9 if res["attn_ms"] > 0 else 0.0
    launches = max(1, res["attn_launches"])
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": ncu_traffic(), "peak_source": peak_src,
                "kernel": "decode_attn_kernel + merge_splits_kernel (split-KV, PDL-chained), per layer",
                "alg_bytes_per_launch": res["attn_bytes"] / launches,
                "avg_launch_us": res["attn_ms"] * 1e3 / launches,
                "frac_of_8TBps": achieved / 8000.0}
    rc = read_ceiling()
    if rc:
        roofline.update({"read_ceiling_gbps": rc, "frac_of_read_ceiling": achieved / rc,
                         "read_ceiling_source": "profiles/hbm_read_probe_r01f.json (4 KiB bulk-load rings, "
                                                "no compute; MEASURED_PEAKS is a read+write copy)"})
    prefetch = None
    if e2e is not None:
        # PCIe link: union of the copy intervals of all PCIe lanes inside the window
        e_steps = max(1, e2e["iterations_timed"])
        link_ms = e2e["pcie_union_ms"]
        kv_bytes = e2e["h2d_bytes_window"] + e2e["d2h_bytes_window"]
        d2h_bytes = e2e["d2h_bytes_window"] + e2e["offload_bytes_window"]
        p2p_gbps = e2e["p2p_bytes_window"] / (e2e["p2p_busy_ms"] * 1e-3) / 1e9 if e2e["p2p_busy_ms"] > 0 else None
        overlap = max(0.0, link_ms + e2e["attn_ms"] - e2e["window_ms"])
        shorter = min(link_ms, e2e["attn_ms"])
        prefetch = {"h2d_gbps": kv_bytes / (link_ms * 1e-3) / 1e9 if link_ms > 0 else None,
                    "d2h_gbps_same_window": d2h_bytes / (link_ms * 1e-3) / 1e9 if link_ms > 0 else None,
                    "h2d_roofline_gbps": 64.0, "h2d_frac_of_roofline": (kv_bytes / (link_ms * 1e-3) / 1e9 / 64.0
                                                                         if link_ms > 0 else None),
                    "p2p_gbps": p2p_gbps, "p2p_roofline_gbps": 770.0,
                    "pcie_busy_ms_per_step": link_ms / e_steps,
                    "attn_ms_per_step": e2e["attn_ms"] / e_steps,
                    "pcie_utilisation": link_ms / max(1e-9, e2e["window_ms"]),
                    "copy_compute_overlap_ms_per_step": overlap / e_steps,
                    "hidden_fraction": overlap / shorter if shorter > 0 else None,
                    "hidden_fraction_def": "overlap of PCIe-busy and attention time / the shorter of the two",
                    "bound": "pcie" if link_ms >= e2e["attn_ms"] else "hbm"}

    full_obj = None
    if full is not None:
        fwin = d.reduce([full["window_ms"]], "MAX")[0]
        ftok = d.reduce([float(full["tokens_timed"])], "SUM")[0]
        f_steps = max(1, full["iterations_timed"])
        f_bytes = full["attn_bytes"] + full["weight_bytes"]
        full_obj = {"value": ftok / (fwin / 1e3) if fwin > 0 else 0.0, "unit": "tokens/s",
                    "ms_per_step": fwin / f_steps,
                    "what": "per step and layer: RMSNorm, QKV GEMM + RoPE, paged attention + KV append, O GEMM + "
                            "residual, RMSNorm, gate/up GEMM + SiLU, down GEMM + residual (bf16, fp32 accumulate; "
                            "GEMMs on tcgen05, synthetic Llama-2-7B-shape weights; after layer 0 each RMSNorm is "
                            "fused into the next GEMM: norm weight folded into its weights, 1/rms per row from the "
                            "residual GEMM's row sums of squares)",
                    "weight_gb_per_step": full["weight_bytes"] / f_steps / 1e9,
                    "kv_gb_per_step": full["attn_bytes"] / f_steps / 1e9,
                    "hbm_gbps": f_bytes / (full["window_ms"] * 1e-3) / 1e9 if full["window_ms"] > 0 else None,
                    "frac_of_hbm_peak": (f_bytes / (full["window_ms"] * 1e-3) / 1e9 / peak
                                         if full["window_ms"] > 0 else None),
                    "gpu_launches": int(full["kernel_launches_timed"])}

    cpu = None
    if d.rank == 0 and d.world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference(cfg, 10_000, S, sample_budget_s=args.cpu_sample_s)
        except Exception as exc:  # baseline is reported, never required
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if d.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": d.world, "steps": K,
            "warmup": W, "ms_per_step": win / max(1, res["iterations_timed"]), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": (f"synthetic: deterministic splitmix64 trace {cfg.get('workload', {}).get('path', '?')}, "
                     "random bf16 KV/q"),
            "config": {"workload": WORKLOAD_NAME, "global_batch": tok / max(1, res["iterations_timed"]),
                       "seq_len": "1K-16K (+ up to 68 generated)", "parallelism": f"pairs{d.world // 2}" if pairs else f"dp{d.world}",
                       "steady_start_iteration": S,
                       "l2": "inputs larger than L2: every step reads ~10-60 GB of KV (L2 is 126 MB)"},
            "e2e": e2e_obj, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks,
            "full_decode_step": full_obj,
            "gpu_launches": int(res["kernel_launches_timed"]),
            "decode_attn_hbm_gbps": achieved, "kv_prefetch": prefetch,
            "virtual_clock_tok_s": res["virtual_decode_tok_s"],
            "bubble_ms_per_step_virtual": res["bubble_ms_timed"] / max(1, res["iterations_timed"]),
            "bubble_measured": {"idle_frac": res["measured_idle_frac"],
                                "ms_per_step": res["measured_bubble_ms"] / max(1, res["iterations_timed"]),
                                "probe": "per-warp %globaltimer start/end of each step's layer-0 launch"},
            "host_decide_ms": res["host_decide_ms"],
            "logical_bytes_moved": res["logical_bytes"],
        }
        print(json.dumps(line), flush=True)
    d.close()


if __name__ == "__main__":
    main()
