"""Python face of the host-side decision path (C++ behind include/asv.h).

Mirrors the reference's entry points on the decode path:
  * run_config_jsonl  ~ `prefixsim run --config X` (experiment_from_json ->
    run_experiment -> log_to_jsonl; reference prefixsim_main.cpp:66-111,
    io.hpp:184-254, io.hpp:279-323), virtual-clock mode;
  * dfs_batch         ~ density_first_search on a pool snapshot
    (reference batch_gen.hpp:126-210); member order = page-table order.
Errors map to the reference's exception types: ValueError for
std::invalid_argument, AssertionError for std::logic_error, RuntimeError for
std::runtime_error, with the same messages.
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from . import _lib


def run_config_jsonl(config, policy: str | None = None) -> str:
    """Run one experiment config (dict or JSON text) and return the schema-1 JSONL log."""
    text = config if isinstance(config, str) else json.dumps(config)
    out = C.c_void_p()
    n = C.c_int64(0)
    h = _lib.lib()
    _lib.check(h.asv_run_config_jsonl(text.encode(), policy.encode() if policy else None,
                                      C.byref(out), C.byref(n)))
    try:
        return C.string_at(out.value, n.value).decode()
    finally:
        h.asv_free(out)


def run_config_jsonl_shard(config, shard_index: int, shard_count: int, policy: str | None = None) -> str:
    """Schema-1 log of one data-parallel shard (request i -> shard i % shard_count)."""
    text = config if isinstance(config, str) else json.dumps(config)
    out = C.c_void_p()
    n = C.c_int64(0)
    h = _lib.lib()
    _lib.check(h.asv_run_config_jsonl_shard(text.encode(), policy.encode() if policy else None,
                                            int(shard_index), int(shard_count), C.byref(out), C.byref(n)))
    try:
        return C.string_at(out.value, n.value).decode()
    finally:
        h.asv_free(out)


def dfs_batch(residents, b_max: int, k_min: int):
    """residents: [(id, prefix_len, kv_blocks)] in insertion order -> (member ids, total_blocks)."""
    arr = np.ascontiguousarray(np.asarray(residents, dtype=np.int64).reshape(-1, 3))
    n = arr.shape[0]
    ids = np.zeros(max(n, 1), dtype=np.int64)
    cnt = C.c_int64(0)
    tot = C.c_int64(0)
    p64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731
    _lib.check(_lib.lib().asv_dfs_batch(p64(arr), n, int(b_max), int(k_min), p64(ids),
                                         C.byref(cnt), C.byref(tot)))
    return ids[:cnt.value].tolist(), int(tot.value)


def load_config(path: str, root: str | None = None) -> dict:
    """Read a config JSON; trace paths are resolved against `root` (default: the repo root)."""
    import os
    root = root or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(path) as f:
        cfg = json.load(f)
    wl = cfg.get("workload", {})
    if wl.get("kind") == "trace" and not os.path.isabs(wl.get("path", "")):
        wl["path"] = os.path.join(root, wl["path"])
    return cfg


def engine_run(config, *, device: int = 0, prefetch_device: int | None = None,
               num_q_heads: int, num_kv_heads: int, num_layers: int, execute_transfers: bool,
               exec_begin: int = 0, exec_end: int = -1, timed_begin: int = 0, copy_begin: int | None = None,
               host_pool_bytes: int = 8 << 30, shard_index: int = 0, shard_count: int = 1,
               pdl: bool = True, run_ahead: int = 256, policy: str | None = None,
               pair_mode: bool = False, full_step: bool = False, intermediate_size: int = 0,
               prefill_offload: bool | None = None, out_dir: str | None = None, return_log: bool = False,
               probe_bubble: bool = False, content_check: bool = False, capture_path: str | None = None,
               capture_every: int = 1, wall_clock: bool = False):
    """Run the decode engine on the GPU (asv_engine_run_ex): reference decisions executed for real.

    Returns the stats dict; with return_log=True, (stats, schema-1 JSONL log).  out_dir: also write
    the reference's run artefacts there (log.jsonl, summary.json, CDF CSVs) plus gpu_stats.json.
    probe_bubble: measure the intra-iteration bubble of every attention launch of the timed window
    (stats["bubble_per_iteration_ms"] lists it per timed iteration).  content_check / capture_path /
    capture_every: the content-check test mode (include/asv.h) writing every executed iteration's
    attention outputs to capture_path (read it with read_capture).  wall_clock: decisions against
    measured iteration times instead of the reference's virtual clock (asv.h wall_clock)."""
    text = config if isinstance(config, str) else json.dumps(config)
    o = _lib.EngineOpts()
    o.decode_device = device
    o.prefetch_device = device if prefetch_device is None else prefetch_device
    o.num_q_heads, o.num_kv_heads, o.num_layers = num_q_heads, num_kv_heads, num_layers
    o.execute_transfers = 1 if execute_transfers else 0
    o.host_pool_bytes = host_pool_bytes
    o.exec_begin, o.exec_end, o.timed_begin = exec_begin, exec_end, timed_begin
    o.copy_begin = exec_begin if copy_begin is None else copy_begin
    o.shard_index, o.shard_count = shard_index, shard_count
    o.pdl = 1 if pdl else 0
    o.run_ahead = run_ahead
    o.pair_mode = 1 if pair_mode else 0
    o.full_step = 1 if full_step else 0
    o.intermediate_size = intermediate_size
    # prefill offloads (prefill GPU -> host pool, D2H; reference cluster_sim.hpp:285-299) belong to the
    # prefill instance's link: by default they are executed when a separate prefill/prefetch GPU exists,
    # and stay virtual when the decode GPU is alone (its PCIe link would carry the prefill instance's
    # traffic too; prefill_offload=True measures exactly that)
    if prefill_offload is None:
        prefill_offload = execute_transfers and o.prefetch_device != o.decode_device and not content_check
    o.execute_prefill_offload = 1 if (execute_transfers and prefill_offload) else 0
    o.probe_bubble = 1 if probe_bubble else 0
    bubbles = None
    if probe_bubble:
        cap = max(1, exec_end - timed_begin) if exec_end >= 0 else 1 << 20
        bubbles = np.zeros(cap, np.float64)
        o.bubble_out = bubbles.ctypes.data
        o.bubble_out_cap = cap
    o.content_check = 1 if content_check else 0
    o.capture_path = capture_path.encode() if capture_path else None
    o.capture_every = capture_every
    o.wall_clock = 1 if wall_clock else 0
    st = _lib.EngineStats()
    h = _lib.lib()

    def stats():
        d = st.as_dict()
        if bubbles is not None:
            d["bubble_per_iteration_ms"] = bubbles[:d["bubble_iterations"]].tolist()
        return d
    if out_dir is None and not return_log:
        _lib.check(h.asv_engine_run(text.encode(), policy.encode() if policy else None, C.byref(o), C.byref(st)))
        return stats()
    buf, n = C.c_void_p(), C.c_int64(0)
    _lib.check(h.asv_engine_run_ex(text.encode(), policy.encode() if policy else None, C.byref(o), C.byref(st),
                                   out_dir.encode() if out_dir else None,
                                   C.byref(buf) if return_log else None, C.byref(n) if return_log else None))
    if not return_log:
        return stats()
    try:
        return stats(), C.string_at(buf.value, n.value).decode()
    finally:
        h.asv_free(buf)


def read_capture(path: str):
    """Records of a capture file (include/asv.h asv_engine_opts.capture_path): dicts
    {seq, ids, lens, head, out}; lens = each request's seq_len decoded from the uploaded plan; out
    float32 [L][b][n_q][128] (head == -1), [L][b][128] (query head `head`) or None (head == -2: no
    content mode, page-table lengths only)."""
    recs = []
    with open(path, "rb") as f:
        data = f.read()
    off = 0
    while off < len(data):
        seq = int(np.frombuffer(data, np.int64, 1, off)[0])
        b, L, n_q, head = (int(x) for x in np.frombuffer(data, np.int32, 4, off + 8))
        off += 24
        ids = np.frombuffer(data, np.int64, b, off).copy()
        off += 8 * b
        lens = np.frombuffer(data, np.int32, b, off).copy()
        off += 4 * b
        if head == -2:
            recs.append({"seq": seq, "ids": ids, "lens": lens, "head": head, "out": None})
            continue
        n = L * b * (n_q if head < 0 else 1) * 128
        raw = np.frombuffer(data, np.uint16, n, off)
        off += 2 * n
        out = (raw.astype(np.uint32) << 16).view(np.float32)
        out = out.reshape((L, b, n_q, 128) if head < 0 else (L, b, 128))
        recs.append({"seq": seq, "ids": ids, "lens": lens, "head": head, "out": out})
    return recs
