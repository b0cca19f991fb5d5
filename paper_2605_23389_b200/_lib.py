"""ctypes binding of libasv.so (the C ABI declared in include/asv.h).

This is the same binding a reference-side maintainer would add:
plain structs and pointers, no torch types crossing the boundary.  Loading is
strict: if the native library is missing the import fails loudly — there is no
CPU or Python fallback anywhere on the product path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# ASV_LIB_PATH: load an alternative build (A/B kernel experiments only)
LIB_PATH = os.environ.get("ASV_LIB_PATH") or os.path.join(_HERE, "libasv.so")


class AttnShape(C.Structure):
    _fields_ = [
        ("num_q_heads", C.c_int32),
        ("num_kv_heads", C.c_int32),
        ("head_dim", C.c_int32),
        ("page_size", C.c_int32),
        ("num_layers", C.c_int32),
    ]


class AttnPlan(C.Structure):
    _fields_ = [
        ("batch", C.c_int32),
        ("total_splits", C.c_int32),
        ("num_items", C.c_int32),
        ("num_pages", C.c_int32),
        ("num_workers", C.c_int32),
        ("off_desc", C.c_int32),
        ("off_split_base", C.c_int32),
        ("off_merge", C.c_int32),
        ("n_merge", C.c_int32),
        ("total_int32", C.c_int32),
        ("max_item_pages", C.c_int32),
        ("append_missing", C.c_int32),
    ]


class AttnArgs(C.Structure):
    _fields_ = [
        ("q", C.c_void_p),
        ("kv_pool", C.c_void_p),
        ("pool_pages", C.c_int64),
        ("layer", C.c_int32),
        ("plan_dev", C.c_void_p),
        ("plan", C.POINTER(AttnPlan)),
        ("k_new", C.c_void_p),
        ("v_new", C.c_void_p),
        ("out", C.c_void_p),
        ("lse", C.c_void_p),
        ("workspace", C.c_void_p),
        ("workspace_bytes", C.c_size_t),
        ("sm_scale", C.c_float),
        ("launch_index", C.c_uint32),
        ("pdl", C.c_int32),
        ("warp_timestamps", C.c_void_p),
        ("kv_dtype", C.c_int32),
        ("defer_merge", C.c_int32),
        ("prev_out", C.c_void_p),
        ("prev_lse", C.c_void_p),
        ("l2_warm_items", C.c_int32),
        ("l2_warm_pages", C.c_int32),
    ]


class LinearArgs(C.Structure):
    _fields_ = [
        ("w", C.c_void_p),
        ("n_out", C.c_int32),
        ("k", C.c_int32),
        ("x", C.c_void_p),
        ("x_rows", C.c_int32),
        ("batch", C.c_int32),
        ("y", C.c_void_p),
        ("y_ld", C.c_int32),
        ("epilogue", C.c_int32),
        ("positions", C.c_void_p),
        ("rope_theta", C.c_float),
        ("q", C.c_void_p),
        ("k_out", C.c_void_p),
        ("v_out", C.c_void_p),
        ("n_q_heads", C.c_int32),
        ("n_kv_heads", C.c_int32),
        ("pdl", C.c_int32),
        ("ss_out", C.c_void_p),
        ("ss_in", C.c_void_p),
        ("ss_parts", C.c_int32),
        ("ss_ld", C.c_int32),
        ("ss_dim", C.c_int32),
        ("ss_eps", C.c_float),
        ("next_w", C.c_void_p),
        ("next_n_out", C.c_int32),
        ("next_k", C.c_int32),
        ("next_epilogue", C.c_int32),
    ]


EPI_STORE, EPI_RESIDUAL, EPI_SILU_MUL, EPI_QKV_ROPE = 0, 1, 2, 3


class EngineOpts(C.Structure):
    _fields_ = [
        ("decode_device", C.c_int32),
        ("prefetch_device", C.c_int32),
        ("num_q_heads", C.c_int32),
        ("num_kv_heads", C.c_int32),
        ("num_layers", C.c_int32),
        ("execute_transfers", C.c_int32),
        ("host_pool_bytes", C.c_int64),
        ("exec_begin", C.c_int64),
        ("exec_end", C.c_int64),
        ("timed_begin", C.c_int64),
        ("shard_index", C.c_int32),
        ("shard_count", C.c_int32),
        ("pdl", C.c_int32),
        ("run_ahead", C.c_int32),
        ("copy_begin", C.c_int64),
        ("pair_mode", C.c_int32),
        ("full_step", C.c_int32),
        ("intermediate_size", C.c_int32),
        ("execute_prefill_offload", C.c_int32),
        ("probe_bubble", C.c_int32),
        ("bubble_out", C.c_void_p),
        ("bubble_out_cap", C.c_int64),
        ("content_check", C.c_int32),
        ("capture_path", C.c_char_p),
        ("capture_every", C.c_int64),
        ("wall_clock", C.c_int32),
    ]


XFER_KINDS = ["prefill_offload", "batch_prefetch", "stray_prefetch", "admit", "evict", "spill", "flush"]


class EngineStats(C.Structure):
    _fields_ = [
        ("iterations_total", C.c_int64),
        ("iterations_timed", C.c_int64),
        ("tokens_timed", C.c_int64),
        ("window_ms", C.c_double),
        ("attn_ms", C.c_double),
        ("attn_bytes", C.c_int64),
        ("attn_launches", C.c_int64),
        ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64),
        ("p2p_bytes", C.c_int64),
        ("h2d_busy_ms", C.c_double),
        ("p2p_busy_ms", C.c_double),
        ("logical_bytes", C.c_int64 * 7),
        ("logical_count", C.c_int64 * 7),
        ("virtual_decode_tok_s", C.c_double),
        ("host_decide_ms", C.c_double),
        ("max_batch", C.c_int64),
        ("pages_decode", C.c_int64),
        ("pages_prefetch", C.c_int64),
        ("bubble_ms_timed", C.c_double),
        ("kernel_launches_timed", C.c_int64),
        ("virtual_window_ms", C.c_double),
        ("h2d_bytes_window", C.c_int64),
        ("d2h_bytes_window", C.c_int64),
        ("p2p_bytes_window", C.c_int64),
        ("measured_idle_frac", C.c_double),
        ("measured_bubble_ms", C.c_double),
        ("pcie_union_ms", C.c_double),
        ("host_wait_ms", C.c_double),
        ("hazard_waits", C.c_int64),
        ("result_d2h_bytes_window", C.c_int64),
        ("weight_bytes", C.c_int64),
        ("offload_bytes", C.c_int64),
        ("offload_bytes_window", C.c_int64),
        ("bubble_iterations", C.c_int64),
        ("bubble_p50_ms", C.c_double),
        ("bubble_p90_ms", C.c_double),
        ("bubble_p99_ms", C.c_double),
        ("bubble_max_ms", C.c_double),
        ("content_inplace_bytes", C.c_int64),
        ("content_iterations_captured", C.c_int64),
    ]

    def as_dict(self):
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            if name in ("logical_bytes", "logical_count"):
                v = {k: int(v[i]) for i, k in enumerate(XFER_KINDS)}
            d[name] = v
        return d


# (name, restype, argtypes) for every symbol include/asv.h declares
SIGNATURES = [
    ("asv_last_error", C.c_char_p, []),
    ("asv_abi_version", C.c_int, []),
    ("asv_struct_size", C.c_int64, [C.c_char_p]),
    ("asv_free", None, [C.c_void_p]),
    ("asv_page_bytes", C.c_int64, [C.POINTER(AttnShape)]),
    ("asv_page_offset", C.c_int64,
     [C.POINTER(AttnShape), C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    ("asv_pool_offset", C.c_int64,
     [C.POINTER(AttnShape), C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    ("asv_pool_group_pages", C.c_int64, [C.POINTER(AttnShape), C.c_int64]),
    ("asv_pool_usable_pages", C.c_int64, [C.POINTER(AttnShape), C.c_int64]),
    ("asv_attn_num_workers", C.c_int, [C.POINTER(AttnShape), C.c_int, C.POINTER(C.c_int32)]),
    ("asv_attn_plan_build", C.c_int,
     [C.POINTER(AttnShape), C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
      C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32), C.c_int64, C.POINTER(AttnPlan)]),
    ("asv_plan_upload", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    ("asv_attn_workspace_bytes", C.c_size_t, [C.POINTER(AttnShape), C.c_int32, C.c_int32]),
    ("asv_attn_workspace_init", C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p]),
    ("asv_decode_attention", C.c_int, [C.POINTER(AttnShape), C.POINTER(AttnArgs), C.c_void_p]),
    ("asv_kv_copy_h2d", C.c_int,
     [C.POINTER(AttnShape), C.c_void_p, C.c_int64, C.POINTER(C.c_int32), C.c_int64, C.POINTER(C.c_void_p),
      C.c_void_p, C.POINTER(C.c_int64)]),
    ("asv_kv_copy_d2h", C.c_int,
     [C.POINTER(AttnShape), C.c_void_p, C.c_int64, C.POINTER(C.c_int32), C.c_int64, C.POINTER(C.c_void_p),
      C.c_void_p, C.POINTER(C.c_int64)]),
    ("asv_kv_copy_d2d", C.c_int,
     [C.POINTER(AttnShape), C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_int32), C.c_void_p, C.c_int64,
      C.c_int32, C.POINTER(C.c_int32), C.c_int64, C.c_void_p, C.POINTER(C.c_int64)]),
    ("asv_linear", C.c_int, [C.POINTER(LinearArgs), C.c_void_p]),
    ("asv_linear_chain_ws_create", C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    ("asv_linear_chain_ws_destroy", None, [C.c_void_p]),
    ("asv_linear_chain", C.c_int, [C.POINTER(LinearArgs), C.c_int32, C.c_void_p, C.c_void_p]),
    ("asv_linear_chain_ws_trace", C.c_int,
     [C.c_void_p, C.c_int32, C.POINTER(C.c_uint64), C.c_int64, C.POINTER(C.c_int64)]),
    ("asv_linear_set_schedule", C.c_int, [C.c_int32, C.c_int32]),
    ("asv_linear_schedule", C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    ("asv_linear_trace", C.c_int, [C.c_int32, C.POINTER(C.c_uint64), C.c_int64, C.POINTER(C.c_int64)]),
    ("asv_rmsnorm", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_float,
                              C.c_int32, C.c_void_p]),
    ("asv_run_config_jsonl", C.c_int,
     [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    ("asv_engine_run", C.c_int,
     [C.c_char_p, C.c_char_p, C.POINTER(EngineOpts), C.POINTER(EngineStats)]),
    ("asv_engine_run_ex", C.c_int,
     [C.c_char_p, C.c_char_p, C.POINTER(EngineOpts), C.POINTER(EngineStats), C.c_char_p, C.POINTER(C.c_void_p),
      C.POINTER(C.c_int64)]),
    ("asv_run_config_jsonl_shard", C.c_int,
     [C.c_char_p, C.c_char_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    ("asv_dfs_batch", C.c_int,
     [C.POINTER(C.c_int64), C.c_int64, C.c_int64, C.c_int64, C.POINTER(C.c_int64),
      C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
]

_lib = None


def lib() -> C.CDLL:
    """Load libasv.so once; raise if it is missing (no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"native library {LIB_PATH} is missing: run __graft_entry__.build() "
                "(make -C paper_2605_23389_b200/csrc); there is no CPU fallback")
        h = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


class AsvError(RuntimeError):
    pass


_ERR_TYPES = {1: ValueError, 2: RuntimeError, 3: AssertionError, 4: AsvError}


def check(rc: int) -> None:
    """Map an ASV_ERR_* code to the Python analogue of the reference's C++ exception."""
    if rc != 0:
        msg = lib().asv_last_error().decode()
        raise _ERR_TYPES.get(rc, AsvError)(msg)
