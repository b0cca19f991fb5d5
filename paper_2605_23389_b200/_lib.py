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
LIB_PATH = os.path.join(_HERE, "libasv.so")


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
    ]


# (name, restype, argtypes) for every symbol include/asv.h declares
SIGNATURES = [
    ("asv_last_error", C.c_char_p, []),
    ("asv_abi_version", C.c_int, []),
    ("asv_free", None, [C.c_void_p]),
    ("asv_page_bytes", C.c_int64, [C.POINTER(AttnShape)]),
    ("asv_page_offset", C.c_int64,
     [C.POINTER(AttnShape), C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    ("asv_attn_num_workers", C.c_int, [C.POINTER(AttnShape), C.c_int, C.POINTER(C.c_int32)]),
    ("asv_attn_plan_build", C.c_int,
     [C.POINTER(AttnShape), C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
      C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32), C.c_int64, C.POINTER(AttnPlan)]),
    ("asv_attn_workspace_bytes", C.c_size_t, [C.POINTER(AttnShape), C.c_int32, C.c_int32]),
    ("asv_attn_workspace_init", C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p]),
    ("asv_decode_attention", C.c_int, [C.POINTER(AttnShape), C.POINTER(AttnArgs), C.c_void_p]),
    ("asv_run_config_jsonl", C.c_int,
     [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
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
