"""Host-side mirror of the decode-attention operator (Python face of include/asv.h).

The reference prices this operator — ``iteration_latency(prefix_lengths, model)``
(reference cost_model.hpp:112-135) returns modeled milliseconds for a batch given
its prefix lengths in running order.  Here the same call shape drives the real
sm_100a kernel: ``plan(seq_lens, ...)`` once per iteration, ``run(layer)`` per
layer.  Argument meaning and errors follow the reference: an empty batch raises
``ValueError("empty batch")`` and a prefix length < 1 raises
``ValueError("prefix lengths must be >= 1")`` (cost_model.hpp:114,122 throw
std::invalid_argument with those messages).

torch is used only for device memory and streams (plumbing); every byte of
compute goes through libasv.so.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _lib

HEAD_DIM = 128
PAGE_SIZE = 16


def _i32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _stream_ptr(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


class Plan:
    """One iteration's split-KV work plan (device copy + host descriptor)."""

    def __init__(self, desc: _lib.AttnPlan, host: torch.Tensor, dev: torch.Tensor):
        self.desc = desc
        self.host = host
        self.dev = dev

    @property
    def batch(self) -> int:
        return self.desc.batch

    @property
    def total_splits(self) -> int:
        return self.desc.total_splits


class PagedDecodeAttention:
    """Paged split-KV decode attention over the ASV page layout (include/asv.h).

    num_layers is the number of layers stored per page; ``run`` attends over one
    layer slice.  The group size num_q_heads / num_kv_heads selects the CUDA-core
    FHFMA path (1) or the mma.sync tensor-core path (2, 4, 5, 8).
    """

    def __init__(self, num_q_heads: int, num_kv_heads: int, num_layers: int,
                 device: int | torch.device = 0, sm_scale: float | None = None,
                 dtype: torch.dtype = torch.bfloat16):
        self.lib = _lib.lib()
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.shape = _lib.AttnShape(num_q_heads, num_kv_heads, HEAD_DIM, PAGE_SIZE, num_layers)
        self.num_q_heads = num_q_heads
        self.num_kv_heads = num_kv_heads
        self.num_layers = num_layers
        if dtype not in (torch.bfloat16, torch.float16):
            raise TypeError("KV dtype must be bfloat16 or float16")
        self.dtype = dtype  # element type of the KV pool, q, k_new / v_new and out
        self.sm_scale = float(sm_scale) if sm_scale is not None else 1.0 / math.sqrt(HEAD_DIM)
        w = C.c_int32(0)
        _lib.check(self.lib.asv_attn_num_workers(C.byref(self.shape), self.device.index or 0, C.byref(w)))
        self.num_workers = int(w.value)
        self.page_bytes = int(self.lib.asv_page_bytes(C.byref(self.shape)))
        self._ws = None
        self._ws_splits = 0
        self._launches = 0
        self.pdl = True

    # ------------------------------------------------------------------ plan
    def plan(self, seq_lens, page_indptr, page_indices, num_workers: int | None = None,
             stream=None) -> Plan:
        seq = np.ascontiguousarray(np.asarray(seq_lens, dtype=np.int32))
        indptr = np.ascontiguousarray(np.asarray(page_indptr, dtype=np.int32))
        indices = np.ascontiguousarray(np.asarray(page_indices, dtype=np.int32))
        b = int(seq.shape[0])
        if b == 0:
            raise ValueError("empty batch")
        nw = int(num_workers) if num_workers is not None else self.num_workers
        npages = int(((seq + 15) // 16).sum())
        cap = 40 * (npages // 2 + b + 1) + 2 * b + 8  # every split holds >= 2 pages or a whole request
        host = torch.empty(cap, dtype=torch.int32, pin_memory=True)
        desc = _lib.AttnPlan()
        hp = C.cast(C.c_void_p(host.data_ptr()), C.POINTER(C.c_int32))
        _lib.check(self.lib.asv_attn_plan_build(C.byref(self.shape), b, _i32p(seq), _i32p(indptr),
                                                 _i32p(indices), nw, hp, cap, C.byref(desc)))
        n = desc.total_int32
        dev = torch.empty(n, dtype=torch.int32, device=self.device)
        with torch.cuda.device(self.device):
            s = stream if stream is not None else torch.cuda.current_stream()
            with torch.cuda.stream(s):
                dev.copy_(host[:n], non_blocking=True)
        self._ensure_workspace(desc.total_splits, stream)
        return Plan(desc, host, dev)

    def _ensure_workspace(self, splits: int, stream=None):
        if self._ws is not None and splits <= self._ws_splits:
            return
        cap = max(splits, 2 * self._ws_splits, 1024)
        nbytes = int(self.lib.asv_attn_workspace_bytes(C.byref(self.shape), 0, cap))
        self._ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self._ws_splits = cap
        with torch.cuda.device(self.device):
            _lib.check(self.lib.asv_attn_workspace_init(C.c_void_p(self._ws.data_ptr()), nbytes,
                                                         C.c_void_p(_stream_ptr(stream))))

    # ------------------------------------------------------------------- run
    def run(self, q: torch.Tensor, kv_pool: torch.Tensor, layer: int, plan: Plan,
            out: torch.Tensor, lse: torch.Tensor | None = None, k_new: torch.Tensor | None = None,
            v_new: torch.Tensor | None = None, stream=None, defer_merge: bool = False,
            prev_out: torch.Tensor | None = None, prev_lse: torch.Tensor | None = None,
            warp_ts: torch.Tensor | None = None) -> torch.Tensor:
        """out[b][n_h][128] (self.dtype) = softmax(q K^T * sm_scale) V for every request of the plan.

        defer_merge / prev_out (include/asv.h): consecutive calls with the same plan may leave the split
        merge of one call to the next — defer_merge=True skips this call's merge kernel (its split
        rows of `out` are written by the next call, which must pass prev_out=out)."""
        b = plan.batch
        if q.dtype != self.dtype or out.dtype != self.dtype:
            raise TypeError(f"q and out must be {self.dtype}")
        if k_new is not None and (k_new.dtype != self.dtype or v_new is None or v_new.dtype != self.dtype):
            raise TypeError(f"k_new and v_new must be {self.dtype}")
        if q.shape[0] < b or out.shape[0] < b:
            raise ValueError("q/out batch smaller than the plan")
        args = _lib.AttnArgs()
        args.q = q.data_ptr()
        args.kv_pool = kv_pool.data_ptr()
        args.pool_pages = kv_pool.numel() * kv_pool.element_size() // self.page_bytes
        args.layer = int(layer)
        args.plan_dev = plan.dev.data_ptr()
        args.plan = C.pointer(plan.desc)
        args.k_new = k_new.data_ptr() if k_new is not None else None
        args.v_new = v_new.data_ptr() if v_new is not None else None
        args.out = out.data_ptr()
        args.lse = lse.data_ptr() if lse is not None else None
        args.workspace = self._ws.data_ptr()
        args.workspace_bytes = self._ws.numel()
        args.sm_scale = self.sm_scale
        args.launch_index = self._launches & 0xFFFFFFFF
        args.pdl = 1 if self.pdl else 0
        args.kv_dtype = 1 if self.dtype == torch.float16 else 0
        args.defer_merge = 1 if defer_merge else 0
        args.prev_out = prev_out.data_ptr() if prev_out is not None else None
        args.prev_lse = prev_lse.data_ptr() if prev_lse is not None else None
        if warp_ts is not None:  # [num_workers][2] uint64 (int64 tensor): %globaltimer start / end per warp
            args.warp_timestamps = warp_ts.data_ptr()
        self._launches += 1
        with torch.cuda.device(self.device):
            _lib.check(self.lib.asv_decode_attention(C.byref(self.shape), C.byref(args),
                                                      C.c_void_p(_stream_ptr(stream))))
        return out

    def l2_warm(self, q: torch.Tensor, kv_pool: torch.Tensor, layer: int, plan: Plan, out: torch.Tensor,
                items: int, pages: int, stream=None) -> None:
        """Measurement experiment (asv.h l2_warm_items): prefetch into L2 the first `pages` pages of the
        first `items` work items a later run(layer, plan) takes first; no attention is computed."""
        args = _lib.AttnArgs()
        args.q = q.data_ptr()
        args.kv_pool = kv_pool.data_ptr()
        args.pool_pages = kv_pool.numel() * kv_pool.element_size() // self.page_bytes
        args.layer = int(layer)
        args.plan_dev = plan.dev.data_ptr()
        args.plan = C.pointer(plan.desc)
        args.out = out.data_ptr()
        args.workspace = self._ws.data_ptr()
        args.workspace_bytes = self._ws.numel()
        args.sm_scale = self.sm_scale
        args.launch_index = self._launches & 0xFFFFFFFF
        args.kv_dtype = 1 if self.dtype == torch.float16 else 0
        args.l2_warm_items, args.l2_warm_pages = int(items), int(pages)
        with torch.cuda.device(self.device):
            _lib.check(self.lib.asv_decode_attention(C.byref(self.shape), C.byref(args),
                                                      C.c_void_p(_stream_ptr(stream))))
