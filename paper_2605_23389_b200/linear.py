"""Host-side face of the decode-step linear layers (include/asv.h asv_linear /
asv_rmsnorm) — the GEMM half of a decode iteration that the reference prices as
the MLP term of iteration_latency (reference cost_model.hpp:60-63, 130-131).

torch is plumbing here (device memory, streams); the math runs in libasv.so
(tcgen05 + TMA kernels, decode_gemm.cu).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib

STORE, RESIDUAL, SILU_MUL, QKV_ROPE = _lib.EPI_STORE, _lib.EPI_RESIDUAL, _lib.EPI_SILU_MUL, _lib.EPI_QKV_ROPE


def _args(x, w, batch, y=None, epilogue=STORE, positions=None, rope_theta=10000.0, q=None, k_out=None, v_out=None,
          n_q_heads=0, n_kv_heads=0, pdl=False, ss_out=None, ss_in=None, ss_eps=1e-5, next_w=None,
          next_epilogue=STORE) -> _lib.LinearArgs:
    if x.dtype != torch.bfloat16 or w.dtype != torch.bfloat16:
        raise TypeError("x and w must be bfloat16")
    n_out, k = w.shape
    a = _lib.LinearArgs()
    a.w, a.n_out, a.k = w.data_ptr(), n_out, k
    a.x, a.x_rows, a.batch = x.data_ptr(), x.shape[0], batch
    a.y = y.data_ptr() if y is not None else None
    a.y_ld = y.shape[-1] if y is not None else 0
    a.epilogue = epilogue
    a.positions = positions.data_ptr() if positions is not None else None
    a.rope_theta = rope_theta
    a.q = q.data_ptr() if q is not None else None
    a.k_out = k_out.data_ptr() if k_out is not None else None
    a.v_out = v_out.data_ptr() if v_out is not None else None
    a.n_q_heads, a.n_kv_heads = n_q_heads, n_kv_heads
    a.pdl = 1 if pdl else 0
    if ss_out is not None:
        a.ss_out, a.ss_ld = ss_out.data_ptr(), ss_out.shape[-1]
    if ss_in is not None:
        a.ss_in, a.ss_parts, a.ss_ld, a.ss_dim, a.ss_eps = ss_in.data_ptr(), ss_in.shape[0], ss_in.shape[-1], k, ss_eps
    if next_w is not None:  # the next linear's weights: L2 prefetch of its first ring stages
        a.next_w, a.next_n_out, a.next_k = next_w.data_ptr(), next_w.shape[0], next_w.shape[1]
        a.next_epilogue = next_epilogue
    return a


def linear_trace(enable: bool | None = None):
    """Measurement only (asv_linear_trace): arm (True) / free (False) the per-CTA timeline of the next
    64 asv_linear launches, or (None) return the armed launches' stamps as uint64 [launches][1024][8]."""
    import numpy as np
    h = _lib.lib()
    if enable is not None:
        _lib.check(h.asv_linear_trace(1 if enable else 0, None, 0, None))
        return None
    cap = 64 * 1024 * 8
    buf = np.zeros(cap, np.uint64)
    n = C.c_int64(0)
    _lib.check(h.asv_linear_trace(0, buf.ctypes.data_as(C.POINTER(C.c_uint64)), cap, C.byref(n)))
    return buf[:n.value].reshape(-1, 1024, 8)


class ChainWorkspace:
    """Cross-CTA counters and partials of asv_linear_chain on one device (include/asv.h)."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        _lib.check(_lib.lib().asv_linear_chain_ws_create(device, C.byref(self.h)))

    def trace(self, enable: bool | None = None):
        """Measurement only: turn the per-CTA phase timeline on / off, or (enable=None) return the last
        launch's stamps as a uint64 array [grid][4 phases][6] (decode_chain.cu kTraceSlots)."""
        import numpy as np
        h = _lib.lib()
        if enable is not None:
            _lib.check(h.asv_linear_chain_ws_trace(self.h, 1 if enable else 0, None, 0, None))
            return None
        cap = 2 * 148 * 4 * 6 * 4
        buf = np.zeros(cap, np.uint64)
        n = C.c_int64(0)
        _lib.check(h.asv_linear_chain_ws_trace(self.h, 1, buf.ctypes.data_as(C.POINTER(C.c_uint64)), cap, C.byref(n)))
        return buf[:n.value].reshape(-1, 4, 6)

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            _lib.lib().asv_linear_chain_ws_destroy(self.h)
            self.h = None


def linear_chain(phases: list[dict], ws: ChainWorkspace, stream=None) -> None:
    """One persistent launch of up to 4 dependent linear layers; each dict holds linear()'s keyword
    arguments (x, w, batch, y, epilogue, ...)."""
    arr = (_lib.LinearArgs * len(phases))(*[_args(**ph) for ph in phases])
    dev = phases[0]["x"].device
    st = (stream or torch.cuda.current_stream(dev)).cuda_stream
    _lib.check(_lib.lib().asv_linear_chain(arr, len(phases), ws.h, C.c_void_p(st)))


def linear(x: torch.Tensor, w: torch.Tensor, batch: int, y: torch.Tensor | None = None,
           epilogue: int = STORE, positions: torch.Tensor | None = None, rope_theta: float = 10000.0,
           q: torch.Tensor | None = None, k_out: torch.Tensor | None = None, v_out: torch.Tensor | None = None,
           n_q_heads: int = 0, n_kv_heads: int = 0, pdl: bool = False, stream=None,
           ss_out: torch.Tensor | None = None, ss_in: torch.Tensor | None = None, ss_eps: float = 1e-5,
           next_w: torch.Tensor | None = None, next_epilogue: int = STORE) -> torch.Tensor | None:
    """y[:batch] = epilogue(x[:batch] @ w.T) on tcgen05 (x has >= batch rounded up to 16 rows).

    Fused RMSNorm: ss_out ([2 * n_out/128][ld] fp32, RESIDUAL only) receives the per-tile sums of
    squares of the updated y rows; a following call with ss_in = that tensor treats x as the raw
    residual stream and scales each output row by rsqrt(mean(x^2) + ss_eps).  next_w: the weights of
    the next linear on the stream and next_epilogue its epilogue (ASV_LINEAR_NEXT_PF: L2 prefetch of the
    stages after its ring; results unchanged)."""
    a = _args(x, w, batch, y, epilogue, positions, rope_theta, q, k_out, v_out, n_q_heads, n_kv_heads, pdl,
              ss_out, ss_in, ss_eps, next_w, next_epilogue)
    st = (stream or torch.cuda.current_stream(x.device)).cuda_stream
    _lib.check(_lib.lib().asv_linear(C.byref(a), C.c_void_p(st)))
    return y


def rmsnorm(h: torch.Tensor, gamma: torch.Tensor, out: torch.Tensor, batch: int, eps: float = 1e-5,
            pdl: bool = False, stream=None) -> torch.Tensor:
    st = (stream or torch.cuda.current_stream(h.device)).cuda_stream
    _lib.check(_lib.lib().asv_rmsnorm(h.data_ptr(), gamma.data_ptr(), out.data_ptr(), h.shape[-1], batch,
                                      out.shape[0], C.c_float(eps), 1 if pdl else 0, C.c_void_p(st)))
    return out
