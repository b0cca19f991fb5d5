"""TEST INFRASTRUCTURE — fp32 CPU restatement of one decode step of one decoder layer.

Used only by bench.py's CPU-baseline leg / `--impl reference` arm (the reference's
CPU path: the reference prices this work, `iteration_latency` cost_model.hpp:112-135,
with the attention term :119-132 and the MLP term :60-63/:130-131; it never
executes it).  The layer is the Llama-2 decoder layer the GPU full step runs
(paper_2605_23389_b200/csrc/executor.cpp layer_front / layer_back):

    x = RMSNorm(h) ; q,k,v = x Wqkv^T (+ rotate-half RoPE at position s)
    o = softmax(q K^T / sqrt(d)) V over the request's s cached tokens (PAPER.md:151-153,
        oracle/attn_oracle.c on all host cores)
    h += o Wo^T ; x = RMSNorm(h) ; h += (silu(x Wg^T) * (x Wu^T)) Wd^T

Weights are random fp32 (timing only: contents do not change the work).  Never
imported by the product package.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(_HERE), "tests"))
import _util as U  # noqa: E402  (oracle loaders)


def rmsnorm(h: np.ndarray, g: np.ndarray, eps: float = 1e-5) -> np.ndarray:
    return h / np.sqrt(np.mean(h * h, axis=-1, keepdims=True) + eps) * g


def rope(x: np.ndarray, pos: np.ndarray, theta: float = 10000.0) -> np.ndarray:
    """rotate-half RoPE over the last dim (128) of [b][heads][128] at per-row positions."""
    d = x.shape[-1]
    inv = theta ** (-np.arange(0, d // 2, dtype=np.float32) * 2.0 / d)
    ang = pos[:, None].astype(np.float32) * inv[None, :]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    x1, x2 = x[..., : d // 2], x[..., d // 2:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


class CpuDecoderLayer:
    """One layer of the decode step on the CPU; `step(lens)` returns its wall time in seconds."""

    def __init__(self, n_q: int, n_kv: int, head_dim: int = 128, threads: int | None = None,
                 full_step: bool = True, intermediate: int | None = None, pool_pages: int = 1024):
        self.n_q, self.n_kv, self.d = n_q, n_kv, head_dim
        self.hidden = n_q * head_dim
        self.inter = intermediate or (11008 if self.hidden == 4096 else 13824 if self.hidden == 5120
                                      else (self.hidden * 8 // 3 + 127) // 128 * 128)
        self.threads = threads or os.cpu_count() or 1
        self.full = full_step
        self.oracle = U.Oracle()
        self.pool_pages = pool_pages
        self.pool = U.random_bf16(5, pool_pages * U.page_bytes(n_kv, 1) // 2).view(np.uint8)
        self.rng = np.random.default_rng(0)
        if full_step:
            r = np.random.default_rng(1)
            H, I = self.hidden, self.inter
            n_qkv = (n_q + 2 * n_kv) * head_dim
            self.w_qkv = r.standard_normal((n_qkv, H), dtype=np.float32) / np.sqrt(H)
            self.w_o = r.standard_normal((H, H), dtype=np.float32) / np.sqrt(H)
            self.w_gu = r.standard_normal((2 * I, H), dtype=np.float32) / np.sqrt(H)
            self.w_d = r.standard_normal((H, I), dtype=np.float32) / np.sqrt(I)
            self.g1 = np.ones(H, np.float32)
            self.g2 = np.ones(H, np.float32)

    def step(self, lens) -> float:
        b = len(lens)
        indptr = np.zeros(b + 1, np.int32)
        indptr[1:] = np.cumsum([(s + 15) // 16 for s in lens])
        indices = self.rng.integers(0, self.pool_pages, int(indptr[-1])).astype(np.int32)
        h = self.rng.standard_normal((b, self.hidden), dtype=np.float32)
        q_bits = U.random_bf16(7, b * self.n_q * self.d)
        t0 = time.perf_counter()
        if self.full:
            x = rmsnorm(h, self.g1)
            qkv = x @ self.w_qkv.T
            pos = np.asarray(lens, np.int64)
            q = rope(qkv[:, : self.n_q * self.d].reshape(b, self.n_q, self.d), pos)
            _k = rope(qkv[:, self.n_q * self.d:(self.n_q + self.n_kv) * self.d].reshape(b, self.n_kv, self.d), pos)
            q_bits = U.f32_to_bf16_bits(q.reshape(-1))
        o, _ = self.oracle.attention(self.n_q, self.n_kv, 1, 0, q_bits, self.pool, lens, indptr, indices,
                                     1.0 / np.sqrt(self.d), self.threads)
        if self.full:
            h = h + o.reshape(b, -1) @ self.w_o.T
            x = rmsnorm(h, self.g2)
            gu = x @ self.w_gu.T
            g, u = gu[:, : self.inter], gu[:, self.inter:]
            act = g / (1.0 + np.exp(-g)) * u
            h = h + act @ self.w_d.T
        return time.perf_counter() - t0
