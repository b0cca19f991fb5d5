"""Test helpers: deterministic inputs, the oracle loaders (TEST INFRASTRUCTURE).

Inputs follow SURVEY §8(d): splitmix64 (reference prng.hpp:10-55) -> U[-1, 1)
-> round-to-nearest-even bf16.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "libasv_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libprefixsim_ref.so")

GOLDEN = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB


def splitmix64(seed: int, n: int) -> np.ndarray:
    """The n outputs of prefixsim::Rng(seed).next_u64() (prng.hpp:14-19), vectorised."""
    with np.errstate(over="ignore"):
        idx = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(seed) + idx * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(M2)
        return z ^ (z >> np.uint64(31))


def uniform_pm1(seed: int, n: int) -> np.ndarray:
    u = (splitmix64(seed, n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return (2.0 * u - 1.0).astype(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u >> np.uint32(16)) & np.uint32(1)) + np.uint32(0x7FFF)
    return ((u + r) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)


def random_bf16(seed: int, n: int) -> np.ndarray:
    return f32_to_bf16_bits(uniform_pm1(seed, n))


def random_f16(seed: int, n: int) -> np.ndarray:
    """IEEE fp16 bits of the same U[-1, 1) draws (fp16 KV variant)."""
    return uniform_pm1(seed, n).astype(np.float16).view(np.uint16)


def swz_off(t: int, d: int) -> int:
    c = d // 8
    return t * 256 + ((c ^ (t & 7)) << 4) + (d % 8) * 2


def page_bytes(n_kv: int, num_layers: int) -> int:
    return num_layers * 2 * n_kv * 4096


def group_pages(n_kv: int, pool_pages: int) -> int:
    """pages per layer-major group: the largest equal split whose layer pitch is < 2 GiB (include/asv.h)."""
    slice_ = 2 * n_kv * 4096
    gmax = ((1 << 31) - 1) // slice_
    return pool_pages // ((pool_pages + gmax - 1) // gmax)


def usable_pages(n_kv: int, pool_pages_: int) -> int:
    """page ids the kernels accept: whole layer-major groups (asv_pool_usable_pages)."""
    g = group_pages(n_kv, pool_pages_)
    return (pool_pages_ // g) * g


def block_view(pool: np.ndarray, n_kv: int, num_layers: int) -> np.ndarray:
    """uint8 LAYER-MAJOR device pool of ONE page group -> [layers][pages][2][n_kv][4096] byte view."""
    assert group_pages(n_kv, pool_pages(pool, n_kv, num_layers)) == pool_pages(pool, n_kv, num_layers), \
        "multi-group pool: use pool_block_offset"
    return pool.reshape(num_layers, -1, 2, n_kv, 4096)


def pool_block_offset(n_kv: int, num_layers: int, pool_pages_: int, page: int, layer: int, kv: int,
                      head: int) -> int:
    """byte offset of block (page, layer, K|V, head) in a grouped layer-major pool (include/asv.h)."""
    g = group_pages(n_kv, pool_pages_)
    slot = (page // g) * g * num_layers + layer * g + page % g
    return slot * 2 * n_kv * 4096 + (kv * n_kv + head) * 4096


def pool_pages(pool: np.ndarray, n_kv: int, num_layers: int) -> int:
    return pool.size // page_bytes(n_kv, num_layers)


def unswizzle_block(block: np.ndarray) -> np.ndarray:
    """4096-byte (16x128 bf16) swizzled block -> [16][128] uint16 row-major."""
    out = np.empty((16, 128), dtype=np.uint16)
    b16 = block.view(np.uint16)
    for t in range(16):
        for c in range(16):
            pc = c ^ (t & 7)
            out[t, c * 8:(c + 1) * 8] = b16[(t * 256 + pc * 16) // 2:(t * 256 + pc * 16) // 2 + 8]
    return out


def make_batch(seq_lens, pool_pages: int, seed: int, append: bool = True):
    """CSR page table over a random permutation of pool pages."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(pool_pages).astype(np.int32)
    indptr = [0]
    indices = []
    pos = 0
    for s in seq_lens:
        n = (s + (1 if append else 0) + 15) // 16
        indices.extend(perm[pos:pos + n])
        pos += n
        indptr.append(len(indices))
    assert pos <= pool_pages, "pool too small for the batch"
    return np.asarray(indptr, np.int32), np.asarray(indices, np.int32)


class Oracle:
    """fp32 CPU attention oracle (oracle/attn_oracle.c) — checker only."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError("oracle/libasv_oracle.so missing: run __graft_entry__.build()")
        self.h = C.CDLL(ORACLE_SO)
        f = self.h.asv_oracle_decode_attention_dt
        f.restype = C.c_int
        f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int64,
                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_float, C.c_void_p,
                      C.c_void_p, C.c_int, C.c_int]

    def content_attention(self, n_q, n_kv, num_layers, ids, lens, sm_scale, threads=None, only_kvh=-1):
        """Expected outputs of a content-mode engine iteration (rows (ids[r], lens[r])), fp32
        [L][b][n_q][128]; with only_kvh >= 0 just that kv head's query heads are filled."""
        f = self.h.asv_oracle_content_attention
        f.restype = C.c_int
        f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_float, C.c_void_p,
                      C.c_int, C.c_int]
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        lens = np.ascontiguousarray(lens, dtype=np.int32)
        out = np.zeros((num_layers, len(ids), n_q, 128), np.float32)
        rc = f(n_q, n_kv, num_layers, ids.ctypes.data, lens.ctypes.data, len(ids), float(sm_scale), out.ctypes.data,
               threads or os.cpu_count() or 1, int(only_kvh))
        assert rc == 0
        return out

    def content_row(self, req, pos, layer, kind, head):
        """bf16 bits of one content row (kind 0 K, 1 V, 2 Q)"""
        f = self.h.asv_oracle_content_row
        f.restype = None
        f.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p]
        out = np.zeros(128, np.uint16)
        f(req, pos, layer, kind, head, out.ctypes.data)
        return out

    def attention(self, n_q, n_kv, num_layers, layer, q_bits, pool, seq_lens, indptr, indices,
                  sm_scale, threads=None, f16=False):
        """q_bits / pool hold bf16 bits (fp16 bits with f16=True)."""
        b = len(seq_lens)
        q_bits = np.ascontiguousarray(q_bits, dtype=np.uint16)
        pool = np.ascontiguousarray(pool, dtype=np.uint8)
        seq = np.ascontiguousarray(seq_lens, dtype=np.int32)
        indptr = np.ascontiguousarray(indptr, dtype=np.int32)
        indices = np.ascontiguousarray(indices, dtype=np.int32)
        out = np.zeros((b, n_q, 128), dtype=np.float32)
        lse = np.zeros((b, n_q), dtype=np.float32)
        rc = self.h.asv_oracle_decode_attention_dt(
            n_q, n_kv, num_layers, layer, q_bits.ctypes.data, pool.ctypes.data,
            pool_pages(pool, n_kv, num_layers), seq.ctypes.data, indptr.ctypes.data, indices.ctypes.data,
            b, float(sm_scale), out.ctypes.data, lse.ctypes.data, threads or os.cpu_count() or 1, 1 if f16 else 0)
        assert rc == 0
        return out, lse


def numpy_attention(n_q, n_kv, num_layers, layer, q_bits, pool, seq_lens, indptr, indices, sm_scale, f16=False):
    """Independent pure-numpy restatement of PAPER Eq. 2 over the paged layout (small cases)."""
    blocks = block_view(pool, n_kv, num_layers)
    g = n_q // n_kv
    widen = (lambda x: np.asarray(x, np.uint16).view(np.float16).astype(np.float32)) if f16 else bf16_bits_to_f32
    q = widen(np.asarray(q_bits, np.uint16)).astype(np.float64)
    b = len(seq_lens)
    out = np.zeros((b, n_q, 128))
    lse = np.zeros((b, n_q))
    for r in range(b):
        s = int(seq_lens[r])
        pages = indices[indptr[r]:indptr[r + 1]]
        for kvh in range(n_kv):
            K = np.concatenate([unswizzle_block(blocks[layer, p, 0, kvh]) for p in pages[:(s + 15) // 16]])[:s]
            V = np.concatenate([unswizzle_block(blocks[layer, p, 1, kvh]) for p in pages[:(s + 15) // 16]])[:s]
            K = widen(K).astype(np.float64)
            V = widen(V).astype(np.float64)
            for h in range(kvh * g, (kvh + 1) * g):
                sc = K @ q[r, h] * sm_scale
                m = sc.max()
                p = np.exp(sc - m)
                out[r, h] = p @ V / p.sum()
                lse[r, h] = m + np.log(p.sum())
    return out, lse


class RefEngine:
    """The UNMODIFIED reference decision path (oracle/_ref, built from /root/reference) — checker only."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise RuntimeError("oracle/_ref/libprefixsim_ref.so missing (reference not built)")
        self.h = C.CDLL(REF_SO)
        for fn in ("ref_run_config_jsonl", "ref_run_config_timed"):
            f = getattr(self.h, fn)
            f.restype = C.c_int
            f.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_longlong),
                          C.POINTER(C.c_double), C.POINTER(C.c_longlong)]
        for fn in ("ref_dfs_batch", "ref_dfs_flat_oracle"):
            f = getattr(self.h, fn)
            f.restype = C.c_int
            f.argtypes = [C.POINTER(C.c_longlong), C.c_longlong, C.c_longlong, C.c_longlong,
                          C.POINTER(C.c_longlong), C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]
        self.h.ref_free.argtypes = [C.c_void_p]
        self.h.ref_last_error.restype = C.c_char_p

    def run_config_jsonl(self, config, policy=None, _fn="ref_run_config_jsonl"):
        """(log, seconds of run_experiment, iterations)"""
        import json as _json
        text = config if isinstance(config, str) else _json.dumps(config)
        out = C.c_void_p()
        n = C.c_longlong(0)
        secs = C.c_double(0)
        its = C.c_longlong(0)
        rc = getattr(self.h, _fn)(text.encode(), policy.encode() if policy else None,
                                  C.byref(out), C.byref(n), C.byref(secs), C.byref(its))
        if rc != 0:
            raise RuntimeError(self.h.ref_last_error().decode())
        try:
            return C.string_at(out.value, n.value).decode(), secs.value, its.value
        finally:
            self.h.ref_free(out)

    def run_config_timed(self, config, policy=None):
        """(log, seconds of the decision engine alone — Simulation::run, no calibration/ingest, iterations)"""
        return self.run_config_jsonl(config, policy, _fn="ref_run_config_timed")

    def dfs(self, residents, b_max, k_min, flat_oracle=False):
        arr = np.ascontiguousarray(np.asarray(residents, dtype=np.int64).reshape(-1, 3))
        n = arr.shape[0]
        ids = np.zeros(max(n, 1), dtype=np.int64)
        cnt = C.c_longlong(0)
        tot = C.c_longlong(0)
        p = lambda a: a.ctypes.data_as(C.POINTER(C.c_longlong))  # noqa: E731
        f = self.h.ref_dfs_flat_oracle if flat_oracle else self.h.ref_dfs_batch
        assert f(p(arr), n, int(b_max), int(k_min), p(ids), C.byref(cnt), C.byref(tot)) == 0
        return ids[:cnt.value].tolist(), int(tot.value)
