"""CPU: pin the attention oracle (TEST INFRASTRUCTURE) before trusting it.

The reference has no numeric attention, so the oracle is pinned by
known-answer cases and by an independent pure-numpy restatement of PAPER Eq. 2.
"""
import math

import numpy as np
import pytest

import _util as U  # noqa: E402


@pytest.fixture(scope="module")
def oracle():
    return U.Oracle()


def _pool(n_kv, L, pages, seed):
    return U.random_bf16(seed, pages * U.page_bytes(n_kv, L) // 2).view(np.uint8).copy()


def test_splitmix_matches_reference_prng():
    # prefixsim::Rng(1).next_u64() first outputs (prng.hpp:14-19), computed by hand
    def ref(seed, n):
        out, s = [], seed
        for _ in range(n):
            s = (s + 0x9E3779B97F4A7C15) & (2**64 - 1)
            z = s
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
            out.append(z ^ (z >> 31))
        return out
    assert U.splitmix64(1, 5).tolist() == ref(1, 5)
    assert U.splitmix64(97, 3).tolist() == ref(97, 3)


def test_swizzle_roundtrip():
    blk = np.zeros(4096, np.uint8)
    vals = np.arange(16 * 128, dtype=np.uint16).reshape(16, 128)
    for t in range(16):
        for d in range(128):
            o = U.swz_off(t, d)
            blk[o:o + 2] = vals[t, d:d + 1].view(np.uint8)
    assert (U.unswizzle_block(blk) == vals).all()


@pytest.mark.parametrize("n_q,n_kv", [(32, 32), (40, 8)])
def test_oracle_matches_numpy_restatement(oracle, n_q, n_kv):
    L, layer = 2, 1
    seq = [1, 16, 17, 70]
    pages = sum((s + 15) // 16 for s in seq) + 3
    pool = _pool(n_kv, L, pages, 5)
    indptr, indices = U.make_batch(seq, pages, 9, append=False)
    q = U.random_bf16(8, len(seq) * n_q * 128).reshape(len(seq), n_q, 128)
    sc = 1 / math.sqrt(128)
    o1, l1 = oracle.attention(n_q, n_kv, L, layer, q, pool, seq, indptr, indices, sc, threads=4)
    o2, l2 = U.numpy_attention(n_q, n_kv, L, layer, q, pool, seq, indptr, indices, sc)
    assert np.abs(o1 - o2).max() < 2e-6
    assert np.abs(l1 - l2).max() < 2e-5


@pytest.mark.parametrize("n_q,n_kv", [(32, 32), (40, 8)])
def test_oracle_fp16_matches_numpy_restatement(oracle, n_q, n_kv):
    """fp16 KV variant: the oracle's exact binary16 widening (subnormals included) vs numpy's."""
    L, layer = 2, 0
    seq = [3, 16, 40]
    pages = sum((s + 15) // 16 for s in seq) + 2
    pool = U.random_f16(6, pages * U.page_bytes(n_kv, L) // 2)
    pool[::97] = np.array([0x0001, 0x03ff, 0x8200, 0x3c00], np.uint16)[np.arange(pool[::97].size) % 4]  # subnormals, 1.0
    pool = pool.view(np.uint8).copy()
    indptr, indices = U.make_batch(seq, pages, 10, append=False)
    q = U.random_f16(9, len(seq) * n_q * 128).reshape(len(seq), n_q, 128)
    sc = 1 / math.sqrt(128)
    o1, l1 = oracle.attention(n_q, n_kv, L, layer, q, pool, seq, indptr, indices, sc, threads=4, f16=True)
    o2, l2 = U.numpy_attention(n_q, n_kv, L, layer, q, pool, seq, indptr, indices, sc, f16=True)
    assert np.abs(o1 - o2).max() < 2e-6
    assert np.abs(l1 - l2).max() < 2e-5


def test_known_answer_single_token(oracle):
    """s = 1: softmax over one key is 1, so O = V_0 exactly."""
    n_kv, L = 4, 1
    pool = _pool(n_kv, L, 2, 3)
    q = U.random_bf16(4, 4 * 128).reshape(1, 4, 128)
    out, _ = oracle.attention(4, 4, L, 0, q, pool, [1], [0, 1], [1], 0.1)
    blocks = U.block_view(pool, n_kv, L)
    for h in range(4):
        v0 = U.bf16_bits_to_f32(U.unswizzle_block(blocks[0, 1, 1, h])[0])
        assert np.array_equal(out[0, h], v0)


def test_known_answer_dominant_key(oracle):
    """One key aligned with q and scaled up dominates: O ~= that key's V."""
    n_kv, L = 1, 1
    pool = np.zeros(2 * U.page_bytes(n_kv, L), np.uint8)
    blocks = U.block_view(pool, n_kv, L)
    q = np.zeros((1, 1, 128), np.float32)
    q[0, 0, 0] = 8.0
    kb = np.zeros((16, 128), np.float32)
    kb[5, 0] = 8.0
    vb = U.uniform_pm1(3, 16 * 128).reshape(16, 128)
    for t in range(16):
        for d in range(128):
            for kv, src in ((0, kb), (1, vb)):
                o = U.swz_off(t, d)
                blocks[0, 0, kv, 0][o:o + 2] = U.f32_to_bf16_bits(src[t, d:d + 1]).view(np.uint8)  # [layer][page]
    out, _ = oracle.attention(1, 1, L, 0, U.f32_to_bf16_bits(q), pool, [16], [0, 1], [0], 1.0)
    v5 = U.bf16_bits_to_f32(U.f32_to_bf16_bits(vb[5]))
    assert np.abs(out[0, 0] - v5).max() < 1e-6


# ---------------------------------------------------------------- content-check restatement
def _np_content_row(req, pos, layer, kind, head):
    """numpy restatement of the content function documented in include/asv.h / attn_oracle.c."""
    G = np.uint64(0x9E3779B97F4A7C15)
    with np.errstate(over="ignore"):
        def mix(z):
            z = np.uint64(z)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            return z ^ (z >> np.uint64(31))
        key = ((((((req << 21) | pos) << 6 | layer) << 2 | kind) << 8) | head)
        seed = mix(np.uint64(key) + G)
        words = [mix(seed + np.uint64(w + 1) * G) for w in range(16)]
    b = np.array(words, dtype=np.uint64).view(np.int8).astype(np.float32)  # little endian: byte j = >> 8j
    return b * (1 / 8 if kind == 2 else 1 / 128)


def test_content_rows_follow_the_documented_function():
    o = U.Oracle()
    for req, pos, layer, kind, head in [(0, 0, 0, 0, 0), (5, 1234, 3, 1, 17), (1 << 20, 77, 1, 2, 31)]:
        got = U.bf16_bits_to_f32(o.content_row(req, pos, layer, kind, head))
        assert np.array_equal(got, _np_content_row(req, pos, layer, kind, head))


@pytest.mark.parametrize("n_q,n_kv", [(4, 4), (8, 2)])
def test_content_attention_matches_numpy_restatement(n_q, n_kv):
    o = U.Oracle()
    ids, lens, L = [3, 11], [1, 37], 2
    got = o.content_attention(n_q, n_kv, L, ids, lens, 0.08838834764831845)
    g = n_q // n_kv
    for l in range(L):
        for r, (i, s) in enumerate(zip(ids, lens)):
            for h in range(n_q):
                q = _np_content_row(i, s, l, 2, h).astype(np.float64)
                K = np.stack([_np_content_row(i, t, l, 0, h // g) for t in range(s)]).astype(np.float64)
                V = np.stack([_np_content_row(i, t, l, 1, h // g) for t in range(s)]).astype(np.float64)
                sc = K @ q * 0.08838834764831845
                p = np.exp(sc - sc.max())
                np.testing.assert_allclose(got[l, r, h], p @ V / p.sum(), rtol=1e-5, atol=1e-6)
    only = o.content_attention(n_q, n_kv, L, ids, lens, 0.08838834764831845, only_kvh=1)
    np.testing.assert_array_equal(only[:, :, g:2 * g], got[:, :, g:2 * g])
    assert not only[:, :, :g].any()
