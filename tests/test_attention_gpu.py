"""Parity of the sm_100a decode-attention kernel (K1+K2+K3) against the fp32 CPU oracle.

Tolerance (bf16 KV, bf16 output; P rounded to bf16 before PV as in FA2/FA3):
    |gpu - oracle| <= ATOL + RTOL * |oracle| elementwise, and rel-L2 <= RL2,
with ATOL = 4e-3, RTOL = 8e-3, RL2 = 5e-3; lse within 2e-3 absolute.
fp16 KV (8 more mantissa bits): ATOL = 1e-3, RTOL = 2e-3, RL2 = 1e-3, lse 5e-4.
The measured max-abs / rel-L2 are printed so runs record the achieved error.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import _util as U  # noqa: E402

ATOL, RTOL, RL2, LSE_ATOL = 4e-3, 8e-3, 5e-3, 2e-3

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def oracle():
    return U.Oracle()


def _run_case(oracle, n_q, n_kv, L, layer, seq_lens, seed=1, num_workers=None, append=True,
              poison_tail=False, const_v=None, repeat=1, f16=False):
    from paper_2605_23389_b200 import PagedDecodeAttention

    dev = torch.device("cuda", 0)
    tdt = torch.float16 if f16 else torch.bfloat16
    rnd = U.random_f16 if f16 else U.random_bf16
    att = PagedDecodeAttention(n_q, n_kv, L, device=0, dtype=tdt)
    pb = att.page_bytes
    need = sum((s + 16) // 16 for s in seq_lens)
    pool_pages = need + 7
    pool = rnd(seed, pool_pages * pb // 2).view(np.uint8).copy()
    indptr, indices = U.make_batch(seq_lens, U.usable_pages(n_kv, pool_pages), seed + 1, append=True)
    blocks = U.block_view(pool, n_kv, L) if (const_v is not None or poison_tail) else None
    if const_v is not None:
        # every element of every V block equal: the swizzle is irrelevant
        cv = (np.array([const_v], np.float16).view(np.uint16) if f16
              else U.f32_to_bf16_bits(np.array([const_v], np.float32)))[0]
        blocks[:, :, 1] = np.full(2048, cv, np.uint16).view(np.uint8)  # [layer][page][V]
    if poison_tail:
        # rows >= seq_len in each last page hold NaN bit patterns; the kernel must ignore them
        nan_row = np.full(128, 0x7FC1, np.uint16)
        for r, s in enumerate(seq_lens):
            last = indices[indptr[r] + (s - 1) // 16]
            for t in range(s % 16 or 16, 16):
                for kv in range(2):
                    for h in range(n_kv):
                        for d in range(128):
                            off = U.swz_off(t, d)
                            blocks[layer, last, kv, h].view(np.uint16)[off // 2] = nan_row[d]
    b = len(seq_lens)
    q_bits = rnd(seed + 2, b * n_q * 128).reshape(b, n_q, 128)
    kn_bits = rnd(seed + 3, b * n_kv * 128).reshape(b, n_kv, 128)
    vn_bits = rnd(seed + 4, b * n_kv * 128).reshape(b, n_kv, 128)

    ref_out, ref_lse = oracle.attention(n_q, n_kv, L, layer, q_bits, pool, seq_lens, indptr, indices,
                                        att.sm_scale, f16=f16)

    pool_d = torch.from_numpy(pool).to(dev)
    q_d = torch.from_numpy(q_bits.view(np.int16)).to(dev).view(tdt)
    kn_d = torch.from_numpy(kn_bits.view(np.int16)).to(dev).view(tdt) if append else None
    vn_d = torch.from_numpy(vn_bits.view(np.int16)).to(dev).view(tdt) if append else None
    out_d = torch.empty(b, n_q, 128, dtype=tdt, device=dev)
    lse_d = torch.empty(b, n_q, dtype=torch.float32, device=dev)
    plan = att.plan(seq_lens, indptr, indices, num_workers=num_workers)
    for _ in range(repeat):
        att.run(q_d, pool_d, layer, plan, out_d, lse_d, kn_d, vn_d)
    torch.cuda.synchronize()
    got = out_d.float().cpu().numpy()
    got_lse = lse_d.cpu().numpy()

    err = np.abs(got - ref_out)
    rel_l2 = float(np.linalg.norm(got - ref_out) / max(np.linalg.norm(ref_out), 1e-30))
    print(f"{'fp16' if f16 else 'bf16'} n_q={n_q} n_kv={n_kv} b={b} splits={plan.total_splits} max_abs={err.max():.3e} "
          f"rel_l2={rel_l2:.3e} lse_max_abs={np.abs(got_lse - ref_lse).max():.3e}")
    atol, rtol, rl2, lse_atol = (1e-3, 2e-3, 1e-3, 5e-4) if f16 else (ATOL, RTOL, RL2, LSE_ATOL)
    assert np.isfinite(got).all()
    assert (err <= atol + rtol * np.abs(ref_out)).all(), f"max abs err {err.max()}"
    assert rel_l2 <= rl2
    assert np.abs(got_lse - ref_lse).max() <= lse_atol

    if append:
        # fused KV append (K3): token row seq_len of (layer, kv head) holds k_new / v_new
        pool_after = pool_d.cpu().numpy()
        npages = U.pool_pages(pool_after, n_kv, L)

        def blk(page, kv, h):  # works for multi-group pools (>= 2 GiB layer pitch) too
            off = U.pool_block_offset(n_kv, L, npages, int(page), layer, kv, h)
            return pool_after[off:off + 4096]
        for r, s in enumerate(seq_lens):
            page = indices[indptr[r] + s // 16]
            t = s % 16
            for h in range(n_kv):
                krow = U.unswizzle_block(blk(page, 0, h))[t]
                vrow = U.unswizzle_block(blk(page, 1, h))[t]
                assert (krow == kn_bits[r, h]).all()
                assert (vrow == vn_bits[r, h]).all()
    return got, ref_out, plan


def test_mha_config1_shape(oracle):
    """C1: Llama-2-7B attention (32 heads, d=128), batch 16, KV lengths 256-2048."""
    rng = np.random.default_rng(7)
    seq = rng.integers(256, 2049, size=16).tolist()
    _run_case(oracle, 32, 32, 2, 1, seq)


def test_mha_edge_lengths(oracle):
    seq = [1, 2, 15, 16, 17, 31, 32, 33, 255, 256, 257]
    _run_case(oracle, 32, 32, 1, 0, seq, seed=11)


def test_mha_long_request_many_splits(oracle):
    _run_case(oracle, 32, 32, 1, 0, [40000, 3], seed=5)


def test_mha_few_workers_cross_item_pipeline(oracle):
    # 4 warps total: every warp walks many items, exercising the cross-item ring
    rng = np.random.default_rng(3)
    seq = rng.integers(1, 900, size=9).tolist()
    _run_case(oracle, 32, 32, 2, 0, seq, seed=21, num_workers=4)


def test_mha_poisoned_tail_rows(oracle):
    _run_case(oracle, 32, 32, 1, 0, [5, 21, 100], seed=31, poison_tail=True, append=False)


def test_constant_v_known_answer(oracle):
    got, ref, _ = _run_case(oracle, 32, 32, 1, 0, [1, 7, 300], seed=41, const_v=0.375, append=False)
    assert np.all(got == np.float32(0.375))


def test_repeat_launch_rearms_work_counters(oracle):
    _run_case(oracle, 32, 32, 1, 0, [3000, 2500, 10], seed=51, repeat=3, append=False)


@pytest.mark.parametrize("n_q,n_kv", [(32, 8), (40, 8), (64, 8), (16, 8)])
def test_gqa_groups(oracle, n_q, n_kv):
    rng = np.random.default_rng(n_q)
    seq = rng.integers(1, 3000, size=12).tolist() + [16, 17]
    _run_case(oracle, n_q, n_kv, 2, 1, seq, seed=61 + n_q)


def test_gqa_poisoned_tail_and_long(oracle):
    _run_case(oracle, 40, 8, 1, 0, [5, 23, 20000], seed=71, poison_tail=True, append=False)


def test_empty_batch_raises():
    from paper_2605_23389_b200 import PagedDecodeAttention

    att = PagedDecodeAttention(32, 32, 1, device=0)
    with pytest.raises(ValueError, match="empty batch"):
        att.plan([], [0], [])
    with pytest.raises(ValueError, match="prefix lengths must be >= 1"):
        att.plan([0], [0, 1], [0])


def test_many_short_requests(oracle):
    """b = 300 requests of 1-40 tokens: hundreds of tiny single-page items."""
    rng = np.random.default_rng(99)
    seq = rng.integers(1, 41, size=300).tolist()
    _run_case(oracle, 32, 32, 1, 0, seq, seed=81)


@pytest.mark.parametrize("n_q,n_kv", [(32, 32), (40, 8)])
def test_pdl_chain_of_layers_matches_oracle(oracle, n_q, n_kv):
    """Several layers launched back to back (PDL, alternating work-counter parity):
    every layer's output must match the oracle for that layer."""
    from paper_2605_23389_b200 import PagedDecodeAttention

    L = 4
    seq = [700, 33, 2048, 15, 4100]
    dev = torch.device("cuda", 0)
    att = PagedDecodeAttention(n_q, n_kv, L, device=0)
    pages = sum((s + 16) // 16 for s in seq) + 3
    pool = U.random_bf16(91, pages * att.page_bytes // 2).view(np.uint8).copy()
    indptr, indices = U.make_batch(seq, pages, 92)
    pool_d = torch.from_numpy(pool).to(dev)
    plan = att.plan(seq, indptr, indices)
    outs, qs = [], []
    for layer in range(L):
        q = U.random_bf16(100 + layer, len(seq) * n_q * 128).reshape(len(seq), n_q, 128)
        qs.append(q)
        out = torch.empty(len(seq), n_q, 128, dtype=torch.bfloat16, device=dev)
        att.run(torch.from_numpy(q.view(np.int16)).to(dev).view(torch.bfloat16), pool_d, layer, plan, out)
        outs.append(out)
    torch.cuda.synchronize()
    for layer in range(L):
        ref, _ = oracle.attention(n_q, n_kv, L, layer, qs[layer], pool, seq, indptr, indices, att.sm_scale)
        got = outs[layer].float().cpu().numpy()
        assert (np.abs(got - ref) <= ATOL + RTOL * np.abs(ref)).all(), f"layer {layer}"


def test_page_id_outside_the_pool_fails_loudly():
    """A page id >= the pool's usable pages traps the kernel (it would otherwise append KV
    outside the pool); run in a subprocess because a trap poisons the CUDA context."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from paper_2605_23389_b200 import PagedDecodeAttention
att = PagedDecodeAttention(32, 32, 1, device=0)
pool = torch.zeros(8 * att.page_bytes, dtype=torch.uint8, device="cuda")
seq = [40]
indptr = np.array([0, 3], np.int32)
indices = np.array([0, 1, 8], np.int32)   # 8 >= 8 pages in the pool
q = torch.zeros(1, 32, 128, dtype=torch.bfloat16, device="cuda")
out = torch.empty_like(q)
kn = torch.zeros(1, 32, 128, dtype=torch.bfloat16, device="cuda")
att.run(q, pool, 0, att.plan(seq, indptr, indices), out, k_new=kn, v_new=kn)
torch.cuda.synchronize()
print("NO ERROR")
'''
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code, root], capture_output=True, text=True, timeout=300)
    assert r.returncode != 0 and "NO ERROR" not in r.stdout, r.stdout + r.stderr


# ---- BASELINE.json full sizes (C2: 1K-16K, C5: up to 128K tokens) against the oracle ----

def test_config2_lengths_full_size(oracle):
    """C2 shape: 7B MHA, batch 8 of KV lengths drawn from 1K-16K (the headline workload's range)."""
    rng = np.random.default_rng(1024)
    seq = rng.integers(1024, 16385, size=8).tolist()
    _run_case(oracle, 32, 32, 1, 0, seq, seed=111)


@pytest.mark.parametrize("n_q,n_kv", [(32, 32), (40, 8)])
def test_config5_max_context_128k(oracle, n_q, n_kv):
    """C5's longest request: 131072 KV tokens (8192 pages, ~250 splits merged) beside two short ones,
    MHA and 13B GQA-8, against the fp32 oracle; plus the fused append at row 131072."""
    _run_case(oracle, n_q, n_kv, 1, 0, [131072, 17, 1000], seed=121)


# ---- fp16 KV (north star: "bf16/fp16 KV"): same kernel family, fp16 FHFMA / HMMA; same tolerance ----

@pytest.mark.parametrize("n_q,n_kv", [(32, 32), (32, 8), (40, 8), (64, 8)])
def test_fp16_kv_matches_oracle(oracle, n_q, n_kv):
    rng = np.random.default_rng(16 + n_q + n_kv)
    seq = rng.integers(1, 3000, size=10).tolist() + [16, 17, 9000]
    _run_case(oracle, n_q, n_kv, 2, 1, seq, seed=161 + n_q, f16=True)


def test_fp16_poisoned_tail_and_known_answer(oracle):
    _run_case(oracle, 32, 32, 1, 0, [5, 21, 100], seed=171, poison_tail=True, append=False, f16=True)
    _run_case(oracle, 40, 8, 1, 0, [5, 23, 700], seed=172, poison_tail=True, append=False, f16=True)
    got, _, _ = _run_case(oracle, 32, 32, 1, 0, [1, 7, 300], seed=173, const_v=0.375, append=False, f16=True)
    assert np.all(got == np.float32(0.375))


def test_dtype_mismatch_is_rejected():
    from paper_2605_23389_b200 import PagedDecodeAttention
    att = PagedDecodeAttention(32, 32, 1, device=0, dtype=torch.float16)
    plan = att.plan([40], [0, 3], [0, 1, 2])
    q = torch.zeros(1, 32, 128, dtype=torch.bfloat16, device="cuda")
    pool = torch.zeros(4 * att.page_bytes, dtype=torch.uint8, device="cuda")
    with pytest.raises(TypeError, match="float16"):
        att.run(q, pool, 0, plan, torch.empty_like(q))


def test_mha_13b_shape_last_layer(oracle):
    """Llama-2-13B MHA shape (40 heads, 40 layers per page: 12.5 MiB pages), the last layer's slice
    (a small batch: the test pool is built in host memory at 12.5 MiB per page)."""
    _run_case(oracle, 40, 40, 40, 39, [1, 200, 513, 700], seed=131)


@pytest.mark.parametrize("n_q,n_kv,seq", [(32, 32, [700, 33, 2048, 15, 4100]), (40, 8, [9000, 64, 3000, 1]),
                                          (32, 32, [20000, 7])])
def test_deferred_merge_chain_matches_oracle(oracle, n_q, n_kv, seq):
    """include/asv.h defer_merge / prev_out: layer l's split rows are merged by layer l+1's launch (its
    warps take them as first work); the last layer merges its own.  Every layer's output (and lse)
    matches the oracle, as with one merge kernel per layer."""
    from paper_2605_23389_b200 import PagedDecodeAttention

    L = 4
    dev = torch.device("cuda", 0)
    att = PagedDecodeAttention(n_q, n_kv, L, device=0)
    pages = sum((s + 16) // 16 for s in seq) + 3
    pool = U.random_bf16(191, pages * att.page_bytes // 2).view(np.uint8).copy()
    indptr, indices = U.make_batch(seq, U.usable_pages(n_kv, pages), 192)
    pool_d = torch.from_numpy(pool).to(dev)
    plan = att.plan(seq, indptr, indices)
    assert plan.desc.n_merge > 0  # split requests exist: the deferral is exercised
    outs, lses, qs = [], [], []
    for layer in range(L):
        q = U.random_bf16(200 + layer, len(seq) * n_q * 128).reshape(len(seq), n_q, 128)
        qs.append(q)
        out = torch.full((len(seq), n_q, 128), float("nan"), dtype=torch.bfloat16, device=dev)
        lse = torch.full((len(seq), n_q), float("nan"), dtype=torch.float32, device=dev)
        att.run(torch.from_numpy(q.view(np.int16)).to(dev).view(torch.bfloat16), pool_d, layer, plan, out, lse,
                defer_merge=layer + 1 < L, prev_out=outs[-1] if outs else None, prev_lse=lses[-1] if lses else None)
        outs.append(out)
        lses.append(lse)
    torch.cuda.synchronize()
    for layer in range(L):
        ref, ref_lse = oracle.attention(n_q, n_kv, L, layer, qs[layer], pool, seq, indptr, indices, att.sm_scale)
        got = outs[layer].float().cpu().numpy()
        assert np.isfinite(got).all(), f"layer {layer}: rows never written"
        assert (np.abs(got - ref) <= ATOL + RTOL * np.abs(ref)).all(), f"layer {layer}"
        assert np.abs(lses[layer].cpu().numpy() - ref_lse).max() <= LSE_ATOL, f"layer {layer} lse"
