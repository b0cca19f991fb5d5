"""GPU: one full decoder layer composed from the C-ABI pieces — RMSNorm, QKV GEMM
with RoPE (tcgen05), paged decode attention with fused KV append, O GEMM +
residual, RMSNorm, gate/up GEMM with SiLU, down GEMM + residual — against a
reference built from torch fp32 linear algebra and the fp32 CPU attention
oracle (oracle/attn_oracle.c), with bf16 rounding at the same points.

The attention attends over the request's s = prefix_len tokens (PAPER Eq. 2 as
the reference prices it, cost_model.hpp:52-56) and appends the step's K/V at
position s for the next step (cluster_sim.hpp:443-447).
Tolerance: |gpu - ref| <= 3e-2 + 3e-2 |ref|, rel-L2 <= 1e-2 on the layer output.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import _util as U  # noqa: E402

pytestmark = pytest.mark.gpu


def _rand(shape, seed, scale=1.0, offset=0.0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return ((torch.rand(shape, generator=g) * 2 - 1) * scale + offset).to(torch.bfloat16).cuda()


def test_decoder_layer_composition_matches_reference():
    from paper_2605_23389_b200 import PagedDecodeAttention
    from paper_2605_23389_b200 import linear as L
    n_q = n_kv = 32
    d, inter = 4096, 11008
    seq = [37, 100, 16]
    b = len(seq)
    rows = 16
    att = PagedDecodeAttention(n_q, n_kv, 1, device=0)
    pages = sum((s + 16) // 16 for s in seq) + 3
    pool = U.random_bf16(3, pages * att.page_bytes // 2).view(np.uint8).copy()
    indptr, indices = U.make_batch(seq, pages, 4, append=True)
    pool_d = torch.from_numpy(pool).cuda()

    h0 = _rand((b, d), 10)
    g1, g2 = _rand((d,), 11, 0.1, 1.0), _rand((d,), 12, 0.1, 1.0)
    wqkv = _rand((3 * d, d), 13, 1 / math.sqrt(d))
    wo = _rand((d, d), 14, 1 / math.sqrt(d))
    wgu = _rand((2 * inter, d), 15, 1 / math.sqrt(d))
    wd = _rand((d, inter), 16, 1 / math.sqrt(inter))
    pos = torch.tensor(seq, dtype=torch.int32, device="cuda")

    # ---- GPU: the decode layer as the engine runs it
    h = h0.clone()
    x = torch.zeros(rows, d, dtype=torch.bfloat16, device="cuda")
    act = torch.zeros(rows, inter, dtype=torch.bfloat16, device="cuda")
    q = torch.empty(b, n_q, 128, dtype=torch.bfloat16, device="cuda")
    kn = torch.empty(b, n_kv, 128, dtype=torch.bfloat16, device="cuda")
    vn = torch.empty(b, n_kv, 128, dtype=torch.bfloat16, device="cuda")
    out = torch.zeros(rows, n_q, 128, dtype=torch.bfloat16, device="cuda")
    plan = att.plan(seq, indptr, indices)
    L.rmsnorm(h, g1, x, b, 1e-5)
    L.linear(x, wqkv, b, None, L.QKV_ROPE, positions=pos, q=q, k_out=kn, v_out=vn, n_q_heads=n_q, n_kv_heads=n_kv)
    att.run(q, pool_d, 0, plan, out, k_new=kn, v_new=vn)
    L.linear(out.view(rows, d), wo, b, h, L.RESIDUAL)
    L.rmsnorm(h, g2, x, b, 1e-5)
    L.linear(x, wgu, b, act, L.SILU_MUL)
    L.linear(act, wd, b, h, L.RESIDUAL)
    torch.cuda.synchronize()

    # ---- reference: torch fp32 + the CPU attention oracle, bf16 at the same points
    def rms(t, g):
        t = t.float()
        return (t * torch.rsqrt(t.pow(2).mean(-1, keepdim=True) + 1e-5) * g.float()).bfloat16()

    y = (rms(h0, g1).float() @ wqkv.float().T).view(b, 3 * n_q, 128)
    inv = 10000.0 ** (-torch.arange(0, 64, device="cuda", dtype=torch.float64) * 2 / 128)
    ang = pos.double()[:, None] * inv[None, :]
    cos, sin = torch.cos(ang).float()[:, None, :], torch.sin(ang).float()[:, None, :]

    def rope(t):
        a, c = t[..., :64], t[..., 64:]
        return torch.cat([a * cos - c * sin, c * cos + a * sin], dim=-1)

    q_r = rope(y[:, :n_q]).bfloat16()
    k_r = rope(y[:, n_q:2 * n_q]).bfloat16()
    v_r = y[:, 2 * n_q:].bfloat16()
    assert float((q.float() - q_r.float()).abs().max()) < 3e-2
    o_r, _ = U.Oracle().attention(n_q, n_kv, 1, 0, q_r.cpu().view(torch.int16).numpy().view(np.uint16), pool, seq,
                                  indptr, indices, att.sm_scale)
    o_r = torch.from_numpy(o_r).cuda().bfloat16().float().view(b, d)
    h1 = (h0.float() + o_r @ wo.float().T).bfloat16()
    gu = (rms(h1, g2).float() @ wgu.float().T).view(b, -1, 2, 64)
    a_r = (torch.nn.functional.silu(gu[:, :, 0].reshape(b, -1)) * gu[:, :, 1].reshape(b, -1)).bfloat16()
    h2 = h1.float() + a_r.float() @ wd.float().T

    err = (h.float() - h2).abs()
    rl2 = float((h.float() - h2).norm() / h2.norm())
    print(f"decoder layer: max_abs={float(err.max()):.3e} rel_l2={rl2:.3e}")
    assert bool((err <= 3e-2 + 3e-2 * h2.abs()).all()) and rl2 <= 1e-2

    # the step's K/V landed at position s of each request's pages (read back from the pool)
    pool_after = pool_d.cpu().numpy()
    blocks = U.block_view(pool_after, n_kv, 1)
    for r, s in enumerate(seq):
        page = indices[indptr[r] + s // 16]
        for kv, src in ((0, kn), (1, vn)):
            row = U.unswizzle_block(blocks[0, page, kv, 5])[s % 16]
            assert np.array_equal(row, src[r, 5].cpu().view(torch.int16).numpy().view(np.uint16))
