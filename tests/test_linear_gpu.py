"""GPU: decode-step linear layers on tcgen05 (asv_linear, asv_rmsnorm) against a
plain torch fp32 reference of the same op (floating-point kernel: the CPU oracle
of this repo covers attention; these layers are SURVEY §8(f) rank 1).

Tolerance (bf16 inputs and output, fp32 accumulation in TMEM):
    |gpu - ref| <= 2e-2 + 2e-2 * |ref| elementwise and rel-L2 <= 8e-3,
where ref is computed in fp32 from the same bf16 inputs and the output is
rounded to bf16 once (rel. rounding error 2^-9).
"""
import math

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ATOL, RTOL, RL2 = 2e-2, 2e-2, 8e-3


def _rand(shape, seed, scale=1.0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return ((torch.rand(shape, generator=g) * 2 - 1) * scale).to(torch.bfloat16).cuda()


def _check(got, ref, what):
    got, ref = got.float(), ref.float()
    err = (got - ref).abs()
    rl2 = float((got - ref).norm() / ref.norm().clamp_min(1e-30))
    print(f"{what}: max_abs={float(err.max()):.3e} rel_l2={rl2:.3e}")
    assert torch.isfinite(got).all()
    assert bool((err <= ATOL + RTOL * ref.abs()).all()), f"{what}: max abs err {float(err.max())}"
    assert rl2 <= RL2, f"{what}: rel-L2 {rl2}"


def _x(batch, k, seed):
    rows = (batch + 15) // 16 * 16
    x = torch.zeros(rows, k, dtype=torch.bfloat16, device="cuda")
    x[:batch] = _rand((batch, k), seed)
    return x


@pytest.mark.parametrize("n_out,k,batch", [(128, 64, 1), (256, 512, 5), (4096, 4096, 16), (1024, 11008, 33),
                                           (12288, 4096, 64), (512, 4096, 256), (384, 1024, 100)])
def test_store_matches_torch(n_out, k, batch):
    from paper_2605_23389_b200 import linear as L
    x = _x(batch, k, 1)
    w = _rand((n_out, k), 2, 1 / math.sqrt(k))
    y = torch.full((batch, n_out), float("nan"), dtype=torch.bfloat16, device="cuda")
    L.linear(x, w, batch, y, L.STORE)
    torch.cuda.synchronize()
    ref = x[:batch].float() @ w.float().T
    _check(y, ref, f"store {n_out}x{k} b{batch}")
    # repeated call: split-K tile counters self-reset
    L.linear(x, w, batch, y, L.STORE)
    torch.cuda.synchronize()
    _check(y, ref, "store (second call)")


@pytest.mark.parametrize("batch", [3, 48])
def test_residual_adds_in_place(batch):
    from paper_2605_23389_b200 import linear as L
    n_out, k = 4096, 4096
    x = _x(batch, k, 3)
    w = _rand((n_out, k), 4, 1 / math.sqrt(k))
    h0 = _rand((batch, n_out), 5)
    h = h0.clone()
    L.linear(x, w, batch, h, L.RESIDUAL)
    torch.cuda.synchronize()
    _check(h, h0.float() + x[:batch].float() @ w.float().T, f"residual b{batch}")


def test_silu_mul_interleaved_gate_up():
    from paper_2605_23389_b200 import linear as L
    inter, k, batch = 11008, 4096, 7
    x = _x(batch, k, 6)
    gate = _rand((inter, k), 7, 1 / math.sqrt(k))
    up = _rand((inter, k), 8, 1 / math.sqrt(k))
    # tile t of the fused weight: 64 gate rows then the 64 up rows of outputs 64t..64t+63
    w = torch.stack([gate.view(-1, 64, k), up.view(-1, 64, k)], dim=1).reshape(2 * inter, k).contiguous()
    y = torch.empty(batch, inter, dtype=torch.bfloat16, device="cuda")
    L.linear(x, w, batch, y, L.SILU_MUL)
    torch.cuda.synchronize()
    xf = x[:batch].float()
    g, u = xf @ gate.float().T, xf @ up.float().T
    _check(y, torch.nn.functional.silu(g) * u, "silu_mul")


@pytest.mark.parametrize("n_q,n_kv,batch", [(32, 32, 4), (40, 8, 19)])
def test_qkv_rope(n_q, n_kv, batch):
    from paper_2605_23389_b200 import linear as L
    k = 128 * n_q
    n_out = 128 * (n_q + 2 * n_kv)
    x = _x(batch, k, 9)
    w = _rand((n_out, k), 10, 1 / math.sqrt(k))
    pos = torch.randint(0, 20000, (batch,), dtype=torch.int32, device="cuda")
    q = torch.empty(batch, n_q, 128, dtype=torch.bfloat16, device="cuda")
    kk = torch.empty(batch, n_kv, 128, dtype=torch.bfloat16, device="cuda")
    v = torch.empty(batch, n_kv, 128, dtype=torch.bfloat16, device="cuda")
    L.linear(x, w, batch, None, L.QKV_ROPE, positions=pos, rope_theta=10000.0, q=q, k_out=kk, v_out=v,
             n_q_heads=n_q, n_kv_heads=n_kv)
    torch.cuda.synchronize()
    y = (x[:batch].float() @ w.float().T).view(batch, n_q + 2 * n_kv, 128)
    inv = 10000.0 ** (-torch.arange(0, 64, device="cuda", dtype=torch.float64) * 2 / 128)
    ang = pos.double()[:, None] * inv[None, :]
    cos, sin = torch.cos(ang).float()[:, None, :], torch.sin(ang).float()[:, None, :]

    def rope(t):
        a, b = t[..., :64], t[..., 64:]
        return torch.cat([a * cos - b * sin, b * cos + a * sin], dim=-1)

    _check(q, rope(y[:, :n_q]), "rope q")
    _check(kk, rope(y[:, n_q:n_q + n_kv]), "rope k")
    _check(v, y[:, n_q + n_kv:], "v")


def test_rmsnorm():
    from paper_2605_23389_b200 import linear as L
    batch, dim = 9, 4096
    h = _rand((batch, dim), 11, 3.0)
    gamma = _rand((dim,), 12)
    out = torch.full((16, dim), 7.0, dtype=torch.bfloat16, device="cuda")
    L.rmsnorm(h, gamma, out, batch, 1e-5)
    torch.cuda.synchronize()
    hf = h.float()
    ref = hf * torch.rsqrt(hf.pow(2).mean(-1, keepdim=True) + 1e-5) * gamma.float()
    _check(out[:batch], ref, "rmsnorm")
    assert not out[batch:].float().abs().any()  # MMA-N padding rows zeroed


def test_bad_arguments_fail_loudly():
    from paper_2605_23389_b200 import _lib
    from paper_2605_23389_b200 import linear as L
    x = _x(4, 128, 1)
    w = _rand((100, 128), 2)  # n_out not a multiple of 128
    with pytest.raises(ValueError, match="multiple of 128"):
        L.linear(x, w, 4, torch.empty(4, 100, dtype=torch.bfloat16, device="cuda"))


def test_pdl_chain_matches_torch():
    """rmsnorm -> o_proj-like residual GEMM -> rmsnorm -> gate/up SiLU GEMM -> down residual GEMM, all
    launched with programmatic dependent launch back to back (weights prefetched before each wait)."""
    from paper_2605_23389_b200 import linear as L
    batch, d, inter = 6, 4096, 11008
    h0 = _rand((batch, d), 21)
    g1, g2 = _rand((d,), 22), _rand((d,), 23)
    wo = _rand((d, d), 24, 1 / math.sqrt(d))
    wgu = _rand((2 * inter, d), 25, 1 / math.sqrt(d))
    wd = _rand((d, inter), 26, 1 / math.sqrt(inter))
    h = h0.clone()
    x = torch.zeros(16, d, dtype=torch.bfloat16, device="cuda")
    act = torch.zeros(16, inter, dtype=torch.bfloat16, device="cuda")
    for _ in range(3):  # repeated: every launch overlaps the previous one's tail
        h.copy_(h0)
        L.rmsnorm(h, g1, x, batch, 1e-5, pdl=True)
        L.linear(x, wo, batch, h, L.RESIDUAL, pdl=True)
        L.rmsnorm(h, g2, x, batch, 1e-5, pdl=True)
        L.linear(x, wgu, batch, act, L.SILU_MUL, pdl=True)
        L.linear(act, wd, batch, h, L.RESIDUAL, pdl=True)
    torch.cuda.synchronize()

    def rms(t, g):
        t = t.float()
        return (t * torch.rsqrt(t.pow(2).mean(-1, keepdim=True) + 1e-5) * g.float()).bfloat16().float()

    r = h0.float()
    r = (r + rms(r.bfloat16(), g1) @ wo.float().T).bfloat16().float()
    xg = rms(r.bfloat16(), g2)
    gu = xg @ wgu.float().T
    gg, uu = gu.view(batch, -1, 2, 64)[:, :, 0].reshape(batch, -1), gu.view(batch, -1, 2, 64)[:, :, 1].reshape(batch, -1)
    a = (torch.nn.functional.silu(gg) * uu).bfloat16().float()
    r = r + a @ wd.float().T
    _check(h, r, "pdl chain")


@pytest.mark.parametrize("batch", [5, 37])
def test_fused_rmsnorm_between_linears(batch):
    """Fused RMSNorm (asv.h ss_*): a RESIDUAL linear leaves per-tile row sums of squares of the
    updated residual stream; the next linear reads that stream raw and scales each output row by
    rsqrt(mean(h^2) + eps) — equal to RMSNorm(h) @ W^T with the norm weight folded into W.
    Checked for the STORE and SILU_MUL consumers against torch fp32."""
    from paper_2605_23389_b200 import linear as L
    d, n2, inter = 4096, 1024, 11008
    rows = (batch + 15) // 16 * 16
    h0 = _rand((rows, d), 71)
    x = _x(batch, d, 72)
    wo, w2 = _rand((d, d), 73, 1 / math.sqrt(d)), _rand((n2, d), 74, 1 / math.sqrt(d))
    wgu = _rand((2 * inter, d), 75, 1 / math.sqrt(d))
    ss = torch.full((2 * d // 128, rows), float("nan"), dtype=torch.float32, device="cuda")
    h = h0.clone()
    L.linear(x, wo, batch, h, L.RESIDUAL, ss_out=ss)
    y = torch.zeros(batch, n2, dtype=torch.bfloat16, device="cuda")
    L.linear(h, w2, batch, y, L.STORE, ss_in=ss)
    act = torch.zeros(batch, inter, dtype=torch.bfloat16, device="cuda")
    L.linear(h, wgu, batch, act, L.SILU_MUL, ss_in=ss)
    torch.cuda.synchronize()
    h1 = (h0[:batch].float() + x[:batch].float() @ wo.float().T).bfloat16()
    _check(h[:batch], h1, "residual")
    # the partial sums are those of the stored bf16 rows, one slot per (tile, half tile, row)
    assert torch.isfinite(ss[:, :batch]).all()
    assert torch.allclose(ss[:, :batch].sum(0), h1.float().pow(2).sum(-1), rtol=1e-4)
    xn = h1.float() * torch.rsqrt(h1.float().pow(2).mean(-1, keepdim=True) + 1e-5)
    _check(y, (xn @ w2.float().T).bfloat16(), "fused rmsnorm -> store")
    gu = (xn @ wgu.float().T).view(batch, -1, 2, 64)
    ref = torch.nn.functional.silu(gu[:, :, 0].reshape(batch, -1)) * gu[:, :, 1].reshape(batch, -1)
    _check(act, ref.bfloat16(), "fused rmsnorm -> silu")


# ------------------------------------------------------------ persistent stream-K chain
@pytest.mark.parametrize("n_out,k,batch", [(128, 64, 1), (256, 512, 5), (4096, 4096, 16), (1024, 11008, 33),
                                           (12288, 4096, 64), (512, 4096, 256), (384, 1024, 100)])
def test_chain_single_phase_matches_torch(n_out, k, batch):
    """asv_linear_chain with one phase = a stream-K GEMM (tiles cut between CTAs, owner reduction)."""
    from paper_2605_23389_b200 import linear as L
    ws = L.ChainWorkspace(0)
    x = _x(batch, k, 1)
    w = _rand((n_out, k), 2, 1 / math.sqrt(k))
    y = torch.full((batch, n_out), float("nan"), dtype=torch.bfloat16, device="cuda")
    ref = x[:batch].float() @ w.float().T
    for i in range(2):  # second call: counters and partial slots are reused
        L.linear_chain([dict(x=x, w=w, batch=batch, y=y, epilogue=L.STORE)], ws)
        torch.cuda.synchronize()
        _check(y, ref, f"chain store {n_out}x{k} b{batch} call {i}")


def _layer_weights(d, inter, n_q, n_kv, seed):
    wo = _rand((d, d), seed, 1 / math.sqrt(d))
    wgu = _rand((2 * inter, d), seed + 1, 1 / math.sqrt(d))
    wd = _rand((d, inter), seed + 2, 1 / math.sqrt(inter))
    wqkv = _rand((128 * (n_q + 2 * n_kv), d), seed + 3, 1 / math.sqrt(d))
    return wo, wgu, wd, wqkv


@pytest.mark.parametrize("batch", [4, 37, 130, 256])
def test_chain_decoder_layer_matches_per_gemm_launches(batch):
    """One chain launch = O+residual(ss_out) -> gate/up SiLU (fused norm) -> down+residual(ss_out) ->
    next QKV+RoPE (fused norm), against the same four GEMMs launched one by one (asv_linear, itself
    checked against torch above) and against torch fp32; repeated launches are bit-identical."""
    from paper_2605_23389_b200 import linear as L
    d, inter, n_q, n_kv = 4096, 11008, 32, 32
    rows = (batch + 15) // 16 * 16
    wo, wgu, wd, wqkv = _layer_weights(d, inter, n_q, n_kv, 40)
    attn = _x(batch, d, 41)
    h0 = torch.zeros(rows, d, dtype=torch.bfloat16, device="cuda")
    h0[:batch] = _rand((batch, d), 42)
    pos = torch.randint(0, 16000, (batch,), dtype=torch.int32, device="cuda")

    def run(chain, ws=None):
        h = h0.clone()
        act = torch.zeros(rows, inter, dtype=torch.bfloat16, device="cuda")
        ss_b = torch.zeros(2 * d // 128, rows, dtype=torch.float32, device="cuda")
        ss_a = torch.zeros(2 * d // 128, rows, dtype=torch.float32, device="cuda")
        q = torch.zeros(batch, n_q, 128, dtype=torch.bfloat16, device="cuda")
        kk = torch.zeros(batch, n_kv, 128, dtype=torch.bfloat16, device="cuda")
        v = torch.zeros(batch, n_kv, 128, dtype=torch.bfloat16, device="cuda")
        phases = [dict(x=attn, w=wo, batch=batch, y=h, epilogue=L.RESIDUAL, ss_out=ss_b, pdl=True),
                  dict(x=h, w=wgu, batch=batch, y=act, epilogue=L.SILU_MUL, ss_in=ss_b, pdl=True),
                  dict(x=act, w=wd, batch=batch, y=h, epilogue=L.RESIDUAL, ss_out=ss_a, pdl=True),
                  dict(x=h, w=wqkv, batch=batch, epilogue=L.QKV_ROPE, positions=pos, q=q, k_out=kk, v_out=v,
                       n_q_heads=n_q, n_kv_heads=n_kv, ss_in=ss_a, pdl=True)]
        if chain:
            L.linear_chain(phases, ws)
        else:
            for ph in phases:
                L.linear(**ph)
        torch.cuda.synchronize()
        return h, act, q, kk, v

    ws = L.ChainWorkspace(0)
    got = run(True, ws)
    want = run(False)
    for name, g, w in zip(("h", "act", "q", "k", "v"), got, want):
        _check(g[:batch], w[:batch].float(), f"chain vs per-GEMM {name} b{batch}")
    again = run(True, ws)
    for g, a in zip(got, again):
        assert torch.equal(g, a), "chain launches are not deterministic"
    # torch fp32 of the residual path (norm weights folded into the weights, as the engine does)
    hf = (h0[:batch].float() + attn[:batch].float() @ wo.float().T).bfloat16().float()
    xg = hf * torch.rsqrt(hf.pow(2).mean(-1, keepdim=True) + 1e-5)
    gu = xg @ wgu.float().T
    gg = gu.view(batch, -1, 2, 64)[:, :, 0].reshape(batch, -1)
    uu = gu.view(batch, -1, 2, 64)[:, :, 1].reshape(batch, -1)
    a = (torch.nn.functional.silu(gg) * uu).bfloat16().float()
    _check(got[1][:batch], a, f"chain act vs torch b{batch}")
    _check(got[0][:batch], hf + a @ wd.float().T, f"chain h vs torch b{batch}")


def test_chain_rejects_mixed_batches():
    from paper_2605_23389_b200 import linear as L
    ws = L.ChainWorkspace(0)
    x = _x(4, 128, 1)
    w = _rand((128, 128), 2)
    y = torch.empty(8, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError, match="same batch"):
        L.linear_chain([dict(x=x, w=w, batch=4, y=y), dict(x=x, w=w, batch=3, y=y)], ws)


def test_next_weights_l2_prefetch_leaves_results_unchanged():
    """asv.h next_w (with ASV_LINEAR_NEXT_PF set, as the A/B runs do): a launch's tail prefetches the next
    linear's first ring stages into L2 — pure data movement, the outputs are bit-identical with and
    without it.  (The knob is read once per process: the test runs the prefetch path only when the
    environment enables it.)"""
    from paper_2605_23389_b200 import linear as L
    batch, d, inter = 6, 4096, 11008
    x = _x(batch, d, 81)
    wo = _rand((d, d), 82, 1 / math.sqrt(d))
    wgu = _rand((2 * inter, d), 83, 1 / math.sqrt(d))
    outs = []
    for nxt in (None, wgu):
        h = _rand((batch, d), 84)
        L.linear(x, wo, batch, h, L.RESIDUAL, pdl=True, next_w=nxt)
        act = torch.zeros(batch, inter, dtype=torch.bfloat16, device="cuda")
        hx = torch.zeros(16, d, dtype=torch.bfloat16, device="cuda")
        hx[:batch] = h
        L.linear(hx, wgu, batch, act, L.SILU_MUL, pdl=True)
        torch.cuda.synchronize()
        outs.append((h.clone(), act.clone()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("epi", ["store", "residual", "silu", "qkv"])
def test_every_schedule_matches_torch(epi):
    """asv_linear_set_schedule forces (K splits = cluster size, ring stages); every schedule the
    automatic choice may pick (decode_gemm.cu linear_plan: splits 1-8, stages 2-8) must give the
    same result as torch — including odd cluster sizes, splits that leave a short last split, and the
    staged-epilogue path (RESIDUAL / QKV with inputs staged in shared memory)."""
    from paper_2605_23389_b200 import _lib
    from paper_2605_23389_b200 import linear as L
    h = _lib.lib()
    k, batch = 1088, 5  # 17 K blocks: uneven splits for most split counts
    n_out = 768 if epi == "qkv" else 512
    x = _x(batch, k, 11)
    w = _rand((n_out, k), 12, 1 / math.sqrt(k))
    acc = x[:batch].float() @ w.float().T
    try:
        for sp in (1, 2, 3, 5, 6, 8):
            for st in (2, 5, 8):
                _lib.check(h.asv_linear_set_schedule(sp, st))
                if epi == "store":
                    y = torch.full((batch, n_out), float("nan"), dtype=torch.bfloat16, device="cuda")
                    L.linear(x, w, batch, y, L.STORE)
                    ref = acc
                elif epi == "residual":
                    y0 = _rand((batch, n_out), 13)
                    y = y0.clone()
                    L.linear(x, w, batch, y, L.RESIDUAL)
                    ref = y0.float() + acc
                elif epi == "silu":
                    y = torch.full((batch, n_out // 2), float("nan"), dtype=torch.bfloat16, device="cuda")
                    L.linear(x, w, batch, y, L.SILU_MUL)
                    a4 = acc.view(batch, n_out // 128, 2, 64)
                    ref = (torch.nn.functional.silu(a4[:, :, 0]) * a4[:, :, 1]).reshape(batch, n_out // 2)
                else:
                    pos = torch.arange(batch, dtype=torch.int32, device="cuda") * 37 + 3
                    q = torch.empty(batch, 2, 128, dtype=torch.bfloat16, device="cuda")
                    kk = torch.empty(batch, 2, 128, dtype=torch.bfloat16, device="cuda")
                    v = torch.empty(batch, 2, 128, dtype=torch.bfloat16, device="cuda")
                    L.linear(x, w, batch, None, L.QKV_ROPE, positions=pos, q=q, k_out=kk, v_out=v,
                             n_q_heads=2, n_kv_heads=2)
                    heads = acc.view(batch, 6, 128)
                    inv = 10000.0 ** (-torch.arange(64, device="cuda").float() * 2 / 128)
                    ang = pos.float()[:, None] * inv[None, :]
                    cs, sn = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
                    lo, hi = heads[:, :4, :64], heads[:, :4, 64:]
                    rot = torch.cat([lo * cs - hi * sn, hi * cs + lo * sn], dim=-1)
                    ref = torch.cat([rot, heads[:, 4:]], dim=1)
                    y = torch.cat([q, kk, v], dim=1)
                torch.cuda.synchronize()
                _check(y, ref, f"{epi} splits {sp} stages {st}")
    finally:
        _lib.check(h.asv_linear_set_schedule(0, 0))
