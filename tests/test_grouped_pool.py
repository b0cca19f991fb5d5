"""Layer-major device pools in page groups (include/asv.h).

A group's layer pitch (group_pages * slice) stays below 2 GiB, the largest
pitch at which the copy engines run a 2-D KV page copy at full PCIe rate
(B200: 54 GB/s below, 29.7 GB/s = one row per copy at >= 2 GiB;
tools/copy_tlb_probe.py).  CPU tests pin the offset arithmetic of the C ABI
against the Python model; GPU tests run the KV copies and the attention kernel
on a three-group pool against byte-exact models and the fp32 oracle.
"""
import ctypes as C

import numpy as np
import pytest

import _util as U


def _shape(n_q, n_kv, L):
    from paper_2605_23389_b200 import _lib
    return _lib.AttnShape(n_q, n_kv, 128, 16, L)


@pytest.mark.parametrize("n_kv,L,pool_pages", [(32, 32, 16448), (32, 32, 8191), (32, 32, 8192), (8, 40, 64900),
                                               (1, 2, 524300), (32, 2, 100)])
def test_group_geometry_matches_model(n_kv, L, pool_pages):
    from paper_2605_23389_b200 import _lib
    h = _lib.lib()
    sh = _shape(n_kv, n_kv, L)
    g = h.asv_pool_group_pages(C.byref(sh), pool_pages)
    assert g == U.group_pages(n_kv, pool_pages)
    assert g * 2 * n_kv * 4096 < 1 << 31
    groups = -(-pool_pages // g) if pool_pages % g else pool_pages // g
    usable = h.asv_pool_usable_pages(C.byref(sh), pool_pages)
    assert usable == (pool_pages // g) * g and pool_pages - usable < groups
    if pool_pages * 2 * n_kv * 4096 < 1 << 31:
        assert g == pool_pages  # a pool that fits one group keeps the plain layer-major layout


def test_pool_offset_matches_model_across_groups():
    from paper_2605_23389_b200 import _lib
    h = _lib.lib()
    n_kv, L, pool_pages = 32, 32, 16448
    sh = _shape(n_kv, n_kv, L)
    usable = h.asv_pool_usable_pages(C.byref(sh), pool_pages)
    rng = np.random.default_rng(3)
    seen = set()
    for page in list(rng.integers(0, usable, 40)) + [0, usable - 1, U.group_pages(n_kv, pool_pages)]:
        for layer in (0, 7, L - 1):
            for kv in (0, 1):
                head, t, d = int(rng.integers(0, n_kv)), int(rng.integers(0, 16)), int(rng.integers(0, 128))
                off = h.asv_pool_offset(C.byref(sh), pool_pages, int(page), layer, kv, head, t, d)
                want = U.pool_block_offset(n_kv, L, pool_pages, int(page), layer, kv, head) + U.swz_off(t, d)
                assert off == want
                assert 0 <= off < pool_pages * U.page_bytes(n_kv, L)
                seen.add(off // 4096)
    assert h.asv_pool_offset(C.byref(sh), pool_pages, usable, 0, 0, 0, 0, 0) == -1  # beyond the last group


def test_groups_tile_the_pool_without_overlap():
    """every (usable page, layer) slice maps to a distinct slice inside the allocation"""
    n_kv, L, pool_pages = 1, 3, 524300
    g = U.group_pages(n_kv, pool_pages)
    usable = (pool_pages // g) * g
    pages = np.arange(usable, dtype=np.int64)
    slots = np.concatenate([(pages // g) * g * L + layer * g + pages % g for layer in range(L)])
    assert len(np.unique(slots)) == len(slots)
    assert slots.max() < pool_pages * L


# ------------------------------------------------------------------ GPU
N_KV, LAYERS, POOL_PAGES = 1, 2, 524300   # slice 8 KiB -> 3 groups of 174766 pages, 8.6 GB pool


@pytest.mark.gpu
def test_kv_copy_roundtrip_on_multigroup_pool():
    torch = pytest.importorskip("torch")
    from paper_2605_23389_b200 import _lib
    h = _lib.lib()
    sh = _shape(8, N_KV, LAYERS)
    pb = U.page_bytes(N_KV, LAYERS)
    g = U.group_pages(N_KV, POOL_PAGES)
    usable = (POOL_PAGES // g) * g
    dev = torch.device("cuda", 0)
    pool = torch.zeros(POOL_PAGES * pb, dtype=torch.uint8, device=dev)
    tokens = 16 * 6 + 5
    npg = (tokens + 15) // 16
    pages = np.array([0, g - 1, g, 2 * g + 17, usable - 1, g + 5, 3], np.int32)[:npg]
    host = torch.empty(npg * pb, dtype=torch.uint8, pin_memory=True)
    host.copy_(torch.from_numpy(U.random_bf16(9, npg * pb // 2).view(np.uint8)))
    ptrs = (C.c_void_p * npg)(*[host.data_ptr() + j * pb for j in range(npg)])
    st = torch.cuda.current_stream().cuda_stream
    moved = C.c_int64(0)
    pp = pages.ctypes.data_as(C.POINTER(C.c_int32))
    _lib.check(h.asv_kv_copy_h2d(C.byref(sh), pool.data_ptr(), POOL_PAGES, pp, tokens, ptrs, st, C.byref(moved)))
    torch.cuda.synchronize()
    assert moved.value == tokens * LAYERS * 2 * N_KV * 256
    src = host.numpy().reshape(npg, LAYERS, 2, N_KV, 4096)
    flat = pool.view(-1)
    for j, p in enumerate(pages):
        rows = min(16, tokens - 16 * j)
        for layer in range(LAYERS):
            for kv in range(2):
                off = U.pool_block_offset(N_KV, LAYERS, POOL_PAGES, int(p), layer, kv, 0)
                got = flat[off:off + 4096].cpu().numpy()
                assert np.array_equal(got[:rows * 256], src[j, layer, kv, 0, :rows * 256])
                assert not got[rows * 256:].any()  # rows beyond the request untouched
    # device -> host round trip of the same request
    back = torch.zeros(npg * pb, dtype=torch.uint8, pin_memory=True)
    bptrs = (C.c_void_p * npg)(*[back.data_ptr() + j * pb for j in range(npg)])
    _lib.check(h.asv_kv_copy_d2h(C.byref(sh), pool.data_ptr(), POOL_PAGES, pp, tokens, bptrs, st, C.byref(moved)))
    torch.cuda.synchronize()
    b = back.numpy().reshape(npg, LAYERS, 2, N_KV, 4096)
    for j in range(npg):
        rows = min(16, tokens - 16 * j)
        assert np.array_equal(b[j, :, :, :, :rows * 256], src[j, :, :, :, :rows * 256])
    # a page id beyond the usable pool is rejected, not written
    bad = np.array([usable], np.int32)
    rc = h.asv_kv_copy_h2d(C.byref(sh), pool.data_ptr(), POOL_PAGES, bad.ctypes.data_as(C.POINTER(C.c_int32)), 16,
                           ptrs, st, C.byref(moved))
    assert rc != 0 and b"usable" in h.asv_last_error()


@pytest.mark.gpu
def test_attention_on_multigroup_pool_matches_oracle():
    torch = pytest.importorskip("torch")
    from paper_2605_23389_b200 import PagedDecodeAttention
    n_q, layer = 8, 1
    pb = U.page_bytes(N_KV, LAYERS)
    g = U.group_pages(N_KV, POOL_PAGES)
    seq = [700, 33, 4096, 16, 1500]
    rng = np.random.default_rng(5)
    # pages spread over all three groups, including both ends of each group
    cand = np.unique(np.concatenate([rng.integers(0, 3 * g, 600), [0, g - 1, g, 2 * g - 1, 2 * g, 3 * g - 1]]))
    cand = rng.permutation(cand).astype(np.int32)
    indptr, indices = [0], []
    pos = 0
    for s in seq:
        n = (s + 16) // 16
        indices.extend(cand[pos:pos + n])
        pos += n
        indptr.append(len(indices))
    indptr, indices = np.asarray(indptr, np.int32), np.asarray(indices, np.int32)
    pool = np.zeros(POOL_PAGES * pb, np.uint8)  # lazily backed: only the written blocks become resident
    blk = U.random_bf16(11, len(indices) * LAYERS * 2 * 2048).view(np.uint8).reshape(len(indices), LAYERS, 2, 4096)
    offs = []
    for j, p in enumerate(indices):
        for l in range(LAYERS):
            for kv in range(2):
                off = U.pool_block_offset(N_KV, LAYERS, POOL_PAGES, int(p), l, kv, 0)
                pool[off:off + 4096] = blk[j, l, kv]
                offs.append(off // 4096)
    b = len(seq)
    q_bits = U.random_bf16(12, b * n_q * 128).reshape(b, n_q, 128)
    att = PagedDecodeAttention(n_q, N_KV, LAYERS, device=0)
    ref, _ = U.Oracle().attention(n_q, N_KV, LAYERS, layer, q_bits, pool, seq, indptr, indices, att.sm_scale)
    dev = torch.device("cuda", 0)
    pool_d = torch.zeros(POOL_PAGES * pb, dtype=torch.uint8, device=dev)
    pool_d.view(-1, 4096)[torch.tensor(offs, device=dev)] = torch.from_numpy(blk.reshape(-1, 4096)).to(dev)
    q_d = torch.from_numpy(q_bits.view(np.int16)).to(dev).view(torch.bfloat16)
    out = torch.empty(b, n_q, 128, dtype=torch.bfloat16, device=dev)
    plan = att.plan(seq, indptr, indices)
    att.run(q_d, pool_d, layer, plan, out)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    err = np.abs(got - ref)
    print(f"multigroup pool: max_abs={err.max():.3e}")
    assert (err <= 4e-3 + 8e-3 * np.abs(ref)).all(), err.max()
