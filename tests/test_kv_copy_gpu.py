"""GPU: KV page moves (asv_kv_copy_*) are byte-exact and move exactly
tokens * kv_bytes_per_token bytes (reference cluster_sim.hpp:239-241).

Host pages are page-major [L][2][n_kv][16][128]; device pools are layer-major
[L][pool_pages][2][n_kv][16][128] (include/asv.h).  For a request with s tokens
only the first s token rows of its pages carry data."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import _util as U  # noqa: E402

pytestmark = pytest.mark.gpu


def _pinned_pages(n, page_bytes, seed):
    t = torch.empty(n * page_bytes, dtype=torch.uint8, pin_memory=True)
    t.copy_(torch.from_numpy(U.random_bf16(seed, n * page_bytes // 2).view(np.uint8)))
    return t


def _host_ptrs(host, n, page_bytes):
    arr = (C.c_void_p * n)(*[host.data_ptr() + j * page_bytes for j in range(n)])
    return arr


def _expected_pool(pool_np, host_np, pages, tokens, n_kv, L):
    """numpy model of an H2D copy: page j -> pool page pages[j], valid rows only."""
    pb = U.page_bytes(n_kv, L)
    blocks = U.block_view(pool_np, n_kv, L)            # [L][pages][2][n_kv][4096]
    src = host_np.reshape(-1, L, 2, n_kv, 4096)        # page-major
    for j, p in enumerate(pages):
        rows = min(16, tokens - 16 * j)
        blocks[:, p, :, :, :rows * 256] = src[j, :, :, :, :rows * 256]
    return pool_np


@pytest.mark.parametrize("n_kv,L,tokens", [(32, 2, 40), (8, 3, 16), (8, 40, 257), (32, 1, 1)])
def test_h2d_d2h_d2d_roundtrip(n_kv, L, tokens):
    from paper_2605_23389_b200 import _lib
    h = _lib.lib()
    shape = _lib.AttnShape(4 * n_kv if n_kv == 8 else n_kv, n_kv, 128, 16, L)
    pb = U.page_bytes(n_kv, L)
    npg = (tokens + 15) // 16
    pool_pages = npg + 5
    dev = torch.device("cuda", 0)
    pool = torch.zeros(pool_pages * pb, dtype=torch.uint8, device=dev)
    host = _pinned_pages(npg, pb, 7)
    pages = np.random.default_rng(1).permutation(pool_pages)[:npg].astype(np.int32)
    pp = pages.ctypes.data_as(C.POINTER(C.c_int32))
    moved = C.c_int64(0)
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(h.asv_kv_copy_h2d(C.byref(shape), pool.data_ptr(), pool_pages, pp, tokens,
                                 _host_ptrs(host, npg, pb), st, C.byref(moved)))
    torch.cuda.synchronize()
    assert moved.value == tokens * L * 2 * n_kv * 256
    want = _expected_pool(np.zeros(pool_pages * pb, np.uint8), host.numpy(), pages, tokens, n_kv, L)
    assert np.array_equal(pool.cpu().numpy(), want)

    # device -> device into a second pool (pair admit), then back to host
    pool2_pages = npg + 3
    pool2 = torch.zeros(pool2_pages * pb, dtype=torch.uint8, device=dev)
    pages2 = np.arange(pool2_pages - npg, pool2_pages, dtype=np.int32)
    _lib.check(h.asv_kv_copy_d2d(C.byref(shape), pool2.data_ptr(), pool2_pages, 0,
                                 pages2.ctypes.data_as(C.POINTER(C.c_int32)), pool.data_ptr(), pool_pages, 0, pp,
                                 tokens, st, C.byref(moved)))
    back = torch.zeros(npg * pb, dtype=torch.uint8, pin_memory=True)
    _lib.check(h.asv_kv_copy_d2h(C.byref(shape), pool2.data_ptr(), pool2_pages,
                                 pages2.ctypes.data_as(C.POINTER(C.c_int32)), tokens, _host_ptrs(back, npg, pb), st,
                                 C.byref(moved)))
    torch.cuda.synchronize()
    assert moved.value == tokens * L * 2 * n_kv * 256
    src = host.numpy().reshape(npg, L, 2, n_kv, 16, 256)
    got = back.numpy().reshape(npg, L, 2, n_kv, 16, 256)
    for j in range(npg):
        rows = min(16, tokens - 16 * j)
        assert np.array_equal(got[j, :, :, :, :rows], src[j, :, :, :, :rows])
        assert not got[j, :, :, :, rows:].any()


@pytest.mark.parametrize("n", [1, 4, 1001, 40 * 2000 + 3])
def test_plan_upload_through_sm_loads_is_exact(n):
    """asv_plan_upload pulls a plan from mapped pinned memory with SM loads (no copy engine)."""
    from paper_2605_23389_b200 import _lib
    h = _lib.lib()
    src = torch.from_numpy(np.random.default_rng(n).integers(-2**31, 2**31 - 1, n + 3, dtype=np.int64)
                           .astype(np.int32)).pin_memory()
    dst = torch.full((n + 3,), -7, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(h.asv_plan_upload(src.data_ptr(), dst.data_ptr(), n, st))
    torch.cuda.synchronize()
    assert torch.equal(dst[:n].cpu(), src[:n])
