"""CPU: the decode-linear schedule (include/asv.h asv_linear_schedule; decode_gemm.cu linear_plan) —
host-only arithmetic, no GPU needed.  Every schedule it picks must be launchable as ONE wave on a
B200 (148 SMs, 228 KiB shared memory and 512 TMEM columns per SM), never leave a K split empty, and
stay inside the kernel's limits; the 7B decode shapes get the schedules measured best on B200
(DESIGN.md §4 L1, profiles/linear_sched_sweep_r02.jsonl)."""
import ctypes as C
import itertools

import pytest

from paper_2605_23389_b200 import _lib

SMS = 148
EPIS = {"store": _lib.EPI_STORE, "residual": _lib.EPI_RESIDUAL, "silu": _lib.EPI_SILU_MUL, "qkv": _lib.EPI_QKV_ROPE}


def schedule(n_out, k, batch, epi, sms=SMS):
    sp, st, sm = C.c_int32(0), C.c_int32(0), C.c_int32(0)
    _lib.check(_lib.lib().asv_linear_schedule(n_out, k, batch, epi, sms, C.byref(sp), C.byref(st), C.byref(sm)))
    return sp.value, st.value, sm.value


@pytest.mark.parametrize("epi", list(EPIS))
def test_every_schedule_is_one_launchable_wave(epi):
    e = EPIS[epi]
    shapes = [128, 384, 1024, 4096, 5120, 12288, 13824, 22016, 27648]
    ks = [64, 128, 1088, 4096, 5120, 11008, 13824]
    for n_out, k, batch in itertools.product(shapes, ks, [1, 4, 16, 17, 33, 64, 100, 128, 256]):
        sp, st, smem = schedule(n_out, k, batch, e)
        kbs = k // 64
        bn = (batch + 15) // 16 * 16
        assert 1 <= sp <= 8 and 2 <= st <= 8, (n_out, k, batch, sp, st)
        per = -(-kbs // sp)
        assert -(-kbs // per) == sp, "a K split would be empty"
        assert smem <= 227 * 1024
        ring = st * (16384 + bn * 128)
        assert smem >= max(ring, bn * 512), "the epilogue's fp32 tile reuses the ring"
        ncols = 32 if bn <= 32 else 64 if bn <= 64 else 128 if bn <= 128 else 256
        per_sm = min((228 * 1024) // (smem + 1024), 512 // ncols)
        ctas = n_out // 128 * sp
        # one wave: the explicit residency model (clusters keep 10% slack for GPC placement)
        assert per_sm >= 1
        if ctas > per_sm * SMS:
            # only possible when even one CTA per tile does not fit in one wave: splits must be 1
            assert sp == 1, (n_out, k, batch, sp, st, ctas, per_sm)
        elif sp > 1:
            assert ctas <= int(per_sm * SMS * 0.9), (n_out, k, batch, sp, st)


def test_schedule_is_deterministic_and_validates():
    a = schedule(12288, 4096, 4, EPIS["qkv"])
    assert a == schedule(12288, 4096, 4, EPIS["qkv"])
    h = _lib.lib()
    sp = C.c_int32(0)
    assert h.asv_linear_schedule(100, 4096, 4, 0, SMS, C.byref(sp), None, None) != 0  # n_out % 128
    assert h.asv_linear_schedule(128, 100, 4, 0, SMS, C.byref(sp), None, None) != 0   # k % 64
    assert h.asv_linear_schedule(128, 64, 0, 0, SMS, C.byref(sp), None, None) != 0    # batch
    assert h.asv_linear_schedule(128, 64, 4, 9, SMS, C.byref(sp), None, None) != 0    # epilogue


def test_7b_decode_schedules_measured_best():
    # batch 4 (bn 16): the QKV and gate/up projections get more, smaller CTAs (more bytes in flight)
    # than round 1's fixed ~100 KiB ring / power-of-two split; O and down keep 8 x 5
    qkv = schedule(12288, 4096, 4, EPIS["qkv"])[:2]
    gu = schedule(22016, 4096, 4, EPIS["silu"])[:2]
    o = schedule(4096, 4096, 4, EPIS["residual"])[:2]
    down = schedule(4096, 11008, 4, EPIS["residual"])[:2]
    assert o == (8, 5) and down == (8, 5)
    assert qkv[0] * 96 > 192 and gu[0] * 172 > 172  # more CTAs than round 1's (2 x 96, 1 x 172)

    def fly(n_out, k, batch, sp, st):
        return n_out // 128 * sp * min(st, -(-(k // 64) // sp)) * (16384 + 16 * 128)
    assert fly(12288, 4096, 4, *qkv) > fly(12288, 4096, 4, 2, 5)
    assert fly(22016, 4096, 4, *gu) > fly(22016, 4096, 4, 1, 5)
