"""CPU: the split-KV work plan (asv_attn_plan_build, K4) — host logic only."""
import ctypes as C

import numpy as np
import pytest

from paper_2605_23389_b200 import _lib

DESC = 40


def build(seq, n_q=32, n_kv=32, workers=1184, append=True, short_table=False):
    h = _lib.lib()
    shape = _lib.AttnShape(n_q, n_kv, 128, 16, 32)
    seq = np.asarray(seq, np.int32)
    npg = (seq + (16 if append else 15)) // 16
    if short_table:
        npg = npg - 1
    indptr = np.concatenate([[0], np.cumsum(npg)]).astype(np.int32)
    indices = np.arange(indptr[-1], dtype=np.int32)[::-1].copy()
    cap = 40 * (int(npg.sum()) // 2 + len(seq) + 1) + 2 * len(seq) + 8
    buf = np.zeros(cap, np.int32)
    plan = _lib.AttnPlan()
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))  # noqa: E731
    rc = h.asv_attn_plan_build(C.byref(shape), len(seq), p(seq), p(indptr), p(indices), workers, p(buf), cap,
                               C.byref(plan))
    _lib.check(rc)
    return plan, buf, indptr, indices


@pytest.mark.parametrize("seq", [[1], [16, 17, 2048], list(range(1, 400, 7)), [131072, 3], [8192] * 13])
def test_splits_cover_every_page_exactly_once(seq):
    plan, buf, indptr, indices = build(seq)
    seq = np.asarray(seq)
    sb = buf[plan.off_split_base:plan.off_split_base + len(seq) + 1]
    seen = {r: [] for r in range(len(seq))}
    sizes = []
    for g in range(plan.total_splits):
        d = buf[plan.off_desc + g * DESC: plan.off_desc + (g + 1) * DESC]
        r, slot, pb, pe, s, ns = d[:6]
        assert s == seq[r] and pe > pb and pe - pb <= 32
        assert ns == sb[r + 1] - sb[r] and sb[r] <= slot < sb[r + 1]
        assert list(d[8:8 + pe - pb]) == list(indices[indptr[r] + pb: indptr[r] + pe])
        seen[r].append((pb, pe))
        sizes.append(pe - pb)
        if d[6] >= 0:  # append page = page holding token index seq
            assert slot == sb[r + 1] - 1 and d[6] == indices[indptr[r] + s // 16]
    for r, spans in seen.items():
        spans.sort()
        npages = (seq[r] + 15) // 16
        assert spans[0][0] == 0 and spans[-1][1] == npages
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert sizes == sorted(sizes, reverse=True), "descriptors must be longest-first (LPT)"
    merges = buf[plan.off_merge:plan.off_merge + plan.n_merge]
    assert sorted(merges) == [r for r in range(len(seq)) if sb[r + 1] - sb[r] > 1]
    assert plan.num_items == plan.total_splits * 32


def test_aligned_batch_gets_two_item_sizes_longest_first():
    """Length-aligned batch: near-equal head items, then the last quarter of every request in
    quarter-size tail items; descriptors are ordered longest first (the dynamic LPT schedule)
    and each request's splits tile its pages exactly."""
    seq = [4096 + i for i in range(16)]
    plan, buf, _, _ = build(seq)
    d = [buf[plan.off_desc + g * DESC: plan.off_desc + g * DESC + 8] for g in range(plan.total_splits)]
    sizes = [int(x[3] - x[2]) for x in d]
    assert sizes == sorted(sizes, reverse=True)
    big = [z for z in sizes if z > sizes[0] // 2]
    small = [z for z in sizes if z <= sizes[0] // 2]
    assert max(big) - min(big) <= 1 and small and max(small) - min(small) <= 1
    assert 3 <= sizes[0] / small[0] <= 5
    for r, s in enumerate(seq):
        spans = sorted((int(x[2]), int(x[3])) for x in d if x[0] == r)
        assert spans[0][0] == 0 and spans[-1][1] == (s + 15) // 16
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_gqa_plan_keeps_equal_items():
    """GQA: no small-item tail (its merge has one row per query head; measured slower on C4)."""
    plan, buf, _, _ = build([4096 + i for i in range(16)], n_q=40, n_kv=8)
    sizes = {int(buf[plan.off_desc + g * DESC + 3] - buf[plan.off_desc + g * DESC + 2])
             for g in range(plan.total_splits)}
    assert max(sizes) - min(sizes) <= 1


def test_gqa_plan_items_per_kv_head():
    plan, _, _, _ = build([1000, 2000], n_q=40, n_kv=8)
    assert plan.num_items == plan.total_splits * 8


def test_plan_errors_follow_reference_messages():
    with pytest.raises(ValueError, match="empty batch"):
        build([])
    with pytest.raises(ValueError, match="prefix lengths must be >= 1"):
        build([5, 0])
    with pytest.raises(ValueError, match="page table shorter"):
        build([40], append=False, short_table=True)
    with pytest.raises(ValueError, match="group size"):
        build([10], n_q=24, n_kv=8)


def test_plan_flags_requests_without_an_append_page():
    """A request whose page list stops at ceil(seq/16) pages (no page for token index seq) is
    counted in append_missing, so a launch that appends K/V rows is rejected rather than
    silently dropping the row (asv_decode_attention checks it)."""
    plan, _, _, _ = build([16, 17, 32, 40], append=True)
    assert plan.append_missing == 0
    plan, _, _, _ = build([16, 17, 32, 40], append=False)
    # seq 16 and 32 end exactly on a page boundary: their append position needs one more page
    assert plan.append_missing == 2
