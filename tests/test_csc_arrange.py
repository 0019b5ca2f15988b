"""Host logic of the pCSC band layout on CPU (no GPU): one warp list arranged by the library's
own arrange_list through the msrep_debug_arrange test hook (DESIGN.md sec. 5 "pCSC").  The
kernel's correctness rests on these invariants: every entry placed exactly once; same-row groups
(32 entries of one row) first; then groups of 32 DISTINCT rows (the warp's plain
read-modify-write scatter needs that); then, if the greedy pass got stuck, segmented groups with
rows non-decreasing and list order within a row (the warp segmented scan needs contiguous runs)."""
import numpy as np
import pytest

import paper_2209_07552_b200 as M

ROWS = 8192


def check_invariants(pk):
    order, same, seg = M.msrep_debug_arrange(pk)
    n = pk.size
    real = order[order >= 0]
    assert np.array_equal(np.sort(real), np.arange(n)), "every entry exactly once"
    rows = np.where(order >= 0, (pk[np.maximum(order, 0)] & (ROWS - 1)).astype(np.int64), -1)
    assert same % 32 == 0 and same <= order.size
    for g in range(0, same, 32):                       # same-row groups: one row, no holes, list order
        grp = order[g:g + 32]
        assert (grp >= 0).all() and len(set(rows[g:g + 32])) == 1
        assert (np.diff(grp) > 0).all()
    end = seg if seg >= 0 else order.size
    assert seg < 0 or (seg % 32 == 0 and seg >= same)
    for g in range(same, end, 32):                      # greedy groups: distinct rows
        r = rows[g:min(g + 32, end)]
        r = r[r >= 0]
        assert len(set(r.tolist())) == r.size, ("duplicate row in a distinct group", g)
    if seg >= 0:                                        # segmented tail: sorted runs, no holes
        tail = order[seg:]
        assert (tail >= 0).all()
        tr = rows[seg:]
        assert (np.diff(tr) >= 0).all()
        for r in np.unique(tr):
            assert (np.diff(tail[tr == r]) > 0).all()
    return order, same, seg


def pack(rows, cols=None):
    rows = np.asarray(rows, np.uint32)
    cols = np.arange(rows.size, dtype=np.uint32) if cols is None else np.asarray(cols, np.uint32)
    return (rows & (ROWS - 1)) | (cols << 13)


def test_distinct_rows_have_no_holes():
    rng = np.random.default_rng(1)
    pk = pack(rng.permutation(4096)[:1000])            # 1000 entries on 1000 distinct rows
    order, same, seg = check_invariants(pk)
    assert same == 0 and seg == -1
    assert (order >= 0).all() and order.size == 1000


def test_heavy_rows_become_same_row_groups():
    rows = np.concatenate([np.full(640, 3), np.full(100, 7), np.arange(100, 400)])
    rng = np.random.default_rng(2)
    pk = pack(rng.permutation(rows))
    order, same, seg = check_invariants(pk)
    assert same >= 20 * 32                              # row 3's full 32-blocks lead the list


def test_few_rows_switch_to_segmented_tail():
    rng = np.random.default_rng(3)
    rows = np.concatenate([np.full(200, r) for r in (11, 12, 13)])
    pk = pack(rng.permutation(rows))
    order, same, seg = check_invariants(pk)
    assert seg >= 0, "the stuck tail on 3 rows should be segmented"
    holes = int((order < 0).sum())
    assert holes <= 31                                  # only the group closed when the greedy pass stuck


def test_short_tail_stays_greedy():
    # a stuck tail that costs few extra groups stays on the greedy (distinct-row) path
    rows = np.concatenate([np.arange(64), [5, 5]])
    order, same, seg = check_invariants(pack(rows))
    assert seg == -1


@pytest.mark.parametrize("seed", range(12))
def test_random_lists_keep_invariants(seed):
    rng = np.random.default_rng(100 + seed)
    kind = seed % 4
    n = int(rng.integers(1, 3000))
    if kind == 0:                                       # uniform rows of a band
        rows = rng.integers(0, ROWS, n)
    elif kind == 1:                                     # a warp's small row range
        rows = rng.integers(0, int(rng.integers(1, 40)), n)
    elif kind == 2:                                     # power-law rows (R-MAT-like skew)
        rows = np.minimum((rng.pareto(1.2, n) * 3).astype(np.int64), ROWS - 1)
    else:                                               # sorted runs, as in a banded matrix's lists
        rows = np.sort(rng.integers(0, int(rng.integers(32, 600)), n))
    check_invariants(pack(rows))


def test_empty_list():
    order, same, seg = M.msrep_debug_arrange(np.zeros(0, np.uint32))
    assert order.size == 0 and same == 0 and seg == -1
