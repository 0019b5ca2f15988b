"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself.

Each pin is chosen so that a plausible mistake (dropped term, wrong sign or
index, transposed operand, off-by-one boundary) fails at least one test:
  * SPEC.md worked values on fixture E (tests/golden/fixture_E.json, cited),
  * closed forms (identity, permutation, diagonal, 27-point stencil, 1xN chain),
  * numpy dense brute force (an independent library primitive),
  * exhaustive invariants (balance <= 1, exact tiling, merge-of-partition = id).
"""
import itertools

import numpy as np
import pytest

import oracle


def E_csr(g, dtype=np.float64):
    return (np.array(g["csr_row_ptr"], np.int64), np.array(g["csr_col_idx"], np.int32),
            np.array(g["csr_val"], dtype))


# ------------------------------------------------------------- conversions
def test_E_coo_to_csr(golden_E):
    g = golden_E
    rp, ci, v = oracle.coo_to_csr(4, g["coo_row"], g["coo_col"], np.array(g["coo_val"]))
    assert rp.tolist() == g["csr_row_ptr"] and ci.tolist() == g["csr_col_idx"]
    assert v.tolist() == g["csr_val"]


def test_E_csr_to_csc(golden_E):
    g = golden_E
    rp, ci, v = E_csr(g)
    cp, ri, cv = oracle.csr_to_csc(4, 4, rp, ci, v)
    assert cp.tolist() == g["csc_col_ptr"] and ri.tolist() == g["csc_row_idx"]
    assert cv.tolist() == g["csc_val"]


def test_empty_matrix_conversion():
    rp, ci, v = oracle.coo_to_csr(3, np.zeros(0, np.int64), np.zeros(0, np.int32), np.zeros(0))
    assert rp.tolist() == [0, 0, 0, 0]


def test_diagonal_csc_equals_csr():
    n = 7
    rp = np.arange(n + 1, dtype=np.int64); ci = np.arange(n, dtype=np.int32)
    v = np.random.default_rng(0).standard_normal(n)
    cp, ri, cv = oracle.csr_to_csc(n, n, rp, ci, v)
    assert np.array_equal(cp, rp) and np.array_equal(ri, ci) and np.array_equal(cv, v)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_roundtrips_bit_exact(dtype):
    rng = np.random.default_rng(11)
    for trial in range(30):
        m, n = rng.integers(1, 40, 2)
        dense = (rng.random((m, n)) < 0.2) * rng.standard_normal((m, n))
        r, c = np.nonzero(dense)                                # row-major = row-sorted
        vals = dense[r, c].astype(dtype)
        rp, ci, v = oracle.coo_to_csr(m, r, c, vals)
        # CSR -> COO -> CSR identity
        ri = oracle.csr_to_coo(m, rp)
        assert np.array_equal(ri, r) and np.array_equal(ci, c)
        assert v.tobytes() == vals.tobytes()
        # double transpose is the identity: CSC(A) read as CSR(A^T), back
        cp, rowi, cv = oracle.csr_to_csc(m, n, rp, ci, v)
        rp2, ci2, v2 = oracle.csr_to_csc(n, m, cp, rowi, cv)
        assert np.array_equal(rp2, rp) and np.array_equal(ci2, ci) and v2.tobytes() == v.tobytes()
        # CSC expands to the transpose's triplets
        cj = oracle.csc_to_coo(n, cp)
        assert sorted(zip(cj.tolist(), rowi.tolist())) == sorted(zip(c.tolist(), r.tolist()))


# ----------------------------------------------------------------- SpMV pins
@pytest.mark.parametrize("fmt", ["csr", "csc", "coo"])
def test_E_spmv_worked_values(golden_E, fmt):
    g = golden_E
    for case in g["spmv"]:
        x = np.array(case["x"], float); y = np.array(case["y"], float)
        if fmt == "csr":
            out = oracle.spmv_csr(4, *E_csr(g), x, y, case["alpha"], case["beta"])
        elif fmt == "csc":
            out = oracle.spmv_csc(4, 4, g["csc_col_ptr"], g["csc_row_idx"], np.array(g["csc_val"]),
                                  x, y, case["alpha"], case["beta"])
        else:
            out = oracle.spmv_coo(4, g["coo_row"], g["coo_col"], np.array(g["coo_val"]), x, y,
                                  case["alpha"], case["beta"])
        assert out.tolist() == case["expect"]


def test_E_nonsymmetric_x_catches_transpose(golden_E):
    # x = e_2 picks column 2: A[:,2] = [2,0,0,0]; a transposed operand would give row 2 (empty).
    g = golden_E
    x = np.array([0, 0, 1, 0], float)
    assert oracle.spmv_csr(4, *E_csr(g), x, np.zeros(4), 1.0, 0.0).tolist() == [2, 0, 0, 0]


def test_identity_closed_form():
    n = 50
    rng = np.random.default_rng(1)
    rp = np.arange(n + 1, dtype=np.int64); ci = np.arange(n, dtype=np.int32); v = np.ones(n)
    x = rng.standard_normal(n); y = rng.standard_normal(n)
    out = oracle.spmv_csr(n, rp, ci, v, x, y, 1.5, -0.5)
    assert np.array_equal(out, 1.5 * x + (-0.5) * y)       # alpha*x + beta*y, one rounding each


def test_permutation_bit_exact():
    n = 97
    rng = np.random.default_rng(2)
    pi = rng.permutation(n)
    rp = np.arange(n + 1, dtype=np.int64); ci = pi.astype(np.int32); v = np.ones(n)
    x = rng.standard_normal(n)
    for f in (lambda: oracle.spmv_csr(n, rp, ci, v, x, np.full(n, np.nan), 1.0, 0.0),
              lambda: oracle.spmv_coo(n, np.arange(n), ci, v, x, np.full(n, np.nan), 1.0, 0.0)):
        assert np.array_equal(f(), x[pi])                 # beta=0: NaN y_in never read (R12)


def test_diagonal_closed_form():
    n = 64
    rng = np.random.default_rng(3)
    d = rng.standard_normal(n); x = rng.standard_normal(n); y = rng.standard_normal(n)
    rp = np.arange(n + 1, dtype=np.int64); ci = np.arange(n, dtype=np.int32)
    out = oracle.spmv_csr(n, rp, ci, d, x, y, 2.0, 0.25)
    assert np.array_equal(out, 2.0 * (d * x) + 0.25 * y)


def stencil27_csr(N):
    """Independent tiny stencil builder (test-local, dense loops)."""
    rows, cols = [], []
    idx = lambda i, j, k: (i * N + j) * N + k
    for i in range(N):
        for j in range(N):
            for k in range(N):
                for di in (-1, 0, 1):
                    for dj in (-1, 0, 1):
                        for dk in (-1, 0, 1):
                            a, b, c = i + di, j + dj, k + dk
                            if 0 <= a < N and 0 <= b < N and 0 <= c < N:
                                rows.append(idx(i, j, k)); cols.append(idx(a, b, c))
    r = np.array(rows); c = np.array(cols)
    v = np.where(r == c, 26.0, -1.0)
    return r, c, v


@pytest.mark.parametrize("N", [2, 3, 5])
def test_stencil_closed_form(N):
    # diag 26, off -1, x = 1  ->  y_i = 27 - k_i, k_i = prod_d (3 - [face in d])
    r, c, v = stencil27_csr(N)
    m = N ** 3
    assert r.size == (3 * N - 2) ** 3
    rp, ci, vv = oracle.coo_to_csr(m, r, c, v)
    out = oracle.spmv_csr(m, rp, ci, vv, np.ones(m), np.zeros(m), 1.0, 0.0)
    g = np.indices((N, N, N)).reshape(3, -1).T
    k = np.prod(3 - ((g == 0) | (g == N - 1)).astype(int) * (1 if N > 1 else 2), axis=1)
    assert np.array_equal(out, 27.0 - k)
    if N >= 3:
        assert set(np.unique(out).tolist()) == {0.0, 9.0, 15.0, 19.0}


def test_alpha_beta_conventions():
    rp = np.array([0, 1], np.int64); ci = np.array([0], np.int32)
    v = np.array([np.nan]); x = np.array([np.nan])
    # alpha == 0: A and x not read, y = beta*y_in
    assert oracle.spmv_csr(1, rp, ci, v, x, np.array([3.0]), 0.0, 2.0).tolist() == [6.0]
    # beta == 0: y_in not read
    v = np.array([2.0]); x = np.array([5.0])
    assert oracle.spmv_csr(1, rp, ci, v, x, np.array([np.nan]), 1.0, 0.0).tolist() == [10.0]


def dense_of(m, n, r, c, v):
    A = np.zeros((m, n))
    np.add.at(A, (r, c), v.astype(np.float64))
    return A


def random_matrix(rng, m, n, density, empty_rows=True):
    mask = rng.random((m, n)) < density
    if empty_rows and m > 2:
        mask[rng.integers(0, m, max(1, m // 5))] = False
    if empty_rows and n > 2:
        mask[:, rng.integers(0, n, max(1, n // 5))] = False
    r, c = np.nonzero(mask)
    v = rng.uniform(-1, 1, r.size)
    return r, c, v


ALPHAS = [0.0, 1.0, -1.0, 2.5]
BETAS = [0.0, 1.0, -1.0, 10.0]


def test_dense_brute_force_all_formats_and_parts():
    """P3: all formats, m,n <= 64, np in 1..9, alpha x beta grid vs numpy dense."""
    rng = np.random.default_rng(1234)
    for trial in range(40):
        m, n = rng.integers(1, 65, 2)
        r, c, v = random_matrix(rng, m, n, [0.01, 0.1, 0.3][trial % 3])
        A = dense_of(m, n, r, c, v)
        rp, ci, vv = oracle.coo_to_csr(m, r, c, v)
        cp, ri, cv = oracle.csr_to_csc(m, n, rp, ci, vv)
        x = rng.uniform(-1, 1, n); y = rng.uniform(-1, 1, m)
        for alpha, beta in itertools.product(ALPHAS, BETAS):
            ref = alpha * (A @ x) + beta * y
            bound = np.abs(alpha) * (np.abs(A) @ np.abs(x)) + np.abs(beta * y)
            outs = [oracle.spmv_csr(m, rp, ci, vv, x, y, alpha, beta),
                    oracle.spmv_csc(m, n, cp, ri, cv, x, y, alpha, beta),
                    oracle.spmv_coo(m, r, c, v, x, y, alpha, beta)]
            np_ = int(rng.integers(1, 10))
            outs += [oracle.exec_csr(m, rp, ci, vv, x, y, alpha, beta, np_),
                     oracle.exec_csc(m, n, cp, ri, cv, x, y, alpha, beta, np_),
                     oracle.exec_coo(m, r, c, v, x, y, alpha, beta, np_)]
            for o in outs:
                assert np.all(np.abs(o - ref) <= 1e-13 * bound + 1e-300), (trial, alpha, beta)


def test_fp32_accumulates_in_fp64_rounds_once():
    # 2^24 + 1 is not representable in fp32; an fp32 accumulator loses the +1s.
    k = 3
    rp = np.array([0, k + 1], np.int64); ci = np.arange(k + 1, dtype=np.int32)
    v = np.array([2.0 ** 24, 1.0, 1.0, 1.0], np.float32); x = np.ones(k + 1, np.float32)
    out = oracle.spmv_csr(1, rp, ci, v, x, np.zeros(1, np.float32), 1.0, 0.0)
    assert out.dtype == np.float32 and out[0] == np.float32(2.0 ** 24 + 4)


# ------------------------------------------------------------- partitioning
def test_boundaries_worked(golden_E):
    for case in golden_E["boundaries"]:
        assert oracle.nnz_boundaries(case["nnz"], case["np"]).tolist() == case["expect"]


def test_balance_exhaustive():
    """sizes differ by <= 1 and tile [0,nnz) exactly, nnz<=1000, np<=64."""
    for nnz in range(0, 1001, 7):
        for np_ in range(1, 65):
            b = oracle.nnz_boundaries(nnz, np_)
            sz = np.diff(b)
            assert b[0] == 0 and b[-1] == nnz and np.all(sz >= 0)
            assert sz.max() - sz.min() <= 1


def test_owner_worked(golden_E):
    for case in golden_E["owners"]:
        assert oracle.owner_linear(golden_E["csr_row_ptr"], case["idx"]) == case["expect"]


def _check_parts(parts, locs, expect):
    for p, loc, e in zip(parts, locs, expect):
        for k in ("start_idx", "end_idx", "start_row", "end_row", "start_flag"):
            assert int(p[k]) == e[k], (k, p, e)
        if "local" in e:
            assert loc.tolist() == e["local"]


def test_E_pcsr_pcsc_pcoo(golden_E):
    g = golden_E
    parts, locs, _ = oracle.partition_ptr(g["csr_row_ptr"], 2)
    _check_parts(parts, locs, g["pcsr_np2"])
    assert [[int(p["owned_begin"]), int(p["owned_end"])] for p in parts] == g["owned_np2"]
    parts5, _, _ = oracle.partition_ptr(g["csr_row_ptr"], 5)
    assert [[int(p["owned_begin"]), int(p["owned_end"])] for p in parts5] == g["owned_np5"]
    parts, locs, _ = oracle.partition_ptr(g["csc_col_ptr"], 2)
    _check_parts(parts, locs, g["pcsc_np2"])
    pc = oracle.partition_coo(4, g["coo_row"], 2)
    _check_parts(pc, [None, None], g["pcoo_np2"])
    # all-same-row COO: part 1 flagged
    pc = oracle.partition_coo(1, [0, 0, 0, 0], 2)
    assert int(pc[1]["start_flag"]) == 1 and int(pc[0]["start_flag"]) == 0


def test_E_kernel_segment_and_csc_accumulators(golden_E):
    g = golden_E
    rp, ci, v = E_csr(g)
    parts, locs, _ = oracle.partition_ptr(rp, 2)
    p, loc = parts[1], locs[1]
    seg = [sum(v[p["start_idx"] + j] * 1.0 for j in range(loc[k], loc[k + 1])) for k in range(len(loc) - 1)]
    assert seg == g["pcsr_np2_kernel_segment_part1"]
    # CSC np=2 accumulators [1,0,0,4] + [2,3,0,5] summed = [3,3,0,9]
    out = oracle.exec_csc(4, 4, g["csc_col_ptr"], g["csc_row_idx"], np.array(g["csc_val"]),
                          np.ones(4), np.zeros(4), 1.0, 0.0, 2)
    assert out.tolist() == (np.array(g["pcsc_np2_accumulators"]).sum(0)).tolist()


def test_shared_row_beta_once(golden_E):
    """S:306 / S:337: a row split across 2 parts gets beta*y_in once -> [20]."""
    s = golden_E["shared_row_1x4"]
    rp = np.array([0, 4], np.int64); ci = np.arange(4, dtype=np.int32); v = np.array(s["val"], float)
    for f in (lambda: oracle.exec_csr(1, rp, ci, v, s["x"], s["y"], s["alpha"], s["beta"], s["np"]),
              lambda: oracle.exec_coo(1, np.zeros(4), ci, v, s["x"], s["y"], s["alpha"], s["beta"], s["np"])):
        assert f().tolist() == s["expect"]
    parts, locs, _ = oracle.partition_ptr(rp, 2)
    assert [int(p["start_flag"]) for p in parts] == [0, 1]
    # the paper's printed merge (Alg. 3 l.9-17) would give 4.0 here (reading R6): keep it failing
    py = s["part_sums"]; y = s["y"][0]; beta = s["beta"]
    y_alg3 = py[0]
    tmp = y_alg3; y_alg3 = py[1]; y_alg3 -= tmp * beta
    assert y_alg3 == 4.0 and s["expect"][0] != y_alg3


@pytest.mark.parametrize("N,np_", [(1, 8), (13, 8), (64, 7), (5, 9)])
def test_chain_row(N, np_):
    """A 1xN all-ones row split over np parts sums to N (reading R10, chains)."""
    rp = np.array([0, N], np.int64); ci = np.arange(N, dtype=np.int32); v = np.ones(N)
    assert oracle.exec_csr(1, rp, ci, v, np.ones(N), np.zeros(1), 1.0, 0.0, np_).tolist() == [N]
    assert oracle.exec_coo(1, np.zeros(N), ci, v, np.ones(N), np.zeros(1), 1.0, 0.0, np_).tolist() == [N]


def test_partition_invariants_and_roundtrip_exhaustive_3x3():
    """Every structure of a 3x3 matrix, np in 1..nnz+2: descriptors valid, owned ranges tile
    [0,m), aux <= m + 2np, merge(partition) == row_ptr."""
    m = n = 3
    for bits in range(1 << 9):
        mask = np.array([(bits >> k) & 1 for k in range(9)], bool).reshape(3, 3)
        r, c = np.nonzero(mask)
        rp, _, _ = oracle.coo_to_csr(m, r, c, np.ones(r.size))
        nnz = int(rp[-1])
        for np_ in range(1, nnz + 3):
            _check_roundtrip(m, rp, np_)


def test_partition_roundtrip_random_5x5_and_larger():
    rng = np.random.default_rng(5)
    for trial in range(300):
        m = int(rng.integers(1, 6)) if trial < 200 else int(rng.integers(6, 80))
        n = int(rng.integers(1, 6)) if trial < 200 else int(rng.integers(6, 80))
        mask = rng.random((m, n)) < rng.choice([0.1, 0.4, 0.8])
        r, c = np.nonzero(mask)
        rp, _, _ = oracle.coo_to_csr(m, r, c, np.ones(r.size))
        for np_ in range(1, min(int(rp[-1]) + 3, 40)):
            _check_roundtrip(m, rp, np_)


def _check_roundtrip(m, rp, np_):
    parts, locs, flat = oracle.partition_ptr(rp, np_)
    nnz = int(rp[-1])
    assert flat.size <= m + 2 * np_
    # exact tiling of [0,nnz) and balance
    assert parts["start_idx"][0] == 0 and parts["end_idx"][-1] == nnz - 1
    assert np.all(parts["start_idx"][1:] == parts["end_idx"][:-1] + 1)
    # owned ranges tile [0,m) disjointly and each row is owned by the part holding row_ptr[r]
    ob, oe = parts["owned_begin"], parts["owned_end"]
    assert ob[0] == 0 and oe[-1] == m and np.all(ob[1:] == oe[:-1]) and np.all(oe >= ob)
    b = oracle.nnz_boundaries(nnz, np_)
    for r in range(m):
        i = int(np.searchsorted(ob, r, side="right") - 1)
        while oe[i] <= r:
            i += 1
        if rp[r] < nnz:
            assert b[i] <= rp[r] < b[i + 1]
        else:
            assert i == np_ - 1
    for i, p in enumerate(parts):
        if p["start_row"] < 0:
            assert p["start_idx"] == p["end_idx"] + 1 and locs[i].tolist() == [0]
            continue
        assert rp[p["start_row"]] <= p["start_idx"] < rp[p["start_row"] + 1]
        assert rp[p["end_row"]] <= p["end_idx"] < rp[p["end_row"] + 1]
        assert p["start_flag"] == (p["start_idx"] > rp[p["start_row"]])
        loc = locs[i]
        assert loc[0] == 0 and loc[-1] == p["end_idx"] - p["start_idx"] + 1 and np.all(np.diff(loc) >= 0)
    # flag inference: part's last row continues iff the next non-empty part is flagged
    nonempty = [p for p in parts if p["start_row"] >= 0]
    for a, bq in zip(nonempty, nonempty[1:]):
        cont = rp[a["end_row"] + 1] > a["end_idx"] + 1
        assert bool(bq["start_flag"]) == bool(cont)
        if cont:
            assert bq["start_row"] == a["end_row"]
    assert np.array_equal(oracle.merge_parts_to_ptr(m, parts, flat), rp)


def test_coo_partition_matches_csr_partition():
    rng = np.random.default_rng(9)
    for trial in range(100):
        m, n = rng.integers(1, 30, 2)
        r, c, v = random_matrix(rng, m, n, 0.2)
        rp, _, _ = oracle.coo_to_csr(m, r, c, v)
        for np_ in range(1, 12):
            pc = oracle.partition_coo(m, r, np_)
            pr, _, _ = oracle.partition_ptr(rp, np_)
            for k in ("start_idx", "end_idx", "start_row", "end_row", "start_flag", "owned_begin",
                      "owned_end"):
                assert np.array_equal(pc[k], pr[k]), (k, trial, np_)


# ------------------------------------------------ Baseline row/column-block split (NEXT f1)
def test_block_split_fixture_E_hand_worked():
    """Baseline row blocks (Sec. 5.1) of SPEC fixture E (row_ptr [0,2,3,3,5]),
    np = 2 -> rows {0,1} | {2,3}: b = [ptr[0], ptr[2], ptr[4]] = [0, 3, 5].  Part 0 holds
    nonzeros 0..2 of rows 0..1 (no flag) and owns rows [0,2); part 1 holds nonzeros 3..4;
    row 2 is empty, so nonzero 3's strict owner is row 3, no flag, owned rows [2,4)
    (R_1 = lower_bound(ptr, 3) = 2: the empty row goes to the part holding the next nonzero)."""
    ptr = np.array([0, 2, 3, 3, 5])
    b = oracle.block_boundaries(ptr, 2)
    assert b.tolist() == [0, 3, 5]
    p = oracle.partition_ptr_b(ptr, b)
    got = [(int(q["start_idx"]), int(q["end_idx"]), int(q["start_row"]), int(q["end_row"]), int(q["start_flag"]),
            int(q["owned_begin"]), int(q["owned_end"])) for q in p]
    assert got == [(0, 2, 0, 1, 0, 0, 2), (3, 4, 3, 3, 0, 2, 4)]


def test_block_split_equals_nnz_split_on_uniform_rows():
    """Closed form: with exactly k nonzeros per row and np | m, row blocks and the nnz split cut
    at the same places (b_i = i*k*m/np), so Alg. 2 yields identical descriptors."""
    for m, k, np_ in [(8, 3, 4), (60, 7, 6), (64, 1, 8)]:
        ptr = np.arange(m + 1, dtype=np.int64) * k
        bb, bn = oracle.block_boundaries(ptr, np_), oracle.nnz_boundaries(m * k, np_)
        assert np.array_equal(bb, bn)
        assert np.array_equal(oracle.partition_ptr_b(ptr, bb), oracle.partition_ptr(ptr, np_)[0])


def test_block_split_whole_rows_no_flags_random():
    """Brute force: part i of the row-block split holds exactly the nonzeros of rows
    [floor(i*m/np), floor((i+1)*m/np)), never shares a row (start_flag = 0), and the COO
    form (counted by scanning row ids) gives the same descriptors."""
    rng = np.random.default_rng(31)
    for _ in range(200):
        m = int(rng.integers(1, 40)); np_ = int(rng.integers(1, 12))
        ptr = np.concatenate([[0], np.cumsum(rng.integers(0, 6, m))]).astype(np.int64)
        b = oracle.block_boundaries(ptr, np_)
        for i in range(np_):
            r0, r1 = i * m // np_, (i + 1) * m // np_
            assert b[i] == ptr[r0] and b[i + 1] == ptr[r1]
        parts = oracle.partition_ptr_b(ptr, b)
        assert (parts["start_flag"] == 0).all()
        rows = oracle.csr_to_coo(m, ptr)
        bc = oracle.block_boundaries_coo(m, rows, np_)
        assert np.array_equal(bc, b)
        pc = oracle.partition_coo_b(m, rows, bc)
        for k in ("start_idx", "end_idx", "start_row", "end_row", "start_flag", "owned_begin", "owned_end"):
            assert np.array_equal(pc[k], parts[k]), k


def test_relative_throughput_fig6_two_class():
    """Fig. 6: 4 of 8 GPUs hold 1/10 of the nonzeros of the other 4 ->
    throughput 'about half (559/1028)'.  The cost model's closed form:
    (4h + 4h/10)/8 / h = 0.55, within 0.01 of the paper's 559/1028 = 0.5438."""
    h = 1000
    sizes = [h] * 4 + [h // 10] * 4
    b = np.concatenate([[0], np.cumsum(sizes)])
    r = oracle.relative_throughput(b)
    assert r == pytest.approx(0.55, abs=1e-12)
    assert abs(r - 559 / 1028) < 0.01
    assert oracle.relative_throughput(oracle.nnz_boundaries(int(b[-1]), 8)) > 0.99
    assert oracle.relative_throughput(np.array([0, 5, 10])) == 1.0


# ------------------------------------------------------------ CG (NEXT f4)
def _spd_stencil(N, diag=30.0):
    """27-point stencil pattern with diagonal `diag`, off-diagonals -1: symmetric and strictly
    diagonally dominant (26 < diag), hence SPD."""
    import gen
    A = gen.stencil27(N, kind=gen.ONES)
    rows = np.repeat(np.arange(A["m"]), np.diff(A["ptr"]))
    A["val"] = np.where(A["idx"] == rows, diag, -1.0)
    return A


def test_cg_identity_one_iteration():
    """A = I: r0 = b, alpha = 1, x1 = b exactly, so CG stops after one iteration."""
    m = 7
    b = np.arange(1.0, m + 1)
    x, it, rr = oracle.cg_csr(m, np.arange(m + 1), np.arange(m, dtype=np.int32), np.ones(m), b, np.zeros(m), 1e-14, 50)
    assert it == 1 and rr == 0.0 and np.array_equal(x, b)


def test_cg_k_distinct_eigenvalues():
    """Textbook property: on an SPD matrix with k distinct eigenvalues CG terminates in at most
    k iterations (in exact arithmetic; here the residual after k steps is at rounding level)."""
    d = np.repeat([1.0, 3.0, 7.0, 10.0], 25)           # k = 4 distinct eigenvalues
    m = d.size
    b = np.linspace(-1, 1, m) + 0.3
    x, it, rr = oracle.cg_csr(m, np.arange(m + 1), np.arange(m, dtype=np.int32), d, b, np.zeros(m), 1e-12, 4)
    assert it <= 4 and rr < 1e-12
    assert np.allclose(x, b / d, rtol=1e-12)


def test_cg_1d_laplacian_n_steps_and_solution():
    """tridiag(-1, 2, -1) of size n (SPD, n distinct eigenvalues): CG reaches the exact solution
    (x* = 1..n, b = A x*) within n iterations, to rounding level."""
    n = 40
    rows, cols, vals = [], [], []
    for i in range(n):
        for j, v in ((i - 1, -1.0), (i, 2.0), (i + 1, -1.0)):
            if 0 <= j < n:
                rows.append(i); cols.append(j); vals.append(v)
    ptr, idx, val = oracle.coo_to_csr(n, np.array(rows), np.array(cols), np.array(vals))
    xs = np.arange(1.0, n + 1)
    b = oracle.spmv_csr(n, ptr, idx, val, xs, np.zeros(n), 1.0, 0.0)
    x, it, rr = oracle.cg_csr(n, ptr, idx, val, b, np.zeros(n), 1e-13, n)
    assert it <= n and rr < 1e-12
    assert np.allclose(x, xs, rtol=1e-10)


def test_cg_spd_stencil_recovers_known_solution():
    """SPD 27-point stencil (diag 30): b = A x* with integer x*, CG from 0 converges to x*."""
    A = _spd_stencil(6)
    m = A["m"]
    xs = (np.arange(m) % 7 - 3).astype(np.float64)
    b = oracle.spmv_csr(m, A["ptr"], A["idx"], A["val"], xs, np.zeros(m), 1.0, 0.0)
    x, it, rr = oracle.cg_csr(m, A["ptr"], A["idx"], A["val"], b, np.zeros(m), 1e-12, 500)
    assert rr <= 1e-12 and 0 < it < 60
    assert np.max(np.abs(x - xs)) < 1e-10


# --------------------------------------------- two-level NUMA split (NEXT f3)
def test_two_level_spec_examples():
    """nnz=12 on groups [3,3] (Summit node) and nnz=16 on [4,4] (DGX-1): 2 per part."""
    assert oracle.two_level_boundaries(12, [3, 3]).tolist() == list(range(0, 13, 2))
    assert oracle.two_level_boundaries(16, [4, 4]).tolist() == list(range(0, 17, 2))
    assert oracle.two_level_boundaries(7, [1]).tolist() == [0, 7]


def test_two_level_differs_from_single_level_counterexample():
    """S:231 claims the composition equals the single-level split; it does not.
    nnz=2 on [1,3]: level 1 gives the groups [0,0) and [0,2); level 2 cuts [0,2) in 3 ->
    [0,0,0,1,2], while floor(i*2/4) = [0,0,1,1,2]."""
    assert oracle.two_level_boundaries(2, [1, 3]).tolist() == [0, 0, 0, 1, 2]
    assert oracle.nnz_boundaries(2, 4).tolist() == [0, 0, 1, 1, 2]


def test_two_level_balance_and_coincidence():
    """Within a group parts differ by <= 1 nonzero; across the whole plan by <= 2; and with
    equal groups whose part count divides nnz the two levels reproduce the single-level cut."""
    rng = np.random.default_rng(41)
    for _ in range(300):
        sizes = rng.integers(1, 5, int(rng.integers(1, 5)))
        nnz = int(rng.integers(0, 200))
        b = oracle.two_level_boundaries(nnz, sizes)
        d = np.diff(b)
        assert b[0] == 0 and b[-1] == nnz and (d >= 0).all()
        assert d.max() - d.min() <= 2
        w = 0
        for s in sizes:
            assert d[w:w + s].max() - d[w:w + s].min() <= 1
            w += s
    for g, per in ((2, 4), (3, 2), (2, 3)):
        nnz = g * per * 7
        assert np.array_equal(oracle.two_level_boundaries(nnz, [per] * g), oracle.nnz_boundaries(nnz, g * per))


# ------------------------------------------------------------ tolerance scale (oracle item 6)
def test_row_bound_worked_E(golden_E):
    """or_row_bound_csr on fixture E with sign-mixed x, negative alpha/beta:
    hand-worked values (tests/golden/row_bound_E.json).  A dropped fabs, a missing |alpha|, a signed
    beta term or a beta term read when beta == 0 each changes one of them."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "row_bound_E.json")) as f:
        G = json.load(f)
    rp, ci, v = E_csr(golden_E)
    x = np.array(G["x"], np.float64)
    for case in G["cases"]:
        y = np.array([float(t) for t in case["y"]], np.float64)
        got = oracle.row_bound_csr(4, rp, ci, v, x, y, case["alpha"], case["beta"])
        assert got.tolist() == case["expect"], case


def test_row_bound_dense_brute_force():
    """bound = |alpha| * (|A| @ |x|) + |beta * y| against numpy dense brute force, m, n <= 64 (P3 style).
    Small-integer data: every partial sum is exact, so the comparison is bit-for-bit; U[-1,1) data
    within 1e-14 relative."""
    rng = np.random.default_rng(4242)
    for trial in range(60):
        m, n = (int(t) for t in rng.integers(1, 65, 2))
        r, c, _ = random_matrix(rng, m, n, [0.02, 0.2, 0.6][trial % 3])
        ints = trial % 2 == 0
        v = rng.integers(-4, 5, r.size).astype(np.float64) if ints else rng.uniform(-1, 1, r.size)
        x = rng.integers(-4, 5, n).astype(np.float64) if ints else rng.uniform(-1, 1, n)
        y = rng.integers(-4, 5, m).astype(np.float64) if ints else rng.uniform(-1, 1, m)
        A = dense_of(m, n, r, c, v)
        rp, ci, vv = oracle.coo_to_csr(m, r, c, v)
        for alpha, beta in [(1.0, 0.0), (-2.0, 0.5), (0.5, -3.0), (0.0, 2.0), (-1.5, -1.0)]:
            ref = abs(alpha) * (np.abs(A) @ np.abs(x)) + (np.abs(beta * y) if beta != 0.0 else 0.0)
            got = oracle.row_bound_csr(m, rp, ci, vv, x, y, alpha, beta)
            if ints:
                assert np.array_equal(got, ref), (trial, alpha, beta)
            else:
                assert np.allclose(got, ref, rtol=1e-14, atol=0.0), (trial, alpha, beta)
            assert np.all(got >= 0.0)


def test_row_bound_fp32_reads_fp32_values():
    """fp32 data: the bound is taken over the stored fp32 values (converted exactly to fp64)."""
    rng = np.random.default_rng(7)
    m, n = 30, 40
    r, c, v = random_matrix(rng, m, n, 0.3)
    v32 = v.astype(np.float32)
    x32 = rng.uniform(-1, 1, n).astype(np.float32)
    y32 = rng.uniform(-1, 1, m).astype(np.float32)
    rp, ci, vv = oracle.coo_to_csr(m, r, c, v32)
    got = oracle.row_bound_csr(m, rp, ci, vv, x32, y32, 1.5, -0.5)
    A = dense_of(m, n, r, c, v32.astype(np.float64))
    ref = 1.5 * (np.abs(A) @ np.abs(x32.astype(np.float64))) + np.abs(-0.5 * y32.astype(np.float64))
    assert np.allclose(got, ref, rtol=1e-14, atol=0.0)


def all_row_pointers(max_m=5, max_len=5):
    """Every row-pointer array of an m x n matrix with m, n <= 5 (the partition depends only on
    row_ptr, so every row-length vector in {0..5}^m, m = 1..5, covers every structure)."""
    for m in range(1, max_m + 1):
        for lens in itertools.product(range(max_len + 1), repeat=m):
            rp = np.zeros(m + 1, np.int64)
            rp[1:] = np.cumsum(lens)
            yield m, rp


def test_partition_roundtrip_exhaustive_5x5():
    """S:253 / S:549: merge(partition) == id and every descriptor invariant, EXHAUSTIVE over all
    row-length vectors with m, n <= 5 (9330 pointer arrays) and np in 1..nnz+2."""
    count = 0
    for m, rp in all_row_pointers():
        for np_ in range(1, int(rp[-1]) + 3):
            _check_roundtrip(m, rp, np_)
            count += 1
    assert count == sum(6 ** m * (2.5 * m + 2) for m in range(1, 6)) == 130635   # sum of (nnz + 2)


# ------------------------------------------------------------ unsorted pCOO
def test_unsorted_coo_fixture_E_hand_worked():
    """Fixture E's triplets in the order (3,3,5) (0,2,2) (1,1,3) (0,0,1) (3,0,4), np = 2: the nnz
    split by position gives parts {0,1} and {2,3,4}; both touch rows 0..3 (reading R25: smallest and
    largest row, no flag, no owned rows).  Partial vectors (x = 1): part 0 -> [2,0,0,5], part 1 ->
    [1,3,0,4]; their sum is the plain SpMV [3,3,0,9] (worked by hand from S:96)."""
    r = np.array([3, 0, 1, 0, 3]); c = np.array([3, 2, 1, 0, 0], np.int32); v = np.array([5.0, 2, 3, 1, 4])
    parts = oracle.partition_coo_unsorted(r, 2)
    assert parts["start_idx"].tolist() == [0, 2] and parts["end_idx"].tolist() == [1, 4]
    assert parts["start_row"].tolist() == [0, 0] and parts["end_row"].tolist() == [3, 3]
    assert parts["start_flag"].tolist() == [0, 0] and parts["owned_end"].tolist() == [0, 0]
    assert oracle.exec_coo_unsorted(4, r, c, v, np.ones(4), np.zeros(4), 1.0, 0.0, 2).tolist() == [3, 3, 0, 9]
    # part 0 alone (its two triplets) is the partial vector [2, 0, 0, 5]
    assert oracle.exec_coo_unsorted(4, r[:2], c[:2], v[:2], np.ones(4), np.zeros(4), 1.0, 0.0, 1).tolist() == [2, 0, 0, 5]
    # beta applied once: alpha 2, beta 10, y 1 -> [16, 16, 10, 28]
    assert oracle.exec_coo_unsorted(4, r, c, v, np.ones(4), np.ones(4), 2.0, 10.0, 5).tolist() == [16, 16, 10, 28]


def test_unsorted_coo_partition_brute_force():
    """Descriptors = positions b_i = floor(i*nnz/np) and the min / max row of each slice (numpy);
    empty parts have rows -1."""
    rng = np.random.default_rng(44)
    for trial in range(200):
        nnz = int(rng.integers(0, 60))
        r = rng.integers(0, 30, nnz)
        np_ = int(rng.integers(1, nnz + 4))
        parts = oracle.partition_coo_unsorted(r, np_)
        b = [(i * nnz) // np_ for i in range(np_ + 1)]
        for i, p in enumerate(parts):
            assert p["start_idx"] == b[i] and p["end_idx"] == b[i + 1] - 1
            sl = r[b[i]:b[i + 1]]
            assert (p["start_row"], p["end_row"]) == ((sl.min(), sl.max()) if sl.size else (-1, -1))
            assert p["start_flag"] == 0 and p["owned_begin"] == 0 and p["owned_end"] == 0


def test_unsorted_coo_exec_permutation_invariant_and_dense():
    """Any triplet order, any np: the unsorted executor equals the sorted-COO SpMV bit for bit on
    small-integer data (every sum exact) and the numpy dense product within tau on U[-1,1)."""
    rng = np.random.default_rng(45)
    for trial in range(40):
        m, n = (int(t) for t in rng.integers(1, 65, 2))
        r, c, _ = random_matrix(rng, m, n, [0.02, 0.2, 0.5][trial % 3])
        ints = trial % 2 == 0
        v = rng.integers(-4, 5, r.size).astype(np.float64) if ints else rng.uniform(-1, 1, r.size)
        x = rng.integers(-4, 5, n).astype(np.float64) if ints else rng.uniform(-1, 1, n)
        y = rng.integers(-4, 5, m).astype(np.float64) if ints else rng.uniform(-1, 1, m)
        perm = rng.permutation(r.size)
        ru, cu, vu = r[perm], c[perm].astype(np.int32), v[perm]
        A = dense_of(m, n, r, c, v)
        for alpha, beta in [(1.0, 0.0), (2.0, 0.5), (-1.0, 1.0), (0.0, 2.0)]:
            ref = oracle.spmv_coo(m, r, c, v, x, y, alpha, beta)
            np_ = int(rng.integers(1, 10))
            got = oracle.exec_coo_unsorted(m, ru, cu, vu, x, y, alpha, beta, np_)
            if ints:
                assert np.array_equal(got, ref), (trial, alpha, beta, np_)
            bound = abs(alpha) * (np.abs(A) @ np.abs(x)) + np.abs(beta * y)
            assert np.all(np.abs(got - (alpha * (A @ x) + beta * y)) <= 1e-13 * bound + 1e-300)
