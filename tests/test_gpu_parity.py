"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Integer-valued inputs (small integers, dyadic alpha/beta) make every summation
order exact, so those cases are compared BIT-FOR-BIT (SURVEY 8(c) pin P5);
U[-1,1) inputs are compared per row within tau * bound (fp64 1e-12, fp32 1e-5).
"""
import itertools

import numpy as np
import pytest

import gen
import oracle
from tests.helpers import (apply_layout, assert_close, coo_of_csr, oracle_ref, row_bound, run_gpu, split_fmt,
                           to_dtype)

pytestmark = pytest.mark.gpu

# coo_col: column-sorted pCOO (merged like pCSC).  The column formats run on row tiles
# over the GPU-transposed slice by default; ":bands" selects the host-built row-band layout.
FMTS = ["csr", "coo", "csc", "coo_col", "csc:bands", "coo_col:bands"]


def as_fmt(A, fmt):
    fmt = split_fmt(fmt)[0]
    if fmt in ("csc", "coo_col"):
        return A if A["fmt"] == "csc" else gen.transpose(A)
    return A if A["fmt"] == "csr" else gen.transpose(A)


def sparse_from_dense_mask(mask, vals):
    r, c = np.nonzero(mask)
    m, n = mask.shape
    rp, ci, v = oracle.coo_to_csr(m, r, c, vals[r, c])
    return gen.Sparse(fmt="csr", m=m, n=n, ptr=rp, idx=ci, val=v)


def check(A, fmt, x, y, alpha, beta, parts=1, exact=False, **kw):
    B = as_fmt(A, fmt)
    got = run_gpu(B, fmt, x, y, alpha, beta, parts=parts, **kw)
    ref = oracle_ref(A, x, y, alpha, beta)
    if exact:
        assert got.dtype == ref.dtype
        assert np.array_equal(got, ref), (fmt, parts, np.nonzero(got != ref)[0][:10])
    else:
        assert_close(got, ref, row_bound(A, x, y, alpha, beta), A["val"].dtype)
    return got


# ------------------------------------------------------------ worked values
@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("parts", [1, 2, 3, 5, 7])
def test_fixture_E(golden_E, fmt, parts):
    g = golden_E
    A = gen.Sparse(fmt="csr", m=4, n=4, ptr=np.array(g["csr_row_ptr"], np.int64),
                   idx=np.array(g["csr_col_idx"], np.int32), val=np.array(g["csr_val"]))
    for case in g["spmv"]:
        got = run_gpu(as_fmt(A, fmt), fmt, np.array(case["x"], float), np.array(case["y"], float),
                      case["alpha"], case["beta"], parts=parts)
        assert got.tolist() == case["expect"]


@pytest.mark.parametrize("fmt", ["csr", "coo"])
def test_shared_row_beta_once(golden_E, fmt):
    s = golden_E["shared_row_1x4"]
    A = gen.Sparse(fmt="csr", m=1, n=4, ptr=np.array([0, 4], np.int64), idx=np.arange(4, dtype=np.int32),
                   val=np.array(s["val"], float))
    got = run_gpu(A, fmt, np.array(s["x"], float), np.array(s["y"], float), s["alpha"], s["beta"], parts=2)
    assert got.tolist() == s["expect"]


# ----------------------------------------------------------- closed forms
@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("n,parts", [(1, 1), (13, 8), (5000, 8), (2047, 3), (2048, 1), (100_000, 9)])
def test_chain_row_all_ones(fmt, n, parts):
    A = gen.Sparse(fmt="csr", m=1, n=n, ptr=np.array([0, n], np.int64), idx=np.arange(n, dtype=np.int32),
                   val=np.ones(n))
    got = run_gpu(as_fmt(A, fmt), fmt, np.ones(n), np.zeros(1), 1.0, 0.0, parts=parts)
    assert got.tolist() == [float(n)]


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("parts", [1, 4])
def test_stencil_closed_form(fmt, parts):
    N = 23
    A = gen.stencil27(N, kind=gen.STENCIL_PIN)
    got = run_gpu(as_fmt(A, fmt), fmt, np.ones(A["m"]), np.zeros(A["m"]), 1.0, 0.0, parts=parts)
    gi = np.indices((N, N, N)).reshape(3, -1).T
    k = np.prod(3 - ((gi == 0) | (gi == N - 1)).astype(int), axis=1)
    assert np.array_equal(got, 27.0 - k)


@pytest.mark.parametrize("fmt", FMTS)
def test_permutation_and_identity_bit_exact(fmt):
    n = 70_001
    rng = np.random.default_rng(7)
    pi = rng.permutation(n)
    A = gen.Sparse(fmt="csr", m=n, n=n, ptr=np.arange(n + 1, dtype=np.int64), idx=pi.astype(np.int32),
                   val=np.ones(n))
    x = rng.standard_normal(n)
    got = run_gpu(as_fmt(A, fmt), fmt, x, np.full(n, np.nan), 1.0, 0.0, parts=3)
    assert np.array_equal(got, x[pi])


# -------------------------------------------------- random, brute-force-ish
@pytest.mark.parametrize("fmt", FMTS)
def test_random_small_all_alpha_beta(fmt):
    rng = np.random.default_rng(100 + FMTS.index(fmt))
    for trial in range(12):
        m, n = (int(v) for v in rng.integers(1, 300, 2))
        mask = rng.random((m, n)) < [0.01, 0.1, 0.3][trial % 3]
        if m > 3:
            mask[rng.integers(0, m, m // 4)] = False
        vals = rng.integers(-4, 5, (m, n)).astype(float)
        vals[vals == 0] = 1.0
        A = sparse_from_dense_mask(mask, vals)
        x = rng.integers(-4, 5, n).astype(float); y = rng.integers(-4, 5, m).astype(float)
        for alpha, beta in itertools.product([0.0, 1.0, -1.0, 2.5], [0.0, 1.0, -1.0, 10.0]):
            parts = int(rng.integers(1, 10))
            check(A, fmt, x, y, alpha, beta, parts=parts, exact=True)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("fmt", FMTS)
def test_random_uniform_tolerance(fmt, dtype):
    rng = np.random.default_rng(5)
    for trial in range(6):
        m, n = (int(v) for v in rng.integers(100, 3000, 2))
        A = to_dtype(gen.kdistinct_csr(m, n, int(rng.integers(1, 60)), seed=trial + 10), dtype)
        x = gen.vector(n, 20 + trial, dtype=dtype); y = gen.vector(m, 40 + trial, dtype=dtype)
        check(A, fmt, x, y, 1.5, 0.5, parts=int(rng.integers(1, 9)))


@pytest.mark.parametrize("fmt", FMTS)
def test_long_and_empty_rows_mix(fmt):
    """Rows longer than a tile (slab-split), runs of empty rows, and part cuts inside long rows."""
    rng = np.random.default_rng(3)
    lens = np.concatenate([[0, 0, 9000, 1, 0, 2048, 2047, 2046, 0, 0, 0], rng.integers(0, 5, 3000),
                           [30000], np.zeros(5000, int), [4097, 3]])
    m, n = lens.size, 40000
    ptr = np.zeros(m + 1, np.int64); ptr[1:] = np.cumsum(lens)
    idx = np.concatenate([np.sort(rng.choice(n, L, replace=False)) for L in lens]).astype(np.int32)
    val = rng.integers(-4, 5, idx.size).astype(float)
    A = gen.Sparse(fmt="csr", m=m, n=n, ptr=ptr, idx=idx, val=val)
    x = rng.integers(-4, 5, n).astype(float); y = rng.integers(-4, 5, m).astype(float)
    for parts in [1, 2, 3, 8, 17]:
        check(A, fmt, x, y, 2.0, -1.0, parts=parts, exact=True)


# --------------------------------------------------------------- edge cases
@pytest.mark.parametrize("fmt", FMTS)
def test_empty_matrix_and_tiny(fmt):
    A = gen.Sparse(fmt="csr", m=5, n=3, ptr=np.zeros(6, np.int64), idx=np.zeros(0, np.int32), val=np.zeros(0))
    y = np.arange(5, dtype=float)
    for parts in [1, 4]:
        got = run_gpu(as_fmt(A, fmt), fmt, np.ones(3), y, 1.0, 2.0, parts=parts)
        assert got.tolist() == (2 * y).tolist()
    # nnz < np: empty parts
    A = gen.Sparse(fmt="csr", m=3, n=3, ptr=np.array([0, 1, 1, 2], np.int64), idx=np.array([2, 0], np.int32),
                   val=np.array([3.0, 4.0]))
    got = run_gpu(as_fmt(A, fmt), fmt, np.array([1.0, 2.0, 5.0]), np.ones(3), 1.0, 1.0, parts=7)
    assert got.tolist() == [16.0, 1.0, 5.0]


@pytest.mark.parametrize("fmt", FMTS)
def test_alpha_zero_beta_zero_do_not_read(fmt):
    A = gen.kdistinct_csr(500, 400, 7, seed=9, kind=gen.SMALLINT)
    x = np.full(400, np.nan)
    y = gen.vector(500, 3)
    got = run_gpu(as_fmt(A, fmt), fmt, x, y, 0.0, 3.0, parts=2)
    assert np.array_equal(got, 3.0 * y)
    x = gen.vector(400, 4, kind=gen.SMALLINT)
    got = run_gpu(as_fmt(A, fmt), fmt, x, np.full(500, np.nan), 1.0, 0.0, parts=2)
    assert np.array_equal(got, oracle_ref(A, x, np.zeros(500), 1.0, 0.0))


def test_unsorted_coo_rejected():
    import paper_2209_07552_b200 as M
    ctx = M.Context()
    with pytest.raises(M.MsrepError) as e:
        ctx.partition("coo", 3, 3, idx=np.array([0, 1, 2], np.int32), val=np.ones(3),
                      coo_row=np.array([0, 2, 1], np.int32))
    assert e.value.status == 3
    with pytest.raises(M.MsrepError) as e:
        ctx.spmv(1.0, 0, 0.0, 0)
    assert e.value.status == 5
    ctx.close()


@pytest.mark.parametrize("fmt", FMTS)
def test_deterministic_and_layout_invariant(fmt):
    A = gen.rmat(14, seed=11)
    x = gen.vector(A["n"], 1); y = gen.vector(A["m"], 2)
    B = as_fmt(A, fmt)
    outs = run_gpu(B, fmt, x, y, 1.5, 0.5, parts=4, repeat=3)
    # no float atomics anywhere (pCSC split bands are reduced over their slots in slot order):
    # every format is bit-reproducible run to run
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    assert_close(outs[0], oracle_ref(A, x, y, 1.5, 0.5), row_bound(A, x, y, 1.5, 0.5), np.float64)


@pytest.mark.parametrize("fmt", FMTS)
def test_host_vector_path_matches_device(fmt):
    A = gen.rmat(13, seed=12, kind=gen.SMALLINT)
    x = gen.vector(A["n"], 1, kind=gen.SMALLINT); y = gen.vector(A["m"], 2, kind=gen.SMALLINT)
    B = as_fmt(A, fmt)
    a = run_gpu(B, fmt, x, y, 2.0, 0.5, parts=3)
    b = run_gpu(B, fmt, x, y, 2.0, 0.5, parts=3, host_path=True)
    assert np.array_equal(a, b)
    assert np.array_equal(a, oracle_ref(A, x, y, 2.0, 0.5))


@pytest.mark.parametrize("fmt", ["csr", "coo", "csc", "coo_col"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_host_vector_pipelined_chunks(fmt, dtype):
    """msrep_spmv_host at one rank and one part runs pipelined: x up whole, y_in up in row chunks,
    chunk k's tiles and split-row fix-up as soon as its y_in is there, its y rows down while later
    chunks go up and compute.  Bit-exact vs the device path and the oracle, for beta != 0 and
    beta == 0 (no y_in copy), every layout the format takes, pageable numpy and pinned torch host
    vectors, with heavy split rows (R-MAT) and with the hot-x cache and compact x (scale 17); the
    result must not depend on what y_host held for beta == 0."""
    import paper_2209_07552_b200 as M
    import torch
    for scale in (13, 17):
        A = to_dtype(gen.rmat(scale, seed=12 + scale, kind=gen.SMALLINT), dtype)
        x = gen.vector(A["n"], 1, kind=gen.SMALLINT).astype(dtype); y = gen.vector(A["m"], 2, kind=gen.SMALLINT).astype(dtype)
        B = as_fmt(A, fmt)
        lays = [M.Y_REPLICATED, M.Y_SHARDED] if fmt in ("csc", "coo_col") else [M.Y_REPLICATED, M.Y_OWNED]
        for beta in (0.5, 0.0):
            ref = oracle_ref(A, x, y, 2.0, beta)
            dev = run_gpu(B, fmt, x, y, 2.0, beta, parts=1)
            assert np.array_equal(dev, ref), (scale, beta)
            for lay in lays:
                for pinned in (False, True):
                    ctx = M.Context(0, 1, None, 0, 1)
                    apply_layout(ctx, fmt)
                    if scale == 17:   # hot-x cache and degree-ordered compact x forced on (x is small here)
                        ctx.set_tuning("hot_x", 1)
                        ctx.set_tuning("compact_x", 2)
                    if fmt in ("coo", "coo_col"):
                        ctx.partition(fmt, B["m"], B["n"], idx=B["idx"], val=B["val"], coo_row=coo_of_csr(B))
                    else:
                        ctx.partition(fmt, B["m"], B["n"], ptr=B["ptr"], idx=B["idx"], val=B["val"])
                    y0 = y.copy() if beta != 0.0 else np.full_like(y, np.nan)
                    if pinned:
                        xh = torch.as_tensor(x).pin_memory(); yh = torch.as_tensor(y0).pin_memory()
                        for _ in range(2):   # twice: the second call reuses the chunking and events
                            yh.copy_(torch.as_tensor(y0))
                            ctx.spmv_host(2.0, xh.data_ptr(), beta, yh.data_ptr(), lay)
                        got = yh.numpy()
                    else:
                        got = y0.copy()
                        ctx.spmv_host(2.0, x, beta, got, lay)
                    st = ctx.stats()
                    ctx.close()
                    assert np.array_equal(got, ref), (scale, beta, lay, pinned)
                    if scale == 17 and fmt == "csr" and dtype == np.float64:
                        assert st["nhot"] > 0 and st["x_compact"] > 0, st


@pytest.mark.parametrize("fmt", ["csr", "csc"])
def test_torch_allocator_hook(fmt):
    """msrep_create's allocator hook (Context(allocator="torch"), the binding's default): every device
    buffer of the partition comes from torch's caching allocator and goes back to it on close;
    results are the same bits as with the library's own cudaMalloc (allocator=None).
    Re-partitioning the same context frees the old layout through the hook."""
    import paper_2209_07552_b200 as M
    import torch
    A = gen.rmat(14, seed=21, kind=gen.SMALLINT)
    B = as_fmt(A, fmt)
    x = gen.vector(A["n"], 22, kind=gen.SMALLINT); y = gen.vector(A["m"], 23, kind=gen.SMALLINT)
    ref = oracle_ref(A, x, y, 1.5, 0.5)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated(0)
    ctx = M.Context(0, 1, None, 0, 2, allocator="torch")
    for _ in range(2):   # the second partition releases the first layout through the hook
        got = run_gpu(B, fmt, x, y, 1.5, 0.5, ctx=ctx)
        assert np.array_equal(got, ref)
        held = torch.cuda.memory_allocated(0) - base
        st = ctx.stats()
        assert held >= st["device_bytes"] > 0, (held, st["device_bytes"])
    ctx.close()
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated(0) - base < st["device_bytes"]   # the layout went back to torch's pool
    # allocator=None: the library's own cudaMalloc / cudaFree, same bits, nothing from torch's pool
    ctx = M.Context(0, 1, None, 0, 2, allocator=None)
    got = run_gpu(B, fmt, x, y, 1.5, 0.5, ctx=ctx)
    assert np.array_equal(got, ref)
    assert torch.cuda.memory_allocated(0) - base < ctx.stats()["device_bytes"]
    ctx.close()


def test_host_vector_pipeline_then_host_resident():
    """One context: a device-resident partition used through the pipelined host-vector path, then
    re-partitioned host-resident (streamed per call on the copy stream) and back -- the two modes
    keep their streams and events apart; every result bit-exact."""
    import paper_2209_07552_b200 as M
    import torch
    A = gen.rmat(13, seed=33, kind=gen.SMALLINT)
    x = gen.vector(A["n"], 34, kind=gen.SMALLINT); y = gen.vector(A["m"], 35, kind=gen.SMALLINT)
    ref = oracle_ref(A, x, y, 1.5, 0.5)
    ctx = M.Context(0, 1, None, 0, 1)
    for res in ("device", "host", "device", "host"):
        kw = {"residency": res, "chunk_bytes": 64 << 10} if res == "host" else {}
        ctx.partition("csr", A["m"], A["n"], ptr=A["ptr"], idx=A["idx"], val=A["val"], **kw)
        yh = y.copy()
        ctx.spmv_host(1.5, x, 0.5, yh)
        assert np.array_equal(yh, ref), ("host path", res)
        yd = torch.as_tensor(y.copy()).cuda()
        ctx.spmv(1.5, torch.as_tensor(x).cuda(), 0.5, yd)
        torch.cuda.synchronize()
        assert np.array_equal(yd.cpu().numpy(), ref), ("device path", res)
    ctx.close()


def test_owned_layout_writes_only_owned_rows():
    import paper_2209_07552_b200 as M
    A = gen.rmat(12, seed=5, kind=gen.SMALLINT)
    x = gen.vector(A["n"], 1, kind=gen.SMALLINT)
    y = np.full(A["m"], 7.0)
    got = run_gpu(A, "csr", x, y, 1.0, 1.0, parts=5, layout=M.Y_OWNED)
    assert np.array_equal(got, oracle_ref(A, x, y, 1.0, 1.0))   # single rank owns every row


# ------------------------------------------------- configs (BASELINE.json)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_config1_random1k(dtype):
    A = to_dtype(gen.make_config("random1k"), dtype)
    assert A.nnz == 10_000
    x = gen.vector(1000, 1, dtype=dtype); y = gen.vector(1000, 2, dtype=dtype)
    for fmt in FMTS:
        check(A, fmt, x, y, 1.5, 0.5)


@pytest.mark.slow
@pytest.mark.parametrize("fmt", ["csr", "coo"])
def test_config2_stencil_full_size(fmt):
    """Full N=127 stencil at the bench launch configuration: closed form + bit-exact integer parity."""
    A = gen.stencil27(127, kind=gen.STENCIL_PIN)
    m = A["m"]
    got = run_gpu(A, fmt, np.ones(m), np.zeros(m), 1.0, 0.0)
    assert set(np.unique(got).tolist()) == {0.0, 9.0, 15.0, 19.0}
    assert int((got == 0).sum()) == 125 ** 3
    A = gen.stencil27(127, kind=gen.SMALLINT)
    x = gen.vector(m, 5, kind=gen.SMALLINT); y = gen.vector(m, 6, kind=gen.SMALLINT)
    check(A, fmt, x, y, 1.5, 0.5, exact=True)
    A = gen.stencil27(127)
    x = gen.vector(m, 5); y = gen.vector(m, 6)
    check(A, fmt, x, y, 1.5, 0.5)


@pytest.mark.slow
@pytest.mark.parametrize("fmt", ["csr", "coo"])
def test_config3_rmat_full_size_bit_exact(fmt):
    A = gen.rmat(24, seed=3, kind=gen.SMALLINT)
    x = gen.vector(A["n"], 7, kind=gen.SMALLINT); y = gen.vector(A["m"], 8, kind=gen.SMALLINT)
    check(A, fmt, x, y, 2.0, 0.5, exact=True)


@pytest.mark.slow
@pytest.mark.parametrize("fmt", ["csr", "coo", "csc"])
def test_config2_stencil_full_size_fp32_bit_exact(fmt):
    """fp32 storage at full size, small-integer data (|y| < 2^24): fp64 accumulation makes every
    order exact, so the fp32 result equals the oracle bit for bit (pin P5)."""
    A = to_dtype(gen.stencil27(127, kind=gen.SMALLINT), np.float32)
    m = A["m"]
    x = gen.vector(m, 5, kind=gen.SMALLINT, dtype=np.float32); y = gen.vector(m, 6, kind=gen.SMALLINT, dtype=np.float32)
    check(A, fmt, x, y, 1.5, 0.5, exact=True)


@pytest.mark.slow
def test_config3_rmat_full_size_fp32_bit_exact():
    A = to_dtype(gen.rmat(24, seed=3, kind=gen.SMALLINT), np.float32)
    x = gen.vector(A["n"], 7, kind=gen.SMALLINT, dtype=np.float32); y = gen.vector(A["m"], 8, kind=gen.SMALLINT, dtype=np.float32)
    check(A, "csr", x, y, 2.0, 0.5, exact=True)


@pytest.mark.slow
@pytest.mark.parametrize("fmt", ["csc", "coo_col", "csc:bands"])
def test_config3_rmat_full_size_column_formats_bit_exact(fmt):
    """R-MAT scale 24 through the pCSC band layout (its heavy first bands are split into slot units)
    and the column-sorted pCOO, fp64, bit-exact."""
    A = gen.rmat(24, seed=3, kind=gen.SMALLINT)
    x = gen.vector(A["n"], 7, kind=gen.SMALLINT); y = gen.vector(A["m"], 8, kind=gen.SMALLINT)
    check(A, fmt, x, y, 2.0, 0.5, exact=True)


@pytest.mark.slow
@pytest.mark.parametrize("fmt", ["csc", "coo"])
def test_config3_rmat_full_size_fp32_other_formats_bit_exact(fmt):
    """R-MAT scale 24 fp32 through pCSC on row tiles (fp32 partial y) and pCOO, bit-exact
    (integer data: every row sum < 2^24)."""
    A = to_dtype(gen.rmat(24, seed=3, kind=gen.SMALLINT), np.float32)
    x = gen.vector(A["n"], 7, kind=gen.SMALLINT, dtype=np.float32); y = gen.vector(A["m"], 8, kind=gen.SMALLINT, dtype=np.float32)
    check(A, fmt, x, y, 2.0, 0.5, exact=True)


@pytest.mark.slow
def test_config4_tallskinny_fp32_bit_exact():
    A = to_dtype(gen.kdistinct_csc(50_000_000, 1_000_000, 500, seed=4, kind=gen.SMALLINT), np.float32)
    x = gen.vector(A["n"], 9, kind=gen.SMALLINT, dtype=np.float32); y = gen.vector(A["m"], 10, kind=gen.SMALLINT, dtype=np.float32)
    check(A, "csc", x, y, 2.0, 0.5, exact=True)


@pytest.mark.slow
@pytest.mark.parametrize("fmt", ["csc", "csc:bands"])
def test_config4_tallskinny_csc_sampled(fmt):
    A = gen.kdistinct_csc(50_000_000, 1_000_000, 500, seed=4, kind=gen.SMALLINT)
    x = gen.vector(A["n"], 9, kind=gen.SMALLINT); y = gen.vector(A["m"], 10, kind=gen.SMALLINT)
    check(A, fmt, x, y, 2.0, 0.5, exact=True)


# ------------------------------------------------------ pCSC row-band layout
def _csc_drop_rows(A, lo, hi):
    """CSC copy of A without the entries whose row is in [lo, hi) (empty row bands)."""
    keep = ~((A["idx"] >= lo) & (A["idx"] < hi))
    cols = np.repeat(np.arange(A["n"]), np.diff(A["ptr"]))[keep]
    ptr = np.zeros(A["n"] + 1, np.int64)
    np.add.at(ptr, cols + 1, 1)
    return gen.Sparse(fmt="csc", m=A["m"], n=A["n"], ptr=np.cumsum(ptr), idx=A["idx"][keep], val=A["val"][keep])


@pytest.mark.parametrize("fmt", ["csc:bands", "csc"])
@pytest.mark.parametrize("parts", [1, 3])
def test_csc_bands_column_chunks_bit_exact(fmt, parts):
    """Several 8192-row bands (ragged last band), > 2^19 columns (two column chunks per
    band), an entirely empty band: bit-exact vs the oracle on integer data."""
    A = gen.kdistinct_csc(3 * 8192 + 17, (1 << 19) + 1000, 2, seed=41, kind=gen.SMALLINT)
    A = _csc_drop_rows(A, 8192, 2 * 8192)
    x = gen.vector(A["n"], 42, kind=gen.SMALLINT); y = gen.vector(A["m"], 43, kind=gen.SMALLINT)
    for alpha, beta in [(1.5, 0.5), (2.0, 0.0), (-1.0, 1.0)]:
        check(A, fmt, x, y, alpha, beta, parts=parts, exact=True)


@pytest.mark.parametrize("fmt", ["csc:bands", "csc"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_csc_bands_uniform_tolerance(fmt, dtype):
    """Dense-ish columns spanning many bands, U[-1,1) values: per-row tolerance."""
    A = to_dtype(gen.kdistinct_csc(100_000, 3000, 400, seed=44), dtype)
    x = gen.vector(A["n"], 45, dtype=dtype); y = gen.vector(A["m"], 46, dtype=dtype)
    check(A, fmt, x, y, 1.5, 0.5, parts=2)


# --------------------------------------------- config 5: SuiteSparse-shaped suite
def _suite_small(shape, kind):
    if shape == "banded":
        return gen.banded(3000, 3000, 70, seed=501, kind=kind)         # 141 per row, rows > one SEG tile
    if shape == "blockdiag":
        return gen.blockdiag(64 * 40, 64, seed=502, kind=kind)          # dense 64x64 blocks
    if shape == "powerlaw":
        return gen.transpose(gen.powerlaw_csc(20000, 20000, 2.13, 5000, seed=503, kind=kind))
    return gen.kdistinct_csr(300, 15000, 500, seed=504, kind=kind)     # short-wide, 500 per row


@pytest.mark.parametrize("shape", ["banded", "blockdiag", "powerlaw", "shortwide"])
@pytest.mark.parametrize("fmt", FMTS)
def test_suite_shapes_bit_exact(shape, fmt):
    """Config 5 shapes at test size, integer data: bit-exact in every format, 1 and 3 parts."""
    A = _suite_small(shape, gen.SMALLINT)
    x = gen.vector(A["n"], 61, kind=gen.SMALLINT); y = gen.vector(A["m"], 62, kind=gen.SMALLINT)
    for parts in (1, 3):
        check(A, fmt, x, y, 1.5, 0.5, parts=parts, exact=True)


@pytest.mark.parametrize("shape", ["banded", "blockdiag", "powerlaw", "shortwide"])
@pytest.mark.parametrize("fmt", FMTS)
def test_suite_shapes_fp32_tolerance(shape, fmt):
    """Config 5 shapes, fp32 storage, U[-1,1): per-row tolerance 1e-5 of sum |a_ij x_j|."""
    A = to_dtype(_suite_small(shape, gen.UNIFORM), np.float32)
    x = gen.vector(A["n"], 63, dtype=np.float32); y = gen.vector(A["m"], 64, dtype=np.float32)
    check(A, fmt, x, y, 1.5, 0.5, parts=2)


@pytest.mark.parametrize("fmt", ["csc:bands", "coo_col:bands", "csc", "coo_unsorted"])
@pytest.mark.parametrize("parts", [1, 3])
def test_csc_split_bands_reproducible(fmt, parts):
    """Heavy bands (R-MAT's first rows; a short-wide matrix with fewer bands than SMs) are cut into
    stage-range units whose partial rows are reduced over slots in slot order: U[-1,1) results are
    bit-identical run to run, and within tau of the oracle."""
    for A in (gen.rmat(16, seed=21), gen.kdistinct_csr(3000, 400_000, 300, seed=22)):
        x = gen.vector(A["n"], 1); y = gen.vector(A["m"], 2)
        outs = run_gpu(as_fmt(A, fmt), fmt, x, y, 1.5, 0.5, parts=parts, repeat=4)
        for o in outs[1:]:
            assert np.array_equal(outs[0], o)
        assert_close(outs[0], oracle_ref(A, x, y, 1.5, 0.5), row_bound(A, x, y, 1.5, 0.5), np.float64)


@pytest.mark.parametrize("fmt", ["csc:bands", "csc"])
@pytest.mark.parametrize("parts", [1, 2])
def test_csc_split_items_short_wide(fmt, parts):
    """Fewer row bands than SMs (m = 3 bands): every band is cut into stage-range units whose
    partial rows go to slots, reduced in slot order at the end of the launch -- integer data,
    bit-exact; and fp32 within tolerance."""
    A = gen.kdistinct_csr(3 * 8192 - 5, 300_000, 40, seed=71, kind=gen.SMALLINT)
    x = gen.vector(A["n"], 72, kind=gen.SMALLINT); y = gen.vector(A["m"], 73, kind=gen.SMALLINT)
    check(A, fmt, x, y, 1.5, 0.5, parts=parts, exact=True)
    check(A, fmt, x, y, 2.0, 0.0, parts=parts, exact=True)
    B = to_dtype(gen.kdistinct_csr(1000, 200_000, 300, seed=74), np.float32)
    xb = gen.vector(B["n"], 75, dtype=np.float32); yb = gen.vector(B["m"], 76, dtype=np.float32)
    check(B, fmt, xb, yb, 1.5, 0.5, parts=parts)


@pytest.mark.parametrize("fmt", ["csr", "coo"])
def test_sell_and_seg_split_launch(fmt):
    """Stencil rows (SELL tiles) stacked over R-MAT rows (SEG tiles / slabs), each a real share of
    the nonzeros: the two tile kinds run as two launches of their own kernel instantiations
    (kernels_per_spmv counts both) -- bit-exact, 1 and 3 parts, device- and host-resident."""
    import paper_2209_07552_b200 as M
    S = gen.stencil27(12, kind=gen.SMALLINT)
    R = gen.rmat(11, seed=141, kind=gen.SMALLINT)
    n = max(S["n"], R["n"])
    A = gen.Sparse(fmt="csr", m=S["m"] + R["m"], n=n,
                   ptr=np.concatenate([S["ptr"], R["ptr"][1:] + S["ptr"][-1]]).astype(np.int64),
                   idx=np.concatenate([S["idx"], R["idx"]]).astype(np.int32),
                   val=np.concatenate([S["val"], R["val"]]))
    x = gen.vector(n, 142, kind=gen.SMALLINT); y = gen.vector(A["m"], 143, kind=gen.SMALLINT)
    ref = oracle_ref(A, x, y, 1.5, 0.5)
    for parts in (1, 3):
        for kw in ({}, {"residency": "host", "chunk_bytes": 32 << 10}):
            ctx = M.Context(0, 1, None, 0, parts)
            got = run_gpu(A, fmt, x, y, 1.5, 0.5, ctx=ctx, **kw)
            st = ctx.stats()
            if parts == 1 and not kw:   # the pipelined host-vector path: row chunks over both tile lists
                for beta in (0.5, 0.0):
                    yh = y.copy()
                    ctx.spmv_host(1.5, x, beta, yh)
                    assert np.array_equal(yh, oracle_ref(A, x, y, 1.5, beta)), ("host path", fmt, beta)
            ctx.close()
            assert np.array_equal(got, ref), (fmt, parts, kw)
            assert st["nsell"] > 0
            if not kw:
                assert st["kernels_per_spmv"] >= 2, st


# ------------------------------------------------ Baseline row/column-block split (NEXT f1)
@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("parts", [2, 5, 8])
def test_block_split_bit_exact(fmt, parts):
    """The paper's Baseline split (whole row / column blocks) through the same kernels and
    merge: bit-exact vs the oracle on integer R-MAT (heavy rows) and a two-class matrix."""
    import paper_2209_07552_b200 as M
    import torch
    for A in (gen.rmat(11, seed=5, kind=gen.SMALLINT), gen.two_class(4000, 3000, 8, 4, 40, 0.1, kind=gen.SMALLINT)):
        B = as_fmt(A, fmt)
        x = gen.vector(A["n"], 81, kind=gen.SMALLINT); y = gen.vector(A["m"], 82, kind=gen.SMALLINT)
        ctx = M.Context(0, 1, None, 0, parts)
        pf = apply_layout(ctx, fmt)
        if pf in ("coo", "coo_col"):
            ctx.partition(pf, B["m"], B["n"], idx=B["idx"], val=B["val"], coo_row=coo_of_csr(B), split="block")
        else:
            ctx.partition(pf, B["m"], B["n"], ptr=B["ptr"], idx=B["idx"], val=B["val"], split="block")
        assert (ctx.parts["start_flag"] == 0).all()
        xd = torch.as_tensor(x).cuda(); yd = torch.as_tensor(y.copy()).cuda()
        ctx.spmv(1.5, xd, 0.5, yd)
        torch.cuda.synchronize()
        assert np.array_equal(yd.cpu().numpy(), oracle_ref(A, x, y, 1.5, 0.5))
        ctx.close()


@pytest.mark.parametrize("k", [1, 3, 6, 8, 12, 16, 20])
@pytest.mark.parametrize("fmt", ["csr", "coo"])
def test_sell_rows_per_lane(k, fmt):
    """Regular short rows become SELL tiles with R = 4 / 2 / 1 rows per lane (R*W <= 32), incl.
    ragged last tiles and a sprinkle of empty rows: bit-exact vs the oracle.  pCOO packs its SELL
    tiles from the window pointer counted on the host."""
    A = gen.kdistinct_csr(32 * 4 * 7 + 45, 5000, k, seed=90 + k, kind=gen.SMALLINT)
    x = gen.vector(A["n"], 91, kind=gen.SMALLINT); y = gen.vector(A["m"], 92, kind=gen.SMALLINT)
    for parts in (1, 3):
        check(A, fmt, x, y, 1.5, 0.5, parts=parts, exact=True)
    # shorter rows mixed in (padding <= 1/8 may still hold or not): still exact
    B = gen.two_class(32 * 4 * 9, 4000, 9, 4, k, 0.5, kind=gen.SMALLINT)
    xb = gen.vector(B["n"], 93, kind=gen.SMALLINT); yb = gen.vector(B["m"], 94, kind=gen.SMALLINT)
    check(B, fmt, xb, yb, 2.0, 0.5, parts=2, exact=True)


def _banded_rows(m, k, span, seed, kind):
    """m rows of k distinct columns each within [r - span/2, r + span/2] (clipped): narrow SELL rows"""
    rng = np.random.default_rng(seed)
    n = m
    ptr = np.arange(m + 1, dtype=np.int64) * k
    idx = np.empty(m * k, dtype=np.int32)
    for r in range(m):
        lo = max(0, min(n - span, r - span // 2))
        idx[r * k:(r + 1) * k] = np.sort(rng.choice(span, size=k, replace=False) + lo)
    val = gen.vector(m * k, seed + 1, kind=kind)
    return gen.Sparse(fmt="csr", m=m, n=n, ptr=ptr, idx=idx, val=val)


@pytest.mark.parametrize("k", [8, 16, 27, 32])
@pytest.mark.parametrize("fmt", ["csr", "coo", "csc", "coo_col"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_narrow_sell_tiles(k, fmt, dtype):
    """Narrow SELL tiles (16-bit column offsets from a per-tile base; fp32 up to 64 entries per lane,
    i.e. R = 2 for 27-point rows) next to 32-bit ones: rows whose columns span < 65536 become
    narrow, a block of rows spanning the whole x stays wide.  Bit-exact vs the oracle for
    MSREP_TUNE_SELL 2 (narrow) and 1 (32-bit only), 1 and 3 parts, device- and host-resident,
    and the SpMM block walk over the same tiles.  The column formats run on row tiles over their
    GPU-transposed slice, whose row spans come from the device (row_span_kernel)."""
    import paper_2209_07552_b200 as M
    import torch
    m = 32 * 4 * 12 + 37
    A = _banded_rows(m, k, 20000, 300 + k, gen.SMALLINT)
    # rows 1024..1279 get a column near the end of a 200K-wide x: those tiles cannot be narrow
    n = 200_000
    idx = A["idx"].copy()
    wide = np.arange(1024, 1280)
    idx[A["ptr"][wide + 1] - 1] = n - 1 - wide
    A = gen.Sparse(fmt="csr", m=m, n=n, ptr=A["ptr"], idx=idx, val=A["val"])
    A = to_dtype(A, dtype)
    x = gen.vector(n, 311, kind=gen.SMALLINT).astype(dtype); y = gen.vector(m, 312, kind=gen.SMALLINT).astype(dtype)
    ref = oracle_ref(A, x, y, 1.5, 0.5)
    for sell in (2, 1):
        for parts in (1, 3):
            for kw in ({}, {"residency": "host", "chunk_bytes": 32 << 10}):
                ctx = M.Context(0, 1, None, 0, parts)
                ctx.set_tuning("sell", sell)
                got = run_gpu(as_fmt(A, fmt), fmt, x, y, 1.5, 0.5, ctx=ctx, **kw)
                st = ctx.stats()
                assert np.array_equal(got, ref), (sell, parts, kw, np.nonzero(got != ref)[0][:8])
                assert st["nsell"] > 0
                if sell == 2:
                    assert 0 < st["nsell_narrow"] < st["nsell"], st
                else:
                    assert st["nsell_narrow"] == 0, st
                if not kw and parts == 1:   # SpMM over the same tiles (4 vectors: 2x, x, -x, 3x)
                    X = np.stack([2 * x, x, -x, 3 * x], 1).astype(dtype)
                    Y = np.stack([y] * 4, 1).astype(dtype)
                    Xd = torch.as_tensor(X).cuda(); Yd = torch.as_tensor(Y).cuda()
                    ctx.spmm(1.5, Xd, 0.5, Yd)
                    torch.cuda.synchronize()
                    got4 = Yd.cpu().numpy()
                    for j in range(4):
                        assert np.array_equal(got4[:, j], oracle_ref(A, X[:, j].copy(), y, 1.5, 0.5)), (sell, j)
                ctx.close()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_narrow_sell_span_boundary(dtype):
    """A SELL tile is narrow iff its columns span <= 65535 (16-bit offsets from the tile's smallest
    column): 128-row blocks (one R = 4 SELL tile each) of 8 columns reaching exactly base + 65535
    are narrow, blocks reaching base + 65536 are not; both bit-exact, including the largest offset
    65535 itself."""
    import paper_2209_07552_b200 as M
    blocks, n = 24, 200_000
    rows_per = 128
    m = blocks * rows_per
    rng = np.random.default_rng(77)
    ptr = np.arange(m + 1, dtype=np.int64) * 8
    idx = np.empty(m * 8, dtype=np.int32)
    for b in range(blocks):
        base = 1000 * b
        reach = 65535 if b % 2 == 0 else 65536   # even blocks narrow, odd blocks wide
        for r in range(b * rows_per, (b + 1) * rows_per):
            mid = np.sort(rng.choice(np.arange(1, reach), size=6, replace=False))
            cols = np.concatenate([[base], base + mid, [base + reach]])
            idx[r * 8:(r + 1) * 8] = cols
    A = to_dtype(gen.Sparse(fmt="csr", m=m, n=n, ptr=ptr, idx=idx, val=gen.vector(m * 8, 78, kind=gen.SMALLINT)), dtype)
    x = gen.vector(n, 79, kind=gen.SMALLINT).astype(dtype); y = gen.vector(m, 80, kind=gen.SMALLINT).astype(dtype)
    ref = oracle_ref(A, x, y, 1.5, 0.5)
    ctx = M.Context(0, 1, None, 0, 1)
    got = run_gpu(A, "csr", x, y, 1.5, 0.5, ctx=ctx)
    st = ctx.stats()
    ctx.close()
    assert np.array_equal(got, ref)
    assert st["nsell"] == blocks and st["nsell_narrow"] == blocks // 2, st


@pytest.mark.parametrize("fmt", ["csc:bands", "coo_col:bands", "csc"])
def test_csc_heavy_rows_same_row_groups(fmt):
    """Rows with thousands of entries inside one band (R-MAT heavy rows, and a dense row): the
    pCSC lists carry same-row groups of 32 (one warp-reduced update) -- bit-exact."""
    A = gen.rmat(14, seed=13, kind=gen.SMALLINT)
    x = gen.vector(A["n"], 95, kind=gen.SMALLINT); y = gen.vector(A["m"], 96, kind=gen.SMALLINT)
    for parts in (1, 3):
        check(A, fmt, x, y, 1.5, 0.5, parts=parts, exact=True)
    n = 50_000
    D = gen.Sparse(fmt="csr", m=3, n=n, ptr=np.array([0, n, n + 7, 2 * n + 7], np.int64),
                   idx=np.concatenate([np.arange(n), np.arange(7) * 11, np.arange(n)]).astype(np.int32),
                   val=np.ones(2 * n + 7))
    xd = gen.vector(n, 97, kind=gen.SMALLINT)
    check(D, fmt, xd, np.zeros(3), 1.0, 0.0, parts=2, exact=True)


@pytest.mark.parametrize("fmt", ["csc:bands", "coo_col:bands", "csc"])
def test_csc_segmented_groups_few_rows(fmt):
    """Warp lists whose entries sit on fewer than 32 rows (40 rows of 700 entries in one band,
    plus sparse light rows): after the same-row groups the greedy distinct-row pass gets stuck and
    the rest of the list becomes row-sorted SEGMENTED groups (one warp segmented scan each) --
    bit-exact on integer data, fp32 within tolerance, 1 and 2 parts."""
    rng = np.random.default_rng(131)
    m, n = 8192, 200_000
    heavy = set(range(0, m, m // 40))
    ptr = [0]; idx = []
    for r in range(m):
        k = 700 if r in heavy else int(rng.integers(0, 3))
        idx.append(np.sort(rng.choice(n, k, replace=False)))
        ptr.append(ptr[-1] + k)
    idx = np.concatenate(idx).astype(np.int32)
    A = gen.Sparse(fmt="csr", m=m, n=n, ptr=np.array(ptr, np.int64), idx=idx,
                   val=rng.integers(-4, 5, idx.size).astype(np.float64))
    x = gen.vector(n, 132, kind=gen.SMALLINT); y = gen.vector(m, 133, kind=gen.SMALLINT)
    for parts in (1, 2):
        check(A, fmt, x, y, 1.5, 0.5, parts=parts, exact=True)
    B = to_dtype(A, np.float32)
    xb = gen.vector(n, 134, dtype=np.float32); yb = gen.vector(m, 135, dtype=np.float32)
    check(B, fmt, xb, yb, 1.5, 0.5, parts=1)


# ------------------------------------------------------------ CG (NEXT f4)
def _spd_stencil(N, diag=30.0, kind=None):
    A = gen.stencil27(N, kind=gen.ONES)
    rows = np.repeat(np.arange(A["m"]), np.diff(A["ptr"]))
    A["val"] = np.where(A["idx"] == rows, diag, -1.0)
    return A


def _cg_gpu(A, fmt, b, parts, dtype, tol, maxit):
    import paper_2209_07552_b200 as M
    import torch
    B = as_fmt(to_dtype(A, dtype), fmt)
    ctx = M.Context(0, 1, None, 0, parts)
    pf = apply_layout(ctx, fmt)
    if pf in ("coo", "coo_col"):
        ctx.partition(pf, B["m"], B["n"], idx=B["idx"], val=B["val"], coo_row=coo_of_csr(B))
    else:
        ctx.partition(pf, B["m"], B["n"], ptr=B["ptr"], idx=B["idx"], val=B["val"])
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    bd = torch.as_tensor(b.astype(dtype)).cuda()
    xd = torch.zeros(A["n"], dtype=tdt, device="cuda")
    it, rr = ctx.cg(bd, xd, tol=tol, maxit=maxit, check_every=1)
    x = xd.cpu().numpy().astype(np.float64)
    ctx.close()
    return x, it, rr


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("parts", [1, 3])
def test_cg_matches_oracle(fmt, parts):
    """msrep_cg on the SPD stencil (diag 30, off -1) with b = A x*: converges to x*, within one
    iteration of the oracle's textbook CG, fp64."""
    A = _spd_stencil(16)
    m = A["m"]
    xs = (np.arange(m) % 7 - 3).astype(np.float64)
    b = oracle.spmv_csr(m, A["ptr"], A["idx"], A["val"], xs, np.zeros(m), 1.0, 0.0)
    xo, ito, rro = oracle.cg_csr(m, A["ptr"], A["idx"], A["val"], b, np.zeros(m), 1e-11, 500)
    x, it, rr = _cg_gpu(A, fmt, b, parts, np.float64, 1e-11, 500)
    assert rr <= 1e-11 and abs(it - ito) <= 1, (it, ito, rr, rro)
    assert np.max(np.abs(x - xs)) < 1e-9
    assert np.max(np.abs(x - xo)) < 1e-9


@pytest.mark.parametrize("fmt", ["csr", "csc", "csc:bands"])
def test_cg_graph_matches_eager(fmt):
    """msrep_cg replays a captured CUDA graph of two iterations (single rank, device-resident);
    with even convergence checks it takes the same iterations and the same iterates, bit for
    bit, as the eager loop (msrep_set_tuning(MSREP_TUNE_CG_GRAPH, 0))."""
    import paper_2209_07552_b200 as M
    import torch
    A = _spd_stencil(14)
    m = A["m"]
    xs = (np.arange(m) % 5 - 2).astype(np.float64)
    b = torch.as_tensor(oracle.spmv_csr(m, A["ptr"], A["idx"], A["val"], xs, np.zeros(m), 1.0, 0.0)).cuda()
    res = []
    for graph in (1, 0):
        B = as_fmt(A, fmt)
        ctx = M.Context(0, 1, None, 0, 2)
        ctx.set_tuning("cg_graph", graph)
        ctx.partition(apply_layout(ctx, fmt), B["m"], B["n"], ptr=B["ptr"], idx=B["idx"], val=B["val"])
        xd = torch.zeros(m, dtype=torch.float64, device="cuda")
        it, rr = ctx.cg(b, xd, tol=1e-11, maxit=300, check_every=4)
        res.append((it, rr, xd.cpu().numpy()))
        ctx.close()
    assert res[0][0] == res[1][0] and res[0][1] == res[1][1], (res[0][:2], res[1][:2])
    assert np.array_equal(res[0][2], res[1][2])
    assert np.max(np.abs(res[0][2] - xs)) < 1e-9


def test_cg_fp32_storage():
    """fp32 storage (fp64 dot products and scalars): converges to x* to fp32 accuracy."""
    A = _spd_stencil(12)
    m = A["m"]
    xs = (np.arange(m) % 5 - 2).astype(np.float64)
    b = oracle.spmv_csr(m, A["ptr"], A["idx"], A["val"], xs, np.zeros(m), 1.0, 0.0)
    x, it, rr = _cg_gpu(A, "csr", b, 2, np.float32, 1e-6, 300)
    assert rr <= 1e-6 and np.max(np.abs(x - xs)) < 1e-4


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("graph", [1, 0])
def test_cg_exact_convergence_no_nan(fmt, graph):
    """Identity matrix: CG converges exactly in one iteration (r = p = 0 afterwards).  The extra
    iterations the graph period / check interval run past that point must be no-ops (alpha, beta
    guarded against 0/0), not a NaN "breakdown"."""
    import paper_2209_07552_b200 as M
    import torch
    m = 5000
    A = gen.Sparse(fmt="csr", m=m, n=m, ptr=np.arange(m + 1, dtype=np.int64), idx=np.arange(m, dtype=np.int32),
                   val=np.ones(m))
    B = as_fmt(A, fmt)
    ctx = M.Context(0, 1, None, 0, 2)
    ctx.set_tuning("cg_graph", graph)
    pf = apply_layout(ctx, fmt)
    if pf in ("coo", "coo_col"):
        ctx.partition(pf, m, m, idx=B["idx"], val=B["val"], coo_row=coo_of_csr(B))
    else:
        ctx.partition(pf, m, m, ptr=B["ptr"], idx=B["idx"], val=B["val"])
    b = (np.arange(m) % 9 - 4).astype(np.float64)
    xd = torch.zeros(m, dtype=torch.float64, device="cuda")
    it, rr = ctx.cg(torch.as_tensor(b).cuda(), xd, tol=0.0, maxit=12, check_every=1)
    assert rr == 0.0 and it >= 1
    assert np.array_equal(xd.cpu().numpy(), b)
    ctx.close()


def test_binding_rejects_bad_arguments():
    """The binding validates what it hands to the C ABI: value dtype, array lengths, and device
    vectors (CUDA, contiguous, the partition's dtype, long enough)."""
    import paper_2209_07552_b200 as M
    import torch
    A = gen.kdistinct_csr(50, 40, 3, seed=3)
    ctx = M.Context(0, 1, None, 0, 1)
    with pytest.raises(ValueError):
        ctx.partition("csr", 50, 40, ptr=A["ptr"], idx=A["idx"], val=A["val"].astype(np.int64))
    with pytest.raises(ValueError):
        ctx.partition("csr", 50, 40, ptr=A["ptr"], idx=A["idx"], val=A["val"][:-1])
    ctx.partition("csr", 50, 40, ptr=A["ptr"], idx=A["idx"], val=A["val"])
    x = torch.zeros(40, dtype=torch.float64, device="cuda"); y = torch.zeros(50, dtype=torch.float64, device="cuda")
    ctx.spmv(1.0, x, 0.0, y)
    for bad_x, bad_y in [(x.float(), y), (x.cpu(), y), (x, y[:49]), (x, torch.zeros(100, dtype=torch.float64,
                                                                                     device="cuda")[::2])]:
        with pytest.raises(ValueError):
            ctx.spmv(1.0, bad_x, 0.0, bad_y)
    with pytest.raises(ValueError):
        ctx.spmv_host(1.0, np.zeros(40, np.float32), 0.0, np.zeros(50))
    with pytest.raises(M.MsrepError):
        ctx.set_tuning("xload", 5)
    ctx.close()


def test_cg_errors():
    import paper_2209_07552_b200 as M
    import torch
    A = gen.kdistinct_csr(20, 30, 3, seed=3)
    ctx = M.Context(0, 1, None, 0, 1)
    ctx.partition("csr", 20, 30, ptr=A["ptr"], idx=A["idx"], val=A["val"])
    with pytest.raises(M.MsrepError) as e:   # not square
        ctx.cg(torch.zeros(20, dtype=torch.float64, device="cuda"), torch.zeros(30, dtype=torch.float64, device="cuda"))
    assert e.value.status == 2
    ctx.close()


# ------------------------------------------------------------ SpMM (NEXT f4)
def _spmm_gpu(A, fmt, X, Y, alpha, beta, parts):
    import paper_2209_07552_b200 as M
    import torch
    B = as_fmt(A, fmt)
    ctx = M.Context(0, 1, None, 0, parts)
    pf = apply_layout(ctx, fmt)
    if pf in ("coo", "coo_col"):
        ctx.partition(pf, B["m"], B["n"], idx=B["idx"], val=B["val"], coo_row=coo_of_csr(B))
    else:
        ctx.partition(pf, B["m"], B["n"], ptr=B["ptr"], idx=B["idx"], val=B["val"])
    Xd = torch.as_tensor(np.ascontiguousarray(X)).cuda()
    Yd = torch.as_tensor(np.ascontiguousarray(Y)).cuda()
    ctx.spmm(alpha, Xd, beta, Yd)
    torch.cuda.synchronize()
    out = Yd.cpu().numpy()
    ctx.close()
    return out


def _spmm_ref(A, X, Y, alpha, beta):
    return np.stack([oracle_ref(A, X[:, j].copy(), Y[:, j].copy(), alpha, beta) for j in range(X.shape[1])], axis=1)


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("k", [2, 4, 8])
def test_spmm_bit_exact(fmt, k):
    """Y = alpha*A*X + beta*Y for k vectors at once equals k oracle SpMVs bit for bit (integer
    data): R-MAT (SEG tiles, slabs, split rows), the stencil (SELL tiles), short regular rows
    (4-row-per-lane SELL), a chain row across parts; 1 and 3 parts; beta = 0 and alpha = 0."""
    cases = [gen.rmat(11, seed=21, kind=gen.SMALLINT), gen.stencil27(9, kind=gen.SMALLINT),
             gen.kdistinct_csr(700, 900, 5, seed=22, kind=gen.SMALLINT),
             gen.Sparse(fmt="csr", m=1, n=3000, ptr=np.array([0, 3000], np.int64), idx=np.arange(3000, dtype=np.int32),
                        val=np.ones(3000))]
    rng = np.random.default_rng(k)
    for A in cases:
        X = rng.integers(-4, 5, (A["n"], k)).astype(np.float64)
        Y = rng.integers(-4, 5, (A["m"], k)).astype(np.float64)
        for parts in (1, 3):
            for alpha, beta in ((1.5, 0.5), (2.0, 0.0), (0.0, -1.0)):
                got = _spmm_gpu(A, fmt, X, Y, alpha, beta, parts)
                assert np.array_equal(got, _spmm_ref(A, X, Y, alpha, beta)), (fmt, k, parts, alpha, beta)


@pytest.mark.parametrize("k", [2, 4, 8])
def test_spmm_fp32_tolerance(k):
    A = to_dtype(gen.rmat(10, seed=23), np.float32)
    rng = np.random.default_rng(30 + k)
    X = rng.uniform(-1, 1, (A["n"], k)).astype(np.float32)
    Y = rng.uniform(-1, 1, (A["m"], k)).astype(np.float32)
    got = _spmm_gpu(A, "csr", X, Y, 1.5, 0.5, 2)
    for j in range(k):
        x, y = X[:, j].copy(), Y[:, j].copy()
        assert_close(got[:, j], oracle_ref(A, x, y, 1.5, 0.5), row_bound(A, x, y, 1.5, 0.5), np.float32)


@pytest.mark.parametrize("fmt", ["csc:bands", "csc"])
@pytest.mark.parametrize("k", [2, 8])
def test_spmm_column_formats_fp32_and_split_bands(fmt, k):
    """pCSC SpMM (one strided band-kernel pass per vector): fp32 within tolerance on a short-wide
    matrix whose bands are split into slot units, and the unsorted pCOO path."""
    A = to_dtype(gen.kdistinct_csr(3000, 200_000, 60, seed=24), np.float32)
    rng = np.random.default_rng(40 + k)
    X = rng.uniform(-1, 1, (A["n"], k)).astype(np.float32)
    Y = rng.uniform(-1, 1, (A["m"], k)).astype(np.float32)
    got = _spmm_gpu(A, fmt, X, Y, 1.5, 0.5, 3)
    for j in range(k):
        x, y = X[:, j].copy(), Y[:, j].copy()
        assert_close(got[:, j], oracle_ref(A, x, y, 1.5, 0.5), row_bound(A, x, y, 1.5, 0.5), np.float32)


def test_spmm_rejects_bad_layout_and_k():
    import paper_2209_07552_b200 as M
    import torch
    A = gen.transpose(gen.kdistinct_csr(50, 40, 3, seed=3))
    ctx = M.Context(0, 1, None, 0, 1)
    ctx.partition("csc", 50, 40, ptr=A["ptr"], idx=A["idx"], val=A["val"])
    with pytest.raises(M.MsrepError) as e:   # OWNED is a row-format layout
        ctx.spmm(1.0, torch.zeros((40, 4), dtype=torch.float64, device="cuda"), 0.0,
                 torch.zeros((50, 4), dtype=torch.float64, device="cuda"), layout=M.Y_OWNED)
    assert e.value.status == 1
    B = gen.kdistinct_csr(50, 40, 3, seed=3)
    ctx.partition("csr", 50, 40, ptr=B["ptr"], idx=B["idx"], val=B["val"])
    with pytest.raises(M.MsrepError) as e:
        ctx.spmm(1.0, torch.zeros((40, 3), dtype=torch.float64, device="cuda"), 0.0,
                 torch.zeros((50, 3), dtype=torch.float64, device="cuda"))
    assert e.value.status == 1
    ctx.close()


# ------------------------------------- fused compute + allgather stores (msrep_spmv_mirror)
@pytest.mark.parametrize("fmt", ["csr", "coo"])
@pytest.mark.parametrize("parts", [1, 3])
def test_spmv_mirror_loopback(fmt, parts):
    """Loopback check of the epilogue's multi-destination stores on one GPU: the mirrors are
    local buffers pre-filled with NaN; after the call y and every mirror equal the oracle
    (bit-exact, integer data), including split rows written by the fix-up (R-MAT heavy rows)
    and SELL tiles (stencil); alpha = 0 copies beta*y into the mirrors."""
    import paper_2209_07552_b200 as M
    import torch
    for A in (gen.rmat(12, seed=31, kind=gen.SMALLINT), gen.stencil27(10, kind=gen.SMALLINT)):
        x = gen.vector(A["n"], 32, kind=gen.SMALLINT); y = gen.vector(A["m"], 33, kind=gen.SMALLINT)
        ctx = M.Context(0, 1, None, 0, parts)
        if fmt == "coo":
            ctx.partition("coo", A["m"], A["n"], idx=A["idx"], val=A["val"], coo_row=coo_of_csr(A))
        else:
            ctx.partition("csr", A["m"], A["n"], ptr=A["ptr"], idx=A["idx"], val=A["val"])
        for alpha, beta in ((1.5, 0.5), (0.0, 2.0)):
            xd = torch.as_tensor(x).cuda(); yd = torch.as_tensor(y.copy()).cuda()
            mirrors = [torch.full((A["m"],), float("nan"), dtype=torch.float64, device="cuda") for _ in range(3)]
            ctx.spmv_mirror(alpha, xd, beta, yd, mirrors)
            torch.cuda.synchronize()
            ref = oracle_ref(A, x, y, alpha, beta)
            assert np.array_equal(yd.cpu().numpy(), ref)
            for mm in mirrors:
                assert np.array_equal(mm.cpu().numpy(), ref)
        ctx.close()


def test_spmv_mirror_rejects():
    import paper_2209_07552_b200 as M
    import torch
    A = gen.transpose(gen.kdistinct_csr(30, 30, 3, seed=3))
    ctx = M.Context(0, 1, None, 0, 1)
    ctx.partition("csc", 30, 30, ptr=A["ptr"], idx=A["idx"], val=A["val"])
    with pytest.raises(M.MsrepError) as e:
        z = torch.zeros(30, dtype=torch.float64, device="cuda")
        ctx.spmv_mirror(1.0, z, 0.0, z.clone(), [z.clone()])
    assert e.value.status == 5
    ctx.close()


@pytest.mark.parametrize("fmt", FMTS)
def test_two_level_split_bit_exact(fmt):
    """The two-level NUMA split (groups [1, 3] and [4, 4] of parts) through the same kernels and
    merge: bit-exact on integer R-MAT (split rows at different cut points than the nnz split)."""
    import paper_2209_07552_b200 as M
    import torch
    A = gen.rmat(11, seed=51, kind=gen.SMALLINT)
    B = as_fmt(A, fmt)
    x = gen.vector(A["n"], 52, kind=gen.SMALLINT); y = gen.vector(A["m"], 53, kind=gen.SMALLINT)
    for groups in ([1, 3], [4, 4]):
        ctx = M.Context(0, 1, None, 0, sum(groups))
        pf = apply_layout(ctx, fmt)
        if pf in ("coo", "coo_col"):
            ctx.partition(pf, B["m"], B["n"], idx=B["idx"], val=B["val"], coo_row=coo_of_csr(B), split=groups)
        else:
            ctx.partition(pf, B["m"], B["n"], ptr=B["ptr"], idx=B["idx"], val=B["val"], split=groups)
        xd = torch.as_tensor(x).cuda(); yd = torch.as_tensor(y.copy()).cuda()
        ctx.spmv(1.5, xd, 0.5, yd)
        torch.cuda.synchronize()
        assert np.array_equal(yd.cpu().numpy(), oracle_ref(A, x, y, 1.5, 0.5)), (fmt, groups)
        ctx.close()


# ---------------------------------------- column formats on row tiles (GPU-transposed slice)
@pytest.mark.parametrize("fmt", ["csc", "coo_col", "coo_unsorted"])
def test_col_row_tiles_repartition_reproducible(fmt):
    """The GPU transposition is a stable sort: partitioning the same matrix twice builds the same
    layout, so U[-1,1) results are bit-identical across partitions (not just across calls); the
    layout is reported (stats col_layout 1; bands 0) and both layouts agree within tau."""
    import paper_2209_07552_b200 as M
    A = gen.rmat(15, seed=151)
    x = gen.vector(A["n"], 152); y = gen.vector(A["m"], 153)
    outs, lays = [], []
    for lay in ("", ":bands", ""):
        ctx = M.Context(0, 1, None, 0, 3)
        outs.append(run_gpu(as_fmt(A, fmt), fmt + lay, x, y, 1.5, 0.5, ctx=ctx))
        lays.append(ctx.stats()["col_layout"])
        ctx.close()
    assert lays == [1, 0, 1]
    assert np.array_equal(outs[0], outs[2])
    for o in outs:
        assert_close(o, oracle_ref(A, x, y, 1.5, 0.5), row_bound(A, x, y, 1.5, 0.5), np.float64)


@pytest.mark.parametrize("m", [1, 2, 255, 256, 257, 65536, 65537])
def test_col_row_tiles_radix_passes(m):
    """Row counts around the radix digit boundaries (0..3 passes of 8 bits, m = 1 needs none) and
    duplicate (row, col) entries in a column: bit-exact on integer data; the rows are tall enough
    that the sort's 4096-entry tiles and ragged last tile are all exercised."""
    rng = np.random.default_rng(m)
    n = 700
    nz = 30_000
    rows = rng.integers(0, m, nz)
    cols = np.sort(rng.integers(0, n, nz))
    ptr = np.zeros(n + 1, np.int64)
    np.add.at(ptr, cols + 1, 1)
    vals = rng.integers(-4, 5, nz).astype(np.float64)
    A = gen.Sparse(fmt="csc", m=m, n=n, ptr=np.cumsum(ptr), idx=rows.astype(np.int32), val=vals)
    x = gen.vector(n, 154, kind=gen.SMALLINT); y = gen.vector(m, 155, kind=gen.SMALLINT)
    for parts in (1, 4):
        check(A, "csc", x, y, 1.5, 0.5, parts=parts, exact=True)
