"""GPU parity of unsorted pCOO (MSREP_COO_UNSORTED; Sec. 3.2.3: "if the elements are
unsorted ... elements in a particular partition can spread among the entire matrix"): the nnz split
by position, per-rank column sort at partition time, the pCSC band kernel, and the column-style
merge.  Integer data: bit-exact against the oracle for any triplet order."""
import numpy as np
import pytest

import gen
import oracle
from tests.helpers import assert_close, oracle_ref, row_bound, run_gpu, shuffled_triplets, to_dtype

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("parts", [1, 2, 3, 5, 7])
def test_unsorted_fixture_E(golden_E, parts):
    g = golden_E
    A = gen.Sparse(fmt="csr", m=4, n=4, ptr=np.array(g["csr_row_ptr"], np.int64),
                   idx=np.array(g["csr_col_idx"], np.int32), val=np.array(g["csr_val"]))
    for case in g["spmv"]:
        got = run_gpu(A, "coo_unsorted", np.array(case["x"], float), np.array(case["y"], float),
                      case["alpha"], case["beta"], parts=parts)
        assert got.tolist() == case["expect"]


@pytest.mark.parametrize("fmt", ["coo_unsorted", "coo_unsorted:bands"])
@pytest.mark.parametrize("parts", [1, 3, 5])
def test_unsorted_rmat_bit_exact(fmt, parts):
    A = gen.rmat(15, seed=81, kind=gen.SMALLINT)
    x = gen.vector(A["n"], 82, kind=gen.SMALLINT); y = gen.vector(A["m"], 83, kind=gen.SMALLINT)
    for alpha, beta in [(1.5, 0.5), (2.0, 0.0), (0.0, -1.0), (-1.0, 1.0)]:
        got = run_gpu(A, fmt, x, y, alpha, beta, parts=parts)
        r, c, v = shuffled_triplets(A)
        assert np.array_equal(got, oracle.exec_coo_unsorted(A["m"], r, c, v, x, y, alpha, beta, parts))
        assert np.array_equal(got, oracle_ref(A, x, y, alpha, beta))


@pytest.mark.parametrize("fmt", ["coo_unsorted", "coo_unsorted:bands"])
def test_unsorted_stencil_and_wide_bit_exact(fmt):
    for A in (gen.stencil27(30, kind=gen.SMALLINT), gen.kdistinct_csr(2000, 300_000, 40, seed=84, kind=gen.SMALLINT)):
        x = gen.vector(A["n"], 85, kind=gen.SMALLINT); y = gen.vector(A["m"], 86, kind=gen.SMALLINT)
        got = run_gpu(A, fmt, x, y, 1.5, 0.5, parts=3)
        assert np.array_equal(got, oracle_ref(A, x, y, 1.5, 0.5))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_unsorted_uniform_tolerance(dtype):
    A = to_dtype(gen.rmat(14, seed=87), dtype)
    x = gen.vector(A["n"], 88, dtype=dtype); y = gen.vector(A["m"], 89, dtype=dtype)
    got = run_gpu(A, "coo_unsorted", x, y, 1.5, 0.5, parts=4)
    assert_close(got, oracle_ref(A, x, y, 1.5, 0.5), row_bound(A, x, y, 1.5, 0.5), dtype)


def test_unsorted_descriptors_and_errors():
    import paper_2209_07552_b200 as M
    A = gen.rmat(12, seed=90, kind=gen.SMALLINT)
    r, c, v = shuffled_triplets(A)
    ctx = M.Context(0, 1, None, 0, 4)
    parts = ctx.partition("coo_unsorted", A["m"], A["n"], idx=c, val=v, coo_row=r)
    ref = oracle.partition_coo_unsorted(r, 4)
    for k in ("start_idx", "end_idx", "start_row", "end_row", "start_flag", "owned_begin", "owned_end"):
        assert np.array_equal(parts[k], ref[k]), k
    with pytest.raises(M.MsrepError):   # row blocks do not exist for an unsorted list
        ctx.partition("coo_unsorted", A["m"], A["n"], idx=c, val=v, coo_row=r, split="block")
    bad = r.copy(); bad[5] = A["m"]
    with pytest.raises(M.MsrepError) as e:
        ctx.partition("coo_unsorted", A["m"], A["n"], idx=c, val=v, coo_row=bad)
    assert e.value.status == 2
    ctx.close()


@pytest.mark.parametrize("fmt", ["coo_unsorted", "coo_unsorted:bands"])
def test_unsorted_host_resident(fmt):
    A = gen.rmat(14, seed=91, kind=gen.SMALLINT)
    x = gen.vector(A["n"], 92, kind=gen.SMALLINT); y = gen.vector(A["m"], 93, kind=gen.SMALLINT)
    got = run_gpu(A, fmt, x, y, 1.5, 0.5, parts=3, residency="host", chunk_bytes=1 << 16)
    assert np.array_equal(got, oracle_ref(A, x, y, 1.5, 0.5))
