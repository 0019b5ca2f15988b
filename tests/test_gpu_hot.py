"""The hot-x cache of the row formats (msrep_set_tuning(MSREP_TUNE_HOT_X)): the
rank's most-gathered columns are served from a shared-memory copy of x.  It changes where x is
read from, never the arithmetic: forced on, forced off and automatic must all give the oracle's
bits on integer data (pin P5), for SpMV, SpMM (which untags the column ids) and the fused mirror
stores, with virtual parts (split rows, head exchange) and with SELL tiles in their own launch."""
import numpy as np
import pytest

import gen
from tests.helpers import assert_close, coo_of_csr, oracle_ref, row_bound, run_gpu

pytestmark = pytest.mark.gpu


def _ctx(hot, parts, compact=1):
    import paper_2209_07552_b200 as M
    ctx = M.Context(0, 1, None, 0, parts)
    ctx.set_tuning("hot_x", hot)
    ctx.set_tuning("compact_x", compact)
    return ctx


@pytest.mark.parametrize("fmt", ["csr", "coo", "csc"])
@pytest.mark.parametrize("parts", [1, 3])
@pytest.mark.parametrize("compact", [1, 2, 0])
def test_hot_x_bit_exact(fmt, parts, compact):
    """Hot cache forced on (also at a 4 KiB size), off and automatic, with and without compact x
    (column-ordered and degree-ordered x'); pCSC on row tiles indexes its column window."""
    A = gen.rmat(18, seed=31, kind=gen.SMALLINT)
    x = gen.vector(A["n"], 32, kind=gen.SMALLINT); y = gen.vector(A["m"], 33, kind=gen.SMALLINT)
    ref = oracle_ref(A, x, y, 1.5, 0.5)
    nhot, ncx = [], []
    for hot in (1, 4, 0, -1):
        ctx = _ctx(hot, parts, compact)
        got = run_gpu(A if fmt != "csc" else gen.transpose(A), fmt, x, y, 1.5, 0.5, ctx=ctx)
        nhot.append(ctx.stats()["nhot"])
        ncx.append(ctx.stats()["x_compact"])
        ctx.close()
        assert np.array_equal(got, ref), (fmt, parts, hot, compact)
    assert nhot[0] > 0 and 0 < nhot[1] <= 4096 // 8 and nhot[2] == 0
    assert all((v > 0) == bool(compact) for v in ncx)


@pytest.mark.parametrize("fmt", ["csr", "coo"])
def test_compact_x_stencil_and_small(fmt):
    """Compact x forced on for SELL-tile matrices (all tiles index x') and a tiny matrix."""
    for A in (gen.stencil27(30, kind=gen.SMALLINT), gen.kdistinct_csr(50, 400, 3, seed=9, kind=gen.SMALLINT)):
        x = gen.vector(A["n"], 32, kind=gen.SMALLINT); y = gen.vector(A["m"], 33, kind=gen.SMALLINT)
        ctx = _ctx(0, 2, 1)
        got = run_gpu(A, fmt, x, y, 1.5, 0.5, ctx=ctx)
        assert ctx.stats()["x_compact"] > 0
        ctx.close()
        assert np.array_equal(got, oracle_ref(A, x, y, 1.5, 0.5))


@pytest.mark.parametrize("cluster", [1, 2])
def test_hot_x_cluster_pairs_bit_exact(cluster):
    """MSREP_TUNE_HOT_CLUSTER = 2: the hot entries are split over the two CTAs of a thread-block
    cluster and read over distributed shared memory -- same bits."""
    A = gen.rmat(17, seed=38, kind=gen.SMALLINT)
    x = gen.vector(A["n"], 39, kind=gen.SMALLINT); y = gen.vector(A["m"], 40, kind=gen.SMALLINT)
    ctx = _ctx(8, 2, 1)
    ctx.set_tuning("hot_cluster", cluster)
    got = run_gpu(A, "csr", x, y, 1.5, 0.5, ctx=ctx)
    st = ctx.stats()
    ctx.close()
    assert st["nhot"] > 0
    assert np.array_equal(got, oracle_ref(A, x, y, 1.5, 0.5))


def test_hot_x_fp32_and_uniform():
    for dtype in (np.float64, np.float32):
        A = gen.rmat(17, seed=34)
        A["val"] = A["val"].astype(dtype)
        x = gen.vector(A["n"], 35, dtype=dtype); y = gen.vector(A["m"], 36, dtype=dtype)
        ctx = _ctx(1, 2, -1)
        got = run_gpu(A, "csr", x, y, 1.5, 0.5, ctx=ctx)
        assert ctx.stats()["nhot"] > 0
        ctx.close()
        assert_close(got, oracle_ref(A, x, y, 1.5, 0.5), row_bound(A, x, y, 1.5, 0.5), dtype)


def test_hot_x_with_sell_split_launch():
    """A stencil block (SELL tiles) next to an R-MAT block (SEG tiles): the SELL tiles run in their
    own launch with raw column ids, the SEG launch uses the hot cache."""
    import paper_2209_07552_b200 as M
    S = gen.stencil27(40, kind=gen.SMALLINT)
    R = gen.rmat(16, seed=37, kind=gen.SMALLINT)
    m = S["m"] + R["m"]
    n = max(S["n"], R["n"])
    ptr = np.concatenate([S["ptr"], S["ptr"][-1] + R["ptr"][1:]])
    A = gen.Sparse(fmt="csr", m=m, n=n, ptr=ptr, idx=np.concatenate([S["idx"], R["idx"]]),
                   val=np.concatenate([S["val"], R["val"]]))
    x = gen.vector(n, 38, kind=gen.SMALLINT); y = gen.vector(m, 39, kind=gen.SMALLINT)
    ctx = _ctx(1, 1)
    got = run_gpu(A, "csr", x, y, 2.0, 0.5, ctx=ctx)
    st = ctx.stats()
    ctx.close()
    assert st["nsell"] > 0 and st["nhot"] > 0
    assert np.array_equal(got, oracle_ref(A, x, y, 2.0, 0.5))


@pytest.mark.parametrize("k", [2, 4, 8])
def test_hot_x_spmm_bit_exact(k):
    import torch
    A = gen.rmat(16, seed=40, kind=gen.SMALLINT)
    m, n = A["m"], A["n"]
    X = np.stack([gen.vector(n, 41 + j, kind=gen.SMALLINT) for j in range(k)], 1)
    Y = np.stack([gen.vector(m, 51 + j, kind=gen.SMALLINT) for j in range(k)], 1)
    ctx = _ctx(1, 3)
    ctx.partition("csr", m, n, ptr=A["ptr"], idx=A["idx"], val=A["val"])
    assert ctx.stats()["nhot"] > 0
    Yd = torch.as_tensor(np.ascontiguousarray(Y)).cuda()
    ctx.spmm(1.5, torch.as_tensor(np.ascontiguousarray(X)).cuda(), 0.5, Yd)
    got = Yd.cpu().numpy()
    ctx.close()
    for j in range(k):
        assert np.array_equal(got[:, j], oracle_ref(A, X[:, j].copy(), Y[:, j].copy(), 1.5, 0.5)), j


def test_hot_x_mirror_bit_exact():
    import torch
    A = gen.rmat(16, seed=60, kind=gen.SMALLINT)
    m, n = A["m"], A["n"]
    x = gen.vector(n, 61, kind=gen.SMALLINT); y = gen.vector(m, 62, kind=gen.SMALLINT)
    ctx = _ctx(1, 2)
    ctx.partition("csr", m, n, ptr=A["ptr"], idx=A["idx"], val=A["val"])
    yd = torch.as_tensor(y).cuda()
    mirrors = [torch.zeros(m, dtype=torch.float64, device="cuda") for _ in range(2)]
    ctx.spmv_mirror(1.5, torch.as_tensor(x).cuda(), 0.5, yd, mirrors)
    ref = oracle_ref(A, x, y, 1.5, 0.5)
    assert np.array_equal(yd.cpu().numpy(), ref)
    for mm in mirrors:
        assert np.array_equal(mm.cpu().numpy(), ref)
    ctx.close()
