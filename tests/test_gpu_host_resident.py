"""GPU parity of the host-resident (out-of-core) mode, MSREP_RESIDENT_HOST (
the paper's timed regime): the device layout is parked in pinned host memory and every
call streams it back in chunks through two staging buffers.  Same kernels, same merge, so the
integer-data cases are compared BIT-FOR-BIT against the oracle (pin P5), with chunk sizes that
force one tile / band per chunk, many chunks, and a single chunk."""
import numpy as np
import pytest

import gen
from tests.helpers import apply_layout, assert_close, coo_of_csr, oracle_ref, row_bound, run_gpu, to_dtype
from tests.test_gpu_parity import FMTS, as_fmt

pytestmark = pytest.mark.gpu

CHUNKS = [1, 64 << 10, 0]   # 1 byte: one tile (or band) per chunk; 64 KiB: many; 0: default (one)


def _ctx_partition(M, B, fmt, parts, **kw):
    ctx = M.Context(0, 1, None, 0, parts)
    fmt = apply_layout(ctx, fmt)
    if fmt in ("coo", "coo_col"):
        ctx.partition(fmt, B["m"], B["n"], idx=B["idx"], val=B["val"], coo_row=coo_of_csr(B), **kw)
    else:
        ctx.partition(fmt, B["m"], B["n"], ptr=B["ptr"], idx=B["idx"], val=B["val"], **kw)
    return ctx


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("parts", [1, 3])
@pytest.mark.parametrize("chunk", CHUNKS)
def test_host_resident_bit_exact(fmt, parts, chunk):
    """R-MAT (SEG tiles, slabs, split rows), the stencil (SELL tiles), a chain row: bit-exact,
    alpha/beta with beta = 0 and alpha = 0; three calls on one context give identical bits
    (the staging buffers are reused across calls)."""
    import paper_2209_07552_b200 as M
    import torch
    cases = [gen.rmat(11, seed=91, kind=gen.SMALLINT), gen.stencil27(11, kind=gen.SMALLINT),
             gen.Sparse(fmt="csr", m=1, n=5000, ptr=np.array([0, 5000], np.int64),
                        idx=np.arange(5000, dtype=np.int32), val=np.ones(5000))]
    for A in cases:
        B = as_fmt(A, fmt)
        x = gen.vector(A["n"], 92, kind=gen.SMALLINT); y = gen.vector(A["m"], 93, kind=gen.SMALLINT)
        ctx = _ctx_partition(M, B, fmt, parts, residency="host", chunk_bytes=chunk)
        st = ctx.stats()
        assert st["residency"] == M.RESIDENT_HOST and st["host_bytes"] > 0
        if chunk == 1:
            assert st["nchunks"] >= 1
        xd = torch.as_tensor(x).cuda()
        for alpha, beta in ((1.5, 0.5), (2.0, 0.0), (0.0, -1.0)):
            outs = []
            for _ in range(3):
                yd = torch.as_tensor(y.copy()).cuda()
                ctx.spmv(alpha, xd, beta, yd)
                torch.cuda.synchronize()
                outs.append(yd.cpu().numpy())
            ref = oracle_ref(A, x, y, alpha, beta)
            for o in outs:
                assert np.array_equal(o, ref), (fmt, parts, chunk, alpha, beta)
        ctx.close()


@pytest.mark.parametrize("fmt", FMTS)
def test_host_resident_many_chunks_counted(fmt):
    """A 64 KiB chunk over a ~6 MB layout gives many chunks; every chunk's kernel is launched
    (kernels_per_spmv counts them) and the result is bit-exact."""
    import paper_2209_07552_b200 as M
    A = gen.rmat(15, seed=94, kind=gen.SMALLINT)
    B = as_fmt(A, fmt)
    ctx = _ctx_partition(M, B, fmt, 2, residency="host", chunk_bytes=64 << 10)
    st = ctx.stats()
    # row formats: chunks are tile ranges; pCSC: whole 8192-row bands (R-MAT scale 15: 4 bands)
    assert st["nchunks"] > (10 if fmt in ("csr", "coo") else 2), st
    assert st["kernels_per_spmv"] >= st["nchunks"]
    x = gen.vector(A["n"], 95, kind=gen.SMALLINT); y = gen.vector(A["m"], 96, kind=gen.SMALLINT)
    got = run_gpu(B, fmt, x, y, 1.5, 0.5, ctx=ctx)
    assert np.array_equal(got, oracle_ref(A, x, y, 1.5, 0.5))
    ctx.close()


@pytest.mark.parametrize("fmt", ["csc:bands", "csc"])
def test_host_resident_csc_split_items(fmt):
    """pCSC with fewer row bands than SMs (split-item units) streamed band range by band range; the
    same matrix on row tiles streamed tile range by tile range."""
    A = gen.kdistinct_csr(3 * 8192 - 5, 300_000, 40, seed=97, kind=gen.SMALLINT)
    x = gen.vector(A["n"], 98, kind=gen.SMALLINT); y = gen.vector(A["m"], 99, kind=gen.SMALLINT)
    for chunk in (1, 1 << 20, 0):
        for parts in (1, 2):
            got = run_gpu(as_fmt(A, fmt), fmt, x, y, 1.5, 0.5, parts=parts, residency="host", chunk_bytes=chunk)
            assert np.array_equal(got, oracle_ref(A, x, y, 1.5, 0.5)), (chunk, parts)


@pytest.mark.parametrize("fmt", FMTS)
def test_host_resident_fp32_tolerance(fmt):
    A = to_dtype(gen.rmat(12, seed=100), np.float32)
    x = gen.vector(A["n"], 101, dtype=np.float32); y = gen.vector(A["m"], 102, dtype=np.float32)
    got = run_gpu(as_fmt(A, fmt), fmt, x, y, 1.5, 0.5, parts=2, residency="host", chunk_bytes=32 << 10)
    assert_close(got, oracle_ref(A, x, y, 1.5, 0.5), row_bound(A, x, y, 1.5, 0.5), np.float32)


@pytest.mark.parametrize("fmt", ["csr", "coo"])
def test_host_resident_spmm_and_cg(fmt):
    """SpMM (k = 4) and CG run over the streamed layout: SpMM bit-exact vs k oracle SpMVs; CG
    takes the same iterates as the device-resident layout (same kernels, same order)."""
    import paper_2209_07552_b200 as M
    import torch
    A = gen.rmat(11, seed=103, kind=gen.SMALLINT)
    rng = np.random.default_rng(104)
    X = rng.integers(-4, 5, (A["n"], 4)).astype(np.float64)
    Y = rng.integers(-4, 5, (A["m"], 4)).astype(np.float64)
    ctx = _ctx_partition(M, A, fmt, 3, residency="host", chunk_bytes=16 << 10)
    Xd = torch.as_tensor(X).cuda(); Yd = torch.as_tensor(Y.copy()).cuda()
    ctx.spmm(1.5, Xd, 0.5, Yd)
    torch.cuda.synchronize()
    ref = np.stack([oracle_ref(A, X[:, j].copy(), Y[:, j].copy(), 1.5, 0.5) for j in range(4)], axis=1)
    assert np.array_equal(Yd.cpu().numpy(), ref)
    ctx.close()
    # CG on the SPD stencil (diag 30, off -1): host- and device-resident give identical iterates
    S = gen.stencil27(10, kind=gen.ONES)
    rows = np.repeat(np.arange(S["m"]), np.diff(S["ptr"]))
    S["val"] = np.where(S["idx"] == rows, 30.0, -1.0)
    b = torch.as_tensor((np.arange(S["m"]) % 5 - 2).astype(np.float64)).cuda()
    res = []
    for kw in ({}, {"residency": "host", "chunk_bytes": 8 << 10}):
        ctx = _ctx_partition(M, S, fmt, 2, **kw)
        xd = torch.zeros(S["m"], dtype=torch.float64, device="cuda")
        it, rr = ctx.cg(b, xd, tol=1e-10, maxit=200, check_every=2)   # even checks: graph and eager loops agree
        res.append((it, rr, xd.cpu().numpy()))
        ctx.close()
    assert res[0][0] == res[1][0] and np.array_equal(res[0][2], res[1][2])


@pytest.mark.parametrize("fmt", ["csr", "csc", "csc:bands"])
def test_host_resident_config2_full_size(fmt):
    """The full N=127 stencil (config 2) streamed from host memory in 64 MiB chunks: closed form
    (interior 0, faces 9, edges 15, corners 19) and bit-exact integer parity."""
    A = gen.stencil27(127, kind=gen.STENCIL_PIN)
    m = A["m"]
    got = run_gpu(as_fmt(A, fmt), fmt, np.ones(m), np.zeros(m), 1.0, 0.0, residency="host", chunk_bytes=64 << 20)
    assert set(np.unique(got).tolist()) == {0.0, 9.0, 15.0, 19.0}
    assert int((got == 0).sum()) == 125 ** 3
    A = gen.stencil27(127, kind=gen.SMALLINT)
    x = gen.vector(m, 5, kind=gen.SMALLINT); y = gen.vector(m, 6, kind=gen.SMALLINT)
    got = run_gpu(as_fmt(A, fmt), fmt, x, y, 1.5, 0.5, residency="host", chunk_bytes=64 << 20)
    assert np.array_equal(got, oracle_ref(A, x, y, 1.5, 0.5))


def test_set_residency_rejects():
    import paper_2209_07552_b200 as M
    ctx = M.Context(0, 1, None, 0, 1)
    with pytest.raises(M.MsrepError) as e:
        M.msrep_set_residency(ctx.h, 7, 0)
    assert e.value.status == 1
    with pytest.raises(M.MsrepError) as e:
        M.msrep_set_residency(ctx.h, M.RESIDENT_HOST, -1)
    assert e.value.status == 1
    ctx.close()


@pytest.mark.parametrize("fmt", ["csr", "csc"])
def test_host_resident_pinned_on_gpu_numa_node(fmt):
    """P:561-567 (Sec. 4.2): the pinned host copy of the partition is allocated on the GPU's own NUMA
    node (sysfs numa_node of the GPU's PCI function); the page's node is read back with
    get_mempolicy.  Boxes without NUMA information report -1 for both."""
    import paper_2209_07552_b200 as M
    A = gen.rmat(14, seed=95, kind=gen.SMALLINT)
    B = A if fmt == "csr" else gen.transpose(A)
    ctx = M.Context(0, 1, None, 0, 1)
    ctx.partition(fmt, A["m"], A["n"], ptr=B["ptr"], idx=B["idx"], val=B["val"], residency="host", chunk_bytes=1 << 20)
    st = ctx.stats()
    ctx.close()
    if st["gpu_numa_node"] >= 0:
        assert st["host_numa_node"] == st["gpu_numa_node"], st
    else:
        assert st["host_numa_node"] in (-1, 0)
