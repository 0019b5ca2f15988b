"""The N > 1 merge executed on ONE B200 (Sec. 4.3; P:529 one worker per
GPU): msrep_create_loopback gives N ranks of this process on cuda:0, each driven by its own host
thread and stream, whose collectives meet in-process instead of in NCCL.  Every device kernel of
the multi-rank path runs for real -- head partials (heads_kernel) + all-gather, the owner fix-up
with routed heads, allgatherv of the owned segments, the fp64 partial-y reduce-scatter and the
shard epilogue, the REPLICATED / OWNED / SHARDED layouts, SpMM k-wide heads, CG with all-reduced
dot products, the fused mirror stores into the peers' y and their fence.  Integer data: each rank's
result equals the single-process oracle BIT FOR BIT."""
import threading

import numpy as np
import pytest

import gen
import oracle
from tests.helpers import apply_layout, coo_of_csr, oracle_ref, shuffled_triplets, split_fmt

pytestmark = pytest.mark.gpu
# column formats on row tiles (default; fp64 / fp32 partial y reduce-scattered) and on row bands
FMTS = ["csr", "coo", "csc", "coo_col", "coo_unsorted", "csc:bands", "coo_unsorted:bands"]


def _run_ranks(world, ppr, body):
    """body(rank, ctx, stream) on `world` threads over one loopback group; returns per-rank results."""
    import torch
    import paper_2209_07552_b200 as M
    ctxs = M.Context.loopback_group(world, 0, ppr)
    out, errs = [None] * world, []

    def run(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                out[r] = body(r, ctxs[r], st)
            st.synchronize()
        except Exception as e:   # noqa: BLE001
            errs.append((r, repr(e)))
    th = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    for c in ctxs:
        c.close()
    assert not errs, errs
    return out


def _partition(ctx, fmt, A, T, split, stream):
    sh = stream.cuda_stream
    fmt = apply_layout(ctx, fmt)
    if fmt == "coo_unsorted":
        r, c, v = shuffled_triplets(A)
        ctx.partition(fmt, A["m"], A["n"], idx=c, val=v, coo_row=r, stream=sh, split=split)
    elif fmt in ("coo", "coo_col"):
        B = T if fmt == "coo_col" else A
        ctx.partition(fmt, A["m"], A["n"], idx=B["idx"], val=B["val"], coo_row=coo_of_csr(B), stream=sh, split=split)
    else:
        B = T if fmt == "csc" else A
        ctx.partition(fmt, A["m"], A["n"], ptr=B["ptr"], idx=B["idx"], val=B["val"], stream=sh, split=split)


def _segments(fmt, A, world, ppr, split):
    import paper_2209_07552_b200 as M
    fmt = split_fmt(fmt)[0]
    ptr = coo = None
    if fmt == "csr":
        ptr = A["ptr"]
    elif fmt == "csc":
        ptr = gen.transpose(A)["ptr"]
    elif fmt == "coo":
        coo = coo_of_csr(A)
    elif fmt == "coo_col":
        coo = coo_of_csr(gen.transpose(A))
    else:
        coo = shuffled_triplets(A)[0]
    seg, _, _ = M.msrep_exchange_plan(M.FORMATS[fmt], A["m"], A["n"], A.nnz, world, ppr, ptr=ptr, coo_row=coo,
                                      split=M.SPLITS[split])
    return seg


CASES = {
    "rmat13": lambda: gen.rmat(13, seed=301, kind=gen.SMALLINT),
    "chain": lambda: gen.Sparse(fmt="csr", m=3, n=5000, ptr=np.array([0, 1, 4999, 5000], np.int64),
                                idx=np.concatenate([[7], np.arange(4998), [3]]).astype(np.int32), val=np.ones(5000)),
    "stencil": lambda: gen.stencil27(14, kind=gen.SMALLINT),
}


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("world,ppr", [(2, 1), (3, 2), (4, 1)])
def test_loopback_spmv_all_layouts_bit_exact(fmt, world, ppr):
    import torch
    import paper_2209_07552_b200 as M
    for name, mk in CASES.items():
        A = mk()
        T = gen.transpose(A)
        x = gen.vector(A["n"], 302, kind=gen.SMALLINT); y = gen.vector(A["m"], 303, kind=gen.SMALLINT)
        splits = ["nnz"] if fmt.startswith("coo_unsorted") else ["nnz", "block"]
        for split in splits:
            seg = _segments(fmt, A, world, ppr, split)
            layouts = [M.Y_REPLICATED, M.Y_SHARDED if split_fmt(fmt)[0] in ("csc", "coo_col", "coo_unsorted") else M.Y_OWNED]
            for alpha, beta in [(1.5, -0.5), (2.0, 0.0), (0.0, 2.0)]:
                ref = oracle_ref(A, x, y, alpha, beta)

                def body(r, ctx, st):
                    _partition(ctx, fmt, A, T, split, st)
                    res = []
                    for lay in layouts:
                        yd = torch.as_tensor(y).cuda()
                        ctx.spmv(alpha, torch.as_tensor(x).cuda(), beta, yd, lay, st.cuda_stream)
                        st.synchronize()
                        res.append(yd.cpu().numpy())
                    yh = y.copy()   # host-vector path, REPLICATED
                    ctx.spmv_host(alpha, x, beta, yh, M.Y_REPLICATED, st.cuda_stream)
                    res.append(yh)
                    return res
                outs = _run_ranks(world, ppr, body)
                for r, (rep, part, host) in enumerate(outs):
                    tag = (name, fmt, split, world, ppr, alpha, beta, r)
                    assert np.array_equal(rep, ref), tag
                    assert np.array_equal(host, ref), tag
                    lo, hi = seg[r]
                    assert np.array_equal(part[lo:hi], ref[lo:hi]), tag


@pytest.mark.parametrize("fmt", ["csr", "coo", "csc", "csc:bands"])
def test_loopback_spmm_bit_exact(fmt):
    import torch
    A = gen.rmat(12, seed=304, kind=gen.SMALLINT)
    T = gen.transpose(A)
    k = 4
    rng = np.random.default_rng(5)
    X = rng.integers(-4, 5, (A["n"], k)).astype(np.float64)
    Y = rng.integers(-4, 5, (A["m"], k)).astype(np.float64)
    ref = np.stack([oracle_ref(A, X[:, j].copy(), Y[:, j].copy(), 1.5, 0.5) for j in range(k)], 1)

    def body(r, ctx, st):
        _partition(ctx, fmt, A, T, "nnz", st)
        Yd = torch.as_tensor(Y.copy()).cuda()
        ctx.spmm(1.5, torch.as_tensor(X).cuda(), 0.5, Yd, stream=st.cuda_stream)
        st.synchronize()
        return Yd.cpu().numpy()
    for out in _run_ranks(3, 2, body):
        assert np.array_equal(out, ref)


def test_loopback_mirror_fused_allgather():
    """msrep_spmv_mirror with the peers' y as mirrors (same device): every rank stores its owned rows
    into every peer's y from the kernel epilogue; after the fence every y is the whole result."""
    import torch
    A = gen.rmat(13, seed=305, kind=gen.SMALLINT)
    x = gen.vector(A["n"], 306, kind=gen.SMALLINT); y = gen.vector(A["m"], 307, kind=gen.SMALLINT)
    ref = oracle_ref(A, x, y, 1.5, 0.5)
    world = 3
    ys = [torch.as_tensor(y.copy()).cuda() for _ in range(world)]
    torch.cuda.synchronize()

    def body(r, ctx, st):
        _partition(ctx, "csr", A, None, "nnz", st)
        ctx.spmv_mirror(1.5, torch.as_tensor(x).cuda(), 0.5, ys[r], [ys[q] for q in range(world) if q != r],
                        st.cuda_stream)
        st.synchronize()
        return True
    _run_ranks(world, 1, body)
    torch.cuda.synchronize()
    for r in range(world):
        assert np.array_equal(ys[r].cpu().numpy(), ref), r


@pytest.mark.parametrize("fmt", ["csr", "csc", "csc:bands"])
def test_loopback_cg(fmt):
    import torch
    S = gen.stencil27(10, kind=gen.ONES)
    rows = np.repeat(np.arange(S["m"]), np.diff(S["ptr"]))
    S["val"] = np.where(S["idx"] == rows, 30.0, -1.0)
    T = gen.transpose(S)
    xs = (np.arange(S["m"]) % 5 - 2).astype(np.float64)
    b = oracle.spmv_csr(S["m"], S["ptr"], S["idx"], S["val"], xs, np.zeros(S["m"]), 1.0, 0.0)

    def body(r, ctx, st):
        _partition(ctx, fmt, S, T, "nnz", st)
        xc = torch.zeros(S["m"], dtype=torch.float64, device="cuda")
        it, rr = ctx.cg(torch.as_tensor(b).cuda(), xc, tol=1e-12, maxit=300, stream=st.cuda_stream)
        return it, rr, xc.cpu().numpy()
    outs = _run_ranks(3, 1, body)
    for it, rr, xv in outs:
        assert rr <= 1e-12 and np.max(np.abs(xv - xs)) < 1e-9
    assert len({o[0] for o in outs}) == 1
    assert all(np.array_equal(outs[0][2], o[2]) for o in outs)   # replicated, identical iterates


@pytest.mark.parametrize("fmt", ["csr", "csc"])
@pytest.mark.parametrize("world,ppr", [(2, 1), (4, 2)])
def test_loopback_partition_slice_rank_local(fmt, world, ppr):
    """bench.py's N > 1 path: every rank holds ONLY the entries of the rows (columns) its nonzero range
    touches -- gen.config_rows-style slices -- and partitions through msrep_partition_slice; the merged
    result equals the oracle bit for bit."""
    import torch
    import paper_2209_07552_b200 as M
    A = gen.rmat(13, seed=308, kind=gen.SMALLINT)
    B = A if fmt == "csr" else gen.transpose(A)
    x = gen.vector(A["n"], 309, kind=gen.SMALLINT); y = gen.vector(A["m"], 310, kind=gen.SMALLINT)
    ref = oracle_ref(A, x, y, 1.5, 0.5)
    outer = A["m"] if fmt == "csr" else A["n"]
    parts = M.msrep_plan(M.FORMATS[fmt], outer, A.nnz, world * ppr, ptr=B["ptr"])

    def body(r, ctx, st):
        mine = parts[r * ppr:(r + 1) * ppr]
        ne = mine[mine["start_row"] >= 0]
        r0, r1 = int(ne["start_row"][0]), int(ne["end_row"][-1]) + 1
        z0, z1 = int(B["ptr"][r0]), int(B["ptr"][r1])
        ctx.partition_slice(fmt, A["m"], A["n"], B["ptr"], B["idx"][z0:z1].copy(), B["val"][z0:z1].copy(), z0,
                            stream=st.cuda_stream)
        yd = torch.as_tensor(y).cuda()
        ctx.spmv(1.5, torch.as_tensor(x).cuda(), 0.5, yd, M.Y_REPLICATED, st.cuda_stream)
        st.synchronize()
        return yd.cpu().numpy()
    for out in _run_ranks(world, ppr, body):
        assert np.array_equal(out, ref)


def test_partition_slice_rejects_short_slice():
    import paper_2209_07552_b200 as M
    A = gen.rmat(10, seed=311, kind=gen.SMALLINT)
    ctx = M.Context(0, 1, None, 0, 1)
    with pytest.raises(M.MsrepError) as e:   # one rank holds everything: a partial slice is rejected
        ctx.partition_slice("csr", A["m"], A["n"], A["ptr"], A["idx"][5:].copy(), A["val"][5:].copy(), 5)
    assert e.value.status == 1
    ctx.close()


@pytest.mark.parametrize("fmt", ["csr", "coo", "csc", "coo_unsorted"])
def test_loopback_hot_and_compact_x(fmt):
    """Per-rank hot-x cache and compact x (forced on: the auto rules need bigger slices) under the
    multi-rank merge: each rank relabels its own columns; results stay bit-exact."""
    import torch
    import paper_2209_07552_b200 as M
    A = gen.rmat(17, seed=312, kind=gen.SMALLINT)   # big enough that every rank has columns of >= 4 gathers per SM
    x = gen.vector(A["n"], 313, kind=gen.SMALLINT); y = gen.vector(A["m"], 314, kind=gen.SMALLINT)
    ref = oracle_ref(A, x, y, 1.5, 0.5)

    def body(r, ctx, st):
        ctx.set_tuning("hot_x", 1)
        ctx.set_tuning("compact_x", 1)
        _partition(ctx, fmt, A, gen.transpose(A) if fmt == "csc" else None, "nnz", st)
        s = ctx.stats()
        yd = torch.as_tensor(y).cuda()
        ctx.spmv(1.5, torch.as_tensor(x).cuda(), 0.5, yd, M.Y_REPLICATED, st.cuda_stream)
        st.synchronize()
        return s["nhot"], s["x_compact"], yd.cpu().numpy()
    outs = _run_ranks(3, 2, body)
    assert all(o[0] > 0 and o[1] > 0 for o in outs), [o[:2] for o in outs]
    for _, _, out in outs:
        assert np.array_equal(out, ref)


@pytest.mark.parametrize("fmt", ["csc", "coo_col", "coo_unsorted", "csc:bands"])
@pytest.mark.parametrize("world,ppr", [(2, 1), (3, 2)])
def test_loopback_column_formats_fp32(fmt, world, ppr):
    """fp32 column formats under the merge: on row tiles each rank's partial y is fp32 and the
    reduce-scatter sums fp32 (rank order); on row bands the partial y is fp64.  Integer data
    (|y| < 2^24): every rank's result equals the oracle bit for bit."""
    import torch
    import paper_2209_07552_b200 as M
    from tests.helpers import to_dtype
    A = to_dtype(gen.rmat(13, seed=315, kind=gen.SMALLINT), np.float32)
    T = gen.transpose(A)
    x = gen.vector(A["n"], 316, kind=gen.SMALLINT, dtype=np.float32)
    y = gen.vector(A["m"], 317, kind=gen.SMALLINT, dtype=np.float32)
    ref = oracle_ref(A, x, y, 1.5, 0.5)

    def body(r, ctx, st):
        _partition(ctx, fmt, A, T, "nnz", st)
        s = ctx.stats()
        yd = torch.as_tensor(y).cuda()
        ctx.spmv(1.5, torch.as_tensor(x).cuda(), 0.5, yd, M.Y_REPLICATED, st.cuda_stream)
        st.synchronize()
        return s["col_layout"], yd.cpu().numpy()
    for lay, out in _run_ranks(world, ppr, body):
        assert lay == (0 if fmt.endswith(":bands") else 1)
        assert out.dtype == np.float32 and np.array_equal(out, ref)
