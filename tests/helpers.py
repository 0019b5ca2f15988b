"""Shared test helpers: run the CUDA path through the C ABI and compare with the oracle."""
import numpy as np

import gen
import oracle

TAU = {np.float64: 1e-12, np.float32: 1e-5}   # north_star per-row tolerance


def coo_of_csr(A):
    return gen.expand_rows(A)


def shuffled_triplets(A, seed=77):
    """The triplets of a CSR gen.Sparse in a seeded random order (row, col, val)."""
    rows = gen.expand_rows(A)
    perm = np.random.default_rng(seed).permutation(A.nnz)
    return rows[perm].copy(), A["idx"][perm].copy(), A["val"][perm].copy()


def to_dtype(A, dtype):
    B = gen.Sparse(A)
    B["val"] = A["val"].astype(dtype)
    return B


def oracle_ref(A, x, y, alpha, beta):
    """Oracle y for a CSR or CSC gen.Sparse (plain definition, fp64 accumulation)."""
    if A["fmt"] == "csr":
        return oracle.spmv_csr(A["m"], A["ptr"], A["idx"], A["val"], x, y, alpha, beta)
    return oracle.spmv_csc(A["m"], A["n"], A["ptr"], A["idx"], A["val"], x, y, alpha, beta)


def row_bound(A, x, y, alpha, beta):
    if A["fmt"] == "csc":
        A = gen.transpose(gen.Sparse(A, val=A["val"].astype(np.float64)))
        x = x.astype(np.float64); y = y.astype(np.float64)
        return oracle.row_bound_csr(A["m"], A["ptr"], A["idx"], A["val"], x, y, alpha, beta)
    return oracle.row_bound_csr(A["m"], A["ptr"], A["idx"], A["val"], x, y, alpha, beta)


def assert_close(got, ref, bound, dtype):
    tau = TAU[np.dtype(dtype).type]
    got = np.asarray(got, np.float64); ref = np.asarray(ref, np.float64)
    err = np.abs(got - ref)
    # fp32 output is rounded once to fp32: allow half an ulp of the result on top of tau*bound
    slack = tau * bound
    if np.dtype(dtype) == np.float32:
        slack = slack + np.abs(ref) * 2.0 ** -24
    bad = ~(err <= slack)
    assert not bad.any(), (f"{bad.sum()} rows out of tolerance; first {np.nonzero(bad)[0][:5]}: "
                           f"got {got[bad][:5]} ref {ref[bad][:5]} bound {bound[bad][:5]}")


# A column format may carry a device-layout suffix: "csc:bands" / "coo_col:bands" /
# "coo_unsorted:bands" select the host-built row bands (csc_band_kernel), "...:tiles" the row tiles
# over the GPU-transposed slice (the default for the column formats).
LAYOUT_SUFFIX = {"bands": 0, "tiles": 1}


def split_fmt(fmt):
    """'csc:bands' -> ('csc', {'col_layout': 0}); 'csr' -> ('csr', {})."""
    base, _, lay = fmt.partition(":")
    return base, ({"col_layout": LAYOUT_SUFFIX[lay]} if lay else {})


def apply_layout(ctx, fmt):
    """set the context's tuning for fmt's layout suffix; return the base format"""
    base, tun = split_fmt(fmt)
    for k, v in tun.items():
        ctx.set_tuning(k, v)
    return base


def run_gpu(A, fmt, x, y, alpha, beta, parts=1, layout=None, host_path=False, ctx=None, repeat=1, **pkw):
    """Partition A (gen.Sparse CSR or CSC) as `fmt` on cuda:0 with `parts` virtual parts; return y."""
    import torch
    import paper_2209_07552_b200 as M
    vdt = A["val"].dtype
    own = ctx is None
    if own:
        ctx = M.Context(0, 1, None, 0, parts)
    fmt = apply_layout(ctx, fmt)
    if fmt == "csr":
        assert A["fmt"] == "csr"
        ctx.partition("csr", A["m"], A["n"], ptr=A["ptr"], idx=A["idx"], val=A["val"], **pkw)
    elif fmt == "coo":
        assert A["fmt"] == "csr"
        ctx.partition("coo", A["m"], A["n"], idx=A["idx"], val=A["val"], coo_row=coo_of_csr(A), **pkw)
    elif fmt == "coo_col":   # column-sorted COO: coo_row carries the sorted column ids
        assert A["fmt"] == "csc"
        ctx.partition("coo_col", A["m"], A["n"], idx=A["idx"], val=A["val"], coo_row=coo_of_csr(A), **pkw)
    elif fmt == "coo_unsorted":   # any triplet order: A is CSR, shuffled with a seeded permutation
        assert A["fmt"] == "csr"
        r, c, v = shuffled_triplets(A)
        ctx.partition("coo_unsorted", A["m"], A["n"], idx=c, val=v, coo_row=r, **pkw)
    else:
        assert A["fmt"] == "csc"
        ctx.partition("csc", A["m"], A["n"], ptr=A["ptr"], idx=A["idx"], val=A["val"], **pkw)
    if layout is None:
        layout = M.Y_REPLICATED
    if host_path:
        yh = np.array(y, dtype=vdt, copy=True)
        ctx.spmv_host(alpha, np.ascontiguousarray(x, vdt), beta, yh, layout)
        out = yh
    else:
        tdt = torch.float64 if vdt == np.float64 else torch.float32
        xd = torch.as_tensor(np.ascontiguousarray(x, vdt)).to("cuda:0")
        outs = []
        for _ in range(repeat):
            yd = torch.as_tensor(np.array(y, dtype=vdt, copy=True)).to("cuda:0")
            ctx.spmv(alpha, xd, beta, yd, layout)
            torch.cuda.synchronize()
            outs.append(yd.cpu().numpy())
        out = outs[0] if repeat == 1 else outs
    if own:
        ctx.close()
    return out
