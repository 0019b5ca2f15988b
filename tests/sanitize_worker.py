"""Small invocations of every kernel of libmsrep, for compute-sanitizer (tests/test_gpu_sanitizer.py):
rows_kernel (SELL, SEG, slab tiles; hot-x cache; compact x; mirror stores), rows_mm_kernel (SpMM),
csc_band_kernel (whole bands and split bands with the slot reduction), the GPU transposition of the
column formats (radix sort, row pointer, permute), fixup / heads, pack, rebase,
the hot-x / compact-x setup kernels, the CG vector kernels.  Checks results against the oracle too,
so a sanitizer run that changes nothing also proves the path ran."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


G = 4096                 # guard elements on both sides of every output buffer
SENT = -12345.678        # their value: any kernel store outside [0, m) changes it


def guarded(host, torch):
    """A device copy of `host` inside a larger buffer whose G leading and trailing elements hold
    SENT; returns (view, check) -- check() is True when no store landed outside the view."""
    a = np.ascontiguousarray(host)
    buf = torch.full((a.size + 2 * G,), SENT, dtype=torch.float64, device="cuda")
    buf[G:G + a.size] = torch.as_tensor(a.reshape(-1)).cuda()
    view = buf[G:G + a.size].view(a.shape)

    def check():
        b = buf.cpu().numpy()
        return bool(np.all(b[:G] == SENT) and np.all(b[G + a.size:] == SENT))
    return view, check


def main():
    import torch
    import gen
    import oracle
    import paper_2209_07552_b200 as M
    torch.cuda.set_device(0)
    fails = 0
    A = gen.rmat(11, seed=5, kind=gen.SMALLINT)          # split rows, SEG tiles, slabs
    S = gen.stencil27(9, kind=gen.SMALLINT)              # SELL tiles
    W = gen.kdistinct_csr(300, 9000, 40, seed=6, kind=gen.SMALLINT)   # short-wide: split pCSC bands
    for name, B in (("rmat", A), ("stencil", S), ("wide", W)):
        m, n = B["m"], B["n"]
        T = gen.transpose(B)
        x = gen.vector(n, 1, kind=gen.SMALLINT); y = gen.vector(m, 2, kind=gen.SMALLINT)
        ref = oracle.spmv_csr(m, B["ptr"], B["idx"], B["val"], x, y, 1.5, 0.5)
        for fmt_tag in ("csr", "coo", "csc", "coo_col", "csc:bands", "coo_col:bands"):
            fmt, _, lay = fmt_tag.partition(":")
            for hot, cx in ((0, 0), (1, 1)):
                ctx = M.Context(0, 1, None, 0, 3)
                ctx.set_tuning("col_layout", 0 if lay == "bands" else -1)
                ctx.set_tuning("hot_x", hot)
                ctx.set_tuning("compact_x", cx)
                ctx.set_tuning("xload", 0)
                C = T if fmt in ("csc", "coo_col") else B
                if fmt in ("coo", "coo_col"):
                    ctx.partition(fmt, m, n, idx=C["idx"], val=C["val"], coo_row=gen.expand_rows(C))
                else:
                    ctx.partition(fmt, m, n, ptr=C["ptr"], idx=C["idx"], val=C["val"])
                yd, yok = guarded(y, torch)
                ctx.spmv(1.5, torch.as_tensor(x).cuda(), 0.5, yd)
                torch.cuda.synchronize()
                if not (np.array_equal(yd.cpu().numpy(), ref) and yok()):
                    print("FAIL", name, fmt_tag, hot, cx, flush=True)
                    fails += 1
                if fmt == "csr":
                    k = 4
                    X = torch.as_tensor(np.stack([x] * k, 1).copy()).cuda()
                    Y, Yok = guarded(np.stack([y] * k, 1), torch)
                    ctx.spmm(1.5, X, 0.5, Y)
                    mirror, mok = guarded(np.zeros(m), torch)
                    yd, yok = guarded(y, torch)
                    ctx.spmv_mirror(1.5, torch.as_tensor(x).cuda(), 0.5, yd, [mirror])
                    torch.cuda.synchronize()
                    if not (np.array_equal(Y.cpu().numpy()[:, 2], ref) and np.array_equal(mirror.cpu().numpy(), ref)
                            and Yok() and mok() and yok()):
                        print("FAIL spmm/mirror", name, hot, cx, flush=True)
                        fails += 1
                ctx.close()
    # CG (vector kernels, graph replay)
    Q = gen.stencil27(6, kind=gen.ONES)
    rows = np.repeat(np.arange(Q["m"]), np.diff(Q["ptr"]))
    Q["val"] = np.where(Q["idx"] == rows, 30.0, -1.0)
    xs = (np.arange(Q["m"]) % 5 - 2).astype(np.float64)
    b = oracle.spmv_csr(Q["m"], Q["ptr"], Q["idx"], Q["val"], xs, np.zeros(Q["m"]), 1.0, 0.0)
    ctx = M.Context(0, 1, None, 0, 2)
    ctx.partition("csr", Q["m"], Q["n"], ptr=Q["ptr"], idx=Q["idx"], val=Q["val"])
    xc = torch.zeros(Q["m"], dtype=torch.float64, device="cuda")
    it, rr = ctx.cg(torch.as_tensor(b).cuda(), xc, tol=1e-12, maxit=100)
    ctx.close()
    if not (rr <= 1e-12 and np.max(np.abs(xc.cpu().numpy() - xs)) < 1e-9):
        print("FAIL cg", it, rr, flush=True)
        fails += 1
    print("sanitize worker:", "OK" if fails == 0 else f"{fails} FAILED", flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
