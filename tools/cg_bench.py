"""CG on the full-size SPD stencil (config 2's 2,048,383-row 27-point pattern, diag 30, off -1)
through msrep_cg, 1 GPU: time per iteration and the bytes it moves (one SpMV + the vector
updates).  Prints one JSON line.   python tools/cg_bench.py [--format csr] [--iters 200]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import paper_2209_07552_b200 as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--format", default="csr")
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--N", type=int, default=127, help="stencil grid edge (127: config 2)")
ap.add_argument("--graph", type=int, default=1, help="MSREP_TUNE_CG_GRAPH (1: CUDA-graph replay, 0: eager)")
a = ap.parse_args()
A = gen.stencil27(a.N, kind=gen.ONES)
rows = np.repeat(np.arange(A["m"]), np.diff(A["ptr"]))
A["val"] = np.where(A["idx"] == rows, 30.0, -1.0)
if a.format in ("csc", "coo_col"):
    A = gen.transpose(A)
ctx = M.Context(0, 1, None, 0, 1)
ctx.set_tuning("cg_graph", a.graph)
coo = a.format in ("coo", "coo_col")
ctx.partition(a.format, A["m"], A["n"], ptr=None if coo else A["ptr"], idx=A["idx"], val=A["val"],
              coo_row=gen.expand_rows(A) if coo else None)
st = ctx.stats()
b = torch.as_tensor(gen.vector(A["m"], 5)).cuda()
x = torch.zeros(A["m"], dtype=torch.float64, device="cuda")
ctx.cg(b, x, tol=0.0, maxit=5)                    # warm-up (workspace allocation)
x.zero_()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
it, rr = ctx.cg(b, x, tol=0.0, maxit=a.iters, check_every=a.iters)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / it
vec_bytes = 12 * A["m"] * 8          # dot(p,Ap) 2, update x,r (4 rd + 2 wr) 6, update p (2 rd + 1 wr) 3, residual ~1
alg = st["alg_bytes_beta0"] + vec_bytes
print(json.dumps({"what": "msrep_cg on the SPD 27-point stencil", "format": a.format,
                  "cuda_graph": bool(a.graph), "m": A["m"], "nnz": A.nnz,
                  "iterations": it, "relres": rr, "ms_per_iter": ms, "spmv_alg_bytes": st["alg_bytes_beta0"],
                  "vector_bytes": vec_bytes, "GBps": alg / (ms * 1e-3) / 1e9,
                  "x_no_allocate": st["x_no_allocate"], "sell_1cta": st["sell_1cta"], "nsell": st["nsell"],
                  "split_launch_tiles": st["ntiles"] - st["nsell"]}), flush=True)
