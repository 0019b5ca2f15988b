"""SpMM (k right-hand sides) vs k SpMVs on one B200: the matrix streamed once for k vectors.
  python tools/spmm_bench.py [--config stencil|rmat] [--format csr|coo]  -> JSON lines"""
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
ap.add_argument("--config", default="stencil")
ap.add_argument("--format", default="csr")
ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()
A = gen.make_config(a.config)
ctx = M.Context(0, 1, None, 0, 1)
coo = a.format == "coo"
ctx.partition(a.format, A["m"], A["n"], ptr=None if coo else A["ptr"], idx=A["idx"], val=A["val"],
              coo_row=gen.expand_rows(A) if coo else None)
st = ctx.stats()


def timed(f):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


x = torch.as_tensor(gen.vector(A["n"], 1)).cuda()
y = torch.as_tensor(gen.vector(A["m"], 2)).cuda()
t1 = timed(lambda: ctx.spmv(1.5, x, 0.5, y))
for k in (2, 4, 8):
    X = torch.rand((A["n"], k), dtype=torch.float64, device="cuda")
    Y = torch.rand((A["m"], k), dtype=torch.float64, device="cuda")
    tk = timed(lambda: ctx.spmm(1.5, X, 0.5, Y))
    mat = st["tile_bytes"]
    vec = (A["n"] + 2 * A["m"]) * k * 8
    print(json.dumps({"workload": f"{a.config}_{a.format}_f64", "k": k, "spmm_ms": tk, "spmv_ms": t1,
                      "speedup_vs_k_spmv": k * t1 / tk, "GFLOPs": 2.0 * A.nnz * k / (tk * 1e-3) / 1e9,
                      "GBps_matrix_plus_XY": (mat + vec) / (tk * 1e-3) / 1e9}), flush=True)
