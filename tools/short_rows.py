"""Per-row cost of short rows: SpMV time per nonzero for matrices of exactly k
uniform random columns per row (k = 2 .. 64, ~6M nonzeros each, the size of one 8-way part of the
two-class study), with SELL tiles on and off; plus the last 8-way part of R-MAT scale 24 (millions
of irregular short rows).  One JSON line per case.   python tools/short_rows.py"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import paper_2209_07552_b200 as M  # noqa: E402


def timed(A, sell, reps=200, n=None):
    ctx = M.Context(0, 1, None, 0, 1)
    ctx.set_tuning("sell", sell)
    ctx.partition("csr", A["m"], A["n"], ptr=A["ptr"], idx=A["idx"], val=A["val"])
    st = ctx.stats()
    x = torch.as_tensor(gen.vector(A["n"], 7)).cuda()
    y = torch.zeros(A["m"], dtype=torch.float64, device="cuda")
    for _ in range(5):
        ctx.spmv(1.0, x, 0.5, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        ctx.spmv(1.0, x, 0.5, y)
    e1.record()
    torch.cuda.synchronize()
    ctx.close()
    ms = e0.elapsed_time(e1) / reps
    return ms, st


torch.cuda.set_device(0)
for k in (2, 4, 6, 8, 12, 16, 24, 32, 64):
    m = 6_250_000 // k
    A = gen.kdistinct_csr(m, 1_420_448, k, seed=600)
    for sell in (1, 0):
        ms, st = timed(A, sell)
        print(json.dumps({"k": k, "m": m, "nnz": A.nnz, "sell": sell, "ms": ms, "ns_per_nnz": ms * 1e6 / A.nnz,
                          "nsell": st["nsell"], "ntiles": st["ntiles"], "tile_bytes": st["tile_bytes"]}), flush=True)
R = gen.make_config("rmat")
plan = M.msrep_plan(M.CSR, R["m"], R.nnz, 8, ptr=R["ptr"])
for j in (0, 7):
    d = plan[j]
    b0, b1 = int(d["start_idx"]), int(d["end_idx"]) + 1
    r0, r1 = int(d["start_row"]), int(d["end_row"]) + 1
    P = gen.Sparse(fmt="csr", m=r1 - r0, n=R["n"], ptr=np.clip(R["ptr"][r0:r1 + 1], b0, b1) - b0,
                   idx=R["idx"][b0:b1].copy(), val=R["val"][b0:b1].copy())
    ms, st = timed(P, 1)
    print(json.dumps({"rmat_part": j, "rows": r1 - r0, "nnz": b1 - b0, "ms": ms, "ns_per_nnz": ms * 1e6 / (b1 - b0),
                      "ntiles": st["ntiles"], "nslabs": st["nslabs"], "nhot": st["nhot"], "x_compact": st["x_compact"]}),
          flush=True)
