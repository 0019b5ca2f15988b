"""Strong-scaling projection on ONE B200 (parallel efficiency per layout).

Only one GPU is available, so an N-GPU run is projected, not measured:
  * compute: for p = 1, 2, 4, 8 the nnz-balanced plan (msrep_plan) is cut into its p parts;
    every part's exact nonzeros are partitioned as a one-rank matrix and its SpMV timed ALONE
    through the library (CUDA events, kernel + fused epilogue) -- T_comp(p) = max over parts;
  * exchange (modelled, NOT measured): OWNED layout (pCSR/pCOO) = one small NCCL all-gather of
    head partials, taken as 15 us of latency; REPLICATED = + allgatherv of the other ranks' owned
    y segments, (m - owned_min) * V bytes into the slowest rank at BW_NVLINK; pCSC = reduce-scatter
    of the fp64 partial y, (1 - 1/p) * m * 8 bytes at BW_NVLINK, + 15 us.
  E(p) = T(1) / (p * T(p)).  One JSON line per (workload, p).

    python tools/scaling_projection.py [--configs stencil:csr,rmat:csr,tallskinny:csc] [--reps 20]
"""
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

BW_NVLINK = 700e9     # bytes/s, effective NCCL bus bandwidth assumed for NVLink 5 (900 GB/s per direction nominal)
LAT = 15e-6           # s, one small NCCL collective


def time_part(A, fmt, d, x, reps):
    """(ms of one part's SpMV ALONE (its nonzeros as a one-rank matrix), its algorithmic bytes)."""
    b0, b1 = int(d["start_idx"]), int(d["end_idx"]) + 1
    if b1 <= b0:
        return 0.0, 0
    o0, o1 = int(d["start_row"]), int(d["end_row"]) + 1          # rows (CSR) / columns (CSC)
    ptr = np.clip(A["ptr"][o0:o1 + 1], b0, b1) - b0
    ctx = M.Context(0, 1, None, 0, 1)
    if fmt == "csr":
        ctx.partition("csr", o1 - o0, A["n"], ptr=ptr, idx=A["idx"][b0:b1], val=A["val"][b0:b1])
        xd = torch.as_tensor(x).cuda()
        yd = torch.zeros(o1 - o0, dtype=torch.float64, device="cuda")
    else:
        ctx.partition("csc", A["m"], o1 - o0, ptr=ptr, idx=A["idx"][b0:b1], val=A["val"][b0:b1])
        xd = torch.as_tensor(x[o0:o1]).cuda()
        yd = torch.zeros(A["m"], dtype=torch.float64, device="cuda")
    for _ in range(10):   # warm: lazy module loading and the first launches stay out of the timing
        ctx.spmv(1.0, xd, 0.0, yd)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        ctx.spmv(1.0, xd, 0.0, yd)
    e1.record()
    torch.cuda.synchronize()
    ab = ctx.stats()["alg_bytes_beta0"]
    ctx.close()
    return e0.elapsed_time(e1) / reps, ab


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="stencil:csr,rmat:csr,tallskinny:csc")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for spec in a.configs.split(","):
        cfg, fmt = spec.split(":")
        A = gen.make_config(cfg)
        if (fmt == "csc") != (A["fmt"] == "csc"):
            A = gen.transpose(A)
        x = gen.vector(A["n"] if fmt == "csr" else A["n"], 7)
        m, V = A["m"], 8
        outer = A["m"] if fmt == "csr" else A["n"]
        t1 = None
        for p in (1, 2, 4, 8):
            plan = M.msrep_plan(M.CSR if fmt == "csr" else M.CSC, outer, A.nnz, p, ptr=A["ptr"])
            tb = [time_part(A, fmt, d, x, a.reps) for d in plan]
            tp = [t for t, _ in tb]
            ab = [b for _, b in tb]
            tc = max(tp)
            if p == 1:
                t1 = tc
            if fmt == "csr":
                owned = [int(d["owned_end"] - d["owned_begin"]) for d in plan]
                ex_owned = LAT if p > 1 else 0.0
                ex_repl = ex_owned + ((m - min(owned)) * V / BW_NVLINK if p > 1 else 0.0)
            else:
                ex_owned = None
                ex_repl = (LAT + (1 - 1 / p) * m * 8 / BW_NVLINK) if p > 1 else 0.0
            out = {"workload": f"{cfg}_{fmt}_f64_m{A['m']}_n{A['n']}_nnz{A.nnz}", "p": p,
                   "part_ms": tp, "t_comp_ms": tc, "imbalance_max_over_mean": tc / (sum(tp) / p),
                   # the nnz split balances nonzeros, not bytes: each part's algorithmic bytes (beta = 0:
                   # matrix + x entries + its y rows) and the rate it streams them at
                   "part_alg_bytes": ab, "bytes_max_over_mean": max(ab) / (sum(ab) / p),
                   "part_GBps": [b / (t * 1e-3) / 1e9 if t > 0 else 0.0 for t, b in tb],
                   "E_comp": t1 / (p * tc),
                   "exchange_model_ms": {"owned": None if ex_owned is None else ex_owned * 1e3,
                                         "replicated": ex_repl * 1e3},
                   "E_owned_projected": None if ex_owned is None else t1 / (p * (tc + ex_owned * 1e3)),
                   "E_replicated_projected": t1 / (p * (tc + ex_repl * 1e3)),
                   "model": f"exchange modelled at {BW_NVLINK / 1e9:.0f} GB/s + {LAT * 1e6:.0f} us; compute measured"}
            print(json.dumps(out), flush=True)
        del A


if __name__ == "__main__":
    main()
