"""tools/part_probe.py CONFIG FMT P K [--sell S ...]: time part K of the P-way nnz plan of a config alone (as in
tools/scaling_projection.py) under tuning variants, with the layout stats -- for chasing a slow part."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import paper_2209_07552_b200 as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config"); ap.add_argument("fmt"); ap.add_argument("p", type=int); ap.add_argument("parts", type=str)
ap.add_argument("--sell", default="2,1"); ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()
torch.cuda.set_device(0)
A = gen.make_config(a.config)
x = gen.vector(A["n"], 7)
plan = M.msrep_plan(M.CSR, A["m"], A.nnz, a.p, ptr=A["ptr"])
for k in map(int, a.parts.split(",")):
    d = plan[k]
    b0, b1 = int(d["start_idx"]), int(d["end_idx"]) + 1
    o0, o1 = int(d["start_row"]), int(d["end_row"]) + 1
    ptr = np.clip(A["ptr"][o0:o1 + 1], b0, b1) - b0
    for sell in map(int, a.sell.split(",")):
        ctx = M.Context(0, 1, None, 0, 1)
        ctx.set_tuning("sell", sell)
        ctx.partition("csr", o1 - o0, A["n"], ptr=ptr, idx=A["idx"][b0:b1], val=A["val"][b0:b1])
        xd = torch.as_tensor(x).cuda(); yd = torch.zeros(o1 - o0, dtype=torch.float64, device="cuda")
        for _ in range(5):
            ctx.spmv(1.0, xd, 0.0, yd)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(a.reps):
            ctx.spmv(1.0, xd, 0.0, yd)
        e1.record(); torch.cuda.synchronize()
        st = ctx.stats()
        print(f"part {k} sell={sell} ms={e0.elapsed_time(e1) / a.reps:.4f} rows={o1 - o0} nnz={b1 - b0} " +
              " ".join(f"{q}={st[q]}" for q in ("ntiles", "nsell", "nsell_narrow", "kernels_per_spmv", "x_no_allocate",
                                                "sell_1cta", "nhot", "x_compact")), flush=True)
        ctx.close()
