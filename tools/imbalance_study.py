"""Fig. 6 / NEXT-f1 study on one B200: the paper's row-block Baseline split
vs msRep's nnz split, with 8 parts.  Every part's SpMV (exactly the nonzeros that rank would
hold, through the library's own kernels) is timed ALONE on the GPU, as if it ran on its own
GPU; a plan's time is the max over its parts (no interconnect).  Reported beside the cost
model's closed form (sum nnz / np) / max nnz.

  python tools/imbalance_study.py [--parts 8] [--nnz 50e6] > gpurun_out/imbalance_study.jsonl
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


def time_part(A, d, x, reps):
    """SpMV time (ms) of one part's nonzeros [start_idx, end_idx] on the GPU, alone."""
    b0, b1 = int(d["start_idx"]), int(d["end_idx"]) + 1
    if b1 <= b0:
        return 0.0, 0
    r0, r1 = int(d["start_row"]), int(d["end_row"]) + 1
    ptr = np.clip(A["ptr"][r0:r1 + 1], b0, b1) - b0
    ctx = M.Context(0, 1, None, 0, 1)
    ctx.partition("csr", r1 - r0, A["n"], ptr=ptr, idx=A["idx"][b0:b1], val=A["val"][b0:b1])
    xd = torch.as_tensor(x).cuda()
    yd = torch.zeros(r1 - r0, dtype=torch.float64, device="cuda")
    for _ in range(5):
        ctx.spmv(1.0, xd, 0.0, yd)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        ctx.spmv(1.0, xd, 0.0, yd)
    e1.record(s)
    torch.cuda.synchronize()
    ctx.close()
    return e0.elapsed_time(e1) / reps, b1 - b0


def study(name, A, parts, reps):
    x = gen.vector(A["n"], 7)
    out = {"matrix": name, "m": A["m"], "matrix_nnz": A.nnz, "parts": parts}
    for split, code in (("block", M.SPLIT_BLOCK), ("nnz", M.SPLIT_NNZ)):
        plan = M.msrep_plan_split(M.CSR, code, A["m"], A.nnz, parts, ptr=A["ptr"])
        t, nz = zip(*(time_part(A, d, x, reps) for d in plan))
        out[split] = {"part_nnz": list(nz), "part_ms": list(t), "plan_ms": max(t),
                      "model_rel": (sum(nz) / parts) / max(nz)}
    out["measured_rel_block_vs_nnz"] = out["nnz"]["plan_ms"] / out["block"]["plan_ms"]
    out["model_rel_block_vs_nnz"] = out["block"]["model_rel"] / out["nnz"]["model_rel"]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parts", type=int, default=8)
    ap.add_argument("--nnz", type=float, default=50e6)
    ap.add_argument("--reps", type=int, default=100)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for ratio in (0.1, 0.25, 0.5, 1.0):
        m = int(a.nnz / (32 * (1 + ratio))) // a.parts * a.parts     # half the rows 64 nnz, half 64*ratio
        A = gen.two_class(m, m, a.parts, a.parts // 2, 64, ratio)
        print(json.dumps(study(f"two_class ratio={ratio}", A, a.parts, a.reps)), flush=True)
    for name, A in (("rmat scale 22", gen.rmat(22, seed=3)), ("powerlaw 10M", gen.transpose(gen.make_config("suite-powerlaw-10M")))):
        print(json.dumps(study(name, A, a.parts, a.reps)), flush=True)


if __name__ == "__main__":
    main()
