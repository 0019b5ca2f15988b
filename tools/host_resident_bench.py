"""Host-resident (out-of-core) SpMV and partition-overhead study on one B200 (
the paper's Fig. part-time).

For each workload:
  * device-resident: partition once (phase breakdown of msrep_partition), K x msrep_spmv;
  * host-resident (MSREP_RESIDENT_HOST): the layout parked in pinned host memory, each call
    streams it H2D in chunks -> ms per SpMV, and the streamed bytes / time as a fraction of the
    measured pinned H2D bandwidth (torch copy of a 1 GiB pinned buffer, best of 5);
  * the paper's per-call regime: partition + one SpMV through the host-vector API, and the
    partition share of it (the paper's "partitioning overhead").
One JSON line per (workload, mode) on stdout.

    python tools/host_resident_bench.py [--configs stencil:csr,rmat:csr,...] [--chunk-mb 256]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gen  # noqa: E402


def h2d_peak_gbs(torch):
    src = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, (1 << 30) / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del src, dst
    return best


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--configs", default="stencil:csr,stencil:coo,stencil:csc,rmat:csr,rmat:coo,tallskinny:csc")
    p.add_argument("--chunk-mb", type=int, default=256)
    p.add_argument("--steps", type=int, default=10)
    a = p.parse_args()
    import torch
    import paper_2209_07552_b200 as M
    torch.cuda.set_device(0)
    peak = h2d_peak_gbs(torch)
    print(json.dumps({"h2d_pinned_peak_gbs": peak, "how": "torch copy 1 GiB pinned -> device, best of 5"}), flush=True)
    for spec in a.configs.split(","):
        cfg, fmt = spec.split(":")
        A = gen.make_config(cfg)
        colwise = fmt in ("csc", "coo_col")
        if colwise != (A["fmt"] == "csc"):
            A = gen.transpose(A)
        coo_row = gen.expand_rows(A) if fmt in ("coo", "coo_col") else None
        x = torch.as_tensor(gen.vector(A["n"], 101)).cuda()
        y = torch.as_tensor(gen.vector(A["m"], 102)).cuda()
        xh = torch.empty(A["n"], dtype=torch.float64, pin_memory=True); xh.copy_(x.cpu())
        yh = torch.empty(A["m"], dtype=torch.float64, pin_memory=True); yh.copy_(y.cpu())
        for res in ("device", "host"):
            ctx = M.Context(0, 1, None, 0, 1)
            t0 = time.perf_counter()
            ctx.partition(fmt, A["m"], A["n"], ptr=None if coo_row is not None else A["ptr"], idx=A["idx"],
                          val=A["val"], coo_row=coo_row, residency=res, chunk_bytes=a.chunk_mb << 20)
            part_wall = (time.perf_counter() - t0) * 1e3
            st = ctx.stats()
            sh = torch.cuda.current_stream().cuda_stream
            for _ in range(3):
                ctx.spmv(1.5, x, 0.5, y, M.Y_REPLICATED, sh)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.steps):
                ctx.spmv(1.5, x, 0.5, y, M.Y_REPLICATED, sh)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            # the paper's per-call regime: host vectors in, y out (partition timed separately above)
            t1 = time.perf_counter()
            ctx.spmv_host(1.5, xh.data_ptr(), 0.5, yh.data_ptr(), M.Y_REPLICATED, sh)
            host_call_ms = (time.perf_counter() - t1) * 1e3
            out = {"workload": f"{cfg}_{fmt}_f64_m{A['m']}_n{A['n']}_nnz{A.nnz}", "residency": res,
                   "ms_per_spmv": ms, "gflops": 2.0 * A.nnz / (ms * 1e-3) / 1e9,
                   "partition_ms": st["partition_ms"], "partition_wall_ms": part_wall,
                   "phase_ms": {"validate": st["phase_ms"][0], "plan": st["phase_ms"][1],
                                "schedule": st["phase_ms"][2], "upload_pack": st["phase_ms"][3]},
                   "spmv_host_call_ms": host_call_ms,
                   "partition_share_of_paper_call": st["partition_ms"] / (st["partition_ms"] + host_call_ms),
                   "tile_bytes": st["tile_bytes"], "device_bytes": st["device_bytes"]}
            if res == "host":
                gbs = st["host_bytes"] / (ms * 1e-3) / 1e9
                out.update({"nchunks": st["nchunks"], "host_bytes": st["host_bytes"], "h2d_gbs": gbs,
                            "frac_of_h2d_peak": gbs / peak, "chunk_mb": a.chunk_mb})
            print(json.dumps(out), flush=True)
            ctx.close()
        del A, coo_row


if __name__ == "__main__":
    main()
