#!/usr/bin/env python
"""bench.py -- msRep nnz-balanced SpMV on B200 (driver contract).

One step = one msrep_spmv (y <- alpha*A*x + beta*y, alpha=1.5, beta=0.5) over
the whole matrix, split nnz-balanced over N GPUs (one process per GPU).
Default workload: BASELINE.json configs[1], the 2,048,383-row 27-point
stencil (54,439,939 nnz), pCSR, fp64.  Metric: GFLOP/s (2*nnz per SpMV,
whole job), with the HBM roofline of the dominant kernel alongside.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config stencil|rmat|tallskinny|random1k]
                  [--format csr|coo|csc] [--dtype f64|f32] [--layout replicated|owned|sharded]
                  [--impl msrep|reference]
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import gen  # noqa: E402

ALPHA, BETA = 1.5, 0.5
METRIC = "SpMV GFLOP/s and HBM GB/s (% of 8 TB/s) at 1/2/4/8 B200, per format"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=2000)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", default="msrep", choices=["msrep", "reference"])
    p.add_argument("--config", default="stencil",
                   choices=["stencil", "rmat", "tallskinny", "random1k"] +
                   [f"suite-{s}-{z}" for s in gen.SUITE_SHAPES for z in gen.SUITE_SIZES])
    p.add_argument("--format", default=None, choices=["csr", "coo", "csc", "coo_col"])
    p.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    p.add_argument("--layout", default=None, choices=["replicated", "owned", "sharded"])
    p.add_argument("--e2e-steps", type=int, default=50)
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--parts-per-rank", type=int, default=1)
    p.add_argument("--fused", action="store_true",
                   help="N>1 row formats: fused allgather (msrep_spmv_mirror into the peers' y over NVLink, "
                        "torch symmetric memory) instead of SpMV + NCCL allgatherv")
    p.add_argument("--split", default="nnz", choices=["nnz", "block"],
                   help="nnz: msRep's nnz-balanced split; block: the paper's row/column-block Baseline")
    a = p.parse_args()
    if a.format is None:
        a.format = "csc" if a.config == "tallskinny" else "csr"
    if a.layout is None:
        a.layout = "replicated"
    return a


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def build_matrix(a):
    """Synthetic matrix of the named config (gen/, seeded): CSR, or CSC for pCSC."""
    A = gen.make_config(a.config)
    colwise = a.format in ("csc", "coo_col")
    if colwise and A["fmt"] == "csr":
        A = gen.transpose(A)
    if not colwise and A["fmt"] == "csc":
        A = gen.transpose(A)
    if a.dtype == "f32":
        A["val"] = A["val"].astype(np.float32)
    return A


def workload_name(a, A):
    return f"{a.config}_{a.format}_{a.dtype}_m{A['m']}_n{A['n']}_nnz{A.nnz}"


class ClockSampler:
    """Samples SM clock + throttle reasons through NVML during the timed region."""

    def __init__(self, dev_index):
        self.samples, self.reasons, self.stop = [], set(), threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        names = {getattr(nv, k): k for k in dir(nv) if k.startswith("nvmlClocksEventReason") or
                 k.startswith("nvmlClocksThrottleReason")}
        while not self.stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h) if hasattr(
                    nv, "nvmlDeviceGetCurrentClocksEventReasons") else nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, nm in names.items():
                    if isinstance(bit, int) and bit and (r & bit) == bit and bit not in (0,):
                        self.reasons.add(nm.replace("nvmlClocksEventReason", "").replace("nvmlClocksThrottleReason", ""))
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self.stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        reasons = sorted(r for r in self.reasons if r not in ("All", "None", "GpuIdle", "ApplicationsClocksSetting"))
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples)}


def host_info():
    """Host facts reported beside the oracle's time (SURVEY 8(d) "oracle timing")."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"host_cpus": os.cpu_count(), "cpu_model": model}


class pinned_core:
    """Pin this process to one core while the single-threaded oracle is timed (restored after)."""

    def __enter__(self):
        self.saved = None
        try:
            self.saved = os.sched_getaffinity(0)
            os.sched_setaffinity(0, {min(self.saved)})
        except (AttributeError, OSError):
            self.saved = None
        return self

    def __exit__(self, *exc):
        if self.saved is not None:
            os.sched_setaffinity(0, self.saved)


def cpu_baseline(A, seconds):
    """The oracle as it stands (single-threaded C), timed on the host on a bounded sample, pinned
    to one core."""
    with pinned_core():
        return _cpu_baseline(A, seconds)


def _cpu_baseline(A, seconds):
    import oracle
    t_end = time.perf_counter() + seconds
    x = gen.vector(A["n"], 101, dtype=A["val"].dtype)
    y = gen.vector(A["m"], 102, dtype=A["val"].dtype)
    reps, flops, t0 = 0, 0.0, time.perf_counter()
    # bounded sample: contiguous row (or column) blocks of ~1/16 of the matrix, cycling
    outer = A["m"] if A["fmt"] == "csr" else A["n"]
    nblk = 16 if A.nnz > 4_000_000 else 1
    while True:
        b = reps % nblk
        r0, r1 = outer * b // nblk, outer * (b + 1) // nblk
        ptr = A["ptr"][r0:r1 + 1] - A["ptr"][r0]
        z0, z1 = int(A["ptr"][r0]), int(A["ptr"][r1])
        if A["fmt"] == "csr":
            oracle.spmv_csr(r1 - r0, ptr, A["idx"][z0:z1], A["val"][z0:z1], x, y[r0:r1], ALPHA, BETA)
        else:
            oracle.spmv_csc(A["m"], r1 - r0, ptr, A["idx"][z0:z1], A["val"][z0:z1], x[r0:r1], y, ALPHA, BETA)
        flops += 2.0 * (z1 - z0)
        reps += 1
        if time.perf_counter() >= t_end:
            break
    dt = time.perf_counter() - t0
    return {"value": flops / dt / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "oracle", **host_info(),
            "sample": f"{reps} single-threaded oracle SpMVs over 1/{nblk} row blocks of the same matrix "
                      f"({flops / 2:.3g} nonzeros total, {dt:.1f} s)"}


def run_reference(a):
    """--impl reference: the oracle (CPU) on bounded samples of the workload, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    A = build_matrix(a)
    import oracle
    x = gen.vector(A["n"], 101, dtype=A["val"].dtype)
    y = gen.vector(A["m"], 102, dtype=A["val"].dtype)
    outer = A["m"] if A["fmt"] == "csr" else A["n"]
    nblk = max(1, int(round(A.nnz / 1_000_000)))    # ~1M nonzeros (~5-10 ms) per step
    def step(i):
        b = i % nblk
        r0, r1 = outer * b // nblk, outer * (b + 1) // nblk
        ptr = A["ptr"][r0:r1 + 1] - A["ptr"][r0]
        z0, z1 = int(A["ptr"][r0]), int(A["ptr"][r1])
        if A["fmt"] == "csr":
            oracle.spmv_csr(r1 - r0, ptr, A["idx"][z0:z1], A["val"][z0:z1], x, y[r0:r1], ALPHA, BETA)
        else:
            oracle.spmv_csc(A["m"], r1 - r0, ptr, A["idx"][z0:z1], A["val"][z0:z1], x[r0:r1], y, ALPHA, BETA)
        return z1 - z0
    with pinned_core():
        for i in range(a.warmup):
            step(i)
        nz, t0 = 0, time.perf_counter()
        for i in range(a.steps):
            nz += step(i)
        dt = time.perf_counter() - t0
    v = 2.0 * nz / dt / 1e9
    out = {"metric": METRIC, "value": v, "unit": "GFLOP/s", "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
           "ms_per_step": dt * 1e3 / max(1, a.steps), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": a.dtype, "data": "synthetic", "impl": "reference",
           "config": {"workload": workload_name(a, A), "format": "p" + a.format.upper(),
                      "sample": f"each step = one 1/{nblk} row block of the matrix (~{A.nnz // nblk} nnz)"},
           "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": 1, "kind": "oracle", **host_info(),
                            "sample": f"{a.steps} steps, 1/{nblk} row blocks, single-threaded oracle pinned to one core"},
           "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import torch.distributed as dist
    import paper_2209_07552_b200 as M

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    A = build_matrix(a)
    fmt = M.FORMATS[a.format]
    layout = {"replicated": M.Y_REPLICATED, "owned": M.Y_OWNED, "sharded": M.Y_SHARDED}[a.layout]
    if world > 1:
        ctx = M.Context.from_torch_dist(device=local, parts_per_rank=a.parts_per_rank)
    else:
        ctx = M.Context(0, 1, None, local, a.parts_per_rank)
    coo = a.format in ("coo", "coo_col")   # COO views carry their sorted major index (rows / columns)
    coo_row = gen.expand_rows(A) if coo else None
    ctx.partition(a.format, A["m"], A["n"], ptr=None if coo else A["ptr"], idx=A["idx"], val=A["val"],
                  coo_row=coo_row, split=a.split)
    del coo_row
    st = ctx.stats()
    vdt = A["val"].dtype
    tdt = torch.float64 if vdt == np.float64 else torch.float32
    V = 8 if vdt == np.float64 else 4
    x = torch.as_tensor(gen.vector(A["n"], 101, dtype=vdt)).cuda()
    y0 = torch.as_tensor(gen.vector(A["m"], 102, dtype=vdt)).cuda()
    y = y0.clone()
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    step = lambda: ctx.spmv(ALPHA, x, BETA, y, layout, sh)
    if a.fused and world > 1 and a.format in ("csr", "coo"):
        # y lives in symmetric memory; every rank stores its owned rows into all peers' y from the
        # SpMV epilogue (msrep_spmv_mirror): the allgather overlaps the SpMV tile by tile
        import torch.distributed._symmetric_memory as symm_mem
        ys = symm_mem.empty(A["m"], dtype=tdt, device=f"cuda:{local}")
        hdl = symm_mem.rendezvous(ys, dist.group.WORLD)
        peers = [hdl.get_buffer(r, (A["m"],), tdt) for r in range(world) if r != rank]
        ys.copy_(y)
        y = ys
        step = lambda: ctx.spmv_mirror(ALPHA, x, BETA, y, peers, sh)

    for _ in range(max(3, a.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    M.msrep_profile_enable(ctx.h, True)
    M.msrep_profile_read(ctx.h, reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    with sampler:
        e0.record(stream)
        for _ in range(a.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    kern_ms, kern_n = M.msrep_profile_read(ctx.h, reset=True)
    M.msrep_profile_enable(ctx.h, False)
    t = torch.tensor([ms, kern_ms / max(1, kern_n)], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, kern_avg_ms = float(t[0]), float(t[1])
    step_ms = ms_max / a.steps
    flops = 2.0 * A.nnz
    value = flops / (step_ms * 1e-3) / 1e9

    # e2e through the public host-vector API: H2D x (and y_in), SpMV, D2H y, every step
    xh = torch.empty(A["n"], dtype=tdt, pin_memory=True)
    xh.copy_(x.cpu())
    yh = torch.empty(A["m"], dtype=tdt, pin_memory=True)
    yh.copy_(y0.cpu())
    seg = st["owned_rows"] if a.layout == "owned" else A["m"]
    for _ in range(3):
        ctx.spmv_host(ALPHA, xh.data_ptr(), BETA, yh.data_ptr(), layout, sh)
    if world > 1:
        dist.barrier()
    ke = a.e2e_steps
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(ke):
        ctx.spmv_host(ALPHA, xh.data_ptr(), BETA, yh.data_ptr(), layout, sh)
    f1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([f0.elapsed_time(f1)], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_step_ms = float(te[0]) / ke
    own_in = st["owned_rows"] if world > 1 else A["m"]
    h2d = A["n"] * V + own_in * V
    d2h = seg * V

    # roofline of the dominant kernel (per rank 0's launch; algorithmic bytes / event-timed duration)
    hbm_peak, peak_kind = load_peaks()
    kname = "csc_band_kernel" if a.format in ("csc", "coo_col") else "rows_kernel"
    traffic = None
    try:   # DRAM bytes per launch of that kernel from a committed `ncu --set full` capture (profiles/)
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f).get(workload_name(a, A))
        if tr and tr.get("kernel") == kname:
            traffic = tr["dram_bytes_per_launch"]
    except Exception:
        traffic = None
    alg_bytes = st["alg_bytes"]
    achieved = alg_bytes / (kern_avg_ms * 1e-3) / 1e9
    step_gbs = alg_bytes / (step_ms * 1e-3) / 1e9

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(A, a.cpu_seconds)
    if rank == 0:
        clocks = sampler.summary()
        out = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": a.dtype, "data": "synthetic (gen/, seeded; no SuiteSparse offline)",
            "config": {"workload": workload_name(a, A), "format": "p" + a.format.upper(), "layout": a.layout,
                       "m": A["m"], "n": A["n"], "nnz": A.nnz, "alpha": ALPHA, "beta": BETA,
                       "parts_per_rank": a.parts_per_rank, "split": a.split,
                       "merge": "fused epilogue stores into peer y (msrep_spmv_mirror)" if (a.fused and world > 1)
                                else "NCCL allgatherv / reduce-scatter",
                       "l2": "no flush: per-step matrix bytes exceed the 126 MB L2 (inputs larger than L2); "
                             "x stays L2-resident across steps as in an iterative solver",
                       "parallelism": f"nnz-balanced dp{world}"},
            "hbm": {"alg_bytes_per_step_rank0": alg_bytes, "step_GBps_rank0": step_gbs,
                    "frac_of_8TBps": step_gbs / 8000.0},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic, "kernel": kname,
                         "kernel_avg_ms": kern_avg_ms, "alg_bytes_per_launch": alg_bytes,
                         "peak_kind": peak_kind + " (MEASURED_PEAKS.json hbm_gbs, a copy)" if peak_kind == "measured"
                         else peak_kind},
            "roofline_gather": {"bound": "x-gather requests", "achieved": A.nnz / (kern_avg_ms * 1e-3) / 1e9,
                                "peak": 272.0, "unit": "G gathers/s",
                                "frac": A.nnz / (kern_avg_ms * 1e-3) / 1e9 / 272.0,
                                "peak_kind": "measured: pure random-gather kernel, L2-resident x (profiles/r1_gatherbench.txt)",
                                "note": "one x gather per nonzero; binds for random column patterns (R-MAT, tall-skinny); "
                                        "coalesced patterns merge requests, so frac > 1 means gathers do not bind"},
            "cpu_baseline": cpu,
            "e2e": {"value": flops / (e2e_step_ms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": e2e_step_ms,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "api": "msrep_spmv_host"},
            "gpu_launches": int(a.steps * st["kernels_per_spmv"]),
            "clocks": clocks,
            "partition_ms": st["partition_ms"],
            "stats_rank0": {k: st[k] for k in ("nnz_rank", "ntiles", "nsell", "nslabs", "nsplit_rows",
                                               "distinct_cols", "kernels_per_spmv", "tile_bytes", "x_no_allocate")},
        }
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
