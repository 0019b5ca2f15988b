#!/usr/bin/env python
"""bench.py -- msRep nnz-balanced SpMV on B200 (driver contract).

One step = one msrep_spmv (y <- alpha*A*x + beta*y, alpha=1.5, beta=0.5) over the whole matrix,
split nnz-balanced over N GPUs (one process per GPU).  Default workload: BASELINE.json configs[2],
the largest single-GPU config -- R-MAT scale 24 (16,777,216 rows, 263,419,028 nnz), pCSR, fp64.
Metric: GFLOP/s (2*nnz per SpMV, whole job), with the HBM roofline of the dominant kernel.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config rmat|stencil|tallskinny|random1k|suite-...]
                  [--format csr|coo|csc|coo_col] [--dtype f64|f32] [--layout replicated|owned|sharded]
                  [--impl msrep|reference] [--hot-x -1|0|1] [--xload -1|0|1]

--gpus N without a torchrun environment re-launches itself under torch.distributed.run with N
ranks (127.0.0.1), and fails with exit code 2 if fewer than N GPUs are visible.  With N > 1
every rank builds only the rows its nonzero range touches (gen.config_rows; rank 0 broadcasts
the pointer array) and partitions through msrep_partition_slice.
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import gen  # noqa: E402

ALPHA, BETA = 1.5, 0.5
METRIC = "SpMV GFLOP/s and HBM GB/s (% of 8 TB/s) at 1/2/4/8 B200, per format"
NVLINK_GBPS = 900.0   # NVLink 5, per direction per GPU (nominal)
T1_CACHE = os.path.join(ROOT, ".bench_cache")


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=2000)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", default="msrep", choices=["msrep", "reference"])
    p.add_argument("--config", default="rmat",
                   choices=["stencil", "rmat", "rmatperm", "tallskinny", "random1k"] +
                   [f"suite-{s}-{z}" for s in gen.SUITE_SHAPES for z in gen.SUITE_SIZES])
    p.add_argument("--format", default=None, choices=["csr", "coo", "csc", "coo_col"])
    p.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    p.add_argument("--layout", default=None, choices=["replicated", "owned", "sharded"])
    p.add_argument("--e2e-steps", type=int, default=50)
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--kernel-times", type=int, default=0, metavar="STEPS",
                   help="after the timed region, profile STEPS SpMVs with torch.profiler (CUPTI) and report "
                        "the average device time of every kernel per SpMV (kernel_times_us)")
    p.add_argument("--parts-per-rank", type=int, default=1)
    p.add_argument("--hot-x", type=int, default=-1,
                   help="MSREP_TUNE_HOT_X: shared-memory hot-x cache (-1 auto, 0 off, 1 on, k > 1: k KiB)")
    p.add_argument("--compact-x", type=int, default=-1, choices=[-1, 0, 1, 2],
                   help="MSREP_TUNE_COMPACT_X: gather the rank's distinct x entries first (-1 auto, 0 off, 1 on)")
    p.add_argument("--sell", type=int, default=None, choices=[0, 1, 2],
                   help="MSREP_TUNE_SELL: 0 SEG tiles only, 1 SELL tiles with 32-bit ids, 2 + narrow SELL tiles")
    p.add_argument("--hot-cluster", type=int, default=1, choices=[1, 2],
                   help="MSREP_TUNE_HOT_CLUSTER: CTAs sharing one hot-x cache over DSMEM")
    p.add_argument("--col-layout", type=int, default=-1, choices=[-1, 0, 1],
                   help="MSREP_TUNE_COL_LAYOUT for pCSC / column-sorted pCOO: -1 auto (row tiles over the GPU-"
                        "transposed slice), 0 row bands (csc_band_kernel), 1 row tiles")
    p.add_argument("--xload", type=int, default=-1, choices=[-1, 0, 1],
                   help="MSREP_TUNE_XLOAD: x-gather L1 policy (-1 timed at partition, 0 allocate, 1 no_allocate)")
    p.add_argument("--fused", action="store_true",
                   help="N>1 row formats: fused allgather (msrep_spmv_mirror into the peers' y over NVLink, "
                        "torch symmetric memory) instead of SpMV + NCCL allgatherv")
    p.add_argument("--split", default="nnz", choices=["nnz", "block"],
                   help="nnz: msRep's nnz-balanced split; block: the paper's row/column-block Baseline")
    a = p.parse_args(argv)
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


def colwise(a):
    return a.format in ("csc", "coo_col")


def build_matrix(a):
    """Synthetic matrix of the named config (gen/, seeded): CSR, or CSC for pCSC."""
    A = gen.make_config(a.config)
    if colwise(a) and A["fmt"] == "csr":
        A = gen.transpose(A)
    if not colwise(a) and A["fmt"] == "csc":
        A = gen.transpose(A)
    if a.dtype == "f32":
        A["val"] = A["val"].astype(np.float32)
    return A


def rank_local_ok(a):
    """Rank-local generation needs the config's native compressed format (no transpose) and a
    pointer format (msrep_partition_slice takes CSR / CSC)."""
    if a.config not in gen.LOCAL_CONFIGS or a.format not in ("csr", "csc"):
        return False
    native = "csc" if a.config == "tallskinny" else "csr"
    return a.format == native


def workload_name(a, m, n, nnz):
    return f"{a.config}_{a.format}_{a.dtype}_m{m}_n{n}_nnz{nnz}"


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


def cpu_baseline(A, seconds, what):
    """The oracle as it stands (single-threaded C), timed on the host on a bounded sample, pinned
    to one core."""
    with pinned_core():
        return _cpu_baseline(A, seconds, what)


def _cpu_baseline(A, seconds, what):
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
            "sample": f"{reps} single-threaded oracle SpMVs over 1/{nblk} blocks of {what} "
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
           "config": {"workload": workload_name(a, A["m"], A["n"], A.nnz), "format": "p" + a.format.upper(),
                      "sample": f"each step = one 1/{nblk} row block of the matrix (~{A.nnz // nblk} nnz)"},
           "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": 1, "kind": "oracle", **host_info(),
                            "sample": f"{a.steps} steps, 1/{nblk} row blocks, single-threaded oracle pinned to one core"},
           "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def spawn(a):
    """--gpus N outside torchrun: relaunch under torch.distributed.run with N local ranks."""
    import torch
    have = torch.cuda.device_count()
    if have < a.gpus:
        print(f"bench.py: --gpus {a.gpus} needs {a.gpus} visible GPUs, found {have}", file=sys.stderr, flush=True)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def build_local(a, rank, world, ppr, dist, torch, M):
    """Rank-local matrix: the pointer array (rank 0 builds it and broadcasts it), then only the rows
    this rank's nonzero range touches.  Returns (fmt, m, n, ptr, r0, r1, idx, val)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    if world > 1:
        head = [None]
        if rank == 0:
            fmt, m, n, ptr = gen.config_pointer(a.config)
            head = [(fmt, m, n, ptr.size)]
        dist.broadcast_object_list(head, src=0)
        fmt, m, n, plen = head[0]
        t = torch.as_tensor(ptr).to(dev) if rank == 0 else torch.empty(plen, dtype=torch.int64, device=dev)
        dist.broadcast(t, src=0)
        ptr = t.cpu().numpy()
        del t
    else:
        fmt, m, n, ptr = gen.config_pointer(a.config)
    outer = n if fmt == "csc" else m
    nnz = int(ptr[-1])
    parts = M.msrep_plan_split(M.FORMATS[fmt], M.SPLITS[a.split], outer, nnz, world * ppr, ptr=ptr)
    mine = parts[rank * ppr:(rank + 1) * ppr]
    ne = mine[mine["start_row"] >= 0]
    if ne.size:
        r0, r1 = int(ne["start_row"][0]), int(ne["end_row"][-1]) + 1
    else:
        r0 = r1 = 0
    idx, val = gen.config_rows(a.config, ptr, r0, r1)
    if a.dtype == "f32":
        val = val.astype(np.float32)
    return fmt, m, n, ptr, r0, r1, idx, val


def t1_cache_path(wl):
    try:
        st = os.stat(os.path.join(ROOT, "paper_2209_07552_b200", "libmsrep.so"))
        tag = f"{int(st.st_mtime)}_{st.st_size}"
    except OSError:
        tag = "nolib"
    return os.path.join(T1_CACHE, f"t1_{wl}_{tag}.json")


def timed(step, steps, stream, torch):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if a.impl == "reference":
        run_reference(a)
        return 0
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(a)
    if world != a.gpus:
        print(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}", file=sys.stderr, flush=True)
        return 2
    if world > 1:   # NCCL communicator lines (nranks, transport) on stderr, for the record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    import torch
    import torch.distributed as dist
    import paper_2209_07552_b200 as M

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if local >= torch.cuda.device_count():   # no CPU fallback: the product path is the CUDA library
        print(f"bench.py: rank {rank} needs CUDA device {local}, found {torch.cuda.device_count()} visible",
              file=sys.stderr, flush=True)
        return 2
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ppr = a.parts_per_rank
    if world > 1:
        ctx = M.Context.from_torch_dist(device=local, parts_per_rank=ppr)
    else:
        ctx = M.Context(0, 1, None, local, ppr)
    ctx.set_tuning("hot_x", a.hot_x)
    ctx.set_tuning("xload", a.xload)
    ctx.set_tuning("compact_x", a.compact_x)
    ctx.set_tuning("hot_cluster", a.hot_cluster)
    if a.sell is not None:
        ctx.set_tuning("sell", a.sell)
    ctx.set_tuning("col_layout", a.col_layout)
    local_gen = rank_local_ok(a)
    A = None
    if local_gen:
        fmt, m, n, ptr, r0, r1, idx, val = build_local(a, rank, world, ppr, dist, torch, M)
        nnz = int(ptr[-1])
        ctx.partition_slice(fmt, m, n, ptr, idx, val, int(ptr[r0]), split=a.split)
        # rank 0's rows for the CPU baseline (the oracle on the same entries this rank holds)
        loc = gen.Sparse(fmt=fmt, m=(r1 - r0) if fmt == "csr" else m, n=n if fmt == "csr" else (r1 - r0),
                         ptr=ptr[r0:r1 + 1] - ptr[r0], idx=idx, val=val)
        cpu_what = "the whole matrix" if world == 1 else f"rank 0's {r1 - r0} {'rows' if fmt == 'csr' else 'columns'}"
        del ptr
    else:
        A = build_matrix(a)
        m, n, nnz = A["m"], A["n"], A.nnz
        coo = a.format in ("coo", "coo_col")   # COO views carry their sorted major index (rows / columns)
        coo_row = gen.expand_rows(A) if coo else None
        ctx.partition(a.format, m, n, ptr=None if coo else A["ptr"], idx=A["idx"], val=A["val"],
                      coo_row=coo_row, split=a.split)
        del coo_row
        loc, cpu_what = A, "the whole matrix"
    st = ctx.stats()
    wl = workload_name(a, m, n, nnz)
    vdt = np.float32 if a.dtype == "f32" else np.float64
    tdt = torch.float64 if vdt == np.float64 else torch.float32
    V = 8 if vdt == np.float64 else 4
    x = torch.as_tensor(gen.vector(n, 101, dtype=vdt)).cuda()
    y0 = torch.as_tensor(gen.vector(m, 102, dtype=vdt)).cuda()
    y = y0.clone()
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    lay = {"replicated": M.Y_REPLICATED, "owned": M.Y_OWNED, "sharded": M.Y_SHARDED}
    layout = lay[a.layout]
    step = lambda: ctx.spmv(ALPHA, x, BETA, y, layout, sh)
    if a.fused and world > 1 and a.format in ("csr", "coo"):
        # y lives in symmetric memory; every rank stores its owned rows into all peers' y from the
        # SpMV epilogue (msrep_spmv_mirror): the allgather overlaps the SpMV tile by tile
        import torch.distributed._symmetric_memory as symm_mem
        ys = symm_mem.empty(m, dtype=tdt, device=f"cuda:{local}")
        hdl = symm_mem.rendezvous(ys, dist.group.WORLD)
        peers = [hdl.get_buffer(r, (m,), tdt) for r in range(world) if r != rank]
        ys.copy_(y)
        y = ys
        step = lambda: ctx.spmv_mirror(ALPHA, x, BETA, y, peers, sh)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(vals):
        t = torch.tensor(vals, device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(v) for v in t]

    for _ in range(max(3, a.warmup)):
        step()
    barrier()
    M.msrep_profile_enable(ctx.h, True)
    M.msrep_profile_read(ctx.h, reset=True)
    sampler = ClockSampler(local)
    with sampler:
        ms = timed(step, a.steps, stream, torch)
    barrier()
    kern_ms, kern_n = M.msrep_profile_read(ctx.h, reset=True)
    M.msrep_profile_enable(ctx.h, False)
    ms_max, kern_avg_ms = max_over_ranks([ms, kern_ms / max(1, kern_n)])
    step_ms = ms_max / a.steps
    flops = 2.0 * nnz
    value = flops / (step_ms * 1e-3) / 1e9

    # a per-call median from individual event pairs (after the timed region, which
    # stays exactly K back-to-back steps): min(K, 50) calls, each bracketed by its own events
    ncall = min(a.steps, 50)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ncall)]
    for e0c, e1c in evs:
        e0c.record(stream)
        step()
        e1c.record(stream)
    torch.cuda.synchronize()
    per_call = sorted(e0c.elapsed_time(e1c) for e0c, e1c in evs)
    per_call_median = max_over_ranks([per_call[len(per_call) // 2]])[0] if per_call else None
    barrier()

    # per-kernel device time of one SpMV in a warm, back-to-back run (not cold-cache like ncu):
    # the split of the step between the tile kernel, the compact-x gather and the fix-up
    ktimes = None
    if a.kernel_times > 0 and rank == 0:
        from torch.profiler import profile, ProfilerActivity
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(a.kernel_times):
                step()
            torch.cuda.synchronize()
        acc = {}
        for ev in prof.events():
            if ev.device_type.name == "CUDA" and ev.device_time > 0:
                nm = ev.name.split("<")[0].split("::")[-1].replace("void ", "").strip() or ev.name[:60]
                acc[nm] = acc.get(nm, 0.0) + ev.device_time
        ktimes = {k: v / a.kernel_times for k, v in sorted(acc.items(), key=lambda kv: -kv[1])}
        barrier()

    # N > 1: the other layout of the format timed the same way (OWNED for the row formats,
    # SHARDED for the column formats: no allgather), merge share and NVLink bytes per rank
    per_layout = {a.layout: {"ms_per_step": step_ms}}
    if world > 1 and not a.fused:
        other = "sharded" if colwise(a) else "owned"
        if other != a.layout:
            st2 = lambda: ctx.spmv(ALPHA, x, BETA, y, lay[other], sh)
            for _ in range(max(3, a.warmup)):
                st2()
            barrier()
            ms2 = max_over_ranks([timed(st2, a.steps, stream, torch)])[0]
            per_layout[other] = {"ms_per_step": ms2 / a.steps}
            barrier()
    for k, d in per_layout.items():
        d["merge_share"] = max(0.0, 1.0 - kern_avg_ms / d["ms_per_step"])
        d["gflops"] = flops / (d["ms_per_step"] * 1e-3) / 1e9
    t1 = None
    cpath = t1_cache_path(wl)
    if world == 1 and rank == 0 and ppr == 1 and a.split == "nnz":
        os.makedirs(T1_CACHE, exist_ok=True)
        with open(cpath, "w") as f:
            json.dump({"t1_ms": step_ms, "workload": wl}, f)
    elif os.path.exists(cpath):
        with open(cpath) as f:
            t1 = json.load(f)["t1_ms"]
    if t1:
        for d in per_layout.values():
            d["E_p"] = t1 / (world * d["ms_per_step"])
    if world > 1:
        if colwise(a):   # reduce-scatter of the fp64 partial y (ring: (1 - 1/p) of it each way) + allgather
            shard = -(-m // world)
            nv_rs = (world - 1) * shard * 8
            nv_ag = (m - min(shard, m)) * V
            nv = {"reduce_scatter_bytes": nv_rs, "allgather_bytes": nv_ag}
            merge_b = nv_rs + (nv_ag if a.layout == "replicated" else 0)
        else:            # allgatherv of the owned y segments: every other rank's rows come in
            ag = (m - st["owned_rows"]) * V
            nv = {"allgatherv_bytes": ag, "head_exchange_bytes": world * ppr * 8}
            merge_b = ag if a.layout == "replicated" else 0
        merge_ms = max(1e-6, step_ms - kern_avg_ms)
        nv["merge_GBps"] = merge_b / (merge_ms * 1e-3) / 1e9
        nv["frac_of_nvlink"] = nv["merge_GBps"] / NVLINK_GBPS
        nv["note"] = f"rank {rank}'s ingress per step over the merge time (step - kernel), vs {NVLINK_GBPS:.0f} GB/s"
    else:
        nv = None

    # e2e through the public host-vector API: H2D x (and y_in), SpMV, D2H y, every step
    xh = torch.empty(n, dtype=tdt, pin_memory=True)
    xh.copy_(x.cpu())
    yh = torch.empty(m, dtype=tdt, pin_memory=True)
    yh.copy_(y0.cpu())
    seg = st["owned_rows"] if a.layout == "owned" else m
    for _ in range(3):
        ctx.spmv_host(ALPHA, xh.data_ptr(), BETA, yh.data_ptr(), layout, sh)
    barrier()
    ke = a.e2e_steps
    e2e_step_ms = max_over_ranks([timed(lambda: ctx.spmv_host(ALPHA, xh.data_ptr(), BETA, yh.data_ptr(), layout, sh),
                                        ke, stream, torch)])[0] / ke
    own_in = st["owned_rows"] if world > 1 else m
    h2d = n * V + own_in * V
    d2h = seg * V

    # roofline of the dominant kernel (rank 0's launch; algorithmic bytes / event-timed duration)
    hbm_peak, peak_kind = load_peaks()
    kname = "csc_band_kernel" if (colwise(a) and st["col_layout"] == 0) else "rows_kernel"
    traffic = None
    try:   # DRAM bytes per launch of that kernel from a committed `ncu --set full` capture (profiles/)
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f).get(wl)
        if tr and tr.get("kernel") == kname and (world == 1 or tr.get("n_gpus", 1) == world):
            traffic = tr["dram_bytes_per_launch"]
    except Exception:
        traffic = None
    alg_bytes, stream_bytes = st["alg_bytes"], st["stream_bytes"]
    # the roofline counts the smaller of the algorithmic bytes and the bytes the built layout
    # streams: pCOO's 4-B row ids are never streamed (the tiles carry u8 keys), narrow SELL tiles
    # carry 2-B column offsets instead of 4-B ids -- a compressed layout is
    # judged against the bytes it really moves, never credited with bytes it skips
    roof_bytes = min(alg_bytes, stream_bytes)
    achieved = roof_bytes / (kern_avg_ms * 1e-3) / 1e9
    step_gbs = alg_bytes / (step_ms * 1e-3) / 1e9

    cpu = None
    if rank == 0 and not a.no_cpu_baseline:
        cpu = cpu_baseline(loc, a.cpu_seconds, cpu_what)
    barrier()
    if rank == 0:
        clocks = sampler.summary()
        out = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": a.dtype, "data": "synthetic (gen/, seeded; no SuiteSparse offline)",
            "config": {"workload": wl, "format": "p" + a.format.upper(), "layout": a.layout,
                       "device_layout": ("row bands" if st["col_layout"] == 0 else "row tiles (slice transposed on the GPU)")
                                        if colwise(a) else "row tiles",
                       "m": m, "n": n, "nnz": nnz, "alpha": ALPHA, "beta": BETA,
                       "parts_per_rank": ppr, "split": a.split,
                       "merge": "fused epilogue stores into peer y (msrep_spmv_mirror)" if (a.fused and world > 1)
                                else "NCCL allgatherv / reduce-scatter",
                       "matrix_build": "rank-local rows (msrep_partition_slice)" if local_gen else "whole matrix per rank",
                       "l2": "no flush: per-step matrix bytes exceed the 126 MB L2 (inputs larger than L2); "
                             "x stays L2-resident across steps as in an iterative solver",
                       "parallelism": f"nnz-balanced dp{world}"},
            "hbm": {"alg_bytes_per_step_rank0": alg_bytes, "stream_bytes_per_step_rank0": stream_bytes,
                    "step_GBps_rank0": step_gbs, "frac_of_8TBps": step_gbs / 8000.0},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic, "kernel": kname,
                         "kernel_avg_ms": kern_avg_ms, "alg_bytes_per_launch": alg_bytes,
                         "bytes_counted": "stream" if stream_bytes < alg_bytes else "alg",
                         "stream_bytes_per_launch": stream_bytes,
                         "frac_of_8TBps": achieved / 8000.0,
                         "peak_kind": peak_kind + " (MEASURED_PEAKS.json hbm_gbs, a copy)" if peak_kind == "measured"
                         else peak_kind},
            "roofline_gather": {"bound": "x-gather requests",
                                "achieved": (st["nnz_rank"] - st["hot_nnz"]) / (kern_avg_ms * 1e-3) / 1e9,
                                "peak": 272.0, "unit": "G gathers/s",
                                "frac": (st["nnz_rank"] - st["hot_nnz"]) / (kern_avg_ms * 1e-3) / 1e9 / 272.0,
                                "hot_x_share": st["hot_nnz"] / max(1, st["nnz_rank"]),
                                "peak_kind": "measured: pure random-gather kernel, L2-resident x (profiles/r1_gatherbench.txt)",
                                "note": "the cold gathers only (one L1TEX->L2 request each; the hot-x share is served "
                                        "from shared memory); binds for random column patterns (R-MAT, tall-skinny); "
                                        "coalesced gathers (stencil) cost far less than one request each"},
            "layouts": per_layout,
            "kernel_times_us": ktimes,
            "per_call_median_ms": per_call_median,
            "nvlink": nv,
            "nccl": {"nranks": world, "version": ".".join(map(str, torch.cuda.nccl.version())),
                     "init_log": "stderr (NCCL_DEBUG=INFO, NCCL_DEBUG_SUBSYS=INIT)"} if world > 1 else None,
            "cpu_baseline": cpu,
            "e2e": {"value": flops / (e2e_step_ms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": e2e_step_ms,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "api": "msrep_spmv_host"},
            "gpu_launches": int(a.steps * st["kernels_per_spmv"]),
            "clocks": clocks,
            "partition_ms": st["partition_ms"],
            "partition_phase_ms": dict(zip(("validate", "plan", "schedule", "upload_pack"), list(st["phase_ms"]))),
            "layout_build_ms": list(st["layout_ms"]),
            "stats_rank0": {k: st[k] for k in ("nnz_rank", "ntiles", "nsell", "nsell_narrow", "nslabs", "nsplit_rows",
                                               "distinct_cols", "kernels_per_spmv", "tile_bytes", "x_no_allocate",
                                               "nhot", "hot_nnz", "x_compact", "x_order", "col_layout")},
        }
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
