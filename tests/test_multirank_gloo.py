"""N>1 host logic on CPU: world_size-2/3 `gloo` process groups run the exchange
step of msrep_spmv (Sec. 4.3; readings R6, R9, R10) with
the library's own multi-rank plan (msrep_plan + msrep_exchange_plan, pure host)
and the collectives the NCCL path issues, in the same shape, for both splits
(msRep's nnz split and the paper's row/column-block Baseline):

  pCSR / pCOO  per-part pure partial sums (oracle, one part at a time, alpha=1, beta=0)
               -> all_gather of parts_per_rank head partials per rank (ncclAllGather)
               -> owner fix-up: alpha*(own sums + routed heads, part order) + beta*y_in
               -> allgatherv of owned segments as one broadcast per rank (ncclBroadcast group)
  pCSC         per-rank fp64 partial py -> sum over ranks (ncclReduceScatter; gloo has no
               reduce-scatter, so all_reduce + take the rank's block) -> alpha/beta epilogue
               on the shard -> allgatherv of shards

Inputs are small integers with dyadic alpha/beta, so every summation order is
exact and the result must equal the single-process oracle bit for bit.  The
device kernels that produce the partial sums are covered by the GPU tests
(virtual parts on one B200, tests/test_gpu_parity.py)."""
import itertools
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ALPHA, BETA = 1.5, -0.5


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cases():
    import gen
    out = []
    # SPEC fixture E: 4x4, 5 nonzeros, shared rows at every small np
    E = {"m": 4, "n": 4, "ptr": np.array([0, 2, 3, 3, 5], np.int64), "idx": np.array([0, 2, 1, 0, 3], np.int32),
         "val": np.array([1, 2, 3, 4, 5], np.float64)}
    out.append(("E", E))
    # one row across every part (chains, reading R10)
    N = 37
    out.append(("chain", {"m": 1, "n": N, "ptr": np.array([0, N], np.int64), "idx": np.arange(N, dtype=np.int32),
                          "val": np.ones(N)}))
    # empty rows, long rows, empty parts (nnz < np)
    out.append(("tiny", {"m": 5, "n": 3, "ptr": np.array([0, 0, 1, 1, 2, 2], np.int64),
                         "idx": np.array([2, 0], np.int32), "val": np.array([3.0, -2.0])}))
    A = gen.rmat(9, seed=3, kind=gen.SMALLINT)
    out.append(("rmat9", {"m": A["m"], "n": A["n"], "ptr": A["ptr"], "idx": A["idx"], "val": A["val"]}))
    B = gen.kdistinct_csr(300, 200, 7, 11, kind=gen.SMALLINT)
    out.append(("kd", {"m": B["m"], "n": B["n"], "ptr": B["ptr"], "idx": B["idx"], "val": B["val"]}))
    return out


def _row_rank(rank, world, vparts, fmt, A, x, y_in, split):
    """One rank of the pCSR/pCOO exchange; returns its full replicated y."""
    import torch
    import torch.distributed as dist
    import oracle
    import paper_2209_07552_b200 as M
    m, n, ptr, idx, val = A["m"], A["n"], A["ptr"], A["idx"], A["val"]
    nnz = idx.size
    np_ = world * vparts
    rows = oracle.csr_to_coo(m, ptr)
    if fmt == "csr":
        parts = M.msrep_plan_split(M.CSR, split, m, nnz, np_, ptr=ptr)
        seg, hrow, hpart = M.msrep_exchange_plan(M.CSR, m, n, nnz, world, vparts, ptr=ptr, split=split)
    else:
        parts = M.msrep_plan_split(M.COO, split, m, nnz, np_, coo_row=rows)
        seg, hrow, hpart = M.msrep_exchange_plan(M.COO, m, n, nnz, world, vparts, coo_row=rows, split=split)
    lo, hi = int(seg[rank, 0]), int(seg[rank, 1])
    acc = np.zeros(m, np.float64)
    head_local = np.zeros(vparts, np.float64)
    for jl in range(vparts):
        d = parts[rank * vparts + jl]
        b0, b1 = int(d["start_idx"]), int(d["end_idx"]) + 1
        if b0 >= b1:
            continue
        r0, r1 = int(d["start_row"]), int(d["end_row"]) + 1
        # the part's own nonzeros only: pure row sums over [b0, b1) (the kernel's job)
        if fmt == "csr":
            lptr = np.clip(ptr[r0:r1 + 1], b0, b1) - b0
            s = oracle.spmv_csr(r1 - r0, lptr, idx[b0:b1], val[b0:b1], x, np.zeros(r1 - r0), 1.0, 0.0)
        else:
            s = oracle.spmv_coo(r1 - r0, rows[b0:b1] - r0, idx[b0:b1], val[b0:b1], x, np.zeros(r1 - r0), 1.0, 0.0)
        first = r0
        if d["start_flag"]:
            head_local[jl] = s[0]
            first = r0 + 1
        for r in range(first, r1):
            assert lo <= r < hi, "a part's non-head rows must be owned by its rank"
            acc[r] += s[r - r0]
    gathered = [torch.zeros(vparts, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(head_local))
    head_all = torch.cat(gathered).numpy()
    for q in range(np_):                       # fix-up on the owner, heads in part order (R10)
        if hpart[q] >= 0 and hpart[q] // vparts == rank:
            assert lo <= hrow[q] < hi
            acc[hrow[q]] += head_all[q]
    y = np.zeros(m, np.float64)
    y[lo:hi] = ALPHA * acc[lo:hi] + BETA * y_in[lo:hi]
    yt = torch.from_numpy(y)
    for r in range(world):                     # allgatherv as one broadcast per rank
        a, b = int(seg[r, 0]), int(seg[r, 1])
        if b > a:
            part = yt[a:b].clone()
            dist.broadcast(part, src=r)
            yt[a:b] = part
    return yt.numpy(), seg


def _csc_rank(rank, world, vparts, A, x, y_in, split):
    import torch
    import torch.distributed as dist
    import oracle
    import paper_2209_07552_b200 as M
    m, n = A["m"], A["n"]
    cp, ri, cv = oracle.csr_to_csc(m, n, A["ptr"], A["idx"], A["val"])
    nnz = ri.size
    np_ = world * vparts
    parts = M.msrep_plan_split(M.CSC, split, n, nnz, np_, ptr=cp)
    seg, hrow, hpart = M.msrep_exchange_plan(M.CSC, m, n, nnz, world, vparts, ptr=cp, split=split)
    assert (hrow == -1).all() and (hpart == -1).all()
    py = np.zeros(m, np.float64)
    for jl in range(vparts):
        d = parts[rank * vparts + jl]
        b0, b1 = int(d["start_idx"]), int(d["end_idx"]) + 1
        if b0 >= b1:
            continue
        c0, c1 = int(d["start_row"]), int(d["end_row"]) + 1
        lptr = np.clip(cp[c0:c1 + 1], b0, b1) - b0
        py += oracle.spmv_csc(m, c1 - c0, lptr, ri[b0:b1], cv[b0:b1], x[c0:c1], np.zeros(m), 1.0, 0.0)
    pt = torch.from_numpy(py)
    dist.all_reduce(pt)
    lo, hi = int(seg[rank, 0]), int(seg[rank, 1])
    y = np.zeros(m, np.float64)
    y[lo:hi] = ALPHA * pt.numpy()[lo:hi] + BETA * y_in[lo:hi]
    yt = torch.from_numpy(y)
    for r in range(world):
        a, b = int(seg[r, 0]), int(seg[r, 1])
        if b > a:
            part = yt[a:b].clone()
            dist.broadcast(part, src=r)
            yt[a:b] = part
    return yt.numpy(), seg


def _worker(rank, world, port, vparts_list, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import gen
    import oracle
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fails = []
    try:
        for name, A in _cases():
            x = gen.vector(A["n"], 7, kind=gen.SMALLINT)
            y_in = gen.vector(A["m"], 8, kind=gen.SMALLINT)
            ref = oracle.spmv_csr(A["m"], A["ptr"], A["idx"], A["val"], x, y_in, ALPHA, BETA)
            for vp, split, fmt in itertools.product(vparts_list, (0, 1), ("csr", "coo", "csc")):
                if fmt == "csc":
                    y, seg = _csc_rank(rank, world, vp, A, x, y_in, split)
                else:
                    y, seg = _row_rank(rank, world, vp, fmt, A, x, y_in, split)
                # segments tile [0, m) in rank order
                ok_tiles = seg[0, 0] == 0 and seg[-1, 1] == A["m"] and all(
                    seg[r, 1] == seg[r + 1, 0] for r in range(world - 1))
                if not ok_tiles or not np.array_equal(y, ref):
                    fails.append((name, fmt, vp, split, bool(ok_tiles)))
    finally:
        dist.destroy_process_group()
    q.put((rank, fails))


@pytest.mark.parametrize("world,vparts", [(2, (1, 2, 3)), (3, (1, 2))])
def test_exchange_gloo_matches_oracle(world, vparts):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, vparts, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, fails in res:
        assert not fails, f"rank {rank}: {fails}"


def test_exchange_plan_routes_heads_to_row_owner():
    """Every flagged part's head goes to the part whose owned range holds that row;
    owned ranges follow R_i = lower_bound(ptr, b_i) (brute force: the part holding
    the row's first nonzero owns it, reading R9)."""
    import gen
    import oracle
    import paper_2209_07552_b200 as M
    for seed in range(6):
        A = gen.rmat(8, seed=seed + 20)
        m, n, ptr, nnz = A["m"], A["n"], A["ptr"], A.nnz
        for world, vp in [(2, 1), (2, 4), (4, 2), (8, 1), (3, 5)]:
            parts = M.msrep_plan(M.CSR, m, nnz, world * vp, ptr=ptr)
            seg, hrow, hpart = M.msrep_exchange_plan(M.CSR, m, n, nnz, world, vp, ptr=ptr)
            b = oracle.nnz_boundaries(nnz, world * vp)
            for j, d in enumerate(parts):
                if d["start_idx"] <= d["end_idx"] and d["start_flag"]:
                    r = int(d["start_row"])
                    assert hrow[j] == r
                    k = int(hpart[j])
                    assert parts[k]["owned_begin"] <= r < parts[k]["owned_end"]
                    # brute force owner: the part containing row r's first nonzero
                    z = int(ptr[r])
                    assert b[k] <= z < b[k + 1]
                else:
                    assert hrow[j] == -1 and hpart[j] == -1
            for r in range(world):
                assert seg[r, 0] == parts[r * vp]["owned_begin"] and seg[r, 1] == parts[(r + 1) * vp - 1]["owned_end"]
