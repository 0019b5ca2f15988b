"""One rank of the multi-GPU parity run (tests/test_gpu_multirank.py, launched by torchrun with N
ranks, one GPU each).  Exercises the NCCL merge of msrep_spmv for real (Sec. 4.3):
head-partial all-gather + owner fix-up + allgatherv (pCSR / pCOO), reduce-scatter + shard
epilogue (+ allgather) (pCSC / column-sorted pCOO), for both splits, 1 and 2 parts per rank, every
layout, plus msrep_spmv_mirror into the peers' y (symmetric memory), SpMM and CG.  Integer data
with dyadic alpha/beta: every result must equal the single-process oracle BIT FOR BIT.  Exit code
0 = all cases passed; failures are printed as "FAIL ..." lines."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    import gen
    import oracle
    import paper_2209_07552_b200 as M

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    fails = []

    def check(tag, got, ref):
        if not np.array_equal(got, ref):
            bad = np.nonzero(got != ref)[0]
            fails.append(f"FAIL rank {rank} {tag}: {bad.size} rows differ, first {bad[:5]} got {got[bad[:3]]} ref {ref[bad[:3]]}")

    mats = {
        "rmat14": gen.rmat(14, seed=91, kind=gen.SMALLINT),
        "chain": gen.Sparse(fmt="csr", m=3, n=5000, ptr=np.array([0, 1, 4999, 5000], np.int64),
                            idx=np.concatenate([[7], np.arange(4998), [3]]).astype(np.int32),
                            val=np.ones(5000)),
        "stencil": gen.stencil27(20, kind=gen.SMALLINT),
    }
    alpha, beta = 1.5, -0.5
    for name, A in mats.items():
        m, n = A["m"], A["n"]
        T = gen.transpose(A)
        x = gen.vector(n, 92, kind=gen.SMALLINT)
        y = gen.vector(m, 93, kind=gen.SMALLINT)
        ref = oracle.spmv_csr(m, A["ptr"], A["idx"], A["val"], x, y, alpha, beta)
        for ppr in (1, 2):
            for split in ("nnz", "block"):
                for fmt in ("csr", "coo", "csc", "coo_col", "coo_unsorted"):
                    if fmt == "coo_unsorted" and split == "block":
                        continue
                    ctx = M.Context.from_torch_dist(device=local, parts_per_rank=ppr)
                    B = T if fmt in ("csc", "coo_col") else A
                    if fmt == "coo_unsorted":
                        perm = np.random.default_rng(5).permutation(A.nnz)
                        ur, uc, uv = gen.expand_rows(A)[perm].copy(), A["idx"][perm].copy(), A["val"][perm].copy()
                        ctx.partition(fmt, m, n, idx=uc, val=uv, coo_row=ur, split=split)
                    elif fmt in ("coo", "coo_col"):
                        ctx.partition(fmt, m, n, idx=B["idx"], val=B["val"], coo_row=gen.expand_rows(B), split=split)
                    else:
                        ctx.partition(fmt, m, n, ptr=B["ptr"], idx=B["idx"], val=B["val"], split=split)
                    st = ctx.stats()
                    seg, _, _ = M.msrep_exchange_plan(M.FORMATS[fmt], m, n, A.nnz, world, ppr,
                                                      ptr=None if fmt.startswith("coo") else B["ptr"],
                                                      coo_row=(ur if fmt == "coo_unsorted" else gen.expand_rows(B))
                                                      if fmt.startswith("coo") else None,
                                                      split=M.SPLITS[split])
                    lo, hi = int(seg[rank][0]), int(seg[rank][1])
                    layouts = ["replicated", "sharded"] if fmt in ("csc", "coo_col", "coo_unsorted") else ["replicated", "owned"]
                    for lay in layouts:
                        yd = torch.as_tensor(y).cuda()
                        ctx.spmv(alpha, torch.as_tensor(x).cuda(), beta, yd,
                                 {"replicated": M.Y_REPLICATED, "owned": M.Y_OWNED, "sharded": M.Y_SHARDED}[lay])
                        torch.cuda.synchronize()
                        got = yd.cpu().numpy()
                        tag = f"{name} {fmt} {split} ppr={ppr} {lay}"
                        if lay == "replicated":
                            check(tag, got, ref)
                        else:
                            check(tag, got[lo:hi], ref[lo:hi])
                    # host-vector path (replicated)
                    yh = y.copy()
                    ctx.spmv_host(alpha, x, beta, yh, M.Y_REPLICATED)
                    check(f"{name} {fmt} {split} ppr={ppr} host", yh, ref)
                    if fmt in ("csr", "coo") and split == "nnz":
                        # SpMM, k = 4, replicated
                        k = 4
                        X = np.stack([gen.vector(n, 100 + j, kind=gen.SMALLINT) for j in range(k)], 1)
                        Y = np.stack([gen.vector(m, 200 + j, kind=gen.SMALLINT) for j in range(k)], 1)
                        Yd = torch.as_tensor(np.ascontiguousarray(Y)).cuda()
                        ctx.spmm(alpha, torch.as_tensor(np.ascontiguousarray(X)).cuda(), beta, Yd)
                        got = Yd.cpu().numpy()
                        for j in range(k):
                            check(f"{name} {fmt} spmm col {j}", got[:, j],
                                  oracle.spmv_csr(m, A["ptr"], A["idx"], A["val"], X[:, j].copy(), Y[:, j].copy(),
                                                  alpha, beta))
                        # fused allgather: every rank stores its owned rows into the peers' y
                        import torch.distributed._symmetric_memory as symm_mem
                        ys = symm_mem.empty(m, dtype=torch.float64, device=f"cuda:{local}")
                        hdl = symm_mem.rendezvous(ys, dist.group.WORLD)
                        peers = [hdl.get_buffer(r, (m,), torch.float64) for r in range(world) if r != rank]
                        ys.copy_(torch.as_tensor(y).cuda())
                        dist.barrier()
                        ctx.spmv_mirror(alpha, torch.as_tensor(x).cuda(), beta, ys, peers)
                        torch.cuda.synchronize()
                        dist.barrier()
                        check(f"{name} {fmt} mirror ppr={ppr}", ys.cpu().numpy(), ref)
                    ctx.close()
    # CG on an SPD stencil (diag 30, off -1), every format: converges to the known solution
    S = gen.stencil27(10, kind=gen.ONES)
    rows = np.repeat(np.arange(S["m"]), np.diff(S["ptr"]))
    S["val"] = np.where(S["idx"] == rows, 30.0, -1.0)
    xs = (np.arange(S["m"]) % 5 - 2).astype(np.float64)
    b = oracle.spmv_csr(S["m"], S["ptr"], S["idx"], S["val"], xs, np.zeros(S["m"]), 1.0, 0.0)
    for fmt in ("csr", "csc"):
        B = gen.transpose(S) if fmt == "csc" else S
        ctx = M.Context.from_torch_dist(device=local, parts_per_rank=1)
        ctx.partition(fmt, S["m"], S["n"], ptr=B["ptr"], idx=B["idx"], val=B["val"])
        xc = torch.zeros(S["m"], dtype=torch.float64, device="cuda")
        it, rr = ctx.cg(torch.as_tensor(b).cuda(), xc, tol=1e-12, maxit=300)
        if not (rr <= 1e-12 and np.max(np.abs(xc.cpu().numpy() - xs)) < 1e-9):
            fails.append(f"FAIL rank {rank} cg {fmt}: it {it} relres {rr}")
        ctx.close()
    for f in fails:
        print(f, flush=True)
    ok = torch.tensor([len(fails)], device="cuda")
    dist.all_reduce(ok)
    dist.destroy_process_group()
    if rank == 0:
        print(f"multirank world={world}: {'OK' if int(ok) == 0 else 'FAILED'}", flush=True)
    return 0 if int(ok) == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
