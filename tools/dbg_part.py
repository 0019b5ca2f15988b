"""Debug: time one part of an nnz-balanced plan alone with both x-gather policies + stats."""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen, paper_2209_07552_b200 as M
cfg, p, j = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
A = gen.make_config(cfg)
plan = M.msrep_plan(M.CSR, A["m"], A.nnz, p, ptr=A["ptr"])
d = plan[j]
b0, b1 = int(d["start_idx"]), int(d["end_idx"]) + 1
o0, o1 = int(d["start_row"]), int(d["end_row"]) + 1
ptr = np.clip(A["ptr"][o0:o1 + 1], b0, b1) - b0
x = torch.as_tensor(gen.vector(A["n"], 7)).cuda()
for pol in (0, 1, -1):
    ctx = M.Context(0, 1, None, 0, 1)
    ctx.set_tuning("xload", pol)
    ctx.partition("csr", o1 - o0, A["n"], ptr=ptr, idx=A["idx"][b0:b1], val=A["val"][b0:b1])
    y = torch.zeros(o1 - o0, dtype=torch.float64, device="cuda")
    for _ in range(3): ctx.spmv(1.0, x, 0.0, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): ctx.spmv(1.0, x, 0.0, y)
    e1.record(); torch.cuda.synchronize()
    st = ctx.stats()
    print(json.dumps({"pol": pol, "ms": e0.elapsed_time(e1) / 20, "rows": o1 - o0, "nnz": b1 - b0,
                      **{k: st[k] for k in ("ntiles", "nsell", "nslabs", "nsplit_rows", "tile_bytes", "x_no_allocate", "distinct_cols")}}), flush=True)
    ctx.close()
