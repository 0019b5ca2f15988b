"""Cost of the fused allgather stores (msrep_spmv_mirror) on one B200 with LOCAL mirrors
(stand-ins for peer buffers): stencil pCSR fp64, 0 / 1 / 3 / 7 mirrors -> ms per SpMV."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import paper_2209_07552_b200 as M  # noqa: E402

A = gen.make_config("stencil")
ctx = M.Context(0, 1, None, 0, 1)
ctx.partition("csr", A["m"], A["n"], ptr=A["ptr"], idx=A["idx"], val=A["val"])
x = torch.as_tensor(gen.vector(A["n"], 1)).cuda()
y = torch.as_tensor(gen.vector(A["m"], 2)).cuda()
for nm in (0, 1, 3, 7):
    mirrors = [torch.empty(A["m"], dtype=torch.float64, device="cuda") for _ in range(nm)]
    f = (lambda: ctx.spmv(1.5, x, 0.5, y)) if nm == 0 else (lambda: ctx.spmv_mirror(1.5, x, 0.5, y, mirrors))
    for _ in range(10):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(200):
        f()
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"mirrors": nm, "ms_per_spmv": e0.elapsed_time(e1) / 200,
                      "mirror_bytes": nm * A["m"] * 8}), flush=True)
