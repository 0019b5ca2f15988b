"""tools/partition_probe.py CONFIG [FMT] [DTYPE] [REPS]: partition a config REPS times in one process and print
the partition phases (stats.phase_ms, stats.layout_ms) -- separates first-touch / allocation effects
from the steady-state cost of msrep_partition."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import paper_2209_07552_b200 as M  # noqa: E402

cfg = sys.argv[1]
fmt = sys.argv[2] if len(sys.argv) > 2 else None
dt = sys.argv[3] if len(sys.argv) > 3 else "f64"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
torch.cuda.set_device(0)
t0 = time.time()
A = gen.make_config(cfg)
if dt == "f32":
    A["val"] = A["val"].astype(np.float32)
fmt = fmt or A["fmt"]
print(f"generate {time.time() - t0:.1f} s  fmt={A['fmt']} nnz={A.nnz}", flush=True)
for r in range(reps):
    ctx = M.Context(0, 1, None, 0, 1)
    t0 = time.time()
    ctx.partition(fmt, A["m"], A["n"], ptr=A["ptr"], idx=A["idx"], val=A["val"])
    wall = time.time() - t0
    st = ctx.stats()
    print(f"rep {r}: wall {wall * 1e3:.0f} ms  partition_ms {st['partition_ms']:.0f}  phases "
          f"{[round(v) for v in st['phase_ms']]}  layout {[round(v) for v in st['layout_ms']]}", flush=True)
    ctx.close()
