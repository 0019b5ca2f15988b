"""Cost of the partition's device allocations on the box: cudaMalloc + cudaFree vs the stream-ordered
pool (cudaMallocAsync / cudaFreeAsync + sync), for the sizes an R-MAT scale-24 partition uses."""
import time
from cuda.bindings import runtime as rt

rt.cudaSetDevice(0)
rt.cudaFree(0)
_, s = rt.cudaStreamCreate()
for gb in (0.25, 1.0, 2.0, 4.0):
    n = int(gb * (1 << 30))
    t0 = time.perf_counter(); e, p = rt.cudaMalloc(n); t1 = time.perf_counter()
    rt.cudaMemsetAsync(p, 0, n, s); rt.cudaStreamSynchronize(s)
    t2 = time.perf_counter(); rt.cudaFree(p); t3 = time.perf_counter()
    e, q = rt.cudaMallocAsync(n, s); t4 = time.perf_counter()
    rt.cudaMemsetAsync(q, 0, n, s); rt.cudaStreamSynchronize(s)
    t5 = time.perf_counter(); rt.cudaFreeAsync(q, s); rt.cudaStreamSynchronize(s); t6 = time.perf_counter()
    print(f"{gb:5.2f} GB  cudaMalloc {1e3*(t1-t0):7.2f} ms  cudaFree {1e3*(t3-t2):7.2f} ms  "
          f"MallocAsync {1e3*(t4-t3):7.2f} ms  FreeAsync+sync {1e3*(t6-t5):7.2f} ms", flush=True)
