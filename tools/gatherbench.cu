// tools/gatherbench.cu -- random x-gather throughput on this B200 (not part of the product):
//   ldg  : per-lane ld.global.nc.L1::no_allocate of x[idx] (the kernels' path), U in flight/thread
//   tma4 : cp.async.bulk.tensor.2d ... tile::gather4 -- x viewed as [n/2][2] fp64 rows of 16 B,
//          one instruction fetches 4 rows into shared memory (8 lanes x 4 = 32 entries per stage)
// Question: is TMA gather4 limited by the same L1TEX -> L2 request rate
// (~1 per SM clock) that bounds the LSU gathers of R-MAT / tall-skinny?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gatherbench tools/gatherbench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}
__global__ void fill(int* idx, double* x, int64_t N, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    idx[i] = (int)(hash32((uint32_t)i * 2654435761u + 12345u) % (uint32_t)n);
    if (i < n) x[i] = (double)(i % 7);
  }
}

template <int U>
__global__ void ldg_gather(const int* __restrict__ idx, const double* __restrict__ x, int64_t N, double* out) {
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < N; b += stride * U) {
    int c[U];
#pragma unroll
    for (int u = 0; u < U; u++) c[u] = b + u * stride < N ? __ldcs(idx + b + u * stride) : 0;
    double v[U];
#pragma unroll
    for (int u = 0; u < U; u++)
      asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v[u]) : "l"(x + c[u]));
#pragma unroll
    for (int u = 0; u < U; u++) acc += v[u];
  }
  if (acc == -1.0) out[0] = acc;
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S>
__global__ void tma4_gather(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx, int64_t N,
                            double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwl = blockDim.x >> 5;
  unsigned char* buf = smem + warp * S * 1024;   // each gather4 destination 128-B aligned
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + nwl * S * 1024) + warp * S;
  const int64_t nchunk = N / 32, gw = blockIdx.x * (int64_t)nwl + warp, nw = (int64_t)gridDim.x * nwl;
  if (lane == 0)
    for (int s = 0; s < S; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto issue = [&](int64_t ch, int s, int myc) {
    // lane 0 arms the stage; lanes 0..7 each gather 4 rows (entries 4l .. 4l+3)
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 512;" ::"r"(sa(&bar[s])) : "memory");
    const int r0 = __shfl_sync(0xffffffffu, myc >> 1, (lane & 7) * 4 + 0);
    const int r1 = __shfl_sync(0xffffffffu, myc >> 1, (lane & 7) * 4 + 1);
    const int r2 = __shfl_sync(0xffffffffu, myc >> 1, (lane & 7) * 4 + 2);
    const int r3 = __shfl_sync(0xffffffffu, myc >> 1, (lane & 7) * 4 + 3);
    if (lane < 8) {
      const uint32_t dst = sa(buf + s * 1024 + lane * 128);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
          "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sa(&bar[s]))
          : "memory");
    }
    (void)ch;
  };
  int cs[S];
  double acc = 0.0;
#pragma unroll
  for (int s = 0; s < S; s++) {
    const int64_t ch = gw + s * nw;
    cs[s] = ch < nchunk ? idx[ch * 32 + lane] : 0;
    if (ch < nchunk) issue(ch, s, cs[s]);
  }
  for (int64_t i = 0;; i += S) {
#pragma unroll
    for (int s = 0; s < S; s++) {
      const int64_t ch = gw + (i + s) * nw;
      if (ch >= nchunk) goto done;
      const uint32_t ph = (uint32_t)((i / S) & 1);
      asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W; }" ::"r"(sa(&bar[s])), "r"(ph) : "memory");
      acc += *reinterpret_cast<const double*>(buf + s * 1024 + (lane >> 2) * 128 + (lane & 3) * 16 + (cs[s] & 1) * 8);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      const int64_t nx = ch + (int64_t)S * nw;
      if (nx < nchunk) {
        cs[s] = idx[nx * 32 + lane];
        issue(nx, s, cs[s]);
      }
    }
  }
done:
  if (acc == -1.0) out[0] = acc;
}

int main(int argc, char** argv) {
  const int64_t N = (int64_t)1 << 27;   // gathers
  cuInit(0);
  auto* encode = &cuTensorMapEncodeTiled;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* idx; double *x, *out;
  cudaMalloc(&idx, N * 4);
  cudaMalloc(&out, 8);
  for (int64_t n : {(int64_t)1 << 20, (int64_t)1 << 24}) {
    cudaMalloc(&x, n * 8);
    fill<<<sms * 8, 256>>>(idx, x, N, n);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms = 0;
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(e0);
      ldg_gather<8><<<sms * 8, 256>>>(idx, x, N, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("ldg   n=%lld  %.3f ms  %.1f G gathers/s  (%s)\n", (long long)n, ms, N / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
    CUtensorMap tm;
    cuuint64_t dims[2] = {2, (cuuint64_t)(n / 2)};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    constexpr int S = 8;
    for (int warps : {8, 16}) {
      const int smem = warps * S * 1024 + warps * S * 8;
      cudaFuncSetAttribute(tma4_gather<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        tma4_gather<S><<<sms * 2, warps * 32, smem>>>(tm, idx, N, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      printf("tma4  n=%lld  warps/CTA=%d  %.3f ms  %.1f G gathers/s  (%s)\n", (long long)n, warps, ms,
             N / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(x);
  }
  return 0;
}
