// tools/membench.cu -- read-bandwidth ceilings on this B200 for the staging
// strategies the SpMV kernels can use (not part of the product):
//   ldg   : grid-stride ld.global.nc.v4 stream, U 16-byte loads in flight per thread
//   tma   : persistent CTAs, 1 producer warp + 8 consumer warps, S-stage ring of
//           CHUNK-byte cp.async.bulk copies (the rows_kernel pipeline, no compute)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench tools/membench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int U>
__global__ void ldg_stream(const int4* __restrict__ a, size_t n16, int* out) {
  int acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride * U) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      size_t j = i + u * stride;
      if (j < n16) asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(a + j));
      else v[u] = make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; u++) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

__global__ void tma_stream(const char* __restrict__ a, size_t bytes, int chunk, int S, int* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = (uint64_t*)(smem + (size_t)S * chunk);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NW = (blockDim.x / 32) - 1;
  if (tid == 0) {
    for (int s = 0; s < S; s++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(&empty[s])), "r"(NW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t nchunks = bytes / chunk;
  if (warp == NW) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      for (int i = 0;; i++) {
        size_t t = blockIdx.x + (size_t)i * gridDim.x;
        if (t >= nchunks) break;
        int s = i % S;
        if (i >= S) {
          uint32_t ph = ((i / S) - 1) & 1;
          asm volatile("{ .reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @P1 bra D; bra W; D: }" ::"r"(saddr(&empty[s])), "r"(ph));
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&full[s])), "r"(chunk));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(saddr(smem + (size_t)s * chunk)), "l"(a + t * chunk), "r"(chunk), "r"(saddr(&full[s])), "l"(pol) : "memory");
      }
    }
    return;
  }
  int acc = 0;
  for (int i = 0;; i++) {
    size_t t = blockIdx.x + (size_t)i * gridDim.x;
    if (t >= nchunks) break;
    int s = i % S;
    uint32_t ph = (i / S) & 1;
    asm volatile("{ .reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @P1 bra D; bra W; D: }" ::"r"(saddr(&full[s])), "r"(ph));
    acc ^= ((const int*)(smem + (size_t)s * chunk))[tid];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(&empty[s])));
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  const size_t bytes = (size_t)1 << 30;   // 1 GiB read per pass
  char* a; int* out;
  cudaMalloc(&a, bytes + 4096); cudaMalloc(&out, 64);
  cudaMemset(a, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](auto launch, const char* name) {
    for (int w = 0; w < 3; w++) launch();
    cudaEventRecord(e0);
    const int R = 10;
    for (int r = 0; r < R; r++) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("%-40s %8.1f GB/s %s\n", name, bytes * (double)R / (ms * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
  };
  for (int bpsm : {4, 8, 16}) {
    char nm[64]; snprintf(nm, 64, "ldg U=8 256thr x %d/SM", bpsm);
    timeit([&] { ldg_stream<8><<<sms * bpsm, 256>>>((const int4*)a, bytes / 16, out); }, nm);
  }
  timeit([&] { ldg_stream<4><<<sms * 8, 256>>>((const int4*)a, bytes / 16, out); }, "ldg U=4 256thr x 8/SM");
  for (int chunk : {8192, 16384, 32768}) {
    for (int S : {2, 3, 4, 6}) {
      for (int ctas : {1, 2}) {
        size_t sm = (size_t)S * chunk + 2 * S * 8;
        if (sm * ctas > 220 * 1024) continue;
        cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        char nm[64]; snprintf(nm, 64, "tma chunk=%dK S=%d ctas/SM=%d", chunk / 1024, S, ctas);
        timeit([&] { tma_stream<<<sms * ctas, 288, sm>>>(a, bytes, chunk, S, out); }, nm);
      }
    }
  }
  return 0;
}
