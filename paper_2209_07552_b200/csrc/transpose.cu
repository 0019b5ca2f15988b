// transpose.cu -- partition-time GPU kernels that put a column-format slice on row tiles.
//
// The column formats (pCSC, column-sorted and unsorted pCOO) hand each rank a contiguous range of
// nonzeros in column order (Alg. 4 / 6).  The paper runs the CSR SpMV
// kernel on such a part "with transpose on"; here the rank's slice is transposed ONCE, at
// partition time and on the GPU ("we offload the most expensive workload to GPUs as specially
// designed kernels"), into the rank-local row-major slice that pack_kernel turns into the
// row tiles rows_kernel walks.  What a call computes for the part is unchanged: y_p = A_p x over
// the part's entries, merged column-style.
//
// The transposition is a STABLE sort of the slice's entries by row: entries of one row keep their
// slice order (column order; for unsorted pCOO the triplet order), so the layout -- and the bits of
// every SpMV on it -- depend only on the input.  LSD radix sort of (row, slice position) pairs,
// 8-bit digits, 4096-entry tiles; per pass:
//   rs_hist_kernel     digit histogram of every tile, stored digit-major [digit][tile]
//   rs_scan_*          exclusive scan of that table (3 kernels): the first output slot of every
//                      (digit, tile) -- digits in order, tiles in order within a digit (stability)
//   rs_scatter_kernel  each warp ranks its 512 consecutive entries 32 at a time (match.any per
//                      digit, lanes in order), per-warp digit counts are prefixed across the tile's
//                      warps, and every entry goes to its slot
// then row_ptr_kernel (the row pointer, by binary search of the sorted rows) and permute_kernel
// (column ids and values in row order).  No atomics on the output positions: deterministic.
#include <cstdint>

#include "internal.h"

namespace msrep {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int RS_THREADS = 256, RS_WARPS = RS_THREADS / 32;
constexpr int RS_IPT = 16;                              // entries per thread per tile
constexpr int RS_TILE = RS_THREADS * RS_IPT;            // 4096 entries per tile
constexpr int RS_WARP_SPAN = RS_TILE / RS_WARPS;        // 512 consecutive entries per warp
constexpr int RS_BINS = 256;
constexpr int SCAN_CHUNK = RS_THREADS * 16;             // scan: entries per block

// warp per column: col[z] = w for z in [lp[w], lp[w+1])
__global__ void expand_cols_kernel(const int64_t* __restrict__ lp, int64_t W, int32_t* __restrict__ col) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < W; w += nw) {
    const int64_t z1 = lp[w + 1];
    for (int64_t z = lp[w] + lane; z < z1; z += 32) col[z] = (int32_t)w;
  }
}

// c[i] = v[i] - base (the rank-local column of a column-sorted / unsorted pCOO entry)
__global__ void rebase_cols_kernel(const int32_t* __restrict__ v, int64_t n, int32_t base, int32_t* __restrict__ c) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c[i] = v[i] - base;
}

__global__ void __launch_bounds__(RS_THREADS) rs_hist_kernel(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                                              uint32_t* __restrict__ hist, int64_t ntiles) {
  __shared__ uint32_t h[RS_BINS];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll 4
  for (int j = 0; j < RS_IPT; j++) {
    const int64_t i = base + j * RS_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & (RS_BINS - 1)], 1u);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// block-wide exclusive scan of one value per thread; returns the block total in *total
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t ws[RS_WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) ws[warp] = incl;
  __syncthreads();
  uint32_t wpre = 0, tot = 0;
  for (int w = 0; w < RS_WARPS; w++) {
    const uint32_t t = ws[w];
    if (w < warp) wpre += t;
    tot += t;
  }
  __syncthreads();   // ws may be reused by the caller's next call
  *total = tot;
  return wpre + incl - v;
}

// bsum[b] = sum of a[b*SCAN_CHUNK .. +SCAN_CHUNK)
__global__ void __launch_bounds__(RS_THREADS) rs_scan_reduce_kernel(const uint32_t* __restrict__ a, int64_t L,
                                                                     uint32_t* __restrict__ bsum) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_CHUNK + (int64_t)threadIdx.x * 16;
  uint32_t v = 0;
#pragma unroll
  for (int j = 0; j < 16; j++)
    if (base + j < L) v += a[base + j];
  uint32_t tot;
  block_excl_scan(v, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// exclusive scan of bsum[0, nb) in place (one block)
__global__ void __launch_bounds__(RS_THREADS) rs_scan_top_kernel(uint32_t* __restrict__ bsum, int64_t nb) {
  uint32_t carry = 0;
  for (int64_t c0 = 0; c0 < nb; c0 += RS_THREADS) {
    const int64_t i = c0 + threadIdx.x;
    const uint32_t v = i < nb ? bsum[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan(v, &tot);
    if (i < nb) bsum[i] = carry + ex;
    carry += tot;
  }
}

// a[i] = bsum[block] + exclusive prefix of a within the block's chunk (in place)
__global__ void __launch_bounds__(RS_THREADS) rs_scan_down_kernel(uint32_t* __restrict__ a, int64_t L,
                                                                   const uint32_t* __restrict__ bsum) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_CHUNK + (int64_t)threadIdx.x * 16;
  uint32_t v[16], s = 0;
#pragma unroll
  for (int j = 0; j < 16; j++) {
    v[j] = base + j < L ? a[base + j] : 0u;
    s += v[j];
  }
  uint32_t tot;
  uint32_t run = bsum[blockIdx.x] + block_excl_scan(s, &tot);
#pragma unroll
  for (int j = 0; j < 16; j++) {
    if (base + j < L) a[base + j] = run;
    run += v[j];
  }
}

// vals_in == nullptr: the value of entry i is i (the first pass: slice positions)
__global__ void __launch_bounds__(RS_THREADS) rs_scatter_kernel(const uint32_t* __restrict__ keys_in,
                                                                 const uint32_t* __restrict__ vals_in, int64_t n,
                                                                 int shift, const uint32_t* __restrict__ offs,
                                                                 int64_t ntiles, uint32_t* __restrict__ keys_out,
                                                                 uint32_t* __restrict__ vals_out) {
  __shared__ uint32_t wc[RS_WARPS][RS_BINS];   // per-warp digit counts, then their prefix over warps
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < RS_WARPS * RS_BINS; i += RS_THREADS) (&wc[0][0])[i] = 0;
  __syncthreads();
  const int64_t tile = blockIdx.x;
  const int64_t base = tile * RS_TILE + (int64_t)warp * RS_WARP_SPAN;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t k[RS_IPT], v[RS_IPT], rk[RS_IPT];
#pragma unroll
  for (int r = 0; r < RS_IPT; r++) {
    const int64_t i = base + r * 32 + lane;
    const bool ok = i < n;
    k[r] = ok ? keys_in[i] : 0u;
    v[r] = ok ? (vals_in ? vals_in[i] : (uint32_t)i) : 0u;
    const uint32_t d = ok ? (k[r] >> shift) & (RS_BINS - 1) : (uint32_t)RS_BINS;   // RS_BINS: past the end
    const uint32_t peers = __match_any_sync(FULL, d);
    const uint32_t before = ok ? wc[warp][d] : 0u;
    __syncwarp();
    if (ok && (peers & lt) == 0) wc[warp][d] = before + __popc(peers);   // the group's lowest lane
    __syncwarp();
    rk[r] = before + __popc(peers & lt);
  }
  __syncthreads();
  {   // digit = thread: exclusive prefix of the per-warp counts in warp order
    uint32_t s = 0;
    for (int w = 0; w < RS_WARPS; w++) {
      const uint32_t t = wc[w][threadIdx.x];
      wc[w][threadIdx.x] = s;
      s += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RS_IPT; r++) {
    const int64_t i = base + r * 32 + lane;
    if (i < n) {
      const uint32_t d = (k[r] >> shift) & (RS_BINS - 1);
      const int64_t dst = (int64_t)offs[(int64_t)d * ntiles + tile] + wc[warp][d] + rk[r];
      keys_out[dst] = k[r];
      vals_out[dst] = v[r];
    }
  }
}

// ptr[r] = number of sorted rows < r, r in [0, m]
__global__ void row_ptr_kernel(const uint32_t* __restrict__ rows, int64_t n, int64_t m, int32_t* __restrict__ ptr) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= m; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)rows[mid] < r) lo = mid + 1; else hi = mid;
    }
    ptr[r] = (int32_t)lo;
  }
}

template <typename VT>
__global__ void permute_kernel(const uint32_t* __restrict__ perm, int64_t n, const int32_t* __restrict__ col_in,
                               const VT* __restrict__ val_in, int32_t* __restrict__ col_out, VT* __restrict__ val_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = perm[i];
    col_out[i] = col_in[p];
    val_out[i] = val_in[p];
  }
}

int grid_of(int64_t n, int per_block) {
  const int64_t g = (n + per_block - 1) / per_block;
  return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

}  // namespace

int64_t transpose_scratch_words(int64_t n) {
  const int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
  const int64_t L = (int64_t)RS_BINS * ntiles;
  return L + (L + SCAN_CHUNK - 1) / SCAN_CHUNK + 64;
}

cudaError_t launch_expand_cols(const int64_t* lp, int64_t W, int32_t* col, cudaStream_t s) {
  if (W <= 0) return cudaSuccess;
  expand_cols_kernel<<<grid_of(W, 8), 256, 0, s>>>(lp, W, col);
  return cudaGetLastError();
}

cudaError_t launch_rebase_cols(const int32_t* v, int64_t n, int32_t base, int32_t* c, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  rebase_cols_kernel<<<grid_of(n, 256), 256, 0, s>>>(v, n, base, c);
  return cudaGetLastError();
}

cudaError_t launch_transpose(const TransposeLaunch& T, cudaStream_t s) {
  const int64_t n = T.n;
  int bits = 0;
  while (bits < 32 && ((int64_t)1 << bits) < T.m) bits++;   // rows < m <= 2^bits
  const int passes = (bits + 7) / 8;
  const uint32_t* kin = T.rows;
  const uint32_t* vin = nullptr;   // pass 0: identity
  const int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
  const int64_t L = (int64_t)RS_BINS * ntiles;
  const int64_t nb = (L + SCAN_CHUNK - 1) / SCAN_CHUNK;
  uint32_t* hist = T.scratch;
  uint32_t* bsum = T.scratch + L;
  const uint32_t* sorted_rows = T.rows;
  const uint32_t* perm = nullptr;
  if (n > 0) {
    for (int p = 0; p < passes; p++) {
      uint32_t* kout = (p & 1) ? T.key_b : T.key_a;
      uint32_t* vout = (p & 1) ? T.perm_b : T.perm_a;
      rs_hist_kernel<<<(unsigned)ntiles, RS_THREADS, 0, s>>>(kin, n, 8 * p, hist, ntiles);
      rs_scan_reduce_kernel<<<(unsigned)nb, RS_THREADS, 0, s>>>(hist, L, bsum);
      rs_scan_top_kernel<<<1, RS_THREADS, 0, s>>>(bsum, nb);
      rs_scan_down_kernel<<<(unsigned)nb, RS_THREADS, 0, s>>>(hist, L, bsum);
      rs_scatter_kernel<<<(unsigned)ntiles, RS_THREADS, 0, s>>>(kin, vin, n, 8 * p, hist, ntiles, kout, vout);
      kin = kout;
      vin = vout;
    }
    sorted_rows = kin;
    perm = vin;
  }
  row_ptr_kernel<<<grid_of(T.m + 1, 256), 256, 0, s>>>(sorted_rows, n, T.m, T.ptr_out);
  if (n > 0) {
    if (!perm) {   // m <= 1: every entry is in row 0 and the slice order stands
      if (T.cols_out != T.cols)
        cudaMemcpyAsync(T.cols_out, T.cols, (size_t)n * 4, cudaMemcpyDeviceToDevice, s);
      cudaMemcpyAsync(T.vals_out, T.vals, (size_t)n * (size_t)T.V, cudaMemcpyDeviceToDevice, s);
    } else if (T.V == 8) {
      permute_kernel<double><<<grid_of(n, 256), 256, 0, s>>>(perm, n, T.cols, (const double*)T.vals, T.cols_out,
                                                             (double*)T.vals_out);
    } else {
      permute_kernel<float><<<grid_of(n, 256), 256, 0, s>>>(perm, n, T.cols, (const float*)T.vals, T.cols_out,
                                                            (float*)T.vals_out);
    }
  }
  return cudaGetLastError();
}

}  // namespace msrep
