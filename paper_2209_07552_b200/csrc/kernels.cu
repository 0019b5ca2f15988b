// kernels.cu -- sm_100a kernels of the msRep hot path (arXiv 2209.07552).
//
// SpMV is HBM-bound (0.17 flop/B in fp64, "memory bound ... main
// cost of SpMV comes from accessing the nonzero elements"), so no tensor cores:
// the design goal is to keep enough bytes in flight to saturate HBM3e.
//
//  rows_kernel  pCSR / pCOO per-GPU SpMV (Alg. 3 / Alg. 7 "Launch:
//               py[i]=<csrSpMVKernel>").  Persistent CTAs
//               walk a static, row-aligned tile schedule built at partition
//               time.  Each tile's val / col_idx / row-pointer (or COO row_idx)
//               slices are staged into shared memory with 1-D TMA bulk copies
//               (cp.async.bulk + mbarrier, L2 evict_first) in an S-stage ring;
//               products val*x[col] are formed in a coalesced pass (x gathered
//               through the read-only path), then a merge-path walk (CSR) or a
//               key-segmented walk (COO) plus a deterministic block segmented
//               scan produces whole-row sums, written as y = alpha*s + beta*y
//               in a coalesced epilogue.  Split rows (rows shared with another
//               part, and rows longer than a tile) are "slab" tiles
//               whose partial goes to a record -- no float atomics, so results
//               are bit-reproducible.
//  fixup_kernel the beta-deferred merge of split rows (reading R6):
//               y_r = alpha*(tail records + head partials, part order) + beta*y_r.
//  cols_kernel  pCSC scatter (Alg. 5; "switch the role of x and
//               y") into a full-length fp64 partial vector py with
//               red.global.add.f64, same TMA tile staging.
#include <climits>
#include <cstdint>

#include "internal.h"

namespace msrep {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int STAGES = 2;

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      " .reg .pred P1;\n"
      "LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra DONE;\n"
      " bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(saddr(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 1-D bulk copy global -> shared (TMA, no tensor map); bytes % 16 == 0, both addresses 16-B aligned.
__device__ __forceinline__ void tma_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar)), "l"(pol)
      : "memory");
}

template <typename T>
__device__ __forceinline__ T ldg_ro(const T* p) { return __ldg(p); }

// ---------------------------------------------------------------- layout
template <typename VT>
struct RowSmem {
  static constexpr int VPA = 16 / (int)sizeof(VT);                       // values per 16 bytes
  static constexpr int VAL_B = (((TILE_ITEMS + VPA) * (int)sizeof(VT)) + 15) & ~15;
  static constexpr int COL_B = (((TILE_ITEMS + 4) * 4) + 15) & ~15;
  static constexpr int AUX_B = (((TILE_ITEMS + 8) * 4) + 15) & ~15;
  static constexpr int STAGE_B = VAL_B + COL_B + AUX_B;
  static constexpr int BUF_OFF = STAGES * STAGE_B;                       // fp64 products / row sums [TILE_ITEMS]
  static constexpr int BAR_OFF = BUF_OFF + TILE_ITEMS * 8;
  static constexpr int DESC_OFF = (BAR_OFF + 2 * STAGES * 8 + 15) & ~15; // full/empty mbarriers, then int4 descriptors
  static constexpr int WK_OFF = DESC_OFF + STAGES * 16;
  static constexpr int WV_OFF = WK_OFF + 32;
  static constexpr int TOTAL = WV_OFF + 64;
};

// Deterministic block-wide exclusive segmented scan of (key, value) pairs whose
// keys are non-decreasing in thread order.  op((ka,va),(kb,vb)) =
// (kb, ka==kb ? va+vb : vb).  Returns the exclusive prefix (INT_MIN key if none).
__device__ __forceinline__ void block_seg_scan(int key, double val, int& pk, double& pv, int* swk, double* swv) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int ik = key;
  double iv = val;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int k2 = __shfl_up_sync(FULL, ik, off);
    double v2 = __shfl_up_sync(FULL, iv, off);
    if (lane >= off && k2 == ik) iv = v2 + iv;
  }
  if (lane == 31) { swk[warp] = ik; swv[warp] = iv; }
  __syncthreads();
  int wk = INT_MIN;
  double wv = 0.0;
  for (int w = 0; w < warp; w++) {
    int k2 = swk[w];
    double v2 = swv[w];
    if (k2 == wk) wv = wv + v2; else { wk = k2; wv = v2; }
  }
  int ek = __shfl_up_sync(FULL, ik, 1);
  double ev = __shfl_up_sync(FULL, iv, 1);
  if (lane == 0) { pk = wk; pv = wv; }
  else { pk = ek; pv = (wk == ek) ? wv + ev : ev; }
}

// Issue the TMA copies of one tile into a stage (thread 0 only).
template <typename VT, bool COO>
__device__ __forceinline__ void issue_row_tile(const RowLaunch& P, int4 d, unsigned char* st, uint64_t* bar,
                                               uint64_t pol) {
  using L = RowSmem<VT>;
  const int nrows = d.z & 0xffff, nnz = d.z >> 16;
  const bool slab = d.w >= 0;
  uint32_t vb = 0, cb = 0, ab = 0;
  int64_t v0 = 0, c0 = 0, a0 = 0;
  if (nnz > 0) {
    v0 = (int64_t)d.y & ~(int64_t)(L::VPA - 1);
    int64_t v1 = ((int64_t)d.y + nnz + L::VPA - 1) & ~(int64_t)(L::VPA - 1);
    vb = (uint32_t)((v1 - v0) * (int64_t)sizeof(VT));
    c0 = (int64_t)d.y & ~(int64_t)3;
    int64_t c1 = ((int64_t)d.y + nnz + 3) & ~(int64_t)3;
    cb = (uint32_t)((c1 - c0) * 4);
    if (COO && !slab) { a0 = c0; ab = cb; }
  }
  if (!COO && !slab) {
    a0 = (int64_t)d.x & ~(int64_t)3;
    int64_t a1 = ((int64_t)d.x + nrows + 1 + 3) & ~(int64_t)3;
    ab = (uint32_t)((a1 - a0) * 4);
  }
  mbar_arrive_expect_tx(bar, vb + cb + ab);
  if (vb) tma_1d(st, (const VT*)P.val + v0, vb, bar, pol);
  if (cb) tma_1d(st + L::VAL_B, P.col + c0, cb, bar, pol);
  if (ab) tma_1d(st + L::VAL_B + L::COL_B, P.aux + a0, ab, bar, pol);
}

// Consumer-only barrier (named barrier 1, the THREADS consumer threads; the
// producer warp never takes part).
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(THREADS) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(bar)) : "memory");
}

// Same as block_seg_scan but synchronising only the consumer warps.
__device__ __forceinline__ void consumer_seg_scan(int key, double val, int& pk, double& pv, int* swk, double* swv) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int ik = key;
  double iv = val;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int k2 = __shfl_up_sync(FULL, ik, off);
    double v2 = __shfl_up_sync(FULL, iv, off);
    if (lane >= off && k2 == ik) iv = v2 + iv;
  }
  if (lane == 31) { swk[warp] = ik; swv[warp] = iv; }
  consumer_sync();
  int wk = INT_MIN;
  double wv = 0.0;
  for (int w = 0; w < warp; w++) {
    int k2 = swk[w];
    double v2 = swv[w];
    if (k2 == wk) wv = wv + v2; else { wk = k2; wv = v2; }
  }
  int ek = __shfl_up_sync(FULL, ik, 1);
  double ev = __shfl_up_sync(FULL, iv, 1);
  if (lane == 0) { pk = wk; pv = wv; }
  else { pk = ek; pv = (wk == ek) ? wv + ev : ev; }
}

constexpr int VEC_UNROLL = 16;

// Warp-specialised persistent kernel: warp THREADS/32 is the TMA producer
// (one elected lane walks this CTA's tiles, waits for a free stage, issues the
// bulk copies); warps 0..THREADS/32-1 consume.  Stages are released per warp
// through an "empty" mbarrier, so vector tiles need no CTA-wide barrier at all.
template <typename VT, bool COO>
__global__ void __launch_bounds__(THREADS + 32, 2) rows_kernel(const RowLaunch P) {
  using L = RowSmem<VT>;
  constexpr int NW = THREADS / 32;
  extern __shared__ __align__(128) unsigned char smem[];
  double* sbuf = reinterpret_cast<double*>(smem + L::BUF_OFF);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  int4* sdesc = reinterpret_cast<int4*>(smem + L::DESC_OFF);
  int* swk = reinterpret_cast<int*>(smem + L::WK_OFF);
  double* swv = reinterpret_cast<double*>(smem + L::WV_OFF);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], NW); }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NW) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int i = 0;; i++) {
        const int t = blockIdx.x + i * gridDim.x;
        if (t >= P.ntiles) break;
        const int s = i % STAGES;
        const int4 d = P.tiles[t];
        if (i >= STAGES) mbar_wait(&empty[s], (uint32_t)(((i / STAGES) - 1) & 1));
        sdesc[s] = d;
        fence_proxy_async();
        issue_row_tile<VT, COO>(P, d, smem + s * L::STAGE_B, &full[s], pol);
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const VT* __restrict__ x = static_cast<const VT*>(P.x);
  VT* __restrict__ y = static_cast<VT*>(P.y);
  const double alpha = P.alpha, beta = P.beta;

  for (int i = 0;; i++) {
    const int t = blockIdx.x + i * gridDim.x;
    if (t >= P.ntiles) break;
    const int s = i % STAGES;
    mbar_wait(&full[s], (uint32_t)((i / STAGES) & 1));
    const int4 d = sdesc[s];
    unsigned char* st = smem + s * L::STAGE_B;
    const int nrows = d.z & 0xffff, nnz = d.z >> 16;
    const VT* sv = reinterpret_cast<const VT*>(st) + (d.y & (L::VPA - 1));
    const int* sc = reinterpret_cast<const int*>(st + L::VAL_B) + (d.y & 3);

    if (!COO && d.w <= -2) {
      // ---- vector tile (pCSR, regular rows): L = 2^(-w-2) lanes per row, products fused into
      // the per-lane sums (no product pass), xor-shuffle tree, coalesced y.  L is chosen at
      // partition time from the tile's row-length profile (host.cpp, tile_mode()).
      const int lg = -d.w - 2;
      const int Lw = 1 << lg, G = THREADS >> lg;
      const int g = tid >> lg, j = tid & (Lw - 1);
      const int* sa = reinterpret_cast<const int*>(st + L::VAL_B + L::COL_B) + (d.x & 3);
      const int base = sa[0];
      const int64_t yrow0 = P.ybase + d.x;
      for (int rp = 0; rp < nrows; rp += G) {
        const int r = rp + g;
        double acc = 0.0, yv = 0.0;
        if (r < nrows) {
          if (beta != 0.0) yv = (double)y[yrow0 + r];
          const int ke = sa[r + 1] - base;
          for (int k = sa[r] - base + j; k < ke; k += VEC_UNROLL * Lw) {
            int cidx[VEC_UNROLL];
            VT xv[VEC_UNROLL];
#pragma unroll
            for (int u = 0; u < VEC_UNROLL; u++) { int kk = k + u * Lw; cidx[u] = kk < ke ? sc[kk] : 0; }
#pragma unroll
            for (int u = 0; u < VEC_UNROLL; u++) { int kk = k + u * Lw; xv[u] = kk < ke ? ldg_ro(x + cidx[u]) : VT(0); }
#pragma unroll
            for (int u = 0; u < VEC_UNROLL; u++) {
              int kk = k + u * Lw;
              if (kk < ke) acc = fma((double)sv[kk], (double)xv[u], acc);
            }
          }
        }
        for (int off = Lw >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(FULL, acc, off);
        if (r < nrows && j == 0) {
          double v = alpha * acc;
          if (beta != 0.0) v += beta * yv;
          y[yrow0 + r] = (VT)v;
        }
      }
    } else if (d.w >= 0) {
      // ---- slab: partial sum of one split row -> record (deterministic order)
      consumer_sync();   // swv reuse guard
      int cidx[8];
      VT xv[8];
#pragma unroll
      for (int u = 0; u < 8; u++) { int k = tid + u * THREADS; cidx[u] = k < nnz ? sc[k] : 0; }
#pragma unroll
      for (int u = 0; u < 8; u++) { int k = tid + u * THREADS; xv[u] = k < nnz ? ldg_ro(x + cidx[u]) : VT(0); }
      double acc = 0.0;
#pragma unroll
      for (int u = 0; u < 8; u++) { int k = tid + u * THREADS; if (k < nnz) acc += (double)sv[k] * (double)xv[u]; }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(FULL, acc, off);
      if (lane == 0) swv[warp] = acc;
      consumer_sync();
      if (tid == 0) {
        double tot = 0.0;
        for (int w = 0; w < NW; w++) tot = tot + swv[w];
        P.rec[d.w] = tot;
      }
    } else {
      // ---- merge-path (CSR) / key-walk (COO) tile: whole rows, irregular lengths
      consumer_sync();   // all consumers are done with the previous tile's sbuf / scratch
      const int64_t yrow0 = P.ybase + d.x;
      double yin[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        int r = tid + u * THREADS;
        yin[u] = (beta != 0.0 && r < nrows) ? (double)y[yrow0 + r] : 0.0;
      }
      // phase A: products, coalesced over the tile's nonzeros, 8 gathers in flight per thread
      {
        int cidx[8];
        VT xv[8];
#pragma unroll
        for (int u = 0; u < 8; u++) { int k = tid + u * THREADS; cidx[u] = k < nnz ? sc[k] : 0; }
#pragma unroll
        for (int u = 0; u < 8; u++) { int k = tid + u * THREADS; xv[u] = k < nnz ? ldg_ro(x + cidx[u]) : VT(0); }
#pragma unroll
        for (int u = 0; u < 8; u++) {
          int k = tid + u * THREADS;
          if (k < nnz) sbuf[k] = (double)sv[k] * (double)xv[u];
        }
      }
      if (COO)
        for (int r = tid; r < nrows; r += THREADS) sbuf[nnz + r] = 0.0;
      consumer_sync();

      double* rsum = sbuf + nnz;   // row sums live after the products (nrows + nnz <= TILE_ITEMS)
      int key;
      double acc = 0.0;
      int first = 0, nseg = 0;
      double firstv = 0.0;
      int k1 = 0, cur = 0;
      if (!COO) {
        // merge path over (row ends, nonzero indices) -- Merrill & Garland style, tile-local
        const int* sa = reinterpret_cast<const int*>(st + L::VAL_B + L::COL_B) + (d.x & 3);
        const int base = sa[0];
        const int items = nrows + nnz;
        const int per = (items + THREADS - 1) / THREADS;
        const int d0 = min(tid * per, items), d1 = min(d0 + per, items);
        int lo = max(0, d0 - nnz), hi = min(d0, nrows);
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          if (sa[mid + 1] - base <= d0 - mid - 1) lo = mid + 1; else hi = mid;
        }
        int xr = lo, yz = d0 - lo;
        first = xr;
        for (int dd = d0; dd < d1; dd++) {
          if (xr < nrows && yz < sa[xr + 1] - base) { acc += sbuf[yz]; yz++; }
          else { rsum[xr] = acc; acc = 0.0; xr++; }
        }
        key = xr;
        nseg = (xr > first) ? 2 : 1;   // >= 2 means the first row was completed here
      } else {
        // key-segmented walk over row_idx - row0 (pCOO row index rebased in-kernel)
        const int* sr = reinterpret_cast<const int*>(st + L::VAL_B + L::COL_B) + (d.y & 3);
        const int rg0 = (int)yrow0;
        const int per = (nnz + THREADS - 1) / THREADS;
        const int k0 = min(tid * per, nnz);
        k1 = min(k0 + per, nnz);
        cur = nrows + 1;
        if (k0 < k1) {
          cur = sr[k0] - rg0;
          nseg = 1;
          for (int k = k0; k < k1; k++) {
            int kk = sr[k] - rg0;
            if (kk != cur) {
              if (nseg == 1) { first = cur; firstv = acc; } else rsum[cur] = acc;
              nseg++;
              cur = kk;
              acc = 0.0;
            }
            acc += sbuf[k];
          }
        }
        key = cur;
      }
      int pk;
      double pv;
      consumer_seg_scan(key, acc, pk, pv, swk, swv);
      if (!COO) {
        if (nseg >= 2 && pk == first) rsum[first] += pv;
      } else {
        if (nseg >= 2) rsum[first] = (pk == first) ? firstv + pv : firstv;
        if (nseg >= 1) {
          const int* sr = reinterpret_cast<const int*>(st + L::VAL_B + L::COL_B) + (d.y & 3);
          bool last_of_row = (k1 >= nnz) || (sr[k1] - (int)yrow0 != cur);
          if (last_of_row) rsum[cur] = (pk == cur) ? pv + acc : acc;
        }
      }
      consumer_sync();
      // coalesced epilogue, alpha and beta applied exactly once per row
#pragma unroll
      for (int u = 0; u < 8; u++) {
        int r = tid + u * THREADS;
        if (r < nrows) {
          double v = alpha * rsum[r];
          if (beta != 0.0) v += beta * yin[u];
          y[yrow0 + r] = (VT)v;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);   // this warp is done with stage s
  }
}

// ------------------------------------------------------------------ pCSC
template <typename VT>
__device__ __forceinline__ void issue_col_tile(const ColLaunch& P, int4 d, unsigned char* st, uint64_t* bar,
                                               uint64_t pol) {
  using L = RowSmem<VT>;
  const int ncols = d.z & 0xffff, nnz = d.z >> 16;
  uint32_t vb = 0, cb = 0, ab = 0;
  int64_t v0 = 0, c0 = 0;
  if (nnz > 0) {
    v0 = (int64_t)d.y & ~(int64_t)(L::VPA - 1);
    int64_t v1 = ((int64_t)d.y + nnz + L::VPA - 1) & ~(int64_t)(L::VPA - 1);
    vb = (uint32_t)((v1 - v0) * (int64_t)sizeof(VT));
    c0 = (int64_t)d.y & ~(int64_t)3;
    int64_t c1 = ((int64_t)d.y + nnz + 3) & ~(int64_t)3;
    cb = (uint32_t)((c1 - c0) * 4);
  }
  int64_t a0 = (int64_t)d.x & ~(int64_t)3;
  int64_t a1 = ((int64_t)d.x + ncols + 1 + 3) & ~(int64_t)3;
  ab = (uint32_t)((a1 - a0) * 4);
  mbar_arrive_expect_tx(bar, vb + cb + ab);
  if (vb) tma_1d(st, (const VT*)P.val + v0, vb, bar, pol);
  if (cb) tma_1d(st + L::VAL_B, P.row + c0, cb, bar, pol);
  tma_1d(st + L::VAL_B + L::COL_B, P.cptr + a0, ab, bar, pol);
}

template <typename VT>
__global__ void __launch_bounds__(THREADS, 2) cols_kernel(const ColLaunch P) {
  using L = RowSmem<VT>;
  extern __shared__ __align__(128) unsigned char smem[];
  double* sx = reinterpret_cast<double*>(smem + L::BUF_OFF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  int4* sdesc = reinterpret_cast<int4*>(smem + L::DESC_OFF);
  const int tid = threadIdx.x;
  const VT* __restrict__ x = static_cast<const VT*>(P.x);
  double* __restrict__ py = P.py;

  uint64_t pol = 0;
  int4 next_desc = make_int4(0, 0, 0, -1);
  if (tid == 0) {
    pol = policy_evict_first();
    for (int s = 0; s < STAGES; s++) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < STAGES; s++) {
      int t = blockIdx.x + s * gridDim.x;
      if (t < P.ntiles) {
        int4 d = P.tiles[t];
        sdesc[s] = d;
        issue_col_tile<VT>(P, d, smem + s * L::STAGE_B, &bars[s], pol);
      }
    }
    int tn = blockIdx.x + STAGES * gridDim.x;
    if (tn < P.ntiles) next_desc = P.tiles[tn];
  }
  for (int i = 0;; i++) {
    const int t = blockIdx.x + i * gridDim.x;
    if (t >= P.ntiles) break;
    const int s = i % STAGES;
    mbar_wait(&bars[s], (uint32_t)((i / STAGES) & 1));
    const int4 dd = sdesc[s];
    unsigned char* st = smem + s * L::STAGE_B;
    const int ncols = dd.z & 0xffff, nnz = dd.z >> 16;
    const VT* sv = reinterpret_cast<const VT*>(st) + (dd.y & (L::VPA - 1));
    const int* sr = reinterpret_cast<const int*>(st + L::VAL_B) + (dd.y & 3);
    const int* sa = reinterpret_cast<const int*>(st + L::VAL_B + L::COL_B) + (dd.x & 3);
    for (int c = tid; c < ncols; c += THREADS) sx[c] = (double)ldg_ro(x + P.xbase + dd.x + c);
    __syncthreads();
    // merge path over (column ends clamped to the tile's nonzero range, nonzero indices)
    const int z0 = dd.y, z1 = dd.y + nnz;
    auto cend = [&](int c) { int e = sa[c + 1]; e = e < z0 ? z0 : (e > z1 ? z1 : e); return e - z0; };
    const int items = ncols + nnz;
    const int per = (items + THREADS - 1) / THREADS;
    const int d0 = min(tid * per, items), d1 = min(d0 + per, items);
    int lo = max(0, d0 - nnz), hi = min(d0, ncols);
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (cend(mid) <= d0 - mid - 1) lo = mid + 1; else hi = mid;
    }
    int xc = lo, yz = d0 - lo;
    for (int q = d0; q < d1; q++) {
      if (xc < ncols && yz < cend(xc)) {
        atomicAdd(py + sr[yz], (double)sv[yz] * sx[xc]);
        yz++;
      } else {
        xc++;
      }
    }
    __syncthreads();
    if (tid == 0) {
      int tn = t + STAGES * gridDim.x;
      if (tn < P.ntiles) {
        sdesc[s] = next_desc;
        fence_proxy_async();
        issue_col_tile<VT>(P, next_desc, st, &bars[s], pol);
        int tnn = tn + STAGES * gridDim.x;
        if (tnn < P.ntiles) next_desc = P.tiles[tnn];
      }
    }
  }
}

// --------------------------------------------------------- small kernels
template <typename VT>
__global__ void fixup_kernel(const FixupLaunch F) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= F.nsplit) return;
  double acc = 0.0;
  for (int k = F.sr_rec[2 * s]; k < F.sr_rec[2 * s + 1]; k++) acc = acc + F.rec[k];
  for (int h = F.sr_head[2 * s]; h < F.sr_head[2 * s + 1]; h++) {
    const int j = F.head_list[h];
    double hv = 0.0;
    if (j >= F.part_lo && j < F.part_hi) {
      const int jl = j - F.part_lo;
      for (int k = F.part_rec[2 * jl]; k < F.part_rec[2 * jl + 1]; k++) hv = hv + F.rec[k];
    } else {
      hv = F.head_all[j];
    }
    acc = acc + hv;
  }
  VT* y = static_cast<VT*>(F.y);
  const int64_t r = F.sr_row[s];
  double v = F.alpha * acc;
  if (F.beta != 0.0) v += F.beta * (double)y[r];
  y[r] = (VT)v;
}

__global__ void heads_kernel(const HeadLaunch H) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= H.nlocal) return;
  double hv = 0.0;
  for (int k = H.part_rec[2 * j]; k < H.part_rec[2 * j + 1]; k++) hv = hv + H.rec[k];
  H.head_local[j] = hv;
}

template <typename VT>
__global__ void scale_kernel(VT* y, int64_t n, double beta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (VT)(beta != 0.0 ? beta * (double)y[i] : 0.0);
}

template <typename VT>
__global__ void axpby_kernel(const double* __restrict__ py, VT* __restrict__ y, int64_t n, double alpha, double beta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = alpha * py[i];
    if (beta != 0.0) v += beta * (double)y[i];
    y[i] = (VT)v;
  }
}

__global__ void rebase_kernel(const int64_t* __restrict__ g, int32_t* __restrict__ l, int64_t n, int64_t lo,
                              int64_t hi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t v = g[i];
    v = v < lo ? lo : (v > hi ? hi : v);
    l[i] = (int32_t)(v - lo);
  }
}

int g_sms = 0;
int num_sms() {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

int elementwise_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms() * 8;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

template <typename K>
cudaError_t set_smem(K kernel, int bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

}  // namespace

int rows_grid(int dtype, int coo, int ntiles) {
  (void)dtype; (void)coo;
  int g = num_sms() * 2;
  return ntiles < g ? (ntiles < 1 ? 1 : ntiles) : g;
}
int cols_grid(int dtype, int ntiles) { return rows_grid(dtype, 0, ntiles); }

cudaError_t launch_rows(const RowLaunch& L, cudaStream_t s) {
  if (L.ntiles == 0) return cudaSuccess;
  cudaError_t e;
  if (L.dtype == 0) {
    int b = RowSmem<double>::TOTAL;
    if (L.coo) { if ((e = set_smem(rows_kernel<double, true>, b))) return e; rows_kernel<double, true><<<L.grid, THREADS + 32, b, s>>>(L); }
    else { if ((e = set_smem(rows_kernel<double, false>, b))) return e; rows_kernel<double, false><<<L.grid, THREADS + 32, b, s>>>(L); }
  } else {
    int b = RowSmem<float>::TOTAL;
    if (L.coo) { if ((e = set_smem(rows_kernel<float, true>, b))) return e; rows_kernel<float, true><<<L.grid, THREADS + 32, b, s>>>(L); }
    else { if ((e = set_smem(rows_kernel<float, false>, b))) return e; rows_kernel<float, false><<<L.grid, THREADS + 32, b, s>>>(L); }
  }
  return cudaGetLastError();
}

cudaError_t launch_cols(const ColLaunch& L, cudaStream_t s) {
  if (L.ntiles == 0) return cudaSuccess;
  cudaError_t e;
  if (L.dtype == 0) {
    int b = RowSmem<double>::TOTAL;
    if ((e = set_smem(cols_kernel<double>, b))) return e;
    cols_kernel<double><<<L.grid, THREADS, b, s>>>(L);
  } else {
    int b = RowSmem<float>::TOTAL;
    if ((e = set_smem(cols_kernel<float>, b))) return e;
    cols_kernel<float><<<L.grid, THREADS, b, s>>>(L);
  }
  return cudaGetLastError();
}

cudaError_t launch_fixup(const FixupLaunch& F, cudaStream_t s) {
  if (F.nsplit == 0) return cudaSuccess;
  int g = (F.nsplit + 127) / 128;
  if (F.dtype == 0) fixup_kernel<double><<<g, 128, 0, s>>>(F);
  else fixup_kernel<float><<<g, 128, 0, s>>>(F);
  return cudaGetLastError();
}

cudaError_t launch_heads(const HeadLaunch& H, cudaStream_t s) {
  if (H.nlocal == 0) return cudaSuccess;
  heads_kernel<<<(H.nlocal + 127) / 128, 128, 0, s>>>(H);
  return cudaGetLastError();
}

cudaError_t launch_scale(void* y, int64_t n, double beta, int dtype, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (dtype == 0) scale_kernel<double><<<elementwise_grid(n), 256, 0, s>>>((double*)y, n, beta);
  else scale_kernel<float><<<elementwise_grid(n), 256, 0, s>>>((float*)y, n, beta);
  return cudaGetLastError();
}

cudaError_t launch_axpby_py(const double* py, void* y, int64_t n, double alpha, double beta, int dtype,
                            cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (dtype == 0) axpby_kernel<double><<<elementwise_grid(n), 256, 0, s>>>(py, (double*)y, n, alpha, beta);
  else axpby_kernel<float><<<elementwise_grid(n), 256, 0, s>>>(py, (float*)y, n, alpha, beta);
  return cudaGetLastError();
}

cudaError_t launch_rebase(const int64_t* g, int32_t* l, int64_t n, int64_t lo, int64_t hi, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  rebase_kernel<<<elementwise_grid(n), 256, 0, s>>>(g, l, n, lo, hi);
  return cudaGetLastError();
}

}  // namespace msrep
