// kernels.cu -- sm_100a kernels of the msRep hot path (arXiv 2209.07552).
//
// SpMV is HBM-bound (0.17 flop/B in fp64, "memory bound ... main
// cost of SpMV comes from accessing the nonzero elements"), so no tensor cores:
// the design goal is to keep enough bytes in flight to saturate HBM3e.
//
//  rows_kernel  pCSR / pCOO per-GPU SpMV (Alg. 3 / Alg. 7 "Launch:
//               py[i]=<csrSpMVKernel>"): ONE persistent
//               launch per SpMV.  Every warp owns a one-slot ring of tile blobs
//               moved by 1-D TMA bulk copies (cp.async.bulk + mbarrier, L2
//               evict_first) and walks a static tile list built at partition
//               time (internal.h): SELL tiles (regular rows, lane = row), SEG
//               tiles (irregular rows, lane-chunked nonzeros with u8 row keys,
//               reduced in registers and joined by one deterministic warp
//               segmented scan) and slabs (pieces of split rows, whose
//               partial goes to a record).  No float atomics: bit-reproducible.
//  rows_mm_kernel  the same walk for a block of k vectors (SpMM).
//  fixup_kernel the beta-deferred merge of split rows (reading R6):
//               y_r = alpha*(tail records + head partials, part order) + beta*y_r.
//  csc_band_kernel  pCSC / column-sorted pCOO scatter (Alg. 5, P:418-423;
//               "switch the role of x and y"): one CTA per row band,
//               fp64 partial y in shared memory with warp-owned rows (plain
//               read-modify-writes, no atomics), stage blobs TMA-streamed by a
//               producer warp, the alpha/beta epilogue (or the py write for the
//               reduce-scatter) fused at band end.
//  cg_*         the vector kernels of msrep_cg.
#include <algorithm>
#include <climits>
#include <mutex>
#include <cstdint>

#include "internal.h"

namespace msrep {
namespace {

constexpr unsigned FULL = 0xffffffffu;

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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(bar)) : "memory");
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
// L2 policies: the matrix stream and y are touched once per SpMV (evict_first,
// .cs); x is re-gathered by every nonzero of its column (evict_last), so the
// y stream must not push it out of L2.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// x gathers (scalar).  NA selects the L1 policy per partition (RowLaunch / ColLaunch .xna, chosen
// by msrep_partition, host.cpp "x-gather L1 policy"): NA = L1::no_allocate, for gathers without
// reuse inside an SM (R-MAT, uniform random: 5-6 % faster, profiles/r1_xload_variants.txt); else
// the read-only path with L1 allocation, for gathers that neighbouring rows / warps re-hit
// (stencil pCOO, banded, block-diagonal, short-wide pCSC).
template <bool NA>
__device__ __forceinline__ double ldx(const double* p, uint64_t pol) {
  double v;
  if constexpr (NA) asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  else asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
template <bool NA>
__device__ __forceinline__ float ldx(const float* p, uint64_t pol) {
  float v;
  if constexpr (NA) asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  else asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}

// ---------------------------------------------------------------- layout
// Every warp owns an independent NS-stage ring of tile blobs in shared memory.
// Lane 0 issues ONE 1-D TMA bulk copy per tile (the blob is contiguous in HBM);
// the warp waits on the stage's mbarrier, computes, and refills the stage --
// no cross-warp synchronisation, so a slow warp never stalls another's loads.
template <typename VT>
struct RStage {
  static constexpr int N = tile_nnz((int)sizeof(VT));
  static constexpr int BYTES = N + N * (int)sizeof(VT) + N * 4;
};

template <int STAGE_B, int NS, int SCRATCH, int NW = WARPS>
struct WLayout {
  static constexpr int DESC_OFF = NS * STAGE_B;                          // int4 per stage
  static constexpr int SCR_OFF = DESC_OFF + NS * 16;                     // per-warp fp64 scratch
  static constexpr int WARP_B = (SCR_OFF + SCRATCH + 15) & ~15;
  static constexpr int BAR_OFF = NW * WARP_B;
  static constexpr int TOTAL = BAR_OFF + NW * NS * 8;
  static constexpr int HOT_OFF = (TOTAL + 15) & ~15;                     // CTA-wide hot x cache (sized per launch)
};

// nonzeros per lane in a full SEG tile / slab (+1 extra slot when ragged): 16 fp64, 32 fp32
template <typename VT>
__host__ __device__ constexpr int qmax() { return tile_nnz((int)sizeof(VT)) / 32; }


// Warp-level exclusive segmented scan of (key, value) pairs with keys
// non-decreasing by lane: op((ka,va),(kb,vb)) = (kb, ka==kb ? va+vb : vb).
// Deterministic (fixed shuffle tree).  Returns INT_MIN as the key of lane 0.
__device__ __forceinline__ void warp_seg_scan(int key, double val, int& pk, double& pv) {
  const int lane = threadIdx.x & 31;
  int ik = key;
  double iv = val;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int k2 = __shfl_up_sync(FULL, ik, off);
    double v2 = __shfl_up_sync(FULL, iv, off);
    if (lane >= off && k2 == ik) iv = v2 + iv;
  }
  int ek = __shfl_up_sync(FULL, ik, 1);
  double ev = __shfl_up_sync(FULL, iv, 1);
  pk = lane == 0 ? INT_MIN : ek;
  pv = lane == 0 ? 0.0 : ev;
}

__device__ __forceinline__ int tile_kind(int4 d) {
  return d.w >= 0 ? KIND_SLAB : (d.w == -2 ? KIND_SELL : (d.w == -3 ? KIND_SELLN : KIND_SEG));
}

__device__ __forceinline__ void issue_blob(const char* blob, int4 d, int kind, int vsize, unsigned char* st,
                                           uint64_t* bar, uint64_t pol) {
  const int bytes = blob_bytes(kind, d.z & 0xffff, d.z >> 16, vsize);
  mbar_arrive_expect_tx(bar, (uint32_t)bytes);
  tma_1d(st, blob + (int64_t)d.y * 16, (uint32_t)bytes, bar, pol);
}

// pCSR / pCOO tile kernel: ONE persistent launch per SpMV.  Every warp owns a
// one-slot TMA ring and walks tiles gw, gw+nw, ... of the rank's tile list
// (SELL tiles first, then SEG / slab tiles; internal.h).
//   SELL: lane = row of 32 consecutive regular rows; all W column indices are
//         read from the slot, then all W x gathers are in flight before the
//         first FMA; padding is masked by the row length.  The slot is refilled
//         after the tile.
//   SEG:  whole rows; the tile is copied from the slot into registers as soon
//         as it lands and the warp's next tile is issued into the slot right
//         away, so that TMA overlaps this tile's x gathers and reduction.  Lane
//         l reduces its contiguous chunk of nonzeros keyed by the uint8
//         tile-local row, rows crossing lanes are joined by one deterministic
//         warp segmented scan, y = alpha*s + beta*y is written coalesced.
//   slab: partial sum of a piece of one split row -> rec[w] (natural order,
//         fixed shuffle tree: bit-reproducible).
#ifndef MSREP_ROW_MINB_F32
#define MSREP_ROW_MINB_F32 2
#endif
#ifndef MSREP_ROW_MINB
#define MSREP_ROW_MINB 2
#endif
template <typename VT>
struct SStage {   // the larger of a full 32-bit-id SELL tile and a full narrow one
  static constexpr int V = (int)sizeof(VT);
  static constexpr int WIDE = SELL_R_MAX * 32 * 2 + SELL_W_MAX * SELL_ROWS * (V + 4);
  static constexpr int NARROW = 16 + SELL_R_MAX * 32 * 2 + selln_w_max(V) * SELL_ROWS * (V + 2);
  static constexpr int BYTES = WIDE > NARROW ? WIDE : NARROW;
};
template <typename VT, bool SELL, bool HOT = false>
using RowLayout = WLayout<(SELL && SStage<VT>::BYTES > RStage<VT>::BYTES) ? SStage<VT>::BYTES : RStage<VT>::BYTES, 1,
                          MAX_TILE_ROWS * 8, HOT ? hot_warps((int)sizeof(VT)) : WARPS>;

// x gather of a SEG / slab column id: tagged ids (bit 31, internal.h HOT_TAG) read the CTA's
// shared-memory copy of the rank's hottest x entries, the others go through L2.  Branch-free: one
// predicated LDS and one predicated LDG into the same register, so all of a lane's gathers stay
// in flight together (a branch per gather serialises the two paths, 1.3 -> 2.2 ms on R-MAT).
// hot-x address of slot s: the slots are spread over the CL CTAs of the cluster, hpc per CTA; hb[r]
// is CTA r's cache base in the shared::cluster window (CL == 1: the CTA's own shared memory)
struct HotRef { uint32_t hb0, hb1, hpc; };
// x[off] from a base pointer with the address formed inside the asm (keeps ptxas from holding a
// 64-bit address per in-flight gather: the narrow SELL tiles keep up to 64 gathers in flight)
__device__ __forceinline__ double ldg_off(const double* xb, uint32_t off) {
  double v;
  asm("{\n\t.reg .u64 ga;\n\tmad.wide.u32 ga, %1, 8, %2;\n\tld.global.nc.f64 %0, [ga];\n\t}" : "=d"(v) : "r"(off), "l"(xb));
  return v;
}
__device__ __forceinline__ float ldg_off(const float* xb, uint32_t off) {
  float v;
  asm("{\n\t.reg .u64 ga;\n\tmad.wide.u32 ga, %1, 4, %2;\n\tld.global.nc.f32 %0, [ga];\n\t}" : "=f"(v) : "r"(off), "l"(xb));
  return v;
}

// The asm of one hot-aware gather, predicated on `on` (0: no load, the result is 0) so that a
// tile's gathers are straight-line code without a branch each.  CL == 2: the slots are split over
// the CTA pair (slot s lives in CTA s / hpc), read through the shared::cluster window.  CL == 1:
// the CTA's own copy, plain LDS; the slot address c * V + base in 32 bits drops the tag bit.
#define MSREP_LDX_PAIR(T, R, SZ, Z, COLD)                                                                \
  asm("{\n\t.reg .pred p, q, g, o;\n\t.reg .u32 ci, sa, hb;\n\t.reg .u64 ga;\n\t"                          \
      "setp.ne.u32 o, %7, 0;\n\tsetp.lt.and.s32 p, %1, 0, o;\n\tsetp.ge.and.s32 g, %1, 0, o;\n\t"         \
      "and.b32 ci, %1, 0x7fffffff;\n\tsetp.ge.u32 q, ci, %4;\n\t"                                          \
      "selp.b32 hb, %3, %2, q;\n\t@q sub.u32 ci, ci, %4;\n\tmad.lo.u32 sa, ci, " SZ ", hb;\n\t"            \
      "mad.wide.u32 ga, %1, " SZ ", %5;\n\tmov." T " %0, " Z ";\n\t@p ld.shared::cluster." T " %0, [sa];\n\t" \
      "@g ld.global.nc" COLD ".L2::cache_hint." T " %0, [ga], %6;\n\t}"                                     \
      : "=" R(v) : "r"(c), "r"(h.hb0), "r"(h.hb1), "r"(h.hpc), "l"(x), "l"(pol), "r"(on))
#define MSREP_LDX_OWN(T, R, SZ, Z, COLD)                                                                 \
  asm("{\n\t.reg .pred p, g, o;\n\t.reg .u32 sa;\n\t.reg .u64 ga;\n\t"                                     \
      "setp.ne.u32 o, %5, 0;\n\tsetp.lt.and.s32 p, %1, 0, o;\n\tsetp.ge.and.s32 g, %1, 0, o;\n\t"         \
      "mad.lo.u32 sa, %1, " SZ ", %2;\n\tmad.wide.u32 ga, %1, " SZ ", %3;\n\tmov." T " %0, " Z ";\n\t"     \
      "@p ld.shared." T " %0, [sa];\n\t@g ld.global.nc" COLD ".L2::cache_hint." T " %0, [ga], %4;\n\t}"   \
      : "=" R(v) : "r"(c), "r"(h.hb0), "l"(x), "l"(pol), "r"(on))
#define MSREP_LDX_COLD(T, R, SZ, Z, COLD)                                                                \
  asm("{\n\t.reg .pred o;\n\t.reg .u64 ga;\n\tsetp.ne.u32 o, %4, 0;\n\tmad.wide.u32 ga, %1, " SZ ", %2;\n\t" \
      "mov." T " %0, " Z ";\n\t@o ld.global.nc" COLD ".L2::cache_hint." T " %0, [ga], %3;\n\t}"           \
      : "=" R(v) : "r"(c), "l"(x), "l"(pol), "r"(on))
#define MSREP_Z64 "0d0000000000000000"
#define MSREP_Z32 "0f00000000"
template <bool NA, int CL>
__device__ __forceinline__ double ldx_sel(const double* x, const HotRef& h, uint32_t c, uint64_t pol, uint32_t on) {
  double v;
  if constexpr (CL == 2) {
    if constexpr (NA) MSREP_LDX_PAIR("f64", "d", "8", MSREP_Z64, ".L1::no_allocate");
    else MSREP_LDX_PAIR("f64", "d", "8", MSREP_Z64, "");
  } else {
    if constexpr (NA) MSREP_LDX_OWN("f64", "d", "8", MSREP_Z64, ".L1::no_allocate");
    else MSREP_LDX_OWN("f64", "d", "8", MSREP_Z64, "");
  }
  return v;
}
template <bool NA, int CL>
__device__ __forceinline__ float ldx_sel(const float* x, const HotRef& h, uint32_t c, uint64_t pol, uint32_t on) {
  float v;
  if constexpr (CL == 2) {
    if constexpr (NA) MSREP_LDX_PAIR("f32", "f", "4", MSREP_Z32, ".L1::no_allocate");
    else MSREP_LDX_PAIR("f32", "f", "4", MSREP_Z32, "");
  } else {
    if constexpr (NA) MSREP_LDX_OWN("f32", "f", "4", MSREP_Z32, ".L1::no_allocate");
    else MSREP_LDX_OWN("f32", "f", "4", MSREP_Z32, "");
  }
  return v;
}
// cold-only gather (no hot cache), predicated like ldx_sel
template <bool NA>
__device__ __forceinline__ double ldx_on(const double* x, uint32_t c, uint64_t pol, uint32_t on) {
  double v;
  if constexpr (NA) MSREP_LDX_COLD("f64", "d", "8", MSREP_Z64, ".L1::no_allocate");
  else MSREP_LDX_COLD("f64", "d", "8", MSREP_Z64, "");
  return v;
}
template <bool NA>
__device__ __forceinline__ float ldx_on(const float* x, uint32_t c, uint64_t pol, uint32_t on) {
  float v;
  if constexpr (NA) MSREP_LDX_COLD("f32", "f", "4", MSREP_Z32, ".L1::no_allocate");
  else MSREP_LDX_COLD("f32", "f", "4", MSREP_Z32, "");
  return v;
}
#undef MSREP_LDX_PAIR
#undef MSREP_LDX_OWN
#undef MSREP_LDX_COLD
#undef MSREP_Z64
#undef MSREP_Z32
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Hot-cache kernels branch around a tile position's gather (the branch is warp-uniform except at
// the ragged extra position, and the slot / global pair stays 5 instructions); the cold-only
// kernels predicate it instead (R-MAT fp32: 1.135 -> 1.038 ms; with the hot cache the predicated
// form was the slower one, 1.085 -> 1.118 ms -- profiles/r2_kernel_ab.txt)
template <bool HOT, bool NA, int CL, typename VT>
__device__ __forceinline__ VT ldx_hot(const VT* x, const HotRef& hbase, uint32_t c, uint64_t pol, bool on) {
  if constexpr (HOT) return on ? ldx_sel<NA, CL>(x, hbase, c, pol, 1u) : VT(0);
  else return ldx_on<NA>(x, c, pol, on ? 1u : 0u);
}

// One SELL tile with R rows per lane (internal.h): all R*W x gathers are in flight before the
// first FMA; padding is masked by the row length, so results equal the plain row sums.  NARROW:
// the column ids are 16-bit offsets from the tile's base (KIND_SELLN), up to selln_w_max entries
// per lane, read from the slot just before each gather.
template <typename VT, int R, bool MIRROR, bool NARROW, class Refill>
__device__ __forceinline__ void sell_tile(const RowLaunch& P, const int4 d, const unsigned char* st, const int lane,
                                          const VT* __restrict__ x, VT* __restrict__ y, double alpha, double beta,
                                          Refill&& refill) {
  constexpr int V = (int)sizeof(VT);
  constexpr int U = NARROW ? selln_w_max(V) : SELL_W_MAX;   // R*W <= U register slots per lane
  const int nrows = d.z & 0xffff, W = d.z >> 16;
  const unsigned char* p = st + (NARROW ? 16 : 0);
  const uint16_t* lens = reinterpret_cast<const uint16_t*>(p);
  const VT* sv = reinterpret_cast<const VT*>(p + align16(R * 32 * 2));
  const int RW = R * W;
  int mylen[R];
  double yv[R];
#pragma unroll
  for (int k = 0; k < R; k++) {
    const int row = k * 32 + lane;
    mylen[k] = lens[k * 32 + lane];
    yv[k] = (beta != 0.0 && row < nrows) ? (double)y[P.ybase + d.x + row] : 0.0;
  }
  VT xs[U];
  double acc[R];
#pragma unroll
  for (int k = 0; k < R; k++) acc[k] = 0.0;
  if constexpr (NARROW) {
    const uint16_t* so = reinterpret_cast<const uint16_t*>(p + align16(R * 32 * 2) + W * R * 32 * V);
    const VT* xb = x + *reinterpret_cast<const uint32_t*>(st);
#pragma unroll
    for (int u = 0; u < U; u++) xs[u] = u < RW ? ldg_off(xb, so[u * 32 + lane]) : VT(0);
  } else {
    const uint32_t* sc = reinterpret_cast<const uint32_t*>(p + align16(R * 32 * 2) + W * R * 32 * V);
    uint32_t c[U];
#pragma unroll
    for (int u = 0; u < U; u++) c[u] = u < RW ? sc[u * 32 + lane] : 0u;   // no loop-carried state
#pragma unroll
    for (int u = 0; u < U; u++) xs[u] = u < RW ? ldg_ro(x + c[u]) : VT(0);
  }
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int k = u % R, t = u / R;           // compile-time after unrolling
    if (u < RW && t < mylen[k]) acc[k] = fma((double)sv[u * 32 + lane], (double)xs[u], acc[k]);
  }
#pragma unroll
  for (int k = 0; k < R; k++) {
    const int row = k * 32 + lane;
    if (row < nrows) {
      double o = alpha * acc[k];
      if (beta != 0.0) o += beta * yv[k];
      const int64_t yi = P.ybase + d.x + row;
      y[yi] = (VT)o;
      if constexpr (MIRROR)
        for (int mi = 0; mi < P.nmirror; mi++) static_cast<VT*>(P.mirror[mi])[yi] = (VT)o;   // fused allgather
    }
  }
  __syncwarp();   // the tile was read in place: refill the slot only now
  refill();
}

template <typename VT, bool SELL, bool MIRROR, bool NA, bool HOT, int CL>
__global__ void __launch_bounds__(HOT ? hot_warps((int)sizeof(VT)) * 32 : WARPS * 32,
                                  HOT ? 1 : (sizeof(VT) == 4 ? MSREP_ROW_MINB_F32 : MSREP_ROW_MINB))
    rows_kernel(const RowLaunch P) {
  using Lay = RowLayout<VT, SELL, HOT>;
  constexpr int NW = HOT ? hot_warps((int)sizeof(VT)) : WARPS;
  constexpr int QMAX = qmax<VT>();
  constexpr int V = (int)sizeof(VT);
  constexpr int YR = MAX_TILE_ROWS / 32;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* st = smem + warp * Lay::WARP_B;
  int4* sdesc = reinterpret_cast<int4*>(st + Lay::DESC_OFF);
  double* rsum = reinterpret_cast<double*>(st + Lay::SCR_OFF);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Lay::BAR_OFF) + warp;
  const int gw = blockIdx.x * NW + warp, nw = gridDim.x * NW;

  const VT* __restrict__ x = static_cast<const VT*>(P.x);
  VT* __restrict__ y = static_cast<VT*>(P.y);
  const double alpha = P.alpha, beta = P.beta;
  const uint64_t xpol = policy_evict_last();
  VT* hx = reinterpret_cast<VT*>(smem + Lay::HOT_OFF);
  // CL == 2: the hot slots are split over the CTA pair of the cluster (slots [r*hpc, (r+1)*hpc) in
  // CTA r), read through distributed shared memory -- twice the hot entries per SM of L1 given up
  HotRef hbase{saddr(hx), saddr(hx), 0x7fffffffu};
  int hlo = 0, hhi = P.nhot;
  if constexpr (HOT && CL == 2) {
    const uint32_t hpc = (uint32_t)((P.nhot + 1) / 2), me = cluster_ctarank();
    hbase = HotRef{mapa_shared(saddr(hx), 0), mapa_shared(saddr(hx), 1), hpc};
    hlo = (int)(me * hpc);
    hhi = min(P.nhot, (int)((me + 1) * hpc));
  }

  uint64_t pol = 0;
  int4 dn = make_int4(0, 0, 0, -1);
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    pol = policy_evict_first();
    if (gw < P.ntiles) {
      const int4 d = P.tiles[gw];
      *sdesc = d;
      issue_blob(P.blob, d, tile_kind(d), V, st, bar, pol);
    }
    if (gw + nw < P.ntiles) dn = P.tiles[gw + nw];
  }
  if constexpr (HOT) {   // the CTA's copy of (its share of) the hot x entries, gathered while the first tiles land
    constexpr int U = 8, T = NW * 32;
    for (int k0 = hlo; k0 < hhi; k0 += U * T) {
      int cs[U];
      VT xs[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int k = k0 + u * T + (int)threadIdx.x;
        cs[u] = k < hhi ? __ldg(P.hot + k) : 0;
      }
#pragma unroll
      for (int u = 0; u < U; u++) xs[u] = __ldg(x + cs[u]);
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int k = k0 + u * T + (int)threadIdx.x;
        if (k < hhi) hx[k - hlo] = xs[u];
      }
    }
    if constexpr (CL == 2) cluster_sync();   // both halves filled before any remote read
    else __syncthreads();
  }
  __syncwarp();

  for (int i = 0;; i++) {
    const int t = gw + i * nw;
    if (t >= P.ntiles) break;
    mbar_wait(bar, (uint32_t)(i & 1));
    const int4 d = *sdesc;
    auto refill = [&]() {
      if (lane == 0) {
        const int tn = t + nw;
        if (tn < P.ntiles) {
          *sdesc = dn;
          issue_blob(P.blob, dn, tile_kind(dn), V, st, bar, pol);
          if (tn + nw < P.ntiles) dn = P.tiles[tn + nw];
        }
      }
    };
    if (SELL && (d.w == -2 || d.w == -3)) {
      // ---- SELL tile (read in place; the slot is refilled after the tile)
      const int R = sell_r(d.z & 0xffff);
      if (d.w == -3) {
        if (R == 1) sell_tile<VT, 1, MIRROR, true>(P, d, st, lane, x, y, alpha, beta, refill);
        else if (R == 2) sell_tile<VT, 2, MIRROR, true>(P, d, st, lane, x, y, alpha, beta, refill);
        else sell_tile<VT, 4, MIRROR, true>(P, d, st, lane, x, y, alpha, beta, refill);
      } else {
        if (R == 1) sell_tile<VT, 1, MIRROR, false>(P, d, st, lane, x, y, alpha, beta, refill);
        else if (R == 2) sell_tile<VT, 2, MIRROR, false>(P, d, st, lane, x, y, alpha, beta, refill);
        else sell_tile<VT, 4, MIRROR, false>(P, d, st, lane, x, y, alpha, beta, refill);
      }
      continue;
    }
    // fp32: the SELL instantiation walks SELL tiles only (the host always launches SEG / slab tiles
    // on their own: a SEG path beside the 64-entry narrow tiles spills, 0.0674 vs 0.0770 ms on the
    // fp32 stencil); fp64: a small share of SEG tiles rides along (no second launch)
    if constexpr (SELL && sizeof(VT) == 4) {
      __trap();
    } else {
    const int nrows = d.z & 0xffff, nnz = d.z >> 16;
    const bool slab = d.w >= 0;
    // ---- stage -> registers (conflict-free 32-lane vectors), then refill the slot
    const int q = slab ? 0 : nnz >> 5, r = nnz & 31;
    const bool extra = !slab && lane < r;
    uint32_t c[QMAX + 1];
    VT v[QMAX + 1];
    uint32_t kp[(QMAX + 4) / 4];   // SEG keys, 4 per register
#pragma unroll
    for (int u = 0; u < (QMAX + 4) / 4; u++) kp[u] = 0u;
    if (slab) {
      const VT* sv = reinterpret_cast<const VT*>(st);
      const uint32_t* sc = reinterpret_cast<const uint32_t*>(st + align16(nnz * V));
#pragma unroll
      for (int u = 0; u < QMAX; u++) {
        const bool on = lane + 32 * u < nnz;
        c[u] = on ? sc[lane + 32 * u] : 0u;   // range-checked at partition
        v[u] = on ? sv[lane + 32 * u] : VT(0);
      }
      c[QMAX] = 0u;
      v[QMAX] = VT(0);
    } else {
      const uint32_t* skw = reinterpret_cast<const uint32_t*>(st) + lane;   // keys, 4 per word
      const VT* sv = reinterpret_cast<const VT*>(st + seg_key_bytes(nnz));
      const uint32_t* sc = reinterpret_cast<const uint32_t*>(st + seg_key_bytes(nnz) + align16(nnz * V));
      const int npos = q + (extra ? 1 : 0);
      static_assert(QMAX % 4 == 0, "the extra key has register word QMAX / 4 to itself");
#pragma unroll
      for (int u = 0; u < QMAX / 4; u++) kp[u] = u * 4 < npos ? skw[u * 32] : 0u;
      if (extra)   // the extra position q moves to register position QMAX (one byte read)
        kp[QMAX / 4] = (uint32_t)st[(q >> 2) * 128 + lane * 4 + (q & 3)] << (8 * (QMAX & 3));
#pragma unroll
      for (int j = 0; j <= QMAX; j++) {
        const bool on = j < QMAX ? j < q : extra;
        const int sl = (j < QMAX ? j : q) * 32 + lane;
        c[j] = on ? sc[sl] : 0u;   // range-checked at partition; padding masked
        v[j] = on ? sv[sl] : VT(0);
      }
    }
    fence_proxy_async();   // order this lane's generic-proxy reads of the slot before the TMA refill
    __syncwarp();          // every lane holds its tile: the slot may be refilled
    refill();
    // ---- x gathers: all in flight before the first use
    VT xv[QMAX + 1];
    if (slab) {
#pragma unroll
      for (int u = 0; u < QMAX; u++) xv[u] = ldx_hot<HOT, NA, CL>(x, hbase, c[u], xpol, lane + 32 * u < nnz);
      double acc = 0.0;
#pragma unroll
      for (int u = 0; u < QMAX; u++) acc = fma((double)v[u], (double)xv[u], acc);   // padding: 0 * 0
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(FULL, acc, off);
      if (lane == 0) P.rec[d.w] = acc;
      continue;
    }
    const int64_t yrow0 = P.ybase + d.x;
    double yin[YR];
#pragma unroll
    for (int u = 0; u < YR; u++) {
      const int rr = lane + 32 * u;
      yin[u] = (beta != 0.0 && rr < nrows) ? (double)__ldcs(y + yrow0 + rr) : 0.0;
    }
#pragma unroll
    for (int j = 0; j <= QMAX; j++) {
      const bool on = j < QMAX ? j < q : extra;
      xv[j] = ldx_hot<HOT, NA, CL>(x, hbase, c[j], xpol, on);
    }
    if (d.w != KIND_W_SEG_DENSE) {   // rows without entries must read 0 (a dense tile writes every row)
      for (int rr = lane; rr < nrows; rr += 32) rsum[rr] = 0.0;
      __syncwarp();
    }
    // ---- walk the lane's chunk: complete rows inside it go straight to rsum
    const int len = q + (extra ? 1 : 0);
    const int key0 = (int)(q > 0 ? (kp[0] & 0xffu) : (kp[QMAX >> 2] >> (8 * (QMAX & 3))) & 0xffu);
    int cur = len > 0 ? key0 : INT_MAX;
    int first = cur, nseg = len > 0 ? 1 : 0;
    double acc = 0.0, firstv = 0.0;
#pragma unroll
    for (int j = 0; j <= QMAX; j++) {
      const bool on = j < QMAX ? j < q : extra;
      if (on) {
        const int k = (int)((kp[j >> 2] >> (8 * (j & 3))) & 0xffu);
        if (k != cur) {
          if (nseg == 1) firstv = acc; else rsum[cur] = acc;
          nseg++;
          cur = k;
          acc = 0.0;
        }
        acc = fma((double)v[j], (double)xv[j], acc);
      }
    }
    // ---- join rows that cross lanes: inclusive run of preceding lanes ending in the same row
    int pk;
    double pv;
    warp_seg_scan(cur, acc, pk, pv);
    const int next_first = __shfl_down_sync(FULL, key0, 1);
    const bool next_has = lane < 31 && (q > 0 || lane + 1 < r);
    if (nseg >= 2) rsum[first] = (pk == first) ? firstv + pv : firstv;
    if (nseg >= 1 && !(next_has && next_first == cur)) rsum[cur] = (pk == cur) ? pv + acc : acc;
    __syncwarp();
    // ---- coalesced epilogue: alpha and beta applied exactly once per row
#pragma unroll
    for (int u = 0; u < YR; u++) {
      const int rr = lane + 32 * u;
      if (rr < nrows) {
        double o = alpha * rsum[rr];
        if (beta != 0.0) o += beta * yin[u];
        __stcs(y + yrow0 + rr, (VT)o);
        if constexpr (MIRROR)
          for (int mi = 0; mi < P.nmirror; mi++) static_cast<VT*>(P.mirror[mi])[yrow0 + rr] = (VT)o;   // fused allgather
      }
    }
    __syncwarp();   // rsum is free
    }
  }
  if constexpr (HOT && CL == 2) cluster_sync();   // the partner CTA may still read this CTA's hot half
}

// ------------------------------------------------------------------ SpMM
// Y <- alpha*A*X + beta*Y for a block of K vectors (X [n x K], Y [m x K], row-major; the
// "easily extended" multi-right-hand-side kernel).  Same tile list, blobs and
// per-warp one-slot TMA ring as rows_kernel: the matrix is streamed once for all K vectors.
// Each nonzero gathers one K-wide row of X (vector loads, L2 evict_last); lanes batch BG
// gathers at a time so K-wide accumulators fit the register budget.
template <typename VT, int K>
__device__ __forceinline__ void ldx_row(const VT* p, VT (&o)[K], uint64_t pol) {
  if constexpr (sizeof(VT) == 8) {
#pragma unroll
    for (int i = 0; i < K; i += 2)
      asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(o[i]), "=d"(o[i + 1]) : "l"(p + i), "l"(pol));
  } else if constexpr (K == 2) {
    asm("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(o[0]), "=f"(o[1]) : "l"(p), "l"(pol));
  } else {
#pragma unroll
    for (int i = 0; i < K; i += 4)
      asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
          : "=f"(o[i]), "=f"(o[i + 1]), "=f"(o[i + 2]), "=f"(o[i + 3]) : "l"(p + i), "l"(pol));
  }
}

// Y row <- alpha * acc + beta * Y row (beta == 0: Y not read)
template <typename VT, int K>
__device__ __forceinline__ void mm_write_row(VT* yrow, const double (&acc)[K], double alpha, double beta) {
#pragma unroll
  for (int j = 0; j < K; j++) {
    double o = alpha * acc[j];
    if (beta != 0.0) o += beta * (double)yrow[j];
    yrow[j] = (VT)o;
  }
}

// a SEG / slab column id of a hot-x partition (tag bit set) -> the column (SpMM gathers K-wide rows
// of X, which the SpMV's shared-memory x cache does not hold); the slot -> column table is copied
// into shared memory at kernel start (a dependent global load per hot gather was 1.5x slower)
__device__ __forceinline__ uint32_t untag(const int* hot_s, uint32_t c) {
  return (c & HOT_TAG) ? (uint32_t)hot_s[c & ~HOT_TAG] : c;
}

template <typename VT, int K, bool SELL>
__global__ void __launch_bounds__(WARPS * 32, MSREP_ROW_MINB) rows_mm_kernel(const RowLaunch P) {
  using Lay = RowLayout<VT, SELL>;
  constexpr int QMAX = qmax<VT>();
  constexpr int V = (int)sizeof(VT);
  constexpr int BG = K >= 8 ? 1 : (K >= 4 ? 2 : 4);   // gathers in flight per lane per batch (SEG / slab)
  constexpr int BS = 32 / K;                          // ... for SELL tiles (no chunk held in registers)
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* st = smem + warp * Lay::WARP_B;
  int4* sdesc = reinterpret_cast<int4*>(st + Lay::DESC_OFF);
  unsigned* written = reinterpret_cast<unsigned*>(st + Lay::SCR_OFF);   // MAX_TILE_ROWS-bit map
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Lay::BAR_OFF) + warp;
  const int gw = blockIdx.x * WARPS + warp, nw = gridDim.x * WARPS;
  const VT* __restrict__ x = static_cast<const VT*>(P.x);
  VT* __restrict__ y = static_cast<VT*>(P.y);
  const double alpha = P.alpha, beta = P.beta;
  const uint32_t xmax = P.xmax;
  const uint64_t xpol = policy_evict_last();
  int* hot_s = reinterpret_cast<int*>(smem + Lay::HOT_OFF);   // P.nhot entries (launch sizes the buffer)
  for (int k = threadIdx.x; k < P.nhot; k += WARPS * 32) hot_s[k] = __ldg(P.hot + k);
  __syncthreads();

  uint64_t pol = 0;
  int4 dn = make_int4(0, 0, 0, -1);
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    pol = policy_evict_first();
    if (gw < P.ntiles) {
      const int4 d = P.tiles[gw];
      *sdesc = d;
      issue_blob(P.blob, d, tile_kind(d), V, st, bar, pol);
    }
    if (gw + nw < P.ntiles) dn = P.tiles[gw + nw];
  }
  __syncwarp();

  for (int i = 0;; i++) {
    const int t = gw + i * nw;
    if (t >= P.ntiles) break;
    mbar_wait(bar, (uint32_t)(i & 1));
    const int4 d = *sdesc;
    auto refill = [&]() {
      if (lane == 0) {
        const int tn = t + nw;
        if (tn < P.ntiles) {
          *sdesc = dn;
          issue_blob(P.blob, dn, tile_kind(dn), V, st, bar, pol);
          if (tn + nw < P.ntiles) dn = P.tiles[tn + nw];
        }
      }
    };
    if (SELL && (d.w == -2 || d.w == -3)) {
      // ---- SELL tile: lane l walks its R rows; element t of row k at (t*R + k)*32 + l
      const int nrows = d.z & 0xffff, W = d.z >> 16, R = sell_r(nrows);
      const bool narrow = d.w == -3;   // 16-bit column offsets from the tile's base (KIND_SELLN)
      const unsigned char* p0 = st + (narrow ? 16 : 0);
      const uint16_t* lens = reinterpret_cast<const uint16_t*>(p0);
      const VT* sv = reinterpret_cast<const VT*>(p0 + align16(R * 32 * 2));
      const uint32_t* sc = reinterpret_cast<const uint32_t*>(p0 + align16(R * 32 * 2) + W * R * 32 * V);
      const uint16_t* so = reinterpret_cast<const uint16_t*>(sc);
      const uint32_t nbase = narrow ? *reinterpret_cast<const uint32_t*>(st) : 0u;
      for (int k = 0; k < R; k++) {
        const int row = k * 32 + lane;
        const int len = row < nrows ? lens[k * 32 + lane] : 0;
        double acc[K];
#pragma unroll
        for (int j = 0; j < K; j++) acc[j] = 0.0;
        for (int e0 = 0; e0 < W; e0 += BS) {
          VT xr[BS][K];
          VT vv[BS];
#pragma unroll
          for (int b = 0; b < BS; b++) {
            const int e = e0 + b;
            const bool on = e < len;
            const int sl = (e * R + k) * 32 + lane;
            const uint32_t cc = on ? min(narrow ? nbase + so[sl] : sc[sl], xmax) : 0u;
            vv[b] = on ? sv[(e * R + k) * 32 + lane] : VT(0);
            if (on) ldx_row<VT, K>(x + (int64_t)cc * K, xr[b], xpol);
            else {
#pragma unroll
              for (int j = 0; j < K; j++) xr[b][j] = VT(0);
            }
          }
#pragma unroll
          for (int b = 0; b < BS; b++)
#pragma unroll
            for (int j = 0; j < K; j++) acc[j] = fma((double)vv[b], (double)xr[b][j], acc[j]);
        }
        if (row < nrows) mm_write_row<VT, K>(y + (P.ybase + d.x + row) * K, acc, alpha, beta);
      }
      __syncwarp();
      refill();
      continue;
    }
    const int nrows = d.z & 0xffff, nnz = d.z >> 16;
    const bool slab = d.w >= 0;
    const int q = slab ? 0 : nnz >> 5, r = nnz & 31;
    const bool extra = !slab && lane < r;
    uint32_t c[QMAX + 1];
    VT v[QMAX + 1];
    uint32_t kp[(QMAX + 4) / 4];
#pragma unroll
    for (int u = 0; u < (QMAX + 4) / 4; u++) kp[u] = 0u;
    if (slab) {
      const VT* sv = reinterpret_cast<const VT*>(st);
      const uint32_t* sc = reinterpret_cast<const uint32_t*>(st + align16(nnz * V));
#pragma unroll
      for (int u = 0; u < QMAX; u++) {
        const bool on = lane + 32 * u < nnz;
        c[u] = on ? sc[lane + 32 * u] : 0u;   // range-checked at partition
        v[u] = on ? sv[lane + 32 * u] : VT(0);
      }
      c[QMAX] = 0u;
      v[QMAX] = VT(0);
    } else {
      const uint32_t* skw = reinterpret_cast<const uint32_t*>(st) + lane;   // keys, 4 per word
      const VT* sv = reinterpret_cast<const VT*>(st + seg_key_bytes(nnz));
      const uint32_t* sc = reinterpret_cast<const uint32_t*>(st + seg_key_bytes(nnz) + align16(nnz * V));
      const int npos = q + (extra ? 1 : 0);
      static_assert(QMAX % 4 == 0, "the extra key has register word QMAX / 4 to itself");
#pragma unroll
      for (int u = 0; u < QMAX / 4; u++) kp[u] = u * 4 < npos ? skw[u * 32] : 0u;
      if (extra)   // the extra position q moves to register position QMAX (one byte read)
        kp[QMAX / 4] = (uint32_t)st[(q >> 2) * 128 + lane * 4 + (q & 3)] << (8 * (QMAX & 3));
#pragma unroll
      for (int j = 0; j <= QMAX; j++) {
        const bool on = j < QMAX ? j < q : extra;
        const int sl = (j < QMAX ? j : q) * 32 + lane;
        c[j] = on ? sc[sl] : 0u;   // range-checked at partition; padding masked
        v[j] = on ? sv[sl] : VT(0);
      }
    }
    fence_proxy_async();   // order this lane's generic-proxy reads of the slot before the TMA refill
    __syncwarp();
    refill();
    if (slab) {
      // ---- slab: K partial sums of one split row -> rec[w*K + j] (natural order, fixed tree)
      double acc[K];
#pragma unroll
      for (int j = 0; j < K; j++) acc[j] = 0.0;
#pragma unroll
      for (int u0 = 0; u0 < QMAX; u0 += BG) {
        VT xr[BG][K];
#pragma unroll
        for (int b = 0; b < BG; b++) {
          if (lane + 32 * (u0 + b) < nnz) ldx_row<VT, K>(x + (int64_t)untag(hot_s, c[u0 + b]) * K, xr[b], xpol);
          else {
#pragma unroll
            for (int j = 0; j < K; j++) xr[b][j] = VT(0);
          }
        }
#pragma unroll
        for (int b = 0; b < BG; b++)
#pragma unroll
          for (int j = 0; j < K; j++) acc[j] = fma((double)v[u0 + b], (double)xr[b][j], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < K; j++) {
        double a = acc[j];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(FULL, a, off);
        if (lane == 0) P.rec[(int64_t)d.w * K + j] = a;
      }
      continue;
    }
    // ---- SEG tile
    const int64_t yrow0 = P.ybase + d.x;
    if (lane < MAX_TILE_ROWS / 32) written[lane] = 0u;
    __syncwarp();
    auto put_row = [&](int row, const double (&a)[K]) {
      mm_write_row<VT, K>(y + (yrow0 + row) * K, a, alpha, beta);
      atomicOr(&written[row >> 5], 1u << (row & 31));
    };
    const int len = q + (extra ? 1 : 0);
    const int key0 = (int)(q > 0 ? (kp[0] & 0xffu) : (kp[QMAX >> 2] >> (8 * (QMAX & 3))) & 0xffu);
    int cur = len > 0 ? key0 : INT_MAX;
    int first = cur, nseg = len > 0 ? 1 : 0;
    double acc[K], firstv[K];
#pragma unroll
    for (int j = 0; j < K; j++) { acc[j] = 0.0; firstv[j] = 0.0; }
#pragma unroll
    for (int j0 = 0; j0 <= QMAX; j0 += BG) {
      VT xr[BG][K];
#pragma unroll
      for (int b = 0; b < BG; b++) {
        const int j = j0 + b;
        const bool on = j <= QMAX && (j < QMAX ? j < q : extra);
        if (on) ldx_row<VT, K>(x + (int64_t)untag(hot_s, c[j <= QMAX ? j : QMAX]) * K, xr[b], xpol);
        else {
#pragma unroll
          for (int jj = 0; jj < K; jj++) xr[b][jj] = VT(0);
        }
      }
#pragma unroll
      for (int b = 0; b < BG; b++) {
        const int j = j0 + b;
        const bool on = j <= QMAX && (j < QMAX ? j < q : extra);
        if (on) {
          const int jc = j <= QMAX ? j : QMAX;
          const int kk = (int)((kp[jc >> 2] >> (8 * (jc & 3))) & 0xffu);
          if (kk != cur) {
            if (nseg == 1) {
#pragma unroll
              for (int jj = 0; jj < K; jj++) firstv[jj] = acc[jj];
            } else {
              put_row(cur, acc);
            }
            nseg++;
            cur = kk;
#pragma unroll
            for (int jj = 0; jj < K; jj++) acc[jj] = 0.0;
          }
#pragma unroll
          for (int jj = 0; jj < K; jj++) acc[jj] = fma((double)v[jc], (double)xr[b][jj], acc[jj]);
        }
      }
    }
    // rows crossing lanes: one deterministic segmented scan per vector
    int pk = INT_MIN;
    double pv[K];
#pragma unroll
    for (int jj = 0; jj < K; jj++) warp_seg_scan(cur, acc[jj], pk, pv[jj]);
    const int next_first = __shfl_down_sync(FULL, key0, 1);
    const bool next_has = lane < 31 && (q > 0 || lane + 1 < r);
    if (nseg >= 2) {
      double h[K];
#pragma unroll
      for (int jj = 0; jj < K; jj++) h[jj] = (pk == first) ? firstv[jj] + pv[jj] : firstv[jj];
      put_row(first, h);
    }
    if (nseg >= 1 && !(next_has && next_first == cur)) {
      double h[K];
#pragma unroll
      for (int jj = 0; jj < K; jj++) h[jj] = (pk == cur) ? pv[jj] + acc[jj] : acc[jj];
      put_row(cur, h);
    }
    __syncwarp();
    // rows of the tile with no nonzero: Y = beta * Y
    for (int rr = lane; rr < nrows; rr += 32)
      if (!((written[rr >> 5] >> (rr & 31)) & 1u)) {
        double z[K];
#pragma unroll
        for (int jj = 0; jj < K; jj++) z[jj] = 0.0;
        mm_write_row<VT, K>(y + (yrow0 + rr) * K, z, alpha, beta);
      }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ pCSC
// pCSC per-GPU kernel (Alg. 5 "Launch": each part scatters its
// columns' contributions into a partial y, "switch the role of x and y",
// P:199).  One CTA per row band (CB_ROWS rows) at a time; the band's fp64
// partial y lives in shared memory and consumer warp w OWNS a contiguous row
// range of it, so the scatter is a plain read-modify-write (no atomics,
// bit-reproducible): every 32-entry step of a warp list holds 32 distinct rows
// (arranged at partition time, internal.h).  A producer lane streams the
// stage blobs with one 1-D TMA each into a CB_NS-stage ring.  Each consumer
// warp is software-pipelined: the next stage's x gathers are in flight while
// it scatters the current one.  At the end of a band every warp writes its own
// rows once: fused y = alpha*acc + beta*y when one rank holds the whole partial
// sum, else acc -> fp64 py for the reduce-scatter.
#ifndef MSREP_CB_NS
#define MSREP_CB_NS 4
#endif
constexpr int CB_NS = MSREP_CB_NS;         // stages
#ifndef MSREP_CB_DEPTH
#define MSREP_CB_DEPTH 2
#endif
constexpr int CB_DEPTH = MSREP_CB_DEPTH;   // stages a consumer warp holds in registers (2 or 3)
constexpr int CB_NC = CB_W * 32;
constexpr int CB_THREADS = CB_NC + 32;     // + one producer warp
constexpr int CB_PER = CB_SEG / 32;        // entries per lane per stage
template <typename VT>
struct CBLayout {
  static constexpr int STAGE = CB_W * CB_SEG * ((int)sizeof(VT) + 4);
  static constexpr int ST_OFF = CB_ROWS * 8;
  static constexpr int DESC_OFF = ST_OFF + CB_NS * STAGE;
  static constexpr int META_OFF = DESC_OFF + CB_NS * 16;   // per stage: [w] same-row groups, [16 + w] first segmented group
  static constexpr int MISC_OFF = META_OFF + CB_NS * 32 * 4;
  static constexpr int BAR_OFF = MISC_OFF + 16;
  static constexpr int TOTAL = BAR_OFF + 2 * CB_NS * 8;
};

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// one consumer warp's share of a stage, in registers
template <typename VT>
struct CBStage {
  int4 d;                 // {band (-1: end), seg | stage << 11, window col base (unit end: slot), flags}
                          // flags: 1 unit end (no entries) | 2 same-row groups | 4 segmented groups
  int hw, sg;             // this warp's same-row groups / first segmented group of the stage's list
  uint32_t pk[CB_PER];
  VT v[CB_PER], xv[CB_PER];
};

template <typename VT, bool NA>
__device__ __forceinline__ void cb_load(CBStage<VT>& S, int it, const unsigned char* smem, const int4* sdesc,
                                        uint64_t* full, uint64_t* empty, const VT* x, uint64_t xpol, int warp,
                                        int lane, int xs) {
  using L = CBLayout<VT>;
  constexpr int V = (int)sizeof(VT);
  const int s = it % CB_NS;
  mbar_wait(&full[s], (uint32_t)((it / CB_NS) & 1));
  S.d = sdesc[s];
  const int* meta = reinterpret_cast<const int*>(smem + L::META_OFF) + s * 32;
  S.hw = (S.d.w & 2) ? meta[warp] : 0;
  S.sg = (S.d.w & 4) ? meta[16 + warp] : INT_MAX;
  const int seg = S.d.y & 0x7ff;
  const unsigned char* st = smem + L::ST_OFF + s * L::STAGE;
  const VT* sv = reinterpret_cast<const VT*>(st) + warp * seg;
  const uint32_t* sp = reinterpret_cast<const uint32_t*>(st + CB_W * seg * V) + warp * seg;
#pragma unroll
  for (int k = 0; k < CB_PER; k++) {
    const int i = k * 32 + lane;
    S.pk[k] = i < seg ? sp[i] : CB_HOLE;
    S.v[k] = i < seg ? sv[i] : VT(0);
  }
  fence_proxy_async();   // the stage's reads are ordered before the producer's next TMA into it
  __syncwarp();
  if (lane == 0) mbar_arrive(&empty[s]);   // the stage is free: the data is in registers
  const VT* xb = x + (int64_t)S.d.z * xs;
#pragma unroll
  for (int k = 0; k < CB_PER; k++)
    S.xv[k] = S.pk[k] != CB_HOLE ? ldx<NA>(xb + (int64_t)(S.pk[k] >> CB_LOG2) * xs, xpol) : VT(0);
}

// CB_PUT rows (row0 + i*stride, i < CB_PUT, those < row_end) receive their full sums a[i]:
// y = alpha*a + beta*y (fused, one rank holds the whole sum), else the fp64 py of the
// reduce-scatter.  The y loads of the batch are all issued before the first store.
constexpr int CB_PUT = 4;
template <typename VT>
__device__ __forceinline__ void cb_put(const ColLaunch& P, int64_t row0, int stride, int64_t row_end,
                                       const double (&a)[CB_PUT]) {
  if (P.fused) {
    VT* y = static_cast<VT*>(P.out);
    double yv[CB_PUT];
#pragma unroll
    for (int i = 0; i < CB_PUT; i++) {
      const int64_t r = row0 + (int64_t)i * stride;
      yv[i] = (P.beta != 0.0 && r < row_end) ? (double)__ldcs(y + r * P.ys) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < CB_PUT; i++) {
      const int64_t r = row0 + (int64_t)i * stride;
      if (r < row_end) {
        double o = P.alpha * a[i];
        if (P.beta != 0.0) o += P.beta * yv[i];
        __stcs(y + r * P.ys, (VT)o);
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < CB_PUT; i++) {
      const int64_t r = row0 + (int64_t)i * stride;
      if (r < row_end) __stcs(static_cast<double*>(P.out) + r, a[i]);
    }
  }
}

template <typename VT, bool NA>
__global__ void __launch_bounds__(CB_THREADS, 1) csc_band_kernel(const ColLaunch P) {
  using L = CBLayout<VT>;
  constexpr int V = (int)sizeof(VT);
  extern __shared__ __align__(128) unsigned char smem[];
  double* acc = reinterpret_cast<double*>(smem);
  int4* sdesc = reinterpret_cast<int4*>(smem + L::DESC_OFF);
  int* misc = reinterpret_cast<int*>(smem + L::MISC_OFF);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + CB_NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < CB_NS; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CB_W);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == CB_W) {   // ---- producer warp: units (fetched dynamically) -> items -> stage blobs
    const uint64_t pol = policy_evict_first();
    int* meta = reinterpret_cast<int*>(smem + L::META_OFF);
    int it = 0;
    auto stage = [&](int4 d, const char* src, int bytes, int hw, int sg) {
      const int s = it % CB_NS;
      if (it >= CB_NS) mbar_wait(&empty[s], (uint32_t)(((it / CB_NS) - 1) & 1));
      if ((d.w & 6) && lane < CB_W) { meta[s * 32 + lane] = hw; meta[s * 32 + 16 + lane] = sg; }
      __syncwarp();
      if (lane == 0) {
        sdesc[s] = d;
        mbar_arrive_expect_tx(&full[s], (uint32_t)bytes);
        if (bytes) tma_1d(smem + L::ST_OFF + s * L::STAGE, src, (uint32_t)bytes, &full[s], pol);
      }
      __syncwarp();
      it++;
    };
    // the next unit is fetched (and its band's item range loaded) one unit ahead, and the item
    // descriptors of a band come in warp-wide batches of 32 -- R-MAT bands average ~3 stages per
    // item, so per-item dependent loads would starve the stage ring
    auto fetch = [&](int4& un, int& i0, int& i1) {
      int u = 0;
      if (lane == 0) u = atomicAdd(&P.ctr[0], 1);
      u = __shfl_sync(FULL, u, 0);
      if (u >= P.nunits) return false;
      un = P.units[u];
      i0 = P.band_item[un.x];
      i1 = P.band_item[un.x + 1];
      return true;
    };
    int4 un;
    int i0, i1;
    // a unit is claimed only when the previous one is fully issued (claiming ahead would hoard units
    // at the tail: banded pCSC 0.27 -> 0.50 ms); the stage ring covers the fetch latency
    while (fetch(un, i0, i1)) {
      const int b = un.x;
      int g = 0;   // band stage index of the item's first stage
      for (int ib = i0; ib < i1 && g < un.z; ib += 32) {
        int4 it4 = make_int4(0, 0, 0, 0);
        int hst_l = 0, sst_l = INT_MAX;
        int64_t off_l = 0;
        if (ib + lane < i1) {
          it4 = P.items[ib + lane];
          hst_l = P.item_hst[ib + lane];
          sst_l = P.item_sst[ib + lane];
          off_l = P.item_off[ib + lane];
        }
        const int nb_items = min(32, i1 - ib);
        for (int t = 0; t < nb_items && g < un.z; t++) {
          const int iy = __shfl_sync(FULL, it4.y, t);
          if (g + iy <= un.y) { g += iy; continue; }
          const int iz = __shfl_sync(FULL, it4.z, t), iw = __shfl_sync(FULL, it4.w, t);
          const int hst = __shfl_sync(FULL, hst_l, t), sst = __shfl_sync(FULL, sst_l, t);
          const int64_t off = __shfl_sync(FULL, off_l, t);
          const int i = ib + t;
          const int q0 = un.y > g ? un.y - g : 0, q1 = min(iy, un.z - g);
          int hw = 0, sgw = INT_MAX;   // lane w < CB_W: warp w's list heads (loaded once per item)
          if (lane < CB_W) {
            if (q0 < hst) hw = P.item_hw[(int64_t)i * CB_W + lane];
            if (q1 > sst) sgw = P.item_sg[(int64_t)i * CB_W + lane];
          }
          const char* src = P.blob + off + (int64_t)q0 * CB_W * CB_SEG * (V + 4);
          for (int q = q0; q < q1; q++) {
            const int seg = q == iy - 1 ? iw : CB_SEG;
            const int bytes = CB_W * seg * (V + 4);
            stage(make_int4(b, seg | (q << 11), iz, (q < hst ? 2 : 0) | (q >= sst ? 4 : 0)), src, bytes, hw, sgw);
            src += bytes;
          }
          g += iy;
        }
      }
      stage(make_int4(b, 0, un.w, 1), nullptr, 0, 0, 0);   // unit end: write out (slot < 0) or park the partial rows
    }
    stage(make_int4(-1, 0, 0, 0), nullptr, 0, 0, 0);
    return;
  }

  // ---- consumer warps
  const VT* __restrict__ x = static_cast<const VT*>(P.x) + P.xbase * P.xs;
  const uint64_t xpol = policy_evict_last();
  for (int r = threadIdx.x; r < CB_ROWS; r += CB_NC) acc[r] = 0.0;
  named_bar_sync(1, CB_NC);
  // CB_DEPTH stages in registers: while stage A is scattered the x gathers of the next stage(s) are
  // in flight
  CBStage<VT> A, B, C;
  int it = 0;
  cb_load<VT, NA>(A, it++, smem, sdesc, full, empty, x, xpol, warp, lane, P.xs);
  if constexpr (CB_DEPTH == 3) {
    if (A.d.x >= 0) cb_load<VT, NA>(B, it++, smem, sdesc, full, empty, x, xpol, warp, lane, P.xs);
    else B = A;
  }
  while (A.d.x >= 0) {
    if constexpr (CB_DEPTH == 3) {
      if (B.d.x >= 0) cb_load<VT, NA>(C, it++, smem, sdesc, full, empty, x, xpol, warp, lane, P.xs);
      else C = B;   // past the terminator: nothing more comes
    } else {
      cb_load<VT, NA>(B, it++, smem, sdesc, full, empty, x, xpol, warp, lane, P.xs);
    }
    // the scatter: 32 distinct rows per step, steps in list order (deterministic)
    if (A.d.w & 6) {   // this stage may hold SAME-ROW groups (heavy rows; first in each list) or
                       // SEGMENTED groups (row-sorted runs; last in each list)
      const int hw = A.hw, sgw = A.sg;
      const int j0 = (A.d.y >> 11) * CB_PER;                                  // list step of k = 0
#pragma unroll
      for (int k = 0; k < CB_PER; k++) {
        if (j0 + k < hw) {   // 32 entries of one heavy row: one warp-reduced update
          double t = (double)A.v[k] * (double)A.xv[k];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(FULL, t, off);
          if (lane == 0) acc[A.pk[k] & (CB_ROWS - 1)] += t;
          __syncwarp();   // visible to the next step's lanes
        } else if (j0 + k >= sgw) {   // rows in contiguous runs: inclusive segmented scan, run ends update
          const bool real = A.pk[k] != CB_HOLE;
          const int key = real ? (int)(A.pk[k] & (CB_ROWS - 1)) : -1 - lane;   // holes: own runs
          double t = real ? (double)A.v[k] * (double)A.xv[k] : 0.0;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const int k2 = __shfl_up_sync(FULL, key, off);
            const double t2 = __shfl_up_sync(FULL, t, off);
            if (lane >= off && k2 == key) t += t2;
          }
          const int kn = __shfl_down_sync(FULL, key, 1);
          if (real && (lane == 31 || kn != key)) acc[key] += t;
          __syncwarp();
        } else {
          if (A.pk[k] != CB_HOLE) {
            double* a = acc + (A.pk[k] & (CB_ROWS - 1));
            *a = fma((double)A.v[k], (double)A.xv[k], *a);
          }
          __syncwarp();   // a row of this step may recur in another lane at the next step
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < CB_PER; k++) {
        if (A.pk[k] != CB_HOLE) {
          double* a = acc + (A.pk[k] & (CB_ROWS - 1));
          *a = fma((double)A.v[k], (double)A.xv[k], *a);
        }
        __syncwarp();   // a row of this step may recur in another lane at the next step
      }
    }
    if (A.d.w & 1) {   // unit complete: this warp writes its rows once and re-zeroes them
      __syncwarp();
      const int b = A.d.x, slot = A.d.z;
      const int lo = P.split[b * (CB_W + 1) + warp], hi = P.split[b * (CB_W + 1) + warp + 1];
      if (slot < 0) {   // the whole band: its rows are complete
        const int64_t r0 = (int64_t)b * CB_ROWS;
        for (int rb = lo + lane; rb < hi; rb += 32 * CB_PUT) {
          double a[CB_PUT];
#pragma unroll
          for (int i = 0; i < CB_PUT; i++) {
            const int r = rb + 32 * i;
            a[i] = r < hi ? acc[r] : 0.0;
            if (r < hi) acc[r] = 0.0;
          }
          cb_put<VT>(P, r0 + rb, 32, r0 + hi, a);
        }
      } else {          // a stage range of a split band: park the partial rows in the unit's slot
        double* sl = P.slots + (int64_t)slot * CB_ROWS;
        for (int r = lo + lane; r < hi; r += 32) {
          __stcg(sl + r, acc[r]);
          acc[r] = 0.0;
        }
        __threadfence();
        named_bar_sync(1, CB_NC);
        if (threadIdx.x == 0)   // after every warp's rows are visible; the band's last unit reduces it
          misc[0] = atomicAdd(&P.tickets[b], 1) == P.bsplit[b].y - 1;
        named_bar_sync(1, CB_NC);
        if (misc[0]) {
          // every unit of the band has parked its rows: y rows = the slots added in slot (= stage)
          // order, whichever CTA comes last -- deterministic; 4 slot loads in flight per step
          __threadfence();
          const int2 bs = P.bsplit[b];
          const int64_t r0 = (int64_t)b * CB_ROWS;
          const int nr = (int)min((int64_t)CB_ROWS, P.m - r0);
          for (int rb = threadIdx.x; rb < nr; rb += CB_NC * CB_PUT) {
            double a[CB_PUT];
#pragma unroll
            for (int i = 0; i < CB_PUT; i++) {
              const int r = rb + CB_NC * i;
              const double* sp = P.slots + (int64_t)bs.x * CB_ROWS + (r < nr ? r : 0);
              double t = 0.0;
              int q = 0;
              for (; q + 4 <= bs.y; q += 4) {
                const double l0 = __ldcg(sp + (int64_t)q * CB_ROWS), l1 = __ldcg(sp + (int64_t)(q + 1) * CB_ROWS);
                const double l2 = __ldcg(sp + (int64_t)(q + 2) * CB_ROWS), l3 = __ldcg(sp + (int64_t)(q + 3) * CB_ROWS);
                t = (((t + l0) + l1) + l2) + l3;
              }
              for (; q < bs.y; q++) t += __ldcg(sp + (int64_t)q * CB_ROWS);
              a[i] = t;
            }
            cb_put<VT>(P, r0 + rb, CB_NC, r0 + nr, a);
          }
          if (threadIdx.x == 0) P.tickets[b] = 0;   // ready for the next launch (stream-ordered)
        }
      }
      named_bar_sync(1, CB_NC);   // every warp's rows are written and zero before the next unit
    }
    A = B;
    if constexpr (CB_DEPTH == 3) B = C;
  }

  // the last CTA to finish resets the work counter for the next launch (every CTA has stopped fetching)
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&P.ctr[1], 1) == (int)gridDim.x - 1) {
      P.ctr[0] = 0;
      __threadfence();
      P.ctr[1] = 0;
    }
  }
}

// ------------------------------------------------------------ tile packing
// Partition-time layout transform (Sec. 4.1, "offload ... to GPUs as specially
// designed kernels"): one warp per tile copies the tile's aux / val / idx into
// its contiguous blob.  aux for pointer kinds = tile-local pointer, i.e.
// clamp(ptr[row0 + j], z0, z1) - z0 for j = 0..nrows (the rebase of Alg. 2 l.12).
__device__ __forceinline__ int pack_col(const PackLaunch& L, int c) {
  if (L.hotslot) {
    const int h = L.hotslot[c];
    if (h >= 0) return (int)(HOT_TAG | (uint32_t)h);
  }
  return L.colmap ? L.colmap[c] : c;
}

__global__ void pack_kernel(const PackLaunch L) {
  const int lane = threadIdx.x & 31;
  const int t = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (t >= L.ntiles) return;
  const int4 d = L.tiles[t];
  const int nrows = d.z & 0xffff, nnz = d.z >> 16;
  char* b = L.blob + (int64_t)L.blob16[t] * 16;
  if (d.w == -3) {   // narrow SELL: as below, column ids as 16-bit offsets from the tile's smallest
    const int W = nnz, R = sell_r(nrows);
    auto colof = [&](int z) { return (uint32_t)(L.colmap ? L.colmap[L.idx[z]] : L.idx[z]); };
    uint32_t lo = 0xffffffffu;
    for (int k = 0; k < R; k++) {
      const int row = k * 32 + lane;
      if (row < nrows)
        for (int z = L.lptr[d.x + row]; z < L.lptr[d.x + row + 1]; z++) lo = min(lo, colof(z));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) lo = min(lo, __shfl_xor_sync(FULL, lo, off));
    if (lane < 4) reinterpret_cast<uint32_t*>(b)[lane] = lane == 0 ? lo : 0u;
    uint16_t* lens = reinterpret_cast<uint16_t*>(b + 16);
    char* vb0 = b + 16 + align16(R * 32 * 2);
    uint16_t* ox = reinterpret_cast<uint16_t*>(vb0 + W * R * 32 * L.vsize);
    for (int k = 0; k < R; k++) {
      const int row = k * 32 + lane;
      const int rs = row < nrows ? L.lptr[d.x + row] : 0;
      const int len = row < nrows ? L.lptr[d.x + row + 1] - rs : 0;
      lens[k * 32 + lane] = (uint16_t)len;
      for (int t = 0; t < W; t++) {
        const bool on = t < len;
        const int sl = (t * R + k) * 32 + lane;
        if (L.vsize == 8) reinterpret_cast<double*>(vb0)[sl] = on ? static_cast<const double*>(L.val)[rs + t] : 0.0;
        else reinterpret_cast<float*>(vb0)[sl] = on ? static_cast<const float*>(L.val)[rs + t] : 0.0f;
        ox[sl] = on ? (uint16_t)(colof(rs + t) - lo) : (uint16_t)0;   // span <= 65535 (host-checked)
      }
    }
    if (lane == 0) {   // zero the 16-byte tail padding of the offsets
      const int used = W * R * 32 * 2;
      for (int q = used; q < align16(used); q++) reinterpret_cast<char*>(ox)[q] = 0;
    }
    return;
  }
  if (d.w == -2) {   // SELL: lane l owns rows l + 32k (k < R); element t of row k at (t*R + k)*32 + l
    const int W = nnz, R = sell_r(nrows);
    uint16_t* lens = reinterpret_cast<uint16_t*>(b);
    char* vb0 = b + align16(R * 32 * 2);
    int* ix = reinterpret_cast<int*>(vb0 + W * R * 32 * L.vsize);
    for (int k = 0; k < R; k++) {
      const int row = k * 32 + lane;
      const int rs = row < nrows ? L.lptr[d.x + row] : 0;
      const int len = row < nrows ? L.lptr[d.x + row + 1] - rs : 0;
      lens[k * 32 + lane] = (uint16_t)len;
      for (int t = 0; t < W; t++) {
        const bool on = t < len;
        const int sl = (t * R + k) * 32 + lane;
        if (L.vsize == 8) reinterpret_cast<double*>(vb0)[sl] = on ? static_cast<const double*>(L.val)[rs + t] : 0.0;
        else reinterpret_cast<float*>(vb0)[sl] = on ? static_cast<const float*>(L.val)[rs + t] : 0.0f;
        ix[sl] = on ? (L.colmap ? L.colmap[L.idx[rs + t]] : L.idx[rs + t]) : 0;
      }
    }
    return;
  }
  const int z0 = d.y;
  if (d.w >= 0) {   // slab: natural order [val][col]
    const int vb = align16(nnz * L.vsize);
    int* ix = reinterpret_cast<int*>(b + vb);
    for (int k = lane; k < nnz; k += 32) {
      if (L.vsize == 8) reinterpret_cast<double*>(b)[k] = static_cast<const double*>(L.val)[z0 + k];
      else reinterpret_cast<float*>(b)[k] = static_cast<const float*>(L.val)[z0 + k];
      ix[k] = pack_col(L, L.idx[z0 + k]);
    }
    return;
  }
  // SEG tile: [key u8][val][col] in lane-chunked slot order (internal.h)
  uint8_t* key = reinterpret_cast<uint8_t*>(b);
  char* vb0 = b + seg_key_bytes(nnz);
  int* ix = reinterpret_cast<int*>(vb0 + align16(nnz * L.vsize));
  if (L.coo) {
    const int64_t r0 = L.row_base + d.x;
    for (int e = lane; e < nnz; e += 32) key[seg_key_off(e, nnz)] = (uint8_t)(L.ptr[z0 + e] - r0);
  } else {
    for (int j = 0; j < nrows; j++) {
      int e0 = L.ptr[d.x + j], e1 = L.ptr[d.x + j + 1];
      e0 = min(max(e0, z0), z0 + nnz) - z0;
      e1 = min(max(e1, z0), z0 + nnz) - z0;
      for (int e = e0 + lane; e < e1; e += 32) key[seg_key_off(e, nnz)] = (uint8_t)j;
    }
  }
  for (int e = lane; e < nnz; e += 32) {
    const int sl = seg_slot(e, nnz);
    if (L.vsize == 8) reinterpret_cast<double*>(vb0)[sl] = static_cast<const double*>(L.val)[z0 + e];
    else reinterpret_cast<float*>(vb0)[sl] = static_cast<const float*>(L.val)[z0 + e];
    ix[sl] = pack_col(L, L.idx[z0 + e]);
  }
}

// hot-x selection (partition time): nonzeros per column of the rank's slice, and the slot table
__global__ void col_degree_kernel(const int32_t* __restrict__ idx, int64_t nz, int32_t* __restrict__ deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nz; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(deg + idx[i], 1);
}
// per-row column span of a row-major slice (narrow SELL eligibility of the transposed column formats)
__global__ void row_span_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ cols, int64_t m,
                                int32_t* __restrict__ lo, int32_t* __restrict__ hi) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= m) return;
  int32_t a = INT_MAX, b = INT_MIN;
  for (int z = ptr[r]; z < ptr[r + 1]; z++) {
    const int32_t q = cols[z];
    a = min(a, q);
    b = max(b, q);
  }
  lo[r] = a;
  hi[r] = b;
}
__global__ void hot_slot_kernel(const int32_t* __restrict__ hot, int nhot, int32_t* __restrict__ slot,
                                const int32_t* __restrict__ val) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nhot) slot[hot[k]] = val ? val[k] : k;
}
// compact x (every SpMV of a compact-x partition): x' rows = x rows of the listed columns
template <typename VT, int K>
// pos != NULL (degree-ordered x'): cols ascending, entry i stored at x' row pos[i] -- the reads of
// x stay in column order (coalesced sectors) and only the stores scatter (into L2-resident x')
__global__ void gather_x_kernel(const VT* __restrict__ x, const int32_t* __restrict__ cols, int64_t n,
                                VT* __restrict__ out, const int32_t* __restrict__ pos) {
  // one compact entry (K values) per thread, 4 independent entries per thread in flight
  constexpr int U = 4;
  const int64_t i0 = (blockIdx.x * (int64_t)blockDim.x) * U + threadIdx.x;
  int32_t c[U];
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int64_t i = i0 + (int64_t)u * blockDim.x;
    c[u] = i < n ? __ldcs(cols + i) : 0;
  }
  VT v[U][K];
#pragma unroll
  for (int u = 0; u < U; u++)
#pragma unroll
    for (int j = 0; j < K; j++) v[u][j] = i0 + (int64_t)u * blockDim.x < n ? __ldg(x + (int64_t)c[u] * K + j) : VT(0);
#pragma unroll
  int64_t o[U];
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int64_t i = i0 + (int64_t)u * blockDim.x;
    o[u] = i < n ? (pos ? (int64_t)__ldcs(pos + i) : i) : 0;
  }
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int64_t i = i0 + (int64_t)u * blockDim.x;
    if (i < n)
#pragma unroll
      for (int j = 0; j < K; j++) out[o[u] * K + j] = v[u][j];
  }
}

// loopback reduce (in-process multi-rank test transport): fixed rank order
__global__ void sum_peers_kernel(const SumLaunch L) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L.count; i += (int64_t)gridDim.x * blockDim.x) {
    if (L.is_int == 1) {
      int a = 0;
      for (int q = 0; q < L.n; q++) a += static_cast<const int*>(L.src[q])[L.off + i];
      static_cast<int*>(L.dst)[i] = a;
    } else if (L.is_int == 2) {   // fp32 partials (column formats on row tiles), summed in rank order
      float a = 0.f;
      for (int q = 0; q < L.n; q++) a += static_cast<const float*>(L.src[q])[L.off + i];
      static_cast<float*>(L.dst)[i] = a;
    } else {
      double a = 0.0;
      for (int q = 0; q < L.n; q++) a += static_cast<const double*>(L.src[q])[L.off + i];
      static_cast<double*>(L.dst)[i] = a;
    }
  }
}

// SpMM on the column formats: a block of k row-major vectors <-> k contiguous vectors, rows [r0, r1)
// (to_planar: dst[j*ld + i] = src[i*k + j]; else dst[i*k + j] = src[j*ld + i])
template <typename VT>
__global__ void planar_kernel(const VT* __restrict__ src, VT* __restrict__ dst, int64_t r0, int64_t r1, int k,
                              int64_t ld, int to_planar) {
  // a thread per row: the planar side is a coalesced vector per j, the row-major side k contiguous values
  for (int64_t i = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r1; i += (int64_t)gridDim.x * blockDim.x) {
    if (to_planar) {
      for (int j = 0; j < k; j++) dst[(int64_t)j * ld + i] = src[i * k + j];
    } else {
      for (int j = 0; j < k; j++) dst[i * k + j] = src[(int64_t)j * ld + i];
    }
  }
}

// --------------------------------------------------------- small kernels
// FIX_G = 8 lanes per (split row, vector j < k): k = 1 for SpMV, the block width for SpMM; records,
// head partials and y are k-wide (record r, vector j at r*k + j; y row-major [m x k]).  The row's
// records are summed G-strided and joined by a fixed shuffle tree (R-MAT's heaviest rows have ~470
// records: one thread summing them serially made the fix-up 30 us; a whole warp per row left most
// lanes idle on its ~5-record average, 16 us per SpMV), then the group's first lane adds the routed
// head partials in part order and applies alpha, beta once.  Fixed order: bit-reproducible.
constexpr int FIX_G = 8;
template <typename VT>
__global__ void fixup_kernel(const FixupLaunch F) {
  constexpr int G = FIX_G;   // lanes per (split row, vector): rows average ~5 records (R-MAT)
  const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int g = threadIdx.x & (G - 1);
  if (t >= (int64_t)F.nsplit * F.k) return;   // whole groups exit together (nsplit*k*G threads, G | 32)
  const unsigned gm = (unsigned)(((1ull << G) - 1) << (threadIdx.x & 31 & ~(G - 1)));
  const int s = F.s0 + (int)(t / F.k), jv = (int)(t % F.k), K = F.k;
  // the row's metadata and its y_in are independent loads: all in flight before the record sum
  const int k0 = F.sr_rec[2 * s], k1 = F.sr_rec[2 * s + 1];
  const int h0 = F.sr_head[2 * s], h1 = F.sr_head[2 * s + 1];
  VT* y = static_cast<VT*>(F.y);
  const int64_t r = F.sr_row[s] * K + jv;
  const double yin = (g == 0 && F.beta != 0.0) ? (double)y[r] : 0.0;
  double acc = 0.0;
  for (int k = k0 + g; k < k1; k += G) acc += F.rec[(int64_t)k * K + jv];
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(gm, acc, off, G);
  if (g != 0) return;
  for (int h = h0; h < h1; h++) {
    const int j = F.head_list[h];
    double hv = 0.0;
    if (j >= F.part_lo && j < F.part_hi) {
      const int jl = j - F.part_lo;
      for (int k = F.part_rec[2 * jl]; k < F.part_rec[2 * jl + 1]; k++) hv = hv + F.rec[(int64_t)k * K + jv];
    } else {
      hv = F.head_all[(int64_t)j * K + jv];
    }
    acc = acc + hv;
  }
  double v = F.alpha * acc;
  if (F.beta != 0.0) v += F.beta * yin;
  y[r] = (VT)v;
  for (int mi = 0; mi < F.nmirror; mi++) static_cast<VT*>(F.mirror[mi])[r] = (VT)v;
}

__global__ void heads_kernel(const HeadLaunch H) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= H.nlocal * H.k) return;
  const int j = t / H.k, jv = t % H.k;
  double hv = 0.0;
  for (int k = H.part_rec[2 * j]; k < H.part_rec[2 * j + 1]; k++) hv = hv + H.rec[(int64_t)k * H.k + jv];
  H.head_local[t] = hv;
}

template <typename VT>
__global__ void scale_kernel(VT* y, int64_t n, double beta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (VT)(beta != 0.0 ? beta * (double)y[i] : 0.0);
}

template <typename VT, typename PT>
__global__ void axpby_kernel(const PT* __restrict__ py, VT* __restrict__ y, int64_t n, double alpha, double beta,
                             int ys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = alpha * (double)py[i];
    if (beta != 0.0) v += beta * (double)y[i * ys];
    y[i * ys] = (VT)v;
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

// ------------------------------------------------------------ CG vector kernels
// Conjugate gradient (Hestenes-Stiefel) on top of msrep_spmv (include/msrep.h
// msrep_cg).  Every kernel works on the rank's owned segment; dot products are
// deterministic: a fixed grid of CG_BLOCKS blocks writes per-block partial sums
// (fixed shuffle tree), one block adds them in index order.
constexpr int CG_BLOCKS = 296, CG_THREADS = 256;

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double ws[CG_THREADS / 32];
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(FULL, v, off);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < CG_THREADS / 32; w++) t += ws[w];
  __syncthreads();
  return t;   // valid in thread 0
}

// r = b - Ax, p = r, partial r.r
template <typename VT>
__global__ void cg_residual_kernel(const VT* __restrict__ b, const VT* __restrict__ ax, VT* __restrict__ r,
                                   VT* __restrict__ p, int64_t n, double* part) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const VT v = (VT)((double)b[i] - (double)ax[i]);
    r[i] = v;
    p[i] = v;
    acc += (double)v * (double)v;
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

template <typename VT>
__global__ void cg_dot_kernel(const VT* __restrict__ a, const VT* __restrict__ b, int64_t n, double* part) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc += (double)a[i] * (double)b[i];
  const double t = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// every block sums the CG_BLOCKS partial sums in the same fixed order (same value everywhere)
__device__ __forceinline__ double sum_parts(const double* part) {
  double t = 0.0;
  for (int i = threadIdx.x; i < CG_BLOCKS; i += blockDim.x) t += part[i];
  __shared__ double tot;
  const double v = block_sum(t);
  if (threadIdx.x == 0) tot = v;
  __syncthreads();
  return tot;
}

// alpha = rs / pAp (pAp = sum of part_in);  x += alpha p;  r -= alpha Ap;  partial r.r -> part_out
template <typename VT>
__global__ void cg_update_xr_kernel(VT* __restrict__ x, VT* __restrict__ r, const VT* __restrict__ p,
                                    const VT* __restrict__ ap, int64_t n, const double* sc, int par,
                                    const double* part_in, double* part_out) {
  // rs == 0: the previous iteration converged exactly (r = p = 0): nothing to do, no 0/0.  pAp == 0
  // with rs > 0 is a breakdown (A not SPD) and still yields inf/NaN for the host check.
  const double rs = sc[par], pap = sum_parts(part_in);
  const double alpha = rs != 0.0 ? rs / pap : 0.0;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = (VT)((double)x[i] + alpha * (double)p[i]);
    const VT v = (VT)((double)r[i] - alpha * (double)ap[i]);
    r[i] = v;
    acc += (double)v * (double)v;
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0) part_out[blockIdx.x] = t;
}

// rs_new = sum of part_in;  beta = rs_new / rs;  p = r + beta p;  rs of the other parity <- rs_new
template <typename VT>
__global__ void cg_update_p_kernel(VT* __restrict__ p, const VT* __restrict__ r, int64_t n, double* sc, int par,
                                   const double* part_in) {
  const double rs_new = sum_parts(part_in);
  const double beta = sc[par] != 0.0 ? rs_new / sc[par] : 0.0;   // converged exactly: p = r = 0
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (VT)((double)r[i] + beta * (double)p[i]);
  if (blockIdx.x == 0 && threadIdx.x == 0) sc[par ^ 1] = rs_new;
}

// *out = sum of part (one block, fixed order)
__global__ void cg_sum_kernel(const double* part, double* out) {
  const double t = sum_parts(part);
  if (threadIdx.x == 0) *out = t;
}

// SM count per device (a process may drive several GPUs)
std::mutex g_kf_mu;
int g_sms[64] = {0};
int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  std::lock_guard<std::mutex> lk(g_kf_mu);
  if (g_sms[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    g_sms[dev] = v > 0 ? v : 148;
  }
  return g_sms[dev];
}

int elementwise_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms() * 8;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

// Per (kernel, device) launch facts, so a launch does not repeat cudaFuncSetAttribute and the
// occupancy query (microseconds of host time that show up between back-to-back small SpMVs).
// Every read and write of the table holds g_kf_mu (contexts may launch from several host threads).
struct KFacts { const void* fn; int dev, smem, occ; };
KFacts g_kf[256];
int g_nkf = 0;
// index of (fn, current device) in g_kf, created on first use; -1 if the table is full
int kfacts_locked(const void* fn, int dev) {
  for (int i = 0; i < g_nkf; i++)
    if (g_kf[i].fn == fn && g_kf[i].dev == dev) return i;
  if (g_nkf == 256) return -1;   // more (kernel, device) pairs than this file has: no caching
  g_kf[g_nkf] = {fn, dev, -1, -1};
  return g_nkf++;
}

template <typename K>
cudaError_t set_smem(K kernel, int bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_kf_mu);
  const int i = kfacts_locked(reinterpret_cast<const void*>(kernel), dev);
  if (i >= 0 && g_kf[i].smem == bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && i >= 0) { g_kf[i].smem = bytes; g_kf[i].occ = -1; }
  return e;
}

template <typename K>
int grid_for(K kernel, int smem_bytes, int ntiles, int warps = WARPS) {
  const int sms = num_sms();
  int dev = 0;
  cudaGetDevice(&dev);
  int occ = -1;
  {
    std::lock_guard<std::mutex> lk(g_kf_mu);
    const int i = kfacts_locked(reinterpret_cast<const void*>(kernel), dev);
    if (i >= 0) occ = g_kf[i].occ;
    if (occ < 0) {
      occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, warps * 32, smem_bytes);
      if (i >= 0) g_kf[i].occ = occ;
    }
  }
  if (occ < 1) occ = 1;
  const int64_t want = ((int64_t)ntiles + warps - 1) / warps;
  const int64_t g = (int64_t)sms * occ;
  return (int)(want < g ? (want < 1 ? 1 : want) : g);
}

constexpr int SELL_1CTA_SMEM = 116 * 1024;   // > half of the SM's 228 KB: one CTA per SM
template <typename VT, bool SELL, bool MIRROR, bool NA, bool HOT, int CL>
cudaError_t launch_rows_k(const RowLaunch& L, cudaStream_t s) {
  using Lay = RowLayout<VT, SELL, HOT>;
  constexpr int nw = HOT ? hot_warps((int)sizeof(VT)) : WARPS;
  static_assert(Lay::HOT_OFF + (HOT ? HOT_AUTO_BYTES : 0) <= 227 * 1024, "rows_kernel shared memory");
  int b = HOT ? Lay::HOT_OFF + ((L.nhot + CL - 1) / CL) * (int)sizeof(VT) : Lay::TOTAL;
  // SELL launches at one CTA per SM (RowLaunch.sell_1cta, picked by timing at partition): the
  // larger L1 holds the in-flight misses of random-column short rows (1.7x faster there), while the
  // stencil's L1-resident gathers prefer two CTAs per SM (profiles/r2_short_rows.jsonl)
  if constexpr (SELL && !HOT) {
    if (L.sell_1cta) b = b > SELL_1CTA_SMEM ? b : SELL_1CTA_SMEM;
  }
  auto kern = rows_kernel<VT, SELL, MIRROR, NA, HOT, CL>;
  cudaError_t e = set_smem(kern, b);
  if (e) return e;
  int g = grid_for(kern, b, L.ntiles, nw);
  if constexpr (CL == 1) {
    kern<<<g, nw * 32, b, s>>>(L);
  } else {   // CTA pairs (one CTA per SM, the two SMs of a TPC) sharing their hot halves over DSMEM
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(nw * 32); cfg.dynamicSmemBytes = (size_t)b; cfg.stream = s;
    cfg.attrs = at; cfg.numAttrs = 1;
    int maxc = 0;
    cfg.gridDim = dim3(CL);
    if (cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg) != cudaSuccess || maxc < 1) { cudaGetLastError(); maxc = 1; }
    g = std::max(CL, std::min(g / CL * CL, maxc * CL));
    cfg.gridDim = dim3(g);
    e = cudaLaunchKernelEx(&cfg, kern, L);
    if (e) return e;
  }
  return cudaGetLastError();
}
template <typename VT, bool SELL, bool MIRROR>
cudaError_t launch_rows_t(const RowLaunch& L, cudaStream_t s) {
  if constexpr (!SELL) {   // the hot x cache serves SEG / slab tiles (SELL launches gather through L2)
    if (L.nhot > 0 && L.hot_cluster == 2)
      return L.xna ? launch_rows_k<VT, false, MIRROR, true, true, 2>(L, s) : launch_rows_k<VT, false, MIRROR, false, true, 2>(L, s);
    if (L.nhot > 0)
      return L.xna ? launch_rows_k<VT, false, MIRROR, true, true, 1>(L, s) : launch_rows_k<VT, false, MIRROR, false, true, 1>(L, s);
  }
  return L.xna ? launch_rows_k<VT, SELL, MIRROR, true, false, 1>(L, s) : launch_rows_k<VT, SELL, MIRROR, false, false, 1>(L, s);
}
template <typename VT, bool SELL>
cudaError_t launch_rows_m(const RowLaunch& L, cudaStream_t s) {
  return L.nmirror > 0 ? launch_rows_t<VT, SELL, true>(L, s) : launch_rows_t<VT, SELL, false>(L, s);
}

#ifndef MSREP_CB_SMEM_MIN
#define MSREP_CB_SMEM_MIN (116 * 1024)
#endif
template <typename VT, bool NA>
cudaError_t launch_cols_k(const ColLaunch& L, cudaStream_t s) {
  // at least MSREP_CB_SMEM_MIN: exactly one CTA per SM (two would share an SM while another idles);
  // no more than the layout needs: the rest of the 256 KB is L1, which holds the x-gather misses
  constexpr int b = CBLayout<VT>::TOTAL > MSREP_CB_SMEM_MIN ? CBLayout<VT>::TOTAL : MSREP_CB_SMEM_MIN;
  cudaError_t e = set_smem(csc_band_kernel<VT, NA>, b);
  if (e) return e;
  const int g = L.nunits < num_sms() ? L.nunits : num_sms();
  if (g < 1) return cudaSuccess;
  csc_band_kernel<VT, NA><<<g, CB_THREADS, b, s>>>(L);
  return cudaGetLastError();
}
template <typename VT>
cudaError_t launch_cols_t(const ColLaunch& L, cudaStream_t s) {
  return L.xna ? launch_cols_k<VT, true>(L, s) : launch_cols_k<VT, false>(L, s);
}

}  // namespace

cudaError_t launch_rows(const RowLaunch& L, cudaStream_t s) {
  if (L.ntiles == 0) return cudaSuccess;
#ifdef MSREP_FORCE_SELL_INST   // tuning experiment: the SELL instantiation for every launch
  if (true) return L.dtype == 0 ? launch_rows_m<double, true>(L, s) : launch_rows_m<float, true>(L, s);
#endif
  if (L.has_sell) return L.dtype == 0 ? launch_rows_m<double, true>(L, s) : launch_rows_m<float, true>(L, s);
  return L.dtype == 0 ? launch_rows_m<double, false>(L, s) : launch_rows_m<float, false>(L, s);
}

cudaError_t launch_cols(const ColLaunch& L, cudaStream_t s) {
  if (L.nunits == 0) return cudaSuccess;
  return L.dtype == 0 ? launch_cols_t<double>(L, s) : launch_cols_t<float>(L, s);
}

cudaError_t launch_pack(const PackLaunch& L, cudaStream_t s) {
  if (L.ntiles == 0) return cudaSuccess;
  const int64_t threads = (int64_t)L.ntiles * 32;
  pack_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(L);
  return cudaGetLastError();
}

cudaError_t launch_fixup(const FixupLaunch& F, cudaStream_t s) {
  if (F.nsplit == 0) return cudaSuccess;
  const int g = (int)(((int64_t)F.nsplit * F.k * FIX_G + 255) / 256);   // FIX_G lanes per (split row, vector)
  if (F.dtype == 0) fixup_kernel<double><<<g, 256, 0, s>>>(F);
  else fixup_kernel<float><<<g, 256, 0, s>>>(F);
  return cudaGetLastError();
}

cudaError_t launch_heads(const HeadLaunch& H, cudaStream_t s) {
  if (H.nlocal == 0) return cudaSuccess;
  heads_kernel<<<(H.nlocal * H.k + 127) / 128, 128, 0, s>>>(H);
  return cudaGetLastError();
}

cudaError_t launch_scale(void* y, int64_t n, double beta, int dtype, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (dtype == 0) scale_kernel<double><<<elementwise_grid(n), 256, 0, s>>>((double*)y, n, beta);
  else scale_kernel<float><<<elementwise_grid(n), 256, 0, s>>>((float*)y, n, beta);
  return cudaGetLastError();
}

cudaError_t launch_axpby_py(const void* py, int py_f32, void* y, int64_t n, double alpha, double beta, int dtype,
                            cudaStream_t s, int ys) {
  if (n <= 0) return cudaSuccess;
  const int g = elementwise_grid(n);
  if (py_f32) axpby_kernel<float, float><<<g, 256, 0, s>>>((const float*)py, (float*)y, n, alpha, beta, ys);
  else if (dtype == 0) axpby_kernel<double, double><<<g, 256, 0, s>>>((const double*)py, (double*)y, n, alpha, beta, ys);
  else axpby_kernel<float, double><<<g, 256, 0, s>>>((const double*)py, (float*)y, n, alpha, beta, ys);
  return cudaGetLastError();
}

cudaError_t launch_planar(const void* src, void* dst, int64_t r0, int64_t r1, int k, int64_t ld, int to_planar,
                          int dtype, cudaStream_t s) {
  if (r1 <= r0) return cudaSuccess;
  const int g = elementwise_grid(r1 - r0);
  if (dtype == 0) planar_kernel<double><<<g, 256, 0, s>>>((const double*)src, (double*)dst, r0, r1, k, ld, to_planar);
  else planar_kernel<float><<<g, 256, 0, s>>>((const float*)src, (float*)dst, r0, r1, k, ld, to_planar);
  return cudaGetLastError();
}

cudaError_t launch_sum_peers(const SumLaunch& L, cudaStream_t s) {
  if (L.count <= 0) return cudaSuccess;
  sum_peers_kernel<<<elementwise_grid(L.count), 256, 0, s>>>(L);
  return cudaGetLastError();
}

cudaError_t launch_col_degree(const int32_t* idx, int64_t nz, int32_t* deg, cudaStream_t s) {
  if (nz <= 0) return cudaSuccess;
  col_degree_kernel<<<elementwise_grid(nz), 256, 0, s>>>(idx, nz, deg);
  return cudaGetLastError();
}

cudaError_t launch_row_span(const int32_t* ptr, const int32_t* cols, int64_t m, int32_t* lo, int32_t* hi, cudaStream_t s) {
  if (m <= 0) return cudaSuccess;
  row_span_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(ptr, cols, m, lo, hi);
  return cudaGetLastError();
}

cudaError_t launch_hot_slots(const int32_t* hot, int nhot, int32_t* slot, cudaStream_t s, const int32_t* val) {
  if (nhot <= 0) return cudaSuccess;
  hot_slot_kernel<<<(nhot + 255) / 256, 256, 0, s>>>(hot, nhot, slot, val);
  return cudaGetLastError();
}

cudaError_t launch_gather_x(const void* x, const int32_t* cols, int64_t n, int k, void* out, int dtype, cudaStream_t s,
                            const int32_t* pos) {
  if (n <= 0) return cudaSuccess;
  const unsigned g = (unsigned)((n + 1023) / 1024);   // 256 threads x 4 entries per block
#define MSREP_GATHER(VT, K) gather_x_kernel<VT, K><<<g, 256, 0, s>>>((const VT*)x, cols, n, (VT*)out, pos)
  if (dtype == 0) {
    if (k == 1) MSREP_GATHER(double, 1);
    else if (k == 2) MSREP_GATHER(double, 2);
    else if (k == 4) MSREP_GATHER(double, 4);
    else MSREP_GATHER(double, 8);
  } else {
    if (k == 1) MSREP_GATHER(float, 1);
    else if (k == 2) MSREP_GATHER(float, 2);
    else if (k == 4) MSREP_GATHER(float, 4);
    else MSREP_GATHER(float, 8);
  }
#undef MSREP_GATHER
  return cudaGetLastError();
}

cudaError_t launch_rebase(const int64_t* g, int32_t* l, int64_t n, int64_t lo, int64_t hi, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  rebase_kernel<<<elementwise_grid(n), 256, 0, s>>>(g, l, n, lo, hi);
  return cudaGetLastError();
}

cudaError_t launch_cg(int op, int dtype, void* a, void* b, void* c, const void* d, int64_t n, double* sc, int par,
                      const double* part_in, double* part_out, cudaStream_t s) {
  const int g = CG_BLOCKS;
  if (op == CG_RESIDUAL) {   // a=b_vec, b=ax, c=r, d=p -> part_out
    if (dtype == 0) cg_residual_kernel<double><<<g, CG_THREADS, 0, s>>>((const double*)a, (const double*)b, (double*)c, (double*)d, n, part_out);
    else cg_residual_kernel<float><<<g, CG_THREADS, 0, s>>>((const float*)a, (const float*)b, (float*)c, (float*)d, n, part_out);
  } else if (op == CG_DOT) {   // a . b -> part_out
    if (dtype == 0) cg_dot_kernel<double><<<g, CG_THREADS, 0, s>>>((const double*)a, (const double*)b, n, part_out);
    else cg_dot_kernel<float><<<g, CG_THREADS, 0, s>>>((const float*)a, (const float*)b, n, part_out);
  } else if (op == CG_UPDATE_XR) {   // a=x, b=r, c=p, d=ap
    if (dtype == 0) cg_update_xr_kernel<double><<<g, CG_THREADS, 0, s>>>((double*)a, (double*)b, (const double*)c, (const double*)d, n, sc, par, part_in, part_out);
    else cg_update_xr_kernel<float><<<g, CG_THREADS, 0, s>>>((float*)a, (float*)b, (const float*)c, (const float*)d, n, sc, par, part_in, part_out);
  } else if (op == CG_UPDATE_P) {   // a=p, b=r
    if (dtype == 0) cg_update_p_kernel<double><<<g, CG_THREADS, 0, s>>>((double*)a, (const double*)b, n, sc, par, part_in);
    else cg_update_p_kernel<float><<<g, CG_THREADS, 0, s>>>((float*)a, (const float*)b, n, sc, par, part_in);
  } else if (op == CG_SUM) {   // part_in -> *sc
    cg_sum_kernel<<<1, CG_THREADS, 0, s>>>(part_in, sc);
  }
  return cudaGetLastError();
}

namespace {
template <typename VT, int K, bool SELL>
cudaError_t launch_rows_mm_t(const RowLaunch& L, cudaStream_t s) {
  const int b = RowLayout<VT, SELL>::HOT_OFF + L.nhot * 4;   // + the hot slot -> column table
  cudaError_t e = set_smem(rows_mm_kernel<VT, K, SELL>, b);
  if (e) return e;
  rows_mm_kernel<VT, K, SELL><<<grid_for(rows_mm_kernel<VT, K, SELL>, b, L.ntiles), WARPS * 32, b, s>>>(L);
  return cudaGetLastError();
}
template <typename VT, int K>
cudaError_t launch_rows_mm_k(const RowLaunch& L, cudaStream_t s) {
  return L.has_sell ? launch_rows_mm_t<VT, K, true>(L, s) : launch_rows_mm_t<VT, K, false>(L, s);
}
}  // namespace

cudaError_t launch_rows_mm(const RowLaunch& L, int k, cudaStream_t s) {
  if (L.ntiles == 0) return cudaSuccess;
  if (L.dtype == 0) {
    if (k == 2) return launch_rows_mm_k<double, 2>(L, s);
    if (k == 4) return launch_rows_mm_k<double, 4>(L, s);
    return launch_rows_mm_k<double, 8>(L, s);
  }
  if (k == 2) return launch_rows_mm_k<float, 2>(L, s);
  if (k == 4) return launch_rows_mm_k<float, 4>(L, s);
  return launch_rows_mm_k<float, 8>(L, s);
}

}  // namespace msrep
