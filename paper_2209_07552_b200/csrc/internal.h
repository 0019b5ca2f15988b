// internal.h -- shared definitions between the host runtime (host.cpp) and the
// sm_100a kernels (kernels.cu) of libmsrep.  Not part of the C ABI.
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace msrep {

// A tile is the unit of work one WARP processes: a row-aligned group of whole
// rows (<= MAX_TILE_ROWS rows, <= TILE_NNZ nonzeros), or a "slab" -- a
// contiguous piece (<= SLAB_NNZ nonzeros) of one split row whose partial sum
// goes to a record instead of y.
#ifndef MSREP_TILE_NNZ
#define MSREP_TILE_NNZ 512
#endif
#ifndef MSREP_TILE_NNZ_F32
#define MSREP_TILE_NNZ_F32 768
#endif
constexpr int TILE_NNZ = MSREP_TILE_NNZ;           // fp64 SEG tiles and slabs (a multiple of 32)
constexpr int TILE_NNZ_F32 = MSREP_TILE_NNZ_F32;   // fp32: ~the bytes of an fp64 tile within the register budget
__host__ __device__ constexpr int tile_nnz(int vsize) { return vsize == 4 ? TILE_NNZ_F32 : TILE_NNZ; }
#ifndef MSREP_MAX_TILE_ROWS
#define MSREP_MAX_TILE_ROWS 128
#endif
constexpr int MAX_TILE_ROWS = MSREP_MAX_TILE_ROWS;   // rows per segment tile (uint8 tile-local row keys: <= 256)
static_assert(MAX_TILE_ROWS % 32 == 0 && MAX_TILE_ROWS <= 256, "SEG row keys are u8");
constexpr int SLAB_NNZ = 512;
#ifndef MSREP_WARPS
#define MSREP_WARPS 8
#endif
constexpr int WARPS = MSREP_WARPS;   // warps per CTA (each with its own TMA ring)

// Hot-x cache (row formats): the rank's most-gathered columns (by nonzero count,
// chosen at partition time) get a slot in a CTA-wide shared-memory copy of x, refilled at every
// launch; SEG / slab tiles carry HOT_TAG | slot instead of the column id for them.  One CTA of
// HOT_WARPS warps per SM holds up to HOT_BYTES of x (sized per partition: HOT_AUTO_BYTES by
// default, MSREP_TUNE_HOT_X KiB when set).
constexpr uint32_t HOT_TAG = 0x80000000u;
#ifndef MSREP_HOT_WARPS
#define MSREP_HOT_WARPS 16
#endif
constexpr int HOT_WARPS = MSREP_HOT_WARPS;
#ifndef MSREP_HOT_WARPS_F32
#define MSREP_HOT_WARPS_F32 12
#endif
// fp32 SEG tiles hold 768 nonzeros (24 per lane): 16 warps x 128 registers spilled, 12 warps get 170
__host__ __device__ constexpr int hot_warps(int vsize) { return vsize == 4 ? MSREP_HOT_WARPS_F32 : HOT_WARPS; }
constexpr int HOT_BYTES = 96 * 1024;
#ifndef MSREP_HOT_AUTO_KB
#define MSREP_HOT_AUTO_KB 32
#endif
constexpr int HOT_AUTO_BYTES = MSREP_HOT_AUTO_KB * 1024;

// Device layout: every tile is one contiguous, 16-byte aligned "blob"; each
// segment is padded to 16 bytes so one TMA bulk copy moves the tile.
//
// SEG tile (pCSR and pCOO irregular rows): [keys][val x nnz][col i32 x nnz]
//   key = tile-local row of the nonzero (u8), 4 per 32-bit word in lane order (seg_key_off:
//   lane l's p-th key at byte (p/4)*128 + 4l + p%4; seg_key_bytes).  Lane-chunked order: lane l owns the
//   contiguous nonzeros [b_l, b_l + len_l) of the tile, b_l = l*q + min(l, r),
//   len_l = q + (l < r), with q = nnz / 32, r = nnz % 32; its j-th nonzero
//   (j < q) sits in slot j*32 + l and its extra one (j == q, l < r) in slot
//   32*q + l.  Every shared-memory read of the kernel is a conflict-free
//   32-lane vector and the lane's products stay in registers.  pCOO tiles use
//   the same layout (row ids rebased at pack time): the paper also runs its
//   CSR kernel on COO input.
// SLAB tile: [val x nnz][col x nnz] in natural order.
// SELL tile (regular pCSR rows): 32*R consecutive rows, R in {1, 2, 4} rows per
//   lane, lane l owning rows l, l+32, ... (R*W <= SELL_W_MAX); element t of
//   the lane's k-th row sits at (t*R + k) * 32 + l (sliced-ELL within the tile,
//   W = longest row, shorter rows padded with val 0 / col 0 and masked in the
//   kernel); aux = the 32*R row lengths (uint16, lane-fastest).  R > 1 keeps
//   tiles of short regular rows big (~1000 elements).  The host only forms a
//   SELL tile when padding is <= 1/8 of its elements.
enum TileKind { KIND_SEG = 0, KIND_SLAB = 2, KIND_SELL = 3, KIND_SELLN = 4 };
constexpr int SELL_ROWS = 32;
constexpr int SELL_W_MAX = 32;    // R * W per lane
// Narrow SELL tile (KIND_SELLN, descriptor w = -3): the same sliced-ELL geometry, but the column
// ids are 16-bit offsets from a per-tile base (every column of the tile within 65535 of the
// smallest one -- banded / stencil rows): [base u32, 12 B pad][lens][val][off u16].  An element
// costs V + 2 bytes instead of V + 4, so the fp32 tiles may hold R * W <= 64 per lane (64 rows of
// a 27-point stencil, the bytes of an fp64 tile).
__host__ __device__ constexpr int selln_w_max(int vsize) { return vsize == 4 ? 64 : 32; }
constexpr int SELL_R_MAX = 4;
__host__ __device__ inline int align16(int b) { return (b + 15) & ~15; }
// rows per lane of a SELL tile of `nrows` rows (1, 2 or 4)
__host__ __device__ inline int sell_r(int nrows) { return nrows <= 32 ? 1 : (nrows <= 64 ? 2 : 4); }
// SEG keys: lane l's p-th nonzero has its u8 key at byte (p/4)*128 + 4*l + p%4, so a lane loads 4
// keys with one 32-bit shared-memory read (a conflict-free 32-lane vector per 4 positions)
__host__ __device__ inline int seg_key_bytes(int nnz) {
  const int npos = (nnz >> 5) + ((nnz & 31) ? 1 : 0);
  return 128 * ((npos + 3) >> 2);
}
__host__ __device__ inline int blob_aux_bytes(int kind, int nrows, int nnz) {
  return kind == KIND_SEG ? seg_key_bytes(nnz)
                          : (kind == KIND_SELL ? align16(sell_r(nrows) * 32 * 2)
                                               : (kind == KIND_SELLN ? 16 + align16(sell_r(nrows) * 32 * 2) : 0));
}
// for KIND_SELL / KIND_SELLN, `nnz` is the slice width W
__host__ __device__ inline int blob_bytes(int kind, int nrows, int nnz, int vsize) {
  if (kind == KIND_SELL) {
    const int r32 = sell_r(nrows) * 32;
    return align16(r32 * 2) + nnz * r32 * (vsize + 4);
  }
  if (kind == KIND_SELLN) {
    const int r32 = sell_r(nrows) * 32;
    return 16 + align16(r32 * 2) + nnz * r32 * vsize + align16(nnz * r32 * 2);
  }
  return blob_aux_bytes(kind, nrows, nnz) + align16(nnz * vsize) + align16(nnz * 4);
}
// slot of element e (0 <= e < nnz) in a SEG tile's lane-chunked order
__host__ __device__ inline int seg_slot(int e, int nnz) {
  const int q = nnz >> 5, r = nnz & 31;
  const int big = r * (q + 1);   // elements owned by the r lanes with q+1 nonzeros
  int lane, j;
  if (e < big) { lane = e / (q + 1); j = e - lane * (q + 1); }
  else { lane = r + (e - big) / q; j = e - (lane * q + r); }
  return j < q ? j * 32 + lane : 32 * q + lane;
}
// byte of element e's key in the SEG key block (seg_key_bytes)
__host__ __device__ inline int seg_key_off(int e, int nnz) {
  const int q = nnz >> 5, r = nnz & 31;
  const int big = r * (q + 1);
  int lane, j;
  if (e < big) { lane = e / (q + 1); j = e - lane * (q + 1); }
  else { lane = r + (e - big) / q; j = e - (lane * q + r); }
  return (j >> 2) * 128 + lane * 4 + (j & 3);   // j == q is the extra position
}

// int4 tile descriptor: x = first row, window-local; y = blob offset in
// 16-byte units; z = nrows | (nnz << 16) (SELL: nrows | (W << 16)); w = kind
// of work (>= 0: slab record index; -1: SEG tile; -4: SEG tile without empty rows; -2: SELL; -3: narrow SELL).
constexpr int KIND_W_SEG_DENSE = -4;
struct TileHost { int32_t row0, nz0, packed, rec; };

struct PackLaunch {        // build the tile blobs from the rank's plain slices (partition time)
  const int4* tiles; const int32_t* blob16; int ntiles;       // tiles: {row0, nz0 (rank-local), packed, w}
  const void* val; const int32_t* idx; const int32_t* ptr;    // ptr: window-local pointer (CSR), or COO row ids
  int coo; int vsize; int64_t row_base;                       // COO: global row of window row 0
  char* blob;
  const int32_t* lptr;                                        // window-local pointer (SELL tiles; CSR: == ptr)
  const int32_t* hotslot;                                     // [n]: hot-x slot of a column, -1 if cold; NULL: no hot x
  const int32_t* colmap;                                      // [n]: compact-x id of a column; NULL: no compact x
};

constexpr int MAX_MIRRORS = 8;   // msrep_spmv_mirror: extra y buffers (peer-mapped or local)

struct RowLaunch {
  const int4* tiles; int ntiles;
  const char* blob;
  const void* x; void* y; int64_t ybase;                     // y row of window row 0
  uint32_t xmax;                                             // n - 1 (clamp for padding lanes)
  double alpha, beta; double* rec;
  int dtype;                                                 // dtype 0 = f64, 1 = f32
  int has_sell;                                              // tiles begin with SELL tiles
  int nmirror; void* mirror[MAX_MIRRORS];                    // y rows are also stored here (msrep_spmv_mirror)
  int xna;                                                   // x gathers with L1::no_allocate (SEG / slab tiles)
  const int32_t* hot; int nhot;                              // hot-x columns by slot (nhot == 0: no hot x)
  int hot_cluster;                                           // 2: slots split over a CTA pair (DSMEM), else 1
  int sell_1cta;                                             // SELL-instantiation launches at one CTA per SM
};

// pCSC row-band layout.  The rank's nonzeros are regrouped
// into bands of CB_ROWS consecutive rows, one CTA per band at a time, the
// band's fp64 partial y in shared memory.  Each of the CB_W consumer warps OWNS
// a contiguous row range of the band (ranges balanced by entry count at
// partition time), so the scatter needs no atomics.  Per (band, column chunk)
// "item", each warp's entries form a "warp list" in CSC order (column-major),
// except that every aligned group of 32 entries is arranged to hold 32
// distinct rows (an entry that would repeat a row of its group is deferred to
// a later group); the lists of an item are padded with holes to one common
// length and cut into stages of CB_SEG entries per warp (the last stage
// shorter, a multiple of 4).  A stage is one contiguous blob
//   [val: CB_W x seg][packed: CB_W x seg]
// moved by one 1-D TMA.  packed = (row & (CB_ROWS-1)) | ((window col - chunk
// base) << CB_LOG2); 0xffffffff marks a hole (never a valid entry: a chunk
// spans CB_CHUNK = 2^19 - 1 columns).
#ifndef MSREP_CB_LOG2
#define MSREP_CB_LOG2 13
#endif
constexpr int CB_LOG2 = MSREP_CB_LOG2;
constexpr int CB_ROWS = 1 << CB_LOG2;      // 8192 rows per band: 64 KB fp64 accumulator
constexpr int CB_W = 15;                   // consumer warps (+1 producer: 16 warps, 128 registers)
constexpr int64_t CB_CHUNK = (1ll << (32 - CB_LOG2)) - 1;
constexpr uint32_t CB_HOLE = 0xffffffffu;
#ifndef MSREP_CB_SEG
#define MSREP_CB_SEG 128
#endif
constexpr int CB_SEG = MSREP_CB_SEG;       // entries per warp per pipeline stage
static_assert(CB_SEG % 32 == 0 && CB_SEG < 2048, "stage descriptors pack seg in 11 bits");
struct ColLaunch {
  const int4* items;          // per item: {band, nstages, window col base, last-stage entries per warp}
  const int64_t* item_off;    // byte offset of each item's first stage blob
  const int32_t* band_item;   // [nb + 1]: items of band b are [band_item[b], band_item[b+1])
  const int32_t* split;       // [nb * (CB_W + 1)]: warp w owns band rows [split[b*(CB_W+1)+w], ...[w+1])
  int nb, band0;              // bands [band0, band0 + nb) (band0 > 0: a host-resident chunk)
  const char* blob;
  const void* x; int64_t xbase;                              // x index of window column 0
  int xs, ys;                 // element strides of x and (fused) y: 1 for SpMV; k for one vector of an SpMM block
  void* out; int64_t m;                                      // fused: y (dtype); else fp64 py
  double alpha, beta;
  int fused; int dtype;
  // Units of work, fetched dynamically (ctr[0]) by the CTAs, largest first: {band, first stage,
  // end stage, slot}, stages counted over the band's items in order.  slot < 0: the whole band,
  // written out at the unit's end; slot >= 0: a stage range of a heavy ("split") band whose
  // partial rows go to slots[slot][CB_ROWS] -- the band's LAST unit to finish (ticket) adds the
  // band's slots in slot order and writes the rows (deterministic, no atomics on values).
  int nunits; const int4* units;
  const int2* bsplit;         // [total bands]: {first slot, slots} of a split band ({0, 0} otherwise)
  double* slots;
  int* tickets;               // [total bands]: units of a split band that have written their slot
  int* ctr;                   // [2]: next unit, finished CTAs (reset by the last CTA)
  const int32_t* item_hst;    // [items]: stages [0, item_hst[i]) may hold same-row groups
  const int32_t* item_hw;     // [items * CB_W]: same-row groups leading warp w's list of item i
  const int32_t* item_sst;    // [items]: stages [item_sst[i], ...) may hold segmented groups
  const int32_t* item_sg;     // [items * CB_W]: first segmented group (list step) of warp w's list
  int xna;                    // x gathers with L1::no_allocate
};

struct FixupLaunch {
  int nsplit, s0;                                     // split rows [s0, s0 + nsplit)
  const int64_t* sr_row; const int32_t* sr_rec;       // sr_rec[2*s], [2*s+1] : record range
  const int32_t* sr_head;                             // sr_head[2*s], [2*s+1]: range into head_list
  const int32_t* head_list;                           // global part ids
  const int32_t* part_rec;                            // part_rec[2*j], [2*j+1]: record range of part j's head (local parts)
  int part_lo, part_hi;                               // local global-part range [lo, hi)
  const double* head_all;                             // head sums of all parts (multi-rank), may be null
  const double* rec;
  void* y; double alpha, beta; int dtype;
  int k;                                              // vectors (1: SpMV; SpMM block width)
  int nmirror; void* mirror[MAX_MIRRORS];             // split-row results are also stored here
};

struct HeadLaunch {
  int nlocal; const int32_t* part_rec; const double* rec; double* head_local;
  int k;
};

// loopback transport (host.cpp LoopGroup): dst[i] = sum over ranks q of src[q][off + i], in rank order
constexpr int MAX_LOOP_RANKS = 8;
struct SumLaunch {
  int n; const void* src[MAX_LOOP_RANKS];
  int64_t off, count;
  void* dst;
  int is_int;   // 1: int32 (the mirror fence), 2: fp32, 0: fp64
};

// kernels.cu entry points (all enqueue on `s`)
cudaError_t launch_rows(const RowLaunch& L, cudaStream_t s);
cudaError_t launch_rows_mm(const RowLaunch& L, int k, cudaStream_t s);   // SpMM, k in {2, 4, 8}
cudaError_t launch_cols(const ColLaunch& L, cudaStream_t s);
cudaError_t launch_fixup(const FixupLaunch& L, cudaStream_t s);
cudaError_t launch_heads(const HeadLaunch& L, cudaStream_t s);
cudaError_t launch_scale(void* y, int64_t count, double beta, int dtype, cudaStream_t s);   // y = beta*y
// y = alpha*py + beta*y (py fp64, or fp32 when py_f32)
cudaError_t launch_axpby_py(const void* py, int py_f32, void* y, int64_t count, double alpha, double beta, int dtype,
                            cudaStream_t s, int ystride = 1);
cudaError_t launch_rebase(const int64_t* gptr, int32_t* lptr, int64_t count, int64_t lo, int64_t hi,
                          cudaStream_t s);                                                  // clamp(gptr,lo,hi)-lo
cudaError_t launch_pack(const PackLaunch& L, cudaStream_t s);
cudaError_t launch_sum_peers(const SumLaunch& L, cudaStream_t s);
// rows [r0, r1) of a k-wide row-major block <-> k planar vectors of leading dimension ld
cudaError_t launch_planar(const void* src, void* dst, int64_t r0, int64_t r1, int k, int64_t ld, int to_planar,
                          int dtype, cudaStream_t s);
cudaError_t launch_col_degree(const int32_t* idx, int64_t nz, int32_t* deg, cudaStream_t s);   // deg[idx[i]]++
cudaError_t launch_row_span(const int32_t* ptr, const int32_t* cols, int64_t m, int32_t* lo, int32_t* hi,
                            cudaStream_t s);   // lo/hi[r] = min/max column of row r (empty: INT_MAX/INT_MIN)
cudaError_t launch_hot_slots(const int32_t* hot, int nhot, int32_t* slot, cudaStream_t s,
                             const int32_t* val = nullptr);   // slot[hot[k]] = val ? val[k] : k
// out[i*k + j] = x[cols[i]*k + j], i < n, j < k (compact x for SpMV k = 1, SpMM k > 1)
cudaError_t launch_gather_x(const void* x, const int32_t* cols, int64_t n, int k, void* out, int dtype, cudaStream_t s,
                            const int32_t* pos = nullptr);   // out[pos ? pos[i] : i] = x[cols[i]]
// transpose.cu: a column-format slice of n entries -> the rank-local row-major slice (stable by
// slice position within a row).  rows = row of each entry (input, also the first pass's keys);
// key_a/key_b/perm_a/perm_b: [n] each; scratch: transpose_scratch_words(n) words;
// outputs cols_out / vals_out [n] in row order and ptr_out [m + 1] (int32 row pointer).
struct TransposeLaunch {
  int64_t n, m;
  int V;
  const uint32_t* rows;
  const int32_t* cols;
  const void* vals;
  uint32_t *key_a, *key_b, *perm_a, *perm_b, *scratch;
  int32_t* cols_out;
  void* vals_out;
  int32_t* ptr_out;
};
int64_t transpose_scratch_words(int64_t n);
cudaError_t launch_transpose(const TransposeLaunch& T, cudaStream_t s);
cudaError_t launch_expand_cols(const int64_t* lp, int64_t W, int32_t* col, cudaStream_t s);   // col[lp[w]..lp[w+1]) = w
cudaError_t launch_rebase_cols(const int32_t* v, int64_t n, int32_t base, int32_t* c, cudaStream_t s);   // c = v - base

// CG vector kernels on an owned segment of n entries (kernels.cu).  sc = device scalars
// {rs (parity 0), rs (parity 1), -, bnorm2}; part_in / part_out = CG_PARTS per-block partial
// sums (every consumer block re-sums part_in in the same fixed order).
enum CgOp { CG_RESIDUAL = 0, CG_DOT = 1, CG_UPDATE_XR = 2, CG_UPDATE_P = 3, CG_SUM = 4 };
constexpr int CG_PARTS = 296;
cudaError_t launch_cg(int op, int dtype, void* a, void* b, void* c, const void* d, int64_t n, double* sc, int par,
                      const double* part_in, double* part_out, cudaStream_t s);

}  // namespace msrep
