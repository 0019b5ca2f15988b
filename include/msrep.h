/*
 * msrep.h -- C ABI of the B200-native msRep hot path (arXiv 2209.07552):
 * nnz-balanced multi-GPU SpMV  y <- alpha*A*x + beta*y  over the paper's
 * augmented formats pCSR, pCSC and pCOO.
 *
 * Citations: P:a-b = PAPER.md lines, S:a-b = SPEC.md lines.
 *
 *   problem statement       y = alpha*A*x + beta*y              P:203-218 (Alg. 1)
 *   nnz split               b_i = floor(i*nnz/np)                P:311-312 (Alg. 2 l.2-3)
 *   pCSR / pCSC / pCOO      Alg. 2 / Alg. 4 / Alg. 6
 *   launch + merge          Alg. 3 / Alg. 5 / Alg. 7
 *   row / column merge      Sec. 4.3
 *   one worker per GPU      Sec. 3.3
 *
 * No exceptions cross this boundary.  Every call returns msrep_status_t; on a
 * failure msrep_last_error() returns a thread-local message.  Arguments are
 * validated before any device work.  All device work is enqueued on the
 * caller's CUDA stream (a cudaStream_t passed as void*; NULL = legacy default
 * stream) and is asynchronous with CUDA semantics unless stated otherwise.
 *
 * Data types: host pointer arrays are int64; device index arrays are int32
 * (m, n < 2^31 and per-rank nnz < 2^31, else MSREP_ERR_TOO_LARGE).  Values are
 * fp64 or fp32 storage; every sum is accumulated in fp64 and rounded once to
 * the storage type (reading R13).
 */
#ifndef MSREP_H_
#define MSREP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSREP_VERSION_MAJOR 0
#define MSREP_VERSION_MINOR 1

typedef struct msrep_ctx_s* msrep_ctx;

/* Storage format of the caller's global matrix (Sec. 2.1).
 * MSREP_COO must be sorted by row (ties by column), "we assume the elements
 * are sorted by rows"; otherwise MSREP_ERR_UNSORTED_COO.
 * MSREP_COO_COL is a COO sorted by column (ties by row), the variant the paper
 * describes and defers (merged "like pCSC", P:597 Fig. col-gather):
 * Alg. 6 runs on the column ids, parts own column ranges, partial y vectors
 * are summed (reduce-scatter).  It uses the pCSC kernel.
 * MSREP_COO_UNSORTED is a COO in any order ("if the elements are
 * unsorted ... elements in a particular partition can spread among the entire
 * matrix"): coo_row = row_idx, idx = col_idx.  The nnz split is by position;
 * a part's descriptor carries its smallest / largest row (DESIGN.md reading
 * R25), no flag, no owned rows; each rank sorts its own triplets by column at
 * partition time and runs the pCSC kernel, and the partial y vectors are
 * merged column-style (reduce-scatter; layouts REPLICATED / SHARDED).  Split:
 * nnz or two-level (no row blocks). */
typedef enum { MSREP_CSR = 0, MSREP_CSC = 1, MSREP_COO = 2, MSREP_COO_COL = 3, MSREP_COO_UNSORTED = 4 } msrep_format;

typedef enum { MSREP_F64 = 0, MSREP_F32 = 1 } msrep_dtype;

/* How the nonzeros are cut into the np parts.
 *  NNZ:   the msRep split b_i = floor(i*nnz/np) (Alg. 2 / 4 / 6 lines 2-3):
 *         every part holds nnz/np nonzeros (+-1), rows/columns may be shared.
 *  BLOCK: the paper's "Baseline" (Sec. 5.1): whole row blocks (CSR, COO) or
 *         column blocks (CSC) [floor(i*outer/np), floor((i+1)*outer/np)),
 *         b_i = ptr[floor(i*outer/np)]; never shares a row, imbalanced when the
 *         nonzeros are (Fig. 6).  Same kernels and merge.
 *  TWO_LEVEL: the paper's NUMA-aware two-level split (Sec. 4.2, Fig.
 *         2level): nonzeros go to NUMA groups in proportion to their part
 *         counts, then each group's range is cut by the floor rule; set with
 *         msrep_set_split_groups.  Not identical to NNZ in general (S:231's
 *         claim is false, reading R20); parts differ by <= 2.
 *         (The matrix is device-resident here, so "placement" is the upload.) */
typedef enum { MSREP_SPLIT_NNZ = 0, MSREP_SPLIT_BLOCK = 1, MSREP_SPLIT_TWO_LEVEL = 2 } msrep_split;

/* Where y ends up after msrep_spmv (reading R19; the paper merges
 * into CPU memory).
 *  REPLICATED: every rank's y[0..m) holds the full result.
 *              pCSR/pCOO: boundary fix-up + allgatherv of owned row segments.
 *              pCSC: reduce-scatter of partial y + epilogue + allgatherv.
 *  OWNED:      pCSR/pCOO only: rank writes exactly its owned rows
 *              [owned_begin of its first part, owned_end of its last part).
 *  SHARDED:    pCSC only: rank writes rows [r*ceil(m/R), min(m,(r+1)*ceil(m/R))).
 * Rows a rank does not write are left untouched. */
typedef enum { MSREP_Y_REPLICATED = 0, MSREP_Y_OWNED = 1, MSREP_Y_SHARDED = 2 } msrep_layout;

typedef enum {
  MSREP_OK = 0,
  MSREP_ERR_INVALID_ARG = 1,
  MSREP_ERR_DIM_MISMATCH = 2,   /* ptr[0] != 0, ptr[last] != nnz, decreasing ptr, index out of range */
  MSREP_ERR_UNSORTED_COO = 3,
  MSREP_ERR_TOO_LARGE = 4,      /* m or n >= 2^31, or a rank's nnz >= 2^31 - 2^16 */
  MSREP_ERR_STATE = 5,          /* spmv before partition, layout invalid for the format, ... */
  MSREP_ERR_OOM = 6,
  MSREP_ERR_CUDA = 7,
  MSREP_ERR_NCCL = 8
} msrep_status_t;

/* One part's descriptor, Alg. 2 / 4 / 6 outputs.
 * For pCSC, start_row/end_row hold start_col/end_col and owned_* are the
 * column-free uniform row shards are not described here (owned_* = 0,0). */
typedef struct {
  int64_t start_idx, end_idx;     /* inclusive nonzero range (Alg. 2 l.2-3); empty part: start_idx == end_idx + 1 */
  int64_t start_row, end_row;     /* strict owners of start_idx / end_idx (reading R3); -1,-1 for an empty part   */
  int32_t start_flag;             /* first row/col is shared with an earlier part (Alg. 2 l.6-10)                  */
  int32_t reserved;               /* 0                                                                             */
  int64_t owned_begin, owned_end; /* rows [R_i, R_{i+1}) this part writes (reading R9; row formats only)            */
} msrep_part_desc;

/* Optional device allocator (NULL -> cudaMalloc/cudaFree). */
typedef struct {
  void* (*alloc)(size_t bytes, void* stream, void* user);
  void (*free)(void* p, size_t bytes, void* stream, void* user);
  void* user;
} msrep_allocator;

/* Per-rank facts about the current partition, for measurement. */
typedef struct {
  int64_t nparts, nranks, parts_per_rank;
  int64_t nnz_rank;          /* nonzeros held by this rank                                   */
  int64_t rows_window;       /* rows the rank's local pointer spans (rows_p)                 */
  int64_t owned_rows;        /* rows this rank writes under OWNED (row formats)              */
  int64_t distinct_cols;     /* X_p: distinct x entries the rank's nonzeros touch            */
  int64_t ntiles, nslabs, nsplit_rows, nheads_local;
  int64_t alg_bytes;         /* algorithmic HBM bytes of one msrep_spmv on this rank, beta!=0 */
  int64_t alg_bytes_beta0;   /* same with beta == 0 (y_in not read)                          */
  int64_t kernels_per_spmv;  /* kernel launches one msrep_spmv makes on this rank (beta!=0)  */
  int64_t device_bytes;      /* device memory held by the partition                          */
  double partition_ms;       /* host + upload time of the last msrep_partition (wall clock)  */
  int64_t tile_bytes;        /* bytes of the rank's tile blobs as stored on the GPU (what one
                                SpMV streams from HBM for A, incl. 16-B / SELL padding)      */
  int64_t nsell;             /* SELL tiles among the rank's tiles (regular pCSR rows)        */
  double phase_ms[4];        /* partition_ms split into: [0] argument validation (O(m + nnz)
                                host scans), [1] plan (split, Alg. 2/4/6 descriptors, local
                                pointer), [2] device layout schedule (host), [3] upload of the
                                slice + GPU-side rebase / packing up to the sync  */
  int64_t residency;         /* msrep_residency of the partition                             */
  int64_t nchunks;           /* MSREP_RESIDENT_HOST: chunks streamed per SpMV (else 0)       */
  int64_t host_bytes;        /* MSREP_RESIDENT_HOST: pinned bytes streamed H2D per SpMV      */
  int64_t x_no_allocate;     /* x-gather L1 policy picked at partition (1: L1::no_allocate; timed
                                both ways on the built layout, or set by MSREP_TUNE_XLOAD)    */
  int64_t nhot;              /* hot-x cache entries (MSREP_TUNE_HOT_X; 0: no cache)          */
  int64_t hot_nnz;           /* nonzeros whose x gather the hot cache serves                 */
  int64_t x_compact;         /* compact-x entries (MSREP_TUNE_COMPACT_X; 0: gathers read x)   */
  int64_t sell_1cta;         /* SELL-tile launches at one CTA per SM (timed with the x-gather
                                policy at partition; 0: two CTAs per SM)                      */
  int64_t gpu_numa_node;     /* NUMA node of the GPU's PCI function (sysfs; -1 unknown)      */
  int64_t host_numa_node;    /* MSREP_RESIDENT_HOST: node of the pinned layout's first page,
                                allocated preferred on gpu_numa_node; else -1    */
  int64_t stream_bytes;      /* bytes the built layout moves per SpMV (beta != 0): tile blobs
                                as stored + x entries + y; pCOO stores u8 tile row keys, not
                                the 4-B row ids alg_bytes counts                              */
  int64_t col_layout;        /* column formats: 1 row tiles (slice transposed on the GPU), 0 row
                                bands (MSREP_TUNE_COL_LAYOUT); row formats: -1                */
  double layout_ms[6];       /* the device-layout build inside phase_ms[2..3] (host wall clock):
                                row tiles: [0] GPU transposition of a column slice (upload, sort,
                                row pointer), [1] tile schedule, [2] slice upload + column degrees
                                + hot / compact-x selection, [3] x-layout tables + pack kernels,
                                [4] tile table / records, [5] before the transposition; row bands:
                                [0..4] counts, sort, list sizing, items / units, list writes    */
  int64_t x_order;           /* compact x order: 0 column, 1 decreasing degree; -1 no compact x */
  int64_t nsell_narrow;      /* narrow SELL tiles among nsell (16-bit column offsets, MSREP_TUNE_SELL 2) */
} msrep_stats;

/* NCCL unique id for the communicator (rank 0 creates it, the caller
 * broadcasts the 128 bytes, e.g. through torch.distributed).  Not needed when
 * nranks == 1. */
msrep_status_t msrep_get_unique_id(uint8_t id[128]);

/* Create a context for one rank (one process per GPU, Sec. 3.3 P:529 reshaped
 * as SPMD).  nranks*parts_per_rank = np partitions; this rank holds parts
 * [rank*parts_per_rank, (rank+1)*parts_per_rank).  parts_per_rank > 1 runs
 * several of the paper's partitions on one GPU ("virtual parts") and exercises
 * the identical merge path; results are bit-identical to the same np spread
 * over more ranks for pCSR/pCOO.  `id` is ignored when nranks == 1.
 * Makes `device` current on the calling thread. */
msrep_status_t msrep_create(msrep_ctx* out, int rank, int nranks, const uint8_t id[128], int device,
                            int parts_per_rank, const msrep_allocator* alloc);

/* Test transport for the multi-rank merge on ONE device: creates nranks (<= 8)
 * contexts of this process on `device`, ranks 0..nranks-1, whose collectives
 * (head-partial all-gather, allgatherv of y, reduce-scatter of the partial y,
 * CG all-reduces, the mirror fence) meet in-process instead of in NCCL: every
 * rank is driven by its own host thread and calls the same sequence of
 * collective API calls, as the NCCL ranks would.  Data movement is stream-
 * ordered device copies and rank-ordered sum kernels, so every device kernel of
 * the N > 1 path runs for real on one GPU.  out[nranks] receives the contexts;
 * destroy each with msrep_destroy.  Errors: MSREP_ERR_INVALID_ARG. */
msrep_status_t msrep_create_loopback(msrep_ctx* out, int nranks, int device, int parts_per_rank);

/* Partition the caller's global matrix with Alg. 2/4/6 and upload this rank's
 * contiguous nonzero range to its GPU (the only host->device transfer of A).
 *   CSR: ptr = row_ptr[m+1], idx = col_idx[nnz], coo_row = NULL
 *   CSC: ptr = col_ptr[n+1], idx = row_idx[nnz], coo_row = NULL
 *   COO: ptr = NULL,         idx = col_idx[nnz], coo_row = row_idx[nnz] (row-sorted)
 *   COO_COL: ptr = NULL,     idx = row_idx[nnz], coo_row = col_idx[nnz] (column-sorted:
 *            coo_row carries the sorted major index)
 *   COO_UNSORTED: ptr = NULL, idx = col_idx[nnz], coo_row = row_idx[nnz], any order
 *   val = [nnz] of dtype.
 * All host arrays are borrowed read-only for the duration of the call (the
 * call synchronises `stream` before returning).  parts_out, if not NULL,
 * receives all np descriptors.  Replaces any previous partition.  Every rank
 * must call it with identical arguments. */
msrep_status_t msrep_partition(msrep_ctx ctx, msrep_format fmt, msrep_dtype dtype, int64_t m, int64_t n,
                               int64_t nnz, const int64_t* ptr, const int32_t* idx, const int32_t* coo_row,
                               const void* val, msrep_part_desc* parts_out, void* stream);

/* The same for a rank that holds only a slice of the entries (each GPU needs only its own
 * partition): ptr is the full pointer array (CSR row_ptr[m+1] / CSC col_ptr[n+1]; every rank needs
 * it to plan all np parts), idx_slice / val_slice hold global nonzero positions
 * [slice_begin, slice_end).  The slice must contain this rank's range [b_{rank*ppr},
 * b_{(rank+1)*ppr}) under the context's split (msrep_plan / msrep_plan_split tell it in advance),
 * else MSREP_ERR_INVALID_ARG.  CSR / CSC only (the COO plan reads the row index at every cut).
 * Otherwise identical to msrep_partition (same layout, same results). */
msrep_status_t msrep_partition_slice(msrep_ctx ctx, msrep_format fmt, msrep_dtype dtype, int64_t m, int64_t n,
                                     int64_t nnz, const int64_t* ptr, const int32_t* idx_slice,
                                     const void* val_slice, int64_t slice_begin, int64_t slice_end,
                                     msrep_part_desc* parts_out, void* stream);

/* y <- alpha*A*x + beta*y on device memory.  alpha, beta: host
 * scalars of the partition's dtype.  x: device [n], identical on every rank
 * (pCSC reads only its column slice).  y: device [m], in/out.  beta == 0:
 * y_in is not read; alpha == 0: y = beta*y_in and A, x are not read
 * (reading R12).  Collective over ranks when nranks > 1 (all ranks must call
 * it with the same layout and scalars). */
msrep_status_t msrep_spmv(msrep_ctx ctx, const void* alpha, const void* x, const void* beta, void* y,
                          msrep_layout layout, void* stream);

/* Fused compute + allgather for the row formats ("epilogue peer
 * stores"): y <- alpha*A*x + beta*y on this rank's owned rows, and every
 * owned row is ALSO stored, tile by tile from the SpMV epilogue (and the
 * split-row fix-up), into each of the `nmirror` (<= 8) device buffers
 * `mirrors` -- the other ranks' y buffers mapped into this process (CUDA IPC
 * / symmetric memory over NVLink), or local buffers.  With every peer's y in
 * `mirrors`, each rank ends with the full y without an allgatherv: the
 * transfer overlaps the SpMV.  When nranks > 1 a one-integer NCCL all-reduce
 * after the kernels fences the stores (every rank's mirror writes are complete
 * when the call's work on `stream` completes).  y_in is read only from `y`
 * (beta != 0).  pCSC / column-sorted pCOO: MSREP_ERR_STATE. */
msrep_status_t msrep_spmv_mirror(msrep_ctx ctx, const void* alpha, const void* x, const void* beta, void* y,
                                 int nmirror, void* const* mirrors, void* stream);

/* End-to-end variant with HOST vectors: copies x[n] and (if beta != 0) y[m]
 * from host memory (pinned recommended) to context-owned device buffers,
 * runs msrep_spmv, and copies back the rows this rank's layout defines into
 * y.  Synchronous: returns after y is written. */
msrep_status_t msrep_spmv_host(msrep_ctx ctx, const void* alpha, const void* x_host, const void* beta,
                               void* y_host, msrep_layout layout, void* stream);

/* Where the rank's partition lives between calls (the
 * paper's own timed regime, "partitioning ... and distributing the
 * partitions to the GPUs" inside every measured call).
 *   MSREP_RESIDENT_DEVICE (default): the device layout is built once and kept
 *     in HBM; msrep_spmv streams it from HBM.
 *   MSREP_RESIDENT_HOST (out-of-core): msrep_partition builds the same device
 *     layout chunk by chunk on the GPU and parks it in pinned host memory;
 *     every msrep_spmv / msrep_spmm / msrep_cg streams it back H2D in chunks of
 *     <= chunk_bytes through two device staging buffers on a copy stream,
 *     the kernel of chunk k overlapping the copy of chunk k+1.  Device memory
 *     held: 2 staging buffers + the per-tile descriptors, whatever the size of
 *     A, so the rank's slice may exceed HBM (the partition step itself needs
 *     the rank's val/idx span of one chunk on the device at a time).
 * chunk_bytes: 0 -> 256 MiB; a chunk always holds at least one tile / row
 * band.  Applies to the next msrep_partition.  Errors: MSREP_ERR_INVALID_ARG
 * (unknown residency, chunk_bytes < 0). */
typedef enum { MSREP_RESIDENT_DEVICE = 0, MSREP_RESIDENT_HOST = 1 } msrep_residency;
msrep_status_t msrep_set_residency(msrep_ctx ctx, msrep_residency residency, int64_t chunk_bytes);

/* Tuning knobs of a context (explicit API, no environment switches).  Each
 * knob keeps the arithmetic identical (same bits); only speed changes.
 *   MSREP_TUNE_XLOAD    x-gather L1 policy of the SpMV kernels, applied by the
 *                       next msrep_partition: -1 (default) time both policies
 *                       on the built layout and keep the faster; 0 allocate in
 *                       L1; 1 ld.global.nc.L1::no_allocate.
 *   MSREP_TUNE_CG_GRAPH msrep_cg replays a CUDA graph of two iterations where
 *                       supported: 1 (default) on, 0 eager launches.
 *   MSREP_TUNE_HOT_X    shared-memory cache of the rank's hottest x entries for
 *                       the row formats, applied by the next
 *                       msrep_partition: -1 (default) when the top columns hold
 *                       enough of the rank's nonzeros, 0 off, 1 on whenever
 *                       any column qualifies, 2..96: on with a cache of that
 *                       many KiB (default size 32 KiB; auto: fp64 only).
 *   MSREP_TUNE_COMPACT_X compact x for the row formats, applied by the next
 *                       msrep_partition: the tiles index the rank's distinct
 *                       columns and every SpMV first gathers x' = x[cols]
 *                       (one launch): -1 (default) when x is >= 32 MB and either the
 *                       column degrees are skewed (x' in decreasing degree when it
 *                       exceeds half the L2, else in column order) or the rank
 *                       touches <= 3/4 of x (x' in column order); 0 off; 1 on,
 *                       column order; 2 on, decreasing column degree (the most-
 *                       gathered entries share cache lines).
 *   MSREP_TUNE_HOT_CLUSTER CTAs sharing one hot-x cache, applied by the next
 *                       msrep_partition: 1 (default) -- every CTA holds the
 *                       whole cache; 2 -- the kernel runs as CTA pairs
 *                       (thread-block clusters) and each CTA holds half of the
 *                       hot entries, read by its partner over distributed shared
 *                       memory (twice the entries, but measured slower on R-MAT).
 *   MSREP_TUNE_SELL     sliced-ELL tiles for runs of regular rows (row formats),
 *                       applied by the next msrep_partition: 2 (default) on,
 *                       with NARROW tiles (16-bit column offsets from a per-tile
 *                       base, fp32: up to 64 entries per lane) wherever a tile's
 *                       columns span <= 65535 (pCSR / pCOO); 1 on, 32-bit column
 *                       ids only; 0 every row goes to SEG tiles / slabs.
 *   MSREP_TUNE_COL_LAYOUT device layout of the column formats (pCSC, column-
 *                       sorted / unsorted pCOO), applied by the next
 *                       msrep_partition: -1 (default) and 1 -- ROW TILES: the
 *                       rank's column-ordered slice is transposed on the GPU at
 *                       partition time (a stable sort by row, "the
 *                       kernel is invoked with transpose on") and walked by the
 *                       row-tile kernel, its partial y merged column-style as
 *                       before; 0 -- ROW BANDS: the column-ordered scatter into
 *                       shared-memory row bands (csc_band_kernel), built on the
 *                       host threads.  Both give the exact sums of the rank's
 *                       entries; the summation order within a row differs.
 * Errors: MSREP_ERR_INVALID_ARG (unknown knob or value). */
typedef enum { MSREP_TUNE_XLOAD = 0, MSREP_TUNE_CG_GRAPH = 1, MSREP_TUNE_HOT_X = 2, MSREP_TUNE_COMPACT_X = 3,
               MSREP_TUNE_HOT_CLUSTER = 4, MSREP_TUNE_SELL = 5, MSREP_TUNE_COL_LAYOUT = 6 } msrep_tuning;
msrep_status_t msrep_set_tuning(msrep_ctx ctx, msrep_tuning knob, int value);

/* Select the split used by the next msrep_partition on this context (default
 * MSREP_SPLIT_NNZ; NNZ or BLOCK here).  All ranks must select the same split. */
msrep_status_t msrep_set_split(msrep_ctx ctx, msrep_split split);
/* Select MSREP_SPLIT_TWO_LEVEL with `ngroups` groups of parts_per_group[g]
 * consecutive parts (sum = nranks*parts_per_rank, else MSREP_ERR_INVALID_ARG),
 * e.g. {4, 4} for a DGX with two NUMA nodes of 4 GPUs. */
msrep_status_t msrep_set_split_groups(msrep_ctx ctx, int ngroups, const int* parts_per_group);

/* Pure host: the np descriptors of Alg. 2/4 (fmt CSR/CSC, ptr = pointer array
 * of length outer+1) or Alg. 6 (fmt COO, coo_row = row_idx[nnz], m = rows).
 * Used for bit-exact parity with the oracle.  No device, no context. */
msrep_status_t msrep_plan(msrep_format fmt, int64_t outer, int64_t nnz, int np, const int64_t* ptr,
                          const int32_t* coo_row, msrep_part_desc* parts_out);
/* The same for either split (msrep_plan == msrep_plan_split(fmt, MSREP_SPLIT_NNZ, ...)). */
msrep_status_t msrep_plan_split(msrep_format fmt, msrep_split split, int64_t outer, int64_t nnz, int np,
                                const int64_t* ptr, const int32_t* coo_row, msrep_part_desc* parts_out);
/* The same for the two-level split (np = sum of parts_per_group[0..ngroups)). */
msrep_status_t msrep_plan_groups(msrep_format fmt, int64_t outer, int64_t nnz, int ngroups, const int* parts_per_group,
                                 const int64_t* ptr, const int32_t* coo_row, msrep_part_desc* parts_out);

/* Pure host: the exchange step of msrep_spmv for nranks > 1 (Sec. 4.3,
 * P:602-607; readings R6, R9, R10) as msrep_spmv performs it, with
 * np = nranks*parts_per_rank parts planned as msrep_plan_split does.
 *   seg_out[2r], seg_out[2r+1]: y rows [lo, hi) rank r writes under OWNED /
 *       SHARDED and broadcasts in the REPLICATED allgatherv (row formats: its
 *       parts' owned rows; pCSC: uniform shards of ceil(m/nranks) rows, the
 *       reduce-scatter blocks).  Array of 2*nranks, required.
 *   head_row_out[j]: the row that receives part j's head partial (its flagged
 *       first row, summed by the owner before alpha/beta), -1 if none. [np] or NULL.
 *   head_part_out[j]: the part whose fix-up adds that partial (rank =
 *       head_part_out[j] / parts_per_rank), -1 if none.  [np] or NULL.
 * pCSC has no head exchange (heads -1): its partial vectors are summed.
 * Errors as msrep_plan.  No device, no context. */
msrep_status_t msrep_exchange_plan(msrep_format fmt, msrep_split split, int64_t m, int64_t n, int64_t nnz,
                                   int nranks, int parts_per_rank, const int64_t* ptr, const int32_t* coo_row,
                                   int64_t* seg_out, int64_t* head_row_out, int32_t* head_part_out);

/* Pure host test hook for the pCSC band layout (DESIGN.md sec. 5 "pCSC"): arranges ONE warp list
 * the way msrep_partition does.  pk[n]: packed entries in list (CSC) order, row = pk & 8191.
 * order_out[cap] receives the arranged list: entry index, or -1 for a hole; *len_out its length
 * (MSREP_ERR_INVALID_ARG if cap is too small); *same_out the number of leading positions in
 * same-row groups (32 entries of one row each); *seg_from_out the first position of the trailing
 * segmented groups (rows non-decreasing, list order within a row), or -1 if there are none.
 * Between them every aligned group of 32 holds distinct rows.  No device, no context. */
msrep_status_t msrep_debug_arrange(const uint32_t* pk, int64_t n, int64_t* order_out, int64_t cap, int64_t* len_out,
                                   int64_t* same_out, int64_t* seg_from_out);

/* Sparse matrix times a block of k dense vectors (SpMM), Y <- alpha*A*X + beta*Y:
 * the multi-right-hand-side extension of the same partition (
 * the paper's conclusion on reuse by other sparse kernels).
 * X: device [n x k], Y: device [m x k], both row-major contiguous (X[c*k + j]),
 * k in {2, 4, 8}.  Row formats (pCSR, pCOO): the matrix is streamed once for
 * all k vectors (layouts REPLICATED / OWNED).  Column formats (pCSC, column-sorted
 * and unsorted pCOO): X and Y are copied to k planar vectors (context workspace,
 * allocated on first use), one band-kernel pass per vector -- each with the
 * column-style merge when nranks > 1 -- and Y is copied back (layouts
 * REPLICATED / SHARDED).
 * Segments are row blocks of Y; beta == 0: Y not read; alpha == 0: Y = beta*Y.
 * Asynchronous on `stream`, collective when nranks > 1. */
msrep_status_t msrep_spmm(msrep_ctx ctx, const void* alpha, const void* X, const void* beta, void* Y, int k,
                          msrep_layout layout, void* stream);

/* Conjugate gradient (Hestenes-Stiefel) for a symmetric positive definite A
 * (m == n) on top of msrep_spmv: the iterative-solver use of SpMV that the
 * paper's applications point to (Sec. 6 "Benefits to applications").
 * b: device [n] (dtype of the partition), identical on every rank; x: device
 * [n], in = x0, out = the iterate, replicated on every rank.  Each iteration:
 * one msrep_spmv into the rank's owned rows (OWNED / SHARDED layout), a
 * deterministic dot p.Ap, the fused update x += a p, r -= a Ap with r.r, and
 * p = r + b p; the vectors are updated on the owned segment only, p is
 * allgathered before each SpMV and the two dot products are all-reduced
 * (NCCL) when nranks > 1.  Scalars stay on the device; the host reads r.r
 * every `check_every` iterations and stops when ||r|| <= tol * ||b|| or after
 * maxit iterations.  iters_out / relres_out (host, may be NULL): iterations
 * done and ||r|| / ||b|| at exit.  Collective; synchronous.  Workspace (4
 * vectors of n) is allocated on first use and freed with the partition.
 * Errors: MSREP_ERR_DIM_MISMATCH (m != n), MSREP_ERR_STATE (no partition, or
 * a NaN residual: breakdown, A not SPD). */
msrep_status_t msrep_cg(msrep_ctx ctx, const void* b, void* x, double tol, int maxit, int check_every,
                        int* iters_out, double* relres_out, void* stream);

msrep_status_t msrep_get_stats(msrep_ctx ctx, msrep_stats* out);

/* Measurement hook (bench.py's roofline): while enabled, every msrep_spmv
 * records a CUDA event pair on the caller's stream around its dominant kernel
 * (the pCSR/pCOO tile kernel, or the pCSC scatter).  msrep_profile_read
 * synchronises those events and returns the summed device time (ms) and the
 * number of timed launches since the last reset. */
msrep_status_t msrep_profile_enable(msrep_ctx ctx, int enable);
msrep_status_t msrep_profile_read(msrep_ctx ctx, double* kernel_ms, int64_t* launches, int reset);

/* NULL-safe; frees device buffers and the communicator. */
msrep_status_t msrep_destroy(msrep_ctx ctx);

/* Thread-local message for the last failure on this thread ("" if none). */
const char* msrep_last_error(void);

int msrep_version(void); /* MSREP_VERSION_MAJOR*100 + MSREP_VERSION_MINOR */

#ifdef __cplusplus
}
#endif
#endif /* MSREP_H_ */
