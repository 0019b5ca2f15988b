// host.cpp -- host runtime of libmsrep: the nnz-balanced partitioner (Alg. 2 /
// 4 / 6), the static tile schedule, device placement of each rank's slice, the
// NCCL merge (Sec. 4.3 reshaped for NVLink), and the C ABI of include/msrep.h.
//
// One process per GPU (Sec. 3.3: "one dedicated CPU thread to manage
// one GPU", reshaped as SPMD ranks).  Each rank computes all np descriptors
// (O(np log m)), keeps only its own contiguous nonzero range on its GPU, and
// exchanges only split-row partials and, for REPLICATED y, its
// owned y segment.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cctype>
#include <climits>
#include <cmath>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include "internal.h"
#include "msrep.h"

using namespace msrep;

namespace {

// NVTX ranges (header-only NVTX v3; free when no tool is attached): the partition phases and the
// steps of msrep_spmv (kernel, head exchange, fix-up, collective) show up by name in nsys / ncu
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};
struct NvtxSeq {   // consecutive ranges (phases); the open one is closed on scope exit, error paths too
  bool on = false;
  void next(const char* name) {
    if (on) nvtxRangePop();
    nvtxRangePushA(name);
    on = true;
  }
  void end() {
    if (on) nvtxRangePop();
    on = false;
  }
  ~NvtxSeq() { end(); }
};

thread_local std::string g_err;

msrep_status_t fail(msrep_status_t s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CUDA_TRY(expr)                                                                             \
  do {                                                                                             \
    cudaError_t e_ = (expr);                                                                       \
    if (e_ != cudaSuccess) return fail(MSREP_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)
#define NCCL_TRY(expr)                                                                             \
  do {                                                                                             \
    ncclResult_t r_ = (expr);                                                                      \
    if (r_ != ncclSuccess) return fail(MSREP_ERR_NCCL, "%s: %s", #expr, ncclGetErrorString(r_));   \
  } while (0)
#define TRY(expr)                                                                                  \
  do {                                                                                             \
    msrep_status_t s_ = (expr);                                                                    \
    if (s_ != MSREP_OK) return s_;                                                                 \
  } while (0)

constexpr int64_t kMaxIdx = (int64_t)1 << 31;

// column-wise formats merge partial y vectors (pCSC, column-sorted pCOO); COO formats carry
// their sorted major index (row ids, or column ids for MSREP_COO_COL) in `coo_row`
inline bool colwise(msrep_format f) { return f == MSREP_CSC || f == MSREP_COO_COL || f == MSREP_COO_UNSORTED; }
inline bool coo_like(msrep_format f) { return f == MSREP_COO || f == MSREP_COO_COL || f == MSREP_COO_UNSORTED; }
constexpr int64_t kMaxRankNnz = kMaxIdx - (1 << 16);
constexpr int64_t COMPACT_X_MIN_BYTES = (int64_t)32 << 20;   // auto compact x when x is >= 32 MB (L2 126 MB)

// ------------------------------------------------------------ descriptors
// Part boundaries b[0..np]: the nnz split b_i = floor(i*nnz/np) (Alg. 2 l.2-3,
// P:311-312), or the paper's "Baseline" row/column blocks (Sec. 5.1):
// b_i = ptr[floor(i*outer/np)] (COO: the first nonzero of row floor(i*m/np)).
void split_bounds(msrep_format fmt, msrep_split split, int64_t outer, int64_t nnz, int np, const int64_t* ptr,
                  const int32_t* row, std::vector<int64_t>& b, const std::vector<int>* groups = nullptr) {
  b.resize((size_t)np + 1);
  if (split == MSREP_SPLIT_TWO_LEVEL) {   // Sec. 4.2: groups by part count, then floor rule inside
    int64_t Dg = 0;
    size_t w = 0;
    for (int sz : *groups) {
      const int64_t c0 = (Dg * nnz) / np, c1 = ((Dg + sz) * nnz) / np;
      for (int i = 0; i < sz; i++) b[w++] = c0 + ((int64_t)i * (c1 - c0)) / sz;
      Dg += sz;
    }
    b[(size_t)np] = nnz;
    return;
  }
  for (int i = 0; i <= np; i++) {
    if (split == MSREP_SPLIT_NNZ) b[(size_t)i] = ((int64_t)i * nnz) / np;
    else if (coo_like(fmt)) {
      const int64_t r = ((int64_t)i * outer) / np;
      b[(size_t)i] = (int64_t)(std::lower_bound(row, row + nnz, (int32_t)std::min<int64_t>(r, INT32_MAX)) - row);
    } else b[(size_t)i] = ptr[((int64_t)i * outer) / np];
  }
}

// Alg. 2/4: BinarySearch -> strict owner upper_bound(ptr, idx) - 1 (reading R3);
// owned range R_i = lower_bound(ptr[0..outer), b_i), R_0 = 0, R_np = outer (R9).
void plan_ptr(int64_t outer, int np, const int64_t* ptr, const std::vector<int64_t>& b, msrep_part_desc* P) {
  for (int i = 0; i < np; i++) {
    const int64_t b0 = b[(size_t)i], b1 = b[(size_t)i + 1];
    msrep_part_desc& d = P[i];
    d.start_idx = b0;
    d.end_idx = b1 - 1;
    d.reserved = 0;
    d.owned_begin = i == 0 ? 0 : (int64_t)(std::lower_bound(ptr, ptr + outer, b0) - ptr);
    d.owned_end = i == np - 1 ? outer : (int64_t)(std::lower_bound(ptr, ptr + outer, b1) - ptr);
    if (b0 == b1) {
      d.start_row = d.end_row = -1;
      d.start_flag = 0;
      continue;
    }
    d.start_row = (int64_t)(std::upper_bound(ptr, ptr + outer + 1, b0) - ptr) - 1;
    d.end_row = (int64_t)(std::upper_bound(ptr, ptr + outer + 1, b1 - 1) - ptr) - 1;
    d.start_flag = b0 > ptr[d.start_row] ? 1 : 0;
  }
}

// Alg. 6 on a row-sorted COO (reading R8): rows read from row_idx at the cuts.
void plan_coo(int64_t m, int np, const int32_t* row, const std::vector<int64_t>& b, msrep_part_desc* P) {
  for (int i = 0; i < np; i++) {
    const int64_t b0 = b[(size_t)i], b1 = b[(size_t)i + 1];
    msrep_part_desc& d = P[i];
    d.start_idx = b0;
    d.end_idx = b1 - 1;
    d.reserved = 0;
    d.owned_begin = i == 0 ? 0 : (b0 == 0 ? 0 : (int64_t)row[b0 - 1] + 1);
    d.owned_end = i == np - 1 ? m : (b1 == 0 ? 0 : (int64_t)row[b1 - 1] + 1);
    if (b0 == b1) {
      d.start_row = d.end_row = -1;
      d.start_flag = 0;
      continue;
    }
    d.start_row = row[b0];
    d.end_row = row[b1 - 1];
    d.start_flag = (b0 > 0 && row[b0 - 1] == row[b0]) ? 1 : 0;
  }
}

// Unsorted COO (Sec. 3.2.3; reading R25): parts are position ranges of the triplet
// list; a part reports the smallest and largest row it touches, no flag, no owned rows (its
// partial y spans the matrix and is merged column-style).
void plan_coo_unsorted(int np, const int32_t* row, const std::vector<int64_t>& b, msrep_part_desc* P) {
  for (int i = 0; i < np; i++) {
    const int64_t b0 = b[(size_t)i], b1 = b[(size_t)i + 1];
    msrep_part_desc& d = P[i];
    d.start_idx = b0;
    d.end_idx = b1 - 1;
    d.reserved = 0;
    d.start_flag = 0;
    d.owned_begin = d.owned_end = 0;
    int64_t lo = -1, hi = -1;
    for (int64_t k = b0; k < b1; k++) {
      if (lo < 0 || row[k] < lo) lo = row[k];
      if (hi < 0 || row[k] > hi) hi = row[k];
    }
    d.start_row = lo;
    d.end_row = hi;
  }
}

// ------------------------------------------------ large host scratch on 2 MB pages
struct HugeBuf {
  void* p = nullptr;
  size_t bytes = 0;
  explicit HugeBuf(size_t n) : bytes(n) {
    p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) { p = nullptr; throw std::bad_alloc(); }
    madvise(p, bytes, MADV_HUGEPAGE);
  }
  ~HugeBuf() { if (p) munmap(p, bytes); }
  HugeBuf(const HugeBuf&) = delete;
  HugeBuf& operator=(const HugeBuf&) = delete;
};

// ------------------------------------------------ host threads for the partition scans
// The partition's O(nnz) host passes run on the host threads, one contiguous index range each
// (Sec. 4.1, "we parallelize the partition process through multi-threading").
int host_threads(int64_t n) {
  if (n < ((int64_t)1 << 20)) return 1;
  return (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
}
template <class F>   // f(lo, hi) over [0, n) in T contiguous ranges
void par_ranges(int64_t n, F&& f) {
  const int T = host_threads(n);
  if (T == 1) { f((int64_t)0, n); return; }
  std::vector<std::thread> th;
  for (int t = 1; t < T; t++) th.emplace_back([&, t] { f(n * t / T, n * (t + 1) / T); });
  f((int64_t)0, n / T);
  for (auto& x : th) x.join();
}
// ------------------------------------------------ NUMA placement of pinned host memory
// Sec. 4.2: host-resident partitions are copied to the GPUs every call, so they should
// live on the GPU's own NUMA node (without it the paper saw no scaling past 3 GPUs on Summit,
// P:849).  The node is the one sysfs reports for the GPU's PCI function; pinned buffers are
// allocated under a preferred-node memory policy (cudaHostAlloc touches and pins the pages, so they
// land there), then the thread's policy is restored.  No libnuma: the two syscalls directly.
constexpr int kMpolDefault = 0, kMpolPreferred = 1, kMpolFNode = 1, kMpolFAddr = 2;

int gpu_numa_node(int device) {
  char bus[64] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) { cudaGetLastError(); return -1; }
  for (char* q = bus; *q; q++) *q = (char)tolower(*q);
  char path[160];
  snprintf(path, sizeof path, "/sys/bus/pci/devices/%s/numa_node", bus);
  FILE* f = fopen(path, "r");
  if (!f) return -1;
  int node = -1;
  if (fscanf(f, "%d", &node) != 1) node = -1;
  fclose(f);
  return node;
}

// node of the page holding p (-1: unknown)
int page_numa_node(const void* p) {
  int node = -1;
  if (!p || syscall(SYS_get_mempolicy, &node, nullptr, 0, const_cast<void*>(p), kMpolFNode | kMpolFAddr) != 0) return -1;
  return node;
}

// cudaHostAlloc with the pages preferred on `node` (node < 0: plain cudaHostAlloc)
cudaError_t host_alloc_on(void** out, size_t bytes, int node) {
  bool bound = false;
  if (node >= 0 && node < 1024) {
    unsigned long mask[1024 / (8 * sizeof(unsigned long))] = {0};
    mask[node / (8 * sizeof(unsigned long))] = 1ul << (node % (8 * sizeof(unsigned long)));
    bound = syscall(SYS_set_mempolicy, kMpolPreferred, mask, (unsigned long)1024) == 0;
  }
  const cudaError_t e = cudaHostAlloc(out, bytes, cudaHostAllocDefault);
  if (bound) syscall(SYS_set_mempolicy, kMpolDefault, nullptr, 0ul);
  return e;
}

// ------------------------------------------------ in-process loopback transport
// msrep_create_loopback: nranks contexts of ONE process on one device, each driven by its own host
// thread, whose collectives meet here instead of in NCCL -- the multi-rank merge (head exchange,
// owner fix-up, allgatherv, reduce-scatter + shard epilogue, CG all-reduces, mirror fence) then
// runs on the device with real ranks on a single GPU.  Protocol per collective: every rank records
// an event after its producing work and publishes its buffers (barrier 1), waits on every peer's
// event and moves / reduces the data it receives with stream-ordered copies and kernels, records a
// second event (barrier 2), and waits on the peers' second events before its stream goes on, so no
// rank overwrites a buffer a peer is still reading.  Sums run in rank order (deterministic).
struct LoopGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> src;   // per rank: the buffer it contributes
  std::vector<void*> dst;         // per rank: the buffer it receives into
  std::vector<cudaEvent_t> ev1, ev2;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      gen++;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

// ---------------------------------------------------------------- memory
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct Ctx {
  int rank = 0, nranks = 1, vparts = 1, np = 1, device = 0;
  int numa_node = -1;               // the GPU's NUMA node (sysfs), for pinned host buffers
  msrep_split split = MSREP_SPLIT_NNZ;
  std::vector<int> groups;          // MSREP_SPLIT_TWO_LEVEL: parts per NUMA group
  ncclComm_t comm = nullptr;
  std::shared_ptr<LoopGroup> loop;  // msrep_create_loopback (else NCCL when nranks > 1)
  double* d_loop_scratch = nullptr; // loopback all-reduce staging
  size_t loop_scratch_bytes = 0;
  msrep_allocator alloc{};
  bool has_alloc = false;

  // partition state
  bool ready = false;
  msrep_format fmt = MSREP_CSR;
  msrep_dtype dtype = MSREP_F64;
  int64_t m = 0, n = 0, nnz = 0;
  std::vector<msrep_part_desc> parts;
  int P0 = 0, P1 = 0;               // local parts [P0, P1)
  int64_t B_lo = 0, B_hi = 0;       // rank nonzero range
  int64_t wlo = 0, whi = 0;         // window rows (cols for CSC)
  int64_t own_lo = 0, own_hi = 0;   // rows this rank writes under OWNED
  bool any_flag = false;            // some part (any rank) has start_flag
  int64_t shard = 0;                // pCSC: ceil(m / nranks)

  std::vector<DevBuf> bufs;
  char* d_blob = nullptr;           // tile blobs [aux][val][idx] (the rank's partition on the GPU)
  int64_t blob_bytes = 0;
  int4* d_tiles = nullptr;
  int ntiles = 0, nsell = 0, nslabs = 0;
  double* d_rec = nullptr;
  int nrec = 0;
  int nsplit = 0;
  int64_t* d_sr_row = nullptr;
  int32_t* d_sr_rec = nullptr;
  int32_t* d_sr_head = nullptr;
  int32_t* d_head_list = nullptr;
  int32_t* d_part_rec = nullptr;
  double* d_head_local = nullptr;
  double* d_head_all = nullptr;
  int* d_fence = nullptr;            // msrep_spmv_mirror completion fence (nranks > 1)
  void* d_py = nullptr;              // column formats, nranks > 1: the partial y of the rank (fp64; row tiles: VT)
  int64_t py_len = 0;
  bool py_f32 = false;              // d_py holds fp32 (an fp32 partition on row tiles)
  // column formats on row tiles (MSREP_TUNE_COL_LAYOUT): the slice transposed at partition time
  bool col_rows = false;
  int64_t ybase = 0;                // y row of tile window row 0 (row formats: wlo; column formats on row tiles: 0)
  int64_t xoff = 0, xn = 0;         // x entries the tiles index: x[xoff + j], j < xn (row formats: 0, n)
  // pCSC row-band layout
  int4* d_citems = nullptr;
  int64_t* d_item_off = nullptr;
  int32_t* d_band_item = nullptr;
  int32_t* d_split = nullptr;
  char* d_cblob = nullptr;
  int64_t cnb = 0, citems = 0;
  int4* d_cunits = nullptr;          // units of work (see CscBands)
  int2* d_bsplit = nullptr;
  double* d_slots = nullptr;
  int* d_tickets = nullptr;
  int* d_ctr = nullptr;
  int64_t nslots = 0;
  int32_t* d_item_hst = nullptr;
  int32_t* d_item_hw = nullptr;
  int32_t* d_item_sst = nullptr;
  int32_t* d_item_sg = nullptr;
  int64_t cunits = 0;
  int nheads_local = 0;

  // CG workspace (msrep_cg): r, p (full length), Ap, partial sums, scalars {rs, pAp, rs_new, bnorm2}
  void* d_cg_r = nullptr;
  void* d_cg_p = nullptr;
  void* d_cg_ap = nullptr;
  double* d_cg_part = nullptr;
  double* d_cg_sc = nullptr;

  // SpMM: k-wide records / head partials (allocated for k <= 8 on first msrep_spmm)
  int mm_k = 0;
  double* d_rec_mm = nullptr;
  double* d_head_local_mm = nullptr;
  double* d_head_all_mm = nullptr;

  // MSREP_RESIDENT_HOST: the device layout parked in pinned host memory, streamed per call
  // in chunks (row formats: tile ranges; pCSC: band ranges) through two staging buffers
  int xna = 0;                      // x-gather L1 policy of the partition (1: L1::no_allocate)
  int sell_1cta = 0;                // SELL launches at one CTA per SM (timed at partition)
  int32_t* d_hot = nullptr;         // hot-x columns by slot (row formats, device-resident)
  int nhot = 0;
  int64_t hot_nnz = 0;              // the rank's nonzeros whose x comes from the hot cache
  int64_t nxc = 0;                  // compact x entries (0: the kernels gather from x itself)
  int x_order = 0;                  // compact x order: 0 column, 1 decreasing degree
  int hot_cluster = 1;              // the partition's hot-x sharing (tune_hot_cluster when built)
  int32_t* d_xcols = nullptr;       // the rank's distinct columns, ascending (compact x -> column)
  int32_t* d_xpos = nullptr;        // degree-ordered x': x' row of d_xcols[i] (NULL: row i)
  void* d_xc = nullptr;             // x' = x[d_xcols], gathered at the start of every SpMV
  void* d_xc_mm = nullptr;          // SpMM: X' (nxc x 8 entries), allocated on first use
  void* d_mm_planar = nullptr;      // SpMM on the column formats: planar X and Y (k <= 8)
  size_t mm_planar_bytes = 0;
  int tune_compact = -1;
  int64_t nsell_narrow = 0;         // narrow SELL tiles (16-bit column offsets)
  int tune_sell = 2;                // SELL tiles for regular rows (0: SEG tiles only, 1: 32-bit ids only, 2: + narrow)
  int tune_hot_cluster = 1;         // CTAs of a cluster sharing one hot-x cache over DSMEM (1 or 2)
  bool split_launch = false;        // SELL tiles and SEG tiles run as two launches (each >= 5-10 % of nnz)
  int residency = MSREP_RESIDENT_DEVICE;
  int64_t chunk_bytes = (int64_t)256 << 20;
  struct Chunk { int32_t t0, t1, u0, u1; int64_t off, bytes; bool has_sell; };
  std::vector<Chunk> chunks;
  char* h_blob = nullptr;           // pinned (cudaHostAlloc)
  int64_t h_bytes = 0;
  char* d_stage[2] = {nullptr, nullptr};
  cudaStream_t cs = nullptr;        // copy stream
  // pipelined msrep_spmv_host (one rank, one part, row tiles in row order): host copies of the tile
  // rows / slab flags and the split rows, the chunking, a D2H stream and per-chunk events
  std::vector<int32_t> h_tile_row0;         // window-local first row of tile t (final tile order)
  std::vector<uint8_t> h_tile_slab;         // tile t is a slab (a piece of a split row)
  std::vector<int64_t> h_sr_row;            // split rows, ascending
  struct HostChunk { int32_t t0, t1, u0, u1; int64_t r0, r1; int32_t s0, s1; };   // SELL / SEG tile ranges
  std::vector<HostChunk> hchunks;           // built on the first pipelined call
  cudaStream_t cs_in = nullptr, cs_out = nullptr;
  std::vector<cudaEvent_t> hev;             // [0]: x in, [1 + k]: y chunk k in, [1 + C + k]: chunk k computed
  cudaStream_t gs = nullptr;        // msrep_cg graph replay stream
  cudaStream_t ss = nullptr;        // side stream of the split SELL / SEG launches
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_go = nullptr, ev_copied[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};

  // partition uploads from pageable caller memory: a pinned two-slot ring (host threads copy
  // into one slot while the DMA drains the other)
  char* h_ring[2] = {nullptr, nullptr};
  cudaEvent_t ring_ev[2] = {nullptr, nullptr};
  bool ring_disabled = false;       // the pinned ring could not be allocated: pageable copies

  // host-vector path buffers
  void* d_hx = nullptr;
  void* d_hy = nullptr;

  msrep_stats stats{};
  // msrep_set_tuning knobs
  int tune_xload = -1;              // -1 auto, 0 allocate, 1 no_allocate
  int tune_cg_graph = 1;
  int tune_hot = -1;                // -1 auto, 0 off, 1 on
  int tune_col_layout = -1;         // column formats: -1 auto (row tiles), 0 row bands, 1 row tiles

  // profiling hook: event pairs around the dominant kernel
  bool prof = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  size_t ev_used = 0;
};

msrep_status_t prof_begin(Ctx* c, cudaStream_t s, cudaEvent_t* end) {
  *end = nullptr;
  if (!c->prof) return MSREP_OK;
  if (c->ev_used == c->ev.size()) {
    cudaEvent_t a, b;
    CUDA_TRY(cudaEventCreate(&a));
    CUDA_TRY(cudaEventCreate(&b));
    c->ev.push_back({a, b});
  }
  auto& p = c->ev[c->ev_used++];
  CUDA_TRY(cudaEventRecord(p.first, s));
  *end = p.second;
  return MSREP_OK;
}

size_t vsz(msrep_dtype t) { return t == MSREP_F64 ? 8 : 4; }

msrep_status_t dalloc(Ctx* c, size_t want, void** out, cudaStream_t s) {
  const size_t bytes = (want + 16 + 255) & ~(size_t)255;   // +16: tile TMA loads round up to 16 B
  void* p = nullptr;
  if (c->has_alloc) {
    p = c->alloc.alloc(bytes, (void*)s, c->alloc.user);
    if (!p) return fail(MSREP_ERR_OOM, "allocator returned NULL for %zu bytes", bytes);
  } else {
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) return fail(e == cudaErrorMemoryAllocation ? MSREP_ERR_OOM : MSREP_ERR_CUDA,
                                      "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
  }
  CUDA_TRY(cudaMemsetAsync(static_cast<char*>(p) + want, 0, bytes - want, s));   // padding only
  c->bufs.push_back({p, bytes});
  *out = p;
  return MSREP_OK;
}

void release_range(Ctx* c, size_t lo, size_t hi) {
  for (size_t i = lo; i < hi; i++) {
    if (c->has_alloc) c->alloc.free(c->bufs[i].p, c->bufs[i].bytes, nullptr, c->alloc.user);
    else cudaFree(c->bufs[i].p);
  }
  c->bufs.erase(c->bufs.begin() + (ptrdiff_t)lo, c->bufs.begin() + (ptrdiff_t)hi);
}

void free_all(Ctx* c) {
  for (auto& b : c->bufs) {
    if (c->has_alloc) c->alloc.free(b.p, b.bytes, nullptr, c->alloc.user);
    else cudaFree(b.p);
  }
  c->bufs.clear();
  if (c->h_blob) cudaFreeHost(c->h_blob);
  c->h_blob = nullptr;
  c->h_bytes = 0;
  c->chunks.clear();
  c->d_stage[0] = c->d_stage[1] = nullptr;
  c->split_launch = false;
  c->ready = false;
  c->d_hx = c->d_hy = nullptr;
  c->d_hot = nullptr;
  c->nhot = 0;
  c->hot_nnz = 0;
  c->nxc = 0;
  c->d_xcols = nullptr;
  c->d_xpos = nullptr;
  c->d_xc = c->d_xc_mm = nullptr;
  c->d_mm_planar = nullptr;
  c->mm_planar_bytes = 0;
  c->d_loop_scratch = nullptr;
  c->loop_scratch_bytes = 0;
  c->d_cg_r = c->d_cg_p = c->d_cg_ap = nullptr;
  c->d_cg_part = c->d_cg_sc = nullptr;
  c->mm_k = 0;
  c->d_rec_mm = c->d_head_local_mm = c->d_head_all_mm = nullptr;
}

// H2D of `bytes` from pageable host memory, enqueued on s.  Large copies go through the pinned
// ring: the host threads fill slot i%2 (after its previous DMA has drained) while the DMA of
// the other slot runs, so the copy proceeds at the pinned H2D rate instead of the driver's
// pageable path (Sec. 4.1 partition optimisation).
constexpr size_t kRingSlot = (size_t)32 << 20;
msrep_status_t h2d(Ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes < ((size_t)8 << 20)) {
    if (bytes) CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return MSREP_OK;
  }
  if (!c->h_ring[0] && !c->ring_disabled) {
    for (int b = 0; b < 2; b++) {
      if (host_alloc_on(reinterpret_cast<void**>(&c->h_ring[b]), kRingSlot, c->numa_node) != cudaSuccess) {
        cudaGetLastError();   // no pinned memory to spare: the driver's pageable path still works
        for (int q = 0; q < 2; q++) {
          if (c->h_ring[q]) cudaFreeHost(c->h_ring[q]);
          if (c->ring_ev[q]) cudaEventDestroy(c->ring_ev[q]);
          c->h_ring[q] = nullptr;
          c->ring_ev[q] = nullptr;
        }
        c->ring_disabled = true;   // do not retry the pinned allocation on every later upload
        break;
      }
      CUDA_TRY(cudaEventCreateWithFlags(&c->ring_ev[b], cudaEventDisableTiming));
      CUDA_TRY(cudaEventRecord(c->ring_ev[b], s));
    }
  }
  if (!c->h_ring[0]) {
    CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return MSREP_OK;
  }
  const char* sp = static_cast<const char*>(src);
  char* dp = static_cast<char*>(dst);
  for (size_t off = 0, i = 0; off < bytes; off += kRingSlot, i++) {
    const int b = (int)(i & 1);
    const size_t len = std::min(kRingSlot, bytes - off);
    CUDA_TRY(cudaEventSynchronize(c->ring_ev[b]));
    char* slot = c->h_ring[b];
    par_ranges((int64_t)len, [&](int64_t lo, int64_t hi) { memcpy(slot + lo, sp + off + lo, (size_t)(hi - lo)); });
    CUDA_TRY(cudaMemcpyAsync(dp + off, slot, len, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaEventRecord(c->ring_ev[b], s));
  }
  return MSREP_OK;
}

template <class T>
msrep_status_t upload(Ctx* c, const T* host, size_t count, T** out, cudaStream_t s) {
  void* p;
  TRY(dalloc(c, count * sizeof(T), &p, s));
  TRY(h2d(c, p, host, count * sizeof(T), s));
  *out = static_cast<T*>(p);
  return MSREP_OK;
}

// ---------------------------------------------------------- tile schedule
struct Schedule {
  std::vector<TileHost> tiles;      // general tiles (merge / COO walk / slabs / pCSC)
  std::vector<TileHost> sell;       // pCSR SELL tiles
  int nrec = 0, nslabs = 0;
  std::vector<int64_t> sr_row;
  std::vector<int32_t> sr_rec, sr_head, head_list, part_rec;
};

struct Packer {
  Schedule& S;
  int64_t wlo;
  const std::vector<int64_t>& lp;   // local pointer over the window (rank-local nonzeros)
  int64_t cur_r0 = -1, cur_r1 = -1;
  const int64_t tnz;                // nonzeros per SEG tile / slab for this value size
  const int32_t* lidx;              // rank-local column ids (host), or
  const int32_t *rlo, *rhi;         // per-window-row column span; both NULL: no narrow SELL tiles
  const int wn;                     // R * W limit of a narrow SELL tile
  explicit Packer(Schedule& s, int64_t w, const std::vector<int64_t>& l, int vsize, const int32_t* li = nullptr,
                  const int32_t* lo = nullptr, const int32_t* hi = nullptr)
      : S(s), wlo(w), lp(l), tnz(tile_nnz(vsize)), lidx(li), rlo(lo), rhi(hi), wn(selln_w_max(vsize)) {}
  int64_t ls(int64_t r) const { return lp[(size_t)(r - wlo)]; }
  int64_t le(int64_t r) const { return lp[(size_t)(r - wlo + 1)]; }
  void flush() {
    if (cur_r0 < 0) return;
    const int64_t nrows = cur_r1 - cur_r0, z0 = ls(cur_r0), nz = le(cur_r1 - 1) - z0;
    bool dense = true;   // no empty row: the kernel writes every row's sum, no scratch zeroing
    for (int64_t r = cur_r0; r < cur_r1 && dense; r++) dense = le(r) > ls(r);
    S.tiles.push_back({(int32_t)(cur_r0 - wlo), (int32_t)z0, (int32_t)(nrows | (nz << 16)), dense ? KIND_W_SEG_DENSE : -1});
    cur_r0 = cur_r1 = -1;
  }
  void add_row(int64_t r) {
    const int64_t len = le(r) - ls(r);
    if (cur_r0 >= 0) {
      const int64_t nz = le(cur_r1 - 1) - ls(cur_r0);
      if (nz + len > tnz || cur_r1 - cur_r0 >= MAX_TILE_ROWS) flush();
    }
    if (cur_r0 < 0) { cur_r0 = r; cur_r1 = r; }
    cur_r1 = r + 1;
  }
  // SELL tile for rows [r, r + 32R) (R rows per lane, whole owned rows < rend) if padding to the
  // longest row is <= 1/8 of the stored elements; tries R = 4, 2, 1.  Narrow (16-bit column
  // offsets, R*W <= wn) when every column of the rows lies within 65535 of the smallest, else
  // R*W <= SELL_W_MAX with 32-bit ids.
  int64_t try_sell(int64_t r, int64_t rend) {
    const bool spans = lidx || rlo;
    const int lim = spans ? std::max(wn, SELL_W_MAX) : SELL_W_MAX;
    for (int R = SELL_R_MAX; R >= 1; R >>= 1) {
      const int64_t e = std::min<int64_t>(r + 32 * R, rend);
      if (R > 1 && e - r <= 32 * (R / 2)) continue;   // a smaller R covers these rows
      int64_t W = 0, sum = 0;
      bool ok = true;
      for (int64_t q = r; q < e && ok; q++) {
        const int64_t len = le(q) - ls(q);
        if (len * R > lim) ok = false;
        W = std::max(W, len);
        sum += len;
      }
      if (!ok || W == 0 || 8 * sum < 7 * W * (e - r)) continue;
      bool narrow = false;
      if (spans && W * R <= wn) {
        int32_t lo = INT32_MAX, hi = INT32_MIN;
        if (lidx) {
          for (int64_t z = ls(r); z < le(e - 1); z++) {
            lo = std::min(lo, lidx[z]);
            hi = std::max(hi, lidx[z]);
          }
        } else {
          for (int64_t q = r; q < e; q++) {
            lo = std::min(lo, rlo[q - wlo]);
            hi = std::max(hi, rhi[q - wlo]);
          }
        }
        narrow = (int64_t)hi - (int64_t)lo <= 65535;
      }
      if (!narrow && W * R > SELL_W_MAX) continue;
      flush();
      S.sell.push_back({(int32_t)(r - wlo), (int32_t)ls(r), (int32_t)((e - r) | (W << 16)), narrow ? -3 : -2});
      return e;
    }
    return -1;
  }
  // slabs over rank-local nonzeros [z0, z1) of row r; with_records: write partial sums to records
  void slabs(int64_t r, int64_t z0, int64_t z1, bool with_records) {
    for (int64_t z = z0; z < z1; z += tnz) {
      const int64_t nz = std::min<int64_t>(tnz, z1 - z);
      S.tiles.push_back({(int32_t)(r - wlo), (int32_t)z, (int32_t)(1 | (nz << 16)), with_records ? S.nrec++ : -1});
      S.nslabs++;
    }
  }
};

// The parts q > j whose flagged head row is part j's last owned row, in part
// order: the chain that continues j's tail row (reading R10).  Only
// empty parts may sit between them.  Part j's fix-up adds their head partials.
void tail_chain(const std::vector<msrep_part_desc>& P, int j, std::vector<int32_t>& chain) {
  chain.clear();
  const msrep_part_desc& d = P[(size_t)j];
  if (d.start_idx > d.end_idx || d.owned_end <= d.owned_begin) return;
  const int64_t last = d.owned_end - 1;
  for (size_t q = (size_t)j + 1; q < P.size(); q++) {
    const msrep_part_desc& e = P[q];
    if (e.start_idx > e.end_idx) continue;
    if (e.start_flag && e.start_row == last) { chain.push_back((int32_t)q); continue; }
    break;
  }
}

// y rows each rank writes (OWNED) and contributes to the allgatherv (REPLICATED):
// row formats: the union of its parts' owned ranges [R_first, R_last) (reading R9);
// pCSC: uniform shards of ceil(m / nranks) rows (the reduce-scatter blocks).
void rank_segments(msrep_format fmt, int64_t m, int nranks, int vparts, const std::vector<msrep_part_desc>& parts,
                   std::vector<int64_t>& lo, std::vector<int64_t>& hi) {
  lo.resize((size_t)nranks);
  hi.resize((size_t)nranks);
  const int64_t shard = (m + nranks - 1) / nranks;
  for (int r = 0; r < nranks; r++) {
    if (colwise(fmt)) {
      lo[(size_t)r] = std::min<int64_t>(m, (int64_t)r * shard);
      hi[(size_t)r] = std::min<int64_t>(m, (int64_t)(r + 1) * shard);
    } else {
      lo[(size_t)r] = parts[(size_t)r * vparts].owned_begin;
      hi[(size_t)r] = parts[(size_t)(r + 1) * vparts - 1].owned_end;
    }
  }
}

// Row formats (pCSR, pCOO): one rank's schedule.  Per local part j, in order:
// head slabs (flagged first row, exported to its owner), the owned rows
// [R_j, R_{j+1}) packed into row-aligned tiles (rows longer than a tile become
// slab-split rows), and the tail row (owned, continues into later parts) as
// slabs whose fix-up adds the head partials of the parts that continue it.
void build_row_schedule(const std::vector<msrep_part_desc>& P, int P0, int P1, int64_t B_lo, int64_t wlo, int V,
                        const std::vector<int64_t>& lp, Schedule& S, bool allow_sell = true,
                        const int32_t* lidx = nullptr, const int32_t* rlo = nullptr, const int32_t* rhi = nullptr) {
  Packer pk(S, wlo, lp, V, lidx, rlo, rhi);
  for (int j = P0; j < P1; j++) {
    const msrep_part_desc& d = P[(size_t)j];
    const bool empty = d.start_idx > d.end_idx;
    const int64_t lz1 = d.end_idx + 1 - B_lo;
    int32_t h0 = S.nrec;
    if (!empty && d.start_flag) {
      const int64_t r = d.start_row, z0 = d.start_idx - B_lo;
      pk.slabs(r, z0, std::min<int64_t>(lz1, pk.le(r)), true);
    }
    S.part_rec.push_back(h0);
    S.part_rec.push_back(S.nrec);
    // tail: the next non-empty part is flagged and starts in our last owned row
    std::vector<int32_t> chain;
    tail_chain(P, j, chain);
    const int64_t tail = chain.empty() ? -1 : d.owned_end - 1;
    const int64_t rend = tail >= 0 ? tail : d.owned_end;
    auto one_row = [&](int64_t r) {
      const int64_t len = pk.le(r) - pk.ls(r);
      if (len > pk.tnz) {
        pk.flush();
        S.sr_row.push_back(r);
        S.sr_rec.push_back(S.nrec);
        pk.slabs(r, pk.ls(r), pk.le(r), true);
        S.sr_rec.push_back(S.nrec);
        S.sr_head.push_back((int32_t)S.head_list.size());
        S.sr_head.push_back((int32_t)S.head_list.size());
      } else {
        pk.add_row(r);
      }
    };
    for (int64_t r = d.owned_begin; r < rend;) {
      if (allow_sell) {   // SELL tiles for regular rows: pCSR, and pCOO too (window pointer uploaded for packing)
        const int64_t e = pk.try_sell(r, rend);
        if (e > r) { r = e; continue; }
      }
      const int64_t e = std::min<int64_t>(r + SELL_ROWS, rend);
      for (; r < e; r++) one_row(r);
    }
    pk.flush();
    if (tail >= 0) {
      S.sr_row.push_back(tail);
      S.sr_rec.push_back(S.nrec);
      pk.slabs(tail, pk.ls(tail), lz1, true);
      S.sr_rec.push_back(S.nrec);
      S.sr_head.push_back((int32_t)S.head_list.size());
      for (int q : chain) S.head_list.push_back(q);
      S.sr_head.push_back((int32_t)S.head_list.size());
    }
  }
}

// pCSC device layout (internal.h "pCSC row-band layout"), built on the host
// threads at partition time: per-row counts -> balanced warp row ranges per
// band -> a stable parallel counting sort by (band, column chunk, warp) -> per
// warp list, the greedy arrangement that gives every aligned group of 32
// entries distinct rows (run twice: once to size the lists, once to write
// them into the stage blobs).
struct CscBands {
  int64_t nb = 0, nch = 1, bytes = 0;     // bands, column chunks, blob bytes
  int64_t chunk = CB_CHUNK;               // columns per chunk
  std::vector<int4> units;                // {band, first stage, end stage, slot (-1: whole band)}
  std::vector<int2> bsplit;               // [nb]: {first slot, slots} of a split band, {0, 0} otherwise
  int64_t nslots = 0;
  std::vector<int32_t> item_hst;          // [items]: stages that may hold same-row groups
  std::vector<int32_t> item_hw;           // [items * CB_W]: same-row groups leading each warp list
  std::vector<int32_t> item_sst;          // [items]: first stage that may hold segmented groups
  std::vector<int32_t> item_sg;           // [items * CB_W]: first segmented group of each warp list
  std::vector<int4> items;                // {band, nstages, window col base, last-stage seg}
  std::vector<int64_t> item_off;          // byte offset of each item's blob
  std::vector<int32_t> band_item;         // [nb + 1]
  std::vector<int32_t> split;             // [nb * (CB_W + 1)]
  std::unique_ptr<char[]> blob;
};

// Group arrangement of one warp list (entries [0, n) of pk/val, CSC order).
// Rows with more entries than the greedy pass has groups first emit full SAME-ROW groups (32
// entries of one row; the kernel detects them and adds one warp-reduced sum),
// the rest go through a greedy pass that emits groups of 32 DISTINCT rows
// (pk & (CB_ROWS-1)); an entry whose row is already in the open group waits in
// `pend` for a later group, and a group that cannot be filled while entries
// remain is closed with holes.  emit(pos, e) receives every output position
// with its entry (e < 0: hole).  Returns the arranged length.
#ifndef MSREP_SEG_RATIO
#define MSREP_SEG_RATIO 3
#endif
constexpr int64_t SEG_RATIO = MSREP_SEG_RATIO;
#ifndef MSREP_CB_SPLIT_DIV
#define MSREP_CB_SPLIT_DIV 1   // pCSC: split a band holding more than share / DIV stages (share = stages / SMs)
#endif
#ifndef MSREP_CB_PIECE_DIV
#define MSREP_CB_PIECE_DIV 2   // ... into units of about share / DIV stages
#endif
   // segmented tail iff greedy groups >= SEG_RATIO x segmented groups
struct ArrangeScratch {
  int64_t same = 0;   // entries the last arrange_list placed in same-row groups
  int64_t seg_from = INT64_MAX;   // list position (a multiple of 32) where its segmented groups start
  std::vector<int64_t> pend, rest;
  std::vector<int> rows;
  std::vector<uint64_t> used;
  std::vector<int32_t> cnt, taken;
};

template <class Emit>
int64_t arrange_list(const uint32_t* pk, int64_t n, ArrangeScratch& A, Emit&& emit) {
  auto rowof = [&](int64_t e) { return (int)(pk[e] & (CB_ROWS - 1)); };
  if (A.cnt.size() != (size_t)CB_ROWS) { A.cnt.assign(CB_ROWS, 0); A.taken.assign(CB_ROWS, 0); }   // zero between lists
  A.rows.clear();
  for (int64_t e = 0; e < n; e++)
    if (A.cnt[(size_t)rowof(e)]++ == 0) A.rows.push_back(rowof(e));
  // A row forces holes in the greedy pass iff it has more entries than the pass has groups
  // (G = remaining entries / 32).  Such "heavy" rows move their full 32-blocks into same-row
  // groups; G shrinks as they leave, so iterate to a fixed point.
  int64_t G = n / 32;
  for (int it = 0; it < 8; it++) {
    int64_t H = 0;
    for (int r : A.rows)
      if (A.cnt[(size_t)r] > std::max<int64_t>(G, 31)) H += A.cnt[(size_t)r] / 32 * 32;
    const int64_t G2 = (n - H) / 32;
    if (G2 == G) break;
    G = G2;
  }
  const int64_t heavy_min = std::max<int64_t>(G, 31) + 1;
  auto nheavy = [&](int r) -> int64_t { return A.cnt[(size_t)r] >= heavy_min ? A.cnt[(size_t)r] / 32 * 32 : 0; };
  int64_t w = 0;
  // 1. same-row groups: the first 32*floor(cnt/32) entries of every heavy row, in list order
  A.rest.clear();
  for (int64_t e = 0; e < n; e++) {
    const int r = rowof(e);
    if (A.taken[(size_t)r] < nheavy(r)) A.taken[(size_t)r]++;
    else A.rest.push_back(e);
  }
  for (int64_t e = 0; e < n; e++) A.taken[(size_t)rowof(e)] = 0;
  {
    // emit heavy entries row by row (rows in first-appearance order, entries in list order),
    // 32 per group: one stable bucket pass
    std::vector<int64_t> order, heavy;
    std::vector<int64_t> start;
    for (int64_t e = 0; e < n; e++) {
      const int r = rowof(e);
      if (nheavy(r) > 0 && A.taken[(size_t)r] == 0) {
        A.taken[(size_t)r] = 1 + (int32_t)order.size();   // 1-based slot of the row
        order.push_back(r);
      }
    }
    start.assign(order.size() + 1, 0);
    for (size_t k = 0; k < order.size(); k++) start[k + 1] = start[k] + nheavy((int)order[k]);
    heavy.assign((size_t)start.back(), 0);
    std::vector<int64_t> fill(start.begin(), start.end() - 1);
    for (int64_t e = 0; e < n; e++) {
      const int r = rowof(e);
      if (nheavy(r) == 0) continue;
      const size_t k = (size_t)A.taken[(size_t)r] - 1;
      if (fill[k] < start[k + 1]) heavy[(size_t)fill[k]++] = e;
    }
    for (int64_t e : heavy) emit(w++, e);
    A.same = (int64_t)heavy.size();
    for (int r : order) A.taken[(size_t)r] = 0;
  }
  // 2. greedy distinct-row groups over the remaining entries.  When a group cannot be filled with
  // distinct rows while entries remain (the rest sits on fewer than 32 rows), the group is closed
  // with holes and everything left is emitted as SEGMENTED groups: sorted by row (list order
  // within a row), so each group's rows form contiguous runs that the kernel reduces with one
  // warp segmented scan -- no more holes, still no atomics.
  A.seg_from = INT64_MAX;
  A.pend.clear();
  if (A.used.size() != (size_t)(CB_ROWS / 64)) A.used.assign(CB_ROWS / 64, 0);   // cleared per group
  int64_t next = 0;
  const int64_t nr = (int64_t)A.rest.size();
  uint32_t grp[32];
  while (next < nr || !A.pend.empty()) {
    int g = 0;
    auto busy = [&](int64_t e) { const uint32_t r = (uint32_t)rowof(e); return (A.used[r >> 6] >> (r & 63)) & 1; };
    auto take = [&](int64_t e) {
      const uint32_t r = (uint32_t)rowof(e);
      A.used[r >> 6] |= 1ull << (r & 63);
      grp[g++] = r;
      emit(w++, e);
    };
    size_t keep = 0;
    for (size_t k = 0; k < A.pend.size(); k++) {   // deferred entries first, order kept
      const int64_t e = A.pend[k];
      if (g < 32 && !busy(e)) take(e); else A.pend[keep++] = e;
    }
    A.pend.resize(keep);
    while (g < 32 && next < nr) {
      const int64_t e = A.rest[(size_t)next++];
      if (busy(e)) A.pend.push_back(e); else take(e);
    }
    const int real = g;
    const bool stuck = g < 32 && (next < nr || !A.pend.empty());
    if (stuck)   // close the group with holes
      for (; g < 32; g++) emit(w++, -1);
    for (int k = 0; k < real; k++) A.used[grp[k] >> 6] &= ~(1ull << (grp[k] & 63));
    if (stuck && A.seg_from == INT64_MAX) {
      // the greedy pass needs about max-entries-per-row more groups for what is left (one entry
      // of a row per group); segmented groups need ceil(left / 32) but cost several distinct
      // groups each (a 5-step shuffle scan): switch only when that wins clearly
      std::vector<int64_t> left(A.pend.begin(), A.pend.end());
      for (int64_t q = next; q < nr; q++) left.push_back(A.rest[(size_t)q]);
      int32_t mx = 0;
      for (int64_t e : left) mx = std::max(mx, ++A.taken[(size_t)rowof(e)]);
      for (int64_t e : left) A.taken[(size_t)rowof(e)] = 0;
      const int64_t seg_groups = ((int64_t)left.size() + 31) / 32;
      if ((int64_t)mx >= SEG_RATIO * seg_groups + SEG_RATIO) {   // segmented groups for everything left: stable by row
        next = nr;
        A.pend.clear();
        std::stable_sort(left.begin(), left.end(), [&](int64_t a, int64_t b) { return rowof(a) < rowof(b); });
        A.seg_from = w;
        for (int64_t e : left) emit(w++, e);
      } else {
        A.seg_from = INT64_MAX - 1;   // decided: greedy (with holes) to the end of the list
      }
    }
  }
  for (int r : A.rows) A.cnt[(size_t)r] = 0;   // leave the scratch zero
  return w;
}

thread_local double g_csc_ms[6];   // sub-phase times of the last build_csc_bands (diagnostics)
msrep_status_t build_csc_bands(const Ctx& c, const std::vector<int64_t>& lp, const int32_t* idx, const void* val,
                               size_t V, int sms, CscBands& B) {
  auto tq = std::chrono::steady_clock::now();
  auto lapq = [&](int k) {
    const auto now = std::chrono::steady_clock::now();
    g_csc_ms[k] = std::chrono::duration<double, std::milli>(now - tq).count();
    tq = now;
  };
  const int64_t W = c.whi - c.wlo;
  const int64_t nz = c.B_hi - c.B_lo;
  const int32_t* rows = idx + c.B_lo;
  const char* vals = static_cast<const char*>(val) + (size_t)c.B_lo * V;
  B.nb = (c.m + CB_ROWS - 1) / CB_ROWS;
  B.nch = std::max<int64_t>(1, (W + CB_CHUNK - 1) / CB_CHUNK);
  // short-wide matrices have fewer bands than SMs: cut the columns into more chunks and let
  // every (band, chunk) item be a unit of work whose partial band is added into py
  const int64_t units = 2 * (int64_t)sms;
  if (B.nb < (int64_t)sms && W > 0) {
    B.nch = std::max(B.nch, std::min<int64_t>((units + B.nb - 1) / B.nb, std::max<int64_t>(1, W / 4096)));
  }
  B.chunk = std::max<int64_t>(1, (W + B.nch - 1) / B.nch);
  B.nch = std::max<int64_t>(1, (W + B.chunk - 1) / B.chunk);
  const int64_t keys = B.nb * B.nch * CB_W;
  if (keys > ((int64_t)1 << 26))
    return fail(MSREP_ERR_TOO_LARGE, "pCSC band layout: %lld (band, chunk, warp) lists > 2^26", (long long)keys);
  int T = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  while (T > 1 && (int64_t)T * keys > ((int64_t)1 << 26)) T--;
  if (nz < (1 << 20)) T = 1;
  auto run = [&](auto&& f) {
    std::vector<std::thread> th;
    for (int t = 1; t < T; t++) th.emplace_back(f, t);
    f(0);
    for (auto& x : th) x.join();
  };
  std::vector<int64_t> cb((size_t)T + 1, W);   // column ranges with ~equal nonzeros per thread
  cb[0] = 0;
  for (int t = 1; t < T; t++) cb[(size_t)t] = std::lower_bound(lp.begin(), lp.end(), nz * t / T) - lp.begin();
  for (int t = 1; t <= T; t++) cb[(size_t)t] = std::max(cb[(size_t)t], cb[(size_t)t - 1]);
  // 0. entries per row -> balanced warp row ranges per band
  std::unique_ptr<int32_t[]> rc(new int32_t[(size_t)std::max<int64_t>(1, c.m)]());
  run([&](int t) {
    for (int64_t z = lp[(size_t)cb[(size_t)t]]; z < lp[(size_t)cb[(size_t)t + 1]]; z++)
      __atomic_fetch_add(&rc[(size_t)rows[z]], 1, __ATOMIC_RELAXED);
  });
  constexpr int SW = CB_W + 1;
  B.split.assign((size_t)(B.nb * SW), 0);
  for (int64_t b = 0; b < B.nb; b++) {
    const int64_t r0 = b * CB_ROWS, nr = std::min<int64_t>(CB_ROWS, c.m - r0);
    int64_t tot = 0;
    for (int64_t o = 0; o < nr; o++) tot += rc[(size_t)(r0 + o)];
    int32_t* sp = &B.split[(size_t)(b * SW)];
    int64_t cum = 0, o = 0;
    for (int w = 1; w < CB_W; w++) {
      const int64_t target = tot * w / CB_W;
      while (o < nr && cum < target) cum += rc[(size_t)(r0 + o++)];
      sp[w] = (int32_t)o;
    }
    sp[0] = 0;
    sp[CB_W] = (int32_t)nr;
  }
  rc.reset();
  lapq(0);
  // warp owning each row (a byte per row): the sort below needs no search per entry
  std::unique_ptr<uint8_t[]> wl(new uint8_t[(size_t)std::max<int64_t>(1, c.m)]);
  run([&](int t) {
    for (int64_t b = B.nb * t / T; b < B.nb * (t + 1) / T; b++) {
      const int32_t* sp = &B.split[(size_t)(b * SW)];
      const int64_t r0 = b * CB_ROWS, nr = std::min<int64_t>(CB_ROWS, c.m - r0);
      int w = 0;
      for (int64_t o = 0; o < nr; o++) {
        while (w < CB_W - 1 && o >= sp[w + 1]) w++;
        wl[(size_t)(r0 + o)] = (uint8_t)w;
      }
    }
  });
  const int64_t nch = B.nch, chunk = B.chunk;
  // 1. stable counting sort by key = (band, column chunk, warp) into temporary (pk, val) arrays
  std::vector<std::vector<int64_t>> off((size_t)T, std::vector<int64_t>((size_t)keys, 0));
  run([&](int t) {
    int64_t* o = off[(size_t)t].data();
    for (int64_t q = cb[(size_t)t]; q < cb[(size_t)t + 1]; q++) {
      const int64_t qc = q / chunk;
      for (int64_t z = lp[(size_t)q]; z < lp[(size_t)q + 1]; z++) {
        const int32_t r = rows[z];
        o[(((int64_t)(r >> CB_LOG2)) * nch + qc) * CB_W + wl[(size_t)r]]++;
      }
    }
  });
  std::vector<int64_t> kbeg((size_t)keys + 1);
  int64_t run_off = 0;
  for (int64_t k = 0; k < keys; k++) {
    kbeg[(size_t)k] = run_off;
    for (int t = 0; t < T; t++) {
      const int64_t cnt = off[(size_t)t][(size_t)k];
      off[(size_t)t][(size_t)k] = run_off;
      run_off += cnt;
    }
  }
  kbeg[(size_t)keys] = run_off;
  // the scatter below writes ~1M random buckets: 2 MB pages cut its TLB misses
  HugeBuf tpk_b((size_t)std::max<int64_t>(1, nz) * 4), tval_b((size_t)std::max<int64_t>(1, nz) * V);
  uint32_t* tpk_p = static_cast<uint32_t*>(tpk_b.p);
  struct { uint32_t* p; uint32_t* get() const { return p; } uint32_t& operator[](size_t i) const { return p[i]; } } tpk{tpk_p};
  struct { char* p; char* get() const { return p; } } tval{static_cast<char*>(tval_b.p)};
  auto scatter = [&](auto vtag) {
    using VT = decltype(vtag);
    const VT* vv = reinterpret_cast<const VT*>(vals);
    VT* tv = reinterpret_cast<VT*>(tval.get());
    run([&](int t) {
      int64_t* o = off[(size_t)t].data();
      for (int64_t q = cb[(size_t)t]; q < cb[(size_t)t + 1]; q++) {
        const int64_t qc = q / chunk;
        const uint32_t qm = (uint32_t)(q - qc * chunk) << CB_LOG2;
        for (int64_t z = lp[(size_t)q]; z < lp[(size_t)q + 1]; z++) {
          const int32_t r = rows[z];
          const int64_t dst = o[(((int64_t)(r >> CB_LOG2)) * nch + qc) * CB_W + wl[(size_t)r]]++;
          tpk[(size_t)dst] = (uint32_t)(r & (CB_ROWS - 1)) | qm;
          tv[(size_t)dst] = vv[(size_t)z];
        }
      }
    });
  };
  if (V == 8) scatter(double{}); else scatter(float{});
  wl.reset();
  off.clear();
  off.shrink_to_fit();
  lapq(1);
  std::atomic<int64_t> next_key{0};
  auto each_key = [&](auto&& f) {
    run([&](int) {
      ArrangeScratch scratch;
      for (;;) {
        const int64_t k0 = next_key.fetch_add(64);
        if (k0 >= keys) break;
        for (int64_t k = k0; k < std::min(keys, k0 + 64); k++) f(k, scratch);
      }
    });
    next_key = 0;
  };
  // 2. arranged length of every list (holes included)
  std::vector<int64_t> alen((size_t)keys, 0), asame((size_t)keys, 0), aseg((size_t)keys, INT64_MAX);
  each_key([&](int64_t k, ArrangeScratch& scr) {
    const int64_t b0 = kbeg[(size_t)k], n = kbeg[(size_t)k + 1] - b0;
    scr.same = 0;
    alen[(size_t)k] = n ? arrange_list(tpk.get() + b0, n, scr, [](int64_t, int64_t) {}) : 0;
    asame[(size_t)k] = scr.same;
    aseg[(size_t)k] = scr.seg_from;
  });
  lapq(2);
  // 3. items: one per non-empty (band, chunk); stage geometry and blob offsets
  B.band_item.assign((size_t)B.nb + 1, 0);
  std::vector<int64_t> key_item((size_t)(B.nb * B.nch), -1);
  int64_t bytes = 0;
  for (int64_t b = 0; b < B.nb; b++) {
    B.band_item[(size_t)b] = (int32_t)B.items.size();
    for (int64_t ch = 0; ch < B.nch; ch++) {
      const int64_t k0 = (b * B.nch + ch) * CB_W;
      int64_t L = 0, H = 0;
      for (int w = 0; w < CB_W; w++) {
        L = std::max(L, alen[(size_t)(k0 + w)]);
        H = std::max(H, asame[(size_t)(k0 + w)]);
      }
      if (L == 0) continue;
      B.item_hst.push_back((int32_t)((H + CB_SEG - 1) / CB_SEG));
      for (int w = 0; w < CB_W; w++) B.item_hw.push_back((int32_t)(asame[(size_t)(k0 + w)] / 32));
      int64_t S0 = INT64_MAX;   // first stage that may hold segmented groups; per warp: first group
      for (int w = 0; w < CB_W; w++) {
        const int64_t a = aseg[(size_t)(k0 + w)] >= INT64_MAX - 1 ? INT64_MAX : aseg[(size_t)(k0 + w)];
        S0 = std::min(S0, a == INT64_MAX ? INT64_MAX : a / CB_SEG);
        B.item_sg.push_back(a == INT64_MAX ? INT32_MAX : (int32_t)(a / 32));
      }
      B.item_sst.push_back(S0 == INT64_MAX ? INT32_MAX : (int32_t)S0);
      const int64_t nst = (L + CB_SEG - 1) / CB_SEG;
      const int64_t last = ((L - (nst - 1) * CB_SEG) + 3) & ~(int64_t)3;
      if (nst >= ((int64_t)1 << 20)) return fail(MSREP_ERR_TOO_LARGE, "pCSC warp list too long (>= 2^20 stages)");
      key_item[(size_t)(b * B.nch + ch)] = (int64_t)B.items.size();
      B.items.push_back(make_int4((int32_t)b, (int32_t)nst, (int32_t)(ch * B.chunk), (int32_t)last));
      B.item_off.push_back(bytes);
      bytes += ((nst - 1) * CB_SEG + last) * CB_W * (int64_t)(V + 4);
    }
  }
  B.band_item[(size_t)B.nb] = (int32_t)B.items.size();
  B.bytes = bytes;
  // Units of work (fetched dynamically by the CTAs, largest first): a whole band, or -- for a band
  // heavier than `per` stages (R-MAT's first bands, short-wide matrices with fewer bands than SMs)
  // -- equal stage ranges of it, each parking its partial rows in a slot; the band's rows are then
  // reduced over its slots in slot order by the band's last unit to finish (deterministic).
  {
    std::vector<int64_t> st((size_t)B.nb, 0);
    int64_t tot = 0;
    for (int64_t b = 0; b < B.nb; b++) {
      for (int32_t i = B.band_item[(size_t)b]; i < B.band_item[(size_t)b + 1]; i++) st[(size_t)b] += B.items[(size_t)i].y;
      tot += st[(size_t)b];
    }
    // a band is split when it holds more than one SM's share of the stages (tot / sms), into
    // pieces of about half a share: with largest-first dynamic fetching the tail is then short
    const int64_t share = std::max<int64_t>(64, (tot + sms - 1) / sms);
    const int64_t per = std::max<int64_t>(16, share / MSREP_CB_PIECE_DIV), cut = share / MSREP_CB_SPLIT_DIV;
    B.bsplit.assign((size_t)B.nb, make_int2(0, 0));
    for (int64_t b = 0; b < B.nb; b++) {
      const int64_t sb = st[(size_t)b];
      const int64_t k = sb > cut ? (sb + per - 1) / per : 1;
      if (k == 1) { B.units.push_back(make_int4((int32_t)b, 0, (int32_t)sb, -1)); continue; }
      B.bsplit[(size_t)b] = make_int2((int32_t)B.nslots, (int32_t)k);
      for (int64_t q = 0; q < k; q++)
        B.units.push_back(make_int4((int32_t)b, (int32_t)(sb * q / k), (int32_t)(sb * (q + 1) / k), (int32_t)(B.nslots + q)));
      B.nslots += k;
    }
  }
  lapq(3);
  B.blob.reset(new char[(size_t)std::max<int64_t>(16, bytes)]);
  // 4. write every list into its item's stage blobs; pad it with holes to the item's length
  each_key([&](int64_t k, ArrangeScratch& scr) {
    const int64_t it = key_item[(size_t)(k / CB_W)];
    if (it < 0) return;
    const int w = (int)(k % CB_W);
    const int4 item = B.items[(size_t)it];
    const int64_t nst = item.y, last = item.w, L = (nst - 1) * CB_SEG + last;
    char* base = B.blob.get() + B.item_off[(size_t)it];
    const int64_t b0 = kbeg[(size_t)k], n = kbeg[(size_t)k + 1] - b0;
    auto put = [&](int64_t pos, int64_t e) {
      const int64_t s = pos / CB_SEG, j = pos % CB_SEG;
      const int64_t seg = s == nst - 1 ? last : CB_SEG;
      char* st = base + s * CB_SEG * CB_W * (int64_t)(V + 4);
      const int64_t slot = (int64_t)w * seg + j;
      uint32_t* pkp = reinterpret_cast<uint32_t*>(st + CB_W * seg * (int64_t)V) + slot;
      if (e >= 0) { *pkp = tpk[(size_t)(b0 + e)]; memcpy(st + slot * (int64_t)V, tval.get() + (size_t)(b0 + e) * V, V); }
      else { *pkp = CB_HOLE; memset(st + slot * (int64_t)V, 0, V); }
    };
    int64_t pos = n ? arrange_list(tpk.get() + b0, n, scr, put) : 0;
    for (; pos < L; pos++) put(pos, -1);
  });
  lapq(4);
  return MSREP_OK;
}

template <class T>
msrep_status_t upload_vec(Ctx* c, const std::vector<T>& v, T** out, cudaStream_t s) {
  return upload(c, v.data(), v.size(), out, s);
}

// Column formats on row tiles (MSREP_TUNE_COL_LAYOUT): the rank's nz_r entries [B_lo, B_hi) of a
// column format, transposed on the GPU into the rank-local row-major slice (transpose.cu):
//   pCSC               rows = idx, columns from the window-local column pointer lp
//   column-sorted pCOO rows = idx, columns = major (coo_row)
//   unsorted pCOO      rows = major (coo_row), columns = idx
// Column ids become window-local (col - c->wlo).  Outputs on the device (allocated here, after the
// caller's mark): t_cols / t_vals in row order and the int32 row pointer t_ptr [m + 1]; on the
// host the same pointer as int64 (lpr), for the tile schedule.  The inputs and sort buffers are
// freed before returning.
msrep_status_t transpose_slice(Ctx* c, msrep_format fmt, const std::vector<int64_t>& lp, const int32_t* idx,
                               const int32_t* coo_row, const void* val, size_t V, cudaStream_t s, int32_t** t_cols,
                               void** t_vals, int32_t** t_ptr, std::vector<int64_t>& lpr) {
  const int64_t nz = c->B_hi - c->B_lo, m = c->m;
  const size_t n1 = (size_t)std::max<int64_t>(1, nz);
  void* q;
  TRY(dalloc(c, n1 * 4, &q, s)); *t_cols = static_cast<int32_t*>(q);
  TRY(dalloc(c, n1 * V, &q, s)); *t_vals = q;
  TRY(dalloc(c, ((size_t)m + 1) * 4, &q, s)); *t_ptr = static_cast<int32_t*>(q);
  const size_t tmp_from = c->bufs.size();
  TransposeLaunch T{};
  T.n = nz; T.m = m; T.V = (int)V;
  int32_t *d_rows, *d_cols;
  const int32_t* rows_h = (fmt == MSREP_COO_UNSORTED ? coo_row : idx) + c->B_lo;
  TRY(upload(c, rows_h, (size_t)nz, &d_rows, s));
  TRY(dalloc(c, n1 * 4, &q, s)); d_cols = static_cast<int32_t*>(q);
  if (fmt == MSREP_CSC) {
    int64_t* d_lp;
    TRY(upload_vec(c, lp, &d_lp, s));
    CUDA_TRY(launch_expand_cols(d_lp, (int64_t)lp.size() - 1, d_cols, s));
  } else {
    const int32_t* cols_h = (fmt == MSREP_COO_UNSORTED ? idx : coo_row) + c->B_lo;
    TRY(h2d(c, d_cols, cols_h, (size_t)nz * 4, s));
    CUDA_TRY(launch_rebase_cols(d_cols, nz, (int32_t)c->wlo, d_cols, s));
  }
  void* d_vals;
  TRY(dalloc(c, n1 * V, &d_vals, s));
  TRY(h2d(c, d_vals, static_cast<const char*>(val) + (size_t)c->B_lo * V, (size_t)nz * V, s));
  uint32_t* sb[4];
  for (auto& b : sb) {
    TRY(dalloc(c, n1 * 4, &q, s));
    b = static_cast<uint32_t*>(q);
  }
  TRY(dalloc(c, (size_t)transpose_scratch_words(nz) * 4, &q, s));
  T.rows = reinterpret_cast<const uint32_t*>(d_rows);
  T.cols = d_cols;
  T.vals = d_vals;
  T.key_a = sb[0]; T.key_b = sb[1]; T.perm_a = sb[2]; T.perm_b = sb[3];
  T.scratch = static_cast<uint32_t*>(q);
  T.cols_out = *t_cols; T.vals_out = *t_vals; T.ptr_out = *t_ptr;
  CUDA_TRY(launch_transpose(T, s));
  std::vector<int32_t> p32((size_t)m + 1);
  CUDA_TRY(cudaMemcpyAsync(p32.data(), *t_ptr, ((size_t)m + 1) * 4, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  release_range(c, tmp_from, c->bufs.size());
  lpr.resize((size_t)m + 1);
  par_ranges(m + 1, [&](int64_t lo, int64_t hi) {
    for (int64_t r = lo; r < hi; r++) lpr[(size_t)r] = p32[(size_t)r];
  });
  return MSREP_OK;
}

ncclDataType_t nccl_type(msrep_dtype t) { return t == MSREP_F64 ? ncclDouble : ncclFloat; }

// ---- collectives of the merge: NCCL, or the loopback group (same buffer semantics)
// loopback phase 1: publish (src, dst) after this rank's work on s, wait for every peer's work
msrep_status_t loop_enter(Ctx* c, const void* src, void* dst, cudaStream_t s) {
  LoopGroup& G = *c->loop;
  CUDA_TRY(cudaEventRecord(G.ev1[(size_t)c->rank], s));
  G.src[(size_t)c->rank] = src;
  G.dst[(size_t)c->rank] = dst;
  G.barrier();
  for (int q = 0; q < G.n; q++)
    if (q != c->rank) CUDA_TRY(cudaStreamWaitEvent(s, G.ev1[(size_t)q], 0));
  return MSREP_OK;
}
// loopback phase 2: every rank has finished reading the peers' buffers before anyone goes on
msrep_status_t loop_leave(Ctx* c, cudaStream_t s) {
  LoopGroup& G = *c->loop;
  CUDA_TRY(cudaEventRecord(G.ev2[(size_t)c->rank], s));
  G.barrier();
  for (int q = 0; q < G.n; q++)
    if (q != c->rank) CUDA_TRY(cudaStreamWaitEvent(s, G.ev2[(size_t)q], 0));
  G.barrier();   // the slots may be republished by the next collective only after every wait above
  return MSREP_OK;
}
msrep_status_t loop_scratch(Ctx* c, size_t bytes, cudaStream_t s) {
  if (c->loop_scratch_bytes >= bytes) return MSREP_OK;
  void* p;
  TRY(dalloc(c, bytes, &p, s));
  c->d_loop_scratch = static_cast<double*>(p);
  c->loop_scratch_bytes = bytes;
  return MSREP_OK;
}
msrep_status_t reduce_peers(Ctx* c, const void* const* srcs, size_t elem_off, size_t count, void* dst, int is_int,
                            cudaStream_t s) {
  SumLaunch L{};
  L.n = c->nranks;
  for (int q = 0; q < c->nranks; q++) L.src[q] = srcs[q];
  L.off = (int64_t)elem_off;
  L.count = (int64_t)count;
  L.dst = dst;
  L.is_int = is_int;
  CUDA_TRY(launch_sum_peers(L, s));
  return MSREP_OK;
}

// recv[q*count .. (q+1)*count) = rank q's send (fp64)
msrep_status_t comm_allgather(Ctx* c, const double* send, double* recv, size_t count, cudaStream_t s) {
  if (!c->loop) {
    NCCL_TRY(ncclAllGather(send, recv, count, ncclDouble, c->comm, s));
    return MSREP_OK;
  }
  TRY(loop_enter(c, send, recv, s));
  for (int q = 0; q < c->nranks; q++)
    if (count) CUDA_TRY(cudaMemcpyAsync(recv + (size_t)q * count, c->loop->src[(size_t)q], count * 8, cudaMemcpyDeviceToDevice, s));
  return loop_leave(c, s);
}
// buf[rank*count .. (rank+1)*count) = sum over ranks of their buf segment (fp64 or fp32, in place)
msrep_status_t comm_reduce_scatter(Ctx* c, void* buf, size_t count, bool f32, cudaStream_t s) {
  const size_t E = f32 ? 4 : 8;
  char* mine = static_cast<char*>(buf) + (size_t)c->rank * count * E;
  if (!c->loop) {
    NCCL_TRY(ncclReduceScatter(buf, mine, count, f32 ? ncclFloat : ncclDouble, ncclSum, c->comm, s));
    return MSREP_OK;
  }
  TRY(loop_enter(c, buf, buf, s));
  // each rank writes only its own segment of its own buffer; peers read the other segments
  TRY(reduce_peers(c, c->loop->src.data(), (size_t)c->rank * count, count, mine, f32 ? 2 : 0, s));
  return loop_leave(c, s);
}
// buf = sum over ranks (in place; fp64 or int32)
msrep_status_t comm_allreduce(Ctx* c, void* buf, size_t count, bool is_int, cudaStream_t s) {
  if (!c->loop) {
    NCCL_TRY(ncclAllReduce(buf, buf, count, is_int ? ncclInt : ncclDouble, ncclSum, c->comm, s));
    return MSREP_OK;
  }
  TRY(loop_scratch(c, count * 8 + 16, s));
  TRY(loop_enter(c, buf, buf, s));
  TRY(reduce_peers(c, c->loop->src.data(), 0, count, c->d_loop_scratch, is_int ? 1 : 0, s));
  TRY(loop_leave(c, s));   // every peer has read this rank's buf: overwrite it now
  CUDA_TRY(cudaMemcpyAsync(buf, c->d_loop_scratch, count * (is_int ? 4 : 8), cudaMemcpyDeviceToDevice, s));
  return MSREP_OK;
}

// allgatherv of per-rank segments of y (in place), as grouped broadcasts.
msrep_status_t allgatherv_y(Ctx* c, void* y, const std::vector<int64_t>& lo, const std::vector<int64_t>& hi,
                            cudaStream_t s, int k = 1) {
  const size_t V = vsz(c->dtype);
  if (c->loop) {   // pull every peer's owned segment into this rank's y
    TRY(loop_enter(c, y, y, s));
    for (int r = 0; r < c->nranks; r++) {
      const int64_t cnt = (hi[(size_t)r] - lo[(size_t)r]) * k;
      if (r == c->rank || cnt <= 0) continue;
      const size_t off = (size_t)lo[(size_t)r] * k * V;
      CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(y) + off, static_cast<const char*>(c->loop->src[(size_t)r]) + off,
                               (size_t)cnt * V, cudaMemcpyDeviceToDevice, s));
    }
    return loop_leave(c, s);
  }
  NCCL_TRY(ncclGroupStart());
  for (int r = 0; r < c->nranks; r++) {
    const int64_t cnt = (hi[(size_t)r] - lo[(size_t)r]) * k;   // rows x k (row-major blocks)
    if (cnt <= 0) continue;
    char* p = static_cast<char*>(y) + (size_t)lo[(size_t)r] * k * V;
    NCCL_TRY(ncclBroadcast(p, p, (size_t)cnt, nccl_type(c->dtype), r, c->comm, s));
  }
  NCCL_TRY(ncclGroupEnd());
  return MSREP_OK;
}

void owned_segments(const Ctx* c, std::vector<int64_t>& lo, std::vector<int64_t>& hi) {
  rank_segments(c->fmt, c->m, c->nranks, c->vparts, c->parts, lo, hi);
}

double get_scalar(const void* p, msrep_dtype t) {
  return t == MSREP_F64 ? *static_cast<const double*>(p) : (double)*static_cast<const float*>(p);
}

}  // namespace

// ======================================================================= ABI
// smallest k in [0, n) with bad(k) != 0 (and that code), or -1
template <class F>
int64_t par_first_bad(int64_t n, int* code, F&& bad) {
  std::atomic<int64_t> first{INT64_MAX};
  par_ranges(n, [&](int64_t lo, int64_t hi) {
    for (int64_t k = lo; k < hi && k < first.load(std::memory_order_relaxed); k++)
      if (bad(k)) {
        int64_t cur = first.load();
        while (k < cur && !first.compare_exchange_weak(cur, k)) {}
        break;
      }
  });
  const int64_t k = first.load();
  if (k == INT64_MAX) return -1;
  *code = bad(k);
  return k;
}

// ------------------------------------------------ main-kernel launch descriptors
RowLaunch row_launch(const Ctx* c, const void* x, void* y, double alpha, double beta) {
  RowLaunch L{};
  L.tiles = c->d_tiles; L.ntiles = c->ntiles;
  L.blob = c->d_blob;
  L.x = static_cast<const char*>(x) + (size_t)c->xoff * vsz(c->dtype); L.y = y; L.ybase = c->ybase;
  L.xmax = c->xn > 0 ? (uint32_t)(c->xn - 1) : 0u;
  L.alpha = alpha; L.beta = beta; L.rec = c->d_rec;
  L.dtype = c->dtype == MSREP_F64 ? 0 : 1; L.has_sell = c->nsell > 0;
  L.xna = c->xna;
  L.hot = c->d_hot; L.nhot = c->nhot; L.hot_cluster = c->hot_cluster; L.sell_1cta = c->sell_1cta;
  if (c->nxc) { L.x = c->d_xc; L.xmax = (uint32_t)(c->nxc - 1); }   // the SpMV gathers x' first (prepare_x)
  return L;
}

// compact x: x' = x[xcols] (k-wide rows for SpMM) on s, before the tile kernel that reads it
msrep_status_t prepare_x(Ctx* c, const void* x, int k, cudaStream_t s) {
  if (!c->nxc) return MSREP_OK;
  void* dst = c->d_xc;
  if (k > 1) {
    if (!c->d_xc_mm) TRY(dalloc(c, (size_t)c->nxc * 8 * vsz(c->dtype), &c->d_xc_mm, s));
    dst = c->d_xc_mm;
  }
  CUDA_TRY(launch_gather_x(static_cast<const char*>(x) + (size_t)c->xoff * k * vsz(c->dtype), c->d_xcols, c->nxc, k, dst,
                           c->dtype == MSREP_F64 ? 0 : 1, s, c->d_xpos));
  return MSREP_OK;
}
ColLaunch col_launch(const Ctx* c, const void* x, void* y, double alpha, double beta) {
  ColLaunch L{};
  L.items = c->d_citems; L.item_off = c->d_item_off; L.band_item = c->d_band_item; L.split = c->d_split;
  L.nb = (int)c->cnb; L.blob = c->d_cblob;
  L.x = x; L.xbase = c->wlo;
  L.xs = 1; L.ys = 1;
  L.nunits = (int)c->cunits; L.units = c->d_cunits; L.bsplit = c->d_bsplit; L.slots = c->d_slots;
  L.tickets = c->d_tickets; L.ctr = c->d_ctr;
  L.item_hst = c->d_item_hst; L.item_hw = c->d_item_hw; L.item_sst = c->d_item_sst; L.item_sg = c->d_item_sg;
  L.fused = c->nranks == 1;
  L.out = L.fused ? y : static_cast<void*>(c->d_py);
  L.m = c->m; L.alpha = alpha; L.beta = beta; L.dtype = c->dtype == MSREP_F64 ? 0 : 1;
  L.xna = c->xna;
  return L;
}

// The device-resident tile walk: one launch, or (split_launch) the SELL tiles [0, nsell) with the
// SELL instantiation and the SEG / slab tiles with the SEG one (k = 1: SpMV, else SpMM).
msrep_status_t launch_row_tiles(Ctx* c, const RowLaunch& L, int k, cudaStream_t s) {
  auto run = [&](const RowLaunch& X, cudaStream_t st) { return k == 1 ? launch_rows(X, st) : launch_rows_mm(X, k, st); };
  if (!c->split_launch) {
    CUDA_TRY(run(L, s));
    return MSREP_OK;
  }
  // SELL tiles and SEG tiles in their own instantiations, forked onto a context side stream so the
  // two launches overlap (each one's tail fills with the other's CTAs) and joined back into s
  if (!c->ss) {
    CUDA_TRY(cudaStreamCreateWithFlags(&c->ss, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  }
  RowLaunch a = L, b = L;
  a.ntiles = c->nsell;
  b.tiles = L.tiles + c->nsell; b.ntiles = L.ntiles - c->nsell; b.has_sell = 0;
  CUDA_TRY(cudaEventRecord(c->ev_fork, s));
  CUDA_TRY(cudaStreamWaitEvent(c->ss, c->ev_fork, 0));
  CUDA_TRY(run(a, c->ss));
  CUDA_TRY(run(b, s));
  CUDA_TRY(cudaEventRecord(c->ev_join, c->ss));
  CUDA_TRY(cudaStreamWaitEvent(s, c->ev_join, 0));
  return MSREP_OK;
}

// x-gather L1 policy.  Whether the L1 should allocate the x lines depends on the matrix: gathers
// that neighbouring rows / warps of an SM re-hit (stencil pCOO, banded, block-diagonal, short-wide
// pCSC) want it; gathers with no reuse inside an SM (R-MAT, uniform random) are 5-6 % faster with
// L1::no_allocate (profiles/r1_xload_variants.txt, r1_suite_sweep.jsonl).  Both policies give
// identical bits, so the partition times the main kernel once with each on the built layout
// (dummy x = 0, y into scratch; 1 warm-up + 3 timed launches) and keeps the faster.
// msrep_set_tuning(MSREP_TUNE_XLOAD, 0|1) forces a policy.  Host-resident and small partitions (< 2^20 nonzeros)
// keep the allocating policy.
msrep_status_t tune_xload(Ctx* c, cudaStream_t s, int64_t nz_r) {
  c->sell_1cta = 0;
  if (c->tune_xload >= 0) { c->xna = c->tune_xload; return MSREP_OK; }
  c->xna = 0;
  if (c->residency == MSREP_RESIDENT_HOST || nz_r < ((int64_t)1 << 20)) return MSREP_OK;
  const size_t V = vsz(c->dtype), mark = c->bufs.size();
  void *dx, *dy;
  if (dalloc(c, (size_t)std::max<int64_t>(1, c->n) * V, &dx, s) != MSREP_OK ||
      dalloc(c, (size_t)std::max<int64_t>(1, c->m) * V, &dy, s) != MSREP_OK) {
    release_range(c, mark, c->bufs.size());   // no room for the probe vectors: keep the default policy
    return MSREP_OK;
  }
  CUDA_TRY(cudaMemsetAsync(dx, 0, (size_t)std::max<int64_t>(1, c->n) * V, s));
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  float best = 0.f;
  int pick = 0;
  // row layouts with SELL tiles also try one CTA per SM for the SELL launches: (policy, occupancy).
  // 2 warm-up + 6 timed launches each; a combination other than the default (allocate, 2 CTAs)
  // must win by 3 % (a noisy pick cost the CG stencil 15 %)
  const bool bands = colwise(c->fmt) && !c->col_rows;
  const int combos = (!bands && c->nsell > 0) ? 4 : 2;
  for (int cb = 0; cb < combos; cb++) {
    const int na = cb & 1;
    c->xna = na;
    c->sell_1cta = cb >> 1;
    float ms = 0.f;
    for (int it = 0; it < 8; it++) {
      if (it == 2) CUDA_TRY(cudaEventRecord(e0, s));
      if (bands) CUDA_TRY(launch_cols(col_launch(c, dx, dy, 1.0, 0.0), s));
      else TRY(launch_row_tiles(c, row_launch(c, dx, dy, 1.0, 0.0), 1, s));
    }
    CUDA_TRY(cudaEventRecord(e1, s));
    CUDA_TRY(cudaEventSynchronize(e1));
    CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    if (cb == 0 || ms < best * (pick == 0 ? 0.97f : 1.0f)) { best = ms; pick = cb; }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  c->xna = pick & 1;
  c->sell_1cta = pick >> 1;
  release_range(c, mark, c->bufs.size());
  return MSREP_OK;
}

// ------------------------------------------------ host-resident streaming
msrep_status_t ensure_copy_stream(Ctx* c) {
  if (c->cs) return MSREP_OK;
  CUDA_TRY(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&c->ev_go, &c->ev_copied[0], &c->ev_copied[1], &c->ev_free[0], &c->ev_free[1]})
    CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  return MSREP_OK;
}

// Stream the pinned layout through the two staging buffers: the copy of chunk k (copy stream)
// waits until the kernel of chunk k-2 (same buffer) has run; the kernel of chunk k (caller's
// stream) waits for its copy.  launch(chunk, base) enqueues on `s` with base = the staging
// buffer minus the chunk's layout offset, so layout offsets index it unchanged.
template <class F>
msrep_status_t stream_chunks(Ctx* c, cudaStream_t s, F&& launch) {
  CUDA_TRY(cudaEventRecord(c->ev_go, s));   // earlier work on s (previous calls' reads) is done first
  CUDA_TRY(cudaStreamWaitEvent(c->cs, c->ev_go, 0));
  for (size_t k = 0; k < c->chunks.size(); k++) {
    const auto& ch = c->chunks[k];
    const int b = (int)(k & 1);
    if (k >= 2) CUDA_TRY(cudaStreamWaitEvent(c->cs, c->ev_free[b], 0));
    CUDA_TRY(cudaMemcpyAsync(c->d_stage[b], c->h_blob + ch.off, (size_t)ch.bytes, cudaMemcpyHostToDevice, c->cs));
    CUDA_TRY(cudaEventRecord(c->ev_copied[b], c->cs));
    CUDA_TRY(cudaStreamWaitEvent(s, c->ev_copied[b], 0));
    TRY(launch(ch, static_cast<const char*>(c->d_stage[b]) - ch.off));
    CUDA_TRY(cudaEventRecord(c->ev_free[b], s));
  }
  return MSREP_OK;
}

msrep_status_t alloc_stages(Ctx* c, cudaStream_t s) {
  int64_t mx = 16;
  for (auto& ch : c->chunks) mx = std::max(mx, ch.bytes);
  for (int b = 0; b < 2; b++) {
    void* p;
    TRY(dalloc(c, (size_t)mx, &p, s));
    c->d_stage[b] = static_cast<char*>(p);
  }
  return MSREP_OK;
}

extern "C" {

const char* msrep_last_error(void) { return g_err.c_str(); }
int msrep_version(void) { return MSREP_VERSION_MAJOR * 100 + MSREP_VERSION_MINOR; }

msrep_status_t msrep_get_unique_id(uint8_t id[128]) {
  if (!id) return fail(MSREP_ERR_INVALID_ARG, "id is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  NCCL_TRY(ncclGetUniqueId(&u));
  memcpy(id, &u, 128);
  return MSREP_OK;
}

msrep_status_t msrep_plan_split(msrep_format fmt, msrep_split split, int64_t outer, int64_t nnz, int np,
                                const int64_t* ptr, const int32_t* coo_row, msrep_part_desc* parts_out) {
  if (np < 1 || outer < 0 || nnz < 0 || !parts_out) return fail(MSREP_ERR_INVALID_ARG, "bad plan arguments");
  if (split != MSREP_SPLIT_NNZ && split != MSREP_SPLIT_BLOCK) return fail(MSREP_ERR_INVALID_ARG, "unknown split %d", (int)split);
  std::vector<int64_t> b;
  if (fmt == MSREP_COO_UNSORTED) {   // positions only; coo_row = the row of each triplet
    if (nnz > 0 && !coo_row) return fail(MSREP_ERR_INVALID_ARG, "unsorted COO plan needs row_idx");
    if (split != MSREP_SPLIT_NNZ) return fail(MSREP_ERR_INVALID_ARG, "unsorted COO takes the nnz split only");
    split_bounds(fmt, split, outer, nnz, np, nullptr, nullptr, b);
    plan_coo_unsorted(np, coo_row, b, parts_out);
  } else if (coo_like(fmt)) {
    if (nnz > 0 && !coo_row) return fail(MSREP_ERR_INVALID_ARG, "COO plan needs its sorted major index");
    split_bounds(fmt, split, outer, nnz, np, nullptr, coo_row, b);
    plan_coo(outer, np, coo_row, b, parts_out);
  } else if (fmt == MSREP_CSR || fmt == MSREP_CSC) {
    if (!ptr) return fail(MSREP_ERR_INVALID_ARG, "plan needs ptr");
    if (ptr[0] != 0 || ptr[outer] != nnz) return fail(MSREP_ERR_DIM_MISMATCH, "ptr[0] != 0 or ptr[outer] != nnz");
    split_bounds(fmt, split, outer, nnz, np, ptr, nullptr, b);
    plan_ptr(outer, np, ptr, b, parts_out);
  } else {
    return fail(MSREP_ERR_INVALID_ARG, "unknown format %d", (int)fmt);
  }
  return MSREP_OK;
}

msrep_status_t msrep_plan(msrep_format fmt, int64_t outer, int64_t nnz, int np, const int64_t* ptr,
                          const int32_t* coo_row, msrep_part_desc* parts_out) {
  return msrep_plan_split(fmt, MSREP_SPLIT_NNZ, outer, nnz, np, ptr, coo_row, parts_out);
}

msrep_status_t msrep_plan_groups(msrep_format fmt, int64_t outer, int64_t nnz, int ngroups, const int* parts_per_group,
                                 const int64_t* ptr, const int32_t* coo_row, msrep_part_desc* parts_out) {
  if (ngroups < 1 || !parts_per_group || outer < 0 || nnz < 0 || !parts_out)
    return fail(MSREP_ERR_INVALID_ARG, "bad two-level plan arguments");
  std::vector<int> g(parts_per_group, parts_per_group + ngroups);
  int np = 0;
  for (int v : g) {
    if (v < 1) return fail(MSREP_ERR_INVALID_ARG, "a group has %d parts", v);
    np += v;
  }
  std::vector<int64_t> b;
  if (coo_like(fmt)) {
    if (nnz > 0 && !coo_row) return fail(MSREP_ERR_INVALID_ARG, "COO plan needs its sorted major index");
    split_bounds(fmt, MSREP_SPLIT_TWO_LEVEL, outer, nnz, np, nullptr, coo_row, b, &g);
    plan_coo(outer, np, coo_row, b, parts_out);
  } else if (fmt == MSREP_CSR || fmt == MSREP_CSC) {
    if (!ptr) return fail(MSREP_ERR_INVALID_ARG, "plan needs ptr");
    if (ptr[0] != 0 || ptr[outer] != nnz) return fail(MSREP_ERR_DIM_MISMATCH, "ptr[0] != 0 or ptr[outer] != nnz");
    split_bounds(fmt, MSREP_SPLIT_TWO_LEVEL, outer, nnz, np, ptr, nullptr, b, &g);
    plan_ptr(outer, np, ptr, b, parts_out);
  } else {
    return fail(MSREP_ERR_INVALID_ARG, "unknown format %d", (int)fmt);
  }
  return MSREP_OK;
}

msrep_status_t msrep_set_split_groups(msrep_ctx h, int ngroups, const int* parts_per_group) {
  if (!h) return fail(MSREP_ERR_INVALID_ARG, "ctx is NULL");
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (ngroups < 1 || !parts_per_group) return fail(MSREP_ERR_INVALID_ARG, "bad groups");
  int np = 0;
  for (int i = 0; i < ngroups; i++) {
    if (parts_per_group[i] < 1) return fail(MSREP_ERR_INVALID_ARG, "group %d has %d parts", i, parts_per_group[i]);
    np += parts_per_group[i];
  }
  if (np != c->np) return fail(MSREP_ERR_INVALID_ARG, "groups hold %d parts, the context has %d", np, c->np);
  c->groups.assign(parts_per_group, parts_per_group + ngroups);
  c->split = MSREP_SPLIT_TWO_LEVEL;
  return MSREP_OK;
}

msrep_status_t msrep_set_tuning(msrep_ctx h, msrep_tuning knob, int value) {
  if (!h) return fail(MSREP_ERR_INVALID_ARG, "ctx is NULL");
  Ctx* c = reinterpret_cast<Ctx*>(h);
  switch (knob) {
    case MSREP_TUNE_XLOAD:
      if (value < -1 || value > 1) return fail(MSREP_ERR_INVALID_ARG, "MSREP_TUNE_XLOAD %d (-1, 0, 1)", value);
      c->tune_xload = value;
      return MSREP_OK;
    case MSREP_TUNE_CG_GRAPH:
      if (value < 0 || value > 1) return fail(MSREP_ERR_INVALID_ARG, "MSREP_TUNE_CG_GRAPH %d (0, 1)", value);
      c->tune_cg_graph = value;
      return MSREP_OK;
    case MSREP_TUNE_COMPACT_X:
      if (value < -1 || value > 2) return fail(MSREP_ERR_INVALID_ARG, "MSREP_TUNE_COMPACT_X %d (-1, 0, 1, 2)", value);
      c->tune_compact = value;
      return MSREP_OK;
    case MSREP_TUNE_HOT_CLUSTER:
      if (value != 1 && value != 2) return fail(MSREP_ERR_INVALID_ARG, "MSREP_TUNE_HOT_CLUSTER %d (1, 2)", value);
      c->tune_hot_cluster = value;
      return MSREP_OK;
    case MSREP_TUNE_SELL:
      if (value < 0 || value > 2) return fail(MSREP_ERR_INVALID_ARG, "MSREP_TUNE_SELL %d (0, 1, 2)", value);
      c->tune_sell = value;
      return MSREP_OK;
    case MSREP_TUNE_COL_LAYOUT:
      if (value < -1 || value > 1) return fail(MSREP_ERR_INVALID_ARG, "MSREP_TUNE_COL_LAYOUT %d (-1, 0, 1)", value);
      c->tune_col_layout = value;
      return MSREP_OK;
    case MSREP_TUNE_HOT_X:
      if (value < -1 || value > HOT_BYTES / 1024)
        return fail(MSREP_ERR_INVALID_ARG, "MSREP_TUNE_HOT_X %d (-1, 0, 1, or 2..%d KiB)", value, HOT_BYTES / 1024);
      c->tune_hot = value;
      return MSREP_OK;
  }
  return fail(MSREP_ERR_INVALID_ARG, "unknown tuning knob %d", (int)knob);
}

msrep_status_t msrep_set_split(msrep_ctx h, msrep_split split) {
  if (!h) return fail(MSREP_ERR_INVALID_ARG, "ctx is NULL");
  if (split != MSREP_SPLIT_NNZ && split != MSREP_SPLIT_BLOCK)
    return fail(MSREP_ERR_INVALID_ARG, "split %d (use msrep_set_split_groups for the two-level split)", (int)split);
  reinterpret_cast<Ctx*>(h)->split = split;
  return MSREP_OK;
}

msrep_status_t msrep_debug_arrange(const uint32_t* pk, int64_t n, int64_t* order_out, int64_t cap, int64_t* len_out,
                                   int64_t* same_out, int64_t* seg_from_out) {
  if (n < 0 || (n > 0 && !pk) || !len_out || !same_out || !seg_from_out || (cap > 0 && !order_out))
    return fail(MSREP_ERR_INVALID_ARG, "bad msrep_debug_arrange arguments");
  ArrangeScratch A;
  std::vector<int64_t> out;
  const int64_t len = n ? arrange_list(pk, n, A, [&](int64_t pos, int64_t e) {
    if ((int64_t)out.size() <= pos) out.resize((size_t)pos + 1, -1);
    out[(size_t)pos] = e;
  }) : 0;
  if (len > cap) return fail(MSREP_ERR_INVALID_ARG, "cap %lld < arranged length %lld", (long long)cap, (long long)len);
  for (int64_t i = 0; i < len; i++) order_out[i] = i < (int64_t)out.size() ? out[(size_t)i] : -1;
  *len_out = len;
  *same_out = A.same;
  *seg_from_out = A.seg_from >= INT64_MAX - 1 ? -1 : A.seg_from;
  return MSREP_OK;
}

msrep_status_t msrep_set_residency(msrep_ctx h, msrep_residency residency, int64_t chunk_bytes) {
  if (!h) return fail(MSREP_ERR_INVALID_ARG, "ctx is NULL");
  if (residency != MSREP_RESIDENT_DEVICE && residency != MSREP_RESIDENT_HOST)
    return fail(MSREP_ERR_INVALID_ARG, "residency %d", (int)residency);
  if (chunk_bytes < 0) return fail(MSREP_ERR_INVALID_ARG, "chunk_bytes < 0");
  Ctx* c = reinterpret_cast<Ctx*>(h);
  c->residency = residency;
  c->chunk_bytes = chunk_bytes ? chunk_bytes : (int64_t)256 << 20;
  return MSREP_OK;
}

msrep_status_t msrep_exchange_plan(msrep_format fmt, msrep_split split, int64_t m, int64_t n, int64_t nnz,
                                   int nranks, int parts_per_rank, const int64_t* ptr, const int32_t* coo_row,
                                   int64_t* seg_out, int64_t* head_row_out, int32_t* head_part_out) {
  if (nranks < 1 || parts_per_rank < 1 || m < 0 || n < 0 || nnz < 0 || !seg_out)
    return fail(MSREP_ERR_INVALID_ARG, "bad exchange-plan arguments");
  const int np = nranks * parts_per_rank;
  const int64_t outer = colwise(fmt) ? n : m;
  std::vector<msrep_part_desc> parts((size_t)np);
  TRY(msrep_plan_split(fmt, split, outer, nnz, np, ptr, coo_row, parts.data()));
  std::vector<int64_t> lo, hi;
  rank_segments(fmt, m, nranks, parts_per_rank, parts, lo, hi);
  for (int r = 0; r < nranks; r++) { seg_out[2 * r] = lo[(size_t)r]; seg_out[2 * r + 1] = hi[(size_t)r]; }
  std::vector<int64_t> hrow((size_t)np, -1);
  std::vector<int32_t> hpart((size_t)np, -1);
  if (!colwise(fmt)) {
    std::vector<int32_t> chain;
    for (int j = 0; j < np; j++) {
      tail_chain(parts, j, chain);
      for (int32_t q : chain) { hrow[(size_t)q] = parts[(size_t)j].owned_end - 1; hpart[(size_t)q] = j; }
    }
    for (int q = 0; q < np; q++)
      if (parts[(size_t)q].start_idx <= parts[(size_t)q].end_idx && parts[(size_t)q].start_flag && hpart[(size_t)q] < 0)
        return fail(MSREP_ERR_STATE, "internal: head of part %d has no owner", q);
  }
  if (head_row_out) memcpy(head_row_out, hrow.data(), hrow.size() * sizeof(int64_t));
  if (head_part_out) memcpy(head_part_out, hpart.data(), hpart.size() * sizeof(int32_t));
  return MSREP_OK;
}

msrep_status_t msrep_create(msrep_ctx* out, int rank, int nranks, const uint8_t id[128], int device,
                            int parts_per_rank, const msrep_allocator* alloc) {
  if (!out) return fail(MSREP_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks || parts_per_rank < 1)
    return fail(MSREP_ERR_INVALID_ARG, "bad rank %d / nranks %d / parts_per_rank %d", rank, nranks, parts_per_rank);
  if (nranks > 1 && !id) return fail(MSREP_ERR_INVALID_ARG, "nranks > 1 needs an NCCL unique id");
  if (alloc && (!alloc->alloc || !alloc->free)) return fail(MSREP_ERR_INVALID_ARG, "allocator needs alloc and free");
  CUDA_TRY(cudaSetDevice(device));
  Ctx* c = new Ctx();
  c->rank = rank;
  c->nranks = nranks;
  c->vparts = parts_per_rank;
  c->np = nranks * parts_per_rank;
  c->device = device;
  c->numa_node = gpu_numa_node(device);
  if (alloc) { c->alloc = *alloc; c->has_alloc = true; }
  if (nranks > 1) {
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclResult_t r = ncclCommInitRank(&c->comm, nranks, u, rank);
    if (r != ncclSuccess) {
      delete c;
      return fail(MSREP_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
  }
  *out = reinterpret_cast<msrep_ctx>(c);
  return MSREP_OK;
}

msrep_status_t msrep_create_loopback(msrep_ctx* out, int nranks, int device, int parts_per_rank) {
  if (!out) return fail(MSREP_ERR_INVALID_ARG, "out is NULL");
  if (nranks < 1 || nranks > MAX_LOOP_RANKS || parts_per_rank < 1)
    return fail(MSREP_ERR_INVALID_ARG, "nranks %d (1..%d) / parts_per_rank %d", nranks, MAX_LOOP_RANKS, parts_per_rank);
  for (int r = 0; r < nranks; r++) out[r] = nullptr;
  CUDA_TRY(cudaSetDevice(device));
  auto G = std::make_shared<LoopGroup>();
  G->n = nranks;
  G->src.assign((size_t)nranks, nullptr);
  G->dst.assign((size_t)nranks, nullptr);
  G->ev1.assign((size_t)nranks, nullptr);
  G->ev2.assign((size_t)nranks, nullptr);
  for (int r = 0; r < nranks; r++) {
    CUDA_TRY(cudaEventCreateWithFlags(&G->ev1[(size_t)r], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&G->ev2[(size_t)r], cudaEventDisableTiming));
  }
  for (int r = 0; r < nranks; r++) {
    Ctx* c = new Ctx();
    c->rank = r;
    c->nranks = nranks;
    c->vparts = parts_per_rank;
    c->np = nranks * parts_per_rank;
    c->device = device;
    c->numa_node = gpu_numa_node(device);
    c->loop = G;
    out[r] = reinterpret_cast<msrep_ctx>(c);
  }
  return MSREP_OK;
}

msrep_status_t msrep_destroy(msrep_ctx h) {
  if (!h) return MSREP_OK;
  Ctx* c = reinterpret_cast<Ctx*>(h);
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  free_all(c);
  for (auto& p : c->ev) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
  if (c->cs) cudaStreamDestroy(c->cs);
  if (c->cs_in) cudaStreamDestroy(c->cs_in);
  if (c->cs_out) cudaStreamDestroy(c->cs_out);
  for (cudaEvent_t e : c->hev) if (e) cudaEventDestroy(e);
  if (c->gs) cudaStreamDestroy(c->gs);
  if (c->ss) cudaStreamDestroy(c->ss);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  for (int b = 0; b < 2; b++) {
    if (c->h_ring[b]) cudaFreeHost(c->h_ring[b]);
    if (c->ring_ev[b]) cudaEventDestroy(c->ring_ev[b]);
  }
  for (cudaEvent_t e : {c->ev_go, c->ev_copied[0], c->ev_copied[1], c->ev_free[0], c->ev_free[1]})
    if (e) cudaEventDestroy(e);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->loop && c->loop.use_count() == 1) {   // the group's last context
    for (auto e : c->loop->ev1) if (e) cudaEventDestroy(e);
    for (auto e : c->loop->ev2) if (e) cudaEventDestroy(e);
  }
  delete c;
  return MSREP_OK;
}

msrep_status_t msrep_partition(msrep_ctx h, msrep_format fmt, msrep_dtype dtype, int64_t m, int64_t n, int64_t nnz,
                               const int64_t* ptr, const int32_t* idx, const int32_t* coo_row, const void* val,
                               msrep_part_desc* parts_out, void* stream) {
  if (!h) return fail(MSREP_ERR_INVALID_ARG, "ctx is NULL");
  Ctx* c = reinterpret_cast<Ctx*>(h);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Nvtx nv_all("msrep_partition");
  const auto t0 = std::chrono::steady_clock::now();
  double phase[4] = {0, 0, 0, 0};
  static const char* kPhase[4] = {"partition: validate", "partition: plan", "partition: schedule", "partition: upload+pack"};
  auto tl = t0;
  NvtxSeq nv_phase;
  nv_phase.next(kPhase[0]);
  auto lap = [&](int k) {
    const auto now = std::chrono::steady_clock::now();
    phase[k] += std::chrono::duration<double, std::milli>(now - tl).count();
    tl = now;
    nv_phase.next(kPhase[k == 3 ? 3 : k + 1]);
  };
  // ---- validation (before any device work)
  if (fmt != MSREP_CSR && fmt != MSREP_CSC && fmt != MSREP_COO && fmt != MSREP_COO_COL && fmt != MSREP_COO_UNSORTED)
    return fail(MSREP_ERR_INVALID_ARG, "format %d", (int)fmt);
  if (fmt == MSREP_COO_UNSORTED && c->split == MSREP_SPLIT_BLOCK)
    return fail(MSREP_ERR_INVALID_ARG, "unsorted COO has no row blocks: use the nnz (or two-level) split");
  if (dtype != MSREP_F64 && dtype != MSREP_F32) return fail(MSREP_ERR_INVALID_ARG, "dtype %d", (int)dtype);
  if (m < 0 || n < 0 || nnz < 0) return fail(MSREP_ERR_INVALID_ARG, "negative dimension");
  if (m >= kMaxIdx || n >= kMaxIdx) return fail(MSREP_ERR_TOO_LARGE, "m, n must be < 2^31");
  if (nnz > 0 && (!idx || !val)) return fail(MSREP_ERR_INVALID_ARG, "idx/val NULL");
  const int64_t outer = colwise(fmt) ? n : m, inner = colwise(fmt) ? m : n;
  if (fmt == MSREP_COO_UNSORTED) {   // any order: only the index ranges are checked
    if (nnz > 0 && !coo_row) return fail(MSREP_ERR_INVALID_ARG, "unsorted COO needs row_idx (coo_row)");
    int code = 0;
    const int64_t k = par_first_bad(nnz, &code, [&](int64_t q) -> int {
      return (coo_row[q] < 0 || coo_row[q] >= m) ? 1 : ((idx[q] < 0 || idx[q] >= n) ? 2 : 0);
    });
    if (k >= 0) return fail(MSREP_ERR_DIM_MISMATCH, "%s index [%lld] out of range", code == 1 ? "row" : "column", (long long)k);
  } else if (coo_like(fmt)) {
    if (nnz > 0 && !coo_row) return fail(MSREP_ERR_INVALID_ARG, "COO needs its sorted major index (coo_row)");
    const char* what = fmt == MSREP_COO ? "(row, col)" : "(col, row)";
    int code = 0;
    const int64_t k = par_first_bad(nnz, &code, [&](int64_t q) -> int {
      if (coo_row[q] < 0 || coo_row[q] >= outer) return 1;
      if (q > 0 && (coo_row[q] < coo_row[q - 1] || (coo_row[q] == coo_row[q - 1] && idx[q] < idx[q - 1]))) return 2;
      return 0;
    });
    if (k >= 0 && code == 1) return fail(MSREP_ERR_DIM_MISMATCH, "major index [%lld] out of range", (long long)k);
    if (k >= 0) return fail(MSREP_ERR_UNSORTED_COO, "COO not sorted by %s at %lld", what, (long long)k);
  } else {
    if (!ptr) return fail(MSREP_ERR_INVALID_ARG, "ptr NULL");
    if (ptr[0] != 0 || ptr[outer] != nnz) return fail(MSREP_ERR_DIM_MISMATCH, "ptr[0] != 0 or ptr[%lld] != nnz", (long long)outer);
    int code = 0;
    const int64_t r = par_first_bad(outer, &code, [&](int64_t q) -> int { return ptr[q + 1] < ptr[q] ? 1 : 0; });
    if (r >= 0) return fail(MSREP_ERR_DIM_MISMATCH, "ptr decreases at %lld", (long long)r);
  }
  lap(0);
  std::vector<msrep_part_desc> parts((size_t)c->np);
  std::vector<int64_t> bnd;
  split_bounds(fmt, c->split, outer, nnz, c->np, ptr, coo_row, bnd, &c->groups);
  if (fmt == MSREP_COO_UNSORTED) plan_coo_unsorted(c->np, coo_row, bnd, parts.data());
  else if (coo_like(fmt)) plan_coo(outer, c->np, coo_row, bnd, parts.data());
  else plan_ptr(outer, c->np, ptr, bnd, parts.data());
  lap(1);
  const int P0 = c->rank * c->vparts, P1 = P0 + c->vparts;
  const int64_t B_lo = bnd[(size_t)P0], B_hi = bnd[(size_t)P1];
  if (B_hi - B_lo >= kMaxRankNnz) return fail(MSREP_ERR_TOO_LARGE, "rank holds %lld nonzeros (>= 2^31 - 2^16)", (long long)(B_hi - B_lo));
  {
    int code = 0;
    const int64_t k = fmt == MSREP_COO_UNSORTED ? -1 : par_first_bad(B_hi - B_lo, &code, [&](int64_t q) -> int {
      return (idx[B_lo + q] < 0 || idx[B_lo + q] >= inner) ? 1 : 0;
    });   // (unsorted COO: both indices were range-checked above)
    if (k >= 0) return fail(MSREP_ERR_DIM_MISMATCH, "index %lld out of range", (long long)(B_lo + k));
  }
  lap(0);

  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(s));
  free_all(c);
  c->fmt = fmt; c->dtype = dtype; c->m = m; c->n = n; c->nnz = nnz;
  c->parts = parts;
  c->P0 = P0; c->P1 = P1; c->B_lo = B_lo; c->B_hi = B_hi;
  c->any_flag = false;
  for (auto& d : parts) c->any_flag |= (d.start_flag != 0);
  if (parts_out) memcpy(parts_out, parts.data(), parts.size() * sizeof(msrep_part_desc));

  // ---- window and local pointer (clamped form of Alg. 2 l.11-12, reading R5)
  const size_t V = vsz(dtype);
  std::vector<int64_t> lp;
  // column formats: row tiles over the slice transposed on the GPU, or the host-built row bands
  const bool col_rows = colwise(fmt) && c->tune_col_layout != 0;
  c->col_rows = col_rows;
  c->ybase = 0;
  c->xoff = 0;
  c->xn = n;
  c->py_f32 = false;
  // unsorted COO (row bands): this rank's triplets, stably counting-sorted by column, are a
  // column-sorted COO slice; from here on the rank builds the same band layout as MSREP_COO_COL
  // (the partial y of its parts spans the matrix and is merged column-style).
  // On row tiles the triplets go to the GPU transposition as they are (triplet order within a row).
  std::vector<int32_t> us_col, us_row;
  std::unique_ptr<char[]> us_val;
  if (fmt == MSREP_COO_UNSORTED && !col_rows) {
    const int64_t nzr = B_hi - B_lo;
    int64_t cmin = n, cmax = -1;
    for (int64_t k = B_lo; k < B_hi; k++) { cmin = std::min<int64_t>(cmin, idx[k]); cmax = std::max<int64_t>(cmax, idx[k]); }
    us_col.resize((size_t)nzr);
    us_row.resize((size_t)nzr);
    us_val.reset(new char[(size_t)std::max<int64_t>(1, nzr) * V]);
    if (nzr > 0) {
      std::vector<int64_t> cnt((size_t)(cmax - cmin + 2), 0);
      for (int64_t k = B_lo; k < B_hi; k++) cnt[(size_t)(idx[k] - cmin + 1)]++;
      for (size_t q = 1; q < cnt.size(); q++) cnt[q] += cnt[q - 1];
      for (int64_t k = B_lo; k < B_hi; k++) {
        const int64_t d = cnt[(size_t)(idx[k] - cmin)]++;
        us_col[(size_t)d] = idx[k];
        us_row[(size_t)d] = coo_row[k];
        memcpy(us_val.get() + (size_t)d * V, static_cast<const char*>(val) + (size_t)k * V, V);
      }
    }
    // global-position views: position B_lo + q of the views is element q of the sorted slice
    coo_row = reinterpret_cast<const int32_t*>(reinterpret_cast<uintptr_t>(us_col.data()) - (uintptr_t)B_lo * 4);
    idx = reinterpret_cast<const int32_t*>(reinterpret_cast<uintptr_t>(us_row.data()) - (uintptr_t)B_lo * 4);
    val = reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(us_val.get()) - (uintptr_t)B_lo * V);
    fmt = MSREP_COO_COL;   // the rank's layout (c->fmt keeps MSREP_COO_UNSORTED)
  }
  if (colwise(fmt)) {
    int64_t lo = -1, hi = -1;
    if (c->fmt == MSREP_COO_UNSORTED && !col_rows) {   // the column window of the sorted slice
      if (B_hi > B_lo) { lo = coo_row[B_lo]; hi = (int64_t)coo_row[B_hi - 1] + 1; }
    } else if (c->fmt == MSREP_COO_UNSORTED) {   // the column window of the triplets
      std::mutex mu;
      int64_t cmin = n, cmax = -1;
      par_ranges(B_hi - B_lo, [&](int64_t a, int64_t b) {
        int64_t l = n, h = -1;
        for (int64_t k = B_lo + a; k < B_lo + b; k++) { l = std::min<int64_t>(l, idx[k]); h = std::max<int64_t>(h, idx[k]); }
        std::lock_guard<std::mutex> g(mu);
        cmin = std::min(cmin, l);
        cmax = std::max(cmax, h);
      });
      if (cmax >= 0) { lo = cmin; hi = cmax + 1; }
    } else {
      for (int j = P0; j < P1; j++) {
        if (parts[(size_t)j].start_idx > parts[(size_t)j].end_idx) continue;
        if (lo < 0) lo = parts[(size_t)j].start_row;
        hi = parts[(size_t)j].end_row + 1;
      }
    }
    if (lo < 0) lo = hi = 0;
    c->wlo = lo; c->whi = hi;
    c->own_lo = c->own_hi = 0;
    c->shard = (m + c->nranks - 1) / c->nranks;
  } else {
    int64_t lo = parts[(size_t)P0].owned_begin;
    for (int j = P0; j < P1; j++) {
      const auto& d = parts[(size_t)j];
      if (d.start_idx <= d.end_idx && d.start_flag) lo = std::min(lo, d.start_row);
    }
    c->wlo = lo;
    c->whi = parts[(size_t)P1 - 1].owned_end;
    c->own_lo = parts[(size_t)P0].owned_begin;
    c->own_hi = parts[(size_t)P1 - 1].owned_end;
  }
  const int64_t W = c->whi - c->wlo;
  if (col_rows && coo_like(fmt)) {
    // no local pointer: the transposition reads the column of every entry
  } else if (coo_like(fmt)) {
    lp.resize((size_t)W + 1);
    // local pointer of a sorted major index: lp[w] = first rank-local k with coo_row >= wlo + w;
    // every row is written by the thread whose range holds the first nonzero at or after it
    const int64_t nzr = B_hi - B_lo;
    const int32_t* cr = coo_row + B_lo;
    par_ranges(nzr, [&](int64_t lo, int64_t hi) {
      for (int64_t k = lo; k < hi; k++) {
        const int64_t prev = k == 0 ? c->wlo - 1 : (int64_t)cr[k - 1];
        for (int64_t r = prev + 1; r <= (int64_t)cr[k]; r++) lp[(size_t)(r - c->wlo)] = k;
      }
    });
    const int64_t last = nzr ? (int64_t)cr[nzr - 1] - c->wlo + 1 : 0;
    for (int64_t w = last; w <= W; w++) lp[(size_t)w] = nzr;
  } else {
    lp.resize((size_t)W + 1);
    for (int64_t w = 0; w <= W; w++) {
      int64_t v = ptr[c->wlo + w];
      lp[(size_t)w] = std::min(std::max(v, B_lo), B_hi) - B_lo;
    }
  }

  const int64_t nz_r = B_hi - B_lo;
  lap(1);
  double layout_ms[6] = {0, 0, 0, 0, 0, 0};   // sub-steps of the layout build (stats.layout_ms)
  auto ts = std::chrono::steady_clock::now();
  auto sub = [&](int k) {
    const auto now = std::chrono::steady_clock::now();
    layout_ms[k] += std::chrono::duration<double, std::milli>(now - ts).count();
    ts = now;
  };
  if (colwise(fmt) && !col_rows) {
    // ---- pCSC: row-band layout built on the host threads, uploaded once
    CscBands CB;
    int sms = 148;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    TRY(build_csc_bands(*c, lp, idx, val, V, sms, CB));
    for (int k = 0; k < 5; k++) layout_ms[k] = g_csc_ms[k];
    lap(2);
    TRY(upload_vec(c, CB.items, &c->d_citems, s));
    TRY(upload_vec(c, CB.item_hst, &c->d_item_hst, s));
    TRY(upload_vec(c, CB.item_hw, &c->d_item_hw, s));
    TRY(upload_vec(c, CB.item_sst, &c->d_item_sst, s));
    TRY(upload_vec(c, CB.item_sg, &c->d_item_sg, s));
    TRY(upload_vec(c, CB.item_off, &c->d_item_off, s));
    TRY(upload_vec(c, CB.band_item, &c->d_band_item, s));
    TRY(upload_vec(c, CB.split, &c->d_split, s));
    // units in band order -> chunk ranges (host-resident: runs of whole bands) -> largest first
    // inside each chunk (the CTAs fetch them in list order)
    std::vector<std::pair<int64_t, int64_t>> uranges;
    if (c->residency == MSREP_RESIDENT_HOST) {
      // park the band blobs in pinned memory; chunks = runs of whole bands of <= chunk_bytes
      CUDA_TRY(host_alloc_on(reinterpret_cast<void**>(&c->h_blob), (size_t)std::max<int64_t>(16, CB.bytes), c->numa_node));
      {
        char* hb = c->h_blob;
        const char* sb = CB.blob.get();
        par_ranges(CB.bytes, [&](int64_t lo, int64_t hi) { memcpy(hb + lo, sb + lo, (size_t)(hi - lo)); });
      }
      c->h_bytes = CB.bytes;
      auto band_off = [&](int64_t b) {
        const int32_t i = CB.band_item[(size_t)b];
        return i < (int32_t)CB.items.size() ? CB.item_off[(size_t)i] : CB.bytes;
      };
      size_t u = 0;
      for (int64_t b = 0; b < CB.nb;) {
        const int64_t off0 = band_off(b);
        int64_t e = b + 1;
        while (e < CB.nb && band_off(e + 1) - off0 <= c->chunk_bytes) e++;
        Ctx::Chunk ch{(int32_t)b, (int32_t)e, (int32_t)u, 0, off0, band_off(e) - off0, false};
        while (u < CB.units.size() && CB.units[u].x < e) u++;
        ch.u1 = (int32_t)u;
        c->chunks.push_back(ch);
        uranges.push_back({ch.u0, ch.u1});
        b = e;
      }
      c->d_cblob = nullptr;
      TRY(ensure_copy_stream(c));
      TRY(alloc_stages(c, s));
    } else {
      uranges.push_back({0, (int64_t)CB.units.size()});
      TRY(upload(c, CB.blob.get(), (size_t)CB.bytes, &c->d_cblob, s));
    }
    for (auto& r : uranges)
      std::stable_sort(CB.units.begin() + r.first, CB.units.begin() + r.second,
                       [](const int4& a, const int4& b) { return a.z - a.y > b.z - b.y; });
    TRY(upload_vec(c, CB.units, &c->d_cunits, s));
    TRY(upload_vec(c, CB.bsplit, &c->d_bsplit, s));
    c->cunits = (int64_t)CB.units.size();
    c->nslots = CB.nslots;
    {
      void* q;
      TRY(dalloc(c, (size_t)std::max<int64_t>(1, CB.nslots) * CB_ROWS * 8, &q, s));
      c->d_slots = static_cast<double*>(q);
      TRY(dalloc(c, (size_t)std::max<int64_t>(1, CB.nb) * 4, &q, s));
      c->d_tickets = static_cast<int*>(q);
      CUDA_TRY(cudaMemsetAsync(q, 0, (size_t)std::max<int64_t>(1, CB.nb) * 4, s));
      TRY(dalloc(c, 16, &q, s));
      c->d_ctr = static_cast<int*>(q);
      CUDA_TRY(cudaMemsetAsync(q, 0, 16, s));
    }
    c->cnb = CB.nb;
    c->citems = (int64_t)CB.items.size();
    c->ntiles = 0; c->nsell = 0; c->nslabs = 0; c->nrec = 0; c->nsplit = 0;
    c->h_tile_row0.clear(); c->h_tile_slab.clear(); c->h_sr_row.clear(); c->hchunks.clear();
    c->blob_bytes = CB.bytes + c->citems * 24 + (CB.nb + 1) * 4 + CB.nb * (CB_W + 1) * 4;
    c->py_len = c->nranks > 1 ? c->shard * c->nranks : 0;
    if (c->py_len) {
      void* pp;
      TRY(dalloc(c, (size_t)c->py_len * 8, &pp, s));
      c->d_py = pp;
      // rows [m, py_len) are never written by the band kernel: zero them once
      CUDA_TRY(cudaMemsetAsync(static_cast<double*>(c->d_py) + m, 0, (size_t)(c->py_len - m) * 8, s));
    }
    CUDA_TRY(cudaStreamSynchronize(s));   // host staging buffers are freed on return
  } else {
    // ---- row tiles: the rank's row slice (row formats) or its column slice transposed on the GPU
    // (column formats: one part of its own with every row of the matrix, no shared rows -- its
    // partial y is merged column-style -- and window-local column ids into x[wlo, whi))
    const bool tr = col_rows;
    const int64_t rwlo = tr ? 0 : c->wlo;
    const int64_t nx = tr ? W : n;   // x entries the tiles index
    c->ybase = rwlo;
    c->xoff = tr ? c->wlo : 0;
    c->xn = nx;
    const size_t mark = c->bufs.size();   // temporaries allocated from here are freed after packing
    std::vector<int64_t> lpr;
    int32_t *t_cols = nullptr, *t_ptr = nullptr;
    void* t_vals = nullptr;
    if (tr) {
      sub(5);
      TRY(transpose_slice(c, fmt, lp, idx, coo_row, val, V, s, &t_cols, &t_vals, &t_ptr, lpr));
      sub(0);
      lap(3);
    }
    const std::vector<int64_t>& LP = tr ? lpr : lp;
    std::vector<msrep_part_desc> tpart(1);
    tpart[0].start_idx = 0;
    tpart[0].end_idx = nz_r - 1;
    tpart[0].start_row = 0;
    tpart[0].end_row = m - 1;
    tpart[0].start_flag = 0;
    tpart[0].owned_begin = 0;
    tpart[0].owned_end = m;
    // ---- schedule
    Schedule S;
    // transposed column formats: the rows' column spans come from the device slice (narrow SELL)
    std::vector<int32_t> span_lo, span_hi;
    if (tr && c->tune_sell == 2 && m > 0) {
      void* q;
      TRY(dalloc(c, (size_t)m * 8, &q, s));
      int32_t* d_span = static_cast<int32_t*>(q);
      CUDA_TRY(launch_row_span(t_ptr, t_cols, m, d_span, d_span + m, s));
      span_lo.resize((size_t)m);
      span_hi.resize((size_t)m);
      CUDA_TRY(cudaMemcpyAsync(span_lo.data(), d_span, (size_t)m * 4, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaMemcpyAsync(span_hi.data(), d_span + m, (size_t)m * 4, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
    }
    auto schedule = [&](bool sell) {
      if (!tr) {
        // narrow SELL tiles (16-bit column offsets) from the host's column ids (MSREP_TUNE_SELL 2)
        build_row_schedule(c->parts, c->P0, c->P1, c->B_lo, c->wlo, (int)V, LP, S, sell,
                           c->tune_sell == 2 ? idx + c->B_lo : nullptr);
        return;
      }
      // one part of its own with no shared rows: rows cut into fixed chunks of 2^18 (the cut never
      // depends on the host's thread count, so neither do the tiles nor the bits), scheduled on the
      // host threads, then concatenated (record indices offset)
      constexpr int64_t CH = (int64_t)1 << 18;
      const int64_t nch = std::max<int64_t>(1, (m + CH - 1) / CH);
      std::vector<Schedule> cs((size_t)nch);
      std::atomic<int64_t> next{0};
      auto work = [&] {
        for (int64_t k; (k = next.fetch_add(1)) < nch;) {
          const int64_t r0 = k * CH, r1 = std::min(m, r0 + CH);
          std::vector<msrep_part_desc> d(1, tpart[0]);
          d[0].start_idx = LP[(size_t)r0];
          d[0].end_idx = LP[(size_t)r1] - 1;
          d[0].start_row = r0; d[0].end_row = r1 - 1;
          d[0].owned_begin = r0; d[0].owned_end = r1;
          build_row_schedule(d, 0, 1, 0, 0, (int)V, LP, cs[(size_t)k], sell, nullptr,
                             span_lo.empty() ? nullptr : span_lo.data(), span_hi.empty() ? nullptr : span_hi.data());
        }
      };
      const int T = (int)std::min<int64_t>(nch, host_threads(nz_r + m));
      std::vector<std::thread> th;
      for (int t = 1; t < T; t++) th.emplace_back(work);
      work();
      for (auto& x : th) x.join();
      for (Schedule& q : cs) {
        const int32_t off = S.nrec;
        for (TileHost t : q.tiles) {
          if (t.rec >= 0) t.rec += off;
          S.tiles.push_back(t);
        }
        S.sell.insert(S.sell.end(), q.sell.begin(), q.sell.end());
        S.sr_row.insert(S.sr_row.end(), q.sr_row.begin(), q.sr_row.end());
        for (int32_t v : q.sr_rec) S.sr_rec.push_back(v + off);
        S.sr_head.insert(S.sr_head.end(), q.sr_head.begin(), q.sr_head.end());   // no head lists: all 0
        S.nrec += q.nrec;
        S.nslabs += q.nslabs;
      }
      S.part_rec = {0, S.nrec};
    };
    schedule(c->tune_sell != 0);
    {
      // A few SELL tiles among many SEG tiles cost more than they save: their presence selects
      // the SELL instantiation of rows_kernel for the whole launch, whose SEG path ran 2.5x
      // slower on an R-MAT part with 1 SELL tile in 195K (profiles/r1_scaling_projection.jsonl,
      // tools/dbg_part.py).  Keep SELL tiles only if they hold >= 10 % of the rank's nonzeros.
      int64_t sell_nz = 0;
      for (const TileHost& t : S.sell)
        sell_nz += LP[(size_t)t.row0 + (size_t)(t.packed & 0xffff)] - LP[(size_t)t.row0];
      if (!S.sell.empty() && sell_nz * 10 < nz_r) {
        S = Schedule{};
        schedule(false);
        sell_nz = 0;
      }
      // ... and SEG / slab tiles get their own launch of the SEG instantiation (forked onto a side
      // stream) when they hold >= 5 % of the nonzeros, and always for fp32 (whose SELL
      // instantiation walks SELL tiles only); a small fp64 share rides in the SELL launch (a
      // second launch put its CTAs in the first one's tail: stencil 0.0914 -> 0.0953 ms)
      c->split_launch = !S.sell.empty() && !S.tiles.empty() && (V == 4 || (nz_r - sell_nz) * 20 >= nz_r);
    }
    sub(1);
    lap(2);
    c->ntiles = (int)(S.tiles.size() + S.sell.size());
    c->nsell = (int)S.sell.size();
    int64_t nsell_narrow = 0;
    for (const TileHost& t : S.sell) nsell_narrow += t.rec == -3 ? 1 : 0;
    c->nsell_narrow = nsell_narrow;
    c->nslabs = S.nslabs;
    c->nrec = S.nrec;
    c->nsplit = (int)S.sr_row.size();

    // ---- tile order (SELL tiles first) and blob offsets
    static_assert(sizeof(TileHost) == sizeof(int4), "tile");
    S.tiles.insert(S.tiles.begin(), S.sell.begin(), S.sell.end());   // one list: SELL tiles first
    const size_t nt = S.tiles.size();
    std::vector<int32_t> blob16(nt);
    int64_t blob_total = 0;
    for (size_t t = 0; t < nt; t++) {
      const TileHost& th = S.tiles[t];
      const int kind = th.rec == -2 ? KIND_SELL : th.rec == -3 ? KIND_SELLN : th.rec >= 0 ? KIND_SLAB : KIND_SEG;
      if (blob_total / 16 >= (int64_t)1 << 31) return fail(MSREP_ERR_TOO_LARGE, "tile blob exceeds 32 GiB");
      blob16[t] = (int32_t)(blob_total / 16);
      blob_total += blob_bytes(kind, th.packed & 0xffff, th.packed >> 16, (int)V);
    }
    // ---- pack groups: all tiles at once (device-resident), or chunks of <= chunk_bytes of
    // layout (host-resident), each with the span of rank-local nonzeros its tiles read
    const bool host_res = c->residency == MSREP_RESIDENT_HOST;
    struct Group { int32_t t0, t1; int64_t z0, z1; };
    std::vector<Group> groups;
    {
      auto tile_end = [&](size_t t) { return t + 1 < nt ? (int64_t)blob16[t + 1] * 16 : blob_total; };
      auto zspan = [&](const TileHost& th, int64_t& z0, int64_t& z1) {
        z0 = th.nz0;
        z1 = (th.rec == -2 || th.rec == -3) ? LP[(size_t)th.row0 + (size_t)(th.packed & 0xffff)] : th.nz0 + (th.packed >> 16);
      };
      const int64_t cap = host_res ? c->chunk_bytes : INT64_MAX;
      size_t t = 0;
      while (t < nt) {
        Group g{(int32_t)t, (int32_t)t, INT64_MAX, 0};
        const int64_t off0 = (int64_t)blob16[t] * 16;
        // host-resident chunks also break where the SELL tiles end (one instantiation per chunk)
        while (t < nt && (t == (size_t)g.t0 || (tile_end(t) - off0 <= cap && !(host_res && t == S.sell.size())))) {
          int64_t z0, z1;
          zspan(S.tiles[t], z0, z1);
          g.z0 = std::min(g.z0, z0);
          g.z1 = std::max(g.z1, z1);
          t++;
        }
        g.t1 = (int32_t)t;
        groups.push_back(g);
        if (host_res) {
          Ctx::Chunk ch{g.t0, g.t1, 0, 0, off0, tile_end(t - 1) - off0, S.tiles[(size_t)g.t0].rec == -2 || S.tiles[(size_t)g.t0].rec == -3};
          c->chunks.push_back(ch);
        }
      }
    }
    int64_t span = 0;
    for (auto& g : groups) span = std::max(span, g.z1 - g.z0);
    if (!host_res || tr) span = nz_r;   // (transposed: the whole slice is on the device already)

    // ---- upload the slice (the only H2D of A) and build the tile blobs on the GPU
    void* vp;
    int32_t *d_idx, *d_aux = nullptr, *d_crow = nullptr;
    int32_t* d_lp = nullptr;   // window-local pointer for SELL packing
    if (tr) {
      vp = t_vals;
      d_idx = t_cols;
      d_aux = d_lp = t_ptr;
    } else {
      TRY(dalloc(c, (size_t)span * V, &vp, s));
      void* ip;
      TRY(dalloc(c, (size_t)span * 4, &ip, s));
      d_idx = static_cast<int32_t*>(ip);
    }
    if (tr) {
      // the row pointer of the transposed slice is on the device (t_ptr)
    } else if (fmt == MSREP_COO) {
      void* ap;
      TRY(dalloc(c, (size_t)span * 4, &ap, s));
      d_crow = static_cast<int32_t*>(ap);
      if (c->nsell) {   // the COO local pointer was counted on the host (plan phase)
        std::vector<int32_t> lp32(lp.begin(), lp.end());
        TRY(upload_vec(c, lp32, &d_lp, s));
      }
    } else {
      // upload the global pointer slice and rebase it on the GPU (Sec. 4.1)
      int64_t* d_g;
      TRY(upload(c, ptr + c->wlo, (size_t)W + 1, &d_g, s));
      void* ap;
      TRY(dalloc(c, ((size_t)W + 1) * 4, &ap, s));
      d_aux = static_cast<int32_t*>(ap);
      CUDA_TRY(launch_rebase(d_g, d_aux, W + 1, B_lo, B_hi, s));
      d_lp = d_aux;
    }
    int4* d_tiles_orig;
    int32_t* d_blob16;
    TRY(upload(c, reinterpret_cast<const int4*>(S.tiles.data()), nt, &d_tiles_orig, s));
    TRY(upload_vec(c, blob16, &d_blob16, s));
    // ---- x layout of the rank (device-resident row formats):
    //  * compact x: the rank's distinct columns in column order; the tiles carry compact column ids
    //    and every SpMV first gathers x' = x[cols] (one sequential pass over x), so the gathers hit
    //    an x' that fits in L2 next to the matrix stream instead of the whole x;
    //  * hot x: the most-gathered columns get slots in a shared-memory copy of x' per CTA; SEG / slab
    //    tiles carry HOT_TAG | slot for them (the SELL instantiation has no hot path).
    std::vector<int32_t> hot, xcols, xcols_col;
    int32_t *d_hotslot = nullptr, *d_colmap = nullptr, *dp_hot_tmp = nullptr;
    bool idx_up = false;
    c->nhot = 0;
    c->hot_nnz = 0;
    c->nxc = 0;
    c->x_order = 0;
    const bool want_hot = !host_res && c->tune_hot != 0 && nz_r > 0 && nx > 0 && (c->nsell == 0 || c->split_launch);
    const bool want_cx = !host_res && nz_r > 0 && nx > 0 &&
                         (c->tune_compact >= 1 || (c->tune_compact == -1 && (int64_t)nx * (int64_t)V >= COMPACT_X_MIN_BYTES));
    if (tr) idx_up = true;
    if (want_hot || want_cx) {
      int sms = 148;
      CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
      if (!idx_up) TRY(h2d(c, d_idx, idx + B_lo, (size_t)nz_r * 4, s));
      idx_up = true;
      void* dp;
      TRY(dalloc(c, (size_t)nx * 4, &dp, s));
      int32_t* d_deg = static_cast<int32_t*>(dp);
      CUDA_TRY(cudaMemsetAsync(d_deg, 0, (size_t)nx * 4, s));
      CUDA_TRY(launch_col_degree(d_idx, nz_r, d_deg, s));
      std::vector<int32_t> deg((size_t)nx);
      CUDA_TRY(cudaMemcpyAsync(deg.data(), d_deg, (size_t)nx * 4, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      // a hot slot costs one gather per CTA per launch: worth it from 4 gathers per SM on
      const int32_t min_deg = 4 * sms;
      std::mutex mu;
      std::vector<std::pair<int64_t, std::vector<int32_t>>> used;
      par_ranges(nx, [&](int64_t lo, int64_t hi) {
        std::vector<int32_t> v, u;
        for (int64_t q = lo; q < hi; q++) {
          if (want_hot && deg[(size_t)q] >= min_deg) v.push_back((int32_t)q);
          if (want_cx && deg[(size_t)q] > 0) u.push_back((int32_t)q);
        }
        std::lock_guard<std::mutex> lk(mu);
        hot.insert(hot.end(), v.begin(), v.end());
        used.push_back({lo, std::move(u)});
      });
      if (want_cx) {
        std::sort(used.begin(), used.end(), [](const auto& p, const auto& q) { return p.first < q.first; });
        for (auto& u : used) xcols.insert(xcols.end(), u.second.begin(), u.second.end());
        // auto: compact x when the column degrees are skewed -- the columns of >= 8x the mean degree
        // hold >= 1/5 of the rank's nonzeros (R-MAT, power-law columns) -- in decreasing degree when
        // x' is too big for the L2 (the warm lines then stay resident together instead of being
        // spread over all of x'), else in column order; for unskewed matrices column order when the
        // rank touches <= 3/4 of x (a uniform matrix that touches every column gains nothing from
        // the extra gather); else no compact x
        bool skewed = false;
        if (!xcols.empty()) {
          const int64_t thr = 8 * (nz_r / (int64_t)xcols.size());
          int64_t heavy = 0;
          for (int32_t q : xcols) heavy += deg[(size_t)q] >= thr ? deg[(size_t)q] : 0;
          skewed = heavy * 5 >= nz_r;
        }
        // degree order pays where x' does not fit in half the L2 (power-law suite: 188 MB, 1.00 -> 0.78 ms);
        // an x' that fits stays in column order, whose gather needs no scatter (R-MAT 59 MB: fp64 step
        // 1.174 -> 1.162, fp32 1.176 -> 1.102, pCSC 1.213 -> 1.159 ms; profiles/r2_kernel_ab.txt #19)
        int l2 = 0;
        if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, c->device) != cudaSuccess || l2 <= 0) l2 = 126 << 20;
        const bool big_x = (int64_t)xcols.size() * (int64_t)V * 2 > (int64_t)l2;
        int mode = c->tune_compact >= 1 ? c->tune_compact
                   : skewed ? (big_x ? 2 : 1) : ((int64_t)xcols.size() * 4 <= (int64_t)nx * 3 ? 1 : 0);
        // narrow SELL tiles need the column order (their 16-bit offsets were checked on column ids)
        if (mode == 2 && nsell_narrow > 0) mode = 1;
        if (mode >= 1) {
          TRY(dalloc(c, (size_t)nx * 4, &dp, s));
          d_colmap = static_cast<int32_t*>(dp);   // column -> compact id (filled from the kept list below)
          c->nxc = (int64_t)xcols.size();
          c->x_order = mode == 2 ? 1 : 0;
          if (mode == 2) {   // degree order: the most-gathered columns share the first lines of x'
            xcols_col = xcols;   // the gather of x' reads x in column order (gather_x_kernel pos)
            // stable by column within a degree: columns of degree >= 2^16 (few) sorted, the rest
            // counting-sorted by degree (descending)
            constexpr int32_t CAP = 1 << 16;
            std::vector<int32_t> out;
            out.reserve(xcols.size());
            std::vector<int64_t> cnt((size_t)CAP + 1, 0);
            for (int32_t q : xcols) {
              if (deg[(size_t)q] >= CAP) out.push_back(q);
              else cnt[(size_t)(CAP - deg[(size_t)q])]++;
            }
            std::sort(out.begin(), out.end(), [&](int32_t a, int32_t b) {
              return deg[(size_t)a] != deg[(size_t)b] ? deg[(size_t)a] > deg[(size_t)b] : a < b;
            });
            int64_t pos = (int64_t)out.size();
            for (auto& v : cnt) { const int64_t t = v; v = pos; pos += t; }
            out.resize(xcols.size());
            for (int32_t q : xcols)
              if (deg[(size_t)q] < CAP) out[(size_t)cnt[(size_t)(CAP - deg[(size_t)q])]++] = q;
            xcols.swap(out);
          }
        } else {
          xcols.clear();
        }
      }
      used.clear();
      if (want_hot) {
        // cache size: MSREP_TUNE_HOT_X = k > 1 asks for k KiB; else HOT_AUTO_BYTES.  Shared memory
        // and L1 share the SM's 256 KB, and the gathers still missing need L1 room in flight
        const int64_t want = c->tune_hot > 1 ? std::min<int64_t>((int64_t)c->tune_hot << 10, HOT_BYTES) : HOT_AUTO_BYTES;
        const size_t H = (size_t)(want / (int64_t)V) * (size_t)c->tune_hot_cluster;   // per CTA x CTAs sharing
        auto hotter = [&](int32_t a, int32_t b) { return deg[(size_t)a] != deg[(size_t)b] ? deg[(size_t)a] > deg[(size_t)b] : a < b; };
        if (hot.size() > H) {
          std::nth_element(hot.begin(), hot.begin() + (ptrdiff_t)H, hot.end(), hotter);
          hot.resize(H);
        }
        std::sort(hot.begin(), hot.end(), hotter);   // slot 0 = the hottest column
        int64_t cap_nz = 0;
        for (int32_t q : hot) cap_nz += deg[(size_t)q];
        // auto: only when the hot columns carry >= 5 % of the rank's gathers (power-law columns)
        // (fp32: the hot instantiation of the fp32 tile walk spills registers, 1.07 -> 1.81 ms on R-MAT,
        // profiles/r2_hot_x_ab.txt -- off unless forced)
        const bool on = c->tune_hot >= 1 ? !hot.empty()
                                         : (V == 8 && cap_nz * 20 >= nz_r && nz_r >= ((int64_t)1 << 20));
        if (on) {
          TRY(dalloc(c, (size_t)nx * 4, &dp, s));
          d_hotslot = static_cast<int32_t*>(dp);
          CUDA_TRY(cudaMemsetAsync(d_hotslot, 0xff, (size_t)nx * 4, s));   // -1: cold
          c->nhot = (int)hot.size();
          c->hot_nnz = cap_nz;
          c->hot_cluster = c->tune_hot_cluster;
          TRY(upload_vec(c, hot, &dp_hot_tmp, s));   // original ids, for the slot table
        } else {
          hot.clear();
        }
      }
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    sub(2);
    const size_t keep_from = c->bufs.size();
    c->d_xcols = nullptr;
    c->d_xpos = nullptr;
    c->d_xc = nullptr;
    if (c->nxc && c->x_order == 1) {
      // degree order: x' row pos[i] holds column xcols_col[i] (ascending), colmap[col] = its x' row
      std::vector<int32_t> pos(xcols_col.size());
      {
        std::vector<int32_t> at((size_t)nx);
        for (size_t i = 0; i < xcols_col.size(); i++) at[(size_t)xcols_col[i]] = (int32_t)i;
        for (size_t k2 = 0; k2 < xcols.size(); k2++) pos[(size_t)at[(size_t)xcols[k2]]] = (int32_t)k2;
      }
      TRY(upload_vec(c, xcols_col, &c->d_xcols, s));
      TRY(upload_vec(c, pos, &c->d_xpos, s));
      CUDA_TRY(launch_hot_slots(c->d_xcols, (int)c->nxc, d_colmap, s, c->d_xpos));   // colmap[xcols_col[i]] = pos[i]
      void* q;
      TRY(dalloc(c, (size_t)c->nxc * V, &q, s));
      c->d_xc = q;
    } else if (c->nxc) {
      TRY(upload_vec(c, xcols, &c->d_xcols, s));
      CUDA_TRY(launch_hot_slots(c->d_xcols, (int)c->nxc, d_colmap, s));   // colmap[xcols[k]] = k
      void* q;
      TRY(dalloc(c, (size_t)c->nxc * V, &q, s));
      c->d_xc = q;
    }
    if (c->nhot) {
      CUDA_TRY(launch_hot_slots(dp_hot_tmp, c->nhot, d_hotslot, s));
      if (c->nxc && c->x_order == 1) {   // degree-ordered x': the hot columns are its first entries
        for (size_t q = 0; q < hot.size(); q++) hot[q] = (int32_t)q;
      } else if (c->nxc) {   // the kernels read x': hot slots are filled from compact ids
        for (auto& q : hot) q = (int32_t)(std::lower_bound(xcols.begin(), xcols.end(), q) - xcols.begin());
      }
      TRY(upload_vec(c, hot, &c->d_hot, s));
    } else {
      c->d_hot = nullptr;
    }
    int64_t pack_bytes = host_res ? 16 : blob_total;
    for (auto& ch : c->chunks) pack_bytes = std::max(pack_bytes, ch.bytes);
    void* bp;
    TRY(dalloc(c, (size_t)std::max<int64_t>(16, pack_bytes), &bp, s));
    char* d_pack = static_cast<char*>(bp);
    if (host_res) {
      CUDA_TRY(host_alloc_on(reinterpret_cast<void**>(&c->h_blob), (size_t)std::max<int64_t>(16, blob_total), c->numa_node));
      c->h_bytes = blob_total;
      c->d_blob = nullptr;
    } else {
      c->d_blob = d_pack;
    }
    for (size_t gi = 0; gi < groups.size(); gi++) {
      const Group& g = groups[gi];
      const int64_t zn = g.z1 - g.z0;
      if (zn > 0 && !tr) {
        TRY(h2d(c, vp, static_cast<const char*>(val) + (size_t)(B_lo + g.z0) * V, (size_t)zn * V, s));
        if (!idx_up) TRY(h2d(c, d_idx, idx + B_lo + g.z0, (size_t)zn * 4, s));
        if (d_crow) TRY(h2d(c, d_crow, coo_row + B_lo + g.z0, (size_t)zn * 4, s));
      }
      const int64_t off0 = (int64_t)blob16[(size_t)g.t0] * 16;
      // pointers shifted by the group's first nonzero / layout offset: tiles index them unchanged
      // (the transposed slice is whole on the device)
      const int64_t zb = tr ? 0 : g.z0;
      PackLaunch PL{d_tiles_orig + g.t0, d_blob16 + g.t0, g.t1 - g.t0,
                    static_cast<const char*>(vp) - (size_t)zb * V, d_idx - zb,
                    d_crow ? d_crow - zb : d_aux, fmt == MSREP_COO, (int)V, rwlo,
                    host_res ? d_pack - off0 : d_pack, d_lp, d_hotslot, d_colmap};
      CUDA_TRY(launch_pack(PL, s));
      if (host_res)
        CUDA_TRY(cudaMemcpyAsync(c->h_blob + off0, d_pack, (size_t)c->chunks[gi].bytes, cudaMemcpyDeviceToHost, s));
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    sub(3);
    std::vector<TileHost> fin(S.tiles);
    for (size_t t = 0; t < fin.size(); t++) fin[t].nz0 = blob16[t];
    c->h_tile_row0.resize(fin.size());
    c->h_tile_slab.resize(fin.size());
    for (size_t t = 0; t < fin.size(); t++) {
      c->h_tile_row0[t] = fin[t].row0;
      c->h_tile_slab[t] = fin[t].rec >= 0 ? 1 : 0;
    }
    c->h_sr_row = S.sr_row;
    c->hchunks.clear();
    CUDA_TRY(cudaStreamSynchronize(s));
    // plain slices are no longer needed: the blobs hold the partition (host-resident: the
    // pinned copy does, and the packing buffer goes too)
    release_range(c, mark, host_res ? c->bufs.size() : keep_from);
    if (host_res) {
      TRY(ensure_copy_stream(c));
      TRY(alloc_stages(c, s));
    }
    TRY(upload(c, reinterpret_cast<const int4*>(fin.data()), fin.size(), &c->d_tiles, s));
    c->blob_bytes = blob_total;
    void* rp;
    TRY(dalloc(c, (size_t)std::max(1, S.nrec) * 8, &rp, s));
    c->d_rec = static_cast<double*>(rp);
    {
      TRY(upload_vec(c, S.sr_row, &c->d_sr_row, s));
      TRY(upload_vec(c, S.sr_rec, &c->d_sr_rec, s));
      TRY(upload_vec(c, S.sr_head, &c->d_sr_head, s));
      TRY(upload_vec(c, S.head_list, &c->d_head_list, s));
      TRY(upload_vec(c, S.part_rec, &c->d_part_rec, s));
      void* hp;
      TRY(dalloc(c, (size_t)c->vparts * 8, &hp, s));
      c->d_head_local = static_cast<double*>(hp);
      if (c->nranks > 1) {
        TRY(dalloc(c, (size_t)c->np * 8, &hp, s));
        c->d_head_all = static_cast<double*>(hp);
        TRY(dalloc(c, 16, &hp, s));
        c->d_fence = static_cast<int*>(hp);
      }
      c->nheads_local = 0;
      if (!tr)
        for (int j = P0; j < P1; j++) c->nheads_local += parts[(size_t)j].start_flag ? 1 : 0;
    }
    if (tr) {   // the rank's partial y for the reduce-scatter (nranks > 1), in the partition's dtype
      c->py_len = c->nranks > 1 ? c->shard * c->nranks : 0;
      c->py_f32 = V == 4;
      if (c->py_len) {
        void* pp;
        TRY(dalloc(c, (size_t)c->py_len * V, &pp, s));
        c->d_py = pp;
        // rows [m, py_len) are never written by the tiles (they cover rows [0, m)): zero them once
        CUDA_TRY(cudaMemsetAsync(static_cast<char*>(pp) + (size_t)m * V, 0, (size_t)(c->py_len - m) * V, s));
      }
    }
  }
  CUDA_TRY(cudaStreamSynchronize(s));
  if (!colwise(fmt) || col_rows) sub(4);
  lap(3);
  nv_phase.end();
  const auto t1 = std::chrono::steady_clock::now();
  TRY(tune_xload(c, s, nz_r));   // outside the partition timer: a measurement, not partitioning

  // ---- stats (X_p by bitmap; outside the partition timer)
  msrep_stats& st = c->stats;
  memset(&st, 0, sizeof st);
  st.nparts = c->np; st.nranks = c->nranks; st.parts_per_rank = c->vparts;
  st.nnz_rank = nz_r;
  st.rows_window = W;
  const bool bands = colwise(fmt) && !c->col_rows;
  st.ntiles = bands ? c->citems : c->ntiles; st.nsell = c->nsell; st.nsell_narrow = bands ? 0 : c->nsell_narrow; st.nslabs = c->nslabs; st.nsplit_rows = c->nsplit; st.nheads_local = c->nheads_local;
  st.partition_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  for (int k = 0; k < 4; k++) st.phase_ms[k] = phase[k];
  st.residency = c->residency;
  st.nchunks = (int64_t)c->chunks.size();
  st.host_bytes = c->h_bytes;
  st.x_no_allocate = c->xna;
  st.nhot = c->nhot;
  st.x_compact = c->nxc;
  st.sell_1cta = c->sell_1cta;
  st.gpu_numa_node = c->numa_node;
  st.host_numa_node = c->h_blob ? page_numa_node(c->h_blob) : -1;
  st.hot_nnz = c->hot_nnz;
  st.col_layout = colwise(fmt) ? (c->col_rows ? 1 : 0) : -1;
  st.x_order = c->nxc ? c->x_order : -1;
  for (int k = 0; k < 6; k++) st.layout_ms[k] = layout_ms[k];
  int64_t X = 0;
  if (colwise(fmt)) {
    X = W;   // pCSC reads x only over its column window
  } else {
    std::vector<uint64_t> bits((size_t)(inner + 63) / 64, 0);
    uint64_t* bw = bits.data();
    par_ranges(B_hi - B_lo, [&](int64_t lo, int64_t hi) {
      for (int64_t k = B_lo + lo; k < B_lo + hi; k++)
        __atomic_fetch_or(&bw[(size_t)idx[k] >> 6], 1ull << (idx[k] & 63), __ATOMIC_RELAXED);
    });
    for (uint64_t w : bits) X += __builtin_popcountll(w);
  }
  st.distinct_cols = X;
  int64_t base;
  int64_t own, ybytes_b1, ybytes_b0;
  if (colwise(fmt)) {
    const int64_t rows_out = c->nranks > 1 ? std::min<int64_t>(c->shard, std::max<int64_t>(0, m - (int64_t)c->rank * c->shard)) : m;
    own = rows_out;
    // the rank's entries + its column pointer + its x window + (p > 1) the fp64 py write and the
    // shard read after the reduce-scatter; p = 1 fuses alpha/beta into the band kernel (no py)
    base = nz_r * (int64_t)(V + 4) + (fmt == MSREP_COO_COL ? nz_r * 4 : (W + 1) * 4) + W * (int64_t)V +
           (c->nranks > 1 ? m * 8 + rows_out * 8 : 0);
    ybytes_b1 = rows_out * (int64_t)V * 2;
    ybytes_b0 = rows_out * (int64_t)V;
  } else {
    own = c->own_hi - c->own_lo;
    base = nz_r * (int64_t)(V + 4) + X * (int64_t)V + (fmt == MSREP_COO ? nz_r * 4 : (W + 1) * 4);
    ybytes_b1 = own * (int64_t)V * 2;
    ybytes_b0 = own * (int64_t)V;
  }
  st.owned_rows = own;
  // what the built layout moves per SpMV: the stored blobs (incl. padding, SEG keys instead of COO
  // row ids), the x entries, y (beta != 0) -- and p > 1 pCSC's py round trip
  st.stream_bytes = c->blob_bytes + (colwise(fmt) ? W : X) * (int64_t)V + ybytes_b1 +
                    (colwise(fmt) && c->nranks > 1 ? m * 8 + own * 8 : 0);
  st.alg_bytes = base + ybytes_b1;
  st.alg_bytes_beta0 = base + ybytes_b0;
  const int64_t nmain = c->chunks.empty() ? 1 : (int64_t)c->chunks.size();   // main-kernel launches
  const bool fixl = c->nsplit > 0;                                            // a fix-up launch per SpMV
  if (bands)
    st.kernels_per_spmv = (c->cunits ? nmain : 0) + (c->nranks > 1 ? 1 /*shard epilogue*/ : 0);
  else if (colwise(fmt))
    st.kernels_per_spmv = (c->ntiles ? nmain + (c->split_launch && c->chunks.empty() ? 1 : 0) : 0) + (fixl ? 1 : 0) +
                          (c->nxc ? 1 : 0) + (c->nranks > 1 ? 1 /*shard epilogue*/ : 0);
  else st.kernels_per_spmv = (c->ntiles ? nmain + (c->split_launch && c->chunks.empty() ? 1 : 0) : 0) + (c->nranks > 1 && c->any_flag ? 1 : 0) + (fixl ? 1 : 0) + (c->nxc ? 1 : 0);
  int64_t db = 0;
  for (auto& b : c->bufs) db += (int64_t)b.bytes;
  st.device_bytes = db;
  st.tile_bytes = c->blob_bytes;
  c->ready = true;
  return MSREP_OK;
}

msrep_status_t msrep_partition_slice(msrep_ctx h, msrep_format fmt, msrep_dtype dtype, int64_t m, int64_t n,
                                     int64_t nnz, const int64_t* ptr, const int32_t* idx_slice,
                                     const void* val_slice, int64_t slice_begin, int64_t slice_end,
                                     msrep_part_desc* parts_out, void* stream) {
  if (!h) return fail(MSREP_ERR_INVALID_ARG, "ctx is NULL");
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (fmt != MSREP_CSR && fmt != MSREP_CSC) return fail(MSREP_ERR_INVALID_ARG, "msrep_partition_slice takes CSR or CSC");
  if (dtype != MSREP_F64 && dtype != MSREP_F32) return fail(MSREP_ERR_INVALID_ARG, "dtype %d", (int)dtype);
  if (m < 0 || n < 0 || nnz < 0 || !ptr) return fail(MSREP_ERR_INVALID_ARG, "bad dimensions or ptr NULL");
  if (m >= kMaxIdx || n >= kMaxIdx) return fail(MSREP_ERR_TOO_LARGE, "m, n must be < 2^31");
  if (slice_begin < 0 || slice_end < slice_begin || slice_end > nnz)
    return fail(MSREP_ERR_INVALID_ARG, "slice [%lld, %lld) outside [0, nnz)", (long long)slice_begin, (long long)slice_end);
  const int64_t outer = fmt == MSREP_CSC ? n : m;
  if (ptr[0] != 0 || ptr[outer] != nnz) return fail(MSREP_ERR_DIM_MISMATCH, "ptr[0] != 0 or ptr[%lld] != nnz", (long long)outer);
  std::vector<int64_t> bnd;
  split_bounds(fmt, c->split, outer, nnz, c->np, ptr, nullptr, bnd, &c->groups);
  const int P0 = c->rank * c->vparts, P1 = P0 + c->vparts;
  const int64_t lo = bnd[(size_t)P0], hi = bnd[(size_t)P1];
  if (lo < hi && (lo < slice_begin || hi > slice_end))
    return fail(MSREP_ERR_INVALID_ARG, "slice [%lld, %lld) does not hold this rank's nonzeros [%lld, %lld)",
                (long long)slice_begin, (long long)slice_end, (long long)lo, (long long)hi);
  if (lo < hi && (!idx_slice || !val_slice)) return fail(MSREP_ERR_INVALID_ARG, "idx/val NULL");
  // msrep_partition reads idx / val of CSR / CSC only at this rank's positions [lo, hi): hand it
  // base addresses that put global position slice_begin at the start of the slices
  const size_t V = vsz(dtype);
  const int32_t* idx = reinterpret_cast<const int32_t*>(reinterpret_cast<uintptr_t>(idx_slice) - (uintptr_t)slice_begin * 4);
  const void* val = reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(val_slice) - (uintptr_t)slice_begin * V);
  return msrep_partition(h, fmt, dtype, m, n, nnz, ptr, idx, nullptr, val, parts_out, stream);
}

msrep_status_t spmv_impl(msrep_ctx h, const void* alpha_p, const void* x, const void* beta_p, void* y,
                         msrep_layout layout, void* stream, int nmirror, void* const* mirrors);

msrep_status_t msrep_spmv(msrep_ctx h, const void* alpha_p, const void* x, const void* beta_p, void* y,
                          msrep_layout layout, void* stream) {
  return spmv_impl(h, alpha_p, x, beta_p, y, layout, stream, 0, nullptr);
}

msrep_status_t msrep_spmv_mirror(msrep_ctx h, const void* alpha_p, const void* x, const void* beta_p, void* y,
                                 int nmirror, void* const* mirrors, void* stream) {
  if (!h) return fail(MSREP_ERR_INVALID_ARG, "ctx is NULL");
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (!c->ready) return fail(MSREP_ERR_STATE, "msrep_spmv_mirror before msrep_partition");
  if (colwise(c->fmt)) return fail(MSREP_ERR_STATE, "msrep_spmv_mirror supports the row formats (pCSR, pCOO)");
  if (nmirror < 0 || nmirror > MAX_MIRRORS || (nmirror > 0 && !mirrors))
    return fail(MSREP_ERR_INVALID_ARG, "nmirror %d (0..%d)", nmirror, MAX_MIRRORS);
  for (int i = 0; i < nmirror; i++)
    if (!mirrors[i]) return fail(MSREP_ERR_INVALID_ARG, "mirror %d is NULL", i);
  TRY(spmv_impl(h, alpha_p, x, beta_p, y, MSREP_Y_OWNED, stream, nmirror, mirrors));
  if (c->nranks > 1) {   // completion fence: every rank's stores into every mirror are done
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CUDA_TRY(cudaMemsetAsync(c->d_fence, 0, sizeof(int), s));
    TRY(comm_allreduce(c, c->d_fence, 1, true, s));
  }
  return MSREP_OK;
}

// The row-tile walk of one SpMV (k = 1) or SpMM (k > 1): device-resident, or streamed in chunks
// from the pinned host copy (MSREP_RESIDENT_HOST)
msrep_status_t row_tiles_pass(Ctx* c, const RowLaunch& L, int k, cudaStream_t s) {
  if (c->residency != MSREP_RESIDENT_HOST) return launch_row_tiles(c, L, k, s);
  return stream_chunks(c, s, [&](const Ctx::Chunk& ch, const char* base) -> msrep_status_t {
    RowLaunch Lc = L;
    Lc.tiles = c->d_tiles + ch.t0; Lc.ntiles = ch.t1 - ch.t0;
    Lc.blob = base; Lc.has_sell = ch.has_sell;
    CUDA_TRY(k == 1 ? launch_rows(Lc, s) : launch_rows_mm(Lc, k, s));
    return MSREP_OK;
  });
}

// the beta-deferred fix-up of the rank's split rows (records + head partials, reading R6/R10)
msrep_status_t fixup_pass(Ctx* c, void* y, double alpha, double beta, int k, int nmirror, void* const* mirrors,
                          double* rec, double* head_all, cudaStream_t s, int s0 = 0, int s1 = -1) {
  FixupLaunch F{};
  F.s0 = s0;
  F.nsplit = (s1 < 0 ? c->nsplit : s1) - s0;   // split rows [s0, s1)
  if (F.nsplit <= 0) return MSREP_OK;
  F.sr_row = c->d_sr_row; F.sr_rec = c->d_sr_rec; F.sr_head = c->d_sr_head; F.head_list = c->d_head_list;
  F.part_rec = c->d_part_rec; F.part_lo = c->P0; F.part_hi = c->P1;
  F.head_all = head_all; F.rec = rec;
  F.y = y; F.alpha = alpha; F.beta = beta; F.dtype = c->dtype == MSREP_F64 ? 0 : 1; F.k = k;
  F.nmirror = nmirror;
  for (int mi = 0; mi < nmirror; mi++) F.mirror[mi] = mirrors[mi];
  CUDA_TRY(launch_fixup(F, s));
  return MSREP_OK;
}

// Column formats (pCSC, column-sorted / unsorted pCOO): vector j of a k-wide row-major block (k = 1:
// SpMV) -- the band kernel with strides k, then for nranks > 1 the reduce-scatter of the fp64
// partial y and the alpha/beta epilogue on this rank's shard [my_lo, my_hi) (Sec. 4.3)
msrep_status_t col_spmv(Ctx* c, double alpha, const void* x, double beta, void* y, int k, int j, int64_t my_lo,
                        int64_t my_hi, cudaStream_t s) {
  const size_t V = vsz(c->dtype);
  const int dt = c->dtype == MSREP_F64 ? 0 : 1;
  if (c->col_rows) {
    // row tiles over the transposed slice (k == 1 here: SpMM passes planar vectors): one rank
    // writes y = alpha*A_p x + beta*y directly; several write their partial y_p (every row, in
    // the partition's dtype) for the reduce-scatter and the alpha/beta epilogue on the shard
    if (k != 1 || j != 0) return fail(MSREP_ERR_STATE, "column format on row tiles: strided vectors");
    const bool one = c->nranks == 1;
    void* out = one ? y : c->d_py;
    const double a = one ? alpha : 1.0, b = one ? beta : 0.0;
    TRY(prepare_x(c, x, 1, s));
    RowLaunch L = row_launch(c, x, out, a, b);
    cudaEvent_t pe;
    TRY(prof_begin(c, s, &pe));
    TRY(row_tiles_pass(c, L, 1, s));
    if (pe) CUDA_TRY(cudaEventRecord(pe, s));
    if (c->nsplit) TRY(fixup_pass(c, out, a, b, 1, 0, nullptr, c->d_rec, c->d_head_all, s));
    if (!one) {
      const char* shard = static_cast<const char*>(c->d_py) + (size_t)c->rank * c->shard * V;
      TRY(comm_reduce_scatter(c, c->d_py, (size_t)c->shard, c->py_f32, s));
      CUDA_TRY(launch_axpby_py(shard, c->py_f32 ? 1 : 0, static_cast<char*>(y) + (size_t)my_lo * V, my_hi - my_lo, alpha,
                               beta, dt, s, 1));
    }
    return MSREP_OK;
  }
  ColLaunch L = col_launch(c, static_cast<const char*>(x) + (size_t)j * V, static_cast<char*>(y) + (size_t)j * V,
                           alpha, beta);
  L.xs = k;
  L.ys = k;
  cudaEvent_t pe;
  TRY(prof_begin(c, s, &pe));
  if (c->residency == MSREP_RESIDENT_HOST) {
    TRY(stream_chunks(c, s, [&](const Ctx::Chunk& ch, const char* base) -> msrep_status_t {
      ColLaunch Lc = L;
      Lc.blob = base;
      Lc.band0 = ch.t0; Lc.nb = ch.t1 - ch.t0;
      Lc.units = L.units + ch.u0; Lc.nunits = ch.u1 - ch.u0;
      CUDA_TRY(launch_cols(Lc, s));
      return MSREP_OK;
    }));
  } else {
    CUDA_TRY(launch_cols(L, s));
  }
  if (pe) CUDA_TRY(cudaEventRecord(pe, s));
  if (c->nranks > 1) {
    const double* shard = static_cast<const double*>(c->d_py) + (size_t)c->rank * c->shard;
    TRY(comm_reduce_scatter(c, c->d_py, (size_t)c->shard, false, s));
    CUDA_TRY(launch_axpby_py(shard, 0, static_cast<char*>(y) + ((size_t)my_lo * k + j) * V, my_hi - my_lo, alpha, beta,
                             dt, s, k));
  }
  return MSREP_OK;
}

msrep_status_t spmv_impl(msrep_ctx h, const void* alpha_p, const void* x, const void* beta_p, void* y,
                         msrep_layout layout, void* stream, int nmirror, void* const* mirrors) {
  if (!h) return fail(MSREP_ERR_INVALID_ARG, "ctx is NULL");
  Nvtx nv_call("msrep_spmv");
  NvtxSeq nv;
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (!c->ready) return fail(MSREP_ERR_STATE, "msrep_spmv before msrep_partition");
  if (!alpha_p || !beta_p) return fail(MSREP_ERR_INVALID_ARG, "alpha/beta NULL");
  if ((c->m > 0 && !y) || (c->n > 0 && !x)) return fail(MSREP_ERR_INVALID_ARG, "x/y NULL");
  if (layout != MSREP_Y_REPLICATED && layout != MSREP_Y_OWNED && layout != MSREP_Y_SHARDED)
    return fail(MSREP_ERR_INVALID_ARG, "layout %d", (int)layout);
  if (colwise(c->fmt) && layout == MSREP_Y_OWNED) return fail(MSREP_ERR_STATE, "OWNED layout is for pCSR/pCOO");
  if (!colwise(c->fmt) && layout == MSREP_Y_SHARDED) return fail(MSREP_ERR_STATE, "SHARDED layout is for pCSC / column-sorted pCOO");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const double alpha = get_scalar(alpha_p, c->dtype), beta = get_scalar(beta_p, c->dtype);
  const size_t V = vsz(c->dtype);
  const int dt = c->dtype == MSREP_F64 ? 0 : 1;
  std::vector<int64_t> seg_lo, seg_hi;
  owned_segments(c, seg_lo, seg_hi);
  const int64_t my_lo = seg_lo[(size_t)c->rank], my_hi = seg_hi[(size_t)c->rank];
  const bool gather = layout == MSREP_Y_REPLICATED && c->nranks > 1;

  if (alpha == 0.0) {   // reading R12: y = beta*y, A and x not read
    CUDA_TRY(launch_scale(static_cast<char*>(y) + (size_t)my_lo * V, my_hi - my_lo, beta, dt, s));
    for (int mi = 0; mi < nmirror; mi++)
      if (my_hi > my_lo)
        CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(mirrors[mi]) + (size_t)my_lo * V, static_cast<char*>(y) + (size_t)my_lo * V,
                                 (size_t)(my_hi - my_lo) * V, cudaMemcpyDefault, s));
    if (gather) TRY(allgatherv_y(c, y, seg_lo, seg_hi, s));
    return MSREP_OK;
  }

  if (colwise(c->fmt)) {
    nv.next("spmv: band kernel + reduce-scatter");
    TRY(col_spmv(c, alpha, x, beta, y, 1, 0, my_lo, my_hi, s));
    if (gather) {
      nv.next("spmv: allgatherv");
      TRY(allgatherv_y(c, y, seg_lo, seg_hi, s));
    }
    return MSREP_OK;
  }

  nv.next("spmv: compact x gather");
  TRY(prepare_x(c, x, 1, s));
  nv.next("spmv: tile kernel");
  RowLaunch L = row_launch(c, x, y, alpha, beta);
  L.nmirror = nmirror;
  for (int mi = 0; mi < nmirror; mi++) L.mirror[mi] = mirrors[mi];
  cudaEvent_t pe;
  TRY(prof_begin(c, s, &pe));
  TRY(row_tiles_pass(c, L, 1, s));
  if (pe) CUDA_TRY(cudaEventRecord(pe, s));
  if (c->nranks > 1 && c->any_flag) {
    nv.next("spmv: head exchange");
    HeadLaunch H{c->vparts, c->d_part_rec, c->d_rec, c->d_head_local, 1};
    CUDA_TRY(launch_heads(H, s));
    TRY(comm_allgather(c, c->d_head_local, c->d_head_all, (size_t)c->vparts, s));
  }
  if (c->nsplit) {
    nv.next("spmv: fix-up");
    TRY(fixup_pass(c, y, alpha, beta, 1, nmirror, mirrors, c->d_rec, c->d_head_all, s));
  }
  if (gather) {
    nv.next("spmv: allgatherv");
    TRY(allgatherv_y(c, y, seg_lo, seg_hi, s));
  }
  return MSREP_OK;
}

msrep_status_t msrep_spmm(msrep_ctx h, const void* alpha_p, const void* X, const void* beta_p, void* Y, int k,
                          msrep_layout layout, void* stream) {
  if (!h) return fail(MSREP_ERR_INVALID_ARG, "ctx is NULL");
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (!c->ready) return fail(MSREP_ERR_STATE, "msrep_spmm before msrep_partition");
  if (k != 2 && k != 4 && k != 8) return fail(MSREP_ERR_INVALID_ARG, "k = %d (must be 2, 4 or 8)", k);
  if (!alpha_p || !beta_p || (c->m > 0 && !Y) || (c->n > 0 && !X)) return fail(MSREP_ERR_INVALID_ARG, "NULL argument");
  if (colwise(c->fmt) ? (layout != MSREP_Y_REPLICATED && layout != MSREP_Y_SHARDED)
                      : (layout != MSREP_Y_REPLICATED && layout != MSREP_Y_OWNED))
    return fail(MSREP_ERR_INVALID_ARG, "layout %d for this format", (int)layout);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const double alpha = get_scalar(alpha_p, c->dtype), beta = get_scalar(beta_p, c->dtype);
  const size_t V = vsz(c->dtype);
  const int dt = c->dtype == MSREP_F64 ? 0 : 1;
  std::vector<int64_t> seg_lo, seg_hi;
  owned_segments(c, seg_lo, seg_hi);
  const int64_t my_lo = seg_lo[(size_t)c->rank], my_hi = seg_hi[(size_t)c->rank];
  const bool gather = layout == MSREP_Y_REPLICATED && c->nranks > 1;
  if (alpha == 0.0) {   // reading R12: Y = beta*Y, A and X not read
    CUDA_TRY(launch_scale(static_cast<char*>(Y) + (size_t)my_lo * k * V, (my_hi - my_lo) * k, beta, dt, s));
    if (gather) TRY(allgatherv_y(c, Y, seg_lo, seg_hi, s, k));
    return MSREP_OK;
  }
  if (colwise(c->fmt) && !(c->col_rows && c->nranks == 1)) {
    // column formats: X and Y go planar (k contiguous vectors), one SpMV pass of the band kernel
    // (and its merge) per vector, and Y back to row-major -- strided gathers / stores of the row-major
    // block directly were slower than k SpMVs (stencil k = 8: 0.64x)
    const size_t nx = (size_t)std::max<int64_t>(1, c->n), ny = (size_t)std::max<int64_t>(1, c->m);
    if (c->mm_planar_bytes < (nx + ny) * (size_t)k * V) {
      void* q;
      TRY(dalloc(c, (nx + ny) * 8 * V, &q, s));   // room for k <= 8
      c->d_mm_planar = q;
      c->mm_planar_bytes = (nx + ny) * 8 * V;
    }
    char* xt = static_cast<char*>(c->d_mm_planar);
    char* yt = xt + nx * (size_t)k * V;
    CUDA_TRY(launch_planar(X, xt, 0, c->n, k, (int64_t)nx, 1, dt, s));
    if (beta != 0.0) CUDA_TRY(launch_planar(Y, yt, my_lo, my_hi, k, (int64_t)ny, 1, dt, s));
    for (int j = 0; j < k; j++)
      TRY(col_spmv(c, alpha, xt + (size_t)j * nx * V, beta, yt + (size_t)j * ny * V, 1, 0, my_lo, my_hi, s));
    CUDA_TRY(launch_planar(yt, Y, my_lo, my_hi, k, (int64_t)ny, 0, dt, s));
    if (gather) TRY(allgatherv_y(c, Y, seg_lo, seg_hi, s, k));
    return MSREP_OK;
  }
  if (c->mm_k < k) {   // k-wide records and head partials, allocated on first use
    void* q;
    TRY(dalloc(c, (size_t)std::max(1, c->nrec) * 8 * 8, &q, s)); c->d_rec_mm = static_cast<double*>(q);
    TRY(dalloc(c, (size_t)c->vparts * 8 * 8, &q, s)); c->d_head_local_mm = static_cast<double*>(q);
    if (c->nranks > 1) { TRY(dalloc(c, (size_t)c->np * 8 * 8, &q, s)); c->d_head_all_mm = static_cast<double*>(q); }
    c->mm_k = 8;
  }
  // row formats, and column formats on row tiles at one rank (y written directly, no merge)
  RowLaunch L{};
  L.tiles = c->d_tiles; L.ntiles = c->ntiles;
  L.blob = c->d_blob;
  L.x = static_cast<const char*>(X) + (size_t)c->xoff * k * V; L.y = Y; L.ybase = c->ybase;
  L.xmax = c->xn > 0 ? (uint32_t)(c->xn - 1) : 0u;
  L.alpha = alpha; L.beta = beta; L.rec = c->d_rec_mm;
  L.dtype = dt; L.has_sell = c->nsell > 0;
  L.hot = c->d_hot; L.nhot = c->nhot;   // SpMM untags hot column ids through the list (no shared-memory cache)
  TRY(prepare_x(c, X, k, s));
  if (c->nxc) { L.x = c->d_xc_mm; L.xmax = (uint32_t)(c->nxc - 1); }
  cudaEvent_t pe;
  TRY(prof_begin(c, s, &pe));
  TRY(row_tiles_pass(c, L, k, s));
  if (pe) CUDA_TRY(cudaEventRecord(pe, s));
  if (c->nranks > 1 && c->any_flag) {
    HeadLaunch H{c->vparts, c->d_part_rec, c->d_rec_mm, c->d_head_local_mm, k};
    CUDA_TRY(launch_heads(H, s));
    TRY(comm_allgather(c, c->d_head_local_mm, c->d_head_all_mm, (size_t)c->vparts * k, s));
  }
  if (c->nsplit) TRY(fixup_pass(c, Y, alpha, beta, k, 0, nullptr, c->d_rec_mm, c->d_head_all_mm, s));
  if (gather) TRY(allgatherv_y(c, Y, seg_lo, seg_hi, s, k));
  return MSREP_OK;
}

// Pipelined host-vector SpMV (one rank, one part, device-resident row tiles -- pCSR, pCOO, or a
// column format on row tiles): x goes up whole (any tile may
// gather any column), then y_in in HOST_CHUNKS row chunks on the copy stream; chunk k's tiles run as
// soon as its y_in is there, its split rows are fixed up right after, and its y rows go down on a
// second copy stream while the next chunks go up and compute (PCIe is full duplex).  Chunks end on
// tile boundaries that are row boundaries and never cut a split row.
#ifndef MSREP_HOST_CHUNKS
#define MSREP_HOST_CHUNKS 16
#endif
constexpr int HOST_CHUNKS = MSREP_HOST_CHUNKS;
bool host_pipeline_ok(const Ctx* c) {
  return c->nranks == 1 && c->vparts == 1 && c->residency == MSREP_RESIDENT_DEVICE && c->ntiles >= 2 * HOST_CHUNKS &&
         (!colwise(c->fmt) || c->col_rows) && (int64_t)c->h_tile_row0.size() == c->ntiles;
}
// Row chunks over both tile lists (SELL tiles [0, nsell) and SEG / slab tiles [nsell, ntiles), each in
// row order): the cuts are tile-start rows of the merged order, so no tile and no split row (its
// slabs share their first row) straddles a cut; chunk k runs its SELL range and its SEG range.
msrep_status_t build_host_chunks(Ctx* c) {
  c->hchunks.clear();
  const int nt = c->ntiles, ns = c->nsell;
  const int32_t* r0s = c->h_tile_row0.data();
  std::vector<int32_t> merged;
  merged.reserve((size_t)nt);
  std::merge(r0s, r0s + ns, r0s + ns, r0s + nt, std::back_inserter(merged));
  std::vector<int32_t> cut{merged.empty() ? 0 : merged[0]};
  for (int k = 1; k < HOST_CHUNKS; k++) {
    const int32_t r = merged[(size_t)((int64_t)k * nt / HOST_CHUNKS)];
    if (r > cut.back()) cut.push_back(r);
  }
  const int64_t rend = c->m;   // one rank, one part: the tiles cover rows [0, m) of y
  for (size_t k = 0; k < cut.size(); k++) {
    const bool last = k + 1 == cut.size();
    const int32_t a = cut[k], b = last ? INT32_MAX : cut[k + 1];
    Ctx::HostChunk hc{};
    hc.t0 = (int32_t)(std::lower_bound(r0s, r0s + ns, a) - r0s);
    hc.t1 = (int32_t)(std::lower_bound(r0s, r0s + ns, b) - r0s);
    hc.u0 = (int32_t)(std::lower_bound(r0s + ns, r0s + nt, a) - r0s);
    hc.u1 = (int32_t)(std::lower_bound(r0s + ns, r0s + nt, b) - r0s);
    if (k == 0) { hc.t0 = 0; hc.u0 = ns; }
    hc.r0 = k == 0 ? 0 : c->ybase + a;
    hc.r1 = last ? rend : c->ybase + b;
    hc.s0 = (int32_t)(std::lower_bound(c->h_sr_row.begin(), c->h_sr_row.end(), hc.r0) - c->h_sr_row.begin());
    hc.s1 = (int32_t)(std::lower_bound(c->h_sr_row.begin(), c->h_sr_row.end(), hc.r1) - c->h_sr_row.begin());
    c->hchunks.push_back(hc);
  }
  // streams of their own (the host-resident mode's copy stream comes with its events: ensure_copy_stream)
  if (!c->cs_in) CUDA_TRY(cudaStreamCreateWithFlags(&c->cs_in, cudaStreamNonBlocking));
  if (!c->cs_out) CUDA_TRY(cudaStreamCreateWithFlags(&c->cs_out, cudaStreamNonBlocking));
  const size_t ne = 1 + 2 * c->hchunks.size() + 1;
  while (c->hev.size() < ne) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->hev.push_back(e);
  }
  return MSREP_OK;
}
msrep_status_t spmv_host_pipelined(Ctx* c, double alpha, const void* x_host, double beta, void* y_host, cudaStream_t s) {
  const size_t V = vsz(c->dtype);
  if (c->hchunks.empty()) TRY(build_host_chunks(c));
  const size_t C = c->hchunks.size();
  cudaEvent_t* ev = c->hev.data();
  // the caller's stream may still use d_hx / d_hy from an earlier call: copies start after it
  CUDA_TRY(cudaEventRecord(ev[2 * C + 1], s));
  CUDA_TRY(cudaStreamWaitEvent(c->cs_in, ev[2 * C + 1], 0));
  CUDA_TRY(cudaStreamWaitEvent(c->cs_out, ev[2 * C + 1], 0));
  if (c->n) CUDA_TRY(cudaMemcpyAsync(c->d_hx, x_host, (size_t)c->n * V, cudaMemcpyHostToDevice, c->cs_in));
  CUDA_TRY(cudaEventRecord(ev[0], c->cs_in));
  for (size_t k = 0; k < C; k++) {
    const Ctx::HostChunk& hc = c->hchunks[k];
    if (beta != 0.0 && hc.r1 > hc.r0)
      CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(c->d_hy) + hc.r0 * V, static_cast<const char*>(y_host) + hc.r0 * V,
                               (size_t)(hc.r1 - hc.r0) * V, cudaMemcpyHostToDevice, c->cs_in));
    CUDA_TRY(cudaEventRecord(ev[1 + k], c->cs_in));
  }
  CUDA_TRY(cudaStreamWaitEvent(s, ev[0], 0));
  TRY(prepare_x(c, c->d_hx, 1, s));
  const RowLaunch L = row_launch(c, c->d_hx, c->d_hy, alpha, beta);
  for (size_t k = 0; k < C; k++) {
    const Ctx::HostChunk& hc = c->hchunks[k];
    CUDA_TRY(cudaStreamWaitEvent(s, ev[1 + k], 0));
    if (hc.t1 > hc.t0) {   // the chunk's SELL tiles
      RowLaunch Lk = L;
      Lk.tiles = c->d_tiles + hc.t0;
      Lk.ntiles = hc.t1 - hc.t0;
      CUDA_TRY(launch_rows(Lk, s));
    }
    if (hc.u1 > hc.u0) {   // its SEG / slab tiles, in the SEG instantiation
      RowLaunch Lk = L;
      Lk.tiles = c->d_tiles + hc.u0;
      Lk.ntiles = hc.u1 - hc.u0;
      Lk.has_sell = 0;
      CUDA_TRY(launch_rows(Lk, s));
    }
    TRY(fixup_pass(c, c->d_hy, alpha, beta, 1, 0, nullptr, c->d_rec, c->d_head_all, s, hc.s0, hc.s1));
    CUDA_TRY(cudaEventRecord(ev[1 + C + k], s));
    CUDA_TRY(cudaStreamWaitEvent(c->cs_out, ev[1 + C + k], 0));
    if (hc.r1 > hc.r0)
      CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(y_host) + hc.r0 * V, static_cast<char*>(c->d_hy) + hc.r0 * V,
                               (size_t)(hc.r1 - hc.r0) * V, cudaMemcpyDeviceToHost, c->cs_out));
  }
  CUDA_TRY(cudaEventRecord(ev[2 * C + 1], c->cs_out));
  CUDA_TRY(cudaStreamWaitEvent(s, ev[2 * C + 1], 0));
  return MSREP_OK;
}

msrep_status_t msrep_spmv_host(msrep_ctx h, const void* alpha, const void* x_host, const void* beta, void* y_host,
                               msrep_layout layout, void* stream) {
  if (!h) return fail(MSREP_ERR_INVALID_ARG, "ctx is NULL");
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (!c->ready) return fail(MSREP_ERR_STATE, "msrep_spmv_host before msrep_partition");
  if (!alpha || !beta) return fail(MSREP_ERR_INVALID_ARG, "alpha/beta NULL");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t V = vsz(c->dtype);
  if (!c->d_hx) {
    TRY(dalloc(c, (size_t)std::max<int64_t>(1, c->n) * V, &c->d_hx, s));
    TRY(dalloc(c, (size_t)std::max<int64_t>(1, c->m) * V, &c->d_hy, s));
  }
  std::vector<int64_t> lo, hi;
  owned_segments(c, lo, hi);
  int64_t r0 = lo[(size_t)c->rank], r1 = hi[(size_t)c->rank];
  if (layout == MSREP_Y_REPLICATED) { r0 = 0; r1 = c->m; }
  const double b = get_scalar(beta, c->dtype);
  const double a = get_scalar(alpha, c->dtype);
  const bool layout_ok = (layout == MSREP_Y_REPLICATED || layout == MSREP_Y_OWNED || layout == MSREP_Y_SHARDED) &&
                         !(colwise(c->fmt) && layout == MSREP_Y_OWNED) && !(!colwise(c->fmt) && layout == MSREP_Y_SHARDED);
  if (a != 0.0 && layout_ok && host_pipeline_ok(c)) {   // (bad layouts take the plain path, which reports them)
    TRY(spmv_host_pipelined(c, a, x_host, b, y_host, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return MSREP_OK;
  }
  if (c->n) CUDA_TRY(cudaMemcpyAsync(c->d_hx, x_host, (size_t)c->n * V, cudaMemcpyHostToDevice, s));
  // y_in: the rows this rank updates (REPLICATED multi-rank: its own segment is enough, peers send the rest)
  const int64_t i0 = lo[(size_t)c->rank], i1 = hi[(size_t)c->rank];
  if (b != 0.0 && i1 > i0)
    CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(c->d_hy) + i0 * V, static_cast<const char*>(y_host) + i0 * V,
                             (size_t)(i1 - i0) * V, cudaMemcpyHostToDevice, s));
  TRY(msrep_spmv(h, alpha, c->d_hx, beta, c->d_hy, layout, stream));
  if (r1 > r0)
    CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(y_host) + r0 * V, static_cast<char*>(c->d_hy) + r0 * V,
                             (size_t)(r1 - r0) * V, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return MSREP_OK;
}

msrep_status_t msrep_cg(msrep_ctx h, const void* b, void* x, double tol, int maxit, int check_every,
                        int* iters_out, double* relres_out, void* stream) {
  if (!h) return fail(MSREP_ERR_INVALID_ARG, "ctx is NULL");
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (!c->ready) return fail(MSREP_ERR_STATE, "msrep_cg before msrep_partition");
  if (c->m != c->n) return fail(MSREP_ERR_DIM_MISMATCH, "CG needs a square matrix (m %lld, n %lld)", (long long)c->m, (long long)c->n);
  if ((c->m > 0 && (!b || !x)) || maxit < 0 || !(tol >= 0.0)) return fail(MSREP_ERR_INVALID_ARG, "bad CG arguments");
  if (check_every < 1) check_every = 1;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t V = vsz(c->dtype);
  const int dt = c->dtype == MSREP_F64 ? 0 : 1;
  if (!c->d_cg_r) {
    void* q;
    TRY(dalloc(c, (size_t)std::max<int64_t>(1, c->m) * V, &q, s)); c->d_cg_r = q;
    TRY(dalloc(c, (size_t)std::max<int64_t>(1, c->m) * V, &q, s)); c->d_cg_p = q;
    TRY(dalloc(c, (size_t)std::max<int64_t>(1, c->m) * V, &q, s)); c->d_cg_ap = q;
    TRY(dalloc(c, (size_t)2 * CG_PARTS * 8, &q, s)); c->d_cg_part = static_cast<double*>(q);
    TRY(dalloc(c, 8 * 8, &q, s)); c->d_cg_sc = static_cast<double*>(q);
  }
  std::vector<int64_t> seg_lo, seg_hi;
  owned_segments(c, seg_lo, seg_hi);
  const int64_t lo = seg_lo[(size_t)c->rank], nloc = seg_hi[(size_t)c->rank] - lo;
  const msrep_layout lay = colwise(c->fmt) ? MSREP_Y_SHARDED : MSREP_Y_OWNED;
  double one64 = 1.0, zero64 = 0.0;
  float one32 = 1.0f, zero32 = 0.0f;
  const void* one = dt == 0 ? (const void*)&one64 : (const void*)&one32;
  const void* zero = dt == 0 ? (const void*)&zero64 : (const void*)&zero32;
  auto off = [&](const void* v) { return static_cast<char*>(const_cast<void*>(v)) + (size_t)lo * V; };
  double* sc = c->d_cg_sc;
  double* p1 = c->d_cg_part;              // partial sums of p.Ap (and of r0.r0, b.b at the start)
  double* p2 = c->d_cg_part + CG_PARTS;   // partial sums of r.r
  auto allreduce_parts = [&](double* part) -> msrep_status_t {   // same partials on every rank
    if (c->nranks > 1) TRY(comm_allreduce(c, part, CG_PARTS, false, s));
    return MSREP_OK;
  };
  // r0 = b - A x0, p0 = r0, rs = r0.r0 (sc[0], parity 0), bnorm2 = b.b (sc[3])
  TRY(msrep_spmv(h, one, x, zero, c->d_cg_ap, lay, stream));
  CUDA_TRY(launch_cg(CG_RESIDUAL, dt, off(b), off(c->d_cg_ap), off(c->d_cg_r), off(c->d_cg_p), nloc, sc, 0, nullptr, p1, s));
  TRY(allreduce_parts(p1));
  CUDA_TRY(launch_cg(CG_SUM, dt, nullptr, nullptr, nullptr, nullptr, 0, sc + 0, 0, p1, nullptr, s));
  CUDA_TRY(launch_cg(CG_DOT, dt, off(b), off(b), nullptr, nullptr, nloc, sc, 0, nullptr, p2, s));
  TRY(allreduce_parts(p2));
  CUDA_TRY(launch_cg(CG_SUM, dt, nullptr, nullptr, nullptr, nullptr, 0, sc + 3, 0, p2, nullptr, s));
  double hs[4] = {0, 0, 0, 0};
  CUDA_TRY(cudaMemcpyAsync(hs, sc, 4 * 8, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  const double bn2 = hs[3], stop = tol * tol * bn2;
  double rs = hs[0];
  int it = 0;
  std::vector<int64_t> lo_v = seg_lo, hi_v = seg_hi;
  // one iteration: SpMV, dot(p, Ap), update x and r (+ r.r), update p (+ rs) -- four launches;
  // the scalars alternate between sc[0] and sc[1] (par), so two iterations are one period
  auto iter = [&](int par, cudaStream_t st) -> msrep_status_t {
    if (c->nranks > 1) TRY(allgatherv_y(c, c->d_cg_p, lo_v, hi_v, st));   // the SpMV needs the whole p
    TRY(msrep_spmv(h, one, c->d_cg_p, zero, c->d_cg_ap, lay, st));        // Ap, owned rows
    CUDA_TRY(launch_cg(CG_DOT, dt, off(c->d_cg_p), off(c->d_cg_ap), nullptr, nullptr, nloc, sc, par, nullptr, p1, st));
    if (c->nranks > 1) TRY(comm_allreduce(c, p1, CG_PARTS, false, st));
    CUDA_TRY(launch_cg(CG_UPDATE_XR, dt, off(x), off(c->d_cg_r), off(c->d_cg_p), off(c->d_cg_ap), nloc, sc, par, p1, p2, st));
    if (c->nranks > 1) TRY(comm_allreduce(c, p2, CG_PARTS, false, st));
    CUDA_TRY(launch_cg(CG_UPDATE_P, dt, off(c->d_cg_p), off(c->d_cg_r), nullptr, nullptr, nloc, sc, par, p2, nullptr, st));
    return MSREP_OK;
  };
  auto check = [&](cudaStream_t st) -> msrep_status_t {   // sc[it & 1] = r.r after iteration it
    CUDA_TRY(cudaMemcpyAsync(hs, sc, 4 * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (std::isnan(hs[it & 1])) return fail(MSREP_ERR_STATE, "CG breakdown at iteration %d (matrix not SPD?)", it);
    rs = hs[it & 1];
    return MSREP_OK;
  };
  // CUDA graph of one period (two iterations, eight launches) replayed on a context stream: the
  // iteration is launch-bound for small systems (pCSR 110K rows: 0.0228 -> 0.0181 ms/iteration;
  // 2M rows: 0.152 -> 0.147, profiles/r1_cg_graph.jsonl).  Single rank, device-resident, row tiles
  // (row formats and column formats on row tiles; a replayed row-band pCSC iteration measured 30 %
  // slower than eager), profiling off;
  // msrep_set_tuning(MSREP_TUNE_CG_GRAPH, 0) disables it.  The convergence check then runs every 2*ceil(check_every/2)
  // iterations; the iterates are the same kernels in the same order as the eager loop.
  const bool graph = c->nranks == 1 && c->residency == MSREP_RESIDENT_DEVICE && (!colwise(c->fmt) || c->col_rows) && !c->prof &&
                     maxit >= 8 && c->tune_cg_graph;
  if (graph && !(rs <= stop)) {
    if (!c->gs) CUDA_TRY(cudaStreamCreateWithFlags(&c->gs, cudaStreamNonBlocking));
    cudaEvent_t ev;
    CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(ev, s));
    CUDA_TRY(cudaStreamWaitEvent(c->gs, ev, 0));   // the setup above precedes the replays
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    CUDA_TRY(cudaStreamBeginCapture(c->gs, cudaStreamCaptureModeThreadLocal));
    msrep_status_t cs = iter(0, c->gs);
    if (cs == MSREP_OK) cs = iter(1, c->gs);
    cudaError_t ce = cudaStreamEndCapture(c->gs, &g);
    if (cs != MSREP_OK) { if (g) cudaGraphDestroy(g); cudaEventDestroy(ev); return cs; }
    CUDA_TRY(ce);
    CUDA_TRY(cudaGraphInstantiate(&ge, g, 0));
    const int ce2 = 2 * ((check_every + 1) / 2);
    msrep_status_t st = MSREP_OK;
    while (st == MSREP_OK && !(rs <= stop) && it + 2 <= maxit) {
      if (cudaGraphLaunch(ge, c->gs) != cudaSuccess) { st = fail(MSREP_ERR_CUDA, "cudaGraphLaunch"); break; }
      it += 2;
      if (it % ce2 == 0 || it + 2 > maxit) st = check(c->gs);
    }
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    if (st != MSREP_OK) { cudaEventDestroy(ev); return st; }
    CUDA_TRY(cudaEventRecord(ev, c->gs));
    CUDA_TRY(cudaStreamWaitEvent(s, ev, 0));       // the caller's stream sees the iterates
    CUDA_TRY(cudaEventDestroy(ev));
  }
  while (!(rs <= stop) && it < maxit) {   // eager loop (and the odd last iteration after graphs)
    TRY(iter(it & 1, s));
    it++;
    if (it % check_every == 0 || it == maxit) TRY(check(s));
  }
  if (c->nranks > 1) TRY(allgatherv_y(c, x, lo_v, hi_v, s));   // x replicated on exit
  CUDA_TRY(cudaStreamSynchronize(s));
  if (iters_out) *iters_out = it;
  if (relres_out) *relres_out = bn2 > 0.0 ? std::sqrt(rs / bn2) : std::sqrt(rs);
  return MSREP_OK;
}

msrep_status_t msrep_profile_enable(msrep_ctx h, int enable) {
  if (!h) return fail(MSREP_ERR_INVALID_ARG, "ctx is NULL");
  reinterpret_cast<Ctx*>(h)->prof = enable != 0;
  return MSREP_OK;
}

msrep_status_t msrep_profile_read(msrep_ctx h, double* kernel_ms, int64_t* launches, int reset) {
  if (!h || !kernel_ms || !launches) return fail(MSREP_ERR_INVALID_ARG, "NULL argument");
  Ctx* c = reinterpret_cast<Ctx*>(h);
  double tot = 0.0;
  for (size_t i = 0; i < c->ev_used; i++) {
    CUDA_TRY(cudaEventSynchronize(c->ev[i].second));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, c->ev[i].first, c->ev[i].second));
    tot += ms;
  }
  *kernel_ms = tot;
  *launches = (int64_t)c->ev_used;
  if (reset) c->ev_used = 0;
  return MSREP_OK;
}

msrep_status_t msrep_get_stats(msrep_ctx h, msrep_stats* out) {
  if (!h || !out) return fail(MSREP_ERR_INVALID_ARG, "NULL argument");
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (!c->ready) return fail(MSREP_ERR_STATE, "no partition");
  *out = c->stats;
  return MSREP_OK;
}

}  // extern "C"
