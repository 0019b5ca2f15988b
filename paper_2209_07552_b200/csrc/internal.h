// internal.h -- shared definitions between the host runtime (host.cpp) and the
// sm_100a kernels (kernels.cu) of libmsrep.  Not part of the C ABI.
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace msrep {

// A tile is the unit of work one CTA processes: a row-aligned group of whole
// rows whose merge items (rows + nonzeros) fit TILE_ITEMS, or a "slab" -- a
// contiguous piece (<= SLAB_NNZ nonzeros) of one split row whose partial sum
// goes to a record instead of y.  For pCSC, tiles are
// column groups / column pieces and every tile scatters into py.
constexpr int TILE_ITEMS = 2048;
constexpr int SLAB_NNZ = 2047;
constexpr int THREADS = 256;

// int4 tile descriptor: x = first row (window-local), y = first nonzero
// (rank-local), z = nrows | (nnz << 16), w = record index (-1: normal tile).
struct TileHost { int32_t row0, nz0, packed, rec; };

struct RowLaunch {
  const int4* tiles; int ntiles;
  const void* val; const int32_t* col; const int32_t* aux;  // aux: local row ptr (CSR) or global row ids (COO)
  const void* x; void* y; int64_t ybase;                     // y row of window row 0
  double alpha, beta; double* rec;
  int coo; int dtype;                                        // dtype 0 = f64, 1 = f32
  int grid;                                                  // persistent CTAs
};

struct ColLaunch {
  const int4* tiles; int ntiles;
  const void* val; const int32_t* row; const int32_t* cptr;   // cptr: rank-local column pointer (window)
  const void* x; int64_t xbase;                              // x index of window column 0
  double* py;
  int dtype; int grid;
};

struct FixupLaunch {
  int nsplit;
  const int64_t* sr_row; const int32_t* sr_rec;       // sr_rec[2*s], [2*s+1] : record range
  const int32_t* sr_head;                             // sr_head[2*s], [2*s+1]: range into head_list
  const int32_t* head_list;                           // global part ids
  const int32_t* part_rec;                            // part_rec[2*j], [2*j+1]: record range of part j's head (local parts)
  int part_lo, part_hi;                               // local global-part range [lo, hi)
  const double* head_all;                             // head sums of all parts (multi-rank), may be null
  const double* rec;
  void* y; double alpha, beta; int dtype;
};

struct HeadLaunch {
  int nlocal; const int32_t* part_rec; const double* rec; double* head_local;
};

// kernels.cu entry points (all enqueue on `s`)
cudaError_t launch_rows(const RowLaunch& L, cudaStream_t s);
cudaError_t launch_cols(const ColLaunch& L, cudaStream_t s);
cudaError_t launch_fixup(const FixupLaunch& L, cudaStream_t s);
cudaError_t launch_heads(const HeadLaunch& L, cudaStream_t s);
cudaError_t launch_scale(void* y, int64_t count, double beta, int dtype, cudaStream_t s);   // y = beta*y
cudaError_t launch_axpby_py(const double* py, void* y, int64_t count, double alpha, double beta, int dtype,
                            cudaStream_t s);                                                // y = alpha*py + beta*y
cudaError_t launch_rebase(const int64_t* gptr, int32_t* lptr, int64_t count, int64_t lo, int64_t hi,
                          cudaStream_t s);                                                  // clamp(gptr,lo,hi)-lo
int rows_grid(int dtype, int coo, int ntiles);
int cols_grid(int dtype, int ntiles);

}  // namespace msrep
