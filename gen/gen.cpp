// gen/gen.cpp -- seeded synthetic sparse-matrix generators.
//
// Shared by the oracle tests and the CUDA path as INPUT ONLY: this file holds
// none of the method's arithmetic (no SpMV, no partitioning, no merge).  Every
// row (or CSC column) is a pure function of (seed, row): a counter-based hash
// (splitmix64 finaliser over the tuple) drives every random choice, so the
// result is identical for any thread count, and the same (row, col) entry has
// the same value whichever format it is emitted in.
//
// Shapes follow SURVEY.md 8(d) (configs 1-5, the paper's Table 2 shapes
// P:628-643 and the power-law selection rule P(k) ~ k^-R).
//
// API pattern: <gen>_count(params, counts[m]) then <gen>_fill(params,
// row_ptr[m+1], col[nnz], val[nnz]); the caller forms row_ptr from counts.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <thread>
#include <vector>

namespace {

inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline uint64_t h2(uint64_t seed, uint64_t a) { return mix64(mix64(seed) ^ a); }
inline uint64_t h3(uint64_t seed, uint64_t a, uint64_t b) { return mix64(h2(seed, a) ^ (b * 0xD6E8FEB86659FD93ull)); }
inline uint64_t h4(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return mix64(h3(seed, a, b) ^ (c * 0xA0761D6478BD642Full));
}
inline double u01(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

// value of entry (r, c): kind 0 = U[-1,1), 1 = integer in {-4..-1,1..4},
// 2 = 1.0, 3 = 27-point-stencil pin (26 on the diagonal, -1 elsewhere).
inline double entry_value(uint64_t seed, int kind, int64_t r, int64_t c) {
  switch (kind) {
    case 0: return 2.0 * u01(h3(seed ^ 0x5A5Aull, (uint64_t)r, (uint64_t)c)) - 1.0;
    case 1: { int v = (int)(h3(seed ^ 0x1234ull, (uint64_t)r, (uint64_t)c) % 8); return v < 4 ? (double)(v - 4) : (double)(v - 3); }
    case 2: return 1.0;
    default: return r == c ? 26.0 : -1.0;
  }
}

int nthreads() {
  const char* e = std::getenv("MSREP_GEN_THREADS");
  if (e && std::atoi(e) > 0) return std::atoi(e);
  unsigned h = std::thread::hardware_concurrency();
  return h ? (int)h : 4;
}

template <class F>
void parallel_rows(int64_t m, F f) {
  int T = nthreads();
  if (m < 4096) T = 1;
  std::atomic<int64_t> next{0};
  const int64_t chunk = 4096;
  auto work = [&]() {
    std::vector<int64_t> scratch;
    for (;;) {
      int64_t r0 = next.fetch_add(chunk);
      if (r0 >= m) break;
      int64_t r1 = std::min(m, r0 + chunk);
      for (int64_t r = r0; r < r1; r++) f(r, scratch);
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < T; t++) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
}

// k distinct uniform columns in [0, n) for outer index r, sorted.
void k_distinct(uint64_t seed, int64_t r, int64_t n, int64_t k, std::vector<int64_t>& s) {
  s.clear();
  if (k >= n) { for (int64_t c = 0; c < n; c++) s.push_back(c); return; }
  uint64_t attempt = 0;
  while ((int64_t)s.size() < k) {
    int64_t need = k - (int64_t)s.size();
    for (int64_t q = 0; q < need; q++) s.push_back((int64_t)(h3(seed, (uint64_t)r, attempt++) % (uint64_t)n));
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
  }
}

// ---------------------------------------------------------------- R-MAT
// Graph500 R-MAT (a,b,c,d) sampled row by row: the row marginal of a cell is
// prod over levels of (a+b | c+d); given the row bits, each column bit is 0
// with probability a/(a+b) (row bit 0) or c/(c+d) (row bit 1).  The number of
// samples landing in row r is Poisson(E * P(r)) (the multinomial's marginal,
// Poisson-approximated); samples are then deduplicated within the row.
struct Rmat { int scale; double edges, a, b, c; uint64_t seed; };

int64_t poisson(uint64_t seed, int64_t r, double lam) {
  if (lam <= 0) return 0;
  if (lam < 40.0) {
    double L = std::exp(-lam), p = 1.0; int64_t k = 0; uint64_t ctr = 0;
    for (;;) { p *= u01(h3(seed ^ 0x77ull, (uint64_t)r, ctr++)); if (p <= L) return k; k++; }
  }
  double u1 = u01(h3(seed ^ 0x99ull, (uint64_t)r, 0)), u2 = u01(h3(seed ^ 0x99ull, (uint64_t)r, 1));
  if (u1 < 1e-300) u1 = 1e-300;
  double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  double v = std::floor(lam + std::sqrt(lam) * z + 0.5);
  return v < 0 ? 0 : (int64_t)v;
}

void rmat_row(const Rmat& P, int64_t r, std::vector<int64_t>& s) {
  double pr = 1.0;
  const double ab = P.a + P.b, cd = 1.0 - ab;
  for (int l = 0; l < P.scale; l++) pr *= ((r >> (P.scale - 1 - l)) & 1) ? cd : ab;
  int64_t deg = poisson(P.seed, r, P.edges * pr);
  const uint32_t t0 = (uint32_t)std::llround(P.a / ab * 65536.0);            // P(col bit 0 | row bit 0)
  const uint32_t t1 = (uint32_t)std::llround(P.c / (1.0 - ab) * 65536.0);    // P(col bit 0 | row bit 1)
  s.resize((size_t)deg);
  for (int64_t q = 0; q < deg; q++) {
    int64_t col = 0;
    uint64_t h = 0;
    for (int l = 0; l < P.scale; l++) {
      if ((l & 3) == 0) h = h4(P.seed, (uint64_t)r, (uint64_t)q, (uint64_t)(l >> 2));
      uint32_t u = (uint32_t)(h & 0xFFFF); h >>= 16;
      int rb = (int)((r >> (P.scale - 1 - l)) & 1);
      int cb = u < (rb ? t1 : t0) ? 0 : 1;
      col = (col << 1) | cb;
    }
    s[(size_t)q] = col;
  }
  std::sort(s.begin(), s.end());
  s.erase(std::unique(s.begin(), s.end()), s.end());
}

// Optional vertex relabelling (the "permuted" R-MAT variant): a 4-round
// Feistel bijection on [0, 2^scale) (scale even or odd handled by cycle-walk).
struct Feistel {
  int bits; uint64_t seed;
  int half() const { return (bits + 1) / 2; }
  uint64_t enc1(uint64_t v) const {
    int hb = half(); uint64_t mask = (1ull << hb) - 1;
    uint64_t L = v >> hb, R = v & mask;
    for (int k = 0; k < 4; k++) { uint64_t F = h3(seed, (uint64_t)k, R) & mask; uint64_t t = R; R = L ^ F; L = t; }
    return (L << hb) | R;
  }
  uint64_t dec1(uint64_t v) const {
    int hb = half(); uint64_t mask = (1ull << hb) - 1;
    uint64_t L = v >> hb, R = v & mask;
    for (int k = 3; k >= 0; k--) { uint64_t t = L; L = R ^ (h3(seed, (uint64_t)k, t) & mask); R = t; }
    return (L << hb) | R;
  }
  uint64_t enc(uint64_t v) const { uint64_t n = 1ull << bits; do { v = enc1(v); } while (v >= n); return v; }
  uint64_t dec(uint64_t v) const { uint64_t n = 1ull << bits; do { v = dec1(v); } while (v >= n); return v; }
};

void rmat_row_perm(const Rmat& P, int permute, int64_t r, std::vector<int64_t>& s) {
  if (!permute) { rmat_row(P, r, s); return; }
  Feistel f{P.scale, P.seed ^ 0xFEEDull};
  rmat_row(P, (int64_t)f.dec((uint64_t)r), s);
  for (auto& c : s) c = (int64_t)f.enc((uint64_t)c);
  std::sort(s.begin(), s.end());
}

// ---------------------------------------------------------- power-law cols
// Column degree k drawn from P(k) ~ k^-R on [1, kmax] by inverse CDF
// (SPEC S:417-418); rows uniform, distinct within a column.  This
// generator emits CSC (outer index = column); the caller converts as needed.
struct PowerLaw { int64_t m; double R; int64_t kmax; uint64_t seed; };

int64_t powerlaw_degree(const PowerLaw& P, int64_t c, const std::vector<double>& cdf) {
  double u = u01(h2(P.seed ^ 0xABCDull, (uint64_t)c));
  auto it = std::lower_bound(cdf.begin(), cdf.end(), u);
  int64_t k = (int64_t)(it - cdf.begin()) + 1;
  return std::min<int64_t>(k, std::min<int64_t>(P.kmax, P.m));
}

std::vector<double> powerlaw_cdf(const PowerLaw& P) {
  std::vector<double> cdf((size_t)P.kmax);
  double s = 0; for (int64_t k = 1; k <= P.kmax; k++) { s += std::pow((double)k, -P.R); cdf[(size_t)k - 1] = s; }
  for (auto& v : cdf) v /= s;
  return cdf;
}

}  // namespace

extern "C" {

// --- config 1 / config 4: exactly k distinct uniform inner indices per outer index.
// transpose=0: outer = row (CSR), value(r,c); transpose=1: outer = column (CSC), value(inner, outer).
void gen_kdistinct_fill(int64_t outer, int64_t inner, int64_t k, uint64_t seed, int kind, int transpose,
                        const int64_t* ptr, int32_t* idx, double* val) {
  parallel_rows(outer, [&](int64_t r, std::vector<int64_t>& s) {
    k_distinct(seed, r, inner, k, s);
    int64_t o = ptr[r];
    for (size_t q = 0; q < s.size(); q++) {
      idx[o + (int64_t)q] = (int32_t)s[q];
      val[o + (int64_t)q] = transpose ? entry_value(seed, kind, s[q], r) : entry_value(seed, kind, r, s[q]);
    }
  });
}

// --- row-dependent k: row r gets ptr[r+1]-ptr[r] distinct uniform columns (two-class imbalance matrices).
void gen_kvar_fill(int64_t outer, int64_t inner, uint64_t seed, int kind, const int64_t* ptr, int32_t* idx, double* val) {
  parallel_rows(outer, [&](int64_t r, std::vector<int64_t>& s) {
    k_distinct(seed, r, inner, ptr[r + 1] - ptr[r], s);
    int64_t o = ptr[r];
    for (size_t q = 0; q < s.size(); q++) { idx[o + (int64_t)q] = (int32_t)s[q]; val[o + (int64_t)q] = entry_value(seed, kind, r, s[q]); }
  });
}

// --- config 2: 27-point stencil on an N^3 grid, lexicographic order (i,j,k), k fastest.
void gen_stencil27_count(int64_t N, int64_t* counts) {
  parallel_rows(N * N * N, [&](int64_t r, std::vector<int64_t>&) {
    int64_t i = r / (N * N), j = (r / N) % N, k = r % N;
    auto c = [N](int64_t v) { return (int64_t)1 + (v > 0) + (v < N - 1); };
    counts[r] = c(i) * c(j) * c(k);
  });
}
void gen_stencil27_fill(int64_t N, uint64_t seed, int kind, const int64_t* ptr, int32_t* idx, double* val) {
  parallel_rows(N * N * N, [&](int64_t r, std::vector<int64_t>&) {
    int64_t i = r / (N * N), j = (r / N) % N, k = r % N, o = ptr[r];
    for (int di = -1; di <= 1; di++) for (int dj = -1; dj <= 1; dj++) for (int dk = -1; dk <= 1; dk++) {
      int64_t a = i + di, b = j + dj, c = k + dk;
      if (a < 0 || a >= N || b < 0 || b >= N || c < 0 || c >= N) continue;
      int64_t col = (a * N + b) * N + c;
      idx[o] = (int32_t)col; val[o] = entry_value(seed, kind, r, col); o++;
    }
  });
}

// --- config 3: R-MAT (Graph500 a,b,c; d = 1-a-b-c), 'edges' samples, deduplicated.
void gen_rmat_count(int scale, double edges, double a, double b, double c, uint64_t seed, int permute,
                    int64_t* counts) {
  Rmat P{scale, edges, a, b, c, seed};
  parallel_rows((int64_t)1 << scale, [&](int64_t r, std::vector<int64_t>& s) {
    rmat_row_perm(P, permute, r, s); counts[r] = (int64_t)s.size();
  });
}
void gen_rmat_fill(int scale, double edges, double a, double b, double c, uint64_t seed, int permute, int kind,
                   const int64_t* ptr, int32_t* idx, double* val) {
  Rmat P{scale, edges, a, b, c, seed};
  parallel_rows((int64_t)1 << scale, [&](int64_t r, std::vector<int64_t>& s) {
    rmat_row_perm(P, permute, r, s);
    int64_t o = ptr[r];
    for (size_t q = 0; q < s.size(); q++) { idx[o + (int64_t)q] = (int32_t)s[q]; val[o + (int64_t)q] = entry_value(seed, kind, r, s[q]); }
  });
}

// --- config 5: banded (half-bandwidth h: columns [r-h, r+h] within [0,n)).
void gen_banded_count(int64_t m, int64_t n, int64_t h, int64_t* counts) {
  parallel_rows(m, [&](int64_t r, std::vector<int64_t>&) {
    int64_t lo = std::max<int64_t>(0, r - h), hi = std::min<int64_t>(n - 1, r + h);
    counts[r] = hi >= lo ? hi - lo + 1 : 0;
  });
}
void gen_banded_fill(int64_t m, int64_t n, int64_t h, uint64_t seed, int kind, const int64_t* ptr, int32_t* idx,
                     double* val) {
  parallel_rows(m, [&](int64_t r, std::vector<int64_t>&) {
    int64_t lo = std::max<int64_t>(0, r - h), hi = std::min<int64_t>(n - 1, r + h), o = ptr[r];
    for (int64_t c = lo; c <= hi; c++) { idx[o] = (int32_t)c; val[o] = entry_value(seed, kind, r, c); o++; }
  });
}

// --- config 5: block-diagonal with dense bs x bs blocks (last block truncated).
void gen_blockdiag_count(int64_t m, int64_t bs, int64_t* counts) {
  parallel_rows(m, [&](int64_t r, std::vector<int64_t>&) {
    int64_t b0 = (r / bs) * bs; counts[r] = std::min<int64_t>(m, b0 + bs) - b0;
  });
}
void gen_blockdiag_fill(int64_t m, int64_t bs, uint64_t seed, int kind, const int64_t* ptr, int32_t* idx, double* val) {
  parallel_rows(m, [&](int64_t r, std::vector<int64_t>&) {
    int64_t b0 = (r / bs) * bs, b1 = std::min<int64_t>(m, b0 + bs), o = ptr[r];
    for (int64_t c = b0; c < b1; c++) { idx[o] = (int32_t)c; val[o] = entry_value(seed, kind, r, c); o++; }
  });
}

// --- config 5: power-law column degrees, emitted as CSC (outer = column).
void gen_powerlaw_csc_count(int64_t m, int64_t n, double R, int64_t kmax, uint64_t seed, int64_t* counts) {
  PowerLaw P{m, R, kmax, seed};
  auto cdf = powerlaw_cdf(P);
  parallel_rows(n, [&](int64_t c, std::vector<int64_t>&) { counts[c] = powerlaw_degree(P, c, cdf); });
}
void gen_powerlaw_csc_fill(int64_t m, int64_t n, double R, int64_t kmax, uint64_t seed, int kind,
                           const int64_t* ptr, int32_t* idx, double* val) {
  PowerLaw P{m, R, kmax, seed};
  auto cdf = powerlaw_cdf(P);
  parallel_rows(n, [&](int64_t c, std::vector<int64_t>& s) {
    int64_t k = powerlaw_degree(P, c, cdf);
    k_distinct(seed ^ 0x5151ull, c, m, k, s);
    int64_t o = ptr[c];
    for (size_t q = 0; q < s.size(); q++) { idx[o + (int64_t)q] = (int32_t)s[q]; val[o + (int64_t)q] = entry_value(seed, kind, s[q], c); }
  });
}

// --- dense vectors: kind 0 = U[-1,1), 1 = integers {-4..4}, 2 = ones.
void gen_vector(int64_t n, uint64_t seed, int kind, double* out) {
  parallel_rows(n, [&](int64_t i, std::vector<int64_t>&) {
    uint64_t h = h2(seed ^ 0xC0FFEEull, (uint64_t)i);
    out[i] = kind == 0 ? 2.0 * u01(h) - 1.0 : kind == 1 ? (double)((int)(h % 9) - 4) : 1.0;
  });
}

// --- transposition (CSR <-> CSC of the same entries) and COO row expansion,
// multithreaded plumbing used to hand the SAME matrix to every format.
// Not the method: the oracle has its own single-threaded conversions.
void gen_expand_ptr(int64_t m, const int64_t* ptr, int32_t* out) {
  parallel_rows(m, [&](int64_t r, std::vector<int64_t>&) { for (int64_t j = ptr[r]; j < ptr[r + 1]; j++) out[j] = (int32_t)r; });
}

// --- rank-local generation: rows (CSC: columns) [r0, r1) only, written from idx / val = the
// buffers of nonzeros [ptr[r0], ptr[r1]) -- each row is a pure function of (seed, row), so a rank
// can build just the rows its nonzero range touches (bench.py with N > 1).
void gen_kdistinct_fill_rows(int64_t outer, int64_t inner, int64_t k, uint64_t seed, int kind, int transpose,
                             int64_t r0, int64_t r1, const int64_t* ptr, int32_t* idx, double* val) {
  (void)outer;
  const int64_t base = ptr[r0];
  parallel_rows(r1 - r0, [&](int64_t q, std::vector<int64_t>& s) {
    const int64_t r = r0 + q;
    k_distinct(seed, r, inner, k, s);
    const int64_t o = ptr[r] - base;
    for (size_t t = 0; t < s.size(); t++) {
      idx[o + (int64_t)t] = (int32_t)s[t];
      val[o + (int64_t)t] = transpose ? entry_value(seed, kind, s[t], r) : entry_value(seed, kind, r, s[t]);
    }
  });
}
void gen_stencil27_fill_rows(int64_t N, uint64_t seed, int kind, int64_t r0, int64_t r1, const int64_t* ptr,
                             int32_t* idx, double* val) {
  const int64_t base = ptr[r0];
  parallel_rows(r1 - r0, [&](int64_t q, std::vector<int64_t>&) {
    const int64_t r = r0 + q;
    int64_t i = r / (N * N), j = (r / N) % N, k = r % N, o = ptr[r] - base;
    for (int di = -1; di <= 1; di++) for (int dj = -1; dj <= 1; dj++) for (int dk = -1; dk <= 1; dk++) {
      int64_t a = i + di, b = j + dj, c = k + dk;
      if (a < 0 || a >= N || b < 0 || b >= N || c < 0 || c >= N) continue;
      int64_t col = (a * N + b) * N + c;
      idx[o] = (int32_t)col; val[o] = entry_value(seed, kind, r, col); o++;
    }
  });
}
void gen_rmat_fill_rows(int scale, double edges, double a, double b, double c, uint64_t seed, int permute, int kind,
                        int64_t r0, int64_t r1, const int64_t* ptr, int32_t* idx, double* val) {
  Rmat P{scale, edges, a, b, c, seed};
  const int64_t base = ptr[r0];
  parallel_rows(r1 - r0, [&](int64_t q, std::vector<int64_t>& s) {
    const int64_t r = r0 + q;
    rmat_row_perm(P, permute, r, s);
    const int64_t o = ptr[r] - base;
    for (size_t t = 0; t < s.size(); t++) { idx[o + (int64_t)t] = (int32_t)s[t]; val[o + (int64_t)t] = entry_value(seed, kind, r, s[t]); }
  });
}

}  // extern "C"

extern "C" {
// Transpose (m x n CSR -> CSC, equivalently CSC -> CSR of the transpose):
// counting sort by inner index, inner order preserved.  Plumbing that hands the
// same matrix to the column format; tests pin it bit-exactly against the
// oracle's own single-threaded conversion.
void gen_transpose(int64_t m, int64_t n, const int64_t* ptr, const int32_t* idx, const double* val,
                   int64_t* tptr, int32_t* tidx, double* tval) {
  int64_t nnz = ptr[m];
  std::vector<int64_t> next((size_t)n + 1, 0);
  for (int64_t c = 0; c <= n; c++) tptr[c] = 0;
  for (int64_t k = 0; k < nnz; k++) tptr[idx[k] + 1]++;
  for (int64_t c = 0; c < n; c++) tptr[c + 1] += tptr[c];
  for (int64_t c = 0; c <= n; c++) next[(size_t)c] = tptr[c];
  for (int64_t r = 0; r < m; r++)
    for (int64_t j = ptr[r]; j < ptr[r + 1]; j++) {
      int64_t d = next[(size_t)idx[j]]++;
      tidx[d] = (int32_t)r; tval[d] = val[j];
    }
}
}  // extern "C"
