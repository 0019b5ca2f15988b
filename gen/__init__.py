"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

Holds none of the method's arithmetic: only matrix/vector generation
(gen/gen.cpp, multithreaded C++, counter-based so every row is a pure function
of (seed, row)).  Recipes: DESIGN.md "Input recipe" / SURVEY.md 8(d).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libgen.so")
_SRC = os.path.join(_HERE, "gen.cpp")

# value kinds (gen.cpp entry_value)
UNIFORM, SMALLINT, ONES, STENCIL_PIN = 0, 1, 2, 3


def build() -> str:
    if (not os.path.exists(_SO)) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread", "-o", _SO, _SRC])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P, I64, D, I, U64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int, ctypes.c_uint64
        sig = {
            "gen_kdistinct_fill": [I64, I64, I64, U64, I, I, P, P, P],
            "gen_stencil27_count": [I64, P],
            "gen_stencil27_fill": [I64, U64, I, P, P, P],
            "gen_rmat_count": [I, D, D, D, D, U64, I, P],
            "gen_rmat_fill": [I, D, D, D, D, U64, I, I, P, P, P],
            "gen_banded_count": [I64, I64, I64, P],
            "gen_banded_fill": [I64, I64, I64, U64, I, P, P, P],
            "gen_blockdiag_count": [I64, I64, P],
            "gen_blockdiag_fill": [I64, I64, U64, I, P, P, P],
            "gen_powerlaw_csc_count": [I64, I64, D, I64, U64, P],
            "gen_powerlaw_csc_fill": [I64, I64, D, I64, U64, I, P, P, P],
            "gen_vector": [I64, U64, I, P],
            "gen_kvar_fill": [I64, I64, U64, I, P, P, P],
            "gen_expand_ptr": [I64, P, P],
            "gen_transpose": [I64, I64, P, P, P, P, P, P],
            "gen_kdistinct_fill_rows": [I64, I64, I64, U64, I, I, I64, I64, P, P, P],
            "gen_stencil27_fill_rows": [I64, U64, I, I64, I64, P, P, P],
            "gen_rmat_fill_rows": [I, D, D, D, D, U64, I, I, I64, I64, P, P, P],
        }
        for k, a in sig.items():
            getattr(L, k).argtypes = a
            getattr(L, k).restype = None
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class Sparse(dict):
    """dict with keys: fmt ('csr'|'csc'), m, n, nnz, ptr (int64), idx (int32), val (float64)."""

    @property
    def nnz(self):
        return int(self["ptr"][-1])


def _finish(fmt, m, n, counts, fill):
    outer = counts.size
    ptr = np.zeros(outer + 1, np.int64)
    np.cumsum(counts, out=ptr[1:])
    nnz = int(ptr[-1])
    idx = np.empty(max(nnz, 1), np.int32)[:nnz]
    val = np.empty(max(nnz, 1), np.float64)[:nnz]
    fill(ptr, idx, val)
    return Sparse(fmt=fmt, m=m, n=n, ptr=ptr, idx=idx, val=val)


def kdistinct_csr(m, n, k, seed, kind=UNIFORM):
    """Config 1: exactly k distinct sorted uniform columns per row (seed 1)."""
    counts = np.full(m, min(k, n), np.int64)
    return _finish("csr", m, n, counts,
                   lambda p, i, v: lib().gen_kdistinct_fill(m, n, k, seed, kind, 0, _p(p), _p(i), _p(v)))


def kdistinct_csc(m, n, k, seed, kind=UNIFORM):
    """Config 4: tall-skinny, exactly k distinct sorted uniform rows per column (seed 4)."""
    counts = np.full(n, min(k, m), np.int64)
    return _finish("csc", m, n, counts,
                   lambda p, i, v: lib().gen_kdistinct_fill(n, m, k, seed, kind, 1, _p(p), _p(i), _p(v)))


def two_class(m, n, nblocks, heavy_blocks, k_heavy, ratio, seed=600, kind=UNIFORM):
    """Fig. 6's imbalance workload: m rows in nblocks equal row blocks; rows of the
    first heavy_blocks blocks get k_heavy distinct uniform columns, the others round(k_heavy*ratio)
    (at least 1), so a row-block split gives two classes of per-GPU nnz with low/high = ratio."""
    blk = np.arange(m, dtype=np.int64) * nblocks // m
    counts = np.where(blk < heavy_blocks, k_heavy, max(1, int(round(k_heavy * ratio)))).astype(np.int64)
    counts = np.minimum(counts, n)
    return _finish("csr", m, n, counts, lambda p, i, v: lib().gen_kvar_fill(m, n, seed, kind, _p(p), _p(i), _p(v)))


def stencil27(N, seed=2, kind=UNIFORM):
    """Config 2: 27-point stencil on an N^3 grid (N=127 -> 2,048,383 rows, (3N-2)^3 nnz)."""
    m = N ** 3
    counts = np.empty(m, np.int64)
    lib().gen_stencil27_count(N, _p(counts))
    return _finish("csr", m, m, counts, lambda p, i, v: lib().gen_stencil27_fill(N, seed, kind, _p(p), _p(i), _p(v)))


def rmat(scale, edges=None, seed=3, kind=UNIFORM, permute=False, a=0.57, b=0.19, c=0.19):
    """Config 3: Graph500 R-MAT, 'edges' samples (default 16 * 2^scale), deduplicated."""
    m = 1 << scale
    edges = float(16 * m if edges is None else edges)
    counts = np.empty(m, np.int64)
    lib().gen_rmat_count(scale, edges, a, b, c, seed, int(permute), _p(counts))
    return _finish("csr", m, m, counts,
                   lambda p, i, v: lib().gen_rmat_fill(scale, edges, a, b, c, seed, int(permute), kind,
                                                        _p(p), _p(i), _p(v)))


def banded(m, n, h, seed=501, kind=UNIFORM):
    counts = np.empty(m, np.int64)
    lib().gen_banded_count(m, n, h, _p(counts))
    return _finish("csr", m, n, counts, lambda p, i, v: lib().gen_banded_fill(m, n, h, seed, kind, _p(p), _p(i), _p(v)))


def blockdiag(m, bs, seed=502, kind=UNIFORM):
    counts = np.empty(m, np.int64)
    lib().gen_blockdiag_count(m, bs, _p(counts))
    return _finish("csr", m, m, counts, lambda p, i, v: lib().gen_blockdiag_fill(m, bs, seed, kind, _p(p), _p(i), _p(v)))


def powerlaw_csc(m, n, R, kmax, seed=503, kind=UNIFORM):
    counts = np.empty(n, np.int64)
    lib().gen_powerlaw_csc_count(m, n, R, kmax, seed, _p(counts))
    return _finish("csc", m, n, counts,
                   lambda p, i, v: lib().gen_powerlaw_csc_fill(m, n, R, kmax, seed, kind, _p(p), _p(i), _p(v)))


def vector(n, seed, kind=UNIFORM, dtype=np.float64):
    out = np.empty(max(n, 1), np.float64)[:n]
    if n:
        lib().gen_vector(n, seed, kind, _p(out))
    return out.astype(dtype, copy=False)


def transpose(A: Sparse) -> Sparse:
    """Same entries in the other compressed format (CSR <-> CSC)."""
    if A["val"].dtype != np.float64:                 # fp32 values round-trip exactly through fp64
        T = transpose(Sparse(A, val=A["val"].astype(np.float64)))
        T["val"] = T["val"].astype(A["val"].dtype)
        return T
    outer, inner = (A["m"], A["n"]) if A["fmt"] == "csr" else (A["n"], A["m"])
    nnz = A.nnz
    tptr = np.zeros(inner + 1, np.int64)
    tidx = np.empty(max(nnz, 1), np.int32)[:nnz]
    tval = np.empty(max(nnz, 1), np.float64)[:nnz]
    lib().gen_transpose(outer, inner, _p(A["ptr"]), _p(A["idx"]), _p(A["val"]), _p(tptr), _p(tidx), _p(tval))
    return Sparse(fmt="csc" if A["fmt"] == "csr" else "csr", m=A["m"], n=A["n"], ptr=tptr, idx=tidx, val=tval)


def expand_rows(A: Sparse) -> np.ndarray:
    """Major index per nonzero: the row of each nonzero of a CSR matrix (row-sorted COO view),
    or the column of each nonzero of a CSC matrix (column-sorted COO view)."""
    out = np.empty(max(A.nnz, 1), np.int32)[:A.nnz]
    lib().gen_expand_ptr(A["ptr"].size - 1, _p(A["ptr"]), _p(out))
    return out


def fit_R(col_degrees):
    """log-log least squares of the column-degree histogram."""
    k, cnt = np.unique(np.asarray(col_degrees), return_counts=True)
    k, cnt = k[k > 0], cnt[k > 0]
    if k.size < 2:
        raise ValueError("fit_R needs at least 2 distinct degrees")
    slope, _ = np.polyfit(np.log(k), np.log(cnt / cnt.sum()), 1)
    return -slope


# ---------------------------------------------------------------- configs
# BASELINE.json configs; 'small' variants are parity-test sizes.
CONFIGS = {
    "random1k": dict(desc="1,000x1,000 random CSR, exactly 10 distinct columns/row, 10k nnz (config 1)"),
    "stencil": dict(desc="27-point 3D stencil N=127: 2,048,383 rows, 54,439,939 nnz (config 2)"),
    "rmat": dict(desc="R-MAT scale 24, 2^28 samples deduplicated, (a,b,c)=(.57,.19,.19) (config 3)"),
    "rmatperm": dict(desc="config 3 with a seeded vertex relabelling of rows and columns (the permuted variant)"),
    "tallskinny": dict(desc="50M x 1M, exactly 500 distinct rows/column, 500M nnz, CSC (config 4)"),
}


def make_config(name, kind=UNIFORM, scale_down=1):
    """Build a named config matrix (CSR, or CSC for tallskinny)."""
    if name == "random1k":
        return kdistinct_csr(1000, 1000, 10, seed=1, kind=kind)
    if name == "stencil":
        return stencil27(127 // scale_down if scale_down > 1 else 127, seed=2, kind=kind)
    if name in ("rmat", "rmatperm"):
        s = 24 - (scale_down.bit_length() - 1 if scale_down > 1 else 0)
        return rmat(s, seed=3, kind=kind, permute=name == "rmatperm")
    if name == "tallskinny":
        return kdistinct_csc(50_000_000 // scale_down, 1_000_000 // scale_down, 500, seed=4, kind=kind)
    if name.startswith("suite-"):
        return suite(name, kind=kind)
    raise KeyError(name)


SUITE_SHAPES = ("banded", "blockdiag", "powerlaw", "shortwide")
SUITE_SIZES = {"1M": 10**6, "10M": 10**7, "100M": 10**8, "1B": 10**9}


def powerlaw_mean_degree(R, kmax):
    k = np.arange(1, kmax + 1, dtype=np.float64)
    w = k ** -R
    return float((k * w).sum() / w.sum())


def suite(name, kind=UNIFORM):
    """BASELINE.json config 5, SuiteSparse-shaped synthetic matrices:
    suite-<shape>-<size>, shape in SUITE_SHAPES, size in SUITE_SIZES (target nnz).
      banded     full band of 141 per row (HV15R-like), square
      blockdiag  dense 64x64 diagonal blocks, square
      powerlaw   power-law column degrees P(k) ~ k^-2.13, kmax 10^5 (wb-edu / Orkut R), square, CSC
      shortwide  exactly 500 distinct uniform columns per row, n = 50 m (transpose of config 4)"""
    _, shape, size = name.split("-")
    target = SUITE_SIZES[size]
    seed = 500 + SUITE_SHAPES.index(shape)
    if shape == "banded":
        m = max(1, target // 141)
        return banded(m, m, 70, seed=seed, kind=kind)
    if shape == "blockdiag":
        m = max(64, target // 64 // 64 * 64)
        return blockdiag(m, 64, seed=seed, kind=kind)
    if shape == "powerlaw":
        R, kmax = 2.13, 100_000
        n = max(1, int(target / powerlaw_mean_degree(R, kmax)))
        return powerlaw_csc(n, n, R, min(kmax, n), seed=seed, kind=kind)
    if shape == "shortwide":
        m = max(1, target // 500)
        return kdistinct_csr(m, 50 * m, 500, seed=seed, kind=kind)
    raise KeyError(name)


# ---------------------------------------------------------- rank-local generation
# A config's pointer array alone (every rank needs it for the plan), then only the rows a rank's
# nonzero range touches: bench.py with N > 1 never builds the whole matrix on a rank.
LOCAL_CONFIGS = ("random1k", "stencil", "rmat", "rmatperm", "tallskinny")


def config_pointer(name):
    """(fmt, m, n, ptr) of a config without its entries (CSR; CSC for tallskinny)."""
    if name == "random1k":
        m, n, k = 1000, 1000, 10
        return "csr", m, n, np.arange(m + 1, dtype=np.int64) * k
    if name == "tallskinny":
        m, n, k = 50_000_000, 1_000_000, 500
        return "csc", m, n, np.arange(n + 1, dtype=np.int64) * k
    if name == "stencil":
        N = 127
        counts = np.empty(N ** 3, np.int64)
        lib().gen_stencil27_count(N, _p(counts))
        m = N ** 3
    elif name in ("rmat", "rmatperm"):
        scale = 24
        m = 1 << scale
        counts = np.empty(m, np.int64)
        lib().gen_rmat_count(scale, float(16 * m), 0.57, 0.19, 0.19, 3, int(name == "rmatperm"), _p(counts))
    else:
        raise KeyError(name)
    ptr = np.zeros(m + 1, np.int64)
    np.cumsum(counts, out=ptr[1:])
    return "csr", m, m, ptr


def config_rows(name, ptr, r0, r1, kind=UNIFORM):
    """idx, val of rows (CSC: columns) [r0, r1) of a config, nonzeros ptr[r0] .. ptr[r1]."""
    nz = int(ptr[r1] - ptr[r0])
    idx = np.empty(max(nz, 1), np.int32)[:nz]
    val = np.empty(max(nz, 1), np.float64)[:nz]
    if nz == 0:
        return idx, val
    L = lib()
    if name == "random1k":
        L.gen_kdistinct_fill_rows(1000, 1000, 10, 1, kind, 0, r0, r1, _p(ptr), _p(idx), _p(val))
    elif name == "tallskinny":
        L.gen_kdistinct_fill_rows(1_000_000, 50_000_000, 500, 4, kind, 1, r0, r1, _p(ptr), _p(idx), _p(val))
    elif name == "stencil":
        L.gen_stencil27_fill_rows(127, 2, kind, r0, r1, _p(ptr), _p(idx), _p(val))
    elif name in ("rmat", "rmatperm"):
        L.gen_rmat_fill_rows(24, float(16 * (1 << 24)), 0.57, 0.19, 0.19, 3, int(name == "rmatperm"), kind, r0, r1,
                             _p(ptr), _p(idx), _p(val))
    else:
        raise KeyError(name)
    return idx, val
