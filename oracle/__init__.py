"""CPU oracle for msRep's hot path (arXiv 2209.07552) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2209_07552_b200``) never imports it and shares no code with it.

This is a thin ctypes wrapper around ``oracle/oracle.c`` (plain single-threaded
C99, fp64 accumulation, no FMA contraction).  Every function cites the PAPER.md
(P:line) / SPEC.md (S:line) passage it follows in ``oracle.c``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

F64, F32 = 0, 1


def build() -> str:
    """Compile oracle.c with gcc (the checker is built, not used, by build())."""
    if (not os.path.exists(_SO)) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
             "-shared", "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        D = ctypes.c_double
        I = ctypes.c_int
        sig = {
            "or_coo_to_csr": [I64, I64, P, P, P, I, P, P, P],
            "or_csr_to_coo": [I64, P, P],
            "or_csr_to_csc": [I64, I64, P, P, P, I, P, P, P],
            "or_csc_to_coo": [I64, P, P],
            "or_spmv_csr": [I64, P, P, P, I, P, P, D, D],
            "or_spmv_csc": [I64, I64, P, P, P, I, P, P, D, D],
            "or_spmv_coo": [I64, I64, P, P, P, I, P, P, D, D],
            "or_row_bound_csr": [I64, P, P, P, I, P, P, D, D, P],
            "or_nnz_boundaries": [I64, I64, P],
            "or_owner_linear": [I64, P, I64],
            "or_partition_ptr": [I64, P, I64, P, P],
            "or_partition_coo": [I64, I64, P, I64, P],
            "or_partition_coo_unsorted": [I64, P, I64, P],
            "or_exec_coo_unsorted": [I64, I64, P, P, P, I, P, P, D, D, I64],
            "or_exec_csr": [I64, P, P, P, I, P, P, D, D, I64],
            "or_exec_coo": [I64, I64, P, P, P, I, P, P, D, D, I64],
            "or_exec_csc": [I64, I64, P, P, P, I, P, P, D, D, I64],
            "or_merge_parts_to_ptr": [I64, I64, P, P, P],
            "or_block_boundaries": [I64, P, I64, P],
            "or_block_boundaries_coo": [I64, I64, P, I64, P],
            "or_relative_throughput": [I64, P],
            "or_two_level_boundaries": [I64, I64, P, P],
            "or_partition_ptr_b": [I64, P, I64, P, P, P],
            "or_partition_coo_b": [I64, P, I64, P, P],
            "or_cg_csr": [I64, P, P, P, P, P, D, I64, P, P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = None
        L.or_owner_linear.restype = I64
        L.or_partition_ptr.restype = I64
        L.or_partition_ptr_b.restype = I64
        L.or_relative_throughput.restype = D
        _lib = L
    return _lib


# numpy record matching the oracle's or_part struct (its own definition)
PART_DTYPE = np.dtype([("start_idx", "<i8"), ("end_idx", "<i8"), ("start_row", "<i8"),
                       ("end_row", "<i8"), ("start_flag", "<i4"), ("pad_", "<i4"),
                       ("owned_begin", "<i8"), ("owned_end", "<i8")])


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _dt(val):
    if val.dtype == np.float64:
        return F64
    if val.dtype == np.float32:
        return F32
    raise TypeError(f"oracle values must be float64 or float32, got {val.dtype}")


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------- conversions
def coo_to_csr(m, row_idx, col_idx, val):
    row_idx = _c(row_idx, np.int64); col_idx = _c(col_idx, np.int32); val = np.ascontiguousarray(val)
    nnz = row_idx.size
    rp = np.zeros(m + 1, np.int64); ci = np.zeros(nnz, np.int32); v = np.zeros(nnz, val.dtype)
    lib().or_coo_to_csr(m, nnz, _p(row_idx), _p(col_idx), _p(val), _dt(val), _p(rp), _p(ci), _p(v))
    return rp, ci, v


def csr_to_coo(m, row_ptr):
    row_ptr = _c(row_ptr, np.int64)
    ri = np.zeros(int(row_ptr[m]), np.int64)
    lib().or_csr_to_coo(m, _p(row_ptr), _p(ri))
    return ri


def csr_to_csc(m, n, row_ptr, col_idx, val):
    row_ptr = _c(row_ptr, np.int64); col_idx = _c(col_idx, np.int32); val = np.ascontiguousarray(val)
    nnz = int(row_ptr[m])
    cp = np.zeros(n + 1, np.int64); ri = np.zeros(nnz, np.int32); v = np.zeros(nnz, val.dtype)
    lib().or_csr_to_csc(m, n, _p(row_ptr), _p(col_idx), _p(val), _dt(val), _p(cp), _p(ri), _p(v))
    return cp, ri, v


def csc_to_coo(n, col_ptr):
    col_ptr = _c(col_ptr, np.int64)
    ci = np.zeros(int(col_ptr[n]), np.int64)
    lib().or_csc_to_coo(n, _p(col_ptr), _p(ci))
    return ci


# ---------------------------------------------------------------------- SpMV
def spmv_csr(m, row_ptr, col_idx, val, x, y, alpha, beta):
    """Alg. 1. Returns a new y; inputs are not modified."""
    row_ptr = _c(row_ptr, np.int64); col_idx = _c(col_idx, np.int32)
    val = np.ascontiguousarray(val); x = _c(x, val.dtype); out = np.array(y, dtype=val.dtype, copy=True)
    lib().or_spmv_csr(m, _p(row_ptr), _p(col_idx), _p(val), _dt(val), _p(x), _p(out), alpha, beta)
    return out


def spmv_csc(m, n, col_ptr, row_idx, val, x, y, alpha, beta):
    """CSC scatter."""
    col_ptr = _c(col_ptr, np.int64); row_idx = _c(row_idx, np.int32)
    val = np.ascontiguousarray(val); x = _c(x, val.dtype); out = np.array(y, dtype=val.dtype, copy=True)
    lib().or_spmv_csc(m, n, _p(col_ptr), _p(row_idx), _p(val), _dt(val), _p(x), _p(out), alpha, beta)
    return out


def spmv_coo(m, row_idx, col_idx, val, x, y, alpha, beta):
    """COO triplet loop."""
    row_idx = _c(row_idx, np.int64); col_idx = _c(col_idx, np.int32)
    val = np.ascontiguousarray(val); x = _c(x, val.dtype); out = np.array(y, dtype=val.dtype, copy=True)
    lib().or_spmv_coo(m, row_idx.size, _p(row_idx), _p(col_idx), _p(val), _dt(val), _p(x), _p(out),
                      alpha, beta)
    return out


def row_bound_csr(m, row_ptr, col_idx, val, x, y_in, alpha, beta):
    row_ptr = _c(row_ptr, np.int64); col_idx = _c(col_idx, np.int32)
    val = np.ascontiguousarray(val); x = _c(x, val.dtype); y_in = _c(y_in, val.dtype)
    b = np.zeros(m, np.float64)
    lib().or_row_bound_csr(m, _p(row_ptr), _p(col_idx), _p(val), _dt(val), _p(x), _p(y_in),
                           alpha, beta, _p(b))
    return b


# ----------------------------------------------------------------- partition
def nnz_boundaries(nnz, np_):
    b = np.zeros(np_ + 1, np.int64)
    lib().or_nnz_boundaries(nnz, np_, _p(b))
    return b


def owner_linear(ptr, idx):
    ptr = _c(ptr, np.int64)
    return int(lib().or_owner_linear(ptr.size - 1, _p(ptr), idx))


def partition_ptr(ptr, np_):
    """Alg. 2 / Alg. 4: returns (parts[np] records, list of local-pointer arrays)."""
    ptr = _c(ptr, np.int64)
    m = ptr.size - 1
    parts = np.zeros(np_, PART_DTYPE)
    nloc = lib().or_partition_ptr(m, _p(ptr), np_, _p(parts), None)
    loc = np.zeros(nloc, np.int64)
    lib().or_partition_ptr(m, _p(ptr), np_, _p(parts), _p(loc))
    out, w = [], 0
    for p in parts:
        k = 1 if p["start_row"] < 0 else int(p["end_row"] - p["start_row"] + 2)
        out.append(loc[w:w + k].copy())
        w += k
    return parts, out, loc


def partition_coo(m, row_idx, np_):
    """Alg. 6 on a row-sorted COO."""
    row_idx = _c(row_idx, np.int64)
    parts = np.zeros(np_, PART_DTYPE)
    lib().or_partition_coo(m, row_idx.size, _p(row_idx), np_, _p(parts))
    return parts


def block_boundaries(ptr, np_):
    """Baseline row/column-block split (Sec. 5.1): b_i = ptr[floor(i*m/np)]."""
    ptr = _c(ptr, np.int64)
    b = np.zeros(np_ + 1, np.int64)
    lib().or_block_boundaries(ptr.size - 1, _p(ptr), np_, _p(b))
    return b


def block_boundaries_coo(m, row_idx, np_):
    row_idx = _c(row_idx, np.int64)
    b = np.zeros(np_ + 1, np.int64)
    lib().or_block_boundaries_coo(m, row_idx.size, _p(row_idx), np_, _p(b))
    return b


def two_level_boundaries(nnz, sizes):
    """Two-level NUMA split (Sec. 4.2): groups get nnz in proportion to their part counts,
    then each group's range is split among its parts by the floor rule."""
    sizes = _c(sizes, np.int64)
    b = np.zeros(int(sizes.sum()) + 1, np.int64)
    lib().or_two_level_boundaries(nnz, sizes.size, _p(sizes), _p(b))
    return b


def relative_throughput(b):
    """Fig. 6 cost model: (sum nnz_i / np) / max nnz_i."""
    b = _c(b, np.int64)
    return float(lib().or_relative_throughput(b.size - 1, _p(b)))


def partition_ptr_b(ptr, b):
    """Alg. 2 / Alg. 4 for given boundaries b[0..np] -> parts (the descriptors only)."""
    ptr = _c(ptr, np.int64); b = _c(b, np.int64)
    parts = np.zeros(b.size - 1, PART_DTYPE)
    lib().or_partition_ptr_b(ptr.size - 1, _p(ptr), b.size - 1, _p(b), _p(parts), None)
    return parts


def partition_coo_b(m, row_idx, b):
    row_idx = _c(row_idx, np.int64); b = _c(b, np.int64)
    parts = np.zeros(b.size - 1, PART_DTYPE)
    lib().or_partition_coo_b(m, _p(row_idx), b.size - 1, _p(b), _p(parts))
    return parts


def cg_csr(m, row_ptr, col_idx, val, b, x0, tol, maxit):
    """Textbook CG (Hestenes-Stiefel) on an SPD CSR matrix, fp64. Returns (x, iterations, relres)."""
    row_ptr = _c(row_ptr, np.int64); col_idx = _c(col_idx, np.int32)
    val = _c(val, np.float64); b = _c(b, np.float64); x = np.array(x0, dtype=np.float64, copy=True)
    it = np.zeros(1, np.int64); rr = np.zeros(1, np.float64)
    lib().or_cg_csr(m, _p(row_ptr), _p(col_idx), _p(val), _p(b), _p(x), float(tol), int(maxit), _p(it), _p(rr))
    return x, int(it[0]), float(rr[0])


def merge_parts_to_ptr(m, parts, loc_flat):
    out = np.zeros(m + 1, np.int64)
    parts = np.ascontiguousarray(parts); loc_flat = _c(loc_flat, np.int64)
    lib().or_merge_parts_to_ptr(m, parts.size, _p(parts), _p(loc_flat), _p(out))
    return out


# --------------------------------------------------------- partitioned exec
def exec_csr(m, row_ptr, col_idx, val, x, y, alpha, beta, np_):
    """Alg. 2 + Alg. 3 with the beta-deferred merge (R6)."""
    row_ptr = _c(row_ptr, np.int64); col_idx = _c(col_idx, np.int32)
    val = np.ascontiguousarray(val); x = _c(x, val.dtype); out = np.array(y, dtype=val.dtype, copy=True)
    lib().or_exec_csr(m, _p(row_ptr), _p(col_idx), _p(val), _dt(val), _p(x), _p(out), alpha, beta, np_)
    return out


def exec_coo(m, row_idx, col_idx, val, x, y, alpha, beta, np_):
    """Alg. 6 + Alg. 7 with the beta-deferred merge."""
    row_idx = _c(row_idx, np.int64); col_idx = _c(col_idx, np.int32)
    val = np.ascontiguousarray(val); x = _c(x, val.dtype); out = np.array(y, dtype=val.dtype, copy=True)
    lib().or_exec_coo(m, row_idx.size, _p(row_idx), _p(col_idx), _p(val), _dt(val), _p(x), _p(out),
                      alpha, beta, np_)
    return out


def partition_coo_unsorted(row_idx, np_):
    """Unsorted COO (Sec. 3.2.3): nnz split by position; per part its smallest and
    largest row, no flag, no owned rows."""
    row_idx = _c(row_idx, np.int64)
    parts = np.zeros(np_, PART_DTYPE)
    lib().or_partition_coo_unsorted(row_idx.size, _p(row_idx), np_, _p(parts))
    return parts


def exec_coo_unsorted(m, row_idx, col_idx, val, x, y, alpha, beta, np_):
    """Unsorted pCOO: per-part full-length partial y, summed in part order (column-style merge)."""
    row_idx = _c(row_idx, np.int64); col_idx = _c(col_idx, np.int32)
    val = np.ascontiguousarray(val); x = _c(x, val.dtype); out = np.array(y, dtype=val.dtype, copy=True)
    lib().or_exec_coo_unsorted(m, row_idx.size, _p(row_idx), _p(col_idx), _p(val), _dt(val), _p(x), _p(out),
                               alpha, beta, np_)
    return out


def exec_csc(m, n, col_ptr, row_idx, val, x, y, alpha, beta, np_):
    """Alg. 4 + Alg. 5 (column merge, R7)."""
    col_ptr = _c(col_ptr, np.int64); row_idx = _c(row_idx, np.int32)
    val = np.ascontiguousarray(val); x = _c(x, val.dtype); out = np.array(y, dtype=val.dtype, copy=True)
    lib().or_exec_csc(m, n, _p(col_ptr), _p(row_idx), _p(val), _dt(val), _p(x), _p(out), alpha, beta, np_)
    return out
