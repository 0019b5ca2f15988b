"""Python binding of libmsrep (include/msrep.h): B200-native nnz-balanced SpMV
over the augmented formats pCSR / pCSC / pCOO of msRep (arXiv 2209.07552).

Argument marshalling only: every step of the hot path runs in the CUDA kernels
of ``csrc/``.  There is no CPU fallback -- importing this package without the
built ``libmsrep.so`` raises.  PyTorch is used by callers for device memory,
streams and ``torch.distributed`` (the NCCL unique-id broadcast); this module
itself needs only ctypes + numpy.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmsrep.so")   # the in-tree build only (tuning builds: tools/variant.sh)

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libmsrep.so not built at {LIB_PATH}: run `make` (or __graft_entry__.build()) first")

_lib = ctypes.CDLL(LIB_PATH)

# enums (include/msrep.h)
CSR, CSC, COO, COO_COL, COO_UNSORTED = 0, 1, 2, 3, 4
SPLIT_NNZ, SPLIT_BLOCK, SPLIT_TWO_LEVEL = 0, 1, 2
SPLITS = {"nnz": SPLIT_NNZ, "block": SPLIT_BLOCK}
F64, F32 = 0, 1
Y_REPLICATED, Y_OWNED, Y_SHARDED = 0, 1, 2
RESIDENT_DEVICE, RESIDENT_HOST = 0, 1
RESIDENCY = {"device": RESIDENT_DEVICE, "host": RESIDENT_HOST}
STATUS = {0: "MSREP_OK", 1: "MSREP_ERR_INVALID_ARG", 2: "MSREP_ERR_DIM_MISMATCH", 3: "MSREP_ERR_UNSORTED_COO",
          4: "MSREP_ERR_TOO_LARGE", 5: "MSREP_ERR_STATE", 6: "MSREP_ERR_OOM", 7: "MSREP_ERR_CUDA",
          8: "MSREP_ERR_NCCL"}
FORMATS = {"csr": CSR, "csc": CSC, "coo": COO, "coo_col": COO_COL, "coo_unsorted": COO_UNSORTED}
TUNE_XLOAD, TUNE_CG_GRAPH, TUNE_HOT_X, TUNE_COMPACT_X, TUNE_HOT_CLUSTER, TUNE_SELL, TUNE_COL_LAYOUT = range(7)
TUNING = {"xload": TUNE_XLOAD, "cg_graph": TUNE_CG_GRAPH, "hot_x": TUNE_HOT_X, "compact_x": TUNE_COMPACT_X,
          "hot_cluster": TUNE_HOT_CLUSTER, "sell": TUNE_SELL, "col_layout": TUNE_COL_LAYOUT}


class PartDesc(ctypes.Structure):
    _fields_ = [("start_idx", ctypes.c_int64), ("end_idx", ctypes.c_int64), ("start_row", ctypes.c_int64),
                ("end_row", ctypes.c_int64), ("start_flag", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("owned_begin", ctypes.c_int64), ("owned_end", ctypes.c_int64)]


PART_DTYPE = np.dtype([("start_idx", "<i8"), ("end_idx", "<i8"), ("start_row", "<i8"), ("end_row", "<i8"),
                       ("start_flag", "<i4"), ("reserved", "<i4"), ("owned_begin", "<i8"), ("owned_end", "<i8")])
assert PART_DTYPE.itemsize == ctypes.sizeof(PartDesc)


class Stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in (
        "nparts", "nranks", "parts_per_rank", "nnz_rank", "rows_window", "owned_rows", "distinct_cols", "ntiles",
        "nslabs", "nsplit_rows", "nheads_local", "alg_bytes", "alg_bytes_beta0", "kernels_per_spmv",
        "device_bytes")] + [("partition_ms", ctypes.c_double), ("tile_bytes", ctypes.c_int64),
                                         ("nsell", ctypes.c_int64),
                                         ("phase_ms", ctypes.c_double * 4), ("residency", ctypes.c_int64),
                                         ("nchunks", ctypes.c_int64), ("host_bytes", ctypes.c_int64),
                                         ("x_no_allocate", ctypes.c_int64), ("nhot", ctypes.c_int64),
                                         ("hot_nnz", ctypes.c_int64), ("x_compact", ctypes.c_int64),
                                         ("sell_1cta", ctypes.c_int64),
                                         ("gpu_numa_node", ctypes.c_int64), ("host_numa_node", ctypes.c_int64),
                                         ("stream_bytes", ctypes.c_int64), ("col_layout", ctypes.c_int64),
                                         ("layout_ms", ctypes.c_double * 6), ("x_order", ctypes.c_int64),
                                         ("nsell_narrow", ctypes.c_int64)]


class Allocator(ctypes.Structure):
    _fields_ = [("alloc", ctypes.c_void_p), ("free", ctypes.c_void_p), ("user", ctypes.c_void_p)]


class MsrepError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msrep_last_error()}")


P, I64, I32, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int
_sig = {
    "msrep_get_unique_id": [P],
    "msrep_create": [ctypes.POINTER(P), I, I, P, I, I, P],
    "msrep_create_loopback": [P, I, I, I],
    "msrep_partition": [P, I, I, I64, I64, I64, P, P, P, P, P, P],
    "msrep_partition_slice": [P, I, I, I64, I64, I64, P, P, P, I64, I64, P, P],
    "msrep_spmv": [P, P, P, P, P, I, P],
    "msrep_spmv_host": [P, P, P, P, P, I, P],
    "msrep_plan": [I, I64, I64, I, P, P, P],
    "msrep_exchange_plan": [I, I, I64, I64, I64, I, I, P, P, P, P, P],
    "msrep_plan_split": [I, I, I64, I64, I, P, P, P],
    "msrep_set_split": [P, I],
    "msrep_set_tuning": [P, I, I],
    "msrep_set_residency": [P, I, I64],
    "msrep_debug_arrange": [P, I64, P, I64, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64)],
    "msrep_cg": [P, P, P, ctypes.c_double, I, I, ctypes.POINTER(I), ctypes.POINTER(ctypes.c_double), P],
    "msrep_spmm": [P, P, P, P, P, I, I, P],
    "msrep_spmv_mirror": [P, P, P, P, P, I, P, P],
    "msrep_plan_groups": [I, I64, I64, I, P, P, P, P],
    "msrep_set_split_groups": [P, I, P],
    "msrep_get_stats": [P, ctypes.POINTER(Stats)],
    "msrep_destroy": [P],
    "msrep_profile_enable": [P, I],
    "msrep_profile_read": [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64), I],
}
for _k, _a in _sig.items():
    getattr(_lib, _k).argtypes = _a
    getattr(_lib, _k).restype = ctypes.c_int
_lib.msrep_last_error.argtypes = []
_lib.msrep_last_error.restype = ctypes.c_char_p
_lib.msrep_version.argtypes = []
_lib.msrep_version.restype = ctypes.c_int

EXPORTED = ["msrep_get_unique_id", "msrep_create", "msrep_create_loopback", "msrep_partition", "msrep_partition_slice", "msrep_spmv", "msrep_spmv_host",
            "msrep_plan", "msrep_plan_split", "msrep_set_split", "msrep_set_tuning", "msrep_set_residency", "msrep_debug_arrange", "msrep_cg", "msrep_spmm", "msrep_spmv_mirror", "msrep_plan_groups", "msrep_set_split_groups", "msrep_exchange_plan", "msrep_get_stats", "msrep_destroy", "msrep_last_error", "msrep_version",
            "msrep_profile_enable", "msrep_profile_read"]


def _check(status, where):
    if status != 0:
        raise MsrepError(status, where)


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if hasattr(a, "data_ptr"):           # torch tensor
        return a.data_ptr()
    return a.ctypes.data


_NP_DTYPE = {F64: np.float64, F32: np.float32}


def _check_vec(t, dtype, count, name):
    """A device vector handed to the library: a CUDA tensor of the partition's dtype, contiguous,
    with >= count elements (a raw int pointer is passed through unchecked)."""
    if t is None or isinstance(t, int):
        return
    import torch
    want = torch.float64 if dtype == F64 else torch.float32
    if not (t.is_cuda and t.is_contiguous() and t.dtype == want and t.numel() >= count):
        raise ValueError(f"{name}: need a contiguous CUDA {want} tensor with >= {count} elements, got "
                         f"{t.dtype} {tuple(t.shape)} on {t.device} (contiguous={t.is_contiguous()})")


def _check_host_vec(a, dtype, count, name):
    if a is None or isinstance(a, int):
        return
    if hasattr(a, "data_ptr"):   # pinned torch tensor
        import torch
        want = torch.float64 if dtype == F64 else torch.float32
        ok = (not a.is_cuda) and a.is_contiguous() and a.dtype == want and a.numel() >= count
    else:
        ok = a.flags["C_CONTIGUOUS"] and a.dtype == _NP_DTYPE[dtype] and a.size >= count
    if not ok:
        raise ValueError(f"{name}: need a contiguous host {_NP_DTYPE[dtype].__name__} array with >= {count} elements")


# ------------------------------------------------------------ C-ABI mirrors
def msrep_last_error() -> str:
    return _lib.msrep_last_error().decode()


def msrep_version() -> int:
    return _lib.msrep_version()


def msrep_get_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(_lib.msrep_get_unique_id(ctypes.cast(buf, P)), "msrep_get_unique_id")
    return bytes(buf)


_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)


def torch_allocator(device=0):
    """An msrep_allocator over torch's CUDA caching allocator (the library's device buffers then come
    from, and go back to, torch's pool).  Returns (struct, keepalive); keep both alive as long as the
    context (Context(allocator="torch") does)."""
    import torch

    def _alloc(nbytes, stream, user):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), device=device, stream=int(stream or 0))
        except Exception:   # reported by the library as MSREP_ERR_OOM
            return None

    def _free(ptr, nbytes, stream, user):
        try:
            if ptr:
                torch.cuda.caching_allocator_delete(ptr)
        except Exception:   # interpreter teardown: the process is ending anyway
            pass

    fa, ff = _ALLOC_FN(_alloc), _FREE_FN(_free)
    st = Allocator(ctypes.cast(fa, ctypes.c_void_p), ctypes.cast(ff, ctypes.c_void_p), None)
    return st, (fa, ff, st)


def msrep_create(rank=0, nranks=1, uid: bytes | None = None, device=0, parts_per_rank=1, alloc=None):
    """alloc: None (cudaMalloc / cudaFree) or an Allocator struct (see torch_allocator)."""
    h = P()
    idbuf = None
    if uid is not None:
        idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    _check(_lib.msrep_create(ctypes.byref(h), rank, nranks, ctypes.cast(idbuf, P) if idbuf is not None else None,
                             device, parts_per_rank, ctypes.byref(alloc) if alloc is not None else None),
           "msrep_create")
    return h


def msrep_partition(ctx, fmt, dtype, m, n, nnz, ptr, idx, coo_row, val, stream=None, want_parts=True, nparts=None):
    """Host numpy arrays in: ptr int64 (CSR/CSC), idx int32, coo_row int32 (COO), val float64/float32."""
    parts = np.zeros(nparts, PART_DTYPE) if (want_parts and nparts) else None
    _check(_lib.msrep_partition(ctx, fmt, dtype, m, n, nnz, _ptr(ptr), _ptr(idx), _ptr(coo_row), _ptr(val),
                                _ptr(parts), stream), "msrep_partition")
    return parts


def _scalar(v, dtype):
    return (ctypes.c_double(v) if dtype == F64 else ctypes.c_float(v))


def msrep_spmv(ctx, alpha, x, beta, y, layout=Y_REPLICATED, stream=None, dtype=F64):
    a, b = _scalar(alpha, dtype), _scalar(beta, dtype)
    _check(_lib.msrep_spmv(ctx, ctypes.byref(a), _ptr(x), ctypes.byref(b), _ptr(y), layout, stream), "msrep_spmv")


def msrep_spmv_host(ctx, alpha, x_host, beta, y_host, layout=Y_REPLICATED, stream=None, dtype=F64):
    a, b = _scalar(alpha, dtype), _scalar(beta, dtype)
    _check(_lib.msrep_spmv_host(ctx, ctypes.byref(a), _ptr(x_host), ctypes.byref(b), _ptr(y_host), layout, stream),
           "msrep_spmv_host")


def msrep_plan(fmt, outer, nnz, np_, ptr=None, coo_row=None):
    parts = np.zeros(np_, PART_DTYPE)
    if ptr is not None:
        ptr = np.ascontiguousarray(ptr, np.int64)
    if coo_row is not None:
        coo_row = np.ascontiguousarray(coo_row, np.int32)
    _check(_lib.msrep_plan(fmt, outer, nnz, np_, _ptr(ptr), _ptr(coo_row), _ptr(parts)), "msrep_plan")
    return parts


def msrep_plan_split(fmt, split, outer, nnz, np_, ptr=None, coo_row=None):
    parts = np.zeros(np_, PART_DTYPE)
    if ptr is not None:
        ptr = np.ascontiguousarray(ptr, np.int64)
    if coo_row is not None:
        coo_row = np.ascontiguousarray(coo_row, np.int32)
    _check(_lib.msrep_plan_split(fmt, split, outer, nnz, np_, _ptr(ptr), _ptr(coo_row), _ptr(parts)),
           "msrep_plan_split")
    return parts


def msrep_plan_groups(fmt, outer, nnz, groups, ptr=None, coo_row=None):
    """Two-level split (Sec. 4.2) descriptors; groups = parts per NUMA group."""
    g = np.ascontiguousarray(groups, np.int32)
    parts = np.zeros(int(g.sum()), PART_DTYPE)
    if ptr is not None:
        ptr = np.ascontiguousarray(ptr, np.int64)
    if coo_row is not None:
        coo_row = np.ascontiguousarray(coo_row, np.int32)
    _check(_lib.msrep_plan_groups(fmt, outer, nnz, g.size, _ptr(g), _ptr(ptr), _ptr(coo_row), _ptr(parts)),
           "msrep_plan_groups")
    return parts


def msrep_set_split_groups(ctx, groups):
    g = np.ascontiguousarray(groups, np.int32)
    _check(_lib.msrep_set_split_groups(ctx, g.size, _ptr(g)), "msrep_set_split_groups")


def msrep_set_split(ctx, split):
    _check(_lib.msrep_set_split(ctx, split), "msrep_set_split")


def msrep_set_tuning(ctx, knob, value):
    """knob: TUNE_XLOAD / TUNE_CG_GRAPH / TUNE_HOT_X (or its TUNING name), value as include/msrep.h."""
    if isinstance(knob, str):
        knob = TUNING[knob]
    _check(_lib.msrep_set_tuning(ctx, int(knob), int(value)), "msrep_set_tuning")


def msrep_set_residency(ctx, residency, chunk_bytes=0):
    _check(_lib.msrep_set_residency(ctx, residency, int(chunk_bytes)), "msrep_set_residency")


def msrep_debug_arrange(pk):
    """Host test hook: the arranged pCSC warp list of packed entries pk (uint32, row = pk & 8191).
    Returns (order, same, seg_from): order[i] = entry index or -1 (hole)."""
    pk = np.ascontiguousarray(pk, np.uint32)
    cap = 64 * max(1, pk.size) + 64
    order = np.empty(cap, np.int64)
    ln, same, seg = I64(), I64(), I64()
    _check(_lib.msrep_debug_arrange(_ptr(pk), pk.size, _ptr(order), cap, ctypes.byref(ln), ctypes.byref(same),
                                    ctypes.byref(seg)), "msrep_debug_arrange")
    return order[:ln.value].copy(), same.value, seg.value


def msrep_exchange_plan(fmt, m, n, nnz, nranks, parts_per_rank, ptr=None, coo_row=None, split=SPLIT_NNZ):
    """Pure host: the multi-rank exchange step msrep_spmv performs (include/msrep.h).
    Returns (seg[nranks, 2] y-row segments per rank, head_row[np], head_part[np])."""
    np_ = nranks * parts_per_rank
    seg = np.zeros(2 * nranks, np.int64)
    hrow = np.zeros(np_, np.int64)
    hpart = np.zeros(np_, np.int32)
    if ptr is not None:
        ptr = np.ascontiguousarray(ptr, np.int64)
    if coo_row is not None:
        coo_row = np.ascontiguousarray(coo_row, np.int32)
    _check(_lib.msrep_exchange_plan(fmt, split, m, n, nnz, nranks, parts_per_rank, _ptr(ptr), _ptr(coo_row), _ptr(seg),
                                    _ptr(hrow), _ptr(hpart)), "msrep_exchange_plan")
    return seg.reshape(nranks, 2), hrow, hpart


def msrep_spmm(ctx, alpha, X, beta, Y, k, layout=Y_REPLICATED, stream=None, dtype=F64):
    """Y (device [m x k], row-major) <- alpha * A * X (device [n x k]) + beta * Y, k in {2, 4, 8}."""
    a, b = _scalar(alpha, dtype), _scalar(beta, dtype)
    _check(_lib.msrep_spmm(ctx, ctypes.byref(a), _ptr(X), ctypes.byref(b), _ptr(Y), int(k), layout, stream),
           "msrep_spmm")


def msrep_spmv_mirror(ctx, alpha, x, beta, y, mirrors, stream=None, dtype=F64):
    """y <- alpha*A*x + beta*y on the owned rows, each row also stored into every buffer in
    `mirrors` (device pointers or tensors: the peers' y, or local buffers)."""
    a, b = _scalar(alpha, dtype), _scalar(beta, dtype)
    arr = (ctypes.c_void_p * max(1, len(mirrors)))(*[_ptr(mm) for mm in mirrors])
    _check(_lib.msrep_spmv_mirror(ctx, ctypes.byref(a), _ptr(x), ctypes.byref(b), _ptr(y), len(mirrors),
                                  ctypes.cast(arr, P), stream), "msrep_spmv_mirror")


def msrep_cg(ctx, b, x, tol=1e-10, maxit=1000, check_every=10, stream=None):
    """CG on the partitioned SPD matrix (include/msrep.h): x (device, in/out) <- iterate.
    Returns (iterations, ||r|| / ||b||)."""
    it, rr = I(), ctypes.c_double()
    _check(_lib.msrep_cg(ctx, _ptr(b), _ptr(x), float(tol), int(maxit), int(check_every), ctypes.byref(it),
                         ctypes.byref(rr), stream), "msrep_cg")
    return it.value, rr.value


def msrep_get_stats(ctx) -> dict:
    s = Stats()
    _check(_lib.msrep_get_stats(ctx, ctypes.byref(s)), "msrep_get_stats")
    return {k: (list(getattr(s, k)) if k in ("phase_ms", "layout_ms") else getattr(s, k)) for k, _ in Stats._fields_}


def msrep_profile_enable(ctx, enable=True):
    _check(_lib.msrep_profile_enable(ctx, int(bool(enable))), "msrep_profile_enable")


def msrep_profile_read(ctx, reset=True):
    ms, n = ctypes.c_double(), I64()
    _check(_lib.msrep_profile_read(ctx, ctypes.byref(ms), ctypes.byref(n), int(bool(reset))), "msrep_profile_read")
    return ms.value, n.value


def msrep_destroy(ctx):
    _check(_lib.msrep_destroy(ctx), "msrep_destroy")


# ------------------------------------------------------------ convenience
class Context:
    """One rank's msrep context.  ``Context.from_torch_dist()`` creates the NCCL
    communicator from an initialised torch.distributed process group (rank 0's
    unique id is broadcast through it).  All device vectors are torch tensors."""

    def __init__(self, rank=0, nranks=1, uid=None, device=0, parts_per_rank=1, allocator="torch"):
        """allocator: "torch" (default: the library's device buffers come from torch's CUDA caching
        allocator) or None (cudaMalloc / cudaFree inside the library)."""
        self.rank, self.nranks, self.device, self.parts_per_rank = rank, nranks, device, parts_per_rank
        self._alloc_keep = None
        st = None
        if allocator == "torch":
            st, self._alloc_keep = torch_allocator(device)
        elif allocator is not None:
            raise ValueError(f"allocator {allocator!r}: None or 'torch'")
        self.h = msrep_create(rank, nranks, uid, device, parts_per_rank, st)
        self.dtype = F64
        self.fmt = CSR
        self.parts = None
        self.m = self.n = self.nnz = 0

    @classmethod
    def loopback_group(cls, nranks, device=0, parts_per_rank=1):
        """nranks contexts on ONE device whose collectives meet in-process (msrep_create_loopback):
        drive each from its own thread with the same call sequence, as NCCL ranks would be."""
        arr = (P * nranks)()
        _check(_lib.msrep_create_loopback(ctypes.cast(arr, P), nranks, device, parts_per_rank), "msrep_create_loopback")
        out = []
        for r in range(nranks):
            c = cls.__new__(cls)
            c.rank, c.nranks, c.device, c.parts_per_rank = r, nranks, device, parts_per_rank
            c.h = P(arr[r])
            c.dtype, c.fmt, c.parts, c.m, c.n, c.nnz = F64, CSR, None, 0, 0, 0
            out.append(c)
        return out

    @classmethod
    def from_torch_dist(cls, device=None, parts_per_rank=1):
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        if device is None:
            device = torch.cuda.current_device()
        uid = None
        if world > 1:
            obj = [msrep_get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        return cls(rank, world, uid, device, parts_per_rank)

    def partition(self, fmt, m, n, ptr=None, idx=None, val=None, coo_row=None, stream=None, split="nnz",
                  residency="device", chunk_bytes=0):
        msrep_set_residency(self.h, RESIDENCY[residency] if isinstance(residency, str) else residency, chunk_bytes)
        if isinstance(fmt, str):
            fmt = FORMATS[fmt]
        if isinstance(split, (list, tuple)):   # two-level: parts per NUMA group
            msrep_set_split_groups(self.h, split)
        else:
            msrep_set_split(self.h, SPLITS[split] if isinstance(split, str) else split)
        val = np.ascontiguousarray(val)
        if val.dtype == np.float64:
            dtype = F64
        elif val.dtype == np.float32:
            dtype = F32
        else:
            raise ValueError(f"val dtype {val.dtype}: the library takes float64 or float32 values")
        idx = np.ascontiguousarray(idx, np.int32)
        nnz = idx.size
        if val.size != nnz:
            raise ValueError(f"val has {val.size} entries, idx {nnz}")
        if coo_row is not None and np.asarray(coo_row).size != nnz:
            raise ValueError(f"coo_row has {np.asarray(coo_row).size} entries, idx {nnz}")
        if ptr is not None:
            ptr = np.ascontiguousarray(ptr, np.int64)
        if coo_row is not None:
            coo_row = np.ascontiguousarray(coo_row, np.int32)
        self.parts = msrep_partition(self.h, fmt, dtype, m, n, nnz, ptr, idx, coo_row, val, stream,
                                     nparts=self.nranks * self.parts_per_rank)
        self.dtype, self.fmt, self.m, self.n, self.nnz = dtype, fmt, m, n, nnz
        return self.parts

    def set_tuning(self, knob, value):
        msrep_set_tuning(self.h, knob, value)

    def partition_slice(self, fmt, m, n, ptr, idx_slice, val_slice, slice_begin, stream=None, split="nnz"):
        """CSR / CSC partition from a slice of the entries: idx_slice / val_slice hold global nonzero
        positions [slice_begin, slice_begin + len) and must cover this rank's range
        (msrep_partition_slice)."""
        msrep_set_residency(self.h, RESIDENT_DEVICE, 0)
        if isinstance(fmt, str):
            fmt = FORMATS[fmt]
        msrep_set_split(self.h, SPLITS[split] if isinstance(split, str) else split)
        val = np.ascontiguousarray(val_slice)
        if val.dtype not in (np.float64, np.float32):
            raise ValueError(f"val dtype {val.dtype}: the library takes float64 or float32 values")
        dtype = F64 if val.dtype == np.float64 else F32
        idx = np.ascontiguousarray(idx_slice, np.int32)
        if val.size != idx.size:
            raise ValueError(f"val slice has {val.size} entries, idx slice {idx.size}")
        ptr = np.ascontiguousarray(ptr, np.int64)
        nnz = int(ptr[-1])
        np_ = self.nranks * self.parts_per_rank
        parts = np.zeros(np_, PART_DTYPE)
        _check(_lib.msrep_partition_slice(self.h, fmt, dtype, m, n, nnz, _ptr(ptr), _ptr(idx), _ptr(val),
                                          int(slice_begin), int(slice_begin) + idx.size, _ptr(parts), stream),
               "msrep_partition_slice")
        self.parts = parts
        self.dtype, self.fmt, self.m, self.n, self.nnz = dtype, fmt, m, n, nnz
        return parts

    def spmv(self, alpha, x, beta, y, layout=Y_REPLICATED, stream=None):
        _check_vec(x, self.dtype, self.n, "x")
        _check_vec(y, self.dtype, self.m, "y")
        if stream is None:
            import torch
            stream = torch.cuda.current_stream().cuda_stream
        msrep_spmv(self.h, alpha, x, beta, y, layout, stream, self.dtype)

    def spmv_host(self, alpha, x_host, beta, y_host, layout=Y_REPLICATED, stream=None):
        _check_host_vec(x_host, self.dtype, self.n, "x_host")
        _check_host_vec(y_host, self.dtype, self.m, "y_host")
        msrep_spmv_host(self.h, alpha, x_host, beta, y_host, layout, stream, self.dtype)

    def stats(self):
        return msrep_get_stats(self.h)

    def spmv_mirror(self, alpha, x, beta, y, mirrors, stream=None):
        _check_vec(x, self.dtype, self.n, "x")
        _check_vec(y, self.dtype, self.m, "y")
        for i, mm in enumerate(mirrors):
            _check_vec(mm, self.dtype, self.m, f"mirrors[{i}]")
        if stream is None:
            import torch
            stream = torch.cuda.current_stream().cuda_stream
        msrep_spmv_mirror(self.h, alpha, x, beta, y, mirrors, stream, self.dtype)

    def spmm(self, alpha, X, beta, Y, layout=Y_REPLICATED, stream=None):
        """X: torch [n, k], Y: torch [m, k] (contiguous, row-major), k in {2, 4, 8}."""
        k = X.shape[1]
        _check_vec(X, self.dtype, self.n * k, "X")
        _check_vec(Y, self.dtype, self.m * k, "Y")
        if Y.dim() != 2 or Y.shape[1] != k:
            raise ValueError(f"Y shape {tuple(Y.shape)} does not match X's k = {k}")
        if stream is None:
            import torch
            stream = torch.cuda.current_stream().cuda_stream
        msrep_spmm(self.h, alpha, X, beta, Y, X.shape[1], layout, stream, self.dtype)

    def cg(self, b, x, tol=1e-10, maxit=1000, check_every=10, stream=None):
        _check_vec(b, self.dtype, self.m, "b")   # m != n is the library's MSREP_ERR_DIM_MISMATCH
        _check_vec(x, self.dtype, self.n, "x")
        if stream is None:
            import torch
            stream = torch.cuda.current_stream().cuda_stream
        return msrep_cg(self.h, b, x, tol, maxit, check_every, stream)

    def close(self):
        if self.h:
            msrep_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
