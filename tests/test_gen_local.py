"""Rank-local generation (bench.py at N > 1): a config's pointer array alone, then only a row range,
must equal the same rows of the whole matrix -- every row is a pure function of (seed, row)."""
import ctypes

import numpy as np

import gen


def _check(name, ranges):
    A = gen.make_config(name)
    fmt, m, n, ptr = gen.config_pointer(name)
    assert fmt == A["fmt"] and (m, n) == (A["m"], A["n"]) and np.array_equal(ptr, A["ptr"])
    for r0, r1 in ranges:
        idx, val = gen.config_rows(name, ptr, r0, r1)
        z0, z1 = int(ptr[r0]), int(ptr[r1])
        assert np.array_equal(idx, A["idx"][z0:z1]) and np.array_equal(val, A["val"][z0:z1]), (name, r0, r1)


def test_random1k_rows():
    _check("random1k", [(0, 1000), (0, 1), (17, 503), (999, 1000), (5, 5)])


def test_stencil_rows():
    _check("stencil", [(0, 4096), (1_000_000, 1_000_300), (2_048_383 - 7, 2_048_383)])


def test_rmat_and_kdistinct_fill_rows_match_whole_fill():
    """The row-range fills of R-MAT and of the k-distinct (tall-skinny) generator, at a small scale
    through the same entry points, equal the whole-matrix fills."""
    L = gen.lib()
    P = ctypes.c_void_p
    A = gen.rmat(12, seed=3)
    for r0, r1 in [(0, 4096), (0, 1), (100, 2000), (4000, 4096)]:
        nz = int(A["ptr"][r1] - A["ptr"][r0])
        idx = np.empty(max(nz, 1), np.int32)[:nz]; val = np.empty(max(nz, 1), np.float64)[:nz]
        L.gen_rmat_fill_rows(12, float(16 * 4096), 0.57, 0.19, 0.19, 3, 0, 0, r0, r1, A["ptr"].ctypes.data_as(P),
                             idx.ctypes.data_as(P), val.ctypes.data_as(P))
        z0 = int(A["ptr"][r0])
        assert np.array_equal(idx, A["idx"][z0:z0 + nz]) and np.array_equal(val, A["val"][z0:z0 + nz])
    C = gen.kdistinct_csc(5000, 300, 40, seed=4)
    for c0, c1 in [(0, 300), (10, 200)]:
        nz = int(C["ptr"][c1] - C["ptr"][c0])
        idx = np.empty(nz, np.int32); val = np.empty(nz, np.float64)
        L.gen_kdistinct_fill_rows(300, 5000, 40, 4, 0, 1, c0, c1, C["ptr"].ctypes.data_as(P), idx.ctypes.data_as(P),
                                  val.ctypes.data_as(P))
        z0 = int(C["ptr"][c0])
        assert np.array_equal(idx, C["idx"][z0:z0 + nz]) and np.array_equal(val, C["val"][z0:z0 + nz])


def test_permuted_rmat_is_a_relabelling():
    """The permuted R-MAT variant (config 3's "permuted variant"): its row-range fill
    equals its whole fill, it holds exactly as many entries as the unpermuted matrix, and its row
    and column degree multisets are the same (a vertex relabelling moves entries, it does not add or
    drop any); heavy rows no longer cluster at low ids."""
    L = gen.lib()
    P = ctypes.c_void_p
    A = gen.rmat(12, seed=3)
    B = gen.rmat(12, seed=3, permute=True)
    assert B.nnz == A.nnz
    assert np.array_equal(np.sort(np.diff(A["ptr"])), np.sort(np.diff(B["ptr"])))
    assert np.array_equal(np.sort(np.bincount(A["idx"], minlength=4096)), np.sort(np.bincount(B["idx"], minlength=4096)))
    assert np.argmax(np.diff(B["ptr"])) != 0 or np.argmax(np.diff(A["ptr"])) != 0
    for r0, r1 in [(0, 4096), (1000, 1100)]:
        nz = int(B["ptr"][r1] - B["ptr"][r0])
        idx = np.empty(max(nz, 1), np.int32)[:nz]; val = np.empty(max(nz, 1), np.float64)[:nz]
        L.gen_rmat_fill_rows(12, float(16 * 4096), 0.57, 0.19, 0.19, 3, 1, 0, r0, r1, B["ptr"].ctypes.data_as(P),
                             idx.ctypes.data_as(P), val.ctypes.data_as(P))
        z0 = int(B["ptr"][r0])
        assert np.array_equal(idx, B["idx"][z0:z0 + nz]) and np.array_equal(val, B["val"][z0:z0 + nz])
