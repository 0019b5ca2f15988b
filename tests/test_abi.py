"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/msrep.h declares, and its host partitioner (msrep_plan, binary search)
is bit-exact against the oracle's linear-scan partitioner."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "msrep.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(msrep_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2209_07552_b200 as M
    lib = ctypes.CDLL(M.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(M.EXPORTED)
    assert M.msrep_version() == 1


def _header_struct_fields(name):
    """(field, C type, array length) of `typedef struct {...} name;` in include/msrep.h, in order"""
    src = open(os.path.join(ROOT, "include", "msrep.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    body = re.search(r"typedef struct \{([^{}]*)\}\s*" + name + ";", src).group(1)
    out = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        ctype, rest = decl.split(None, 1)
        for f in rest.split(","):
            m = re.match(r"\s*(\w+)(?:\[(\d+)\])?", f)
            out.append((m.group(1), ctype, int(m.group(2)) if m.group(2) else 1))
    return out


def test_binding_structs_match_header():
    """The ctypes mirrors of msrep_stats / msrep_part_desc have the header's fields, in order, with
    the same types and sizes: a missing field would let msrep_get_stats write past the buffer."""
    import paper_2209_07552_b200 as M
    sizes = {"int64_t": 8, "double": 8, "int32_t": 4}
    for cls, name in ((M.Stats, "msrep_stats"), (M.PartDesc, "msrep_part_desc")):
        hdr = _header_struct_fields(name)
        py = [(f, t) for f, t in cls._fields_]
        assert [f for f, _, _ in hdr] == [f for f, _ in py], name
        for (f, ct, n), (_, t) in zip(hdr, py):
            assert ctypes.sizeof(t) == sizes[ct] * n, (name, f)
        assert ctypes.sizeof(cls) == sum(sizes[ct] * n for _, ct, n in hdr), name


def test_library_is_sm100a_and_uses_tma():
    import shutil
    import subprocess
    import paper_2209_07552_b200 as M
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-sass", M.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UBLKCP" in out          # cp.async.bulk (1-D TMA) staging in the SpMV kernels
    # the pCSC scatter is a plain read-modify-write into warp-owned shared-memory rows (no CAS
    # loops); global fp64 adds appear only where short-wide matrices add partial bands into py
    assert "ATOMS.CAST" not in out


def _parts_equal(a, b):
    for k in ("start_idx", "end_idx", "start_row", "end_row", "start_flag", "owned_begin", "owned_end"):
        assert np.array_equal(a[k], b[k]), k


def test_plan_bit_exact_vs_oracle_random():
    import paper_2209_07552_b200 as M
    rng = np.random.default_rng(17)
    for trial in range(300):
        m = int(rng.integers(0, 60))
        lens = rng.integers(0, 6, m) * (rng.random(m) < 0.6)
        if trial % 7 == 0 and m:
            lens[rng.integers(0, m)] = 200
        ptr = np.zeros(m + 1, np.int64); ptr[1:] = np.cumsum(lens)
        nnz = int(ptr[-1])
        for np_ in list(range(1, 10)) + [nnz + 1, nnz + 5, 64]:
            ours = M.msrep_plan(M.CSR, m, nnz, np_, ptr=ptr)
            ref, _, _ = oracle.partition_ptr(ptr, np_)
            _parts_equal(ours, ref)
            rows = np.repeat(np.arange(m), lens)
            ours = M.msrep_plan(M.COO, m, nnz, np_, coo_row=rows)
            _parts_equal(ours, oracle.partition_coo(m, rows, np_))


def test_plan_worked_values(golden_E):
    import paper_2209_07552_b200 as M
    g = golden_E
    p = M.msrep_plan(M.CSR, 4, 5, 2, ptr=np.array(g["csr_row_ptr"]))
    for got, e in zip(p, g["pcsr_np2"]):
        for k in ("start_idx", "end_idx", "start_row", "end_row", "start_flag"):
            assert int(got[k]) == e[k]
    p = M.msrep_plan(M.CSC, 4, 5, 2, ptr=np.array(g["csc_col_ptr"]))
    for got, e in zip(p, g["pcsc_np2"]):
        for k in ("start_idx", "end_idx", "start_row", "end_row", "start_flag"):
            assert int(got[k]) == e[k]
    p = M.msrep_plan(M.CSR, 4, 5, 5, ptr=np.array(g["csr_row_ptr"]))
    assert [[int(a["owned_begin"]), int(a["owned_end"])] for a in p] == g["owned_np5"]


def test_plan_large_bit_exact():
    import gen
    import paper_2209_07552_b200 as M
    A = gen.rmat(16, seed=3)
    for np_ in (1, 2, 4, 8, 64):
        ours = M.msrep_plan(M.CSR, A["m"], A.nnz, np_, ptr=A["ptr"])
        ref, _, _ = oracle.partition_ptr(A["ptr"], np_)
        _parts_equal(ours, ref)


def test_plan_errors():
    import paper_2209_07552_b200 as M
    with pytest.raises(M.MsrepError) as e:
        M.msrep_plan(M.CSR, 2, 3, 2, ptr=np.array([0, 1, 2]))     # ptr[m] != nnz
    assert e.value.status == 2
    with pytest.raises(M.MsrepError) as e:
        M.msrep_plan(M.CSR, 2, 2, 0, ptr=np.array([0, 1, 2]))
    assert e.value.status == 1
    assert "bad plan" in M.msrep_last_error()


def test_create_rejects_bad_args_without_device():
    import paper_2209_07552_b200 as M
    with pytest.raises(M.MsrepError) as e:
        M.msrep_create(rank=2, nranks=2)
    assert e.value.status == 1


def test_block_split_plan_bit_exact_vs_oracle():
    """msrep_plan_split(BLOCK) (binary searches) == the oracle's Baseline row/column blocks
    (linear scans) on random CSR / CSC / COO structures, including empty rows and np > m."""
    import paper_2209_07552_b200 as M
    rng = np.random.default_rng(23)
    for trial in range(300):
        m = int(rng.integers(0, 50)); np_ = int(rng.integers(1, 12))
        lens = rng.integers(0, 7, m) * (rng.random(m) < 0.7)
        ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        nnz = int(ptr[-1])
        ours = M.msrep_plan_split(M.CSR, M.SPLIT_BLOCK, m, nnz, np_, ptr=ptr)
        ref = oracle.partition_ptr_b(ptr, oracle.block_boundaries(ptr, np_))
        _parts_equal(ours, ref)
        ours = M.msrep_plan_split(M.CSC, M.SPLIT_BLOCK, m, nnz, np_, ptr=ptr)
        _parts_equal(ours, ref)
        rows = oracle.csr_to_coo(m, ptr)
        ours = M.msrep_plan_split(M.COO, M.SPLIT_BLOCK, m, nnz, np_, coo_row=rows)
        refc = oracle.partition_coo_b(m, rows, oracle.block_boundaries_coo(m, rows, np_))
        _parts_equal(ours, refc)


def test_coo_col_plan_matches_csc_and_oracle():
    """Column-sorted pCOO: Alg. 6 on the sorted column ids gives exactly the pCSC
    descriptors of Alg. 4 on the same matrix, and the oracle's linear-scan Alg. 6."""
    import paper_2209_07552_b200 as M
    rng = np.random.default_rng(29)
    for trial in range(200):
        n = int(rng.integers(0, 40)); np_ = int(rng.integers(1, 10))
        lens = rng.integers(0, 6, n) * (rng.random(n) < 0.7)
        cp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        nnz = int(cp[-1])
        cols = oracle.csr_to_coo(n, cp)
        for split in (M.SPLIT_NNZ, M.SPLIT_BLOCK):
            a = M.msrep_plan_split(M.COO_COL, split, n, nnz, np_, coo_row=cols)
            b = M.msrep_plan_split(M.CSC, split, n, nnz, np_, ptr=cp)
            for k in ("start_idx", "end_idx", "start_row", "end_row", "start_flag"):
                assert np.array_equal(a[k], b[k]), k
        ref = oracle.partition_coo(n, cols, np_)
        _parts_equal(M.msrep_plan(M.COO_COL, n, nnz, np_, coo_row=cols), ref)


def test_two_level_plan_bit_exact_vs_oracle():
    """msrep_plan_groups == the oracle's two-level boundaries fed to its Alg. 2 / Alg. 6."""
    import paper_2209_07552_b200 as M
    rng = np.random.default_rng(43)
    for trial in range(200):
        m = int(rng.integers(1, 50))
        groups = [int(v) for v in rng.integers(1, 5, int(rng.integers(1, 4)))]
        lens = rng.integers(0, 7, m) * (rng.random(m) < 0.7)
        ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        nnz = int(ptr[-1])
        b = oracle.two_level_boundaries(nnz, groups)
        _parts_equal(M.msrep_plan_groups(M.CSR, m, nnz, groups, ptr=ptr), oracle.partition_ptr_b(ptr, b))
        rows = oracle.csr_to_coo(m, ptr)
        _parts_equal(M.msrep_plan_groups(M.COO, m, nnz, groups, coo_row=rows), oracle.partition_coo_b(m, rows, b))


def test_plan_bit_exact_vs_oracle_exhaustive_5x5():
    """The library's binary-search partitioner (msrep_plan, CSR and row-sorted COO) equals the
    oracle's linear scan on every row-pointer array with m, n <= 5 and np in 1..nnz+2."""
    import itertools
    import paper_2209_07552_b200 as M
    for m in range(1, 6):
        for lens in itertools.product(range(6), repeat=m):
            ptr = np.zeros(m + 1, np.int64)
            ptr[1:] = np.cumsum(lens)
            nnz = int(ptr[-1])
            rows = np.repeat(np.arange(m), lens).astype(np.int32)
            for np_ in range(1, nnz + 3):
                ref, _, _ = oracle.partition_ptr(ptr, np_)
                _parts_equal(M.msrep_plan(M.CSR, m, nnz, np_, ptr=ptr), ref)
                _parts_equal(M.msrep_plan(M.COO, m, nnz, np_, coo_row=rows), ref)


def test_plan_unsorted_coo_matches_oracle():
    """msrep_plan(MSREP_COO_UNSORTED) == the oracle's unsorted-COO descriptors (positions, min/max
    row), random orders and np up to nnz + 3."""
    import paper_2209_07552_b200 as M
    rng = np.random.default_rng(46)
    for trial in range(200):
        nnz = int(rng.integers(0, 80))
        rows = rng.integers(0, 40, nnz).astype(np.int32)
        for np_ in (1, 2, 3, 7, nnz + 3):
            _parts_equal(M.msrep_plan(M.COO_UNSORTED, 40, nnz, np_, coo_row=rows),
                         oracle.partition_coo_unsorted(rows, np_))
