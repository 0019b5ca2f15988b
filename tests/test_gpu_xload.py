"""The x-gather L1 policy picked at partition time (host.cpp tune_xload) changes only caching:
both policies, and the automatic pick, must give the same bits as the oracle (integer data,
pin P5) for every format, on matrices above the tuner's 2^20-nonzero threshold."""
import numpy as np
import pytest

import gen
from tests.helpers import oracle_ref, run_gpu
from tests.test_gpu_parity import FMTS, as_fmt

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fmt", FMTS)
def test_xload_policies_bit_identical(fmt):
    import paper_2209_07552_b200 as M
    cases = [gen.rmat(17, seed=111, kind=gen.SMALLINT), gen.stencil27(40, kind=gen.SMALLINT)]
    for A in cases:
        assert A["idx"].size >= (1 << 20)
        x = gen.vector(A["n"], 112, kind=gen.SMALLINT); y = gen.vector(A["m"], 113, kind=gen.SMALLINT)
        ref = oracle_ref(A, x, y, 1.5, 0.5)
        picks = []
        for forced in (0, 1, -1):
            ctx = M.Context(0, 1, None, 0, 2)
            ctx.set_tuning("xload", forced)   # msrep_set_tuning(MSREP_TUNE_XLOAD, ...)
            got = run_gpu(as_fmt(A, fmt), fmt, x, y, 1.5, 0.5, ctx=ctx)
            picks.append(ctx.stats()["x_no_allocate"])
            ctx.close()
            assert np.array_equal(got, ref), (fmt, forced)
        assert picks[0] == 0 and picks[1] == 1 and picks[2] in (0, 1)


@pytest.mark.parametrize("fmt", ["csr", "coo"])
def test_sell_occupancy_pick_bit_identical(fmt):
    """Short regular rows with random columns (SELL tiles): the partition times the SELL launches
    at two and at one CTA per SM (stats sell_1cta) -- occupancy changes nothing in the bits."""
    A = gen.kdistinct_csr(400_000, 1_400_000, 6, seed=114, kind=gen.SMALLINT)
    x = gen.vector(A["n"], 115, kind=gen.SMALLINT); y = gen.vector(A["m"], 116, kind=gen.SMALLINT)
    import paper_2209_07552_b200 as M
    ctx = M.Context(0, 1, None, 0, 1)
    got = run_gpu(A, fmt, x, y, 1.5, 0.5, ctx=ctx)
    st = ctx.stats()
    ctx.close()
    assert st["nsell"] > 0 and st["sell_1cta"] in (0, 1)
    assert np.array_equal(got, oracle_ref(A, x, y, 1.5, 0.5))
