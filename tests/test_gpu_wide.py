"""GPU parity of SURVEY 8(f) f4 (gbla_reduce_wide: primes 2 < p < 2^31) against the
wide-field oracle (oracle/wide.py, pinned by brute-force Gauss-Jordan of M*sigma)."""
import numpy as np
import pytest

import gbla_gen
import oracle
from oracle import wide

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gb():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a GPU")
    import paper_1602_06097_b200 as gb
    return gb


@pytest.fixture(scope="module")
def ctx(gb):
    return gb.Context(0)


def _np(t):
    import torch
    return t.view(torch.int32).cpu().numpy().view(np.uint32).astype(np.int64)


def check(gb, ctx, M):
    W = wide.reduce(M)
    h = gb.gbla_reduce_wide(ctx, M.m, M.n, M.row_ptr, M.col, M.val, M.p)
    npiv, mN, nN = h.dims()
    assert (npiv, mN, nN) == (W.npiv, W.nonpivot_row.size, M.n - W.npiv), M.name
    sig, prow, nprow = h.maps()
    assert np.array_equal(_np(sig), W.sigma) and np.array_equal(_np(prow), W.pivot_row)
    assert np.array_equal(_np(nprow), W.nonpivot_row)
    r, pc, R, Dn = h.wide()
    assert np.array_equal(_np(Dn), W.dnew), M.name
    assert h.opcount()[0] == W.modmac
    assert r == W.rank and np.array_equal(_np(pc), W.pivcol) and np.array_equal(_np(R), W.R), M.name
    h.free()
    return W


def test_wide_random_suite(gb, ctx):
    for p in (3, 65521, 1048573, 8388593, 2147483647):
        for s in range(10):
            check(gb, ctx, gbla_gen.random_wide(int(4 + 9 * s), int(6 + 11 * s), 0.05 + 0.04 * (s % 5), p, 500 * s + 7))


def test_wide_f4_shapes(gb, ctx):
    """F4-shaped patterns (c0, scaled c1 / c3) with values redrawn below 2^23 and 2^31, and the
    16-bit case equal to the u16 pipeline."""
    c0 = gbla_gen.f4_matrix("c0")
    check(gb, ctx, gbla_gen.widen(c0, 8388593, seed=1))
    check(gb, ctx, gbla_gen.widen(c0, 2147483647, seed=2))
    check(gb, ctx, gbla_gen.widen(gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS["c1"], 0.02)), 1048573, seed=3))
    check(gb, ctx, gbla_gen.widen(gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS["c3"], 0.015)), 4194301, seed=4))
    res = oracle.reduce(c0)
    Wc0 = gbla_gen.WideCSR(c0.m, c0.n, c0.p, c0.row_ptr, c0.col.astype(np.uint32), c0.val.astype(np.uint32))
    h = gb.gbla_reduce_wide(ctx, Wc0.m, Wc0.n, Wc0.row_ptr, Wc0.col, Wc0.val, Wc0.p)
    r, pc, R, Dn = h.wide()
    assert r == res.rank and np.array_equal(_np(R), res.R) and np.array_equal(_np(Dn), res.dnew)
    assert h.opcount()[0] == res.modmac
    h.free()


def test_wide_errors(gb, ctx):
    M = gbla_gen.random_wide(10, 12, 0.3, 1048573, 5)
    for p, st in ((1048575, 2), (2147483659, 2), (2, 2)):
        with pytest.raises(gb.GblaError) as e:
            gb.gbla_reduce_wide(ctx, M.m, M.n, M.row_ptr, M.col, M.val, p)
        assert e.value.status == st
    bad = M.val.copy(); bad[0] = 1048573                       # value >= p
    with pytest.raises(gb.GblaError) as e:
        gb.gbla_reduce_wide(ctx, M.m, M.n, M.row_ptr, M.col, bad, 1048573)
    assert e.value.status == 1
    h = gb.gbla_reduce_wide(ctx, M.m, M.n, M.row_ptr, M.col, M.val, 1048573)
    with pytest.raises(gb.GblaError) as e:                     # u16 calls reject a wide handle
        gb.gbla_echelon_D(h)
    assert e.value.status == 3
    h.free()
