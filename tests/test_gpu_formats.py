"""GPU: the device decoder of the paper's binary formats (gbla_file_decode; SURVEY 8(f) f3,
P:230-314) against the CPU reference codec (oracle/formats.py), and the decoded matrices reduced
end to end against the oracle."""
import struct

import numpy as np
import pytest

import gbla_gen
import oracle
from conftest import csr_from_dense
from oracle import formats as fm

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


def _np(t, dt):
    import torch
    view = {np.uint64: torch.int64, np.uint32: torch.int32, np.uint16: torch.int16}[dt]
    return t.view(view).cpu().numpy().view(dt)


def _check(M, dec):
    m, n, p, rp, col, val = dec
    assert (m, n, p) == (M.m, M.n, M.p)
    assert np.array_equal(_np(rp, np.uint64), M.row_ptr.astype(np.uint64))
    assert np.array_equal(_np(col, np.uint32), M.col.astype(np.uint32))
    assert np.array_equal(_np(val, np.uint16), M.val.astype(np.uint16))


def test_decode_both_formats(gb, ctx):
    cases = [gbla_gen.f4_matrix("c0"), csr_from_dense(np.zeros((3, 4), np.int64), 7),
             csr_from_dense([[2, 0, 5]], 7)]
    cases += list(gbla_gen.random_suite(30, seed0=91))
    cases += [gbla_gen.gb_like_matrix(2000, 5000, 24, 60, 65521, seed=s, run=r) for s, r in ((1, 4), (2, 16), (3, 1))]
    cases.append(gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS["c1"], 0.05)))
    for M in cases:
        _check(M, gb.file_decode(ctx, fm.write_format1(M), 1))
        _check(M, gb.file_decode(ctx, fm.write_format2(M), 2))
    # every pdata width / the paper's type code 011
    M = cases[-2]
    for tc in (0b011, 0b100, 0b110):
        _check(M, gb.file_decode(ctx, fm.write_format2(M, typecode=tc), 2))
    info = gb.file_info(fm.write_format2(M), 2)
    assert info["version"] == 1 and info["typecode"] == 0b010 and info["m"] == M.m


def test_decoded_matrix_reduces(gb, ctx):
    """Format 2 file -> device decode -> gbla_reduce: R and rank equal the oracle's on c0 and on a
    gb-like matrix (rows m_i f_j)."""
    for M in (gbla_gen.f4_matrix("c0"), gbla_gen.gb_like_matrix(1500, 3000, 20, 50, 32003, seed=7, run=8)):
        res = oracle.reduce(M)
        m, n, p, rp, col, val = gb.file_decode(ctx, fm.write_format2(M), 2)
        h = gb.gbla_reduce(ctx, m, n, rp, col, val, p)
        r, pc, R = h.rref()
        assert r == res.rank and np.array_equal(pc.cpu().numpy(), res.pivcol)
        assert np.array_equal(R.cpu().numpy(), res.R)
        h.free()


def test_decode_errors(gb, ctx):
    M = gbla_gen.gb_like_matrix(200, 800, 5, 20, 7, seed=4, run=4)
    b2 = fm.write_format2(M)

    def status(data, fmt):
        with pytest.raises(gb.GblaError) as e:
            gb.file_decode(ctx, data, fmt)
        return e.value.status

    assert status(b2[:-1], 2) == 1                              # truncated: sizes do not add up
    bad = bytearray(b2)
    struct.pack_into("<Q", bad, 20, M.nnz + 1)                  # nnz that the rows do not add up to
    assert status(bytes(bad), 2) == 1
    bad = bytearray(b2)
    bad[3] = 7                                                   # unknown version
    assert status(bytes(bad), 2) == 1
    struct.pack_into("<Q", bad := bytearray(b2), 12, 65537)      # p >= 2^16
    assert status(bytes(bad), 2) == 2
    # a run head whose length slot became a single column (masked): the run has no length
    o = 28 + 8 * M.m + 8
    toks = np.frombuffer(b2, "<u8", count=struct.unpack_from("<Q", b2, o - 8)[0], offset=o)
    j = int(np.nonzero((toks & (1 << 31)) == 0)[0][1])          # the length slot of the first run
    bad = bytearray(b2)
    struct.pack_into("<Q", bad, o + 8 * j, int(toks[j]) | (1 << 31))
    assert status(bytes(bad), 2) == 1
    b1 = bytearray(fm.write_format1(M))
    b1[20] = 0; b1[21] = 0                                       # a zero value (format 1 stores nonzeros)
    m, n, p, rp, col, val = gb.file_decode(ctx, bytes(b1), 1)   # decodes; the splice rejects it
    with pytest.raises(gb.GblaError) as e:
        gb.gbla_splice(ctx, m, n, rp, col, val, p)
    assert e.value.status == 1
