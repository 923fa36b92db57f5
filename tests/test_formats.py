"""Pins for the CPU reference codec of the paper's binary formats (oracle/formats.py; P:230-314,
Table `tab:bin_formats` P:241-270).  -m "not gpu"."""
import struct

import numpy as np
import pytest

import gbla_gen
from conftest import csr_from_dense
from oracle import formats as fm


def _eq(M, dec):
    m, n, p, rp, col, val = dec
    assert (m, n, p) == (M.m, M.n, M.p)
    assert np.array_equal(rp.astype(np.uint64), M.row_ptr.astype(np.uint64))
    assert np.array_equal(col.astype(np.uint32), M.col.astype(np.uint32))
    assert np.array_equal(val.astype(np.uint16), M.val.astype(np.uint16))


def test_colid_runs_paper_rule():
    # "If s > 1 several non zero elements are consecutive on a row and if f is the first one, then
    # we store f s ... If s = 1 then we use a mask" (reading: f | 2^31)
    assert fm.encode_colids([5, 6, 7, 8]) == [5, 4]
    assert fm.encode_colids([9]) == [9 | (1 << 31)]
    assert fm.encode_colids([0, 1, 4, 5, 6, 100]) == [0, 2, 4, 3, 100 | (1 << 31)]
    assert fm.decode_colids([0, 2, 4, 3, 100 | (1 << 31)], 6) == [0, 1, 4, 5, 6, 100]
    with pytest.raises(ValueError):
        fm.decode_colids([5, 4], 3)
    rng = np.random.default_rng(1)
    for _ in range(300):
        c = np.unique(rng.integers(0, 2000, int(rng.integers(0, 60))))
        assert fm.decode_colids(fm.encode_colids(c), c.size) == c.tolist()


def test_format1_layout_and_round_trip():
    M = csr_from_dense([[2, 0, 5]], 7)                          # 1 x 3, row [(0,2), (2,5)]
    b = fm.write_format1(M)
    assert b == struct.pack("<IIIQ", 1, 3, 7, 2) + struct.pack("<HH", 2, 5) + struct.pack("<II", 0, 2) + \
        struct.pack("<I", 2)
    _eq(M, fm.read_format1(b))
    E = csr_from_dense(np.zeros((3, 4), np.int64), 7)           # empty rows: rows = [0, 0, 0]
    _eq(E, fm.read_format1(fm.write_format1(E)))
    for M in gbla_gen.random_suite(60, seed0=5):
        _eq(M, fm.read_format1(fm.write_format1(M)))
    bad = bytearray(fm.write_format1(csr_from_dense([[1, 1], [0, 1]], 7)))
    bad[-4:] = struct.pack("<I", 5)                             # sum of rows != nnz
    with pytest.raises(ValueError):
        fm.read_format1(bytes(bad))


def test_format2_dedup_and_round_trip():
    # "the coefficients in all lines of this type correspond to the same polynomial"
    M = csr_from_dense([[2, 1, 5, 0, 0], [0, 0, 2, 1, 5]], 7)
    b = fm.write_format2(M)
    bb, m, n, p, nnz = struct.unpack_from("<IIIQQ", b, 0)
    assert (bb & 7, bb >> 24, m, n, p, nnz) == (0b010, 1, 2, 5, 7, 6)
    o = 28 + 16                                                  # after rows, polmap
    assert np.frombuffer(b, "<u4", 2, 28 + 8).tolist() == [0, 0]          # polmap: one polynomial
    (k,) = struct.unpack_from("<Q", b, o)
    assert k == 4                                               # two runs (f, s) of 3 columns
    assert np.frombuffer(b, "<u8", 4, o + 8).tolist() == [0, 3, 2, 3]
    pnb, pnnz = struct.unpack_from("<IQ", b, o + 8 + 32)
    assert (pnb, pnnz) == (1, 3)
    _eq(M, fm.read_format2(b))
    T = csr_from_dense([[3, 1, 0]] * 10, 7)                     # 10 rows, one polynomial
    assert struct.unpack_from("<IQ", fm.write_format2(T), 28 + 80 + 8 + 8 * 10 * 2)[0:2] == (1, 2)
    for M in gbla_gen.random_suite(60, seed0=6):
        _eq(M, fm.read_format2(fm.write_format2(M)))
    # the paper's worked type code 011 also reads as 16-bit data (reading R23)
    b11 = bytearray(fm.write_format2(M))
    b11[0] = (b11[0] & ~7) | 0b011
    _eq(M, fm.read_format2(bytes(b11)))


def test_format2_smaller_on_repeated_polynomials():
    G = gbla_gen.gb_like_matrix(16 * 64, 4000, 16, 40, 65521, seed=3, run=16)   # horizontal runs
    f1, f2 = fm.write_format1(G), fm.write_format2(G)
    _eq(G, fm.read_format2(f2))
    assert len(f2) < len(f1) / 2


def test_format2_without_dedup_reads_back():
    for M in list(gbla_gen.random_suite(30, seed0=8)) + [gbla_gen.f4_matrix("c0")]:
        _eq(M, fm.read_format2(fm.write_format2_nodedup(M)))
