"""The paper's two binary matrix formats (Table `tab:bin_formats` P:241-270) --
TEST INFRASTRUCTURE ONLY (the CPU reference codec the device decoder is checked against; only
tests/ and bench.py may import it).

Readings of the passages the paper leaves open (R20/R23-R26):
  * little-endian throughout (unstated);
  * Format 2 type code: the lowest 3 bits of b are u | (v << 1), u = 1 iff signed, data of
    8 * 2^v bits; the paper's own example "011" for an unsigned 16-bit type contradicts
    "u = 1 iff signed", so a reader accepts both 010 and 011 as 16-bit data (and 000 / 001 as 8-bit,
    100 / 101 as 32-bit); the writer emits 010.  The highest 8 bits of b hold the format version
    ("on the highest bits a mask is used to store a file format version"): 1;
  * column ids: a run of s > 1 consecutive columns starting at f is stored as two
    consecutive 64-bit colid slots f, s; a single column f as one slot f | 2^31 (the paper writes
    "f AND (1 << 31)", which would destroy f: OR is the only reading consistent with "we lose a bit
    for the number of rows");
  * polynomial data: rows whose value sequences are identical share one polynomial
    (exact equality), polmap[i] = its number, prow[j] = its length, pdata = the polynomials
    concatenated in order of first use.
"""
from __future__ import annotations

import struct

import numpy as np

MASK = 1 << 31
VERSION = 1


def _rows(M):
    rp = M.row_ptr.astype(np.int64)
    return [(M.col[rp[i]:rp[i + 1]].astype(np.int64), M.val[rp[i]:rp[i + 1]].astype(np.int64)) for i in range(M.m)]


# ------------------------------------------------------------------------------- Format 1
def write_format1(M) -> bytes:
    """Table 2, Format 1: m, n, p (u32), nnz (u64), data (u16 x nnz), cols (u32 x nnz), rows (u32 x m)."""
    rp = M.row_ptr.astype(np.int64)
    out = [struct.pack("<IIIQ", M.m, M.n, M.p, int(rp[-1]) if M.m else 0),
           np.ascontiguousarray(M.val, "<u2").tobytes(), np.ascontiguousarray(M.col, "<u4").tobytes(),
           np.diff(rp).astype("<u4").tobytes()]
    return b"".join(out)


def read_format1(buf: bytes):
    """Inverse of write_format1: (m, n, p, row_ptr u64[m+1], col u32[nnz], val u16[nnz])."""
    if len(buf) < 20:
        raise ValueError("format 1: truncated header")
    m, n, p, nnz = struct.unpack_from("<IIIQ", buf, 0)
    o = 20
    need = o + 2 * nnz + 4 * nnz + 4 * m
    if len(buf) != need:
        raise ValueError(f"format 1: {len(buf)} bytes, expected {need}")
    val = np.frombuffer(buf, "<u2", nnz, o).copy(); o += 2 * nnz
    col = np.frombuffer(buf, "<u4", nnz, o).copy(); o += 4 * nnz
    rows = np.frombuffer(buf, "<u4", m, o).astype(np.uint64)
    rp = np.zeros(m + 1, np.uint64)
    rp[1:] = np.cumsum(rows)
    if m and int(rp[-1]) != nnz:
        raise ValueError("format 1: sum of row lengths != nnz")
    return m, n, p, rp, col, val


# ------------------------------------------------------------------------------- Format 2
def encode_colids(cols) -> list[int]:
    """Run compression of one row's strictly increasing column ids."""
    out = []
    cols = [int(c) for c in cols]
    i = 0
    while i < len(cols):
        j = i
        while j + 1 < len(cols) and cols[j + 1] == cols[j] + 1:
            j += 1
        s = j - i + 1
        if s > 1:
            out += [cols[i], s]
        else:
            out.append(cols[i] | MASK)
        i = j + 1
    return out


def decode_colids(tokens, expected: int) -> list[int]:
    out = []
    i = 0
    while i < len(tokens):
        t = int(tokens[i])
        if t & MASK:
            out.append(t & ~MASK)
            i += 1
        else:
            if i + 1 >= len(tokens):
                raise ValueError("colid: run without length")
            s = int(tokens[i + 1])
            out += list(range(t, t + s))
            i += 2
    if len(out) != expected:
        raise ValueError(f"colid: decoded {len(out)} columns, expected {expected}")
    return out


def write_format2(M, typecode: int = 0b010) -> bytes:
    """Table 2, Format 2 with polynomial deduplication (exact value sequences) and run-compressed
    column ids; pdata elements of 8 * 2^v bits for typecode = u | (v << 1) (010 / 011: 16-bit)."""
    if M.m >= 2 ** 31:
        raise ValueError("format 2: m >= 2^31")
    rows = _rows(M)
    polys, polmap, tokens = {}, [], []
    plist = []
    for cols, vals in rows:
        key = tuple(vals.tolist())
        if key not in polys:
            polys[key] = len(plist)
            plist.append(key)
        polmap.append(polys[key])
        tokens += encode_colids(cols)
    pnnz = sum(len(q) for q in plist)
    nnz = int(M.row_ptr[-1]) if M.m else 0
    b = (VERSION << 24) | typecode
    out = [struct.pack("<IIIQQ", b, M.m, M.n, M.p, nnz),
           np.array([len(c) for c, _ in rows], "<u4").tobytes(), np.array(polmap, "<u4").tobytes(),
           struct.pack("<Q", len(tokens)), np.array(tokens, "<u8").tobytes(),
           struct.pack("<IQ", len(plist), pnnz), np.array([len(q) for q in plist], "<u4").tobytes(),
           np.array([v for q in plist for v in q], {0: "<u1", 1: "<u2", 2: "<u4", 3: "<u8"}[(typecode >> 1) & 3]).tobytes()]
    return b"".join(out)


def read_format2(buf: bytes):
    """Inverse of write_format2: (m, n, p, row_ptr, col, val); accepts the type codes of the
    module docstring (8-, 16-, 32-bit unsigned or signed data)."""
    b, m, n, p, nnz = struct.unpack_from("<IIIQQ", buf, 0)
    if (b >> 24) not in (0, VERSION):
        raise ValueError("format 2: unknown version")
    v = (b >> 1) & 3
    width = {0: "<u1", 1: "<u2", 2: "<u4", 3: "<u8"}[v]
    o = 28
    rows = np.frombuffer(buf, "<u4", m, o).astype(np.int64); o += 4 * m
    polmap = np.frombuffer(buf, "<u4", m, o).astype(np.int64); o += 4 * m
    (k,) = struct.unpack_from("<Q", buf, o); o += 8
    tokens = np.frombuffer(buf, "<u8", k, o); o += 8 * k
    pnb, pnnz = struct.unpack_from("<IQ", buf, o); o += 12
    prow = np.frombuffer(buf, "<u4", pnb, o).astype(np.int64); o += 4 * pnb
    pdata = np.frombuffer(buf, width, pnnz, o).astype(np.int64)
    pstart = np.concatenate([[0], np.cumsum(prow)])
    rp = np.zeros(m + 1, np.uint64)
    rp[1:] = np.cumsum(rows)
    if int(rp[-1]) != nnz:
        raise ValueError("format 2: sum of row lengths != nnz")
    # tokens of each row: parse sequentially
    cols, vals = [], []
    t = 0
    for i in range(m):
        got = []
        while len(got) < rows[i]:
            x = int(tokens[t])
            if x & MASK:
                got.append(x & ~MASK); t += 1
            else:
                got += list(range(x, x + int(tokens[t + 1]))); t += 2
        if len(got) != rows[i] or prow[polmap[i]] != rows[i]:
            raise ValueError(f"format 2: row {i} inconsistent")
        cols += got
        vals += pdata[pstart[polmap[i]]:pstart[polmap[i]] + rows[i]].tolist()
    return m, n, p, rp, np.array(cols, np.uint32), np.array(vals, np.uint16)


def write_format2_nodedup(M, typecode: int = 0b010) -> bytes:
    """Format 2 without polynomial deduplication (polmap = identity, pdata = the values in row
    order), column runs encoded vectorized -- the same byte layout, for large synthetic matrices
    whose coefficients are i.i.d. (nothing to deduplicate) in benchmarks."""
    rp = M.row_ptr.astype(np.int64)
    col = M.col.astype(np.int64)
    nnz = col.size
    if nnz:
        rowid = np.repeat(np.arange(M.m), np.diff(rp))
        brk = np.ones(nnz, bool)
        brk[1:] = (col[1:] != col[:-1] + 1) | (rowid[1:] != rowid[:-1])
        starts = np.nonzero(brk)[0]
        lens = np.diff(np.append(starts, nnz))
        single = lens == 1
        ntok = np.where(single, 1, 2)
        off = np.concatenate([[0], np.cumsum(ntok)[:-1]])
        tokens = np.zeros(int(ntok.sum()), np.uint64)
        tokens[off[single]] = col[starts[single]].astype(np.uint64) | np.uint64(MASK)
        tokens[off[~single]] = col[starts[~single]].astype(np.uint64)
        tokens[off[~single] + 1] = lens[~single].astype(np.uint64)
    else:
        tokens = np.zeros(0, np.uint64)
    rows = np.diff(rp).astype("<u4")
    w = {0: "<u1", 1: "<u2", 2: "<u4", 3: "<u8"}[(typecode >> 1) & 3]
    out = [struct.pack("<IIIQQ", (VERSION << 24) | typecode, M.m, M.n, M.p, nnz), rows.tobytes(),
           np.arange(M.m, dtype="<u4").tobytes(), struct.pack("<Q", tokens.size), tokens.astype("<u8").tobytes(),
           struct.pack("<IQ", M.m, nnz), rows.tobytes(), M.val.astype(w).tobytes()]
    return b"".join(out)
