"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the Faugere-Lachartre method: it only
draws matrices.  It is the single place both sides take inputs from
(SURVEY.md §8(d) G1-G8).

Configs c0..c4 are BASELINE.json's ``configs`` (index = config number).
Fields marked "proposal" in SURVEY.md §8(d) are fixed here and restated in
DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libgblagen.so")


class _Params(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int64), ("n", ctypes.c_int64), ("npiv", ctypes.c_int64),
        ("rank_planted", ctypes.c_int64), ("k", ctypes.c_int64), ("run", ctypes.c_int64),
        ("band", ctypes.c_int64), ("band_np", ctypes.c_int64), ("chain", ctypes.c_int64),
        ("share", ctypes.c_double), ("lead_frac", ctypes.c_double),
        ("p", ctypes.c_uint32), ("pad_", ctypes.c_uint32), ("seed", ctypes.c_uint64),
    ]


class _Out(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int64), ("n", ctypes.c_int64), ("nnz", ctypes.c_int64),
        ("row_ptr", ctypes.POINTER(ctypes.c_uint64)), ("col", ctypes.POINTER(ctypes.c_uint32)),
        ("val", ctypes.POINTER(ctypes.c_uint16)), ("piv", ctypes.POINTER(ctypes.c_uint32)),
        ("npiv", ctypes.c_int64),
    ]


def build(force: bool = False) -> str:
    """Compile the generator (plain C, gcc)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-Wall", "-shared", "-fPIC", _SRC, "-o", _LIB])
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.gen_f4.argtypes = [ctypes.POINTER(_Params), ctypes.POINTER(_Out)]
        lib.gen_f4.restype = ctypes.c_int
        lib.gen_random.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_uint32,
                                   ctypes.c_uint64, ctypes.POINTER(_Out)]
        lib.gen_random.restype = ctypes.c_int
        lib.gen_free.argtypes = [ctypes.POINTER(_Out)]
        _lib = lib
    return _lib


@dataclass
class CSR:
    """Host CSR matrix over GF(p): row_ptr u64[m+1], col u32[nnz], val u16[nnz]."""
    m: int
    n: int
    p: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    piv: np.ndarray | None = None   # generator's pivot columns (F4 configs only)
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def to_dense(self) -> np.ndarray:
        a = np.zeros((self.m, self.n), dtype=np.int64)
        for i in range(self.m):
            s, e = int(self.row_ptr[i]), int(self.row_ptr[i + 1])
            a[i, self.col[s:e]] = self.val[s:e]
        return a


def _take(out: _Out, p: int, name: str) -> CSR:
    m, n, nnz = out.m, out.n, out.nnz
    rp = np.ctypeslib.as_array(out.row_ptr, shape=(m + 1,)).copy()
    col = np.ctypeslib.as_array(out.col, shape=(max(nnz, 1),))[:nnz].copy()
    val = np.ctypeslib.as_array(out.val, shape=(max(nnz, 1),))[:nnz].copy()
    piv = None
    if out.npiv > 0 and bool(out.piv):
        piv = np.ctypeslib.as_array(out.piv, shape=(out.npiv,)).copy()
    _load().gen_free(ctypes.byref(out))
    return CSR(m=m, n=n, p=p, row_ptr=rp, col=col, val=val, piv=piv, name=name)


@dataclass(frozen=True)
class F4Config:
    name: str
    m: int
    n: int
    npiv: int
    p: int
    seed: int
    density: float
    run: int
    band: int            # W for pivot rows (0: unbanded, runs up to the last column)
    band_np: int         # W for non-pivot rows
    share: float
    rank_planted: int
    lead_frac: float     # >0: non-pivot leads among pivot columns < lead_frac*n
    chain: int = 4096    # pattern-sharing chain restart period (proposal)

    @property
    def k(self) -> int:
        return int(round(self.density * self.n))

    @property
    def mN(self) -> int:
        return self.m - self.npiv

    @property
    def nN(self) -> int:
        return self.n - self.npiv


# BASELINE.json configs[0..4].
CONFIGS = {
    "c0": F4Config("c0", 1500, 1800, 1200, 65521, 0, 0.03, 4, 300, 0, 0.70, 250, 0.10),
    "c1": F4Config("c1", 45000, 55000, 38000, 65521, 1, 0.02, 8, 4000, 4000, 0.80, 6500, 0.0),
    "c2": F4Config("c2", 200000, 250000, 160000, 65521, 2, 0.01, 16, 10000, 10000, 0.70, 38000, 0.0),
    "c3": F4Config("c3", 60000, 80000, 40000, 32003, 3, 0.05, 32, 0, 0, 0.70, 19000, 0.05),
    "c4": F4Config("c4", 1000000, 1000000, 850000, 65521, 4, 0.002, 16, 40000, 40000, 0.70, 140000, 0.0),
}


def scaled(cfg: F4Config, scale: float, name: str | None = None) -> F4Config:
    """Same recipe at a fraction of the size (rows, columns, band, rank)."""
    f = lambda x: max(1, int(round(x * scale)))
    return F4Config(name or f"{cfg.name}@{scale:g}", f(cfg.m), f(cfg.n), f(cfg.npiv), cfg.p, cfg.seed,
                    cfg.density, cfg.run, f(cfg.band) if cfg.band else 0,
                    f(cfg.band_np) if cfg.band_np else 0, cfg.share, f(cfg.rank_planted),
                    cfg.lead_frac, cfg.chain)


def f4_matrix(cfg: F4Config | str) -> CSR:
    """Generate the F4-shaped matrix of a config (deterministic in cfg.seed)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    P = _Params(m=cfg.m, n=cfg.n, npiv=cfg.npiv, rank_planted=cfg.rank_planted, k=cfg.k,
                run=cfg.run, band=cfg.band, band_np=cfg.band_np, chain=cfg.chain,
                share=cfg.share, lead_frac=cfg.lead_frac, p=cfg.p, pad_=0, seed=cfg.seed)
    out = _Out()
    rc = _load().gen_f4(ctypes.byref(P), ctypes.byref(out))
    if rc != 0:
        raise ValueError(f"gen_f4 rejected config {cfg}")
    return _take(out, cfg.p, cfg.name)


def random_matrix(m: int, n: int, density: float, p: int, seed: int) -> CSR:
    """Plain random sparse matrix (non-monic rows, zero rows allowed)."""
    out = _Out()
    _load().gen_random(m, n, float(density), p, seed, ctypes.byref(out))
    return _take(out, p, f"rand{m}x{n}d{density:g}p{p}s{seed}")


def random_suite(count: int, seed0: int = 0, max_m: int = 100, max_n: int = 150,
                 primes=(3, 251, 32003, 65521)):
    """The randomized small-matrix suite (SPEC-style acceptance shapes)."""
    rng = np.random.default_rng(seed0)
    for i in range(count):
        m = int(rng.integers(1, max_m + 1))
        n = int(rng.integers(1, max_n + 1))
        d = float(rng.choice([0.01, 0.03, 0.1, 0.2, 0.4]))
        p = int(primes[i % len(primes)])
        yield random_matrix(m, n, d, p, seed0 * 100003 + i)


def gb_like_matrix(m: int, n: int, npoly: int, plen: int, p: int, seed: int, run: int = 4) -> CSR:
    """Rows of the form m_i * f_j: npoly base polynomials f_j (plen monic coefficients on
    a run-structured support), each row a random base polynomial shifted by a random column offset
    (monomial multiplication moves the support, the coefficients stay), plus a few unique rows.
    Exercises Format 2's polynomial deduplication and column-run compression; rows in random
    order, some duplicates of a (shift, polynomial) pair allowed.  Input generation only."""
    rng = np.random.default_rng(seed)
    span = 4 * plen
    bases = []
    for _ in range(npoly):
        offs = set()
        while len(offs) < plen:
            start = int(rng.integers(0, span - run))
            for u in range(int(rng.integers(1, run + 1))):
                offs.add(start + u)
        offs = sorted(offs)[:plen]
        offs = [o - offs[0] for o in offs]
        vals = rng.integers(1, p, len(offs))
        vals[0] = 1
        bases.append((np.array(offs, np.int64), vals.astype(np.int64)))
    rows = []
    for i in range(m):
        if i % 17 == 16:                                   # a unique row now and then
            k = int(rng.integers(1, plen + 1))
            c = np.sort(rng.choice(n, k, replace=False)).astype(np.int64)
            v = rng.integers(1, p, k)
            rows.append((c, v))
            continue
        offs, vals = bases[int(rng.integers(0, npoly))]
        sh = int(rng.integers(0, max(1, n - int(offs[-1]))))
        rows.append((offs + sh, vals))
    rp = np.zeros(m + 1, np.uint64)
    rp[1:] = np.cumsum([len(c) for c, _ in rows])
    col = np.concatenate([c for c, _ in rows]).astype(np.uint32) if m else np.zeros(0, np.uint32)
    val = np.concatenate([v for _, v in rows]).astype(np.uint16) if m else np.zeros(0, np.uint16)
    return CSR(m=m, n=n, p=p, row_ptr=rp, col=col, val=val, name=f"gblike{m}x{n}s{seed}")


# ---- residues below 2^31 (input generation only) --------------------------------
@dataclass
class WideCSR:
    """Host CSR over GF(p), p < 2^31: row_ptr u64[m+1], col u32[nnz], val u32[nnz]."""
    m: int
    n: int
    p: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if self.m else 0

    def dense(self) -> np.ndarray:
        a = np.zeros((self.m, self.n), np.int64)
        for i in range(self.m):
            s, e = int(self.row_ptr[i]), int(self.row_ptr[i + 1])
            a[i, self.col[s:e].astype(np.int64)] = self.val[s:e]
        return a


def random_wide(m: int, n: int, density: float, p: int, seed: int) -> WideCSR:
    """Random sparse matrix with residues in [1, p) (input generation only; zero rows allowed)."""
    rng = np.random.default_rng(seed)
    rp, cols, vals = [0], [], []
    for _ in range(m):
        k = int(rng.binomial(n, density))
        c = np.sort(rng.choice(n, k, replace=False)) if k else np.zeros(0, np.int64)
        cols.append(c)
        vals.append(rng.integers(1, p, c.size))
        rp.append(rp[-1] + c.size)
    col = np.concatenate(cols).astype(np.uint32) if cols else np.zeros(0, np.uint32)
    val = np.concatenate(vals).astype(np.uint32) if vals else np.zeros(0, np.uint32)
    return WideCSR(m, n, p, np.array(rp, np.uint64), col, val, f"wide{m}x{n}p{p}s{seed}")


def widen(M, p: int, seed: int) -> WideCSR:
    """An F4-shaped matrix's pattern (a gbla_gen CSR) with values redrawn in [1, p)."""
    rng = np.random.default_rng(seed)
    val = rng.integers(1, p, M.col.size).astype(np.uint32)
    return WideCSR(M.m, M.n, p, M.row_ptr.astype(np.uint64), M.col.astype(np.uint32), val,
                   f"{M.name}-p{p}")
