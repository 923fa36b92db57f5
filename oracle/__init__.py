"""CPU oracle for the Faugere-Lachartre reduction -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_1602_06097_b200``) never imports it and fails loudly
when its CUDA library is missing.

The arithmetic lives in ``gbla_oracle.c`` (plain C, each function citing the
PAPER.md passage it follows); this module only marshals numpy arrays.

Parity status: every function here is pinned by ``tests/test_oracle_pins.py``
(see DESIGN.md §"Oracle pins").  No function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gbla_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
NONE = 0xFFFFFFFF

_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(dtype=np.uint16, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, plain C + pthreads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-Wall", "-shared", "-fPIC", "-pthread", _SRC, "-o", _LIB])
    return _LIB


_lib = None


def _nullable(t):
    def from_param(obj):
        if obj is None:
            return None
        return t.from_param(obj)
    return type("Nullable", (), {"from_param": staticmethod(from_param)})


def _load():
    global _lib
    if _lib is not None:
        return _lib
    build()
    L = ctypes.CDLL(_LIB)
    i64, u32 = ctypes.c_int64, ctypes.c_uint32
    L.orc_is_prime.argtypes = [u32]; L.orc_is_prime.restype = ctypes.c_int
    L.orc_inv.argtypes = [u32, u32]; L.orc_inv.restype = u32
    L.orc_validate.argtypes = [i64, i64, _u64p, _u32p, _u16p, u32]; L.orc_validate.restype = ctypes.c_int
    L.orc_splice.argtypes = [i64, i64, _u64p, _u32p, _u32p, _u32p, _u32p, _u32p,
                             ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.orc_splice.restype = ctypes.c_int
    n32 = _nullable(_u32p)
    L.orc_quadrants.argtypes = [i64, i64, _u64p, _u32p, _u16p, u32, _u32p, _u32p, i64, _u32p, i64,
                                n32, n32, n32, n32]
    L.orc_dnew.argtypes = [i64, i64, _u64p, _u32p, _u16p, u32, _u32p, _u32p, i64, _u32p, i64,
                           _i64p, i64, _u16p, _nullable(_u16p), _nullable(_u64p), ctypes.c_int]
    L.orc_trsm.argtypes = [_u32p, _u32p, _u32p, i64, i64, u32]
    L.orc_sub_mul.argtypes = [_u32p, _u32p, _u32p, _u32p, i64, i64, i64, u32]
    L.orc_rref.argtypes = [_u32p, i64, i64, u32, _u32p, ctypes.c_int]; L.orc_rref.restype = i64
    L.orc_multiline.argtypes = [_u32p, _u32p, i64, _u32p, _u32p]; L.orc_multiline.restype = i64
    L.orc_ml_axpy.argtypes = [_u32p, _u32p, u32, u32, u32, u32, _u32p, _u32p, i64, u32]
    _lib = L
    return L


def default_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


# ----------------------------------------------------------------- field
def is_prime(p: int) -> bool:
    return bool(_load().orc_is_prime(p))


def inv(a: int, p: int) -> int:
    return int(_load().orc_inv(a % p, p))


def validate(M) -> int:
    return int(_load().orc_validate(M.m, M.n, M.row_ptr, M.col, M.val, M.p))


# ----------------------------------------------------------------- Step 1
@dataclass
class Splice:
    m: int
    n: int
    p: int
    npiv: int
    mN: int
    lead: np.ndarray          # u32[m], NONE for zero rows
    sigma: np.ndarray         # u32[n]
    pivot_row: np.ndarray     # u32[npiv]
    nonpivot_row: np.ndarray  # u32[mN]

    @property
    def nN(self) -> int:
        return self.n - self.npiv


def splice(M) -> Splice:
    """Step 1, readings R1-R7 (see gbla_oracle.c:orc_splice)."""
    L = _load()
    if L.orc_validate(M.m, M.n, M.row_ptr, M.col, M.val, M.p) != 0:
        raise ValueError("invalid input matrix / modulus")
    lead = np.empty(M.m, np.uint32)
    sigma = np.empty(M.n, np.uint32)
    prow = np.empty(max(M.n, 1), np.uint32)
    nprow = np.empty(max(M.m, 1), np.uint32)
    npiv, mN = ctypes.c_int64(), ctypes.c_int64()
    L.orc_splice(M.m, M.n, M.row_ptr, M.col, lead, sigma, prow, nprow, ctypes.byref(npiv), ctypes.byref(mN))
    return Splice(M.m, M.n, M.p, npiv.value, mN.value, lead, sigma, prow[:npiv.value].copy(),
                  nprow[:mN.value].copy())


def quadrants(M, S: Splice):
    """Dense A, B, C, D (uint32 residues, sigma column order). Small inputs only."""
    A = np.zeros((S.npiv, S.npiv), np.uint32)
    B = np.zeros((S.npiv, S.nN), np.uint32)
    C = np.zeros((S.mN, S.npiv), np.uint32)
    D = np.zeros((S.mN, S.nN), np.uint32)
    _load().orc_quadrants(M.m, M.n, M.row_ptr, M.col, M.val, M.p, S.sigma, _pad(S.pivot_row),
                          S.npiv, _pad(S.nonpivot_row), S.mN, A, B, C, D)
    return A, B, C, D


def _pad(a):
    return a if a.size else np.zeros(1, a.dtype)


# ------------------------------------------------------ Alg 2 (new order)
def dnew_rows(M, S: Splice, targets=None, want_x: bool = False, threads: int | None = None):
    """D_new rows (u16, nN wide), C' rows (u16, npiv wide) and modMAC counts
    for the given targets (indices into the non-pivot rows), by Alg 2."""
    if targets is None:
        targets = np.arange(S.mN, dtype=np.int64)
    targets = np.ascontiguousarray(targets, dtype=np.int64)
    nt = targets.size
    dnew = np.zeros((max(nt, 1), max(S.nN, 1)), np.uint16)
    x = np.zeros((max(nt, 1), max(S.npiv, 1)), np.uint16) if want_x else None
    ops = np.zeros(max(nt, 1), np.uint64)
    if nt:
        _load().orc_dnew(M.m, M.n, M.row_ptr, M.col, M.val, M.p, S.sigma, _pad(S.pivot_row), S.npiv,
                         _pad(S.nonpivot_row), S.mN, targets, nt, dnew, x, ops,
                         threads or default_threads())
    dnew = dnew[:nt, :S.nN]
    if x is not None:
        x = x[:nt, :S.npiv]
    return dnew, x, ops[:nt]


# ---------------------------------------------------- standard order parts
def trsm(A: np.ndarray, B: np.ndarray, p: int) -> np.ndarray:
    """Step 2: B' = A^-1 B."""
    A = np.ascontiguousarray(A, np.uint32); B = np.ascontiguousarray(B, np.uint32)
    npiv, nN = B.shape
    Bp = np.zeros((max(npiv, 1), max(nN, 1)), np.uint32)
    if npiv and nN:
        _load().orc_trsm(A, B, Bp, npiv, nN, p)
    return Bp[:npiv, :nN]


def sub_mul(D: np.ndarray, X: np.ndarray, Y: np.ndarray, p: int) -> np.ndarray:
    """Step 3: D - X*Y mod p."""
    D = np.ascontiguousarray(D, np.uint32); X = np.ascontiguousarray(X, np.uint32)
    Y = np.ascontiguousarray(Y, np.uint32)
    rows, cols = D.shape
    inner = X.shape[1]
    out = np.zeros((max(rows, 1), max(cols, 1)), np.uint32)
    if rows and cols:
        if inner == 0:
            return D.copy()
        _load().orc_sub_mul(D, X, Y, out, rows, inner, cols, p)
    return out[:rows, :cols]


# ------------------------------------------------------------- Step 4 RREF
def rref(D: np.ndarray, p: int, threads: int | None = None):
    """Canonical RREF (reading R13). Returns (rank, R[rank x cols] u16, pivcol u32[rank])."""
    a = np.ascontiguousarray(D, dtype=np.uint32).copy()
    rows, cols = a.shape
    if rows == 0 or cols == 0:
        return 0, np.zeros((0, cols), np.uint16), np.zeros(0, np.uint32)
    pc = np.zeros(max(rows, 1), np.uint32)
    r = int(_load().orc_rref(a, rows, cols, p, pc, threads or default_threads()))
    return r, a[:r].astype(np.uint16), pc[:r].copy()


# ------------------------------------------------------------- multiline
def multiline(r1, r2):
    r1 = np.ascontiguousarray(r1, np.uint32); r2 = np.ascontiguousarray(r2, np.uint32)
    n = r1.size
    pos = np.zeros(max(n, 1), np.uint32); val = np.zeros(max(2 * n, 2), np.uint32)
    l = int(_load().orc_multiline(r1, r2, n, pos, val))
    return pos[:l].copy(), val[:2 * l].copy()


def ml_axpy(d1, d2, l11, l12, l21, l22, pos, val, p):
    d1 = np.ascontiguousarray(d1, np.uint32).copy(); d2 = np.ascontiguousarray(d2, np.uint32).copy()
    pos = np.ascontiguousarray(pos, np.uint32); val = np.ascontiguousarray(val, np.uint32)
    _load().orc_ml_axpy(d1, d2, l11, l12, l21, l22, _pad(pos), _pad(val), pos.size, p)
    return d1, d2


# ----------------------------------------------------------- whole pipeline
@dataclass
class Result:
    splice: Splice
    dnew: np.ndarray          # mN x nN u16
    rank: int
    R: np.ndarray             # rank x nN u16
    pivcol: np.ndarray        # u32[rank]
    modmac: int               # sparse-phase modMACs (Alg 2 count)
    x: np.ndarray | None = None
    extra: dict = field(default_factory=dict)

    @property
    def rank_M(self) -> int:
        return self.splice.npiv + self.rank


def reduce(M, want_x: bool = False, threads: int | None = None) -> Result:
    """Whole pipeline (new order, fully reduced echelon of D):
    Step 1 -> Alg 2 -> RREF(D_new)."""
    S = splice(M)
    dn, x, ops = dnew_rows(M, S, want_x=want_x, threads=threads)
    rank, R, pc = rref(dn, M.p, threads=threads)
    return Result(S, dn, rank, R, pc, int(ops.sum()), x)


def full_rref(M, res: Result | None = None, threads: int | None = None):
    """the fully reduced row echelon form of the WHOLE M in its original column
    order, by the paper's route: Step 2 B' = A^-1 B (orc_trsm), the second
    reduction of the pivot rows by R, B'' = B' - B'[:, pivcol(R)] R (orc_sub_mul), and
    Step 5: the columns back in the original order, rows sorted by pivot column.  The
    pivot rows become [1 at their pivot column | B''] and the R rows [0 | R].
    Returns (rank(M), RREF(M) as a dense u16 array rank(M) x n, pivot columns u32[rank(M)]).
    Small inputs only (dense quadrants).  Pinned by the textbook Gauss-Jordan RREF of M
    (tests/pins.py brute_rref) -- the RREF is unique."""
    if res is None:
        res = reduce(M, threads=threads)
    S = res.splice
    p = M.p
    A, B, _, _ = quadrants(M, S)
    Bp = trsm(A, B, p)                                                     # Step 2
    Bpp = sub_mul(Bp, Bp[:, res.pivcol.astype(np.int64)], res.R.astype(np.uint32), p) if res.rank else Bp
    inv_sigma = np.empty(M.n, np.int64)                                   # sigma index -> original column
    inv_sigma[S.sigma.astype(np.int64)] = np.arange(M.n)
    pcol, ncol = inv_sigma[:S.npiv], inv_sigma[S.npiv:]
    rank_M = S.npiv + res.rank
    out = np.zeros((rank_M, M.n), np.uint16)
    piv = np.concatenate([pcol, ncol[res.pivcol.astype(np.int64)]]).astype(np.int64)
    out[np.arange(S.npiv), pcol] = 1                                       # Step 5: original columns
    out[:S.npiv, ncol] = Bpp
    out[S.npiv:, ncol] = res.R
    order = np.argsort(piv, kind="stable")                                 # rows by pivot column
    return rank_M, out[order], piv[order].astype(np.uint32)


def rref_digest(rank: int, nN: int, pivcol: np.ndarray, R: np.ndarray) -> str:
    """SHA-256 of LE bytes (u32 rank, u32 nN, u32 pivcol[rank], u16 R row-major)."""
    h = hashlib.sha256()
    h.update(np.array([rank, nN], dtype="<u4").tobytes())
    h.update(np.ascontiguousarray(pivcol, dtype="<u4").tobytes())
    h.update(np.ascontiguousarray(R, dtype="<u2").tobytes())
    return h.hexdigest()


def array_digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u2").tobytes()).hexdigest()
