"""SURVEY 8(f) f4 oracle -- wider prime fields ("the float type for p < 2^23" and 32-bit
residues) -- TEST INFRASTRUCTURE ONLY (only tests/ may import it).

The same reduction as gbla_oracle.c, written out in numpy for residues below 2^31 (products below
2^62 fit int64; every operation is reduced mod p at once -- no delayed reduction), for small
inputs only:
  Step 1 (readings R1-R7): every nonzero row made monic by the inverse of its leading
    value (Python's pow(a, -1, p)), P = the leading columns, the pivot row of a column = the
    candidate of minimum (weight, row id), sigma = P ascending then the other columns ascending;
  Alg 2 (R8/R9): per target, lambda = acc[j] captured, acc -= lambda * pivot row j, for
    j ascending from the target's lead; the modMAC count adds nnz(row_j) - 1 per nonzero lambda;
  Step 4 (R13): canonical RREF of D_new by textbook Gauss-Jordan.
Pinned (tests/test_oracle_pins.py) by the brute-force Gauss-Jordan of the whole M*sigma
(tests/pins.py, rank additivity, R = the bottom-right block) and by equality with the C oracle
for p < 2^16.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class WideResult:
    npiv: int
    sigma: np.ndarray
    pivot_row: np.ndarray
    nonpivot_row: np.ndarray
    dnew: np.ndarray          # mN x nN (int64 residues)
    rank: int
    R: np.ndarray             # rank x nN
    pivcol: np.ndarray
    modmac: int

    @property
    def rank_M(self) -> int:
        return self.npiv + self.rank


def _rref(a: np.ndarray, p: int):
    a = a.copy() % p
    rows, cols = a.shape
    r, piv = 0, []
    for c in range(cols):
        if r >= rows:
            break
        nz = np.nonzero(a[r:, c])[0]
        if nz.size == 0:
            continue
        s = r + int(nz[0])
        if s != r:
            a[[r, s]] = a[[s, r]]
        a[r] = (a[r] * pow(int(a[r, c]), -1, p)) % p
        for i in np.nonzero(a[:, c])[0]:
            if i != r:
                a[i] = (a[i] - (int(a[i, c]) * a[r]) % p) % p
        piv.append(c)
        r += 1
    return r, a[:r].copy(), np.array(piv, np.int64)


def reduce(M) -> WideResult:
    """M: a gbla_gen.WideCSR (row_ptr u64, col u32, val u32, p < 2^31)."""
    p = M.p
    rows = []
    lead, weight = np.full(M.m, -1, np.int64), np.zeros(M.m, np.int64)
    for i in range(M.m):                                          # Step 1: monic rows (R6)
        s, e = int(M.row_ptr[i]), int(M.row_ptr[i + 1])
        c = M.col[s:e].astype(np.int64)
        v = M.val[s:e].astype(np.int64) % p
        if c.size:
            v = (v * pow(int(v[0]), -1, p)) % p
            lead[i], weight[i] = c[0], c.size
        rows.append((c, v))
    best = {}
    for i in range(M.m):                                          # min (weight, id) per lead (R1)
        if lead[i] >= 0:
            k = (weight[i], i)
            if lead[i] not in best or k < best[lead[i]]:
                best[lead[i]] = k
    P = sorted(best)
    Pset = set(P)
    N = [c for c in range(M.n) if c not in Pset]
    sigma = np.empty(M.n, np.int64)
    sigma[P] = np.arange(len(P))
    sigma[N] = len(P) + np.arange(len(N))
    npiv = len(P)
    pivot_row = np.array([best[c][1] for c in P], np.int64)
    piv_set = set(pivot_row.tolist())
    nonpivot = np.array([i for i in range(M.m) if i not in piv_set], np.int64)

    def dense_row(i):
        d = np.zeros(M.n, np.int64)
        c, v = rows[i]
        d[sigma[c]] = v
        return d

    A = np.array([dense_row(i) for i in pivot_row]).reshape(npiv, M.n)
    w = np.array([rows[i][0].size for i in pivot_row], np.int64)
    mN, nN = nonpivot.size, M.n - npiv
    dnew = np.zeros((mN, nN), np.int64)
    ops = 0
    for t, i in enumerate(nonpivot):                              # Alg 2
        acc = dense_row(i)
        l0 = int(sigma[lead[i]]) if lead[i] >= 0 else npiv
        for j in range(l0, npiv):
            lam = int(acc[j])                                     # captured before use (R9)
            if lam:
                acc = (acc - lam * A[j]) % p                      # subtract (R8)
                ops += int(w[j]) - 1
        dnew[t] = acc[npiv:]
    rank, R, pc = _rref(dnew, p)
    return WideResult(npiv, sigma, pivot_row, nonpivot, dnew, rank, R, pc, ops)
