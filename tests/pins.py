"""Independent pins for the oracle (test helpers; no oracle code here).

``brute_rref`` is a textbook dense Gauss-Jordan elimination mod p over the
WHOLE matrix (numpy int64, vectorized row operations).  It is a different
algorithm from the oracle's splice -> Alg 2 -> RREF(D_new) pipeline and is
used to pin it.
"""
from __future__ import annotations

import numpy as np


def brute_rref(a: np.ndarray, p: int):
    """Canonical RREF of a dense integer matrix mod p.
    Returns (rank, R (rank x cols, int64), pivot columns list)."""
    a = np.array(a, dtype=np.int64) % p
    rows, cols = a.shape
    r = 0
    piv = []
    for c in range(cols):
        if r >= rows:
            break
        nz = np.nonzero(a[r:, c])[0]
        if nz.size == 0:
            continue
        s = r + int(nz[0])
        if s != r:
            a[[r, s]] = a[[s, r]]
        inv = pow(int(a[r, c]), p - 2, p)          # Fermat: p prime
        a[r] = (a[r] * inv) % p
        f = a[:, c].copy()
        f[r] = 0
        nzr = np.nonzero(f)[0]
        if nzr.size:
            a[nzr] = (a[nzr] - (f[nzr, None] * a[r][None, :]) % p) % p
        piv.append(c)
        r += 1
    return r, a[:r].copy(), piv


def dense_sigma(M, sigma: np.ndarray) -> np.ndarray:
    """Dense M with columns permuted by sigma (column c goes to sigma[c])."""
    d = M.to_dense()
    out = np.zeros_like(d)
    out[:, sigma.astype(np.int64)] = d
    return out


def matmul_mod(X: np.ndarray, Y: np.ndarray, p: int) -> np.ndarray:
    """Exact X*Y mod p for residues (chunked so int64 never overflows)."""
    X = np.asarray(X, np.int64) % p
    Y = np.asarray(Y, np.int64) % p
    out = np.zeros((X.shape[0], Y.shape[1]), np.int64)
    step = max(1, (2 ** 62) // ((p - 1) ** 2 + 1) // 2)
    for k0 in range(0, X.shape[1], step):
        out = (out + X[:, k0:k0 + step] @ Y[k0:k0 + step, :]) % p
    return out


def rank_mod(a: np.ndarray, p: int) -> int:
    return brute_rref(a, p)[0]
