"""Generator checks (-m "not gpu"): determinism and the config shapes."""
import json
import os

import numpy as np

import gbla_gen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _csr_digest(M):
    import hashlib
    h = hashlib.sha256()
    for a, dt in ((M.row_ptr, "<u8"), (M.col, "<u4"), (M.val, "<u2")):
        h.update(np.ascontiguousarray(a, dtype=dt).tobytes())
    return h.hexdigest()


def test_c0_is_deterministic_and_matches_golden(c0_matrix):
    with open(os.path.join(GOLD, "c0_oracle.json")) as f:
        g = json.load(f)
    assert _csr_digest(c0_matrix) == g["csr_sha256"]
    assert _csr_digest(gbla_gen.f4_matrix("c0")) == g["csr_sha256"]


def test_c0_shape(c0_matrix):
    M, cfg = c0_matrix, gbla_gen.CONFIGS["c0"]
    assert (M.m, M.n) == (cfg.m, cfg.n)
    rp = M.row_ptr.astype(np.int64)
    lens = np.diff(rp)
    assert lens.min() > 0
    assert np.all(M.val[rp[:-1]] == 1)                       # monic rows
    leads = M.col[rp[:-1]]
    assert np.array_equal(np.unique(leads), M.piv)           # P = generator pivots
    for i in range(M.m):
        c = M.col[rp[i]:rp[i + 1]].astype(np.int64)
        assert np.all(np.diff(c) > 0)
    assert np.all((M.val > 0) & (M.val < M.p))


def test_scaled_configs_generate():
    for name in ("c1", "c2", "c3", "c4"):
        cfg = gbla_gen.scaled(gbla_gen.CONFIGS[name], 0.01 if name != "c4" else 0.002)
        M = gbla_gen.f4_matrix(cfg)
        leads = np.unique(M.col[M.row_ptr[:-1].astype(np.int64)])
        assert leads.size == cfg.npiv
        assert M.m == cfg.m and M.n == cfg.n


def test_random_matrix_deterministic():
    a = gbla_gen.random_matrix(30, 40, 0.2, 251, 9)
    b = gbla_gen.random_matrix(30, 40, 0.2, 251, 9)
    assert np.array_equal(a.col, b.col) and np.array_equal(a.val, b.val)
