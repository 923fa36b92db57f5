"""Pins for the CPU oracle (-m "not gpu").

Each oracle function is checked against something other than itself:
values the paper prints, SPEC worked examples (derived),
closed forms (A*B' = B, C'*A = C), invariants (rank(M) = n_piv + rank(D_new),
RREF idempotence and row-permutation invariance) and an independent
brute-force dense Gauss-Jordan over the whole M*sigma (tests/pins.py).
"""
import json
import os

import numpy as np
import pytest

import gbla_gen
import oracle
from conftest import csr_from_dense
from pins import brute_rref, dense_sigma, matmul_mod

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _json(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# --------------------------------------------------------------- field
def test_field_primes_and_inverses():
    ex = _json("spec_examples.json")["field"]
    assert oracle.is_prime(65521) and oracle.is_prime(32003) and oracle.is_prime(3)
    assert not oracle.is_prime(65523) and not oracle.is_prime(32001) and not oracle.is_prime(1)
    # 65521 is the largest 16-bit prime
    assert not any(oracle.is_prime(q) for q in range(65522, 65536))
    assert oracle.inv(2, 65521) == ex["inv_2_65521"]
    assert (40000 + 40000) % 65521 == ex["add_40000_40000_65521"]
    assert oracle.inv(0, 65521) == 0
    # exhaustive inverse check for small primes, sampled for 65521 / 32003
    for p in (3, 5, 7, 251, 257):
        for a in range(1, p):
            assert a * oracle.inv(a, p) % p == 1
    rng = np.random.default_rng(0)
    for p in (32003, 65521):
        for a in rng.integers(1, p, 500):
            assert int(a) * oracle.inv(int(a), p) % p == 1


# ------------------------------------------------------------- multiline
def test_multiline_paper_example():
    ex = _json("multiline_example.json")
    pos, val = oracle.multiline(ex["r1"], ex["r2"])
    assert pos.tolist() == ex["ml_pos"]
    assert val.tolist() == ex["ml_val"]
    # no-useless-column and <=1 padding zero per column
    v = val.reshape(-1, 2)
    assert np.all((v != 0).any(axis=1))
    assert int((v == 0).sum()) <= len(pos)


def test_multiline_axpy_equals_four_scalar_axpys():
    rng = np.random.default_rng(1)
    for p in (7, 251, 65521):
        for _ in range(20):
            n = 40
            r1 = rng.integers(0, p, n) * (rng.random(n) < 0.4)
            r2 = rng.integers(0, p, n) * (rng.random(n) < 0.4)
            d1 = rng.integers(0, p, n); d2 = rng.integers(0, p, n)
            l = [int(x) for x in rng.integers(0, p, 4)]
            pos, val = oracle.multiline(r1, r2)
            o1, o2 = oracle.ml_axpy(d1, d2, l[0], l[1], l[2], l[3], pos, val, p)
            e1 = (d1 - l[0] * r1 - l[1] * r2) % p
            e2 = (d2 - l[2] * r1 - l[3] * r2) % p
            assert np.array_equal(o1, e1) and np.array_equal(o2, e2)


# ---------------------------------------------------------------- splice
def test_splice_identity_and_tie_rule():
    I = csr_from_dense(np.eye(5, dtype=np.int64), 7)
    S = oracle.splice(I)
    assert S.npiv == 5 and S.mN == 0
    assert S.sigma.tolist() == list(range(5))
    A, B, C, D = oracle.quadrants(I, S)
    assert np.array_equal(A, np.eye(5))
    ex = _json("spec_examples.json")["splice_tie"]
    M = csr_from_dense(ex["M"], ex["p"])
    R = oracle.reduce(M)
    assert R.splice.npiv == ex["npiv"]
    assert R.splice.pivot_row.tolist() == [ex["pivot_row"]]
    assert R.dnew.tolist() == ex["dnew"]                      # 3 - 1*2 = 1
    assert R.rank_M == ex["rank_M"]


def test_splice_normalizes_rows():
    ex = _json("spec_examples.json")["normalize"]
    M = csr_from_dense([ex["row"]], ex["p"])
    S = oracle.splice(M)
    A, B, C, D = oracle.quadrants(M, S)
    assert np.concatenate([A[0], B[0]]).tolist() == ex["monic"]


def test_splice_properties_random():
    for M in gbla_gen.random_suite(60, seed0=3):
        S = oracle.splice(M)
        dense = M.to_dense()
        leads = {int(np.nonzero(r)[0][0]) for r in dense if r.any()}
        assert S.npiv == len(leads)                                      # distinct leads
        assert sorted(S.sigma.tolist()) == list(range(M.n))              # bijection
        # pivot rows: lead maps to its sigma index; minimum weight, lowest id
        w = (dense != 0).sum(axis=1)
        for i, r in enumerate(S.pivot_row):
            lc = int(np.nonzero(dense[r])[0][0])
            assert S.sigma[lc] == i
            cands = [q for q in range(M.m) if dense[q].any() and int(np.nonzero(dense[q])[0][0]) == lc]
            assert int(r) == min(cands, key=lambda q: (w[q], q))
        # permute back: [A B; C D] rows/cols back = row-normalized input
        A, B, C, D = oracle.quadrants(M, S)
        top = np.hstack([A, B]).astype(np.int64); bot = np.hstack([C, D]).astype(np.int64)
        for i, r in enumerate(S.pivot_row):
            row = dense[r] % M.p
            inv = pow(int(row[np.nonzero(row)[0][0]]), M.p - 2, M.p)
            assert np.array_equal(top[i][S.sigma], (row * inv) % M.p)
        for i, r in enumerate(S.nonpivot_row):
            row = dense[r] % M.p
            if row.any():
                row = (row * pow(int(row[np.nonzero(row)[0][0]]), M.p - 2, M.p)) % M.p
            assert np.array_equal(bot[i][S.sigma], row)
        # A upper unitriangular
        if S.npiv:
            assert np.all(np.diag(A) == 1) and not np.tril(A, -1).any()


# ------------------------------------------------------------ TRSM / C'
def test_trsm_examples_and_closed_form():
    ex = _json("spec_examples.json")["trsm"]
    Bp = oracle.trsm(np.array(ex["A"]), np.array(ex["B"]), ex["p"])
    assert Bp.tolist() == ex["Bp"]
    assert np.array_equal(oracle.trsm(np.eye(3, dtype=np.uint32), np.arange(6).reshape(3, 2), 7),
                          np.arange(6).reshape(3, 2))
    for M in gbla_gen.random_suite(40, seed0=5):
        S = oracle.splice(M)
        A, B, C, D = oracle.quadrants(M, S)
        Bp = oracle.trsm(A, B, M.p)
        assert np.array_equal(matmul_mod(A, Bp, M.p), B.astype(np.int64))       # A * B' = B


def test_cprime_closed_form_and_order_equivalence():
    for M in gbla_gen.random_suite(60, seed0=7):
        S = oracle.splice(M)
        A, B, C, D = oracle.quadrants(M, S)
        dn, x, ops = oracle.dnew_rows(M, S, want_x=True)
        p = M.p
        assert np.array_equal(matmul_mod(x, A, p), C.astype(np.int64))           # C' * A = C
        # new order == standard order == Schur complement
        Bp = oracle.trsm(A, B, p)
        std = oracle.sub_mul(D, C, Bp, p)
        new4 = oracle.sub_mul(D, x.astype(np.uint32), B, p)
        assert np.array_equal(dn.astype(np.uint32), std)
        assert np.array_equal(dn.astype(np.uint32), new4)
        # modMAC count: every nonzero lambda applies nnz(row_j) - 1 products
        w = np.diff(M.row_ptr.astype(np.int64))
        exp = int(((x != 0) * (w[S.pivot_row.astype(np.int64)] - 1)[None, :]).sum()) if S.npiv else 0
        assert int(ops.sum()) == exp


def test_update_trivial_cases():
    # C = 0 -> D unchanged; 1x1 quadrants -> d - c*b
    D = np.array([[3, 4]], np.uint32)
    assert np.array_equal(oracle.sub_mul(D, np.zeros((1, 2), np.uint32), np.ones((2, 2), np.uint32), 7), D)
    assert oracle.sub_mul(np.array([[5]]), np.array([[3]]), np.array([[4]]), 7).tolist() == [[(5 - 12) % 7]]


# ------------------------------------------------------------------ RREF
def test_rref_examples():
    ex = _json("spec_examples.json")["rref"]
    r, R, pc = oracle.rref(np.array(ex["D"]), ex["p"])
    assert r == ex["rank"] and R.tolist() == ex["R"] and pc.tolist() == ex["pivcol"]
    r, R, pc = oracle.rref(np.zeros((4, 5), np.uint32), 7)
    assert r == 0


def test_rref_against_brute_force_and_invariances():
    rng = np.random.default_rng(11)
    for t in range(60):
        p = [3, 251, 32003, 65521][t % 4]
        rows, cols = int(rng.integers(1, 40)), int(rng.integers(1, 50))
        D = rng.integers(0, p, (rows, cols)) * (rng.random((rows, cols)) < rng.choice([0.1, 0.5, 1.0]))
        r, R, pc = oracle.rref(D, p)
        br, bR, bpc = brute_rref(D, p)
        assert r == br and np.array_equal(R.astype(np.int64), bR) and pc.tolist() == bpc
        # idempotence and row-permutation invariance
        r2, R2, _ = oracle.rref(R, p)
        assert r2 == r and np.array_equal(R2, R)
        perm = rng.permutation(rows)
        r3, R3, _ = oracle.rref(D[perm], p)
        assert r3 == r and np.array_equal(R3, R)
    # threads do not change the result
    D = rng.integers(0, 65521, (64, 80))
    assert np.array_equal(oracle.rref(D, 65521, threads=1)[1], oracle.rref(D, 65521, threads=7)[1])


# ------------------------------------------------------- whole pipeline
def _check_against_brute(M, res):
    """R = bottom-right block of RREF(M*sigma); first npiv columns are pivots;
    rank(M) = npiv + rank(D_new) (SURVEY §8(c) proof, O9)."""
    S = res.splice
    Ms = dense_sigma(M, S.sigma)
    br, bR, bpc = brute_rref(Ms, M.p)
    assert br == S.npiv + res.rank
    assert bpc[:S.npiv] == list(range(S.npiv))
    assert [c - S.npiv for c in bpc[S.npiv:]] == res.pivcol.tolist()
    assert np.array_equal(bR[S.npiv:, S.npiv:], res.R.astype(np.int64))
    # rank in original column order is the same
    assert brute_rref(M.to_dense(), M.p)[0] == br


def test_pipeline_random_suite_against_brute_force():
    n = 0
    for M in gbla_gen.random_suite(300, seed0=13):
        res = oracle.reduce(M, threads=2)
        _check_against_brute(M, res)
        n += 1
    assert n == 300


def test_pipeline_c0_against_brute_force(c0_matrix, c0_oracle):
    res = c0_oracle
    cfg = gbla_gen.CONFIGS["c0"]
    assert res.splice.npiv == cfg.npiv and res.splice.mN == cfg.mN       # G8 self-check
    assert res.rank == cfg.rank_planted                                   # planted rank
    assert abs(c0_matrix.nnz / (cfg.m * cfg.n) - cfg.density) / cfg.density < 0.1
    _check_against_brute(c0_matrix, res)


def test_pipeline_threads_and_row_order_invariance(c0_matrix, c0_oracle):
    """R and rank do not depend on row order (proof in SURVEY §8(c)); D_new
    does not depend on the oracle's thread count."""
    M = c0_matrix
    rng = np.random.default_rng(2)
    perm = rng.permutation(M.m)
    rp = np.zeros(M.m + 1, np.uint64)
    lens = np.diff(M.row_ptr.astype(np.int64))[perm]
    rp[1:] = np.cumsum(lens)
    cols, vals = [], []
    for r in perm:
        s, e = int(M.row_ptr[r]), int(M.row_ptr[r + 1])
        cols.append(M.col[s:e]); vals.append(M.val[s:e])
    M2 = gbla_gen.CSR(M.m, M.n, M.p, rp, np.concatenate(cols), np.concatenate(vals))
    r2 = oracle.reduce(M2, threads=3)
    assert r2.rank == c0_oracle.rank
    assert np.array_equal(r2.R, c0_oracle.R) and np.array_equal(r2.pivcol, c0_oracle.pivcol)
    r1 = oracle.reduce(M, threads=1)
    assert np.array_equal(r1.dnew, c0_oracle.dnew) and r1.modmac == c0_oracle.modmac


def test_validate_rejects_bad_input():
    M = csr_from_dense([[1, 2], [0, 3]], 7)
    assert oracle.validate(M) == 0
    bad = gbla_gen.CSR(2, 2, 7, M.row_ptr.copy(), M.col[::-1].copy(), M.val.copy())
    assert oracle.validate(bad) != 0
    assert oracle.validate(gbla_gen.CSR(2, 2, 8, M.row_ptr, M.col, M.val)) != 0   # 8 not prime
    badv = M.val.copy(); badv[0] = 7
    assert oracle.validate(gbla_gen.CSR(2, 2, 7, M.row_ptr, M.col, badv)) == 4         # val >= p
    zero = M.val.copy(); zero[1] = 0
    assert oracle.validate(gbla_gen.CSR(2, 2, 7, M.row_ptr, M.col, zero)) == 4         # explicit zero
    wide = M.col.copy(); wide[-1] = 2
    assert oracle.validate(gbla_gen.CSR(2, 2, 7, M.row_ptr, wide, M.val)) == 3         # col >= n
    assert oracle.validate(bad) == 3                                                    # unsorted columns
    assert oracle.validate(gbla_gen.CSR(2, 2, 7, np.array([0, 2, 3], np.uint64), np.array([0, 0, 1], np.uint32),
                                        np.array([1, 2, 3], np.uint16))) == 3       # duplicate column
    assert oracle.validate(gbla_gen.CSR(2, 2, 7, np.array([0, 2, 1], np.uint64), M.col, M.val)) == 2   # row_ptr
    with pytest.raises(ValueError):
        oracle.splice(gbla_gen.CSR(2, 2, 7, M.row_ptr, M.col, zero))


def test_modmac_count_hand_derived():
    """The sparse-phase modMAC count (the numerator of the bench metric) on hand-worked Alg 2 runs
    (reading R8/R9: lambda captured before use, subtract lambda * row_j, count
    nnz(row_j) - 1 per nonzero lambda), not by re-typing the oracle's formula."""
    # SPEC tie example [[1,2],[1,3]] mod 7: pivot row 0 (equal weights, lower id); the target
    # [1,3] takes lambda = 1 once against a 2-entry row: 1 modMAC, D_new = [3 - 2] = [1]
    R = oracle.reduce(csr_from_dense([[1, 2], [1, 3]], 7))
    assert R.modmac == 1 and R.dnew.tolist() == [[1]]
    # three pivots, p = 7, pivot rows r0 = [1,2,0,0,1], r1 = [0,1,3,0,0], r2 = [0,0,1,4,0]; target
    # t = [1,1,1,1,1]: lambda_0 = 1 -> t = [0,6,1,1,0] (+2), lambda_1 = 6 -> [0,0,4,1,0] (+1),
    # lambda_2 = 4 -> [0,0,0,6,0] (+1): 4 modMACs, D_new = [6, 0]
    rows = [[1, 2, 0, 0, 1], [0, 1, 3, 0, 0], [0, 0, 1, 4, 0]]
    R = oracle.reduce(csr_from_dense(rows + [[1, 1, 1, 1, 1]], 7))
    assert R.splice.npiv == 3 and R.modmac == 4 and R.dnew.tolist() == [[6, 0]]
    assert R.rank == 1 and R.R.tolist() == [[1, 0]] and R.rank_M == 4
    # a zero lambda is skipped (no count): t = [1,2,6,0,1] -> [0,0,6,0,0] (+2), lambda_1 = 0,
    # lambda_2 = 6 -> [0,0,0,4,0] (+1): 3 modMACs, D_new = [4, 0]
    R = oracle.reduce(csr_from_dense(rows + [[1, 2, 6, 0, 1]], 7))
    assert R.modmac == 3 and R.dnew.tolist() == [[4, 0]]
    # both targets together: counts add, rows independent
    R = oracle.reduce(csr_from_dense(rows + [[1, 1, 1, 1, 1], [1, 2, 6, 0, 1]], 7))
    assert R.modmac == 7 and R.dnew.tolist() == [[6, 0], [4, 0]] and R.rank == 1


def test_full_rref_of_M_against_textbook_gauss_jordan(c0_matrix, c0_oracle):
    """f2: the paper's route to RREF(M) in the original column order (B' = A^-1 B,
    B'' = B' - B'[:, pivcol] R, Step 5 re-arrangement) equals the textbook Gauss-Jordan RREF of M
    (unique) on the random suite, on matrices whose pivot rows are reduced by R, and on c0."""
    from pins import brute_rref
    cases = list(gbla_gen.random_suite(120, seed0=33))
    cases.append(c0_matrix)
    for M in cases:
        dense = np.zeros((M.m, M.n), np.int64)
        for i in range(M.m):
            s, e = int(M.row_ptr[i]), int(M.row_ptr[i + 1])
            dense[i, M.col[s:e].astype(np.int64)] = M.val[s:e]
        r, R, piv = brute_rref(dense, M.p)
        res = c0_oracle if M is c0_matrix else None
        rk, RM, pc = oracle.full_rref(M, res)
        assert rk == r, M.name
        assert np.array_equal(RM.astype(np.int64), R), M.name
        assert pc.tolist() == piv, M.name


def test_wide_field_oracle_pins(c0_matrix, c0_oracle):
    """f4 oracle (oracle/wide.py, p < 2^31): against the brute-force Gauss-Jordan of the whole M*sigma
    (the first n_piv columns are pivots, rank(M) = n_piv + rank(D_new), R = the bottom-right block)
    for p up to 2^31 - 1, and equal to the C oracle (D_new, modMACs, R) for p < 2^16."""
    from oracle import wide
    from pins import brute_rref
    for p in (3, 65521, 1048573, 8388593, 2147483647):
        for s in range(12):
            M = gbla_gen.random_wide(int(5 + 7 * s), int(8 + 9 * s), 0.15 + 0.02 * (s % 4), p, 1000 * s + p % 977)
            W = wide.reduce(M)
            dense = M.dense()
            perm = np.argsort(W.sigma)                              # column of sigma index k
            r, RR, piv = brute_rref(dense[:, perm], p)
            assert r == W.rank_M
            assert piv[:W.npiv] == list(range(W.npiv))
            assert np.array_equal(RR[W.npiv:, W.npiv:], W.R)
    # equal to the C oracle on 16-bit primes (c0 and a random suite)
    W = wide.reduce(gbla_gen.WideCSR(c0_matrix.m, c0_matrix.n, c0_matrix.p, c0_matrix.row_ptr,
                                     c0_matrix.col.astype(np.uint32), c0_matrix.val.astype(np.uint32)))
    assert W.modmac == c0_oracle.modmac and np.array_equal(W.dnew, c0_oracle.dnew)
    assert W.rank == c0_oracle.rank and np.array_equal(W.R, c0_oracle.R)
    for M in gbla_gen.random_suite(20, seed0=17):
        res = oracle.reduce(M)
        W = wide.reduce(gbla_gen.WideCSR(M.m, M.n, M.p, M.row_ptr, M.col.astype(np.uint32), M.val.astype(np.uint32)))
        assert W.modmac == res.modmac and np.array_equal(W.dnew, res.dnew) and np.array_equal(W.R, res.R)
