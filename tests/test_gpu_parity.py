"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Bar: bit-exact for everything (integer arithmetic mod p): maps, quadrants,
C', B', D_new, modMAC counts, rank, R and pivot columns.
Run on a B200 via gpurun: python -m pytest tests -m gpu -x -q
"""
import json
import os

import numpy as np
import pytest

import gbla_gen
import oracle
from conftest import csr_from_dense

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


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


def to_dev(M):
    import torch
    return (torch.from_numpy(M.row_ptr.astype(np.uint64)).cuda(), torch.from_numpy(M.col.astype(np.uint32)).cuda(),
            torch.from_numpy(M.val.astype(np.uint16)).cuda())


def np_(t):
    return t.cpu().numpy()


def gpu_reduce(gb, ctx, M, flags=0):
    rp, c, v = to_dev(M)
    h = gb.gbla_reduce(ctx, M.m, M.n, rp, c, v, M.p, flags=flags)
    return h


def check_full(gb, ctx, M, res=None, flags=0, check_dnew=True, keep=False):
    if res is None:
        res = oracle.reduce(M, want_x=True)
    S = res.splice
    rp, c, v = to_dev(M)
    h = gb.gbla_splice(ctx, M.m, M.n, rp, c, v, M.p)
    npiv, mN, nN = h.dims()
    assert (npiv, mN, nN) == (S.npiv, S.mN, S.nN)
    sig, prow, nprow = h.maps()
    assert np.array_equal(np_(sig), S.sigma) and np.array_equal(np_(prow), S.pivot_row)
    assert np.array_equal(np_(nprow), S.nonpivot_row)
    if flags & gb.GBLA_ORDER_STANDARD:
        gb.gbla_reduce_B(h)
        gb.gbla_update_D(h)
    else:
        gb.gbla_reduce_C(h, fused=True, int_pipe=bool(flags & gb.GBLA_SPARSE_INT))
    if check_dnew:
        assert np.array_equal(np_(h.D()), res.dnew), "D_new differs"
    if not (flags & gb.GBLA_ORDER_STANDARD):
        assert h.opcount()[0] == res.modmac
    r = gb.gbla_echelon_D(h, flags & (gb.GBLA_DENSE_INT | gb.GBLA_DENSE_TC))
    rank, pc, R = h.rref()
    assert r == rank == res.rank
    assert np.array_equal(np_(pc), res.pivcol)
    assert np.array_equal(np_(R), res.R)
    if keep:
        return h
    h.free()


def test_splice_quadrants_random_suite(gb, ctx):
    for M in gbla_gen.random_suite(80, seed0=21):
        S = oracle.splice(M)
        A, B, C, D = oracle.quadrants(M, S)
        rp, c, v = to_dev(M)
        h = gb.gbla_splice(ctx, M.m, M.n, rp, c, v, M.p)
        sig, prow, nprow = h.maps()
        assert np.array_equal(np_(sig), S.sigma)
        assert np.array_equal(np_(prow), S.pivot_row)
        assert np.array_equal(np_(nprow), S.nonpivot_row)
        for name, ref in (("A", A), ("B", B), ("C", C), ("D", D)):
            assert np.array_equal(np_(h.quadrant(name)).astype(np.uint32), ref), name
        h.free()


def test_multilines_match_oracle_definition(gb, ctx):
    """a2: the device two-row multilines of A|B equal the oracle's multiline
    (Definition, pinned by the paper's example P:524-556) of every
    pair of sigma-ordered pivot rows."""
    cases = list(gbla_gen.random_suite(30, seed0=31)) + [gbla_gen.f4_matrix("c0")]
    for M in cases:
        S = oracle.splice(M)
        A, B, C, D = oracle.quadrants(M, S)
        AB = np.hstack([A, B]).astype(np.uint32)
        rp, c, v = to_dev(M)
        h = gb.gbla_splice(ctx, M.m, M.n, rp, c, v, M.p)
        ptr, col, val = (np_(t) for t in h.multilines())
        assert ptr.size == (S.npiv + 1) // 2 + 1
        for k in range((S.npiv + 1) // 2):
            r1 = AB[2 * k]
            r2 = AB[2 * k + 1] if 2 * k + 1 < S.npiv else np.zeros_like(r1)
            pos, mv = oracle.multiline(r1, r2)
            q0, q1 = int(ptr[k]), int(ptr[k + 1])
            assert np.array_equal(col[q0:q1], pos), (k, col[q0:q1], pos)
            packed = mv[0::2].astype(np.uint64) | (mv[1::2].astype(np.uint64) << 16)
            assert np.array_equal(val[q0:q1].astype(np.uint64), packed), k
        h.free()


def test_multiline_column_runs(gb, ctx):
    """a2: the column runs of the device multilines (gbla_get_multiline_runs) decode to exactly the
    multiline columns, and are the maximal runs of the paper's run rule (the reference
    codec's encode_colids) cut only at the pair's diagonal-block end and its first N column."""
    from oracle import formats as fm
    cases = list(gbla_gen.random_suite(30, seed0=37)) + [gbla_gen.f4_matrix("c0")]
    cases.append(gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS["c3"], 0.02)))
    for M in cases:
        S = oracle.splice(M)
        rp, c, v = to_dev(M)
        h = gb.gbla_splice(ctx, M.m, M.n, rp, c, v, M.p)
        ptr, col, val = (np_(t) for t in h.multilines())
        rptr, rcol, rlen, rslot = (np_(t).astype(np.int64) for t in h.multiline_runs())
        for k in range((S.npiv + 1) // 2):
            q0, q1 = int(ptr[k]), int(ptr[k + 1])
            cols = col[q0:q1].astype(np.int64)
            runs = list(range(int(rptr[k]), int(rptr[k + 1])))
            dec = np.concatenate([np.arange(rcol[r], rcol[r] + rlen[r]) for r in runs]) if runs else np.zeros(0)
            assert np.array_equal(dec, cols), k
            assert all(np.array_equal(cols[rslot[r]:rslot[r] + rlen[r]], np.arange(rcol[r], rcol[r] + rlen[r]))
                       for r in runs), k
            # the run rule on the pieces between the cut points
            cuts = sorted({0, int(np.searchsorted(cols, min(2 * k + 2, S.npiv))), int(np.searchsorted(cols, S.npiv)),
                           cols.size})
            exp = []
            for a, b in zip(cuts[:-1], cuts[1:]):
                t = fm.encode_colids(cols[a:b])
                i = 0
                while i < len(t):
                    if t[i] & fm.MASK:
                        exp.append((t[i] & ~fm.MASK, 1)); i += 1
                    else:
                        exp.append((t[i], t[i + 1])); i += 2
            assert [(int(rcol[r]), int(rlen[r])) for r in runs] == exp, k
        h.free()


def test_pipeline_random_suite_new_order(gb, ctx):
    for M in gbla_gen.random_suite(150, seed0=23):
        check_full(gb, ctx, M)


def test_int_pipe_over_column_runs(gb, ctx, c0_matrix, c0_oracle, monkeypatch):
    """The INT-pipe engine walking the multilines' column runs (GBLA_INT_RUNS=1) gives the same
    D_new, op counts and R as the oracle (c0, a random suite, scaled c1)."""
    monkeypatch.setenv("GBLA_INT_RUNS", "1")
    check_full(gb, ctx, c0_matrix, c0_oracle, flags=gb.GBLA_SPARSE_INT)
    for M in list(gbla_gen.random_suite(30, seed0=41)) + [gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS["c1"], 0.03))]:
        check_full(gb, ctx, M, flags=gb.GBLA_SPARSE_INT)
    monkeypatch.delenv("GBLA_INT_RUNS")


def test_pipeline_random_suite_int_pipe(gb, ctx):
    for M in gbla_gen.random_suite(80, seed0=29):
        check_full(gb, ctx, M, flags=gb.GBLA_SPARSE_INT | gb.GBLA_DENSE_INT)


def test_pipeline_random_suite_standard_order(gb, ctx):
    for M in gbla_gen.random_suite(60, seed0=25):
        check_full(gb, ctx, M, flags=gb.GBLA_ORDER_STANDARD)


def test_unfused_cprime_bprime(gb, ctx, monkeypatch):
    for M in list(gbla_gen.random_suite(40, seed0=27)) + [gbla_gen.f4_matrix("c0"),
                                                          gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS["c1"], 0.03))]:
        S = oracle.splice(M)
        A, B, C, D = oracle.quadrants(M, S)
        dn, x, ops = oracle.dnew_rows(M, S, want_x=True)
        rp, c, v = to_dev(M)
        h = gb.gbla_splice(ctx, M.m, M.n, rp, c, v, M.p)
        gb.gbla_reduce_C(h, fused=False)
        assert np.array_equal(np_(h.cprime()), x)
        gb.gbla_update_D(h)
        assert np.array_equal(np_(h.D()), dn)
        assert h.opcount()[0] == int(ops.sum())
        h.free()
        bp = oracle.trsm(A, B, M.p)
        # TRSM on the tensor cores (default) and on the INT pipe (K8); D -= C B' by the sparse rows of
        # C (INT pipe) and by K11 on the densified C
        for trsm_int, upd in (("0", "tc"), ("1", "int"), ("0", "int"), ("0", None)):
            monkeypatch.setenv("GBLA_TRSM_INT", trsm_int)
            if upd:
                monkeypatch.setenv("GBLA_UPDATE_BP", upd)
            h = gb.gbla_splice(ctx, M.m, M.n, rp, c, v, M.p)
            gb.gbla_reduce_B(h)
            assert np.array_equal(np_(h.bprime()).astype(np.uint32), bp)
            gb.gbla_update_D(h)
            assert np.array_equal(np_(h.D()), dn)
            h.free()
            monkeypatch.delenv("GBLA_UPDATE_BP", raising=False)
        monkeypatch.delenv("GBLA_TRSM_INT")
        for ip in (False, True):
            h = gb.gbla_splice(ctx, M.m, M.n, rp, c, v, M.p)
            gb.gbla_reduce_C(h, fused=True, keep_cprime=True, int_pipe=ip)
            assert np.array_equal(np_(h.cprime()), x)
            assert np.array_equal(np_(h.D()), dn)
            assert h.opcount()[0] == int(ops.sum())
            h.free()
            h = gb.gbla_splice(ctx, M.m, M.n, rp, c, v, M.p)
            gb.gbla_reduce_C(h, fused=False, int_pipe=ip)
            assert np.array_equal(np_(h.cprime()), x)
            gb.gbla_update_D(h)
            assert np.array_equal(np_(h.D()), dn)
            h.free()


def test_c0_full(gb, ctx, c0_matrix, c0_oracle):
    check_full(gb, ctx, c0_matrix, c0_oracle)
    check_full(gb, ctx, c0_matrix, c0_oracle, flags=gb.GBLA_ORDER_STANDARD)
    check_full(gb, ctx, c0_matrix, c0_oracle, flags=gb.GBLA_DENSE_INT)
    check_full(gb, ctx, c0_matrix, c0_oracle, flags=gb.GBLA_SPARSE_INT)


def test_scaled_configs_tc_vs_int(gb, ctx):
    """The tensor-core block path and the INT-pipe AXPY path on every config
    shape at reduced scale (several 128-blocks, ragged tails): D_new, counts,
    R against the oracle."""
    for name, sc in (("c1", 0.05), ("c2", 0.02), ("c3", 0.03), ("c4", 0.004)):
        cfg = gbla_gen.scaled(gbla_gen.CONFIGS[name], sc)
        M = gbla_gen.f4_matrix(cfg)
        res = oracle.reduce(M)
        check_full(gb, ctx, M, res)
        check_full(gb, ctx, M, res, flags=gb.GBLA_SPARSE_INT | gb.GBLA_DENSE_INT)


def test_xt_batches(gb, ctx, monkeypatch):
    """The sparse phase in batches of target tiles (how c4 fits in HBM): forcing
    2-tile batches must not change D_new, the op count or R."""
    monkeypatch.setenv("GBLA_XT_BATCH", "2")
    for name, sc in (("c1", 0.05), ("c3", 0.03), ("c4", 0.004)):
        M = gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS[name], sc))
        check_full(gb, ctx, M, oracle.reduce(M))
    monkeypatch.setenv("GBLA_DIST_EMULATE", "3")
    M = gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS["c1"], 0.05))
    res = oracle.reduce(M)
    h = gpu_reduce(gb, ctx, M)
    r, pc, R = h.rref()
    assert r == res.rank and np.array_equal(np_(pc), res.pivcol) and np.array_equal(np_(R), res.R)
    assert h.opcount()[0] == res.modmac
    h.free()


def test_long_accumulations_are_chunked(gb, ctx):
    """Unbanded A|B with more than 128 blocks of 128 pivots: a target's block sweep and the D update
    accumulate more than 128 tile pairs, which must be split into exact s32 chunks (K <= 16,384).
    Sampled D_new rows (leftmost leads: the longest lists) against the oracle's Alg 2."""
    import torch
    cfg = gbla_gen.scaled(gbla_gen.CONFIGS["c3"], 0.42)
    M = gbla_gen.f4_matrix(cfg)
    S = oracle.splice(M)
    assert (S.npiv + 127) // 128 > 129
    rp, c, v = to_dev(M)
    h = gb.gbla_splice(ctx, M.m, M.n, rp, c, v, M.p)
    gb.gbla_reduce_C(h, fused=True)
    D = h.D()
    ld = S.lead[S.nonpivot_row]
    lead_sig = np.where(ld < M.n, S.sigma[np.minimum(ld, M.n - 1)], M.n)
    t = np.sort(np.argsort(lead_sig, kind="stable")[:8])
    dn, _, _ = oracle.dnew_rows(M, S, targets=t)
    got = D.view(torch.int16)[torch.from_numpy(t).cuda().long()].cpu().numpy().view(np.uint16)
    assert np.array_equal(got, dn)
    h.free()


def test_window_step_with_lead_scan(gb, ctx, c0_matrix, c0_oracle, monkeypatch):
    """GBLA_WIN_LEAD=1: the fused window step also computes the next window's leading columns after a
    grid barrier (instead of k_lead2)."""
    monkeypatch.setenv("GBLA_WIN_LEAD", "1")
    check_full(gb, ctx, c0_matrix, c0_oracle)
    M = gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS["c1"], 0.05))
    check_full(gb, ctx, M, oracle.reduce(M))


def test_gather_after_the_whole_panel(gb, ctx, c0_matrix, c0_oracle, monkeypatch):
    """GBLA_EARLY_GATHER=0: the next step's F gather waits for the whole panel (the default waits on
    the panel's flag, set before its T solve)."""
    monkeypatch.setenv("GBLA_EARLY_GATHER", "0")
    check_full(gb, ctx, c0_matrix, c0_oracle)
    M = gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS["c1"], 0.05))
    check_full(gb, ctx, M, oracle.reduce(M))


def test_window_step_in_two_launches(gb, ctx, c0_matrix, c0_oracle, monkeypatch):
    """GBLA_WIN_FUSED=0: the Rn window and the window update as two launches (the default fuses
    them into one persistent kernel with column-tile flags); both must give the oracle's R."""
    monkeypatch.setenv("GBLA_WIN_FUSED", "0")
    check_full(gb, ctx, c0_matrix, c0_oracle)
    M = gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS["c1"], 0.05))
    check_full(gb, ctx, M, oracle.reduce(M))


def test_echelon_without_lookahead(gb, ctx, c0_matrix, c0_oracle, monkeypatch):
    """The echelon's look-ahead (next panel on a side stream beside the rest of
    the trailing update) and the serial schedule give the same R."""
    monkeypatch.setenv("GBLA_NO_LOOKAHEAD", "1")
    check_full(gb, ctx, c0_matrix, c0_oracle)
    M = gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS["c3"], 0.03))
    check_full(gb, ctx, M, oracle.reduce(M))


def test_host_input_and_host_copy(gb, ctx, c0_matrix, c0_oracle):
    M = c0_matrix
    h = gb.gbla_reduce(ctx, M.m, M.n, M.row_ptr, M.col, M.val, M.p)     # numpy => GBLA_HOST_INPUT
    r, pc, R = h.rref_to_host()
    assert r == c0_oracle.rank and np.array_equal(pc, c0_oracle.pivcol) and np.array_equal(R, c0_oracle.R)
    h.free()


def test_c1_full_size_against_golden(gb, ctx):
    """c1 (bench workload) at full size: counts and digests written by the
    oracle (tests/golden/make_golden.py), plus sampled D_new rows computed by
    the oracle one by one."""
    g = json.load(open(os.path.join(GOLD, "c1_oracle.json")))
    M = gbla_gen.f4_matrix("c1")
    h = gpu_reduce(gb, ctx, M)
    npiv, mN, nN = h.dims()
    assert (npiv, mN, nN) == (g["npiv"], g["mN"], g["nN"])
    assert h.opcount()[0] == g["modmac_sparse"]
    r, pc, R = h.rref()
    assert r == g["rank_D"]
    assert oracle.rref_digest(r, nN, np_(pc), np_(R)) == g["rref_sha256"]
    h.free()
    # D_new: digest + sampled rows by the oracle
    rp, c, v = to_dev(M)
    h = gb.gbla_splice(ctx, M.m, M.n, rp, c, v, M.p)
    gb.gbla_reduce_C(h, fused=True)
    D = np_(h.D())
    assert oracle.array_digest(D) == g["dnew_sha256"]
    S = oracle.splice(M)
    rng = np.random.default_rng(5)
    t = np.sort(rng.choice(S.mN, 24, replace=False))
    dn, _, ops = oracle.dnew_rows(M, S, targets=t)
    assert np.array_equal(D[t], dn)
    h.free()


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_standard_order_full_size_against_golden(gb, ctx, name):
    """The standard order (Step 2 TRSM on the tensor cores, Step 3 D - C B' by K11) at
    full size: its D_new is the new order's (the oracle's golden digest), hundreds of tiles wide."""
    g = json.load(open(os.path.join(GOLD, name + "_oracle.json")))
    M = gbla_gen.f4_matrix(name)
    rp, c, v = to_dev(M)
    h = gb.gbla_splice(ctx, M.m, M.n, rp, c, v, M.p)
    gb.gbla_reduce_B(h)
    gb.gbla_update_D(h)
    assert oracle.array_digest(np_(h.D())) == g["dnew_sha256"]
    h.free()


def test_c3_full_size_against_golden(gb, ctx):
    """c3 (dense-D-heavy, 60,000 x 80,000, p = 32003) at full size through the default path (super-
    panels of 4: deferred K = 512 flushes on CTA pairs, lead-sorted rows, prefix slots, back
    elimination): the modMAC count, the R digest and the D_new digest written by the oracle
    (tests/golden/make_golden.py c3: 2.2 h on 8 cores), bit-exact."""
    g = json.load(open(os.path.join(GOLD, "c3_oracle.json")))
    M = gbla_gen.f4_matrix("c3")
    h = gpu_reduce(gb, ctx, M)
    npiv, mN, nN = h.dims()
    assert (npiv, mN, nN) == (g["npiv"], g["mN"], g["nN"])
    assert h.opcount()[0] == g["modmac_sparse"]
    r, pc, R = h.rref()
    assert r == g["rank_D"]
    assert oracle.rref_digest(r, nN, np_(pc), np_(R)) == g["rref_sha256"]
    h.free()
    rp, c, v = to_dev(M)
    h = gb.gbla_splice(ctx, M.m, M.n, rp, c, v, M.p)
    gb.gbla_reduce_C(h, fused=True)
    assert oracle.array_digest(np_(h.D())) == g["dnew_sha256"]
    h.free()


def test_edge_cases(gb, ctx):
    cases = [
        np.eye(6, dtype=np.int64),                        # A = I, no C|D
        np.zeros((4, 5), dtype=np.int64),                 # all zero rows, npiv = 0
        np.array([[0, 0, 3, 1], [0, 0, 0, 0], [0, 0, 6, 2]]),   # zero row + dependent
        np.array([[1, 2], [1, 3]]),                       # SPEC tie example
        np.array([[5]]),                                  # 1x1
        np.ones((7, 3), dtype=np.int64),                  # wide dependence
        np.triu(np.ones((9, 9), dtype=np.int64)),         # dense upper triangular
    ]
    for a in cases:
        for p in (3, 7, 65521):
            M = csr_from_dense(a, p)
            check_full(gb, ctx, M)
    # odd / even pivot counts with the multiline pairing, dense D
    rng = np.random.default_rng(3)
    for npiv in (1, 2, 3, 63, 64, 65, 129):
        n, m = npiv + 70, npiv + 90
        a = np.zeros((m, n), dtype=np.int64)
        a[:npiv, :npiv] = np.triu(rng.integers(0, 65521, (npiv, npiv)))
        np.fill_diagonal(a[:npiv, :npiv], 1)
        a[:npiv, npiv:] = rng.integers(0, 65521, (npiv, 70))
        a[npiv:, :] = rng.integers(0, 65521, (90, n))
        check_full(gb, ctx, csr_from_dense(a, 65521))


def test_errors(gb, ctx):
    M = csr_from_dense([[1, 2], [0, 3]], 7)
    rp, c, v = to_dev(M)
    with pytest.raises(gb.GblaError) as e:
        gb.gbla_splice(ctx, M.m, M.n, rp, c, v, 8)
    assert e.value.status == 2
    import torch
    bad_c = torch.flip(c, [0]).contiguous()
    with pytest.raises(gb.GblaError) as e:
        gb.gbla_splice(ctx, M.m, M.n, rp, bad_c, v, 7)
    assert e.value.status == 1
    bad_v = v.clone(); bad_v[0] = 7
    with pytest.raises(gb.GblaError) as e:
        gb.gbla_splice(ctx, M.m, M.n, rp, c, bad_v, 7)
    assert e.value.status == 1
    h = gb.gbla_splice(ctx, M.m, M.n, rp, c, v, 7)
    with pytest.raises(gb.GblaError) as e:
        gb.gbla_update_D(h)                        # nothing to update with
    assert e.value.status == 3
    gb.gbla_reduce_B(h)
    gb.gbla_reduce_C(h, fused=False)
    with pytest.raises(gb.GblaError) as e:
        gb.gbla_update_D(h)                        # both: would apply A^-1 twice
    assert e.value.status == 3
    h.free()


def test_modgemm_tc_and_int_against_numpy(gb, ctx):
    """K11 alone: exact C - A*B mod p for ragged shapes (several tiles and a
    ragged tail), both engines, with and without a row-index gather."""
    import torch
    from pins import matmul_mod
    rng = np.random.default_rng(8)
    shapes = [(1, 1, 1), (5, 7, 3), (128, 64, 128), (129, 65, 127), (300, 200, 128), (1000, 333, 77), (77, 1030, 128),
              (130, 70, 129), (257, 300, 384), (200, 129, 512), (1, 64, 500)]
    for p in (3, 251, 32003, 65521):
        for rows, cols, K in shapes:
            A = rng.integers(0, p, (rows, K)); B = rng.integers(0, p, (K, cols))
            C0 = rng.integers(0, p, (rows + 3, cols))
            perm = rng.permutation(rows + 3)[:rows].astype(np.uint32)
            exp = C0.copy()
            exp[perm] = (C0[perm] - matmul_mod(A, B, p)) % p
            for engine in (0, 1):
                tA = torch.from_numpy(A.astype(np.uint16)).cuda()
                tB = torch.from_numpy(B.astype(np.uint16)).cuda()
                tC = torch.from_numpy(C0.astype(np.uint16)).cuda()
                gb.gbla_modgemm(ctx, p, tA, tB, tC, rowidx=torch.from_numpy(perm).cuda(), engine=engine)
                assert np.array_equal(tC.cpu().numpy().astype(np.int64), exp), (p, rows, cols, K, engine)
    # worst case for the s32 limb accumulators: all entries p - 1, K = 128 and K = 512 (multi-K)
    p = 65521
    for K in (128, 512):
        A = np.full((128, K), p - 1); B = np.full((K, 64), p - 1); C0 = np.zeros((128, 64), np.int64)
        tC = torch.from_numpy(C0.astype(np.uint16)).cuda()
        gb.gbla_modgemm(ctx, p, torch.from_numpy(A.astype(np.uint16)).cuda(),
                        torch.from_numpy(B.astype(np.uint16)).cuda(), tC)
        assert np.array_equal(tC.cpu().numpy().astype(np.int64), (C0 - matmul_mod(A, B, p)) % p), K


def test_echelon_engines_agree_c0_and_dense(gb, ctx, c0_matrix, c0_oracle):
    check_full(gb, ctx, c0_matrix, c0_oracle, flags=gb.GBLA_DENSE_TC)
    check_full(gb, ctx, c0_matrix, c0_oracle, flags=gb.GBLA_DENSE_INT)
    # dense random D with rank deficiency (dense-D-heavy shape, like c3)
    rng = np.random.default_rng(4)
    for p in (32003, 65521):
        base = rng.integers(0, p, (150, 400))
        comb = rng.integers(0, p, (100, 150))
        from pins import matmul_mod
        dep = matmul_mod(comb, base, p)
        a = np.vstack([base, dep])[rng.permutation(250)]
        M = csr_from_dense(np.hstack([np.zeros((250, 0), np.int64), a]), p)
        res = oracle.reduce(M)
        assert res.rank_M == 150
        for f in (gb.GBLA_DENSE_TC, gb.GBLA_DENSE_INT):
            check_full(gb, ctx, M, res, flags=f)


def check_ref(gb, h, res, p):
    """GBLA_ECHELON_REF output against the oracle: same rank and pivot columns, leading 1s, zeros
    left of every pivot and below it, and RREF(R_ref) (computed by the oracle) = the oracle's R."""
    r, pc, R = h.rref()
    R, pc = np_(R), np_(pc)
    assert r == res.rank and np.array_equal(pc, res.pivcol)
    if r:
        rows = np.arange(r)
        assert np.all(R[rows, pc] == 1)
        cols = np.arange(R.shape[1])
        assert not np.any(R[cols[None, :] < pc[:, None]])              # zero left of the pivot
        below = R[:, pc]                                                  # column pc[i] of row j
        assert not np.any(np.tril(below, -1))                             # zero below every pivot
    r2, R2, pc2 = oracle.rref(R, p)
    assert r2 == res.rank and np.array_equal(pc2, res.pivcol) and np.array_equal(R2, res.R)
    return R


def test_echelon_ref_mode(gb, ctx, c0_matrix, c0_oracle, monkeypatch):
    """the row echelon form without back elimination (GBLA_ECHELON_REF), on both
    trailing-update engines, with look-ahead and super-panels, and with emulated ranks.  On a
    multi-panel D it must really skip the back elimination (R_ref != R somewhere)."""
    cases = [(c0_matrix, c0_oracle)]
    for name, sc in (("c1", 0.05), ("c3", 0.03)):
        M = gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS[name], sc))
        cases.append((M, oracle.reduce(M)))
    for i, (M, res) in enumerate(cases):
        for f in (gb.GBLA_DENSE_TC, gb.GBLA_DENSE_INT):
            h = gpu_reduce(gb, ctx, M, flags=f | gb.GBLA_ECHELON_REF)
            R = check_ref(gb, h, res, M.p)
            if i == 1:
                assert not np.array_equal(R, res.R), "REF mode did a full reduction"
            h.free()
    M, res = cases[2]
    monkeypatch.setenv("GBLA_SP", "4")                                    # deferred updates
    h = gpu_reduce(gb, ctx, M, flags=gb.GBLA_ECHELON_REF)
    check_ref(gb, h, res, M.p)
    h.free()
    monkeypatch.delenv("GBLA_SP")
    monkeypatch.setenv("GBLA_DIST_EMULATE", "3")
    for mode in ("panels", "replicated"):
        monkeypatch.setenv("GBLA_DIST_ECHELON", mode)
        h = gpu_reduce(gb, ctx, M, flags=gb.GBLA_ECHELON_REF)
        check_ref(gb, h, res, M.p)
        h.free()
    monkeypatch.delenv("GBLA_DIST_ECHELON")
    monkeypatch.delenv("GBLA_DIST_EMULATE")


def _csr_dense(rp, col, val, rows, n):
    import torch
    rp = rp.view(torch.int64).cpu().numpy(); col = col.view(torch.int32).cpu().numpy().astype(np.int64)
    val = val.view(torch.int16).cpu().numpy().view(np.uint16)
    out = np.zeros((rows, n), np.uint16)
    for i in range(rows):
        s, e = rp[i], rp[i + 1]
        c = col[s:e]
        assert np.all(np.diff(c) > 0), "columns not ascending"
        out[i, c] = val[s:e]
    return out


def test_full_rref_of_M(gb, ctx, c0_matrix, c0_oracle):
    """SURVEY 8(f) f2 (gbla_rref_M): RREF of the whole M in the original column order (B' = A^-1 B
    by the tensor-core sparse phase on the targets e_k, B'' = B' - B'[:, pivcol] R by K11, Step 5
    re-arrangement) bit-exact against the oracle's route (itself pinned against textbook
    Gauss-Jordan of M) on c0, a random suite (p in {3, 251, 32003, 65521}, zero rows, all-pivot and
    no-pivot cases) and scaled c1 / c3 (several 128-pivot blocks, K = rank > 512 in chunks)."""
    cases = [(c0_matrix, c0_oracle)]
    cases += [(M, None) for M in gbla_gen.random_suite(40, seed0=71)]
    for name, sc in (("c1", 0.05), ("c3", 0.05)):
        cases.append((gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS[name], sc)), None))
    cases.append((csr_from_dense(np.eye(7, dtype=np.int64) * 3, 7), None))          # all pivots, no D
    cases.append((csr_from_dense(np.zeros((4, 5), np.int64), 7), None))              # no pivots
    for M, res in cases:
        if res is None:
            res = oracle.reduce(M)
        rk, RM, pc = oracle.full_rref(M, res)
        h = gpu_reduce(gb, ctx, M)
        r, rp, col, val = h.rref_M()
        assert r == rk == res.rank_M, M.name
        got = _csr_dense(rp, col, val, r, M.n)
        assert np.array_equal(got, RM), M.name
        h.free()
    # call order: before the echelon, and after a row-echelon-only echelon
    rp_, c_, v_ = to_dev(c0_matrix)
    h = gb.gbla_splice(ctx, c0_matrix.m, c0_matrix.n, rp_, c_, v_, c0_matrix.p)
    with pytest.raises(gb.GblaError) as e:
        h.rref_M()
    assert e.value.status == 3
    h.free()
    h = gpu_reduce(gb, ctx, c0_matrix, flags=gb.GBLA_ECHELON_REF)
    with pytest.raises(gb.GblaError) as e:
        h.rref_M()
    assert e.value.status == 3
    h.free()


def test_one_rank_nccl_communicator(gb, monkeypatch):
    """The real multi-GPU code path on one GPU (a one-rank NCCL communicator, gbla_ctx_set_comm with
    world 1): C1 broadcast of M, the row-sharded sparse phase with the op-count all-reduce, then
    either echelon mode: "replicated" (C7: pack, grouped in-place all-gathers of the slot-ordered
    D_new rounds, unpack; then the single-GPU echelon) or "panels" (the distributed echelon:
    lead-count all-reduce, candidate all-gather, pivot-row all-reduce, R by broadcasts) -- every
    ncclBroadcast / ncclAllGather / ncclAllReduce call site runs with its real buffers, counts and
    types.  R, rank and op counts against the oracle; REF mode too; then detach and reduce again
    on the single-GPU path."""
    ctx1 = gb.Context(0)
    ctx1.set_comm(gb.nccl_unique_id(), 0, 1)
    cases = [gbla_gen.f4_matrix("c0")]
    for name, sc in (("c1", 0.05), ("c3", 0.03), ("c2", 0.02)):
        cases.append(gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS[name], sc)))
    for mode in ("replicated", "panels"):
        monkeypatch.setenv("GBLA_DIST_ECHELON", mode)
        for M in cases:
            res = oracle.reduce(M)
            h = gpu_reduce(gb, ctx1, M)
            r, pc, R = h.rref()
            assert r == res.rank and np.array_equal(np_(pc), res.pivcol) and np.array_equal(np_(R), res.R), \
                (mode, M.name)
            assert h.opcount()[0] == res.modmac
            h.free()
        h = gpu_reduce(gb, ctx1, cases[1], flags=gb.GBLA_ECHELON_REF)
        check_ref(gb, h, oracle.reduce(cases[1]), cases[1].p)
        h.free()
    monkeypatch.delenv("GBLA_DIST_ECHELON")
    # the INT-pipe echelon is single-GPU: with a communicator gbla_reduce keeps D whole on every rank
    h = gpu_reduce(gb, ctx1, cases[0], flags=gb.GBLA_DENSE_INT)
    r, pc, R = h.rref()
    res0 = oracle.reduce(cases[0])
    assert r == res0.rank and np.array_equal(np_(R), res0.R)
    h.free()
    ctx1.set_comm(None, 0, 1)
    check_full(gb, ctx1, cases[0], oracle.reduce(cases[0], want_x=True))
    ctx1.close()


def test_super_panels_rref_exact(gb, ctx, monkeypatch):
    """The default echelon schedule of c2-c4 (GBLA_SP = 4 panels per super-panel: per-panel updates
    left of the deferred columns, one K = 512 multi-K flush per super-panel over the rows whose
    leading column is left of the super-panel's end, per-panel fix-ups of the selected rows, the
    back elimination into earlier pivot rows), in full RREF mode and with look-ahead, bit-exact
    against the oracle's R at scaled c2, c3 and c4 with several super-panels; also
    2 panels per super-panel and a partial last super-panel."""
    monkeypatch.setenv("GBLA_BACKSUB", "0")         # the Gauss-Jordan back elimination in the panels
    for name, sc in (("c2", 0.05), ("c3", 0.1), ("c4", 0.012)):
        M = gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS[name], sc))
        res = oracle.reduce(M)
        assert res.rank > 2 * 4 * 128, (name, res.rank)             # several super-panels of 4 panels
        for sp in ("4", "2", "3"):
            monkeypatch.setenv("GBLA_SP", sp)
            check_full(gb, ctx, M, res, check_dnew=(sp == "4"))
    monkeypatch.delenv("GBLA_SP")


def test_sharded_sparse_phase_emulated_ranks(gb, ctx, c0_matrix, c0_oracle, monkeypatch):
    """Multi-GPU row sharding (dist.cu), with G ranks emulated on one GPU
    (GBLA_DIST_EMULATE): each shard sweeps only its cyclic target tiles, the
    packed D_new blocks are all-gathered (device copies instead of NCCL) and
    the echelon runs on the gathered D.  R, rank and op count must not depend
    on G."""
    cases = [(c0_matrix, c0_oracle)]
    for name, sc in (("c1", 0.05), ("c3", 0.03)):
        M = gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS[name], sc))
        cases.append((M, oracle.reduce(M)))
    for M, res in cases:
        for G in (2, 3, 8):
            for mode in ("panels", "replicated"):
                monkeypatch.setenv("GBLA_DIST_EMULATE", str(G))
                monkeypatch.setenv("GBLA_DIST_ECHELON", mode)
                h = gpu_reduce(gb, ctx, M)
                r, pc, R = h.rref()
                assert r == res.rank and np.array_equal(np_(pc), res.pivcol) and np.array_equal(np_(R), res.R)
                assert h.opcount()[0] == res.modmac
                h.free()
    monkeypatch.delenv("GBLA_DIST_EMULATE")
    monkeypatch.delenv("GBLA_DIST_ECHELON")


def test_backsub_rref_exact(gb, ctx, c0_matrix, c0_oracle, monkeypatch):
    """K14: the RREF through a row echelon form and one triangular solve RREF = U_sq^-1 U (the K5'
    sweep on the reversed, transposed pivot block; R13), forced on every config shape at
    reduced scale (several 128-pivot blocks, long accumulations folded every 128 tile pairs on the
    unbanded triangle), with forced 1- and 3-tile batches of target tiles, and on c0: R, rank and
    pivot columns bit-exact against the oracle; the Gauss-Jordan path (GBLA_BACKSUB=0) agrees."""
    monkeypatch.setenv("GBLA_BACKSUB", "1")
    check_full(gb, ctx, c0_matrix, c0_oracle)
    for name, sc in (("c1", 0.05), ("c2", 0.03), ("c3", 0.06), ("c4", 0.01)):
        M = gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS[name], sc))
        res = oracle.reduce(M)
        h = check_full(gb, ctx, M, res, check_dnew=False, keep=True)
        assert h.kernel_work()["backsub"] > 0, name          # the solve ran (non-pivot columns exist)
        h.free()
        if name in ("c1", "c3"):
            for b in ("1", "3"):
                monkeypatch.setenv("GBLA_XT_BATCH", b)
                check_full(gb, ctx, M, res, check_dnew=False)
            monkeypatch.delenv("GBLA_XT_BATCH")
    monkeypatch.setenv("GBLA_BACKSUB", "0")
    check_full(gb, ctx, c0_matrix, c0_oracle)


def test_backsub_prefix_scans(gb, ctx, c0_matrix, c0_oracle, monkeypatch):
    """Row echelon panels walking only the rows whose initial lead is left of the window / panel end
    (the default for mN >= 65,536, forced here with GBLA_REF_PREFIX at reduced scale): R, rank and
    pivot columns bit-exact against the oracle on c0 and scaled c1/c2/c4 shapes."""
    monkeypatch.setenv("GBLA_BACKSUB", "1")
    monkeypatch.setenv("GBLA_REF_PREFIX", "1")
    check_full(gb, ctx, c0_matrix, c0_oracle)
    for name, sc in (("c1", 0.05), ("c2", 0.03), ("c4", 0.01)):
        M = gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS[name], sc))
        check_full(gb, ctx, M, oracle.reduce(M), check_dnew=False)


def test_backsub_edge_cases(gb, ctx, monkeypatch):
    """K14 on the degenerate shapes: rank 0 and 1 (nothing above a pivot), a full-rank square D (no
    non-pivot column: only the pivot columns are cleared), a single non-pivot column, dense random
    D over small and large p, all bit-exact against the oracle."""
    monkeypatch.setenv("GBLA_BACKSUB", "1")
    from pins import matmul_mod
    rng = np.random.default_rng(11)
    npiv = 130
    for p in (3, 251, 65521):
        for (mn, nn, rk) in ((5, 7, 0), (6, 9, 1), (40, 40, 40), (40, 41, 40), (150, 260, 137), (300, 300, 150)):
            a = np.zeros((npiv + mn, npiv + nn), dtype=np.int64)
            a[:npiv, :npiv] = np.triu(rng.integers(0, p, (npiv, npiv)))
            np.fill_diagonal(a[:npiv, :npiv], 1)
            a[:npiv, npiv:] = rng.integers(0, p, (npiv, nn))
            base = rng.integers(0, p, (max(rk, 1), npiv + nn))
            comb = rng.integers(0, p, (mn, max(rk, 1))) if rk else np.zeros((mn, 1), np.int64)
            a[npiv:, :] = matmul_mod(comb, base, p)
            M = csr_from_dense(a, p)
            res = oracle.reduce(M)
            if p > 3:
                assert res.rank == rk, (p, mn, nn, rk, res.rank)
            check_full(gb, ctx, M, res)


def test_backsub_choice(gb, ctx, monkeypatch):
    """Default choice of the echelon route (echelon.cu use_bsub): a staircase D_new (rows leading in
    distinct columns: the c1/c2/c4 shapes) takes the row echelon form + back substitution, a dense
    D_new (rows leading in the same few columns: c3) the Gauss-Jordan panels."""
    monkeypatch.delenv("GBLA_BACKSUB", raising=False)
    for name, sc, want in (("c2", 0.03, True), ("c3", 0.06, False)):
        M = gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS[name], sc))
        res = oracle.reduce(M)
        h = check_full(gb, ctx, M, res, check_dnew=False, keep=True)
        assert (h.kernel_work()["backsub"] > 0) == want, name
        h.free()
