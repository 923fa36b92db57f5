"""Full-size parity on BASELINE.json's larger configs (c2, c3, c4), in the launch
configuration bench.py uses (gbla_splice -> fused gbla_reduce_C -> gbla_echelon_D,
default engines).  The oracle cannot reduce these whole in test time, so:

* D_new: sampled target rows, each computed one by one by the oracle (Alg 2,
  oracle.dnew_rows) and compared bit for bit (leftmost leads, which reduce
  through the most pivots, plus uniform samples);
* R: the structure of a reduced row echelon form (pivot columns strictly
  increasing, identity in the pivot columns, zeros left of each pivot) on
  sampled rows / columns, and rank(D) = the planted rank (SURVEY.md §8(c)
  "Planted rank");
* rowspace(D_new) within rowspace(R): for random y, v = y^T D_new must equal
  sum_k v[pivcol_k] R_k (false accept <= 1/p per trial).  Both products are
  computed by cuBLAS in float64, exact here (every partial sum < 2^53), so no
  libgbla kernel checks itself.
Unpinned at these sizes: rowspace(R) within rowspace(D_new)
beyond the rank equality, and D_new rows outside the sample.
"""
import numpy as np
import pytest

import gbla_gen
import oracle

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


def _i32(t):
    """uint16 CUDA tensor -> int32 values (torch has few uint16 CUDA kernels)."""
    import torch
    return t.view(torch.int16).to(torch.int32) & 0xFFFF


def _rowspace_check(Dh, pc, R, p, trials=2, seed=0):
    """Dh: D_new on the host (numpy u16), streamed to the GPU in row blocks."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    mN, nN = Dh.shape
    for _ in range(trials):
        y = torch.randint(0, p, (mN,), generator=g, device="cuda", dtype=torch.int64).double()
        v = torch.zeros(nN, dtype=torch.float64, device="cuda")
        for r0 in range(0, mN, 4096):                      # sums < mN * p^2 < 2^53
            blk = torch.from_numpy(Dh[r0:r0 + 4096].view(np.int16)).cuda()
            v += y[r0:r0 + 4096] @ (blk.to(torch.int32) & 0xFFFF).double()
        v = torch.remainder(v, p)
        coef = v[pc.view(torch.int32).long()]
        w = torch.zeros(nN, dtype=torch.float64, device="cuda")
        for r0 in range(0, R.shape[0], 4096):
            w += coef[r0:r0 + 4096] @ _i32(R[r0:r0 + 4096]).double()
        w = torch.remainder(w, p)
        assert torch.equal(v, w), "a random combination of D_new rows is not in the row space of R"


def _rref_structure(pc, R, rng):
    import torch
    rank = pc.numel()
    pcl = pc.view(torch.int32).long()
    assert bool((pcl[1:] > pcl[:-1]).all()), "pivot columns not strictly increasing"
    cols = torch.from_numpy(rng.choice(rank, min(rank, 512), replace=False)).cuda()
    Ri = R.view(torch.int16)
    sub = (Ri[:, pcl[cols]].to(torch.int32) & 0xFFFF).long()   # rank x 512: identity columns
    exp = torch.zeros_like(sub)
    exp[cols, torch.arange(cols.numel(), device="cuda")] = 1
    assert torch.equal(sub, exp), "R is not the identity in its pivot columns"
    for k in rng.choice(rank, min(rank, 256), replace=False):
        c = int(pcl[k])
        assert int(Ri[k, c]) == 1 and not bool((Ri[k, :c] != 0).any()), f"row {k} not zero left of its pivot"


@pytest.mark.parametrize("name", ["c3", "c2", "c4"])
def test_full_size_sampled(gb, ctx, name):
    import torch
    cfg = gbla_gen.CONFIGS[name]
    M = gbla_gen.f4_matrix(cfg)
    S = oracle.splice(M)
    rp = torch.from_numpy(M.row_ptr).cuda()
    col = torch.from_numpy(M.col).cuda()
    val = torch.from_numpy(M.val).cuda()
    h = gb.gbla_splice(ctx, M.m, M.n, rp, col, val, M.p)
    npiv, mN, nN = h.dims()
    assert (npiv, mN, nN) == (S.npiv, S.mN, S.nN) == (cfg.npiv, cfg.m - cfg.npiv, cfg.n - cfg.npiv)
    sig, prow, nprow = h.maps()
    assert np.array_equal(sig.cpu().numpy(), S.sigma) and np.array_equal(prow.cpu().numpy(), S.pivot_row)
    gb.gbla_reduce_C(h, fused=True)
    Dv = h.D(clone=False)                                  # D_new (library buffer), copied to the host
    Dh = np.empty(tuple(Dv.shape), np.uint16)
    for r0 in range(0, Dv.shape[0], 8192):
        Dh[r0:r0 + 8192] = Dv[r0:r0 + 8192].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    del Dv
    # sampled rows against the oracle (leftmost leads first: they take the longest sweep)
    rng = np.random.default_rng(11)
    ld = S.lead[S.nonpivot_row]
    lead_sig = np.where(ld < M.n, S.sigma[np.minimum(ld, M.n - 1)], M.n)
    order = np.argsort(lead_sig, kind="stable")
    t = np.unique(np.concatenate([order[:6], rng.choice(S.mN, 6, replace=False)]))
    dn, _, ops = oracle.dnew_rows(M, S, targets=t)
    assert np.array_equal(Dh[t], dn), "sampled D_new rows differ"
    rank = gb.gbla_echelon_D(h)
    r, pc, R = h.rref()
    assert r == rank == cfg.rank_planted, (r, cfg.rank_planted)
    _rref_structure(pc, R, rng)
    _rowspace_check(Dh, pc, R, M.p)
    h.free()
