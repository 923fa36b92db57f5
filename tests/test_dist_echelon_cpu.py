"""The distributed echelon's protocol (panel.cu: panels_dist)
run by 2 and 3 gloo ranks on the CPU, in numpy, against the oracle's RREF.

Each rank owns the rows of the target tiles T = rank, rank + G, ... (tiles of
TILE rows) and never touches another rank's rows.  Per panel, exactly the
exchanges of the CUDA path: an all-reduce of the lead counts of the window
(C3a), the same panel-width rule as k_width, an all-gather of every rank's
candidate slices (C3b), the same panel factorization on every rank, an
all-reduce of the selected rows' full tails (C4, each from its owner, zeros
elsewhere), and a local update of own rows; R from every rank's pivot rows
(C6).  The panel factorization here is a plain dense Gauss-Jordan of the
candidates' window (what k_panel2 computes), so this checks the protocol -
window rule, candidate choice, replicated transform, back elimination of
earlier pivot rows - not the kernels (those are checked against the oracle on
the GPU with emulated ranks)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

PK, PW, TILE = 8, 16, 4        # pivots per panel, widest window, rows per target tile (small: many panels)
NONE = 1 << 30


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def panel_width(cnt, wmax):
    """k_width: widest w (multiple of 4 here, as the 32 of the kernels) with <= PK rows leading before w;
    dense (more than PK rows before min(PK, wmax)) -> min(PK, wmax)."""
    w128 = min(PK, wmax)
    if sum(cnt[:w128]) > PK:
        return w128, True
    width, cum = w128, 0
    for c in range(wmax + 1):
        if c >= w128 and cum <= PK and (c == wmax or c % 4 == 0):
            width = c
        if c < wmax:
            cum += cnt[c]
    return width, False


def rref_rows(V, p):
    """Gauss-Jordan of the rows of V (k x w) mod p: T with T @ V = the basis (rows with pivots), the
    pivot columns, and the candidates the basis replaces (T is supported on them only)."""
    V = V.copy() % p
    k = V.shape[0]
    E = np.eye(k, dtype=np.int64)
    perm = list(range(k))
    piv, r = [], 0
    for c in range(V.shape[1]):
        nz = [i for i in range(r, k) if V[i, c]]
        if not nz:
            continue
        i = nz[0]
        V[[r, i]] = V[[i, r]]
        E[[r, i]] = E[[i, r]]
        perm[r], perm[i] = perm[i], perm[r]
        iv = pow(int(V[r, c]), p - 2, p)
        V[r] = V[r] * iv % p
        E[r] = E[r] * iv % p
        for j in range(k):
            if j != r and V[j, c]:
                g = V[j, c]
                V[j] = (V[j] - g * V[r]) % p
                E[j] = (E[j] - g * E[r]) % p
        piv.append(c)
        r += 1
    assert not E[:r][:, [j for j in range(k) if j not in perm[:r]]].any()
    return E[:r], piv, perm[:r]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for seed, p, kind in ((1, 251, "staircase"), (2, 65521, "staircase"), (3, 7, "dense"), (4, 32003, "dense")):
            rng = np.random.default_rng(seed)
            m, n = 40, 56
            if kind == "staircase":                       # leads spread, rank deficient (dependent rows)
                D = np.zeros((m, n), np.int64)
                for i in range(m - 6):
                    l = rng.integers(0, n - 8)
                    D[i, l] = rng.integers(1, p)
                    D[i, l + 1:] = rng.integers(0, p, n - l - 1)
                for i in range(m - 6, m):
                    a, b = rng.choice(m - 6, 2, replace=False)
                    D[i] = (D[a] + rng.integers(1, p) * D[b]) % p
            else:
                base = rng.integers(0, p, (30, n))
                D = np.vstack([base, (rng.integers(0, p, (m - 30, 30)) @ base) % p])
            D = D[rng.permutation(m)] % p
            order = np.argsort([np.nonzero(r)[0][0] if r.any() else n for r in D], kind="stable")
            owner = np.empty(m, np.int64)
            owner[order] = (np.arange(m) // TILE) % world
            mine = owner == rank
            rowpiv = np.full(m, -1)
            c0 = 0
            while c0 < n:
                wmax = min(PW, n - c0)
                lead = np.full(m, NONE)
                for i in np.nonzero(mine & (rowpiv < 0))[0]:
                    nz = np.nonzero(D[i, c0:c0 + wmax])[0]
                    if nz.size:
                        lead[i] = nz[0]
                cnt = torch.zeros(wmax, dtype=torch.int64)
                for l in lead[lead < wmax]:
                    cnt[l] += 1
                dist.all_reduce(cnt)                       # C3a
                width, dense = panel_width(cnt.tolist(), wmax)
                own = [(int(lead[i]), int(i)) for i in np.nonzero(lead < width)[0]]
                allc = [None] * world
                dist.all_gather_object(allc, [(l, i, D[i, c0:c0 + width].tolist()) for l, i in own])   # C3b
                cands = sorted(c for block in allc for c in block)
                rids = [i for _, i, _ in cands]
                if cands:
                    V = np.array([v for _, _, v in cands], np.int64)
                    T, piv, heads = rref_rows(V, p)
                else:
                    T, piv, heads = np.zeros((0, 0), np.int64), [], []
                kp = len(piv)
                S = np.zeros((len(rids), n - c0), np.int64)   # C4: candidates' tails from their owners
                for j, i in enumerate(rids):
                    if mine[i]:
                        S[j] = D[i, c0:]
                St = torch.from_numpy(S)
                dist.all_reduce(St)
                Rn = (T @ St.numpy()) % p if kp else np.zeros((0, n - c0), np.int64)
                pcs = [c0 + c for c in piv]
                selected = [rids[j] for j in heads]       # the basis rows replace the candidates they combine
                for i in np.nonzero(mine)[0]:
                    if i in selected:
                        continue
                    F = D[i, pcs]
                    if F.any():
                        D[i, c0:] = (D[i, c0:] - F @ Rn) % p
                for b, i in enumerate(selected):
                    if mine[i]:
                        D[i, c0:] = Rn[b]
                        rowpiv[i] = pcs[b]
                c0 += width
            rows = [(int(rowpiv[i]), D[i].tolist()) for i in np.nonzero(mine & (rowpiv >= 0))[0]]
            allr = [None] * world
            dist.all_gather_object(allr, rows)                 # C6
            R = sorted(r for block in allr for r in block)
            out.append((seed, p, kind, [c for c, _ in R], [r for _, r in R]))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_echelon_protocol_matches_oracle(world):
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for case in range(4):
        seed, p, kind, pcs, R = res[0][case]
        for r in range(1, world):
            assert res[r][case][3] == pcs and res[r][case][4] == R      # every rank assembles the same R
        # the oracle on the same matrix
        rng = np.random.default_rng(seed)
        m, n = 40, 56
        if kind == "staircase":
            D = np.zeros((m, n), np.int64)
            for i in range(m - 6):
                l = rng.integers(0, n - 8)
                D[i, l] = rng.integers(1, p)
                D[i, l + 1:] = rng.integers(0, p, n - l - 1)
            for i in range(m - 6, m):
                a, b = rng.choice(m - 6, 2, replace=False)
                D[i] = (D[a] + rng.integers(1, p) * D[b]) % p
        else:
            base = rng.integers(0, p, (30, n))
            D = np.vstack([base, (rng.integers(0, p, (m - 30, 30)) @ base) % p])
        D = D[rng.permutation(m)] % p
        rank, Ro, pivcol = oracle.rref(D.astype(np.uint32), p)
        assert rank == len(pcs) and pivcol.tolist() == pcs, (kind, p)
        assert np.array_equal(np.array(R, np.int64).reshape(rank, n), Ro.astype(np.int64)), (kind, p)
