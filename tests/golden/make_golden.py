"""Write tests/golden/<cfg>_oracle.json from the CPU oracle ONLY.

Usage: python tests/golden/make_golden.py c0 c1 [--threads N]

Stored values: n_piv, mN, nN, rank(D_new), sparse-phase modMAC count, the
SHA-256 digests of D_new (u16 row-major) and of the canonical RREF
(oracle.rref_digest), and the input CSR digest (so a generator change is
detected).  Nothing here touches the CUDA path.
"""
import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import gbla_gen  # noqa: E402
import oracle  # noqa: E402


def csr_digest(M) -> str:
    h = hashlib.sha256()
    for a, dt in ((M.row_ptr, "<u8"), (M.col, "<u4"), (M.val, "<u2")):
        h.update(np.ascontiguousarray(a, dtype=dt).tobytes())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=oracle.default_threads())
    a = ap.parse_args()
    for name in a.configs:
        M = gbla_gen.f4_matrix(name)
        t0 = time.time()
        S = oracle.splice(M)
        dn, _, ops = oracle.dnew_rows(M, S, threads=a.threads)
        t1 = time.time()
        rank, R, pc = oracle.rref(dn, M.p, threads=a.threads)
        t2 = time.time()
        out = {
            "config": name,
            "written_by": "tests/golden/make_golden.py (oracle/ only)",
            "csr_sha256": csr_digest(M),
            "m": M.m, "n": M.n, "nnz": M.nnz, "p": M.p,
            "npiv": S.npiv, "mN": S.mN, "nN": S.nN,
            "rank_D": rank, "rank_M": S.npiv + rank,
            "modmac_sparse": int(ops.sum()),
            "dnew_sha256": oracle.array_digest(dn),
            "rref_sha256": oracle.rref_digest(rank, S.nN, pc, R),
            "oracle_seconds": {"splice+dnew": round(t1 - t0, 2), "rref": round(t2 - t1, 2)},
            "threads": a.threads,
        }
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"{name}_oracle.json")
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
        print(json.dumps(out))


if __name__ == "__main__":
    main()
