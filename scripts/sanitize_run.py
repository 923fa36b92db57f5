#!/usr/bin/env python
"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck / synccheck, one tool per
process): c0 through gbla_reduce (sweep, update, panels with look-ahead, K11), a scaled c3 with
super-panels (CTA-pair multi-K flushes, prefix-slot updates) and f2 (gbla_rref_M), each checked
against the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    import gbla_gen
    import oracle
    import paper_1602_06097_b200 as gb
    ctx = gb.Context(0)
    cases = [gbla_gen.f4_matrix("c0")]
    if "--small" not in sys.argv:
        cases.append(gbla_gen.f4_matrix(gbla_gen.scaled(gbla_gen.CONFIGS["c3"], 0.04)))
    for i, M in enumerate(cases):
        if i == 1:
            os.environ["GBLA_SP"] = "4"
        res = oracle.reduce(M)
        rp, col, val = (torch.from_numpy(a).cuda() for a in (M.row_ptr, M.col, M.val))
        h = gb.gbla_reduce(ctx, M.m, M.n, rp, col, val, M.p)
        r, pc, R = h.rref()
        assert r == res.rank and np.array_equal(R.cpu().numpy(), res.R), M.name
        rk, _, _, _ = h.rref_M()
        assert rk == res.rank_M
        h.free()
        print("ok", M.name, r, rk, flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
