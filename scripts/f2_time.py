#!/usr/bin/env python
"""Time SURVEY 8(f) f2 (gbla_rref_M: RREF of the whole M in the original column order) after a
gbla_reduce, on the given configs (default c1 c3).  CUDA events on the library stream; prints
one JSON line per config: reduce ms, rref_M ms, rank(M), nnz of RREF(M)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import gbla_gen
    import paper_1602_06097_b200 as gb
    ctx = gb.Context(0)
    for name in (sys.argv[1:] or ["c1", "c3"]):
        M = gbla_gen.f4_matrix(name)
        rp, col, val = (torch.from_numpy(a).cuda() for a in (M.row_ptr, M.col, M.val))
        st = torch.cuda.current_stream()
        for it in range(3):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(st)
            h = gb.gbla_reduce(ctx, M.m, M.n, rp, col, val, M.p, stream=st)
            e[1].record(st)
            r, rpo, co, vo = h.rref_M(stream=st)
            e[2].record(st)
            torch.cuda.synchronize()
            if it == 2:
                print(json.dumps({"config": name, "reduce_ms": round(e[0].elapsed_time(e[1]), 2),
                                  "rref_M_ms": round(e[1].elapsed_time(e[2]), 2), "rank_M": r,
                                  "nnz_rref_M": int(co.numel()), "npiv": h.dims()[0]}), flush=True)
            h.free()
    ctx.close()


if __name__ == "__main__":
    main()
