#!/usr/bin/env python
"""Time Step 2 (gbla_reduce_B) and the standard-order update (gbla_update_D) on the
given configs (default c1), tensor-core TRSM (default) against the INT-pipe K8 (GBLA_TRSM_INT=1).
The library's phase timers (CUDA events on its stream); one JSON line per config and engine."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import gbla_gen
    import paper_1602_06097_b200 as gb
    ctx = gb.Context(0)
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    engines = ("0",) if "--tc-only" in sys.argv else ("0", "1")
    for name in (args or ["c1"]):
        M = gbla_gen.f4_matrix(name)
        rp, col, val = (torch.from_numpy(a).cuda() for a in (M.row_ptr, M.col, M.val))
        for eng in engines:
            os.environ["GBLA_TRSM_INT"] = eng
            best = None
            for it in range(3):
                h = gb.gbla_splice(ctx, M.m, M.n, rp, col, val, M.p)
                gb.gbla_reduce_B(h)
                gb.gbla_update_D(h)
                torch.cuda.synchronize()
                ph = h.phase_ms()
                if best is None or ph["reduce_B"] < best["reduce_B"]:
                    best = ph
                npiv, mN, nN = h.dims()
                h.free()
            print(json.dumps({"config": name, "trsm": "int (K8)" if eng == "1" else "tensor cores",
                              "npiv": npiv, "nN": nN, "reduce_B_ms": round(best["reduce_B"], 2),
                              "update_D_ms": round(best["update_D"], 2)}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
