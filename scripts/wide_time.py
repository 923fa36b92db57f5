#!/usr/bin/env python
"""Time SURVEY 8(f) f4 (gbla_reduce_wide) on an F4-shaped pattern with residues redrawn below a wide
prime (default: c1's pattern, p = 8388593 < 2^23).  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import gbla_gen
    import paper_1602_06097_b200 as gb
    name = sys.argv[1] if len(sys.argv) > 1 else "c1"
    p = int(sys.argv[2]) if len(sys.argv) > 2 else 8388593
    W = gbla_gen.widen(gbla_gen.f4_matrix(name), p, seed=1)
    ctx = gb.Context(0)
    rp = torch.from_numpy(W.row_ptr.view(np.int64)).cuda().view(torch.uint64)
    col = torch.from_numpy(W.col.view(np.int32)).cuda().view(torch.uint32)
    val = torch.from_numpy(W.val.view(np.int32)).cuda().view(torch.uint32)
    st = torch.cuda.current_stream()
    for it in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        h = gb.gbla_reduce_wide(ctx, W.m, W.n, rp, col, val, p, stream=st)
        e1.record(st)
        torch.cuda.synchronize()
        r = h.wide()[0]
        ops = h.opcount()[0]
        h.free()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"config": name, "p": p, "ms": round(ms, 2), "rank_D": r, "sparse_modmac": ops,
                      "Gop_s": round(ops / ms / 1e6, 1)}), flush=True)
    ctx.close()


import numpy as np  # noqa: E402

if __name__ == "__main__":
    main()
