#!/usr/bin/env python
"""Time gbla_reduce on one config under several environment settings (one process,
one generated matrix).  Usage:
    python scripts/env_sweep.py c4 "GBLA_SWEEP_GROUP=8" "GBLA_SWEEP_GROUP=16,GBLA_BSUB_GROUP=16" ...
An empty setting ("") is the default.  Prints one JSON line per setting with the step times and
the per-kernel CUDA-event times (GBLA_KERNEL_TIMERS)."""
import gc
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("GBLA_KERNEL_TIMERS", "1")

import torch  # noqa: E402

import gbla_gen  # noqa: E402
import paper_1602_06097_b200 as gb  # noqa: E402


def main():
    cfg_name = sys.argv[1]
    steps = int(os.environ.get("ENV_SWEEP_STEPS", "2"))
    settings = sys.argv[2:] or [""]
    M = gbla_gen.f4_matrix(gbla_gen.CONFIGS[cfg_name])
    rp = torch.from_numpy(M.row_ptr).cuda()
    col = torch.from_numpy(M.col).cuda()
    val = torch.from_numpy(M.val).cuda()
    ctx = gb.Context(0)
    stream = torch.cuda.current_stream()
    gc.collect()
    gc.disable()
    base = dict(os.environ)
    ref = None
    for s in settings:
        os.environ.clear()
        os.environ.update(base)
        for kv in filter(None, s.split(",")):
            k, v = kv.split("=", 1)
            os.environ[k] = v
        ms, kms = [], []
        for i in range(steps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            h = gb.gbla_reduce(ctx, M.m, M.n, rp, col, val, M.p, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            rank, pc, R = h.rref()
            sig = (rank, int(pc.to(torch.int64).sum().item()),
                   int(R[:, : min(R.shape[1], 256)].to(torch.int64).sum().item()) if rank else 0)
            if ref is None:
                ref = sig
            ok = sig == ref
            if i > 0:                       # first call of a setting is its warm-up
                ms.append(round(e0.elapsed_time(e1), 3))
                kms.append({k: round(v[0], 2) for k, v in h.kernel_ms().items()})
            h.free()
            torch.cuda.empty_cache()
        print(json.dumps({"config": cfg_name, "setting": s or "default", "ms": ms, "kernel_ms": kms,
                          "same_result": ok}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
