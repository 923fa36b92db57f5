#!/usr/bin/env python
"""Device decode throughput of the paper's Format 2 (and Format 1) on a config's matrix
(gbla_file_decode): file bytes / decode time (host -> device copies of the sections
included, CUDA events around the call), the copies alone beside it.  Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import gbla_gen
    import paper_1602_06097_b200 as gb
    from oracle import formats as fm
    name = sys.argv[1] if len(sys.argv) > 1 else "c1"
    M = gbla_gen.f4_matrix(name)
    ctx = gb.Context(0)
    for fmt, data in ((2, fm.write_format2_nodedup(M)), (1, fm.write_format1(M))):
        pinned = torch.empty(len(data), dtype=torch.uint8).pin_memory()
        pinned.numpy()[:] = np.frombuffer(data, np.uint8)
        import ctypes
        info = gb.file_info(data, fmt)
        rp = torch.empty(info["m"] + 1, dtype=torch.uint64, device="cuda")
        col = torch.empty(info["nnz"], dtype=torch.uint32, device="cuda")
        val = torch.empty(info["nnz"], dtype=torch.uint16, device="cuda")
        lib = gb.load_library()
        ts = []
        for it in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            gb._check(lib.gbla_file_decode(ctx._h, ctypes.c_void_p(pinned.data_ptr()), len(data), fmt,
                                           ctypes.c_void_p(rp.data_ptr()), ctypes.c_void_p(col.data_ptr()),
                                           ctypes.c_void_p(val.data_ptr()), gb._stream_ptr(None)))
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        t = min(ts[1:])
        ok = bool(torch.equal(col.view(torch.int32).cpu(), torch.from_numpy(M.col.view(np.int32))))
        print(json.dumps({"config": name, "format": fmt, "file_bytes": len(data), "nnz": info["nnz"],
                          "decode_ms": round(t * 1e3, 3), "GB_per_s": round(len(data) / t / 1e9, 2),
                          "cols_match": ok, "note": "pinned host image, section H2D copies inside the timing"}),
              flush=True)
    ctx.close()


import numpy as np  # noqa: E402

if __name__ == "__main__":
    main()
