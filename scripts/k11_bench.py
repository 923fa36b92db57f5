#!/usr/bin/env python
"""K11 (modular GEMM C -= A B mod p on tcgen05, u8 limbs) microbenchmark through the C ABI
(gbla_modgemm_bench): the shapes of the echelon's trailing updates (c2: 40,000 rows, widths up
to 90,000, K = 128 per panel and K = 512 for the deferred super-panel flush).  Prints one JSON
line per shape: ms per launch, T modMAC/s, int8 TOPS (4 u8 MACs x 2 ops per modMAC) and the
D bytes (u16 read + write) per second."""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_1602_06097_b200 as gb
    if os.environ.get("GBLA_LIB"):
        gb.load_library(os.environ["GBLA_LIB"])   # a variant build (experiments)
    ctx = gb.Context(0)
    shapes = [(40000, 45056, 512), (40000, 45056, 128), (16384, 16384, 512), (8192, 90112, 512)]
    if len(sys.argv) > 1:
        shapes = [tuple(int(x) for x in s.split("x")) for s in sys.argv[1:]]
    for rows, cols, K in shapes:
        ms = gb.modgemm_bench(ctx, 65521, rows, cols, K, reps=5)
        kk = (K + 127) // 128 * 128
        mm = rows * cols * kk
        print(json.dumps({"rows": rows, "cols": cols, "K": kk, "ms": round(ms, 4),
                          "T_modmac_s": round(mm / ms / 1e9, 2), "int8_TOPS": round(mm * 8 / ms / 1e9, 1),
                          "D_GBs": round(rows * cols * 4 / ms / 1e6, 1)}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
