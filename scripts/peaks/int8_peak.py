#!/usr/bin/env python
"""Measured int8 tensor peak of this B200 (the denominator of the dense-D
roofline): torch._int_mm (cuBLASLt int8 x int8 -> int32) on
8192^3, 2*N^3 ops per call, best of 10 (burst) and back to back for 4 s
(sustained), the way MEASURED_PEAKS.json measures bf16.  Prints one JSON line."""
import json
import time

import torch


def main():
    n = 8192
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    burst = 2 * n ** 3 / (best / 1e3) / 1e12
    t_end = time.time() + 4.0
    calls = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() < t_end:
        for _ in range(20):
            torch._int_mm(a, b)
        calls += 20
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sus = 2 * n ** 3 * calls / (e0.elapsed_time(e1) / 1e3) / 1e12
    print(json.dumps({"int8_tops_burst": round(burst, 1), "int8_tops_sustained": round(sus, 1),
                      "how": "torch._int_mm int8 8192^3 (2*N^3 ops): best of 10 / back to back 4 s",
                      "gpu": torch.cuda.get_device_name()}))


if __name__ == "__main__":
    main()
