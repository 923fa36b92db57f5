#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
total device time, launches and share per kernel.  Usage:
    python scripts/launch_summary.py gpurun_out/launches.csv [steps]
With `steps` the per-step times are printed too (the launch list covers
warm-up + timed steps of the same command)."""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}[unit]
        rows.append((name, v * scale))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for n, ms in rows:
        tot[n] += ms
        cnt[n] += 1
    T = sum(tot.values())
    print(f"launches {len(rows)}  total device time {T:.3f} ms  ({T / steps:.3f} ms per step over {steps} steps)")
    for n, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{ms:10.3f} ms {ms / steps:9.3f} ms/step {cnt[n]:6d}  {100 * ms / T:5.1f}%  {n}")


if __name__ == "__main__":
    main()
