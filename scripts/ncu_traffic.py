#!/usr/bin/env python
"""Per-kernel-family DRAM traffic for bench.py's roofline "traffic" field, from a
launch list (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) or one `ncu --set full` capture of the SAME bench
config.  Usage (here, no GPU needed):
    python scripts/ncu_traffic.py <launches.csv | prof.ncu-rep> profiles/ncu_traffic.json <config>
Merges {config: {family: {kernel, dram_bytes_per_launch, duration_ms_per_launch,
launches_captured, source}}} into the JSON (other configs are kept)."""
import csv
import io
import json
import subprocess
import sys

FAMILIES = [("k_sweep<1>", "backsub"), ("k_sweep", "sweep"), ("k_update_tc", "update"), ("k_panel", "panel"),
            ("k_modgemm_ws<0", "trailing"), ("k_modgemm_mk2", "trailing"), ("k_modgemm_win", "trailing"),
            ("k_modgemm_ws<1", "rnew")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TSCALE = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}


def family(name):
    for key, fam in FAMILIES:
        if key in name:
            return fam
    return None


def from_launch_list(path, out):
    """A launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv):
    per family, the mean DRAM bytes and duration per launch over every captured launch."""
    lines = [ln for ln in open(path) if ln.startswith('"')]
    recs = {}
    for r in csv.DictReader(lines):
        rec = recs.setdefault(r["ID"], {"name": r["Kernel Name"]})
        unit = r["Metric Unit"]
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Name"].startswith("dram__bytes"):
            v *= SCALE.get(unit, 1)
        elif r["Metric Name"] == "gpu__time_duration.sum":
            v *= TSCALE.get(unit, 1e-6)
        rec[r["Metric Name"]] = v
    acc = {}
    for rec in recs.values():
        fam = family(rec["name"])
        if fam is None or "dram__bytes_read.sum" not in rec:
            continue
        a = acc.setdefault(fam, {"kernel": rec["name"].split("(")[0], "bytes": 0.0, "ms": 0.0, "n": 0})
        a["bytes"] += rec["dram__bytes_read.sum"] + rec["dram__bytes_write.sum"]
        a["ms"] += rec.get("gpu__time_duration.sum", 0.0)
        a["n"] += 1
    res = {fam: {"kernel": a["kernel"], "dram_bytes_per_launch": round(a["bytes"] / a["n"]),
                 "duration_ms_per_launch": round(a["ms"] / a["n"], 4), "launches_captured": a["n"],
                 "source": path.split("/")[-1]} for fam, a in acc.items()}
    return res


def main():
    rep, out, cfg = sys.argv[1], sys.argv[2], sys.argv[3]
    res = from_launch_list(rep, out) if rep.endswith(".csv") else from_capture(rep)
    try:
        db = json.load(open(out))
    except Exception:
        db = {}
    if db and not all(isinstance(v, dict) and "kernel" not in v for v in db.values()):
        db = {}                                        # an old single-config file
    db[cfg] = res
    json.dump(db, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


def from_capture(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    acc = {}
    for r in rows[2:]:
        fam = family(r[col["Kernel Name"]])
        if fam is None:
            continue
        rd = float(r[col["dram__bytes_read.sum"]]) * SCALE[units[col["dram__bytes_read.sum"]]]
        wr = float(r[col["dram__bytes_write.sum"]]) * SCALE[units[col["dram__bytes_write.sum"]]]
        t = float(r[col["gpu__time_duration.sum"]]) * TSCALE[units[col["gpu__time_duration.sum"]]]
        k = "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
        tp = float(r[col[k]]) if k in col and r[col[k]] else None
        a = acc.setdefault(fam, {"kernel": r[col["Kernel Name"]].split("(")[0], "bytes": 0.0, "ms": 0.0, "n": 0,
                                 "tensor": []})
        a["bytes"] += rd + wr
        a["ms"] += t
        a["n"] += 1
        if tp is not None:
            a["tensor"].append(tp)
    res = {}
    for fam, a in acc.items():
        res[fam] = {"kernel": a["kernel"], "dram_bytes_per_launch": round(a["bytes"] / a["n"]),
                    "duration_ms_per_launch": round(a["ms"] / a["n"], 4),
                    "tensor_pipe_pct_of_active": round(sum(a["tensor"]) / len(a["tensor"]), 2) if a["tensor"] else None,
                    "launches_captured": a["n"], "source": rep.split("/")[-1]}
    return res


if __name__ == "__main__":
    main()
