#!/usr/bin/env python
"""bench.py -- Faugere-Lachartre reduction (GBLA, arXiv 1602.06097) on B200.

One STEP = one gbla_reduce over the bench workload (default BASELINE.json
configs[2] = c2, 200,000 x 250,000, p = 65521: the largest config that fits
one GPU with room to spare; --config c1 for the Katsura-12-scale matrix):
splice -> sparse phase (Alg 2, fused reduce_C + update_D) -> fully reduced
echelon of D, device-resident CSR in, device-resident R + rank out.

metric  nnz-AXPY Gop/s mod p: exact sparse-phase modMAC count (Alg 2 count,
        equal to the oracle's) / whole-step time.  ms_per_step is the F4
        matrix reduction time.
e2e     the same metric through the C ABI with HOST buffers: pinned-host CSR
        copied in by the library (GBLA_HOST_INPUT) and R + pivcol copied back
        to host, inside the timed region.
--impl reference   the CPU oracle (oracle/, plain C) on the box's host cores,
        each step a bounded sample of the config's targets (same metric, unit).

Multi-GPU (torchrun, N > 1): see DESIGN.md §"Multi-GPU"; one process per GPU.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")


def _peaks():
    try:
        return json.load(open(MEASURED)), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 9:
                for k, nm in enumerate(names):
                    if r[5 + k].lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, bounded samples."""
    world, rank, _ = _dist()
    if world > 1 and rank != 0:
        return
    import gbla_gen
    import oracle
    cfg = gbla_gen.CONFIGS[args.config]
    M = gbla_gen.f4_matrix(cfg)
    S = oracle.splice(M)
    threads = oracle.default_threads()
    rng = np.random.default_rng(123)
    per_step = args.ref_targets
    for _ in range(args.warmup):
        oracle.dnew_rows(M, S, targets=np.sort(rng.choice(S.mN, max(8, per_step // 8), replace=False)),
                         threads=threads)
    times, ops = [], 0
    for _ in range(args.steps):
        t = np.sort(rng.choice(S.mN, per_step, replace=False))
        t0 = time.perf_counter()
        _, _, o = oracle.dnew_rows(M, S, targets=t, threads=threads)
        times.append(time.perf_counter() - t0)
        ops += int(o.sum())
    tot = sum(times)
    gops = ops / tot / 1e9
    sample = (f"oracle Alg 2 (sparse phase) on {per_step} random targets of {args.config} per step "
              f"(of mN={S.mN}); splice not timed; RREF not included")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gops, 4), "unit": "Gop/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(tot / args.steps * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64 accumulate, u16 residues", "data": "synthetic",
        "config": {"workload": cfg.name, "m": cfg.m, "n": cfg.n, "npiv": cfg.npiv, "p": cfg.p,
                   "density": cfg.density, "band": cfg.band, "rank_planted": cfg.rank_planted,
                   "flags": args.flags, "parallelism": f"CPU oracle on {threads} host threads (rank 0 only)"},
        "cpu_baseline": {"value": round(gops, 4), "unit": "Gop/s", "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(gops, 4), "unit": "Gop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "nnz-AXPY Gop/s mod p (F4 matrix reduction, gbla_reduce)"

# kernel families timed by the library (gbla_get_kernel_ms) and how each is bounded
KERNEL_NAMES = {"sweep": "k_sweep<0> (K5', C' = C A^-1 block forward substitution, tcgen05)",
                "update": "k_update_tc (K7', D -= C' B, tcgen05)",
                "panel": "k_panel2 (K10, panel echelon form, one CTA)",
                "trailing": "K11 trailing update (k_modgemm_mk2 CTA-pair K = 512 flushes + k_modgemm_ws / "
                            "k_modgemm_win K = 128 window updates)",
                "rnew": "k_modgemm_ws<STORE> (K11 new pivot rows)",
                "backsub": "K14 back substitution RREF = U_sq^-1 U (k_sweep<1> on the pivot block of the row echelon "
                           "form; band / C-tile setup included)"}
TRAFFIC = os.path.join(ROOT, "profiles", "ncu_traffic.json")
INT8_PEAK = os.path.join(ROOT, "profiles", "r02_int8_peak.json")      # scripts/peaks/int8_peak.py on a B200
IMAD_PEAK = os.path.join(ROOT, "profiles", "r02_imad_peak.json")      # scripts/peaks/imad_peak.cu on a B200


def _int8_peak(peaks, peak_src):
    """Dense int8 tensor peak (TOPS): measured torch._int_mm 8192^3 (burst / sustained) if the
    measurement is committed, else 2 x the measured bf16 peak (nominal int8:bf16 = 2)."""
    try:
        m = json.load(open(INT8_PEAK))
        return float(m["int8_tops_burst"]), float(m["int8_tops_sustained"]), \
            "measured torch._int_mm int8 8192^3 on a B200 (profiles/r02_int8_peak.json)"
    except Exception:
        return 2.0 * float(peaks["bf16_tflops"]), 2.0 * float(peaks["bf16_tflops_sustained"]), \
            f"2 x {peak_src} bf16 (MEASURED_PEAKS.json; nominal int8:bf16 = 2; int8 not measured)"


def _imad_peak(sm_count, sm_mhz):
    try:
        m = json.load(open(IMAD_PEAK))
        return float(m["int_modmac_T_per_s"]), "measured acc += (u64)a*b microbenchmark (profiles/r02_imad_peak.json)"
    except Exception:
        return sm_count * 32 * sm_mhz * 1e6 / 1e12, f"derived: {sm_count} SMs x 32 IMAD.WIDE/clk x {sm_mhz:.0f} MHz"


def roofline(kms, kwork, peaks, peak_src, sm_count, config, kexec=None):
    """Roofline of the dominant kernel family (largest CUDA-event time over the timed steps), against
    WHOLE-GPU peaks.  Tensor-core families: achieved = algorithmic modMACs (gbla_get_kernel_work,
    DESIGN.md §6) x 4 u8 MACs (limb split) x 2 ops / family time, against the dense int8 peak
    (the sustained figure: these kernels run inside a long step; burst beside it).  The panel K10
    (one CTA, INT pipe + mma.sync): modMACs / time against the whole GPU's measured INT-pipe modMAC
    rate.  traffic = ncu DRAM bytes per launch of that family in a launch list of the SAME config."""
    dom = max(kms, key=lambda k: kms[k][0])
    ms, n = kms[dom]
    work = kwork[dom]
    try:
        tr = json.load(open(TRAFFIC)).get(config, {}).get(dom)
    except Exception:
        tr = None
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    sec = ms / 1e3 if ms > 0 else float("inf")
    if dom == "panel":
        peak, src = _imad_peak(sm_count, sm_mhz)
        ach = work / sec / 1e12
        out = {"bound": "alu", "achieved": round(ach, 5), "peak": round(peak, 3), "unit": "Tmodmac/s",
               "peak_source": src + "; the kernel is ONE CTA by design (latency/barrier bound)"}
    else:
        burst, sustained, src = _int8_peak(peaks, peak_src)
        ach = work * 4 * 2 / sec / 1e12
        out = {"bound": "tensor", "achieved": round(ach, 2), "peak": round(sustained, 1), "unit": "TOPS",
               "peak_source": src + " (sustained; burst " + f"{burst:.0f})",
               "frac_of_burst": round(ach / burst, 4) if burst else None,
               "modmac_per_s_T": round(work / sec / 1e12, 3)}
        if kexec and kexec.get(dom):
            # the dense 128 x 128 band tiles the family executes (any density): executed int8 rate
            ex = kexec[dom] * 2 / sec / 1e12
            out["executed_TOPS"] = round(ex, 1)
            out["executed_frac"] = round(ex / sustained, 4)
            out["algorithmic_over_executed"] = round(work * 4 / kexec[dom], 4)
        if dom == "trailing" and kwork.get("trailing_elems"):
            byts = 4.0 * kwork["trailing_elems"]          # u16 read + write per D entry of every update
            out["hbm_algorithmic_GBs"] = round(byts / sec / 1e9, 1)
            out["hbm_frac"] = round(byts / sec / 1e9 / float(peaks["hbm_gbs"]), 4)
    out.update({"kernel": KERNEL_NAMES[dom], "frac": round(out["achieved"] / out["peak"], 5) if out["peak"] else 0.0,
                "kernel_ms_total": round(ms, 3), "launches": n, "algorithmic_modmac": int(work),
                "algorithmic_modmac_per_launch": int(work / max(n, 1)),
                "traffic": (tr["dram_bytes_per_launch"] if tr else None),
                "traffic_source": (f"profiles/{tr['source']} ({config} launch list: ncu dram__bytes_read+write per "
                                   f"launch of the family)" if tr else None)})
    return out


def cpu_baseline(cfg_name: str, M, targets: int):
    import oracle
    S = oracle.splice(M)
    threads = oracle.default_threads()
    rng = np.random.default_rng(7)
    t = np.sort(rng.choice(S.mN, min(targets, S.mN), replace=False))
    t0 = time.perf_counter()
    _, _, o = oracle.dnew_rows(M, S, targets=t, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": round(int(o.sum()) / dt / 1e9, 4), "unit": "Gop/s", "cores": threads, "kind": "oracle",
            "sample": f"oracle Alg 2 (sparse phase only) on {t.size} random targets of {cfg_name} "
                      f"(of mN={S.mN}), {dt:.1f} s wall on {threads} threads"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", help="BASELINE.json config (c2: the largest single-GPU headline)")
    ap.add_argument("--flags", type=int, default=0, help="gbla_reduce flags")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-targets", type=int, default=384)
    ap.add_argument("--ref-targets", type=int, default=96)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    os.environ.setdefault("GBLA_KERNEL_TIMERS", "1")    # per-kernel CUDA events on the library's stream
    import torch
    import gbla_gen
    import paper_1602_06097_b200 as gb

    world, rank, local = _dist()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    cfg = gbla_gen.CONFIGS[args.config]
    M = gbla_gen.f4_matrix(cfg)              # host, seeded; with N > 1 only rank 0's copy is used
    rp = torch.from_numpy(M.row_ptr).cuda()
    col = torch.from_numpy(M.col).cuda()
    val = torch.from_numpy(M.val).cuda()
    ctx = gb.Context(dev)
    if world > 1:
        # NCCL communicator inside libgbla; the ncclUniqueId travels over torch.distributed.
        # gbla_reduce then broadcasts rank 0's CSR (C1), shards the target tiles, all-gathers D_new.
        uid = [gb.nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(uid, src=0)
        ctx.set_comm(uid[0], rank, world)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    def step():
        h = gb.gbla_reduce(ctx, M.m, M.n, rp, col, val, M.p, flags=args.flags, stream=stream)
        return h

    # libgbla allocates device memory through torch (a Python callback per buffer): keep the Python
    # garbage collector from running inside those callbacks in the middle of a reduction
    gc.collect()
    gc.disable()
    for _ in range(max(args.warmup, 0)):
        step().free()
    torch.cuda.synchronize()
    launches0 = gb.kernel_launches()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    phases = []
    kms = {k: [0.0, 0] for k in gb.Mat.KERNELS}
    kwork = {k: 0 for k in list(gb.Mat.KERNELS) + ["trailing_elems"]}
    kexec = {k: 0 for k in gb.Mat.KERNELS}
    kms_steps = []
    ops = dense_ops = 0
    rank_d = None
    clocks = ClockSampler(dev)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for i in range(args.steps):
        flush.zero_()                                 # L2 flush between timed steps
        ev[i][0].record(stream)
        h = step()
        ev[i][1].record(stream)
        phases.append(h.phase_ms())
        step_k = {}
        for k, (ms_k, n_k) in h.kernel_ms().items():
            kms[k][0] += ms_k
            kms[k][1] += n_k
            step_k[k] = round(ms_k, 2)
        kms_steps.append(step_k)
        for k, w in h.kernel_work().items():
            kwork[k] += w
        for k, w in h.kernel_exec().items():
            kexec[k] += w
        ops, dense_ops = h.opcount()
        rank_d = h.dims(), h.rank()
        h.free()
    torch.cuda.synchronize()
    clk = clocks.stop()
    gc.enable()
    launches = gb.kernel_launches() - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = statistics.mean(step_ms)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()

    # ---- e2e through the C ABI with pinned host buffers
    e2e = None
    if args.e2e_steps > 0:           # collective when N > 1 (every rank runs it; rank 0's input is used)
        hp = [torch.from_numpy(a).pin_memory() for a in (M.row_ptr, M.col, M.val)]
        hn = [t.numpy() for t in hp]
        (npiv, mN, nN), rk = rank_d
        h2d = M.row_ptr.nbytes + M.col.nbytes + M.val.nbytes
        d2h = rk * nN * 2 + rk * 4
        # results land in pinned host buffers (allocated once, outside the timed region)
        out_pc = torch.empty(max(rk, 1), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
        out_R = torch.empty((max(rk, 1), max(nN, 1)), dtype=torch.int16).pin_memory().numpy().view(np.uint16)
        e_ms = []
        gc.collect()
        gc.disable()
        for i in range(args.e2e_steps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h = gb.gbla_reduce(ctx, M.m, M.n, hn[0], hn[1], hn[2], M.p, flags=args.flags, stream=stream)
            r, pc_h, R_h = h.rref_to_host(stream=stream, out=(out_pc, out_R))
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) * 1e3
            h.free()
            if i > 0:
                e_ms.append(dt)
        gc.enable()
        em = statistics.mean(e_ms)
        if world > 1:
            t = torch.tensor([em], device="cuda", dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            em = float(t.item())
        e2e = {"value": round(ops / (em / 1e3) / 1e9, 4), "unit": "Gop/s", "ms_per_step": round(em, 3),
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "note": "host wall clock around gbla_reduce(GBLA_HOST_INPUT, pinned) + gbla_copy_rref_to_host"}

    if rank == 0:
        peaks, peak_src = _peaks()
        ph = {k: round(statistics.mean(p[k] for p in phases), 3) for k in phases[0]}
        dims = rank_d[0] if rank_d else (0, 0, 0)
        roof = roofline(kms, kwork, peaks, peak_src, torch.cuda.get_device_properties(dev).multi_processor_count,
                        cfg.name, kexec)
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_baseline(cfg.name, M, args.cpu_targets)
        line = {
            "metric": METRIC, "value": round(ops / (ms / 1e3) / 1e9, 4), "unit": "Gop/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u16", "dtype_note": "exact arithmetic on u16 residues mod p (no rounding): tensor-core "
                                          "products on u8 limbs with s32 accumulation, u64 delayed reduction on "
                                          "the INT pipe",
            "data": "synthetic",
            "config": {"workload": cfg.name, "m": cfg.m, "n": cfg.n, "npiv": cfg.npiv, "p": cfg.p,
                       "density": cfg.density, "band": cfg.band, "rank_planted": cfg.rank_planted,
                       "flags": args.flags, "l2": "flushed (256 MiB write) between timed steps; inputs > L2",
                       "parallelism": (f"{world} GPUs: C1 broadcast of M, target tiles sharded (sparse phase), "
                                       f"row-sharded distributed echelon (NCCL all-reduce / all-gather per "
                                       f"panel, R assembled by broadcasts)") if world > 1 else "1 GPU"},
            "value_note": "exact sparse-phase (Alg 2) modMAC count / WHOLE gbla_reduce time (splice + sparse phase "
                          "+ echelon): conservative; SURVEY 8(d)'s sparse-phase-only rate is value_sparse_phase",
            "value_sparse_phase": round(ops / (statistics.mean(p["reduce_C"] for p in phases) / 1e3) / 1e9, 2),
            "sparse_modmac_per_step": ops, "dense_modmac_per_step": dense_ops,
            "rank_D": rank_d[1], "npiv": rank_d[0][0],
            "phase_ms": ph, "step_ms": [round(x, 3) for x in step_ms],
            "kernel_ms_per_step": {k: round(v[0] / args.steps, 3) for k, v in kms.items()},
            "phase_ms_steps": [{k: round(v, 2) for k, v in p.items() if v} for p in phases],
            "kernel_ms_steps": kms_steps,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "gpu_launches_per_step": round(launches / max(args.steps, 1), 1),
            "clocks": clk, "peaks_source": peak_src,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
