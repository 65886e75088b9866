#!/usr/bin/env python
"""Benchmark of the FHR hot path (BASELINE.json metric: hyperspectral voxel*lambda
reconstructed per second on 1xB200, plus % roofline).

One step = the whole hot path on one batch of synthetic input already resident
in HBM: subspace_decompose (n_iter Lee-Seung iterations from the seeded init)
-> fbp of the K subspace sinograms -> synthesize x^h over all slices and bins.
value = N_x * N_k * ranks / (max-over-ranks time per step).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl hsnct|reference]

--impl reference times the fp64 CPU oracle (the tier's reference arm) on a bounded
sample of the same workload.  Under torchrun every rank runs an independent
replica of the workload (weak scaling, no data-path collective).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "hyperspectral voxel\u00b7\u03bb reconstructed/sec (1\u00d7B200) + % roofline per stage"  # BASELINE.json
UNIT = "voxel\u00b7\u03bb/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    # default: C5, the largest single-GPU configuration (BASELINE.json's metric names none)
    ap.add_argument("--config", type=int, default=5, help="BASELINE.json configs[i-1] (6: the paper's Table I shape)")
    ap.add_argument("--impl", default="hsnct", choices=["hsnct", "reference"])
    ap.add_argument("--n-iter", type=int, default=None, help="override NMF iterations (testing only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dhr", action="store_true")
    ap.add_argument("--no-fmd", action="store_true")
    ap.add_argument("--no-mbir", action="store_true")
    ap.add_argument("--no-counts", action="store_true")
    ap.add_argument("--mbir-iters", type=int, default=10, help="SQS iterations of the MBIR extra (NEXT-3)")
    ap.add_argument("--shard", action="store_true",
                    help="N > 1: split the config's slices over the ranks (strong scaling; one NCCL "
                         "all-reduce of B, H and two scalars per NMF iteration, NEXT-4) instead of replicas")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def max_over_ranks(x: float, world: int, device=None) -> float:
    """Max of a scalar over all ranks (NCCL on GPU, gloo on CPU)."""
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm_gbs=d.get("hbm_gbs", 6650.0), sm_max_mhz=d.get("sm_max_mhz", 1965.0),
                    source="measured (MEASURED_PEAKS.json)")
    return dict(hbm_gbs=6650.0, sm_max_mhz=1965.0, source="fallback (B200_PROFILING.md)")


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a moment to start: wait for its first sample so that the timed
            # region (which starts when this returns) is sampled from its beginning
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < 5.0:
                time.sleep(0.005)
        except Exception:
            self.proc = None
        self.k0 = len(self.lines)  # samples from here on fall inside the timed region
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            t0 = time.perf_counter()  # a very short timed region: take the next sample too
            while len(self.lines) <= self.k0 and time.perf_counter() - t0 < 0.1:
                time.sleep(0.002)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[getattr(self, "k0", 0):]:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def workload_desc(cfg, n_iter):
    return (f"C{cfg.idx}: {cfg.Nc}x{cfg.Nc}x{cfg.Nr} volume, {cfg.Nv} views over 180 deg, "
            f"Nk={cfg.Nk}, K={cfg.K}, {n_iter} NMF iterations, {cfg.M} materials, "
            f"Poisson {cfg.counts:g} counts/bin")


def config_dict(cfg, n_iter, world, shard=False):
    """The `config` object of BOTH arms' JSON lines (identical by construction)."""
    par = (f"slice-sharded x{world} (one all-reduce of B, H, 2 scalars per NMF iteration)" if shard
           else f"replicas x{world}")
    return {"workload": workload_desc(cfg, n_iter), "config_index": cfg.idx,
            "Nc": cfg.Nc, "Nr": cfg.Nr, "Nv": cfg.Nv, "Nk": cfg.Nk, "K": cfg.K,
            "n_iter": n_iter, "parallelism": par,
            "l2": f"inputs larger than L2 (Y = {4 * cfg.Np * cfg.Nk / 1e6:.0f} MB > 126 MB), no flush"}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------- CPU oracle
def oracle_sample(cfg, n_iter, nthreads=0, budget_s=12.0):
    """Bounded oracle sample of one step of config cfg, on the box's host cores.

    C1, C2 (one slice): the FULL step -- n_iter NMF iterations, FBP, synthesis of every bin --
    when it fits the budget (C1 always; C2 about 15-30 s), else as below.
    C3-C5: the slice-reduced problem synthdata.reduced(cfg, 2) (same N_v, N_c, N_k, K, counts:
    the per-element cost of every stage is shape-independent) -- as many NMF iterations as fit
    half the budget, FBP of both slices and synthesis of one slice x all bins -- each stage's
    time scaled by the fraction of the full step's work it did.
    Returns dict(t_full, t_sample, fraction, desc, threads)."""
    import oracle
    import synthdata as sd
    full_ok = cfg.Nr == 1 and cfg.Np * cfg.Nk * n_iter <= 2.5e10
    pc = cfg if full_ok else sd.reduced(cfg, min(cfg.Nr, 2))
    pr = sd.make_problem(pc)
    Y, V0, D0 = pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy()
    threads = nthreads or oracle.max_threads()
    t_all0 = time.perf_counter()
    if full_ok:
        it_s = n_iter
    else:
        t0 = time.perf_counter()
        oracle.nmf(Y, V0, D0, 1, nthreads=nthreads)
        t1 = time.perf_counter() - t0
        it_s = max(1, min(n_iter, int(0.5 * budget_s / max(t1, 1e-6))))
    t0 = time.perf_counter()
    V, D = oracle.nmf(Y, V0, D0, it_s, nthreads=nthreads)
    t_nmf = time.perf_counter() - t0
    f_nmf = (pc.Np * it_s) / (cfg.Np * n_iter)
    t0 = time.perf_counter()
    X = oracle.fbp(V, pc.Nv, pc.Nr, pc.Nc, nthreads=nthreads)
    t_fbp = time.perf_counter() - t0
    f_fbp = pc.Nr / cfg.Nr
    ns = 1 if not full_ok else pc.Nr
    t0 = time.perf_counter()
    oracle.synthesize(X, D, 0, ns, nthreads=nthreads)
    t_syn = time.perf_counter() - t0
    f_syn = ns / cfg.Nr
    t_sample = time.perf_counter() - t_all0
    t_full = t_nmf / f_nmf + t_fbp / f_fbp + t_syn / f_syn
    if full_ok:
        desc = (f"oracle (fp64 C, OpenMP, {threads} threads, {cpu_model()}): the full {cfg.name} step "
                f"({n_iter} NMF iterations, FBP, synthesis of all {cfg.Nk} bins), not extrapolated")
    else:
        desc = (f"oracle (fp64 C, OpenMP, {threads} threads, {cpu_model()}) on the slice-reduced {cfg.name} "
                f"problem (N_r = {pc.Nr}, same N_v/N_c/N_k/K): {it_s} of {n_iter} NMF iterations "
                f"({t_nmf / it_s:.3f} s/iter on {pc.Np} rows), FBP of {pc.Nr} slices, synthesis of {ns} slice; "
                f"each stage EXTRAPOLATED by its work fraction (NMF x{1 / f_nmf:.0f}, FBP x{1 / f_fbp:g}, "
                f"synthesis x{1 / f_syn:g}) to the full step")
    frac = t_sample / t_full
    return dict(t_full=t_full, t_sample=t_sample, fraction=frac, desc=desc, threads=threads,
                extrapolated=not full_ok)


def run_reference(args, cfg, n_iter, rank, world):
    if rank != 0:
        return 0
    for _ in range(args.warmup):
        pass  # the oracle has no warm-up state; warm-up steps are skipped deliberately
    samples = []
    t_start = time.perf_counter()
    for _ in range(args.steps):
        samples.append(oracle_sample(cfg, n_iter))
    wall = time.perf_counter() - t_start
    T_full = statistics.mean(s["t_full"] for s in samples)
    T_sample = statistics.mean(s["t_sample"] for s in samples)
    value = cfg.Nx * cfg.Nk / T_full
    smp = samples[-1]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            # a step is the bounded sample (its measured time); value is the full step's rate
            "ms_per_step": T_sample * 1e3, "full_step_ms_extrapolated": T_full * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Bragg-edge ellipse phantom, Poisson counts, -log)",
            "config": config_dict(cfg, n_iter, world, args.shard),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": smp["threads"], "kind": "oracle",
                             "sample": smp["desc"], "extrapolated": smp["extrapolated"],
                             "sample_fraction_of_step": smp["fraction"], "wall_s": wall},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------- GPU arm
def run_hsnct(args, cfg, n_iter, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import synthdata as sd
    from paper_2410_22500_b200 import Hsnct

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    peaks = load_peaks()

    # uint8 counts y, y0 as well (NEXT-1 extra; Y is their Eq. 2 decode, bit for bit)
    pr = sd.make_problem(cfg, device=dev, return_counts=not args.no_counts and not args.shard)
    Y, V0, D0 = pr["Y"], pr["V0"], pr["D0"]
    shard = args.shard  # at N = 1 the split iteration without a collective (a path check)
    gcfg = cfg  # the global workload (the metric counts its voxel*lambda)
    if shard:
        # this rank's slices [r0, r1): all views of them, local row order (v, r - r0, c); the
        # extras below (DHR, FMD, e2e, CPU baseline) are single-GPU measurements and skipped
        from paper_2410_22500_b200.sharded import slice_range, slice_rows
        r0, r1 = slice_range(cfg.Nr, rank, world)
        if world > 1:
            rows = slice_rows(cfg.Nv, cfg.Nr, cfg.Nc, r0, r1).to(dev)
            Y, V0 = Y.index_select(0, rows), V0.index_select(0, rows)
            pr["Y"], pr["V0"] = Y, V0
            torch.cuda.empty_cache()
        cfg = sd.reduced(cfg, r1 - r0)
        args.no_dhr = args.no_fmd = args.no_e2e = args.no_cpu = args.no_mbir = args.no_counts = True
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=local_rank)
    V = torch.empty_like(V0)
    D = torch.empty_like(D0)
    X = torch.empty((cfg.K, cfg.Nr, cfg.Nc, cfg.Nc), dtype=torch.float32, device=dev)
    # x^h: one window buffer reused across windows when the volume exceeds the budget
    win = max(1, min(cfg.Nr, (8 << 30) // (cfg.Nc * cfg.Nc * cfg.Nk * 4)))
    Xh = torch.empty((win * cfg.Nc * cfg.Nc, cfg.Nk), dtype=torch.float32, device=dev)
    import paper_2410_22500_b200.hsnct as hm
    ws_nmf = h.workspace(hm.OP_DECOMPOSE)
    ws_fbp = h.workspace(hm.OP_FBP)
    stream = torch.cuda.current_stream(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    red = torch.empty(h.nmf_red_size(), dtype=torch.float64, device=dev) if shard else None

    def step(rec=None):
        V.copy_(V0)
        D.copy_(D0)
        if rec is not None:
            rec[0].record(stream)
        if shard:
            from paper_2410_22500_b200.sharded import sharded_subspace_decompose
            sharded_subspace_decompose(h, Y, V, D, n_iter, ws=ws_nmf, red=red)
        else:
            h.subspace_decompose(Y, V, D, n_iter, ws=ws_nmf)
        if rec is not None:
            rec[1].record(stream)
        h.fbp(V, X, ws=ws_fbp)
        if rec is not None:
            rec[2].record(stream)
        for s0 in range(0, cfg.Nr, win):
            ns = min(win, cfg.Nr - s0)
            h.synthesize(X, D, s0, ns, 0, cfg.Nk, Xh=Xh[:ns * cfg.Nc * cfg.Nc])
        if rec is not None:
            rec[3].record(stream)

    for _ in range(args.warmup):
        step()
    h.sync()
    torch.cuda.synchronize()
    # events around the decompose call's input preparation and its iterations (the dominant
    # kernel's own launch), recorded on the launching stream inside the timed steps
    h.debug_nmf_timing(True)
    nmf_times = []
    recs = [[ev() for _ in range(4)] for _ in range(args.steps)]
    l0 = h.kernel_launches
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        e0, e1 = ev(), ev()
        e0.record(stream)
        for i in range(args.steps):
            step(recs[i])
            if not shard:
                nmf_times.append(h.debug_nmf_times())  # waits for the step (outside the device timing)
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = h.kernel_launches - l0
    h.sync()
    ms_total = e0.elapsed_time(e1)
    ms_step = max_over_ranks(ms_total / args.steps, world, dev)
    t_nmf = statistics.mean(r[0].elapsed_time(r[1]) for r in recs) * 1e-3
    t_fbp = statistics.mean(r[1].elapsed_time(r[2]) for r in recs) * 1e-3
    t_syn = statistics.mean(r[2].elapsed_time(r[3]) for r in recs) * 1e-3
    # replicas: every rank does the whole workload; sharded: the ranks share one workload
    value = gcfg.Nx * gcfg.Nk * (1 if shard else world) / (ms_step * 1e-3)

    # rooflines (algorithmic bytes)
    Np, Nk, K, Nx = cfg.Np, cfg.Nk, cfg.K, cfg.Nx
    nmf_bytes_iter = 4.0 * Np * Nk + 8.0 * Np * K
    nmf_gbs = nmf_bytes_iter * n_iter / t_nmf / 1e9
    syn_bytes = 4.0 * Nx * Nk + 4.0 * K * Nx
    syn_gbs = syn_bytes / t_syn / 1e9
    fbp_bytes = 4.0 * K * Np + 4.0 * K * Nx
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    plan = h.debug_plan()
    if os.path.exists(tp):
        tr = json.load(open(tp)).get(f"C{cfg.idx}", {})
        if tr.get("plan") == plan:
            traffic = tr.get("nmf_iter_dram_bytes")
    h.debug_nmf_timing(False)
    if nmf_times:  # the dominant kernel's own launch (all n_iter iterations), CUDA events
        t_prep = statistics.mean(t[0] for t in nmf_times) * 1e-3
        t_iters = statistics.mean(t[1] for t in nmf_times) * 1e-3
        kgbs = nmf_bytes_iter * n_iter / t_iters / 1e9
        kname = f"{plan} (the iterations' launch; input preparation {t_prep * 1e3:.1f} ms per call excluded)"
    else:  # sharded: the whole decompose call
        t_prep, t_iters, kgbs = None, None, nmf_gbs
        kname = f"subspace_decompose ({plan}; input preparation + G init once per call)"
    roof = {"bound": "hbm", "kernel": kname,
            "achieved": kgbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": kgbs / peaks["hbm_gbs"], "traffic": traffic,
            "algorithmic_bytes_per_unit": nmf_bytes_iter, "unit_of_work": "one NMF iteration",
            "units_per_launch": n_iter, "peak_source": peaks["source"]}
    if roof["frac"] > 1.0:
        # MEASURED_PEAKS' hbm_gbs is a copy (read + write) figure; the row pass is a pure read
        # stream, which HBM3e serves faster than a copy (ncu: 7.16 TB/s of DRAM reads for this
        # kernel at C5, profiles/r02/session4/ncu_mma_c5.txt)
        roof["note"] = ("frac > 1: the peak is the measured copy (read+write) bandwidth; a read-only stream "
                        "exceeds it (ncu DRAM read rate of this kernel: 7.16 TB/s)")
    stages = {"nmf_s": t_nmf, "nmf_per_iter_us": t_nmf / n_iter * 1e6, "fbp_s": t_fbp,
              "nmf_prep_s": t_prep, "nmf_iters_s": t_iters,
              "nmf_hbm_frac_incl_prep": nmf_gbs / peaks["hbm_gbs"],
              "synth_s": t_syn, "nmf_hbm_frac": kgbs / peaks["hbm_gbs"],
              "synth_hbm_frac": syn_gbs / peaks["hbm_gbs"],
              "fbp_hbm_frac": fbp_bytes / t_fbp / 1e9 / peaks["hbm_gbs"],
              "nmf_share_of_step": t_nmf / (ms_step * 1e-3)}

    # per-kernel FBP timing (outside the timed region): the ramp filter is bound by HBM, the
    # backprojection by the shared-memory crossbar (its staged detector windows)
    h.debug_fbp_timing(True)
    rt = []
    for _ in range(3):
        h.fbp(V, X, ws=ws_fbp)
        rt.append(h.debug_fbp_times())
    h.debug_fbp_timing(False)
    t_ramp = statistics.median(r[0] for r in rt) * 1e-3
    t_bp = statistics.median(r[1] for r in rt) * 1e-3
    kc = K if K <= 8 else 16
    ramp_bytes = 4.0 * K * Np + 4.0 * kc * Np                  # read V, write Q
    bp_smem_bytes = 2.0 * 4 * K * Nx * cfg.Nv                  # two detector samples per voxel, view, channel
    smem_peak = 148 * 128 * peaks["sm_max_mhz"] * 1e6 / 1e9    # GB/s: 128 B/clk/SM (B300_MICROARCH.md)
    fp32_peak = 148 * 128 * 2 * peaks["sm_max_mhz"] * 1e6 / 1e12  # TFLOP/s: 128 FMA/clk/SM
    P = 1 << max(1, (2 * cfg.Nc - 1).bit_length())
    ramp_flops = (cfg.Nv * cfg.Nr) * ((K + 1) // 2) * (2 * 5.0 * P * math.log2(P) + 2.0 * P)
    bp_fma = 2.0 * K * Nx * cfg.Nv
    stages.update({
        "ramp_s": t_ramp, "backproject_s": t_bp,
        "ramp_roofline": {"bound": "hbm", "achieved": ramp_bytes / t_ramp / 1e9, "peak": peaks["hbm_gbs"],
                          "unit": "GB/s", "frac": ramp_bytes / t_ramp / 1e9 / peaks["hbm_gbs"],
                          # the FFT arithmetic that actually bounds it: 5 P log2 P flop per complex
                          # transform, forward + inverse, one per channel pair and detector row,
                          # plus the real filter product; against the FP32 FMA peak
                          "alu_tflops": ramp_flops / t_ramp / 1e12, "alu_peak_tflops": fp32_peak,
                          "alu_frac": ramp_flops / t_ramp / 1e12 / fp32_peak},
        "backproject_roofline": {"bound": "smem", "achieved": bp_smem_bytes / t_bp / 1e9, "peak": smem_peak,
                                 "unit": "GB/s", "frac": bp_smem_bytes / t_bp / 1e9 / smem_peak,
                                 "fma_frac": bp_fma / t_bp / (fp32_peak * 0.5e12),
                                 "hbm_frac": (4.0 * kc * Np + 4.0 * K * Nx) / t_bp / 1e9 / peaks["hbm_gbs"],
                                 "peak_source": "148 SMs x 128 B/clk x max SM clock"},
        "synth_roofline": {"bound": "hbm", "achieved": syn_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                           "frac": syn_gbs / peaks["hbm_gbs"]},
    })

    # GPU DHR baseline on the same data (outside the timed region): EVERY bin of EVERY slice
    # (BASELINE config 5: "timed against GPU DHR (per-bin FBP over all 1600 bins) on the same
    # data"), written window by window into the x^h window buffer
    dhr = None
    if not args.no_dhr and rank == 0:
        ws_d = h.workspace(hm.OP_DHR, h.workspace_bytes(hm.OP_DHR) * min(cfg.Nr, 4))

        def dhr_all():
            for s0 in range(0, cfg.Nr, win):
                ns = min(win, cfg.Nr - s0)
                h.dhr(Y, s0, ns, 0, cfg.Nk, Xh=Xh[:ns * cfg.Nc * cfg.Nc], ws=ws_d)
        h.dhr(Y, 0, 1, 0, cfg.Nk, Xh=Xh[:cfg.Nc * cfg.Nc], ws=ws_d)  # warm-up
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record(stream)
        dhr_all()
        b.record(stream)
        torch.cuda.synchronize()
        t = a.elapsed_time(b) * 1e-3
        dhr = {"value": cfg.Nx * cfg.Nk / t, "unit": UNIT, "ms": t * 1e3,
               "sample": f"full volume: all {cfg.Nr} slices x {cfg.Nk} bins, one run after a one-slice warm-up",
               "fhr_over_dhr_time": (ms_step * 1e-3) / t}
        del ws_d

    # FMD back half (NEXT-2, outside the timed step): Eq. 7-9 on this step's X and D with the
    # phantom's pure-material regions as the user regions
    fmd = None
    if not args.no_fmd and rank == 0:
        nm = min(cfg.M, cfg.K)
        lab = torch.as_tensor(sd.region_labels(pr), dtype=torch.int32).to(dev).contiguous()
        # outputs and workspace allocated once, outside the timed call
        T = torch.empty((nm, cfg.K), dtype=torch.float32, device=dev)
        Xm = torch.empty((nm, cfg.Nr, cfg.Nc, cfg.Nc), dtype=torch.float32, device=dev)
        Dm = torch.empty((nm, cfg.Nk), dtype=torch.float32, device=dev)
        wsf = h.workspace(hm.OP_FMD)
        for _ in range(2):
            h.fmd_transform(X, lab, nm, T=T, ws=wsf)
            h.fmd_materials(X, T, Xm=Xm, ws=wsf)
            h.fmd_spectra(D, T, Dm=Dm)
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record(stream)
        h.fmd_transform(X, lab, nm, T=T, ws=wsf)
        h.fmd_materials(X, T, Xm=Xm, ws=wsf)
        h.fmd_spectra(D, T, Dm=Dm)
        b.record(stream)
        h.sync()
        t = a.elapsed_time(b) * 1e-3
        fmd = {"ms": t * 1e3, "voxels_per_s": cfg.Nx / t, "n_mat": nm,
               "note": "transform (Eq. 7) + per-voxel NNLS (Eq. 8) + spectra (Eq. 9), not in the metric"}
        del lab, Xm, Dm, T, wsf

    # MBIR of the subspace sinograms (NEXT-3, Eq. 5; outside the timed step and the metric):
    # hsnct_mbir from x0 = max(FBP, 0) of this step's V; per-iteration time from two call lengths,
    # the projector timed alone through hsnct_project (the same kernel and launch shape)
    mbir = None
    if not args.no_mbir and rank == 0 and args.mbir_iters > 1:
        nmb = args.mbir_iters
        wsm = h.workspace(hm.OP_MBIR)
        wsp = h.workspace(hm.OP_PROJECT)
        X0 = X.clamp(min=0)
        Xm = torch.empty_like(X0)
        Pm = torch.empty_like(V)
        # R26: sigma_v = 5% of the rms of V, sigma_x = 20% of the mean positive x0; svMBIR's
        # QGGMRF defaults p = 1.2, q = 2, T = 1 (the cost does not depend on the values)
        sv = 0.05 * float(V.double().pow(2).mean().sqrt())
        sx = 0.2 * float(X0[X0 > 0].double().mean()) if bool((X0 > 0).any()) else 1.0
        sx = sx if sx > 0 else 1.0

        def t_mbir(n):
            Xm.copy_(X0)
            torch.cuda.synchronize()
            a, b = ev(), ev()
            a.record(stream)
            h.mbir(V, Xm, n, sv, sx, ws=wsm)
            b.record(stream)
            h.sync()
            return a.elapsed_time(b) * 1e-3
        t_mbir(1)
        t1, tn = t_mbir(1), t_mbir(nmb)
        per = (tn - t1) / (nmb - 1)
        h.project(Xm, Pm, ws=wsp)
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record(stream)
        h.project(Xm, Pm, ws=wsp)
        b.record(stream)
        torch.cuda.synchronize()
        t_pr = a.elapsed_time(b) * 1e-3
        K = cfg.K
        kp = K + (K & 1)
        # the projector's shared-memory reads: 3 taps of kp floats per (bin, line, view, slice)
        pr_smem = 3.0 * 4 * kp * cfg.Nc * cfg.Nc * cfg.Nv * cfg.Nr
        smem_pk = 148 * 128 * peaks["sm_max_mhz"] * 1e6 / 1e9
        mbir = {"n_iter": nmb, "ms_per_iter": per * 1e3, "ms_total": tn * 1e3, "setup_ms": (t1 - per) * 1e3,
                "voxels_x_iter_per_s": K * cfg.Nx / per, "sigma_v": sv, "sigma_x": sx, "p": 1.2, "q": 2.0, "T": 1.0,
                "project_ms": t_pr * 1e3,
                "project_roofline": {"bound": "smem", "achieved": pr_smem / t_pr / 1e9, "peak": smem_pk,
                                     "unit": "GB/s", "frac": pr_smem / t_pr / 1e9 / smem_pk},
                "note": "x0 = max(FBP, 0); one iteration = projector (e = y - A x) + backprojector (A^T e) + SQS "
                        "update; not in the metric"}
        # the paper's Table II comparison on this data: FHR = NMF + N_s MBIR
        # reconstructions + expansion, DHR = N_k FBP reconstructions; all terms measured in this run
        # (MBIR at nmb SQS iterations from the FBP start); the per-bin-MBIR DHR is extrapolated
        # from the K-channel MBIR time by N_k / K (the MBIR kernels are linear in the channel count)
        if dhr is not None:
            fhr_mbir = stages["nmf_s"] + tn + stages["synth_s"]
            mbir["table2"] = {
                "fhr_mbir_s": fhr_mbir, "dhr_fbp_s": dhr["ms"] * 1e-3,
                "dhr_over_fhr_mbir": dhr["ms"] * 1e-3 / fhr_mbir,
                "dhr_mbir_s_extrapolated": tn * cfg.Nk / K,
                "dhr_mbir_over_fhr_mbir": tn * cfg.Nk / K / fhr_mbir,
                "paper": "Table II (simulated, hardware not stated): DHR (FBP per bin) 817.44 min, FHR (NMF + 9 MBIR "
                         "+ expansion) 62.96 min -> 13.0x",
                "note": f"FHR = this run's NMF ({n_iter} iterations) + MBIR of the K subspace sinograms ({nmb} SQS "
                        "iterations) + synthesis of all bins; DHR = the full-volume GPU DHR above"}
        del wsm, wsp, X0, Xm, Pm

    # counts-domain input (NEXT-1, outside the timed step): one-iteration decompositions from the
    # fp32 Y and from the uint8 counts (the input preparation is the only difference; results are
    # bit-identical), and the full decomposition from counts
    counts = None
    if not args.no_counts and rank == 0 and "y" in pr:
        yc, y0c = pr["y"], pr["y0"]

        def t_dec(fn, n):
            V.copy_(V0)
            D.copy_(D0)
            torch.cuda.synchronize()
            a, b = ev(), ev()
            a.record(stream)
            fn(n)
            b.record(stream)
            h.sync()
            return a.elapsed_time(b) * 1e-3
        f_y = lambda n: h.subspace_decompose(Y, V, D, n, ws=ws_nmf)  # noqa: E731
        f_c = lambda n: h.subspace_decompose_counts(yc, y0c, V, D, n, ws=ws_nmf)  # noqa: E731
        t_dec(f_c, 1)
        t1y, t1c = t_dec(f_y, 1), t_dec(f_c, 1)
        tfull = t_dec(f_c, n_iter)
        counts = {"decompose_1it_ms_fp32_input": t1y * 1e3, "decompose_1it_ms_counts_input": t1c * 1e3,
                  "prep_saving_ms": (t1y - t1c) * 1e3, "decompose_ms_counts_input": tfull * 1e3,
                  "input_bytes_fp32": 4 * cfg.Np * cfg.Nk, "input_bytes_counts": cfg.Np * cfg.Nk + cfg.Nr * cfg.Nc * cfg.Nk,
                  "note": "hsnct_subspace_decompose_counts: Eq. 2 decoded inside the Y+ preparation; the "
                          "iterations read the fp32 Y+ as before (bit-identical V, D)"}
        counts["note"] = ("hsnct_subspace_decompose_counts: Eq. 2 decoded inside the input preparation; the "
                          "iterations read the prepared operand as before (bit-identical V, D)")
        del yc, y0c
    # host copies of the counts for the counts-domain end-to-end line (NEXT-1 e2e)
    ych = (pr["y"].cpu(), pr["y0"].cpu()) if (not args.no_e2e and "y" in pr) else None
    pr.pop("y", None)
    pr.pop("y0", None)

    # end to end through the public API on page-locked HOST buffers (hsnct_fhr_stream): the
    # timed region holds, every step, the H2D copy of Y, V0, D0, the three stages, and the D2H
    # copy of ALL of x^h (window by window into a two-window host ring, overlapped with the
    # synthesis of the next window) plus V and D
    e2e = None
    e2e_ok = not args.no_e2e
    if e2e_ok:
        # host memory for the pinned copy of Y (and the counts, the ring): every local rank holds
        # its own; skip the end-to-end leg rather than drive the box out of memory
        try:
            import psutil
            local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
            need = 1.25 * Y.numel() * Y.element_size() + (4 << 30)
            avail = psutil.virtual_memory().available / max(1, local_world)
            if need > 0.9 * avail:
                e2e_ok = False
                sys.stderr.write(f"[bench] e2e skipped: needs {need / 2**30:.0f} GiB of host memory per rank, "
                                 f"{avail / 2**30:.0f} GiB available\n")
        except ImportError:
            pass
        if world > 1:  # one decision for all ranks (the leg has barriers)
            flag = torch.tensor([1 if e2e_ok else 0], dtype=torch.int32, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            e2e_ok = bool(flag.item())
    if e2e_ok:
        Yh = Y.cpu().pin_memory()
        V0h, D0h = V0.cpu().pin_memory(), D0.cpu().pin_memory()
        del Y, Xh, ws_nmf, ws_fbp
        pr.pop("Y", None)
        h.release_workspaces()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        wsl = h.fhr_stream_window_slices()
        ring = h.fhr_stream_ring(wsl)
        import paper_2410_22500_b200.hsnct as hm2
        ws_e = torch.empty(hm2.lib().hsnct_fhr_stream_bytes(h._h, wsl), dtype=torch.uint8, device=dev)
        Vh, Dh = torch.empty_like(V0h), torch.empty_like(D0h)
        got = [0]

        def on_window(s0, ns, xh):
            got[0] += ns

        h.fhr_stream(Yh, V0h, D0h, n_iter, window_slices=wsl, ring=ring, on_window=on_window, V=Vh, D=Dh,
                     ws=ws_e)  # warm-up
        n_e2e = max(1, min(args.steps, 2))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        got[0] = 0
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            h.fhr_stream(Yh, V0h, D0h, n_iter, window_slices=wsl, ring=ring, on_window=on_window, V=Vh, D=Dh,
                         ws=ws_e)
        t_e2e = max_over_ranks((time.perf_counter() - t0) / n_e2e, world, dev)
        assert got[0] == n_e2e * cfg.Nr
        e2e = {"value": cfg.Nx * cfg.Nk * world / t_e2e, "unit": UNIT,
               "h2d_bytes_per_step": 4 * (Np * Nk + Np * K + K * Nk),
               "d2h_bytes_per_step": 4 * (Nx * Nk + Np * K + K * Nk), "ms_per_step": t_e2e * 1e3,
               "steps": n_e2e, "window_slices": wsl,
               "path": "hsnct_fhr_stream (H2D, decompose, fbp, windowed synthesis + D2H into a pinned ring)",
               "timer": "host wall clock around the blocking call (max over ranks)"}
        del ws_e, Yh
        # the same end to end from the detector counts (hsnct_fhr_stream_counts): H2D of uint8 y, y0
        # (1 + 1/N_v bytes per element) instead of fp32 Y; Eq. 2 decoded on the device
        if ych is not None:
            yh, y0h = ych[0].pin_memory(), ych[1].pin_memory()
            ych = None
            ws_c = torch.empty(hm2.lib().hsnct_fhr_stream_counts_bytes(h._h, wsl), dtype=torch.uint8, device=dev)
            h.fhr_stream_counts(yh, y0h, V0h, D0h, n_iter, window_slices=wsl, ring=ring, on_window=on_window,
                                V=Vh, D=Dh, ws=ws_c)  # warm-up
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            got[0] = 0
            t0 = time.perf_counter()
            for _ in range(n_e2e):
                h.fhr_stream_counts(yh, y0h, V0h, D0h, n_iter, window_slices=wsl, ring=ring, on_window=on_window,
                                    V=Vh, D=Dh, ws=ws_c)
            t_c = max_over_ranks((time.perf_counter() - t0) / n_e2e, world, dev)
            assert got[0] == n_e2e * cfg.Nr
            e2e["counts_input"] = {
                "value": cfg.Nx * cfg.Nk * world / t_c, "unit": UNIT, "ms_per_step": t_c * 1e3,
                "h2d_bytes_per_step": Np * Nk + cfg.Nr * cfg.Nc * Nk + 4 * (Np * K + K * Nk),
                "d2h_bytes_per_step": 4 * (Nx * Nk + Np * K + K * Nk), "steps": n_e2e,
                "path": "hsnct_fhr_stream_counts (H2D of uint8 y, y0, Eq. 2 in the decomposition's input "
                        "preparation, then as hsnct_fhr_stream)"}
            del ws_c, yh, y0h
        del ring

    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:  # the CPU baseline: rank 0 at N = 1 only
        smp = oracle_sample(cfg, n_iter)
        cpu = {"value": cfg.Nx * cfg.Nk / smp["t_full"], "unit": UNIT, "cores": smp["threads"], "kind": "oracle",
               "sample": smp["desc"], "extrapolated": smp["extrapolated"], "sample_s": smp["t_sample"]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong" if shard else "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded Bragg-edge ellipse phantom, Poisson counts, -log)",
                "config": config_dict(gcfg, n_iter, world, shard),
                "roofline": roof, "stages": stages, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "gpu_dhr": dhr, "fmd": fmd, "mbir": mbir, "counts": counts, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    import synthdata as sd
    cfg = sd.CONFIGS[args.config]
    n_iter = args.n_iter if args.n_iter is not None else cfg.n_iter
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        return run_reference(args, cfg, n_iter, rank, world)
    return run_hsnct(args, cfg, n_iter, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
