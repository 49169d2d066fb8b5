#!/usr/bin/env python
"""Benchmark of the hot path (BASELINE.json metric) on synthetic C5 inputs.

One step = one whole time-to-solution of config C5 (1024^2 P1 grid, k = 400,
32 strips, l = 1, t = 4 double sweeps LRL+RLR+BTB+TBT, MPGMRES to 1e-6):
helm_assemble -> sweep_setup x 4 -> mpgmres_solve (every iteration: sources,
one batched 4-direction sweep_apply launch, SpMM, BCGS2 + block QR, host LSQ)
-> x.  `value` = sweep-preconditioner applies per second over the whole step
(t x iterations / step time, setup included); ms_per_step is the
time-to-solution.  Inputs (c, f) are resident in HBM when the timed region
starts; the two factor sets (one per strip axis, shared by LRL/RLR and
BTB/TBT) are GBs, far larger than the 126 MB L2, so no explicit flush.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 5]

N > 1 (torchrun): independent replicas per rank ("replicas only", DESIGN.md
§8; scaling weak), timed by CUDA events, max over ranks.
--impl reference: the CPU oracle (oracle/) timed on this host; one step =
one batched t = 4 sweep apply of the same C5 workload (measured, no
extrapolation; factor sets built before timing).
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sweep-precond applies/s + MPGMRES time-to-solve; HBM GB/s as % of peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-north-star", action="store_true")
    ap.add_argument("--clock-interval-ms", type=int, default=50, help="nvidia-smi sampling period during the timed region")
    ap.add_argument("--mode", default="replicas", choices=["replicas", "directions"],
                    help="N > 1: independent replicas per rank (default), or the direction-parallel "
                         "solve (mpgmres_solve_dist: the t directions split over the ranks of a group, "
                         "NCCL all-gather of the new columns each iteration)")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0, interval_ms=50):
        self.index = index
        self.interval_ms = int(interval_ms)
        self.proc = None
        self.lines = []          # (host time, csv line)
        self.window = None       # (t0, t1) of the timed region

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.interval_ms)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        # let the exit of the nvidia-smi client settle before anything else is timed
        time.sleep(0.5)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if self.window is not None:
            inside = [(t, ln) for t, ln in lines if self.window[0] <= t <= self.window[1]]
            lines = inside if inside else lines[-1:]
        for _, ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def reduce_over_ranks(local_ms, local_applies, pg=None, dev=None):
    """Replicas: the job's time is the MAX of the per-rank device times, its
    work the SUM of the per-rank applies (each rank solves its own copy)."""
    if pg is None:
        return float(local_ms), int(local_applies)
    import torch
    tt = torch.tensor([float(local_ms)], dtype=torch.float64, device=dev)
    aa = torch.tensor([int(local_applies)], dtype=torch.int64, device=dev)
    pg.all_reduce(tt, op=pg.ReduceOp.MAX)
    pg.all_reduce(aa, op=pg.ReduceOp.SUM)
    return float(tt.item()), int(aa.item())


def run_ours(args):
    import numpy as np
    import torch

    import paper_2408_11929_b200 as hs
    from helm_inputs import make_config

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    cfg = make_config(args.config)
    names = cfg.dirs
    t = len(names)
    dp = direction_groups(args, ws, rank, t, pg)       # None: replicas
    my_names = names if dp is None else hs.partition_directions(names, dp["size"])[dp["rank"]]
    c_dev = torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev)
    f_dev = torch.tensor(cfg.f.ravel(), dtype=torch.complex128, device=dev)
    b = torch.zeros(cfg.n, dtype=torch.complex128, device=dev)
    x = torch.zeros(cfg.n, dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)

    last = {}
    # one stream per strip axis: the x- and y-strip factorisations run concurrently
    setup_streams = {0: torch.cuda.Stream(dev).cuda_stream, 1: torch.cuda.Stream(dev).cuda_stream}

    def step():
        prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, c_dev)
        t0 = time.perf_counter()
        dirs = hs.make_sweeps(prob, my_names, n_strips=cfg.n_strips, overlap=cfg.overlap, streams=setup_streams)
        t1 = time.perf_counter()
        prob.load_vector(f_dev, b)
        if dp is None:
            _, st = hs.mpgmres_solve(prob, dirs, b, x, tol=cfg.tol, maxit=cfg.maxit)
        else:
            _, st = hs.mpgmres_solve_dist(prob, dirs, dp["size"], dp["rank"], b, x, dp["cb"], tol=cfg.tol,
                                          maxit=cfg.maxit)
        last.update(st=st, setup_s=t1 - t0, dirs_info=[d.info() for d in dirs])
        return st

    # the clock sampler runs from before the warm-up; only its samples inside the
    # timed region are reported
    gc.collect()
    sampler = ClockSampler(local, args.clock_interval_ms)
    sampler.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    l0 = hs.kernel_launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()   # no cyclic collection inside the timed region (as timeit does); refcount frees still run
    tw0 = time.monotonic()
    ev0.record(stream)
    its, sweep_ms, spmv_ms, orth_ms, setup_s = [], 0.0, 0.0, 0.0, 0.0
    for _ in range(args.steps):
        st = step()
        its.append(st["iterations"])
        sweep_ms += st["sweep_ms"]
        spmv_ms += st["spmv_ms"]
        orth_ms += st["orth_ms"]
        setup_s += last["setup_s"]
    ev1.record(stream)
    torch.cuda.synchronize()
    gc.enable()
    sampler.mark(tw0, time.monotonic())
    launches = hs.kernel_launches() - l0
    clocks = sampler.stop()
    # replicas: each rank's solve applies t preconditioners per iteration; direction-
    # parallel: a group's solve applies t per iteration, t / size of them on each rank
    local_t = t if dp is None else len(my_names)
    total_ms, applies = reduce_over_ranks(ev0.elapsed_time(ev1), sum(its) * local_t, pg, dev)
    value = applies / (total_ms / 1e3)
    ms_step = total_ms / args.steps
    st = last["st"]
    # roofline of the dominant kernel (k_sweep_apply, one launch per iteration)
    model_bytes = sum(i.model_bytes_per_apply for i in last["dirs_info"])
    n_sweeps = sum(its)
    avg_sweep_ms = sweep_ms / max(n_sweeps, 1)
    achieved = model_bytes / (avg_sweep_ms / 1e3) / 1e9
    peak, peak_kind = measured_peaks()
    traffic = None
    tp = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            tr = json.load(fh)
        if tr.get("config") == cfg.name:
            traffic = tr.get("dram_bytes_per_launch")
    out = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "applies/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 3),
        "higher_is_better": True,
        "scaling": "strong" if (dp is not None and dp["size"] == ws) else "weak",
        "vs_baseline": None,
        "dtype": "c128 (f64 complex)",
        "data": "synthetic (helm_inputs seeded recipe of " + cfg.name + ")",
        "config": {"workload": f"{cfg.name}: P1 {cfg.nx}x{cfg.ny} k={cfg.omega:g}, N={cfg.n_strips} strips l={cfg.overlap}, "
                               f"t={t} ({'+'.join(names)}), MPGMRES tol {cfg.tol:g}, x0=0; step = assemble + "
                               "4 sweep setups + solve",
                   "n_unknowns": cfg.n,
                   "parallelism": ("single GPU" if ws == 1 else f"replicas x{ws}" if dp is None else
                                   f"direction-parallel: {ws // dp['size']} group(s) of {dp['size']} ranks "
                                   f"x {t // dp['size']} direction(s), NCCL all-gather of Z and AZ per iteration"),
                   "l2_policy": "no flush: two factor sets (x / y strips) of %.2f GB in all >> 126 MB L2" % (
                       sum({i.axis: i.factor_bytes for i in last["dirs_info"]}.values()) / 1e9)},
        "time_to_solution_ms": round(ms_step, 3),
        "iterations": its[-1],
        "setup_ms_avg": round(setup_s / args.steps * 1e3, 3),
        "sweep_apply_ms_avg": round(avg_sweep_ms, 4),
        "spmm_ms_avg": round(spmv_ms / max(n_sweeps, 1), 4),
        "orth_ms_avg": round(orth_ms / max(n_sweeps, 1), 4),
        "true_rel_res": st["true_rel_res"],
        "roofline": {"kernel": hs.sweep_kernel_name() + " (t=4 batched double sweeps, one cooperative launch per iteration)",
                     "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "model_bytes_per_launch": model_bytes,
                     "model": "SURVEY 8(d): sum over local solves of 16(2 n_c w^2 + 3 n_c w)"},
        "setup_roofline": (lambda fl: {
            "bound": "fp64", "achieved": round(fl / (setup_s / args.steps) / 1e12, 2), "peak": FP64_PEAK_TFLOPS,
            "unit": "TFLOP/s", "frac": round(fl / (setup_s / args.steps) / 1e12 / FP64_PEAK_TFLOPS, 4),
            "flops_per_step": fl, "peak_source": "measured FP64 FMA throughput, tools/bench_fp64 (profiles/r02_fp64_peak.txt)",
            "model": "both axes: sum over strips of 8 w^3 (3 n_c + 4 K + K (K-1)); setup wall time of the step's sweep_setup calls"})(
            setup_flops(cfg, last["dirs_info"][0].n_segments)),
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if not args.no_north_star and ws == 1:
        out["north_star"] = north_star_kernels(cfg, names, peak)
    if not args.no_e2e:
        e2e = run_e2e(args, cfg, names, my_names, dp)
        # replicas: the job's end-to-end time is the max over ranks, its work the sum
        e_ms, e_app = reduce_over_ranks(e2e.pop("_ms_total"), e2e.pop("_applies"), pg, dev)
        e2e["value"] = round(e_app / (e_ms / 1e3), 3)
        e2e["ms_per_step"] = round(e_ms / args.steps, 3)
        out["e2e"] = e2e
    if rank == 0 and not args.no_cpu_baseline and ws == 1:
        out["cpu_baseline"] = oracle_baseline(cfg, names)
    if rank == 0:
        print(json.dumps(out))
    if pg:
        pg.barrier()
        pg.destroy_process_group()


FP64_PEAK_TFLOPS = 34.1   # measured: tools/bench_fp64 on this pool's B200 (profiles/r02_fp64_peak.txt)


def setup_flops(cfg, n_segments):
    """Algorithmic FP64 flops of the strip factorisations (sweep_setup) of BOTH
    strip axes, complex multiply-add = 8 flops (DESIGN.md §5 "Setup"):
      rows        n_c x (inverse S_c^-1, 8 w^3; bottom-up inverse, 8 w^3; the
                  X[lo][hi] chain product, 8 w^3)                 = 24 w^3 n_c
      separators  K x (Schur update, inverse, G_k, F_k: 4 x 8 w^3)  = 32 w^3 K
      explicit R^-1 rows  K (K - 1) block products                 =  8 w^3 K (K - 1)
    summed over the strips' widths w (interior strips cells + 2l + 1 nodes)."""
    total = 0.0
    for axis in (0, 1):
        n_axis = cfg.nx if axis == 0 else cfg.ny
        nc = (cfg.ny if axis == 0 else cfg.nx) + 1
        base, extra = divmod(n_axis, cfg.n_strips)
        p = [0]
        for s in range(cfg.n_strips):
            p.append(p[-1] + base + (1 if s < extra else 0))
        K = n_segments - 1
        for s in range(cfg.n_strips):
            a, b = max(p[s] - cfg.overlap, 0), min(p[s + 1] + cfg.overlap, n_axis)
            w = b - a + 1
            total += 8.0 * w ** 3 * (3 * nc + 4 * K + K * (K - 1))
    return total


def direction_groups(args, ws, rank, t, pg):
    """--mode directions: ranks form groups of `size` = the largest divisor of t
    that divides ws (<= t); each group solves the problem with its directions
    split over its ranks (mpgmres_solve_dist), the groups are replicas."""
    if args.mode != "directions" or ws == 1:
        return None
    import paper_2408_11929_b200 as hs
    size = max(d for d in range(1, t + 1) if t % d == 0 and ws % d == 0)
    groups = [pg.new_group(ranks=list(range(g0, g0 + size))) for g0 in range(0, ws, size)]
    grp = groups[rank // size]
    return {"size": size, "rank": rank % size, "group": grp, "cb": hs.torch_allgather(grp)}


def run_e2e(args, cfg, names, my_names=None, dp=None):
    """Same metric through the C ABI with HOST buffers: pinned host c and f are
    copied in, x is copied back, every step, inside the timed region.  Same
    --warmup / --steps as the device arm; timed with CUDA events on the
    launching stream, synchronised on both sides (x is on the host at the end)."""
    import torch

    import paper_2408_11929_b200 as hs

    t = len(names)
    c_h = torch.tensor(cfg.c.ravel(), dtype=torch.float64).pin_memory()
    f_h = torch.tensor(cfg.f.ravel(), dtype=torch.complex128).pin_memory()
    x_h = torch.zeros(cfg.n, dtype=torch.complex128).pin_memory()
    b_d = torch.zeros(cfg.n, dtype=torch.complex128, device="cuda")
    stream = torch.cuda.current_stream()
    setup_streams = {0: torch.cuda.Stream().cuda_stream, 1: torch.cuda.Stream().cuda_stream}

    my_names = my_names or names

    def step():
        prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, c_h.numpy())
        # b = M1 f needs only the grid: issued before the setups, so that the host-to-device
        # copy of f runs beside the factorisation kernels of the setup streams
        prob.load_vector(f_h.numpy(), b_d)
        dirs = hs.make_sweeps(prob, my_names, n_strips=cfg.n_strips, overlap=cfg.overlap, streams=setup_streams)
        if dp is None:
            _, st = hs.mpgmres_solve(prob, dirs, b_d, x_h.numpy(), tol=cfg.tol, maxit=cfg.maxit)
        else:
            _, st = hs.mpgmres_solve_dist(prob, dirs, dp["size"], dp["rank"], b_d, x_h.numpy(), dp["cb"],
                                          tol=cfg.tol, maxit=cfg.maxit)
        return st["iterations"]

    for _ in range(args.warmup):
        step()
    gc.collect()
    gc.disable()   # no cyclic collection inside the timed region (as timeit does); refcount frees still run
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record(stream)
    its, step_wall = [], []
    for _ in range(args.steps):
        s0 = time.perf_counter()
        its.append(step())
        step_wall.append(round(1e3 * (time.perf_counter() - s0), 2))
    e1.record(stream)
    torch.cuda.synchronize()
    gc.enable()
    wall = time.perf_counter() - w0
    ms = e0.elapsed_time(e1)
    return {"_ms_total": ms, "_applies": sum(its) * len(my_names), "unit": "applies/s",
            "h2d_bytes_per_step": 8 * cfg.n + 16 * cfg.n, "d2h_bytes_per_step": 16 * cfg.n,
            "host_wall_ms_per_step": round(wall / len(its) * 1e3, 3), "host_wall_ms_each_step": step_wall,
            # isolated host-side stalls (one step of 10-300 ms in ~3% of the steps on this pool's boxes,
            # DESIGN.md §7) inflate the mean; `value` stays the mean over all K steps
            "host_wall_ms_median_step": round(sorted(step_wall)[len(step_wall) // 2], 2),
            "steps": len(its), "warmup": args.warmup,
            "path": "helm_assemble(host c) + helm_load_vector(host f) + sweep_setup x4 + mpgmres_solve(x to host)"}


def north_star_kernels(cfg, names, peak):
    """The north star's per-kernel numbers on this config, measured with CUDA
    events on the launching stream (warm, 2 warm-up + 10 timed launches each):
    SpMV (1 column) and SpMM (t = 4) against the SURVEY 8(d) byte model
    16 nnz + 2 t 16 n, and the batched sweep apply at t = 1 (LRL), 2 (+BTB),
    4 (+RLR, TBT) as applies/s and model GB/s.  Inputs exceed L2 (factor sets
    of GBs; the SpMM's 252 MB > 126 MB)."""
    import torch

    import paper_2408_11929_b200 as hs
    from helm_inputs import random_vector

    dev = torch.device("cuda")
    stream = torch.cuda.current_stream()
    prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev))
    dirs = dict(zip(names, hs.make_sweeps(prob, names, n_strips=cfg.n_strips, overlap=cfg.overlap)))
    # a batch of fewer directions leaves SMs free for more, shorter segments (P CTAs per
    # direction): measured best P for C5 is 49 at t = 1, 41 at t = 2, 36 at t = 4
    # (DESIGN.md §5); the t = 4 handles above use the automatic 36
    seg_for_t = {1: 49, 2: 41}
    extra = {t_: dict(zip(names[:1] if t_ == 1 else ["LRL", "BTB"],
                          hs.make_sweeps(prob, ["LRL"] if t_ == 1 else ["LRL", "BTB"], n_strips=cfg.n_strips,
                                         overlap=cfg.overlap, n_segments=seg_for_t[t_])))
             for t_ in seg_for_t} if cfg.n_strips > 1 and cfg.nx >= 512 else {}
    # assembled nonzeros of the 7-point P1 stencil on the grid (7,346,177 for C5)
    nx, ny = cfg.nx, cfg.ny
    nnz = (nx + 1) * (ny + 1) + 2 * (nx * (ny + 1) + (nx + 1) * ny + nx * ny)

    def timed(fn, reps=10, warm=2):
        for _ in range(warm):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    out = {"nnz": nnz}
    for ncol in (1, 4):
        X = torch.tensor(random_vector(cfg.n, 5, ncol), device=dev)
        Y = torch.zeros_like(X)
        ms = timed(lambda: prob.spmv(X, Y, ncol), reps=50)
        model = 16 * nnz + 2 * ncol * 16 * cfg.n
        out["spmv" if ncol == 1 else "spmm_t4"] = {
            "ms": round(ms, 5), "model_bytes": model, "achieved_gbs": round(model / (ms / 1e3) / 1e9, 1),
            "frac_of_peak": round(model / (ms / 1e3) / 1e9 / peak, 4)}
    r = torch.tensor(random_vector(cfg.n, 6), device=dev)
    for combo in (["LRL"], ["LRL", "BTB"], ["LRL", "RLR", "BTB", "TBT"]):
        src = extra.get(len(combo), dirs)
        ds = [src[nm] for nm in combo]
        Z = torch.zeros((len(ds), cfg.n), dtype=torch.complex128, device=dev)
        ms = timed(lambda: hs.sweep_apply(ds, r, Z, ldr=0), reps=10)
        model = sum(d.info().model_bytes_per_apply for d in ds)
        out[f"sweep_apply_t{len(ds)}"] = {
            "dirs": "+".join(combo), "ms": round(ms, 4), "applies_per_s": round(len(ds) / (ms / 1e3), 1),
            "model_bytes": model, "achieved_gbs": round(model / (ms / 1e3) / 1e9, 1),
            "frac_of_peak": round(model / (ms / 1e3) / 1e9 / peak, 4), "kernel": hs.sweep_kernel_name(),
            "segments": ds[0].info().n_segments}
    # opt-in inexact separator solve (sweep_set_precision(32), not the headline: the
    # preconditioner is then ~1e-7 off the exact strip solves; x stays complex128)
    ds = [dirs[nm] for nm in names]
    Z = torch.zeros((len(ds), cfg.n), dtype=torch.complex128, device=dev)
    b = torch.zeros(cfg.n, dtype=torch.complex128, device=dev)
    prob.load_vector(torch.tensor(cfg.f.ravel(), dtype=torch.complex128, device=dev), b)
    x64 = torch.zeros_like(b)
    _, st64 = hs.mpgmres_solve(prob, ds, b, x64, tol=cfg.tol, maxit=cfg.maxit)
    for d in ds:
        d.set_precision(32)
    ms32 = timed(lambda: hs.sweep_apply(ds, r, Z, ldr=0), reps=10)
    x32 = torch.zeros_like(b)
    _, st32 = hs.mpgmres_solve(prob, ds, b, x32, tol=cfg.tol, maxit=cfg.maxit)
    for d in ds:
        d.set_precision(64)
    out["inexact_separator_fp32"] = {
        "sweep_apply_t4_ms": round(ms32, 4), "applies_per_s": round(len(ds) / (ms32 / 1e3), 1),
        "iterations": st32["iterations"], "iterations_exact": st64["iterations"],
        "true_rel_res": st32["true_rel_res"],
        "x_rel_diff_vs_exact": float(torch.linalg.norm(x32 - x64) / torch.linalg.norm(x64)),
        "what": "opt-in sweep_set_precision(32): complex64 separator-inverse rows, FP32 separator mat-vec"}
    return out


def host_info():
    """Host description for the CPU numbers."""
    info = {"os_cpu_count": os.cpu_count()}
    try:
        info["nproc"] = len(os.sched_getaffinity(0))
    except Exception:
        info["nproc"] = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        from threadpoolctl import threadpool_info
        info["blas"] = [{k: d.get(k) for k in ("internal_api", "num_threads")} for d in threadpool_info()]
    except Exception:
        info["blas"] = None
    info["OMP_NUM_THREADS"] = os.environ.get("OMP_NUM_THREADS")
    return info


def oracle_baseline(cfg, names):
    """The CPU oracle as it stands, timed on this host on a bounded sample of
    the same workload, measured (not extrapolated): the C5 assembly, the
    splu factor set of the x strips (LRL's 32 strips), and one full LRL double
    sweep (2N - 1 = 63 strip solves).  `value` is the oracle's measured apply
    rate (applies/s, factor set built); its setup times are reported beside it."""
    from helm_inputs import random_vector
    from oracle import p1, sweep

    t0 = time.perf_counter()
    A = p1.assemble(cfg)
    t_asm = time.perf_counter() - t0
    t1 = time.perf_counter()
    P = sweep.make_preconditioner(cfg, A, names[0])
    t_fac = time.perf_counter() - t1
    r = random_vector(cfg.n, 77)
    t2 = time.perf_counter()
    c2 = time.process_time()
    P.apply(r)
    t_apply = time.perf_counter() - t2
    cores = (time.process_time() - c2) / t_apply   # threads actually busy (process CPU time / wall)
    sample_s = time.perf_counter() - t0
    return {"value": round(1.0 / t_apply, 4), "unit": "applies/s", "cores": round(cores, 2), "kind": "oracle",
            "sample": f"{cfg.name}: oracle assembly ({t_asm:.1f} s) + splu of the {cfg.n_strips} x-strips "
                      f"({t_fac:.1f} s) + one {names[0]} double sweep of {2 * cfg.n_strips - 1} strip solves "
                      f"({t_apply:.2f} s); {sample_s:.1f} s of CPU work in all, single process",
            "oracle_apply_s": round(t_apply, 3), "oracle_assembly_s": round(t_asm, 3),
            "oracle_factor_one_axis_s": round(t_fac, 3), "host": host_info()}


def _ref_worker_init(cfg_num, name):
    global _REF_P, _REF_R
    from helm_inputs import make_config, random_vector
    from oracle import p1, sweep
    cfg = make_config(cfg_num)
    A = p1.assemble(cfg)
    _REF_P = sweep.make_preconditioner(cfg, A, name)
    _REF_R = random_vector(cfg.n, 78)


def _ref_worker_apply(_):
    t0 = time.perf_counter()
    _REF_P.apply(_REF_R)
    return time.perf_counter() - t0


def run_reference(args):
    """The reference arm: the CPU oracle (oracle/, numpy/scipy splu) as it
    stands, on this host, on the same config / metric / unit.  Untimed
    preparation: assembly and the splu factor sets of both strip axes.  One
    step = one batched t = 4 sweep apply (LRL, RLR, BTB, TBT, each 2N - 1
    strip solves), applied one after another as in the paper's serial MATLAB
    runs.  value = t / step time (applies/s).  Also measured: the
    t-process mode (a pool of t worker processes, one direction each, "applied
    in parallel").  Under torchrun only rank 0 runs."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from helm_inputs import make_config, random_vector
    from oracle import p1, sweep
    cfg = make_config(args.config)
    names = cfg.dirs
    t = len(names)
    tp0 = time.perf_counter()
    A = p1.assemble(cfg)
    t_asm = time.perf_counter() - tp0
    tf0 = time.perf_counter()
    precs = sweep.make_preconditioners(cfg, A, names)
    t_fac = time.perf_counter() - tf0
    r = random_vector(cfg.n, 78)

    def step():
        for P in precs:
            P.apply(r)

    for _ in range(args.warmup):
        step()
    times = []
    cpu0 = time.process_time()
    for _ in range(args.steps):
        s0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - s0)
    cores = (time.process_time() - cpu0) / sum(times)   # threads actually busy (process CPU time / wall)
    ms = 1e3 * sum(times) / len(times)
    value = t / (ms / 1e3)
    del precs
    # t-process mode: one worker per direction, the t applies run concurrently
    par = None
    try:
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor
        ctx = mp.get_context("fork")
        pools = [ProcessPoolExecutor(1, mp_context=ctx, initializer=_ref_worker_init, initargs=(args.config, nm))
                 for nm in names]
        w0 = time.perf_counter()
        for f in [pl.submit(_ref_worker_apply, 0) for pl in pools]:
            f.result()          # first call includes each worker's setup
        t_par_setup = time.perf_counter() - w0
        pt = []
        for _ in range(args.steps):
            s0 = time.perf_counter()
            for f in [pl.submit(_ref_worker_apply, 0) for pl in pools]:
                f.result()
            pt.append(time.perf_counter() - s0)
        for pl in pools:
            pl.shutdown()
        par = {"value": round(t / (sum(pt) / len(pt)), 4), "unit": "applies/s", "processes": t,
               "ms_per_step": round(1e3 * sum(pt) / len(pt), 1), "setup_plus_first_apply_s": round(t_par_setup, 1)}
    except Exception as e:  # pragma: no cover - host without fork / memory
        par = {"unavailable": str(e)[:200]}
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "applies/s", "n_gpus": ws,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 1),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64 complex)",
           "data": "synthetic (helm_inputs seeded recipe of " + cfg.name + ")",
           "config": {"workload": f"{cfg.name}: P1 {cfg.nx}x{cfg.ny} k={cfg.omega:g}, N={cfg.n_strips} strips "
                                  f"l={cfg.overlap}, t={t} ({'+'.join(names)}); CPU oracle (numpy/scipy splu); "
                                  "step = one batched t-direction sweep apply, factor sets built before timing",
                      "n_unknowns": cfg.n},
           "cpu_baseline": {"value": round(value, 5), "unit": "applies/s", "cores": round(cores, 2), "kind": "oracle",
                            "sample": f"per step: {t} double sweeps x {2 * cfg.n_strips - 1} strip solves on the full "
                                      f"{cfg.name} grid, serial (paper-like, P:L241); untimed preparation: assembly "
                                      f"{t_asm:.1f} s + splu factor sets of both axes {t_fac:.1f} s",
                            "host": host_info()},
           "t_process_mode": par,
           "oracle_setup_s": {"assembly": round(t_asm, 2), "factor_both_axes": round(t_fac, 2)},
           "e2e": {"value": round(value, 5), "unit": "applies/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
