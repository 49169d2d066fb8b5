"""Round report (SURVEY §8(d) "What to report"): per config and per t, the
sweep applies/s and model GB/s (% of the measured HBM peak), SpMV/SpMM time and
model GB/s, MPGMRES iterations, setup and solve time.  Markdown on stdout.

  python tools/report.py [--configs 1,2,3,4,5] [--reps 5]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2408_11929_b200 as hs
from helm_inputs import make_config

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3,4,5")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(root, "MEASURED_PEAKS.json")) else 6650.0
dev = torch.device("cuda:0")
TS = {1: ["LRL"], 2: ["LRL", "BTB"], 4: ["LRL", "RLR", "BTB", "TBT"]}


def timed(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


print(f"peak HBM (MEASURED_PEAKS.json): {peak} GB/s\n")
print("| cfg | n | t | kernel | apply ms | applies/s | model GB/s | % peak | SpMM(t) us | SpMM GB/s | its | setup ms | solve ms |")
print("|---|---:|---:|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|")
for c in [int(x) for x in a.configs.split(",")]:
    cfg = make_config(c)
    for t in (1, 2, 4):
        if t > len(cfg.dirs) and t != 4:
            pass
        names = TS[t] if t < 4 else cfg.dirs if len(cfg.dirs) == 4 else None
        if names is None:
            continue
        prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev))
        # setup and solve are timed on their second call (the first one pays module
        # loading and the Krylov workspace allocation)
        for _ in range(2):
            dirs = None
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dirs = hs.make_sweeps(prob, names, n_strips=cfg.n_strips, overlap=cfg.overlap)
            torch.cuda.synchronize()
            setup_ms = (time.perf_counter() - t0) * 1e3
        r = torch.randn(cfg.n, dtype=torch.complex128, device=dev)
        Z = torch.zeros((t, cfg.n), dtype=torch.complex128, device=dev)
        ms = timed(lambda: hs.sweep_apply(dirs, r, Z, ldr=0), a.reps)
        kern = hs.sweep_kernel_name()
        model = sum(d.info().model_bytes_per_apply for d in dirs)
        X = torch.randn((t, cfg.n), dtype=torch.complex128, device=dev)
        Y = torch.zeros_like(X)
        sp_ms = timed(lambda: prob.spmv(X, Y, ncols=t), 20)
        sp_bytes = 16 * 4 * cfg.n + 2 * t * 16 * cfg.n   # 4 stored diagonals + t columns in and out
        b = torch.zeros(cfg.n, dtype=torch.complex128, device=dev)
        prob.load_vector(torch.tensor(cfg.f.ravel(), device=dev), b)
        for _ in range(2):
            x = torch.zeros(cfg.n, dtype=torch.complex128, device=dev)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            _, st = hs.mpgmres_solve(prob, dirs, b, x, tol=cfg.tol, maxit=cfg.maxit)
            torch.cuda.synchronize()
            solve_ms = (time.perf_counter() - t1) * 1e3
        gbs = model / ms / 1e6
        print(f"| {cfg.name} | {cfg.n} | {t} | {kern} | {ms:.3f} | {t * 1e3 / ms:.1f} | {gbs:.0f} | {gbs / peak * 100:.1f} | "
              f"{sp_ms * 1e3:.1f} | {sp_bytes / sp_ms / 1e6:.0f} | {st['iterations']} | {setup_ms:.1f} | {solve_ms:.1f} |",
              flush=True)
        del dirs, prob
