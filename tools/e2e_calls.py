"""The e2e step of bench.py (host buffers, no synchronisation between the calls)
with a host timer around every call: which call do the isolated stalls sit in?"""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2408_11929_b200 as hs
from helm_inputs import make_config

cfg = make_config(5)
names = cfg.dirs
c_h = torch.tensor(cfg.c.ravel(), dtype=torch.float64).pin_memory()
f_h = torch.tensor(cfg.f.ravel(), dtype=torch.complex128).pin_memory()
x_h = torch.zeros(cfg.n, dtype=torch.complex128).pin_memory()
b_d = torch.zeros(cfg.n, dtype=torch.complex128, device="cuda")
streams = {0: torch.cuda.Stream().cuda_stream, 1: torch.cuda.Stream().cuda_stream}
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200


def step():
    T = []
    t = time.perf_counter()
    prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, c_h.numpy())
    T.append(time.perf_counter() - t); t = time.perf_counter()
    dirs = hs.make_sweeps(prob, names, n_strips=cfg.n_strips, overlap=cfg.overlap, streams=streams)
    T.append(time.perf_counter() - t); t = time.perf_counter()
    prob.load_vector(f_h.numpy(), b_d)
    T.append(time.perf_counter() - t); t = time.perf_counter()
    _, st = hs.mpgmres_solve(prob, dirs, b_d, x_h.numpy(), tol=cfg.tol, maxit=cfg.maxit)
    T.append(time.perf_counter() - t); t = time.perf_counter()
    del dirs, prob
    T.append(time.perf_counter() - t)
    T.append(st["solve_s"]); T.append(st["sweep_ms"] * 1e-3); T.append(st["orth_ms"] * 1e-3)
    return T


for _ in range(3):
    step()
gc.collect(); gc.disable()
torch.cuda.synchronize()
Ts = [step() for _ in range(n)]
tot = sorted(sum(T[:5]) for T in Ts)
med = tot[len(tot) // 2]
print(f"{n} e2e steps: median {1e3*med:.2f} ms, max {1e3*tot[-1]:.2f} ms, mean {1e3*sum(tot)/n:.2f} ms")
lab = ["assemble", "setup", "load", "solve", "destroy", "solve_s", "sweep", "orth"]
print("median step:", {k: round(1e3 * sorted(T[i] for T in Ts)[n // 2], 2) for i, k in enumerate(lab)})
for i, T in enumerate(Ts):
    if sum(T[:5]) > 1.05 * med:
        print("  slow step", i, {k: round(1e3 * v, 2) for k, v in zip(lab, T)})
