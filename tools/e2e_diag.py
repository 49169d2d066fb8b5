"""Where does the end-to-end (host-buffer) step spend its time vs the device step?
Host wall time per phase, synchronised; C5."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2408_11929_b200 as hs
from helm_inputs import make_config

cfg = make_config(5)
names = cfg.dirs
dev = torch.device("cuda:0")
c_d = torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev)
f_d = torch.tensor(cfg.f.ravel(), dtype=torch.complex128, device=dev)
c_h = torch.tensor(cfg.c.ravel(), dtype=torch.float64).pin_memory()
f_h = torch.tensor(cfg.f.ravel(), dtype=torch.complex128).pin_memory()
x_h = torch.zeros(cfg.n, dtype=torch.complex128).pin_memory()
b_d = torch.zeros(cfg.n, dtype=torch.complex128, device=dev)
x_d = torch.zeros(cfg.n, dtype=torch.complex128, device=dev)
streams = {0: torch.cuda.Stream().cuda_stream, 1: torch.cuda.Stream().cuda_stream}


def step(host):
    T = {}
    torch.cuda.synchronize(); t = time.perf_counter()
    prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, c_h.numpy() if host else c_d)
    torch.cuda.synchronize(); T["assemble"] = time.perf_counter() - t; t = time.perf_counter()
    dirs = hs.make_sweeps(prob, names, n_strips=cfg.n_strips, overlap=cfg.overlap, streams=streams)
    torch.cuda.synchronize(); T["setup"] = time.perf_counter() - t; t = time.perf_counter()
    prob.load_vector(f_h.numpy() if host else f_d, b_d)
    torch.cuda.synchronize(); T["load"] = time.perf_counter() - t; t = time.perf_counter()
    _, st = hs.mpgmres_solve(prob, dirs, b_d, x_h.numpy() if host else x_d, tol=cfg.tol, maxit=cfg.maxit)
    torch.cuda.synchronize(); T["solve"] = time.perf_counter() - t; t = time.perf_counter()
    del dirs, prob
    torch.cuda.synchronize(); T["destroy"] = time.perf_counter() - t
    return T


for host in (False, True, False, True):
    for _ in range(2):
        step(host)
    Ts = [step(host) for _ in range(3)]
    print("host" if host else "dev ", {k: round(1e3 * sum(T[k] for T in Ts) / 3, 2) for k in Ts[0]}, flush=True)


# per-step outliers of the host-buffer step: 150 steps, phases of every step above 1.15x the median
Ts = [step(True) for _ in range(150)]
tot = sorted(sum(T.values()) for T in Ts)
med = tot[len(tot) // 2]
print(f"host-buffer steps: median {1e3*med:.2f} ms, max {1e3*tot[-1]:.2f} ms", flush=True)
for i, T in enumerate(Ts):
    if sum(T.values()) > 1.15 * med:
        print("  outlier step", i, {k: round(1e3 * v, 2) for k, v in T.items()}, flush=True)
Ts = [step(False) for _ in range(150)]
tot = sorted(sum(T.values()) for T in Ts)
med = tot[len(tot) // 2]
print(f"device-buffer steps: median {1e3*med:.2f} ms, max {1e3*tot[-1]:.2f} ms", flush=True)
for i, T in enumerate(Ts):
    if sum(T.values()) > 1.15 * med:
        print("  outlier step", i, {k: round(1e3 * v, 2) for k, v in T.items()}, flush=True)
