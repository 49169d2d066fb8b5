"""Time the setup pieces of one C5 step (assembly, 4 sweep setups, load vector,
solve) with host clocks around synchronous calls."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2408_11929_b200 as hs
from helm_inputs import make_config

num = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = make_config(num)
dev = torch.device("cuda:0")
c = torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev)
f = torch.tensor(cfg.f.ravel(), dtype=torch.complex128, device=dev)
b = torch.zeros(cfg.n, dtype=torch.complex128, device=dev)
x = torch.zeros(cfg.n, dtype=torch.complex128, device=dev)
for rep in range(int(os.environ.get("REPS", "3"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, c)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ts = []
    if os.environ.get("PAR_SETUP"):
        a = time.perf_counter()
        dirs = hs.make_sweeps(prob, cfg.dirs, n_strips=cfg.n_strips, overlap=cfg.overlap)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - a)
    else:
        dirs = []
        for nm in cfg.dirs:
            a = time.perf_counter()
            dirs.append(hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap))
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - a)
    t2 = time.perf_counter()
    prob.load_vector(f, b)
    _, st = hs.mpgmres_solve(prob, dirs, b, x, tol=cfg.tol)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    del dirs
    torch.cuda.synchronize()
    t35 = time.perf_counter()
    del prob
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"rep {rep}: assemble {1e3*(t1-t0):.1f} ms | setups " + " ".join(f"{1e3*v:.1f}" for v in ts) +
          f" ms | solve {1e3*(t3-t2):.1f} ms (sweep {st['sweep_ms']:.1f}, orth {st['orth_ms']:.1f}, it {st['iterations']}) "
          f"| destroy sweeps {1e3*(t35-t3):.1f} problem {1e3*(t4-t35):.1f} ms", flush=True)
