"""Profile driver for the SpMV / SpMM kernel (k_spmm) on C5: warm-up, then
timed helm_spmv calls with 1 and 4 columns (CUDA events); prints model GB/s
(16 nnz + 2 t 16 n).  Under ncu: -k regex:k_spmm -s 2 -c 2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2408_11929_b200 as hs
from helm_inputs import make_config, random_vector

cfg = make_config(5)
dev = torch.device("cuda:0")
prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev))
nnz = cfg.n + 2 * (cfg.nx * (cfg.ny + 1) + (cfg.nx + 1) * cfg.ny + cfg.nx * cfg.ny)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for ncol in (1, 4):
    X = torch.tensor(random_vector(cfg.n, 5, ncol), device=dev)
    Y = torch.zeros_like(X)
    prob.spmv(X, Y, ncol)     # warm-up launch (profiled launch order: t=1 warm, t=4 warm, then timed)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        prob.spmv(X, Y, ncol)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    model = 16 * nnz + 2 * ncol * 16 * cfg.n
    print(f"C5 SpMM t={ncol}: {ms * 1e3:.1f} us, model {model / 1e6:.1f} MB -> {model / ms / 1e6:.0f} GB/s")
