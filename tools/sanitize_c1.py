"""Small C1 run of every hot-path call for compute-sanitizer (one tool per
gpurun call): assembly, load vector, both axes' sweep setups, one batched
4-direction apply, an SpMM and a full MPGMRES solve (t = 2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2408_11929_b200 as hs
from helm_inputs import make_config, random_vector

cfg = make_config(1)
dev = torch.device("cuda:0")
prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev))
names = ["LRL", "RLR", "BTB", "TBT"]
dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap) for nm in names]
r = torch.tensor(random_vector(cfg.n, 1), device=dev)
Z = torch.zeros((4, cfg.n), dtype=torch.complex128, device=dev)
hs.sweep_apply(dirs, r, Z, ldr=0)
W = torch.zeros_like(Z)
prob.spmv(Z, W, 4)
b = torch.zeros(cfg.n, dtype=torch.complex128, device=dev)
prob.load_vector(torch.tensor(cfg.f.ravel(), device=dev), b)
x = torch.zeros(cfg.n, dtype=torch.complex128, device=dev)
_, st = hs.mpgmres_solve(prob, [dirs[0], dirs[2]], b, x, tol=cfg.tol)
torch.cuda.synchronize()
print("sanitize_c1 done: iterations", st["iterations"], "kernel", hs.sweep_kernel_name(), "launches", hs.kernel_launches())
