"""Compare the fast sweep kernel with the general (TMA-ring) kernel and the
oracle goldens, per direction and batched, for one config."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2408_11929_b200 as hs
from helm_inputs import make_config, random_vector

num = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nseg = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = make_config(num)
dev = torch.device("cuda:0")
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", f"oracle_C{num}.npz"))
prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev))
dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap, n_segments=nseg) for nm in cfg.dirs]
print("P =", dirs[0].info().n_segments, "w =", dirs[0].info().wmax)
r = torch.tensor(random_vector(cfg.n, int(g["r_seed"])), device=dev)
idx = g["idx"]


def run(ds):
    Z = torch.zeros((len(ds), cfg.n), dtype=torch.complex128, device=dev)
    hs.sweep_apply(ds, r, Z, ldr=0)
    return Z.cpu().numpy()


kern = os.environ.get("HELM_SWEEP_KERNEL", "default")
Zb = run(dirs)
for k, nm in enumerate(cfg.dirs):
    Zs = run([dirs[k]])[0]
    e_b = np.linalg.norm(Zb[k][idx] - g["z"][k]) / np.linalg.norm(g["z"][k])
    e_s = np.linalg.norm(Zs[idx] - g["z"][k]) / np.linalg.norm(g["z"][k])
    print(f"{kern} {nm}: batched vs oracle {e_b:.2e}  alone vs oracle {e_s:.2e}  batched vs alone "
          f"{np.linalg.norm(Zb[k]-Zs)/np.linalg.norm(Zs):.2e}")
