import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2408_11929_b200 as hs
from helm_inputs import make_config
cfg = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
dev = torch.device("cuda:0")
c = torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev)
prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, c)
for rep in range(3):
    if rep == 2: hs.set_knob("setup_timing", 1)
    d = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap) for nm in ("LRL", "BTB")]
    torch.cuda.synchronize()
    del d
