cat > /tmp/c4d.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2408_11929_b200 as hs
from helm_inputs import make_config, random_vector
cfg = make_config(4)
dev = torch.device("cuda:0")
prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev))
r = torch.tensor(random_vector(cfg.n, 41), device=dev)
outs = []
for rep in range(3):
    dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap, n_segments=33) for nm in ["LRL"]]
    Z = torch.zeros((1, cfg.n), dtype=torch.complex128, device=dev)
    hs.sweep_apply(dirs, r, Z, ldr=0)
    outs.append(Z.cpu().numpy()); del dirs
print("setup-to-setup max diff", [float(np.max(np.abs(outs[k] - outs[0]))) for k in range(3)], flush=True)
PY
for v in; do echo "== $v"; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so python /tmp/c4d.py; done
echo "== now"; python /tmp/c4d.py
