cat > /tmp/orth.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2408_11929_b200 as hs
from helm_inputs import make_config
cfg = make_config(5)
dev = torch.device("cuda:0")
c = torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev)
f = torch.tensor(cfg.f.ravel(), dtype=torch.complex128, device=dev)
prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, c)
dirs = hs.make_sweeps(prob, cfg.dirs, n_strips=cfg.n_strips, overlap=cfg.overlap)
b = torch.zeros(cfg.n, dtype=torch.complex128, device=dev); prob.load_vector(f, b)
x = torch.zeros_like(b)
hs.mpgmres_solve(prob, dirs, b, x, tol=cfg.tol)
hs.set_knob("orth_prof", 1)
x.zero_()
_, st = hs.mpgmres_solve(prob, dirs, b, x, tol=cfg.tol)
print(st)
PY
python /tmp/orth.py 2>&1 | tail -16
