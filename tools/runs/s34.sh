cat > /tmp/c4.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2408_11929_b200 as hs
from helm_inputs import make_config, random_vector
from oracle import p1, sweep
cfg = make_config(4)
dev = torch.device("cuda:0")
prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev))
A = p1.assemble(cfg)
precs = sweep.make_preconditioners(cfg, A, cfg.dirs)
r = random_vector(cfg.n, 41)
for nseg in [33, 36]:
    dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap, n_segments=nseg if nm in ("BTB","TBT") else 33) for nm in cfg.dirs]
    Z = torch.zeros((len(dirs), cfg.n), dtype=torch.complex128, device=dev)
    hs.sweep_apply(dirs, torch.tensor(r, device=dev), Z, ldr=0)
    Zh = Z.cpu().numpy()
    errs = []
    for k, P in enumerate(precs):
        z = P.apply(r); errs.append(float(np.max(np.abs(Zh[k] - z)) / np.max(np.abs(z))))
    print("y-strips P", nseg, "err_inf per dir", ["%.3e" % e for e in errs], flush=True)
    del dirs
PY
echo "== new GJ"; python /tmp/c4.py
echo "== old GJ"; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_oldgj.so python /tmp/c4.py
