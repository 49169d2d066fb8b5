sed -i 's/for nseg in \[33, 36\]:/for nseg in [33]:/' /tmp/c4.py 2>/dev/null
cat > /tmp/c4.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2408_11929_b200 as hs
from helm_inputs import make_config, random_vector
from oracle import p1, sweep
cfg = make_config(4)
dev = torch.device("cuda:0")
prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev))
A = p1.assemble(cfg)
precs = sweep.make_preconditioners(cfg, A, cfg.dirs)
r = random_vector(cfg.n, 41)
dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap, n_segments=33) for nm in cfg.dirs]
Z = torch.zeros((len(dirs), cfg.n), dtype=torch.complex128, device=dev)
hs.sweep_apply(dirs, torch.tensor(r, device=dev), Z, ldr=0)
Zh = Z.cpu().numpy()
print(hs.sweep_kernel_name(), ["%.4e" % (float(np.max(np.abs(Zh[k] - P.apply(r))) / np.max(np.abs(P.apply(r))))) for k, P in enumerate(precs)], flush=True)
PY
for v in at_e29c264 at_aa1f410; do echo "== $v"; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so python /tmp/c4.py; done
echo "== now"; python /tmp/c4.py
