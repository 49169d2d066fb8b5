cat > /tmp/st.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2408_11929_b200 as hs
from helm_inputs import make_config
cfg = make_config(5)
dev = torch.device("cuda:0")
c = torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev)
prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, c)
d = hs.Sweep(prob, "LRL", n_strips=cfg.n_strips, overlap=cfg.overlap); torch.cuda.synchronize(); del d
hs.set_knob("setup_timing", 1)
d = hs.Sweep(prob, "LRL", n_strips=cfg.n_strips, overlap=cfg.overlap); torch.cuda.synchronize(); del d
PY
HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_gjp.so python /tmp/st.py 2>&1 | tail -2
