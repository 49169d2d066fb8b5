cat > /tmp/st.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2408_11929_b200 as hs
from helm_inputs import make_config
cfg = make_config(5)
dev = torch.device("cuda:0")
c = torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev)
prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, c)
for rep in range(2):
    d = hs.Sweep(prob, "LRL", n_strips=cfg.n_strips, overlap=cfg.overlap)
    torch.cuda.synchronize(); del d
hs.set_knob("setup_timing", 1)
d = hs.Sweep(prob, "LRL", n_strips=cfg.n_strips, overlap=cfg.overlap)
torch.cuda.synchronize(); del d
PY
for v in r4 r6 r9fg; do echo "== $v"; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so python /tmp/st.py 2>&1 | tail -2; done
echo "== r9"; python /tmp/st.py 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/prof_setup.py 5 2>&1 | tail -1
