cat > /tmp/st4.py <<'PY'
import sys, torch, time
sys.path.insert(0, '.')
import paper_2408_11929_b200 as hs
from helm_inputs import make_config
cfg = make_config(4)
dev = torch.device("cuda:0")
c = torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev)
prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, c)
d = hs.Sweep(prob, "LRL", n_strips=cfg.n_strips, overlap=cfg.overlap); torch.cuda.synchronize(); del d
hs.set_knob("setup_timing", 1)
d = hs.Sweep(prob, "LRL", n_strips=cfg.n_strips, overlap=cfg.overlap); torch.cuda.synchronize(); del d
hs.set_knob("setup_timing", 0)
ts = []
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    dirs = hs.make_sweeps(prob, cfg.dirs, n_strips=cfg.n_strips, overlap=cfg.overlap)
    torch.cuda.synchronize(); ts.append(1e3 * (time.perf_counter() - t)); del dirs
print(f"C4 both axes setup {min(ts):.2f} ms", flush=True)
PY
python /tmp/st4.py 2>&1 | grep -v "k_reduced\]"
timeout 900 python -m pytest tests -m gpu -x -q -k "wide or C4 or fullsize or general" 2>&1 | tail -2
