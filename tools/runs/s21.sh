cat > /tmp/sc.py <<'PY'
import sys, time, torch
sys.path.insert(0, '.')
import paper_2408_11929_b200 as hs
from helm_inputs import make_config
cfg = make_config(5)
dev = torch.device("cuda:0")
c = torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev)
prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, c)
for ch in [1, 2, 4, 8, 0]:
    hs.set_knob("setup_chunks", ch)
    ts = []
    for rep in range(4):
        torch.cuda.synchronize(); t = time.perf_counter()
        dirs = hs.make_sweeps(prob, cfg.dirs, n_strips=cfg.n_strips, overlap=cfg.overlap)
        torch.cuda.synchronize(); ts.append(1e3 * (time.perf_counter() - t)); del dirs
    print(f"chunks {ch}: both axes {min(ts[1:]):.2f} ms (all {['%.1f' % x for x in ts]})", flush=True)
PY
python /tmp/sc.py
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
