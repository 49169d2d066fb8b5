import os, sys, time, threading
sys.path.insert(0, "/root/repo")
import torch
import paper_2408_11929_b200 as hs
from helm_inputs import make_config
cfg = make_config(5)
dev = torch.device("cuda:0")
c = torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev)
streams = {0: torch.cuda.Stream().cuda_stream, 1: torch.cuda.Stream().cuda_stream}
T0 = time.perf_counter()
log = []
def run(ax, names, prob):
    for nm in names:
        a = time.perf_counter()
        s = hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap, stream=streams[ax])
        b = time.perf_counter()
        log.append((nm, round((a - T0) * 1e3, 1), round((b - T0) * 1e3, 1)))
        keep.append(s)
for rep in range(3):
    prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, c)
    keep = []
    log.clear()
    torch.cuda.synchronize()
    T0 = time.perf_counter()
    th = [threading.Thread(target=run, args=(0, ["LRL", "RLR"], prob)), threading.Thread(target=run, args=(1, ["BTB", "TBT"], prob))]
    for t in th: t.start()
    for t in th: t.join()
    print(rep, sorted(log, key=lambda x: x[1]), round((time.perf_counter() - T0) * 1e3, 1))
    del keep, prob
