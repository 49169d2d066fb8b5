"""The paper's iteration tables (Tables 1-5) recomputed on the GPU in
the five-point paper-calibration mode (helm_assemble_fd5): the paper's source,
N strips with one extra mesh line per internal boundary, tol 1e-6, x0 = 0.
Gather: the P:L93 literal "recent" rule (default) or "core" (--core).
    python tools/fd5_tables_gpu.py [--core] [--tables 1,2,3,4,5]"""
import argparse
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2408_11929_b200 as hs
from helm_inputs import HelmConfig
from oracle import fd5   # the paper's source formula only (test / tool infrastructure)

ap = argparse.ArgumentParser()
ap.add_argument("--core", action="store_true")
ap.add_argument("--tables", default="1,2,3,4,5")
a = ap.parse_args()
gather = 1 if a.core else 0
dev = torch.device("cuda:0")


def solve(e, k, names, N=8):
    n = 2 ** e
    cfg = HelmConfig("fd5", n, n, 1.0, 1.0, k, np.ones((n + 1, n + 1)), np.zeros((n + 1, n + 1), np.complex128), N, 1, names)
    prob = hs.Problem(n, n, 1.0 / n, k, disc="fd5")
    dirs = [hs.Sweep(prob, nm, n_strips=N, overlap=1, gather=gather) for nm in names]
    b = torch.zeros(cfg.n, dtype=torch.complex128, device=dev)
    prob.load_vector(torch.tensor(fd5.source(cfg), device=dev), b)
    x = torch.zeros(cfg.n, dtype=torch.complex128, device=dev)
    t0 = time.perf_counter()
    _, st = hs.mpgmres_solve(prob, dirs, b, x, tol=1e-6, maxit=150)
    return st["iterations"] if st["converged"] else f">{st['iterations']}", time.perf_counter() - t0


tabs = set(int(t) for t in a.tables.split(","))
print(f"# gather = {'core' if gather else 'recent (P:L93)'}")
if 1 in tabs:
    paper = {50: [20, 9, 31, 18], 100: [18, 8, 29, 18], 200: [17, 9, 31, 18]}
    print("## Table 1 (h = 2^-9, N = 8): LRL / LRL+BTB / LR+RL / LR+BT+RL+TB")
    for k in (50, 100, 200):
        its = [solve(9, float(k), c)[0] for c in (["LRL"], ["LRL", "BTB"], ["LR", "RL"], ["LR", "BT", "RL", "TB"])]
        print(f"k={k}: gpu {its}  paper {paper[k]}")
if 2 in tabs:
    ks = list(range(40, 641, 40))
    pl = [20, 18, 18, 17, 17, 18, 18, 18, 19, 20, 21, 23, 23, 26, 27, 29]
    pb = [9, 8, 8, 9, 9, 10, 10, 11, 13, 13, 14, 16, 17, 19, 22, 27]
    print("## Table 2 (h = 2^-9, N = 8): k, LRL gpu/paper, LRL+BTB gpu/paper")
    for k, l, b2 in zip(ks, pl, pb):
        print(f"k={k}: LRL {solve(9, float(k), ['LRL'])[0]}/{l}  LRL+BTB {solve(9, float(k), ['LRL', 'BTB'])[0]}/{b2}")
if 3 in tabs:
    pl, pb = [8, 10, 12, 15, 19, 22], [8, 10, 10, 11, 11, 12]
    print("## Table 3 (10 ppw, N = 8): h, k, LRL gpu/paper, LRL+BTB gpu/paper")
    for e, l, b2 in zip(range(5, 10), pl, pb):   # h = 2^-10 with N = 8: 131-node strips (> 119, unsupported)
        k = 2 * math.pi * 2 ** e / 10
        print(f"h=2^-{e} k={k:.1f}: LRL {solve(e, k, ['LRL'])[0]}/{l}  LRL+BTB {solve(e, k, ['LRL', 'BTB'])[0]}/{b2}")
if 4 in tabs:
    pl, pb = [21, 10, 12, 15, 20, 24], [25, 10, 8, 8, 9, 10]
    print("## Table 4 (k = 50, N = 8): h, LRL gpu/paper, LRL+BTB gpu/paper")
    for e, l, b2 in zip(range(5, 10), pl, pb):
        print(f"h=2^-{e}: LRL {solve(e, 50.0, ['LRL'])[0]}/{l}  LRL+BTB {solve(e, 50.0, ['LRL', 'BTB'])[0]}/{b2}")
if 5 in tabs:
    paper = {50: ([17, 20, 24, 37, 60], [8, 9, 10, 13, 15]), 100: ([16, 18, 22, 33, 52], [7, 8, 10, 13, 19])}
    print("## Table 5 (h = 2^-9): N, LRL gpu/paper (GPU solve s), LRL+BTB gpu/paper (GPU solve s)")
    for k in (50, 100):
        # N = 4 gives 131-node strips (> 119, unsupported by the wide-strip factorisation)
        for N, l, b2 in zip((8, 16, 32, 64), *[v[1:] for v in paper[k]]):
            i1, t1 = solve(9, float(k), ["LRL"], N)
            i2, t2 = solve(9, float(k), ["LRL", "BTB"], N)
            print(f"k={k} N={N}: LRL {i1}/{l} ({t1:.3f} s)  LRL+BTB {i2}/{b2} ({t2:.3f} s)")
