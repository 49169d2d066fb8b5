"""Quick GPU diagnostics: run each hot-path piece on small inputs and print
relative differences against the oracle (never raises on mismatch)."""
import os
import sys
import time
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2408_11929_b200 as hs
from helm_inputs import make_config, random_vector, small_problem
from oracle import krylov, p1, sweep

DEV = torch.device("cuda:0")


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def gp(cfg):
    return hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=DEV))


def step(name, fn):
    t0 = time.time()
    try:
        out = fn()
        print(f"[ok ] {name}: {out}  ({time.time()-t0:.2f}s)", flush=True)
    except Exception as e:
        print(f"[ERR] {name}: {e}", flush=True)
        traceback.print_exc()


cfg = small_problem(24, 20, 12.0, seed=5, variable_c=True, n_strips=3, overlap=1)
A = p1.assemble(cfg)


def t_asm():
    prob = gp(cfg)
    d = torch.zeros(4 * cfg.n, dtype=torch.complex128, device=DEV)
    prob.diagonals(d)
    d = d.cpu().numpy().reshape(4, cfg.n)
    g = np.arange(cfg.n)
    s = cfg.nx + 1
    errs = []
    for k, off in enumerate([0, 1, s, s + 1]):
        ok = g + off < cfg.n
        errs.append(np.abs(d[k][ok] - np.asarray(A[g[ok], g[ok] + off]).ravel()).max())
    b = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    prob.load_vector(torch.tensor(cfg.f.ravel(), device=DEV), b)
    X = random_vector(cfg.n, 1, 2)
    Y = torch.zeros((2, cfg.n), dtype=torch.complex128, device=DEV)
    prob.spmv(torch.tensor(X, device=DEV), Y, 2)
    return dict(diag_err=errs, b=rel(b.cpu().numpy(), p1.load_vector(cfg)),
                spmv=[rel(Y[c].cpu().numpy(), A @ X[c]) for c in range(2)])


step("assembly/load/spmv", t_asm)


def t_sweep(names, nseg, n_strips=3, overlap=1, c=cfg, AA=A):
    prob = gp(c)
    dirs = [hs.Sweep(prob, nm, n_strips=n_strips, overlap=overlap, n_segments=nseg) for nm in names]
    R = random_vector(c.n, 2, len(names))
    Z = torch.zeros((len(names), c.n), dtype=torch.complex128, device=DEV)
    hs.sweep_apply(dirs, torch.tensor(R, device=DEV), Z)
    torch.cuda.synchronize()
    out = {}
    for k, nm in enumerate(names):
        P = sweep.make_preconditioner(c, AA, nm, n_strips=n_strips, overlap=overlap)
        out[nm] = rel(Z[k].cpu().numpy(), P.apply(R[k]))
    return out


for nseg in (1, 2, 3):
    step(f"sweep LRL nseg={nseg}", lambda nseg=nseg: t_sweep(["LRL"], nseg))
    step(f"sweep all4 nseg={nseg}", lambda nseg=nseg: t_sweep(["LRL", "RLR", "BTB", "TBT"], nseg))
step("sweep N=1", lambda: t_sweep(["LRL"], 2, n_strips=1))

c1 = make_config(1)
A1 = p1.assemble(c1)
step("C1 sweeps auto", lambda: t_sweep(["LRL", "BTB"], 0, n_strips=4, overlap=0, c=c1, AA=A1))


def t_solve():
    prob = gp(c1)
    dirs = [hs.Sweep(prob, nm, n_strips=4, overlap=0) for nm in c1.dirs]
    b = torch.zeros(c1.n, dtype=torch.complex128, device=DEV)
    prob.load_vector(torch.tensor(c1.f.ravel(), device=DEV), b)
    x = torch.zeros(c1.n, dtype=torch.complex128, device=DEV)
    _, st = hs.mpgmres_solve(prob, dirs, b, x, tol=1e-6)
    precs = [sweep.make_preconditioner(c1, A1, nm).apply for nm in c1.dirs]
    xo, so = krylov.mpgmres(A1, precs, p1.load_vector(c1), tol=1e-6)
    return dict(it=st["iterations"], it_ref=so.iterations, x=rel(x.cpu().numpy(), xo), st=st["status"],
                true=st["true_rel_res"])


step("C1 mpgmres", t_solve)
print("launches", hs.kernel_launches())
