"""Full-size GPU parity on C1-C5 in the launch configuration bench.py times.

Expected values are oracle-only (tests/golden/oracle_C<k>.npz, written by
tools/make_golden.py, which calls nothing but oracle/ and helm_inputs): one
double-sweep apply per direction on a seeded r, sampled at 512 seeded nodes,
and the MPGMRES solve (iteration count, residual history, x at the same
nodes).  Tolerances: preconditioner 1e-10, x 1e-8 at equal iteration count,
count +-1 (BASELINE.json north star).  Properties that hold at any size
(linearity, the most-recent-gather residual identity) are checked on the
whole vector.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2408_11929_b200 as hs
from helm_inputs import make_config, random_vector
from oracle import p1, sweep

DEV = torch.device("cuda:0")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def setup(num):
    cfg = make_config(num)
    prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=DEV))
    dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap) for nm in cfg.dirs]
    return cfg, prob, dirs


@pytest.mark.parametrize("num", [1, 2, 3, 4, 5])
def test_fullsize_sweep_and_solve(num):
    g = np.load(os.path.join(GOLDEN, f"oracle_C{num}.npz"))
    cfg, prob, dirs = setup(num)
    assert list(g["dirs"]) == cfg.dirs
    idx = g["idx"]
    r = random_vector(cfg.n, int(g["r_seed"]))
    Z = torch.zeros((len(dirs), cfg.n), dtype=torch.complex128, device=DEV)
    hs.sweep_apply(dirs, torch.tensor(r, device=DEV), Z, ldr=0)
    Zs = Z.cpu().numpy()[:, idx]
    for k in range(len(dirs)):
        assert rel(Zs[k], g["z"][k]) <= 1e-10, (cfg.name, cfg.dirs[k], rel(Zs[k], g["z"][k]))
    b = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    prob.load_vector(torch.tensor(cfg.f.ravel(), device=DEV), b)
    assert abs(float(torch.linalg.norm(b)) - float(g["b_norm"])) <= 1e-13 * float(g["b_norm"])
    x = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    _, st = hs.mpgmres_solve(prob, dirs, b, x, tol=cfg.tol, maxit=cfg.maxit)
    it_ref = int(g["iterations"])
    assert abs(st["iterations"] - it_ref) <= 1, (cfg.name, st["iterations"], it_ref)
    assert st["true_rel_res"] <= 10 * cfg.tol
    if st["iterations"] == it_ref:
        assert rel(x.cpu().numpy()[idx], g["x"]) <= 1e-8
        h, hr = np.array(st["history"]), g["history"]
        assert np.max(np.abs(h - hr) / hr) <= 1e-6
        assert abs(float(torch.linalg.norm(x)) - float(g["x_norm"])) <= 1e-8 * float(g["x_norm"])


def test_fullsize_linearity_c5():
    """Linearity of the batched t = 4 apply at full C5 size (property check)."""
    cfg, prob, dirs = setup(5)
    r1 = torch.tensor(random_vector(cfg.n, 31), device=DEV)
    r2 = torch.tensor(random_vector(cfg.n, 32), device=DEV)
    a, bb = complex(0.7, -0.2), complex(-1.3, 0.4)
    Z = [torch.zeros((4, cfg.n), dtype=torch.complex128, device=DEV) for _ in range(3)]
    hs.sweep_apply(dirs, r1, Z[0], ldr=0)
    hs.sweep_apply(dirs, r2, Z[1], ldr=0)
    hs.sweep_apply(dirs, (a * r1 + bb * r2).contiguous(), Z[2], ldr=0)
    lhs = Z[2]
    rhs = a * Z[0] + bb * Z[1]
    assert float(torch.linalg.norm(lhs - rhs) / torch.linalg.norm(rhs)) <= 1e-12


def test_fullsize_repeatable_c5():
    """Deterministic: two applies on the same input are bitwise identical."""
    cfg, prob, dirs = setup(5)
    r = torch.tensor(random_vector(cfg.n, 33), device=DEV)
    Z1 = torch.zeros((4, cfg.n), dtype=torch.complex128, device=DEV)
    Z2 = torch.zeros_like(Z1)
    hs.sweep_apply(dirs, r, Z1, ldr=0)
    hs.sweep_apply(dirs, r, Z2, ldr=0)
    assert torch.equal(Z1, Z2)


@pytest.mark.parametrize("num", [4, 5])
def test_fullsize_full_vector(num):
    """The production configuration compared over the WHOLE vector: C4 (x-strips
    99 nodes wide: the general kernel) and C5 (P = 33, m = 30-31, w = 35: the
    two-chain kernel as bench.py launches it), all four directions batched in
    one launch, against the oracle computed here (splu strip factors, one set
    per axis): max |dz| <= 1e-10 ||z||_inf and the relative 2-norm <= 1e-10."""
    cfg, prob, dirs = setup(num)
    A = p1.assemble(cfg)
    precs = sweep.make_preconditioners(cfg, A, cfg.dirs)
    r = random_vector(cfg.n, 41)
    Z = torch.zeros((len(dirs), cfg.n), dtype=torch.complex128, device=DEV)
    hs.sweep_apply(dirs, torch.tensor(r, device=DEV), Z, ldr=0)
    Zh = Z.cpu().numpy()
    for k, P in enumerate(precs):
        z = P.apply(r)
        err_inf = float(np.max(np.abs(Zh[k] - z)) / np.max(np.abs(z)))
        assert err_inf <= 1e-10, (cfg.name, cfg.dirs[k], err_inf)
        assert rel(Zh[k], z) <= 1e-10, (cfg.name, cfg.dirs[k], rel(Zh[k], z))
