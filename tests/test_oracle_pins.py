"""Pins of the CPU oracle against what the paper and the mathematics fix
(SURVEY.md §8(c) Pin-1 .. Pin-14).  CPU only.

None of these re-types the oracle's formula: each checks an independent fact
(closed-form stencil rows from hand algebra, a symmetry, a conservation
identity, a manufactured solution's convergence order, a brute-force dense
solve, an exactness property of the method, a textbook algorithm, or the cost
formula printed in the paper).
"""
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from helm_inputs import make_config, small_problem
from oracle import krylov, p1, strips, sweep

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _const_cfg(n, k):
    cfg = small_problem(n, n, k, seed=0)
    cfg.c[:] = 1.0
    return cfg


# ---------------------------------------------------------------- Pin-1 / 2 / 3



@pytest.mark.parametrize("k", [2.0, 7.5])
def test_pin1_closed_form_rows(k):
    """Pin-1: assembled rows equal the closed-form P1 rows (hand algebra,
    tests/golden/p1_stencil_closed_form.txt, expressed in t = k^2 h^2 and
    s = k h)."""
    n = 8
    cfg = _const_cfg(n, k)
    A = p1.assemble(cfg).tocsr()
    h = cfg.h
    t = k * k * h * h
    s = k * h
    where = {"interior": (4, 4), "bottom": (4, 0), "top": (4, n), "left": (0, 4),
             "right": (n, 4), "corner00": (0, 0), "cornerNN": (n, n),
             "cornerN0": (n, 0), "corner0N": (0, n)}
    env = {"t": t, "s": s}
    gold = {}
    with open(os.path.join(GOLDEN, "p1_stencil_closed_form.txt")) as fh:
        for line in fh:
            line = line.split("#")[0].strip()
            if not line:
                continue
            name, di, dj, re_expr, im_expr = line.split()
            gold.setdefault(name, []).append((int(di), int(dj), eval(re_expr, {}, env), eval(im_expr, {}, env)))
    for name, entries in gold.items():
        i, j = where[name]
        g = p1.node(cfg, i, j)
        row = A.getrow(g).toarray().ravel()
        expected = np.zeros(cfg.n, dtype=np.complex128)
        for di, dj, re, im in entries:
            expected[p1.node(cfg, i + di, j + dj)] = re + 1j * im
        np.testing.assert_allclose(row, expected, rtol=0, atol=1e-14, err_msg=name)


def test_pin1b_variable_c_closed_form_rows():
    """Pin-1b (A5 / D3, variable wave speed): on a 2 x 2-cell grid with nine
    nodal c values (non-linear in i, j), the assembled rows equal the rows
    derived by hand in tests/golden/p1_variable_c_closed_form.txt, where every
    k_T = omega / mean(c at the triangle's vertices) and k_e = omega / mean(c at
    the edge's ends) was worked out as a fraction.  A centroid, harmonic-mean,
    nodal-k or wrong-triangle reading changes these numbers."""
    from helm_inputs import HelmConfig
    c = np.array([[1.0, 3.0, 2.0], [4.0, 1.0, 5.0], [2.0, 6.0, 3.0]])     # [j][i]
    cfg = HelmConfig("pin1b", 2, 2, 1.0, 1.0, 6.0, c, np.zeros((3, 3), np.complex128), 1, 0, ["LRL"])
    A = p1.assemble(cfg).tocsr()
    rows = {}
    with open(os.path.join(GOLDEN, "p1_variable_c_closed_form.txt")) as fh:
        for line in fh:
            line = line.split("#")[0].strip()
            if not line:
                continue
            i, j, di, dj, re_expr, im_expr = line.split()
            rows.setdefault((int(i), int(j)), []).append((int(di), int(dj), eval(re_expr), eval(im_expr)))
    assert len(rows) == 4
    for (i, j), entries in rows.items():
        row = A.getrow(p1.node(cfg, i, j)).toarray().ravel()
        expected = np.zeros(cfg.n, dtype=np.complex128)
        for di, dj, re, im in entries:
            expected[p1.node(cfg, i + di, j + dj)] = re + 1j * im
        np.testing.assert_allclose(row, expected, rtol=0, atol=1e-14, err_msg=str((i, j)))


@pytest.mark.parametrize("axis", [0, 1])
@pytest.mark.parametrize("overlap", [0, 1])
def test_pin_d7_strip_is_its_own_impedance_problem(axis, overlap):
    """D7 interface term (Eq. 4): the transmission operator on an
    interface is B = d/dn - i k, the operator of the physical boundary condition
    Eq. 1b.  So each local matrix A_s must equal the D4 assembly of the
    strip's rectangle posed as its OWN impedance problem (all of its boundary
    edges impedance edges, with k_e from the same nodal c), which Pin-1 / Pin-1b
    / Pin-4 fix independently.  A wrong sign or scale of the interface term
    i k_e B_e, or a missing / extra interface edge, fails here.  Every strip of a
    16 x 12 variable-c grid, both axes, overlap 0 and 1."""
    from helm_inputs import HelmConfig
    cfg = small_problem(16, 12, 9.0, seed=21, variable_c=True, n_strips=4, overlap=overlap)
    _, sts = strips.strips(cfg, axis, 4, overlap)
    for st in sts:
        As = strips.restrict(strips.local_matrix_global(cfg, axis, st), st.nodes).toarray()
        if axis == 0:
            c_sub = cfg.c[:, st.a:st.b + 1]
            sub = HelmConfig("sub", st.b - st.a, cfg.ny, (st.b - st.a) * cfg.h, cfg.Ly, cfg.omega,
                             np.ascontiguousarray(c_sub), np.zeros_like(c_sub, np.complex128), 1, 0, ["LRL"])
        else:
            c_sub = cfg.c[st.a:st.b + 1, :]
            sub = HelmConfig("sub", cfg.nx, st.b - st.a, cfg.Lx, (st.b - st.a) * cfg.h, cfg.omega,
                             np.ascontiguousarray(c_sub), np.zeros_like(c_sub, np.complex128), 1, 0, ["LRL"])
        assert abs(sub.h - cfg.h) < 1e-15
        Asub = p1.assemble(sub).toarray()
        assert As.shape == Asub.shape
        scale = np.abs(Asub).max()
        assert np.abs(As - Asub).max() <= 1e-14 * scale, (axis, overlap, st.s)


def test_pin2_complex_symmetric_not_hermitian():
    cfg = small_problem(10, 7, 6.0, seed=3, variable_c=True)
    A = p1.assemble(cfg)
    assert abs(A - A.T).max() == 0.0
    assert abs(A - A.conj().T).max() > 1e-3


def test_pin3_row_sums():
    """Pin-3: K annihilates constants, so A 1 = k^2 M 1 + i k B 1; interior
    rows sum to k^2 h^2 (area of the node's patch h^2 times k^2)."""
    k = 5.0
    cfg = _const_cfg(12, k)
    A = p1.assemble(cfg)
    one = np.ones(cfg.n)
    rs = A @ one
    h = cfg.h
    i, j = np.meshgrid(np.arange(1, 12), np.arange(1, 12))
    g = p1.node(cfg, i.ravel(), j.ravel())
    np.testing.assert_allclose(rs[g], k * k * h * h, rtol=1e-13)
    # total: k^2 |Omega| + i k |dOmega|
    np.testing.assert_allclose(rs.sum(), k * k * 1.0 + 1j * k * 4.0, rtol=1e-12)


# ---------------------------------------------------------------- Pin-4

def test_pin4_plane_wave_second_order():
    """Pin-4: plane wave u* = exp(i k (x cos 0.3 + y sin 0.3)) solves Eq. 1a
    with f = 0; impedance data g = du*/dn - i k u*.  The P1 error in max norm
    must decrease at order >= 1.95 from nx = 64 to 128 (k = 10)."""
    k, th = 10.0, 0.3
    d = np.array([math.cos(th), math.sin(th)])
    u = lambda x, y: np.exp(1j * k * (x * d[0] + y * d[1]))
    grad = lambda x, y: (1j * k * d[0] * u(x, y), 1j * k * d[1] * u(x, y))
    errs = []
    for n in (32, 64, 128):
        cfg = _const_cfg(n, k)
        A = p1.assemble(cfg)
        b = p1.manufactured_rhs(cfg, u, grad, k)
        uh = spla.spsolve(A.tocsc(), b)
        x, y = p1.node_xy(cfg)
        errs.append(np.max(np.abs(uh - u(x, y))))
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert orders[-1] >= 1.95, (errs, orders)
    assert orders[0] >= 1.9, (errs, orders)


# ---------------------------------------------------------------- Pin-5 / 5b

def test_pin5_dense_bruteforce():
    """Pin-5: dense numpy.linalg.solve on a tiny grid agrees with the sparse
    global solve and with every strip's SuperLU solve."""
    cfg = small_problem(12, 9, 8.0, seed=5, variable_c=True, n_strips=3, overlap=1)
    A = p1.assemble(cfg)
    r = cfg.f.ravel()
    xd = np.linalg.solve(A.toarray(), r)
    xs = spla.spsolve(A.tocsc(), r)
    assert np.linalg.norm(xd - xs) / np.linalg.norm(xd) < 1e-12
    for axis in (0, 1):
        _, sts = strips.strips(cfg, axis, 3, 1)
        for st in sts:
            S = sweep.StripSolver(cfg, axis, st, A)
            rl = r[st.nodes]
            dense = np.linalg.solve(S.As.toarray(), rl)
            assert np.linalg.norm(S.solve(rl) - dense) / np.linalg.norm(dense) < 1e-12


def test_pin5b_c1_load_vector_closed_form():
    """Pin-5b: b = M1 f at the C1 centre node equals
    h^2 [1/2 + (4 e^{-h^2/(2 sigma^2)} + 2 e^{-h^2/sigma^2}) / 12]
    (centre weight h^2/2, 4 axis neighbours at distance h and the 2 "/"
    neighbours at distance sqrt(2) h, each weighted h^2/12)."""
    cfg = make_config(1)
    b = p1.load_vector(cfg)
    h, sg = cfg.h, 0.02
    bc = h * h * (0.5 + (4 * math.exp(-h * h / (2 * sg * sg)) + 2 * math.exp(-h * h / (sg * sg))) / 12.0)
    assert abs(b[p1.node(cfg, 32, 32)] - bc) < 1e-18
    assert abs(bc - 2.041483e-4) < 1e-9
    # the mass matrix integrates constants exactly: 1^T M1 1 = |Omega|
    assert abs(p1.mass_unit(cfg).sum() - 1.0) < 1e-13


# ---------------------------------------------------------------- D7 / D8 consistency

def test_local_matrix_equals_global_off_interface():
    """D7: A_s = A[I_s, I_s] except in rows/columns on the interface lines; A_s is
    complex symmetric; N = 1 gives A_1 = A."""
    cfg = small_problem(16, 12, 7.0, seed=2, variable_c=True)
    A = p1.assemble(cfg).tocsr()
    for axis in (0, 1):
        p, sts = strips.strips(cfg, axis, 4, 1)
        for st in sts:
            As = strips.restrict(strips.local_matrix_global(cfg, axis, st), st.nodes).toarray()
            Ar = A[st.nodes][:, st.nodes].toarray()
            assert np.abs(As - As.T).max() == 0.0
            keep = np.ones(st.nodes.size, dtype=bool)
            for L, has in ((st.a, st.low_iface), (st.b, st.high_iface)):
                if has:
                    keep &= ~np.isin(st.nodes, strips.line_nodes(cfg, axis, L))
            assert np.abs((As - Ar)[np.ix_(keep, keep)]).max() < 1e-13
    _, one = strips.strips(cfg, 0, 1, 0)
    A1 = strips.local_matrix_global(cfg, 0, one[0])
    assert abs(A1 - A).max() < 1e-13


@pytest.mark.parametrize("overlap", [0, 1, 2])
def test_transmission_consistency(overlap):
    """S:L225 / D8: the exact solution u* = A^{-1} b restricted to any strip
    satisfies that strip's local system when both interface corrections are
    built from u* itself: A_s R_s u* = R_s b + C^low(u*) + C^high(u*)."""
    cfg = small_problem(20, 15, 9.0, seed=4, variable_c=True)
    A = p1.assemble(cfg)
    b = cfg.f.ravel()
    u = spla.spsolve(A.tocsc(), b)
    for axis in (0, 1):
        _, sts = strips.strips(cfg, axis, 3, overlap)
        for st in sts:
            S = sweep.StripSolver(cfg, axis, st, A)
            lhs = S.As @ u[st.nodes]
            rhs = b[st.nodes].astype(np.complex128)
            for side in S.corr:
                rhs = rhs + (S.corr[side] @ u)[st.nodes]
            assert np.abs(lhs - rhs).max() <= 1e-10 * np.abs(b).max()


def test_correction_five_point_support():
    """D8: each interface row of (Atilde_s - A) touches exactly the 3 nodes on
    the interface line and the 2 outer-line nodes of the '/' mesh
    ((a-1, c), (a-1, c-1) on the low side; (b+1, c), (b+1, c+1) on the high side)."""
    cfg = small_problem(16, 12, 6.0, seed=7, variable_c=True)
    A = p1.assemble(cfg)
    _, sts = strips.strips(cfg, 0, 4, 1)
    st = sts[1]
    S = sweep.StripSolver(cfg, 0, st, A)
    j = 5
    for side, L, outer in (("low", st.a, [(st.a - 1, j), (st.a - 1, j - 1)]),
                           ("high", st.b, [(st.b + 1, j), (st.b + 1, j + 1)])):
        row = S.corr[side].getrow(p1.node(cfg, L, j)).toarray().ravel()
        nz = set(np.nonzero(np.abs(row) > 0)[0].tolist())
        exp = {int(p1.node(cfg, L, jj)) for jj in (j - 1, j, j + 1)} | {int(p1.node(cfg, i, jj)) for i, jj in outer}
        assert nz == exp


# ---------------------------------------------------------------- Pin-6 .. Pin-10

@pytest.mark.parametrize("name", ["LRL", "RLR", "BTB", "TBT", "LR", "TB"])
def test_pin6_single_strip_is_exact(name):
    cfg = small_problem(12, 10, 9.0, seed=1, variable_c=True)
    A = p1.assemble(cfg)
    r = cfg.f.ravel()
    x = spla.spsolve(A.tocsc(), r)
    P = sweep.make_preconditioner(cfg, A, name, n_strips=1, overlap=1)
    assert np.linalg.norm(P.apply(r) - x) / np.linalg.norm(x) < 1e-13


@pytest.mark.parametrize("overlap,n", [(0, 12), (1, 12), (2, 15)])
@pytest.mark.parametrize("name", ["LRL", "RLR", "BTB", "TBT"])
def test_pin7_exact_schur_double_sweep_is_exact(name, overlap, n):
    """Pin-7: with exact Schur complements (exact DtN data) the
    double sweep is A^{-1}; MPGMRES then converges in one iteration."""
    cfg = small_problem(n, n, 9.0, seed=1, variable_c=True, n_strips=3, overlap=overlap)
    A = p1.assemble(cfg)
    r = cfg.f.ravel()
    x = spla.spsolve(A.tocsc(), r)
    P = sweep.make_preconditioner(cfg, A, name, exact_schur=True)
    z = P.apply(r)
    assert np.linalg.norm(z - x) / np.linalg.norm(x) < 1e-13
    _, st = krylov.mpgmres(A, [P.apply], r, tol=1e-10, maxit=5)
    assert st.iterations == 1 and st.converged


def test_inexact_sweep_is_not_exact():
    """Control for Pin-7: the Robin (Eq. 4) sweep is only an approximation."""
    cfg = small_problem(12, 12, 9.0, seed=1, variable_c=True, n_strips=3, overlap=1)
    A = p1.assemble(cfg)
    r = cfg.f.ravel()
    x = spla.spsolve(A.tocsc(), r)
    z = sweep.make_preconditioner(cfg, A, "LRL").apply(r)
    assert np.linalg.norm(z - x) / np.linalg.norm(x) > 1e-4


@pytest.mark.parametrize("name", ["LRL", "RLR", "BTB", "TBT", "LR", "RL", "BT", "TB"])
def test_pin8_linearity(name):
    cfg = small_problem(16, 16, 8.0, seed=3, variable_c=True, n_strips=4, overlap=1)
    A = p1.assemble(cfg)
    rng = np.random.default_rng(8)
    r1 = rng.standard_normal(cfg.n) + 1j * rng.standard_normal(cfg.n)
    r2 = rng.standard_normal(cfg.n) + 1j * rng.standard_normal(cfg.n)
    a, bb = 0.3 - 1.1j, -2.0 + 0.5j
    P = sweep.make_preconditioner(cfg, A, name)
    lhs = P.apply(a * r1 + bb * r2)
    rhs = a * P.apply(r1) + bb * P.apply(r2)
    assert np.linalg.norm(lhs - rhs) / np.linalg.norm(rhs) < 1e-12


@pytest.mark.parametrize("N", [1, 2, 4])
def test_pin9_solve_count(N):
    cfg = small_problem(16, 16, 8.0, seed=3, n_strips=N, overlap=1)
    A = p1.assemble(cfg)
    for name, expect in (("LRL", 2 * N - 1), ("TB", N)):
        P = sweep.make_preconditioner(cfg, A, name)
        P.apply(cfg.f.ravel())
        assert P.n_solves == expect


@pytest.mark.parametrize("overlap", [0, 1])
def test_pin10_transposition_symmetry(overlap):
    """Pin-10: the '/' mesh is invariant under x <-> y, so on a square grid
    with c symmetric, BTB(r) = T LRL(T r) and TBT(r) = T RLR(T r)."""
    n = 16
    cfg = small_problem(n, n, 8.0, seed=9, n_strips=4, overlap=overlap)
    cfg.c = 0.5 * (cfg.c + cfg.c.T)
    A = p1.assemble(cfg)
    T = lambda v: v.reshape(n + 1, n + 1).T.ravel()
    assert abs(A - A[np.argsort(T(np.arange(cfg.n)))][:, np.argsort(T(np.arange(cfg.n)))]).max() < 1e-14
    r = cfg.f.ravel()
    for xname, yname in (("LRL", "BTB"), ("RLR", "TBT")):
        zx = sweep.make_preconditioner(cfg, A, xname).apply(T(r))
        zy = sweep.make_preconditioner(cfg, A, yname).apply(r)
        assert np.linalg.norm(zy - T(zx)) / np.linalg.norm(zy) < 1e-13


def test_gather_recent_vs_core_differ_only_in_overlap():
    """A16: the two gathers agree outside the overlap bands."""
    cfg = small_problem(16, 12, 8.0, seed=3, n_strips=4, overlap=1)
    A = p1.assemble(cfg)
    r = cfg.f.ravel()
    Pr = sweep.make_preconditioner(cfg, A, "LRL", gather="recent")
    Pc = sweep.make_preconditioner(cfg, A, "LRL", gather="core")
    zr, zc = Pr.apply(r), Pc.apply(r)
    i = np.arange(cfg.n) % (cfg.nx + 1)
    band = np.zeros(cfg.n, dtype=bool)
    for s in range(1, 4):
        band |= np.abs(i - Pr.p[s]) <= 1
    assert np.abs(zr - zc)[~band].max() == 0.0
    assert np.abs(zr - zc)[band].max() > 0.0


# ---------------------------------------------------------------- Pin-11 .. Pin-14

def test_pin11_t1_is_textbook_gmres():
    cfg = small_problem(12, 12, 8.0, seed=11, n_strips=3, overlap=1)
    A = p1.assemble(cfg)
    b = cfg.f.ravel()
    P = sweep.make_preconditioner(cfg, A, "LRL")
    xs = krylov.gmres_textbook(A, P.apply, b, 6)
    _, st = krylov.mpgmres(A, [P.apply], b, tol=1e-30, maxit=6, keep_x_history=True)
    for a, c in zip(xs, st.x_history):
        assert np.linalg.norm(a - c) / np.linalg.norm(a) < 1e-10


@pytest.mark.parametrize("t", [2, 4])
def test_pin12_paper_inner_product_count(t):
    """(k - 1/2) t^2 + (3/2) t inner products at iteration k."""
    cfg = small_problem(16, 16, 8.0, seed=12, n_strips=4, overlap=1)
    A = p1.assemble(cfg)
    names = ["LRL", "BTB"] if t == 2 else ["LRL", "RLR", "BTB", "TBT"]
    precs = [sweep.make_preconditioner(cfg, A, nm).apply for nm in names]
    _, st = krylov.mpgmres(A, precs, cfg.f.ravel(), tol=1e-14, maxit=4, mode="paper")
    assert st.deflations == 0
    for k, ip in enumerate(st.inner_products, start=1):
        assert ip == (k - 0.5) * t * t + 1.5 * t
    assert st.matvecs == t * st.iterations and st.prec_applies == t * st.iterations


def test_pin13_complete_dominates():
    """Pin-13: on a tiny system with t = 2, the complete MPGMRES
    residual (brute-force least squares over the enumerated word space) is <=
    the selective residual and <= each single-preconditioner GMRES residual."""
    cfg = small_problem(6, 6, 5.0, seed=13, n_strips=2, overlap=0)
    A = p1.assemble(cfg)
    b = cfg.f.ravel()
    P1 = sweep.make_preconditioner(cfg, A, "LR").apply
    P2 = sweep.make_preconditioner(cfg, A, "BT").apply
    K = 3
    comp = krylov.complete_mpgmres_residuals(A, [P1, P2], b, K)
    _, sel = krylov.mpgmres(A, [P1, P2], b, tol=1e-30, maxit=K)
    _, g1 = krylov.mpgmres(A, [P1], b, tol=1e-30, maxit=K)
    _, g2 = krylov.mpgmres(A, [P2], b, tol=1e-30, maxit=K)
    for k in range(K):
        assert comp[k] <= sel.history[k] * (1 + 1e-10)
        assert comp[k] <= g1.history[k] * (1 + 1e-10)
        assert comp[k] <= g2.history[k] * (1 + 1e-10)
    assert comp[1] < sel.history[1] * 0.999   # the complete space is strictly larger


def test_pin14_arnoldi_relation_and_monotonicity():
    cfg = small_problem(16, 16, 10.0, seed=14, n_strips=4, overlap=1)
    A = p1.assemble(cfg)
    b = cfg.f.ravel()
    precs = [sweep.make_preconditioner(cfg, A, nm).apply for nm in ["LRL", "RLR", "BTB", "TBT"]]
    x, st, (V, Z, H) = krylov.mpgmres(A, precs, b, tol=1e-8, maxit=30, return_basis=True)
    assert st.converged
    h = np.array(st.history)
    assert np.all(np.diff(h) <= 1e-14)
    assert np.abs(V.conj().T @ V - np.eye(V.shape[1])).max() < 1e-12
    AZ = A @ Z
    rel = np.linalg.norm(AZ - V[:, :H.shape[0]] @ H) / (sp.linalg.norm(A) * np.linalg.norm(Z))
    assert rel < 1e-12
    assert abs(st.true_rel_res - h[-1]) < 1e-8


@pytest.mark.parametrize("name", ["LRL", "RLR", "BTB", "TBT"])
def test_recent_gather_keeps_last_solves_equations(name):
    """P:L93 "values from the most recent subdomain solve": after the double
    sweep, z equals u_{sigma m} wherever no later-written strip overwrote it,
    so the global residual r - A z vanishes on every row whose whole stencil
    lies in such a region and off the interface lines (there each u_s solves
    A_s u_s = R_s r + corrections with A_s = A).  A wrong overwrite order
    breaks this on the overlap-adjacent lines."""
    n = 16
    cfg = small_problem(n, n, 8.0, seed=21, variable_c=True, n_strips=4, overlap=1)
    A = p1.assemble(cfg)
    r = cfg.f.ravel()
    P = sweep.make_preconditioner(cfg, A, name)
    z = P.apply(r)
    res = np.abs(r - A @ z)
    axis = P.axis
    line_of = (np.arange(cfg.n) % (n + 1)) if axis == 0 else (np.arange(cfg.n) // (n + 1))
    owner = -np.ones(n + 1, dtype=int)          # strip whose u is in z on each line
    for s in reversed(P.sigma):                 # written sigma_N first ... sigma_1 last
        st = P.strips[s]
        owner[st.a:st.b + 1] = s
    checked = 0
    for L in range(1, n):
        s = owner[L]
        st = P.strips[s]
        if owner[L - 1] == s and owner[L + 1] == s and L not in (st.a, st.b):
            rows = line_of == L
            assert res[rows].max() <= 1e-10 * np.abs(r).max(), (name, L)
            checked += 1
    assert checked >= n - 8


def test_selection_rule_examples():
    """P:L154 (and S:L342-344, tagged [PAPER]): k = 1 -> every preconditioner
    gets v1; t = 2, V2 = [a b] (a from M1, b from M2) -> sources (b, a);
    t = 4, V2 = [a b c d] -> all get a + b + c + d."""
    rng = np.random.default_rng(0)
    v1 = rng.standard_normal(5)
    a, b, c, d = (rng.standard_normal(5) for _ in range(4))
    assert all(np.array_equal(s, v1) for s in krylov._select_sources(1, 3, v1[:, None], [-1], v1))
    s = krylov._select_sources(2, 2, np.column_stack([a, b]), [0, 1], v1)
    assert np.array_equal(s[0], b) and np.array_equal(s[1], a)
    s = krylov._select_sources(2, 4, np.column_stack([a, b, c, d]), [0, 1, 2, 3], v1)
    assert all(np.allclose(x, a + b + c + d) for x in s)
    s = krylov._select_sources(3, 2, np.column_stack([b]), [1], v1)   # deflated: survivor feeds both
    assert np.array_equal(s[0], b) and np.array_equal(s[1], b)


def test_duplicate_preconditioner_deflates_to_gmres():
    """Deflation (D10 step 5-6, A19, A21): MPGMRES with [M, M] builds exactly
    GMRES's space (the second column deflates every iteration), so its
    residual history equals t = 1 GMRES with M."""
    cfg = small_problem(12, 12, 8.0, seed=22, n_strips=3, overlap=1)
    A = p1.assemble(cfg)
    b = cfg.f.ravel()
    M = sweep.make_preconditioner(cfg, A, "LRL").apply
    _, g = krylov.mpgmres(A, [M], b, tol=1e-9, maxit=40)
    x2, d = krylov.mpgmres(A, [M, M], b, tol=1e-9, maxit=40)
    assert d.deflations == d.iterations
    assert d.iterations == g.iterations
    np.testing.assert_allclose(d.history, g.history, rtol=1e-6)


def test_shared_strip_solvers_are_identical():
    """make_preconditioners factors each axis once and reuses the strip solvers
    for the other order (test / bench infrastructure): the applies are bit for
    bit those of independently built preconditioners."""
    cfg = small_problem(20, 16, 8.0, seed=4, variable_c=True, n_strips=3, overlap=1)
    A = p1.assemble(cfg)
    names = ["LRL", "RLR", "BTB", "TBT"]
    shared = sweep.make_preconditioners(cfg, A, names)
    assert shared[0].solvers is shared[1].solvers and shared[2].solvers is shared[3].solvers
    r = np.random.default_rng(3).standard_normal(cfg.n) + 0j
    for nm, P in zip(names, shared):
        assert np.array_equal(P.apply(r), sweep.make_preconditioner(cfg, A, nm).apply(r)), nm
