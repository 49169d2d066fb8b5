"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs (SURVEY §8(c) parity metrics).

  b and A x          relative 2-norm <= 1e-14  (we allow 1e-13: different summation order)
  preconditioner     relative 2-norm <= 1e-10  (BASELINE.json north star)
  MPGMRES            same iteration count +-1; x at equal k <= 1e-8 (A23)

Sizes: full C1-C3; C4/C5 recipes at reduced grids that the oracle finishes in
seconds but that still span several segments, separators and a ragged last
segment; full-size C4/C5 are covered by test_gpu_fullsize.py.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2408_11929_b200 as hs
from helm_inputs import make_config, random_vector, small_problem
from oracle import krylov, p1, sweep

DEV = torch.device("cuda:0")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def elementwise(a, b):
    """max_i |a_i - b_i| / ||b||_inf (element-wise bound beside the 2-norm one)."""
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


KERNEL_KNOB = {"dual": 0, "fast": 2, "general": 3}


@pytest.fixture
def knob():
    """Set library knobs (helm_set_knob) for one test; all reset to 0 afterwards."""
    touched = []

    def set_(name, value):
        touched.append(name)
        hs.set_knob(name, value)

    yield set_
    for name in touched:
        hs.set_knob(name, 0)


def gpu_problem(cfg):
    return hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=DEV))


def to_dev(x):
    return torch.tensor(np.ascontiguousarray(x), dtype=torch.complex128, device=DEV)


CFGS = {
    "C1": lambda: make_config(1),
    "C2": lambda: make_config(2),
    "C3": lambda: make_config(3),
    "C4s": lambda: make_config(4, nx=384),        # 384 x 128 recipe of C4 (variable c)
    "C5s": lambda: make_config(5, nx=256),        # 256^2, N = 32 strips of 8 cells
    "var": lambda: small_problem(40, 33, 25.0, seed=5, variable_c=True, n_strips=5, overlap=1),
}


@pytest.mark.parametrize("name", ["C1", "var", "C4s"])
def test_assembly_and_load_vector(name):
    cfg = CFGS[name]()
    A = p1.assemble(cfg).tocsr()
    prob = gpu_problem(cfg)
    diag = torch.zeros(4 * cfg.n, dtype=torch.complex128, device=DEV)
    prob.diagonals(diag)
    d = diag.cpu().numpy().reshape(4, cfg.n)
    g = np.arange(cfg.n)
    s = cfg.nx + 1
    for k, off in enumerate([0, 1, s, s + 1]):
        ok = g + off < cfg.n
        ref = np.asarray(A[g[ok], g[ok] + off]).ravel()
        got = d[k][ok]
        # entries that do not exist (row ends) must be exactly zero on both sides
        assert np.abs(got - ref).max() <= 1e-13 * np.abs(A.data).max(), (name, k)
    b_ref = p1.load_vector(cfg)
    b = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    prob.load_vector(to_dev(cfg.f.ravel()), b)
    assert rel(b.cpu().numpy(), b_ref) <= 1e-14


@pytest.mark.parametrize("ncols", [1, 2, 4, 5])
def test_spmm(ncols):
    cfg = CFGS["var"]()
    A = p1.assemble(cfg)
    prob = gpu_problem(cfg)
    X = random_vector(cfg.n, 3, ncols)
    Y = torch.zeros((ncols, cfg.n), dtype=torch.complex128, device=DEV)
    prob.spmv(to_dev(X), Y, ncols)
    for c in range(ncols):
        assert rel(Y[c].cpu().numpy(), A @ X[c]) <= 1e-14


def _oracle_precs(cfg, A, names, gather="recent", n_strips=None, overlap=None):
    return [sweep.make_preconditioner(cfg, A, nm, n_strips=n_strips, overlap=overlap, gather=gather) for nm in names]


@pytest.mark.parametrize("name", ["C1", "var", "C2", "C4s", "C5s"])
@pytest.mark.parametrize("nseg", [0, 1, 3])
def test_sweep_apply_parity(name, nseg):
    """All four double sweeps batched in one launch vs the oracle, per direction
    (<= 1e-10), with per-direction sources (ldr = n)."""
    cfg = CFGS[name]()
    if name == "C1" and nseg == 3:
        nseg = 2
    A = p1.assemble(cfg)
    names = ["LRL", "RLR", "BTB", "TBT"]
    prob = gpu_problem(cfg)
    dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap, n_segments=nseg) for nm in names]
    R = random_vector(cfg.n, 11, len(names))
    Z = torch.zeros((len(names), cfg.n), dtype=torch.complex128, device=DEV)
    hs.sweep_apply(dirs, to_dev(R), Z)
    Zh = Z.cpu().numpy()
    for k, P in enumerate(_oracle_precs(cfg, A, names)):
        z_ref = P.apply(R[k])
        assert rel(Zh[k], z_ref) <= 1e-10, (name, names[k], rel(Zh[k], z_ref))
        assert elementwise(Zh[k], z_ref) <= 1e-10, (name, names[k], elementwise(Zh[k], z_ref))


@pytest.mark.parametrize("kernel", ["dual", "fast", "general"])
@pytest.mark.parametrize("nseg", [16, 30])
def test_short_segments(kernel, nseg, knob):
    """Degenerate segment lengths: C1 (65 cross rows) with 16 / 30 segments has
    segments of 1-4 rows (odd and even, the step loop's tail, the ring across
    solves with very short phases) -- every kernel vs the oracle."""
    knob("sweep_kernel", KERNEL_KNOB[kernel])
    cfg = CFGS["C1"]()
    A = p1.assemble(cfg)
    names = ["LRL", "BTB"]
    prob = gpu_problem(cfg)
    dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap, n_segments=nseg) for nm in names]
    R = random_vector(cfg.n, 13, len(names))
    Z = torch.zeros((len(names), cfg.n), dtype=torch.complex128, device=DEV)
    hs.sweep_apply(dirs, to_dev(R), Z)
    assert hs.sweep_kernel_name().endswith({"dual": "dual", "fast": "fast", "general": "apply"}[kernel])
    Zh = Z.cpu().numpy()
    for k, P in enumerate(_oracle_precs(cfg, A, names)):
        assert rel(Zh[k], P.apply(R[k])) <= 1e-10, (kernel, nseg, names[k])


@pytest.mark.parametrize("wide_xinv", [False, True])
def test_wide_strips(wide_xinv, knob):
    """Block rows wider than 36 nodes (x-strips of 83 nodes): the general kernel,
    with the explicit separator-inverse rows formed in global memory (default)
    or with the reducer CTA's separator solve (no_wide_xinv knob) -- vs the oracle."""
    if not wide_xinv:
        knob("no_wide_xinv", 1)
    cfg = small_problem(160, 48, 12.0, seed=31, variable_c=True, n_strips=2, overlap=1)
    A = p1.assemble(cfg)
    names = ["LRL", "RLR", "BTB", "TBT"]
    prob = gpu_problem(cfg)
    dirs = [hs.Sweep(prob, nm, n_strips=2, overlap=1, n_segments=4) for nm in names]
    assert dirs[0].info().wmax > 36
    R = random_vector(cfg.n, 19, len(names))
    Z = torch.zeros((len(names), cfg.n), dtype=torch.complex128, device=DEV)
    hs.sweep_apply(dirs, to_dev(R), Z)
    assert hs.sweep_kernel_name() == "k_sweep_apply"
    Zh = Z.cpu().numpy()
    for k, P in enumerate(_oracle_precs(cfg, A, names, n_strips=2, overlap=1)):
        assert rel(Zh[k], P.apply(R[k])) <= 1e-10, (wide_xinv, names[k], rel(Zh[k], P.apply(R[k])))


@pytest.mark.parametrize("kernel", ["dual", "fast", "general"])
@pytest.mark.parametrize("name", ["var", "C2", "C5s"])
def test_sweep_kernels_parity(kernel, name, knob):
    """Every sweep kernel (sweep_kernel knob, read per call) against the oracle:
    two-chain block kernel (default), single-chain register-streaming kernel,
    general TMA-ring kernel."""
    knob("sweep_kernel", KERNEL_KNOB[kernel])
    cfg = CFGS[name]()
    A = p1.assemble(cfg)
    names = ["LRL", "RLR", "BTB", "TBT"]
    prob = gpu_problem(cfg)
    dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap) for nm in names]
    R = random_vector(cfg.n, 12, len(names))
    Z = torch.zeros((len(names), cfg.n), dtype=torch.complex128, device=DEV)
    hs.sweep_apply(dirs, to_dev(R), Z)
    Zh = Z.cpu().numpy()
    for k, P in enumerate(_oracle_precs(cfg, A, names)):
        z_ref = P.apply(R[k])
        assert rel(Zh[k], z_ref) <= 1e-10, (kernel, name, names[k], rel(Zh[k], z_ref))
        assert elementwise(Zh[k], z_ref) <= 1e-10, (kernel, name, names[k])


@pytest.mark.parametrize("names", [["LR", "RL", "BT", "TB"]])
def test_single_sweeps_and_broadcast(names):
    cfg = CFGS["var"]()
    A = p1.assemble(cfg)
    prob = gpu_problem(cfg)
    dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=1, n_segments=2) for nm in names]
    r = random_vector(cfg.n, 12)
    Z = torch.zeros((len(names), cfg.n), dtype=torch.complex128, device=DEV)
    hs.sweep_apply(dirs, to_dev(r), Z, ldr=0)
    for k, P in enumerate(_oracle_precs(cfg, A, names, overlap=1)):
        assert rel(Z[k].cpu().numpy(), P.apply(r)) <= 1e-10


def test_eight_directions_split_batch():
    """t = 8 with 33 segments needs 8 x 33 CTAs, more than the SMs: the apply
    runs as two co-resident half batches; every direction must equal its
    single-direction apply bit for bit (single applies are oracle-tested above)."""
    cfg = CFGS["C3"]()
    names = ["LRL", "RLR", "BTB", "TBT", "LR", "RL", "BT", "TB"]
    prob = gpu_problem(cfg)
    dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap) for nm in names]
    assert dirs[0].info().n_segments * len(names) > 148
    r = to_dev(random_vector(cfg.n, 21))
    Z = torch.zeros((len(names), cfg.n), dtype=torch.complex128, device=DEV)
    hs.sweep_apply(dirs, r, Z, ldr=0)
    for k, d in enumerate(dirs):
        z1 = torch.zeros((1, cfg.n), dtype=torch.complex128, device=DEV)
        hs.sweep_apply([d], r, z1, ldr=0)
        assert torch.equal(Z[k], z1[0]), names[k]


def test_core_gather_and_overlap0():
    cfg = small_problem(48, 36, 20.0, seed=8, variable_c=True, n_strips=4, overlap=0)
    A = p1.assemble(cfg)
    prob = gpu_problem(cfg)
    for gather, gname in ((0, "recent"), (1, "core")):
        dirs = [hs.Sweep(prob, nm, n_strips=4, overlap=0, gather=gather, n_segments=3) for nm in ["LRL", "TBT"]]
        r = random_vector(cfg.n, 13)
        Z = torch.zeros((2, cfg.n), dtype=torch.complex128, device=DEV)
        hs.sweep_apply(dirs, to_dev(r), Z, ldr=0)
        for k, P in enumerate(_oracle_precs(cfg, A, ["LRL", "TBT"], gather=gname, n_strips=4, overlap=0)):
            assert rel(Z[k].cpu().numpy(), P.apply(r)) <= 1e-10


def test_single_strip_is_exact_solve():
    cfg = small_problem(30, 30, 15.0, seed=9, variable_c=True)
    A = p1.assemble(cfg)
    import scipy.sparse.linalg as spla
    prob = gpu_problem(cfg)
    d = [hs.Sweep(prob, "LRL", n_strips=1, overlap=1, n_segments=4)]
    r = random_vector(cfg.n, 14)
    Z = torch.zeros((1, cfg.n), dtype=torch.complex128, device=DEV)
    hs.sweep_apply(d, to_dev(r), Z, ldr=0)
    assert rel(Z[0].cpu().numpy(), spla.spsolve(A.tocsc(), r)) <= 1e-11


@pytest.mark.parametrize("name,t", [("C1", 2), ("var", 4), ("C2", 4), ("C5s", 1), ("C5s", 2), ("C4s", 4)])
def test_mpgmres_parity(name, t):
    cfg = CFGS[name]()
    names = {1: ["LRL"], 2: ["LRL", "BTB"], 4: ["LRL", "RLR", "BTB", "TBT"]}[t]
    A = p1.assemble(cfg)
    b_ref = p1.load_vector(cfg)
    precs = _oracle_precs(cfg, A, names)
    x_ref, st_ref = krylov.mpgmres(A, [P.apply for P in precs], b_ref, tol=cfg.tol, maxit=200)
    prob = gpu_problem(cfg)
    dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap) for nm in names]
    b = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    prob.load_vector(to_dev(cfg.f.ravel()), b)
    x = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    _, st = hs.mpgmres_solve(prob, dirs, b, x, tol=cfg.tol, maxit=200)
    assert abs(st["iterations"] - st_ref.iterations) <= 1, (st["iterations"], st_ref.iterations)
    assert st["true_rel_res"] <= 10 * cfg.tol
    if st["iterations"] == st_ref.iterations:
        assert rel(x.cpu().numpy(), x_ref) <= 1e-8
        h = np.array(st["history"])
        assert np.max(np.abs(h - np.array(st_ref.history)) / np.array(st_ref.history)) <= 1e-6
    else:  # A23: compare at equal k
        x2, _ = krylov.mpgmres(A, [P.apply for P in precs], b_ref, tol=1e-300, maxit=st["iterations"])
        assert rel(x.cpu().numpy(), x2) <= 1e-8


@pytest.mark.parametrize("names", [["LRL", "LRL"], ["LRL", "BTB", "LRL", "BTB"]])
def test_mpgmres_deflation(names):
    """Duplicate preconditioners (D10 step 5, A21): the duplicate columns deflate
    in every iteration (||w|| <= 1e-10 ||A z||) inside the fused
    orthogonalisation -- zero V slots, intra-block projections through them --
    and the iterates match the oracle run with the same preconditioners."""
    cfg = CFGS["var"]()
    A = p1.assemble(cfg)
    b_ref = p1.load_vector(cfg)
    precs = _oracle_precs(cfg, A, names)
    x_ref, st_ref = krylov.mpgmres(A, [P.apply for P in precs], b_ref, tol=cfg.tol, maxit=200)
    prob = gpu_problem(cfg)
    dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap) for nm in names]
    b = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    prob.load_vector(to_dev(cfg.f.ravel()), b)
    x = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    _, st = hs.mpgmres_solve(prob, dirs, b, x, tol=cfg.tol, maxit=200)
    ndup = len(names) - len(set(names))
    assert st_ref.deflations == ndup * st_ref.iterations
    assert st["deflations"] == ndup * st["iterations"], (st["deflations"], st["iterations"])
    assert abs(st["iterations"] - st_ref.iterations) <= 1
    if st["iterations"] == st_ref.iterations:
        assert rel(x.cpu().numpy(), x_ref) <= 1e-8


@pytest.mark.parametrize("nx,ny,n_strips,overlap", [(4, 4, 2, 0), (6, 6, 2, 1), (3, 7, 1, 0)])
def test_tiny_grids(nx, ny, n_strips, overlap):
    """Smallest grids the method admits (strips of max(2l+1, 2) cells, 3-row
    cross directions, a single strip): every direction's apply and a t = 3
    solve (sum rule, A17/P:L154) against the oracle."""
    cfg = small_problem(nx, ny, 3.0, seed=nx * 10 + ny, variable_c=True, n_strips=n_strips, overlap=overlap)
    A = p1.assemble(cfg)
    names = ["LRL", "RLR", "BTB"]
    prob = gpu_problem(cfg)
    dirs = [hs.Sweep(prob, nm, n_strips=n_strips, overlap=overlap) for nm in names]
    R = random_vector(cfg.n, 17, len(names))
    Z = torch.zeros((len(names), cfg.n), dtype=torch.complex128, device=DEV)
    hs.sweep_apply(dirs, to_dev(R), Z)
    precs = _oracle_precs(cfg, A, names, n_strips=n_strips, overlap=overlap)
    for k, P in enumerate(precs):
        assert rel(Z[k].cpu().numpy(), P.apply(R[k])) <= 1e-10, names[k]
    b_ref = cfg.f.ravel()
    x_ref, st_ref = krylov.mpgmres(A, [P.apply for P in precs], b_ref, tol=1e-8, maxit=50)
    x = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    _, st = hs.mpgmres_solve(prob, dirs, to_dev(b_ref), x, tol=1e-8, maxit=50)
    assert abs(st["iterations"] - st_ref.iterations) <= 1
    assert rel(A @ x.cpu().numpy(), b_ref) <= 1e-7


def test_host_buffers_end_to_end():
    """The C ABI accepts host pointers (the end-to-end path stages them)."""
    cfg = CFGS["C1"]()
    prob = hs.Problem.from_config(cfg)
    b = np.zeros(cfg.n, dtype=np.complex128)
    b = prob.load_vector(cfg.f.ravel(), b)
    assert rel(b, p1.load_vector(cfg)) <= 1e-14
    dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap) for nm in cfg.dirs]
    x = np.zeros(cfg.n, dtype=np.complex128)
    x, st = hs.mpgmres_solve(prob, dirs, b, x, tol=cfg.tol)
    assert st["converged"] == 1
    A = p1.assemble(cfg)
    assert np.linalg.norm(p1.load_vector(cfg) - A @ x) / np.linalg.norm(b) <= 1e-5
    # oracle parity of the host-buffer path (A23: x at equal k)
    precs = _oracle_precs(cfg, A, cfg.dirs)
    x_ref, st_ref = krylov.mpgmres(A, [P.apply for P in precs], p1.load_vector(cfg), tol=cfg.tol, maxit=200)
    assert abs(st["iterations"] - st_ref.iterations) <= 1
    if st["iterations"] != st_ref.iterations:
        x_ref, _ = krylov.mpgmres(A, [P.apply for P in precs], p1.load_vector(cfg), tol=1e-300, maxit=st["iterations"])
    assert rel(x, x_ref) <= 1e-8
    # a host-buffer sweep apply, element-wise against the oracle
    r = random_vector(cfg.n, 23)
    Zh = np.zeros((len(dirs), cfg.n), dtype=np.complex128)
    Zh = hs.sweep_apply(dirs, r, Zh, ldr=0)
    for k, P in enumerate(precs):
        assert elementwise(Zh[k], P.apply(r)) <= 1e-10


def test_status_paths():
    """Error and early-exit paths of the ABI: directions of another problem size
    (HELM_EDIM), more than 8 directions (HELM_EINVAL), maxit reached
    (HELM_ENOCONV with the last iterate), and b = 0 (x = 0, no iteration)."""
    cfg = CFGS["C1"]()
    prob = gpu_problem(cfg)
    other = hs.Problem.from_config(CFGS["var"]())
    d1 = hs.Sweep(prob, "LRL", n_strips=4, overlap=0)
    d2 = hs.Sweep(other, "LRL", n_strips=5, overlap=1)
    r = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    Z = torch.zeros((2, cfg.n), dtype=torch.complex128, device=DEV)
    with pytest.raises(hs.HelmError) as ei:
        hs.sweep_apply([d1, d2], r, Z, ldr=0)
    assert ei.value.code == 2
    Z9 = torch.zeros((9, cfg.n), dtype=torch.complex128, device=DEV)
    with pytest.raises(hs.HelmError) as ei:
        hs.sweep_apply([d1] * 9, r, Z9, ldr=0)
    assert ei.value.code == 1
    b = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    prob.load_vector(to_dev(cfg.f.ravel()), b)
    x = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    _, st = hs.mpgmres_solve(prob, [d1], b, x, tol=1e-12, maxit=3)
    assert st["status"] == "HELM_ENOCONV" and st["iterations"] == 3 and len(st["history"]) == 3
    assert st["true_rel_res"] < 1.0 and torch.linalg.norm(x).item() > 0
    z0 = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    x0 = torch.ones(cfg.n, dtype=torch.complex128, device=DEV)
    _, st0 = hs.mpgmres_solve(prob, [d1], z0, x0, tol=1e-6)
    assert st0["iterations"] == 0 and torch.count_nonzero(x0).item() == 0


def test_invalid_arguments_raise():
    cfg = CFGS["C1"]()
    prob = gpu_problem(cfg)
    with pytest.raises(hs.HelmError) as ei:
        hs.Sweep(prob, "LRL", n_strips=40, overlap=1)     # 64/40 cells per strip: too thin
    assert ei.value.code == 1
    with pytest.raises(hs.HelmError):
        hs.Sweep(prob, "LRL", n_strips=4, overlap=1, n_segments=100)
    d = [hs.Sweep(prob, "LRL", n_strips=4, overlap=0)]
    b = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    x = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    with pytest.raises(hs.HelmError):
        hs.mpgmres_solve(prob, d, b, x, tol=2.0)


@pytest.mark.parametrize("names", [["LR", "RL"], ["LR", "BT", "RL", "TB"]])
def test_single_sweep_solves(names):
    """The paper's single-sweep combinations as MPGMRES solves (P:L154-156,
    Table 1 columns LR+RL and LR+BT+RL+TB): iteration count +-1 and x at equal
    k against the oracle."""
    cfg = CFGS["C2"]()
    A = p1.assemble(cfg)
    b_ref = p1.load_vector(cfg)
    precs = _oracle_precs(cfg, A, names)
    x_ref, st_ref = krylov.mpgmres(A, [P.apply for P in precs], b_ref, tol=cfg.tol, maxit=200)
    prob = gpu_problem(cfg)
    dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap) for nm in names]
    b = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    prob.load_vector(to_dev(cfg.f.ravel()), b)
    x = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    _, st = hs.mpgmres_solve(prob, dirs, b, x, tol=cfg.tol, maxit=200)
    assert st["converged"] == 1
    assert abs(st["iterations"] - st_ref.iterations) <= 1, (names, st["iterations"], st_ref.iterations)
    if st["iterations"] != st_ref.iterations:
        x_ref, _ = krylov.mpgmres(A, [P.apply for P in precs], b_ref, tol=1e-300, maxit=st["iterations"])
    assert rel(x.cpu().numpy(), x_ref) <= 1e-8


def test_problem_reused_across_t():
    """One problem handle, solves with t = 4 (maxit 3), t = 2, t = 4, t = 1: the
    cached Krylov workspace is sized in columns and for the largest t seen
    (a later solve with another t must not overrun V / Z / C1)."""
    cfg = CFGS["var"]()
    A = p1.assemble(cfg)
    b_ref = p1.load_vector(cfg)
    prob = gpu_problem(cfg)
    all_names = ["LRL", "RLR", "BTB", "TBT"]
    dirs = {nm: hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap) for nm in all_names}
    oracle = {nm: P for nm, P in zip(all_names, _oracle_precs(cfg, A, all_names))}
    b = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    prob.load_vector(to_dev(cfg.f.ravel()), b)
    for names, maxit, tol in ((all_names, 3, cfg.tol), (["LRL", "BTB"], 200, cfg.tol),
                              (all_names, 200, cfg.tol), (["LRL"], 200, 1e-10)):
        x = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
        _, st = hs.mpgmres_solve(prob, [dirs[nm] for nm in names], b, x, tol=tol, maxit=maxit)
        precs = [oracle[nm].apply for nm in names]
        x_ref, st_ref = krylov.mpgmres(A, precs, b_ref, tol=tol, maxit=maxit)
        assert abs(st["iterations"] - st_ref.iterations) <= 1, (names, st["iterations"], st_ref.iterations)
        if st["iterations"] != st_ref.iterations:
            x_ref, _ = krylov.mpgmres(A, precs, b_ref, tol=1e-300, maxit=st["iterations"])
        assert rel(x.cpu().numpy(), x_ref) <= 1e-8, names


def test_nonfinite_guard():
    """Failure detection: a NaN in b reaches the Krylov block; the solve stops
    with HELM_ENONFINITE instead of deflating the column silently."""
    cfg = CFGS["C1"]()
    prob = gpu_problem(cfg)
    d = [hs.Sweep(prob, "LRL", n_strips=4, overlap=0)]
    b = torch.ones(cfg.n, dtype=torch.complex128, device=DEV)
    b[17] = complex(float("nan"), 0.0)
    x = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    with pytest.raises(hs.HelmError) as ei:
        hs.mpgmres_solve(prob, d, b, x, tol=1e-6, maxit=5)
    assert ei.value.code == 8


def test_binding_checks_tensor_dtype_and_size():
    cfg = CFGS["C1"]()
    prob = gpu_problem(cfg)
    with pytest.raises(ValueError):
        prob.load_vector(to_dev(cfg.f.ravel()), torch.zeros(cfg.n, dtype=torch.complex64, device=DEV))
    with pytest.raises(ValueError):
        prob.load_vector(to_dev(cfg.f.ravel()), torch.zeros(cfg.n - 1, dtype=torch.complex128, device=DEV))


@pytest.mark.parametrize("kernel", ["dual", "fast", "general"])
def test_overlap2(kernel, knob):
    """Overlap l = 2 (two extra mesh lines per internal boundary, SURVEY §8(f) #4,
    P:L152 generalised): all four double sweeps vs the oracle on every kernel."""
    knob("sweep_kernel", KERNEL_KNOB[kernel])
    cfg = small_problem(60, 44, 18.0, seed=12, variable_c=True, n_strips=5, overlap=2)
    A = p1.assemble(cfg)
    names = ["LRL", "RLR", "BTB", "TBT"]
    prob = gpu_problem(cfg)
    dirs = [hs.Sweep(prob, nm, n_strips=5, overlap=2, n_segments=3) for nm in names]
    R = random_vector(cfg.n, 29, len(names))
    Z = torch.zeros((len(names), cfg.n), dtype=torch.complex128, device=DEV)
    hs.sweep_apply(dirs, to_dev(R), Z)
    Zh = Z.cpu().numpy()
    for k, P in enumerate(_oracle_precs(cfg, A, names, n_strips=5, overlap=2)):
        z = P.apply(R[k])
        assert rel(Zh[k], z) <= 1e-10 and elementwise(Zh[k], z) <= 1e-10, (kernel, names[k])


@pytest.mark.parametrize("name", ["C2", "C5s"])
def test_inexact_separator_fp32(name):
    """Opt-in inexact separator solve (sweep_set_precision(32)):
    the apply stays within 1e-5 of the oracle's exact sweep; MPGMRES with the
    inexact preconditioners converges with at most one extra iteration and its
    x satisfies the same residual tolerance; switching back to 64 bits restores
    the exact (1e-10) apply."""
    cfg = CFGS[name]()
    A = p1.assemble(cfg)
    names = ["LRL", "RLR", "BTB", "TBT"]
    prob = gpu_problem(cfg)
    dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap) for nm in names]
    precs = _oracle_precs(cfg, A, names)
    R = random_vector(cfg.n, 31, len(names))
    Z = torch.zeros((len(names), cfg.n), dtype=torch.complex128, device=DEV)
    for d in dirs:
        d.set_precision(32)
    hs.sweep_apply(dirs, to_dev(R), Z)
    Zh = Z.cpu().numpy()
    errs = [rel(Zh[k], P.apply(R[k])) for k, P in enumerate(precs)]
    assert max(errs) <= 1e-5 and max(errs) > 1e-12, errs          # inexact, and really used
    b = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    prob.load_vector(to_dev(cfg.f.ravel()), b)
    x = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    _, st = hs.mpgmres_solve(prob, dirs, b, x, tol=cfg.tol)
    x_ref, st_ref = krylov.mpgmres(A, [P.apply for P in precs], p1.load_vector(cfg), tol=cfg.tol, maxit=200)
    assert st["converged"] == 1 and st["iterations"] <= st_ref.iterations + 1
    assert st["true_rel_res"] <= 10 * cfg.tol
    assert rel(x.cpu().numpy(), x_ref) <= 1e-4
    for d in dirs:
        d.set_precision(64)
    hs.sweep_apply(dirs, to_dev(R), Z)
    assert max(rel(Z[k].cpu().numpy(), P.apply(R[k])) for k, P in enumerate(precs)) <= 1e-10


@pytest.mark.parametrize("chunks", [2, 3])
def test_setup_chunks(chunks, knob):
    """The setup_chunks schedule (strips pipelined on forked streams) forms the same
    factors: the batched apply equals the one-pass setup's bitwise and the oracle's."""
    cfg = CFGS["C2"]()
    names = ["LRL", "BTB"]
    prob = gpu_problem(cfg)
    R = to_dev(random_vector(cfg.n, 5, len(names)))
    Zs = []
    for ch in (1, chunks):
        knob("setup_chunks", ch)
        dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap) for nm in names]
        Z = torch.zeros((len(names), cfg.n), dtype=torch.complex128, device=DEV)
        hs.sweep_apply(dirs, R, Z)
        Zs.append(Z.cpu().numpy())
    assert np.array_equal(Zs[0], Zs[1])
    A = p1.assemble(cfg)
    Rh = R.cpu().numpy()
    for k, P in enumerate(_oracle_precs(cfg, A, names)):
        assert elementwise(Zs[1][k], P.apply(Rh[k])) <= 1e-10


@pytest.mark.parametrize("name", ["C2", "C5s"])
def test_two_level_separator_solve(name, knob):
    """The two-chain kernel's opt-in two-level separator solve (fine groups + coarse
    Schur system, sep_two_level knob, >= 8 separators) against the full explicit
    R^-1 rows (the default) and the oracle, element-wise."""
    cfg = CFGS[name]()
    names = ["LRL", "RLR", "BTB", "TBT"]
    prob = gpu_problem(cfg)
    R = to_dev(random_vector(cfg.n, 7, len(names)))
    Zs = []
    for two in (1, 0):
        knob("sep_two_level", two)
        dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap) for nm in names]
        assert dirs[0].info().n_segments - 1 >= 8
        Z = torch.zeros((len(names), cfg.n), dtype=torch.complex128, device=DEV)
        hs.sweep_apply(dirs, R, Z)
        assert hs.sweep_kernel_name() == "k_sweep_dual"
        Zs.append(Z.cpu().numpy())
        del dirs
    A = p1.assemble(cfg)
    Rh = R.cpu().numpy()
    for k, P in enumerate(_oracle_precs(cfg, A, names)):
        z_ref = P.apply(Rh[k])
        assert elementwise(Zs[0][k], z_ref) <= 1e-10, (name, k, elementwise(Zs[0][k], z_ref))
        assert elementwise(Zs[0][k], Zs[1][k]) <= 1e-11


@pytest.mark.parametrize("wide", [False, True])
def test_setup_reports_unfactorable_strip(wide):
    """Failure detection: a NaN wave speed poisons a strip block, no pivot
    compares > 0, and sweep_setup returns HELM_ESINGULAR instead of factors full of NaN --
    on the register-row Gauss-Jordan (strips <= 36 nodes) and on the blocked shared-memory
    one (wider strips)."""
    if wide:
        cfg = small_problem(160, 48, 12.0, seed=31, variable_c=True, n_strips=2, overlap=1)
    else:
        cfg = small_problem(40, 33, 25.0, seed=5, variable_c=True, n_strips=5, overlap=1)
    c = cfg.c.copy().ravel()
    c[c.size // 2] = np.nan
    prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, torch.tensor(c, dtype=torch.float64, device=DEV))
    with pytest.raises(hs.HelmError) as ei:
        hs.Sweep(prob, "LRL", n_strips=cfg.n_strips, overlap=cfg.overlap, n_segments=3)
    assert ei.value.code == 3, ei.value   # HELM_ESINGULAR
    # the library is still usable afterwards
    good = gpu_problem(cfg)
    d = hs.Sweep(good, "LRL", n_strips=cfg.n_strips, overlap=cfg.overlap, n_segments=3)
    assert d.info().wmax > 36 if wide else d.info().wmax <= 36
