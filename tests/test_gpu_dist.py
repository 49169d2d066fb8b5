"""Direction-parallel MPGMRES (mpgmres_solve_dist) on one GPU.

* nranks = 1: identical to mpgmres_solve (bitwise).
* Two ranks emulated by two host threads on the one GPU (this pool has one GPU
  per call): each rank owns two of LRL, RLR, BTB, TBT, its own problem and sweep
  handles and stream; the all-gather callback is a host barrier plus device
  copies of the peer's columns.  No kernel waits on another rank's kernel (the
  ranks synchronise on the host only).  x, the iteration count and the residual
  history must equal the single-process t = 4 solve, and the oracle's.
"""
import ctypes
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2408_11929_b200 as hs
from helm_inputs import make_config
from oracle import krylov, p1, sweep

DEV = torch.device("cuda:0")
NAMES = ["LRL", "RLR", "BTB", "TBT"]


def setup_rank(cfg, names, stream):
    with torch.cuda.stream(stream):
        prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega,
                          torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=DEV), stream=stream.cuda_stream)
        dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap, stream=stream.cuda_stream)
                for nm in names]
        b = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
        prob.load_vector(torch.tensor(cfg.f.ravel(), device=DEV), b, stream=stream.cuda_stream)
        x = torch.zeros(cfg.n, dtype=torch.complex128, device=DEV)
    stream.synchronize()
    return prob, dirs, b, x


def test_dist_one_rank_is_mpgmres_solve():
    cfg = make_config(2)
    s = torch.cuda.Stream()
    prob, dirs, b, x = setup_rank(cfg, NAMES, s)
    _, st = hs.mpgmres_solve(prob, dirs, b, x, tol=cfg.tol, stream=s.cuda_stream)
    x1 = torch.zeros_like(x)
    cb = hs.ALLGATHER_FN(lambda *a: 1)            # never called with one rank
    _, st1 = hs.mpgmres_solve_dist(prob, dirs, 1, 0, b, x1, cb, tol=cfg.tol, stream=s.cuda_stream)
    s.synchronize()
    assert st1["iterations"] == st["iterations"] and torch.equal(x1, x)


class HostAllGather:
    """All-gather between ranks emulated as host threads on one GPU."""

    def __init__(self, nranks):
        self.nranks = nranks
        self.bar = threading.Barrier(nranks)
        self.slots = {}

    def callback(self, rank):
        def cb(ctx, send, recv, nbytes, stream):
            try:
                st = torch.cuda.ExternalStream(int(stream))
                st.synchronize()                      # this rank's columns are written
                self.slots[rank] = send
                self.bar.wait()
                with torch.cuda.stream(st):
                    for r in range(self.nranks):
                        if r == rank:
                            continue
                        src = torch.as_tensor(hs._Bytes(self.slots[r], nbytes, True), device="cuda")
                        dst = torch.as_tensor(hs._Bytes(recv + r * nbytes, nbytes, True), device="cuda")
                        dst.copy_(src)
                st.synchronize()
                self.bar.wait()                       # no rank reuses its buffers before the peers copied
                return 0
            except Exception:
                import traceback
                traceback.print_exc()
                self.bar.abort()
                return 1

        return hs.ALLGATHER_FN(cb)


@pytest.mark.parametrize("num", [2, 5])
def test_dist_two_ranks_emulated(num):
    cfg = make_config(num)
    # reference: single process, all four directions
    s0 = torch.cuda.Stream()
    prob0, dirs0, b0, x0 = setup_rank(cfg, NAMES, s0)
    _, st0 = hs.mpgmres_solve(prob0, dirs0, b0, x0, tol=cfg.tol, stream=s0.cuda_stream)
    s0.synchronize()
    parts = hs.partition_directions(NAMES, 2)
    ag = HostAllGather(2)
    cbs = [ag.callback(r) for r in range(2)]
    res = [None, None]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    ranks = [setup_rank(cfg, parts[r], streams[r]) for r in range(2)]

    def run(r):
        prob, dirs, b, x = ranks[r]
        res[r] = hs.mpgmres_solve_dist(prob, dirs, 2, r, b, x, cbs[r], tol=cfg.tol, stream=streams[r].cuda_stream)
        streams[r].synchronize()

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for r in range(2):
        x, st = res[r]
        assert st["iterations"] == st0["iterations"], (r, st["iterations"], st0["iterations"])
        assert st["history"] == st0["history"]
        assert torch.equal(x, x0), r
    if num == 2:   # and the oracle (A23)
        A = p1.assemble(cfg)
        precs = sweep.make_preconditioners(cfg, A, NAMES)
        xr, sr = krylov.mpgmres(A, [P.apply for P in precs], p1.load_vector(cfg), tol=cfg.tol, maxit=200)
        assert abs(sr.iterations - st0["iterations"]) <= 1
        if sr.iterations == st0["iterations"]:
            assert np.linalg.norm(x0.cpu().numpy() - xr) / np.linalg.norm(xr) <= 1e-8
