"""Oracle: directional double (and single) sweeps.  TEST INFRASTRUCTURE ONLY.

Forward sweep (Eq. 2a-2c) and backward sweep (Eq. 3a-3c)
over the strips of oracle.strips, with the zeroth-order transmission operator
of Eq. 4 realised algebraically (D8).  Written step by step in the paper's
order:

  sweep order sigma = (1..N) for LRL/BTB, (N..1) for RLR/TBT; "prev"/"next"
  are the neighbours in sigma.
  Forward:  v_{s1} = A_{s1}^{-1} R r;  v_{sm} = A_{sm}^{-1}(R r + C^prev(v_{s(m-1)}))
            (Eq. 2b data from the previous subdomain, Eq. 2c homogeneous).
  Backward: u_{sN} = v_{sN} ("u_N = v_N");
            u_{sm} = A_{sm}^{-1}(R r + C^prev(v_{s(m-1)}) + C^next(u_{s(m+1)}))
            for m = N-1..1 (Eq. 3b: data from v_{s-1}; Eq. 3c: from u_{s+1}).
  => 2N - 1 local solves per double sweep (Pin-9).
  Gather "recent" ("the values from the most recent subdomain solve"):
  write u_{sN}, u_{s(N-1)}, ..., u_{s1} in that order, each overwriting.
  Gather "core" (A16 variant): node line L belongs to the strip with
  p_{s-1} <= L < p_s (last strip also takes p_N).

Local solves use SciPy's SuperLU (splu) on each strip matrix: the paper's
"using \\ for subdomain problems".

Exact-Schur test mode (D12): each A_s is replaced by the exact Schur
complement of A onto I_s, so the transmission data are exact DtN data and the
double sweep equals A^{-1} (the "nilpotent" exact sweep of P:L57-58).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import fd5
from . import p1
from . import strips as st_mod


class StripSolver:
    """One strip's local operator: either SuperLU of A_s (D7) or, in exact-Schur
    mode, a dense LU of the exact Schur complement (D12)."""

    def __init__(self, cfg, axis, strip, A, exact_schur=False, disc="p1"):
        self.strip = strip
        nodes = strip.nodes
        if not exact_schur:
            if disc == "fd5":    # five-point rows, ghost-point Robin interface rows (oracle/fd5.py)
                Atilde = fd5.local_matrix_global(cfg, axis, strip, A)
            else:                # P1 strip assembly with interface impedance edges (D7)
                Atilde = st_mod.local_matrix_global(cfg, axis, strip)
            self.Atilde = Atilde
            self.As = st_mod.restrict(Atilde, nodes)
            self.lu = spla.splu(self.As.tocsc())
            self.dense = None
        else:
            Ad = A.toarray()
            inside = np.zeros(cfg.n, dtype=bool)
            inside[nodes] = True
            out = np.where(~inside)[0]
            S = Ad[np.ix_(nodes, nodes)]
            if out.size:
                S = S - Ad[np.ix_(nodes, out)] @ np.linalg.solve(Ad[np.ix_(out, out)], Ad[np.ix_(out, nodes)])
            T = np.zeros((cfg.n, cfg.n), dtype=np.complex128)
            T[np.ix_(nodes, nodes)] = S
            self.Atilde = sp.csr_matrix(T)
            self.As = S
            self.lu = None
            self.dense = S
        self.corr = {}
        for side in ("low", "high"):
            has = strip.low_iface if side == "low" else strip.high_iface
            if has:
                self.corr[side] = st_mod.correction_operator(cfg, axis, strip, A, self.Atilde, side)

    def solve(self, rhs_local):
        if self.lu is not None:
            return self.lu.solve(rhs_local)
        return np.linalg.solve(self.dense, rhs_local)


class SweepPreconditioner:
    """z = M^{-1} r for one direction (LRL, RLR, BTB, TBT or the single sweeps
    LR, RL, BT, TB), built once ("factored once") and applied many times."""

    def __init__(self, cfg, A, axis, order, n_strips, overlap, double=True,
                 gather="recent", exact_schur=False, solvers_from=None, disc="p1"):
        self.cfg = cfg
        self.axis = axis
        self.order = order
        self.double = double
        self.gather = gather
        self.p, self.strips = st_mod.strips(cfg, axis, n_strips, overlap)
        if solvers_from is not None:
            # the same strips factored once serve both orders (LRL / RLR): the
            # strip solvers depend only on (axis, N, overlap), not on the order
            assert (solvers_from.axis, len(solvers_from.strips)) == (axis, n_strips)
            assert all(np.array_equal(a.nodes, b.nodes) for a, b in zip(solvers_from.strips, self.strips))
            self.solvers = solvers_from.solvers
        else:
            self.solvers = [StripSolver(cfg, axis, s, A, exact_schur, disc) for s in self.strips]
        N = n_strips
        self.sigma = list(range(N)) if order == 0 else list(range(N - 1, -1, -1))
        # "prev" interface of a strip = the side facing sigma's predecessor
        self.prev_side = "low" if order == 0 else "high"
        self.next_side = "high" if order == 0 else "low"
        self.n_solves = 0

    def _extend(self, s, v_local):
        v = np.zeros(self.cfg.n, dtype=np.complex128)
        v[self.strips[s].nodes] = v_local
        return v

    def _corr(self, s, side, v_local_of_neighbour, neighbour):
        """C_s^{side}(v) restricted to strip s's nodes (D8)."""
        vhat = self._extend(neighbour, v_local_of_neighbour)
        return (self.solvers[s].corr[side] @ vhat)[self.strips[s].nodes]

    def forward(self, r):
        sig = self.sigma
        N = len(sig)
        v = {}
        for m in range(N):
            s = sig[m]
            rhs = r[self.strips[s].nodes].astype(np.complex128)
            if m > 0:
                rhs = rhs + self._corr(s, self.prev_side, v[sig[m - 1]], sig[m - 1])
            v[s] = self.solvers[s].solve(rhs)
            self.n_solves += 1
        return v

    def backward(self, r, v):
        sig = self.sigma
        N = len(sig)
        u = {sig[N - 1]: v[sig[N - 1]]}
        for m in range(N - 2, -1, -1):
            s = sig[m]
            rhs = r[self.strips[s].nodes].astype(np.complex128)
            if m > 0:
                rhs = rhs + self._corr(s, self.prev_side, v[sig[m - 1]], sig[m - 1])
            rhs = rhs + self._corr(s, self.next_side, u[sig[m + 1]], sig[m + 1])
            u[s] = self.solvers[s].solve(rhs)
            self.n_solves += 1
        return u

    def gather_recent(self, sols, order_written):
        z = np.zeros(self.cfg.n, dtype=np.complex128)
        for s in order_written:
            z[self.strips[s].nodes] = sols[s]
        return z

    def gather_core(self, sols):
        z = np.zeros(self.cfg.n, dtype=np.complex128)
        n_axis = st_mod.axis_len(self.cfg, self.axis)
        N = len(self.strips)
        for s, st in enumerate(self.strips):
            hi = self.p[s + 1] if s == N - 1 else self.p[s + 1] - 1
            for L in range(self.p[s], hi + 1):
                nodes = st_mod.line_nodes(self.cfg, self.axis, L)
                loc = np.searchsorted(st.nodes, nodes)
                z[nodes] = sols[s][loc]
        assert n_axis == self.p[-1]
        return z

    def apply(self, r):
        r = np.asarray(r, dtype=np.complex128)
        v = self.forward(r)
        if self.double:
            u = self.backward(r, v)
            if self.gather == "core":
                return self.gather_core(u)
            # u_{sigma N} first, then u_{sigma(N-1)}, ..., u_{sigma 1}: most recent wins
            return self.gather_recent(u, list(reversed(self.sigma)))
        if self.gather == "core":
            return self.gather_core(v)
        # single sweep: v_{sigma 1}, ..., v_{sigma N} in solve order
        return self.gather_recent(v, list(self.sigma))


DIRS = {"LRL": (0, 0, True), "RLR": (0, 1, True), "BTB": (1, 0, True), "TBT": (1, 1, True),
        "LR": (0, 0, False), "RL": (0, 1, False), "BT": (1, 0, False), "TB": (1, 1, False)}


def make_preconditioner(cfg, A, name, n_strips=None, overlap=None, gather="recent",
                        exact_schur=False, solvers_from=None, disc="p1"):
    """``solvers_from``: an existing preconditioner on the same strips (same axis,
    N, overlap) whose factored strip solvers are reused -- no arithmetic change.
    ``disc``: "p1" (the hot path, D4/D7) or "fd5" (the paper's five-point
    scheme, oracle/fd5.py; A must then be fd5.assemble(cfg))."""
    axis, order, double = DIRS[name]
    return SweepPreconditioner(cfg, A, axis, order,
                               cfg.n_strips if n_strips is None else n_strips,
                               cfg.overlap if overlap is None else overlap,
                               double=double, gather=gather, exact_schur=exact_schur,
                               solvers_from=solvers_from, disc=disc)


def make_preconditioners(cfg, A, names, **kw):
    """make_preconditioner for several directions, factoring each set of strips
    (axis) once."""
    out, by_axis = [], {}
    for nm in names:
        ax = DIRS[nm][0]
        P = make_preconditioner(cfg, A, nm, solvers_from=by_axis.get(ax), **kw)
        by_axis.setdefault(ax, P)
        out.append(P)
    return out
