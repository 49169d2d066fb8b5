"""Oracle: five-point finite differences, the paper's own discretisation
(paper-calibration mode).  TEST INFRASTRUCTURE ONLY.

P:L152 (§4): "we make use of the standard five-point finite different
approximation on a regular Cartesian grid"; the benchmark source
f(x, y) = 3e4 exp(-200 k ((x-0.5)^2 + (y-0.5)^2)); the problem is Eq. 1a-1b
(P:L23-32), Delta u + k^2 u = f with du/dn - i k u = 0 on dOmega.

Reading (FD5 readings; SPEC helmholtz_fd, which the paper leaves
open): the system is A u = b with b = f sampled at every grid node and
  interior row     (u_E + u_W + u_N + u_S - 4 u) / h^2 + k^2 u
  boundary rows    ghost-point elimination of the centred normal derivative
                   through Eq. 1b: u_ghost = u_inward + 2 i k h u, so the
                   inward neighbour gets 2/h^2 and the diagonal + 2 i k / h
                   (both eliminations at a corner: + 4 i k / h).
Strip local matrices (Eq. 2-4 with the zeroth-order B = d/dn - i k of Eq. 4):
the global rows, except on an interface line, where the same ghost-point
elimination is applied towards the outside of the strip (the outward
neighbour is dropped, the inward one doubled, + 2 i k / h on the diagonal).
The transmission data then enter through the algebraic correction
(Atilde_s - A) v on the interface rows (oracle/strips.py D8), which equals
-(2/h) B(v) with B evaluated by the centred difference on the neighbour's
solution (SPEC strip_decomp trace_rhs).

The matrix is not symmetric (boundary rows couple inward with 2/h^2, the
inward row couples back with 1/h^2).  Unit wave speed (k given).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import p1


def source(cfg):
    """f = 3e4 exp(-200 k |x - (1/2, 1/2)|^2) at every node."""
    x, y = p1.node_xy(cfg)
    k = cfg.omega
    return 3.0e4 * np.exp(-200.0 * k * ((x - 0.5) ** 2 + (y - 0.5) ** 2)) + 0j


def assemble(cfg):
    """Global five-point matrix with ghost-point impedance rows (k = omega, c = 1)."""
    nx, ny, h, k = cfg.nx, cfg.ny, cfg.h, cfg.omega
    n = cfg.n
    I, J = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1))
    I = I.ravel()
    J = J.ravel()
    g = p1.node(cfg, I, J)
    rows, cols, vals = [g], [g], [np.full(n, -4.0 / h ** 2 + k * k + 0j)]
    for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1)):
        ii, jj = I + di, J + dj
        inside = (ii >= 0) & (ii <= nx) & (jj >= 0) & (jj <= ny)
        # a neighbour outside the grid is a ghost node: eliminated through Eq. 1b,
        # it adds 1/h^2 to the opposite (inward) neighbour and 2 i k / h to the diagonal
        rows.append(g[inside]); cols.append(p1.node(cfg, ii[inside], jj[inside]))
        vals.append(np.full(int(inside.sum()), 1.0 / h ** 2 + 0j))
        out = ~inside
        oi, oj = I[out] - di, J[out] - dj          # the inward neighbour of a ghost
        rows.append(g[out]); cols.append(p1.node(cfg, oi, oj))
        vals.append(np.full(int(out.sum()), 1.0 / h ** 2 + 0j))
        rows.append(g[out]); cols.append(g[out])
        vals.append(np.full(int(out.sum()), 2j * k / h))
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(n, n)).tocsr()


def local_matrix_global(cfg, axis, st, A):
    """Atilde_s: the global rows of the strip's nodes with the ghost-point
    Robin elimination of Eq. 4 on its interface lines, in global indexing
    (zero outside I_s)."""
    h, k = cfg.h, cfg.omega
    A = A.tocsr()
    n = cfg.n
    inside = np.zeros(n, dtype=bool)
    inside[st.nodes] = True
    x_idx = np.arange(n) % (cfg.nx + 1)
    y_idx = np.arange(n) // (cfg.nx + 1)
    line = x_idx if axis == 0 else y_idx
    step = 1 if axis == 0 else cfg.nx + 1            # global index step along the axis
    R = sp.diags(inside.astype(np.float64)) @ A     # the strip's rows
    R = R.tolil()
    for L, has, d in ((st.a, st.low_iface, -1), (st.b, st.high_iface, +1)):
        if not has:
            continue
        for q in np.where((line == L) & inside)[0]:
            outer, inner = q + d * step, q - d * step
            R[q, outer] = 0.0
            R[q, inner] = R[q, inner] + 1.0 / h ** 2
            R[q, q] = R[q, q] + 2j * k / h
    R = R.tocsr()
    R = R @ sp.diags(inside.astype(np.float64))     # columns outside I_s are exactly the dropped ones
    R.eliminate_zeros()
    return R.tocsr()
