"""Oracle: strip decomposition, local matrices and transmission corrections.
TEST INFRASTRUCTURE ONLY.

Follows P:L64 ("a simple sweep over N sequential subdomains with overlap"),
Fig. 1, P:L152 ("add one layer of mesh points for every internal
boundary ... overlap ... of width 2h") and Eq. 4 (zeroth-order
transmission operator B = d/dn - i k), in the discrete reading SURVEY D6-D8:

D6  strips along axis x (lines i = const; LRL/RLR) or y (lines j = const;
    BTB/TBT).  Partition lines p_0 = 0 < ... < p_N = n_axis, cell runs differ
    by <= 1, larger runs first (A12).  Strip s (0-based) spans lines
    a_s = max(p_s - l, 0) .. b_s = min(p_{s+1} + l, n_axis) over the full cross
    range; l = overlap (A11).
D7  local matrix A_s = the D4 assembly restricted to the strip's cells, the
    physical dOmega edges of those cells, and impedance edges i k_e B_e along
    line a_s (if s > 0) and line b_s (if s < N-1)  (Eq. 4 discretised, A13).
    Atilde_s = that assembly in global indexing.
D8  transmission correction for strip s and a neighbour solution v (extended
    by zero, v_hat):  C_s^Gamma(v) = [(Atilde_s - A) v_hat] restricted to the
    rows on interface line Gamma  (algebraic form of Eq. 2b, 3b, 3c).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import p1


@dataclass
class Strip:
    s: int
    a: int               # first line (along the axis)
    b: int               # last line
    nodes: np.ndarray    # sorted global node indices of I_s
    low_iface: bool      # has an interface on line a (s > 0)
    high_iface: bool     # has an interface on line b (s < N-1)


def partition_lines(n_axis: int, n_strips: int):
    """p_0 = 0 < p_1 < ... < p_N = n_axis; runs differ by <= 1, larger first (D6, A12)."""
    base, extra = divmod(n_axis, n_strips)
    runs = [base + (1 if s < extra else 0) for s in range(n_strips)]
    return np.concatenate([[0], np.cumsum(runs)]).astype(np.int64)


def axis_len(cfg, axis):
    return cfg.nx if axis == 0 else cfg.ny


def line_nodes(cfg, axis, L):
    """Global indices of the nodes on line L (i = L for axis 0, j = L for axis 1)."""
    if axis == 0:
        return p1.node(cfg, L, np.arange(cfg.ny + 1))
    return p1.node(cfg, np.arange(cfg.nx + 1), L)


def line_edges(cfg, axis, L):
    """The mesh edges lying on line L, as (m, 2) node pairs (interface edges, D7)."""
    nodes = line_nodes(cfg, axis, L)
    return np.stack([nodes[:-1], nodes[1:]], axis=1)


def strips(cfg, axis, n_strips, overlap):
    """Strip geometry (D6).  Raises ValueError for invalid decompositions
    (every strip needs >= max(2l+1, 2) cells along the axis)."""
    n_axis = axis_len(cfg, axis)
    if n_strips < 1:
        raise ValueError("n_strips must be >= 1")
    p = partition_lines(n_axis, n_strips)
    if np.min(np.diff(p)) < max(2 * overlap + 1, 2) and n_strips > 1:
        raise ValueError("strip too thin for the requested overlap")
    out = []
    for s in range(n_strips):
        a = max(p[s] - overlap, 0)
        b = min(p[s + 1] + overlap, n_axis)
        if axis == 0:
            I, J = np.meshgrid(np.arange(a, b + 1), np.arange(cfg.ny + 1))
        else:
            I, J = np.meshgrid(np.arange(cfg.nx + 1), np.arange(a, b + 1))
        nodes = np.sort(p1.node(cfg, I.ravel(), J.ravel()))
        out.append(Strip(s, a, b, nodes, s > 0, s < n_strips - 1))
    return p, out


def strip_cell_mask(cfg, axis, st: Strip):
    mask = np.zeros((cfg.ny, cfg.nx), dtype=bool)
    if axis == 0:
        mask[:, st.a:st.b] = True
    else:
        mask[st.a:st.b, :] = True
    return mask


def local_matrix_global(cfg, axis, st: Strip):
    """Atilde_s (D7) in global indexing."""
    extra = []
    if st.low_iface:
        extra.append(line_edges(cfg, axis, st.a))
    if st.high_iface:
        extra.append(line_edges(cfg, axis, st.b))
    extra = np.concatenate(extra) if extra else None
    return p1.assemble_general(cfg, strip_cell_mask(cfg, axis, st), extra)


def restrict(M, nodes):
    """M[I_s, I_s] for a global-indexed sparse matrix."""
    return M.tocsr()[nodes][:, nodes].tocsc()


def correction_operator(cfg, axis, st: Strip, A, Atilde, side):
    """The linear map v_hat -> C_s^Gamma(v_hat) (D8) as a sparse n x n matrix:
    rows of (Atilde_s - A) on interface line Gamma (side 'low' = line a_s,
    'high' = line b_s); all other rows zero."""
    L = st.a if side == "low" else st.b
    rows = line_nodes(cfg, axis, L)
    D = (Atilde - A).tocsr()
    sel = sp.diags(np.isin(np.arange(cfg.n), rows).astype(np.float64))
    return (sel @ D).tocsr()
