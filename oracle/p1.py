"""Oracle: P1 discretisation of the impedance Helmholtz problem.  TEST INFRASTRUCTURE ONLY.

Model problem (Eq. 1a-1b):  Delta u + k^2 u = f in Omega,
du/dn - i k u = 0 on dOmega, with k = omega / c.

Weak form (paper sign, reading A3): for all test functions phi,
    -int grad u . grad phi + int k^2 u phi + i int_{dOmega} k u phi = int f phi,
so the matrix is  A = -K + sum_T k_T^2 M_T + i sum_e k_e B_e and
b = M1 f (consistent unit-coefficient mass times nodal f, reading A4 / D5).

Mesh (D1, D2): nodes (i, j) at (i h, j h), global index g = j (nx+1) + i; each
cell [i, i+1] x [j, j+1] is split along the "/" diagonal (i,j)-(i+1,j+1) into
    T_L = {(i,j), (i+1,j), (i+1,j+1)}   and   T_U = {(i,j), (i+1,j+1), (i,j+1)}.
Coefficients (D3, reading A5): k_T = omega / mean(c at the 3 vertices),
k_e = omega / mean(c at the 2 endpoints).

Everything here is written element by element from the textbook P1 formulas;
the only library primitive is scipy.sparse's COO -> CSR summation.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def node(cfg, i, j):
    """Global node index g = j (nx+1) + i  (D1)."""
    return np.asarray(j) * (cfg.nx + 1) + np.asarray(i)


def triangles(cfg):
    """All triangles as (ntri, 3) node-index arrays plus their (ntri,) cell
    coordinates (ci, cj).  Order: for every cell (row-major in j, then i),
    T_L then T_U (D2)."""
    nx, ny = cfg.nx, cfg.ny
    cj, ci = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    ci = ci.ravel()
    cj = cj.ravel()
    p00 = node(cfg, ci, cj)
    p10 = node(cfg, ci + 1, cj)
    p11 = node(cfg, ci + 1, cj + 1)
    p01 = node(cfg, ci, cj + 1)
    TL = np.stack([p00, p10, p11], axis=1)
    TU = np.stack([p00, p11, p01], axis=1)
    tri = np.empty((2 * ci.size, 3), dtype=np.int64)
    tri[0::2] = TL
    tri[1::2] = TU
    tci = np.repeat(ci, 2)
    tcj = np.repeat(cj, 2)
    return tri, tci, tcj


def node_xy(cfg):
    g = np.arange(cfg.n)
    i = g % (cfg.nx + 1)
    j = g // (cfg.nx + 1)
    return i * cfg.h, j * cfg.h


def p1_local_matrices(xy):
    """Textbook P1 element matrices for one triangle with vertex coordinates
    xy (3, 2): stiffness K_ab = |T| grad(phi_a) . grad(phi_b) and consistent
    mass M = |T|/12 [[2,1,1],[1,2,1],[1,1,2]]."""
    Mcoord = np.column_stack([np.ones(3), xy])          # phi_a = c0 + c1 x + c2 y
    coef = np.linalg.inv(Mcoord)                         # column a: coefficients of phi_a
    grads = coef[1:, :].T                                 # (3, 2)
    area = 0.5 * abs(np.linalg.det(Mcoord))
    K = area * grads @ grads.T
    M = area / 12.0 * np.array([[2.0, 1.0, 1.0], [1.0, 2.0, 1.0], [1.0, 1.0, 2.0]])
    return K, M


def boundary_edge_local(length):
    """P1 boundary mass on an edge: B_e = |e|/6 [[2,1],[1,2]]  (D4)."""
    return length / 6.0 * np.array([[2.0, 1.0], [1.0, 2.0]])


def element_k(cfg, tri):
    """k_T = omega / mean(c over the triangle's 3 vertices)  (D3, A5)."""
    c = cfg.c.ravel()
    return cfg.omega / (c[tri].sum(axis=1) / 3.0)


def edge_k(cfg, edges):
    """k_e = omega / mean(c over the edge's 2 endpoints)  (D3, A5)."""
    c = cfg.c.ravel()
    return cfg.omega / ((c[edges[:, 0]] + c[edges[:, 1]]) / 2.0)


def physical_edges(cfg):
    """Edges on dOmega (D4: the impedance edges of Eq. 1b) as (nedge, 2) node
    pairs, together with the cell (ci, cj) each edge belongs to."""
    nx, ny = cfg.nx, cfg.ny
    e, ci, cj = [], [], []
    i = np.arange(nx)
    # bottom j = 0, cell (i, 0); top j = ny, cell (i, ny-1)
    e.append(np.stack([node(cfg, i, 0), node(cfg, i + 1, 0)], 1)); ci.append(i); cj.append(np.zeros_like(i))
    e.append(np.stack([node(cfg, i, ny), node(cfg, i + 1, ny)], 1)); ci.append(i); cj.append(np.full_like(i, ny - 1))
    j = np.arange(ny)
    # left i = 0, cell (0, j); right i = nx, cell (nx-1, j)
    e.append(np.stack([node(cfg, 0, j), node(cfg, 0, j + 1)], 1)); ci.append(np.zeros_like(j)); cj.append(j)
    e.append(np.stack([node(cfg, nx, j), node(cfg, nx, j + 1)], 1)); ci.append(np.full_like(j, nx - 1)); cj.append(j)
    return np.concatenate(e), np.concatenate(ci), np.concatenate(cj)


def assemble_general(cfg, cell_mask=None, extra_edges=None):
    """Assemble  -K + sum_T k_T^2 M_T + i sum_e k_e B_e  in GLOBAL indexing over
    the cells selected by ``cell_mask`` ((ny, nx) bool; None = all cells), the
    physical boundary edges belonging to those cells, and the additional
    impedance edges ``extra_edges`` ((m, 2) node pairs; the interface edges of
    D7).  Returns an n x n scipy CSR matrix (complex128)."""
    tri, tci, tcj = triangles(cfg)
    if cell_mask is None:
        sel = np.ones(tri.shape[0], dtype=bool)
    else:
        sel = cell_mask[tcj, tci]
    tri = tri[sel]
    x, y = node_xy(cfg)
    kT = element_k(cfg, tri)
    rows, cols, vals = [], [], []
    # Element matrices from the vertex coordinates (p1_local_matrices).  The
    # mesh is uniform, so triangles fall into two shapes (T_L, T_U); each shape's
    # K and M is computed once from its own coordinates and applied to all
    # triangles of that shape with their own k_T^2.
    xy = np.stack([x[tri], y[tri]], axis=2)                     # (ntri, 3, 2)
    rel = np.round((xy - xy[:, :1, :]) / cfg.h).astype(np.int64).reshape(-1, 6)
    uniq, inv = np.unique(rel, axis=0, return_inverse=True)
    inv = inv.ravel()
    for u in range(uniq.shape[0]):
        K, M = p1_local_matrices(uniq[u].reshape(3, 2).astype(np.float64) * cfg.h)
        m = inv == u
        tr = tri[m]
        k2 = kT[m] ** 2
        for a in range(3):
            for bb in range(3):
                rows.append(tr[:, a])
                cols.append(tr[:, bb])
                vals.append(-K[a, bb] + k2 * M[a, bb] + 0j)
    # physical impedance edges of the selected cells
    pe, pci, pcj = physical_edges(cfg)
    if cell_mask is not None:
        pe = pe[cell_mask[pcj, pci]]
    edges = pe if extra_edges is None or len(extra_edges) == 0 else np.concatenate([pe, np.asarray(extra_edges)])
    if edges.shape[0]:
        ke = edge_k(cfg, edges)
        B = boundary_edge_local(cfg.h)
        for a in range(2):
            for bb in range(2):
                rows.append(edges[:, a])
                cols.append(edges[:, bb])
                vals.append(1j * ke * B[a, bb])
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = np.concatenate(vals)
    return sp.coo_matrix((vals, (rows, cols)), shape=(cfg.n, cfg.n)).tocsr()


def assemble(cfg):
    """The global matrix A (D4): all cells, all physical impedance edges."""
    return assemble_general(cfg)


def mass_unit(cfg):
    """M1: consistent P1 mass matrix with unit coefficient (D5)."""
    tri, _, _ = triangles(cfg)
    area = 0.5 * cfg.h * cfg.h
    M = area / 12.0 * np.array([[2.0, 1.0, 1.0], [1.0, 2.0, 1.0], [1.0, 1.0, 2.0]])
    rows, cols, vals = [], [], []
    for a in range(3):
        for bb in range(3):
            rows.append(tri[:, a]); cols.append(tri[:, bb]); vals.append(np.full(tri.shape[0], M[a, bb]))
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(cfg.n, cfg.n)).tocsr()


def load_vector(cfg, f_nodes=None):
    """b = M1 f_I, f_I = nodal values of the complex source (D5, reading A4)."""
    f = cfg.f.ravel() if f_nodes is None else np.asarray(f_nodes).ravel()
    return mass_unit(cfg) @ f


def manufactured_rhs(cfg, u_exact, grad_exact, k):
    """Manufactured-solution load (D5): f = 0 and inhomogeneous impedance data
    g = du*/dn - i k u* on dOmega.  The weak form gives
    -K u + k^2 M u + i k B u = -int_{dOmega} g phi, so b = -G with
    G_q = sum_{edges e containing q} (h/6)(2 g_q + g_other), g evaluated per edge
    with that edge's outward normal (handles corners).  Constant k only."""
    pe, _, _ = physical_edges(cfg)
    x, y = node_xy(cfg)
    nx, ny = cfg.nx, cfg.ny
    G = np.zeros(cfg.n, dtype=np.complex128)
    # normals per edge side
    nb = pe.shape[0]
    counts = [nx, nx, ny, ny]
    normals = [(0.0, -1.0), (0.0, 1.0), (-1.0, 0.0), (1.0, 0.0)]
    start = 0
    for cnt, (nxn, nyn) in zip(counts, normals):
        ed = pe[start:start + cnt]
        start += cnt
        for a, o in ((0, 1), (1, 0)):
            q = ed[:, a]
            r = ed[:, o]
            gq = grad_exact(x[q], y[q])[0] * nxn + grad_exact(x[q], y[q])[1] * nyn - 1j * k * u_exact(x[q], y[q])
            gr = grad_exact(x[r], y[r])[0] * nxn + grad_exact(x[r], y[r])[1] * nyn - 1j * k * u_exact(x[r], y[r])
            np.add.at(G, q, cfg.h / 6.0 * (2.0 * gq + gr))
    assert start == nb
    return -G
