// p1_entries.cuh -- entries of the P1 Helmholtz matrix (global A and strip
// matrices A_s), computed per entry in gather form (deterministic, no atomics).
//
// A = -K + sum_T k_T^2 M_T + i sum_e k_e B_e     (Eq. 1a-1b)
// on the "/" mesh (D2): cell (ci,cj) -> T_L = {(ci,cj),(ci+1,cj),(ci+1,cj+1)}
// (right angle at (ci+1,cj)) and T_U = {(ci,cj),(ci+1,cj+1),(ci,cj+1)} (right
// angle at (ci,cj+1)).  Right isosceles P1 element: stiffness 1 at the right-
// angle vertex, 1/2 at the hypotenuse ends, -1/2 along a leg, 0 across the
// hypotenuse; mass h^2/24 [2 1 1; 1 2 1; 1 1 2]; edge mass h/6 [2 1; 1 2].
// k_T = omega / mean(c at vertices), k_e = omega / mean(c at ends) (D3, A5).
//
// A "selection" restricts the assembly to the cells of one strip plus its
// interface impedance edges (D7; Eq. 4 with the zeroth-order condition of
// P:L88-92): that is the strip's local matrix in global indexing.
#pragma once
#include "common.cuh"

struct GridView {
  int nx, ny;
  double h, omega;
  const double* c;  // nodal wave speed
};

struct CellSel {
  int axis;      // -1 = all cells, 0 = x-strip (cells ci in [lo,hi)), 1 = y-strip (cj in [lo,hi))
  int lo, hi;    // along-axis line range of the strip (cells lo..hi-1)
  int if_lo;     // impedance interface edges on line lo
  int if_hi;     // impedance interface edges on line hi
};

__host__ __device__ inline CellSel sel_all() { return CellSel{-1, 0, 0, 0, 0}; }

__device__ __forceinline__ double cnode(const GridView& g, int i, int j) {
  return g.c ? g.c[(long)j * (g.nx + 1) + i] : 1.0;
}

__device__ __forceinline__ bool cell_in(const GridView& g, const CellSel& s, int ci, int cj) {
  if (ci < 0 || cj < 0 || ci >= g.nx || cj >= g.ny) return false;
  if (s.axis == 0) return ci >= s.lo && ci < s.hi;
  if (s.axis == 1) return cj >= s.lo && cj < s.hi;
  return true;
}

// k_T^2 for T_L (upper = 0) or T_U (upper = 1) of cell (ci, cj)
__device__ __forceinline__ double kT2(const GridView& g, int ci, int cj, int upper) {
  double c0 = cnode(g, ci, cj), c2 = cnode(g, ci + 1, cj + 1);
  double c1 = upper ? cnode(g, ci, cj + 1) : cnode(g, ci + 1, cj);
  double k = g.omega / ((c0 + c1 + c2) / 3.0);
  return k * k;
}

__device__ __forceinline__ double kedge(const GridView& g, int i0, int j0, int i1, int j1) {
  return g.omega / ((cnode(g, i0, j0) + cnode(g, i1, j1)) / 2.0);
}

// element contribution of one triangle to a diagonal entry: -Kdiag + k^2 h^2/12
__device__ __forceinline__ double tri_diag(const GridView& g, const CellSel& s, int ci, int cj,
                                           int upper, double kdiag) {
  if (!cell_in(g, s, ci, cj)) return 0.0;
  return -kdiag + kT2(g, ci, cj, upper) * g.h * g.h / 12.0;
}
// ... to a leg entry: +1/2 + k^2 h^2/24; to a hypotenuse entry: k^2 h^2/24
__device__ __forceinline__ double tri_off(const GridView& g, const CellSel& s, int ci, int cj,
                                          int upper, double kneg) {
  if (!cell_in(g, s, ci, cj)) return 0.0;
  return kneg + kT2(g, ci, cj, upper) * g.h * g.h / 24.0;
}

// is the physical boundary edge owned by cell (ci,cj) selected?
__device__ __forceinline__ bool pedge(const GridView& g, const CellSel& s, int ci, int cj) {
  return cell_in(g, s, ci, cj);
}
// is the vertical edge (L,j)-(L,j+1) an interface edge of the selection?
__device__ __forceinline__ bool iface_v(const CellSel& s, int L) {
  return s.axis == 0 && ((s.if_lo && L == s.lo) || (s.if_hi && L == s.hi));
}
// horizontal edge (i,L)-(i+1,L)
__device__ __forceinline__ bool iface_h(const CellSel& s, int L) {
  return s.axis == 1 && ((s.if_lo && L == s.lo) || (s.if_hi && L == s.hi));
}

// Diagonal entry of node (i, j).
__device__ inline cplx entry_C(const GridView& g, const CellSel& s, int i, int j) {
  double re = 0.0, im = 0.0;
  // the 6 triangles around (i,j) with the node's stiffness diagonal
  re += tri_diag(g, s, i, j, 0, 0.5);          // T_L(i,j): hypotenuse end
  re += tri_diag(g, s, i, j, 1, 0.5);          // T_U(i,j): hypotenuse end
  re += tri_diag(g, s, i - 1, j, 0, 1.0);      // T_L(i-1,j): right angle
  re += tri_diag(g, s, i - 1, j - 1, 0, 0.5);  // T_L(i-1,j-1): hypotenuse end
  re += tri_diag(g, s, i - 1, j - 1, 1, 0.5);  // T_U(i-1,j-1): hypotenuse end
  re += tri_diag(g, s, i, j - 1, 1, 1.0);      // T_U(i,j-1): right angle
  const double eb = g.h / 3.0;                 // B_e diagonal 2h/6
  // physical impedance edges (owned by a cell) touching (i,j)
  if (j == 0) {
    if (i > 0 && pedge(g, s, i - 1, 0)) im += kedge(g, i - 1, 0, i, 0) * eb;
    if (i < g.nx && pedge(g, s, i, 0)) im += kedge(g, i, 0, i + 1, 0) * eb;
  }
  if (j == g.ny) {
    if (i > 0 && pedge(g, s, i - 1, g.ny - 1)) im += kedge(g, i - 1, j, i, j) * eb;
    if (i < g.nx && pedge(g, s, i, g.ny - 1)) im += kedge(g, i, j, i + 1, j) * eb;
  }
  if (i == 0) {
    if (j > 0 && pedge(g, s, 0, j - 1)) im += kedge(g, 0, j - 1, 0, j) * eb;
    if (j < g.ny && pedge(g, s, 0, j)) im += kedge(g, 0, j, 0, j + 1) * eb;
  }
  if (i == g.nx) {
    if (j > 0 && pedge(g, s, g.nx - 1, j - 1)) im += kedge(g, i, j - 1, i, j) * eb;
    if (j < g.ny && pedge(g, s, g.nx - 1, j)) im += kedge(g, i, j, i, j + 1) * eb;
  }
  // interface impedance edges (strip selections only)
  if (iface_v(s, i)) {
    if (j > 0) im += kedge(g, i, j - 1, i, j) * eb;
    if (j < g.ny) im += kedge(g, i, j, i, j + 1) * eb;
  }
  if (iface_h(s, j)) {
    if (i > 0) im += kedge(g, i - 1, j, i, j) * eb;
    if (i < g.nx) im += kedge(g, i, j, i + 1, j) * eb;
  }
  return cmk(re, im);
}

// East entry: (i,j)-(i+1,j), requires i < nx.
__device__ inline cplx entry_E(const GridView& g, const CellSel& s, int i, int j) {
  if (i >= g.nx) return cmk(0.0, 0.0);
  double re = tri_off(g, s, i, j, 0, 0.5) + tri_off(g, s, i, j - 1, 1, 0.5);  // two legs
  double im = 0.0;
  const double eo = g.h / 6.0;
  if (j == 0 && pedge(g, s, i, 0)) im += kedge(g, i, j, i + 1, j) * eo;
  if (j == g.ny && pedge(g, s, i, g.ny - 1)) im += kedge(g, i, j, i + 1, j) * eo;
  if (iface_h(s, j)) im += kedge(g, i, j, i + 1, j) * eo;
  return cmk(re, im);
}

// North entry: (i,j)-(i,j+1), requires j < ny.
__device__ inline cplx entry_N(const GridView& g, const CellSel& s, int i, int j) {
  if (j >= g.ny) return cmk(0.0, 0.0);
  double re = tri_off(g, s, i, j, 1, 0.5) + tri_off(g, s, i - 1, j, 0, 0.5);  // two legs
  double im = 0.0;
  const double eo = g.h / 6.0;
  if (i == 0 && pedge(g, s, 0, j)) im += kedge(g, i, j, i, j + 1) * eo;
  if (i == g.nx && pedge(g, s, g.nx - 1, j)) im += kedge(g, i, j, i, j + 1) * eo;
  if (iface_v(s, i)) im += kedge(g, i, j, i, j + 1) * eo;
  return cmk(re, im);
}

// North-east entry: (i,j)-(i+1,j+1) across the hypotenuse of cell (i,j).
__device__ inline cplx entry_NE(const GridView& g, const CellSel& s, int i, int j) {
  if (i >= g.nx || j >= g.ny) return cmk(0.0, 0.0);
  double re = tri_off(g, s, i, j, 0, 0.0) + tri_off(g, s, i, j, 1, 0.0);
  return cmk(re, 0.0);
}

// ---- generic strip coordinates: along-axis position pa, cross row c.
// axis 0: node (i, j) = (pa, c); axis 1: node (i, j) = (c, pa).
// "along" coupling (pa,c)-(pa+1,c); "cross" coupling (pa,c)-(pa,c+1);
// "diag" coupling (pa,c)-(pa+1,c+1) (the "/" diagonal is symmetric under i<->j).
__device__ __forceinline__ cplx gen_diag(const GridView& g, const CellSel& s, int axis, int pa, int c) {
  return axis == 0 ? entry_C(g, s, pa, c) : entry_C(g, s, c, pa);
}
__device__ __forceinline__ cplx gen_along(const GridView& g, const CellSel& s, int axis, int pa, int c) {
  return axis == 0 ? entry_E(g, s, pa, c) : entry_N(g, s, c, pa);
}
__device__ __forceinline__ cplx gen_cross(const GridView& g, const CellSel& s, int axis, int pa, int c) {
  return axis == 0 ? entry_N(g, s, pa, c) : entry_E(g, s, c, pa);
}
__device__ __forceinline__ cplx gen_ne(const GridView& g, const CellSel& s, int axis, int pa, int c) {
  return axis == 0 ? entry_NE(g, s, pa, c) : entry_NE(g, s, c, pa);
}
