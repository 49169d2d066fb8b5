"""Oracle: multipreconditioned GMRES.  TEST INFRASTRUCTURE ONLY.

Selective MPGMRES ("augment the search space by t additional vectors
at each iteration") with the paper's selection rules (for t = 2 "apply
the preconditioner only to the previous vector corresponding to the other
preconditioner"; for t > 2 "apply the preconditioner to the sum of all vectors
at the previous iteration"; at k = 1 all act on r0/||r0||), written
step by step as SURVEY D10:

  x0 = 0, beta = ||b||, V_1 = [b / beta] (origin tag: none)
  iteration k:
    1. sources by the selection rule (cross rule uses origin tags; after a
       deflation the surviving column feeds both, A19)
    2. Z_k[:, i] = M_i^{-1} src_i
    3. W = A Z_k                                   (t matvecs)
    4. BCGS2 against V_1..k: C1 = V^H W, W -= V C1; C2 = V^H W, W -= V C2;
       H block = C1 + C2      (block classical Gram-Schmidt, 2 passes; A20)
    5. intra-block CGS2 over W's columns i = 1..t (two projection passes
       against the already-accepted new columns); column i is dropped if its
       final norm <= 1e-10 * ||A z_i|| (its norm straight out of the matvec).
       Kept columns become V_{k+1} with origin tag i; their norms / projection
       coefficients are the new rows of H~.
    6. every Z column is kept (A21): a dropped column's H~ column has no new
       subdiagonal row, so A Z = V H~ stays exact.
    7. y = argmin ||beta e1 - H~ y|| ("minimises the Euclidean norm of
       the residual"); rho_k = ||beta e1 - H~ y|| / beta; stop if rho_k <= tol.
  finish: x = Z y.

Inner products use <u, v> = u^H v.  "paper" mode (single-pass block CGS and
single-pass intra-block CGS) exists to check the cost statement of P:L142:
(k - 1/2) t^2 + (3/2) t inner products per iteration (Pin-12).

The projected least-squares problem is solved with numpy.linalg.lstsq (a
library primitive standing in for "Householder QR of H~", reading A22).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

DEFLATION_TOL = 1e-10


@dataclass
class SolveStats:
    iterations: int = 0
    converged: bool = False
    exhausted: bool = False
    history: list = field(default_factory=list)      # rho_k per iteration
    matvecs: int = 0
    prec_applies: int = 0
    inner_products: list = field(default_factory=list)  # per iteration
    true_rel_res: float = float("nan")
    deflations: int = 0
    x_history: list = field(default_factory=list)


def _select_sources(k, t, Vblk, tags, v1):
    """Selection rule (D10 step 1; A19)."""
    if k == 1:
        return [v1] * t
    if Vblk.shape[1] == 0:
        raise RuntimeError("search space exhausted")
    if t == 1:
        return [Vblk[:, -1]]
    if t == 2:
        by_tag = {tags[c]: Vblk[:, c] for c in range(Vblk.shape[1])}
        if 0 in by_tag and 1 in by_tag:
            return [by_tag[1], by_tag[0]]   # M1 <- column from M2, M2 <- column from M1
        surv = Vblk[:, 0]
        return [surv, surv]
    s = Vblk.sum(axis=1)
    return [s] * t


def mpgmres(A, precs, b, tol=1e-6, maxit=200, mode="bcgs2", keep_x_history=False,
            return_basis=False):
    """Selective MPGMRES (D10).  ``A``: callable or matrix; ``precs``: list of
    callables r -> M_i^{-1} r.  Returns (x, SolveStats)."""
    Aop = A if callable(A) else (lambda v: A @ v)
    t = len(precs)
    b = np.asarray(b, dtype=np.complex128)
    n = b.size
    stats = SolveStats()
    beta = np.linalg.norm(b)
    if beta == 0.0:
        stats.converged = True
        return np.zeros(n, dtype=np.complex128), stats
    V = [b / beta]
    tags = [-1]
    blk_start = 0            # first column of V_k (the newest block)
    Zcols = []
    Hcols = []               # list of dense columns (variable length, padded later)
    two = mode == "bcgs2"
    y = None
    for k in range(1, maxit + 1):
        Vmat = np.column_stack(V)
        Vblk = Vmat[:, blk_start:]
        srcs = _select_sources(k, t, Vblk, tags[blk_start:], V[0])
        Zk = [precs[i](srcs[i]) for i in range(t)]
        stats.prec_applies += t
        W = np.column_stack([Aop(z) for z in Zk]).astype(np.complex128)
        stats.matvecs += t
        nAz = np.linalg.norm(W, axis=0)
        m = Vmat.shape[1]
        ip = 0
        # 4. block classical Gram-Schmidt against V_1..k (two passes in bcgs2)
        C1 = Vmat.conj().T @ W
        ip += m * t
        W = W - Vmat @ C1
        Hblk = C1
        if two:
            C2 = Vmat.conj().T @ W
            ip += m * t
            W = W - Vmat @ C2
            Hblk = C1 + C2
        # 5. intra-block CGS (two passes in bcgs2), deflation
        R = np.zeros((t, t), dtype=np.complex128)
        kept = []
        newV = []
        for i in range(t):
            w = W[:, i].copy()
            for _ in range(2 if two else 1):
                if kept:
                    Q = np.column_stack([newV[kept.index(j)] for j in kept])
                    c = Q.conj().T @ w
                    ip += len(kept)
                    w = w - Q @ c
                    R[kept, i] += c
            nrm = np.linalg.norm(w)
            ip += 1
            if nrm <= DEFLATION_TOL * nAz[i]:
                stats.deflations += 1
                continue
            R[i, i] = nrm
            kept.append(i)
            newV.append(w / nrm)
        stats.inner_products.append(ip)
        # 6. new H~ columns: rows 0..m-1 from Hblk, then one row per kept column
        for i in range(t):
            col = np.concatenate([Hblk[:, i], R[kept, i]])
            Hcols.append(col)
            Zcols.append(Zk[i])
        blk_start = m
        for j, i in enumerate(kept):
            V.append(newV[j])
            tags.append(i)
        # 7. projected least squares
        nrows = len(V)
        H = np.zeros((nrows, len(Hcols)), dtype=np.complex128)
        for c, col in enumerate(Hcols):
            H[:col.size, c] = col
        rhs = np.zeros(nrows, dtype=np.complex128)
        rhs[0] = beta
        y = np.linalg.lstsq(H, rhs, rcond=None)[0]
        rho = np.linalg.norm(rhs - H @ y) / beta
        stats.history.append(rho)
        stats.iterations = k
        if keep_x_history:
            stats.x_history.append(np.column_stack(Zcols) @ y)
        if rho <= tol:
            stats.converged = True
            break
        if not kept:
            stats.exhausted = True
            break
    x = np.column_stack(Zcols) @ y
    stats.true_rel_res = np.linalg.norm(b - Aop(x)) / beta
    if return_basis:
        return x, stats, (np.column_stack(V), np.column_stack(Zcols), H)
    return x, stats


def gmres_textbook(A, M, b, maxit):
    """Textbook right-preconditioned GMRES: Arnoldi with modified
    Gram-Schmidt on the Krylov space of A M^{-1}; x_k = Z_k y_k.  Returns the
    list of iterates x_1..x_maxit (for Pin-11)."""
    Aop = A if callable(A) else (lambda v: A @ v)
    b = np.asarray(b, dtype=np.complex128)
    beta = np.linalg.norm(b)
    V = [b / beta]
    Z = []
    H = np.zeros((maxit + 1, maxit), dtype=np.complex128)
    xs = []
    for j in range(maxit):
        z = M(V[j])
        Z.append(z)
        w = Aop(z)
        for i in range(j + 1):
            H[i, j] = np.vdot(V[i], w)
            w = w - H[i, j] * V[i]
        H[j + 1, j] = np.linalg.norm(w)
        V.append(w / H[j + 1, j])
        e1 = np.zeros(j + 2, dtype=np.complex128)
        e1[0] = beta
        y = np.linalg.lstsq(H[: j + 2, : j + 1], e1, rcond=None)[0]
        xs.append(np.column_stack(Z) @ y)
    return xs


def complete_mpgmres_residuals(A, precs, b, kmax):
    """Complete MPGMRES: at iteration k the search space is
    span{ p(M_1^{-1}A, ..., M_t^{-1}A) M_i^{-1} r0 } over all words of length
    < k in t non-commuting letters -- built here by brute-force enumeration of
    the words (small problems only).  Returns min-residual norms / ||b|| for
    k = 1..kmax."""
    Aop = A if callable(A) else (lambda v: A @ v)
    b = np.asarray(b, dtype=np.complex128)
    beta = np.linalg.norm(b)
    t = len(precs)
    frontier = [precs[i](b) for i in range(t)]          # words of length 1
    basis = list(frontier)
    out = []
    for k in range(1, kmax + 1):
        Zb = np.column_stack(basis)
        AZ = np.column_stack([Aop(z) for z in basis])
        # orthonormal basis of range(AZ) via SVD (rank-revealing)
        U, sv, _ = np.linalg.svd(AZ, full_matrices=False)
        r = int(np.sum(sv > sv[0] * 1e-12))
        U = U[:, :r]
        res = b - U @ (U.conj().T @ b)
        out.append(np.linalg.norm(res) / beta)
        if k < kmax:
            new = []
            for z in frontier:
                Az = Aop(z)
                for i in range(t):
                    new.append(precs[i](Az))
            frontier = new
            basis = basis + frontier
    return out
