"""Seeded synthetic inputs for the five workloads (BASELINE.json configs).

This module is shared by the CPU oracle (``oracle/``) and the CUDA path
(``paper_2408_11929_b200``).  It holds NONE of the method's arithmetic: it only
produces the *inputs* of the problem -- grid geometry, the nodal wave speed
c(x, y), the angular frequency omega, the nodal complex source f(x, y) and the
strip/preconditioner parameters.  Everything derived from them (wavenumbers
per element/edge, the P1 matrix, the load vector b = M1 f, strips, factors) is
computed independently by each side.

Readings used (SURVEY.md §8(c) A6–A11):
  * A6  source amplitudes 1 (C1, C2, C4, C5) or e^{i phi} (C3); C4 sigma = 2h.
  * A7  seeds: numpy.random.default_rng(11929 + c), c = config number (1..5).
  * A8  "seeded random interior location" ~ U[0.1, 0.9]^2.
  * A9  C4 medium recipe (12 layers + smoothed Gaussian perturbation, 10 ppw).
  * A10 C4 "surface" source at (1.5, 0.98).
  * A11 overlap l: C1 0 ("non-overlapping"), C3 1 ("1-line overlap"), others 1.
  * A17/A18 preconditioner lists: t=2 -> LRL, BTB; t=4 -> LRL, RLR, BTB, TBT.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import math

import numpy as np

# direction codes: (axis, order). axis 0 = x (strips are vertical slabs, L/R),
# axis 1 = y (horizontal slabs, B/T). order 0 = increasing (LRL / BTB),
# order 1 = decreasing (RLR / TBT).
DIRECTIONS = {
    "LRL": (0, 0),
    "RLR": (0, 1),
    "BTB": (1, 0),
    "TBT": (1, 1),
}


@dataclass
class HelmConfig:
    name: str
    nx: int
    ny: int
    Lx: float
    Ly: float
    omega: float
    c: np.ndarray            # (ny+1, nx+1) nodal wave speed, float64
    f: np.ndarray            # (ny+1, nx+1) nodal complex source, complex128
    n_strips: int
    overlap: int
    dirs: list = field(default_factory=list)
    tol: float = 1e-6
    maxit: int = 200

    @property
    def h(self) -> float:
        return self.Lx / self.nx

    @property
    def n(self) -> int:
        return (self.nx + 1) * (self.ny + 1)

    @property
    def t(self) -> int:
        return len(self.dirs)


def _grid(nx, ny, h):
    x = np.arange(nx + 1) * h
    y = np.arange(ny + 1) * h
    X, Y = np.meshgrid(x, y)  # shape (ny+1, nx+1), [j, i]
    return X, Y


def gaussian(X, Y, x0, y0, sigma):
    """exp(-|x - x0|^2 / (2 sigma^2)) sampled at the nodes."""
    return np.exp(-((X - x0) ** 2 + (Y - y0) ** 2) / (2.0 * sigma * sigma))


def _c4_speed(nx, ny, h, rng):
    """A9: 12 equal-thickness layers, speeds ~ U[1.5, 4.5]; xi = white N(0,1)
    smoothed by a Gaussian filter of std (0.05/sqrt 2)/h nodes (covariance
    ~ exp(-r^2/(2*0.05^2))), scaled to max|xi| = 1; c = c_layer (1 + 0.1 xi)."""
    from scipy.ndimage import gaussian_filter

    speeds = rng.uniform(1.5, 4.5, 12)
    j = np.arange(ny + 1)
    layer = np.minimum((12 * j) // ny, 11)
    c_layer = speeds[layer][:, None] * np.ones((1, nx + 1))
    xi = rng.standard_normal((ny + 1, nx + 1))
    xi = gaussian_filter(xi, sigma=(0.05 / math.sqrt(2.0)) / h, mode="reflect")
    xi = xi / np.max(np.abs(xi))
    return c_layer * (1.0 + 0.1 * xi)


def make_config(num: int, *, nx: int | None = None, dirs=None) -> HelmConfig:
    """Build config C<num> (1..5) exactly as SURVEY.md §8(d) states.

    ``nx`` optionally overrides the grid size (for quick tests on a smaller
    grid of the same recipe); ``dirs`` overrides the preconditioner list.
    """
    rng = np.random.default_rng(11929 + num)
    if num == 1:
        n = nx or 64
        h = 1.0 / n
        X, Y = _grid(n, n, h)
        f = gaussian(X, Y, 0.5, 0.5, 0.02).astype(np.complex128)
        cfg = HelmConfig("C1", n, n, 1.0, 1.0, 20.0, np.ones_like(X), f, 4, 0,
                         ["LRL", "BTB"])
    elif num == 2:
        n = nx or 256
        h = 1.0 / n
        X, Y = _grid(n, n, h)
        x0 = rng.uniform(0.1, 0.9, size=2)
        f = gaussian(X, Y, x0[0], x0[1], h).astype(np.complex128)
        cfg = HelmConfig("C2", n, n, 1.0, 1.0, 100.0, np.ones_like(X), f, 8, 1,
                         ["LRL", "RLR", "BTB", "TBT"])
    elif num == 3:
        n = nx or 512
        h = 1.0 / n
        X, Y = _grid(n, n, h)
        pos = rng.uniform(0.1, 0.9, size=(3, 2))
        phi = rng.uniform(0.0, 2.0 * math.pi, 3)
        f = np.zeros_like(X, dtype=np.complex128)
        for m in range(3):
            f += np.exp(1j * phi[m]) * gaussian(X, Y, pos[m, 0], pos[m, 1], 2 * h)
        cfg = HelmConfig("C3", n, n, 1.0, 1.0, 200.0, np.ones_like(X), f, 16, 1,
                         ["LRL", "RLR", "BTB", "TBT"])
    elif num == 4:
        ny_ = (nx // 3) if nx else 512
        nx_ = 3 * ny_
        h = 1.0 / ny_
        X, Y = _grid(nx_, ny_, h)
        c = _c4_speed(nx_, ny_, h, rng)
        omega = 2.0 * math.pi * float(c.min()) / (10.0 * h)
        f = gaussian(X, Y, 1.5, 0.98, 2 * h).astype(np.complex128)
        cfg = HelmConfig("C4", nx_, ny_, 3.0, 1.0, omega, c, f, 16, 1,
                         ["LRL", "RLR", "BTB", "TBT"])
    elif num == 5:
        n = nx or 1024
        h = 1.0 / n
        X, Y = _grid(n, n, h)
        f = gaussian(X, Y, 0.5, 0.5, 2 * h).astype(np.complex128)
        cfg = HelmConfig("C5", n, n, 1.0, 1.0, 400.0, np.ones_like(X), f, 32, 1,
                         ["LRL", "RLR", "BTB", "TBT"])
    else:
        raise ValueError(f"unknown config {num}")
    if dirs is not None:
        cfg.dirs = list(dirs)
    return cfg


def random_vector(n: int, seed: int, ncols: int | None = None) -> np.ndarray:
    """Seeded complex128 test vector(s) with N(0,1) real and imaginary parts."""
    rng = np.random.default_rng(seed)
    shape = (n,) if ncols is None else (ncols, n)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def small_problem(nx: int, ny: int, omega: float, *, seed: int = 0,
                  variable_c: bool = False, n_strips: int = 2, overlap: int = 1,
                  dirs=("LRL", "BTB")) -> HelmConfig:
    """Tiny seeded problems for tests (uniform or random smooth c)."""
    rng = np.random.default_rng(seed)
    h = 1.0 / ny
    X, Y = _grid(nx, ny, h)
    if variable_c:
        c = 1.0 + 0.3 * rng.uniform(0.0, 1.0, size=X.shape)
    else:
        c = np.ones_like(X)
    f = (rng.standard_normal(X.shape) + 1j * rng.standard_normal(X.shape))
    return HelmConfig(f"small{nx}x{ny}", nx, ny, nx * h, 1.0, omega, c, f,
                      n_strips, overlap, list(dirs))
