"""ORACLE (test infrastructure only) -- multigrid hierarchy for the shifted operator.

A_1 = H_s (fine, Eq. 2.6 with readings A1/A2)
A_{l+1} = R_l A_l P_l   Galerkin coarse operator, intergrid per the
                        chosen scheme (level-dependent by default)
Option REDISCRETIZE (north_star item 4 literal, reading A13): full-weighting
average of (omega^2 kappa^2, gamma/omega) to the coarse grid and the same
stencil at h_{l+1} = 2 h_l (P:323 mentions re-discretisation as the alternative
the paper does not use).
Smoother: additive Vanka (vanka.py), damping per level from Table 5.1
(P:761-780); the last value is reused beyond the table (reading A9).
Coarsest level: direct LU solve.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .operators import COMPACT4, fine_operator, sigma_fields
from .intergrid import LEVDEP, LIN, coarse_nodes, level_scheme, prolongation, restriction
from .vanka import ELEMENT, JACOBI, PLUS, RB, vanka_operator

GALERKIN = "galerkin"
REDISCRETIZE = "rediscretize"

# Table 5.1: per-level damping, fine level first.
DAMPING = {
    (2, JACOBI): [0.89, 0.9, 0.3, 0.71],
    (2, ELEMENT): [0.97, 0.66, 0.48, 0.88],
    (2, PLUS): [0.87, 0.57, 0.55, 0.74],
    (2, RB): [0.83, 0.5, 0.4, 0.65],
    (3, JACOBI): [0.6, 0.4, 0.3, 0.5],
    (3, ELEMENT): [1.1, 0.7, 0.45, 0.6],
    (3, PLUS): [0.92, 0.55, 0.45, 0.55],
}


@dataclass
class Options:
    dim: int
    cells: tuple
    h: float
    levels: int = 4
    nu1: int = 1
    nu2: int = 1
    cycle: str = "V"              # "V" or "W"
    fine_stencil: str = COMPACT4
    intergrid: str = LEVDEP
    coarse_op: str = GALERKIN
    smoother: str = RB
    damping: list = None

    def damping_at(self, level):
        d = self.damping if self.damping is not None else DAMPING[(self.dim, self.smoother)]
        return d[min(level, len(d) - 1)]


@dataclass
class Hierarchy:
    opts: Options
    omega: float
    alpha: float
    nodes: list = field(default_factory=list)    # per level, x first
    A: list = field(default_factory=list)        # per level operator (level 0 = H_s)
    R: list = field(default_factory=list)        # level l -> l+1
    P: list = field(default_factory=list)        # level l+1 -> l
    B: list = field(default_factory=list)        # Vanka operator per smoothing level
    cnt: list = field(default_factory=list)
    H: object = None                             # unshifted fine operator
    coarse_lu: object = None
    sigma: np.ndarray = None
    sigma_s: np.ndarray = None

    @property
    def levels(self):
        return len(self.A)


def _fw_average(nodes, field_):
    """Full-weighting average (row-normalised truncated lin R) -- REDISCRETIZE."""
    R = restriction(nodes, LIN)
    s = np.asarray(R.sum(axis=1)).ravel()
    return (R @ field_) / s


def build_hierarchy(opts: Options, kappa, omega, gamma, alpha, build_smoothers=True):
    """Setup (not part of time-to-solve)."""
    nodes = tuple(c + 1 for c in opts.cells)
    if opts.dim not in (2, 3) or len(nodes) != opts.dim:
        raise ValueError("dim")
    for c in opts.cells:
        if c < 4 or c % (2 ** (opts.levels - 1)) != 0:
            raise ValueError("cells must be divisible by 2^(levels-1)")
    sigma, sigma_s = sigma_fields(kappa, gamma, omega, alpha)
    hier = Hierarchy(opts, omega, alpha, sigma=sigma, sigma_s=sigma_s)
    hier.H = fine_operator(nodes, opts.h, sigma, opts.fine_stencil)
    A = fine_operator(nodes, opts.h, sigma_s, opts.fine_stencil)
    hier.nodes.append(nodes)
    hier.A.append(A)
    w2k2 = (np.asarray(kappa, float) ** 2 * omega ** 2).ravel()
    g = (np.asarray(gamma, float) / omega).ravel()
    h = opts.h
    for l in range(opts.levels - 1):
        rk, pk = level_scheme(opts.intergrid, l)
        R = restriction(nodes, rk)
        P = prolongation(nodes, pk)
        cn = tuple(coarse_nodes(n) for n in nodes)
        if opts.coarse_op == GALERKIN:
            Ac = (R @ A @ P).tocsr()
        else:
            w2k2 = _fw_average(nodes, w2k2)
            g = _fw_average(nodes, g)
            h = 2.0 * h
            Ac = fine_operator(cn, h, w2k2 * (1.0 - 1j * (g + alpha)), opts.fine_stencil)
        hier.R.append(R)
        hier.P.append(P)
        hier.nodes.append(cn)
        hier.A.append(Ac)
        nodes, A = cn, Ac
    if build_smoothers:
        for l in range(opts.levels - 1):
            B, cnt = vanka_operator(hier.A[l], hier.nodes[l], opts.smoother)
            hier.B.append(B)
            hier.cnt.append(cnt)
    Ac = hier.A[-1]
    if Ac.shape[0] <= 6000:
        hier.coarse_lu = ("dense", sla.lu_factor(Ac.toarray()))
    else:
        hier.coarse_lu = ("sparse", spla.splu(Ac.tocsc()))
    return hier


def coarse_solve(hier, r):
    kind, lu = hier.coarse_lu
    if kind == "dense":
        return sla.lu_solve(lu, r)
    return lu.solve(r)


def operator_complexity(hier):
    """Eq. 3.7: sum_l nnz(H_c^l) / nnz(H).  nnz counts stored
    entries of the SciPy products (exact cancellations are dropped by SciPy)."""
    nnz = [A.count_nonzero() for A in hier.A]
    return sum(nnz) / nnz[0]


def stencil_radius(A, nodes):
    """Largest Chebyshev distance between coupled nodes (P:364-365 stencil growth)."""
    A = A.tocoo()
    dim = len(nodes)
    strides = np.cumprod((1,) + tuple(nodes[:-1]))
    rr = np.zeros(A.nnz, dtype=np.int64)
    for a in range(dim - 1, -1, -1):
        ra = (A.row // strides[a]) % nodes[a]
        ca = (A.col // strides[a]) % nodes[a]
        rr = np.maximum(rr, np.abs(ra - ca))
    return int(rr.max())
