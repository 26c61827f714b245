"""ORACLE (test infrastructure only) -- discretisation of Eq. 1.1.

H = L - diag(sigma) M   (Eq. 2.2 in 2D, Eq. 2.3 in 3D)
sigma   = omega^2 kappa^2 (1 - i gamma/omega)                  (Eq. 1.1)
sigma_s = omega^2 kappa^2 (1 - i (gamma/omega + alpha))        (Eq. 2.6,
          read as "the shift adds attenuation" with kappa^2 pointwise:
          SURVEY §8(c) A1, A2; readings R1, R2)

Grid: nodes = cells + 1 per axis, all nodes unknown, x-fastest linear index,
neighbours outside the domain are dropped (homogeneous Dirichlet by
truncation; reading A4/A5).  sigma multiplies row j (evaluated at the row's
centre node).
"""
from __future__ import annotations

import itertools

import numpy as np
import scipy.sparse as sp

COMPACT4 = "compact4"
FD2 = "fd2"


def node_coords(nodes):
    """Per-axis integer coordinates (x first) of every node, x-fastest order."""
    grids = np.meshgrid(*[np.arange(n) for n in nodes[::-1]], indexing="ij")
    # grids[k] is the coordinate along numpy axis k == physical axis dim-1-k
    return [g.ravel() for g in grids[::-1]]


def stencil_matrix(nodes, offsets, coefs):
    """Sparse A with A[j, j+o] = coefs[o][j] for every offset o whose neighbour
    j+o lies inside the grid (truncation = homogeneous Dirichlet).

    nodes: per-axis node counts (x first).  offsets: list of integer tuples
    (x first).  coefs: list of scalars or length-N arrays (value for row j).
    """
    nodes = tuple(int(n) for n in nodes)
    N = int(np.prod(nodes))
    coords = node_coords(nodes)
    strides = np.cumprod((1,) + nodes[:-1])
    rows, cols, vals = [], [], []
    for o, c in zip(offsets, coefs):
        mask = np.ones(N, dtype=bool)
        shift = 0
        for a, oa in enumerate(o):
            mask &= (coords[a] + oa >= 0) & (coords[a] + oa < nodes[a])
            shift += oa * int(strides[a])
        r = np.nonzero(mask)[0]
        v = np.broadcast_to(np.asarray(c, dtype=np.complex128), (N,))[r]
        rows.append(r)
        cols.append(r + shift)
        vals.append(v)
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = np.concatenate(vals)
    return sp.csr_matrix((vals, (rows, cols)), shape=(N, N))


def L_stencil(dim, h, kind=COMPACT4):
    """Offsets/coefficients of L.  COMPACT4: Eq. 2.2 / Eq. 2.3.
    FD2: the standard 2nd-order 5/7-point Laplacian (option a11)."""
    offs, cf = [], []
    if kind == FD2:
        offs.append((0,) * dim)
        cf.append(2.0 * dim / h ** 2)
        for a in range(dim):
            for s in (-1, 1):
                o = [0] * dim
                o[a] = s
                offs.append(tuple(o))
                cf.append(-1.0 / h ** 2)
        return offs, cf
    if dim == 2:
        # (1/h^2) [-1/6 -2/3 -1/6; -2/3 10/3 -2/3; -1/6 -2/3 -1/6]
        table = {0: 10.0 / 3.0, 1: -2.0 / 3.0, 2: -1.0 / 6.0}
        for o in itertools.product((-1, 0, 1), repeat=2):
            offs.append(o)
            cf.append(table[sum(abs(x) for x in o)] / h ** 2)
        return offs, cf
    # 3D: -1/(6h^2) * { [0 1 0;1 2 1;0 1 0], [1 2 1;2 -24 2;1 2 1], [0 1 0;1 2 1;0 1 0] }
    planes = {
        -1: np.array([[0, 1, 0], [1, 2, 1], [0, 1, 0]], float),
        0: np.array([[1, 2, 1], [2, -24, 2], [1, 2, 1]], float),
        1: np.array([[0, 1, 0], [1, 2, 1], [0, 1, 0]], float),
    }
    for oz in (-1, 0, 1):
        for oy in (-1, 0, 1):
            for ox in (-1, 0, 1):
                w = planes[oz][oy + 1, ox + 1]
                if w != 0.0:
                    offs.append((ox, oy, oz))
                    cf.append(-w / (6.0 * h ** 2))
    return offs, cf


def M_stencil(dim, kind=COMPACT4):
    """Offsets/coefficients of M: Eq. 2.2 (2D: 2/3 centre, 1/12 axis) and Eq. 2.3
    (3D: (1/12)*[6 centre, 1 on the six faces]).  FD2: identity."""
    if kind == FD2:
        return [(0,) * dim], [1.0]
    centre = 2.0 / 3.0 if dim == 2 else 0.5
    offs, cf = [(0,) * dim], [centre]
    for a in range(dim):
        for s in (-1, 1):
            o = [0] * dim
            o[a] = s
            offs.append(tuple(o))
            cf.append(1.0 / 12.0)
    return offs, cf


def sigma_fields(kappa, gamma, omega, alpha):
    """sigma (for H) and sigma_s (for H_s), flattened x-fastest (A1/A2)."""
    k2w2 = (np.asarray(kappa, float) ** 2 * omega ** 2).ravel()
    g = (np.asarray(gamma, float) / omega).ravel()
    sigma = k2w2 * (1.0 - 1j * g)
    sigma_s = k2w2 * (1.0 - 1j * (g + alpha))
    return sigma, sigma_s


def fine_operator(nodes, h, sigma, kind=COMPACT4):
    """H = L - diag(sigma) M on the grid."""
    dim = len(nodes)
    lo, lc = L_stencil(dim, h, kind)
    mo, mc = M_stencil(dim, kind)
    L = stencil_matrix(nodes, lo, lc)
    M = stencil_matrix(nodes, mo, mc)
    return (L - sp.diags(np.asarray(sigma, np.complex128)) @ M).tocsr()


def apply_helmholtz(A, x):
    """y = A x (plain sparse matvec)."""
    return A @ np.asarray(x, np.complex128).ravel()
