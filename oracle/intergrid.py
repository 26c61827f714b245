"""ORACLE (test infrastructure only) -- intergrid operators (§3.1).

1D restriction weights centred at fine node 2I (coarse node I == fine node 2I):
  lin  [1 2 1]/4          -> 2D (1/16)[1 2 1]^T[1 2 1]          Eq. 3.1
  cub  [1 4 6 4 1]/16     -> 2D (1/256) outer([1 4 6 4 1])      Eq. 3.2
dD operators are Kronecker products (Eqs. 3.5-3.6).  Truncated at
the boundary without renormalisation (reading A5).
P = 2^d R^T of the P-kind weights ("P = 4 R^T" in 2D; 8 R^T in 3D, P:399
"defined similarly", reading A6).
Level-dependent scheme (Eqs. 3.3-3.4): (R,P) = (cub,cub) for
1->2 and (lin,cub) for k->k+1, k>1.
"""
from __future__ import annotations

from functools import reduce

import numpy as np
import scipy.sparse as sp

LIN = "lin"
CUB = "cub"
WEIGHTS = {LIN: np.array([1.0, 2.0, 1.0]) / 4.0,
           CUB: np.array([1.0, 4.0, 6.0, 4.0, 1.0]) / 16.0}

LEVDEP = "levdep"
LINEAR = "linear"
CUBIC = "cubic"
MIXED = "mixed"


def coarse_nodes(n_fine):
    assert (n_fine - 1) % 2 == 0, "cells must be even"
    return (n_fine - 1) // 2 + 1


def restriction_1d(n_fine, kind):
    """R[I, 2I+k] = w_k for 2I+k inside the grid (truncated)."""
    w = WEIGHTS[kind]
    r = len(w) // 2
    nc = coarse_nodes(n_fine)
    rows, cols, vals = [], [], []
    for I in range(nc):
        for k in range(-r, r + 1):
            i = 2 * I + k
            if 0 <= i < n_fine:
                rows.append(I)
                cols.append(i)
                vals.append(w[k + r])
    return sp.csr_matrix((vals, (rows, cols)), shape=(nc, n_fine))


def restriction(nodes, kind):
    """dD restriction = kron over axes; x fastest => kron(R_z, R_y, R_x)."""
    mats = [restriction_1d(n, kind) for n in nodes]   # x first
    return reduce(lambda a, b: sp.kron(a, b, format="csr"), mats[::-1]).tocsr()


def prolongation(nodes, kind):
    """P = 2^d R^T."""
    d = len(nodes)
    return (2.0 ** d * restriction(nodes, kind).T).tocsr()


def level_scheme(scheme, level):
    """(R kind, P kind) for the transfer level -> level+1 (0-based level)."""
    if scheme == LEVDEP:
        return (CUB, CUB) if level == 0 else (LIN, CUB)
    if scheme == LINEAR:
        return (LIN, LIN)
    if scheme == CUBIC:
        return (CUB, CUB)
    if scheme == MIXED:
        return (LIN, CUB)
    raise ValueError(scheme)
