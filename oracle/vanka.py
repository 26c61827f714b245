"""ORACLE (test infrastructure only) -- additive Vanka smoother (§3.2-3.3).

S = I - w (sum_i V_i^T W_i H_i^{-1} V_i) A,   H_i = V_i A V_i^T     Eq. 3.8

Patches (Figs. 3.1/3.2):
  element : the 2^d vertices of one cell, one patch per cell
  plus    : centre + axis neighbours (5 in 2D / 7 in 3D)
  rb      : centre + same-colour neighbours of the compact stencil;
            2D X-shape centre + (+-1,+-1)
  jacobi  : one node (1x1 Vanka == damped Jacobi)
Boundary treatment: for every kind except element, one patch per
node, clipped to the domain (the "intersection of an entire patch with the
domain"); the weight of node j is 1/cnt_j with cnt_j = number of patches
that contain j.  Element patches get the 1/cnt weights too
(reading A7).  Patch matrices use the same shapes on every level with entries
taken from that level's operator (reading A8).  H_i^{-1} is a dense inverse
(LAPACK LU with partial pivoting via numpy.linalg.inv).
"""
from __future__ import annotations

import itertools

import numpy as np
import scipy.sparse as sp

from .operators import node_coords

ELEMENT = "element"
PLUS = "plus"
RB = "rb"
JACOBI = "jacobi"


def _patch_offsets(dim, kind):
    if kind == JACOBI:
        return [(0,) * dim]
    if kind == PLUS:
        offs = [(0,) * dim]
        for a in range(dim):
            for s in (-1, 1):
                o = [0] * dim
                o[a] = s
                offs.append(tuple(o))
        return offs
    if kind == RB:
        # same red-black colour within the compact (3^d) stencil: even coordinate sum
        offs = [o for o in itertools.product((-1, 0, 1), repeat=dim)
                if sum(abs(x) for x in o) % 2 == 0]
        offs.sort(key=lambda o: (sum(abs(x) for x in o), o))
        return offs
    if kind == ELEMENT:
        return list(itertools.product((0, 1), repeat=dim))
    raise ValueError(kind)


def patches(nodes, kind):
    """Index sets X_i.  Returns a list of (k, P_k) with P_k an int array
    (n_patches_k, k) of node indices: patches grouped by (clipped) size."""
    nodes = tuple(nodes)
    dim = len(nodes)
    N = int(np.prod(nodes))
    coords = node_coords(nodes)
    strides = np.cumprod((1,) + nodes[:-1])
    offs = _patch_offsets(dim, kind)
    if kind == ELEMENT:
        centres = np.ones(N, dtype=bool)
        for a in range(dim):
            centres &= coords[a] < nodes[a] - 1
        centres = np.nonzero(centres)[0]
    else:
        centres = np.arange(N)
    members = np.full((centres.size, len(offs)), -1, dtype=np.int64)
    for k, o in enumerate(offs):
        ok = np.ones(centres.size, dtype=bool)
        shift = 0
        for a, oa in enumerate(o):
            ca = coords[a][centres] + oa
            ok &= (ca >= 0) & (ca < nodes[a])
            shift += oa * int(strides[a])
        members[ok, k] = centres[ok] + shift
    sizes = (members >= 0).sum(axis=1)
    groups = []
    for s in np.unique(sizes):
        sel = members[sizes == s]
        # compact each row (keep patch-local order, drop clipped entries)
        order = np.argsort(sel < 0, axis=1, kind="stable")
        rows = np.take_along_axis(sel, order, axis=1)[:, :s]
        groups.append((int(s), np.ascontiguousarray(rows)))
    return groups


def patch_counts(nodes, kind):
    """cnt_j = number of patches containing node j."""
    N = int(np.prod(nodes))
    cnt = np.zeros(N, dtype=np.int64)
    for _, P in patches(nodes, kind):
        cnt += np.bincount(P.ravel(), minlength=N)
    return cnt


def patch_matrices(A, P):
    """Dense H_i = V_i A V_i^T for every patch row of P (n, k) -> (n, k, k)."""
    A = A.tocsr()
    n, k = P.shape
    H = np.empty((n, k, k), dtype=np.complex128)
    for a in range(k):
        for b in range(k):
            H[:, a, b] = np.asarray(A[P[:, a], P[:, b]]).ravel()
    return H


def vanka_operator(A, nodes, kind):
    """B = sum_i V_i^T W_i H_i^{-1} V_i as a sparse matrix (Eq. 3.8 without the
    damping and the trailing A), W_i(j,j) = 1/cnt_j."""
    N = int(np.prod(nodes))
    groups = patches(nodes, kind)
    cnt = np.zeros(N, dtype=np.int64)
    for _, P in groups:
        cnt += np.bincount(P.ravel(), minlength=N)
    rows, cols, vals = [], [], []
    for k, P in groups:
        Hinv = np.linalg.inv(patch_matrices(A, P))
        for a in range(k):
            for b in range(k):
                rows.append(P[:, a])
                cols.append(P[:, b])
                vals.append(Hinv[:, a, b] / cnt[P[:, a]])
    B = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(N, N))
    return B, cnt
