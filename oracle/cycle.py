"""ORACLE (test infrastructure only) -- multigrid cycle (§2.2, Alg. 2.1).

Alg. 2.1 with step 3 replaced by one recursive call (V-cycle) or
two (W-cycle); the coarsest level is solved directly (LU).
Relaxation (Eq. 3.8): u <- u + w_l B_l (f - A_l u).
"""
from __future__ import annotations

import numpy as np

from .hierarchy import coarse_solve


def smooth(hier, level, f, u):
    """One additive-Vanka relaxation on ``level``."""
    w = hier.opts.damping_at(level)
    return u + w * (hier.B[level] @ (f - hier.A[level] @ u))


def cycle(hier, level, f, u):
    """u <- MG(level, f, u), Alg. 2.1 applied recursively."""
    if level == hier.levels - 1:
        return coarse_solve(hier, f)
    A = hier.A[level]
    for _ in range(hier.opts.nu1):                        # step 1
        u = smooth(hier, level, f, u)
    rc = hier.R[level] @ (f - A @ u)                      # step 2
    ec = np.zeros(rc.shape, np.complex128)
    for _ in range(2 if hier.opts.cycle == "W" else 1):   # step 3 (recursive)
        ec = cycle(hier, level + 1, rc, ec)
    u = u + hier.P[level] @ ec                            # step 4
    for _ in range(hier.opts.nu2):                        # step 5
        u = smooth(hier, level, f, u)
    return u


def vcycle(hier, f, u=None):
    """One preconditioner application x = MG(f) (zero initial guess by default)."""
    f = np.asarray(f, np.complex128).ravel()
    u = np.zeros_like(f) if u is None else np.asarray(u, np.complex128).ravel()
    return cycle(hier, 0, f, u)
