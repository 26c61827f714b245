"""ORACLE (test infrastructure only) -- restarted flexible GMRES ("(flexible)
GMRES [saad1993flexible]"; P:824 GMRES(5)).

Saad's FGMRES(m) with right preconditioning, modified Gram-Schmidt Arnoldi and
Givens rotations; x0 = 0.  One iteration = one preconditioner
application.  Stop when the estimated relative residual |g_{j+1}|/||q|| < tol,
then form x and check the true relative residual; restart if it is not below
tol (reading A17).  c_f per Eq. 5.1 with a 5-iteration warm-up.
"""
from __future__ import annotations

import numpy as np


def convergence_factor(history, warmup=5):
    """c_f = (||r_k|| / ||r_0||)^(1/k), counted after ``warmup`` iterations (Eq. 5.1)."""
    h = np.asarray(history, float)
    if h.size <= warmup + 1:
        return float("nan")
    k = h.size - 1 - warmup
    return float((h[-1] / h[warmup]) ** (1.0 / k))


def fgmres_solve(A, q, precond, restart=20, tol=1e-6, maxiter=500, x0=None):
    """Solve A x = q.  ``A`` sparse (or callable), ``precond(v) -> z``.

    Returns (x, info) with info = dict(iterations, converged, history (estimated
    relres after each iteration, history[0] = 1), true_relres, restarts)."""
    matvec = A if callable(A) else (lambda v: A @ v)
    q = np.asarray(q, np.complex128).ravel()
    n = q.size
    x = np.zeros(n, np.complex128) if x0 is None else np.asarray(x0, np.complex128).ravel().copy()
    qnorm = np.linalg.norm(q)
    history = [1.0]
    its = 0
    converged = False
    true_rel = 1.0
    restarts = 0
    if qnorm == 0.0:
        return np.zeros(n, np.complex128), dict(iterations=0, converged=True, history=history,
                                                 true_relres=0.0, restarts=0)
    while its < maxiter:
        r = q - matvec(x)
        beta = np.linalg.norm(r)
        true_rel = beta / qnorm
        if true_rel < tol:
            converged = True
            break
        V = np.zeros((restart + 1, n), np.complex128)
        Z = np.zeros((restart, n), np.complex128)
        Hs = np.zeros((restart + 1, restart), np.complex128)
        cs = np.zeros(restart, np.complex128)
        sn = np.zeros(restart, np.complex128)
        g = np.zeros(restart + 1, np.complex128)
        g[0] = beta
        V[0] = r / beta
        j_end = 0
        stop = False
        for j in range(restart):
            Z[j] = precond(V[j])
            w = matvec(Z[j])
            for i in range(j + 1):                       # modified Gram-Schmidt
                Hs[i, j] = np.vdot(V[i], w)
                w = w - Hs[i, j] * V[i]
            Hs[j + 1, j] = np.linalg.norm(w)
            breakdown = Hs[j + 1, j] == 0.0
            if not breakdown:
                V[j + 1] = w / Hs[j + 1, j]
            for i in range(j):                           # previous rotations
                t = cs[i] * Hs[i, j] + sn[i] * Hs[i + 1, j]
                Hs[i + 1, j] = -np.conj(sn[i]) * Hs[i, j] + np.conj(cs[i]) * Hs[i + 1, j]
                Hs[i, j] = t
            a, b = Hs[j, j], Hs[j + 1, j]
            den = np.sqrt(abs(a) ** 2 + abs(b) ** 2)
            if den == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            elif abs(a) == 0.0:
                cs[j], sn[j] = 0.0, 1.0
            else:
                cs[j] = abs(a) / den
                sn[j] = (a / abs(a)) * np.conj(b) / den
            Hs[j, j] = cs[j] * a + sn[j] * b
            Hs[j + 1, j] = 0.0
            g[j + 1] = -np.conj(sn[j]) * g[j]
            g[j] = cs[j] * g[j]
            its += 1
            history.append(abs(g[j + 1]) / qnorm)
            j_end = j + 1
            if abs(g[j + 1]) / qnorm < tol or breakdown or its >= maxiter:
                stop = True
                break
        y = np.zeros(j_end, np.complex128)
        for i in range(j_end - 1, -1, -1):               # back substitution
            y[i] = (g[i] - Hs[i, i + 1:j_end] @ y[i + 1:j_end]) / Hs[i, i]
        x = x + y @ Z[:j_end]
        restarts += 1
        if stop:
            r = q - matvec(x)
            true_rel = np.linalg.norm(r) / qnorm
            if true_rel < tol:
                converged = True
                break
    return x, dict(iterations=its, converged=converged, history=history,
                   true_relres=float(true_rel), restarts=restarts)
