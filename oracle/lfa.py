"""ORACLE (test infrastructure only) -- 2D local Fourier analysis (§2.4, §4).

Helmholtz symbol (Eq. 4.2):
    H~ = a + 2b cos t1 + 2b cos t2 + 4c cos t1 cos t2,
    a = 10/(3h^2) - 2 sigma/3,  b = -2/(3h^2) - sigma/12,  c = -1/(6h^2)
Vanka smoother symbol (Eq. 4.1):
    S~ = 1 - w (V^T W Phi^H H_i^{-1} Phi V) H~,  V = ones(N), W = I/N
with Phi and H_i of Eqs. 4.3-4.7 (element P:599-610, plus P:611-622, RB
P:623-637); Jacobi = 1x1 patch.
Intergrid symbols: bilinear (1/4)(1+cos t1)(1+cos t2),
bicubic (1/64) prod (3 + 4 cos t + cos 2t).
Two-grid symbol (Eq. 2.7) over the 4 harmonics (Def. 2.3),
H~_c = R~ H~ P~ with P~ = R~^T (the scale of P cancels in P H_c^{-1} R).
mu_loc = sup over T_high of |S~| (Def. 2.1), rho_loc = sup over T_low of
rho(TG~) (Def. 2.2), sampled at midpoints ("256x256 values").
Resonant samples with |H~_c| h^2 <= 1e-2 are excluded (the paper is silent;
reading A11).
"""
from __future__ import annotations

import numpy as np

PATCH_KINDS = ("jacobi", "element", "plus", "rb")


def abc(sigma, h):
    return 10.0 / (3 * h * h) - 2.0 * sigma / 3.0, -2.0 / (3 * h * h) - sigma / 12.0, \
        -1.0 / (6 * h * h)


def helmholtz_symbol(t1, t2, sigma, h):
    a, b, c = abc(sigma, h)
    return a + 2 * b * np.cos(t1) + 2 * b * np.cos(t2) + 4 * c * np.cos(t1) * np.cos(t2)


def _patch(kind, sigma, h):
    """(offsets, H_i) of Eqs. 4.3-4.7; offsets are the patch node positions."""
    a, b, c = abc(sigma, h)
    if kind == "jacobi":
        return [(0, 0)], np.array([[a]], complex)
    if kind == "element":
        offs = [(0, 0), (1, 0), (0, 1), (1, 1)]
        H = np.array([[a, b, b, c], [b, a, c, b], [b, c, a, b], [c, b, b, a]], complex)
        return offs, H
    if kind == "plus":
        offs = [(0, -1), (-1, 0), (0, 0), (1, 0), (0, 1)]
        H = np.array([[a, c, b, c, 0], [c, a, b, 0, c], [b, b, a, b, b],
                      [c, 0, b, a, c], [0, c, b, c, a]], complex)
        return offs, H
    if kind == "rb":
        offs = [(-1, -1), (1, -1), (0, 0), (-1, 1), (1, 1)]
        H = np.array([[a, 0, c, 0, 0], [0, a, c, 0, 0], [c, c, a, c, c],
                      [0, 0, c, a, 0], [0, 0, c, 0, a]], complex)
        return offs, H
    raise ValueError(kind)


def smoother_symbol(kind, t1, t2, sigma, h, w):
    """S~(theta) of Eq. 4.1 (vectorised over t1, t2 arrays)."""
    offs, H = _patch(kind, sigma, h)
    Hinv = np.linalg.inv(H)
    N = len(offs)
    t1 = np.asarray(t1, float)
    t2 = np.asarray(t2, float)
    phi = np.stack([np.exp(1j * (o[0] * t1 + o[1] * t2)) for o in offs], axis=-1)  # (..., N)
    # V^T W Phi^H Hinv Phi V = (1/N) sum_{k,l} conj(phi_k) Hinv[k,l] phi_l
    Bsym = np.einsum("...k,kl,...l->...", np.conj(phi), Hinv, phi) / N
    return 1.0 - w * Bsym * helmholtz_symbol(t1, t2, sigma, h)


def restriction_symbol(kind, t1, t2):
    if kind == "lin":
        return 0.25 * (1 + np.cos(t1)) * (1 + np.cos(t2))
    if kind == "cub":
        return (3 + 4 * np.cos(t1) + np.cos(2 * t1)) * (3 + 4 * np.cos(t2) + np.cos(2 * t2)) / 64.0
    raise ValueError(kind)


def _midpoints(lo, hi, n):
    step = (hi - lo) / n
    return lo + step * (np.arange(n) + 0.5)


def mu_loc(kind, sigma, h, w, n=256):
    """Smoothing factor (Def. 2.1) on n x n midpoint samples of [-pi/2, 3pi/2)^2."""
    t = _midpoints(-np.pi / 2, 3 * np.pi / 2, n)
    T1, T2 = np.meshgrid(t, t, indexing="ij")
    high = ~((np.abs(T1) < np.pi / 2) & (np.abs(T2) < np.pi / 2))
    S = smoother_symbol(kind, T1[high], T2[high], sigma, h, w)
    return float(np.abs(S).max())


def rho_loc(kind, sigma, h, w, intergrid=("cub", "cub"), nu1=1, nu2=1, n=256, excl=1e-2):
    """Two-grid factor (Def. 2.2, Eq. 2.7) on n x n midpoint samples of T_low."""
    t = _midpoints(-np.pi / 2, np.pi / 2, n)
    T1, T2 = np.meshgrid(t, t, indexing="ij")
    T1 = T1.ravel()
    T2 = T2.ravel()
    harm = [(T1, T2), (T1 + np.pi, T2 + np.pi), (T1 + np.pi, T2), (T1, T2 + np.pi)]
    Hd = np.stack([helmholtz_symbol(a, b, sigma, h) for a, b in harm], axis=-1)        # (M,4)
    Sd = np.stack([smoother_symbol(kind, a, b, sigma, h, w) for a, b in harm], axis=-1)
    Rr = np.stack([restriction_symbol(intergrid[0], a, b) for a, b in harm], axis=-1)
    Pp = np.stack([restriction_symbol(intergrid[1], a, b) for a, b in harm], axis=-1)
    Hc = np.sum(Rr * Hd * Pp, axis=-1)                                                   # (M,)
    keep = np.abs(Hc) * h * h > excl
    Hd, Sd, Rr, Pp, Hc = Hd[keep], Sd[keep], Rr[keep], Pp[keep], Hc[keep]
    M = Hd.shape[0]
    eye = np.broadcast_to(np.eye(4, dtype=complex), (M, 4, 4))
    CGC = eye - (Pp[:, :, None] / Hc[:, None, None]) * (Rr * Hd)[:, None, :]
    S = Sd[:, :, None] * eye
    TG = np.linalg.matrix_power(S, nu2) @ CGC @ np.linalg.matrix_power(S, nu1)
    return float(np.abs(np.linalg.eigvals(TG)).max())


def argmin_damping(fn, ws):
    vals = np.array([fn(w) for w in ws])
    return float(ws[int(np.argmin(vals))]), float(vals.min())
