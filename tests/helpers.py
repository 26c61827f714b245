"""Shared test helpers: build the oracle and the CUDA hierarchy from one seeded
problem (paper_2511_16808_b200.media), and compare vectors."""
from __future__ import annotations

import numpy as np

from paper_2511_16808_b200 import media

# Table 5.1, fine level first
DAMPING = {
    (2, "jacobi"): [0.89, 0.9, 0.3, 0.71],
    (2, "element"): [0.97, 0.66, 0.48, 0.88],
    (2, "plus"): [0.87, 0.57, 0.55, 0.74],
    (2, "rb"): [0.83, 0.5, 0.4, 0.65],
    (3, "jacobi"): [0.6, 0.4, 0.3, 0.5],
    (3, "element"): [1.1, 0.7, 0.45, 0.6],
    (3, "plus"): [0.92, 0.55, 0.45, 0.55],
}


def problem(dim, cells, ppw=10.0, sponge=4, hetero=True, seed=0):
    """Small seeded problem with a sponge and (optionally) a smooth random
    slowness field so that every per-node coefficient differs."""
    cells = tuple(cells)
    h = 1.0 / cells[0]
    nodes = tuple(c + 1 for c in cells)
    rng = np.random.default_rng(seed)
    kappa = np.ones(nodes[::-1])
    if hetero:
        kappa = 1.0 + 0.3 * rng.random(nodes[::-1])
    omega = media.omega_ppw(1.0 / kappa.max(), h, ppw)
    gamma = media.sponge_gamma(cells, sponge, 2.0 * omega)
    q = media.point_source(cells, h)
    return media.Problem(dim, cells, h, kappa, gamma, omega, q)


def build_pair(prob, alpha=0.3, levels=3, smoother=None, intergrid="levdep", coarse_op="galerkin",
               fine_stencil="compact4", cycle="V", dtype="c128", nu1=1, nu2=1, oracle=True):
    from paper_2511_16808_b200 import hmg
    from oracle.hierarchy import Options as OOptions, build_hierarchy
    dim = prob.dim
    smoother = smoother or ("rb" if dim == 2 else "element")
    damping = DAMPING[(dim, smoother)]
    opts = hmg.Options(dim=dim, cells=prob.cells, h=prob.h, levels=levels, nu1=nu1, nu2=nu2, cycle=cycle,
                       fine_stencil=fine_stencil, intergrid=intergrid, coarse_op=coarse_op, smoother=smoother,
                       damping=damping, dtype=dtype)
    gh = hmg.Hierarchy(opts, prob.kappa, prob.omega, prob.gamma, alpha)
    oh = None
    if oracle:
        oo = OOptions(dim=dim, cells=prob.cells, h=prob.h, levels=levels, nu1=nu1, nu2=nu2, cycle=cycle,
                      fine_stencil=fine_stencil, intergrid=intergrid, coarse_op=coarse_op, smoother=smoother,
                      damping=damping)
        oh = build_hierarchy(oo, prob.kappa, prob.omega, prob.gamma, alpha)
    return gh, oh


def to_dev(a, dtype="c128"):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, np.complex128).ravel()))
    return t.to(torch.complex64 if dtype == "c64" else torch.complex128).cuda()


def to_host(t):
    return t.detach().cpu().numpy().astype(np.complex128)


def rel_err(a, b):
    """max |a - b| / max |b| (elementwise comparison normalised by the scale)."""
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / (den if den > 0 else 1.0))


def stencil_from_sparse(A, nodes, r):
    """Oracle sparse matrix -> [K, N] coefficient array in the library's
    hmg_copy_stencil layout (offset index x-fastest over -r..r)."""
    A = A.tocoo()
    dim = len(nodes)
    N = int(np.prod(nodes))
    strides = np.cumprod((1,) + tuple(nodes[:-1]))
    w = 2 * r + 1
    K = w ** dim
    out = np.zeros((K, N), np.complex128)
    k = np.zeros(A.nnz, np.int64)
    mult = 1
    for a in range(dim):
        ra = (A.row // strides[a]) % nodes[a]
        ca = (A.col // strides[a]) % nodes[a]
        d = ca - ra
        assert np.all(np.abs(d) <= r), "oracle stencil wider than the radius"
        k += (d + r) * mult
        mult *= w
    np.add.at(out, (k, A.row), A.data)
    return out
