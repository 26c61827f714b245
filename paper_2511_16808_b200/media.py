"""Seeded synthetic inputs (media, absorbing layer, source, frequency).

This module is shared by the CUDA path's harness (tests, bench) and by the
CPU oracle.  It holds NONE of the method's arithmetic: it only produces the
problem data of Eq. 1.1 -- slowness kappa, attenuation gamma,
angular frequency omega and the source q -- with the shapes and structure of
the paper's workloads (§5; SURVEY.md §8(d) input recipe).

Conventions (SURVEY.md §8(c) readings A4, A14, A15, A16):
  * grid: ``cells`` per axis (x first), nodes = cells + 1, all nodes unknown,
    node index x-fastest.  Numpy arrays are shaped ``nodes[::-1]`` (z, y, x) so
    that ``ravel()`` gives the x-fastest linear index.
  * omega = 2*pi*v_min / (ppw * h)  ("10 grid points per
    wavelength", measured on the shortest wavelength).
  * absorbing layer: gamma = gamma_max * ((W - d)/W)^2 for
    d < W, d = min over axes of min(i, n_a - 1 - i) in nodes; 0 inside.
  * source: q = 1/h^d at one node ("point source").
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Problem", "sponge_gamma", "point_source", "omega_ppw", "config_problem",
    "homogeneous_problem", "linear_kappa2_problem", "layered2d_velocity",
    "thrust3d_velocity", "random_complex",
]


@dataclass
class Problem:
    """One Helmholtz problem instance (inputs of build_hierarchy + RHS)."""
    dim: int
    cells: tuple            # per axis, x first
    h: float
    kappa: np.ndarray       # slowness, shape nodes[::-1], float64
    gamma: np.ndarray       # attenuation (rad/s, same units as omega), float64
    omega: float
    q: np.ndarray           # complex128 RHS, shape nodes[::-1]
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def nodes(self):
        return tuple(c + 1 for c in self.cells)

    @property
    def n(self):
        return int(np.prod(self.nodes))


def _nodes(cells):
    return tuple(int(c) + 1 for c in cells)


def sponge_gamma(cells, width, gamma_max):
    """Quadratic absorbing-layer profile (reading A14 of the paper's "layer of
    ... grid cells of increasing attenuation")."""
    nodes = _nodes(cells)
    d = None
    for ax, n in enumerate(nodes):
        i = np.arange(n)
        da = np.minimum(i, n - 1 - i)
        shape = [1] * len(nodes)
        shape[len(nodes) - 1 - ax] = n
        da = da.reshape(shape)
        d = da if d is None else np.minimum(d, da)
    d = np.broadcast_to(d, nodes[::-1]).astype(np.float64)
    g = np.where(d < width, gamma_max * ((width - d) / width) ** 2, 0.0)
    return np.ascontiguousarray(g)


def point_source(cells, h, at=None):
    """q = 1/h^d at node ``at`` (x-first index tuple); default the centre node."""
    nodes = _nodes(cells)
    dim = len(nodes)
    if at is None:
        at = tuple((n - 1) // 2 for n in nodes)
    q = np.zeros(nodes[::-1], dtype=np.complex128)
    q[tuple(at[::-1])] = 1.0 / h ** dim
    return q


def omega_ppw(v_min, h, ppw):
    """omega for ``ppw`` points per shortest wavelength."""
    return 2.0 * math.pi * v_min / (ppw * h)


def homogeneous_problem(dim, n_cells, ppw=10.0, sponge=16, gamma_max_over_omega=2.0,
                        name="homogeneous"):
    """Configs 0, 1, 3 (and the paper's constant-model tables): unit cube, kappa=1."""
    cells = (n_cells,) * dim if np.isscalar(n_cells) else tuple(n_cells)
    h = 1.0 / cells[0]
    nodes = _nodes(cells)
    kappa = np.ones(nodes[::-1])
    omega = omega_ppw(1.0, h, ppw)
    gamma = sponge_gamma(cells, sponge, gamma_max_over_omega * omega)
    q = point_source(cells, h)
    return Problem(dim, cells, h, kappa, gamma, omega, q, name=name,
                   meta=dict(sponge=sponge, ppw=ppw, gmax=gamma_max_over_omega))


def linear_kappa2_problem(n_cells, ppw=10.0, sponge=20, gamma_max_over_omega=1.0):
    """PAPER.md:903-905 "Linear" model: kappa^2 varies linearly in the vertical
    direction over [0.25, 1] on [0,1]^2 (orientation: 0.25 at the top row y=0)."""
    cells = (n_cells, n_cells)
    h = 1.0 / n_cells
    nodes = _nodes(cells)
    y = np.arange(nodes[1]) / n_cells
    k2 = 0.25 + 0.75 * y
    kappa = np.sqrt(np.broadcast_to(k2[:, None], nodes[::-1])).copy()
    omega = omega_ppw(1.0, h, ppw)  # v_min = 1/kappa_max = 1
    gamma = sponge_gamma(cells, sponge, gamma_max_over_omega * omega)
    q = point_source(cells, h)
    return Problem(2, cells, h, kappa, gamma, omega, q, name="linear")


def _smooth_noise(rng, shape, sigma):
    from scipy.ndimage import gaussian_filter
    g = gaussian_filter(rng.standard_normal(shape), sigma=sigma, mode="reflect")
    return g / g.std()


def layered2d_velocity(nx_cells, nz_cells, h, seed=2, n_layers=12, vmin=1500.0, vmax=4500.0,
                       n_faults=2, pert=0.05):
    """Config 2 medium: dipping layers + normal faults +
    Gaussian-smoothed perturbation.  Returns velocity shaped (nz+1, nx+1)."""
    rng = np.random.default_rng(seed)
    nx, nz = nx_cells + 1, nz_cells + 1
    X, Z = nx_cells * h, nz_cells * h
    z0 = np.sort(rng.uniform(0.05, 0.95, n_layers - 1) * Z)
    s = rng.uniform(-0.15, 0.15, n_layers - 1)
    vint = np.sort(rng.uniform(vmin, vmax, n_layers - 2))
    vel_layers = np.concatenate([[vmin], vint, [vmax]])
    faults = []
    for _ in range(n_faults):
        xf = rng.uniform(0.2, 0.8) * X
        dip = math.radians(rng.uniform(60.0, 80.0))
        throw = rng.uniform(50.0, 300.0)
        faults.append((xf, dip, throw))
    x = np.arange(nx) * h
    z = np.arange(nz) * h
    XX, ZZ = np.meshgrid(x, z)          # (nz, nx)
    zeff = ZZ.copy()
    for xf, dip, throw in faults:
        hang = XX > xf + zeff / math.tan(dip)
        zeff = np.where(hang, zeff - throw, zeff)
    idx = np.zeros(XX.shape, dtype=np.int64)
    for k in range(n_layers - 1):
        zk = z0[k] + s[k] * (XX - X / 2)
        idx += (zeff > zk)
    v = vel_layers[idx]
    g = _smooth_noise(rng, (nz, nx), 3.0)
    v = np.clip(v * (1.0 + pert * g), vmin, vmax)
    return v


def thrust3d_velocity(cells, h, seed=4, n_layers=20, vmin=2000.0, vmax=6000.0, pert=0.03):
    """Config 4 medium: folded layers + one thrust fault +
    smoothed perturbation.  Returns velocity shaped (nz+1, ny+1, nx+1)."""
    rng = np.random.default_rng(seed)
    nx, ny, nz = (c + 1 for c in cells)
    X, Y, Z = (c * h for c in cells)
    m = n_layers - 1
    z0 = np.sort(rng.uniform(0.08, 0.95, m) * Z)
    A = rng.uniform(50.0, 400.0, m)
    lx = rng.uniform(3000.0, 12000.0, m)
    ly = rng.uniform(3000.0, 12000.0, m)
    phi = rng.uniform(0, 2 * math.pi, m)
    psi = rng.uniform(0, 2 * math.pi, m)
    vint = np.sort(rng.uniform(vmin, vmax, n_layers - 2))
    vel_layers = np.concatenate([[vmin], vint, [vmax]])
    xt = rng.uniform(0.3, 0.7) * X
    zt = rng.uniform(0.5, 0.9) * Z
    dip = math.radians(rng.uniform(20.0, 35.0))
    throw = rng.uniform(300.0, 800.0)
    x = np.arange(nx) * h
    y = np.arange(ny) * h
    z = np.arange(nz) * h
    v = np.empty((nz, ny, nx))
    zf = zt - (x - xt) * math.tan(dip)                  # (nx,)
    for iz in range(nz):
        zeff = np.where(z[iz] < zf, z[iz] + throw, z[iz])[None, :]   # (1, nx)
        idx = np.zeros((ny, nx), dtype=np.int64)
        for k in range(m):
            zk = z0[k] + A[k] * np.sin(2 * math.pi * x[None, :] / lx[k] + phi[k]) * \
                np.sin(2 * math.pi * y[:, None] / ly[k] + psi[k])
            idx += (zeff > zk)
        v[iz] = vel_layers[idx]
    g = _smooth_noise(rng, (nz, ny, nx), 3.0)
    v = np.clip(v * (1.0 + pert * g), vmin, vmax)
    return v


def config_problem(cfg, n=None, scale=1):
    """Problem for BASELINE.json configs[cfg].

    cfg 0: 2D 128^2, cfg 1: 2D n^2 (n in 512..4096), cfg 2: 2D 2048x640 layered,
    cfg 3: 3D 256^3 (or n^3), cfg 4: 3D 768^2x384 thrust (``scale`` divides the
    cell counts for scaled replicas; h is multiplied by ``scale``).
    """
    if cfg == 0:
        p = homogeneous_problem(2, 128, sponge=16, gamma_max_over_omega=2.0, name="config0")
        return p
    if cfg == 1:
        n = n or 4096
        return homogeneous_problem(2, n, sponge=16, gamma_max_over_omega=2.0, name=f"config1_N{n}")
    if cfg == 3:
        n = n or 256
        return homogeneous_problem(3, n, sponge=16, gamma_max_over_omega=2.0, name=f"config3_N{n}")
    if cfg == 2:
        cx, cz = 2048 // scale, 640 // scale
        h = 12.5 * scale
        v = layered2d_velocity(cx, cz, h, seed=2)
        cells = (cx, cz)
        kappa = 1.0 / v
        omega = omega_ppw(1500.0, h, 10.0)
        W = max(32 // scale, 4)
        gamma = sponge_gamma(cells, W, 2.0 * omega)
        q = point_source(cells, h, at=(cx // 2, W + 2))
        return Problem(2, cells, h, kappa, gamma, omega, q, name=f"config2_s{scale}",
                       meta=dict(sponge=W))
    if cfg == 4:
        cells = (768 // scale, 768 // scale, 384 // scale)
        h = 25.0 * scale
        v = thrust3d_velocity(cells, h, seed=4)
        kappa = 1.0 / v
        omega = omega_ppw(2000.0, h, 8.0)
        W = max(24 // scale, 4)
        gamma = sponge_gamma(cells, W, 2.0 * omega)
        q = point_source(cells, h, at=(cells[0] // 2, cells[1] // 2, W + 2))
        return Problem(3, cells, h, kappa, gamma, omega, q, name=f"config4_s{scale}",
                       meta=dict(sponge=W))
    raise ValueError(f"unknown config {cfg}")


def random_complex(shape, seed):
    """Seeded complex128 test vector, entries ~ N(0,1) + i N(0,1)."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
