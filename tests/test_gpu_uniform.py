"""Uniform-box coefficient compression (k_uniform.cuh).

In a homogeneous medium every level's coefficients are identical at every node of an
interior box, and the kernels read one shared copy there.  The values and the
arithmetic are those of the stored path, so the output must be BIT-identical to a
hierarchy built with HMG_NO_UNIFORM=1 (stored planes everywhere).  Also checked:
the box found on the fine level is exactly the region the sponge profile (reading
A14) and the RB patch reach predict, and heterogeneous media get no box.
"""
import numpy as np
import pytest

from helpers import DAMPING, problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _pair(monkeypatch, p, levels, alpha, smoother, dtype):
    from paper_2511_16808_b200 import hmg
    opts = hmg.Options(dim=p.dim, cells=p.cells, h=p.h, levels=levels, smoother=smoother,
                       damping=DAMPING[(p.dim, smoother)], dtype=dtype)
    monkeypatch.delenv("HMG_NO_UNIFORM", raising=False)
    gu = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, alpha)
    monkeypatch.setenv("HMG_NO_UNIFORM", "1")
    gs = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, alpha)
    monkeypatch.delenv("HMG_NO_UNIFORM")
    return gu, gs


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("case", ["2d", "3d"])
def test_uniform_bit_identical(monkeypatch, case, dtype):
    import torch
    from paper_2511_16808_b200 import media
    if case == "2d":
        p, L, alpha, m, sm = media.config_problem(0), 4, 0.15, 10, "rb"
    else:
        p, L, alpha, m, sm = media.homogeneous_problem(3, 32, sponge=4), 3, 0.5, 10, "element"
    gu, gs = _pair(monkeypatch, p, L, alpha, sm, dtype)
    n0, lo, hi = gu.uniform_box(0)
    assert n0 > 0 and gs.uniform_box(0)[0] == 0
    assert gu.uniform_box(1)[0] > 0                 # the Galerkin level 1 is compressed too
    cdt = torch.complex64 if dtype == "c64" else torch.complex128
    q = torch.from_numpy(p.q.ravel()).to(cdt).cuda()
    x = torch.from_numpy(media.random_complex(p.n, 3)).to(cdt).cuda()
    for shifted in (False, True):
        yu, ys = torch.empty_like(x), torch.empty_like(x)
        gu.apply_helmholtz(x, yu, shifted=shifted)
        gs.apply_helmholtz(x, ys, shifted=shifted)
        assert torch.equal(yu, ys)
    for lvl in range(L - 1):
        N = gu.level_nodes(lvl)[0]
        f = torch.from_numpy(media.random_complex(N, 5 + lvl)).to(cdt).cuda()
        uu = torch.from_numpy(media.random_complex(N, 7 + lvl)).to(cdt).cuda()
        us = uu.clone()
        gu.smooth(f, uu, level=lvl)
        gs.smooth(f, us, level=lvl)
        assert torch.equal(uu, us), f"level {lvl}"
    zu, zs = torch.zeros_like(q), torch.zeros_like(q)
    gu.vcycle(q, zu)
    gs.vcycle(q, zs)
    assert torch.equal(zu, zs)
    xu, xs = torch.zeros_like(q), torch.zeros_like(q)
    ru = gu.fgmres_solve(q, xu, restart=m, tol=1e-6, maxiter=500)
    rs = gs.fgmres_solve(q, xs, restart=m, tol=1e-6, maxiter=500)
    assert ru.converged and ru.iterations == rs.iterations and ru.history == rs.history
    assert torch.equal(xu, xs)


def test_uniform_box_matches_sponge_geometry():
    """Config 0: gamma = 0 exactly for nodes at distance d >= W = 16 from the boundary
    (reading A14), so sigma is uniform on [16, 113)^2; the RB factors of node j also
    read sigma at j's diagonal neighbours, so the fine-level box is [17, 112)^2."""
    from paper_2511_16808_b200 import hmg, media
    p = media.config_problem(0)
    gh = hmg.Hierarchy(hmg.Options(dim=2, cells=p.cells, h=p.h, levels=4, damping=DAMPING[(2, "rb")]),
                       p.kappa, p.omega, p.gamma, 0.15)
    n, lo, hi = gh.uniform_box(0)
    assert (lo, hi) == ((17, 17), (112, 112)) and n == 95 * 95
    n1, lo1, hi1 = gh.uniform_box(1)
    assert 0 < n1 and lo1[0] > 8 and hi1[0] < 57          # inside the coarse image of the sponge
    assert gh.uniform_box(3)[0] == 0                      # coarsest: dense inverse, no box


def test_heterogeneous_has_no_box():
    from paper_2511_16808_b200 import hmg
    p = problem(2, (32, 32))          # random smooth kappa: every node differs
    gh = hmg.Hierarchy(hmg.Options(dim=2, cells=p.cells, h=p.h, levels=3, damping=DAMPING[(2, "rb")]),
                       p.kappa, p.omega, p.gamma, 0.3)
    assert all(gh.uniform_box(l)[0] == 0 for l in range(3))
