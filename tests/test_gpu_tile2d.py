"""Shared-memory tiled 2D Galerkin-level stencil (k_stored_op2d_pair<..., TILE>; DESIGN.md
§5.2) against the gather it replaces (HMG_NO_TILE2D=1 at build): the same terms in the same
order, so every coarse-level residual, smoothing step and V-cycle must be
BIT-identical -- inside the uniform box, through the coefficient dictionary and on stored
planes (heterogeneous medium), for ragged tiles (level sizes not multiples of 64 x 16)."""
import pytest

from helpers import DAMPING, problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.parametrize("smoother", ["rb", "element", "plus"])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("case", ["homogeneous", "hetero"])
def test_tile2d_bit_identical(monkeypatch, case, dtype, smoother):
    import torch
    from paper_2511_16808_b200 import hmg, media
    if case == "homogeneous":
        p = media.homogeneous_problem(2, (272, 144), sponge=12)
    else:
        p = problem(2, (200, 136))
    opts = hmg.Options(dim=2, cells=p.cells, h=p.h, levels=4, smoother=smoother,
                       damping=DAMPING[(2, smoother)], dtype=dtype)
    monkeypatch.delenv("HMG_NO_TILE2D", raising=False)
    ga = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.5)
    monkeypatch.setenv("HMG_NO_TILE2D", "1")
    gb = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.5)
    monkeypatch.delenv("HMG_NO_TILE2D")
    cdt = torch.complex64 if dtype == "c64" else torch.complex128
    for lvl in range(1, 3):
        N = ga.level_nodes(lvl)[0]
        f = torch.from_numpy(media.random_complex(N, 3 + lvl)).to(cdt).cuda()
        x = torch.from_numpy(media.random_complex(N, 9 + lvl)).to(cdt).cuda()
        ra, rb = torch.empty_like(x), torch.empty_like(x)
        ga.residual(f, x, ra, level=lvl, shifted=True)
        gb.residual(f, x, rb, level=lvl, shifted=True)
        assert torch.equal(ra, rb), f"residual level {lvl}"
        ua, ub = x.clone(), x.clone()
        ga.smooth(f, ua, level=lvl)
        gb.smooth(f, ub, level=lvl)
        assert torch.equal(ua, ub), f"smooth level {lvl}"
    q = torch.from_numpy(p.q.ravel()).to(cdt).cuda()
    za, zb = torch.zeros_like(q), torch.zeros_like(q)
    ga.vcycle(q, za)
    gb.vcycle(q, zb)
    assert torch.equal(za, zb)
