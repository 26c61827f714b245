"""The z-marching staged 3D kernels (k_stage3d.cuh) against the
node-parallel gather kernels they replace (HMG_NO_STAGE3D=1 at build): same values,
same grouping of the stencil sums, so the outputs must be BIT-identical -- on ragged
grids (no dimension a multiple of the 32 x 8 x 32 tile), homogeneous (uniform box)
and heterogeneous media, both precisions, through the operator, one smoothing step,
the V-cycle and FGMRES.  Parity of either against the oracle is test_gpu_parity.py."""
import pytest

from helpers import DAMPING, problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("medium,cells,stencil", [
    ("homogeneous", (40, 24, 36), "compact4"),
    ("hetero", (20, 12, 68), "compact4"),
    ("hetero", (36, 20, 12), "fd2"),
])
def test_stage3d_bit_identical(monkeypatch, medium, cells, stencil, dtype):
    import torch
    from paper_2511_16808_b200 import hmg, media
    if medium == "homogeneous":
        p = media.homogeneous_problem(3, cells[0], sponge=4)
        p = media.Problem(3, cells, p.h, *_homog(cells, p.h, p.omega))
    else:
        p = problem(3, cells)
    opts = hmg.Options(dim=3, cells=p.cells, h=p.h, levels=3, smoother="element", fine_stencil=stencil,
                       damping=DAMPING[(3, "element")], dtype=dtype)
    monkeypatch.delenv("HMG_NO_STAGE3D", raising=False)
    ga = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.5)
    monkeypatch.setenv("HMG_NO_STAGE3D", "1")
    gb = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.5)
    monkeypatch.delenv("HMG_NO_STAGE3D")
    cdt = torch.complex64 if dtype == "c64" else torch.complex128
    x = torch.from_numpy(media.random_complex(p.n, 1)).to(cdt).cuda()
    f = torch.from_numpy(media.random_complex(p.n, 2)).to(cdt).cuda()
    for shifted in (False, True):
        ya, yb = torch.empty_like(x), torch.empty_like(x)
        ga.apply_helmholtz(x, ya, shifted=shifted)
        gb.apply_helmholtz(x, yb, shifted=shifted)
        assert torch.equal(ya, yb)
        ga.residual(f, x, ya, shifted=shifted)
        gb.residual(f, x, yb, shifted=shifted)
        assert torch.equal(ya, yb)
    ua, ub = x.clone(), x.clone()
    ga.smooth(f, ua)
    gb.smooth(f, ub)
    assert torch.equal(ua, ub)
    q = torch.from_numpy(p.q.ravel()).to(cdt).cuda()
    za, zb = torch.zeros_like(q), torch.zeros_like(q)
    ga.vcycle(q, za)
    gb.vcycle(q, zb)
    assert torch.equal(za, zb)
    xa, xb = torch.zeros_like(q), torch.zeros_like(q)
    ra = ga.fgmres_solve(q, xa, restart=10, tol=1e-6, maxiter=300)
    rb = gb.fgmres_solve(q, xb, restart=10, tol=1e-6, maxiter=300)
    assert ra.iterations == rb.iterations and ra.history == rb.history
    assert torch.equal(xa, xb)


def _homog(cells, h, omega):
    """kappa = 1 with a 4-node sponge on a non-cubic grid, centre source."""
    from paper_2511_16808_b200 import media
    import numpy as np
    nodes = tuple(c + 1 for c in cells)
    kappa = np.ones(nodes[::-1])
    gamma = media.sponge_gamma(cells, 4, 2.0 * omega)
    q = media.point_source(cells, h)
    return kappa, gamma, omega, q


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("cells,intergrid", [((20, 12, 68), "levdep"), ((24, 16, 36), "linear")])
def test_zblock3_transfers_bit_identical(monkeypatch, dtype, cells, intergrid):
    """3D restriction (fine level, 4 coarse planes per thread, each fine plane reduced once) and
    prolongation (4 coarse planes per thread, coarse windows reused) against the per-node kernels
    (HMG_NO_ZBLOCK3=1): bit-identical restrictions, prolongations, V-cycles; ragged plane counts."""
    import torch
    from paper_2511_16808_b200 import hmg, media
    p = problem(3, cells)
    opts = hmg.Options(dim=3, cells=p.cells, h=p.h, levels=3, smoother="element", intergrid=intergrid,
                       damping=DAMPING[(3, "element")], dtype=dtype)
    monkeypatch.delenv("HMG_NO_ZBLOCK3", raising=False)
    ga = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.5)
    monkeypatch.setenv("HMG_NO_ZBLOCK3", "1")
    gb = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.5)
    monkeypatch.delenv("HMG_NO_ZBLOCK3")
    cdt = torch.complex64 if dtype == "c64" else torch.complex128
    for lvl in range(2):
        nf, nc = ga.level_nodes(lvl)[0], ga.level_nodes(lvl + 1)[0]
        r = torch.from_numpy(media.random_complex(nf, 1 + lvl)).to(cdt).cuda()
        ca, cb = torch.zeros(nc, dtype=cdt, device="cuda"), torch.zeros(nc, dtype=cdt, device="cuda")
        ga.restrict(r, ca, level=lvl)
        gb.restrict(r, cb, level=lvl)
        assert torch.equal(ca, cb), lvl
        e = torch.from_numpy(media.random_complex(nc, 5 + lvl)).to(cdt).cuda()
        ua, ub = r.clone(), r.clone()
        ga.prolong_add(e, ua, level=lvl)
        gb.prolong_add(e, ub, level=lvl)
        assert torch.equal(ua, ub), lvl
    q = torch.from_numpy(p.q.ravel()).to(cdt).cuda()
    za, zb = torch.zeros_like(q), torch.zeros_like(q)
    ga.vcycle(q, za)
    gb.vcycle(q, zb)
    assert torch.equal(za, zb)
