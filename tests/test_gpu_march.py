"""The 2D c64 warp-marching fine operator (k_fine_op2d_march) against the
node-parallel kernels it replaces (HMG_NO_FMARCH=1 at build): the same per-node grouping of
the stencil sums, so the outputs must be BIT-identical -- on ragged grids (strip width 60,
segment height 32: sizes that leave partial strips and segments), homogeneous (uniform box)
and heterogeneous media, through H x, H_s x, the residual, the V-cycle and FGMRES (the
FGMRES matvec uses the fp64-sigma instance).  Parity against the oracle: test_gpu_parity.py."""
import numpy as np
import pytest

from helpers import DAMPING, problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.parametrize("medium,cells,stencil", [
    ("homogeneous", (128, 128), "compact4"),
    ("hetero", (120, 68), "compact4"),
    ("hetero", (8, 40), "compact4"),
    ("hetero", (64, 32), "fd2"),
])
def test_march_bit_identical(monkeypatch, medium, cells, stencil):
    import torch
    from paper_2511_16808_b200 import hmg, media
    if medium == "homogeneous":
        p = media.config_problem(0)
    else:
        p = problem(2, cells)
    L = 3
    opts = hmg.Options(dim=2, cells=p.cells, h=p.h, levels=L, smoother="rb", fine_stencil=stencil,
                       damping=DAMPING[(2, "rb")], dtype="c64")
    monkeypatch.delenv("HMG_NO_FMARCH", raising=False)
    ga = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.3)
    monkeypatch.setenv("HMG_NO_FMARCH", "1")
    gb = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.3)
    monkeypatch.delenv("HMG_NO_FMARCH")
    x = torch.from_numpy(media.random_complex(p.n, 1)).to(torch.complex64).cuda()
    f = torch.from_numpy(media.random_complex(p.n, 2)).to(torch.complex64).cuda()
    for shifted in (False, True):
        ya, yb = torch.empty_like(x), torch.empty_like(x)
        ga.apply_helmholtz(x, ya, shifted=shifted)
        gb.apply_helmholtz(x, yb, shifted=shifted)
        assert torch.equal(ya, yb)
        ga.residual(f, x, ya, shifted=shifted)
        gb.residual(f, x, yb, shifted=shifted)
        assert torch.equal(ya, yb)
    q = torch.from_numpy(p.q.ravel()).to(torch.complex64).cuda()
    za, zb = torch.zeros_like(q), torch.zeros_like(q)
    ga.vcycle(q, za)
    gb.vcycle(q, zb)
    assert torch.equal(za, zb)
    xa, xb = torch.zeros_like(q), torch.zeros_like(q)
    ra = ga.fgmres_solve(q, xa, restart=10, tol=1e-6, maxiter=300)
    rb = gb.fgmres_solve(q, xb, restart=10, tol=1e-6, maxiter=300)
    assert ra.iterations == rb.iterations and ra.history == rb.history
    assert torch.equal(xa, xb)


@pytest.mark.parametrize("n", [256, 304])
def test_rb_fast_path_bit_identical(monkeypatch, n):
    """The RB sweep's constant-coefficient instance for warps inside the uniform box (MODE 1 of
    k_rb2d_march2) against the generic instance everywhere (HMG_NO_RB_FAST=1): bit-identical
    smoothing steps, V-cycles and FGMRES solves (config-1 family, c64)."""
    import torch
    from paper_2511_16808_b200 import hmg, media
    p = media.config_problem(1, n=n) if n == 256 else media.homogeneous_problem(2, n, sponge=16)
    opts = hmg.Options(dim=2, cells=p.cells, h=p.h, levels=4, smoother="rb", damping=DAMPING[(2, "rb")], dtype="c64")
    monkeypatch.delenv("HMG_NO_RB_FAST", raising=False)
    ga = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.25)
    monkeypatch.setenv("HMG_NO_RB_FAST", "1")
    gb = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.25)
    monkeypatch.delenv("HMG_NO_RB_FAST")
    assert ga.uniform_box(0)[0] > 0
    f = torch.from_numpy(media.random_complex(p.n, 2)).to(torch.complex64).cuda()
    u = torch.from_numpy(media.random_complex(p.n, 3)).to(torch.complex64).cuda()
    ua, ub = u.clone(), u.clone()
    ga.smooth(f, ua)
    gb.smooth(f, ub)
    assert torch.equal(ua, ub)
    q = torch.from_numpy(p.q.ravel()).to(torch.complex64).cuda()
    za, zb = torch.zeros_like(q), torch.zeros_like(q)
    ga.vcycle(q, za)
    gb.vcycle(q, zb)
    assert torch.equal(za, zb)
    xa, xb = torch.zeros_like(q), torch.zeros_like(q)
    ra = ga.fgmres_solve(q, xa, restart=20, tol=1e-6, maxiter=400)
    rb = gb.fgmres_solve(q, xb, restart=20, tol=1e-6, maxiter=400)
    assert ra.iterations == rb.iterations and torch.equal(xa, xb)


@pytest.mark.parametrize("dim,vbz", [(2, 2), (2, 4), (3, 2), (3, 4)])
def test_vanka_blocked_bit_identical(monkeypatch, dim, vbz):
    """The register-blocked assembled-Vanka stencil (k_vanka_stencil_blk, BZ nodes per thread
    along the slow axis) against the one-node gather (HMG_VANKA_BZ=1): bit-identical smoothing
    steps on every smoothing level and V-cycles (2D element patches, 3D element patches; c64)."""
    import torch
    from paper_2511_16808_b200 import hmg, media
    if dim == 2:
        p, sm, L = problem(2, (256, 136)), "element", 3
    else:
        p, sm, L = problem(3, (24, 20, 132)), "element", 3
    opts = hmg.Options(dim=dim, cells=p.cells, h=p.h, levels=L, smoother=sm, damping=DAMPING[(dim, sm)], dtype="c64")
    monkeypatch.setenv("HMG_VANKA_BZ", str(vbz))
    ga = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.4)
    monkeypatch.setenv("HMG_VANKA_BZ", "1")
    gb = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.4)
    monkeypatch.delenv("HMG_VANKA_BZ")
    for lvl in range(L - 1):
        N = ga.level_nodes(lvl)[0]
        f = torch.from_numpy(media.random_complex(N, 5 + lvl)).to(torch.complex64).cuda()
        u = torch.from_numpy(media.random_complex(N, 7 + lvl)).to(torch.complex64).cuda()
        ua, ub = u.clone(), u.clone()
        ga.smooth(f, ua, level=lvl)
        gb.smooth(f, ub, level=lvl)
        assert torch.equal(ua, ub), lvl
    q = torch.from_numpy(p.q.ravel()).to(torch.complex64).cuda()
    za, zb = torch.zeros_like(q), torch.zeros_like(q)
    ga.vcycle(q, za)
    gb.vcycle(q, zb)
    assert torch.equal(za, zb)


@pytest.mark.parametrize("medium,n", [("homogeneous", 512), ("hetero", 520)])
def test_stored_march_bit_identical(monkeypatch, medium, n):
    """The warp-marching stored-stencil residual (k_stored_op2d_march, opt-in HMG_SMARCH=8, levels
    with >= 256 rows) against the register-blocked gather (default): bit-identical level-1
    residuals, V-cycles and FGMRES solves (c64; uniform box and heterogeneous medium)."""
    import torch
    from paper_2511_16808_b200 import hmg, media
    p = media.config_problem(1, n=n) if medium == "homogeneous" else problem(2, (n, 264))
    opts = hmg.Options(dim=2, cells=p.cells, h=p.h, levels=4, smoother="rb", damping=DAMPING[(2, "rb")], dtype="c64")
    monkeypatch.setenv("HMG_SMARCH", "8")
    ga = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.25)
    monkeypatch.delenv("HMG_SMARCH")
    gb = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.25)
    N1 = ga.level_nodes(1)[0]
    x = torch.from_numpy(media.random_complex(N1, 2)).to(torch.complex64).cuda()
    f = torch.from_numpy(media.random_complex(N1, 3)).to(torch.complex64).cuda()
    ra, rb = torch.empty_like(x), torch.empty_like(x)
    ga.residual(f, x, ra, level=1, shifted=True)
    gb.residual(f, x, rb, level=1, shifted=True)
    assert torch.equal(ra, rb)
    ga.apply_helmholtz(x, ra, level=1, shifted=True)
    gb.apply_helmholtz(x, rb, level=1, shifted=True)
    assert torch.equal(ra, rb)
    q = torch.from_numpy(p.q.ravel()).to(torch.complex64).cuda()
    za, zb = torch.zeros_like(q), torch.zeros_like(q)
    ga.vcycle(q, za)
    gb.vcycle(q, zb)
    assert torch.equal(za, zb)
    xa, xb = torch.zeros_like(q), torch.zeros_like(q)
    r1 = ga.fgmres_solve(q, xa, restart=20, tol=1e-6, maxiter=600)
    r2 = gb.fgmres_solve(q, xb, restart=20, tol=1e-6, maxiter=600)
    assert r1.iterations == r2.iterations and torch.equal(xa, xb)


@pytest.mark.parametrize("medium,cells,stencil", [
    ("homogeneous", (256, 256), "compact4"),
    ("hetero", (120, 68), "compact4"),
    ("hetero", (8, 40), "compact4"),
    ("hetero", (64, 32), "fd2"),
])
def test_residual_restrict_fused_bit_identical(monkeypatch, medium, cells, stencil):
    """The fused fine residual + bicubic restriction (k_fine_resrestrict2d_march: residual
    never written) against the residual kernel followed by k_restrict_pair (HMG_NO_RRFUSE=1):
    bit-identical V-cycles and FGMRES solves on ragged grids (strip 56, segment 32)."""
    import torch
    from paper_2511_16808_b200 import hmg, media
    p = media.config_problem(1, n=cells[0]) if medium == "homogeneous" else problem(2, cells)
    opts = hmg.Options(dim=2, cells=p.cells, h=p.h, levels=3, smoother="rb", fine_stencil=stencil,
                       damping=DAMPING[(2, "rb")], dtype="c64")
    monkeypatch.delenv("HMG_NO_RRFUSE", raising=False)
    ga = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.3)
    monkeypatch.setenv("HMG_NO_RRFUSE", "1")
    gb = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.3)
    monkeypatch.delenv("HMG_NO_RRFUSE")
    for seed in (1, 2):
        f = torch.from_numpy(media.random_complex(p.n, seed)).to(torch.complex64).cuda()
        za, zb = torch.zeros_like(f), torch.zeros_like(f)
        ga.vcycle(f, za)
        gb.vcycle(f, zb)
        assert torch.equal(za, zb)
        u = torch.from_numpy(media.random_complex(p.n, seed + 10)).to(torch.complex64).cuda()
        ua, ub = u.clone(), u.clone()
        ga.vcycle(f, ua, x_is_zero=False)
        gb.vcycle(f, ub, x_is_zero=False)
        assert torch.equal(ua, ub)
    q = torch.from_numpy(p.q.ravel()).to(torch.complex64).cuda()
    xa, xb = torch.zeros_like(q), torch.zeros_like(q)
    r1 = ga.fgmres_solve(q, xa, restart=10, tol=1e-6, maxiter=400)
    r2 = gb.fgmres_solve(q, xb, restart=10, tol=1e-6, maxiter=400)
    assert r1.iterations == r2.iterations and torch.equal(xa, xb)
