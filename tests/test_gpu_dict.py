"""Coefficient dictionary (k_dict.cuh).

Outside the uniform box of a sponge-bordered homogeneous medium a node's Galerkin
stencil and assembled Vanka operator depend only on the damping profile around it,
so a level carries few distinct coefficient vectors; the kernels read a 2-byte class
index per node and a class table instead of the per-node planes.  Same values, same
arithmetic order: every output must be BIT-identical to a hierarchy built with
HMG_NO_DICT=1 (the planes), on the uniform-box path (dictionary outside the box) and
with HMG_NO_UNIFORM=1 (dictionary on every node), through the stand-alone kernels
and the persistent coarse tail.  Heterogeneous media keep their planes.
"""
import pytest

from helpers import DAMPING

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _build(monkeypatch, p, levels, smoother, dtype, alpha, env):
    from paper_2511_16808_b200 import hmg
    for k in ("HMG_NO_DICT", "HMG_NO_UNIFORM"):
        monkeypatch.delenv(k, raising=False)
    for k in env:
        monkeypatch.setenv(k, "1")
    opts = hmg.Options(dim=p.dim, cells=p.cells, h=p.h, levels=levels, smoother=smoother,
                       damping=DAMPING[(p.dim, smoother)], dtype=dtype)
    g = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, alpha)
    for k in env:
        monkeypatch.delenv(k)
    return g


CASES = {
    "2d": lambda media: (media.config_problem(0), 4, 0.15, "rb"),
    # 3D, 4 levels: levels >= 1 run in the persistent coarse tail (3D default)
    "3d": lambda media: (media.homogeneous_problem(3, 32, sponge=4), 4, 0.5, "element"),
    "3d_r2": lambda media: (media.homogeneous_problem(3, 48, sponge=8), 3, 0.5, "element"),
}


@pytest.mark.parametrize("uniform", [True, False], ids=["box", "nobox"])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("case", sorted(CASES))
def test_dict_bit_identical(monkeypatch, case, dtype, uniform):
    import torch
    from paper_2511_16808_b200 import media
    p, L, alpha, sm = CASES[case](media)
    base = [] if uniform else ["HMG_NO_UNIFORM"]
    gd = _build(monkeypatch, p, L, sm, dtype, alpha, base)
    gs = _build(monkeypatch, p, L, sm, dtype, alpha, base + ["HMG_NO_DICT"])
    # the levels with a stored stencil / Vanka operator use dictionaries; the planes build has none
    for lvl in range(L - 1):
        cn, bn = gd.dict_classes(lvl)
        assert gs.dict_classes(lvl) == (0, 0)
        if lvl > 0:
            assert cn > 0, f"level {lvl}: no stencil dictionary"
        if sm == "element" or lvl > 0:
            assert bn > 0, f"level {lvl}: no Vanka-operator dictionary"
    cdt = torch.complex64 if dtype == "c64" else torch.complex128
    for lvl in range(L - 1):
        N = gd.level_nodes(lvl)[0]
        f = torch.from_numpy(media.random_complex(N, 5 + lvl)).to(cdt).cuda()
        x = torch.from_numpy(media.random_complex(N, 9 + lvl)).to(cdt).cuda()
        rd, rs = torch.empty_like(x), torch.empty_like(x)
        gd.residual(f, x, rd, level=lvl, shifted=True)
        gs.residual(f, x, rs, level=lvl, shifted=True)
        assert torch.equal(rd, rs), f"residual level {lvl}"
        ud = torch.from_numpy(media.random_complex(N, 7 + lvl)).to(cdt).cuda()
        us = ud.clone()
        gd.smooth(f, ud, level=lvl)
        gs.smooth(f, us, level=lvl)
        assert torch.equal(ud, us), f"smooth level {lvl}"
    q = torch.from_numpy(p.q.ravel()).to(cdt).cuda()
    zd, zs = torch.zeros_like(q), torch.zeros_like(q)
    gd.vcycle(q, zd)
    gs.vcycle(q, zs)
    assert torch.equal(zd, zs)
    xd, xs = torch.zeros_like(q), torch.zeros_like(q)
    rd = gd.fgmres_solve(q, xd, restart=10, tol=1e-6, maxiter=300)
    rs = gs.fgmres_solve(q, xs, restart=10, tol=1e-6, maxiter=300)
    assert rd.converged and rd.iterations == rs.iterations and rd.history == rs.history
    assert torch.equal(xd, xs)


def test_dict_heterogeneous_keeps_planes():
    """A layered medium with a random perturbation (config 2's generator at 1/8 scale):
    nearly every node's coefficients differ, so no level gets a dictionary."""
    from paper_2511_16808_b200 import hmg, media
    p = media.config_problem(2, scale=8)
    opts = hmg.Options(dim=2, cells=p.cells, h=p.h, levels=3, smoother="rb",
                       damping=DAMPING[(2, "rb")], dtype="c64")
    g = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, 0.5)
    for lvl in range(2):
        assert g.dict_classes(lvl) == (0, 0)
