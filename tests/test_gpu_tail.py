"""The persistent coarse tail (k_coarse_tail: the small levels of a one-rank
V(1,1) cycle in one launch -- a cooperative grid with a software grid barrier, or ONE
thread-block cluster of 16 / 8 blocks with the hardware cluster barrier) against the per-kernel
cycle (HMG_TAIL_NODES=0, HMG_TAIL_CLUSTER_NODES=0): the same per-node arithmetic, so V-cycles and
FGMRES solves must be BIT-identical -- 2D RB and Element, 3D Element and Plus, both precisions, homogeneous (uniform
boxes) and heterogeneous media, and multi-RHS batches after a buffer reallocation."""
import pytest

from helpers import DAMPING, problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _pair(monkeypatch, p, L, sm, dtype, alpha, thr="300000", mode="grid"):
    """(hierarchy with the tail in `mode`, hierarchy with the per-kernel cycle); mode: "grid"
    (cooperative launch, software barrier) or "cluster16" / "cluster8" (one cluster)."""
    from paper_2511_16808_b200 import hmg
    opts = hmg.Options(dim=p.dim, cells=p.cells, h=p.h, levels=L, smoother=sm, damping=DAMPING[(p.dim, sm)],
                       dtype=dtype)
    if mode == "grid":
        monkeypatch.setenv("HMG_TAIL_NODES", thr)
        monkeypatch.setenv("HMG_TAIL_CLUSTER_NODES", "0")
    else:
        monkeypatch.setenv("HMG_TAIL_NODES", "0")
        monkeypatch.setenv("HMG_TAIL_CLUSTER_NODES", thr)
        monkeypatch.setenv("HMG_TAIL_CLUSTER", mode[len("cluster"):])
    ga = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, alpha)
    monkeypatch.setenv("HMG_TAIL_NODES", "0")
    monkeypatch.setenv("HMG_TAIL_CLUSTER_NODES", "0")
    gb = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, alpha)
    for k in ("HMG_TAIL_NODES", "HMG_TAIL_CLUSTER_NODES", "HMG_TAIL_CLUSTER"):
        monkeypatch.delenv(k, raising=False)
    return ga, gb


@pytest.mark.parametrize("mode", ["grid", "cluster16", "cluster8"])
@pytest.mark.parametrize("case,dtype", [("2d_rb", "c64"), ("2d_rb", "c128"), ("2d_element", "c64"),
                                        ("2d_hetero", "c128"), ("3d_element", "c64"), ("3d_plus", "c128")])
def test_tail_bit_identical(monkeypatch, case, dtype, mode):
    import torch
    from paper_2511_16808_b200 import media
    if case == "2d_rb":
        p, L, sm, al, m = media.config_problem(1, n=256), 5, "rb", 0.25, 20
    elif case == "2d_element":
        p, L, sm, al, m = media.config_problem(0), 4, "element", 0.25, 10
    elif case == "2d_hetero":
        p, L, sm, al, m = problem(2, (128, 96)), 4, "rb", 0.3, 10
    elif case == "3d_element":
        p, L, sm, al, m = media.homogeneous_problem(3, 32, sponge=4), 4, "element", 0.5, 10
    else:
        p, L, sm, al, m = problem(3, (16, 16, 32)), 3, "plus", 0.65, 10
    # a threshold that puts every coarse level in the tail
    ga, gb = _pair(monkeypatch, p, L, sm, dtype, al, thr="100000000", mode=mode)
    cdt = torch.complex64 if dtype == "c64" else torch.complex128
    q = torch.from_numpy(p.q.ravel()).to(cdt).cuda()
    for seed in (0, 1):
        f = q if seed == 0 else torch.from_numpy(media.random_complex(p.n, 4)).to(cdt).cuda()
        za, zb = torch.zeros_like(f), torch.zeros_like(f)
        ga.vcycle(f, za)
        gb.vcycle(f, zb)
        assert torch.equal(za, zb)
    xa, xb = torch.zeros_like(q), torch.zeros_like(q)
    ra = ga.fgmres_solve(q, xa, restart=m, tol=1e-6, maxiter=500)
    rb = gb.fgmres_solve(q, xb, restart=m, tol=1e-6, maxiter=500)
    assert ra.converged and ra.iterations == rb.iterations and torch.equal(xa, xb)


@pytest.mark.parametrize("mode", ["grid", "cluster16"])
def test_tail_after_batch_realloc(monkeypatch, mode):
    """A multi-RHS batch reallocates the coarse-level vectors; single solves afterwards still
    equal the per-kernel path (the tail's level table follows the new buffers)."""
    import torch
    from paper_2511_16808_b200 import media
    p = media.config_problem(0)
    ga, gb = _pair(monkeypatch, p, 4, "rb", "c128", 0.15, thr="100000000", mode=mode)
    q = torch.from_numpy(p.q.ravel()).cuda()
    Q = torch.stack([q, q.roll(3000)])
    X = torch.zeros_like(Q)
    ga.fgmres_solve_batch(Q, X, restart=10, tol=1e-6, maxiter=300)
    xa, xb = torch.zeros_like(q), torch.zeros_like(q)
    ra = ga.fgmres_solve(q, xa, restart=10, tol=1e-6, maxiter=300)
    rb = gb.fgmres_solve(q, xb, restart=10, tol=1e-6, maxiter=300)
    assert ra.iterations == rb.iterations and torch.equal(xa, xb)
