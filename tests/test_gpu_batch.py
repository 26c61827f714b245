"""Multi-RHS batched solves (hmg_fgmres_solve_batch).

The batch applies one batched preconditioner per step (fine level per right-hand
side, coarser levels once for all of them) with the per-RHS arithmetic of the
single solve, so every batched solution must equal the single solve's bit for
bit, with the same iteration count; one case is also checked against the oracle."""
import numpy as np
import pytest

from helpers import DAMPING, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _rhs(p, nr, seed):
    """nr right-hand sides: the config's point source, then seeded random sources."""
    from paper_2511_16808_b200 import media
    qs = [p.q.ravel().astype(np.complex128)]
    for k in range(1, nr):
        qs.append(media.random_complex(p.n, seed + k))
    return np.stack(qs)


def _batch_vs_single(p, levels, alpha, restart, dtype, nr, smoother=None, cycle="V", zero_rhs=None):
    import torch
    from paper_2511_16808_b200 import hmg
    smoother = smoother or ("rb" if p.dim == 2 else "element")
    gh = hmg.Hierarchy(hmg.Options(dim=p.dim, cells=p.cells, h=p.h, levels=levels, smoother=smoother, cycle=cycle,
                                   damping=DAMPING[(p.dim, smoother)], dtype=dtype), p.kappa, p.omega, p.gamma, alpha)
    cdt = torch.complex64 if dtype == "c64" else torch.complex128
    Q = _rhs(p, nr, 100)
    if zero_rhs is not None:
        Q[zero_rhs] = 0
    q = torch.from_numpy(Q).to(cdt).cuda()
    x = torch.zeros_like(q)
    reps = gh.fgmres_solve_batch(q, x, restart=restart, tol=1e-6, maxiter=500)
    assert len(reps) == nr
    for k in range(nr):
        xs = torch.zeros_like(q[k])
        rs = gh.fgmres_solve(q[k].clone(), xs, restart=restart, tol=1e-6, maxiter=500)
        assert reps[k].iterations == rs.iterations, (k, reps[k].iterations, rs.iterations)
        assert reps[k].converged and rs.converged
        assert reps[k].history == rs.history
        assert torch.equal(x[k], xs), k
    return gh, Q, x, reps


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_batch_config0_bit_identical(dtype):
    from paper_2511_16808_b200 import media
    p = media.config_problem(0)
    _batch_vs_single(p, 4, 0.15, 10, dtype, 3)


@pytest.mark.parametrize("nr", [5, 9])
def test_batch_chunking(nr):
    """5 = 4 + 1 and 9 = 8 + 1 right-hand sides through the batched kernels."""
    from paper_2511_16808_b200 import media
    p = media.homogeneous_problem(2, 64, sponge=8)
    _batch_vs_single(p, 3, 0.3, 10, "c64", nr)


def test_batch_zero_rhs_and_wcycle():
    """A zero right-hand side converges at once and leaves the batch; W-cycles batch too."""
    from paper_2511_16808_b200 import media
    p = media.homogeneous_problem(2, 64, sponge=8)
    _, _, x, reps = _batch_vs_single(p, 3, 0.3, 5, "c128", 3, cycle="W", zero_rhs=1)
    assert reps[1].iterations == 0 and float(x[1].abs().max()) == 0.0


def test_batch_3d_element():
    from paper_2511_16808_b200 import media
    p = media.homogeneous_problem(3, 16, sponge=4)
    _batch_vs_single(p, 3, 0.5, 10, "c64", 3)


def test_batch_matches_oracle():
    """Each batched solution against the oracle's FGMRES on the same right-hand side."""
    from paper_2511_16808_b200 import media
    from oracle.cycle import vcycle
    from oracle.fgmres import fgmres_solve
    from oracle.hierarchy import Options as OOptions, build_hierarchy
    p = media.config_problem(0)
    _, Q, x, reps = _batch_vs_single(p, 4, 0.15, 10, "c128", 2)
    oh = build_hierarchy(OOptions(dim=2, cells=p.cells, h=p.h, levels=4, smoother="rb",
                                  damping=DAMPING[(2, "rb")]), p.kappa, p.omega, p.gamma, 0.15)
    for k in range(2):
        xo, info = fgmres_solve(oh.H, Q[k], lambda v: vcycle(oh, v), restart=10, tol=1e-6, maxiter=500)
        assert abs(reps[k].iterations - info["iterations"]) <= 1
        assert rel_err(x[k].cpu().numpy(), xo) <= 1e-4


def test_batch_errors():
    import torch
    from paper_2511_16808_b200 import hmg, media
    p = media.homogeneous_problem(2, 16, sponge=2)
    gh = hmg.Hierarchy(hmg.Options(dim=2, cells=p.cells, h=p.h, levels=2, damping=DAMPING[(2, "rb")]),
                       p.kappa, p.omega, p.gamma, 0.3)
    q = torch.zeros(2 * p.n + 1, dtype=torch.complex128, device="cuda")
    with pytest.raises(ValueError):
        gh.fgmres_solve_batch(q, torch.zeros_like(q))
