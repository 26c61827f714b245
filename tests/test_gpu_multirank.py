"""Slab-partitioned solve on ONE GPU through the LOCAL backend:
k virtual ranks, one host thread each, halos by stream-ordered device copies.
The partitioned operator, transfers, smoothing and V-cycle must equal the
single-slab results bit for bit (per-node arithmetic is identical; ghost rows
hold the neighbours' data); FGMRES (dots summed per rank, then across ranks)
must match the single-GPU iteration count within +-1 and the oracle's."""
import threading

import numpy as np
import pytest

from helpers import DAMPING, problem, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def run_ranks(P, fn):
    """Run fn(rank, comm) in P threads; re-raise the first exception."""
    from paper_2511_16808_b200 import hmg
    group = hmg.LocalGroup(P)
    comms = [group.rank(r) for r in range(P)]
    out, err = [None] * P, []

    def body(r):
        try:
            out[r] = fn(r, comms[r])
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if err:
        raise err[0]
    return out


def opts_for(p, levels, dtype, smoother=None):
    from paper_2511_16808_b200 import hmg
    sm = smoother or ("rb" if p.dim == 2 else "element")
    return hmg.Options(dim=p.dim, cells=p.cells, h=p.h, levels=levels, smoother=sm, damping=DAMPING[(p.dim, sm)],
                       dtype=dtype)


def rows(v, lo, hi, p):
    """Slab-axis rows [lo, hi) of a flat x-fastest vector."""
    return np.ascontiguousarray(np.asarray(v).reshape(p.nodes[::-1])[lo:hi]).ravel()


@pytest.mark.parametrize("P,dim,cells,levels,dtype", [
    (2, 2, (64, 64), 4, "c128"),
    (3, 2, (64, 96), 4, "c64"),
    (2, 3, (16, 16, 32), 3, "c128"),
])
def test_partitioned_equals_single(P, dim, cells, levels, dtype):
    import torch
    from paper_2511_16808_b200 import hmg, media
    p = problem(dim, cells, sponge=4)
    alpha = 0.3 if dim == 2 else 0.5
    cdt = torch.complex64 if dtype == "c64" else torch.complex128
    single = hmg.Hierarchy(opts_for(p, levels, dtype), p.kappa, p.omega, p.gamma, alpha)
    x = media.random_complex(p.n, 3)
    f = media.random_complex(p.n, 4)
    xd = torch.from_numpy(x).to(cdt).cuda()
    fd = torch.from_numpy(f).to(cdt).cuda()
    y1 = torch.empty_like(xd)
    single.apply_helmholtz(xd, y1)
    v1 = torch.zeros_like(xd)
    single.vcycle(fd, v1)
    q = torch.from_numpy(p.q.ravel()).to(cdt).cuda()
    s1 = torch.zeros_like(q)
    r1 = single.fgmres_solve(q, s1, restart=10, tol=1e-6, maxiter=400)
    torch.cuda.synchronize()
    y1, v1, s1 = y1.cpu().numpy(), v1.cpu().numpy(), s1.cpu().numpy()

    def rank_fn(r, comm):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            h = hmg.Hierarchy(opts_for(p, levels, dtype), p.kappa, p.omega, p.gamma, alpha, stream=st.cuda_stream,
                              comm=comm)
            lo, hi = h.level_rows(0)
            xl = torch.from_numpy(rows(xd.cpu().numpy(), lo, hi, p)).cuda()
            fl = torch.from_numpy(rows(fd.cpu().numpy(), lo, hi, p)).cuda()
            ql = torch.from_numpy(rows(q.cpu().numpy(), lo, hi, p)).cuda()
            yl = torch.empty_like(xl)
            h.apply_helmholtz(xl, yl, stream=st.cuda_stream)
            vl = torch.zeros_like(xl)
            h.vcycle(fl, vl, stream=st.cuda_stream)
            sl = torch.zeros_like(ql)
            rep = h.fgmres_solve(ql, sl, restart=10, tol=1e-6, maxiter=400, stream=st.cuda_stream)
            st.synchronize()
            return lo, hi, yl.cpu().numpy(), vl.cpu().numpy(), sl.cpu().numpy(), rep

    res = run_ranks(P, rank_fn)
    los = [r[0] for r in res]
    assert los[0] == 0 and res[-1][1] == p.nodes[-1]
    for a, b in zip(res[:-1], res[1:]):
        assert a[1] == b[0]
    for lo, hi, yl, vl, sl, rep in res:
        assert np.array_equal(yl, rows(y1, lo, hi, p)), "partitioned H x differs"
        assert np.array_equal(vl, rows(v1, lo, hi, p)), "partitioned V-cycle differs"
        assert rep.converged and abs(rep.iterations - r1.iterations) <= 1
    sol = np.concatenate([r[4] for r in res])
    assert rel_err(sol, s1) <= (1e-5 if dtype == "c128" else 1e-3)
    its = {r[5].iterations for r in res}
    assert len(its) == 1, "ranks disagree on the iteration count"
