"""Per-stream workspaces (include/hmg.h "Ownership"; "concurrent solves on
one hierarchy"): two host threads solve different right-hand sides on ONE hierarchy, each on its
own CUDA stream, at the same time; every result must equal, bit for bit, the same solve run
alone on the default stream (one workspace per stream, coefficients shared)."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_concurrent_streams_bit_identical(dtype):
    import torch
    from paper_2511_16808_b200 import hmg, media
    p = media.config_problem(0)
    gh = hmg.Hierarchy(hmg.Options(dim=2, cells=p.cells, h=p.h, levels=4, damping=[0.83, 0.5, 0.4, 0.65],
                                   dtype=dtype), p.kappa, p.omega, p.gamma, 0.15)
    cdt = torch.complex64 if dtype == "c64" else torch.complex128
    rng = np.random.default_rng(5)
    Q = []
    for k in range(4):
        q = np.zeros(p.n, np.complex128)
        q[rng.integers(2000, p.n - 2000)] = 1.0 / p.h ** 2
        Q.append(torch.from_numpy(q).to(cdt).cuda())
    # reference: one after the other on the default stream
    ref = []
    for q in Q:
        x = torch.zeros_like(q)
        r = gh.fgmres_solve(q, x, restart=10, tol=1e-6, maxiter=300)
        z = torch.zeros_like(q)
        gh.vcycle(q, z)
        ref.append((r.iterations, x.clone(), z.clone()))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(2)]
    out = [None] * 4
    err = []

    def worker(t):
        try:
            with torch.cuda.stream(streams[t]):
                for k in (t, t + 2):
                    x = torch.zeros_like(Q[k])
                    r = gh.fgmres_solve(Q[k], x, restart=10, tol=1e-6, maxiter=300, stream=streams[t])
                    z = torch.zeros_like(Q[k])
                    gh.vcycle(Q[k], z, stream=streams[t])
                    streams[t].synchronize()
                    out[k] = (r.iterations, x, z)
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not err, err
    for k in range(4):
        assert out[k][0] == ref[k][0]
        assert torch.equal(out[k][1], ref[k][1]) and torch.equal(out[k][2], ref[k][2])
