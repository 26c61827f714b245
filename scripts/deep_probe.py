"""Iterations vs V-cycle depth on the config-4 generator (3D heterogeneous)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_16808_b200 import hmg, media
for scale, levels in ((4, (4, 5)), (2, (5, 6))):
    p = media.config_problem(4, scale=scale)
    for L in levels:
        gh = hmg.Hierarchy(hmg.Options(dim=3, cells=p.cells, h=p.h, levels=L, smoother="element",
                                       damping=[1.1, 0.7, 0.45, 0.6], dtype="c64"), p.kappa, p.omega, p.gamma, 0.5)
        q = torch.from_numpy(p.q.ravel()).to(torch.complex64).cuda()
        x = torch.zeros_like(q)
        r = gh.fgmres_solve(q, x, restart=20, tol=1e-6, maxiter=1500)
        print(json.dumps(dict(scale=scale, cells=p.cells, levels=L, its=r.iterations, conv=r.converged,
                              relres=r.relres_true, s=r.seconds, hist=[round(h, 6) for h in r.history[::40]])),
              flush=True)
        del gh
        torch.cuda.empty_cache()
