import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2511_16808_b200 import hmg, media
p = media.config_problem(4, scale=2)
qc = media.point_source(p.cells, p.h, at=(192, 192, 96))
for name, q_, alpha, L in (("src centre a.5", qc, 0.5, 5), ("src top a.8", p.q, 0.8, 5), ("src top a.5 L3-ish(4)", p.q, 0.5, 4)):
    try:
        gh = hmg.Hierarchy(hmg.Options(dim=3, cells=p.cells, h=p.h, levels=L, smoother="element",
                                       damping=[1.1, 0.7, 0.45, 0.6], dtype="c64"), p.kappa, p.omega, p.gamma, alpha)
    except Exception as e:
        print(name, "build failed", e); continue
    q = torch.from_numpy(q_.ravel()).to(torch.complex64).cuda()
    x = torch.zeros_like(q)
    r = gh.fgmres_solve(q, x, restart=20, tol=1e-6, maxiter=600)
    print(json.dumps(dict(case=name, its=r.iterations, conv=r.converged, relres=r.relres_true,
                          hist=[round(h, 6) for h in r.history[::50]])), flush=True)
    del gh
    torch.cuda.empty_cache()
