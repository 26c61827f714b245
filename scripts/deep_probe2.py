import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2511_16808_b200 import hmg, media
p = media.config_problem(4, scale=2)
for dt, L, sm in (("c128", 5, "element"), ("c64", 5, "jacobi"), ("c64", 5, "element")):
    damp = [1.1, 0.7, 0.45, 0.6] if sm == "element" else [0.6, 0.4, 0.3, 0.5]
    gh = hmg.Hierarchy(hmg.Options(dim=3, cells=p.cells, h=p.h, levels=L, smoother=sm, damping=damp, dtype=dt),
                       p.kappa, p.omega, p.gamma, 0.5)
    cdt = torch.complex64 if dt == "c64" else torch.complex128
    q = torch.from_numpy(p.q.ravel()).to(cdt).cuda()
    x = torch.zeros_like(q)
    r = gh.fgmres_solve(q, x, restart=20, tol=1e-6, maxiter=300)
    # where is the final residual concentrated?
    y = torch.empty_like(x)
    gh.residual(q, x, y)
    rr = y.abs().cpu().numpy().reshape(p.nodes[::-1])
    zmax = np.unravel_index(np.argmax(rr), rr.shape)
    prof = [float(rr[k].max()) for k in range(0, rr.shape[0], 12)]
    print(json.dumps(dict(dt=dt, L=L, sm=sm, its=r.iterations, conv=r.converged, relres=r.relres_true,
                          argmax_zyx=[int(v) for v in zmax], max_by_z=[f"{v:.2e}" for v in prof],
                          qn=float(np.abs(p.q).max()))), flush=True)
    del gh
    torch.cuda.empty_cache()
