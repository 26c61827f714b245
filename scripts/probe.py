"""A few preconditioner applications and FGMRES steps on a BASELINE workload, for ncu captures.

    python scripts/probe.py [--config 1|3] [--n 4096] [--dtype c64] [--iters 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--dtype", default="c64")
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    import torch
    from paper_2511_16808_b200 import hmg, media
    if a.config == 3:
        n = a.n or 256
        p = media.config_problem(3, n=n)
        L, alpha, sm, damp, m = n.bit_length() - 4, 0.5, "element", [1.1, 0.7, 0.45, 0.6], 10
    else:
        n = a.n or 4096
        p = media.config_problem(1, n=n)
        L, alpha, sm, damp, m = n.bit_length() - 4, 0.25, "rb", [0.83, 0.5, 0.4, 0.65], 20
    gh = hmg.Hierarchy(hmg.Options(dim=p.dim, cells=p.cells, h=p.h, levels=L, smoother=sm, damping=damp,
                                   dtype=a.dtype), p.kappa, p.omega, p.gamma, alpha)
    cdt = torch.complex64 if a.dtype == "c64" else torch.complex128
    q = torch.from_numpy(p.q.ravel()).to(cdt).cuda()
    x = torch.zeros_like(q)
    r = gh.fgmres_solve(q, x, restart=m, tol=1e-6, maxiter=a.iters)
    torch.cuda.synchronize()
    print("ok", r.iterations)


if __name__ == "__main__":
    main()
