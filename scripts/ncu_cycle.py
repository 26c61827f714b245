"""One V-cycle of a BASELINE config between cudaProfilerStart/Stop (for
``ncu --profile-from-start off``): the kernels of one preconditioner application
after a warm-up solve.

    ncu --profile-from-start off --set full -o /tmp/c3 python scripts/ncu_cycle.py --config 3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--n", type=int, default=0)
    a = ap.parse_args()
    import torch
    from paper_2511_16808_b200 import hmg, media
    if a.config == 3:
        p, kw = media.config_problem(3), dict(levels=6, alpha=0.5, dtype="c64")
    elif a.config == 4:
        p, kw = media.config_problem(4, scale=2), dict(levels=6, alpha=0.6, dtype="c64")
    else:
        n = a.n or 4096
        p, kw = media.config_problem(1, n=n), dict(levels=n.bit_length() - 4, alpha=0.25, dtype="c64")
    sm = "rb" if p.dim == 2 else "element"
    damp = [0.83, 0.5, 0.4, 0.65] if p.dim == 2 else [1.1, 0.7, 0.45, 0.6]
    gh = hmg.Hierarchy(hmg.Options(dim=p.dim, cells=p.cells, h=p.h, levels=kw["levels"], smoother=sm, damping=damp,
                                   dtype=kw["dtype"]), p.kappa, p.omega, p.gamma, kw["alpha"])
    q = torch.from_numpy(p.q.ravel()).to(torch.complex64).cuda()
    z = torch.zeros_like(q)
    gh.vcycle(q, z)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    gh.vcycle(q, z)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
