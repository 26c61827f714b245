"""A few preconditioner applications (one V-cycle each) on the bench workload, for ncu captures.

    python scripts/vcycle_probe.py [--n 4096] [--dtype c64] [--cycles 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--dtype", default="c64")
    ap.add_argument("--cycles", type=int, default=3)
    a = ap.parse_args()
    import torch
    from paper_2511_16808_b200 import hmg, media
    p = media.config_problem(1, n=a.n)
    gh = hmg.Hierarchy(hmg.Options(dim=2, cells=p.cells, h=p.h, levels=a.n.bit_length() - 4, smoother="rb",
                                   damping=[0.83, 0.5, 0.4, 0.65], dtype=a.dtype), p.kappa, p.omega, p.gamma, 0.25)
    cdt = torch.complex64 if a.dtype == "c64" else torch.complex128
    f = torch.from_numpy(p.q.ravel()).to(cdt).cuda()
    x = torch.zeros_like(f)
    for _ in range(a.cycles):
        gh.vcycle(f, x, x_is_zero=True)
    torch.cuda.synchronize()
    print("ok", float(x.abs().max()))


if __name__ == "__main__":
    main()
