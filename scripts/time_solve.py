"""Median device-timed time-to-solve of one configuration (graph mode, as bench.py).

    python scripts/time_solve.py --config 1 --n 4096 [--dtype c64] [--reps 3]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--dtype", default="c64")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    import torch
    from paper_2511_16808_b200 import hmg, media
    if a.config == 3:
        p, L, alpha, m = media.config_problem(3), 6, 0.5, 10
    elif a.config == 4:
        p, L, alpha, m = media.config_problem(4, scale=2), 6, 0.6, 20
    else:
        p, L, alpha, m = media.config_problem(1, n=a.n), a.n.bit_length() - 4, 0.25, 20
    sm = "rb" if p.dim == 2 else "element"
    damp = [0.83, 0.5, 0.4, 0.65] if p.dim == 2 else [1.1, 0.7, 0.45, 0.6]
    g = hmg.Hierarchy(hmg.Options(dim=p.dim, cells=p.cells, h=p.h, levels=L, smoother=sm, damping=damp,
                                  dtype=a.dtype), p.kappa, p.omega, p.gamma, alpha)
    cdt = torch.complex64 if a.dtype == "c64" else torch.complex128
    q = torch.from_numpy(p.q.ravel()).to(cdt).cuda()
    x = torch.zeros_like(q)
    reps = [g.fgmres_solve(q, x, restart=m, tol=1e-6, maxiter=4000) for _ in range(a.reps + 1)]
    sec = statistics.median(r.seconds for r in reps[1:])
    print(json.dumps(dict(tag=a.tag or os.environ.get("TAG", ""), config=a.config, n=a.n, dtype=a.dtype,
                          iterations=reps[-1].iterations, seconds=round(sec, 5),
                          ms_per_iteration=round(1e3 * sec / reps[-1].iterations, 4))), flush=True)


if __name__ == "__main__":
    main()
