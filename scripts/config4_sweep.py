"""Config 4 (BASELINE configs[4] generator: folded layers + thrust fault, seed 4) at 1/2 scale
(384 x 384 x 192 cells, h = 50 m): shift alpha, depth and coarse-level damping swept on the GPU
to settle the round-1 finding that alpha = 0.5 stalls there (VERDICT r01 "Next round" 6).

    python scripts/config4_sweep.py [--scale 2] [--out profiles/r02_config4_sweep.jsonl]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=2)
    ap.add_argument("--maxiter", type=int, default=500)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_config4_sweep.jsonl"))
    a = ap.parse_args()
    import torch
    from paper_2511_16808_b200 import hmg, media
    p = media.config_problem(4, scale=a.scale)
    q = torch.from_numpy(p.q.ravel()).to(torch.complex64).cuda()
    out = open(a.out, "w")
    runs = []
    for L in (5, 6):
        for alpha in (0.5, 0.6, 0.7, 0.8, 1.0):
            runs.append((L, alpha, [1.1, 0.7, 0.45, 0.6]))
    # damping beyond level 4 ("not very sensitive"): the level-3 value vs the level-2 value reused
    for alpha in (0.5, 0.7):
        runs.append((6, alpha, [1.1, 0.7, 0.45, 0.6, 0.45, 0.45]))
        runs.append((6, alpha, [1.1, 0.7, 0.45, 0.45]))
    for L, alpha, damp in runs:
        t0 = time.time()
        try:
            gh = hmg.Hierarchy(hmg.Options(dim=3, cells=p.cells, h=p.h, levels=L, smoother="element", damping=damp,
                                           dtype="c64"), p.kappa, p.omega, p.gamma, alpha)
            setup = time.time() - t0
            x = torch.zeros_like(q)
            r = gh.fgmres_solve(q, x, restart=20, tol=1e-6, maxiter=a.maxiter)
            rec = {"levels": L, "alpha": alpha, "damping": damp, "iterations": r.iterations,
                   "converged": bool(r.converged), "relres_true": r.relres_true, "c_f": r.c_f,
                   "solve_s": r.seconds, "setup_s": round(setup, 1)}
        except Exception as e:  # noqa: BLE001
            rec = {"levels": L, "alpha": alpha, "damping": damp, "error": str(e)}
        rec.update({"cells": list(p.cells), "h": p.h, "unknowns": p.n})
        print(json.dumps(rec), flush=True)
        out.write(json.dumps(rec) + "\n")
        out.flush()
        gh = None
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
