"""Config 4 generator at 1/2 scale (384 x 384 x 192 cells, 28.6 M unknowns) solved
slab-partitioned over P virtual ranks on one GPU (LOCAL backend: the partitioned build --
setup windows, kept rows, gathered coarse level -- and the partitioned cycle with halos and
allreduced dots), against the single-GPU solve of the same problem: iterations and solution.

    python scripts/config4_partitioned.py [--ranks 4] [--alpha 0.6] [--levels 6]
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=4)
    ap.add_argument("--alpha", type=float, default=0.6)
    ap.add_argument("--levels", type=int, default=6)
    ap.add_argument("--scale", type=int, default=2)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    from paper_2511_16808_b200 import hmg, media
    p = media.config_problem(4, scale=a.scale)
    opts = hmg.Options(dim=3, cells=p.cells, h=p.h, levels=a.levels, smoother="element",
                       damping=[1.1, 0.7, 0.45, 0.6], dtype="c64")
    q = torch.from_numpy(p.q.ravel()).to(torch.complex64).cuda()
    t0 = time.time()
    single = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, a.alpha)
    x1 = torch.zeros_like(q)
    r1 = single.fgmres_solve(q, x1, restart=20, tol=1e-6, maxiter=1000)
    t_single = time.time() - t0
    x1h = x1.cpu().numpy().reshape(p.nodes[::-1])
    del single
    torch.cuda.empty_cache()
    group = hmg.LocalGroup(a.ranks)
    comms = [group.rank(r) for r in range(a.ranks)]
    res = [None] * a.ranks
    err = []

    def body(r):
        try:
            torch.cuda.set_device(0)
            gh = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, a.alpha, comm=comms[r])
            lo, hi = gh.level_rows(0)
            qs = torch.from_numpy(np.ascontiguousarray(p.q[lo:hi]).ravel()).to(torch.complex64).cuda()
            xs = torch.zeros_like(qs)
            rep = gh.fgmres_solve(qs, xs, restart=20, tol=1e-6, maxiter=1000)
            torch.cuda.synchronize()
            res[r] = (lo, hi, rep.iterations, bool(rep.converged), rep.relres_true, xs.cpu().numpy())
            del gh
        except BaseException as e:  # noqa: BLE001
            err.append(repr(e))

    t0 = time.time()
    th = [threading.Thread(target=body, args=(r,)) for r in range(a.ranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    t_part = time.time() - t0
    out = {"cells": list(p.cells), "unknowns": p.n, "levels": a.levels, "alpha": a.alpha, "ranks": a.ranks,
           "single": {"iterations": r1.iterations, "converged": bool(r1.converged), "relres": r1.relres_true,
                      "wall_s": round(t_single, 1)}, "errors": err}
    if not err:
        xp = np.concatenate([r[5].reshape(-1, p.nodes[1], p.nodes[0]) for r in res], axis=0)
        out["partitioned"] = {"rows": [[r[0], r[1]] for r in res], "iterations": [r[2] for r in res],
                              "converged": all(r[3] for r in res), "relres": res[0][4], "wall_s": round(t_part, 1),
                              "solution_rel_diff": float(np.abs(xp - x1h).max() / np.abs(x1h).max())}
    print(json.dumps(out))
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
