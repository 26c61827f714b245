"""(Test infrastructure: lives under tests/ because it runs the oracle.)
Writes the at-scale oracle goldens under tests/golden/ (VERDICT r01 "Next round" 1):
FGMRES + V(1,1) solves of BASELINE.json configurations at sizes the CPU oracle
finishes in minutes, recorded so that the -m gpu tests can compare the CUDA path
with them without re-running the oracle (tests/test_gpu_golden.py).

Every number written here comes from oracle/ only (no CUDA path is imported);
the inputs are the seeded generators of paper_2511_16808_b200.media, and their
SHA-256 is stored so that a drifting generator fails the test instead of
silently comparing different problems.

    python tests/tools/make_golden.py CASE [CASE ...]      (cases: see CASES)

Per case: iterations, the full history of estimated relative residuals, the
true relative residual, restarts; one V-cycle z = MG(q) and the FGMRES solution
x at 256 seeded sample nodes (+ the source node and the corners) together with
max|z|, max|x| and their 2-norms.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

RB2 = [0.83, 0.5, 0.4, 0.65]    # Table 5.1, 2D RB row
EL3 = [1.1, 0.7, 0.45, 0.6]     # Table 5.1, 3D element row

# name -> (problem factory args, levels, alpha, restart, smoother, damping)
CASES = {
    # BASELINE configs[1] at N = 1024: 7 levels, alpha 0.25 (219 iterations)
    "config1_n1024": (dict(cfg=1, n=1024), 7, 0.25, 20, "rb", RB2),
    # configs[3] family scaled to 128^3 cells: 5 levels, alpha 0.5, FGMRES(10) (29)
    "config3_n128": (dict(cfg=3, n=128), 5, 0.5, 10, "element", EL3),
    # configs[4] generator (seed 4) at 1/4 scale: 192 x 192 x 96 cells, h = 100 m, 5 levels
    # (SURVEY §8(d) "full parity on a scaled replica ... 192x192x96 cells, h = 100 m, 5 levels")
    "config4_s4": (dict(cfg=4, scale=4), 5, 0.5, 20, "element", EL3),
    # the same replica with the shift frozen for config 4 by the 1/2-scale sweep (reading R16)
    "config4_s4_a06": (dict(cfg=4, scale=4), 5, 0.6, 20, "element", EL3),
}


def problem(spec):
    from paper_2511_16808_b200 import media
    spec = dict(spec)
    return media.config_problem(spec.pop("cfg"), **spec)


def input_sha(p):
    h = hashlib.sha256()
    for a in (p.kappa, p.gamma, p.q):
        h.update(np.ascontiguousarray(a).tobytes())
    h.update(repr((p.cells, float(p.h), float(p.omega))).encode())
    return h.hexdigest()


def sample_nodes(p, n=256, seed=123):
    rng = np.random.default_rng(seed)
    N = p.n
    idx = set(int(i) for i in rng.integers(0, N, size=n))
    idx.add(int(np.argmax(np.abs(p.q.ravel()))))      # the source node
    idx.update([0, N - 1])
    return sorted(idx)


def run(name, maxiter=3000):
    from threadpoolctl import threadpool_limits
    from oracle.cycle import vcycle
    from oracle.fgmres import fgmres_solve
    from oracle.hierarchy import Options, build_hierarchy
    spec, levels, alpha, m, sm, damp = CASES[name]
    p = problem(spec)
    t0 = time.time()
    oh = build_hierarchy(Options(dim=p.dim, cells=p.cells, h=p.h, levels=levels, smoother=sm, damping=damp),
                         p.kappa, p.omega, p.gamma, alpha)
    setup_s = time.time() - t0
    q = p.q.ravel()
    idx = sample_nodes(p)
    with threadpool_limits(1):
        z = vcycle(oh, q)
        t0 = time.time()
        x, info = fgmres_solve(oh.H, q, lambda v: vcycle(oh, v), restart=m, tol=1e-6, maxiter=maxiter)
        solve_s = time.time() - t0
    pack = lambda v: [[float(v[i].real), float(v[i].imag)] for i in idx]
    rec = {
        "_source": "tests/tools/make_golden.py (oracle/ only, complex128)",
        "case": name, "problem": {k: v for k, v in spec.items()}, "cells": list(p.cells), "h": p.h,
        "omega": p.omega, "levels": levels, "alpha": alpha, "restart": m, "smoother": sm, "damping": damp,
        "tol": 1e-6, "input_sha256": input_sha(p),
        "iterations": int(info["iterations"]), "converged": bool(info["converged"]),
        "restarts": int(info["restarts"]), "true_relres": float(info["true_relres"]),
        "history": [float(v) for v in info["history"]],
        "samples": idx,
        "vcycle": {"values": pack(z), "max_abs": float(np.abs(z).max()), "norm2": float(np.linalg.norm(z))},
        "solution": {"values": pack(x), "max_abs": float(np.abs(x).max()), "norm2": float(np.linalg.norm(x))},
        "oracle_setup_s": round(setup_s, 1), "oracle_solve_s": round(solve_s, 1),
    }
    out = os.path.join(ROOT, "tests", "golden", f"at_scale_{name}.json")
    with open(out, "w") as fh:
        json.dump(rec, fh, indent=1)
    print(name, rec["iterations"], rec["converged"], f"setup {setup_s:.0f}s solve {solve_s:.0f}s", flush=True)


if __name__ == "__main__":
    for c in sys.argv[1:] or list(CASES):
        run(c)
