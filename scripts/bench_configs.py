"""Time-to-solve on every BASELINE.json configuration (report, not the bench contract).

    python scripts/bench_configs.py [--out profiles/r01_configs.jsonl] [--only 0,1,2,3,4]

One warm-up solve, then the median of 3 device-timed solves per configuration
(CUDA events inside hmg_fgmres_solve; setup excluded as in the paper,
P:1026-1027).  Config 4 runs as the 1/2-scale replica of the same generator
(384^2 x 192 cells, h = 50 m): the full 768^2 x 384 grid's replicated fp64
setup does not fit one GPU.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

RB2 = [0.83, 0.5, 0.4, 0.65]
EL3 = [1.1, 0.7, 0.45, 0.6]


def cases():
    from paper_2511_16808_b200 import media
    yield "config0 2D 128^2 c128 L4 a.15 FGMRES(10)", lambda: media.config_problem(0), dict(levels=4, alpha=0.15,
                                                                                            restart=10, dtype="c128")
    for n in (512, 1024, 2048, 4096):
        for dt in ("c64", "c128"):
            yield (f"config1 2D {n}^2 {dt} L{n.bit_length() - 4} a.25 FGMRES(20)",
                   (lambda n=n: media.config_problem(1, n=n)),
                   dict(levels=n.bit_length() - 4, alpha=0.25, restart=20, dtype=dt))
    yield "config2 2D 2048x640 layered c128 L7 a.5 FGMRES(20)", lambda: media.config_problem(2), dict(
        levels=7, alpha=0.5, restart=20, dtype="c128")
    yield "config3 3D 256^3 c64 L6 a.5 FGMRES(10)", lambda: media.config_problem(3), dict(
        levels=6, alpha=0.5, restart=10, dtype="c64")
    # config 4 at 1/2 scale with the shift frozen by the sweep (reading R16: alpha 0.6)
    yield "config4 3D 384^2x192 (1/2 scale) thrust c64 L6 a.6 FGMRES(20)", lambda: media.config_problem(4, scale=2), dict(
        levels=6, alpha=0.6, restart=20, dtype="c64")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_configs.jsonl"))
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    import torch
    from paper_2511_16808_b200 import hmg
    only = [c for c in args.only.split(",") if c]
    out = open(args.out, "a")
    for name, mk, kw in cases():
        if only and not any(name.startswith(f"config{c}") for c in only):
            continue
        p = mk()
        sm = "rb" if p.dim == 2 else "element"
        opts = hmg.Options(dim=p.dim, cells=p.cells, h=p.h, levels=kw["levels"], smoother=sm,
                           damping=RB2 if p.dim == 2 else EL3, dtype=kw["dtype"])
        t0 = time.time()
        gh = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, kw["alpha"])
        torch.cuda.synchronize()
        setup = time.time() - t0
        cdt = torch.complex64 if kw["dtype"] == "c64" else torch.complex128
        q = torch.from_numpy(p.q.ravel()).to(cdt).cuda()
        x = torch.zeros_like(q)
        reps = [gh.fgmres_solve(q, x, restart=kw["restart"], tol=1e-6, maxiter=4000) for _ in range(4)]
        secs = statistics.median(r.seconds for r in reps[1:])
        r = reps[-1]
        rec = dict(config=name, unknowns=p.n, iterations=r.iterations, converged=r.converged,
                   relres_true=r.relres_true, time_to_solve_s=secs,
                   unknown_updates_per_s=p.n * r.iterations / secs, setup_s=round(setup, 2),
                   ms_per_iteration=1e3 * secs / max(r.iterations, 1))
        print(json.dumps(rec), flush=True)
        out.write(json.dumps(rec) + "\n")
        del gh
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
