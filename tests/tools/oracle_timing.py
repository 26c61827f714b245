"""(Test infrastructure: lives under tests/ because it runs the oracle.)
Oracle (CPU, SciPy, complex128) timed on the GPU box's host, beside the GPU numbers
(SURVEY §8(d) "Oracle timing beside it").  Setup and solve are reported separately.
Small cases are solved in full; for the large ones the first restart cycle (m iterations)
is timed and the full solve is extrapolated with the GPU's iteration count for the same
configuration (labelled "extrapolated").

    python tests/tools/oracle_timing.py [--out profiles/r01_oracle_timing.jsonl] [--budget-s 900]
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

RB2 = [0.83, 0.5, 0.4, 0.65]
EL3 = [1.1, 0.7, 0.45, 0.6]


def host_info():
    model = platform.processor()
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    from threadpoolctl import threadpool_info
    blas = [{"api": i.get("internal_api"), "threads": i.get("num_threads")} for i in threadpool_info()]
    return {"cpu_model": model, "affinity_cores": len(os.sched_getaffinity(0)), "blas": blas,
            "python": platform.python_version()}


def cases():
    from paper_2511_16808_b200 import media
    # name, problem factory, options, restart, GPU iterations or None = solve in full
    yield "config0 2D 128^2 L4 a.15 FGMRES(10)", lambda: media.config_problem(0), dict(levels=4, alpha=0.15), 10, None
    yield "config1 2D 512^2 L6 a.25 FGMRES(20)", lambda: media.config_problem(1, n=512), dict(levels=6, alpha=0.25), 20, None
    yield "config1 2D 1024^2 L7 a.25 FGMRES(20)", lambda: media.config_problem(1, n=1024), dict(levels=7, alpha=0.25), 20, 219
    yield "config1 2D 4096^2 L9 a.25 FGMRES(20)", lambda: media.config_problem(1, n=4096), dict(levels=9, alpha=0.25), 20, 872
    yield "config2 2D 2048x640 L7 a.5 FGMRES(20)", lambda: media.config_problem(2), dict(levels=7, alpha=0.5), 20, 409
    yield "config3-family 3D 64^3 L4 a.5 FGMRES(10)", lambda: media.homogeneous_problem(3, 64, sponge=16), dict(levels=4, alpha=0.5), 10, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_oracle_timing.jsonl"))
    ap.add_argument("--budget-s", type=float, default=900.0)
    args = ap.parse_args()
    from threadpoolctl import threadpool_limits
    from oracle.cycle import vcycle
    from oracle.fgmres import fgmres_solve
    from oracle.hierarchy import Options, build_hierarchy
    info = host_info()
    out = open(args.out, "w")
    out.write(json.dumps({"host": info}) + "\n")
    print(json.dumps({"host": info}), flush=True)
    t_start = time.time()
    for name, mk, kw, m, gpu_its in cases():
        if time.time() - t_start > args.budget_s:
            break
        p = mk()
        sm = "rb" if p.dim == 2 else "element"
        opts = Options(dim=p.dim, cells=p.cells, h=p.h, levels=kw["levels"], smoother=sm,
                       damping=RB2 if p.dim == 2 else EL3)
        t0 = time.perf_counter()
        hier = build_hierarchy(opts, p.kappa, p.omega, p.gamma, kw["alpha"])   # setup may use BLAS threads
        setup = time.perf_counter() - t0
        maxiter = m if gpu_its else 2000
        with threadpool_limits(1):                                          # sparse solve: one core
            t0 = time.perf_counter()
            _, res = fgmres_solve(hier.H, p.q.ravel(), lambda v: vcycle(hier, v), restart=m, tol=1e-6,
                                  maxiter=maxiter)
            solve = time.perf_counter() - t0
        its = res["iterations"]
        rec = {"config": name, "unknowns": p.n, "setup_s": round(setup, 2), "solve_s": round(solve, 2),
               "iterations_timed": its, "s_per_iteration": solve / max(its, 1),
               "unknown_updates_per_s": p.n * its / solve, "solve_threads": 1}
        if gpu_its:
            rec["extrapolated_full_solve_s"] = round(solve / its * gpu_its, 1)
            rec["extrapolated_with_gpu_iterations"] = gpu_its
        else:
            rec["converged"] = bool(res["converged"])
        print(json.dumps(rec), flush=True)
        out.write(json.dumps(rec) + "\n")
        out.flush()


if __name__ == "__main__":
    main()
