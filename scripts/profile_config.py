"""Per-kernel breakdown (CUDA-event profile, algorithmic bytes) of one solve of a BASELINE config.

    python scripts/profile_config.py --config 3
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    a = ap.parse_args()
    import torch
    from paper_2511_16808_b200 import hmg, media
    if a.config == 3:
        p, kw = media.config_problem(3), dict(levels=6, alpha=0.5, restart=10, dtype="c64")
    elif a.config == 4:   # 1/2-scale replica, alpha frozen by reading R16
        p, kw = media.config_problem(4, scale=2), dict(levels=6, alpha=0.6, restart=20, dtype="c64")
    elif a.config == 1:
        p, kw = media.config_problem(1, n=4096), dict(levels=9, alpha=0.25, restart=20, dtype="c64")
    elif a.config == 2:
        p, kw = media.config_problem(2), dict(levels=7, alpha=0.5, restart=20, dtype="c128")
    else:
        p, kw = media.config_problem(0), dict(levels=4, alpha=0.15, restart=10, dtype="c128")
    sm = "rb" if p.dim == 2 else "element"
    damp = [0.83, 0.5, 0.4, 0.65] if p.dim == 2 else [1.1, 0.7, 0.45, 0.6]
    gh = hmg.Hierarchy(hmg.Options(dim=p.dim, cells=p.cells, h=p.h, levels=kw["levels"], smoother=sm, damping=damp,
                                   dtype=kw["dtype"]), p.kappa, p.omega, p.gamma, kw["alpha"])
    cdt = torch.complex64 if kw["dtype"] == "c64" else torch.complex128
    q = torch.from_numpy(p.q.ravel()).to(cdt).cuda()
    x = torch.zeros_like(q)
    r = gh.fgmres_solve(q, x, restart=kw["restart"], tol=1e-6, maxiter=4000)
    hmg.profile_begin()
    r = gh.fgmres_solve(q, x, restart=kw["restart"], tol=1e-6, maxiter=4000)
    prof = hmg.profile_report()
    tot = sum(v["ms"] for v in prof.values())
    rows = sorted(prof.items(), key=lambda kv: -kv[1]["ms"])
    print(json.dumps({"config": a.config, "iterations": r.iterations, "kernel_ms": round(tot, 2)}))
    for k, v in rows[:40]:
        print(f"{k:32s} {v['ms']:9.2f} ms {v['launches']:6d} {v['bytes'] / (v['ms'] * 1e-3) / 1e9 if v['ms'] else 0:9.1f} GB/s")


if __name__ == "__main__":
    main()
