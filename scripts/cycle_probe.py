"""Where the V-cycle time goes at the bench size: the whole preconditioner
application as it runs (graph replay, CUDA events, median of 50) against the
profiled per-kernel times by level (events around every launch, no graph).

    python scripts/cycle_probe.py [--n 4096]
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
    ap.add_argument("--n", type=int, default=4096)
    a = ap.parse_args()
    import torch
    from paper_2511_16808_b200 import hmg, media
    p = media.config_problem(1, n=a.n)
    L = a.n.bit_length() - 4
    gh = hmg.Hierarchy(hmg.Options(dim=2, cells=p.cells, h=p.h, levels=L, damping=[0.83, 0.5, 0.4, 0.65],
                                   dtype="c64"), p.kappa, p.omega, p.gamma, 0.25)
    f = torch.from_numpy(p.q.ravel()).to(torch.complex64).cuda()
    x = torch.zeros_like(f)
    s = torch.cuda.current_stream()
    for _ in range(5):
        gh.vcycle(f, x)
    ms = []
    for _ in range(50):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        gh.vcycle(f, x)
        e1.record(s)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    hmg.profile_begin()
    for _ in range(10):
        gh.vcycle(f, x)
    prof = hmg.profile_report()
    by_level = {}
    for k, v in prof.items():
        lvl = int(k.rsplit("@L", 1)[1]) if "@L" in k else -1
        by_level[lvl] = by_level.get(lvl, 0.0) + v["ms"] / 10
    rec = {"vcycle_ms_graph": statistics.median(ms), "profiled_ms_by_level": {str(k): round(v, 4) for k, v in sorted(by_level.items())}}
    l01 = by_level.get(0, 0) + by_level.get(1, 0)
    rec["graph_minus_profiled_L0_L1_ms"] = round(statistics.median(ms) - l01, 4)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
