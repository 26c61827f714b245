"""Benchmark: FGMRES + additive-Vanka V-cycle time-to-solve on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--n 4096] [--dtype c64|c128]

One STEP = one full solve H x = q from x0 = 0 to a true relative residual
< 1e-6 (FGMRES(20) right-preconditioned by one V(1,1)-cycle, BASELINE.json
configs[1]: 2D homogeneous, N x N cells, 10 points per wavelength, 16-node
sponge, centre point source, log2(N) - 3 levels, alpha = 0.25).
Setup (hmg_build_hierarchy) is excluded, as in the paper.

value = unknown-updates/s = (fine unknowns x FGMRES iterations) / time-to-solve.
With --gpus N > 1 (torchrun, one process per GPU) the SAME problem is
slab-partitioned over the N GPUs (y-slabs, NCCL halo exchange
and dot-product allreduce inside libhmg, coarse levels replicated), i.e. strong
scaling.  Time is measured with CUDA events on the solve stream, barrier +
synchronize on both sides, max over ranks.  Inputs (>= 134 MB per vector at N=4096, GBs of working set) are larger
than the 126 MB L2.

--impl reference times the CPU oracle (oracle/, SciPy, as it stands) on the
host cores on a bounded sample of the SAME workload: the oracle hierarchy of the
4096^2 problem is built once (setup reported, not timed), then each step is one
FGMRES(20) iteration (maxiter = 1).  The default run's cpu_baseline does the same
with 2 iterations.

--gpus N > 1 without a torchrun environment re-launches this script under
`python -m torch.distributed.run --nproc-per-node N` (127.0.0.1 rendezvous);
--dry-run stops every rank right after the rendezvous (CPU test of the launch).
Extra keys of the JSON line: "c128" (the same 4096^2 solve in complex128),
"config3" (BASELINE configs[3], 3D 256^3, c64), "multi_rhs" (4 sources batched).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FGMRES+V-cycle time-to-solve (s), unknown-updates/s, % HBM roofline @1-8 GPU"
UNIT = "unknown-updates/s"
ALPHA = {512: 0.25, 1024: 0.25, 2048: 0.25, 4096: 0.25}
DAMP_RB = [0.83, 0.5, 0.4, 0.65]   # Table 5.1, last value reused
RESTART, TOL = 20, 1e-6


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "of measured (MEASURED_PEAKS.json hbm_gbs: STREAM-style copy, the only HBM figure)"
    return 6650.0, "of fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 8:
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def build_problem(n):
    from paper_2511_16808_b200 import media
    return media.config_problem(1, n=n)


def levels_for(n):
    return max(2, n.bit_length() - 1 - 3)   # log2(N) - 3, coarsest 17^2


def run_ours(args):
    import numpy as np
    import torch
    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dist = None
    comm = None
    from paper_2511_16808_b200 import hmg
    if ws > 1:
        import torch.distributed as dist
        from paper_2511_16808_b200 import dist as hd
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = hd.nccl_comm()                # libhmg's own NCCL communicator (halos, dots, allgather)
    n = args.n
    p = build_problem(n)
    L = levels_for(n)
    alpha = ALPHA.get(n, 0.25)
    opts = hmg.Options(dim=2, cells=p.cells, h=p.h, levels=L, damping=DAMP_RB, dtype=args.dtype)
    stream = torch.cuda.current_stream()
    t0 = time.time()
    gh = hmg.Hierarchy(opts, p.kappa, p.omega, p.gamma, alpha, comm=comm)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    cdt = torch.complex64 if args.dtype == "c64" else torch.complex128
    lo, hi = gh.level_rows(0)                # this rank's slab of rows (all rows on one GPU)
    q = torch.from_numpy(np.ascontiguousarray(p.q[lo:hi]).ravel()).to(cdt).cuda()
    x = torch.zeros_like(q)
    N = p.n                                  # unknowns of the WHOLE problem

    reps = []
    for _ in range(args.warmup):
        reps.append(gh.fgmres_solve(q, x, restart=RESTART, tol=TOL, maxiter=args.maxiter))
    # ---------------------------------------------------------------- timed region
    clk = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk.start()
    l0 = hmg.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    its = []
    for k in range(args.steps):
        ev[k][0].record(stream)
        r = gh.fgmres_solve(q, x, restart=RESTART, tol=TOL, maxiter=args.maxiter)
        ev[k][1].record(stream)
        its.append(r.iterations)
        reps.append(r)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = hmg.launch_count() - l0
    clocks = clk.stop()
    ms = [a.elapsed_time(b) for a, b in ev]
    ms_step = sum(ms) / len(ms)
    if dist:
        t = torch.tensor([ms_step], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    iters = its[-1]
    converged = all(r.converged for r in reps)
    value = N * iters / (ms_step * 1e-3)     # whole-problem unknown-updates / max-over-ranks time

    # ---------------------------------------------------------------- e2e: host buffers through the C-ABI
    # host wall clock around the C-ABI call that takes HOST buffers (copies inside the call)
    qh = q.cpu().pin_memory()
    xh = torch.zeros_like(qh).pin_memory()
    e_ms = []
    for k in range(max(2, min(args.steps, 3))):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        re = gh.fgmres_solve_host(qh, xh, restart=RESTART, tol=TOL, maxiter=args.maxiter)
        torch.cuda.synchronize()
        e_ms.append((time.perf_counter() - t0) * 1e3)
    e_ms = sum(e_ms) / len(e_ms)
    if dist:
        t = torch.tensor([e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    e2e = {"value": N * re.iterations / (e_ms * 1e-3), "unit": UNIT,
           "time_to_solve_s": e_ms * 1e-3, "clock": "host wall clock (time.perf_counter), mean of the samples",
           "h2d_bytes_per_step": qh.numel() * qh.element_size(),
           "d2h_bytes_per_step": xh.numel() * xh.element_size()}

    # ---------------------------------------------------------------- multi-RHS batch
    multi = None
    if ws == 1 and args.nrhs > 1:
        multi = multi_rhs(gh, p, n, args, cdt, stream, value)

    # ---------------------------------------------------------------- live per-kernel roofline (one extra solve)
    hmg.profile_begin()
    gh.fgmres_solve(q, x, restart=RESTART, tol=TOL, maxiter=args.maxiter)
    prof = hmg.profile_report()
    peak, peak_src = _peaks()
    kern = sorted(prof.items(), key=lambda kv: -kv[1]["ms"])
    tot_ms = sum(v["ms"] for v in prof.values())
    top_name, top = kern[0]
    per_launch_bytes = top["bytes"] / top["launches"]
    avg_ms = top["ms"] / top["launches"]
    achieved = per_launch_bytes / (avg_ms * 1e-3) / 1e9
    traffic, traffic_ratio = None, None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        tj = json.load(open(tf))
        traffic = tj.get(f"{top_name}|{args.dtype}|{n}")
        traffic_ratio = tj.get(f"{top_name}|{args.dtype}|{n}|ratio")
    table = {k: {"launches": v["launches"], "ms_total": round(v["ms"], 3),
                 "share": round(v["ms"] / tot_ms, 4) if tot_ms else None,
                 "GBps": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1) if v["ms"] > 0 else None}
             for k, v in kern}
    roofline = {"bound": "hbm", "kernel": top_name, "achieved": round(achieved, 1), "peak": peak,
                "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                "traffic_source": "profiles/ncu_traffic.json: mean ncu dram__bytes_read.sum + dram__bytes_write.sum "
                                  "per launch over one restart cycle's launches (ncu --set full)",
                "traffic_over_algorithmic": traffic_ratio,
                "bytes_per_launch": per_launch_bytes, "avg_launch_ms": avg_ms,
                "share_of_step": round(top["ms"] / tot_ms, 4) if tot_ms else None}
    # whole-solve modelled HBM fraction: algorithmic bytes of every kernel / device time
    all_bytes = sum(v["bytes"] for v in prof.values())

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak",
        "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic",
        "time_to_solve_s": ms_step * 1e-3, "iterations": iters, "converged": converged,
        "config": {"workload": f"BASELINE configs[1]: 2D homogeneous {n}x{n} cells ({N} unknowns), 10 ppw, "
                               f"16-node sponge, centre source, {L}-level V(1,1) RB-Vanka + lev-dep Galerkin, "
                               f"alpha={alpha}, FGMRES({RESTART}) to {TOL}",
                   "cells": [n, n], "levels": L, "alpha": alpha, "restart": RESTART, "tol": TOL,
                   "parallelism": (f"slab-partitioned over {ws} GPUs (y-slabs, NCCL halos + allreduce, "
                                   f"coarse levels replicated)") if ws > 1 else "single GPU",
                   "l2": "inputs larger than L2 (every vector >= 134 MB at N=4096; no flush needed)",
                   "precision": ("c64: fine-level vectors, Krylov basis and all coefficients stored in fp32 complex; "
                                 "coarse-level vectors, FGMRES iterate / RHS / restart residual in fp64; arithmetic "
                                 "fp64 except the fine post-sweep residual (fp32, difference form) -- DESIGN.md 4.1")
                   if args.dtype == "c64" else "c128: fp64 complex storage and arithmetic",
                   "setup_s": round(setup_s, 2)},
        "clocks": clocks, "e2e": e2e, "gpu_launches": launches,
        "roofline": roofline,
        "solve_hbm_frac_modelled": round(all_bytes / (tot_ms * 1e-3) / 1e9 / peak, 4) if tot_ms else None,
        "kernel_time_per_step_ms": round(tot_ms, 3),
        "kernel_launches_per_step": int(sum(v["launches"] for v in prof.values())),
        "kernels": table,
    }
    if multi:
        out["multi_rhs"] = multi
    if ws == 1 and not args.no_extra:
        del gh
        torch.cuda.empty_cache()
        out["c128"] = extra_c128(n, args)
        torch.cuda.empty_cache()
        out["config3"] = extra_config3(args)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.cpu_n, args.cpu_iters)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


def multi_rhs(gh, p, n, args, cdt, stream, single_value):
    """nrhs point sources at seeded positions in the interior (many shots on one
    medium) solved as ONE batch (hmg_fgmres_solve_batch): one warm-up
    batch, one timed batch (CUDA events).  Aggregate unknown-updates/s over all
    right-hand sides, and the ratio to the single-RHS value of the same run."""
    import numpy as np
    import torch
    rng = np.random.default_rng(11)
    N = p.n
    Q = np.zeros((args.nrhs, N), np.complex128)
    Q[0] = p.q.ravel()
    nodes = n + 1
    for k in range(1, args.nrhs):
        ix, iy = rng.integers(32, nodes - 32, size=2)
        Q[k, iy * nodes + ix] = p.q.ravel().max()
    q = torch.from_numpy(Q).to(cdt).cuda()
    x = torch.zeros_like(q)
    gh.fgmres_solve_batch(q, x, restart=RESTART, tol=TOL, maxiter=args.maxiter)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    reps = gh.fgmres_solve_batch(q, x, restart=RESTART, tol=TOL, maxiter=args.maxiter)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    its = [r.iterations for r in reps]
    v = N * sum(its) / (ms * 1e-3)
    return {"nrhs": args.nrhs, "value": v, "unit": UNIT, "batch_time_s": ms * 1e-3, "iterations": its,
            "converged": all(r.converged for r in reps), "vs_single_rhs": round(v / single_value, 3),
            "sources": "config-1 centre source + seeded interior point sources (numpy default_rng(11))"}


def _timed_solves(gh, q, restart, nsolve, maxiter):
    """1 warm-up solve, then nsolve solves timed with CUDA events on the stream; median."""
    import torch
    x = torch.zeros_like(q)
    gh.fgmres_solve(q, x, restart=restart, tol=TOL, maxiter=maxiter)
    stream = torch.cuda.current_stream()
    ms, r = [], None
    for _ in range(nsolve):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        r = gh.fgmres_solve(q, x, restart=restart, tol=TOL, maxiter=maxiter)
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return statistics.median(ms), r


def extra_c128(n, args):
    """BASELINE configs[1] names complex64 AND complex128: the same solve in c128."""
    import torch
    from paper_2511_16808_b200 import hmg
    p = build_problem(n)
    gh = hmg.Hierarchy(hmg.Options(dim=2, cells=p.cells, h=p.h, levels=levels_for(n), damping=DAMP_RB,
                                   dtype="c128"), p.kappa, p.omega, p.gamma, ALPHA.get(n, 0.25))
    q = torch.from_numpy(p.q.ravel()).cuda()
    ms, r = _timed_solves(gh, q, RESTART, 2, args.maxiter)
    return {"dtype": "c128", "time_to_solve_s": ms * 1e-3, "iterations": r.iterations, "converged": bool(r.converged),
            "value": p.n * r.iterations / (ms * 1e-3), "unit": UNIT,
            "timing": "median of 2 device-timed solves after 1 warm-up"}


def extra_config3(args):
    """BASELINE configs[3]: 3D homogeneous 256^3 cells, 6 levels, element Vanka, alpha 0.5,
    FGMRES(10), c64 -- the paper's 3D timing experiment setting."""
    import torch
    from paper_2511_16808_b200 import hmg, media
    p = media.config_problem(3)
    t0 = time.time()
    gh = hmg.Hierarchy(hmg.Options(dim=3, cells=p.cells, h=p.h, levels=6, smoother="element",
                                   damping=[1.1, 0.7, 0.45, 0.6], dtype="c64"), p.kappa, p.omega, p.gamma, 0.5)
    torch.cuda.synchronize()
    setup = time.time() - t0
    q = torch.from_numpy(p.q.ravel()).to(torch.complex64).cuda()
    ms, r = _timed_solves(gh, q, 10, 3, args.maxiter)
    return {"workload": "BASELINE configs[3]: 3D 256^3 cells (16974593 unknowns), 6-level V(1,1) element Vanka, "
                        "lev-dep Galerkin, alpha 0.5, FGMRES(10) to 1e-6, c64",
            "time_to_solve_s": ms * 1e-3, "ms_per_iteration": ms / max(r.iterations, 1), "iterations": r.iterations,
            "converged": bool(r.converged), "value": p.n * r.iterations / (ms * 1e-3), "unit": UNIT,
            "setup_s": round(setup, 2), "timing": "median of 3 device-timed solves after 1 warm-up"}


_ORACLE = {}
_ORACLE_SETUP = {}


def _oracle_sample(n, iters):
    """Oracle (as it stands) on config 1 at n x n: setup untimed (built once; its
    time is kept in _ORACLE_SETUP), then a fixed number of FGMRES iterations timed
    (the first iterations of the first restart cycle); returns
    (unknown-updates/s, seconds, N, iterations)."""
    from threadpoolctl import threadpool_limits
    from oracle.cycle import vcycle
    from oracle.fgmres import fgmres_solve
    from oracle.hierarchy import Options as OOptions, build_hierarchy
    p = build_problem(n)
    L = levels_for(n)
    with threadpool_limits(1):
        if n not in _ORACLE:
            ts = time.perf_counter()
            _ORACLE[n] = build_hierarchy(OOptions(dim=2, cells=p.cells, h=p.h, levels=L, damping=DAMP_RB), p.kappa,
                                         p.omega, p.gamma, ALPHA.get(n, 0.25))
            _ORACLE_SETUP[n] = time.perf_counter() - ts
        oh = _ORACLE[n]
        t0 = time.perf_counter()
        _, info = fgmres_solve(oh.H, p.q.ravel(), lambda v: vcycle(oh, v), restart=RESTART, tol=TOL,
                               maxiter=iters)
        dt = time.perf_counter() - t0
    N = p.n
    return N * info["iterations"] / dt, dt, N, info["iterations"]


def cpu_baseline(n, iters):
    v, dt, N, it = _oracle_sample(n, iters)
    return {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"oracle (SciPy, complex128, 1 thread) on the bench workload itself (config 1, {n}x{n} cells, "
                      f"{N} unknowns): the first {it} FGMRES({RESTART}) iterations timed ({dt:.1f} s); setup "
                      f"{_ORACLE_SETUP.get(n, 0):.0f} s, not timed (P:1026-1027)",
            "setup_s": round(_ORACLE_SETUP.get(n, 0), 1)}


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    n = args.cpu_n
    rates, secs = [], []
    for k in range(args.warmup + args.steps):
        v, dt, N, it = _oracle_sample(n, args.cpu_iters)
        if k >= args.warmup:
            rates.append(v)
            secs.append(dt)
    value = sum(rates) / len(rates)
    ws = int(os.environ.get("WORLD_SIZE", args.gpus))
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / len(secs),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
           "data": "synthetic",
           "config": {"workload": f"BASELINE configs[1], the bench workload itself ({n}x{n} cells), bounded sample: "
                                  f"{args.cpu_iters} FGMRES({RESTART}) iteration(s) per step (the full N=4096 solve "
                                  f"is hours in SciPy)", "cells": [n, n], "levels": levels_for(n),
                      "oracle_setup_s": round(_ORACLE_SETUP.get(n, 0), 1)},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": f"{n}x{n}, {args.cpu_iters} iteration(s) per step, setup "
                                      f"({_ORACLE_SETUP.get(n, 0):.0f} s) excluded"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def relaunch(args):
    """--gpus N > 1 outside torchrun: re-run this script under torch.distributed.run,
    one process per GPU, rendezvous on 127.0.0.1 (the driver's own launch line)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dry_run(args):
    """Rendezvous only (CPU): every rank reports itself, rank 0 the world size."""
    ws, rank, local = _dist()
    import torch.distributed as dist
    rec = {"dry_run": True, "rank": rank, "world_size": ws, "local_rank": local, "gpus": args.gpus}
    if ws > 1:
        dist.init_process_group("gloo")
        t = __import__("torch").tensor([1])
        dist.all_reduce(t)
        rec["ranks_seen"] = int(t.item())
        for r in range(ws):  # one rank at a time: the ranks share one stdout pipe
            if r == rank:
                os.write(1, (json.dumps(rec) + "\n").encode())
            dist.barrier()
        dist.destroy_process_group()
    else:
        rec["ranks_seen"] = 1
        os.write(1, (json.dumps(rec) + "\n").encode())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--dtype", default="c64", choices=["c64", "c128"])
    ap.add_argument("--maxiter", type=int, default=4000)
    ap.add_argument("--cpu-n", type=int, default=4096, help="oracle sample grid (default: the bench workload)")
    ap.add_argument("--cpu-iters", type=int, default=None,
                    help="oracle FGMRES iterations per sample (default: 2 for cpu_baseline, 1 per reference step)")
    ap.add_argument("--no-extra", action="store_true", help="skip the c128 and config3 extra keys")
    ap.add_argument("--dry-run", action="store_true", help="launch / rendezvous only (no CUDA)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nrhs", type=int, default=4, help="batch size of the multi-RHS line (<= 1: skip)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.dry_run:
        dry_run(args)
        return
    if args.impl == "reference":
        if args.cpu_iters is None:
            args.cpu_iters = 1
        run_reference(args)
    else:
        if args.cpu_iters is None:
            args.cpu_iters = 2
        run_ours(args)


if __name__ == "__main__":
    main()
