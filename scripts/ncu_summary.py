"""Summarise ncu outputs into profiles/ (tracked).

    python scripts/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launches.md
    python scripts/ncu_summary.py full gpurun_out/prof.ncu-rep profiles/r01_ncu_full.md [--traffic-key NAME]
        [--traffic-kernel SUBSTRING]   (largest per-launch DRAM bytes among kernels matching SUBSTRING)

`launches`: the `--metrics gpu__time_duration.sum` launch list (cold-cache,
serialised: compare SHARES, not absolute times) aggregated per kernel.
`full`: the key `--set full` metrics per captured launch (DRAM bytes and
throughput, occupancy, pipe utilisation, top stall reasons).
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys


def short(name):
    name = re.sub(r"\(.*$", "", name)           # drop the parameter list
    return name.replace("void ", "").replace("hmg::", "")


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    unit = "ns"
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = d.get("Metric Unit", unit)
        v = float(d["Metric Value"].replace(",", ""))
        k = short(d["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = [f"# ncu launch list summary ({os.path.basename(src)})", "",
           f"{len(data)} launches captured; times are cold-cache and serialised (compare shares).", "",
           f"| kernel | launches | total ({unit}) | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {n} | {t:,.0f} | {t / tot:.1%} |")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out[:20]))


WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("launch__grid_size", "grid"),
]
STALLS = ["long_scoreboard", "barrier", "short_scoreboard", "wait", "math_pipe_throttle", "mio_throttle",
          "lg_throttle", "not_selected", "selected", "no_instruction", "dispatch_stall", "drain", "membar"]


def full(src, dst, traffic_key=None, traffic_kernel=None):
    raw = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = [f"# ncu --set full summary ({os.path.basename(src)})", ""]
    traffic = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = short(d.get("Kernel Name", "?"))
        out.append(f"## `{name}`  grid {d.get('Grid Size', '')} block {d.get('Block Size', '')}")
        for m, lab in WANT:
            if m in d:
                out.append(f"- {lab}: {d[m]} {u.get(m, '')}")
        st = []
        for s_ in STALLS:
            m = f"smsp__pcsamp_warps_issue_stalled_{s_}"
            if m in d and d[m] not in ("", "0"):
                st.append((float(d[m].replace(",", "")), s_))
        st.sort(reverse=True)
        if st:
            tot = sum(v for v, _ in st)
            out.append("- stall samples: " + ", ".join(f"{n} {v / tot:.0%}" for v, n in st[:5]))
        out.append("")
        try:
            rd = float(d["dram__bytes_read.sum"].replace(",", "")) * _scale(u["dram__bytes_read.sum"])
            wr = float(d["dram__bytes_write.sum"].replace(",", "")) * _scale(u["dram__bytes_write.sum"])
            traffic.setdefault(name, []).append(rd + wr)
        except (KeyError, ValueError):
            pass
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out[:40]))
    if traffic_key:
        tf = os.path.join(os.path.dirname(dst), "ncu_traffic.json")
        cur = json.load(open(tf)) if os.path.exists(tf) else {}
        # mean DRAM read+write bytes per captured launch of the matching kernel (the roofline's
        # `achieved` is an average over launches too)
        cand = [v for k, v in traffic.items() if not traffic_kernel or traffic_kernel in k]
        allv = [x for v in cand for x in v]
        if allv:
            cur[traffic_key] = sum(allv) / len(allv)
            cur[traffic_key + "|launches"] = len(allv)
        json.dump(cur, open(tf, "w"), indent=1)


def _scale(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)


if __name__ == "__main__":
    kind, src, dst = sys.argv[1:4]
    key = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
    kk = sys.argv[sys.argv.index("--traffic-kernel") + 1] if "--traffic-kernel" in sys.argv else None
    os.makedirs(os.path.dirname(dst) or ".", exist_ok=True)
    if kind == "launches":
        launches(src, dst)
    else:
        full(src, dst, key, kk)
