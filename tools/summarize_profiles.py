#!/usr/bin/env python3
"""Summarise a round's GPU evidence into profiles/<tag>_summary.md.

Inputs (from gpurun_out/): an ncu launch list CSV (gpu__time_duration.sum per launch of the
bench's timed region) and `ncu --set full` reports of K2 (sweep_kernel) and K1 (toeplitz_apply).
Usage: python tools/summarize_profiles.py r01 gpurun_out/launches_r01.csv gpurun_out/prof_k2_r01.ncu-rep \
       gpurun_out/prof_k1_r01.ncu-rep
"""
import collections
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("fib::<unnamed>::", "").replace("void ", "").strip()
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {c} | {t:.3f} | {100 * t / tot:.1f}% |")
    out.append(f"| **total** | {sum(v[0] for v in agg.values())} | {tot:.3f} | 100% |")
    return "\n".join(out)


WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
]


def ncu_table(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for n, launch in enumerate(rows[2:]):
        name = launch[h.index("Kernel Name")].split("(")[0].replace("fib::<unnamed>::", "")
        out.append(f"\nlaunch {n}: `{name}`\n\n| metric | unit | value |\n|---|---|---|")
        for w in WANT:
            if w in h:
                i = h.index(w)
                out.append(f"| {w} | {units[i]} | {launch[i]} |")
        stalls = [(h[i], float(launch[i] or 0)) for i in range(len(h))
                  if h[i].startswith("smsp__average_warps_issue_stalled_") and h[i].endswith("_per_issue_active.ratio")]
        stalls = sorted(stalls, key=lambda x: -x[1])[:5]
        out.append("\ntop stall reasons (warps per issue): " + ", ".join(
            f"{s.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
            for s, v in stalls))
    return "\n".join(out)


def main():
    tag, launches, *reps = sys.argv[1:]
    md = [f"# GPU evidence, {tag}", "", "## Launch list of `bench.py --steps 1 --warmup 3 --profile` (timed region)",
          "", "Cold-cache, serialised ncu timings: compare shares, not absolutes.", "", launch_table(launches)]
    for r in reps:
        md += ["", f"## `ncu --set full` — {os.path.basename(r)}", ncu_table(r)]
    out = os.path.join(ROOT, "profiles", f"{tag}_summary.md")
    open(out, "w").write("\n".join(md) + "\n")
    print(out)


if __name__ == "__main__":
    main()
