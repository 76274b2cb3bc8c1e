#!/usr/bin/env python3
"""Per-kernel SASS instruction counts of the built library (cuobjdump -sass): the tensor-pipe and copy
instructions that prove the design (DMMA for K1 / the history products, UBLKCP / UBLKPF for the bulk copies
and prefetches, LDGSTS for cp.async, SHFL, BAR), written to profiles/<tag>/sass_summary.md.
usage: python tools/sass_summary.py r02"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2507_02809_b200", "libfracinv_b200.so")
OPS = ["DMMA", "DFMA", "DADD", "DMUL", "UBLKCP", "UBLKPF", "LDGSTS", "LDG", "STG", "LDS", "STS", "SHFL", "BAR", "ATOMG", "RED"]


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    counts, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", line)
        if cur and m:
            op = m.group(1)
            counts[cur]["_total"] += 1
            for o in OPS:
                if op == o:
                    counts[cur][o] += 1
    dem = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
    rows = ["| kernel | SASS instructions | " + " | ".join(OPS) + " |", "|---|---|" + "---|" * len(OPS)]
    for (name, c), d in sorted(zip(counts.items(), dem), key=lambda x: -x[0][1]["_total"]):
        short = d.replace("(anonymous namespace)::", "").replace("void ", "")
        short = re.sub(r"\(.*", "", short).replace("fib::", "")
        rows.append(f"| `{short[:60]}` | {c['_total']} | " + " | ".join(str(c[o]) for o in OPS) + " |")
    out = os.path.join(ROOT, "profiles", tag, "sass_summary.md")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        f.write(f"# SASS summary ({tag}): `cuobjdump -sass paper_2507_02809_b200/libfracinv_b200.so`, sm_100a\n\n")
        f.write("Static instruction counts per kernel (not executed counts).  DMMA = FP64 tensor-pipe MMA "
                "(mma.sync.m8n8k4.f64; tcgen05 has no f64 kind); UBLKCP / UBLKPF = cp.async.bulk copy / L2 "
                "prefetch; LDGSTS = cp.async.\n\n")
        f.write("\n".join(rows) + "\n")
    print(out)


if __name__ == "__main__":
    main()
