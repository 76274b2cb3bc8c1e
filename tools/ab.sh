#!/bin/bash
# A/B timing of library variants on one box: abx/<name>.so copied over the package library in turn,
# ROUNDS passes over the list, one tools/sweep_timing.py line per run (tuning aid).
# usage: tools/ab.sh v0 v1 ...   (ROUNDS, CFG from the environment; CMD overrides the timing command)
set -u
LIB=paper_2507_02809_b200/libfracinv_b200.so
cp "$LIB" /tmp/ab_orig.so
for r in $(seq "${ROUNDS:-2}"); do
  for v in "$@"; do
    cp "abx/$v.so" "$LIB"
    echo -n "$v "
    timeout 300 ${CMD:-python tools/sweep_timing.py} 2>/dev/null | tail -1
  done
done
cp /tmp/ab_orig.so "$LIB"
