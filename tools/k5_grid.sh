#!/bin/bash
# K5 grid-size sweep: config-4 P^-1 device time on the smooth (Arnoldi) and random inputs per FI_TAU_GRID,
# with the per-phase trace; then the tau-PCG parity tests at the chosen grid.  usage: bash tools/k5_grid.sh "148 96 74"
mkdir -p gpurun_out
for g in ${1:-148 96 74 65}; do
  echo "== grid $g"
  FI_TAU_GRID=$g CFG=${CFG:-4} timeout 300 python tools/smooth_papply.py 2>&1 | tail -1
  FI_TAU_GRID=$g FI_ITER_TRACE=1 CFG=${CFG:-4} timeout 300 python tools/smooth_papply.py 2>&1 | grep -v "^{" | tail -4
done
