#!/bin/bash
# K5 A/B: config-4 (and 3) P^-1 device time on the smooth (Arnoldi) and random inputs with the phase trace,
# then the tau-PCG parity tests and the 2D goldens.  usage: bash tools/k5_check.sh [pytest -k expr]
mkdir -p gpurun_out
for c in 4 3; do
  CFG=$c timeout 300 python tools/smooth_papply.py 2>&1 | tail -1
done
FI_ITER_TRACE=1 CFG=4 timeout 300 python tools/smooth_papply.py 2>&1 | grep -v "^{" | tail -4
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_iterative.py tests/test_gpu_parity_large.py tests/test_gpu_goldens.py -k "${1:-tau or config2 or config3 or solve_matches or forward}" 2>&1 | tail -3
