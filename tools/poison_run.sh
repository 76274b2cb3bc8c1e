#!/bin/bash
# Uninitialised-read check in place of compute-sanitizer (closed on this GPU pool): the GPU test files with every
# device allocation poisoned (FI_POISON=1: 0xff bytes = NaN doubles / ~0 counters), one file at a time under its
# own timeout.  A kernel that reads scratch it never wrote, or code relying on zeroed allocations, fails the
# parity asserts (or spins).  usage: bash tools/poison_run.sh [files]   (round 2 found: K5 left the pad columns of
# its output unwritten; fixed)
cd "$(dirname "$0")/.."
for f in ${@:-tests/test_gpu_*.py}; do
  echo "== $f"
  FI_POISON=1 timeout ${T:-420} python -m pytest "$f" -m gpu -q -x -k "not unpreconditioned" 2>&1 | tail -2
  echo "rc=${PIPESTATUS[0]}"
done
