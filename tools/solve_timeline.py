"""Kernel timeline of one config-1 GMRES solve through torch.profiler (CUPTI): busy time per
kernel name and the idle gaps between consecutive kernels on the library stream (diagnostic).
usage: python tools/solve_timeline.py"""
import collections
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_02809_b200 import fracinv as F  # noqa: E402
from paper_2507_02809_b200.configs import NOISE, RESTART, SEED_BASE, TOL, baseline_problem  # noqa: E402

ctx = F.Context(0)
A = F.SystemOperator(baseline_problem(F, 1), ctx=ctx)
P = F.BlockTriangularPreconditioner(A)
mu = F.forward_solve(A, P).mu
z = F.build_rhs(A, F.add_gaussian_noise(mu, NOISE[1], SEED_BASE + 1)).z
b = torch.from_numpy(z).cuda()
opts = F.GmresOptions(TOL[1], 0, RESTART)
for _ in range(3):
    F.gmres(A, P, b, opts)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    F.gmres(A, P, b, opts)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
busy = collections.Counter()
cnt = collections.Counter()
for e in ev:
    busy[e.name.split("(")[0][:60]] += e.time_range.elapsed_us()
    cnt[e.name.split("(")[0][:60]] += 1
t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
print(f"span {(t1 - t0) / 1e3:.3f} ms, {len(ev)} device activities")
for e in ev[:8]:
    print(f"  +{(e.time_range.start - t0) / 1e3:8.3f} ms  {e.time_range.elapsed_us():8.1f} us  {e.name[:70]}")
for k, v in busy.most_common(14):
    print(f"  {v / 1e3:8.3f} ms  x{cnt[k]:4d}  {k}")
# gaps: union of busy intervals
iv = sorted((e.time_range.start, e.time_range.end) for e in ev)
gaps, end, big = 0.0, iv[0][1], []
for s, e in iv[1:]:
    if s > end:
        gaps += s - end
        big.append((s - end, s - t0))
    end = max(end, e)
big.sort(reverse=True)
print(f"idle {gaps / 1e3:.3f} ms; largest gaps (us, at ms): " +
      ", ".join(f"{g:.0f}@{at / 1e3:.2f}" for g, at in big[:12]))
