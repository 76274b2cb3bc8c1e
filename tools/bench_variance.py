"""Run-to-run spread of the config-1 solve rate (diagnostic for bench.py): several timed passes of
K device-resident solves, with and without an nvidia-smi -lms 100 sampler running beside them.
usage: python tools/bench_variance.py [passes] [K]"""
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_02809_b200 import fracinv as F  # noqa: E402
from paper_2507_02809_b200.configs import NOISE, RESTART, SEED_BASE, TOL, baseline_problem  # noqa: E402

passes = int(sys.argv[1]) if len(sys.argv) > 1 else 4
K = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ctx = F.Context(0)
A = F.SystemOperator(baseline_problem(F, 1), ctx=ctx)
P = F.BlockTriangularPreconditioner(A)
mu = F.forward_solve(A, P).mu
z = F.build_rhs(A, F.add_gaussian_noise(mu, NOISE[1], SEED_BASE + 1)).z
b = torch.from_numpy(z).cuda()
opts = F.GmresOptions(TOL[1], 0, RESTART)
stream = torch.cuda.ExternalStream(ctx.stream)
for _ in range(3):
    F.gmres(A, P, b, opts)
torch.cuda.synchronize()
for sampler in (False, True, False):
    proc = None
    if sampler:
        proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "100"],
                                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        time.sleep(0.5)
    rates = []
    for _ in range(passes):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        it = 0
        for _ in range(K):
            _, rep = F.gmres(A, P, b, opts)
            it += rep.iterations
        e1.record(stream)
        torch.cuda.synchronize()
        rates.append(it / (e0.elapsed_time(e1) * 1e-3))
    if proc:
        proc.terminate()
    print(("sampler " if sampler else "quiet   ") + " ".join(f"{r:.1f}" for r in rates), flush=True)
