"""Config 4 unpreconditioned GMRES(50), maxit 2000, tol 1e-8 (BASELINE configs[4]) on the golden's observation;
saves the report, history and recovered f to gpurun_out/unprec4.npz.  usage: python tools/unprec4.py"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_02809_b200 import fracinv as F  # noqa: E402
from paper_2507_02809_b200.configs import RESTART, baseline_problem  # noqa: E402

g = np.load(os.path.join(ROOT, "tests", "golden", "oracle_config4.npz"))
A = F.SystemOperator(baseline_problem(F, 4))
z = torch.from_numpy(F.build_rhs(A, g["mu_eps"]).z).cuda()
t0 = time.perf_counter()
x, rep = F.gmres(A, None, z, F.GmresOptions(1e-8, 2000, RESTART))
torch.cuda.synchronize()
t = time.perf_counter() - t0
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez(os.path.join(ROOT, "gpurun_out", "unprec4.npz"), f=x[-A.N:].cpu().numpy(), iterations=rep.iterations,
         history=np.array(rep.residual_history), converged=rep.converged, final_true_residual=rep.final_true_residual,
         seconds=t)
print(f"unpreconditioned config 4: {rep.iterations} iterations, converged {rep.converged}, final true residual "
      f"{rep.final_true_residual:.6e}, last history {rep.residual_history[-1]:.6e}, {t:.1f} s")
