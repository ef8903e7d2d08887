"""Compare the e_k trajectory of the strip kernel in use with the oracle on one
small problem (diagnostics): python tools/s6small.py n1 n2 r mode"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_07422_b200 as ir  # noqa: E402
from oracle import ircur_oracle as orc  # noqa: E402

n1, n2, r, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
D = orc.baseline_problem_blocked(n1, n2, r, 0.2, 70 + r, dtype=np.float32)[0]
linf = float(np.abs(D).max()) * 0.5
kw = dict(rank=r, eps=1e-5, zeta0=linf, gamma=0.7, mode=mode, max_iter=80)
ref = orc.solve(D.astype(np.float64), seed=5, **kw)
out = ir.solve(D, ir.SolverConfig(seed=ir.RngSeed(5), **kw), device=0)
print("iters", out[2].iterations, "ref", ref.iterations)
for k, (a, b) in enumerate(zip(out[2].errors, ref.errors)):
    print(f"{k:2d} {a:.6e} {b:.6e} {a / b - 1:+.2e}")
