"""Quick fp32 check of the strip kernel in use against the oracle (diagnostics)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2010_07422_b200 as ir  # noqa: E402
from oracle import ircur_oracle as orc  # noqa: E402
import parity  # noqa: E402

cases = [(300, 280, 3, 0.1, "resampled"), (1000, 900, 5, 0.2, "resampled"), (2000, 2000, 5, 0.2, "fixed"),
         (600, 5000, 10, 0.2, "resampled"), (10000, 10000, 5, 0.2, "resampled")]
for n1, n2, r, alpha, mode in cases:
    D, L, S, linf = orc.baseline_problem_blocked(n1, n2, r, alpha, 7, dtype=np.float32)[0], None, None, None
    D64 = D.astype(np.float64)
    linf = float(np.abs(D64).max()) * 0.5
    kw = dict(rank=r, eps=1e-5, zeta0=linf, gamma=0.7, mode=mode, max_iter=60)
    t0 = time.time()
    out = ir.solve(D, ir.SolverConfig(seed=ir.RngSeed(3), **kw), device=0)
    t1 = time.time()
    ref = orc.solve(D64, seed=3, record_x=True, **kw)

    def resolve(mi, e):
        return ir.solve(D, ir.SolverConfig(seed=ir.RngSeed(3), **{**kw, "max_iter": mi, "eps": e}), device=0)
    try:
        rec = parity.check(out, ref, True, resolve=resolve, name=f"{n1}x{n2}")
        print("OK", rec, f"{t1 - t0:.2f}s", flush=True)
    except AssertionError as e:
        print("FAIL", parity.STATS[-1], str(e)[:300], flush=True)
