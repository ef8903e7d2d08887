"""e2e (solve from pinned host D) per call after device-resident solves, as
bench.py runs it, with the overlapped or the sequential loop."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2010_07422_b200 as ir
from paper_2010_07422_b200 import gen

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
os.environ["IRCUR_OVERLAP"] = sys.argv[2] if len(sys.argv) > 2 else "1"
n1, n2, r, al, dts, _ = bench.CONFIGS[name]
if name in bench.VIDEO:
    f, h, w = bench.VIDEO[name]
    Dv, _, _ = gen.video_problem(frames=f, height=h, width=w, rank=r, seed=bench.DATA_SEED)
    D = torch.from_numpy(np.ascontiguousarray(Dv, dtype=np.float32)).cuda()
    linf = None
else:
    D, linf, _ = gen.baseline_problem_device(n1, n2, r, al, bench.DATA_SEED, dtype=torch.float32)
cfg = ir.SolverConfig(rank=r, eps=bench.EPS, zeta0=linf, gamma=bench.GAMMA, mode="resampled",
                      max_iter=bench.MAX_ITER, seed=ir.RngSeed(bench.SOLVER_SEED))
for _ in range(8):
    res = ir.solve_device(D, cfg, profile="deferred")
torch.cuda.synchronize()
Dh = torch.empty(D.shape, dtype=D.dtype, pin_memory=True)
Dh.copy_(D)
del D, res
ir.clear_cache()
torch.cuda.synchronize()
torch.cuda.empty_cache()
ts = []
for _ in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cur, sp, tr = ir.solve(Dh, cfg)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
    del cur, sp, tr
print(f"{name} overlap={os.environ['IRCUR_OVERLAP']} e2e ms={np.round(ts, 2).tolist()}", flush=True)
