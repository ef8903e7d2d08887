"""Timeline of the overlapped loop (IRCUR_OVERLAP=1) for a bench config:
per iteration the chain (core .. SVD) and strips intervals on the two
streams, from ircur_get_timeline."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("IRCUR_OVERLAP", "1")
import numpy as np
import torch

import bench
import paper_2010_07422_b200 as ir
from paper_2010_07422_b200 import gen

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
n1, n2, r, al, dts, _ = bench.CONFIGS[name]
if name in bench.VIDEO:  # video-like configs: zeta0 = max|D|
    f, h, w = bench.VIDEO[name]
    Dv, _, _ = gen.video_problem(frames=f, height=h, width=w, rank=r, seed=bench.DATA_SEED)
    D, linf = torch.from_numpy(np.ascontiguousarray(Dv, dtype=np.float32)).cuda(), None
else:
    D, linf, _ = gen.baseline_problem_device(n1, n2, r, al, bench.DATA_SEED, dtype=torch.float32)
cfg = ir.SolverConfig(rank=r, eps=bench.EPS, zeta0=linf, gamma=bench.GAMMA, mode="resampled",
                      max_iter=bench.MAX_ITER, seed=ir.RngSeed(bench.SOLVER_SEED))
for _ in range(2):
    res = ir.solve_device(D, cfg, profile="deferred")
it = res.trace.iterations
ms = np.zeros(5 * it, dtype=np.float32)
rc = res.ctx.lib.ircur_get_timeline(res.ctx.h, it, ms.ctypes.data_as(C.POINTER(C.c_float)))
assert rc == 0, res.ctx.lib.ircur_last_error()
t = ms.reshape(it, 5) * 1e3
print(f"{name}: {it} iterations; us relative to the first chain start")
print("  k  chain_start chain_end  strips_start strips_end  sampled_end   strips_us  chain_us  "
      "strips(k-1)->sampled(k)end  sampled(k)end->core(k+1)")
for k in range(it):
    cs, ce, ss, se, sm = t[k]
    prev_se = t[k - 1][3] if k > 0 else float("nan")
    nxt_cs = t[k + 1][0] if k + 1 < it else float("nan")
    print(f"{k:3d} {cs:11.1f} {ce:9.1f} {ss:13.1f} {se:10.1f} {sm:11.1f} {se - ss:11.1f} {ce - cs:9.1f} "
          f"{sm - prev_se:26.1f} {nxt_cs - sm:24.1f}")
