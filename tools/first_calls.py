import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench, paper_2010_07422_b200 as ir
from paper_2010_07422_b200 import gen
f, h, w = bench.VIDEO["cfg3"]
Dv, _, _ = gen.video_problem(frames=f, height=h, width=w, rank=2, seed=0)
Dh = torch.from_numpy(np.ascontiguousarray(Dv, dtype=np.float32)).pin_memory()
cfg = ir.SolverConfig(rank=2, eps=1e-5, zeta0=None, gamma=0.7, mode="resampled", max_iter=100, seed=ir.RngSeed(1))
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = ir.solve_device(Dh, cfg, profile=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    p = res.profile
    it = res.trace.iterations
    print(i, f"{(t1-t0)*1e3:.2f} ms", "host", {k: round(v, 2) for k, v in (p.get('host_ms') or {}).items()},
          "gaps", {k: round(v, 3) for k, v in p['gaps_ms'].items()}, "strips", round(float(p['strips_ms'][:it].sum()), 3),
          "chain", round(float(p['svd_ms'][:it].sum()), 3), "ov", p.get("overlapped"), flush=True)
