import os, sys, time
sys.path.insert(0, "/root/repo")
import torch, numpy as np
import paper_2010_07422_b200 as ir
from paper_2010_07422_b200 import gen, solver
import cProfile, pstats
probs, cfgs = [], []
for p in range(512):
    D, linf, _ = gen.baseline_problem_device(2000, 2000, 5, 0.2, 1000 + p, dtype=torch.float32)
    probs.append(D); cfgs.append(ir.SolverConfig(rank=5, eps=1e-5, zeta0=linf, gamma=0.7, mode="resampled", max_iter=100, seed=ir.RngSeed(1000 + p)))
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); st = {}
    res = ir.solve_batch_device(probs, cfgs, stats=st, svd_cs=int(os.environ.get("SVDCS", "0")))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"total {1e3*(t1-t0):.1f} ms prepare {1e3*st['prepare_s']:.1f} run {1e3*st['batched_run_s']:.1f}", flush=True)
pr = cProfile.Profile(); pr.enable()
res = ir.solve_batch_device(probs, cfgs, stats={}); torch.cuda.synchronize()
pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
