"""Same-process A/B of the sequential and the overlapped loop (IRCUR_OVERLAP)
for one bench config: per-solve time (CUDA events around solve_device, as
bench.py), the device marks before the loop and the loop span."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2010_07422_b200 as ir
from paper_2010_07422_b200 import gen

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
n1, n2, r, al, dts, _ = bench.CONFIGS[name]
D, linf, _ = gen.baseline_problem_device(n1, n2, r, al, bench.DATA_SEED, dtype=torch.float32)
cfg = ir.SolverConfig(rank=r, eps=bench.EPS, zeta0=linf, gamma=bench.GAMMA, mode="resampled",
                      max_iter=bench.MAX_ITER, seed=ir.RngSeed(bench.SOLVER_SEED))
st = torch.cuda.current_stream()
for rnd in range(2):
    for ov in ("0", "1"):
        os.environ["IRCUR_OVERLAP"] = ov
        ir.clear_cache()
        for _ in range(3):
            res = ir.solve_device(D, cfg, profile="deferred")
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        ev[0].record(st)
        for i in range(reps):
            res = ir.solve_device(D, cfg, profile="deferred")
            ev[i + 1].record(st)
        torch.cuda.synchronize()
        ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(reps)]
        marks = np.full(5, -1.0, dtype=np.float32)
        res.ctx.lib.ircur_get_marks(res.ctx.h, marks.ctypes.data_as(C.POINTER(C.c_float)))
        it = res.trace.iterations
        p = res.read_profile()
        line = (f"overlap={ov} iters={it} solve_ms={np.round(ms, 3).tolist()} marks={np.round(marks, 3).tolist()} "
                f"strips={np.sum(p['strips_ms'][:it]):.3f} svd={np.sum(p['svd_ms'][:it]):.3f}")
        if ov == "1":
            tl = np.zeros(4 * it, dtype=np.float32)
            res.ctx.lib.ircur_get_timeline(res.ctx.h, it, tl.ctypes.data_as(C.POINTER(C.c_float)))
            line += f" loop_span={tl.reshape(it, 4)[-1, 3]:.3f}"
        print(line, flush=True)
