"""Where the end-to-end solve(pinned host D) time goes (diagnostics)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2010_07422_b200 as ir
from paper_2010_07422_b200 import gen, solver

n1, n2, r, alpha, dts, _ = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg5"]
D, linf, _ = gen.baseline_problem_device(n1, n2, r, alpha, bench.DATA_SEED, dtype=torch.float32)
cfg = ir.SolverConfig(rank=r, eps=bench.EPS, zeta0=linf, gamma=bench.GAMMA, mode="resampled",
                      max_iter=bench.MAX_ITER, seed=ir.RngSeed(bench.SOLVER_SEED))
Dh = torch.empty(D.shape, dtype=D.dtype, pin_memory=True)
Dh.copy_(D)
del D
torch.cuda.synchronize()
for rep in range(3):
    t = [time.perf_counter()]
    Dd = solver._device_matrix(Dh, None, None); torch.cuda.synchronize(); t.append(time.perf_counter())
    res = ir.solve_device(Dd, cfg, fetch_factors="copy"); torch.cuda.synchronize(); t.append(time.perf_counter())
    cur, sp = solver._host_results(res.ctx, res.trace.iterations - 1, n1, n2, res.handle); t.append(time.perf_counter())
    del Dd, res, cur, sp
    torch.cuda.synchronize(); t.append(time.perf_counter())
    print(f"rep {rep}: h2d {1e3*(t[1]-t[0]):.1f} ms, solve {1e3*(t[2]-t[1]):.1f} ms, results {1e3*(t[3]-t[2]):.1f} ms, "
          f"free {1e3*(t[4]-t[3]):.1f} ms", flush=True)
