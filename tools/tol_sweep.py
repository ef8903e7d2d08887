"""Core-SVD tolerance sweep (diagnostics): steps, time and result drift.

    python tools/tol_sweep.py cfg5 1e-6 1e-7 ...          (the floor, IRCUR_SVD_TOL32/64)
    TOL_VAR=SCALE python tools/tol_sweep.py cfg5 1e-8 1e-5  (the e_{k-lag} scale, IRCUR_SVD_TOLSCALE32/64)
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
import paper_2010_07422_b200 as ir
from paper_2010_07422_b200 import gen

name = sys.argv[1]
n1, n2, r, alpha, dts, _ = bench.CONFIGS[name]
tdt = torch.float32 if dts == "f32" else torch.float64
D, linf, _ = gen.baseline_problem_device(n1, n2, r, alpha, bench.DATA_SEED, dtype=tdt)
cfg = ir.SolverConfig(rank=r, eps=bench.EPS, zeta0=linf, gamma=bench.GAMMA, mode="resampled",
                      max_iter=bench.MAX_ITER, seed=ir.RngSeed(bench.SOLVER_SEED))
out = {}
for tol in sys.argv[2:]:
    var = "TOLSCALE" if os.environ.get("TOL_VAR") == "SCALE" else "TOL"
    os.environ[f"IRCUR_SVD_{var}32"] = tol
    os.environ[f"IRCUR_SVD_{var}64"] = tol
    ir.solve_device(D, cfg, profile=True)
    ts = []
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); res = ir.solve_device(D, cfg, profile=True); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    p = res.profile
    Pt, Qt = res.handle.Pt.double(), res.handle.Qt.double()
    # sample of L = P Q on random blocks
    g = torch.Generator(device="cpu").manual_seed(0)
    ri = torch.randint(0, n1, (512,), generator=g).cuda(); ci = torch.randint(0, n2, (512,), generator=g).cuda()
    Lb = (Pt[:, ri].T @ Qt[:, ci]).cpu().numpy()
    out[tol] = (res.trace.iterations, res.trace.errors[-1], Lb)
    print(f"tol={tol}: iters={res.trace.iterations} e_last={res.trace.errors[-1]:.6e} ms={np.median(ts):.2f} "
          f"svd={p['svd_ms'].sum():.2f} steps={int(p['svd_steps'].sum())} per-k={list(p['svd_steps'])}", flush=True)
    ir.clear_cache()
ref = out[sys.argv[2]][2]
for tol, (it, e, Lb) in out.items():
    print(f"tol={tol}: rel L-block diff vs first = {np.linalg.norm(Lb - ref) / np.linalg.norm(ref):.3e}")
