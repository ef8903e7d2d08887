"""Run solves of a bench config (for ncu captures / per-iteration breakdowns).

    python tools/prof_run.py cfg5 [--colmajor 0|1] [--solves 2] [--detail]
"""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
import paper_2010_07422_b200 as ir
from paper_2010_07422_b200 import gen

ap = argparse.ArgumentParser()
ap.add_argument("config"); ap.add_argument("--colmajor", default="auto")
ap.add_argument("--solves", type=int, default=2); ap.add_argument("--detail", action="store_true")
ap.add_argument("--mode", default="resampled")
a = ap.parse_args()
n1, n2, r, alpha, dts, _ = bench.CONFIGS[a.config]
tdt = torch.float32 if dts == "f32" else torch.float64
if a.config in bench.VIDEO:  # video-like configs: zeta0 = max|D|
    f, h, w = bench.VIDEO[a.config]
    Dv, _, _ = gen.video_problem(frames=f, height=h, width=w, rank=r, seed=bench.DATA_SEED)
    D, linf = torch.from_numpy(np.ascontiguousarray(Dv, dtype=np.float32)).cuda(), None
else:
    D, linf, amp = gen.baseline_problem_device(n1, n2, r, alpha, bench.DATA_SEED, dtype=tdt)
cfg = ir.SolverConfig(rank=r, eps=bench.EPS, zeta0=linf, gamma=bench.GAMMA, mode=a.mode,
                      max_iter=bench.MAX_ITER, seed=ir.RngSeed(bench.SOLVER_SEED))
cm = a.colmajor if a.colmajor == "auto" else a.colmajor == "1"
for i in range(a.solves):
    st = torch.cuda.Event(enable_timing=True); en = torch.cuda.Event(enable_timing=True)
    st.record(); res = ir.solve_device(D, cfg, colmajor=cm, profile=True); en.record(); en.synchronize()
    p = res.profile
    print(f"solve {i}: {st.elapsed_time(en):.2f} ms, iters {res.trace.iterations}, colmajor {res.colmajor}, "
          f"strips {p['strips_ms'].sum():.2f} svd {p['svd_ms'].sum():.2f} core {p['core_ms'].sum():.2f} "
          f"fin {p['finalize_ms'].sum():.2f} ms", flush=True)
    import ctypes as C
    cyc = (C.c_longlong * 32)()
    res.ctx.lib.ircur_get_svd_phase_cycles(res.ctx.h, cyc, 1)
    names = ["product", "reduce", "ritz", "rotate", "nextblk", "gather", "final", "loop"]
    tot = sum(cyc[:8]) or 1
    print("  svd phases (Mcycles, CTA0/thread0): " + " ".join(f"{n}={c/1e6:.2f}({c/tot*100:.0f}%)" for n, c in zip(names, cyc[:8])))
    print(f"  ritz: chol={cyc[8]/1e6:.2f} solves={cyc[9]/1e6:.2f} jacobi={cyc[10]/1e6:.2f} Mcyc, "
          f"eig calls={cyc[14]} sweeps={cyc[13]}; final extraction={cyc[11]/1e6:.2f} Mcyc "
          f"(its jacobi {cyc[12]/1e6:.2f})")
    fn = ["UV", "H2sum", "jacobi", "rotate+norms", "outputs", "QJ", "sync", "W+Wr"]
    print("  final extraction (Mcycles): " + " ".join(f"{n}={c/1e6:.2f}" for n, c in zip(fn, cyc[24:32])))
    sn = ["stage_wait", "pass1", "reduce", "override+write", "pass2", "sync+issue", "lvec+loop"]
    ver = os.environ.get("IRCUR_STRIPS_VER", "5")
    if ver == "6":
        sn = ["wait+barA", "strip+issue", "pass1", "barB", "reduce+barC", "a3+barD", "pass2", "sums"]
    if ver == "5":
        sn = ["fresh+wait_full", "wait_MMA1", "phaseA", "residual(prev)", "issue_loads", "-", "-", "loop"]
    elif ver != "1":
        sn = ["stage(issue+wait)", "pass1", "sync_after_pass1", "reduce+write+sync", "pass2", "final_sync", "loop"]
    nph = 8 if ver in ("5", "6") else 7
    stot = sum(cyc[16:16 + nph]) or 1
    print("  strips phases (Mcycles, CTA0/thread0): " + " ".join(
        f"{n}={c/1e6:.2f}({c/stot*100:.0f}%)" for n, c in zip(sn, [cyc[16 + k] for k in range(nph)])))
    if a.detail and i == a.solves - 1:
        for k in range(res.trace.iterations):
            print(f"  k={k:2d} e={res.trace.errors[k]:.3e} svd_steps={p['svd_steps'][k]:3d} svd={p['svd_ms'][k]:.3f} "
                  f"strips={p['strips_ms'][k]:.3f} core={p['core_ms'][k]:.3f} ms")
