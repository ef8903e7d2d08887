"""Diagnostics run on the GPU box: per-fixture parity numbers (no asserts)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from conftest import golden_names, load_golden, solver_kwargs
import paper_2010_07422_b200 as ir
from oracle import ircur_oracle as orc

def rel(a, b):
    nb = np.linalg.norm(b); return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)

for name in golden_names():
    D, meta, g = load_golden(name)
    kw = solver_kwargs(meta); seed = kw.pop("seed", 0)
    cfg = ir.SolverConfig(seed=ir.RngSeed(seed), **kw)
    try:
        t = time.time(); cur, sp, tr = ir.solve(D, cfg, device=0); dt = time.time() - t
    except Exception as e:
        print(f"{name}: EXC {type(e).__name__}: {e}"); continue
    n = min(tr.iterations, meta["iterations"])
    e = np.asarray(tr.errors[:n]); re = g["errors"][:n]
    erel = np.max(np.abs(e - re) / np.maximum(np.abs(re), 1e-300)) if n else 0
    out = f"{name}: it {tr.iterations}/{meta['iterations']} conv {tr.converged}/{meta['converged']} erel {erel:.2e} t={dt*1e3:.1f}ms"
    if tr.iterations == meta["iterations"] and meta["iterations"] > 0:
        out += " C %.1e R %.1e Sr %.1e Sc %.1e sig %.1e" % (rel(cur.C, g["C"]), rel(cur.R, g["R"]),
            rel(sp.row_values, g["S_rows"]), rel(sp.col_values, g["S_cols"]), rel(cur.core_pinv.sigma, g["sigma"]))
    print(out, flush=True)
