"""Generate tests/golden/*.npz by running the REAL reference package.

TEST INFRASTRUCTURE.  Run in the build container, where the read-only
reference is importable:

    python oracle/make_golden.py          # writes tests/golden/

Each fixture stores the solver inputs (D itself for small cases, or the
generator arguments for the 1000x1000 BASELINE cfg1 case), the
SolverConfig fields, and everything `ircur.solver.solve` returned
(solver.py:304-416): C, R, S strips, the core pinv factor, the final index
sets and the full trace.  Nothing here is imported at run time by the
product or by the GPU tests' product path.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")
sys.path.insert(0, HERE)

from ircur_oracle import baseline_problem  # noqa: E402


def _ref():
    sys.path.insert(0, REF_SRC)
    import ircur  # noqa: F401
    from ircur.solver import SolverConfig, solve
    from ircur.sampling import RngSeed
    from ircur.synth import SyntheticSpec, gen_low_rank, make_problem
    return SolverConfig, solve, RngSeed, SyntheticSpec, gen_low_rank, make_problem


def run_case(name, D, cfg_kw, store_D=True, gen=None):
    SolverConfig, solve, RngSeed, *_ = _ref()
    seed = cfg_kw.pop("seed", 0)
    cfg = SolverConfig(seed=RngSeed(seed), **cfg_kw)
    cur, sp, tr = solve(D, cfg)
    meta = dict(cfg_kw, seed=seed, shape=list(D.shape), dtype=str(D.dtype),
                iterations=tr.iterations, converged=tr.converged, gen=gen)
    arrs = dict(
        C=cur.C, R=cur.R, S_rows=sp.row_values, S_cols=sp.col_values,
        W=cur.core_pinv.W, sigma=cur.core_pinv.sigma, V=cur.core_pinv.V,
        inv_sigma=cur.core_pinv.inv_sigma,
        rows=cur.rows.indices, cols=cur.cols.indices,
        errors=np.asarray(tr.errors, dtype=np.float64),
        thresholds=np.asarray(tr.thresholds, dtype=np.float64),
        sampled_rows=np.asarray(tr.sampled_rows, dtype=np.int64),
        sampled_cols=np.asarray(tr.sampled_cols, dtype=np.int64),
        meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8),
    )
    if store_D:
        arrs["D"] = D
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **arrs)
    print(f"{name}: {D.shape} iters={tr.iterations} conv={tr.converged} "
          f"e={tr.errors[-1]:.3e} -> {os.path.getsize(path)} B")


def main():
    os.makedirs(OUT, exist_ok=True)
    SolverConfig, solve, RngSeed, SyntheticSpec, gen_low_rank, make_problem = _ref()

    # BASELINE-generator problems (Gaussian factors, Bernoulli support,
    # +-10 mean|L| outliers), zeta0 = max|L|, gamma = 0.7.
    for name, n1, n2, r, alpha, mode, seed in [
        ("bl_sq120_r3_resampled", 120, 120, 3, 0.1, "resampled", 11),
        ("bl_sq120_r3_fixed", 120, 120, 3, 0.1, "fixed", 11),
        ("bl_rect90x60_r2_resampled", 90, 60, 2, 0.1, "resampled", 12),
        ("bl_rect50x140_r3_fixed", 50, 140, 3, 0.15, "fixed", 13),
        ("bl_sq200_r5_resampled", 200, 200, 5, 0.2, "resampled", 14),
    ]:
        D, L, S, linf = baseline_problem(n1, n2, r, alpha, seed)
        run_case(name, D, dict(rank=r, zeta0=linf, gamma=0.7, mode=mode,
                               max_iter=100, seed=seed + 100))
    # fp32 input (reference upcasts to fp64, matcore.py:70-77)
    D, L, S, linf = baseline_problem(150, 150, 4, 0.2, 15)
    run_case("bl_sq150_r4_f32_resampled", D.astype(np.float32),
             dict(rank=4, zeta0=linf, gamma=0.7, mode="resampled", max_iter=100,
                  seed=115))
    # BASELINE cfg1 at its own size: D regenerated from the generator args.
    D, L, S, linf = baseline_problem(1000, 1000, 5, 0.1, 0)
    run_case("cfg1_n1000_r5_resampled", D,
             dict(rank=5, zeta0=linf, gamma=0.7, mode="resampled", max_iter=100, seed=1),
             store_D=False, gen=dict(n1=1000, n2=1000, rank=5, alpha=0.1, seed=0))

    # Reference-suite style edge cases (test_solver.py:286-433).
    run_case("zero_9x7", np.zeros((9, 7)), dict(rank=2, seed=0))
    run_case("tiny_1x1", np.array([[2.5]]), dict(rank=1, seed=92))
    rng = np.random.default_rng(7)
    small = np.outer(rng.standard_normal(3), rng.standard_normal(3))
    run_case("tiny_3x3_rank5", small, dict(rank=5, seed=93))
    L = gen_low_rank(60, 2, RngSeed(94))
    run_case("overrank_60_r5", L, dict(rank=5, seed=95))
    L = gen_low_rank(40, 3, RngSeed(90), n_cols=25)
    run_case("rect_40x25_exact", L, dict(rank=3, seed=91))
    inst = make_problem(SyntheticSpec(60, 3, 0.2, RngSeed(33)))
    run_case("maxiter1_60", inst.D, dict(rank=3, max_iter=1, seed=34))
    inst = make_problem(SyntheticSpec(100, 4, 0.1, RngSeed(50)))
    run_case("refgen_100_fixed", inst.D,
             dict(rank=4, zeta0=2.0 * float(np.abs(inst.L).max()), mode="fixed", seed=51))
    run_case("refgen_100_resampled", inst.D,
             dict(rank=4, zeta0=2.0 * float(np.abs(inst.L).max()), mode="resampled", seed=51))
    inst = make_problem(SyntheticSpec(300, 5, 0.1, RngSeed(30)))
    run_case("refgen_300_zeta_none", inst.D, dict(rank=5, gamma=0.65, seed=31))


if __name__ == "__main__":
    main()
