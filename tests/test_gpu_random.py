"""GPU parity on a seeded sweep of random problem shapes and settings.

The fixed cases (test_gpu_parity.py, test_gpu_configs.py) pin the golden
fixtures and the BASELINE configurations.  This sweep covers the space
between them against the oracle:
- aspect ratios from 20 x 600 to 600 x 20;
- ranks 1..6, so the SVD block kk = min(r + 2, |I|, |J|) runs through both
  the register-resident small solvers and the shared-memory path;
- fixed and resampled modes, zeta0 given or max|D|;
- several gamma / eps schedules, fp64 and fp32.

fp64 must match to 1e-9 with identical iterations, index sets and convergence;
fp32 to 1e-4 with the iteration count within one (the module docstring of
test_gpu_parity.py).  The cases are seeded, so the sweep is deterministic.
"""

import numpy as np
import pytest

from oracle import ircur_oracle as orc
import parity

pytestmark = pytest.mark.gpu

TOL64, TOL32 = 1e-9, 1e-4


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def ir():
    import paper_2010_07422_b200 as m
    from paper_2010_07422_b200 import _build
    _build.build()
    return m


def _case(i: int):
    rng = np.random.default_rng(7000 + i)
    shapes = [(20, 600), (600, 20), (37, 41), (400, 90), (90, 400), (256, 256), (513, 129), (64, 500)]
    n1, n2 = shapes[i % len(shapes)]
    r = int(rng.integers(1, 7))
    alpha = float(rng.choice([0.0, 0.05, 0.2]))
    f32 = bool(i % 4 == 3)
    mode = "fixed" if i % 3 == 2 else "resampled"
    gamma = float(rng.choice([0.6, 0.7, 0.8]))
    eps = float(rng.choice([1e-5, 1e-7]))
    use_zeta = bool(rng.integers(0, 2))
    return n1, n2, r, alpha, f32, mode, gamma, eps, use_zeta


@pytest.mark.parametrize("i", range(40))
def test_random_problem_matches_oracle(ir, i):
    n1, n2, r, alpha, f32, mode, gamma, eps, use_zeta = _case(i)
    D, L, S, linf = orc.baseline_problem(n1, n2, r, alpha, seed=100 + i)
    zeta0 = linf if use_zeta else None
    kw = dict(rank=r, eps=eps, zeta0=zeta0, gamma=gamma, mode=mode, max_iter=150)
    Dm = D.astype(np.float32) if f32 else D
    ref = orc.solve(np.asarray(Dm, dtype=np.float64), seed=9 + i, record_x=True, **kw)

    def resolve(mi, e):
        return ir.solve(Dm, ir.SolverConfig(seed=ir.RngSeed(9 + i), **{**kw, "max_iter": mi, "eps": e}), device=0)

    out = resolve(kw["max_iter"], eps)
    parity.check(out, ref, f32, resolve=resolve, name=f"random_{i}")
    cur = out[0]
    if not f32:
        np.testing.assert_allclose(cur.core_pinv.sigma, ref.sigma, rtol=TOL64,
                                   atol=1e-12 * max(ref.sigma.max(), 1e-300))
