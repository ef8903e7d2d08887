"""Batched independent problems (ircur_batch_prepare + ircur_batched_run;
BASELINE.json cfg4, the reference's trial pool cli.py:117-125): one launch
per phase per iteration over all problems.

* Each problem's results are bitwise those of its own solve with the same
  SVD cluster size (IRCUR_SVD_CS), whatever else is in the batch;
* against the CPU oracle (tests/parity.py bar) at the cfg4 shape;
* problems that stop early, a den == 0 problem, and fixed mode in a batch.
"""

import numpy as np
import pytest

from oracle import ircur_oracle as orc
import parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ir():
    import paper_2010_07422_b200 as m
    from paper_2010_07422_b200 import _build
    _build.build()
    return m


def _problems(ir, n, count, r=5, alpha=0.2, mode="resampled", seed0=1000, eps=1e-5):
    probs, cfgs = [], []
    for p in range(count):
        D, _, _, linf = orc.baseline_problem(n, n, r, alpha, seed0 + p)
        probs.append(D.astype(np.float32))
        cfgs.append(ir.SolverConfig(rank=r, eps=eps, zeta0=linf, gamma=0.7, mode=mode, max_iter=100,
                                    seed=ir.RngSeed(seed0 + p)))
    return probs, cfgs


@pytest.mark.parametrize("cs", [1, 5])
def test_batched_equals_own_solves(ir, monkeypatch, cs):
    probs, cfgs = _problems(ir, 2000, 6)
    cfgs[2] = ir.SolverConfig(rank=5, eps=1e-3, zeta0=cfgs[2].zeta0, gamma=0.7, mode="resampled", max_iter=100,
                              seed=ir.RngSeed(1002))  # stops early: the batch runs on without it
    bat = ir.solve_batch(probs, cfgs, device=0, svd_cs=cs)
    monkeypatch.setenv("IRCUR_SVD_CS", str(cs))
    ir.clear_cache()
    one = [ir.solve(D, c, device=0, overlap=False) for D, c in zip(probs, cfgs)]
    assert bat[2][2].iterations < bat[0][2].iterations
    for (c1, s1, t1), (c2, s2, t2) in zip(one, bat):
        assert t1.iterations == t2.iterations and t1.converged == t2.converged
        assert t1.errors == t2.errors
        assert t1.thresholds == t2.thresholds and t1.sampled_rows == t2.sampled_rows
        np.testing.assert_array_equal(c1.C, c2.C)
        np.testing.assert_array_equal(c1.R, c2.R)
        np.testing.assert_array_equal(s1.row_values, s2.row_values)
        np.testing.assert_array_equal(c1.core_pinv.sigma, c2.core_pinv.sigma)
    ir.clear_cache()


@pytest.mark.parametrize("mode", ["resampled", "fixed"])
def test_batched_matches_oracle(ir, mode):
    probs, cfgs = _problems(ir, 2000, 4, mode=mode, seed0=1100)
    bat = ir.solve_batch(probs, cfgs, device=0)
    for i, ((cur, sp, tr), D, c) in enumerate(zip(bat, probs, cfgs)):
        kw = dict(rank=c.rank, eps=c.eps, zeta0=c.zeta0, gamma=c.gamma, mode=c.mode, max_iter=c.max_iter)
        ref = orc.solve(D.astype(np.float64), seed=1100 + i, record_x=True, **kw)

        def resolve(mi, e, D=D, kw=kw, i=i):
            return ir.solve_batch([D], [ir.SolverConfig(seed=ir.RngSeed(1100 + i), **{**kw, "max_iter": mi,
                                                                                        "eps": e})], device=0)[0]

        parity.check((cur, sp, tr), ref, True, resolve=resolve, name=f"batched_{mode}_{i}")


def test_batched_zero_slab_problem(ir):
    """A problem whose first sampled slabs are zero takes the den == 0 exit
    (solver.py:335-341) inside a batch; the others run normally."""
    probs, cfgs = _problems(ir, 600, 3, r=3, seed0=1200)
    n1, n2 = probs[1].shape
    m1, m2 = ir.sample_count(n1, 3, 4.0), ir.sample_count(n2, 3, 4.0)
    I0, J0 = ir.draw_index_sets(n1, n2, m1, m2, cfgs[1].seed, 1)[0]
    probs[1] = probs[1].copy()
    probs[1][I0, :] = 0.0
    probs[1][:, J0] = 0.0
    bat = ir.solve_batch(probs, cfgs, device=0)
    assert bat[1][2].errors == [0.0] and bat[1][2].converged and not bat[1][0].C.any()
    for i in (0, 2):
        ref = ir.solve(probs[i], cfgs[i], device=0, overlap=False)
        assert ref[2].iterations == bat[i][2].iterations


def test_batched_nonfinite_problem_raises(ir):
    """A non-finite entry in one problem of a batch raises the reference's
    error (matcore.require_finite, matcore.py:70-77) naming that problem; the
    same contexts then solve a clean batch."""
    probs, cfgs = _problems(ir, 600, 3, r=3, seed0=1300)
    bad = [p.copy() for p in probs]
    bad[2][5, 7] = np.nan
    with pytest.raises(ValueError, match="non-finite") as ei:
        ir.solve_batch(bad, cfgs, device=0)
    assert "problem 2" in str(ei.value)
    bat = ir.solve_batch(probs, cfgs, device=0)
    for i in range(3):
        ref = ir.solve(probs[i], cfgs[i], device=0, overlap=False)
        assert ref[2].iterations == bat[i][2].iterations
        assert ref[2].errors == bat[i][2].errors
