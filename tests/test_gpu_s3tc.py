"""strips3_kernel's tensor-core residual (tcgen05 tf32, kernels_strips3.cu).

The residual pass of the default fp32 strip kernel, r = c - <Res_line,
Fnew(:, x)> (solver.py:262-280, 393-400), runs on the tensor cores for row
strips of at least 32768 positions (cfg5).  IRCUR_S3_TC=2 forces it wherever
it fits, which is how the small cases here reach it; the full-size path is
covered by tests/test_gpu_cfg5_oracle.py.

* against the CPU oracle at the bar of the FFMA kernels (tests/parity.py);
* against the FFMA residual on the same problem: same iterations, same index
  sets, e_k within fp32 round-off of each other (the split is exact, the only
  rounding is the fp32 accumulator's);
* ragged tiles, odd line counts, r = 1 and r = 10, fixed mode;
* a batched problem and a row-sharded solve take the same residual as the
  problem's own solve (bitwise e_k);
* the selection rule: small problems keep the FFMA residual by default.
"""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import ircur_oracle as orc
import parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ir():
    import paper_2010_07422_b200 as m
    from paper_2010_07422_b200 import _build
    _build.build()
    return m


def _counter(res, which) -> int:
    v = C.c_longlong(-1)
    assert res.ctx.lib.ircur_debug_counter(res.ctx.h, which, C.byref(v)) == 0
    return int(v.value)


CASES = [(2000, 2000, 5, 0.2, "resampled"), (1000, 900, 10, 0.2, "resampled"), (600, 5000, 10, 0.2, "fixed"),
         (1500, 1300, 3, 0.1, "resampled"), (333, 4100, 1, 0.1, "resampled"), (10000, 10000, 5, 0.2, "resampled")]


@pytest.mark.parametrize("n1,n2,r,alpha,mode", CASES)
def test_tc_residual_matches_oracle_and_ffma(ir, monkeypatch, n1, n2, r, alpha, mode):
    D = orc.baseline_problem_blocked(n1, n2, r, alpha, 70 + r, dtype=np.float32)[0]
    linf = float(np.abs(D).max()) * 0.5
    kw = dict(rank=r, eps=1e-5, zeta0=linf, gamma=0.7, mode=mode, max_iter=80)
    ref = orc.solve(D.astype(np.float64), seed=5, record_x=True, **kw)
    Dd = torch.from_numpy(D).cuda()

    def resolve(mi, e):
        return ir.solve(Dd, ir.SolverConfig(seed=ir.RngSeed(5), **{**kw, "max_iter": mi, "eps": e}), device=0)

    monkeypatch.setenv("IRCUR_S3_TC", "0")
    ffma = resolve(kw["max_iter"], kw["eps"])
    monkeypatch.setenv("IRCUR_S3_TC", "2")
    res = ir.solve_device(Dd, ir.SolverConfig(seed=ir.RngSeed(5), **kw))
    assert _counter(res, 2) == 3 and _counter(res, 4) == 1  # no silent fallback
    out = resolve(kw["max_iter"], kw["eps"])
    parity.check(out, ref, True, resolve=resolve, name=f"s3tc_{n1}x{n2}_r{r}_{mode}")
    again = resolve(kw["max_iter"], kw["eps"])  # run to run: bitwise
    assert again[2].errors == out[2].errors
    np.testing.assert_array_equal(again[0].C, out[0].C)
    # the two residuals see the same thresholded strips: e_k agrees to fp32 round-off
    assert out[2].iterations == ffma[2].iterations
    assert out[2].sampled_rows == ffma[2].sampled_rows and out[2].thresholds == ffma[2].thresholds
    e_tc, e_ff = np.asarray(out[2].errors), np.asarray(ffma[2].errors)
    # e^2 = |residual|^2 / |D|^2: the two differ by the fp32 round-off of the residual entries (< 3e-7 |D| rms)
    assert np.all(np.abs(e_tc ** 2 - e_ff ** 2) <= 1e-5 * e_ff ** 2 + (3e-7) ** 2)
    ir.clear_cache()


def test_small_problems_keep_the_ffma_residual_by_default(ir, monkeypatch):
    monkeypatch.delenv("IRCUR_S3_TC", raising=False)
    D, _, _, linf = orc.baseline_problem(800, 700, 4, 0.1, 3)
    Dd = torch.from_numpy(D.astype(np.float32)).cuda()
    res = ir.solve_device(Dd, ir.SolverConfig(rank=4, eps=1e-5, zeta0=linf, gamma=0.7, max_iter=30,
                                              seed=ir.RngSeed(2)))
    assert _counter(res, 2) == 3 and _counter(res, 4) == 0
    ir.clear_cache()


def test_wide_row_strip_takes_the_tc_residual_by_default(ir, monkeypatch):
    monkeypatch.delenv("IRCUR_S3_TC", raising=False)
    n1, n2, r = 300, 40000, 3
    D = orc.baseline_problem_blocked(n1, n2, r, 0.1, 9, dtype=np.float32)[0]
    linf = float(np.abs(D).max()) * 0.5
    kw = dict(rank=r, eps=1e-5, zeta0=linf, gamma=0.7, mode="resampled", max_iter=60)
    ref = orc.solve(D.astype(np.float64), seed=4, record_x=True, **kw)
    Dd = torch.from_numpy(D).cuda()

    def resolve(mi, e):
        return ir.solve(Dd, ir.SolverConfig(seed=ir.RngSeed(4), **{**kw, "max_iter": mi, "eps": e}), device=0)

    res = ir.solve_device(Dd, ir.SolverConfig(seed=ir.RngSeed(4), **kw))
    assert _counter(res, 2) == 3 and _counter(res, 4) == 1
    parity.check(resolve(kw["max_iter"], kw["eps"]), ref, True, resolve=resolve, name="s3tc_default_300x40000")
    ir.clear_cache()


def test_batched_takes_the_same_residual(ir, monkeypatch):
    monkeypatch.setenv("IRCUR_S3_TC", "2")
    probs, cfgs = [], []
    for p in range(4):
        D, _, _, linf = orc.baseline_problem(1500, 1500, 5, 0.2, 2000 + p)
        probs.append(D.astype(np.float32))
        cfgs.append(ir.SolverConfig(rank=5, eps=1e-5, zeta0=linf, gamma=0.7, mode="resampled", max_iter=100,
                                    seed=ir.RngSeed(2000 + p)))
    bat = ir.solve_batch(probs, cfgs, device=0, svd_cs=1)
    monkeypatch.setenv("IRCUR_SVD_CS", "1")
    ir.clear_cache()
    one = [ir.solve(D, c, device=0, overlap=False) for D, c in zip(probs, cfgs)]
    for (c1, s1, t1), (c2, s2, t2) in zip(one, bat):
        assert t1.iterations == t2.iterations and t1.converged == t2.converged
        assert t1.errors == t2.errors
        np.testing.assert_array_equal(c1.C, c2.C)
        np.testing.assert_array_equal(c1.R, c2.R)
    ir.clear_cache()


@pytest.mark.parametrize("world", [1, 3])
def test_sharded_takes_the_same_residual(ir, monkeypatch, world):
    from paper_2010_07422_b200.dist import gather_program, run_lockstep, shard_rows, solve_shard_program
    monkeypatch.setenv("IRCUR_S3_TC", "2")
    n1, n2, r = 700, 900, 4
    D = orc.baseline_problem_blocked(n1, n2, r, 0.1, 31, dtype=np.float32)[0]
    linf = float(np.abs(D).max()) * 0.5
    cfg = ir.SolverConfig(rank=r, eps=1e-5, zeta0=linf, gamma=0.7, mode="resampled", max_iter=80, seed=ir.RngSeed(6))
    Dd = torch.from_numpy(D).cuda()
    cur1, sp1, tr1 = ir.solve(Dd, cfg)
    progs = []
    for rank in range(world):
        r0, nl = shard_rows(n1, world, rank)
        progs.append(solve_shard_program(Dd[r0:r0 + nl], cfg, n1=n1, row0=r0))
    res = run_lockstep(progs)
    out = run_lockstep([gather_program(x) for x in res])
    ref = orc.solve(D.astype(np.float64), seed=6, rank=r, eps=1e-5, zeta0=linf, gamma=0.7, mode="resampled",
                    max_iter=80)
    for cur, sp, tr in out:
        assert tr.iterations == tr1.iterations == ref.iterations
        if world == 1:
            assert tr.errors == tr1.errors
            np.testing.assert_array_equal(cur.C, cur1.C)
        else:  # the all-reduced sums round differently from one GPU's: oracle bar
            np.testing.assert_allclose(tr.errors, ref.errors, rtol=2e-3, atol=3e-7)
            assert np.linalg.norm(cur.C - ref.C) <= 1e-4 * np.linalg.norm(ref.C)
    ir.clear_cache()
