"""The sampled-factor kernel (kernels_sampled.cu) against the strip kernel.

Iteration k + 1's core can be computed from P_k(I_{k+1}, :) and
Q_k(:, J_{k+1}) produced by the sampled-factor kernel instead of gathered
from the strips' full factors.  With IRCUR_SAMPLED_CHECK=1 the sequential
loop runs the sampled kernel after every strip launch and the next core
kernel counts the gathered entries that differ from it: the count must be 0
(bitwise equal), for fp32 with the column-major copy (the strips3_kernel
path the sampled kernel reproduces).
"""

import ctypes as C

import numpy as np
import pytest

from oracle import ircur_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ir():
    import paper_2010_07422_b200 as m
    from paper_2010_07422_b200 import _build
    _build.build()
    return m


def _mismatches(res) -> int:
    v = C.c_longlong(-1)
    assert res.ctx.lib.ircur_debug_counter(res.ctx.h, 0, C.byref(v)) == 0
    return int(v.value)


@pytest.mark.parametrize("r", [2, 5, 10])
@pytest.mark.parametrize("mode", ["resampled", "fixed"])
@pytest.mark.parametrize("colmajor", ["sampled", "full"])
def test_sampled_factors_equal_strip_factors(ir, monkeypatch, r, mode, colmajor):
    monkeypatch.setenv("IRCUR_SAMPLED_CHECK", "1")
    monkeypatch.setenv("IRCUR_OVERLAP", "0")  # the check runs in the sequential loop
    ir.clear_cache()  # the flag is read when a context is created
    try:
        D, L, S, linf = orc.baseline_problem(900, 700, r, 0.1, seed=40 + r)
        cfg = ir.SolverConfig(rank=r, zeta0=linf, gamma=0.7, mode=mode, max_iter=60, seed=ir.RngSeed(3))
        import torch
        res = ir.solve_device(torch.from_numpy(D.astype(np.float32)).cuda(), cfg, colmajor=colmajor)
        assert res.trace.iterations > 3
        assert _mismatches(res) == 0
    finally:
        monkeypatch.delenv("IRCUR_SAMPLED_CHECK")
        monkeypatch.delenv("IRCUR_OVERLAP")
        ir.clear_cache()


def test_check_detects_a_different_summation_order(ir, monkeypatch):
    """Control for the check itself: without the column-major copy the strips
    run on the cluster kernel (a different summation order), whose factors
    differ from the sampled kernel's in the last bits, and the counter sees it."""
    import torch
    monkeypatch.setenv("IRCUR_SAMPLED_CHECK", "1")
    monkeypatch.setenv("IRCUR_OVERLAP", "0")  # the check runs in the sequential loop
    ir.clear_cache()
    try:
        D, L, S, linf = orc.baseline_problem(900, 700, 5, 0.1, seed=45)
        cfg = ir.SolverConfig(rank=5, zeta0=linf, gamma=0.7, mode="resampled", max_iter=60, seed=ir.RngSeed(3))
        res = ir.solve_device(torch.from_numpy(D.astype(np.float32)).cuda(), cfg, colmajor=False)
        assert _mismatches(res) > 0
    finally:
        monkeypatch.delenv("IRCUR_SAMPLED_CHECK")
        monkeypatch.delenv("IRCUR_OVERLAP")
        ir.clear_cache()


def _flag(res, which):
    v = C.c_longlong(-1)
    assert res.ctx.lib.ircur_debug_counter(res.ctx.h, which, C.byref(v)) == 0
    return int(v.value)


@pytest.mark.parametrize("n,r,mode,colmajor", [(1500, r, m, cm) for r in (2, 5, 10) for m in ("resampled", "fixed")
                                               for cm in ("sampled", "full")] + [(10000, 5, "resampled", "sampled")])
def test_overlapped_loop_equals_sequential(ir, monkeypatch, n, r, mode, colmajor):
    """The two-stream loop (SVD of k + 1 next to the strips of k, IRCUR_OVERLAP)
    gives bitwise the sequential loop's results with the same SVD tolerance
    lag (IRCUR_SVD_ERRLAG=2): trace, strips, core.  The 10^4 case has more
    strip tiles than CTAs in both loops, whose strip grids differ (the
    overlapped one leaves the SVD cluster's SMs free): the per-tile den and
    residual sums keep e_k independent of the grid."""
    import torch
    D = orc.baseline_problem_blocked(n, n - 200, r, 0.1, 60 + r)[0] if n > 2000 else None
    if D is None:
        D, L, S, linf = orc.baseline_problem(n, n - 200, r, 0.1, seed=60 + r)
    else:
        linf = float(np.abs(D).max()) * 0.5
    Dd = torch.from_numpy(D.astype(np.float32)).cuda()
    cfg = ir.SolverConfig(rank=r, zeta0=linf, gamma=0.7, mode=mode, max_iter=60, seed=ir.RngSeed(4))
    out = []
    try:
        for env in ({"IRCUR_SVD_ERRLAG": "2", "IRCUR_OVERLAP": "0"}, {"IRCUR_OVERLAP": "1"}):
            for k, v in env.items():
                monkeypatch.setenv(k, v)
            ir.clear_cache()
            res = ir.solve_device(Dd, cfg, colmajor=colmajor)
            assert _flag(res, 1) == int(env["IRCUR_OVERLAP"])
            cur, sp, tr = ir.solve(Dd, cfg, colmajor=colmajor)
            out.append((cur, sp, tr))
            for k in env:
                monkeypatch.delenv(k)
    finally:
        ir.clear_cache()
    (c1, s1, t1), (c2, s2, t2) = out
    assert t1.iterations == t2.iterations and t1.errors == t2.errors and t1.converged == t2.converged
    assert t1.iterations > 3
    np.testing.assert_array_equal(c1.C, c2.C)
    np.testing.assert_array_equal(c1.R, c2.R)
    np.testing.assert_array_equal(s1.row_values, s2.row_values)
    np.testing.assert_array_equal(s1.col_values, s2.col_values)
    np.testing.assert_array_equal(c1.core_pinv.sigma, c2.core_pinv.sigma)


@pytest.mark.parametrize("dtype,colmajor,want", [("f32", "sampled", 1), ("f32", "full", 1),
                                                 ("f32", False, 0), ("f64", "sampled", 0)])
def test_default_loop_selection(ir, monkeypatch, dtype, colmajor, want):
    """With no environment override the overlapped loop runs wherever it is
    eligible (fp32, one GPU, strips3_kernel on every set: needs the column
    copy), and the sequential loop elsewhere; both match the oracle."""
    import torch
    monkeypatch.delenv("IRCUR_OVERLAP", raising=False)
    monkeypatch.delenv("IRCUR_SVD_ERRLAG", raising=False)
    ir.clear_cache()
    D, L, S, linf = orc.baseline_problem(800, 600, 4, 0.1, seed=77)
    Dm = D.astype(np.float32) if dtype == "f32" else D
    cfg = ir.SolverConfig(rank=4, zeta0=linf, gamma=0.7, mode="resampled", max_iter=60, seed=ir.RngSeed(5))
    try:
        res = ir.solve_device(torch.from_numpy(Dm).cuda(), cfg, colmajor=colmajor)
        assert _flag(res, 1) == want
        cur, sp, tr = ir.solve(Dm, cfg, device=0, colmajor=colmajor)
    finally:
        ir.clear_cache()
    ref = orc.solve(np.asarray(Dm, dtype=np.float64), rank=4, zeta0=linf, gamma=0.7, mode="resampled",
                    max_iter=60, seed=5)
    np.testing.assert_array_equal(cur.rows.indices, ref.rows)
    np.testing.assert_array_equal(cur.cols.indices, ref.cols)
    tol = 1e-4 if dtype == "f32" else 1e-9
    assert abs(tr.iterations - ref.iterations) <= (1 if dtype == "f32" else 0)
    if tr.iterations == ref.iterations:
        assert np.linalg.norm(cur.C - ref.C) <= tol * np.linalg.norm(ref.C)
        assert np.linalg.norm(sp.row_values - ref.S_rows) <= tol * max(np.linalg.norm(ref.S_rows), 1.0)


def test_loop_choice_does_not_change_fp32_results(ir):
    """overlap=False (solve_batch's choice) and the default overlapped loop
    give bitwise the same fp32 results: both use the SVD tolerance lag 2."""
    D, L, S, linf = orc.baseline_problem(1200, 1000, 5, 0.2, seed=91)
    Dm = D.astype(np.float32)
    cfg = ir.SolverConfig(rank=5, zeta0=linf, gamma=0.7, mode="resampled", max_iter=60, seed=ir.RngSeed(8))
    out = []
    for ov in (None, False, True):
        res = ir.solve_device(Dm, cfg, device=0, overlap=ov)
        assert _flag(res, 1) == (0 if ov is False else 1)
        out.append(ir.solve(Dm, cfg, device=0, overlap=ov))
    for cur, sp, tr in out[1:]:
        assert tr.errors == out[0][2].errors and tr.iterations == out[0][2].iterations
        np.testing.assert_array_equal(cur.C, out[0][0].C)
        np.testing.assert_array_equal(sp.col_values, out[0][1].col_values)


@pytest.mark.parametrize("mode", ["resampled", "fixed"])
def test_chain0_beside_prep_pass_is_bitwise_neutral(ir, monkeypatch, mode):
    """With zeta0 given, ircur_solve queues iteration 0's core, Gram and SVD
    ahead of the prep pass (which runs beside the SVD cluster).  Results are
    bitwise those of the plain order (IRCUR_PRE_CHAIN0=0); a NaN in D still
    raises, and zeta0 = None (max|D| needed first) takes the plain order."""
    import torch
    D, L, S, linf = orc.baseline_problem(1500, 1300, 6, 0.1, seed=93)
    Dd = torch.from_numpy(D.astype(np.float32)).cuda()
    cfg = ir.SolverConfig(rank=6, zeta0=linf, gamma=0.7, mode=mode, max_iter=60, seed=ir.RngSeed(6))
    out = []
    for knob in ("0", "1"):
        monkeypatch.setenv("IRCUR_PRE_CHAIN0", knob)
        res = ir.solve_device(Dd, cfg)
        assert _flag(res, 1) == 1
        out.append(ir.solve(Dd, cfg))
    (c1, s1, t1), (c2, s2, t2) = out
    assert t1.errors == t2.errors and t1.iterations == t2.iterations and t1.iterations > 3
    np.testing.assert_array_equal(c1.C, c2.C)
    np.testing.assert_array_equal(c1.R, c2.R)
    np.testing.assert_array_equal(s1.row_values, s2.row_values)
    np.testing.assert_array_equal(c1.core_pinv.sigma, c2.core_pinv.sigma)
    Dn = Dd.clone()
    Dn[700, 11] = float("nan")
    with pytest.raises(ValueError):
        ir.solve(Dn, cfg)
    cur, sp, tr = ir.solve(Dd, cfg)  # the context is still usable after the error
    assert tr.errors == t1.errors
    monkeypatch.delenv("IRCUR_PRE_CHAIN0")


@pytest.mark.parametrize("n1,n2,r,max_iter,eps,mode", [
    (300, 260, 16, 30, 1e-5, "resampled"),   # the largest rank the overlapped loop takes
    (80, 700, 3, 1, 1e-5, "resampled"),      # one iteration: no next chain, no pre-launched chain(1) run
    (500, 400, 4, 2, 1e-5, "resampled"),     # chain(1) pre-launched and consumed, then stop
    (600, 600, 5, 40, 0.5, "resampled"),     # converges at once: speculative chains are discarded
    (700, 90, 2, 50, 1e-6, "fixed"),         # tall and thin, fixed sets
    (64, 900, 6, 50, 1e-6, "resampled"),     # wide and short
])
def test_overlapped_edge_cases_equal_sequential(ir, n1, n2, r, max_iter, eps, mode):
    """Edge cases of the two-stream loop and of the chains queued beside the
    prep pass, bitwise against the sequential loop (both use the fp32 SVD
    tolerance lag 2)."""
    import torch
    D, L, S, linf = orc.baseline_problem(n1, n2, r, 0.1, seed=n1 + n2 + r)
    Dd = torch.from_numpy(D.astype(np.float32)).cuda()
    cfg = ir.SolverConfig(rank=r, zeta0=linf, gamma=0.7, eps=eps, mode=mode, max_iter=max_iter,
                          seed=ir.RngSeed(r + max_iter))
    seq = ir.solve(Dd, cfg, overlap=False)
    res = ir.solve_device(Dd, cfg)
    ov_ran = _flag(res, 1)
    ovl = ir.solve(Dd, cfg)
    (c1, s1, t1), (c2, s2, t2) = seq, ovl
    assert t1.errors == t2.errors and t1.iterations == t2.iterations and t1.converged == t2.converged
    np.testing.assert_array_equal(c1.C, c2.C)
    np.testing.assert_array_equal(c1.R, c2.R)
    np.testing.assert_array_equal(s1.row_values, s2.row_values)
    np.testing.assert_array_equal(s1.col_values, s2.col_values)
    np.testing.assert_array_equal(c1.core_pinv.sigma, c2.core_pinv.sigma)
    if r <= 16 and ov_ran == 0:
        pytest.skip("strips3_kernel not selected for this shape: sequential loop both times")


@pytest.mark.parametrize("mode", ["resampled", "fixed"])
def test_observer_after_overlapped_run_equals_fresh_context(ir, mode):
    """An observer solve (ircur_iterate, one iteration per call) on a cached
    context that just ran an overlapped fp32 solve must not inherit its
    state: the overlapped run's run-ahead leaves position maps of the next
    parity set and a different SVD tolerance lag.  The observer
    trajectory must equal the same observer solve on a fresh context, and
    the plain (non-observer) solve."""
    from oracle.ircur_oracle import baseline_problem
    D = baseline_problem(900, 800, 5, 0.2, 21)[0].astype(np.float32)
    kw = dict(rank=5, gamma=0.7, eps=1e-6, mode=mode, max_iter=60)
    seen = []

    def obs(k, zeta, cur, sparse, e):
        seen.append((k, e, cur.C.copy(), cur.R.copy()))

    ir.clear_cache()
    fresh_plain = ir.solve(D, ir.SolverConfig(seed=ir.RngSeed(11), **kw), device=0)
    ir.clear_cache()
    fresh = ir.solve(D, ir.SolverConfig(seed=ir.RngSeed(11), **kw), observer=obs, device=0)
    fresh_seen, seen[:] = list(seen), []
    ir.clear_cache()
    ir.solve(D, ir.SolverConfig(seed=ir.RngSeed(3), **kw), device=0)  # overlapped run first
    again = ir.solve(D, ir.SolverConfig(seed=ir.RngSeed(11), **kw), observer=obs, device=0)
    assert again[2].errors == fresh[2].errors == fresh_plain[2].errors
    assert len(seen) == len(fresh_seen)
    for (k1, e1, C1, R1), (k2, e2, C2, R2) in zip(seen, fresh_seen):
        assert k1 == k2 and e1 == e2
        np.testing.assert_array_equal(C1, C2)
        np.testing.assert_array_equal(R1, R2)
    np.testing.assert_array_equal(again[0].C, fresh_plain[0].C)
    np.testing.assert_array_equal(again[1].row_values, fresh_plain[1].row_values)
    ir.clear_cache()
