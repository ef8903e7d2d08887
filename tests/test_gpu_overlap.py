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
        ir.clear_cache()


def test_check_detects_a_different_summation_order(ir, monkeypatch):
    """Control for the check itself: without the column-major copy the strips
    run on the cluster kernel (a different summation order), whose factors
    differ from the sampled kernel's in the last bits, and the counter sees it."""
    import torch
    monkeypatch.setenv("IRCUR_SAMPLED_CHECK", "1")
    ir.clear_cache()
    try:
        D, L, S, linf = orc.baseline_problem(900, 700, 5, 0.1, seed=45)
        cfg = ir.SolverConfig(rank=5, zeta0=linf, gamma=0.7, mode="resampled", max_iter=60, seed=ir.RngSeed(3))
        res = ir.solve_device(torch.from_numpy(D.astype(np.float32)).cuda(), cfg, colmajor=False)
        assert _mismatches(res) > 0
    finally:
        monkeypatch.delenv("IRCUR_SAMPLED_CHECK")
        ir.clear_cache()
