"""The tensor-core strip kernels against the CPU oracle: kernels_strips5.cu
(tcgen05, IRCUR_STRIPS_VER=5) and kernels_strips6.cu (warp-level mma.sync,
IRCUR_STRIPS_VER=6).

Same bar as the default fp32 kernels (tests/parity.py): index sets, thresholds
and (within one) iteration counts; e_k; C, R, S strips at 1e-4; support flips
only at fp32 ties.  The kernel that ran is read back (ircur_debug_counter 2),
so a silent fallback to the FFMA kernels fails the test.  Tolerances tighter
than 1e-6 select the FFMA kernel (the 3-term tf32 residual floor, ~4e-7).
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


def _kernel(res) -> int:
    v = C.c_longlong(-1)
    assert res.ctx.lib.ircur_debug_counter(res.ctx.h, 2, C.byref(v)) == 0
    return int(v.value)


CASES = [(2000, 2000, 5, 0.2, "resampled"), (1000, 900, 10, 0.2, "resampled"), (600, 5000, 10, 0.2, "fixed"),
         (1500, 1300, 3, 0.1, "resampled"), (10000, 10000, 5, 0.2, "resampled")]


@pytest.mark.parametrize("ver", [5, 6])
@pytest.mark.parametrize("n1,n2,r,alpha,mode", CASES)
def test_tensor_core_strips_match_oracle(ir, monkeypatch, ver, n1, n2, r, alpha, mode):
    monkeypatch.setenv("IRCUR_STRIPS_VER", str(ver))
    D = orc.baseline_problem_blocked(n1, n2, r, alpha, 70 + r, dtype=np.float32)[0]
    linf = float(np.abs(D).max()) * 0.5
    kw = dict(rank=r, eps=1e-5, zeta0=linf, gamma=0.7, mode=mode, max_iter=80)
    ref = orc.solve(D.astype(np.float64), seed=5, record_x=True, **kw)
    Dd = torch.from_numpy(D).cuda()

    def resolve(mi, e):
        return ir.solve(Dd, ir.SolverConfig(seed=ir.RngSeed(5), **{**kw, "max_iter": mi, "eps": e}), device=0)

    res = ir.solve_device(Dd, ir.SolverConfig(seed=ir.RngSeed(5), **kw))
    assert _kernel(res) == ver
    out = resolve(kw["max_iter"], kw["eps"])
    parity.check(out, ref, True, resolve=resolve, name=f"strips{ver}_{n1}x{n2}_r{r}_{mode}")
    again = resolve(kw["max_iter"], kw["eps"])  # run to run: bitwise
    assert again[2].errors == out[2].errors
    np.testing.assert_array_equal(again[0].C, out[0].C)
    ir.clear_cache()


@pytest.mark.parametrize("ver", [5, 6])
def test_tight_tolerance_takes_the_ffma_kernel(ir, monkeypatch, ver):
    monkeypatch.setenv("IRCUR_STRIPS_VER", str(ver))
    D, _, _, linf = orc.baseline_problem(800, 700, 4, 0.1, 3)
    Dd = torch.from_numpy(D.astype(np.float32)).cuda()
    res = ir.solve_device(Dd, ir.SolverConfig(rank=4, eps=1e-7, zeta0=linf, gamma=0.7, max_iter=30,
                                              seed=ir.RngSeed(2)))
    assert _kernel(res) == 3
    res = ir.solve_device(Dd, ir.SolverConfig(rank=4, eps=1e-5, zeta0=linf, gamma=0.7, max_iter=30,
                                              seed=ir.RngSeed(2)))
    assert _kernel(res) == ver
    ir.clear_cache()
