"""CUR -> compact SVD on the device (ircur_factors_to_svd) against the
reference algorithm (oracle.cur_to_svd, a restatement of convert.py:21-48)
on the golden fixtures.  W and V are unique up to per-component signs, so
the comparison uses sigma, the reconstructed product and orthonormality."""

import numpy as np
import pytest

from conftest import golden_names, load_golden, solver_kwargs
from oracle import ircur_oracle as orc

pytestmark = pytest.mark.gpu


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def ir():
    import paper_2010_07422_b200 as m
    from paper_2010_07422_b200 import _build
    _build.build()
    return m


CASES = [n for n in golden_names() if not n.startswith(("zero", "tiny", "maxiter1"))]


@pytest.mark.parametrize("name", CASES)
def test_factors_to_svd_matches_reference_algorithm(ir, name):
    D, meta, g = load_golden(name)
    kw = solver_kwargs(meta)
    seed = kw.pop("seed", 0)
    cur, _, _ = ir.solve(D, ir.SolverConfig(seed=ir.RngSeed(seed), **kw), device=0)
    Wr, sr, Vr = orc.cur_to_svd(g["C"], g["W"], g["sigma"], g["V"], g["inv_sigma"], g["R"])
    tol = 1e-4 if D.dtype == np.float32 else 1e-9
    for svd in (ir.factors_to_svd(cur), ir.cur_to_svd(cur.C, cur.core_pinv, cur.R, device=0)):
        assert svd.sigma.size == sr.size
        np.testing.assert_allclose(svd.sigma, sr, rtol=tol, atol=tol * sr[0])
        assert rel((svd.W * svd.sigma) @ svd.V.T, (Wr * sr) @ Vr.T) <= tol
        k = svd.sigma.size
        assert np.abs(svd.W.T @ svd.W - np.eye(k)).max() <= 1e-9
        assert np.abs(svd.V.T @ svd.V - np.eye(k)).max() <= 1e-9
        assert np.all(np.diff(svd.sigma) <= 0)


def test_cur_to_svd_validates_shapes(ir):
    D, meta, g = load_golden("bl_sq120_r3_resampled")
    core = ir.PinvFactor(W=g["W"], sigma=g["sigma"], V=g["V"], inv_sigma=g["inv_sigma"])
    with pytest.raises(ValueError):
        ir.cur_to_svd(g["C"][:, :-1], core, g["R"], device=0)
    with pytest.raises(ValueError):
        ir.cur_to_svd(g["C"], core, g["R"][:-1], device=0)
