"""Pin the CPU oracle (oracle/ircur_oracle.py) to the reference's own outputs.

The fixtures under tests/golden/ were produced by running the unmodified
reference `ircur.solver.solve` (oracle/make_golden.py).  Index sets,
thresholds, iteration counts and convergence flags must agree exactly; the
floating-point outputs may differ only by BLAS association order.
"""

import numpy as np
import pytest

from conftest import golden_names, load_golden, solver_kwargs
from oracle import ircur_oracle as orc

TOL = 1e-10  # relative Frobenius, fp64 vs fp64 with different association


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.mark.parametrize("name", golden_names())
def test_oracle_matches_reference_golden(name):
    D, meta, g = load_golden(name)
    res = orc.solve(D, **solver_kwargs(meta))
    assert res.iterations == meta["iterations"]
    assert res.converged == meta["converged"]
    np.testing.assert_array_equal(res.rows, g["rows"])
    np.testing.assert_array_equal(res.cols, g["cols"])
    assert res.thresholds == list(g["thresholds"])
    assert res.sampled_rows == list(g["sampled_rows"])
    assert res.sampled_cols == list(g["sampled_cols"])
    e_ref = g["errors"]
    e = np.asarray(res.errors)
    assert np.all(np.abs(e - e_ref) <= 1e-9 * np.maximum(np.abs(e_ref), 1e-300) + 1e-15)
    for key, mine in (("C", res.C), ("R", res.R), ("S_rows", res.S_rows),
                      ("S_cols", res.S_cols), ("sigma", res.sigma)):
        assert rel(mine, g[key]) <= TOL, key
    # singular vectors are sign-ambiguous: compare W diag(sigma) V^T
    assert rel((res.W * res.sigma) @ res.V.T, (g["W"] * g["sigma"]) @ g["V"].T) <= TOL
    np.testing.assert_array_equal(res.inv_sigma > 0, g["inv_sigma"] > 0)


def test_sample_count_known_answers():
    # test_sampling.py:11-34
    assert orc.sample_count(1000, 5, 4) == 139
    assert orc.sample_count(10, 5, 0.01) == 5
    assert orc.sample_count(20, 10, 100) == 20


def test_hard_threshold_known_answers():
    # test_solver.py:43-60
    X = np.array([[3.0, -1.0], [0.5, 2.0]])
    np.testing.assert_array_equal(orc.hard_threshold(X, 1.0), [[3.0, 0.0], [0.0, 2.0]])
    X = np.array([[0.0, -2.0], [1e-300, 0.0]])
    np.testing.assert_array_equal(orc.hard_threshold(X, 0.0), X)
    assert orc.hard_threshold(np.array([[1.0]]), 1.0)[0, 0] == 0.0
