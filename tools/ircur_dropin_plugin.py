"""pytest plugin: the reference package's own tests with `ircur.solve`
replaced by the B200 drop-in.

    PYTHONPATH=/root/repo/tools:/root/repo IRCUR_REF_SRC=<reference>/pkg/src \\
        python -m pytest -p ircur_dropin_plugin -p no:cacheprovider -c /dev/null \\
        --rootdir=/tmp/dropin <reference>/pkg/tests

Needs a CUDA device and an importable copy of the reference package.  The
reference's test modules bind `from ircur.solver import solve` at import
time, so the patch must happen in a plugin loaded before collection (a
conftest next to the tests cannot be added: the tree is read-only).

The drop-in accepts the reference's own SolverConfig / RngSeed (duck-typed:
same fields, `seed.generator()`), and this adapter converts its results
into the reference's dataclasses so isinstance checks and __post_init__
validation behave as with the original solve.
"""

from __future__ import annotations

import os
import sys

REF = os.environ.get("IRCUR_REF_SRC", "/root/reference/pkg/src")
if REF not in sys.path:
    sys.path.insert(0, REF)

import ircur  # noqa: E402
import ircur.solver as rsolver  # noqa: E402
from ircur.matcore import PinvFactor as RPinvFactor  # noqa: E402
from ircur.sampling import IndexSet as RIndexSet  # noqa: E402

import paper_2010_07422_b200 as b200  # noqa: E402

_reference_solve = rsolver.solve


def _to_reference(cur, sparse, trace=None):
    rows = RIndexSet(cur.rows.indices, cur.rows.bound)
    cols = RIndexSet(cur.cols.indices, cur.cols.bound)
    core = RPinvFactor(W=cur.core_pinv.W, sigma=cur.core_pinv.sigma, V=cur.core_pinv.V,
                       inv_sigma=cur.core_pinv.inv_sigma)
    rc = rsolver.CurFactors(C=cur.C, core_pinv=core, R=cur.R, rows=rows, cols=cols)
    rs = rsolver.SparseEstimate(row_values=sparse.row_values, col_values=sparse.col_values, rows=rows,
                                cols=cols)
    if trace is None:
        return rc, rs
    rt = rsolver.SolverTrace(errors=list(trace.errors), thresholds=list(trace.thresholds),
                             iterations=trace.iterations, converged=trace.converged,
                             seconds=list(trace.seconds), allocated=list(trace.allocated),
                             sampled_rows=list(trace.sampled_rows), sampled_cols=list(trace.sampled_cols))
    return rc, rs, rt


CALLS = {"solve": 0}


def solve(D, config, observer=None):
    """ircur.solver.solve signature, B200 arithmetic."""
    CALLS["solve"] += 1
    obs = None
    if observer is not None:
        def obs(k, zeta, cur, sparse, e):
            rc, rs = _to_reference(cur, sparse)
            observer(k, zeta, rc, rs, e)
    cur, sparse, trace = b200.solve(D, config, obs)
    return _to_reference(cur, sparse, trace)


def pytest_configure(config):
    rsolver.solve = solve
    ircur.solve = solve
    for name, mod in list(sys.modules.items()):
        if name.startswith("ircur") and getattr(mod, "solve", None) is _reference_solve:
            mod.solve = solve


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"drop-in: {CALLS['solve']} ircur.solve calls ran on the B200 library")
