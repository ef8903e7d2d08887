"""Parity checks shared by the `-m gpu` suites (test infrastructure).

`check(out, ref, f32, resolve=...)` applies the north_star bar
(BASELINE.json) to one B200 solve against the CPU oracle
(`oracle/ircur_oracle.py`, pinned to the real reference's golden vectors):

* index sets and thresholds identical; iteration count identical (fp64) or
  within one (fp32);
* e_k within ERR_RTOL64 / ERR_RTOL32 relative (+ ERR_ATOL32 absolute for
  fp32 round-off) over the shared iterations;
* C, R, S_rows, S_cols within 1e-9 (fp64) / 1e-4 (fp32) relative Frobenius;
* outlier-support decisions (the S masks, solver.py:153-168): a "flip" is an
  entry kept by one side and zeroed by the other.  fp64 may flip only inside
  the tie band | |x| - zeta_k | <= 1e-12 zeta_k of the oracle's
  pre-threshold value x = d - l; fp32 flips are counted and must lie within
  FLIP_BAND32 of the threshold relative to the operands (|d| + |l|), i.e.
  be fp32 rounding ties, not wrong decisions.

fp32 runs whose iteration count differs by one from the oracle's are NOT
skipped: `resolve(max_iter, eps)` re-runs the B200 solve pinned to the
oracle's count (max_iter = ref.iterations, eps = 1e-300, so the loop stops
exactly there) and the strips of that same iteration are compared.

Every check appends a record to STATS; conftest writes them to
gpurun_out/parity_stats.json at session end (flip counts, worst relative
errors), which is how the fp32 flip counts are reported.
"""

from __future__ import annotations

import numpy as np

TOL64, TOL32 = 1e-9, 1e-4
ERR_RTOL64 = 1e-9
ERR_RTOL32 = 2e-4
# fp32: e_k also carries the round-off of the residual itself.  Each residual
# entry c - l is a difference of values ~|d|; with the tensor-core strips
# (3-term tf32 products, ~3 * 2^-22 relative each) e cannot be resolved below
# ~3 * 2^-22 (||D(I,:)|| + ||D(:,J)||) / den ~ 4e-7 (the FFMA kernel's floor
# is ~2^-24 of it); allow 1e-6 absolute.
ERR_ATOL32 = 1e-6
TIE_BAND64 = 1e-12
FLIP_BAND32 = 1e-5

STATS: list = []


def rel(a, b) -> float:
    a = np.asarray(a)
    b = np.asarray(b)
    nb = float(np.linalg.norm(b))
    return float(np.linalg.norm(a - b)) / (nb if nb > 0 else 1.0)


def flip_stats(S_mine, S_ref, X_ref, D_ref, zeta):
    """(flips, worst distance to the threshold relative to zeta, worst
    distance relative to the operands |d| + |l|) over the flipped entries.
    X_ref = d - l is the oracle's pre-threshold strip, D_ref the data strip
    (R + S_rows or C + S_cols: Phase II is c = d - s)."""
    S_mine = np.asarray(S_mine)
    S_ref = np.asarray(S_ref)
    m = (S_mine != 0) != (S_ref != 0)
    n = int(np.count_nonzero(m))
    if n == 0 or X_ref is None:
        return n, 0.0, 0.0
    x = np.asarray(X_ref)[m]
    d = np.asarray(D_ref)[m]
    gap = np.abs(np.abs(x) - zeta)
    scale = np.abs(d) + np.abs(d - x)  # |d| + |l|
    return n, float(gap.max() / zeta), float((gap / np.maximum(scale, 1e-300)).max())


def check(out, ref, f32: bool, *, name: str = "", resolve=None, sigma=True, x_ref=True):
    """Compare out = (CurFactors, SparseEstimate, SolverTrace) with an
    OracleResult (or an object with the same fields).  All measurements are
    recorded in STATS before any assertion fires."""
    cur, sp, tr = out
    rec = {"case": name, "dtype": "f32" if f32 else "f64", "iters": tr.iterations,
           "ref_iters": ref.iterations, "converged": tr.converged, "ref_converged": ref.converged}
    STATS.append(rec)
    n = min(tr.iterations, ref.iterations)
    e, re = np.asarray(tr.errors[:n]), np.asarray(ref.errors[:n])
    dev = np.abs(e - re) / np.maximum(np.abs(re), 1e-300)
    rec["err_max_rel"] = float(dev.max()) if n else 0.0
    same_thr = list(tr.thresholds[:n]) == list(ref.thresholds[:n])
    same_sizes = (list(tr.sampled_rows[:n]) == list(ref.sampled_rows[:n])
                  and list(tr.sampled_cols[:n]) == list(ref.sampled_cols[:n]))
    first = (cur, sp, tr)
    if tr.iterations != ref.iterations and resolve is not None and ref.iterations > 0:
        cur, sp, tr = resolve(ref.iterations, 1e-300)
        rec["aligned_rerun"] = True
    aligned = tr.iterations == ref.iterations
    tol = TOL32 if f32 else TOL64
    if aligned and ref.iterations > 0:
        for key, a, b in (("C", cur.C, ref.C), ("R", cur.R, ref.R),
                          ("S_rows", sp.row_values, ref.S_rows), ("S_cols", sp.col_values, ref.S_cols)):
            rec["rel_" + key] = rel(a, b)
        zeta = ref.thresholds[ref.iterations - 1]
        X_rows = getattr(ref, "X_rows", None) if x_ref else None
        X_cols = getattr(ref, "X_cols", None) if x_ref else None
        fr = flip_stats(sp.row_values, ref.S_rows, X_rows, np.asarray(ref.R) + np.asarray(ref.S_rows), zeta)
        fc = flip_stats(sp.col_values, ref.S_cols, X_cols, np.asarray(ref.C) + np.asarray(ref.S_cols), zeta)
        rec["flips"] = fr[0] + fc[0]
        rec["support"] = int(np.count_nonzero(ref.S_rows) + np.count_nonzero(ref.S_cols))
        rec["flip_gap_over_zeta"] = max(fr[1], fc[1])
        rec["flip_gap_over_operand"] = max(fr[2], fc[2])
        if sigma:
            rec["rel_sigma"] = rel(cur.core_pinv.sigma, ref.sigma)
    # ---- assertions
    assert same_thr, "thresholds differ"
    assert same_sizes, "per-iteration |I_k| / |J_k| differ"
    if f32:
        c, s2, t = first
        assert abs(t.iterations - ref.iterations) <= 1, rec
        assert t.converged == ref.converged or t.iterations != ref.iterations, rec
    else:
        assert first[2].iterations == ref.iterations and first[2].converged == ref.converged, rec
    np.testing.assert_allclose(e, re, rtol=ERR_RTOL32 if f32 else ERR_RTOL64, atol=ERR_ATOL32 if f32 else 1e-15)
    assert aligned, ("no way to compare the strips at the oracle's iteration", rec)
    np.testing.assert_array_equal(cur.rows.indices, ref.rows)
    np.testing.assert_array_equal(cur.cols.indices, ref.cols)
    if ref.iterations == 0:
        return rec
    for key in ("C", "R", "S_rows", "S_cols"):
        assert rec["rel_" + key] <= tol, (key, rec)
    if sigma:
        assert rec["rel_sigma"] <= tol, rec
    if f32:
        assert rec["flip_gap_over_operand"] <= FLIP_BAND32, rec
    elif x_ref and getattr(ref, "X_rows", None) is not None:
        assert rec["flip_gap_over_zeta"] <= TIE_BAND64, rec
    else:
        assert rec["flips"] == 0, rec
    return rec
