"""GPU parity: the B200 solve (through the C-ABI) vs the reference's golden
vectors and the CPU oracle, on the same seeded inputs.

fp64 inputs run fp64 kernels and must match to 1e-9 (relative Frobenius for
C, R, S strips and W Sigma V^T; relative for e_k), with identical index
sets, thresholds, iteration counts and convergence flags — the tolerance
BASELINE.json's north_star states.  fp32 inputs run fp32 strip kernels
against the reference's fp64 arithmetic on the same fp32 values: 1e-4
relative Frobenius on L/S (north_star), iteration count within one.
"""

import numpy as np
import pytest
import torch

from conftest import golden_names, load_golden, solver_kwargs
import parity

pytestmark = pytest.mark.gpu

TOL64 = 1e-9
TOL32 = 1e-4


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def ir():
    import paper_2010_07422_b200 as m
    from paper_2010_07422_b200 import _build
    _build.build()
    return m


def _cfg(ir, meta):
    kw = solver_kwargs(meta)
    seed = kw.pop("seed", 0)
    return ir.SolverConfig(seed=ir.RngSeed(seed), **kw)


@pytest.mark.parametrize("name", golden_names())
def test_solve_matches_reference_golden(ir, name):
    """Against the real reference's vectors, and (for the support-flip and
    aligned-iteration checks of tests/parity.py) against the oracle pinned
    to them.  An fp32 run that stops one iteration away from the reference
    is re-run pinned to the reference's count, never skipped."""
    from oracle import ircur_oracle as orc
    D, meta, g = load_golden(name)
    cfg = _cfg(ir, meta)
    f32 = D.dtype == np.float32
    tol = TOL32 if f32 else TOL64

    def resolve(mi, e):
        kw = solver_kwargs(meta)
        seed = kw.pop("seed", 0)
        kw.update(max_iter=mi, eps=e)
        return ir.solve(D, ir.SolverConfig(seed=ir.RngSeed(seed), **kw), device=0)

    out = ir.solve(D, cfg, device=0)
    cur, sparse, trace = out
    if not f32:
        assert trace.iterations == meta["iterations"]
        assert trace.converged == meta["converged"]
        np.testing.assert_array_equal(cur.rows.indices, g["rows"])
        np.testing.assert_array_equal(cur.cols.indices, g["cols"])
        assert trace.thresholds == list(g["thresholds"])
        e = np.asarray(trace.errors)
        ref_e = g["errors"]
        assert np.all(np.abs(e - ref_e) <= TOL64 * np.abs(ref_e) + 1e-14), (e, ref_e)
    if meta["iterations"] == 0:
        assert trace.errors == [0.0]
        return
    kw = solver_kwargs(meta)
    ref = orc.solve(np.asarray(D, dtype=np.float64), record_x=True, **kw)
    parity.check(out, ref, f32, resolve=resolve, name="golden_" + name)
    if trace.iterations != meta["iterations"]:
        cur, sparse, trace = resolve(meta["iterations"], 1e-300)
    for key, mine in (("C", cur.C), ("R", cur.R), ("S_rows", sparse.row_values),
                      ("S_cols", sparse.col_values)):
        assert rel(mine, g[key]) <= tol, (key, rel(mine, g[key]))
    assert rel(cur.core_pinv.sigma, g["sigma"]) <= tol
    mine_core = (cur.core_pinv.W * cur.core_pinv.sigma) @ cur.core_pinv.V.T
    ref_core = (g["W"] * g["sigma"]) @ g["V"].T
    assert rel(mine_core, ref_core) <= tol
    np.testing.assert_array_equal(cur.core_pinv.inv_sigma > 0, g["inv_sigma"] > 0)


def test_intersection_blocks_agree_bitwise(ir):
    # SparseEstimate invariant (solver.py:117-129; test_solver.py:169-177)
    D, meta, g = load_golden("bl_sq200_r5_resampled")
    seen = []

    def obs(k, zeta, cur, sparse, e):
        a = sparse.row_values[:, sparse.cols.indices]
        b = sparse.col_values[sparse.rows.indices, :]
        seen.append(np.array_equal(a, b) and np.array_equal(cur.R[:, cur.cols.indices],
                                                            cur.C[cur.rows.indices, :]))

    cfg = _cfg(ir, meta)
    _, _, trace = ir.solve(D, cfg, observer=obs, device=0)
    assert seen and all(seen)
    assert trace.iterations == meta["iterations"]


@pytest.mark.parametrize("mode", ["fixed", "resampled"])
def test_bitwise_run_to_run_determinism(ir, mode):
    from oracle.ircur_oracle import baseline_problem
    D = baseline_problem(180, 170, 4, 0.15, 3)[0]
    cfg = ir.SolverConfig(rank=4, gamma=0.7, mode=mode, seed=ir.RngSeed(4))
    a = ir.solve(D, cfg, device=0)
    b = ir.solve(D, cfg, device=0)
    assert a[2].errors == b[2].errors
    np.testing.assert_array_equal(a[0].C, b[0].C)
    np.testing.assert_array_equal(a[0].R, b[0].R)
    np.testing.assert_array_equal(a[1].row_values, b[1].row_values)
    np.testing.assert_array_equal(a[1].col_values, b[1].col_values)


def test_nonfinite_rejected(ir):
    D = np.ones((40, 30))
    D[3, 4] = np.nan
    with pytest.raises(ValueError):
        ir.solve(D, ir.SolverConfig(rank=2), device=0)
    D[3, 4] = np.inf
    with pytest.raises(ValueError):
        ir.solve(D.astype(np.float32), ir.SolverConfig(rank=2), device=0)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("mode", ["resampled", "fixed"])
def test_colmajor_copy_and_strided_paths_agree(ir, dtype, mode):
    """Full copy, sampled copy (incl. on-demand extension past the covered
    sets) and the strided gather from row-major D give identical bits."""
    from oracle.ircur_oracle import baseline_problem
    D = baseline_problem(150, 130, 3, 0.1, 8)[0].astype(dtype)
    cfg = ir.SolverConfig(rank=3, gamma=0.7, eps=1e-9, mode=mode, seed=ir.RngSeed(9))
    ref = ir.solve(D, cfg, device=0, colmajor="full")
    assert ref[2].iterations > 6
    for cm in (False, "sampled", "sampled:1", "sampled:3"):
        b = ir.solve(D, cfg, device=0, colmajor=cm)
        assert b[2].errors == ref[2].errors, cm
        for x, y in ((b[0].C, ref[0].C), (b[0].R, ref[0].R), (b[1].col_values, ref[1].col_values)):
            np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("overlap", [True, False])
def test_sampled_copy_extensions_agree(ir, overlap):
    """A sampled copy that covers fewer sets than the loop runs is extended on
    the way: by gathering the new columns from the row-major D into the copy's
    free lines (extend_cover), or by a full prep pass when those run out.  Both
    happen here (6 -> 10 sets does not fit the first allocation, 10 -> 14 does);
    the results are those of the full copy, bit for bit, on either loop."""
    from oracle.ircur_oracle import baseline_problem_blocked
    D = baseline_problem_blocked(3000, 2500, 5, 0.2, 75, dtype=np.float32)[0]
    linf = float(np.abs(D).max()) * 0.5
    cfg = ir.SolverConfig(rank=5, gamma=0.7, eps=1e-5, zeta0=linf, mode="resampled", max_iter=80, seed=ir.RngSeed(5))
    ref = ir.solve(D, cfg, device=0, colmajor="full", overlap=overlap)
    assert ref[2].iterations > 16 and ref[2].converged
    for cm in ("sampled:6", "sampled:15", "sampled"):
        b = ir.solve(D, cfg, device=0, colmajor=cm, overlap=overlap)
        assert b[2].iterations == ref[2].iterations and b[2].errors == ref[2].errors, cm
        for x, y in ((b[0].C, ref[0].C), (b[0].R, ref[0].R), (b[1].col_values, ref[1].col_values)):
            np.testing.assert_array_equal(x, y)
    ir.clear_cache()


def test_materialize_matches_oracle(ir):
    from oracle import ircur_oracle as orc
    D, meta, g = load_golden("bl_sq120_r3_resampled")
    cur, _, _ = ir.solve(D, _cfg(ir, meta), device=0)
    L_ref = orc.materialize(g["C"], g["V"], g["inv_sigma"], g["W"], g["R"])
    assert rel(ir.materialize(cur), L_ref) <= TOL64


@pytest.mark.parametrize("decay", [0.9, 0.99, 1.0])
@pytest.mark.parametrize("mode", ["resampled", "fixed"])
def test_no_spectral_gap_matches_oracle(ir, decay, mode):
    """Cores whose singular values have no gap at r (rank-8 data, r = 4,
    geometric decay or exactly equal): the block subspace SVD must still
    reproduce LAPACK's top-r triplets through the whole trace."""
    from oracle import ircur_oracle as orc
    rng = np.random.default_rng(17)
    n1, n2, k = 260, 230, 8
    A = np.linalg.qr(rng.standard_normal((n1, k)))[0]
    B = np.linalg.qr(rng.standard_normal((n2, k)))[0]
    s = 50.0 * decay ** np.arange(k)
    D = (A * s) @ B.T
    mask = rng.random((n1, n2)) < 0.05
    D = D + np.where(mask, rng.uniform(-5, 5, (n1, n2)), 0.0)
    zeta0 = float(np.abs((A * s) @ B.T).max())
    kw = dict(rank=4, eps=1e-12, zeta0=zeta0, gamma=0.7, mode=mode, max_iter=12, seed=3)
    ref = orc.solve(D, **kw)
    cfg = ir.SolverConfig(rank=4, eps=1e-12, zeta0=zeta0, gamma=0.7, mode=mode, max_iter=12,
                          seed=ir.RngSeed(3))
    cur, sp, tr = ir.solve(D, cfg, device=0)
    assert tr.iterations == ref.iterations
    np.testing.assert_allclose(tr.errors, ref.errors, rtol=1e-8)
    np.testing.assert_allclose(cur.core_pinv.sigma, ref.sigma, rtol=1e-9)
    assert rel(cur.C, ref.C) <= TOL64 and rel(cur.R, ref.R) <= TOL64
    assert rel(sp.row_values, ref.S_rows) <= TOL64


@pytest.mark.parametrize("colmajor", ["sampled", "full", False])
def test_zero_slabs_early_exit(ir, colmajor):
    """solver.py:335-341: when D(I_0,:) and D(:,J_0) are identically zero the
    solve returns the zero state, even if D is nonzero elsewhere.  The
    sampled prep pass computes these norms itself; every copy mode must
    agree with the reference's oracle."""
    from oracle import ircur_oracle as orc
    n1, n2, r = 300, 280, 3
    cfg = ir.SolverConfig(rank=r, zeta0=1.0, mode="resampled", max_iter=20, seed=ir.RngSeed(4))
    m1, m2 = ir.sample_count(n1, r, 4.0), ir.sample_count(n2, r, 4.0)
    I0, J0 = ir.draw_index_sets(n1, n2, m1, m2, cfg.seed, 1)[0]
    D = np.random.default_rng(0).standard_normal((n1, n2))
    D[I0, :] = 0.0
    D[:, J0] = 0.0
    ref = orc.solve(D, rank=r, zeta0=1.0, mode="resampled", max_iter=20, seed=4)
    cur, sp, tr = ir.solve(D, cfg, device=0, colmajor=colmajor)
    assert ref.iterations == 0 or ref.errors == [0.0]
    assert tr.errors == [0.0] and tr.converged and not cur.C.any()
    D[I0[0], 5] = 1e-30  # one tiny nonzero entry in the row slab: no early exit
    ref = orc.solve(D, rank=r, zeta0=1.0, mode="resampled", max_iter=20, seed=4)
    cur, sp, tr = ir.solve(D, cfg, device=0, colmajor=colmajor)
    assert tr.iterations == ref.iterations == 1 and tr.thresholds == [1.0]
    assert tr.errors == ref.errors


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
@pytest.mark.parametrize("colmajor", ["sampled", "full", False])
def test_nonfinite_rejected_in_full_tiles(ir, bad, colmajor):
    """NaN/Inf inside a full 64 x 64 prep tile (the vectorised scan paths)."""
    D = np.random.default_rng(1).standard_normal((256, 320)).astype(np.float32)
    D[130, 200] = bad
    with pytest.raises(ValueError, match="non-finite"):
        ir.solve(D, ir.SolverConfig(rank=2, zeta0=1.0), device=0, colmajor=colmajor)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("colmajor", ["sampled", "full", False])
def test_zeta0_none_uses_exact_max_abs(ir, dtype, colmajor):
    """zeta0=None takes max|D| (solver.py:342-344) from the prep pass: the
    first threshold must equal numpy's max|D| exactly, for a maximum that
    is negative, inside a full tile or in an edge tile."""
    rng = np.random.default_rng(2)
    for where in ((70, 80), (255, 319), (3, 317)):
        D = rng.standard_normal((256, 320)).astype(dtype)
        D[where] = -7.25
        cfg = ir.SolverConfig(rank=2, mode="fixed", max_iter=2)
        tr = ir.solve(D, cfg, device=0, colmajor=colmajor)[2]
        assert tr.thresholds[0] == float(np.abs(D).max()) == 7.25


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("colmajor", [0, 1, 2])
@pytest.mark.parametrize("offset", [0, 1])
def test_slab_sqnorms_match_numpy(ir, dtype, colmajor, offset):
    """ircur_slab_sqnorms (the den of solver.py:331-341) against numpy, for
    every copy mode, on an unaligned strided view of D (odd leading
    dimension, start off the 16-byte grid) and lines longer than one
    8192-element work unit."""
    from paper_2010_07422_b200 import _capi
    from paper_2010_07422_b200.solver import Context
    n1, n2, r = 700, 9000, 3
    rng = np.random.default_rng(5)
    base = torch.from_numpy(rng.standard_normal((n1, n2 + 3)).astype(dtype)).cuda()
    D = base[:, offset:offset + n2]
    sets = ir.draw_index_sets(n1, n2, 40, 300, ir.RngSeed(9), 2)
    ctx = Context(0, _capi.F32 if dtype == np.float32 else _capi.F64, n1, n2, r, 40, 300, 2)
    ctx.set_indices(sets)
    ctx.prepare(D, colmajor, cover=1)
    Dn = D.double().cpu().numpy()
    for s, (I, J) in enumerate(sets):
        a, b = ctx.slab_sqnorms(s)
        assert a == pytest.approx(float((Dn[I, :] ** 2).sum()), rel=1e-12)
        assert b == pytest.approx(float((Dn[:, J] ** 2).sum()), rel=1e-12)
    ctx.close()


@pytest.mark.parametrize("colmajor", ["sampled", "full", False])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_streamed_host_input_matches_device_input(ir, monkeypatch, colmajor, dtype):
    """A host D is copied in row chunks with the prep pass queued behind each
    chunk (solver._stream_in); the results must be bitwise those of the same
    D passed as a device tensor, and NaN in the last chunk is still
    rejected.  Streaming is forced on a small matrix (several chunks,
    a ragged last chunk)."""
    from paper_2010_07422_b200 import solver
    monkeypatch.setattr(solver, "_STREAM_MIN_BYTES", 0)
    monkeypatch.setattr(solver, "_STREAM_CHUNKS", 5)
    n1, n2, r = 700, 520, 3
    rng = np.random.default_rng(11)
    L = rng.standard_normal((n1, r)) @ rng.standard_normal((r, n2))
    S = np.where(rng.random((n1, n2)) < 0.05, 10.0 * rng.standard_normal((n1, n2)), 0.0)
    D = (L + S).astype(dtype)
    cfg = ir.SolverConfig(rank=r, mode="resampled", max_iter=30, seed=ir.RngSeed(5))
    a = ir.solve(D, cfg, device=0, colmajor=colmajor)
    b = ir.solve(torch.from_numpy(D).cuda(), cfg, device=0, colmajor=colmajor)
    assert a[2].iterations == b[2].iterations and a[2].errors == b[2].errors
    np.testing.assert_array_equal(a[0].C, b[0].C)
    np.testing.assert_array_equal(a[0].R, b[0].R)
    np.testing.assert_array_equal(a[1].row_values, b[1].row_values)
    D[n1 - 3, 7] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        ir.solve(D, cfg, device=0, colmajor=colmajor)


def test_prepare_rows_rejects_out_of_order_chunks(ir):
    """ircur_prepare_rows_async chunks must start at row 0 and continue in
    order (include/ircur_b200.h)."""
    from paper_2010_07422_b200 import _capi
    from paper_2010_07422_b200.solver import Context
    D = torch.randn(256, 64, device="cuda")
    ctx = Context(0, _capi.F32, 256, 64, 2, 16, 16, 4)
    ctx.set_indices(ir.draw_index_sets(256, 64, 16, 16, ir.RngSeed(1), 1))
    with pytest.raises(Exception):
        ctx.prepare_rows_async(D, 0, 1, 64, 128)  # no pass started at row 0
    ctx.prepare_rows_async(D, 0, 1, 0, 64)
    with pytest.raises(Exception):
        ctx.prepare_rows_async(D, 0, 1, 128, 256)  # gap
    ctx.prepare_rows_async(D, 0, 1, 64, 256)
    assert ctx.prepare_wait() == float(D.abs().max())
    ctx.close()


@pytest.mark.parametrize("colmajor", ["auto", "sampled", "full", False, True])
@pytest.mark.parametrize("mode", ["resampled", "fixed"])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_native_solve_matches_python_sequence(ir, monkeypatch, colmajor, mode, dtype):
    """ircur_solve (the host sequence in the library) against the Python
    sequence of solve_device (IRCUR_NATIVE=0): same draws, copy plan,
    thresholds, iterations and bitwise results."""
    n1, n2, r = 400, 350, 3
    rng = np.random.default_rng(21)
    D = (rng.standard_normal((n1, r)) @ rng.standard_normal((r, n2))
         + np.where(rng.random((n1, n2)) < 0.05, 8.0, 0.0)).astype(dtype)
    for zeta0 in (None, 9.0):
        cfg = ir.SolverConfig(rank=r, mode=mode, max_iter=25, zeta0=zeta0, seed=ir.RngSeed(8))
        monkeypatch.setenv("IRCUR_NATIVE", "0")
        a = ir.solve(D, cfg, device=0, colmajor=colmajor)
        monkeypatch.delenv("IRCUR_NATIVE")
        b = ir.solve(D, cfg, device=0, colmajor=colmajor)
        assert a[2].iterations == b[2].iterations and a[2].errors == b[2].errors
        assert a[2].thresholds == b[2].thresholds and a[2].converged == b[2].converged
        assert a[2].sampled_rows == b[2].sampled_rows and a[2].sampled_cols == b[2].sampled_cols
        np.testing.assert_array_equal(a[0].rows.indices, b[0].rows.indices)
        np.testing.assert_array_equal(a[0].C, b[0].C)
        np.testing.assert_array_equal(a[0].R, b[0].R)
        np.testing.assert_array_equal(a[1].col_values, b[1].col_values)
        np.testing.assert_array_equal(a[0].core_pinv.sigma, b[0].core_pinv.sigma)


def test_native_solve_zero_slabs(ir):
    """The den == 0 early exit through ircur_solve (solver.py:335-341)."""
    n1, n2, r = 300, 280, 3
    cfg = ir.SolverConfig(rank=r, zeta0=1.0, mode="resampled", max_iter=20, seed=ir.RngSeed(4))
    m1, m2 = ir.sample_count(n1, r, 4.0), ir.sample_count(n2, r, 4.0)
    I0, J0 = ir.draw_index_sets(n1, n2, m1, m2, cfg.seed, 1)[0]
    D = np.random.default_rng(0).standard_normal((n1, n2))
    D[I0, :] = 0.0
    D[:, J0] = 0.0
    cur, sp, tr = ir.solve(D, cfg, device=0)
    assert tr.errors == [0.0] and tr.converged and tr.iterations == 0 and not cur.C.any()
