"""Parity and properties at the BASELINE.json configurations.

* cfg2 (1e4 x 1e4, r = 5, alpha = 0.2) in fp64 and fp32: full trace against
  the CPU oracle (the reference algorithm) on the same data.
* cfg3 (video-like 25344 x 1000, r = 2): against the oracle.
* cfg4 (problems of the 512 x 2000^2 batch, per-problem seeds 1000 + p):
  against the oracle, solved one by one and through solve_batch.
* cfg5 (1e5 x 1e5 fp32, r = 10, 40 GB): too large for the oracle on the
  test box, so size-independent properties: convergence, recovery of the
  generator's known L on random blocks, bitwise run-to-run determinism, and
  the I x J intersection of the strips agreeing bitwise.
"""

import numpy as np
import pytest
import torch

from oracle import ircur_oracle as orc
import parity

pytestmark = pytest.mark.gpu

TOL64, TOL32 = 1e-9, 1e-4


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def ir():
    import paper_2010_07422_b200 as m
    from paper_2010_07422_b200 import _build
    _build.build()
    return m


def _solve_both(ir, D, rank, zeta0, seed, gamma=0.7, eps=1e-5, max_iter=100, mode="resampled"):
    ref = orc.solve(np.asarray(D, dtype=np.float64) if D.dtype == np.float32 else D, rank=rank, eps=eps,
                    zeta0=zeta0, gamma=gamma, mode=mode, max_iter=max_iter, seed=seed, record_x=True)
    kw = dict(rank=rank, eps=eps, zeta0=zeta0, gamma=gamma, mode=mode, max_iter=max_iter)

    def resolve(mi, e):
        return ir.solve(D, ir.SolverConfig(**{**kw, "max_iter": mi, "eps": e}, seed=ir.RngSeed(seed)), device=0)

    return ref, resolve(max_iter, eps), resolve


def _check(ref, out, f32, resolve=None, name=""):
    parity.check(out, ref, f32, resolve=resolve, name=name)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_cfg2_matches_oracle(ir, dtype):
    D, linf, _ = orc.baseline_problem_blocked(10000, 10000, 5, 0.2, 0, dtype=dtype)
    ref, out, resolve = _solve_both(ir, D, 5, linf, 1)
    _check(ref, out, dtype == np.float32, resolve, f"cfg2_{np.dtype(dtype).name}")
    ir.clear_cache()


def test_cfg3_video_matches_oracle(ir):
    from paper_2010_07422_b200.gen import video_problem
    D, L, S = video_problem(seed=0)
    ref, out, resolve = _solve_both(ir, D, 2, None, 1)
    _check(ref, out, True, resolve, "cfg3_video")
    # the foreground is recovered: S on the sampled rows has the blocks' support
    cur, sp, tr = out
    assert tr.converged
    ir.clear_cache()


@pytest.mark.parametrize("p", [0, 1])
def test_cfg4_problems_match_oracle(ir, p):
    D, _, _, linf = orc.baseline_problem(2000, 2000, 5, 0.2, 1000 + p)
    D = D.astype(np.float32)
    ref, out, resolve = _solve_both(ir, D, 5, linf, 1000 + p)
    _check(ref, out, True, resolve, f"cfg4_p{p}")


def test_cfg4_batch_equals_one_by_one(ir):
    """solve_batch's threaded path (several problems in flight on separate
    streams) gives bitwise the results of sequential solves."""
    probs, cfgs = [], []
    for p in range(6):
        D, _, _, linf = orc.baseline_problem(2000, 2000, 5, 0.2, 1000 + p)
        probs.append(D.astype(np.float32))
        cfgs.append(ir.SolverConfig(rank=5, eps=1e-5, zeta0=linf, gamma=0.7, mode="resampled", max_iter=100,
                                    seed=ir.RngSeed(1000 + p)))
    seq = [ir.solve(D, c, device=0) for D, c in zip(probs, cfgs)]
    bat = ir.solve_batch(probs, cfgs, device=0, streams=3, batched=False)
    for (c1, s1, t1), (c2, s2, t2) in zip(seq, bat):
        assert t1.errors == t2.errors and t1.iterations == t2.iterations
        np.testing.assert_array_equal(c1.C, c2.C)
        np.testing.assert_array_equal(s1.row_values, s2.row_values)


def test_cfg5_full_size_properties(ir):
    from paper_2010_07422_b200 import gen
    n, r = 100000, 10
    D, linf, _ = gen.baseline_problem_device(n, n, r, 0.2, 0, dtype=torch.float32)
    cfg = ir.SolverConfig(rank=r, eps=1e-5, zeta0=linf, gamma=0.7, mode="resampled", max_iter=100,
                          seed=ir.RngSeed(1))
    res = ir.solve_device(D, cfg)
    tr = res.trace
    assert tr.converged and tr.iterations <= 40 and tr.errors[-1] <= 1e-5
    assert all(b < a for a, b in zip(tr.errors[1:], tr.errors[2:]))  # monotone after the first step
    # recovery of the generator's L = W V^T on random blocks
    W, V, _ = gen.factors(n, n, r, 0)
    rng = np.random.default_rng(5)
    Pt, Qt = res.handle.Pt.double(), res.handle.Qt.double()
    for _ in range(3):
        ri = np.sort(rng.choice(n, 300, replace=False))
        ci = np.sort(rng.choice(n, 300, replace=False))
        Lb = (Pt[:, torch.from_numpy(ri).cuda()].T @ Qt[:, torch.from_numpy(ci).cuda()]).cpu().numpy()
        assert rel(Lb, W[ri] @ V[ci].T) <= 1e-4
    errors = list(tr.errors)
    # the I x J block of the final strips: C(I,:) and R(:,J) agree bitwise
    cur, sp = ir.solver._host_results(res.ctx, tr.iterations - 1, n, n, res.handle)
    I, J = cur.rows.indices, cur.cols.indices
    np.testing.assert_array_equal(cur.C[I, :], cur.R[:, J])
    np.testing.assert_array_equal(sp.col_values[I, :], sp.row_values[:, J])
    del cur, sp
    # run-to-run determinism
    res2 = ir.solve_device(D, cfg)
    assert list(res2.trace.errors) == errors
    del D, res, res2
    ir.clear_cache()
    torch.cuda.empty_cache()


def test_concurrent_streams_beyond_cache_limit(ir):
    """More host threads/streams than the context cache holds
    (solver._CACHE_MAX): contexts a solve is running on are leased and never
    evicted under it; every result equals the sequential solve."""
    import threading
    from paper_2010_07422_b200 import solver
    probs, cfgs = [], []
    for p in range(12):
        D, _, _, linf = orc.baseline_problem(600, 500, 3, 0.2, 2000 + p)
        probs.append(torch.from_numpy(D.astype(np.float32)).cuda())
        cfgs.append(ir.SolverConfig(rank=3, eps=1e-5, zeta0=linf, gamma=0.7, mode="resampled", max_iter=60,
                                    seed=ir.RngSeed(2000 + p)))
    seq = [ir.solve_device(D, c, fetch_factors="copy").trace.errors for D, c in zip(probs, cfgs)]
    nthreads = solver._CACHE_MAX + 4
    streams = [torch.cuda.Stream() for _ in range(nthreads)]
    out = [None] * len(probs)

    def worker(w):
        with torch.cuda.stream(streams[w]):
            for i in range(w, len(probs), nthreads):
                out[i] = ir.solve(probs[i].cpu().numpy(), cfgs[i], device=0)[2].errors
            streams[w].synchronize()

    th = [threading.Thread(target=worker, args=(w,)) for w in range(nthreads)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert out == seq


def test_concurrent_threads_same_stream_same_shape(ir):
    """The reference's threaded trial pool (cli.py:117-125, _run_trial
    cli.py:76-97) solves same-shaped problems from several threads on the
    default stream: each solve must get its own context (a shared one
    mixed index sets and core factors across threads)."""
    import threading
    probs, cfgs = [], []
    for p in range(12):
        D, _, _, linf = orc.baseline_problem(50, 50, 2, 0.2, 3000 + p)
        probs.append(D)
        cfgs.append(ir.SolverConfig(rank=2, zeta0=linf, gamma=0.7, mode="fixed", max_iter=30,
                                    c_rows=1.0 + (p % 2), c_cols=1.0 + (p % 2), seed=ir.RngSeed(3000 + p)))
    seq = [ir.solve(D, c, device=0) for D, c in zip(probs, cfgs)]
    out = [None] * len(probs)

    def worker(w):
        for i in range(w, len(probs), 4):
            out[i] = ir.solve(probs[i], cfgs[i], device=0)

    th = [threading.Thread(target=worker, args=(w,)) for w in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for (c1, s1, t1), (c2, s2, t2) in zip(seq, out):
        assert t1.errors == t2.errors
        np.testing.assert_array_equal(c1.rows.indices, c2.rows.indices)
        np.testing.assert_array_equal(c1.C, c2.C)
        np.testing.assert_array_equal(c1.core_pinv.W, c2.core_pinv.W)
