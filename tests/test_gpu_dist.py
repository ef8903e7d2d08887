"""Row-sharded device path (ircur_shard_* C-ABI) on one GPU.

Ranks are emulated in one process by the lockstep driver of
paper_2010_07422_b200/dist.py: each rank has its own library context over
its rows of D, and the all-reduces are done between phases by torch ops on
the same stream, so no kernel ever waits on another rank's kernel.
  * one shard: the split row-strip launches (partial sums, then finish)
    reproduce the single-GPU fused kernel bit for bit;
  * 2 and 3 shards: the oracle within the north-star tolerances (the Q sums
    are reassociated across shards, so not bitwise).
"""

import numpy as np
import pytest
import torch

from oracle import ircur_oracle as orc
import parity
import paper_2010_07422_b200 as ir
from paper_2010_07422_b200.dist import gather_program, run_lockstep, shard_rows, solve_shard_program

pytestmark = pytest.mark.gpu


def _problem(n1, n2, rank, seed=11, alpha=0.1):
    D, _, _, linf = orc.baseline_problem(n1, n2, rank, alpha, seed)
    return D, linf


def _cfg(rank, linf, mode="resampled", eps=1e-9, max_iter=80):
    return ir.SolverConfig(rank=rank, eps=eps, zeta0=linf, gamma=0.7, mode=mode, max_iter=max_iter,
                           seed=ir.RngSeed(2))


def _sharded(Dd, cfg, world):
    n1 = Dd.shape[0]
    progs = []
    for g in range(world):
        r0, nl = shard_rows(n1, world, g)
        progs.append(solve_shard_program(Dd[r0:r0 + nl], cfg, n1=n1, row0=r0))
    res = run_lockstep(progs)
    assert len({r.launched for r in res}) == 1
    return res, run_lockstep([gather_program(r) for r in res])


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.mark.parametrize("mode", ["resampled", "fixed"])
def test_one_shard_bitwise_equals_single_gpu(mode):
    D, linf = _problem(240, 200, 4)
    cfg = _cfg(4, linf, mode)
    Dd = torch.from_numpy(D).cuda()
    cur1, sp1, tr1 = ir.solve(Dd, cfg)
    _, out = _sharded(Dd, cfg, 1)
    cur, sp, tr = out[0]
    assert tr.iterations == tr1.iterations and tr.converged == tr1.converged
    assert tr.errors == tr1.errors
    for a, b in ((cur.C, cur1.C), (cur.R, cur1.R), (sp.row_values, sp1.row_values),
                 (sp.col_values, sp1.col_values), (cur.core_pinv.sigma, cur1.core_pinv.sigma)):
        np.testing.assert_array_equal(a, b)
    ir.clear_cache()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", ["resampled", "fixed"])
def test_sharded_fp64_matches_oracle(world, mode):
    D, linf = _problem(301, 257, 4)
    cfg = _cfg(4, linf, mode)
    ref = orc.solve(D, rank=4, eps=cfg.eps, zeta0=linf, gamma=0.7, mode=mode, max_iter=cfg.max_iter, seed=2)
    _, out = _sharded(torch.from_numpy(D).cuda(), cfg, world)
    for cur, sp, tr in out:
        assert tr.iterations == ref.iterations and tr.converged == ref.converged
        np.testing.assert_allclose(tr.errors, ref.errors, rtol=1e-9, atol=1e-15)
        np.testing.assert_array_equal(cur.rows.indices, ref.rows)
        np.testing.assert_array_equal(cur.cols.indices, ref.cols)
        for a, b in ((cur.C, ref.C), (cur.R, ref.R), (sp.row_values, ref.S_rows), (sp.col_values, ref.S_cols)):
            assert _rel(a, b) < 1e-9
        np.testing.assert_allclose(cur.core_pinv.sigma, ref.sigma, rtol=1e-9)
    ir.clear_cache()


def test_sharded_fp32_matches_oracle():
    D, linf = _problem(400, 380, 5, alpha=0.2)
    D32 = D.astype(np.float32)
    cfg = _cfg(5, linf, eps=1e-5)
    ref = orc.solve(D32.astype(np.float64), rank=5, eps=1e-5, zeta0=linf, gamma=0.7, mode="resampled",
                    max_iter=cfg.max_iter, seed=2, record_x=True)
    Dd = torch.from_numpy(D32).cuda()

    def resolve(mi, e):
        c = ir.SolverConfig(rank=5, eps=e, zeta0=linf, gamma=0.7, mode="resampled", max_iter=mi,
                            seed=ir.RngSeed(2))
        return _sharded(Dd, c, 2)[1][0]

    _, out = _sharded(Dd, cfg, 2)
    parity.check(out[0], ref, True, resolve=resolve, name="sharded2_f32")
    ir.clear_cache()


def test_sharded_nonfinite_raises():
    D, linf = _problem(120, 100, 3)
    D[-1, 5] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        _sharded(torch.from_numpy(D).cuda(), _cfg(3, linf), 2)
    ir.clear_cache()


@pytest.fixture(scope="module")
def gloo1():
    """A one-rank torch.distributed group (gloo) for the driver's own
    exchanges; the native loop brings its own NCCL communicator."""
    import os

    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    fresh = not dist.is_initialized()
    if fresh:
        dist.init_process_group("gloo", rank=0, world_size=1)
    yield
    if fresh:
        dist.destroy_process_group()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("mode", ["resampled", "fixed"])
def test_native_shard_loop_bitwise_equals_python_loop(gloo1, dtype, mode):
    """ircur_shard_run (the loop in the library, NCCL all-reduces) issues the
    same phases and collectives as the Python driver: bitwise the same trace,
    strips and core, the same number of launched iterations; a second solve
    reuses the communicator."""
    from paper_2010_07422_b200.dist import run_collective

    D, linf = _problem(300, 260, 4, seed=17)
    cfg = _cfg(4, linf, mode, eps=1e-5 if dtype == np.float32 else 1e-9)
    Dd = torch.from_numpy(D.astype(dtype)).cuda()
    outs = []
    for native in (False, True, True):
        res = run_collective(solve_shard_program(Dd, cfg, n1=300, row0=0, native=native, overlap=False))
        outs.append((res.launched, run_collective(gather_program(res))))
    (l0, (c0, s0, t0)) = outs[0]
    for li, (ci, si, ti) in outs[1:]:
        assert li == l0
        assert ti.iterations == t0.iterations and ti.converged == t0.converged and ti.errors == t0.errors
        for a, b in ((ci.C, c0.C), (ci.R, c0.R), (si.row_values, s0.row_values), (si.col_values, s0.col_values),
                     (ci.core_pinv.sigma, c0.core_pinv.sigma)):
            np.testing.assert_array_equal(a, b)
    ir.clear_cache()


@pytest.mark.parametrize("split", ["0", "1"])
@pytest.mark.parametrize("mode", ["resampled", "fixed"])
def test_native_overlapped_shard_loop_equals_single_gpu(gloo1, monkeypatch, mode, split):
    """The library's overlapped sharded loop (chain of k + 1 beside the strips
    of k, sampled Q partials and U all-reduced on one communicator, Q partials
    and the 4 sums on the other) at one rank: bitwise the single-GPU solve
    (the split strip launches and the sampled-factor kernel reproduce the
    fused kernels; both runs use the fp32 SVD tolerance lag of 2).  At one
    rank the row strip runs fused; IRCUR_SHARD_SPLIT=1 keeps the partial /
    all-reduce / finish sequence the N > 1 loop runs."""
    import ctypes as C

    monkeypatch.setenv("IRCUR_SHARD_SPLIT", split)

    from paper_2010_07422_b200.dist import run_collective

    D, linf = _problem(2000, 1800, 5, seed=19, alpha=0.2)
    cfg = _cfg(5, linf, mode, eps=1e-5)
    Dd = torch.from_numpy(D.astype(np.float32)).cuda()
    cur1, sp1, tr1 = ir.solve(Dd, cfg)
    res = run_collective(solve_shard_program(Dd, cfg, n1=2000, row0=0, native=True, overlap=True))
    ov = C.c_longlong(0)
    assert res.engine.lib.ircur_debug_counter(res.engine.h, 1, C.byref(ov)) == 0
    assert ov.value == 1, "the overlapped sharded loop did not run"
    cur, sp, tr = run_collective(gather_program(res))
    assert tr.iterations == tr1.iterations and tr.converged == tr1.converged
    assert tr.errors == tr1.errors
    for a, b in ((cur.C, cur1.C), (cur.R, cur1.R), (sp.row_values, sp1.row_values), (sp.col_values, sp1.col_values),
                 (cur.core_pinv.sigma, cur1.core_pinv.sigma)):
        np.testing.assert_array_equal(a, b)
    ir.clear_cache()


@pytest.mark.parametrize("split", ["0", "1"])
def test_run_ahead_reaching_the_column_cover(gloo1, monkeypatch, split):
    """With a loose eps the host's run-ahead (3 iterations) reaches the last
    set the sampled column copy covers (3/4 of the schedule's estimate + 2)
    although the solve has finished.  The single-GPU loops stop there; the
    sharded loop, whose ranks must launch the same count, goes on without
    extending the copy.  Results: the full copy's and the single GPU's, bit
    for bit."""
    from paper_2010_07422_b200.dist import run_collective
    from paper_2010_07422_b200.solver import _cover_sets

    monkeypatch.setenv("IRCUR_SHARD_SPLIT", split)
    D, linf = _problem(2000, 1800, 5, seed=23, alpha=0.2)
    cfg = _cfg(5, linf, "resampled", eps=1e-3)
    Dd = torch.from_numpy(D.astype(np.float32)).cuda()
    full = ir.solve(Dd, cfg, colmajor="full")
    assert full[2].converged and full[2].iterations + 3 >= _cover_sets(cfg) > full[2].iterations
    outs = [ir.solve(Dd, cfg, overlap=ov) for ov in (True, False)]
    res = run_collective(solve_shard_program(Dd, cfg, n1=2000, row0=0, native=True, overlap=True))
    outs.append(run_collective(gather_program(res)))
    again = ir.solve(Dd, cfg)  # (the contexts stay usable)
    outs.append(again)
    for cur, sp, tr in outs:
        assert tr.iterations == full[2].iterations and tr.converged and tr.errors == full[2].errors
        for a, b in ((cur.C, full[0].C), (cur.R, full[0].R), (sp.col_values, full[1].col_values)):
            np.testing.assert_array_equal(a, b)
    ir.clear_cache()


def test_native_sharded_loop_extends_the_column_copy(gloo1):
    """A sampled copy that covers 6 sets, extended while the library's sharded
    loop runs (gathers from the row-major shard, or a second prep pass when
    the copy's free lines run out): bitwise the single-GPU solve."""
    from paper_2010_07422_b200.dist import run_collective

    D, linf = _problem(2000, 1800, 5, seed=29, alpha=0.2)
    cfg = _cfg(5, linf, "resampled", eps=1e-5)
    Dd = torch.from_numpy(D.astype(np.float32)).cuda()
    cur1, sp1, tr1 = ir.solve(Dd, cfg)
    assert tr1.iterations > 14

    def sharded(ov, cm):
        res = run_collective(solve_shard_program(Dd, cfg, n1=2000, row0=0, native=True, overlap=ov, colmajor=cm))
        return run_collective(gather_program(res))

    for ov in (True, False):
        # (the sequential sharded loop takes its SVD tolerance from e_{k-1}, the overlapped
        # loops from e_{k-2}: each is compared with the full copy on its own loop)
        ref = (cur1, sp1, tr1) if ov else sharded(ov, "full")
        cur, sp, tr = sharded(ov, "sampled:6")
        assert tr.iterations == ref[2].iterations and tr.converged == ref[2].converged
        assert tr.errors == ref[2].errors, ov
        for a, b in ((cur.C, ref[0].C), (cur.R, ref[0].R), (sp.col_values, ref[1].col_values)):
            np.testing.assert_array_equal(a, b)
    ir.clear_cache()


def test_native_loop_edge_cases(gloo1):
    """fp64 with the default overlap request takes the library's sequential
    loop (the overlapped one is fp32); a den == 0 problem leaves the loop
    before it starts, after its chain(0) was queued beside the prep pass, and
    the next solve on the same context is unaffected."""
    from paper_2010_07422_b200.dist import run_collective

    D, linf = _problem(240, 220, 4, seed=23)
    cfg = _cfg(4, linf, "resampled", eps=1e-9)
    Dd = torch.from_numpy(D).cuda()
    a = run_collective(gather_program(run_collective(solve_shard_program(Dd, cfg, n1=240, row0=0, native=False))))
    b = run_collective(gather_program(run_collective(solve_shard_program(Dd, cfg, n1=240, row0=0, native=True))))
    assert a[2].errors == b[2].errors
    np.testing.assert_array_equal(a[0].C, b[0].C)
    # fp32: the zero-slab exit with a pre-launched chain, then a normal solve
    cfg32 = _cfg(4, linf, "resampled", eps=1e-5)
    n1, n2 = D.shape
    m1, m2 = ir.sample_count(n1, 4, 4.0), ir.sample_count(n2, 4, 4.0)
    I0, J0 = ir.draw_index_sets(n1, n2, m1, m2, cfg32.seed, 1)[0]
    Z = D.astype(np.float32).copy()
    Z[I0, :] = 0.0
    Z[:, J0] = 0.0
    z = run_collective(gather_program(run_collective(solve_shard_program(
        torch.from_numpy(Z).cuda(), cfg32, n1=n1, row0=0, native=True))))
    assert z[2].errors == [0.0] and z[2].converged
    D32 = torch.from_numpy(D.astype(np.float32)).cuda()
    one = ir.solve(D32, cfg32)
    sh = run_collective(gather_program(run_collective(solve_shard_program(D32, cfg32, n1=n1, row0=0, native=True))))
    assert sh[2].errors == one[2].errors
    np.testing.assert_array_equal(sh[0].C, one[0].C)
    ir.clear_cache()
