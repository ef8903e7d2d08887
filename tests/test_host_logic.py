"""Host-side logic of the drop-in (no GPU): index draws, config validation,
threshold schedule, colmajor rule, generator restatements."""

import numpy as np
import pytest

from oracle import ircur_oracle as orc
import paper_2010_07422_b200 as ir
from paper_2010_07422_b200 import sampling
from paper_2010_07422_b200.solver import _copy_plan, _want_colmajor


def test_sorted_unique_equals_np_unique():
    rng = np.random.default_rng(0)
    for n, m in ((10, 50), (1000, 139), (100000, 461), (1, 3)):
        x = rng.integers(0, n, size=m)
        np.testing.assert_array_equal(sampling.sorted_unique(x), np.unique(x))
    np.testing.assert_array_equal(sampling.sorted_unique(np.array([], dtype=np.int64)), np.array([], dtype=np.int64))


@pytest.mark.parametrize("mode", ["fixed", "resampled"])
@pytest.mark.parametrize("shape", [(1000, 1000), (90, 60), (25344, 1000), (1, 1)])
def test_draw_order_equals_oracle_index_stream(mode, shape):
    n1, n2 = shape
    r, seed, max_iter = 3, 7, 6
    m1 = ir.sample_count(n1, r, 4.0)
    m2 = ir.sample_count(n2, r, 4.0)
    sets = ir.draw_index_sets(n1, n2, m1, m2, ir.RngSeed(seed), max_iter if mode == "resampled" else 1)
    ref = orc.index_stream(n1, n2, r, 4.0, 4.0, mode, max_iter, seed)
    for k in range(max_iter):
        I, J = sets[k if mode == "resampled" else 0]
        np.testing.assert_array_equal(I, ref[k][0])
        np.testing.assert_array_equal(J, ref[k][1])


def test_sample_count_matches_oracle():
    for n in (1, 2, 10, 1000, 10000, 25344, 100000):
        for r in (1, 2, 5, 10):
            for c in (0.5, 4.0):
                assert ir.sample_count(n, r, c) == orc.sample_count(n, r, c)


def test_solver_config_validation_messages():
    with pytest.raises(ValueError, match="rank"):
        ir.SolverConfig(rank=0)
    with pytest.raises(ValueError, match="eps"):
        ir.SolverConfig(rank=1, eps=0.0)
    with pytest.raises(ValueError, match="zeta0"):
        ir.SolverConfig(rank=1, zeta0=-1.0)
    with pytest.raises(ValueError, match="gamma"):
        ir.SolverConfig(rank=1, gamma=1.0)
    with pytest.raises(ValueError, match="mode"):
        ir.SolverConfig(rank=1, mode="other")
    with pytest.raises(ValueError, match="max_iter"):
        ir.SolverConfig(rank=1, max_iter=0)


def test_threshold_schedule_bits():
    cfg = ir.SolverConfig(rank=2, zeta0=3.7, gamma=0.7)
    for k in range(30):
        assert ir.threshold_at(cfg, k) == 0.7**k * 3.7  # the reference's expression, same bits
    with pytest.raises(ValueError):
        ir.threshold_at(cfg, -1)
    with pytest.raises(ValueError):
        ir.threshold_at(ir.SolverConfig(rank=2), 0)


def test_colmajor_rule(monkeypatch):
    monkeypatch.delenv("IRCUR_COLMAJOR", raising=False)
    assert _want_colmajor("auto", 100000, 100000, 461, 4, "resampled")
    assert _want_colmajor("auto", 10000, 10000, 185, 4, "resampled")
    assert not _want_colmajor("auto", 1000, 10**6, 10, 4, "resampled")
    assert _want_colmajor(True, 10, 10**6, 1, 4, "fixed") and not _want_colmajor(False, 10, 10, 5, 4, "fixed")
    monkeypatch.setenv("IRCUR_COLMAJOR", "0")
    assert not _want_colmajor(True, 10, 10, 5, 4, "fixed")


def test_blocked_generator_equals_reference_generator():
    D, L, S, linf = orc.baseline_problem(300, 170, 4, 0.2, 5)
    Db, linf_b, a = orc.baseline_problem_blocked(300, 170, 4, 0.2, 5, block_rows=64)
    np.testing.assert_array_equal(Db, D)
    assert linf_b == linf


def test_copy_plan(monkeypatch):
    monkeypatch.delenv("IRCUR_COLMAJOR", raising=False)
    cfg = ir.SolverConfig(rank=10, eps=1e-5, gamma=0.7, mode="resampled", max_iter=100)
    n = 100000
    m = ir.sample_count(n, 10, 4.0)
    sets = ir.draw_index_sets(n, n, m, m, ir.RngSeed(1), 100)
    mode, cover = _copy_plan("auto", n, m, sets, cfg)
    est = int(np.ceil(np.log(1e-5) / np.log(0.7)))  # 33: the schedule's iteration estimate
    assert mode == 2 and cover == (3 * est + 3) // 4 + 2 == 27  # (capi.cu cover_sets_for, the same rule)
    assert _copy_plan("full", n, m, sets, cfg) == (1, 0)
    assert _copy_plan(False, n, m, sets, cfg) == (0, 0)
    assert _copy_plan("sampled:3", n, m, sets, cfg) == (2, 3)
    fixed = ir.SolverConfig(rank=10, mode="fixed")
    assert _copy_plan(True, n, m, sets[:1], fixed) == (2, 1)
    # small n: the union of the sets covers most columns -> full copy
    sets2 = ir.draw_index_sets(200, 200, 60, 60, ir.RngSeed(1), 100)
    assert _copy_plan(True, 200, 60, sets2, cfg) == (1, 0)
    monkeypatch.setenv("IRCUR_COLMAJOR", "0")
    assert _copy_plan(True, n, m, sets, cfg) == (0, 0)


@pytest.mark.parametrize("shape,r,seed,stream", [((100000, 100000), 10, 1, 0), ((10000, 10000), 5, 7, 3),
                                                 ((1, 1), 1, 0, 0), ((2, 3), 2, 5, 1), ((1000, 97), 4, 11, 0),
                                                 ((25344, 1000), 2, 2, 0)])
def test_c_draws_equal_numpy(shape, r, seed, stream):
    """ircur_draw_index_sets (PCG64 + bounded Lemire + bitmap unique in C)
    reproduces numpy's integers()/unique sequence exactly."""
    from paper_2010_07422_b200.sampling import draw_index_sets_numpy
    n1, n2 = shape
    m1, m2 = ir.sample_count(n1, r, 4.0), ir.sample_count(n2, r, 4.0)
    s = ir.RngSeed(seed, stream)
    fast = ir.draw_index_sets(n1, n2, m1, m2, s, 60)
    ref = draw_index_sets_numpy(n1, n2, m1, m2, s, 60)
    for (a, b), (c, d) in zip(fast, ref):
        np.testing.assert_array_equal(a, c)
        np.testing.assert_array_equal(b, d)
        assert a.dtype == np.int64 and b.dtype == np.int64


def test_c_draws_continue_from_state():
    """Drawing n0 sets and then the rest from the returned PCG64 state gives
    the sequence of one call (the overlapped draws of solve_device)."""
    from paper_2010_07422_b200.sampling import draw_index_sets_from, pcg_words
    n, r = 50000, 7
    m = ir.sample_count(n, r, 4.0)
    s = ir.RngSeed(3, 2)
    whole = ir.draw_index_sets(n, n, m, m, s, 40)
    first, st = draw_index_sets_from(pcg_words(s), n, n, m, m, 17)
    rest, _ = draw_index_sets_from(st, n, n, m, m, 23)
    first.extend_drawn(rest)
    assert len(first) == 40 and first.rows.shape == (40, m)
    for (a, b), (c, d) in zip(first, whole):
        np.testing.assert_array_equal(a, c)
        np.testing.assert_array_equal(b, d)


@pytest.mark.parametrize("n1,n2,m1,m2,n_sets", [(2**31 + 12345, 3 * 2**30 + 7, 40, 30, 37),
                                                (100000, 100000, 461, 461, 49), (1, 5000, 3, 60, 25)])
def test_c_draws_chunked_with_rejections_equal_numpy(n1, n2, m1, m2, n_sets):
    """The threaded draws (chunks started at their rejection-free stream
    positions, redrawn where Lemire rejections shifted them) equal numpy's
    sequential integers()/unique stream, and the returned PCG64 state is
    numpy's state after the same draws.  At n ~ 2^31 about every second
    draw is rejected, so nearly every chunk is redrawn."""
    from paper_2010_07422_b200.sampling import draw_index_sets_from, pcg_words
    s = ir.RngSeed(13, 1)
    fast, st = draw_index_sets_from(pcg_words(s), n1, n2, m1, m2, n_sets)
    g = s.generator()
    for a, b in fast:
        np.testing.assert_array_equal(a, np.unique(g.integers(0, n1, m1)))
        np.testing.assert_array_equal(b, np.unique(g.integers(0, n2, m2)))
    ref = g.bit_generator.state
    m64 = (1 << 64) - 1
    want = [ref["state"]["state"] & m64, ref["state"]["state"] >> 64, ref["state"]["inc"] & m64,
            ref["state"]["inc"] >> 64, int(ref["has_uint32"])]
    assert [int(x) for x in st[:5]] == want
    if ref["has_uint32"]:
        assert int(st[5]) == int(ref["uinteger"])


def test_native_copy_code_matches_copy_plan(monkeypatch):
    """solver._native_copy_code (the code ircur_solve receives) makes the
    same copy-plan decision as solver._copy_plan for every colmajor form;
    code 3 is the covered-column rule, evaluated here like ircur_solve does."""
    from paper_2010_07422_b200.solver import _copy_plan, _cover_sets, _native_copy_code
    monkeypatch.delenv("IRCUR_COLMAJOR", raising=False)
    monkeypatch.delenv("IRCUR_NATIVE", raising=False)
    for (n, m, ns) in ((100000, 461, 49), (200, 60, 100), (10000, 185, 49)):
        sets = ir.draw_index_sets(n, n, m, m, ir.RngSeed(1), ns)
        for mode in ("resampled", "fixed"):
            cfg = ir.SolverConfig(rank=10, mode=mode, eps=1e-5, gamma=0.7)
            for cm in ("auto", "sampled", "full", False, True, 0, 1):
                want = _copy_plan(cm, n, m, sets, cfg)
                code = _native_copy_code(cm, n, m, cfg)
                assert code is not None
                cover = 1 if mode == "fixed" else max(1, min(len(sets), _cover_sets(cfg)))
                if code == 3:
                    u = len(set(np.concatenate([sets[k][1] for k in range(cover)]).tolist()))
                    got = (1, 0) if u > 0.7 * n else (2, cover)
                else:
                    got = (code, cover if code == 2 else 0)
                assert got == want, (n, mode, cm, got, want)
    monkeypatch.setenv("IRCUR_NATIVE", "0")
    assert _native_copy_code("auto", 1000, 10, ir.SolverConfig(rank=2)) is None
    monkeypatch.delenv("IRCUR_NATIVE")
    assert _native_copy_code("sampled:3", 1000, 10, ir.SolverConfig(rank=2)) is None
