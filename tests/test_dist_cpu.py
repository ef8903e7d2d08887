"""Row-sharded orchestration on CPU.

The rank programs of paper_2010_07422_b200/dist.py run with the test-only
numpy engine (tests/shard_engine_np.py) in place of the GPU context:
  * in one process through the lockstep driver (several shard counts,
    ranks that observe the device stop at different times);
  * in two processes over torch.distributed gloo (world_size 2), through
    the same `run_collective` driver the NCCL path uses.
Results are compared with the oracle (the reference algorithm restated).
"""

import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ircur_oracle as orc
from paper_2010_07422_b200 import RngSeed, SolverConfig
from paper_2010_07422_b200.dist import (gather_program, run_collective, run_lockstep, shard_rows,
                                        solve_shard_program)
from shard_engine_np import NumpyShardEngine, numpy_engine

N1, N2, RANK, ALPHA = 150, 130, 3, 0.1


def _problem(n1=N1, n2=N2, rank=RANK, seed=3):
    D, _, _, linf = orc.baseline_problem(n1, n2, rank, ALPHA, seed)
    return D, linf


def _cfg(linf, mode="resampled", max_iter=60):
    return SolverConfig(rank=RANK, eps=1e-9, zeta0=linf, gamma=0.7, mode=mode, max_iter=max_iter,
                        seed=RngSeed(5))


def _oracle(D, cfg):
    return orc.solve(D, rank=cfg.rank, eps=cfg.eps, zeta0=cfg.zeta0, gamma=cfg.gamma, mode=cfg.mode,
                     max_iter=cfg.max_iter, seed=5)


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def _check_against_oracle(cur, sparse, trace, ref):
    assert trace.iterations == ref.iterations
    assert trace.converged == ref.converged
    np.testing.assert_allclose(trace.errors, ref.errors, rtol=1e-8, atol=1e-14)
    np.testing.assert_array_equal(cur.rows.indices, ref.rows)
    np.testing.assert_array_equal(cur.cols.indices, ref.cols)
    for a, b in ((cur.C, ref.C), (cur.R, ref.R), (sparse.row_values, ref.S_rows),
                 (sparse.col_values, ref.S_cols)):
        assert a.shape == b.shape
        assert _rel(a, b) < 1e-9
    np.testing.assert_allclose(cur.core_pinv.sigma, ref.sigma, rtol=1e-9)


def _lockstep(D, cfg, world, engine=numpy_engine):
    n1 = D.shape[0]
    progs = []
    for g in range(world):
        r0, nl = shard_rows(n1, world, g)
        progs.append(solve_shard_program(D[r0:r0 + nl], cfg, n1=n1, row0=r0, engine_factory=engine))
    res = run_lockstep(progs)
    out = run_lockstep([gather_program(r) for r in res])
    return res, out


def test_shard_rows_partition():
    for n1 in (7, 100, 100001):
        for world in (1, 2, 3, 8):
            if n1 < world:
                continue
            spans = [shard_rows(n1, world, g) for g in range(world)]
            assert spans[0][0] == 0
            for (a, na), (b, _) in zip(spans, spans[1:]):
                assert a + na == b
            assert sum(n for _, n in spans) == n1
            assert max(n for _, n in spans) - min(n for _, n in spans) <= 1
    with pytest.raises(ValueError):
        shard_rows(3, 4, 0)


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("mode", ["resampled", "fixed"])
def test_lockstep_matches_oracle(world, mode):
    D, linf = _problem()
    cfg = _cfg(linf, mode)
    ref = _oracle(D, cfg)
    res, out = _lockstep(D, cfg, world)
    assert len({r.launched for r in res}) == 1  # identical collective counts on every rank
    for cur, sparse, trace in out:
        _check_against_oracle(cur, sparse, trace, ref)


class _LaggyEngine(NumpyShardEngine):
    """Reports device progress late (by a rank-dependent number of polls),
    like ranks whose hosts see the mapped stop flag at different times."""

    def __init__(self, *a, lag=0, **k):
        super().__init__(*a, **k)
        self.lag, self.hist = lag, []

    def poll(self):
        self.hist.append(super().poll())
        return self.hist[max(0, len(self.hist) - 1 - self.lag)]


def test_lockstep_stop_rule_with_lagging_ranks():
    D, linf = _problem()
    cfg = _cfg(linf)
    ref = _oracle(D, cfg)

    def factory(lag):
        def make(D_local, n1, row0, cfg, m_rows, m_cols, **_):
            return _LaggyEngine(D_local, n1, row0, cfg, m_rows, m_cols, lag=lag), D_local
        return make

    n1 = D.shape[0]
    progs = []
    for g in range(3):
        r0, nl = shard_rows(n1, 3, g)
        progs.append(solve_shard_program(D[r0:r0 + nl], cfg, n1=n1, row0=r0, engine_factory=factory(g * 2),
                                         ahead=2))
    res = run_lockstep(progs)
    assert len({r.launched for r in res}) == 1
    assert res[0].launched <= ref.iterations + 2
    cur, sparse, trace = run_lockstep([gather_program(r) for r in res])[0]
    _check_against_oracle(cur, sparse, trace, ref)


def test_lockstep_max_iter_and_zero_matrix():
    D, linf = _problem()
    cfg = _cfg(linf, max_iter=4)
    ref = _oracle(D, cfg)
    _, out = _lockstep(D, cfg, 2)
    cur, sparse, trace = out[0]
    assert trace.iterations == 4 and not trace.converged
    _check_against_oracle(cur, sparse, trace, ref)
    Z = np.zeros((40, 30))
    _, out = _lockstep(Z, SolverConfig(rank=2, zeta0=1.0), 2)
    cur, sparse, trace = out[0]
    assert trace.converged and trace.errors == [0.0] and not cur.C.any()


def test_lockstep_nonfinite_raises_on_every_rank():
    D, linf = _problem()
    D = D.copy()
    D[-1, 0] = np.nan  # only the last shard sees it
    n1 = D.shape[0]
    progs = [solve_shard_program(D[r0:r0 + nl], _cfg(linf), n1=n1, row0=r0, engine_factory=numpy_engine)
             for r0, nl in (shard_rows(n1, 2, g) for g in range(2))]
    first = [next(p) for p in progs]
    assert all(op == "max" for op, _ in first)
    acc = torch.maximum(first[0][1], first[1][1])
    for p, (_, t) in zip(progs, first):
        t.copy_(acc)
        with pytest.raises(ValueError, match="non-finite"):
            p.send(None)


# --------------------------------------------------------------- gloo (2 ranks)
def _gloo_worker(rank, world, port, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        D, linf = _problem()
        cfg = _cfg(linf)
        r0, nl = shard_rows(D.shape[0], world, rank)
        res = run_collective(solve_shard_program(D[r0:r0 + nl], cfg, n1=D.shape[0], row0=r0,
                                                 engine_factory=numpy_engine))
        cur, sparse, trace = run_collective(gather_program(res))
        np.savez(f"{path}.{rank}.npz", C=cur.C, R=cur.R, Sr=sparse.row_values, Sc=sparse.col_values,
                 sigma=cur.core_pinv.sigma, errors=np.array(trace.errors), iters=trace.iterations,
                 conv=trace.converged, launched=res.launched, rows=cur.rows.indices, cols=cur.cols.indices)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_matches_oracle():
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "out")
        mp.spawn(_gloo_worker, args=(2, port, path), nprocs=2, join=True)
        outs = [np.load(f"{path}.{r}.npz") for r in range(2)]
    D, linf = _problem()
    ref = _oracle(D, _cfg(linf))
    assert int(outs[0]["launched"]) == int(outs[1]["launched"])
    for o in outs:
        assert int(o["iters"]) == ref.iterations and bool(o["conv"]) == ref.converged
        np.testing.assert_allclose(o["errors"], ref.errors, rtol=1e-8, atol=1e-14)
        np.testing.assert_array_equal(o["rows"], ref.rows)
        for k, b in (("C", ref.C), ("R", ref.R), ("Sr", ref.S_rows), ("Sc", ref.S_cols)):
            assert _rel(o[k], b) < 1e-9
