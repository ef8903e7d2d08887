"""Row-sharded IRCUR across GPUs (one process per GPU).

SURVEY.md section 8(e) / BASELINE.json cfg5: D is split by rows, rank g owns
rows [row0_g, row0_g + n_g).  Index sets, thresholds and the core SVD are
replicated; everything that touches D is rank-local.  Per iteration three
all-reduces (SUM) cross the NVLink fabric:

  U      |I| x |J| fp64    the thresholded core; each rank fills its rows of I
  Qpart  r x n2            local partial sums of Q_{k+1} = W_r^T R
  scal   4 fp64            {den_I, res_I, den_J, res_J} for e_k (solver.py:393-400)

The per-rank work is a *program*: a generator that enqueues the library
phases (ircur_shard_phase) and yields a collective request at each exchange
point.  A driver services the requests.  `run_collective` uses
torch.distributed (NCCL on GPUs, gloo in the CPU tests); `run_lockstep`
advances several programs in one process and reduces their buffers
directly.  Lockstep runs enqueue work for each rank in turn, and no kernel
waits on another rank's kernel.

Requests are `("sum" | "max", tensor)`, reduced in place, or
`("gather", obj)`, where the driver sends back the list of every rank's
object.

Run-ahead: as on a single GPU, a rank enqueues up to `ahead` iterations past
the last one the device has finished.  Kernels after the stop are no-ops.
Each rank must issue the same collectives, so after the device reports the
stop at iteration K every rank keeps launching (no-op) iterations until
exactly min(max_iter, K + ahead) have been issued.  That number depends only
on K, which all ranks share.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .sampling import IndexSet, draw_index_sets, sample_count
from .types import CurFactors, PinvFactor, SolverConfig, SolverTrace, SparseEstimate

__all__ = ["shard_rows", "solve_shard_program", "run_collective", "run_lockstep", "solve_sharded",
           "ShardResult", "SHARD_CORE", "SHARD_FACTOR", "SHARD_RESID", "SHARD_STOP"]

SHARD_CORE, SHARD_FACTOR, SHARD_RESID, SHARD_STOP = 0, 1, 2, 3
FIXED, RESAMPLED = 0, 1


def shard_rows(n1: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous row ranges: (row0, n_rows) of `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    if n1 < world:
        raise ValueError(f"cannot split {n1} rows over {world} ranks")
    base, extra = divmod(n1, world)
    return rank * base + min(rank, extra), base + (1 if rank < extra else 0)


@dataclass
class ShardResult:
    """One rank's view after a sharded solve.  Strips are local: C and S_cols
    hold the rank's rows of D, R and S_rows its rows of I."""

    trace: SolverTrace
    cfg: SolverConfig
    engine: object
    sets: list
    row0: int
    n1: int
    n2: int
    zero_state: bool = False
    launched: int = 0


def _gpu_engine(D_local, n1: int, row0: int, config: SolverConfig, m_rows: int, m_cols: int,
                device=None, compute_dtype=None):
    """Default engine: a libircur_b200 context on this rank's GPU."""
    import torch

    from . import _capi
    from .solver import _context, _device_matrix, _release

    Dd = _device_matrix(D_local, device, compute_dtype)
    nloc, n2 = int(Dd.shape[0]), int(Dd.shape[1])
    dev = Dd.device.index
    dtype = _capi.F32 if Dd.dtype == torch.float32 else _capi.F64
    stream = torch.cuda.current_stream(dev).cuda_stream
    ctx = _context(dev, dtype, n1, n2, config.rank, m_rows, m_cols, config.max_iter, stream, row0, nloc)
    _release(ctx)  # one driving thread per rank: no lease needed against concurrent eviction
    return ctx, Dd


def solve_shard_program(D_local, config: SolverConfig, *, n1: int, row0: int, colmajor="auto",
                        ahead: int = 3, engine_factory=None, device=None, compute_dtype=None, profile=False,
                        native: bool = False, overlap: bool = True):
    """Generator: this rank's share of a row-sharded `solve` (solver.py:304-416).

    D_local holds rows [row0, row0 + D_local.shape[0]) of the n1 x n2 matrix.
    Returns (via StopIteration.value) a ShardResult.  profile=True records
    the strip launches' events (engine.profile(iterations)["strips_ms"]).
    native=True runs the iteration loop inside the library (ircur_shard_run:
    the same phases, collectives and run-ahead, issued from C++ over NCCL
    communicators the driver sets up with a ("native_comm", engine) request);
    the prep exchanges before the loop go through the driver as usual.  With
    overlap (fp32) the library runs the two-stream schedule: the SVD of k + 1
    beside the strips of k, one communicator per stream.
    """
    cfg = config
    if len(getattr(D_local, "shape", ())) != 2:
        raise ValueError("expected a 2-D row shard")
    nloc, n2 = int(D_local.shape[0]), int(D_local.shape[1])
    if n1 * n2 == 0 or nloc == 0:
        raise ValueError("D must be nonempty")
    m_rows = sample_count(n1, cfg.rank, cfg.c_rows)
    m_cols = sample_count(n2, cfg.rank, cfg.c_cols)
    resampled = cfg.mode == "resampled"
    sets = draw_index_sets(n1, n2, m_rows, m_cols, cfg.seed, cfg.max_iter if resampled else 1)
    make = engine_factory or _gpu_engine
    eng, Dd = make(D_local, n1, row0, cfg, m_rows, m_cols, device=device, compute_dtype=compute_dtype)
    if hasattr(eng, "set_profiling"):  # strip-kernel events (engine.profile) for the bench roofline
        eng.set_profiling(bool(profile))
    from .solver import _copy_plan

    cm, cover = _copy_plan(colmajor, n2, m_cols, sets, cfg)
    eng.set_indices(sets)
    if native and overlap and cfg.zeta0 is not None and cm != 0 and hasattr(eng, "shard_pre_chain"):
        # chain(0) / chain(1) of the library's overlapped loop beside the prep pass
        yield ("native_comm", eng)
        eng.shard_pre_chain(Dd, cfg.zeta0, cfg.gamma, RESAMPLED if resampled else FIXED, cfg.max_iter)
    # matcore.require_finite / inf_norm over all shards: every rank raises together
    bad, max_abs = 0.0, 0.0
    try:
        max_abs = eng.prepare(Dd, cm, cover)
    except ValueError as e:
        if "non-finite" not in str(e):
            raise
        bad = 1.0
    flag = eng.host_tensor([bad, max_abs])
    yield ("max", flag)
    if float(flag[0]) != 0.0:
        raise ValueError("matrix contains non-finite entries")
    max_abs = float(flag[1])
    a, b = eng.slab_sqnorms(0)
    den = eng.host_tensor([a, b])
    yield ("sum", den)
    rows0, cols0 = sets[0]
    if np.sqrt(float(den[0])) + np.sqrt(float(den[1])) == 0.0:  # solver.py:335-341
        tr = SolverTrace()
        tr.errors.append(0.0)
        tr.converged = True
        return ShardResult(tr, cfg, eng, sets, row0, n1, n2, zero_state=True)
    if cfg.zeta0 is None:
        cfg = replace(cfg, zeta0=max_abs)  # solver.py:342-344
    zetas = [cfg.gamma**k * cfg.zeta0 for k in range(cfg.max_iter)]
    mode = RESAMPLED if resampled else FIXED
    if native:
        yield ("native_comm", eng)
        iters, conv, errors, ms, launched = eng.shard_run(zetas, cfg.eps, mode, cfg.max_iter, ahead, overlap)
        return _shard_result(cfg, eng, sets, row0, n1, n2, zetas, resampled, iters, conv, errors, ms, launched)
    eng.shard_reset()
    U, Qp, scal = eng.shard_buffers()
    launched, stop_at = 0, cfg.max_iter
    while launched < stop_at:
        done, seen = eng.poll()
        if done:
            stop_at = min(stop_at, seen + ahead)
            if launched >= stop_at:
                break
        elif launched >= seen + ahead:
            continue  # spin: the device is `ahead` iterations behind
        k = launched
        s = k if resampled else 0
        eng.shard_phase(SHARD_CORE, k, s, zetas[k], cfg.eps, cfg.max_iter)
        yield ("sum", U)
        eng.shard_phase(SHARD_FACTOR, k, s, zetas[k], cfg.eps, cfg.max_iter)
        yield ("sum", Qp)
        eng.shard_phase(SHARD_RESID, k, s, zetas[k], cfg.eps, cfg.max_iter)
        yield ("sum", scal)
        eng.shard_phase(SHARD_STOP, k, s, zetas[k], cfg.eps, cfg.max_iter)
        launched += 1
    iters, conv, errors, ms = eng.shard_finish(zetas, mode)
    return _shard_result(cfg, eng, sets, row0, n1, n2, zetas, resampled, iters, conv, errors, ms, launched)


def _shard_result(cfg, eng, sets, row0, n1, n2, zetas, resampled, iters, conv, errors, ms, launched):
    tr = SolverTrace()
    tr.errors = [float(e) for e in errors]
    tr.seconds = [float(t) / 1e3 for t in ms]
    tr.iterations = iters
    tr.converged = conv
    tr.thresholds = zetas[:iters]
    tr.allocated = [0] * iters
    tr.sampled_rows = [int(sets[k if resampled else 0][0].size) for k in range(iters)]
    tr.sampled_cols = [int(sets[k if resampled else 0][1].size) for k in range(iters)]
    return ShardResult(tr, cfg, eng, sets, row0, n1, n2, launched=launched)


def gather_program(res: ShardResult):
    """Generator: all-gather the local strips into the reference's host
    results (CurFactors, SparseEstimate, SolverTrace) on every rank."""
    cfg = res.cfg
    if res.zero_state:
        from .solver import _zero_results

        I, J = res.sets[0]
        parts = yield ("gather", None)
        cur, sparse = _zero_results(res.n1, res.n2, IndexSet(I, res.n1), IndexSet(J, res.n2), cfg.rank)
        return cur, sparse, res.trace
    last = (res.trace.iterations - 1) if cfg.mode == "resampled" else 0
    C_loc, R_loc, Sr_loc, Sc_loc = res.engine.strips(last)
    parts = yield ("gather", (res.row0, C_loc, R_loc, Sr_loc, Sc_loc))
    parts = sorted(parts, key=lambda p: p[0])
    Cm = np.concatenate([p[1] for p in parts], axis=0)
    Rm = np.concatenate([p[2] for p in parts], axis=0)
    Sr = np.concatenate([p[3] for p in parts], axis=0)
    Sc = np.concatenate([p[4] for p in parts], axis=0)
    W, s, V, inv = res.engine.core()
    I, J = res.sets[last]
    rows, cols = IndexSet(I, res.n1), IndexSet(J, res.n2)
    cur = CurFactors(C=Cm, core_pinv=PinvFactor(W=W, sigma=s, V=V, inv_sigma=inv), R=Rm, rows=rows,
                     cols=cols, device=None)
    return cur, SparseEstimate(Sr, Sc, rows, cols), res.trace


# ------------------------------------------------------------------ drivers
def run_collective(program, group=None):
    """Run one rank's program, servicing its requests with torch.distributed
    collectives on `group` (NCCL for CUDA tensors, gloo for CPU)."""
    import torch.distributed as dist

    try:
        req = next(program)
        while True:
            op, payload = req
            if op == "native_comm":  # an NCCL communicator over the group for the engine's native loop
                _native_comm(payload, group)
                req = program.send(None)
                continue
            if op == "gather":
                out = [None] * dist.get_world_size(group)
                dist.all_gather_object(out, payload, group=group)
                req = program.send(out)
                continue
            rop = dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX
            dist.all_reduce(payload, op=rop, group=group)
            req = program.send(None)
    except StopIteration as stop:
        return stop.value


def _native_comm(eng, group) -> None:
    """Give `eng` (a library context) a communicator over `group` unless it
    already holds one for this group: the decision is all-reduced, so every
    rank takes part in the (collective) initialisation or none does."""
    import torch
    import torch.distributed as dist

    from .solver import nccl_unique_id

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    key = getattr(eng, "_comm_key", None)
    have = key is not None and key[0] == world and key[1] == rank and getattr(eng, "_comm_group", None) is group
    need = torch.tensor([0 if have else 1], dtype=torch.int64, device=f"cuda:{eng.device}"
                        if dist.get_backend(group) == "nccl" else "cpu")
    dist.all_reduce(need, op=dist.ReduceOp.MAX, group=group)
    if int(need.item()) == 0:
        return
    obj = [nccl_unique_id(2) if rank == 0 else None]
    src = 0 if group is None else dist.get_global_rank(group, 0)
    dist.broadcast_object_list(obj, src=src, group=group)
    eng.shard_comm_init(obj[0], world, rank)
    eng._comm_group = group


def run_lockstep(programs):
    """Run several rank programs in one process.  At every exchange point all
    programs must present the same request; it is reduced across them in
    place (sum/max over the tensors) before they resume."""
    n = len(programs)
    results = [None] * n
    reqs = []
    live = []
    for i, p in enumerate(programs):
        try:
            reqs.append(next(p))
            live.append(True)
        except StopIteration as stop:
            results[i] = stop.value
            reqs.append(None)
            live.append(False)
    while any(live):
        if not all(live):
            raise RuntimeError("rank programs diverged: some finished while others wait in a collective")
        ops = {r[0] for r in reqs}
        if len(ops) != 1:
            raise RuntimeError(f"rank programs diverged: requests {sorted(ops)}")
        op = ops.pop()
        if op == "native_comm":
            raise NotImplementedError("the native sharded loop needs one process per GPU (run_collective)")
        sends = [None] * n
        if op == "gather":
            sends = [[r[1] for r in reqs]] * n
        else:
            ts = [r[1] for r in reqs]
            acc = ts[0].clone()
            for t in ts[1:]:
                if op == "sum":
                    acc += t.to(acc.device)
                else:
                    acc = acc.maximum(t.to(acc.device))
            for t in ts:
                t.copy_(acc)
        for i, p in enumerate(programs):
            try:
                reqs[i] = p.send(sends[i])
            except StopIteration as stop:
                results[i] = stop.value
                reqs[i] = None
                live[i] = False
    return results


def solve_sharded(D_local, config: SolverConfig, observer=None, *, n1: int, row0: int, group=None,
                  gather: bool = True, colmajor="auto", device=None, compute_dtype=None, native: bool = False):
    """Row-sharded drop-in for `ircur.solve` inside a torch.distributed job:
    every rank passes its row shard of D.  With gather=True every rank gets
    the reference's (CurFactors, SparseEstimate, SolverTrace) on the host;
    otherwise the local ShardResult (factors stay on the device)."""
    if observer is not None:
        raise NotImplementedError("observer callbacks are supported by the single-GPU solve only")
    res = run_collective(solve_shard_program(D_local, config, n1=n1, row0=row0, colmajor=colmajor,
                                             device=device, compute_dtype=compute_dtype, native=native), group)
    if not gather:
        return res
    return run_collective(gather_program(res), group)
