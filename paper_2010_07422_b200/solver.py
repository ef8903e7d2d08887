"""`solve(D, config, observer=None)` on a B200 — drop-in for `ircur.solver.solve`.

Reference: /root/reference/pkg/src/ircur/solver.py:304-416.  The Python
layer keeps the reference's signature, types, draw order, threshold schedule
and error behaviour; every arithmetic step of the loop runs in
libircur_b200.so (sm_100a kernels) through the C-ABI in
include/ircur_b200.h:

    require_finite / inf_norm  (matcore.py:70-91)   -> ircur_prepare
    pre-loop den == 0 check    (solver.py:331-341)  -> ircur_slab_sqnorms
    loop body + stop rule      (solver.py:358-414)  -> ircur_run / ircur_iterate
    returned C, R, S strips    (solver.py:375-391)  -> ircur_get_strips
    PinvFactor of the core     (matcore.py:142-165) -> ircur_get_core
    materialize                (solver.py:211-213)  -> ircur_materialize_factors

PyTorch provides device memory and the CUDA stream only.  There is no CPU
fallback: without a CUDA device or without the built library, solve raises.
"""

from __future__ import annotations

import ctypes as C
import os
from collections import OrderedDict
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _capi
from .sampling import DrawnSets, IndexSet, LazyDrawnSets, draw_index_sets, draw_index_sets_from, pcg_words, sample_count
from .types import CurFactors, PinvFactor, SolverConfig, SolverTrace, SparseEstimate

__all__ = ["solve", "solve_device", "solve_batch", "materialize", "materialize_device", "threshold_at",
           "Context", "DeviceResult"]


def threshold_at(config: SolverConfig, k: int) -> float:
    """gamma**k * zeta0 (solver.py:171-177)."""
    if k < 0:
        raise ValueError(f"k must be >= 0, got {k}")
    if config.zeta0 is None:
        raise ValueError("config.zeta0 is unresolved (None)")
    return config.gamma**k * config.zeta0


# --------------------------------------------------------------- context
def _ptr(t) -> int:
    return int(t.data_ptr())


class Context:
    """One libircur_b200 solver context (device workspace + stream)."""

    def __init__(self, device: int, dtype: int, n1: int, n2: int, rank: int, max_rows: int,
                 max_cols: int, max_iter: int, row0: int = 0, local_rows: int | None = None,
                 stream: int | None = None):
        self.lib = _capi.load()
        self.device, self.dtype, self.n1, self.n2, self.rank = device, dtype, n1, n2, rank
        self.max_rows, self.max_cols, self.max_iter = max_rows, max_cols, max_iter
        self.row0 = row0
        self.local_rows = n1 if local_rows is None else local_rows
        self.stream = stream if stream is not None else torch.cuda.current_stream(device).cuda_stream
        h = C.c_void_p()
        _capi.check(self.lib.ircur_ctx_create(C.byref(h), device, dtype, n1, n2, rank, max_rows,
                                              max_cols, max_iter, row0, self.local_rows,
                                              C.c_void_p(self.stream)))
        self.h = h
        self._busy = 0  # solves currently running on this context (solver._context leases)
        self._D = None
        self.sets: list = []
        self.colmajor = False

    def close(self) -> None:
        if self.h is not None and self.h.value:
            self.lib.ircur_ctx_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prepare(self, D: torch.Tensor, colmajor, cover: int = 0) -> float:
        """Finite check + max|D| (+ column-major copy): colmajor 0/False none,
        1/True full copy, 2 only the columns of the J sets [0, cover)
        (index sets must be uploaded first)."""
        self._D = D
        mode = int(colmajor)
        self.colmajor = mode
        ok = C.c_int(0)
        mx = C.c_double(0.0)
        if mode == 2:
            _capi.check(self.lib.ircur_prepare_sampled(self.h, C.c_void_p(_ptr(D)), D.stride(0), int(cover),
                                                       C.byref(ok), C.byref(mx)))
        else:
            _capi.check(self.lib.ircur_prepare(self.h, C.c_void_p(_ptr(D)), D.stride(0), mode,
                                               C.byref(ok), C.byref(mx)))
        return float(mx.value)

    def prepare_async(self, D: torch.Tensor, colmajor, cover: int = 0) -> None:
        """Queue the prep pass (see prepare) without waiting; prepare_wait
        returns its max|D| (ValueError on NaN/Inf)."""
        self._D = D
        mode = int(colmajor)
        self.colmajor = mode
        _capi.check(self.lib.ircur_prepare_async(self.h, C.c_void_p(_ptr(D)), D.stride(0), mode, int(cover)))

    def prepare_rows_async(self, D: torch.Tensor, colmajor, cover: int, r0: int, r1: int) -> None:
        """One row chunk [r0, r1) of the prep pass (chunks in order from 0)."""
        self._D = D
        mode = int(colmajor)
        self.colmajor = mode
        _capi.check(self.lib.ircur_prepare_rows_async(self.h, C.c_void_p(_ptr(D)), D.stride(0), mode, int(cover),
                                                      int(r0), int(r1)))

    def prepare_wait(self) -> float:
        ok = C.c_int(0)
        mx = C.c_double(0.0)
        _capi.check(self.lib.ircur_prepare_wait(self.h, C.byref(ok), C.byref(mx)))
        return float(mx.value)

    def slab_sqnorms_async(self, s: int) -> None:
        _capi.check(self.lib.ircur_slab_sqnorms_async(self.h, s))

    def set_indices(self, sets) -> None:
        n = len(sets)
        pre = getattr(sets, "rows", None)
        if pre is not None and pre.shape == (n, self.max_rows) and sets.cols.shape == (n, self.max_cols):
            rows, cols, rc, cc = sets.rows, sets.cols, sets.row_counts, sets.col_counts
        else:
            rows = np.zeros((n, self.max_rows), dtype=np.int64)
            cols = np.zeros((n, self.max_cols), dtype=np.int64)
            rc = np.zeros(n, dtype=np.int32)
            cc = np.zeros(n, dtype=np.int32)
            for s, (I, J) in enumerate(sets):
                rows[s, :I.size] = I
                cols[s, :J.size] = J
                rc[s], cc[s] = I.size, J.size
        p64 = C.POINTER(C.c_int64)
        p32 = C.POINTER(C.c_int32)
        _capi.check(self.lib.ircur_set_indices(self.h, n, rows.ctypes.data_as(p64), rc.ctypes.data_as(p32),
                                               cols.ctypes.data_as(p64), cc.ctypes.data_as(p32)))
        self.sets = sets

    def append_indices(self, sets) -> None:
        """Upload more sets after the current ones (a DrawnSets)."""
        p64, p32 = C.POINTER(C.c_int64), C.POINTER(C.c_int32)
        _capi.check(self.lib.ircur_append_indices(self.h, len(sets), sets.rows.ctypes.data_as(p64),
                                                  sets.row_counts.ctypes.data_as(p32),
                                                  sets.cols.ctypes.data_as(p64),
                                                  sets.col_counts.ctypes.data_as(p32)))
        self.sets = list(self.sets) + list(sets)

    def slab_sqnorms(self, s: int) -> tuple[float, float]:
        a, b = C.c_double(), C.c_double()
        _capi.check(self.lib.ircur_slab_sqnorms(self.h, s, C.byref(a), C.byref(b)))
        return a.value, b.value

    def run(self, zetas, eps: float, mode: int, max_iter: int):
        z = np.ascontiguousarray(zetas, dtype=np.float64)
        errors = np.zeros(max_iter, dtype=np.float64)
        ms = np.zeros(max_iter, dtype=np.float32)
        it, conv = C.c_int(0), C.c_int(0)
        pd = C.POINTER(C.c_double)
        _capi.check(self.lib.ircur_run(self.h, z.ctypes.data_as(pd), eps, mode, max_iter, C.byref(it),
                                       C.byref(conv), errors.ctypes.data_as(pd),
                                       ms.ctypes.data_as(C.POINTER(C.c_float))))
        n = it.value
        return n, bool(conv.value), errors[:n], ms[:n]

    def set_target_eps(self, eps: float) -> None:
        _capi.check(self.lib.ircur_set_target_eps(self.h, float(eps)))

    def iterate(self, k: int, s: int, zeta: float) -> float:
        e = C.c_double()
        _capi.check(self.lib.ircur_iterate(self.h, k, s, zeta, C.byref(e)))
        return e.value

    def strips(self, set_idx: int, on_device: bool = False):
        I, J = self.sets[set_idx]
        mI = int(np.count_nonzero((I >= self.row0) & (I < self.row0 + self.local_rows)))
        nJ = J.size
        shapes = [(self.local_rows, nJ), (mI, self.n2), (mI, self.n2), (self.local_rows, nJ)]
        if on_device:
            outs = [torch.empty(s, dtype=torch.float64, device=f"cuda:{self.device}") for s in shapes]
            ptrs = [C.c_void_p(_ptr(t)) for t in outs]
        else:
            # page-locked host arrays (torch's caching host allocator): the
            # write-out kernels store into them directly at PCIe speed, where
            # first-touch pageable memory runs at a few GB/s
            outs = [torch.empty(s, dtype=torch.float64, pin_memory=True).numpy() for s in shapes]
            ptrs = [C.c_void_p(o.ctypes.data) for o in outs]
        _capi.check(self.lib.ircur_get_strips(self.h, *ptrs))
        return outs  # C, R, S_rows, S_cols

    def core(self):
        k, m, n = C.c_int(), C.c_int(), C.c_int()
        _capi.check(self.lib.ircur_get_core(self.h, None, None, None, None, C.byref(k), C.byref(m), C.byref(n)))
        k, m, n = k.value, m.value, n.value
        W = np.zeros((m, k)); V = np.zeros((n, k)); s = np.zeros(k); inv = np.zeros(k)
        vp = lambda a: C.c_void_p(a.ctypes.data)  # noqa: E731
        _capi.check(self.lib.ircur_get_core(self.h, vp(W), vp(s), vp(V), vp(inv), None, None, None))
        return W, s, V, inv

    def set_profiling(self, on: bool) -> None:
        _capi.check(self.lib.ircur_set_profiling(self.h, int(on)))

    def set_overlap(self, overlap) -> None:
        """None: library default; True / False: overlapped (where eligible) / sequential loop."""
        _capi.check(self.lib.ircur_set_overlap(self.h, -1 if overlap is None else int(bool(overlap))))

    def profile(self, n_iters: int) -> dict:
        li, kl = C.c_int(), C.c_longlong()
        arrs = [np.zeros(max(n_iters, 1), dtype=np.float32) for _ in range(4)]
        pf = C.POINTER(C.c_float)
        _capi.check(self.lib.ircur_get_profile(self.h, n_iters, C.byref(li), C.byref(kl),
                                               *[a.ctypes.data_as(pf) for a in arrs]))
        steps = np.zeros(max(n_iters, 1), dtype=np.int32)
        _capi.check(self.lib.ircur_get_svd_steps(self.h, n_iters, steps.ctypes.data_as(C.POINTER(C.c_int))))
        marks = np.full(5, -1.0, dtype=np.float32)
        _capi.check(self.lib.ircur_get_marks(self.h, marks.ctypes.data_as(pf)))
        ov = C.c_longlong(0)
        _capi.check(self.lib.ircur_debug_counter(self.h, 1, C.byref(ov)))
        # overlapped loop: svd_ms is the chain (core, Gram, SVD) beside the strips; core_ms is 0
        return dict(launched_iters=li.value, kernel_launches=kl.value, svd_steps=steps[:n_iters],
                    overlapped=bool(ov.value),
                    gaps_ms=dict(zip(("upload_to_prep", "prep", "prep_to_slab_end", "slab_to_run",
                                      "run_to_first_kernel"), [float(x) for x in marks])),
                    core_ms=arrs[0][:n_iters], svd_ms=arrs[1][:n_iters],
                    strips_ms=arrs[2][:n_iters], finalize_ms=arrs[3][:n_iters])

    # ---- row-sharded loop (include/ircur_b200.h, "Row-sharded loop")
    def shard_buffers(self):
        """(U fp64, Qpart, scal[:4]) as zero-copy torch views of the context's
        exchange buffers, for the caller's all-reduce."""
        u, q, sc = C.c_void_p(), C.c_void_p(), C.c_void_p()
        nu, nq = C.c_int64(), C.c_int64()
        _capi.check(self.lib.ircur_shard_buffers(self.h, C.byref(u), C.byref(nu), C.byref(q), C.byref(nq),
                                                 C.byref(sc)))
        qdt = "<f4" if self.dtype == _capi.F32 else "<f8"
        return (_device_view(u.value, nu.value, "<f8", self.device),
                _device_view(q.value, nq.value, qdt, self.device),
                _device_view(sc.value, 4, "<f8", self.device))

    def host_tensor(self, vals) -> torch.Tensor:
        """A small fp64 tensor on this context's device (scalar all-reduces)."""
        return torch.tensor(vals, dtype=torch.float64, device=f"cuda:{self.device}")

    def shard_reset(self) -> None:
        _capi.check(self.lib.ircur_shard_reset(self.h))

    def shard_phase(self, phase: int, k: int, s: int, zeta: float, eps: float, max_iter: int) -> None:
        _capi.check(self.lib.ircur_shard_phase(self.h, phase, k, s, zeta, eps, max_iter))

    def shard_comm_init(self, uids: bytes, nranks: int, rank: int) -> None:
        """Give this context its NCCL communicators (a collective: every rank
        calls it with the same ids from nccl_unique_id(), 128 bytes each; two
        ids give the overlapped loop one communicator per stream)."""
        n = len(uids) // 128
        buf = C.create_string_buffer(bytes(uids), 128 * n)
        _capi.check(self.lib.ircur_shard_comm_init(self.h, buf, n, nranks, rank))
        self._comm_key = (nranks, rank, bytes(uids))

    def shard_pre_chain(self, D, zeta0: float, gamma: float, mode: int, max_iter: int) -> None:
        """Queue chain(0) / chain(1) of the overlapped sharded loop before the
        prep pass (ircur_shard_pre_chain); D is this rank's device shard."""
        _capi.check(self.lib.ircur_shard_pre_chain(self.h, C.c_void_p(D.data_ptr()), int(D.stride(0)), float(zeta0),
                                                   float(gamma), int(mode), int(max_iter)))

    def shard_run(self, zetas, eps: float, mode: int, max_iter: int, ahead: int, overlap: bool = True):
        """The whole sharded loop in the library (ircur_shard_run):
        (iterations, converged, errors, ms, launched)."""
        z = np.ascontiguousarray(zetas, dtype=np.float64)
        errors = np.zeros(max_iter, dtype=np.float64)
        ms = np.zeros(max_iter, dtype=np.float32)
        it, conv, la = C.c_int(0), C.c_int(0), C.c_int(0)
        pd = C.POINTER(C.c_double)
        _capi.check(self.lib.ircur_shard_run(self.h, z.ctypes.data_as(pd), float(eps), int(mode), int(max_iter),
                                             int(ahead), 1 if overlap else 0, C.byref(it), C.byref(conv),
                                             errors.ctypes.data_as(pd), ms.ctypes.data_as(C.POINTER(C.c_float)),
                                             C.byref(la)))
        n = it.value
        return n, bool(conv.value), errors[:n], ms[:n], la.value

    def poll(self) -> tuple[bool, int]:
        d, it = C.c_int(), C.c_int()
        _capi.check(self.lib.ircur_poll(self.h, C.byref(d), C.byref(it)))
        return bool(d.value), it.value

    def shard_finish(self, zetas, mode: int):
        z = np.ascontiguousarray(zetas, dtype=np.float64)
        n = len(z)
        errors = np.zeros(n, dtype=np.float64)
        ms = np.zeros(n, dtype=np.float32)
        it, conv = C.c_int(0), C.c_int(0)
        pd = C.POINTER(C.c_double)
        _capi.check(self.lib.ircur_shard_finish(self.h, z.ctypes.data_as(pd), mode, C.byref(it), C.byref(conv),
                                                errors.ctypes.data_as(pd), ms.ctypes.data_as(C.POINTER(C.c_float))))
        n = it.value
        return n, bool(conv.value), errors[:n], ms[:n]

    def factor_views(self):
        """(P^T, Q) as zero-copy views of the context's final factor buffers
        (valid until the next solve on this context)."""
        pp, qq = C.c_void_p(), C.c_void_p()
        lp, lq = C.c_int64(), C.c_int64()
        _capi.check(self.lib.ircur_factor_buffers(self.h, C.byref(pp), C.byref(lp), C.byref(qq), C.byref(lq)))
        ts = "<f4" if self.dtype == _capi.F32 else "<f8"
        r = self.rank
        Pt = _device_view(pp.value, r * lp.value, ts, self.device).view(r, lp.value)[:, :self.local_rows]
        Qt = _device_view(qq.value, r * lq.value, ts, self.device).view(r, lq.value)[:, :self.n2]
        return Pt, Qt

    def factors(self):
        tdt = torch.float32 if self.dtype == _capi.F32 else torch.float64
        dev = f"cuda:{self.device}"
        Pt = torch.empty((self.rank, self.local_rows), dtype=tdt, device=dev)
        Qt = torch.empty((self.rank, self.n2), dtype=tdt, device=dev)
        _capi.check(self.lib.ircur_get_factors(self.h, C.c_void_p(_ptr(Pt)), C.c_void_p(_ptr(Qt))))
        return Pt, Qt


class _CudaArray:
    """__cuda_array_interface__ wrapper so torch can view a library buffer."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr), False),
                                         "strides": None, "version": 3}


def _device_view(ptr: int, n: int, typestr: str, device: int) -> torch.Tensor:
    return torch.as_tensor(_CudaArray(ptr, n, typestr), device=f"cuda:{device}")


_CACHE: "OrderedDict[tuple, Context]" = OrderedDict()
_CACHE_MAX = 4
_CACHE_LOCK = __import__("threading").RLock()


def _context(device, dtype, n1, n2, rank, m_rows, m_cols, max_iter, stream, row0=0,
             local_rows=None) -> Context:
    local_rows = n1 if local_rows is None else local_rows
    key = (device, dtype, n1, n2, rank, m_rows, m_cols, max_iter, stream, row0, local_rows)
    with _CACHE_LOCK:
        ctx = _context_locked(key, device, dtype, n1, n2, rank, m_rows, m_cols, max_iter, stream, row0,
                              local_rows)
        ctx._busy += 1  # leased until _release: never evicted while a solve runs on it
        return ctx


def _release(ctx: Context) -> None:
    with _CACHE_LOCK:
        ctx._busy -= 1


def _evict_idle(keep: int) -> None:
    """Close least-recently-used contexts that no solve is running on until
    at most `keep` remain (contexts in use stay; the cache then grows)."""
    while len(_CACHE) > keep:
        victim = next((k for k, c in _CACHE.items() if c._busy == 0), None)
        if victim is None:
            return
        _CACHE.pop(victim).close()


def _context_locked(key, device, dtype, n1, n2, rank, m_rows, m_cols, max_iter, stream, row0,
                    local_rows) -> Context:
    # A context serves one solve at a time: threads solving problems of the
    # same shape on the same stream (e.g. the reference's threaded trial
    # pool, cli.py:117-125, all on the default stream) each get their own.
    slot = 0
    while True:
        ctx = _CACHE.get(key + (slot,))
        if ctx is None:
            break
        if ctx._busy == 0:
            _CACHE.move_to_end(key + (slot,))
            return ctx
        slot += 1
    key = key + (slot,)
    _evict_idle(_CACHE_MAX - 1)
    try:
        ctx = Context(device, dtype, n1, n2, rank, m_rows, m_cols, max_iter, row0, local_rows, stream=stream)
    except MemoryError:
        _evict_idle(0)  # out of memory: drop every idle context, then retry once
        torch.cuda.empty_cache()
        ctx = Context(device, dtype, n1, n2, rank, m_rows, m_cols, max_iter, row0, local_rows, stream=stream)
    _CACHE[key] = ctx
    return ctx


def clear_cache() -> None:
    """Close every cached context no solve is currently running on."""
    with _CACHE_LOCK:
        _evict_idle(0)


# ------------------------------------------------------------ device input
def _device_matrix(D, device, compute_dtype) -> torch.Tensor:
    """D as a row-major CUDA tensor in the storage/compute dtype (fp32 stays
    fp32, everything else becomes fp64 as in matcore.require_finite)."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2010_07422_b200.solve needs a CUDA device (no CPU fallback)")
    if isinstance(D, torch.Tensor):
        t = D
    else:
        a = np.asarray(D)
        if a.dtype != np.float32:
            a = np.asarray(a, dtype=np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a))
    if t.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={t.ndim}")
    want = compute_dtype
    if want is None:
        want = torch.float32 if t.dtype == torch.float32 else torch.float64
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    t = t.to(device=dev, dtype=want)
    if t.numel() and (t.stride(1) != 1 or t.stride(0) < t.shape[1]):
        t = t.contiguous()
    return t


_STREAM_CHUNKS = 16          # row chunks of a host D streamed in under the prep pass
_STREAM_MIN_BYTES = 256 << 20
_copy_streams: dict = {}


def _host_source(D, device, compute_dtype):
    """(host tensor, device dtype) when D is a contiguous host matrix worth
    streaming in chunks (the prep pass then runs under the copy), else None."""
    if isinstance(D, torch.Tensor):
        if D.is_cuda:
            return None
        t = D
    elif isinstance(D, np.ndarray) and D.dtype in (np.float32, np.float64):
        t = torch.from_numpy(D)
    else:
        return None
    if t.ndim != 2 or not t.is_contiguous() or t.numel() * t.element_size() < _STREAM_MIN_BYTES:
        return None
    want = compute_dtype or (torch.float32 if t.dtype == torch.float32 else torch.float64)
    if t.dtype != want:
        return None
    return t, want


def _stream_in(Dh: torch.Tensor, Dd: torch.Tensor, ctx: "Context", cm: int, cover: int) -> None:
    """Copy host rows into Dd chunk by chunk on a side stream and queue each
    chunk's prep pass on the context stream behind its copy."""
    dev = Dd.device
    cs = _copy_streams.get(dev.index)
    if cs is None:
        cs = _copy_streams[dev.index] = torch.cuda.Stream(device=dev)
    cur = torch.cuda.current_stream(dev)
    cs.wait_stream(cur)  # Dd's allocation / earlier users
    Dd.record_stream(cs)
    n1 = Dd.shape[0]
    step = max(64, -(-n1 // _STREAM_CHUNKS))
    step = -(-step // 64) * 64
    for r0 in range(0, n1, step):
        r1 = min(n1, r0 + step)
        with torch.cuda.stream(cs):
            Dd[r0:r1].copy_(Dh[r0:r1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        cur.wait_event(ev)
        ctx.prepare_rows_async(Dd, cm, cover, r0, r1)


def _want_colmajor(colmajor, n1, n2, m_cols, dtype_size, mode) -> bool:
    env = os.environ.get("IRCUR_COLMAJOR")
    if env is not None:
        return env not in ("0", "false", "False", "")
    if colmajor != "auto":
        return bool(colmajor)
    # The copy costs one extra write of D (~n1*n2*s at ~4.8 TB/s); without it
    # every iteration gathers the column strip in 32-byte sectors.  Measured
    # at n = 1e5, |J| = 461 (fp32): copy 10.8 ms extra vs 1.35 ms saved per
    # iteration, i.e. break-even after ~8 iterations; the break-even scales
    # with n2 / |J|.  IRCUR converges in ~20-25 iterations.
    return n2 < 600 * m_cols


class _Ticker:
    """Host wall-clock marks between the phases of solve_device (profiling)."""

    def __init__(self, on: bool):
        import time
        self.on, self.clock = on, time.perf_counter
        self.t = self.clock() if on else 0.0
        self.marks: dict = {}

    def __call__(self, name: str) -> None:
        if self.on:
            t = self.clock()
            self.marks[name] = (t - self.t) * 1e3
            self.t = t


def _cover_estimate(cfg: SolverConfig) -> int:
    """Iterations the threshold schedule needs to reach eps: ceil(log eps / log gamma)."""
    return int(np.ceil(np.log(cfg.eps) / np.log(cfg.gamma)))


def _cover_sets(cfg: SolverConfig) -> int:
    """J sets the prep pass copies column-major (capi.cu cover_sets_for, the same
    rule): 3/4 of the schedule's estimate + 2.  Measured iteration counts are
    ~0.7 of the estimate, and the library extends the copy set by set (a gather
    from the row-major D) if the loop runs longer."""
    return (3 * _cover_estimate(cfg) + 3) // 4 + 2


def _copy_plan(colmajor, n2: int, m_cols: int, sets, cfg: SolverConfig) -> tuple[int, int]:
    """Which column-major copy the prep pass builds: (mode, cover) with mode
    0 = none, 1 = full copy of D, 2 = only the columns of the J sets
    [0, cover) (extended automatically if the loop runs longer).  cover is
    _cover_sets: 3/4 of the iteration count the threshold schedule needs to
    reach eps (log eps / log gamma) plus 2."""
    env = os.environ.get("IRCUR_COLMAJOR")
    if env is not None:
        colmajor = {"0": False, "1": "full", "2": "sampled"}.get(env, env)
    if colmajor in (False, 0, "0", "false", "False", "none", ""):
        return 0, 0
    if colmajor == "auto" and not _want_colmajor("auto", 0, n2, m_cols, 0, cfg.mode):
        return 0, 0
    if colmajor in ("full", 1) and colmajor is not True:
        return 1, 0
    if cfg.mode == "fixed":
        cover = 1
    else:
        cover = max(1, min(len(sets), _cover_sets(cfg)))
    if isinstance(colmajor, str) and colmajor.startswith("sampled"):
        if ":" in colmajor:  # "sampled:K" covers the first K sets (tests of the extension path)
            cover = max(1, min(len(sets), int(colmajor.split(":")[1])))
        return 2, cover
    mark = np.zeros(n2, dtype=bool)
    padded = getattr(sets, "cols", None)
    if padded is not None:
        # rows of sets.cols are padded with zeros past their counts; column
        # 0 can only be a set's first (smallest) entry
        mark[padded[:cover].ravel()] = True
        mark[0] = bool((padded[:cover, 0] == 0).any())
    else:
        for k in range(cover):
            mark[sets[k][1]] = True
    return (1, 0) if np.count_nonzero(mark) > 0.7 * n2 else (2, cover)


@dataclass
class DeviceHandle:
    """Final rank-r factors on the device: L = P Q with P^T (r x n1) and Q (r x n2)."""

    Pt: torch.Tensor
    Qt: torch.Tensor
    dtype: int


class _LazyDeviceHandle:
    """DeviceHandle whose P^T / Q views of the context's factor buffers are
    made on first use (torch.as_tensor over __cuda_array_interface__ costs
    tens of microseconds, which adds up over the 512 results of a batch).
    The views alias the same buffers whenever they are made: valid until the
    context's next solve, like DeviceHandle's."""

    def __init__(self, ctx: "Context", dtype: int):
        self._ctx = ctx
        self.dtype = dtype
        self._views = None

    def _get(self):
        if self._views is None:
            self._views = self._ctx.factor_views()
        return self._views

    @property
    def Pt(self) -> torch.Tensor:
        return self._get()[0]

    @property
    def Qt(self) -> torch.Tensor:
        return self._get()[1]


@dataclass
class DeviceResult:
    trace: SolverTrace
    cfg: SolverConfig
    ctx: Context | None
    rows: IndexSet
    cols: IndexSet
    handle: DeviceHandle | None
    zero_state: bool = False
    profile: dict | None = None
    colmajor: bool = False
    sets: list | None = None

    def read_profile(self) -> dict | None:
        """Per-kernel event times of a solve run with profile="deferred"
        (valid until the next solve on the same context)."""
        if self.profile is None and self.ctx is not None:
            host = getattr(self, "_host_ms", None)
            self.profile = self.ctx.profile(self.trace.iterations)
            if host is not None:
                self.profile["host_ms"] = host
        return self.profile


def solve_device(D, config: SolverConfig, observer=None, *, device=None, compute_dtype=None,
                 colmajor="auto", fetch_factors=True, profile=False, overlap=None) -> DeviceResult:
    """Run the loop on the device; results stay on the device (see solve).

    The returned DeviceResult reads its strips/core from the cached library
    context, and with fetch_factors=True its `handle` holds zero-copy views
    of the context's final factors: both stay valid until the next solve on
    the same context (same device, shape, dtype and stream).  Pass
    fetch_factors="copy" for private factor tensors.  profile=True reads the
    per-kernel event times into result.profile; profile="deferred" records
    the events but leaves the read-back to result.read_profile(), keeping
    it out of the caller's timed region.  overlap: None = the library
    default (the overlapped loop where eligible), False = the sequential loop
    (concurrent solves sharing one GPU), True = overlapped where eligible.
    """
    leases: list = []
    try:
        return _solve_device(D, config, observer, device=device, compute_dtype=compute_dtype, colmajor=colmajor,
                             fetch_factors=fetch_factors, profile=profile, overlap=overlap, _leases=leases)
    finally:
        for c in leases:
            _release(c)


def _solve_device(D, config: SolverConfig, observer=None, *, device=None, compute_dtype=None,
                  colmajor="auto", fetch_factors=True, profile=False, overlap=None,
                  _leases=None) -> DeviceResult:
    """See solve_device."""
    cfg = config
    tick = _Ticker(profile)
    src = _host_source(D, device, compute_dtype) if torch.cuda.is_available() else None
    if src is not None:  # host D: allocate here, stream the rows in under the prep pass
        Dh, want = src
        Dd = torch.empty(tuple(Dh.shape), dtype=want,
                         device=torch.device("cuda", device if device is not None else torch.cuda.current_device()))
    else:
        Dh = None
        Dd = _device_matrix(D, device, compute_dtype)
    if Dd.numel() == 0:
        raise ValueError("D must be nonempty")
    n1, n2 = int(Dd.shape[0]), int(Dd.shape[1])
    dev = Dd.device.index
    dtype = _capi.F32 if Dd.dtype == torch.float32 else _capi.F64
    m_rows = sample_count(n1, cfg.rank, cfg.c_rows)
    m_cols = sample_count(n2, cfg.rank, cfg.c_cols)
    resampled = cfg.mode == "resampled"
    n_sets = cfg.max_iter if resampled else 1
    pcg = pcg_words(cfg.seed) if max(n1, n2) <= 2**32 else None
    code = _native_copy_code(colmajor, n2, m_cols, cfg) if (Dh is None and observer is None and pcg is not None
                                                           and profile in (False, "deferred")) else None
    if code is not None:  # the whole host sequence in one library call (ircur_solve)
        stream = torch.cuda.current_stream(dev).cuda_stream
        ctx = _context(dev, dtype, n1, n2, cfg.rank, m_rows, m_cols, cfg.max_iter, stream)
        _leases.append(ctx)
        ctx.set_profiling(bool(profile))
        ctx.set_overlap(overlap)
        return _solve_native(ctx, Dd, cfg, pcg, code, fetch_factors, dtype, n1, n2, m_rows, m_cols, profile)
    # Draw the sets the prep pass needs first; the rest of the sequence is
    # drawn by a worker thread while the (host-blocking) prep pass runs.
    n_first = min(n_sets, _cover_sets(cfg)) if resampled else n_sets
    if pcg is None:
        sets, pcg_next = draw_index_sets(n1, n2, m_rows, m_cols, cfg.seed, n_sets), None
        n_first = n_sets
    else:
        sets, pcg_next = draw_index_sets_from(pcg, n1, n2, m_rows, m_cols, n_first)
    tick("draw")
    stream = torch.cuda.current_stream(dev).cuda_stream
    ctx = _context(dev, dtype, n1, n2, cfg.rank, m_rows, m_cols, cfg.max_iter, stream)
    _leases.append(ctx)
    ctx.set_profiling(bool(profile))
    ctx.set_overlap(overlap)
    ctx.set_indices(sets)
    tick("set_indices")
    cm, cover = _copy_plan(colmajor, n2, m_cols, sets, cfg)
    rest = None
    if n_first < n_sets:
        import threading

        box = {}
        worker = threading.Thread(target=lambda: box.update(
            r=draw_index_sets_from(pcg_next, n1, n2, m_rows, m_cols, n_sets - n_first)[0]))
        worker.start()
    try:
        # the pass over D runs while the host draws and uploads the tail of
        # the index sequence and queues the den == 0 check
        if Dh is not None:
            _stream_in(Dh, Dd, ctx, cm, cover)
        else:
            ctx.prepare_async(Dd, cm, cover)
    finally:
        if n_first < n_sets:
            worker.join()
            rest = box["r"]
    if rest is not None:
        ctx.append_indices(rest)
        sets.extend_drawn(rest)
    ctx.slab_sqnorms_async(0)
    tick("queue")
    max_abs = ctx.prepare_wait()  # ValueError on NaN/Inf (matcore.py:75-76)
    tick("prepare")
    a, b = ctx.slab_sqnorms(0)
    tick("slab")
    rows0, cols0 = sets[0]
    trace = SolverTrace()
    if np.sqrt(a) + np.sqrt(b) == 0.0:
        # solver.py:335-341: sampled slabs identically zero
        trace.errors.append(0.0)
        trace.converged = True
        return DeviceResult(trace, cfg, None, IndexSet(rows0, n1), IndexSet(cols0, n2), None, True)
    if cfg.zeta0 is None:
        cfg = replace(cfg, zeta0=max_abs)  # solver.py:342-344
    zetas = [cfg.gamma**k * cfg.zeta0 for k in range(cfg.max_iter)]
    mode = _capi.RESAMPLED if resampled else _capi.FIXED
    prof = None
    if observer is None:
        iters, conv, errors, ms = ctx.run(zetas, cfg.eps, mode, cfg.max_iter)
        tick("run")
        if profile and profile != "deferred":
            prof = ctx.profile(iters)
            tick("profile")
        trace.errors = [float(e) for e in errors]
        trace.seconds = [float(t) / 1e3 for t in ms]
    else:
        iters, conv = 0, False
        ctx.set_target_eps(cfg.eps)
        for k in range(cfg.max_iter):
            s = k if resampled else 0
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record()
            e = ctx.iterate(k, s, zetas[k])
            ev1.record()
            ev1.synchronize()
            iters = k + 1
            trace.errors.append(float(e))
            trace.seconds.append(ev0.elapsed_time(ev1) / 1e3)
            cur, sparse = _host_results(ctx, s, n1, n2, None)
            observer(k + 1, zetas[k], cur, sparse, float(e))
            if e <= cfg.eps:
                conv = True
                break
    trace.iterations = iters
    trace.converged = conv
    trace.thresholds = zetas[:iters]
    trace.allocated = [0] * iters
    last = (iters - 1) if resampled else 0
    trace.sampled_rows = [int(sets[k if resampled else 0][0].size) for k in range(iters)]
    trace.sampled_cols = [int(sets[k if resampled else 0][1].size) for k in range(iters)]
    I, J = sets[last]
    handle = None
    if fetch_factors:
        # zero-copy views into the context (valid until its next solve);
        # fetch_factors="copy" returns private tensors instead
        Pt, Qt = ctx.factors() if fetch_factors == "copy" else ctx.factor_views()
        handle = DeviceHandle(Pt, Qt, dtype)
        tick("factors")
    res = DeviceResult(trace, cfg, ctx, IndexSet(I, n1), IndexSet(J, n2), handle)
    if prof is not None:
        prof["host_ms"] = tick.marks
    res.profile = prof
    res._host_ms = tick.marks if profile else None
    res.colmajor = cm
    res.sets = sets
    return res


def _native_copy_code(colmajor, n2: int, m_cols: int, cfg: SolverConfig):
    """_copy_plan's rule as an ircur_solve code (0 none, 1 full, 2 sampled,
    3 by the covered-column share), or None for the forms only the Python
    sequence handles (IRCUR_COLMAJOR / IRCUR_NATIVE=0 overrides, "sampled:K")."""
    if os.environ.get("IRCUR_COLMAJOR") is not None or os.environ.get("IRCUR_NATIVE", "1") == "0":
        return None
    if colmajor in (False, 0, "0", "false", "False", "none", ""):
        return 0
    if colmajor == "auto" and not _want_colmajor("auto", 0, n2, m_cols, 0, cfg.mode):
        return 0
    if colmajor in ("full", 1) and colmajor is not True:
        return 1
    if cfg.mode == "fixed" and colmajor in ("sampled", True, "auto"):
        return 2 if colmajor == "sampled" else 3
    if colmajor == "sampled":
        return 2
    if colmajor is True or colmajor == "auto":
        return 3
    return None


def _solve_native(ctx: Context, Dd: torch.Tensor, cfg: SolverConfig, pcg, code: int, fetch_factors, dtype: int,
                  n1: int, n2: int, m_rows: int, m_cols: int, profile) -> DeviceResult:
    """solve_device through ircur_solve: draws, copy plan, prep pass, den
    check, schedule and loop run in the library (no interpreter work per
    phase, so several host threads can drive independent problems)."""
    resampled = cfg.mode == "resampled"
    n_sets = cfg.max_iter if resampled else 1
    rows = np.empty((n_sets, m_rows), dtype=np.int64)
    cols = np.empty((n_sets, m_cols), dtype=np.int64)
    rc = np.zeros(n_sets, dtype=np.int32)
    cc = np.zeros(n_sets, dtype=np.int32)
    errors = np.zeros(max(cfg.max_iter, 1), dtype=np.float64)
    ms = np.zeros(max(cfg.max_iter, 1), dtype=np.float32)
    it, conv, cm, zs = C.c_int(0), C.c_int(0), C.c_int(0), C.c_int(0)
    z0 = C.c_double(0.0)
    p64, p32 = C.POINTER(C.c_int64), C.POINTER(C.c_int32)
    ctx._D = Dd
    _capi.check(ctx.lib.ircur_solve(
        ctx.h, C.c_void_p(_ptr(Dd)), Dd.stride(0), pcg.ctypes.data_as(C.POINTER(C.c_uint64)),
        float(cfg.zeta0) if cfg.zeta0 is not None else -1.0, float(cfg.gamma), float(cfg.eps),
        _capi.RESAMPLED if resampled else _capi.FIXED, cfg.max_iter, code, rows.ctypes.data_as(p64),
        rc.ctypes.data_as(p32), cols.ctypes.data_as(p64), cc.ctypes.data_as(p32), C.byref(it), C.byref(conv),
        errors.ctypes.data_as(C.POINTER(C.c_double)), ms.ctypes.data_as(C.POINTER(C.c_float)), C.byref(z0),
        C.byref(cm), C.byref(zs)))
    sets = DrawnSets([(rows[k, :rc[k]], cols[k, :cc[k]]) for k in range(n_sets)], rows, rc, cols, cc)
    ctx.sets = sets
    ctx.colmajor = cm.value
    trace = SolverTrace()
    if zs.value:  # solver.py:335-341: sampled slabs identically zero
        trace.errors.append(0.0)
        trace.converged = True
        r0, c0 = sets[0]
        return DeviceResult(trace, cfg, None, IndexSet(r0, n1), IndexSet(c0, n2), None, True)
    if cfg.zeta0 is None:
        cfg = replace(cfg, zeta0=z0.value)  # solver.py:342-344
    iters = it.value
    zetas = [cfg.gamma**k * cfg.zeta0 for k in range(iters)]
    trace.errors = [float(e) for e in errors[:iters]]
    trace.seconds = [float(t) / 1e3 for t in ms[:iters]]
    trace.iterations = iters
    trace.converged = bool(conv.value)
    trace.thresholds = zetas
    trace.allocated = [0] * iters
    trace.sampled_rows = [int(rc[k if resampled else 0]) for k in range(iters)]
    trace.sampled_cols = [int(cc[k if resampled else 0]) for k in range(iters)]
    I, J = sets[(iters - 1) if resampled else 0]
    handle = None
    if fetch_factors:
        Pt, Qt = ctx.factors() if fetch_factors == "copy" else ctx.factor_views()
        handle = DeviceHandle(Pt, Qt, dtype)
    res = DeviceResult(trace, cfg, ctx, IndexSet(I, n1), IndexSet(J, n2), handle)
    res.profile = None
    res._host_ms = None
    res.colmajor = cm.value
    res.sets = sets
    if profile and profile != "deferred":
        res.read_profile()
    return res


def _host_results(ctx: Context, set_idx: int, n1: int, n2: int, handle):
    I, J = ctx.sets[set_idx]
    Cm, Rm, Sr, Sc = ctx.strips(set_idx)
    W, s, V, inv = ctx.core()
    rows, cols = IndexSet(I, n1), IndexSet(J, n2)
    cur = CurFactors(C=Cm, core_pinv=PinvFactor(W=W, sigma=s, V=V, inv_sigma=inv), R=Rm, rows=rows,
                     cols=cols, device=handle)
    return cur, SparseEstimate(Sr, Sc, rows, cols)


def _zero_results(n1, n2, rows: IndexSet, cols: IndexSet, rank: int):
    """_zero_state (solver.py:283-301): L_0 = 0, S_0 = 0 in factor form."""
    m, n = rows.size, cols.size
    k = min(rank, m, n)
    W = np.eye(m, k)
    V = np.eye(n, k)
    z = np.zeros(k)
    cur = CurFactors(C=np.zeros((n1, n)), core_pinv=PinvFactor(W, z.copy(), V, z.copy()),
                     R=np.zeros((m, n2)), rows=rows, cols=cols, device=None)
    return cur, SparseEstimate(np.zeros((m, n2)), np.zeros((n1, n)), rows, cols)


def solve(D, config: SolverConfig, observer=None, *, device=None, compute_dtype=None,
          colmajor="auto", overlap=None):
    """Drop-in for ircur.solver.solve (solver.py:304-416).

    Returns (CurFactors, SparseEstimate, SolverTrace) with float64 host
    arrays.  Extra keyword arguments (not in the reference): `device` (CUDA
    ordinal), `compute_dtype` (torch dtype; default keeps fp32 input in fp32
    and runs everything else in fp64) and `colmajor` (build the column-major
    copy of D used by the column-strip kernel: True/False/"auto") and
    `overlap` (loop selection, see solve_device).
    """
    leases: list = []  # the context stays leased until its results are read back
    try:
        res = _solve_device(D, config, observer, device=device, compute_dtype=compute_dtype,
                            colmajor=colmajor, fetch_factors="copy", overlap=overlap, _leases=leases)
        n1, n2 = res.rows.bound, res.cols.bound
        if res.zero_state:
            cur, sparse = _zero_results(n1, n2, res.rows, res.cols, config.rank)
            return cur, sparse, res.trace
        last = (res.trace.iterations - 1) if res.cfg.mode == "resampled" else 0
        cur, sparse = _host_results(res.ctx, last, n1, n2, res.handle)
        return cur, sparse, res.trace
    finally:
        for c in leases:
            _release(c)


_BATCH_POOL: list = []  # contexts of the batched path, reused across calls of the same shape


def _batchable(Ds, configs) -> bool:
    if not Ds or os.environ.get("IRCUR_BATCHED", "1") == "0":
        return False
    c0 = configs[0]
    shape = tuple(Ds[0].shape)
    for D, c in zip(Ds, configs):
        dt = D.dtype if isinstance(D, torch.Tensor) else np.asarray(D).dtype
        if dt not in (np.float32, torch.float32) or tuple(D.shape) != shape or len(shape) != 2:
            return False
        if (c.rank, c.mode, c.max_iter, c.c_rows, c.c_cols) != (c0.rank, c0.mode, c0.max_iter, c0.c_rows, c0.c_cols):
            return False
        if c.rank > 16 or max(shape) > 2**32:
            return False
    return True


_PCG_CACHE: dict = {}


def _pcg_cached(seed):
    """pcg_words of a RngSeed (cached: a batch reuses the same seeds)."""
    key = (type(seed).__name__, getattr(seed, "seed", None), getattr(seed, "stream", None))
    w = _PCG_CACHE.get(key) if key[1] is not None else None
    if w is None:
        w = pcg_words(seed)
        if w is None:
            raise ValueError("batched problems need PCG64 seeds")
        if key[1] is not None and len(_PCG_CACHE) < 100000:
            _PCG_CACHE[key] = w
    return w


def solve_batch_device(Ds, configs, *, device=None, svd_cs: int = 0, colmajor="auto", stats=None):
    """Independent fp32 problems of one shape and schedule (BASELINE.json cfg4;
    the reference's trial pool, cli.py:117-125) solved together: every
    problem's host sequence (draws, copy plan, prep pass, den check) runs in
    the library, then ircur_batched_run issues ONE launch per phase per
    iteration over all of them (core, Gram + SVD with one cluster per
    problem, strips, stop test).  Each problem's results equal its own
    sequential solve with the same SVD cluster size (IRCUR_SVD_CS = svd_cs;
    0 = the smallest that fits).  Returns a DeviceResult per problem."""
    import concurrent.futures as cf
    import time as _time

    t_start = _time.perf_counter()
    dev = device if device is not None else torch.cuda.current_device()
    n = len(Ds)
    c0 = configs[0]
    Dds = [_device_matrix(D, dev, torch.float32) for D in Ds]
    n1, n2 = int(Dds[0].shape[0]), int(Dds[0].shape[1])
    m_rows = sample_count(n1, c0.rank, c0.c_rows)
    m_cols = sample_count(n2, c0.rank, c0.c_cols)
    resampled = c0.mode == "resampled"
    n_sets = c0.max_iter if resampled else 1
    main = torch.cuda.current_stream(dev)
    stream = main.cuda_stream
    # the per-problem host sequences (draws, prep pass, den check: host syncs)
    # run on `workers` threads, each with its own stream and contexts
    workers = max(1, min(int(os.environ.get("IRCUR_BATCH_PREP_THREADS", "16")), n))
    key = (dev, n1, n2, c0.rank, m_rows, m_cols, c0.max_iter)
    with _CACHE_LOCK:
        pool = [c for c in _BATCH_POOL if c._key == key]
        wstreams = []
        for c in pool:
            if c._wstream not in wstreams:
                wstreams.append(c._wstream)
        while len(wstreams) < workers:
            wstreams.append(torch.cuda.Stream(device=dev))
        while len(pool) < n:
            w = len(pool) % workers
            ctx = Context(dev, _capi.F32, n1, n2, c0.rank, m_rows, m_cols, c0.max_iter,
                          stream=wstreams[w].cuda_stream)
            ctx._key = key
            ctx._wstream = wstreams[w]
            _BATCH_POOL.append(ctx)
            pool.append(ctx)
    ctxs = pool[:n]
    ready = torch.cuda.Event()
    ready.record(main)  # the problems' device copies are ordered before every prep pass
    for ws in {id(c._wstream): c._wstream for c in ctxs}.values():
        ws.wait_event(ready)
    p64, p32 = C.POINTER(C.c_int64), C.POINTER(C.c_int32)
    pd = C.POINTER(C.c_double)
    pi = C.POINTER(C.c_int)
    out = [None] * n
    preps = [None] * n
    # every problem's host sequence (draws, copy plan, prep pass, den check)
    # in one library call, on `workers` library threads
    rows = np.empty((n, n_sets, m_rows), dtype=np.int64)
    cols = np.empty((n, n_sets, m_cols), dtype=np.int64)
    rc = np.zeros((n, n_sets), dtype=np.int32)
    cc = np.zeros((n, n_sets), dtype=np.int32)
    pcg = np.stack([_pcg_cached(c.seed) for c in configs])
    z0in = np.array([float(c.zeta0) if c.zeta0 is not None else -1.0 for c in configs])
    gam = np.array([float(c.gamma) for c in configs])
    eps = np.array([float(c.eps) for c in configs])
    z0 = np.zeros(n)
    cm = np.zeros(n, dtype=np.int32)
    zs = np.zeros(n, dtype=np.int32)
    dptr = (C.c_void_p * n)(*[_ptr(Dd) for Dd in Dds])
    harr = (C.c_void_p * n)(*[c.h.value for c in ctxs])
    for ctx, Dd in zip(ctxs, Dds):
        ctx._D = Dd
    code = _native_copy_code(colmajor, n2, m_cols, c0)
    failed = C.c_int(-1)
    t_setup = _time.perf_counter()
    _capi.check(_capi.load().ircur_batch_prepare_many(
        harr, n, dptr, Dds[0].stride(0), pcg.ctypes.data_as(C.POINTER(C.c_uint64)), z0in.ctypes.data_as(pd),
        gam.ctypes.data_as(pd), eps.ctypes.data_as(pd), _capi.RESAMPLED if resampled else _capi.FIXED,
        c0.max_iter, 3 if code is None else code, rows.ctypes.data_as(p64), rc.ctypes.data_as(p32),
        cols.ctypes.data_as(p64), cc.ctypes.data_as(p32), z0.ctypes.data_as(pd), cm.ctypes.data_as(pi),
        zs.ctypes.data_as(pi), workers, C.byref(failed)))
    for i in range(n):
        cfg, ctx = configs[i], ctxs[i]
        sets = LazyDrawnSets(rows[i], rc[i], cols[i], cc[i])
        ctx.sets = sets
        ctx.colmajor = int(cm[i])
        if zs[i]:  # solver.py:335-341
            tr = SolverTrace()
            tr.errors.append(0.0)
            tr.converged = True
            r0, c_0 = sets[0]
            out[i] = DeviceResult(tr, cfg, None, IndexSet(r0, n1), IndexSet(c_0, n2), None, True)
            continue
        if cfg.zeta0 is None:
            cfg = replace(cfg, zeta0=float(z0[i]))
        preps[i] = (i, ctx, cfg, sets, int(cm[i]))
    live = [x for x in preps if x is not None]
    t_prep = _time.perf_counter()
    if live:
        nl = len(live)
        arr = (C.c_void_p * nl)(*[c.h.value for _, c, _, _, _ in live])
        its = np.zeros(nl, dtype=np.int32)
        cvs = np.zeros(nl, dtype=np.int32)
        errs = np.zeros((nl, c0.max_iter), dtype=np.float64)
        sms = C.c_float(0.0)
        _capi.check(_capi.load().ircur_batched_run(arr, nl, C.c_void_p(stream), int(svd_cs),
                                                   its.ctypes.data_as(C.POINTER(C.c_int)),
                                                   cvs.ctypes.data_as(C.POINTER(C.c_int)),
                                                   errs.ctypes.data_as(C.POINTER(C.c_double)), c0.max_iter,
                                                   C.byref(sms) if stats is not None else None))
        if stats is not None:
            stats["strip_ms"] = float(sms.value)
            stats["prepare_s"] = t_prep - t_start
            stats["batched_run_s"] = _time.perf_counter() - t_prep
        for j, (i, ctx, cfg, sets, cmv) in enumerate(live):
            iters = int(its[j])
            tr = SolverTrace()
            tr.errors = [float(e) for e in errs[j, :iters]]
            tr.seconds = [0.0] * iters
            tr.iterations = iters
            tr.converged = bool(cvs[j])
            tr.thresholds = [cfg.gamma**k * cfg.zeta0 for k in range(iters)]
            tr.allocated = [0] * iters
            rcs, ccs = sets.row_counts, sets.col_counts
            tr.sampled_rows = [int(rcs[k if resampled else 0]) for k in range(iters)]
            tr.sampled_cols = [int(ccs[k if resampled else 0]) for k in range(iters)]
            I, J = sets[(iters - 1) if resampled else 0]
            res = DeviceResult(tr, cfg, ctx, IndexSet(I, n1), IndexSet(J, n2), _LazyDeviceHandle(ctx, _capi.F32))
            res.profile = None
            res._host_ms = None
            res.colmajor = cmv
            res.sets = sets
            out[i] = res
        if stats is not None:
            stats["results_s"] = _time.perf_counter() - t_prep - stats["batched_run_s"]
    if stats is not None:
        stats["setup_s"] = t_setup - t_start
    return out


def solve_batch(Ds, configs, *, device=None, streams: int = 4, compute_dtype=None, colmajor="auto",
                batched=None, svd_cs: int = 0):
    """Independent problems (BASELINE.json cfg4: 512 x 2000^2).

    fp32 problems of one shape and schedule go through the batched path
    (solve_batch_device: one launch per phase per iteration over all of
    them); anything else is solved concurrently by `streams` host threads,
    each driving its own CUDA stream and library context.  Returns the list
    of (CurFactors, SparseEstimate, SolverTrace) in input order."""
    import concurrent.futures as cf

    global _CACHE_MAX
    Ds = list(Ds)
    configs = list(configs) if isinstance(configs, (list, tuple)) else [configs] * len(Ds)
    if len(configs) != len(Ds):
        raise ValueError("need one config per problem")
    dev = device if device is not None else torch.cuda.current_device()
    if (batched if batched is not None else True) and compute_dtype in (None, torch.float32) and \
            _batchable(Ds, configs):
        res = solve_batch_device(Ds, configs, device=dev, svd_cs=svd_cs, colmajor=colmajor)
        outs = []
        for r_ in res:
            n1, n2 = r_.rows.bound, r_.cols.bound
            if r_.zero_state:
                cur, sparse = _zero_results(n1, n2, r_.rows, r_.cols, r_.cfg.rank)
            else:
                last = (r_.trace.iterations - 1) if r_.cfg.mode == "resampled" else 0
                cur, sparse = _host_results(r_.ctx, last, n1, n2, r_.handle)
            outs.append((cur, sparse, r_.trace))
        return outs
    nstreams = max(1, min(streams, len(Ds)))
    pool_streams = [torch.cuda.Stream(device=dev) for _ in range(nstreams)]
    with _CACHE_LOCK:
        _CACHE_MAX = max(_CACHE_MAX, nstreams + 2)
    out = [None] * len(Ds)

    def worker(w):
        st = pool_streams[w]
        with torch.cuda.device(dev), torch.cuda.stream(st):
            for i in range(w, len(Ds), nstreams):
                # the sequential loop: the overlapped one sizes its strip grid for a GPU of its own
                out[i] = solve(Ds[i], configs[i], device=dev, compute_dtype=compute_dtype, colmajor=colmajor,
                               overlap=False)
            st.synchronize()

    with cf.ThreadPoolExecutor(nstreams) as ex:
        list(ex.map(worker, range(nstreams)))
    return out


# ------------------------------------------------------------ materialise
def materialize_device(cur_or_handle, out_dtype=torch.float64) -> torch.Tensor:
    """Full L = C U^+ R = P Q streamed by the K=rank writer (solver.py:211-213)."""
    h = cur_or_handle.device if isinstance(cur_or_handle, CurFactors) else cur_or_handle
    if h is None:
        raise ValueError("CurFactors carry no device factors (zero state or foreign object)")
    lib = _capi.load()
    r, n1 = h.Pt.shape
    n2 = h.Qt.shape[1]
    L = torch.empty((n1, n2), dtype=out_dtype, device=h.Pt.device)
    od = _capi.F32 if out_dtype == torch.float32 else _capi.F64
    stream = torch.cuda.current_stream(h.Pt.device).cuda_stream
    _capi.check(lib.ircur_materialize_factors(C.c_void_p(_ptr(h.Pt)), h.Pt.stride(0),
                                              C.c_void_p(_ptr(h.Qt)), h.Qt.stride(0), n1, n2, r,
                                              h.dtype, C.c_void_p(_ptr(L)), L.stride(0), od,
                                              C.c_void_p(stream)))
    return L


def materialize(cur: CurFactors) -> np.ndarray:
    """Dense L as a float64 host array (test scale), like the reference."""
    if cur.device is None:
        if not cur.C.any() and not cur.R.any():
            return np.zeros(cur.shape)
        raise ValueError("CurFactors carry no device factors")
    return materialize_device(cur, torch.float64).cpu().numpy()


def nccl_unique_id(n: int = 1) -> bytes:
    """n NCCL unique ids (128 bytes each) for Context.shard_comm_init."""
    buf = C.create_string_buffer(128 * n)
    _capi.check(_capi.load().ircur_nccl_unique_id(buf, 128 * n))
    return buf.raw

