"""ctypes binding of libircur_b200.so (the C-ABI in include/ircur_b200.h).

This is the "thin C-ABI/ctypes layer" of the design: plain pointers and
sizes cross it, no torch types.  Errors come back as negative status codes
plus ircur_last_error() and are mapped to the exceptions the reference
raises (ValueError for bad input, matcore.py:70-77 / solver.py:320-321).

There is no fallback: if the shared library is missing or fails to load,
every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libircur_b200.so")

OK, EINVAL, ENONFINITE, ECUDA, ENCCL, ENOMEM, EEMPTY = 0, -1, -2, -3, -4, -5, -6
F32, F64 = 0, 1
FIXED, RESAMPLED = 0, 1
SHARD_CORE, SHARD_FACTOR, SHARD_RESID, SHARD_STOP = 0, 1, 2, 3

# (name, restype, argtypes) — mirrors include/ircur_b200.h one to one.
_vp, _i, _i64, _d = C.c_void_p, C.c_int, C.c_int64, C.c_double
_pi, _pd, _pf, _pi64, _pu64 = (C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_float),
                               C.POINTER(C.c_int64), C.POINTER(C.c_uint64))
PROTOTYPES = [
    ("ircur_abi_version", _i, []),
    ("ircur_last_error", C.c_char_p, []),
    ("ircur_ctx_create", _i, [C.POINTER(_vp), _i, _i, _i64, _i64, _i, _i, _i, _i, _i64, _i64, _vp]),
    ("ircur_ctx_destroy", _i, [_vp]),
    ("ircur_prepare", _i, [_vp, _vp, _i64, _i, _pi, _pd]),
    ("ircur_prepare_sampled", _i, [_vp, _vp, _i64, _i, _pi, _pd]),
    ("ircur_prepare_async", _i, [_vp, _vp, _i64, _i, _i]),
    ("ircur_prepare_rows_async", _i, [_vp, _vp, _i64, _i, _i, _i64, _i64]),
    ("ircur_prepare_wait", _i, [_vp, _pi, _pd]),
    ("ircur_draw_index_sets", _i, [_pu64, _i64, _i64, _i, _i, _i, _pi64, C.POINTER(C.c_int32), _pi64,
                                   C.POINTER(C.c_int32), _pu64]),
    ("ircur_set_indices", _i, [_vp, _i, _pi64, C.POINTER(C.c_int32), _pi64, C.POINTER(C.c_int32)]),
    ("ircur_append_indices", _i, [_vp, _i, _pi64, C.POINTER(C.c_int32), _pi64, C.POINTER(C.c_int32)]),
    ("ircur_slab_sqnorms", _i, [_vp, _i, _pd, _pd]),
    ("ircur_slab_sqnorms_async", _i, [_vp, _i]),
    ("ircur_run", _i, [_vp, _pd, _d, _i, _i, _pi, _pi, _pd, _pf]),
    ("ircur_solve", _i, [_vp, _vp, _i64, _pu64, _d, _d, _d, _i, _i, _i, _pi64, C.POINTER(C.c_int32), _pi64,
                         C.POINTER(C.c_int32), _pi, _pi, _pd, _pf, _pd, _pi, _pi]),
    ("ircur_iterate", _i, [_vp, _i, _i, _d, _pd]),
    ("ircur_shard_buffers", _i, [_vp, C.POINTER(_vp), _pi64, C.POINTER(_vp), _pi64, C.POINTER(_vp)]),
    ("ircur_shard_reset", _i, [_vp]),
    ("ircur_shard_phase", _i, [_vp, _i, _i, _i, _d, _d, _i]),
    ("ircur_poll", _i, [_vp, _pi, _pi]),
    ("ircur_nccl_unique_id", _i, [_vp, _i64]),
    ("ircur_shard_comm_init", _i, [_vp, _vp, _i, _i, _i]),
    ("ircur_shard_pre_chain", _i, [_vp, _vp, _i64, _d, _d, _i, _i]),
    ("ircur_shard_run", _i, [_vp, _pd, _d, _i, _i, _i, _i, _pi, _pi, _pd, _pf, _pi]),
    ("ircur_shard_finish", _i, [_vp, _pd, _i, _pi, _pi, _pd, _pf]),
    ("ircur_get_strips", _i, [_vp, _vp, _vp, _vp, _vp]),
    ("ircur_get_core", _i, [_vp, _vp, _vp, _vp, _vp, _pi, _pi, _pi]),
    ("ircur_get_factors", _i, [_vp, _vp, _vp]),
    ("ircur_factor_buffers", _i, [_vp, C.POINTER(_vp), _pi64, C.POINTER(_vp), _pi64]),
    ("ircur_materialize", _i, [_vp, _vp, _i64, _i]),
    ("ircur_set_profiling", _i, [_vp, _i]),
    ("ircur_get_marks", _i, [_vp, _pf]),
    ("ircur_debug_counter", _i, [_vp, _i, C.POINTER(C.c_longlong)]),
    ("ircur_get_timeline", _i, [_vp, _i, _pf]),
    ("ircur_set_overlap", _i, [_vp, _i]),
    ("ircur_set_target_eps", _i, [_vp, _d]),
    ("ircur_get_profile", _i, [_vp, _i, _pi, C.POINTER(C.c_longlong), _pf, _pf, _pf, _pf]),
    ("ircur_get_svd_steps", _i, [_vp, _i, _pi]),
    ("ircur_get_svd_phase_cycles", _i, [_vp, C.POINTER(C.c_longlong), _i]),
    ("ircur_materialize_factors", _i, [_vp, _i64, _vp, _i64, _i64, _i64, _i, _i, _vp, _i64, _i, _vp]),
    ("ircur_bin_block_to_rowmajor", _i, [_vp, _i64, _i64, _i64, _vp, _i64, _i, _i64, _i64, _i64, _vp, _vp]),
    ("ircur_rowmajor_to_bin_block", _i, [_vp, _i64, _i, _i64, _i64, _vp, _vp]),
    ("ircur_video_frames", _i, [_vp, _i64, _vp, _i64, _vp, _i64, _i, _i64, _i, _i, _i64, _i, _i, _vp, _vp, _vp,
                                _vp]),
    ("ircur_cur_to_factors", _i, [_vp, _i64, _vp, _i64, _vp, _vp, _i64, _i64, _i, _i, _i, _vp, _i64, _vp, _i64,
                              _vp]),
    ("ircur_batch_prepare", _i, [_vp, _vp, _i64, _pu64, _d, _d, _d, _i, _i, _i, _pi64, C.POINTER(C.c_int32), _pi64,
                             C.POINTER(C.c_int32), _pd, _pi, _pi]),
    ("ircur_batch_prepare_many", _i, [_vp, _i, _vp, _i64, _pu64, _pd, _pd, _pd, _i, _i, _i, _pi64,
                                      C.POINTER(C.c_int32), _pi64, C.POINTER(C.c_int32), _pd, _pi, _pi, _i, _pi]),
    ("ircur_batched_run", _i, [_vp, _i, _vp, _i, _pi, _pi, _pd, _i, _pf]),
    ("ircur_factors_to_svd", _i, [_vp, _i64, _vp, _i64, _i64, _i64, _i, _i, _vp, _vp, _vp, _pi, _vp]),
    ("ircur_gen_baseline", _i, [_vp, _i, _i64, _i64, _i64, _i64, _i64, _i, _vp, _vp, _d, _d,
                                _pu64, _pd, _pi64, _vp]),
]

_lib = None


class IrcurError(RuntimeError):
    """A CUDA/NCCL-level failure inside libircur_b200."""


def load() -> C.CDLL:
    """Load (once) and type the shared library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2010_07422_b200._build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in PROTOTYPES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = load().ircur_last_error().decode(errors="replace")
    if rc in (EINVAL, ENONFINITE, EEMPTY):
        raise ValueError(msg)
    if rc == ENOMEM:
        raise MemoryError(msg)
    raise IrcurError(f"libircur_b200 error {rc}: {msg}")


def exported_symbols() -> list[str]:
    return [name for name, _, _ in PROTOTYPES]
