"""BASELINE.json synthetic problems generated on the device.

Draw-for-draw the same matrix as `oracle.ircur_oracle.baseline_problem`
(numpy PCG64): the Gaussian factors W, V come from numpy on the host (small,
n x r), then the device reproduces the Generator's `random()` mask draws and
`uniform()` value draws by jumping the PCG64 stream to each cell's draw
index (ircur_gen_baseline in csrc/kernels_prep.cu).  That keeps the n = 1e5
configuration (40 GB fp32) bit-identical to what numpy would produce, for
any row sharding.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _capi

M64 = (1 << 64) - 1
Q24 = 16777216.0


def _pcg_words(rng: np.random.Generator) -> np.ndarray:
    st = rng.bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    return np.array([s & M64, s >> 64, inc & M64, inc >> 64], dtype=np.uint64)


def factors(n1: int, n2: int, rank: int, seed: int):
    """Host Gaussian factors + the PCG64 state after drawing them."""
    rng = np.random.default_rng(seed)
    W = rng.standard_normal((n1, rank))
    V = rng.standard_normal((n2, rank))
    return W, V, _pcg_words(rng)


def _call(D, dtype, ldd, n1, n2, row0, nrows, rank, Wd, Vd, alpha, amp_a, pcg, stream):
    lib = _capi.load()
    mx = C.c_double(0.0)
    q = C.c_int64(0)
    _capi.check(lib.ircur_gen_baseline(
        C.c_void_p(D), dtype, ldd, n1, n2, row0, nrows, rank, C.c_void_p(Wd.data_ptr()),
        C.c_void_p(Vd.data_ptr()), alpha, amp_a, pcg.ctypes.data_as(C.POINTER(C.c_uint64)),
        C.byref(mx), C.byref(q), C.c_void_p(stream)))
    return mx.value, q.value


def baseline_problem_device(n1: int, n2: int, rank: int, alpha: float, seed: int,
                            dtype=torch.float32, amp: float = 10.0, device=None,
                            row0: int = 0, nrows: int | None = None, stats_reduce=None):
    """Rows [row0, row0+nrows) of D on the device plus (max|L|, a=mean|L|).

    `stats_reduce(max_abs, qsum) -> (max_abs, qsum)` lets a multi-GPU caller
    combine the per-shard statistics (max and an exact int64 sum) so every
    shard uses the same outlier amplitude.
    """
    nrows = n1 - row0 if nrows is None else nrows
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    W, V, pcg = factors(n1, n2, rank, seed)
    Wd = torch.from_numpy(W).to(dev)
    Vd = torch.from_numpy(V).to(dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    dt = _capi.F32 if dtype == torch.float32 else _capi.F64
    mx, q = _call(None, dt, n2, n1, n2, row0, nrows, rank, Wd, Vd, alpha, 0.0, pcg, stream)
    if stats_reduce is not None:
        mx, q = stats_reduce(mx, q)
    a = float(q) / Q24 / (n1 * n2)
    D = torch.empty((nrows, n2), dtype=dtype, device=dev)
    _call(D.data_ptr(), dt, n2, n1, n2, row0, nrows, rank, Wd, Vd, alpha, amp * a, pcg, stream)
    return D, mx, a


def video_problem(frames: int = 1000, height: int = 144, width: int = 176, rank: int = 2, n_blocks: int = 12,
                  block: int = 16, seed: int = 0, dtype=np.float32):
    """BASELINE.json cfg3: a video-like matrix, one frame per
    column, pixel (x, y) at row y + x * height (the reference's frame
    layout, mio.py:162-174).  Low-rank background = `rank` Gaussian-blurred
    (sigma = 8 px) N(0,1) fields times per-frame weights following random
    walks (step 0.01); sparse foreground = `n_blocks` moving block x block
    squares of U[0.5, 1] intensity with constant velocities |v| <= 3
    px/frame, wrapping at the borders.  Host numpy (a data source for
    parity tests and the cfg3 bench line, not part of the hot path).
    Returns (D, L, S)."""
    from scipy.ndimage import gaussian_filter

    rng = np.random.default_rng(seed)
    fields = np.stack([gaussian_filter(rng.standard_normal((width, height)), sigma=8.0, mode="wrap")
                       for _ in range(rank)])
    fields /= np.abs(fields).max(axis=(1, 2), keepdims=True)
    F = fields.reshape(rank, width * height).T          # row = y + x * height
    w = 1.0 + np.cumsum(0.01 * rng.standard_normal((rank, frames)), axis=1)
    L = F @ w
    S = np.zeros((width * height, frames))
    pos = rng.uniform(0, [width, height], size=(n_blocks, 2))
    ang = rng.uniform(0, 2 * np.pi, n_blocks)
    spd = rng.uniform(0.5, 3.0, n_blocks)
    vel = np.stack([spd * np.cos(ang), spd * np.sin(ang)], axis=1)
    inten = rng.uniform(0.5, 1.0, n_blocks)
    xs = np.arange(block)
    for t in range(frames):
        p = (pos + t * vel)
        for b in range(n_blocks):
            x = (int(p[b, 0]) + xs) % width
            y = (int(p[b, 1]) + xs) % height
            rows = (y[None, :] + x[:, None] * height).ravel()
            S[rows, t] = inten[b]
    D = (L + S).astype(dtype)
    return D, L, S
