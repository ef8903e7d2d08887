"""Video background / foreground separation outputs on the device
(reference: cli.py:185-230 run_video, mio.py:160-200 frame helpers).

D holds one frame per column, pixel (x, y) at row y + x * height (the
reference's frames_to_matrix layout).  After a solve, `video_frames`
evaluates L(:, t) = P Q(:, t) for a chunk of frames, the foreground
|D - L| rescaled per frame to [0, 255] (cli.py:224-227), and returns both as
uint8 frames (t, y, x) rounded and clamped like matrix_to_frames
(mio.py:177-187); ircur_video_frames (csrc/video.cu) does the work.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np
import torch

from . import _capi

__all__ = ["frames_to_matrix", "video_frames", "run_video_device", "write_pgm"]


def frames_to_matrix(pixels: np.ndarray) -> np.ndarray:
    """(frames, height, width) -> pixels x frames float64 (mio.py:160-174 layout)."""
    f, h, w = pixels.shape
    return np.ascontiguousarray(pixels.transpose(1, 2, 0).reshape((h * w, f), order="F").astype(np.float64))


def write_pgm(frame: np.ndarray, path) -> None:
    """One (height, width) uint8 frame as binary PGM (P5, maxval 255), mio.py:190-200."""
    frame = np.asarray(frame, dtype=np.uint8)
    h, w = frame.shape
    with open(path, "wb") as fh:
        fh.write(f"P5\n{w} {h}\n255\n".encode("ascii"))
        fh.write(frame.tobytes(order="C"))


def video_frames(D: torch.Tensor, handle, height: int, width: int, start: int, stop: int):
    """uint8 (background, foreground) frames [start, stop) as host arrays (t, y, x)."""
    if D.dtype != handle.Pt.dtype:
        raise ValueError("D and the factors must have the same dtype")
    n1, n2 = D.shape
    if n1 != height * width:
        raise ValueError(f"matrix with {n1} rows does not match {width}x{height} frames")
    if not 0 <= start <= stop <= n2:
        raise ValueError("frame range out of bounds")
    nt = stop - start
    dev = D.device
    bg = torch.empty((nt, height, width), dtype=torch.uint8, device=dev)
    fg = torch.empty((nt, height, width), dtype=torch.uint8, device=dev)
    peaks = torch.empty(max(nt, 1), dtype=torch.int64, device=dev)
    dt = _capi.F32 if D.dtype == torch.float32 else _capi.F64
    stream = torch.cuda.current_stream(dev).cuda_stream
    _capi.check(_capi.load().ircur_video_frames(
        C.c_void_p(handle.Pt.data_ptr()), handle.Pt.stride(0), C.c_void_p(handle.Qt.data_ptr()),
        handle.Qt.stride(0), C.c_void_p(D.data_ptr()), D.stride(0), dt, n1, height, width, start, nt,
        handle.Pt.shape[0], C.c_void_p(peaks.data_ptr()), C.c_void_p(bg.data_ptr()), C.c_void_p(fg.data_ptr()),
        C.c_void_p(stream)))
    return bg.cpu().numpy(), fg.cpu().numpy()


def run_video_device(D, config, height: int, width: int, *, chunk: int = 100, out_dir=None, device=None):
    """run_video (cli.py:185-230) from the frames matrix: solve, then write
    background/ foreground PGM frames per chunk when out_dir is given.
    Returns (trace, background, foreground) with the frames as uint8 arrays
    (all frames when out_dir is None)."""
    from .solver import _device_matrix, solve_device

    Dd = _device_matrix(D, device, None)
    res = solve_device(Dd, config, fetch_factors="copy")
    n_frames = Dd.shape[1]
    bgs, fgs = [], []
    for s in range(0, n_frames, chunk):
        e = min(s + chunk, n_frames)
        bg, fg = video_frames(Dd, res.handle, height, width, s, e)
        if out_dir is not None:
            bdir, fdir = Path(out_dir) / "background", Path(out_dir) / "foreground"
            bdir.mkdir(parents=True, exist_ok=True)
            fdir.mkdir(parents=True, exist_ok=True)
            for t in range(s, e):
                write_pgm(bg[t - s], bdir / f"frame_{t:05d}.pgm")
                write_pgm(fg[t - s], fdir / f"frame_{t:05d}.pgm")
        else:
            bgs.append(bg)
            fgs.append(fg)
    if out_dir is not None:
        return res.trace, None, None
    return res.trace, np.concatenate(bgs), np.concatenate(fgs)
