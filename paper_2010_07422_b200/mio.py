"""BIN matrix files straight into (row-sharded) device memory.

Reference format (mio.py:66-121): magic "IRCM", little-endian int32 rows
and cols, then rows*cols little-endian float64 in column-major order.  The
reference reads the whole file into host memory and returns a float64
array; here column blocks stream through page-locked buffers to the GPU,
where ircur_bin_block_to_rowmajor (csrc/mio.cu) transposes them into the
row-major D the solver uses (optionally only rows [row0, row0 + nrows) for a
row-sharded rank, optionally cast to float32) and looks for the first
non-finite value.  Validation and errors follow the reference's reader:
FormatError (a ValueError) with the byte offset for truncated headers, bad
magic, negative dimensions, truncated payloads, trailing bytes and
non-finite values (the first in file order).
"""

from __future__ import annotations

import ctypes as C
import os
import struct
from pathlib import Path

import numpy as np
import torch

from . import _capi

__all__ = ["BIN_MAGIC", "FormatError", "read_matrix_device", "write_matrix_device", "bin_shape"]

BIN_MAGIC = b"IRCM"
_HDR = struct.Struct("<4sii")
_BLOCK_BYTES = 256 << 20  # staging per column block


class FormatError(ValueError):
    """Malformed matrix file; same message and fields as the reference's
    mio.FormatError (path, byte offset)."""

    def __init__(self, message: str, path=None, offset: int | None = None):
        loc = f"{path}: " if path is not None else ""
        at = f" (byte offset {offset})" if offset is not None else ""
        super().__init__(f"{loc}{message}{at}")
        self.path = path
        self.offset = offset


def bin_shape(path) -> tuple[int, int]:
    """(rows, cols) of a BIN file after the reference's header/size checks."""
    path = Path(path)
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(_HDR.size)
    if len(head) < _HDR.size:
        raise FormatError("truncated header", path=path, offset=len(head))
    magic, rows, cols = _HDR.unpack(head)
    if magic != BIN_MAGIC:
        raise FormatError(f"bad magic {magic!r}", path=path, offset=0)
    if rows < 0 or cols < 0:
        raise FormatError(f"negative dimensions {rows}x{cols}", path=path, offset=4)
    expected = _HDR.size + 8 * rows * cols
    if size < expected:
        raise FormatError(f"truncated payload, expected {expected} bytes", path=path, offset=size)
    if size > expected:
        raise FormatError("trailing bytes after payload", path=path, offset=expected)
    return rows, cols


def read_matrix_device(path, *, dtype=torch.float64, device=None, row0: int = 0, nrows: int | None = None,
                       block_cols: int | None = None) -> torch.Tensor:
    """Rows [row0, row0 + nrows) of a BIN matrix as a row-major CUDA tensor."""
    path = Path(path)
    rows, cols = bin_shape(path)
    nrows = rows - row0 if nrows is None else nrows
    if row0 < 0 or nrows < 0 or row0 + nrows > rows:
        raise ValueError(f"row range [{row0}, {row0 + nrows}) outside 0..{rows}")
    if dtype not in (torch.float32, torch.float64):
        raise ValueError("dtype must be torch.float32 or torch.float64")
    if not torch.cuda.is_available():
        raise RuntimeError("read_matrix_device needs a CUDA device")
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    D = torch.empty((nrows, cols), dtype=dtype, device=dev)
    if nrows == 0 or cols == 0:
        return D
    lib = _capi.load()
    cb = block_cols or max(1, min(cols, _BLOCK_BYTES // (8 * nrows)))
    host = [torch.empty(nrows * cb, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    stage = [torch.empty(nrows * cb, dtype=torch.float64, device=dev) for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    bad = torch.full((1,), -1, dtype=torch.int64, device=dev)  # all ones: "no non-finite value"
    stream = torch.cuda.current_stream(dev)
    dt = _capi.F64 if dtype == torch.float64 else _capi.F32
    contiguous = row0 == 0 and nrows == rows
    with open(path, "rb", buffering=0) as fh:
        for b, j0 in enumerate(range(0, cols, cb)):
            k = b & 1
            nc = min(cb, cols - j0)
            done[k].synchronize()  # the copy out of this host buffer finished
            hv = memoryview(host[k].numpy()).cast("B")
            if contiguous:
                fh.seek(_HDR.size + 8 * j0 * rows)
                fh.readinto(hv[:8 * nrows * nc])
            else:
                for j in range(nc):
                    fh.seek(_HDR.size + 8 * ((j0 + j) * rows + row0))
                    fh.readinto(hv[8 * nrows * j:8 * nrows * (j + 1)])
            stage[k][:nrows * nc].copy_(host[k][:nrows * nc], non_blocking=True)
            done[k].record(stream)
            _capi.check(lib.ircur_bin_block_to_rowmajor(
                C.c_void_p(stage[k].data_ptr()), nrows, nrows, nc,
                C.c_void_p(D.data_ptr() + j0 * D.element_size()), cols, dt, rows, row0, j0,
                C.c_void_p(bad.data_ptr()), C.c_void_p(stream.cuda_stream)))
    first = int(bad.item())
    if first != -1:
        raise FormatError("non-finite value", path=path, offset=_HDR.size + 8 * (first & ((1 << 63) - 1)))
    return D


def write_matrix_device(D: torch.Tensor, path, *, block_cols: int | None = None) -> Path:
    """Write a 2-D CUDA tensor (row-major, fp32/fp64) in the reference's BIN
    format; the values are written as float64 like mio.write_matrix."""
    path = Path(path)
    if D.ndim != 2 or D.stride(1) != 1:
        raise ValueError("expected a 2-D tensor with unit column stride")
    if D.dtype not in (torch.float32, torch.float64):
        raise ValueError("dtype must be float32 or float64")
    rows, cols = D.shape
    lib = _capi.load()
    dev = D.device
    stream = torch.cuda.current_stream(dev)
    cb = block_cols or max(1, min(cols, _BLOCK_BYTES // (8 * max(rows, 1))))
    stage = torch.empty(max(rows, 1) * cb, dtype=torch.float64, device=dev)
    host = torch.empty(max(rows, 1) * cb, dtype=torch.float64, pin_memory=True)
    dt = _capi.F64 if D.dtype == torch.float64 else _capi.F32
    with open(path, "wb") as fh:
        fh.write(_HDR.pack(BIN_MAGIC, rows, cols))
        for j0 in range(0, cols, cb):
            nc = min(cb, cols - j0)
            _capi.check(lib.ircur_rowmajor_to_bin_block(
                C.c_void_p(D.data_ptr() + j0 * D.element_size()), D.stride(0), dt, rows, nc,
                C.c_void_p(stage.data_ptr()), C.c_void_p(stream.cuda_stream)))
            host[:rows * nc].copy_(stage[:rows * nc])
            fh.write(memoryview(host[:rows * nc].numpy()).cast("B"))
    return path
