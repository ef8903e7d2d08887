"""CUR -> compact SVD (reference: convert.py:21-48, `cur_to_svd` and
`factors_to_svd`), on the device.

The solver's iterate is already held as L = P Q with P = C V Sigma^+ and
Q = W_r^T R (the product C U^+ R of the reference), so the conversion needs
only r-wide work: ircur_factors_to_svd (csrc/convert.cu) takes Cholesky-QR
factors of P and Q^T, the SVD of the r x r middle factor, and applies the
rotations; singular values below 1e-14 sigma_max are dropped like the
reference's COMPACT_DROP.  Results are float64 host arrays (SvdFactors), like
the reference's; W and V are unique up to the sign of each column pair.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _capi
from .types import CurFactors, PinvFactor, SvdFactors

__all__ = ["cur_to_svd", "factors_to_svd", "factors_to_svd_device"]


def factors_to_svd_device(Pt: torch.Tensor, Qt: torch.Tensor):
    """(W, sigma, V) as CUDA fp64 tensors from device factors P^T (r x n1) and
    Q (r x n2), both fp32 or both fp64 with unit column stride."""
    if Pt.dtype != Qt.dtype or Pt.dtype not in (torch.float32, torch.float64):
        raise ValueError("P and Q must both be float32 or float64")
    if Pt.shape[0] != Qt.shape[0] or Pt.stride(1) != 1 or Qt.stride(1) != 1:
        raise ValueError("expected P^T (r x n1) and Q (r x n2) with unit column stride")
    r, n1 = Pt.shape
    n2 = Qt.shape[1]
    dev = Pt.device
    W = torch.empty((n1, r), dtype=torch.float64, device=dev)
    V = torch.empty((n2, r), dtype=torch.float64, device=dev)
    s = torch.empty(r, dtype=torch.float64, device=dev)
    k = C.c_int()
    dt = _capi.F32 if Pt.dtype == torch.float32 else _capi.F64
    stream = torch.cuda.current_stream(dev).cuda_stream
    _capi.check(_capi.load().ircur_factors_to_svd(
        C.c_void_p(Pt.data_ptr()), Pt.stride(0), C.c_void_p(Qt.data_ptr()), Qt.stride(0), n1, n2, r, dt,
        C.c_void_p(W.data_ptr()), C.c_void_p(s.data_ptr()), C.c_void_p(V.data_ptr()), C.byref(k),
        C.c_void_p(stream)))
    kk = k.value
    return W[:, :kk], s[:kk], V[:, :kk]


def cur_to_svd(C_: np.ndarray, core_pinv: PinvFactor, R: np.ndarray, *, device=None) -> SvdFactors:
    """Drop-in for convert.cur_to_svd(C, core_pinv, R) (convert.py:21-48)."""
    C_ = np.asarray(C_)
    R = np.asarray(R)
    if C_.ndim != 2 or R.ndim != 2:
        raise ValueError("C and R must be 2-D matrices")
    if C_.shape[1] != core_pinv.V.shape[0]:
        raise ValueError(f"C has {C_.shape[1]} columns but the core expects {core_pinv.V.shape[0]}")
    if R.shape[0] != core_pinv.W.shape[0]:
        raise ValueError(f"R has {R.shape[0]} rows but the core expects {core_pinv.W.shape[0]}")
    if not torch.cuda.is_available():
        raise RuntimeError("cur_to_svd needs a CUDA device (no CPU fallback)")
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    Cd = torch.from_numpy(np.ascontiguousarray(C_, dtype=np.float64)).to(dev)
    Rd = torch.from_numpy(np.ascontiguousarray(R, dtype=np.float64)).to(dev)
    VS = torch.from_numpy(np.asarray(core_pinv.V, dtype=np.float64) * np.asarray(core_pinv.inv_sigma)).to(dev)
    if VS.shape[1] == 0:
        n1, n2 = C_.shape[0], R.shape[1]
        return SvdFactors(W=np.zeros((n1, 0)), sigma=np.zeros(0), V=np.zeros((n2, 0)))
    n1, nJ = C_.shape
    mI, n2 = R.shape
    kk = VS.shape[1]
    Pt = torch.empty((kk, n1), dtype=torch.float64, device=dev)
    Qt = torch.empty((kk, n2), dtype=torch.float64, device=dev)
    W_ = torch.from_numpy(np.ascontiguousarray(core_pinv.W, dtype=np.float64)).to(dev)
    VS = VS.contiguous()
    stream = torch.cuda.current_stream(dev).cuda_stream
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    # P^T = (C V Sigma^+)^T and Q = W^T R: the library's skinny products
    _capi.check(_capi.load().ircur_cur_to_factors(vp(Cd), nJ, vp(Rd), n2, vp(VS), vp(W_), n1, n2, mI, nJ, kk,
                                                  vp(Pt), n1, vp(Qt), n2, C.c_void_p(stream)))
    W, s, V = factors_to_svd_device(Pt, Qt)
    return SvdFactors(W=W.cpu().numpy(), sigma=s.cpu().numpy(), V=V.cpu().numpy())


def factors_to_svd(cur: CurFactors) -> SvdFactors:
    """Drop-in for convert.factors_to_svd(cur).  Uses the device factors the
    solve returned with `cur` when present (no re-upload of C and R)."""
    h = getattr(cur, "device", None)
    if h is not None:
        W, s, V = factors_to_svd_device(h.Pt, h.Qt)
        return SvdFactors(W=W.cpu().numpy(), sigma=s.cpu().numpy(), V=V.cpu().numpy())
    return cur_to_svd(cur.C, cur.core_pinv, cur.R)
