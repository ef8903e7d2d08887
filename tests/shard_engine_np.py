"""Test-only numpy stand-in for a row-sharded libircur_b200 context.

It implements the per-phase contract of include/ircur_b200.h ("Row-sharded
loop") in fp64 numpy, with exchange buffers shaped like the device ones,
so the host orchestration in paper_2010_07422_b200/dist.py (program,
collectives, run-ahead and stop rule, gathers) can be exercised on CPU
with gloo and checked against the oracle.  It is never used by the product
path.  The math follows the device kernels: P = C V Sigma^+ and Q = W_r^T R
with the core overrides P(I,:) = U V Sigma^+ and Q(:,J) = W_r^T U
(reference: solver.py:358-400, matcore.py:128-189).
"""

from __future__ import annotations

import numpy as np
import torch


def _keep(d, l, zeta):
    """c = d - T_zeta(d - l), strict |x| > zeta (solver.py:162-168, 380-382)."""
    x = d - l
    s = np.where(np.abs(x) > zeta, x, 0.0)
    return d - s, s


class NumpyShardEngine:
    def __init__(self, D_local, n1, row0, cfg, m_rows, m_cols):
        self.D = np.asarray(D_local, dtype=np.float64)
        self.n1, self.row0 = n1, row0
        self.nloc, self.n2 = self.D.shape
        self.r = cfg.rank
        self.max_rows, self.max_cols = m_rows, m_cols
        self.ldq = (self.n2 + 3) & ~3
        self._U = torch.zeros(m_rows * m_cols, dtype=torch.float64)
        self._Qp = torch.zeros(self.r * self.ldq, dtype=torch.float64)
        self._scal = torch.zeros(4, dtype=torch.float64)
        self.sets = []

    # ---- setup
    def prepare(self, D, colmajor, cover=0):
        if not np.isfinite(self.D).all():
            raise ValueError("matrix contains non-finite entries")
        return float(np.abs(self.D).max())

    def host_tensor(self, vals):
        return torch.tensor(vals, dtype=torch.float64)

    def set_indices(self, sets):
        self.sets = sets

    def _local(self, s):
        I, J = self.sets[s]
        m = (I >= self.row0) & (I < self.row0 + self.nloc)
        lo = int(np.argmax(m)) if m.any() else 0
        return I[m] - self.row0, lo, J

    def slab_sqnorms(self, s):
        il, _, J = self._local(s)
        return float((self.D[il] ** 2).sum()), float((self.D[:, J] ** 2).sum())

    def shard_reset(self):
        self.P = np.zeros((self.nloc, self.r))
        self.Q = np.zeros((self.r, self.n2))
        self.done = self.iters = self.conv = 0
        self.errors = []

    def shard_buffers(self):
        return self._U, self._Qp, self._scal

    def poll(self):
        return bool(self.done), self.iters

    # ---- phases
    def shard_phase(self, phase, k, s, zeta, eps, max_iter):
        if self.done:
            if phase == 0:
                self._U.zero_()
            return
        il, lo, J = self._local(s)
        I_all = self.sets[s][0]
        mI, nJ, ml = I_all.size, J.size, il.size
        U = self._U.numpy().reshape(self.max_rows, self.max_cols)
        if phase == 0:
            U[:] = 0.0
            c, _ = _keep(self.D[np.ix_(il, J)], self.P[il] @ self.Q[:, J], zeta)
            U[lo:lo + ml, :nJ] = c
        elif phase == 1:
            Uc = U[:mI, :nJ].copy()
            Wf, sig, Vt = np.linalg.svd(Uc, full_matrices=False)
            kk = min(self.r, mI, nJ)
            W, sig, V = Wf[:, :kk], sig[:kk], Vt[:kk].T
            inv = np.zeros(kk)
            if kk and sig[0] > 0:
                keep = sig > 1e-12 * sig[0]
                inv[keep] = 1.0 / sig[keep]
            Wr = np.zeros((mI, self.r)); Wr[:, :kk] = W
            VS = np.zeros((nJ, self.r)); VS[:, :kk] = V * inv
            self.core_f = (W, sig, V, inv)
            self.Wr, self.VS = Wr, VS
            self.PI = Uc @ VS
            self.QJ = (Wr.T @ Uc).T
            # column strip (local rows), complete
            dc = self.D[:, J]
            C, _ = _keep(dc, self.P @ self.Q[:, J], zeta)
            Pn = C @ VS
            Pn[il] = self.PI[lo:lo + ml]
            self.den_c = float((dc ** 2).sum())
            self.res_c = float(((C - Pn @ self.QJ.T) ** 2).sum())
            self.P_new = Pn
            # row strip: local partial sums of Q
            dr = self.D[il]
            R, _ = _keep(dr, self.P[il] @ self.Q, zeta)
            self.R = R
            self.den_r = float((dr ** 2).sum())
            Qp = self._Qp.numpy().reshape(self.r, self.ldq)
            Qp[:] = 0.0
            Qp[:, :self.n2] = Wr[lo:lo + ml].T @ R
        elif phase == 2:
            Qn = self._Qp.numpy().reshape(self.r, self.ldq)[:, :self.n2].copy()
            Qn[:, J] = self.QJ.T
            res_r = float(((self.R - self.PI[lo:lo + ml] @ Qn) ** 2).sum())
            self.Q_new = Qn
            self._scal[:] = torch.tensor([self.den_r, res_r, self.den_c, self.res_c], dtype=torch.float64)
        elif phase == 3:
            d = self._scal.numpy()
            e = (np.sqrt(d[1]) + np.sqrt(d[3])) / (np.sqrt(d[0]) + np.sqrt(d[2]))
            self.errors.append(float(e))
            self.iters = k + 1
            self.last = (s, zeta, self.P, self.Q)  # the L this iteration thresholded against
            self.P, self.Q = self.P_new, self.Q_new
            if e <= eps:
                self.conv = self.done = 1
            elif k + 1 >= max_iter:
                self.done = 1

    def shard_finish(self, zetas, mode):
        n = self.iters
        return n, bool(self.conv), np.array(self.errors[:n]), np.zeros(n, dtype=np.float32)

    # ---- results of the last iteration (ircur_get_strips / ircur_get_core)
    def strips(self, s):
        il, _, J = self._local(s)
        _, zeta, P, Q = self.last
        C, Sc = _keep(self.D[:, J], P @ Q[:, J], zeta)
        R, Sr = _keep(self.D[il], P[il] @ Q, zeta)
        return C, R, Sr, Sc

    def core(self):
        return self.core_f


def numpy_engine(D_local, n1, row0, cfg, m_rows, m_cols, device=None, compute_dtype=None):
    return NumpyShardEngine(D_local, n1, row0, cfg, m_rows, m_cols), D_local
