"""CPU oracle for the IRCUR hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy (float64) restatement of the reference
package's solver loop (`/root/reference/pkg/src/ircur/solver.py`) and the
dense kernels it calls (`matcore.py`), written independently for this repo.
It exists so that the B200 product can be checked against the reference's
algorithm on machines where the reference itself is absent (the GPU box).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it, and only as the checker or as the
timed CPU baseline.  The product package `paper_2010_07422_b200` never
imports it.

Parity pin: `oracle/make_golden.py` runs the real reference (importable in
the build container from /root/reference/pkg/src) on seeded inputs and
commits the results under `tests/golden/`; `tests/test_oracle_golden.py`
checks this restatement against those vectors (bitwise for indices,
thresholds and iteration counts; <=1e-12 relative for the floating-point
outputs, which differ only by BLAS association order).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

PINV_CUTOFF = 1e-12  # matcore.py:22


# --------------------------------------------------------------- sampling
def sample_count(n: int, r: int, c: float) -> int:
    """m = min(n, max(r, ceil(c r ln n)))  — sampling.py:86-90."""
    if n < 1 or r < 1 or c <= 0:
        raise ValueError("need n >= 1, r >= 1, c > 0")
    return min(n, max(r, math.ceil(c * r * math.log(n))))


def seed_generator(seed: int, stream: int = 0) -> np.random.Generator:
    """RngSeed.generator — sampling.py:37-40."""
    return np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(stream,)))


def sample_indices(n: int, m: int, gen: np.random.Generator) -> np.ndarray:
    """With-replacement draws then sort+dedup — sampling.py:93-104."""
    if m < 1 or m > n:
        raise ValueError("need 1 <= m <= n")
    return np.unique(gen.integers(0, n, size=m))


def index_stream(n1, n2, rank, c_rows, c_cols, mode, max_iter, seed, stream=0):
    """Every (I_k, J_k) the reference loop would use, in its draw order:
    rows then cols before the loop (solver.py:325-329), then again at the top
    of every k>0 iteration in resampled mode (solver.py:362-364)."""
    gen = seed_generator(seed, stream)
    m1 = sample_count(n1, rank, c_rows)
    m2 = sample_count(n2, rank, c_cols)
    rows = sample_indices(n1, m1, gen)
    cols = sample_indices(n2, m2, gen)
    out = [(rows, cols)]
    for _ in range(1, max_iter):
        if mode == "resampled":
            rows = sample_indices(n1, m1, gen)
            cols = sample_indices(n2, m2, gen)
        out.append((rows, cols))
    return out


# ------------------------------------------------------------ dense kernels
def hard_threshold(X: np.ndarray, zeta: float) -> np.ndarray:
    """keep x iff |x| > zeta (strict) — solver.py:153-168."""
    if zeta < 0:
        raise ValueError("zeta must be >= 0")
    return np.where(np.abs(X) > zeta, X, 0.0)


def truncated_svd(M: np.ndarray, r: int):
    """Top-min(r, min shape) triplets via LAPACK gesdd — matcore.py:128-139."""
    U, s, Vt = np.linalg.svd(M, full_matrices=False)
    k = min(r, s.size)
    return U[:, :k], s[:k], Vt[:k, :].T


def pinv_inverse(sigma: np.ndarray, rel_cutoff: float = PINV_CUTOFF) -> np.ndarray:
    """1/sigma where sigma > cutoff*sigma_max else 0 — matcore.py:156-165."""
    inv = np.zeros_like(sigma)
    smax = sigma[0] if sigma.size else 0.0
    if smax > 0.0:
        kept = sigma > rel_cutoff * smax
        inv[kept] = 1.0 / sigma[kept]
    return inv


def frob(M: np.ndarray) -> float:
    return float(np.linalg.norm(M, "fro")) if M.size else 0.0  # matcore.py:80-84


@dataclass
class OracleResult:
    C: np.ndarray
    R: np.ndarray
    S_rows: np.ndarray
    S_cols: np.ndarray
    W: np.ndarray
    sigma: np.ndarray
    V: np.ndarray
    inv_sigma: np.ndarray
    rows: np.ndarray
    cols: np.ndarray
    errors: list = field(default_factory=list)
    thresholds: list = field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    sampled_rows: list = field(default_factory=list)
    sampled_cols: list = field(default_factory=list)
    # record_x=True: the pre-threshold strips D - L of the final iteration
    # (the |x| > zeta decisions of solver.py:375-377), for support-flip checks
    X_rows: np.ndarray | None = None
    X_cols: np.ndarray | None = None


def _eval_rows(C, W, V, inv, R, rows):
    # (C[I',:] V diag(inv)) W^T R — solver.py:180-186 / matcore.py:185-189
    t = (C[rows, :] @ V) * inv
    return (t @ W.T) @ R


def _eval_cols(C, W, V, inv, R, cols):
    # C (V diag(inv) (W^T R[:,J'])) — solver.py:189-195 / matcore.py:179-183
    t = (W.T @ R[:, cols]) * inv[:, None]
    return C @ (V @ t)


def solve(D, rank, eps=1e-5, zeta0=None, gamma=0.65, c_rows=4.0, c_cols=4.0,
          mode="fixed", max_iter=200, seed=0, stream=0, upcast=True,
          on_iter=None, record_x=False) -> OracleResult:
    """Algorithm 1 exactly as the reference loop runs it (solver.py:304-416),
    in float64 regardless of D's dtype (matcore.require_finite, :70-77).

    upcast=False keeps a float32 D as is and upcasts each gathered strip
    instead (the same fp64 values; used only to time bounded CPU samples of
    matrices whose fp64 copy would not fit in host memory).  on_iter(k,
    seconds) is called after every iteration; returning True stops the loop
    (bounded timing samples).  record_x keeps the final iteration's
    pre-threshold strips D - L (X_rows, X_cols) for support-flip checks."""
    import time as _time
    if upcast:
        D = np.asarray(D, dtype=np.float64)
    else:
        D = np.asarray(D)
    if D.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    if upcast and not np.isfinite(D).all():
        raise ValueError("matrix contains non-finite entries")
    if D.size == 0:
        raise ValueError("D must be nonempty")
    n1, n2 = D.shape
    f64 = lambda a: np.asarray(a, dtype=np.float64)  # noqa: E731
    sets = index_stream(n1, n2, rank, c_rows, c_cols, mode, max_iter, seed, stream)
    rows, cols = sets[0]
    d_rows = f64(D[rows, :])
    d_cols = f64(D[:, cols])
    den = frob(d_rows) + frob(d_cols)
    res = OracleResult(None, None, None, None, None, None, None, None, rows, cols)
    if den == 0.0:  # solver.py:335-341 / _zero_state :283-301
        k = min(rank, rows.size, cols.size)
        res.C = np.zeros((n1, cols.size)); res.R = np.zeros((rows.size, n2))
        res.S_rows = np.zeros((rows.size, n2)); res.S_cols = np.zeros((n1, cols.size))
        W, s, V = truncated_svd(np.zeros((rows.size, cols.size)), rank)
        res.W, res.sigma, res.V, res.inv_sigma = W, s, V, pinv_inverse(s)
        res.errors = [0.0]
        res.converged = True
        return res
    if zeta0 is None:
        zeta0 = float(max(np.max(D), -np.min(D)))  # inf_norm, matcore.py:87-91
    l_rows = np.zeros((rows.size, n2))
    l_cols = np.zeros((n1, cols.size))
    fac = None
    for k in range(max_iter):
        t0 = _time.perf_counter()
        if mode == "resampled" and k > 0:  # solver.py:362-370
            rows, cols = sets[k]
            d_rows = f64(D[rows, :])
            d_cols = f64(D[:, cols])
            den = frob(d_rows) + frob(d_cols)
            C, W, V, inv, R = fac
            l_rows = _eval_rows(C, W, V, inv, R, rows)
            l_cols = _eval_cols(C, W, V, inv, R, cols)
            l_cols[rows, :] = l_rows[:, cols]
        zeta = gamma ** k * zeta0  # solver.py:372
        x_rows, x_cols = d_rows - l_rows, d_cols - l_cols
        s_rows = hard_threshold(x_rows, zeta)
        s_cols = hard_threshold(x_cols, zeta)
        C = d_cols - s_cols  # solver.py:380-382
        R = d_rows - s_rows
        W, s, V = truncated_svd(R[:, cols], rank)
        inv = pinv_inverse(s)
        fac = (C, W, V, inv, R)
        l_rows = _eval_rows(C, W, V, inv, R, rows)  # solver.py:393-400
        l_cols = _eval_cols(C, W, V, inv, R, cols)
        l_cols[rows, :] = l_rows[:, cols]
        e = (frob(d_rows - l_rows - s_rows) + frob(d_cols - l_cols - s_cols)) / den
        res.errors.append(e)
        res.thresholds.append(zeta)
        res.sampled_rows.append(rows.size)
        res.sampled_cols.append(cols.size)
        res.iterations = k + 1
        res.C, res.R, res.S_rows, res.S_cols = C, R, s_rows, s_cols
        res.W, res.sigma, res.V, res.inv_sigma = W, s, V, inv
        res.rows, res.cols = rows, cols
        if record_x:
            res.X_rows, res.X_cols = x_rows, x_cols
        if e <= eps:
            res.converged = True
            break
        if on_iter is not None and on_iter(k, _time.perf_counter() - t0):
            break
    return res


def materialize(C, V, inv_sigma, W, R):
    """Full L = C V diag(inv) W^T R — solver.py:211-213."""
    return C @ (V @ ((W.T @ R) * inv_sigma[:, None]))


# ----------------------------------------------- BASELINE.json generators
def baseline_problem(n1: int, n2: int, rank: int, alpha: float, seed: int,
                     amp: float = 10.0):
    """BASELINE.json configs 1/2/4/5 restated (Gaussian factors, Bernoulli(alpha)
    support, outliers U[-amp*a, amp*a] with a = mean|L|), in float64.

    Draw order from one numpy Generator (PCG64): W (n1 x r) and V (n2 x r)
    standard normals, then one `random()` per cell for the mask, then one
    `uniform()` per cell for the value (row-major).  L is accumulated
    elementwise in t order (multiply, then add); a = mean|L| is taken as an
    exact integer sum of |L| quantised to 2^-24, so it does not depend on
    summation order.  The device generator (ircur_gen_baseline) reproduces D
    bit for bit from the same PCG64 state.  Returns D, L, S, max|L|.
    """
    rng = np.random.default_rng(seed)
    W = rng.standard_normal((n1, rank))
    V = rng.standard_normal((n2, rank))
    L = W[:, 0:1] * V[:, 0][None, :]
    for t in range(1, rank):
        L = L + W[:, t:t + 1] * V[:, t][None, :]
    a = mean_abs_quantised(L)
    A = amp * a
    mask = rng.random((n1, n2)) < alpha
    vals = rng.uniform(-A, A, size=(n1, n2))
    S = np.where(mask, vals, 0.0)
    D = L + S
    return D, L, S, float(np.abs(L).max())


def _L_rows(W, V, r0, r1):
    L = W[r0:r1, 0:1] * V[:, 0][None, :]
    for t in range(1, W.shape[1]):
        L = L + W[r0:r1, t:t + 1] * V[:, t][None, :]
    return L


def baseline_problem_blocked(n1: int, n2: int, rank: int, alpha: float, seed: int,
                             amp: float = 10.0, dtype=np.float64, block_rows: int = 256,
                             threads: int | None = None):
    """Same D as baseline_problem (bit for bit, then cast to `dtype`), built
    in row blocks with PCG64.advance so large matrices (n = 1e5) fit in host
    memory and generate on all cores.  Returns D, max|L|, a."""
    import concurrent.futures as cf
    import os as _os
    rng = np.random.default_rng(seed)
    W = rng.standard_normal((n1, rank))
    V = rng.standard_normal((n2, rank))
    state = rng.bit_generator.state
    blocks = [(r0, min(n1, r0 + block_rows)) for r0 in range(0, n1, block_rows)]
    nt = threads or (_os.cpu_count() or 1)

    def stats(b):
        L = _L_rows(W, V, *b)
        return float(np.abs(L).max()), int(np.rint(np.abs(L) * 16777216.0).astype(np.int64).sum())

    with cf.ThreadPoolExecutor(nt) as ex:
        st = list(ex.map(stats, blocks))
    linf = max(s[0] for s in st)
    q = sum(s[1] for s in st)
    a = float(q) / 16777216.0 / (n1 * n2)
    A = amp * a
    D = np.empty((n1, n2), dtype=dtype)

    def fill(b):
        r0, r1 = b
        g1 = np.random.PCG64()
        g1.state = state
        g1.advance(r0 * n2)
        mask = np.random.Generator(g1).random((r1 - r0, n2)) < alpha
        g2 = np.random.PCG64()
        g2.state = state
        g2.advance(n1 * n2 + r0 * n2)
        vals = np.random.Generator(g2).uniform(-A, A, size=(r1 - r0, n2))
        D[r0:r1] = _L_rows(W, V, r0, r1) + np.where(mask, vals, 0.0)

    with cf.ThreadPoolExecutor(nt) as ex:
        list(ex.map(fill, blocks))
    return D, linf, a


def mean_abs_quantised(L: np.ndarray) -> float:
    """mean|L| from an exact int64 sum of rint(|L| * 2^24) (order-free)."""
    q = np.rint(np.abs(L) * 16777216.0).astype(np.int64).sum()
    return float(q) / 16777216.0 / L.size


# ------------------------------------------------------------ CUR -> SVD
def cur_to_svd(C, W, sigma, V, inv_sigma, R, compact_drop=1e-14):
    """Compact SVD of C U^+ R as convert.py:21-48 computes it: thin QRs of C
    and R^T, SVD of the middle factor r_c U^+ r_r^T (U^+ applied through
    the factored pinv, matcore.py:185-189), singular values below
    compact_drop * sigma_max dropped.  Returns (W, sigma, V)."""
    q_c, r_c = np.linalg.qr(np.asarray(C, dtype=np.float64), mode="reduced")
    q_r, r_r = np.linalg.qr(np.asarray(R, dtype=np.float64).T, mode="reduced")
    middle = ((r_c @ V) * inv_sigma) @ W.T @ r_r.T
    w_u, s, v_u_t = np.linalg.svd(middle, full_matrices=False)
    Wc, Vc = q_c @ w_u, q_r @ v_u_t.T
    smax = s[0] if s.size else 0.0
    if smax > 0.0:
        keep = s >= compact_drop * smax
        Wc, s, Vc = Wc[:, keep], s[keep], Vc[:, keep]
    return Wc, s, Vc
