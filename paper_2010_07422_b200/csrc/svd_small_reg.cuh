// Register-resident small dense kernels of the core SVD (one warp, kk <= 8).
//
// The kk x kk Rayleigh-Ritz problems of the block subspace iteration
// (ritz_small: Cholesky of V^T V, two triangular solves, Jacobi eigensolver,
// back substitution) and the final Jacobi of the extraction step are
// latency chains.  The shared-memory versions in kernels_svd.cu spend a named
// barrier and several dependent shared-memory round trips per Jacobi round.
// For small blocks (kk = r + 2 <= 8, i.e. r <= 6: cfg1-cfg4) lane i holds
// row i (or column i) of each matrix in registers; the round loop is fully
// unrolled, so every register index and pair is a compile-time constant and
// all exchanges are warp shuffles.  Measured on one warp (tools/ritz_iso.cu):
// kk = 7 Rayleigh-Ritz 19k vs 29k cycles, kk = 4 8k vs 15k.  Larger blocks
// (cfg5: kk = 12) keep the shared-memory kernels, whose code size and
// registers stay independent of kk.
//
// Same arithmetic as the shared-memory kernels: right-looking Cholesky with
// 1/sqrt of the pivot, forward substitution with four partial sums
// (tri_forward), cyclic Jacobi with round-robin pairing, the tangent in fp32
// and c = (1 + t^2)^-1/2, s = t c in fp64, rotations skipped below the
// threshold, eigenpairs sorted by decreasing eigenvalue.
#pragma once

namespace ircur {
namespace sreg {

__host__ __device__ constexpr int circ(int pos, int rd, int nrd) { return pos == 0 ? 0 : ((pos - 1 + rd) % nrd) + 1; }

__device__ __forceinline__ double shf(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

// 1/sqrt(x) for normal x > 0: MUFU approximation + two Newton steps (no
// slow-path branch, so the warp stays converged around the shuffles)
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double h = fma(-x * y, y, 1.0);
  y = fma(0.5 * y, h, y);
  h = fma(-x * y, y, 1.0);
  return fma(0.5 * y, h, y);
}

// Rotation (c, s) annihilating hpq, or (1, 0) below the threshold; branch
// free (every lane evaluates every pair of a round).
__device__ __forceinline__ void rot_params(double hpp, double hqq, double hpq, double thr, double isc, double& c,
                                           double& s) {
  const float d = (float)((hqq - hpp) * isc), h2 = (float)(2.0 * hpq * isc);
  float rt;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(rt) : "f"(fmaf(d, d, h2 * h2)));
  const float tf = __fdividef(h2, fabsf(d) + rt) * (d >= 0.f ? 1.f : -1.f);
  const double t = (double)tf;
  const double cc = rsqrt_nr(fma(t, t, 1.0));
  const bool rot = fabs(hpq) > 1e-300 && fabs(hpq) > thr;
  c = rot ? cc : 1.0;
  s = rot ? t * cc : 0.0;
}

// Cyclic Jacobi on the symmetric matrix whose row `lane` is h (lanes >= KK
// idle); z accumulates the rotations (Z <- Z J, row `lane` of Z).  Returns
// the sweeps run.
template <int KK>
__device__ __forceinline__ int jacobi(double (&h)[KK], double (&z)[KK], int lane, double thr_rel, int max_sweeps) {
  constexpr int NP = KK + (KK & 1), NR = NP - 1, NS = NP / 2;
  const bool row = lane < KK;
  double dg = 0.0;
#pragma unroll
  for (int j = 0; j < KK; ++j) dg = (j == lane) ? h[j] : dg;
  double scale = row ? fabs(dg) : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
  const double thr = thr_rel * scale;
  const double isc = scale > 0.0 ? 1.0 / scale : 1.0;
  auto offmax = [&]() {
    double off = 0.0;
#pragma unroll
    for (int j = 0; j < KK; ++j) off = (row && j != lane) ? fmax(off, fabs(h[j])) : off;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) off = fmax(off, __shfl_xor_sync(0xffffffffu, off, o));
    return off;
  };
  double off = offmax();
  int sweeps = 0;
  for (; sweeps < max_sweeps && off > thr; ++sweeps) {
#pragma unroll
    for (int rd = 0; rd < NR; ++rd) {
      double pc[NS], ps[NS];
      // H <- H J (columns p, q of my row), Z <- Z J; pair parameters from the
      // round's starting H (disjoint pairs leave each other's 2x2 blocks alone)
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const int p0 = circ(k, rd, NR), q0 = circ(NP - 1 - k, rd, NR);
        const int p = p0 < q0 ? p0 : q0, q = p0 < q0 ? q0 : p0;
        pc[k] = 1.0;
        ps[k] = 0.0;
        if (q < KK) {
          rot_params(shf(h[p], p), shf(h[q], q), shf(h[q], p), thr, isc, pc[k], ps[k]);
          const double c = pc[k], s = ps[k];
          const double hp = h[p], hq = h[q];
          h[p] = c * hp - s * hq;
          h[q] = c * hq + s * hp;
          const double zp = z[p], zq = z[q];
          z[p] = c * zp - s * zq;
          z[q] = c * zq + s * zp;
        }
      }
      // H <- J^T H: my row mixes with my partner's (first of a pair: +s)
      const int pos = lane == 0 ? 0 : ((lane - 1 - rd + NR) % NR) + 1;
      const int ppos = NP - 1 - pos;
      int partner = circ(ppos, rd, NR);
      const int slot = pos < ppos ? pos : ppos;
      partner = (row && partner < KK) ? partner : lane;
      double c = 1.0, s = 0.0;
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        c = (k == slot) ? pc[k] : c;
        s = (k == slot) ? ps[k] : s;
      }
      s = lane > partner ? -s : s;
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        const double ph = shf(h[j], partner);
        h[j] = c * h[j] - s * ph;
      }
    }
    off = offmax();
  }
  return sweeps;
}

// Eigenvalues of lane's row (diagonal after Jacobi) -> rank by decreasing
// value (ties by index), written to lam[rank]; Z columns permuted the same
// way into Zs (row `lane`, ld HL).
template <int KK>
__device__ __forceinline__ void sort_out(const double (&h)[KK], const double (&z)[KK], int lane, double* lam,
                                         double* Zs, int HL) {
  double li = 0.0;
#pragma unroll
  for (int j = 0; j < KK; ++j) li = (j == lane) ? h[j] : li;
  int rk = 0;
#pragma unroll
  for (int j = 0; j < KK; ++j) {
    const double lj = shf(li, j);
    rk += (lj > li) || (lj == li && j < lane);
  }
  if (lane < KK) lam[rk] = li;
#pragma unroll
  for (int j = 0; j < KK; ++j) {
    const int rj = __shfl_sync(0xffffffffu, rk, j);
    if (lane < KK) Zs[lane * HL + rj] = z[j];
  }
}

// x = L^{-1} b in place, lane = column of b; L row i in lane i (m[k], k <= i),
// linv = 1 / L_ii of the lane.  Four partial sums as tri_forward.
template <int KK>
__device__ __forceinline__ void fwd(const double (&m)[KK], double linv, double (&x)[KK]) {
#pragma unroll
  for (int i = 0; i < KK; ++i) {
    double s[4] = {x[i], 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < i; ++k) {
      const int u = (k < (i & ~3)) ? (k & 3) : 0;  // tri_forward: remainder terms go to s0
      s[u] = fma(-shf(m[k], i), x[k], s[u]);
    }
    x[i] = ((s[0] + s[1]) + (s[2] + s[3])) * shf(linv, i);
  }
}

// Rayleigh-Ritz on (Hp, M) (both kk x kk, ld KK, symmetric): lanes 0..31 of
// one warp.  Writes T = L^{-T} Z (ld HL), lam (descending); scratch W, Zs
// (kk x HL).  Returns 0 if chol(M) broke down.
template <int KK>
__device__ int ritz(const double* Hp, const double* M, double* T, double* lam, double* W, double* Zs, int HL,
                    double thr_rel, int max_sweeps, int* sweeps_out) {
  const int lane = threadIdx.x & 31;
  const bool row = lane < KK;
  // ---- Cholesky M = L L^T (row `lane`)
  double m[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) m[k] = (row && k <= lane) ? M[lane * KK + k] : 0.0;
  double linv = 1.0;
  int ok = 1;
#pragma unroll
  for (int j = 0; j < KK; ++j) {
    double d = shf(m[j], j);
    ok &= d > 1e-300;
    d = d > 1e-300 ? d : 1.0;
    const double ir = rsqrt_nr(d);
    linv = lane == j ? ir : linv;
    m[j] = lane == j ? d * ir : (lane > j ? m[j] * ir : m[j]);
#pragma unroll
    for (int k = j + 1; k < KK; ++k) {
      const double lkj = shf(m[j], k);
      m[k] = (lane >= k && row) ? fma(-m[j], lkj, m[k]) : m[k];
    }
  }
  if (!ok) return 0;
  // ---- H = L^{-1} Hp L^{-T}: column `lane` of L^{-1} Hp, transpose, again
  double x[KK];
#pragma unroll
  for (int i = 0; i < KK; ++i) x[i] = row ? Hp[i * KK + lane] : 0.0;
  fwd<KK>(m, linv, x);
  if (row)
#pragma unroll
    for (int i = 0; i < KK; ++i) W[i * HL + lane] = x[i];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < KK; ++j) x[j] = row ? W[lane * HL + j] : 0.0;
  __syncwarp();
  fwd<KK>(m, linv, x);  // x = column `lane` of L^{-1} K^T
  if (row)
#pragma unroll
    for (int i = 0; i < KK; ++i) W[i * HL + lane] = x[i];
  __syncwarp();
  double h[KK], z[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) {
    h[j] = row ? 0.5 * (W[lane * HL + j] + x[j]) : 0.0;
    z[j] = (j == lane) ? 1.0 : 0.0;
  }
  const int sw = jacobi<KK>(h, z, lane, thr_rel, max_sweeps);
  if (sweeps_out) *sweeps_out = sw;
  sort_out<KK>(h, z, lane, lam, Zs, HL);
  __syncwarp();
  // ---- T = L^{-T} Zs (column `lane`), back substitution as ritz_small
  double t[KK];
#pragma unroll
  for (int i = 0; i < KK; ++i) t[i] = row ? Zs[i * HL + lane] : 0.0;
#pragma unroll
  for (int i = KK - 1; i >= 0; --i) {
    double s[4] = {t[i], 0.0, 0.0, 0.0};
#pragma unroll
    for (int k2 = i + 1; k2 < KK; ++k2) {
      const int u = (k2 - (i + 1)) < ((KK - (i + 1)) & ~3) ? ((k2 - (i + 1)) & 3) : 0;
      s[u] = fma(-shf(m[i], k2), t[k2], s[u]);
    }
    t[i] = ((s[0] + s[1]) + (s[2] + s[3])) * shf(linv, i);
  }
  if (row)
#pragma unroll
    for (int i = 0; i < KK; ++i) T[i * HL + lane] = t[i];
  return 1;
}

// Symmetric eigenproblem of H (kk x kk rows, ld HL): sorted eigenvectors into
// Zs (ld HL), eigenvalues into lam.  One warp.
template <int KK>
__device__ int eig(const double* H, int HL, double* Zs, double* lam, double thr_rel, int max_sweeps) {
  const int lane = threadIdx.x & 31;
  const bool row = lane < KK;
  double h[KK], z[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) {
    h[j] = row ? H[lane * HL + j] : 0.0;
    z[j] = (j == lane) ? 1.0 : 0.0;
  }
  const int sw = jacobi<KK>(h, z, lane, thr_rel, max_sweeps);
  sort_out<KK>(h, z, lane, lam, Zs, HL);
  return sw;
}

}  // namespace sreg

#define IRCUR_SREG_CASES(X) X(3) X(4) X(5) X(6) X(7) X(8)

__host__ __device__ constexpr bool sreg_supported(int kk) { return kk >= 3 && kk <= 8; }

__device__ __noinline__ int ritz_reg(int kk, const double* Hp, const double* M, double* T, double* lam, double* W,
                                     double* Zs, int HL, double thr_rel, int max_sweeps, int* sweeps_out) {
  switch (kk) {
#define IRCUR_RC(K) \
  case K:           \
    return sreg::ritz<K>(Hp, M, T, lam, W, Zs, HL, thr_rel, max_sweeps, sweeps_out);
    IRCUR_SREG_CASES(IRCUR_RC)
#undef IRCUR_RC
    default:
      return -1;
  }
}

__device__ __noinline__ int eig_reg(int kk, const double* H, int HL, double* Zs, double* lam, double thr_rel,
                                    int max_sweeps) {
  switch (kk) {
#define IRCUR_EC(K) \
  case K:           \
    return sreg::eig<K>(H, HL, Zs, lam, thr_rel, max_sweeps);
    IRCUR_SREG_CASES(IRCUR_EC)
#undef IRCUR_EC
    default:
      return -1;
  }
}

}  // namespace ircur
