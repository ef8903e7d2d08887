// Exact top-r SVD / pseudo-inverse of the |I| x |J| core (sm_100a).
//
// Replaces matcore.truncated_svd (LAPACK gesdd, matcore.py:128-139) and
// PinvFactor.from_svd (cutoff sigma > 1e-12 sigma_max, matcore.py:156-165).
// Only the top k = min(r, |I|, |J|) triplets are consumed, so instead of a
// full dense SVD the core is factorised by block subspace iteration on the
// Gram matrix G = U^T U with Rayleigh-Ritz extraction every step,
// warm-started from the previous iterate's Q(:,J) and iterated until the
// Ritz residuals reach fp64 round-off; a final Rayleigh-Ritz step on U
// itself resolves small singular values to absolute fp64 accuracy, so the
// pinv cutoff behaves like LAPACK's.  Block size kk = min(2r, |I|, |J|, 32).
//
// Layout: one thread-block cluster per core.  CTA q owns rows [lo_q, hi_q)
// of G (resident in its shared memory for the whole call) and of the n x kk
// block V; the full V is replicated in every CTA's shared memory and
// re-assembled through L2 after each step; the small kk x kk sums go through
// DSMEM in a fixed rank order, so every CTA holds bitwise-identical reduced
// values and takes identical branches (deterministic, run to run).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "ircur_common.cuh"
#include "launchers.cuh"

namespace cg = cooperative_groups;

namespace ircur {

constexpr int kSvdNT = 512;
constexpr int kSvdNW = kSvdNT / 32;
constexpr int kKMax = 32;

// ------------------------------------------------------------------ gram
// G = U^T U (n x n), 32x32 output tile per CTA, K = m in 32-row chunks.
__global__ void __launch_bounds__(256) gram_kernel(const double* __restrict__ U, int ldu, int m, int n,
                                                   double* __restrict__ G, int ldg, const int* done) {
  if (done && *done) return;
  __shared__ double A[32][33];
  __shared__ double B[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // ty 0..7
  const int a0 = blockIdx.y * 32, b0 = blockIdx.x * 32;
  double acc[4] = {0, 0, 0, 0};
  for (int i0 = 0; i0 < m; i0 += 32) {
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
      const int i = i0 + ty + k;
      A[ty + k][tx] = (i < m && a0 + tx < n) ? U[(int64_t)i * ldu + a0 + tx] : 0.0;
      B[ty + k][tx] = (i < m && b0 + tx < n) ? U[(int64_t)i * ldu + b0 + tx] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int i = 0; i < 32; ++i) {
      const double bv = B[i][tx];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = fma(A[i][ty + 8 * u], bv, acc[u]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int ra = a0 + ty + 8 * u, cb = b0 + tx;
    if (ra < n && cb < n) G[(int64_t)ra * ldg + cb] = acc[u];
  }
}

// ------------------------------------------------------------ layout
// Shared-memory layout in doubles; identical on host (size) and device.
struct SvdLayout {
  int n, m, kk, KP, HL, per, mper, rowsmax, ldgq, S, gq_smem;
  int oV, oGq, oP, oBq, oXq, oH, oH2, oZ, oRed, oRout, oLam, oCs, oW, total;
};

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

__host__ __device__ inline SvdLayout svd_layout(int n, int m, int kk, int cs) {
  SvdLayout L;
  L.n = n; L.m = m; L.kk = kk;
  L.KP = kk | 1;
  L.HL = kk + 1;
  L.per = ceil_div(n, cs);
  L.mper = ceil_div(m, cs);
  L.rowsmax = L.per > L.mper ? L.per : L.mper;
  L.ldgq = n | 1;
  const int tasks = ceil_div(L.rowsmax, 8) * ceil_div(kk, 16);
  int S = kSvdNW / (tasks > 0 ? tasks : 1);
  S = S < 1 ? 1 : (S > 4 ? 4 : S);
  L.S = S;
  int off = 0;
  L.oV = off; off += n * L.KP;
  L.oP = off; off += S * L.rowsmax * L.KP;
  L.oBq = off; off += L.rowsmax * L.KP;
  L.oXq = off; off += L.rowsmax * L.KP;
  L.oH = off; off += kk * L.HL;
  L.oH2 = off; off += kk * L.HL;
  L.oZ = off; off += kk * L.HL;
  L.oRed = off; off += kk * kk + 2 * kk;
  L.oRout = off; off += kk * kk + 2 * kk;
  L.oLam = off; off += kk;
  L.oCs = off; off += 4 * kKMax;
  L.oW = off; off += 2 * kKMax + 8;   // warp scratch / flags (as doubles)
  const int base = off;
  L.oGq = base;
  const size_t with_g = (size_t)(base + L.per * L.ldgq) * sizeof(double);
  L.gq_smem = with_g <= (size_t)227 * 1024 ? 1 : 0;
  L.total = L.gq_smem ? base + L.per * L.ldgq : base;
  return L;
}

// ------------------------------------------------------------ helpers
__device__ __forceinline__ double hash_uniform(uint64_t a, uint64_t b) {
  uint64_t z = a * 0x9E3779B97F4A7C15ull ^ (b + 0x632BE59BD9B4E019ull) * 0xBF58476D1CE4E5B9ull;
  z ^= z >> 31; z *= 0x94D049BB133111EBull; z ^= z >> 29; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 32;
  return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;  // [-1, 1)
}

struct Sm {
  SvdLayout L;
  double *V, *Gq, *P, *Bq, *Xq, *H, *H2, *Z, *red, *rout, *lam, *cs, *ws;
  int* flags;
};

__device__ __forceinline__ void cluster_sum(cg::cluster_group& cl, Sm& S, int len) {
  cl.sync();
  const int CS = (int)cl.num_blocks();
  for (int e = threadIdx.x; e < len; e += kSvdNT) {
    double s = *cl.map_shared_rank(S.red + e, 0);
    for (int q = 1; q < CS; ++q) s += *cl.map_shared_rank(S.red + e, q);
    S.rout[e] = s;
  }
  cl.sync();
}

// Out(nr x kk, ld KP) = A(nr x n, lda) * V(n x kk, ld KP).  Warp tile:
// 8 rows x 16 cols, lane = (row pair, col pair) so that the A loads are
// 4-way and the V loads 8-way broadcasts; the inner dimension is split in S
// contiguous chunks whose partial tiles are summed in a fixed order.
// A may live in shared or global memory (generic pointer).
__device__ void tiled_product(const double* A, int lda, int nr, int n, const double* V, int KP, int kk,
                              double* Out, double* partial, int S) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int li = lane >> 3, lc = lane & 7;
  const int rt_n = ceil_div(nr, 8), ct_n = ceil_div(kk, 16);
  const int tasks = rt_n * ct_n * S;
  const int chunk = ceil_div(n, S);
  for (int task = w; task < tasks; task += kSvdNW) {
    const int ks = task % S;
    const int t2 = task / S;
    const int rt = t2 % rt_n, ct = t2 / rt_n;
    const int i0 = rt * 8 + li * 2, c0 = ct * 16 + lc * 2;
    const int ia = min(i0, nr - 1), ib = min(i0 + 1, nr - 1);
    const int ca = min(c0, kk - 1), cb = min(c0 + 1, kk - 1);
    const int j0 = ks * chunk, j1 = min(n, j0 + chunk);
    const double* Aa = A + (int64_t)ia * lda;
    const double* Ab = A + (int64_t)ib * lda;
    double s00 = 0.0, s01 = 0.0, s10 = 0.0, s11 = 0.0;
#pragma unroll 4
    for (int j = j0; j < j1; ++j) {
      const double a0 = Aa[j], a1 = Ab[j];
      const double v0 = V[j * KP + ca], v1 = V[j * KP + cb];
      s00 = fma(a0, v0, s00);
      s01 = fma(a0, v1, s01);
      s10 = fma(a1, v0, s10);
      s11 = fma(a1, v1, s11);
    }
    double* P = partial + (size_t)ks * nr * KP;
    if (i0 < nr) {
      if (c0 < kk) P[i0 * KP + c0] = s00;
      if (c0 + 1 < kk) P[i0 * KP + c0 + 1] = s01;
    }
    if (i0 + 1 < nr) {
      if (c0 < kk) P[(i0 + 1) * KP + c0] = s10;
      if (c0 + 1 < kk) P[(i0 + 1) * KP + c0 + 1] = s11;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nr * kk; e += kSvdNT) {
    const int i = e / kk, c = e - i * kk;
    double s = partial[i * KP + c];
    for (int ks = 1; ks < S; ++ks) s += partial[(size_t)ks * nr * KP + i * KP + c];
    Out[i * KP + c] = s;
  }
  __syncthreads();
}

// Cyclic Jacobi eigen-decomposition of the symmetric kk x kk S.H (round-robin
// parallel ordering, J^T H J for all disjoint pairs of a round in one pass).
// On exit S.lam holds eigenvalues in decreasing order and S.Z the matching
// eigenvectors (columns).  Executed identically by every CTA of the cluster.
__device__ void jacobi_eig(Sm& S, int kk) {
  const int tid = threadIdx.x;
  const int HL = S.L.HL;
  double* H = S.H;
  double* Hn = S.H2;
  for (int e = tid; e < kk * kk; e += kSvdNT) {
    const int i = e / kk, j = e - i * kk;
    S.Z[i * HL + j] = (i == j) ? 1.0 : 0.0;
  }
  const int np = (kk + 1) / 2;
  const int nply = 2 * np;
  int* pairs = reinterpret_cast<int*>(S.cs + 2 * kKMax);  // [kKMax] partner of each index
  double scale = 0.0;
  for (int i = 0; i < kk; ++i) scale = fmax(scale, fabs(H[i * HL + i]));
  const double thr = 4e-16 * scale;
  __syncthreads();
  for (int sweep = 0; sweep < 30; ++sweep) {
    // early exit: any off-diagonal above threshold?
    if (tid == 0) S.flags[0] = 0;
    __syncthreads();
    for (int e = tid; e < kk * kk; e += kSvdNT) {
      const int i = e / kk, j = e - i * kk;
      if (i < j && fabs(H[i * HL + j]) > thr) S.flags[0] = 1;
    }
    __syncthreads();
    if (S.flags[0] == 0) break;
    for (int rd = 0; rd < nply - 1; ++rd) {
      if (tid < np) {
        const int pa = tid == 0 ? 0 : ((tid - 1 + rd) % (nply - 1)) + 1;
        const int pb = ((nply - 2 - tid + rd) % (nply - 1)) + 1;
        const int p = min(pa, pb), q = max(pa, pb);
        double c = 1.0, s = 0.0;
        if (q < kk) {
          const double hpq = H[p * HL + q];
          if (fabs(hpq) > 1e-300 && fabs(hpq) > thr) {
            const double hpp = H[p * HL + p], hqq = H[q * HL + q];
            const double tau = (hqq - hpp) / (2.0 * hpq);
            const double t = fabs(tau) > 1e150 ? 0.5 / tau
                                               : (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
          }
          pairs[p] = q;
          pairs[q] = p;
          S.cs[2 * p] = c;  S.cs[2 * p + 1] = s;     // p is the "first" of its pair
          S.cs[2 * q] = c;  S.cs[2 * q + 1] = -s;    // sign flip marks the second
        } else if (p < kk) {
          pairs[p] = p;
          S.cs[2 * p] = 1.0; S.cs[2 * p + 1] = 0.0;
        }
      }
      __syncthreads();
      // new H = J^T H J; each entry from the 2x2 block of its row and column pairs
      for (int e = tid; e < kk * kk; e += kSvdNT) {
        const int a = e / kk, b = e - a * kk;
        const int pa_ = pairs[a], pb_ = pairs[b];
        const double ca = S.cs[2 * a], sa = S.cs[2 * a + 1];
        const double cb = S.cs[2 * b], sb = S.cs[2 * b + 1];
        // row rotation: new row a = ca * row a - sa * row partner(a)   (sa < 0 for the second)
        const double r_b = ca * H[a * HL + b] - sa * H[pa_ * HL + b];
        const double r_pb = ca * H[a * HL + pb_] - sa * H[pa_ * HL + pb_];
        Hn[a * HL + b] = cb * r_b - sb * r_pb;
      }
      for (int e = tid; e < kk * kk; e += kSvdNT) {
        const int i = e / kk, b = e - i * kk;
        const int pb_ = pairs[b];
        const double cb = S.cs[2 * b], sb = S.cs[2 * b + 1];
        if (sb != 0.0 && b < pb_) {
          const double zp = S.Z[i * HL + b], zq = S.Z[i * HL + pb_];
          S.Z[i * HL + b] = cb * zp - sb * zq;
          S.Z[i * HL + pb_] = sb * zp + cb * zq;
        }
      }
      __syncthreads();
      double* t = H; H = Hn; Hn = t;
    }
  }
  // sort (descending, stable) via rank computation
  int* perm = pairs;
  __syncthreads();
  if (tid < kk) {
    const double li = H[tid * HL + tid];
    int rk = 0;
    for (int j = 0; j < kk; ++j) {
      const double lj = H[j * HL + j];
      rk += (lj > li) || (lj == li && j < tid);
    }
    perm[kKMax + rk] = tid;
  }
  __syncthreads();
  if (tid < kk) S.lam[tid] = H[perm[kKMax + tid] * HL + perm[kKMax + tid]];
  for (int e = tid; e < kk * kk; e += kSvdNT) {
    const int i = e / kk, j = e - i * kk;
    Hn[i * HL + j] = S.Z[i * HL + perm[kKMax + j]];
  }
  __syncthreads();
  for (int e = tid; e < kk * kk; e += kSvdNT) {
    const int i = e / kk, j = e - i * kk;
    S.Z[i * HL + j] = Hn[i * HL + j];
  }
  __syncthreads();
}

// X(nr x kk, ld KP) <- X Z  using tmp (nr x KP)
__device__ void rotate_rows(double* X, int nr, int KP, int kk, const double* Z, int HL, double* tmp) {
  for (int e = threadIdx.x; e < nr * kk; e += kSvdNT) {
    const int i = e / kk, c = e - i * kk;
    double s = 0.0;
    for (int j = 0; j < kk; ++j) s = fma(X[i * KP + j], Z[j * HL + c], s);
    tmp[i * KP + c] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nr * kk; e += kSvdNT) {
    const int i = e / kk, c = e - i * kk;
    X[i * KP + c] = tmp[i * KP + c];
  }
  __syncthreads();
}

// Cholesky of the kk x kk Gram in G (ld kk) into Lo (lower, ld HL) by warp 0;
// returns 0 on breakdown (non-positive pivot).
__device__ int cholesky_warp(const double* Gr, double* Lo, int HL, int kk, int* flag) {
  const int lane = threadIdx.x & 31;
  if ((threadIdx.x >> 5) == 0) {
    int ok = 1;
    for (int j = 0; j < kk; ++j) {
      double p = 0.0;
      for (int k2 = lane; k2 < j; k2 += 32) p = fma(Lo[j * HL + k2], Lo[j * HL + k2], p);
      p = warp_sum(p);
      double d = Gr[j * kk + j] - p;
      if (!(d > 1e-300)) { ok = 0; d = 1.0; }
      const double ljj = sqrt(d);
      for (int i = j + 1 + lane; i < kk; i += 32) {
        double s2 = Gr[i * kk + j];
        for (int k2 = 0; k2 < j; ++k2) s2 = fma(-Lo[i * HL + k2], Lo[j * HL + k2], s2);
        Lo[i * HL + j] = s2 / ljj;
      }
      if (lane == 0) Lo[j * HL + j] = ljj;
      __syncwarp();
    }
    if (lane == 0) *flag = ok;
  }
  __syncthreads();
  return *flag;
}

// rows of X (nr x kk, ld KP): x <- x L^{-T}
__device__ void trsm_rows(double* X, int nr, int KP, int kk, const double* Lo, int HL) {
  for (int i = threadIdx.x; i < nr; i += kSvdNT) {
    for (int c = 0; c < kk; ++c) {
      double s = X[i * KP + c];
      for (int k2 = 0; k2 < c; ++k2) s = fma(-X[i * KP + k2], Lo[c * HL + k2], s);
      X[i * KP + c] = s / Lo[c * HL + c];
    }
  }
  __syncthreads();
}

// Block-local CGS2 with random replacement on the FULL V (n x kk) — robust
// fallback when the Cholesky-QR start breaks down (rank-deficient start).
__device__ void cgs2_full(Sm& S, int n, int KP, int kk, uint64_t salt) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  double* dots = S.red;
  for (int c = 0; c < kk; ++c) {
    for (int attempt = 0; attempt < 4; ++attempt) {
      double p = 0.0;
      for (int j = tid; j < n; j += kSvdNT) p = fma(S.V[j * KP + c], S.V[j * KP + c], p);
      p = warp_sum(p);
      if (lane == 0) S.ws[w] = p;
      __syncthreads();
      double nrm0 = 0.0;
      for (int i = 0; i < kSvdNW; ++i) nrm0 += S.ws[i];
      __syncthreads();
      for (int pass = 0; pass < 2; ++pass) {
        for (int k = w; k < c; k += kSvdNW) {
          double d = 0.0;
          for (int j = lane; j < n; j += 32) d = fma(S.V[j * KP + k], S.V[j * KP + c], d);
          d = warp_sum(d);
          if (lane == 0) dots[k] = d;
        }
        __syncthreads();
        for (int j = tid; j < n; j += kSvdNT) {
          double v = S.V[j * KP + c];
          for (int k = 0; k < c; ++k) v = fma(-dots[k], S.V[j * KP + k], v);
          S.V[j * KP + c] = v;
        }
        __syncthreads();
      }
      p = 0.0;
      for (int j = tid; j < n; j += kSvdNT) p = fma(S.V[j * KP + c], S.V[j * KP + c], p);
      p = warp_sum(p);
      if (lane == 0) S.ws[w] = p;
      __syncthreads();
      double nrm = 0.0;
      for (int i = 0; i < kSvdNW; ++i) nrm += S.ws[i];
      __syncthreads();
      if (nrm > 1e-20 * nrm0 && nrm > 1e-280) {
        const double inv = 1.0 / sqrt(nrm);
        for (int j = tid; j < n; j += kSvdNT) S.V[j * KP + c] *= inv;
        __syncthreads();
        break;
      }
      for (int j = tid; j < n; j += kSvdNT)
        S.V[j * KP + c] = hash_uniform(salt + 1000003ull * (uint64_t)(attempt + 1), (uint64_t)j * 64 + c);
      __syncthreads();
    }
  }
}

// Full-V orthonormalisation (redundant in every CTA): Cholesky-QR twice,
// CGS2 fallback on breakdown.
__device__ void orthonormalize_full(Sm& S, int n, int KP, int kk, uint64_t salt) {
  const int HL = S.L.HL;
  for (int pass = 0; pass < 2; ++pass) {
    for (int e = threadIdx.x; e < kk * kk; e += kSvdNT) {
      const int c1 = e / kk, c2 = e - c1 * kk;
      double s = 0.0;
      if (c2 <= c1)
        for (int j = 0; j < n; ++j) s = fma(S.V[j * KP + c1], S.V[j * KP + c2], s);
      S.rout[e] = s;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kk * kk; e += kSvdNT) {
      const int c1 = e / kk, c2 = e - c1 * kk;
      if (c2 > c1) S.rout[e] = S.rout[c2 * kk + c1];
    }
    __syncthreads();
    if (!cholesky_warp(S.rout, S.H2, HL, kk, S.flags + 1)) {
      cgs2_full(S, n, KP, kk, salt);
      return;
    }
    trsm_rows(S.V, n, KP, kk, S.H2, HL);
  }
}

template <typename T>
__global__ void __launch_bounds__(kSvdNT, 1) svd_kernel(const __grid_constant__ SvdArgs a) {
  if (a.done && *a.done) return;
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks();
  const int q = (int)cl.block_rank();
  const int n = a.n, m = a.m, r = a.r, kk = a.kk;
  const int reff = min(r, min(m, n));
  extern __shared__ __align__(16) double svsm[];
  Sm S;
  S.L = svd_layout(n, m, kk, CS);
  const SvdLayout& L = S.L;
  const int KP = L.KP, HL = L.HL;
  S.V = svsm + L.oV; S.P = svsm + L.oP; S.Bq = svsm + L.oBq; S.Xq = svsm + L.oXq;
  S.H = svsm + L.oH; S.H2 = svsm + L.oH2; S.Z = svsm + L.oZ; S.red = svsm + L.oRed;
  S.rout = svsm + L.oRout; S.lam = svsm + L.oLam; S.cs = svsm + L.oCs; S.ws = svsm + L.oW;
  S.flags = reinterpret_cast<int*>(svsm + L.oW + kKMax);
  S.Gq = svsm + L.oGq;
  const int lo = min(n, q * L.per), hi = min(n, lo + L.per), nr = hi - lo;
  const int mlo = min(m, q * L.mper), mhi = min(m, mlo + L.mper), mr = mhi - mlo;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

  // ---- 0. G rows of this CTA into shared memory; starting block V
  const double* Gq = a.G + (int64_t)lo * a.ldg;
  int ldgq = a.ldg;
  if (L.gq_smem) {
    for (int e = tid; e < nr * n; e += kSvdNT) {
      const int i = e / n, j = e - i * n;
      S.Gq[i * L.ldgq + j] = a.G[(int64_t)(lo + i) * a.ldg + j];
    }
    Gq = S.Gq;
    ldgq = L.ldgq;
  }
  const T* warm = reinterpret_cast<const T*>(a.warm);
  for (int e = tid; e < n * kk; e += kSvdNT) {
    const int j = e / kk, c = e - j * kk;
    double v = 0.0;
    if (warm && c < a.warm_cols) v = (double)warm[(int64_t)j * a.warm_ld + c];
    else v = hash_uniform(0x5EEDull + a.salt, (uint64_t)j * 64 + c);
    S.V[j * KP + c] = v;
  }
  __syncthreads();
  orthonormalize_full(S, n, KP, kk, a.salt);

  double prev_res = 1e300;
  int stall = 0;
  int step = 0;
  for (; step < a.maxsteps; ++step) {
    // ---- 1. B_q = G(lo:hi, :) V
    tiled_product(Gq, ldgq, nr, n, S.V, KP, kk, S.Bq, S.P, L.S);
    // ---- 2. H = V^T G V (partial over my rows) -> cluster sum
    for (int e = tid; e < kk * kk; e += kSvdNT) {
      const int c1 = e / kk, c2 = e - c1 * kk;
      double s = 0.0;
      for (int i = 0; i < nr; ++i) s = fma(S.V[(lo + i) * KP + c1], S.Bq[i * KP + c2], s);
      S.red[e] = s;
    }
    cluster_sum(cl, S, kk * kk);
    for (int e = tid; e < kk * kk; e += kSvdNT) {
      const int c1 = e / kk, c2 = e - c1 * kk;
      S.H[c1 * HL + c2] = 0.5 * (S.rout[c1 * kk + c2] + S.rout[c2 * kk + c1]);
    }
    __syncthreads();
    jacobi_eig(S, kk);
    // ---- 3. Ritz rotation of my rows: Xq <- V_q Z ; P <- B_q Z
    for (int e = tid; e < nr * kk; e += kSvdNT) {
      const int i = e / kk, c = e - i * kk;
      double sv = 0.0, sb = 0.0;
      for (int j = 0; j < kk; ++j) {
        const double z = S.Z[j * HL + c];
        sv = fma(S.V[(lo + i) * KP + j], z, sv);
        sb = fma(S.Bq[i * KP + j], z, sb);
      }
      S.Xq[i * KP + c] = sv;
      S.P[i * KP + c] = sb;
    }
    __syncthreads();
    // ---- 4. residuals ||B z_c - lam_c V z_c||^2 and the next block
    //      Vn_c = B z_c / lam_c (significant lam) or V z_c (negligible lam)
    const double lam0 = S.lam[0];
    const double sig_thr = 1e-10 * fabs(lam0);
    if (tid < kk) {
      const int c = tid;
      const double lc = S.lam[c];
      double rs = 0.0;
      for (int i = 0; i < nr; ++i) {
        const double d = S.P[i * KP + c] - lc * S.Xq[i * KP + c];
        rs = fma(d, d, rs);
      }
      S.red[kk * kk + c] = rs;
    }
    for (int e = tid; e < nr * kk; e += kSvdNT) {
      const int i = e / kk, c = e - i * kk;
      const double lc = S.lam[c];
      S.Bq[i * KP + c] = (lc > sig_thr && lc > 0.0) ? S.P[i * KP + c] / lc : S.Xq[i * KP + c];
    }
    __syncthreads();
    for (int e = tid; e < kk * kk; e += kSvdNT) {
      const int c1 = e / kk, c2 = e - c1 * kk;
      double s = 0.0;
      for (int i = 0; i < nr; ++i) s = fma(S.Bq[i * KP + c1], S.Bq[i * KP + c2], s);
      S.red[e] = s;
    }
    cluster_sum(cl, S, kk * kk + kk);
    double resmax = 0.0;
    for (int c = 0; c < reff; ++c) resmax = fmax(resmax, sqrt(S.rout[kk * kk + c]));
    const bool conv = !(lam0 > 0.0) || resmax <= a.tol * lam0;
    if (resmax > 0.5 * prev_res) ++stall; else stall = 0;
    prev_res = resmax;
    const bool give_up = (stall >= 3 && resmax <= 1e-11 * lam0);
    if (conv || give_up || step + 1 == a.maxsteps) {
      for (int e = tid; e < nr * kk; e += kSvdNT) {
        const int i = e / kk, c = e - i * kk;
        a.scratch[(int64_t)(lo + i) * kKMax + c] = S.Xq[i * KP + c];
      }
      break;
    }
    // ---- 5. Cholesky-QR of the next block (Gram = I + E^T E, well posed)
    const int ok = cholesky_warp(S.rout, S.H2, HL, kk, S.flags + 1);
    if (ok) trsm_rows(S.Bq, nr, KP, kk, S.H2, HL);
    // ---- 6. all-gather the new block through global scratch (L2)
    for (int e = tid; e < nr * kk; e += kSvdNT) {
      const int i = e / kk, c = e - i * kk;
      a.scratch[(int64_t)(lo + i) * kKMax + c] = S.Bq[i * KP + c];
    }
    __threadfence();
    cl.sync();
    for (int e = tid; e < n * kk; e += kSvdNT) {
      const int j = e / kk, c = e - j * kk;
      S.V[j * KP + c] = a.scratch[(int64_t)j * kKMax + c];
    }
    __syncthreads();
    if (!ok) orthonormalize_full(S, n, KP, kk, a.salt + 77ull * (step + 1));
    cl.sync();  // nobody overwrites scratch before every CTA has copied it
  }
  __threadfence();
  cl.sync();
  for (int e = tid; e < n * kk; e += kSvdNT) {
    const int j = e / kk, c = e - j * kk;
    S.V[j * KP + c] = a.scratch[(int64_t)j * kKMax + c];
  }
  __syncthreads();
  if (q == 0 && tid == 0 && a.steps_out) *a.steps_out = step + 1;

  // ---- 7. Rayleigh-Ritz on U itself: Y = U V (my m-rows), H2 = Y^T Y
  tiled_product(a.U + (int64_t)mlo * a.ldu, a.ldu, mr, n, S.V, KP, kk, S.Xq, S.P, L.S);
  for (int e = tid; e < kk * kk; e += kSvdNT) {
    const int c1 = e / kk, c2 = e - c1 * kk;
    double s = 0.0;
    for (int i = 0; i < mr; ++i) s = fma(S.Xq[i * KP + c1], S.Xq[i * KP + c2], s);
    S.red[e] = s;
  }
  cluster_sum(cl, S, kk * kk);
  for (int e = tid; e < kk * kk; e += kSvdNT) {
    const int c1 = e / kk, c2 = e - c1 * kk;
    S.H[c1 * HL + c2] = 0.5 * (S.rout[c1 * kk + c2] + S.rout[c2 * kk + c1]);
  }
  __syncthreads();
  jacobi_eig(S, kk);
  rotate_rows(S.Xq, mr, KP, kk, S.Z, HL, S.P);
  rotate_rows(S.V + lo * KP, nr, KP, kk, S.Z, HL, S.P);  // only my rows are written out
  for (int c = tid; c < kk; c += kSvdNT) {
    double s = 0.0;
    for (int i = 0; i < mr; ++i) s = fma(S.Xq[i * KP + c], S.Xq[i * KP + c], s);
    S.red[c] = s;
  }
  cluster_sum(cl, S, kk);
  if (tid < kk) S.lam[tid] = sqrt(S.rout[tid]);  // sigma
  __syncthreads();
  const double smax = S.lam[0];
  // ---- 8. outputs
  T* Wr = reinterpret_cast<T*>(a.Wr);
  T* PI = reinterpret_cast<T*>(a.PI);
  T* VS = reinterpret_cast<T*>(a.VS);
  T* QJ = reinterpret_cast<T*>(a.QJ);
  if (q == 0 && tid < r) {
    const int c = tid;
    double sg = 0.0, iv = 0.0;
    if (c < reff) {
      sg = S.lam[c];
      if (smax > 0.0 && sg > 1e-12 * smax) iv = 1.0 / sg;
    }
    a.sigma[c] = sg;
    a.inv[c] = iv;
  }
  int ndef = 0;
  for (int c = 0; c < reff; ++c) ndef += !(S.lam[c] > 1e-14 * smax && S.lam[c] > 0.0);
  for (int e = tid; e < mr * r; e += kSvdNT) {
    const int i = e / r, c = e - i * r;
    double wv = 0.0, piv = 0.0;
    if (c < reff) {
      const double sg = S.lam[c];
      const double y = S.Xq[i * KP + c];
      if (sg > 1e-14 * smax && sg > 0.0) wv = y / sg;
      const double iv = (smax > 0.0 && sg > 1e-12 * smax) ? 1.0 / sg : 0.0;
      piv = y * iv;
    }
    a.W[(int64_t)(mlo + i) * r + c] = wv;
    PI[(int64_t)(mlo + i) * r + c] = (T)piv;
  }
  for (int e = tid; e < nr * r; e += kSvdNT) {
    const int i = e / r, c = e - i * r;
    double vv = 0.0, vs = 0.0;
    if (c < reff) {
      vv = S.V[(lo + i) * KP + c];
      const double sg = S.lam[c];
      const double iv = (smax > 0.0 && sg > 1e-12 * smax) ? 1.0 / sg : 0.0;
      vs = vv * iv;
    }
    a.V[(int64_t)(lo + i) * r + c] = vv;
    VS[(int64_t)(lo + i) * r + c] = (T)vs;
  }
  __threadfence();
  cl.sync();
  if (ndef > 0 && q == 0) {
    // CGS2 completion of W's deficient columns with unit-vector candidates
    double* dots = S.red;
    for (int c = 0; c < reff; ++c) {
      const double sg = S.lam[c];
      if (sg > 1e-14 * smax && sg > 0.0) continue;
      for (int cand = 0; cand < m; ++cand) {
        const int e0 = (c + cand) % m;
        for (int i = tid; i < m; i += kSvdNT) a.W[(int64_t)i * r + c] = (i == e0) ? 1.0 : 0.0;
        __syncthreads();
        for (int pass = 0; pass < 2; ++pass) {
          for (int k2 = w; k2 < reff; k2 += kSvdNW) {
            double d = 0.0;
            if (k2 != c) {
              for (int i = lane; i < m; i += 32) d = fma(a.W[(int64_t)i * r + k2], a.W[(int64_t)i * r + c], d);
              d = warp_sum(d);
            }
            if (lane == 0) dots[k2] = d;
          }
          __syncthreads();
          for (int i = tid; i < m; i += kSvdNT) {
            double v = a.W[(int64_t)i * r + c];
            for (int k2 = 0; k2 < reff; ++k2) v = fma(-dots[k2], a.W[(int64_t)i * r + k2], v);
            a.W[(int64_t)i * r + c] = v;
          }
          __syncthreads();
        }
        double p = 0.0;
        for (int i = tid; i < m; i += kSvdNT) p = fma(a.W[(int64_t)i * r + c], a.W[(int64_t)i * r + c], p);
        p = warp_sum(p);
        if (lane == 0) S.ws[w] = p;
        __syncthreads();
        double nrm = 0.0;
        for (int i = 0; i < kSvdNW; ++i) nrm += S.ws[i];
        __syncthreads();
        if (nrm > 1e-8) {
          const double inv = 1.0 / sqrt(nrm);
          for (int i = tid; i < m; i += kSvdNT) a.W[(int64_t)i * r + c] *= inv;
          __syncthreads();
          break;
        }
      }
    }
    __threadfence();
  }
  cl.sync();
  for (int e = tid; e < mr * r; e += kSvdNT) {
    const int i = e / r, c = e - i * r;
    Wr[(int64_t)(mlo + i) * r + c] = (T)a.W[(int64_t)(mlo + i) * r + c];
  }
  // QJ(j, c) = sum_i W(i, c) U(i, j) for my n-rows: lanes over j (coalesced U rows)
  for (int j0 = lo + w * 32; j0 < hi; j0 += kSvdNW * 32) {
    const int j = j0 + lane;
    double acc[kMaxRank];
#pragma unroll
    for (int c = 0; c < kMaxRank; ++c) acc[c] = 0.0;
    if (j < hi) {
      for (int i = 0; i < m; ++i) {
        const double u = a.U[(int64_t)i * a.ldu + j];
        const double* wrow = a.W + (int64_t)i * r;
#pragma unroll
        for (int c = 0; c < kMaxRank; ++c)
          if (c < r) acc[c] = fma(wrow[c], u, acc[c]);
      }
#pragma unroll
      for (int c = 0; c < kMaxRank; ++c)
        if (c < r) QJ[(int64_t)j * r + c] = (T)acc[c];
    }
  }
}

size_t svd_smem_bytes(int n, int m, int kk, int cs) {
  return (size_t)svd_layout(n, m, kk, cs).total * sizeof(double);
}

// ~32 rows of G per CTA, more CTAs (up to 16) until G's row block fits in
// shared memory next to the replicated V.
int svd_pick_cluster(int n, int m, int kk) {
  int cs = (n + 31) / 32;
  if (cs < 1) cs = 1;
  if (cs > 16) cs = 16;
  while (cs < 16 && !svd_layout(n, m, kk, cs).gq_smem) ++cs;
  return cs;
}

template <typename T>
cudaError_t launch_svd(const SvdArgs& a, int cs, cudaStream_t st) {
  dim3 gg((unsigned)((a.n + 31) / 32), (unsigned)((a.n + 31) / 32));
  gram_kernel<<<gg, 256, 0, st>>>(a.U, a.ldu, a.m, a.n, const_cast<double*>(a.G), a.ldg, a.done);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t smem = svd_smem_bytes(a.n, a.m, a.kk, cs);
  static bool attr = false;
  if (!attr) {
    e = cudaFuncSetAttribute(svd_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(svd_kernel<T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cs, 1, 1);
  cfg.blockDim = dim3(kSvdNT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = cs;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, svd_kernel<T>, a);
}

template cudaError_t launch_svd<float>(const SvdArgs&, int, cudaStream_t);
template cudaError_t launch_svd<double>(const SvdArgs&, int, cudaStream_t);

}  // namespace ircur
