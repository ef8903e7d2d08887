// Exact top-r SVD / pseudo-inverse of the |I| x |J| core (sm_100a).
//
// Replaces matcore.truncated_svd (LAPACK gesdd, matcore.py:128-139) and
// PinvFactor.from_svd (cutoff sigma > 1e-12 sigma_max, matcore.py:156-165).
// Only the top k = min(r, |I|, |J|) triplets are consumed, so instead of a
// full dense SVD the core is factorised by block subspace iteration on the
// Gram matrix G = U^T U with Rayleigh-Ritz extraction, warm-started from the
// previous iterate's Q(:,J), iterated until the Ritz residuals reach fp64
// round-off, then finished by a Rayleigh-Ritz step on U itself (so small
// singular values are resolved in absolute fp64 accuracy and the pinv cutoff
// behaves like LAPACK's).  Block size kk = min(2r, |I|, |J|, 32).
//
// Layout: one thread-block cluster per core; CTA q owns rows [lo_q, hi_q) of
// the n x kk block V; the full V is replicated in every CTA's shared memory;
// small cluster-wide sums go through DSMEM in a fixed rank order, so every
// CTA holds bitwise-identical reduced values and takes identical branches.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "ircur_common.cuh"
#include "launchers.cuh"

namespace cg = cooperative_groups;

namespace ircur {

constexpr int kSvdNT = 512;
constexpr int kKMax = 32;
constexpr int kHLd = kKMax + 1;

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

// ------------------------------------------------------------ helpers
__device__ __forceinline__ double hash_uniform(uint64_t a, uint64_t b) {
  uint64_t z = a * 0x9E3779B97F4A7C15ull ^ (b + 0x632BE59BD9B4E019ull) * 0xBF58476D1CE4E5B9ull;
  z ^= z >> 31; z *= 0x94D049BB133111EBull; z ^= z >> 29; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 32;
  return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;  // [-1, 1)
}

struct SvdSmem {
  double* V;      // n x KP (full, replicated)
  double* Bq;     // per x KP
  double* Xq;     // per x KP (scratch rows)
  double* H;      // 32 x 33
  double* Z;      // 32 x 33
  double* red;    // partial sums exposed to the cluster (kKMax*kHLd + 2*kKMax)
  double* rout;   // reduced sums
  double* lam;    // 32
  double* cs;     // 64 (rotation c,s per pair)
  double* wsum;   // kSvdNT/32 * kKMax (warp partials)
  int* perm;      // 32
  int* flags;     // 8
};

__device__ __forceinline__ void cluster_sum(cg::cluster_group& cl, SvdSmem& S, int L) {
  cl.sync();
  const int CS = (int)cl.num_blocks();
  for (int e = threadIdx.x; e < L; e += kSvdNT) {
    double s = *cl.map_shared_rank(S.red + e, 0);
    for (int q = 1; q < CS; ++q) s += *cl.map_shared_rank(S.red + e, q);
    S.rout[e] = s;
  }
  cl.sync();
}

// Cyclic Jacobi eigen-decomposition of the symmetric kk x kk matrix in S.H
// (round-robin parallel ordering).  On exit S.lam holds eigenvalues sorted in
// decreasing order and S.Z the matching eigenvectors (columns).  Executed
// redundantly and identically by every CTA of the cluster.
__device__ void jacobi_eig(SvdSmem& S, int kk) {
  const int tid = threadIdx.x;
  for (int e = tid; e < kk * kHLd; e += kSvdNT) {
    const int i = e / kHLd, j = e - i * kHLd;
    S.Z[e] = (i == j) ? 1.0 : 0.0;
  }
  const int np = (kk + 1) / 2;
  const int nply = 2 * np;  // even number of players
  __syncthreads();
  // rotation threshold: absolute, a few ulps of the largest diagonal entry
  // (a relative test on tiny/zero eigenvalues never settles under round-off)
  double scale = 0.0;
  for (int i = 0; i < kk; ++i) scale = fmax(scale, fabs(S.H[i * kHLd + i]));
  const double thr = 4e-16 * scale;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (tid == 0) S.flags[0] = 0;
    __syncthreads();
    for (int rd = 0; rd < nply - 1; ++rd) {
      if (tid < np) {
        int pa = tid == 0 ? 0 : ((tid - 1 + rd) % (nply - 1)) + 1;
        int pb = ((nply - 2 - tid + rd) % (nply - 1)) + 1;
        if (tid == 0) pb = ((nply - 2 + rd) % (nply - 1)) + 1;
        int p = min(pa, pb), q = max(pa, pb);
        double c = 1.0, s = 0.0;
        if (q < kk) {
          const double hpq = S.H[p * kHLd + q];
          const double hpp = S.H[p * kHLd + p], hqq = S.H[q * kHLd + q];
          if (fabs(hpq) > 1e-300 && fabs(hpq) > thr) {
            const double tau = (hqq - hpp) / (2.0 * hpq);
            const double t = fabs(tau) > 1e150 ? 0.5 / tau
                                               : (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            S.flags[0] = 1;
          }
        }
        S.cs[4 * tid] = c;
        S.cs[4 * tid + 1] = s;
        reinterpret_cast<int*>(S.cs)[8 * tid + 4] = p;  // pack p,q after c,s
        reinterpret_cast<int*>(S.cs)[8 * tid + 5] = q;
      }
      __syncthreads();
      // rows: H <- J^T H
      for (int e = tid; e < np * kk; e += kSvdNT) {
        const int pr = e / kk, j = e - pr * kk;
        const int p = reinterpret_cast<int*>(S.cs)[8 * pr + 4], q = reinterpret_cast<int*>(S.cs)[8 * pr + 5];
        const double c = S.cs[4 * pr], s = S.cs[4 * pr + 1];
        if (q < kk && s != 0.0) {
          const double hp = S.H[p * kHLd + j], hq = S.H[q * kHLd + j];
          S.H[p * kHLd + j] = c * hp - s * hq;
          S.H[q * kHLd + j] = s * hp + c * hq;
        }
      }
      __syncthreads();
      // columns: H <- H J, Z <- Z J
      for (int e = tid; e < np * kk; e += kSvdNT) {
        const int pr = e / kk, i = e - pr * kk;
        const int p = reinterpret_cast<int*>(S.cs)[8 * pr + 4], q = reinterpret_cast<int*>(S.cs)[8 * pr + 5];
        const double c = S.cs[4 * pr], s = S.cs[4 * pr + 1];
        if (q < kk && s != 0.0) {
          double hp = S.H[i * kHLd + p], hq = S.H[i * kHLd + q];
          S.H[i * kHLd + p] = c * hp - s * hq;
          S.H[i * kHLd + q] = s * hp + c * hq;
          hp = S.Z[i * kHLd + p];
          hq = S.Z[i * kHLd + q];
          S.Z[i * kHLd + p] = c * hp - s * hq;
          S.Z[i * kHLd + q] = s * hp + c * hq;
        }
      }
      __syncthreads();
    }
    if (S.flags[0] == 0) break;
    __syncthreads();
  }
  // sort eigenvalues (descending, stable) via rank computation
  if (tid < kk) {
    const double li = S.H[tid * kHLd + tid];
    int rk = 0;
    for (int j = 0; j < kk; ++j) {
      const double lj = S.H[j * kHLd + j];
      rk += (lj > li) || (lj == li && j < tid);
    }
    S.perm[rk] = tid;
  }
  __syncthreads();
  if (tid < kk) S.lam[tid] = S.H[S.perm[tid] * kHLd + S.perm[tid]];
  // permute Z columns into S.H (as scratch), then copy back
  for (int e = tid; e < kk * kk; e += kSvdNT) {
    const int i = e / kk, j = e - i * kk;
    S.H[i * kHLd + j] = S.Z[i * kHLd + S.perm[j]];
  }
  __syncthreads();
  for (int e = tid; e < kk * kk; e += kSvdNT) {
    const int i = e / kk, j = e - i * kk;
    S.Z[i * kHLd + j] = S.H[i * kHLd + j];
  }
  __syncthreads();
}

// rows X (nr x KP) <- X * Z(:, 0:kk) in place, row-parallel (uses Xs scratch row per thread)
__device__ __forceinline__ void rotate_rows(double* X, int nr, int KP, int kk, const double* Z, double* tmp) {
  // tmp: nr x KP scratch
  for (int e = threadIdx.x; e < nr * kk; e += kSvdNT) {
    const int i = e / kk, c = e - i * kk;
    double s = 0.0;
    for (int j = 0; j < kk; ++j) s = fma(X[i * KP + j], Z[j * kHLd + c], s);
    tmp[i * KP + c] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nr * kk; e += kSvdNT) {
    const int i = e / kk, c = e - i * kk;
    X[i * KP + c] = tmp[i * KP + c];
  }
  __syncthreads();
}

// Block-local CGS2 with random replacement on the FULL V (n x kk), executed
// identically by every CTA (no cluster communication).
__device__ void orthonormalize_full(SvdSmem& S, int n, int KP, int kk, uint64_t salt) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  constexpr int NW = kSvdNT / 32;
  for (int c = 0; c < kk; ++c) {
    for (int attempt = 0; attempt < 4; ++attempt) {
      // original norm
      double p = 0.0;
      for (int j = tid; j < n; j += kSvdNT) p = fma(S.V[j * KP + c], S.V[j * KP + c], p);
      p = warp_sum(p);
      if (lane == 0) S.wsum[w] = p;
      __syncthreads();
      double nrm0 = 0.0;
      for (int i = 0; i < NW; ++i) nrm0 += S.wsum[i];
      __syncthreads();
      for (int pass = 0; pass < 2; ++pass) {
        // dots with previous columns: warp w handles k = w, w+NW, ...
        for (int k = w; k < c; k += NW) {
          double d = 0.0;
          for (int j = lane; j < n; j += 32) d = fma(S.V[j * KP + k], S.V[j * KP + c], d);
          d = warp_sum(d);
          if (lane == 0) S.lam[k] = d;
        }
        __syncthreads();
        for (int j = tid; j < n; j += kSvdNT) {
          double v = S.V[j * KP + c];
          for (int k = 0; k < c; ++k) v = fma(-S.lam[k], S.V[j * KP + k], v);
          S.V[j * KP + c] = v;
        }
        __syncthreads();
      }
      p = 0.0;
      for (int j = tid; j < n; j += kSvdNT) p = fma(S.V[j * KP + c], S.V[j * KP + c], p);
      p = warp_sum(p);
      if (lane == 0) S.wsum[w] = p;
      __syncthreads();
      double nrm = 0.0;
      for (int i = 0; i < NW; ++i) nrm += S.wsum[i];
      __syncthreads();
      if (nrm > 1e-20 * nrm0 && nrm > 1e-280) {
        const double inv = 1.0 / sqrt(nrm);
        for (int j = tid; j < n; j += kSvdNT) S.V[j * KP + c] *= inv;
        __syncthreads();
        break;
      }
      // replace with a fresh pseudo-random column and retry
      for (int j = tid; j < n; j += kSvdNT)
        S.V[j * KP + c] = hash_uniform(salt + 1000003ull * (uint64_t)(attempt + 1), (uint64_t)j * 64 + c);
      __syncthreads();
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(kSvdNT, 1) svd_kernel(const __grid_constant__ SvdArgs a) {
  if (a.done && *a.done) return;
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks();
  const int q = (int)cl.block_rank();
  const int n = a.n, m = a.m, r = a.r, kk = a.kk;
  const int KP = kk | 1;
  const int reff = min(r, min(m, n));
  const int per = (n + CS - 1) / CS;
  const int lo = min(n, q * per), hi = min(n, lo + per), nr = hi - lo;
  const int mper = (m + CS - 1) / CS;
  const int mlo = min(m, q * mper), mhi = min(m, mlo + mper), mr = mhi - mlo;
  const int rowsmax = max(per, mper);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  constexpr int NW = kSvdNT / 32;

  extern __shared__ __align__(16) double svsm[];
  SvdSmem S;
  S.V = svsm;
  S.Bq = S.V + (size_t)n * KP;
  S.Xq = S.Bq + (size_t)rowsmax * KP;
  S.H = S.Xq + (size_t)rowsmax * KP;
  S.Z = S.H + kKMax * kHLd;
  S.red = S.Z + kKMax * kHLd;
  S.rout = S.red + (kKMax * kHLd + 2 * kKMax);
  S.lam = S.rout + (kKMax * kHLd + 2 * kKMax);
  S.cs = S.lam + kKMax;
  S.wsum = S.cs + 4 * kKMax;
  S.perm = reinterpret_cast<int*>(S.wsum + NW * kKMax);
  S.flags = S.perm + kKMax;

  // ---- 0. starting block: warm columns (previous Q(:,J)) + pseudo-random
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
    // ---- 1. B_q = G(lo:hi, :) V   (warp per row, lanes over the inner index)
    for (int i = w; i < nr; i += NW) {
      double acc[kKMax];
#pragma unroll
      for (int c = 0; c < kKMax; ++c) acc[c] = 0.0;
      const double* grow = a.G + (int64_t)(lo + i) * a.ldg;
      for (int j = lane; j < n; j += 32) {
        const double g = grow[j];
        const double* vr = S.V + j * KP;
#pragma unroll
        for (int c = 0; c < kKMax; ++c)
          if (c < kk) acc[c] = fma(g, vr[c], acc[c]);
      }
#pragma unroll
      for (int c = 0; c < kKMax; ++c) {
        if (c < kk) {
          const double s = warp_sum(acc[c]);
          if (lane == 0) S.Bq[i * KP + c] = s;
        }
      }
    }
    __syncthreads();
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
      S.H[c1 * kHLd + c2] = 0.5 * (S.rout[c1 * kk + c2] + S.rout[c2 * kk + c1]);
    }
    __syncthreads();
    jacobi_eig(S, kk);
    // ---- 3. Ritz rotation of my rows: Xq <- V_q Z, then V_q <- B_q Z
    for (int e = tid; e < nr * kk; e += kSvdNT) {
      const int i = e / kk, c = e - i * kk;
      double sv = 0.0;
      for (int j = 0; j < kk; ++j) sv = fma(S.V[(lo + i) * KP + j], S.Z[j * kHLd + c], sv);
      S.Xq[i * KP + c] = sv;
    }
    __syncthreads();
    // rotated B (separate pass so Bq reads above are complete)
    for (int e = tid; e < nr * kk; e += kSvdNT) {
      const int i = e / kk, c = e - i * kk;
      double sb = 0.0;
      for (int j = 0; j < kk; ++j) sb = fma(S.Bq[i * KP + j], S.Z[j * kHLd + c], sb);
      S.V[(lo + i) * KP + c] = sb;  // V rows of mine now hold B Z (V Z kept in Xq)
    }
    __syncthreads();
    // ---- 4. residuals ||B z_c - lam_c V z_c||^2 and the next block
    //      Vn_c = B z_c / lam_c  (significant lam) or V z_c (negligible lam)
    const double lam0 = S.lam[0];
    for (int e = tid; e < kk * kk + kk; e += kSvdNT) S.red[e] = 0.0;
    __syncthreads();
    if (tid < kk) {
      const int c = tid;
      const double lc = S.lam[c];
      double rs = 0.0;
      for (int i = 0; i < nr; ++i) {
        const double d = S.V[(lo + i) * KP + c] - lc * S.Xq[i * KP + c];
        rs = fma(d, d, rs);
      }
      S.red[kk * kk + c] = rs;
    }
    __syncthreads();
    const double sig_thr = 1e-10 * fabs(lam0);
    for (int e = tid; e < nr * kk; e += kSvdNT) {
      const int i = e / kk, c = e - i * kk;
      const double lc = S.lam[c];
      double v = S.Xq[i * KP + c];
      if (lc > sig_thr && lc > 0.0) v = S.V[(lo + i) * KP + c] / lc;
      S.Bq[i * KP + c] = v;  // Bq now holds the (un-orthonormalised) next block rows
    }
    __syncthreads();
    for (int e = tid; e < kk * kk; e += kSvdNT) {
      const int c1 = e / kk, c2 = e - c1 * kk;
      double s = 0.0;
      for (int i = 0; i < nr; ++i) s = fma(S.Bq[i * KP + c1], S.Bq[i * KP + c2], s);
      S.red[e] = s;
    }
    cluster_sum(cl, S, kk * kk + kk);
    // convergence (identical in all CTAs)
    double resmax = 0.0;
    for (int c = 0; c < reff; ++c) resmax = fmax(resmax, sqrt(S.rout[kk * kk + c]));
    const bool conv = !(lam0 > 0.0) || resmax <= a.tol * lam0;
    if (resmax > 0.5 * prev_res) ++stall; else stall = 0;
    prev_res = resmax;
    const bool give_up = (stall >= 3 && resmax <= 1e-11 * lam0);
    if (conv || give_up || step + 1 == a.maxsteps) {
      // final block = current Ritz vectors V Z (in Xq) -> gather into V
      for (int e = tid; e < nr * kk; e += kSvdNT) {
        const int i = e / kk, c = e - i * kk;
        a.scratch[(int64_t)(lo + i) * kKMax + c] = S.Xq[i * KP + c];
      }
      break;
    }
    // ---- 5. CholQR of the next block: Gram (in rout) = L L^T; Vn <- Vn L^{-T}
    if (w == 0) {
      // Cholesky of the Gram (in rout) into S.H (lower), one warp
      int ok = 1;
      for (int j = 0; j < kk; ++j) {
        double p = 0.0;
        for (int k2 = lane; k2 < j; k2 += 32) p = fma(S.H[j * kHLd + k2], S.H[j * kHLd + k2], p);
        p = warp_sum(p);
        double d = S.rout[j * kk + j] - p;
        if (!(d > 0.0)) { ok = 0; d = 1e-300; }
        const double ljj = sqrt(d);
        for (int i = j + 1 + lane; i < kk; i += 32) {
          double s2 = S.rout[i * kk + j];
          for (int k2 = 0; k2 < j; ++k2) s2 = fma(-S.H[i * kHLd + k2], S.H[j * kHLd + k2], s2);
          S.H[i * kHLd + j] = s2 / ljj;
        }
        if (lane == 0) S.H[j * kHLd + j] = ljj;
        __syncwarp();
      }
      if (lane == 0) S.flags[1] = ok;
    }
    __syncthreads();
    for (int i = tid; i < nr; i += kSvdNT) {
      // solve x L^T = v  (forward substitution over columns)
      for (int c = 0; c < kk; ++c) {
        double s = S.Bq[i * KP + c];
        for (int k2 = 0; k2 < c; ++k2) s -= S.Bq[i * KP + k2] * S.H[c * kHLd + k2];
        S.Bq[i * KP + c] = s / S.H[c * kHLd + c];
      }
    }
    __syncthreads();
    // ---- 6. all-gather the new block through global scratch
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
    if (S.flags[1] == 0) {
      // Cholesky broke down (should not happen: Gram = I + E^T E); restore
      // orthonormality with the robust block-local CGS2.
      orthonormalize_full(S, n, KP, kk, a.salt + 77ull * (step + 1));
    }
    cl.sync();  // scratch may be overwritten next step only after all copies
  }
  // gather the final Ritz block
  __threadfence();
  cl.sync();
  for (int e = tid; e < n * kk; e += kSvdNT) {
    const int j = e / kk, c = e - j * kk;
    S.V[j * KP + c] = a.scratch[(int64_t)j * kKMax + c];
  }
  __syncthreads();
  if (q == 0 && tid == 0 && a.steps_out) *a.steps_out = step + 1;

  // ---- 7. Rayleigh-Ritz on U itself: Y = U V (my m-rows), H2 = Y^T Y
  for (int i = w; i < mr; i += NW) {
    double acc[kKMax];
#pragma unroll
    for (int c = 0; c < kKMax; ++c) acc[c] = 0.0;
    const double* urow = a.U + (int64_t)(mlo + i) * a.ldu;
    for (int j = lane; j < n; j += 32) {
      const double u = urow[j];
      const double* vr = S.V + j * KP;
#pragma unroll
      for (int c = 0; c < kKMax; ++c)
        if (c < kk) acc[c] = fma(u, vr[c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < kKMax; ++c) {
      if (c < kk) {
        const double s = warp_sum(acc[c]);
        if (lane == 0) S.Xq[i * KP + c] = s;
      }
    }
  }
  __syncthreads();
  for (int e = tid; e < kk * kk; e += kSvdNT) {
    const int c1 = e / kk, c2 = e - c1 * kk;
    double s = 0.0;
    for (int i = 0; i < mr; ++i) s = fma(S.Xq[i * KP + c1], S.Xq[i * KP + c2], s);
    S.red[e] = s;
  }
  cluster_sum(cl, S, kk * kk);
  for (int e = tid; e < kk * kk; e += kSvdNT) {
    const int c1 = e / kk, c2 = e - c1 * kk;
    S.H[c1 * kHLd + c2] = 0.5 * (S.rout[c1 * kk + c2] + S.rout[c2 * kk + c1]);
  }
  __syncthreads();
  jacobi_eig(S, kk);
  // Y_q <- Y_q Z ; V (full) <- V Z
  rotate_rows(S.Xq, mr, KP, kk, S.Z, S.Bq);
  rotate_rows(S.V + lo * KP, nr, KP, kk, S.Z, S.Bq);  // only my rows are written out
  // sigma_c = ||Y_c|| (cluster sum of column norms)
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
  // deficient columns need an orthonormal completion of W (rare)
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
    for (int c = 0; c < reff; ++c) {
      const double sg = S.lam[c];
      if (sg > 1e-14 * smax && sg > 0.0) continue;
      for (int cand = 0; cand < m; ++cand) {
        const int e0 = (c + cand) % m;
        for (int i = tid; i < m; i += kSvdNT) a.W[(int64_t)i * r + c] = (i == e0) ? 1.0 : 0.0;
        __syncthreads();
        for (int pass = 0; pass < 2; ++pass) {
          for (int k2 = w; k2 < reff; k2 += NW) {
            double d = 0.0;
            if (k2 != c) {
              for (int i = lane; i < m; i += 32) d = fma(a.W[(int64_t)i * r + k2], a.W[(int64_t)i * r + c], d);
              d = warp_sum(d);
            }
            if (lane == 0) S.cs[k2] = (k2 == c) ? 0.0 : d;
          }
          __syncthreads();
          for (int i = tid; i < m; i += kSvdNT) {
            double v = a.W[(int64_t)i * r + c];
            for (int k2 = 0; k2 < reff; ++k2) v = fma(-S.cs[k2], a.W[(int64_t)i * r + k2], v);
            a.W[(int64_t)i * r + c] = v;
          }
          __syncthreads();
        }
        double p = 0.0;
        for (int i = tid; i < m; i += kSvdNT) p = fma(a.W[(int64_t)i * r + c], a.W[(int64_t)i * r + c], p);
        p = warp_sum(p);
        if (lane == 0) S.wsum[w] = p;
        __syncthreads();
        double nrm = 0.0;
        for (int i = 0; i < NW; ++i) nrm += S.wsum[i];
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
  // Wr (storage precision copy of W) for my m-rows
  for (int e = tid; e < mr * r; e += kSvdNT) {
    const int i = e / r, c = e - i * r;
    Wr[(int64_t)(mlo + i) * r + c] = (T)a.W[(int64_t)(mlo + i) * r + c];
  }
  // QJ(j, c) = sum_i W(i, c) U(i, j) for my n-rows: lanes over j (coalesced U rows)
  for (int j0 = lo + w * 32; j0 < hi; j0 += NW * 32) {
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
  const int KP = kk | 1;
  const int per = (n + cs - 1) / cs, mper = (m + cs - 1) / cs;
  const int rowsmax = per > mper ? per : mper;
  size_t d = (size_t)n * KP + 2 * (size_t)rowsmax * KP + 2 * kKMax * kHLd +
             2 * (kKMax * kHLd + 2 * kKMax) + kKMax + 4 * kKMax + (kSvdNT / 32) * kKMax;
  return d * sizeof(double) + 2 * kKMax * sizeof(int) + 64;
}

template <typename T>
cudaError_t launch_svd(const SvdArgs& a, int cs, cudaStream_t st) {
  // Gram first
  dim3 gg((unsigned)((a.n + 31) / 32), (unsigned)((a.n + 31) / 32));
  gram_kernel<<<gg, 256, 0, st>>>(a.U, a.ldu, a.m, a.n, const_cast<double*>(a.G), a.ldg, a.done);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t smem = svd_smem_bytes(a.n, a.m, a.kk, cs);
  static size_t attr_smem = 0;
  if (smem > attr_smem) {
    e = cudaFuncSetAttribute(svd_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute(svd_kernel<T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr_smem = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cs, 1, 1);
  cfg.blockDim = dim3(kSvdNT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, svd_kernel<T>, a);
}

template cudaError_t launch_svd<float>(const SvdArgs&, int, cudaStream_t);
template cudaError_t launch_svd<double>(const SvdArgs&, int, cudaStream_t);

}  // namespace ircur
