// CUR -> compact SVD on the device (reference: convert.py:21-48).
//
// The reference takes thin QRs of C (n1 x |J|) and R^T (n2 x |I|) and the
// SVD of the |J| x |I| middle factor.  On the device the low-rank iterate
// is already held as L = P Q with P = C V Sigma^+ (n1 x r) and Q = W_r^T R
// (r x n2) (the same product in exact arithmetic), so the compact SVD only
// needs r-wide work:
//   Gp = P^T P, Gq = Q Q^T                (streaming Gram kernels, fp64)
//   Gp = Rp^T Rp, Gq = Rq^T Rq            (Cholesky, one CTA)
//   M = Rp Rq^T = Wm S Vm^T               (one-sided Jacobi SVD, one CTA)
//   W = P (Rp^-1 Wm), V = Q^T (Rq^-1 Vm)  (streaming apply kernels)
// and singular values below 1e-14 sigma_max are dropped (COMPACT_DROP,
// convert.py:18).  Every reduction has a fixed order (deterministic).
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/ircur_b200.h"
#include "ircur_common.cuh"

namespace ircur {

constexpr int kCvMaxR = 16;
constexpr int kCvNT = 256;
constexpr int kCvBlocks = 256;  // partial Gram blocks (fixed: deterministic sum order)

// partial[b][a*k + c] = sum_{x in block b's stride} X[a][x] X[c][x]
template <typename T>
__global__ void __launch_bounds__(kCvNT) tall_gram_kernel(const T* __restrict__ X, int64_t ldx, int64_t n, int k,
                                                          double* __restrict__ partial) {
  __shared__ double sh[kCvNT / 32][kCvMaxR * kCvMaxR];
  double acc[kCvMaxR * (kCvMaxR + 1) / 2];
  for (int i = 0; i < k * (k + 1) / 2; ++i) acc[i] = 0.0;
  for (int64_t x = (int64_t)blockIdx.x * kCvNT + threadIdx.x; x < n; x += (int64_t)gridDim.x * kCvNT) {
    double v[kCvMaxR];
    for (int a = 0; a < k; ++a) v[a] = (double)X[a * ldx + x];
    int e = 0;
    for (int a = 0; a < k; ++a)
      for (int c = a; c < k; ++c, ++e) acc[e] = fma(v[a], v[c], acc[e]);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int e = 0;
  for (int a = 0; a < k; ++a)
    for (int c = a; c < k; ++c, ++e) {
      const double s = warp_sum(acc[e]);
      if (lane == 0) sh[w][a * k + c] = s;
    }
  __syncthreads();
  for (int i = threadIdx.x; i < k * k; i += kCvNT) {
    const int a = i / k, c = i - a * k;
    double s = 0.0;
    if (c >= a)
      for (int ww = 0; ww < kCvNT / 32; ++ww) s += sh[ww][i];
    partial[(int64_t)blockIdx.x * k * k + i] = s;
  }
}

// Small dense part on one CTA (thread 0 does the O(r^3) work; r <= 16).
// Outputs A1 = Rp^-1 Wm, A2 = Rq^-1 Vm (k x k, fp64), sigma (k, descending),
// and the count kept after the compact drop.
__global__ void __launch_bounds__(32) small_svd_kernel(const double* __restrict__ pp, const double* __restrict__ pq,
                                                       int nblk, int k, double* A1, double* A2, double* sigma,
                                                       int* kept, int* status) {
  if (threadIdx.x != 0) return;
  double Gp[kCvMaxR][kCvMaxR], Gq[kCvMaxR][kCvMaxR];
  for (int a = 0; a < k; ++a)
    for (int c = a; c < k; ++c) {
      double sp = 0.0, sq = 0.0;
      for (int b = 0; b < nblk; ++b) {  // fixed block order
        sp += pp[(int64_t)b * k * k + a * k + c];
        sq += pq[(int64_t)b * k * k + a * k + c];
      }
      Gp[a][c] = Gp[c][a] = sp;
      Gq[a][c] = Gq[c][a] = sq;
    }
  // upper Cholesky G = R^T R (a zero pivot leaves a zero row: rank-deficient factor)
  auto chol = [&](double (*G)[kCvMaxR], double (*Rm)[kCvMaxR]) {
    for (int a = 0; a < k; ++a)
      for (int c = 0; c < k; ++c) Rm[a][c] = 0.0;
    for (int j = 0; j < k; ++j) {
      double d = G[j][j];
      for (int i = 0; i < j; ++i) d -= Rm[i][j] * Rm[i][j];
      const double rjj = d > 0.0 ? sqrt(d) : 0.0;
      Rm[j][j] = rjj;
      for (int c = j + 1; c < k; ++c) {
        double s = G[j][c];
        for (int i = 0; i < j; ++i) s -= Rm[i][j] * Rm[i][c];
        Rm[j][c] = rjj > 0.0 ? s / rjj : 0.0;
      }
    }
  };
  double Rp[kCvMaxR][kCvMaxR], Rq[kCvMaxR][kCvMaxR];
  chol(Gp, Rp);
  chol(Gq, Rq);
  // M = Rp Rq^T, then one-sided Jacobi on the columns of M (M = Wm S Vm^T)
  double Mx[kCvMaxR][kCvMaxR], Vm[kCvMaxR][kCvMaxR];
  for (int a = 0; a < k; ++a)
    for (int c = 0; c < k; ++c) {
      double s = 0.0;
      for (int i = 0; i < k; ++i) s += Rp[a][i] * Rq[c][i];
      Mx[a][c] = s;
      Vm[a][c] = a == c ? 1.0 : 0.0;
    }
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < k; ++p)
      for (int q = p + 1; q < k; ++q) {
        double app = 0.0, aqq = 0.0, apq = 0.0;
        for (int i = 0; i < k; ++i) {
          app += Mx[i][p] * Mx[i][p];
          aqq += Mx[i][q] * Mx[i][q];
          apq += Mx[i][p] * Mx[i][q];
        }
        if (apq == 0.0 || fabs(apq) <= 1e-17 * sqrt(app * aqq)) continue;
        off = fmax(off, fabs(apq) / sqrt(app * aqq));
        const double zeta = (aqq - app) / (2.0 * apq);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int i = 0; i < k; ++i) {
          const double mp = Mx[i][p], mq = Mx[i][q];
          Mx[i][p] = c * mp - s * mq;
          Mx[i][q] = s * mp + c * mq;
          const double vp = Vm[i][p], vq = Vm[i][q];
          Vm[i][p] = c * vp - s * vq;
          Vm[i][q] = s * vp + c * vq;
        }
      }
    if (off <= 1e-15) break;
  }
  // sigma = column norms, Wm = normalised columns; order by decreasing sigma
  double sg[kCvMaxR];
  int ord[kCvMaxR];
  for (int c = 0; c < k; ++c) {
    double s = 0.0;
    for (int i = 0; i < k; ++i) s += Mx[i][c] * Mx[i][c];
    sg[c] = sqrt(s);
    ord[c] = c;
  }
  for (int a = 1; a < k; ++a)  // insertion sort, ties by index
    for (int b = a; b > 0 && sg[ord[b]] > sg[ord[b - 1]]; --b) {
      const int t = ord[b];
      ord[b] = ord[b - 1];
      ord[b - 1] = t;
    }
  const double smax = k > 0 ? sg[ord[0]] : 0.0;
  int nk = 0;
  for (int c = 0; c < k; ++c)
    if (smax > 0.0 && sg[ord[c]] >= 1e-14 * smax) ++nk;
  // A1 = Rp^-1 Wm, A2 = Rq^-1 Vm by back substitution (upper triangular)
  for (int cc = 0; cc < k; ++cc) {
    const int c = ord[cc];
    const double sc = sg[c];
    double wm[kCvMaxR], vm[kCvMaxR], x1[kCvMaxR], x2[kCvMaxR];
    for (int i = 0; i < k; ++i) {
      wm[i] = sc > 0.0 ? Mx[i][c] / sc : 0.0;
      vm[i] = Vm[i][c];
    }
    // sign convention: the largest |entry| of Wm's column is positive
    int im = 0;
    for (int i = 1; i < k; ++i)
      if (fabs(wm[i]) > fabs(wm[im])) im = i;
    if (wm[im] < 0.0)
      for (int i = 0; i < k; ++i) {
        wm[i] = -wm[i];
        vm[i] = -vm[i];
      }
    for (int i = k - 1; i >= 0; --i) {
      double s1 = wm[i], s2 = vm[i];
      for (int j = i + 1; j < k; ++j) {
        s1 -= Rp[i][j] * x1[j];
        s2 -= Rq[i][j] * x2[j];
      }
      x1[i] = Rp[i][i] > 0.0 ? s1 / Rp[i][i] : 0.0;
      x2[i] = Rq[i][i] > 0.0 ? s2 / Rq[i][i] : 0.0;
    }
    for (int i = 0; i < k; ++i) {
      A1[i * k + cc] = x1[i];
      A2[i * k + cc] = x2[i];
    }
    sigma[cc] = sc;
  }
  *kept = nk;
  *status = 0;
}

// Y (n x k_out, row-major fp64) = X^T A[:, :k_out] for X given as k rows of length n
template <typename T>
__global__ void __launch_bounds__(kCvNT) tall_apply_kernel(const T* __restrict__ X, int64_t ldx, int64_t n, int k,
                                                           const double* __restrict__ A, const int* kept,
                                                           double* __restrict__ Y, int ldy) {
  __shared__ double sa[kCvMaxR * kCvMaxR];
  for (int i = threadIdx.x; i < k * k; i += kCvNT) sa[i] = A[i];
  __syncthreads();
  const int ko = *kept;
  for (int64_t x = (int64_t)blockIdx.x * kCvNT + threadIdx.x; x < n; x += (int64_t)gridDim.x * kCvNT) {
    double v[kCvMaxR];
    for (int a = 0; a < k; ++a) v[a] = (double)X[a * ldx + x];
    for (int c = 0; c < ko; ++c) {
      double s = 0.0;
      for (int a = 0; a < k; ++a) s = fma(v[a], sa[a * k + c], s);
      Y[x * ldy + c] = s;
    }
  }
}

}  // namespace ircur

using namespace ircur;

extern "C" int ircur_factors_to_svd(const void* Pt, int64_t ldp, const void* Q, int64_t ldq, int64_t n1, int64_t n2,
                                    int rank, int dtype, double* W, double* sigma, double* V, int* k_out,
                                    void* stream) {
  if (!Pt || !Q || !W || !sigma || !V || !k_out || rank < 1 || rank > kCvMaxR || n1 < 1 || n2 < 1 ||
      ldp < n1 || ldq < n2 || (dtype != IRCUR_F32 && dtype != IRCUR_F64))
    return IRCUR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int k = rank;
  double* buf = nullptr;  // partials (2 x blocks x k^2) | A1 | A2 | kept | status
  const size_t np = (size_t)kCvBlocks * k * k;
  const size_t bytes = (2 * np + 2 * (size_t)k * k) * sizeof(double) + 4 * sizeof(int);
  if (cudaMallocAsync(&buf, bytes, st) != cudaSuccess) return IRCUR_ENOMEM;
  double* pp = buf;
  double* pq = pp + np;
  double* A1 = pq + np;
  double* A2 = A1 + k * k;
  int* kept = reinterpret_cast<int*>(A2 + k * k);
  int* status = kept + 1;
  if (dtype == IRCUR_F32) {
    tall_gram_kernel<float><<<kCvBlocks, kCvNT, 0, st>>>((const float*)Pt, ldp, n1, k, pp);
    tall_gram_kernel<float><<<kCvBlocks, kCvNT, 0, st>>>((const float*)Q, ldq, n2, k, pq);
  } else {
    tall_gram_kernel<double><<<kCvBlocks, kCvNT, 0, st>>>((const double*)Pt, ldp, n1, k, pp);
    tall_gram_kernel<double><<<kCvBlocks, kCvNT, 0, st>>>((const double*)Q, ldq, n2, k, pq);
  }
  small_svd_kernel<<<1, 32, 0, st>>>(pp, pq, kCvBlocks, k, A1, A2, sigma, kept, status);
  if (dtype == IRCUR_F32) {
    tall_apply_kernel<float><<<kCvBlocks, kCvNT, 0, st>>>((const float*)Pt, ldp, n1, k, A1, kept, W, k);
    tall_apply_kernel<float><<<kCvBlocks, kCvNT, 0, st>>>((const float*)Q, ldq, n2, k, A2, kept, V, k);
  } else {
    tall_apply_kernel<double><<<kCvBlocks, kCvNT, 0, st>>>((const double*)Pt, ldp, n1, k, A1, kept, W, k);
    tall_apply_kernel<double><<<kCvBlocks, kCvNT, 0, st>>>((const double*)Q, ldq, n2, k, A2, kept, V, k);
  }
  int hk = 0;
  cudaMemcpyAsync(&hk, kept, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(buf, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return IRCUR_ECUDA;
  *k_out = hk;
  return IRCUR_OK;
}

// ------------------------------------------------------------------------
// The factored form of host C / R (convert.py:21-48 multiplies them out):
//   P^T (k x n1) = (C V diag(inv_sigma))^T,  Q (k x n2) = W^T R
// Both are tall-skinny products with k <= 16 outputs per row / column, HBM
// bound on reading C and R once: a block stages a 32 x 32 tile of C in
// shared memory (coalesced rows), each thread owns one row of C and k
// accumulators; for Q each thread owns one column of R (coalesced across
// the warp) and walks the rows with W^T in shared memory.  Fixed summation
// order (ascending j / i), so results are deterministic.
namespace ircur {
namespace {
constexpr int kCfRows = 128;  // rows of C per block
constexpr int kCfChunk = 32;  // columns of C per staged tile

template <int K>
__global__ void __launch_bounds__(kCfRows) cur_p_kernel(const double* C, int64_t ldc, int64_t n1, int nJ,
                                                        const double* VS, double* Pt, int64_t ldp) {
  __shared__ double tile[kCfRows][kCfChunk + 1];
  __shared__ double vs[kCfChunk][K];
  const int64_t r0 = (int64_t)blockIdx.x * kCfRows;
  const int tid = threadIdx.x;
  double acc[K];
#pragma unroll
  for (int t = 0; t < K; ++t) acc[t] = 0.0;
  for (int j0 = 0; j0 < nJ; j0 += kCfChunk) {
    const int jn = nJ - j0 < kCfChunk ? nJ - j0 : kCfChunk;
    for (int e = tid; e < kCfRows * kCfChunk; e += kCfRows) {
      const int rr = e / kCfChunk, jj = e - rr * kCfChunk;
      tile[rr][jj] = (r0 + rr < n1 && jj < jn) ? C[(r0 + rr) * ldc + j0 + jj] : 0.0;
    }
    for (int e = tid; e < kCfChunk * K; e += kCfRows) {
      const int jj = e / K, t = e - jj * K;
      vs[jj][t] = jj < jn ? VS[(int64_t)(j0 + jj) * K + t] : 0.0;
    }
    __syncthreads();
    for (int jj = 0; jj < jn; ++jj) {
      const double c = tile[tid][jj];
#pragma unroll
      for (int t = 0; t < K; ++t) acc[t] = fma(c, vs[jj][t], acc[t]);
    }
    __syncthreads();
  }
  if (r0 + tid < n1) {
#pragma unroll
    for (int t = 0; t < K; ++t) Pt[t * ldp + r0 + tid] = acc[t];
  }
}

template <int K>
__global__ void __launch_bounds__(256) cur_q_kernel(const double* R, int64_t ldr, int mI, int64_t n2,
                                                    const double* W, double* Qt, int64_t ldq) {
  extern __shared__ double wsm[];  // mI x K
  for (int e = threadIdx.x; e < mI * K; e += blockDim.x) wsm[e] = W[e];
  __syncthreads();
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n2) return;
  double acc[K];
#pragma unroll
  for (int t = 0; t < K; ++t) acc[t] = 0.0;
  for (int i = 0; i < mI; ++i) {
    const double rv = R[(int64_t)i * ldr + x];
#pragma unroll
    for (int t = 0; t < K; ++t) acc[t] = fma(wsm[i * K + t], rv, acc[t]);
  }
#pragma unroll
  for (int t = 0; t < K; ++t) Qt[t * ldq + x] = acc[t];
}
}  // namespace
}  // namespace ircur

extern "C" int ircur_cur_to_factors(const double* C, int64_t ldc, const double* R, int64_t ldr,
                                    const double* VS, const double* W, int64_t n1, int64_t n2, int mI,
                                    int nJ, int k, double* Pt, int64_t ldp, double* Qt, int64_t ldq,
                                    void* stream) {
  using namespace ircur;
  if (k < 1 || k > kMaxRank || n1 < 0 || n2 < 0 || mI < 0 || nJ < 0 || ldc < nJ || ldr < n2 || ldp < n1 ||
      ldq < n2)
    return IRCUR_EINVAL;
  if ((size_t)mI * k * sizeof(double) > 48 * 1024) return IRCUR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned gp = (unsigned)((n1 + kCfRows - 1) / kCfRows), gq = (unsigned)((n2 + 255) / 256);
  const size_t qsm = (size_t)mI * k * sizeof(double);
  IRCUR_DISPATCH_RANK(k, KK, {
    if (n1 > 0) cur_p_kernel<KK><<<gp, kCfRows, 0, st>>>(C, ldc, n1, nJ, VS, Pt, ldp);
    if (n2 > 0) cur_q_kernel<KK><<<gq, 256, qsm, st>>>(R, ldr, mI, n2, W, Qt, ldq);
  });
  return cudaGetLastError() == cudaSuccess ? IRCUR_OK : IRCUR_ECUDA;
}
