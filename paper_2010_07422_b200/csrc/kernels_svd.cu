// Exact top-r SVD / pseudo-inverse of the |I| x |J| core (sm_100a).
//
// Replaces matcore.truncated_svd (LAPACK gesdd, matcore.py:128-139) and
// PinvFactor.from_svd (cutoff sigma > 1e-12 sigma_max, matcore.py:156-165).
// Only the top k = min(r, |I|, |J|) triplets are consumed, so instead of a
// full dense SVD the core is factorised by block subspace iteration on the
// Gram matrix G = U^T U with a Rayleigh-Ritz step every iteration,
// warm-started from the previous iterate's Q(:,J), until the Ritz residuals
// reach round-off (scaled by the previous e_k); a final
// Rayleigh-Ritz step on U itself (converged Jacobi) resolves small singular
// values to absolute fp64 accuracy, so the pinv cutoff behaves like LAPACK's.
// Block size kk = min(2r, |I|, |J|, 32).
//
// One thread-block cluster per core.  CTA q owns rows [lo_q, hi_q) of G
// (resident in its shared memory for the whole call) and of the n x kk block
// V.  The full V lives in a double-buffered L2 scratch and is read through
// L1 by the G-row-block product.  Per step there are exactly two
// cluster-wide synchronisations: one DSMEM reduction (fixed rank order) of
// [V^T G V | V^T V | previous Ritz residuals], and the publication of the
// next block.  The Cholesky-QR of the block is folded into the Rayleigh-Ritz
// problem (generalised eigenproblem through chol(V^T V)); the kk x kk
// eigenproblem runs on four warps under a named barrier.  Every CTA holds
// bitwise-identical reduced values and takes identical branches
// (deterministic run to run).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "ircur_common.cuh"
#include "launchers.cuh"
#include <mutex>

#include "svd_small_reg.cuh"

namespace cg = cooperative_groups;

namespace ircur {

constexpr int kSvdNT = 512;
constexpr int kSvdNW = kSvdNT / 32;
constexpr int kKMax = 32;
constexpr int kEigNT = 128;  // threads running the small dense kernels
constexpr int kLdV = kKMax;  // leading dimension of V in the L2 scratch

// ------------------------------------------------------------------ gram
// G = U^T U (n x n) on the FP64 tensor cores (mma.sync m8n8k4 f64).  One CTA
// per 32 x 32 tile of the upper triangle; warp w owns the 8 x 8 blocks
// (w / 2, 2 (w % 2) + {0, 1}) and runs K = m in steps of 4 rows.  K streams in
// 32-row chunks through a kGramNS-stage cp.async pipeline.  Exact symmetry:
// below-diagonal blocks of a diagonal tile are not computed, and a diagonal
// 8 x 8 block writes its upper triangle and the mirror of it.  (The CUDA-core
// version — one DFMA per shared load, latency-bound at 23 us for 460^2 — is
// what this replaces.)
constexpr int kGramNS = 8;
constexpr int kGramLd = 33;
constexpr int kGramSmem = kGramNS * 2 * 32 * kGramLd * (int)sizeof(double);

__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void gram_body(const double* __restrict__ U, int ldu, int m, int n,
                                          double* __restrict__ G, int ldg, const int* done, int bx) {
  if (done && *done) return;
  extern __shared__ double gram_sm[];
  auto As = [&](int st, int r, int c) -> double& { return gram_sm[((st * 2) * 32 + r) * kGramLd + c]; };
  auto Bs = [&](int st, int r, int c) -> double& { return gram_sm[((st * 2 + 1) * 32 + r) * kGramLd + c]; };
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // blockIdx.x -> (ta <= tb) in row-major order of the upper triangle
  const int nt = (n + 31) / 32;
  if (bx >= nt * (nt + 1) / 2) return;
  int ta = 0, rem = bx;
  while (rem >= nt - ta) { rem -= nt - ta; ++ta; }
  const int tb = ta + rem;
  const int a0 = ta * 32, b0 = tb * 32;
  const int nch = (m + 31) / 32;
  auto issue = [&](int ch) {
    if (ch < nch) {
      const int st = ch % kGramNS;
      const int c = tid & 31;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int r = (tid >> 5) + 8 * k, i = ch * 32 + r;
        const bool va = i < m && a0 + c < n, vb = i < m && b0 + c < n;
        const double* pa = va ? U + (int64_t)i * ldu + a0 + c : U;
        const double* pb = vb ? U + (int64_t)i * ldu + b0 + c : U;
        const unsigned da = (unsigned)__cvta_generic_to_shared(&As(st, r, c));
        const unsigned db = (unsigned)__cvta_generic_to_shared(&Bs(st, r, c));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(da), "l"(pa), "r"(va ? 8 : 0));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(db), "l"(pb), "r"(vb ? 8 : 0));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  const int br = warp >> 1, bc0 = (warp & 1) * 2;  // block row, first block column (8 x 8 blocks)
  const bool diag = ta == tb;
  const bool on0 = !diag || bc0 >= br, on1 = !diag || bc0 + 1 >= br;
  const int g = lane >> 2, q = lane & 3;  // fragment row / column group
  double acc0[2] = {0.0, 0.0}, acc1[2] = {0.0, 0.0};
#pragma unroll
  for (int c = 0; c < kGramNS - 1; ++c) issue(c);
  for (int c = 0; c < nch; ++c) {
    issue(c + kGramNS - 1);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kGramNS - 1));
    __syncthreads();
    const int st = c % kGramNS;
    if (on0 || on1) {
#pragma unroll
      for (int k0 = 0; k0 < 32; k0 += 4) {
        const double av = As(st, k0 + q, br * 8 + g);
        const double bv0 = Bs(st, k0 + q, bc0 * 8 + g);
        const double bv1 = Bs(st, k0 + q, bc0 * 8 + 8 + g);
        if (on0) dmma_8x8x4(acc0, av, bv0);
        if (on1) dmma_8x8x4(acc1, av, bv1);
      }
    }
    __syncthreads();
  }
  auto store = [&](const double (&acc)[2], int bc) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = a0 + br * 8 + g, cc = b0 + bc * 8 + 2 * q + h;
      if (r >= n || cc >= n) continue;
      if (diag && bc == br) {  // diagonal block: upper triangle and its mirror
        if (cc < r) continue;
        G[(int64_t)r * ldg + cc] = acc[h];
        G[(int64_t)cc * ldg + r] = acc[h];
      } else {
        G[(int64_t)r * ldg + cc] = acc[h];
        G[(int64_t)cc * ldg + r] = acc[h];
      }
    }
  };
  if (on0) store(acc0, bc0);
  if (on1) store(acc1, bc0 + 1);
}

__global__ void __launch_bounds__(256) gram_kernel(const double* __restrict__ U, int ldu, int m, int n,
                                                   double* __restrict__ G, int ldg, const int* done) {
  gram_body(U, ldu, m, n, G, ldg, done, (int)blockIdx.x);
}
// batched problems (ircur_batched_run): problem blockIdx.y, its core / Gram from the SVD arguments
__global__ void __launch_bounds__(256) gram_kernel_batched(const SvdArgs* __restrict__ as) {
  const SvdArgs& a = as[blockIdx.y];
  gram_body(a.U, a.ldu, a.m, a.n, const_cast<double*>(a.G), a.ldg, a.done, (int)blockIdx.x);
}

// ------------------------------------------------------------ layout
// Shared-memory layout in doubles; identical on host (size) and device.
struct SvdLayout {
  int n, m, kk, KP, HL, per, mper, rowsmax, ldgq, S, gq_smem, RL;
  int oVq, oGq, oP, oBq, oXq, oH, oH2, oZ, oLc, oT, oRed, oRout, oRes, oResq, oLam, oCs, oW, oPt, total;
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
  L.RL = 2 * kk * kk + kk;  // reduction record: H' | M | residuals
  int off = 0;
  L.oVq = off; off += L.rowsmax * L.KP;
  L.oP = off; off += S * L.rowsmax * L.KP;
  L.oBq = off; off += L.rowsmax * L.KP;
  L.oXq = off; off += L.rowsmax * L.KP;
  L.oH = off; off += kk * L.HL;
  L.oH2 = off; off += kk * L.HL;
  L.oZ = off; off += kk * L.HL;
  L.oLc = off; off += kk * L.HL;
  L.oT = off; off += kk * L.HL;
  L.oRed = off; off += 2 * L.RL;
  L.oRout = off; off += L.RL;
  L.oRes = off; off += kk;
  L.oResq = off; off += 2 * kKMax;
  L.oLam = off; off += kk;
  L.oCs = off; off += 4 * kKMax;
  L.oW = off; off += 2 * kKMax + 8;
  L.oPt = off; off += kKMax * kKMax * 3 / 4;  // partner table (1024 ints) + entry table (1024 shorts)
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
  double *Vq, *Gq, *P, *Bq, *Xq, *H, *H2, *Z, *Lc, *T, *red, *rout, *res, *resq, *lam, *cs, *ws;
  int* flags;
  int* ptab;
};

// named barrier for the first kEigNT threads
__device__ __forceinline__ void eig_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kEigNT) : "memory"); }

// fixed-rank-order DSMEM reduction of red[buf][0:len) -> rout (one cluster sync;
// red is double-buffered so peers may still be reading the other buffer)
__device__ __forceinline__ void cluster_sum(cg::cluster_group& cl, Sm& S, int buf, int len) {
  double* src = S.red + buf * S.L.RL;
  cl.sync();
  const int CS = (int)cl.num_blocks();
  for (int e = threadIdx.x; e < len; e += kSvdNT) {
    double v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = q < CS ? *cl.map_shared_rank(src + e, q) : 0.0;
    double s = v[0];
#pragma unroll
    for (int q = 1; q < 16; ++q)
      if (q < CS) s += v[q];
    S.rout[e] = s;
  }
  __syncthreads();
}

// Out(nr x kk, ld KP) = A(nr x n, lda) * V(n x kk, ld ldv).  Warp tile:
// 8 rows x 16 cols, lane = (row pair, col pair) so that the A loads are
// 4-way and the V loads 8-way broadcasts; the inner dimension is split in S
// contiguous chunks whose partial tiles are summed in a fixed order.  A and
// V may live in shared or global memory (generic pointers).
__device__ void tiled_product(const double* A, int lda, int nr, int n, const double* V, int ldv, int KP,
                              int kk, double* Out, double* partial, int S) {
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
#pragma unroll 8
    for (int j = j0; j < j1; ++j) {
      const double a0 = Aa[j], a1 = Ab[j];
      const double v0 = V[(int64_t)j * ldv + ca], v1 = V[(int64_t)j * ldv + cb];
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

// Cyclic Jacobi eigen-decomposition of the symmetric kk x kk S.H on the first
// kEigNT threads.  Parallel (round-robin, circle method) ordering: in every
// round one thread per disjoint pair (p, q) computes the rotation and
// publishes (c, s) and the partner of p and q; then every thread applies
// J^T H J and Z J to its fixed set of <= 8 matrix entries (kept in
// registers as indices).  Two named barriers per round; the off-diagonal
// maximum that decides the next sweep is reduced inside the last round.
// On exit S.lam holds the eigenvalues in decreasing order and S.Z the
// matching eigenvectors.  `thr_rel` is the stopping threshold relative to the
// largest diagonal entry, `max_sweeps` caps the work (an inexact Z only costs
// the subspace iteration an extra step; the final extraction runs to
// convergence).  Caller: the first kEigNT threads.
constexpr int kEigCPT = 8;  // columns per thread (kk <= 32, 128 threads: >= 4 row groups)

__device__ __forceinline__ int circle_player(int pos, int rd, int nrd) {
  if (pos == 0) return 0;
  int x = pos - 1 + rd;
  x -= (x >= nrd) ? nrd : 0;
  return x + 1;
}

__device__ __forceinline__ double approx_sqrtf_d(float x) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ void jacobi_eig(Sm& S, int kk, double thr_rel, int max_sweeps, long long* dbg = nullptr,
                           bool reg = false) {
  if (reg && sreg_supported(kk)) {  // one warp, registers (svd_small_reg.cuh)
    if (threadIdx.x < 32) {
      const int sw = eig_reg(kk, S.H, S.L.HL, S.Z, S.lam, thr_rel, max_sweeps);
      if (dbg && blockIdx.x == 0 && threadIdx.x == 0) dbg[13] += sw;
    }
    eig_sync();
    return;
  }
  const int tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
  const int HL = S.L.HL;
  double* H = S.H;
  double* Hn = S.H2;
  double* Z = S.Z;
  double* Zn = S.T;  // free while the eigenproblem is solved
  const int nply = kk + (kk & 1);
  const int nrd = nply - 1;
  int* prt = S.ptab;  // partner of each index in the current round (itself when idle)
  // entry mapping: thread -> row a, columns b = g, g + ng, g + 2 ng, ...
  const int ng = kEigNT / kk;  // row groups (>= 4)
  const int a = tid % kk, g = tid / kk;
  const bool act = g < ng;
  const int ncol = act ? (kk - g + ng - 1) / ng : 0;  // <= kEigCPT
#pragma unroll
  for (int v = 0; v < kEigCPT; ++v)
    if (v < ncol) {
      const int b = g + v * ng;
      Z[a * HL + b] = (a == b) ? 1.0 : 0.0;
    }
  double scale = 0.0;
  for (int i = 0; i < kk; ++i) scale = fmax(scale, fabs(H[i * HL + i]));
  const double thr = thr_rel * scale;
  const double isc = scale > 0.0 ? 1.0 / scale : 1.0;  // keeps the fp32 tangent in range
  double off = 0.0;
#pragma unroll
  for (int v = 0; v < kEigCPT; ++v)
    if (v < ncol) {
      const int b = g + v * ng;
      if (a != b) off = fmax(off, fabs(H[a * HL + b]));
    }
  double* offw = S.ws + 16;  // 2 x 4 warp maxima (double-buffered by sweep)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) off = fmax(off, __shfl_xor_sync(0xffffffffu, off, o));
  if (lane == 0) offw[wq] = off;
  eig_sync();
  off = fmax(fmax(offw[0], offw[1]), fmax(offw[2], offw[3]));
  for (int sweep = 0; sweep < max_sweeps && off > thr; ++sweep) {
    if (dbg && blockIdx.x == 0 && tid == 0) dbg[13] += 1;
    double offl = 0.0;
    const bool rec = dbg && blockIdx.x == 0 && tid == 0;
    for (int rd = 0; rd < nrd; ++rd) {
      if (tid < nply / 2) {
        int p = circle_player(tid, rd, nrd), q = circle_player(nply - 1 - tid, rd, nrd);
        if (p > q) { const int t = p; p = q; q = t; }
        if (q < kk) {
          const double hpq = H[p * HL + q], hpp = H[p * HL + p], hqq = H[q * HL + q];
          double c = 1.0, s = 0.0;
          if (fabs(hpq) > 1e-300 && fabs(hpq) > thr) {
            // tan(theta) in fp32 (only the convergence rate depends on it);
            // c = (1 + t^2)^{-1/2}, s = t c in fp64 from that t keep the
            // transform orthogonal to fp64 round-off.
            const float d = (float)((hqq - hpp) * isc), h2 = (float)(2.0 * hpq * isc);
            const float rt = (float)approx_sqrtf_d(fmaf(d, d, h2 * h2));
            const float tf = __fdividef(h2, fabsf(d) + rt) * (d >= 0.f ? 1.f : -1.f);
            const double t = (double)tf;
            c = rsqrt(fma(t, t, 1.0));
            s = t * c;
          }
          S.cs[2 * p] = c;  S.cs[2 * p + 1] = s;     // first of the pair
          S.cs[2 * q] = c;  S.cs[2 * q + 1] = -s;    // second (sign flip)
          prt[p] = q;
          prt[q] = p;
        } else {  // p pairs with the padding index of an odd kk
          S.cs[2 * p] = 1.0; S.cs[2 * p + 1] = 0.0;
          prt[p] = p;
        }
      }
      eig_sync();
      const bool lastrd = rd == nrd - 1;
      if (act) {
        // row a:  H' = J^T H J  restricted to (a, b):  rows a, pa then columns b, pb
        const int pa = prt[a];
        const double ca = S.cs[2 * a], sa = S.cs[2 * a + 1];
        const double* Ha = H + a * HL;
        const double* Hpa = H + pa * HL;
        const double* Za = Z + a * HL;
#pragma unroll 4
        for (int v = 0; v < ncol; ++v) {
          const int b = g + v * ng;
          const int pb = prt[b];
          const double cb = S.cs[2 * b], sb = S.cs[2 * b + 1];
          const double r_b = ca * Ha[b] - sa * Hpa[b];
          const double r_pb = ca * Ha[pb] - sa * Hpa[pb];
          const double hn = cb * r_b - sb * r_pb;
          Hn[a * HL + b] = hn;
          Zn[a * HL + b] = cb * Za[b] - sb * Za[pb];  // Z <- Z J
          if (lastrd && a != b) offl = fmax(offl, fabs(hn));
        }
      }
      if (lastrd) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) offl = fmax(offl, __shfl_xor_sync(0xffffffffu, offl, o));
        if (lane == 0) offw[4 * (sweep & 1) + wq] = offl;
      }
      eig_sync();
      double* t = H; H = Hn; Hn = t;
      t = Z; Z = Zn; Zn = t;
    }
    const double* ow = offw + 4 * (sweep & 1);
    off = fmax(fmax(ow[0], ow[1]), fmax(ow[2], ow[3]));
  }
  if (Z != S.Z) {
    for (int e = tid; e < kk * kk; e += kEigNT) {
      const int i = e / kk, j = e - i * kk;
      S.Z[i * HL + j] = Z[i * HL + j];
    }
    eig_sync();
  }
  int* perm = reinterpret_cast<int*>(S.cs + 2 * kKMax) + kKMax;
  if (tid < kk) {
    const double li = H[tid * HL + tid];
    int rk = 0;
    for (int j = 0; j < kk; ++j) {
      const double lj = H[j * HL + j];
      rk += (lj > li) || (lj == li && j < tid);
    }
    perm[rk] = tid;
  }
  eig_sync();
  if (tid < kk) S.lam[tid] = H[perm[tid] * HL + perm[tid]];
  for (int e = tid; e < kk * kk; e += kEigNT) {
    const int i = e / kk, j = e - i * kk;
    Hn[i * HL + j] = S.Z[i * HL + perm[j]];
  }
  eig_sync();
  for (int e = tid; e < kk * kk; e += kEigNT) {
    const int i = e / kk, j = e - i * kk;
    S.Z[i * HL + j] = Hn[i * HL + j];
  }
  eig_sync();
}

// Cholesky M = Lc Lc^T of the kk x kk Gram M (ld kk), right-looking, by warp
// 0 of the eig threads with lane i owning row i (column values broadcast by
// shuffles); the reciprocal diagonal is kept in column kk.  Returns 0 on
// breakdown.  Caller: first kEigNT threads.
__device__ int cholesky_warp(const double* M, double* Lc, int HL, int kk, int* flag) {
  const int tid = threadIdx.x;
  if (tid < 32) {
    const int i = tid;
    const bool row = i < kk;
    if (row)
      for (int k = 0; k <= i; ++k) Lc[i * HL + k] = M[i * kk + k];
    __syncwarp();
    int ok = 1;
    for (int j = 0; j < kk; ++j) {
      double d = Lc[j * HL + j];
      const bool bad = !(d > 1e-300);
      if (bad) { d = 1.0; ok = 0; }
      const double ir = rsqrt(d);  // 1 / L_jj (division-free)
      double lij = 0.0;
      if (row && i > j) {
        lij = Lc[i * HL + j] * ir;
        Lc[i * HL + j] = lij;
      }
      if (i == j) {
        Lc[j * HL + j] = d * ir;
        Lc[j * HL + kk] = ir;
      }
      for (int k0 = j + 1; k0 < kk; k0 += 4) {
        double lk[4], lv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + u;
          lk[u] = __shfl_sync(0xffffffffu, lij, k & 31);
          lv[u] = (row && k < kk && k <= i) ? Lc[i * HL + k] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + u;
          if (row && k < kk && k <= i) Lc[i * HL + k] = fma(-lij, lk[u], lv[u]);
        }
      }
      __syncwarp();
    }
    if (tid == 0) *flag = ok;
  }
  eig_sync();
  return *flag;
}

// x_i = (b_i - sum_{k<i} L_ik x_k) * Linv_i for i = 0..kk-1 (forward) with the
// inner products split over four independent partial sums.
__device__ __forceinline__ void tri_forward(const double* Lc, int HL, int kk, const double* b, int bstride,
                                            double* x, int xstride) {
  for (int i = 0; i < kk; ++i) {
    double s0 = b[i * bstride], s1 = 0.0, s2 = 0.0, s3 = 0.0;
    const double* Li = Lc + i * HL;
    int k2 = 0;
    for (; k2 + 3 < i; k2 += 4) {
      s0 = fma(-Li[k2], x[k2 * xstride], s0);
      s1 = fma(-Li[k2 + 1], x[(k2 + 1) * xstride], s1);
      s2 = fma(-Li[k2 + 2], x[(k2 + 2) * xstride], s2);
      s3 = fma(-Li[k2 + 3], x[(k2 + 3) * xstride], s3);
    }
    for (; k2 < i; ++k2) s0 = fma(-Li[k2], x[k2 * xstride], s0);
    x[i * xstride] = ((s0 + s1) + (s2 + s3)) * Li[kk];
  }
}

// Rayleigh-Ritz on (H', M): H = Lc^{-1} H' Lc^{-T}, eig(H) = Z Lambda Z^T,
// T = Lc^{-T} Z so that V T has orthonormal columns and diagonalises V^T G V.
// Caller: first kEigNT threads.  Returns 0 if chol(M) broke down.
__device__ int ritz_small(Sm& S, int kk, const double* Hp, const double* M, double thr_rel, int max_sweeps,
                          long long* dbg = nullptr, bool reg = false) {
  const int tid = threadIdx.x, HL = S.L.HL;
  const bool rec = dbg && blockIdx.x == 0 && tid == 0;
  long long t0 = clock64();
  if (reg && sreg_supported(kk)) {  // one warp, registers (svd_small_reg.cuh)
    if (tid < 32) {
      int sw = 0;
      const int ok = ritz_reg(kk, Hp, M, S.T, S.lam, S.H2, S.Z, HL, thr_rel, max_sweeps, &sw);
      if (tid == 0) {
        S.flags[1] = ok;
        if (rec) {
          dbg[10] += clock64() - t0;
          dbg[13] += sw;
          dbg[14] += 1;
        }
      }
    }
    eig_sync();
    return S.flags[1];
  }
  if (!cholesky_warp(M, S.Lc, HL, kk, S.flags + 1)) return 0;
  if (rec) { const long long t1 = clock64(); dbg[8] += t1 - t0; t0 = t1; }
  // K = Lc^{-1} H' (column c: stride HL down the rows), then H^T = Lc^{-1} K^T
  if (tid < kk) tri_forward(S.Lc, HL, kk, Hp + tid, kk, S.H2 + tid, HL);
  eig_sync();
  if (tid < kk) tri_forward(S.Lc, HL, kk, S.H2 + tid * HL, 1, S.T + tid * HL, 1);
  eig_sync();
  for (int e = tid; e < kk * kk; e += kEigNT) {
    const int i = e / kk, j = e - i * kk;
    S.H[i * HL + j] = 0.5 * (S.T[i * HL + j] + S.T[j * HL + i]);
  }
  eig_sync();
  if (rec) { const long long t1 = clock64(); dbg[9] += t1 - t0; t0 = t1; }
  jacobi_eig(S, kk, thr_rel, max_sweeps, dbg);
  if (rec) { const long long t1 = clock64(); dbg[10] += t1 - t0; t0 = t1; dbg[14] += 1; }
  if (tid < kk) {  // T = Lc^{-T} Z (back substitution, column c = tid)
    const int c = tid;
    for (int i = kk - 1; i >= 0; --i) {
      double s0 = S.Z[i * HL + c], s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int k2 = i + 1;
      for (; k2 + 3 < kk; k2 += 4) {
        s0 = fma(-S.Lc[k2 * HL + i], S.T[k2 * HL + c], s0);
        s1 = fma(-S.Lc[(k2 + 1) * HL + i], S.T[(k2 + 1) * HL + c], s1);
        s2 = fma(-S.Lc[(k2 + 2) * HL + i], S.T[(k2 + 2) * HL + c], s2);
        s3 = fma(-S.Lc[(k2 + 3) * HL + i], S.T[(k2 + 3) * HL + c], s3);
      }
      for (; k2 < kk; ++k2) s0 = fma(-S.Lc[k2 * HL + i], S.T[k2 * HL + c], s0);
      S.T[i * HL + c] = ((s0 + s1) + (s2 + s3)) * S.Lc[i * HL + kk];
    }
  }
  eig_sync();
  return 1;
}

// X(nr x kk, ld KP) <- X R (R kk x kk, ld HL) using tmp
__device__ void rotate_rows(double* X, int nr, int KP, int kk, const double* Rm, int HL, double* tmp) {
  for (int e = threadIdx.x; e < nr * kk; e += kSvdNT) {
    const int i = e / kk, c = e - i * kk;
    double s = 0.0;
    for (int j = 0; j < kk; ++j) s = fma(X[i * KP + j], Rm[j * HL + c], s);
    tmp[i * KP + c] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nr * kk; e += kSvdNT) {
    const int i = e / kk, c = e - i * kk;
    X[i * KP + c] = tmp[i * KP + c];
  }
  __syncthreads();
}

// CGS2 with random replacement on the FULL V (n x kk, ld kLdV) in global
// memory, by one CTA — the rare path for a rank-deficient starting block.
__device__ void cgs2_global(Sm& S, double* V, int n, int kk, uint64_t salt) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  double* dots = S.rout;
  for (int c = 0; c < kk; ++c) {
    for (int attempt = 0; attempt < 4; ++attempt) {
      double p = 0.0;
      for (int j = tid; j < n; j += kSvdNT) p = fma(V[j * kLdV + c], V[j * kLdV + c], p);
      p = warp_sum(p);
      if (lane == 0) S.ws[w] = p;
      __syncthreads();
      double nrm0 = 0.0;
      for (int i = 0; i < kSvdNW; ++i) nrm0 += S.ws[i];
      __syncthreads();
      for (int pass = 0; pass < 2; ++pass) {
        for (int k = w; k < c; k += kSvdNW) {
          double d = 0.0;
          for (int j = lane; j < n; j += 32) d = fma(V[j * kLdV + k], V[j * kLdV + c], d);
          d = warp_sum(d);
          if (lane == 0) dots[k] = d;
        }
        __syncthreads();
        for (int j = tid; j < n; j += kSvdNT) {
          double v = V[j * kLdV + c];
          for (int k = 0; k < c; ++k) v = fma(-dots[k], V[j * kLdV + k], v);
          V[j * kLdV + c] = v;
        }
        __syncthreads();
      }
      p = 0.0;
      for (int j = tid; j < n; j += kSvdNT) p = fma(V[j * kLdV + c], V[j * kLdV + c], p);
      p = warp_sum(p);
      if (lane == 0) S.ws[w] = p;
      __syncthreads();
      double nrm = 0.0;
      for (int i = 0; i < kSvdNW; ++i) nrm += S.ws[i];
      __syncthreads();
      if (nrm > 1e-20 * nrm0 && nrm > 1e-280) {
        const double inv = 1.0 / sqrt(nrm);
        for (int j = tid; j < n; j += kSvdNT) V[j * kLdV + c] *= inv;
        __syncthreads();
        break;
      }
      for (int j = tid; j < n; j += kSvdNT)
        V[j * kLdV + c] = hash_uniform(salt + 1000003ull * (uint64_t)(attempt + 1), (uint64_t)j * 64 + c);
      __syncthreads();
    }
  }
}

template <typename T, bool REG>
__device__ __forceinline__ void svd_body(const SvdArgs& a) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double svsm[];
  {  // one skip decision for the whole cluster: in the overlapped loop the stop
     // flag can be set (finalize on the other stream) while the CTAs start, and a
     // CTA that exits alone would leave the others reading its shared memory.
     // (The flag borrows the first word of the dynamic shared memory, which the
     // kernel only uses after the second cluster barrier.)
    int* s_done = reinterpret_cast<int*>(svsm);
    if (threadIdx.x == 0) *s_done = (a.done && *(volatile const int*)a.done) ? 1 : 0;
    cl.sync();
    const int d0 = *cl.map_shared_rank(s_done, 0);
    cl.sync();  // every CTA has read rank 0's flag before any of them exits
    if (d0) return;
  }
  const int CS = (int)cl.num_blocks();
  const int q = (int)cl.block_rank();
  const int n = a.n, m = a.m, r = a.r, kk = a.kk;
  const int reff = min(r, min(m, n));
  Sm S;
  S.L = svd_layout(n, m, kk, CS);
  const SvdLayout& L = S.L;
  const int KP = L.KP, HL = L.HL, RL = L.RL;
  S.Vq = svsm + L.oVq; S.P = svsm + L.oP; S.Bq = svsm + L.oBq; S.Xq = svsm + L.oXq;
  S.H = svsm + L.oH; S.H2 = svsm + L.oH2; S.Z = svsm + L.oZ; S.Lc = svsm + L.oLc; S.T = svsm + L.oT;
  S.red = svsm + L.oRed; S.rout = svsm + L.oRout; S.res = svsm + L.oRes; S.lam = svsm + L.oLam;
  S.resq = svsm + L.oResq;
  S.cs = svsm + L.oCs; S.ws = svsm + L.oW;
  S.flags = reinterpret_cast<int*>(svsm + L.oW + kKMax);
  S.ptab = reinterpret_cast<int*>(svsm + L.oPt);
  S.Gq = svsm + L.oGq;
  const int lo = min(n, q * L.per), hi = min(n, lo + L.per), nr = hi - lo;
  const int mlo = min(m, q * L.mper), mhi = min(m, mlo + L.mper), mr = mhi - mlo;
  const int tid = threadIdx.x;
  const bool eigt = tid < kEigNT;
  const double eprev = a.prev_err ? fmin(1.0, fabs(*a.prev_err)) : 1.0;
  const double tol = fmax(a.tol, a.tol_scale * eprev);
  double* scr[2] = {a.scratch, a.scratch + (size_t)n * kLdV};

  // ---- 0. G rows of this CTA into shared memory; starting block (my rows)
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
  int gbuf = 0;
  for (int e = tid; e < nr * kk; e += kSvdNT) {
    const int i = e / kk, c = e - i * kk;
    const int j = lo + i;
    double v;
    if (warm && c < a.warm_cols) v = (double)warm[(int64_t)j * a.warm_ld + c];
    else v = hash_uniform(0x5EEDull + a.salt, (uint64_t)j * 64 + c);
    S.Vq[i * KP + c] = v;
    scr[gbuf][(int64_t)j * kLdV + c] = v;
  }
  for (int c = tid; c < kk; c += kSvdNT) S.res[c] = 0.0;
  __threadfence();
  cl.sync();

  int step = 0, buf = 0, redo = 0;
  bool gx_valid = false;  // S.P holds G X for the final Ritz block X (my rows)
  double prev_res = 1e300;
  int stall = 0;
  double* scrX = a.scratch + 2 * (size_t)n * kLdV;  // Ritz block X of the latest step
  long long tph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tc = clock64();
#define PH(i) do { if (a.dbg) { const long long _t = clock64(); tph[i] += _t - tc; tc = _t; } } while (0)
  for (;;) {
    PH(7);
    // ---- 1. B_q = G(lo:hi, :) V   (V through L1 from the L2 scratch)
    tiled_product(Gq, ldgq, nr, n, scr[gbuf], kLdV, KP, kk, S.Bq, S.P, L.S);
    PH(0);
    // ---- 2. one reduction: [V^T B | V^T V]
    double* rb = S.red + buf * RL;
    for (int e = tid; e < 2 * kk * kk; e += kSvdNT) {
      const int which = e / (kk * kk);
      const int e2 = e - which * kk * kk;
      const int c1 = e2 / kk, c2 = e2 - c1 * kk;
      const double* Y = which == 0 ? S.Bq : S.Vq;
      double s = 0.0;
      for (int i = 0; i < nr; ++i) s = fma(S.Vq[i * KP + c1], Y[i * KP + c2], s);
      rb[e] = s;
    }
    cluster_sum(cl, S, buf, 2 * kk * kk);
    buf ^= 1;
    PH(1);
    // ---- 3. Rayleigh-Ritz (generalised through chol(V^T V))
    if (eigt) {
      const int ok = ritz_small(S, kk, S.rout, S.rout + kk * kk, a.jac_thr, a.sweeps, a.dbg, REG);
      if (tid == 0) S.flags[7] = ok;
    }
    __syncthreads();
    if (!S.flags[7]) {
      // rank-deficient block: CTA 0 orthonormalises the shared copy robustly
      if (q == 0) cgs2_global(S, scr[gbuf], n, kk, a.salt + 77ull * (redo + 1));
      __threadfence();
      cl.sync();
      for (int e = tid; e < nr * kk; e += kSvdNT) {
        const int i = e / kk, c = e - i * kk;
        S.Vq[i * KP + c] = scr[gbuf][(int64_t)(lo + i) * kLdV + c];
      }
      __syncthreads();
      gx_valid = false;
      if (++redo > 3) {
        for (int e = tid; e < nr * kk; e += kSvdNT) {
          const int i = e / kk, c = e - i * kk;
          scrX[(int64_t)(lo + i) * kLdV + c] = S.Vq[i * KP + c];
        }
        break;
      }
      continue;
    }
    PH(2);
    // ---- 4. Ritz vectors X_q = V_q T (orthonormal), Y_q = B_q T (= G X)
    for (int e = tid; e < nr * kk; e += kSvdNT) {
      const int i = e / kk, c = e - i * kk;
      double sx = 0.0, sy = 0.0;
      for (int j = 0; j < kk; ++j) {
        const double t = S.T[j * HL + c];
        sx = fma(S.Vq[i * KP + j], t, sx);
        sy = fma(S.Bq[i * KP + j], t, sy);
      }
      S.Xq[i * KP + c] = sx;
      S.P[i * KP + c] = sy;
      scrX[(int64_t)(lo + i) * kLdV + c] = sx;
    }
    gx_valid = true;
    __syncthreads();
    PH(3);
    // ---- 5. this step's Ritz residuals (my rows) and the next block
    double* rq = S.resq + (step & 1) * kKMax;
    const double lam0 = S.lam[0];
    const double sig_thr = 1e-10 * fabs(lam0);
    for (int c = tid; c < kk; c += kSvdNT) {
      const double lc = S.lam[c];
      double rs = 0.0;
      for (int i = 0; i < nr; ++i) {
        const double d = S.P[i * KP + c] - lc * S.Xq[i * KP + c];
        rs = fma(d, d, rs);
      }
      rq[c] = rs;
    }
    double* sc = scr[gbuf ^ 1];
    for (int e = tid; e < nr * kk; e += kSvdNT) {
      const int i = e / kk, c = e - i * kk;
      const double lc = S.lam[c];
      const double v = (lc > sig_thr && lc > 0.0) ? S.P[i * KP + c] / lc : S.Xq[i * KP + c];
      S.Vq[i * KP + c] = v;
      sc[(int64_t)(lo + i) * kLdV + c] = v;
    }
    PH(4);
    // ---- 6. publish X and the next block; residuals of THIS step from every
    // CTA's shared memory (fixed rank order: identical on all CTAs)
    __threadfence();
    cl.sync();
    if (tid < reff) {
      double v[16];
#pragma unroll
      for (int qq = 0; qq < 16; ++qq) v[qq] = qq < CS ? *cl.map_shared_rank(rq + tid, qq) : 0.0;
      double rs = v[0];
#pragma unroll
      for (int qq = 1; qq < 16; ++qq)
        if (qq < CS) rs += v[qq];
      S.res[tid] = sqrt(rs);
    }
    __syncthreads();
    double resmax = 0.0;
    for (int c = 0; c < reff; ++c) resmax = fmax(resmax, S.res[c]);
    bool conv = !(lam0 > 0.0) || resmax <= tol * lam0;
    if (resmax > 0.5 * prev_res) ++stall; else stall = 0;
    prev_res = resmax;
    if (stall >= 3 && resmax <= 1e-11 * lam0) conv = true;
    gbuf ^= 1;
    ++step;
    PH(5);
    if (conv || step >= a.maxsteps) break;
  }
  if (q == 0 && tid == 0 && a.steps_out) *a.steps_out = step;
  PH(6);
  if (a.dbg && q == 0 && tid == 0)
    for (int i = 0; i < 8; ++i) a.dbg[i] += tph[i];
#undef PH

  // ---- 7. Rayleigh-Ritz on U itself: Y = U V (my m-rows), H2 = Y^T Y
  const long long tfin0 = clock64();
  long long tf = tfin0;
#define FPH(i) do { if (a.dbg && q == 0 && tid == 0) { const long long _t = clock64(); a.dbg[24 + (i)] += _t - tf; tf = _t; } } while (0)
  const double* Vf = scrX;  // published before the loop's last cluster sync
  // keep G X of the last step (my n-rows): QJ = G (X Z) Sigma^-1 = (G X) Z Sigma^-1
  if (gx_valid) {
    for (int e = tid; e < nr * kk; e += kSvdNT) {
      const int i = e / kk, c = e - i * kk;
      S.Bq[i * KP + c] = S.P[i * KP + c];
    }
    __syncthreads();
  }
  tiled_product(a.U + (int64_t)mlo * a.ldu, a.ldu, mr, n, Vf, kLdV, KP, kk, S.Xq, S.P, L.S);
  FPH(0);
  {
    double* rb = S.red + buf * RL;
    for (int e = tid; e < kk * kk; e += kSvdNT) {
      const int c1 = e / kk, c2 = e - c1 * kk;
      double s = 0.0;
      for (int i = 0; i < mr; ++i) s = fma(S.Xq[i * KP + c1], S.Xq[i * KP + c2], s);
      rb[e] = s;
    }
    cluster_sum(cl, S, buf, kk * kk);
    buf ^= 1;
  }
  FPH(1);
  if (eigt) {
    for (int e = tid; e < kk * kk; e += kEigNT) {
      const int c1 = e / kk, c2 = e - c1 * kk;
      S.H[c1 * HL + c2] = 0.5 * (S.rout[c1 * kk + c2] + S.rout[c2 * kk + c1]);
    }
    eig_sync();
    const long long tj0 = clock64();
    jacobi_eig(S, kk, 4e-16, 30, nullptr, REG);
    if (a.dbg && q == 0 && tid == 0) a.dbg[12] += clock64() - tj0;
  }
  __syncthreads();
  FPH(2);
  rotate_rows(S.Xq, mr, KP, kk, S.Z, HL, S.P);
  // rotated V: my rows into Vq and into the other scratch buffer (for QJ)
  double* Vr = scr[0];  // free: both block buffers are dead after the loop
  for (int e = tid; e < nr * kk; e += kSvdNT) {
    const int i = e / kk, c = e - i * kk;
    double s = 0.0;
    for (int j = 0; j < kk; ++j) s = fma(Vf[(int64_t)(lo + i) * kLdV + j], S.Z[j * HL + c], s);
    S.Vq[i * KP + c] = s;
    Vr[(int64_t)(lo + i) * kLdV + c] = s;
  }
  {
    double* rb = S.red + buf * RL;
    for (int c = tid; c < kk; c += kSvdNT) {
      double s = 0.0;
      for (int i = 0; i < mr; ++i) s = fma(S.Xq[i * KP + c], S.Xq[i * KP + c], s);
      rb[c] = s;
    }
    __threadfence();
    cluster_sum(cl, S, buf, kk);  // also publishes Vr
    buf ^= 1;
  }
  if (tid < kk) S.lam[tid] = sqrt(S.rout[tid]);  // sigma
  __syncthreads();
  FPH(3);
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
      vv = S.Vq[i * KP + c];
      const double sg = S.lam[c];
      const double iv = (smax > 0.0 && sg > 1e-12 * smax) ? 1.0 / sg : 0.0;
      vs = vv * iv;
    }
    a.V[(int64_t)(lo + i) * r + c] = vv;
    VS[(int64_t)(lo + i) * r + c] = (T)vs;
  }
  FPH(4);
  // QJ = U^T W = G V Sigma^{-1} for my n-rows (zero for deficient columns)
  if (gx_valid) rotate_rows(S.Bq, nr, KP, kk, S.Z, HL, S.P);
  else tiled_product(Gq, ldgq, nr, n, Vr, kLdV, KP, kk, S.Bq, S.P, L.S);
  for (int e = tid; e < nr * r; e += kSvdNT) {
    const int i = e / r, c = e - i * r;
    double v = 0.0;
    if (c < reff) {
      const double sg = S.lam[c];
      if (sg > 1e-14 * smax && sg > 0.0) v = S.Bq[i * KP + c] / sg;
    }
    QJ[(int64_t)(lo + i) * r + c] = (T)v;
  }
  __threadfence();
  FPH(5);
  cl.sync();
  FPH(6);
  if (ndef > 0 && q == 0) {
    // CGS2 completion of W's deficient columns with unit-vector candidates
    double* dots = S.rout;
    const int lane = tid & 31, w = tid >> 5;
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
  FPH(7);
#undef FPH
  if (a.dbg && q == 0 && tid == 0) a.dbg[11] += clock64() - tfin0;
}

template <typename T, bool REG>
__global__ void __launch_bounds__(kSvdNT, 1) svd_kernel(const __grid_constant__ SvdArgs a) {
  svd_body<T, REG>(a);
}
// batched problems: one cluster per problem (cluster id along x)
template <typename T, bool REG>
__global__ void __launch_bounds__(kSvdNT, 1) svd_kernel_batched(const SvdArgs* __restrict__ as) {
  cg::cluster_group cl = cg::this_cluster();
  svd_body<T, REG>(as[blockIdx.x / cl.num_blocks()]);
}

size_t svd_smem_bytes(int n, int m, int kk, int cs) {
  return (size_t)svd_layout(n, m, kk, cs).total * sizeof(double);
}

// ~32 rows of G per CTA; more CTAs (up to 16) while that lets G's row block
// stay resident in shared memory.
int svd_pick_cluster(int n, int m, int kk) {
  int cs = (n + 31) / 32;
  if (cs < 1) cs = 1;
  if (cs > 16) cs = 16;
  int c2 = cs;
  while (c2 < 16 && !svd_layout(n, m, kk, c2).gq_smem) ++c2;
  if (svd_layout(n, m, kk, c2).gq_smem) cs = c2;
  return cs;
}

template <typename T>
cudaError_t launch_svd(const SvdArgs& a, int cs, cudaStream_t st, cudaEvent_t after_gram) {
  const int nt = (a.n + 31) / 32;
  static std::atomic<unsigned long long> gram_devs{0};  // once per device
  cudaError_t e = smem_attr_once(gram_devs, gram_kernel, kGramSmem);
  if (e != cudaSuccess) return e;
  gram_kernel<<<(unsigned)(nt * (nt + 1) / 2), 256, kGramSmem, st>>>(a.U, a.ldu, a.m, a.n,
                                                                     const_cast<double*>(a.G), a.ldg, a.done);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (after_gram) {  // (overlapped loop: gates the previous iteration's strips)
    e = cudaEventRecord(after_gram, st);
    if (e != cudaSuccess) return e;
  }
  const size_t smem = svd_smem_bytes(a.n, a.m, a.kk, cs);
  // kk <= 8 (r <= 6): the kernel with the register-resident small solvers;
  // larger blocks: the shared-memory solvers only (its registers and code
  // are not shared with the small-kk paths)
  const bool reg = a.small_reg && sreg_supported(a.kk);
  auto kern = reg ? svd_kernel<T, true> : svd_kernel<T, false>;
  static std::atomic<unsigned long long> devs_reg{0}, devs_std{0};  // once per device
  e = reg ? smem_attr_once(devs_reg, svd_kernel<T, true>, 227 * 1024, true)
          : smem_attr_once(devs_std, svd_kernel<T, false>, 227 * 1024, true);
  if (e != cudaSuccess) return e;
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
  return cudaLaunchKernelEx(&cfg, kern, a);
}

bool svd_reg_path(const SvdArgs& a) { return a.small_reg && sreg_supported(a.kk); }

// Gram + SVD of n problems, one launch each: Gram blocks (tile, problem),
// one cs-CTA cluster per problem.  Every problem shares cs, the register
// path choice and the dynamic shared memory size (the largest).
template <typename T>
cudaError_t launch_svd_batched(const SvdArgs* d_args, int n, int max_n, int cs, size_t smem, bool reg,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int nt = (max_n + 31) / 32;
  static std::atomic<unsigned long long> gram_devs{0};
  cudaError_t e = smem_attr_once(gram_devs, gram_kernel_batched, kGramSmem);
  if (e != cudaSuccess) return e;
  gram_kernel_batched<<<dim3((unsigned)(nt * (nt + 1) / 2), (unsigned)n), 256, kGramSmem, st>>>(d_args);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  auto kern = reg ? svd_kernel_batched<T, true> : svd_kernel_batched<T, false>;
  static std::atomic<unsigned long long> devs_reg{0}, devs_std{0};
  e = reg ? smem_attr_once(devs_reg, svd_kernel_batched<T, true>, 227 * 1024, true)
          : smem_attr_once(devs_std, svd_kernel_batched<T, false>, 227 * 1024, true);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(cs * n), 1, 1);
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
  return cudaLaunchKernelEx(&cfg, kern, d_args);
}
template cudaError_t launch_svd_batched<float>(const SvdArgs*, int, int, int, size_t, bool, cudaStream_t);
template cudaError_t launch_svd_batched<double>(const SvdArgs*, int, int, int, size_t, bool, cudaStream_t);

template cudaError_t launch_svd<float>(const SvdArgs&, int, cudaStream_t, cudaEvent_t);
template cudaError_t launch_svd<double>(const SvdArgs&, int, cudaStream_t, cudaEvent_t);

}  // namespace ircur
