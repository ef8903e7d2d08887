// The next iteration's sampled factor entries, ahead of the strips (fp32).
//
// Iteration k + 1's core needs only P_k(I_{k+1}, :) and Q_k(:, J_{k+1}) — the
// new factors at the next sampled rows and columns, which are drawn in
// advance (solver.py:362-370 uses them through L_k(I_{k+1}, J_{k+1})).  This
// kernel computes exactly those entries from iteration k's inputs (the old
// factors, the core SVD's W / V Sigma^+ and the overrides), so that core,
// Gram matrix and SVD of iteration k + 1 can run while the strip kernel of
// iteration k still streams the full strips.
//
// The arithmetic is that of strips3_kernel (kernels_strips3.cu) for one
// position: l = <A_line, B(:, x)> as lowrank_entry, e = d - T_zeta(d - l),
// then 16 partial sums (warp w of the strip kernel takes line pairs
// kp = w, w + 16, ...; in each pair line 2kp before 2kp + 1; the padding line
// of an odd count adds fma(0, 0, acc)) added in warp order, and the override
// of the other index set.  The results are therefore bitwise the strip
// kernel's values at those positions (checked by the core kernel's verify
// mode, tests/test_gpu_overlap.py).
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "kernels_iter.cuh"
#include "launchers.cuh"

namespace ircur {

constexpr int kSmpW = 16;    // partial sums per position (strips3_kernel's warps)
constexpr int kSmpPos = 16;  // positions per 256-thread block

template <int R>
__global__ void __launch_bounds__(256) sampled_factors_kernel(const __grid_constant__ SampledArgs a) {
  if (*a.done) return;
  const SampledStrip& s = a.s[blockIdx.y];
  __shared__ float red[kSmpPos][kSmpW][R];
  const int pl = threadIdx.x / kSmpW, w = threadIdx.x - pl * kSmpW;
  const int p = blockIdx.x * kSmpPos + pl;
  const bool live = p < s.npos;
  const int64_t x = live ? (int64_t)s.pos[p] - s.pos_off : 0;
  float acc[R];
#pragma unroll
  for (int t = 0; t < R; ++t) acc[t] = 0.f;
  if (live) {
    float b[R];
#pragma unroll
    for (int t = 0; t < R; ++t) b[t] = s.B[t * s.ldb + x];
    const int np = (s.nk + 1) / 2;
    auto elem = [&](int k) {
      const float d = s.src[(int64_t)(s.lines[k] - s.line_off) * s.line_stride + x * s.pos_stride];
      const float* A = s.lineA + (int64_t)k * R;
      float l = __fmul_rn(A[0], b[0]);
#pragma unroll
      for (int t = 1; t < R; ++t) l = __fmaf_rn(A[t], b[t], l);
      const float xd = __fmaf_rn(l, -1.f, d);
      const float sv = fabsf(xd) > a.zt ? xd : 0.f;
      return __fmaf_rn(sv, -1.f, d);
    };
    for (int kp = w; kp < np; kp += kSmpW) {
      const int k0 = 2 * kp, k1 = k0 + 1;
      const float e0 = elem(k0);
      const float e1 = k1 < s.nk ? elem(k1) : 0.f;
      const float* W0 = s.lineW + (int64_t)k0 * R;
      const float* W1 = s.lineW + (int64_t)k1 * R;
#pragma unroll
      for (int t = 0; t < R; ++t) {
        acc[t] = __fmaf_rn(W0[t], e0, acc[t]);
        acc[t] = __fmaf_rn(k1 < s.nk ? W1[t] : 0.f, e1, acc[t]);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < R; ++t) red[pl][w][t] = acc[t];
  __syncthreads();
  if (live && w < R) {  // thread (position, t): fixed warp order, then the override
    const int t = w;
    const int o = s.omap[x];
    float v;
    if (o >= 0) {
      v = s.zero_override ? 0.f : s.otherF[(int64_t)o * R + t];
    } else {
      v = red[pl][0][t];
#pragma unroll
      for (int ww = 1; ww < kSmpW; ++ww) v += red[pl][ww][t];
    }
    s.out[(int64_t)p * R + t] = v;
  }
}

// Staged variant: a block takes kSmpP positions of one strip.  Phase 1
// computes every thresholded element e(line, position) in parallel into
// shared memory (the element gathers and line loads are independent, so
// they overlap), phase 2 forms the 16 ordered partial sums per (position, t)
// from shared memory, phase 3 adds them in warp order.  Same operations in
// the same order as sampled_factors_kernel, so the same bits; several times
// more parallel memory traffic in flight.
constexpr int kSmpP = 4;
constexpr int kSmpB = 4;     // element gathers in flight per thread
constexpr int kSmpThreads = 512;

__host__ __device__ inline size_t sampled_staged_smem(int nk, int R) {
  const int nk2 = nk + (nk & 1);
  return ((size_t)nk2 * kSmpP + 2 * (size_t)nk2 * R + (size_t)kSmpP * R + (size_t)kSmpP * kSmpW * R) *
             sizeof(float) + (size_t)nk2 * sizeof(int);
}

// n floats global -> shared, 16-byte vectors when both sides allow it
__device__ __forceinline__ void smp_stage(float* dst, const float* __restrict__ src, int n, int tid, int nt) {
  if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
    const int n4 = n >> 2;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (int i = tid; i < n4; i += nt) d4[i] = __ldg(s4 + i);
    for (int i = 4 * n4 + tid; i < n; i += nt) dst[i] = __ldg(src + i);
  } else {
    for (int i = tid; i < n; i += nt) dst[i] = __ldg(src + i);
  }
}

template <int R>
__global__ void __launch_bounds__(kSmpThreads) sampled_staged_kernel(const __grid_constant__ SampledArgs a) {
  if (*a.done) return;
  const SampledStrip& s = a.s[blockIdx.y];
  const int p0 = blockIdx.x * kSmpP;
  if (p0 >= s.npos) return;
  const int nk = s.nk, nk2 = nk + (nk & 1);
  extern __shared__ __align__(16) float smp_sm[];
  float* sW = smp_sm;               // [nk2][R] line weights (row nk zero)
  float* sA = sW + nk2 * R;         // [nk2][R] old factor at the lines
  float* sE = sA + nk2 * R;         // [nk2][kSmpP] thresholded elements
  float* sB = sE + nk2 * kSmpP;     // [kSmpP][R] old factor at the positions
  float* red = sB + kSmpP * R;      // [kSmpP][kSmpW][R] partial sums
  int* sL = reinterpret_cast<int*>(red + kSmpP * kSmpW * R);  // [nk] line indices
  __shared__ int64_t xs[kSmpP];
  const int tid = threadIdx.x, nt = blockDim.x;
  // round 1: positions and line indices
  if (tid < kSmpP) xs[tid] = p0 + tid < s.npos ? (int64_t)s.pos[p0 + tid] - s.pos_off : -1;
  for (int i = tid; i < nk; i += nt) sL[i] = s.lines[i] - s.line_off;
  __syncthreads();
  // round 2: the element gathers (kept in registers) and, while they are in
  // flight, the line vectors and the old factor at the positions
  const int ne = nk * kSmpP;
  constexpr int kMaxE = 2;  // register batches of kSmpB gathers before the staging loads
  float d[kMaxE][kSmpB];
#pragma unroll
  for (int b = 0; b < kMaxE; ++b)
#pragma unroll
    for (int u = 0; u < kSmpB; ++u) {
      const int i = tid + (b * kSmpB + u) * nt;
      const int k = i / kSmpP, p = i - k * kSmpP;
      d[b][u] = i < ne && xs[p] >= 0 ? s.src[(int64_t)sL[k] * s.line_stride + xs[p] * s.pos_stride] : 0.f;
    }
  smp_stage(sW, s.lineW, nk * R, tid, nt);
  smp_stage(sA, s.lineA, nk * R, tid, nt);
  if (nk & 1) {
    for (int i = tid; i < R; i += nt) sW[nk * R + i] = 0.f;
    for (int i = tid; i < kSmpP; i += nt) sE[nk * kSmpP + i] = 0.f;
  }
  for (int i = tid; i < kSmpP * R; i += nt) {
    const int p = i / R, t = i - p * R;
    sB[i] = xs[p] >= 0 ? s.B[t * s.ldb + xs[p]] : 0.f;
  }
  __syncthreads();
  // phase 1: e(k, p) = d - T_zeta(d - <A_k, B(:, x_p)>), as strips3_kernel
  auto elem = [&](int i, float dv) {
    const int k = i / kSmpP, p = i - k * kSmpP;
    float e = 0.f;
    if (xs[p] >= 0) {
      const float* A = sA + k * R;
      const float* bb = sB + p * R;
      float l = __fmul_rn(A[0], bb[0]);
#pragma unroll
      for (int t = 1; t < R; ++t) l = __fmaf_rn(A[t], bb[t], l);
      const float xd = __fmaf_rn(l, -1.f, dv);
      const float sv = fabsf(xd) > a.zt ? xd : 0.f;
      e = __fmaf_rn(sv, -1.f, dv);
    }
    sE[i] = e;
  };
#pragma unroll
  for (int b = 0; b < kMaxE; ++b)
#pragma unroll
    for (int u = 0; u < kSmpB; ++u) {
      const int i = tid + (b * kSmpB + u) * nt;
      if (i < ne) elem(i, d[b][u]);
    }
  // (sets larger than kMaxE * kSmpB * nt / kSmpP lines: the rest in batches)
  for (int base = tid + kMaxE * kSmpB * nt; base < ne; base += kSmpB * nt) {
    float dd[kSmpB];
#pragma unroll
    for (int u = 0; u < kSmpB; ++u) {
      const int i = base + u * nt;
      const int k = i / kSmpP, p = i - k * kSmpP;
      dd[u] = i < ne && xs[p] >= 0 ? s.src[(int64_t)sL[k] * s.line_stride + xs[p] * s.pos_stride] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kSmpB; ++u) {
      const int i = base + u * nt;
      if (i < ne) elem(i, dd[u]);
    }
  }
  __syncthreads();
  // phase 2: partial w sums line pairs kp = w, w + 16, ...; 2kp before 2kp + 1
  const int npair = nk2 / 2;
  for (int i = tid; i < kSmpP * R * kSmpW; i += blockDim.x) {
    const int w = i % kSmpW, t = (i / kSmpW) % R, p = i / (kSmpW * R);
    float acc = 0.f;
    for (int kp = w; kp < npair; kp += kSmpW) {
      const int k0 = 2 * kp, k1 = k0 + 1;
      acc = __fmaf_rn(sW[k0 * R + t], sE[k0 * kSmpP + p], acc);
      acc = __fmaf_rn(sW[k1 * R + t], sE[k1 * kSmpP + p], acc);
    }
    red[(p * kSmpW + w) * R + t] = acc;
  }
  __syncthreads();
  // phase 3: fixed warp order, then the override of the other index set
  for (int i = tid; i < kSmpP * R; i += blockDim.x) {
    const int p = i / R, t = i - p * R;
    if (xs[p] < 0) continue;
    const int o = s.omap[xs[p]];
    float v;
    if (o >= 0) {
      v = s.zero_override ? 0.f : s.otherF[(int64_t)o * R + t];
    } else {
      v = red[(p * kSmpW) * R + t];
#pragma unroll
      for (int ww = 1; ww < kSmpW; ++ww) v += red[(p * kSmpW + ww) * R + t];
    }
    s.out[(int64_t)(p0 + p) * R + t] = v;
  }
}

cudaError_t launch_sampled_factors(const SampledArgs& a, int R, cudaStream_t st) {
  const int n = a.s[0].npos > a.s[1].npos ? a.s[0].npos : a.s[1].npos;
  if (n == 0) return cudaSuccess;
  if (R > kSmpW) return cudaErrorNotSupported;  // one thread per factor entry in the final sum
  const int nk = a.s[0].nk > a.s[1].nk ? a.s[0].nk : a.s[1].nk;
  const size_t smem = sampled_staged_smem(nk, R);
  static const bool legacy = std::getenv("IRCUR_SAMPLED_LEGACY") != nullptr;  // A/B knob
  cudaError_t e = cudaErrorInvalidValue;
  if (!legacy && smem <= 200 * 1024) {
    dim3 grid((unsigned)((n + kSmpP - 1) / kSmpP), 2);
    IRCUR_DISPATCH_RANK(R, RR, {
      static std::atomic<unsigned long long> devs{0};
      const cudaError_t attr = smem_attr_once(devs, sampled_staged_kernel<RR>, 200 * 1024);
      if (attr != cudaSuccess) return attr;
      sampled_staged_kernel<RR><<<grid, kSmpThreads, smem, st>>>(a);
      e = cudaGetLastError();
    });
    return e;
  }
  dim3 grid((unsigned)((n + kSmpPos - 1) / kSmpPos), 2);
  IRCUR_DISPATCH_RANK(R, RR, {
    sampled_factors_kernel<RR><<<grid, kSmpPos * kSmpW, 0, st>>>(a);
    e = cudaGetLastError();
  });
  return e;
}

}  // namespace ircur
