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
      v = s.otherF[(int64_t)o * R + t];
    } else {
      v = red[pl][0][t];
#pragma unroll
      for (int ww = 1; ww < kSmpW; ++ww) v += red[pl][ww][t];
    }
    s.out[(int64_t)p * R + t] = v;
  }
}

cudaError_t launch_sampled_factors(const SampledArgs& a, int R, cudaStream_t st) {
  const int n = a.s[0].npos > a.s[1].npos ? a.s[0].npos : a.s[1].npos;
  if (n == 0) return cudaSuccess;
  if (R > kSmpW) return cudaErrorNotSupported;  // one thread per factor entry in the final sum
  dim3 grid((unsigned)((n + kSmpPos - 1) / kSmpPos), 2);
  cudaError_t e = cudaErrorInvalidValue;
  IRCUR_DISPATCH_RANK(R, RR, {
    sampled_factors_kernel<RR><<<grid, kSmpPos * kSmpW, 0, st>>>(a);
    e = cudaGetLastError();
  });
  return e;
}

}  // namespace ircur
