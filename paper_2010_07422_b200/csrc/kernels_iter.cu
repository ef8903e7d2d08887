// IRCUR per-iteration kernels for sm_100a: core gather/threshold, the fused
// row+column strip kernel (Phase I, Phase II factor reduction and stopping
// residual in one HBM pass), the stop check, the final strip write-out and
// the streaming rank-r materialiser.
//
// Reference semantics (file:line in /root/reference/pkg/src/ircur):
//   Phase I  s = T_zeta(d - l)          solver.py:375-377 (strict |x| > zeta, :153-168)
//   Phase II C = d_cols - s, R = ...     solver.py:380-382
//   residual e = (|R - L(I,:)| + |C - L(:,J)|) / den   solver.py:393-400
//   L(I',:) = C(I',:) V diag(inv) W^T R  solver.py:180-195, reassociated as P(I',:) Q
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "kernels_iter.cuh"

namespace cg = cooperative_groups;

namespace ircur {

// ------------------------------------------------------------------ core
template <typename T, int R>
__device__ __forceinline__ void core_body(const CoreArgs<T>& a, int bx) {
  if (*a.done) return;
  const int idx = bx * blockDim.x + threadIdx.x;
  const int total = a.mI * a.nJ;
  if (idx >= total) return;
  const int k1 = idx / a.nJ, k2 = idx - k1 * a.nJ;
  const int64_t il = (int64_t)a.I[k1] - a.row0;
  const int j = a.J[k2];
  T pa[R], qb[R];
  if (a.presampled) {
#pragma unroll
    for (int t = 0; t < R; ++t) {
      pa[t] = a.PoldI[(int64_t)k1 * R + t];
      qb[t] = a.QoldJ[(int64_t)k2 * R + t];
    }
  } else {
#pragma unroll
    for (int t = 0; t < R; ++t) {
      pa[t] = a.Pt[t * a.ldp + il];
      qb[t] = a.Qt[t * a.ldq + j];
    }
  }
  if (k2 == 0) {
    if (!a.presampled) {
#pragma unroll
      for (int t = 0; t < R; ++t) {
        if (a.verify && a.PoldI[(int64_t)k1 * R + t] != pa[t]) atomicAdd(a.mismatches, 1u);
        a.PoldI[(int64_t)k1 * R + t] = pa[t];
      }
    }
    a.rowmap[il] = a.upos0 + k1;
  }
  if (k1 == 0) {
    if (!a.presampled) {
#pragma unroll
      for (int t = 0; t < R; ++t) {
        if (a.verify && a.QoldJ[(int64_t)k2 * R + t] != qb[t]) atomicAdd(a.mismatches, 1u);
        a.QoldJ[(int64_t)k2 * R + t] = qb[t];
      }
    }
    a.colmap[j] = k2;
  }
  const T l = lowrank_entry<T, R>(pa, qb);
  const T d = a.D[il * a.ldd + j];
  T s;
  const T c = keep_value(d, l, a.zt, s);
  a.U[(int64_t)(a.upos0 + k1) * a.ldu + k2] = (double)c;
}

template <typename T, int R>
__global__ void __launch_bounds__(256) core_kernel(CoreArgs<T> a) { core_body<T, R>(a, (int)blockIdx.x); }

// batched problems (ircur_batched_run): problem blockIdx.y
template <typename T, int R>
__global__ void __launch_bounds__(256) core_kernel_batched(const CoreArgs<T>* __restrict__ as) {
  core_body<T, R>(as[blockIdx.y], (int)blockIdx.x);
}

// ------------------------------------------------------------- finalize
constexpr int kFinNT = 512;

__device__ __forceinline__ void finalize_body(const FinalizeArgs& a) {
  if (*a.done) return;
  __shared__ double sh[4][kFinNT / 32];
  const int tid = threadIdx.x;
  // the strips of this iteration are finished: reset the position maps
  if (!a.sums_out) {
    for (int e = tid; e < a.mI; e += kFinNT) a.rowmap[a.I[e] - a.row0] = -1;
    for (int e = tid; e < a.nJ; e += kFinNT) a.colmap[a.J[e]] = -1;
  }
  // deterministic: each thread sums a fixed strided subset (loads unrolled,
  // adds in order), then a fixed butterfly per warp and a fixed warp order.
  double v[4] = {0, 0, 0, 0};
#pragma unroll 4
  for (int c = tid; c < a.ncta_rows; c += kFinNT) {
    const double4 p = *reinterpret_cast<const double4*>(a.partials + 4 * c);
    v[0] += p.x;
    v[1] += p.y;
    v[2] += p.z;
    v[3] += p.w;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double ws = warp_sum(v[q]);
    if ((tid & 31) == 0) sh[q][tid >> 5] = ws;
  }
  __syncthreads();
  if (tid == 0) {
    double s[4] = {0, 0, 0, 0};
    for (int q = 0; q < 4; ++q)
      for (int i = 0; i < kFinNT / 32; ++i) s[q] += sh[q][i];
    if (a.sums_out) {  // row-sharded: local sums, all-reduced by the caller
      for (int q = 0; q < 4; ++q) a.sums_out[q] = s[q];
      return;
    }
    const double den = sqrt(s[0]) + sqrt(s[2]);
    const double e = (sqrt(s[1]) + sqrt(s[3])) / den;
    a.errors[a.k] = e;
    *a.iters = a.k + 1;
    int fin = 0;
    if (e <= a.eps) {
      *a.converged = 1;
      fin = 1;
    } else if (a.k + 1 >= a.max_iter) {
      fin = 1;
    }
    if (fin) *a.done = 1;
    if (a.host_iters) {  // iteration count visible before the stop flag (ircur_poll reads done first)
      *a.host_iters = a.k + 1;
      __threadfence_system();
      if (fin) {
        *a.host_done = 1;
        __threadfence_system();
      }
    }
  }
}

__global__ void __launch_bounds__(kFinNT) finalize_kernel(FinalizeArgs a) { finalize_body(a); }
__global__ void __launch_bounds__(kFinNT) finalize_kernel_batched(const FinalizeArgs* __restrict__ as) {
  finalize_body(as[blockIdx.x]);
}

// --------------------------------------------------------------- writeout
template <typename T, int R>
__global__ void writeout_rows_kernel(WriteoutArgs<T> a) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)a.mI * a.n2;
  if (idx >= total) return;
  const int k1 = (int)(idx / a.n2);
  const int64_t x = idx - (int64_t)k1 * a.n2;
  const int64_t il = a.I[k1] - a.row0;
  T pa[R], qb[R];
#pragma unroll
  for (int t = 0; t < R; ++t) {
    pa[t] = a.Pt[t * a.ldp + il];
    qb[t] = a.Qt[t * a.ldq + x];
  }
  const T l = lowrank_entry<T, R>(pa, qb);
  const T d = a.D[il * a.ldd + x];
  T s;
  const T c = keep_value(d, l, a.zt, s);
  if (a.R) a.R[idx] = (double)c;
  if (a.Srows) a.Srows[idx] = (double)s;
}

template <typename T, int R>
__global__ void writeout_cols_kernel(WriteoutArgs<T> a) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = a.nloc * a.nJ;
  if (idx >= total) return;
  const int64_t x = idx / a.nJ;
  const int k2 = (int)(idx - x * a.nJ);
  const int j = a.J[k2];
  T pa[R], qb[R];
#pragma unroll
  for (int t = 0; t < R; ++t) {
    pa[t] = a.Pt[t * a.ldp + x];
    qb[t] = a.Qt[t * a.ldq + j];
  }
  const T l = lowrank_entry<T, R>(pa, qb);
  const T d = a.D[x * a.ldd + j];
  T s;
  const T c = keep_value(d, l, a.zt, s);
  if (a.C) a.C[idx] = (double)c;
  if (a.Scols) a.Scols[idx] = (double)s;
}

// ------------------------------------------------------------ materialise
// L = P Q for local rows: each thread owns 4 consecutive columns (Q in
// registers), the CTA walks a chunk of rows with P rows staged in smem.
// Pure HBM write stream (solver.py:211-213 replaced by a K=rank writer).
constexpr int kMatNT = 256;
constexpr int kMatRows = 32;

template <typename T, typename O, int R>
__global__ void __launch_bounds__(kMatNT) materialize_kernel(const T* Pt, int64_t ldp, const T* Qt,
                                                             int64_t ldq, int64_t nloc, int64_t n2,
                                                             O* L, int64_t ldl) {
  __shared__ T ps[kMatRows][R];
  const int64_t y0 = ((int64_t)blockIdx.x * kMatNT + threadIdx.x) * 4;
  const int64_t xr0 = (int64_t)blockIdx.y * kMatRows;
  for (int e = threadIdx.x; e < kMatRows * R; e += kMatNT) {
    const int rr = e / R, t = e - rr * R;
    ps[rr][t] = (xr0 + rr < nloc) ? Pt[t * ldp + xr0 + rr] : T(0);
  }
  T q[4][R];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int t = 0; t < R; ++t) q[u][t] = (y0 + u < n2) ? Qt[t * ldq + y0 + u] : T(0);
  __syncthreads();
  const int nrows = (int)((nloc - xr0) < (int64_t)kMatRows ? (nloc - xr0) : (int64_t)kMatRows);
  // 16-byte stores when the row segment is whole and aligned (the common case)
  const bool vec = y0 + 3 < n2 && (ldl & 3) == 0 && ((reinterpret_cast<uintptr_t>(L) & 15) == 0);
  for (int rr = 0; rr < nrows; ++rr) {
    O* out = L + (xr0 + rr) * ldl + y0;
    O v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = (O)lowrank_entry<T, R>(ps[rr], q[u]);
    if (vec) {
      if constexpr (sizeof(O) == 4) {
        *reinterpret_cast<float4*>(out) = make_float4((float)v[0], (float)v[1], (float)v[2], (float)v[3]);
      } else {
        reinterpret_cast<double2*>(out)[0] = make_double2((double)v[0], (double)v[1]);
        reinterpret_cast<double2*>(out)[1] = make_double2((double)v[2], (double)v[3]);
      }
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (y0 + u < n2) out[u] = v[u];
    }
  }
}

// ----------------------------------------------------------------- launchers
template <typename T>
cudaError_t launch_core(const CoreArgs<T>& a, int R, cudaStream_t st) {
  const int total = a.mI * a.nJ;
  if (total == 0) return cudaSuccess;
  const int blocks = (total + 255) / 256;
  IRCUR_DISPATCH_RANK(R, RR, core_kernel<T, RR><<<blocks, 256, 0, st>>>(a));
  return cudaGetLastError();
}


cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t st) {
  finalize_kernel<<<1, kFinNT, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_finalize_batched(const FinalizeArgs* d_args, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  finalize_kernel_batched<<<n, kFinNT, 0, st>>>(d_args);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_core_batched(const CoreArgs<T>* d_args, int n, int max_total, int R, cudaStream_t st) {
  if (n <= 0 || max_total <= 0) return cudaSuccess;
  dim3 grid((unsigned)((max_total + 255) / 256), (unsigned)n);
  IRCUR_DISPATCH_RANK(R, RR, core_kernel_batched<T, RR><<<grid, 256, 0, st>>>(d_args));
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_writeout(const WriteoutArgs<T>& a, int R, cudaStream_t st) {
  const int64_t tr = (int64_t)a.mI * a.n2;
  const int64_t tc = a.nloc * a.nJ;
  if (tr > 0 && (a.R || a.Srows)) {
    const unsigned blocks = (unsigned)((tr + 255) / 256);
    IRCUR_DISPATCH_RANK(R, RR, writeout_rows_kernel<T, RR><<<blocks, 256, 0, st>>>(a));
  }
  if (tc > 0 && (a.C || a.Scols)) {
    const unsigned blocks = (unsigned)((tc + 255) / 256);
    IRCUR_DISPATCH_RANK(R, RR, writeout_cols_kernel<T, RR><<<blocks, 256, 0, st>>>(a));
  }
  return cudaGetLastError();
}

template <typename T, typename O>
cudaError_t launch_materialize(const T* Pt, int64_t ldp, const T* Qt, int64_t ldq, int64_t nloc,
                               int64_t n2, O* L, int64_t ldl, int R, cudaStream_t st) {
  if (nloc == 0 || n2 == 0) return cudaSuccess;
  dim3 grid((unsigned)((n2 + kMatNT * 4 - 1) / (kMatNT * 4)),
            (unsigned)((nloc + kMatRows - 1) / kMatRows));
  IRCUR_DISPATCH_RANK(R, RR,
                      (materialize_kernel<T, O, RR><<<grid, kMatNT, 0, st>>>(Pt, ldp, Qt, ldq, nloc, n2, L, ldl)));
  return cudaGetLastError();
}

#define IRCUR_INST(T)                                                                      \
  template cudaError_t launch_core<T>(const CoreArgs<T>&, int, cudaStream_t);              \
  template cudaError_t launch_core_batched<T>(const CoreArgs<T>*, int, int, int, cudaStream_t); \
  template cudaError_t launch_writeout<T>(const WriteoutArgs<T>&, int, cudaStream_t);      \
  template cudaError_t launch_materialize<T, float>(const T*, int64_t, const T*, int64_t,  \
                                                    int64_t, int64_t, float*, int64_t, int, \
                                                    cudaStream_t);                          \
  template cudaError_t launch_materialize<T, double>(const T*, int64_t, const T*, int64_t, \
                                                     int64_t, int64_t, double*, int64_t,   \
                                                     int, cudaStream_t);
IRCUR_INST(float)
IRCUR_INST(double)

}  // namespace ircur
