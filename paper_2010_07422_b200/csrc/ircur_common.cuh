// Shared device helpers for the IRCUR B200 kernels (sm_100a).
//
// The single most important invariant lives here: every kernel that needs
// an entry of the low-rank iterate L_k(i,j) = sum_t P(i,t) Q(t,j) evaluates
// it with the SAME rounded operation chain (mul, then fma in t order), and
// then applies the SAME threshold/difference sequence.  That makes the core
// U = (D-S)(I,J), the row strip R = (D-S)(I,:) and the column strip
// C = (D-S)(:,J) agree bitwise on the I x J intersection — the property the
// reference obtains with _sync_intersection (solver.py:216-221) and asserts
// in test_solver.py:169-177.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ircur {

constexpr int kMaxRank = 16;

// ---- scalar ops with explicit rounding (no contraction differences) ------
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// Pair of values for two adjacent positions.  float uses the sm_100 packed
// FFMA2/FMUL2/FADD2 instructions; each lane of a packed op is the same IEEE
// operation as the scalar one, so results are bitwise identical to the
// scalar chain used by the core kernel.
template <typename T> struct Pair;
template <> struct Pair<float> {
  float2 v;
  __device__ __forceinline__ static Pair splat(float a) { return {make_float2(a, a)}; }
};
template <> struct Pair<double> {
  double2 v;
  __device__ __forceinline__ static Pair splat(double a) { return {make_double2(a, a)}; }
};
__device__ __forceinline__ Pair<float> pmul(Pair<float> a, Pair<float> b) { return {__fmul2_rn(a.v, b.v)}; }
__device__ __forceinline__ Pair<float> pfma(Pair<float> a, Pair<float> b, Pair<float> c) { return {__ffma2_rn(a.v, b.v, c.v)}; }
__device__ __forceinline__ Pair<double> pmul(Pair<double> a, Pair<double> b) {
  return {make_double2(__dmul_rn(a.v.x, b.v.x), __dmul_rn(a.v.y, b.v.y))};
}
__device__ __forceinline__ Pair<double> pfma(Pair<double> a, Pair<double> b, Pair<double> c) {
  return {make_double2(__fma_rn(a.v.x, b.v.x, c.v.x), __fma_rn(a.v.y, b.v.y, c.v.y))};
}

// d - x per lane with one rounding (fma(x, -1, d) == d - x exactly rounded,
// i.e. bitwise the scalar sub_rn of each lane).
__device__ __forceinline__ Pair<float> psub(Pair<float> d, Pair<float> x) {
  return {__ffma2_rn(x.v, make_float2(-1.f, -1.f), d.v)};
}
__device__ __forceinline__ Pair<double> psub(Pair<double> d, Pair<double> x) {
  return {make_double2(__dsub_rn(d.v.x, x.v.x), __dsub_rn(d.v.y, x.v.y))};
}

// Threshold value in storage precision such that, for every value x of type
// T, (|x| > zt) <=> ((double)|x| > zeta).  For float this is zeta rounded
// toward -inf (computed on the host); for double it is zeta itself.
template <typename T> struct Zeta { T v; };

// Phase I + Phase II for one entry: s = T_zeta(d - l), c = d - s
// (solver.py:375-382).  Strict |x| > zeta (solver.py:153-168).
template <typename T>
__device__ __forceinline__ T keep_value(T d, T l, T zt, T& s_out) {
  T x = sub_rn(d, l);
  T s = (fabs(x) > zt) ? x : T(0);
  s_out = s;
  return sub_rn(d, s);
}

// keep_value for two adjacent entries (same per-lane operations).
template <typename T>
__device__ __forceinline__ Pair<T> keep_pair(Pair<T> d, Pair<T> l, T zt) {
  const Pair<T> x = psub(d, l);
  Pair<T> sv;
  sv.v.x = (fabs(x.v.x) > zt) ? x.v.x : T(0);
  sv.v.y = (fabs(x.v.y) > zt) ? x.v.y : T(0);
  return psub(d, sv);
}

// L_k(i,j) as the shared chain.  a: R values of the row factor, b: R values
// of the column factor (both in registers/shared memory).
template <typename T, int R>
__device__ __forceinline__ T lowrank_entry(const T* a, const T* b) {
  T l = mul_rn(a[0], b[0]);
#pragma unroll
  for (int t = 1; t < R; ++t) l = fma_rn(a[t], b[t], l);
  return l;
}

// ---- misc ----------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide deterministic fp64 sum (fixed tree), result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh /* >= NT/32 */) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) s += sh[i];
  }
  return s;
}

// Non-negative double as orderable uint64 (for atomicMax of |x|).
__device__ __forceinline__ unsigned long long dbits(double x) {
  return (unsigned long long)__double_as_longlong(x);
}

// First position p in sorted a[0..n) with a[p] >= key.
__device__ __forceinline__ int lower_bound_i32(const int* a, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Dispatch a runtime rank to a compile-time template argument.
#define IRCUR_DISPATCH_RANK(r, R, ...)                     \
  switch (r) {                                             \
    case 1: { constexpr int R = 1; __VA_ARGS__; } break;   \
    case 2: { constexpr int R = 2; __VA_ARGS__; } break;   \
    case 3: { constexpr int R = 3; __VA_ARGS__; } break;   \
    case 4: { constexpr int R = 4; __VA_ARGS__; } break;   \
    case 5: { constexpr int R = 5; __VA_ARGS__; } break;   \
    case 6: { constexpr int R = 6; __VA_ARGS__; } break;   \
    case 7: { constexpr int R = 7; __VA_ARGS__; } break;   \
    case 8: { constexpr int R = 8; __VA_ARGS__; } break;   \
    case 9: { constexpr int R = 9; __VA_ARGS__; } break;   \
    case 10: { constexpr int R = 10; __VA_ARGS__; } break; \
    case 11: { constexpr int R = 11; __VA_ARGS__; } break; \
    case 12: { constexpr int R = 12; __VA_ARGS__; } break; \
    case 13: { constexpr int R = 13; __VA_ARGS__; } break; \
    case 14: { constexpr int R = 14; __VA_ARGS__; } break; \
    case 15: { constexpr int R = 15; __VA_ARGS__; } break; \
    case 16: { constexpr int R = 16; __VA_ARGS__; } break; \
    default: break;                                        \
  }

}  // namespace ircur
