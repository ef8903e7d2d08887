// Per-solve passes over D and the BASELINE synthetic generator (sm_100a).
//
//   prep     : one read of D -> non-finite flag, max|D|, optional column-major
//              copy Dt for the column strip (matcore.require_finite,
//              matcore.py:70-77, and inf_norm, matcore.py:87-91).
//   slab norm: ||D(I,:)||^2, ||D(:,J)||^2 for the den == 0 early exit
//              (solver.py:331-341).
//   generator: BASELINE.json configs — W V^T + Bernoulli/uniform outliers,
//              drawing the SAME PCG64 stream numpy's Generator.random() /
//              .uniform() would (see oracle.ircur_oracle.baseline_problem).
#include <cuda_runtime.h>
#include <stdint.h>

#include "ircur_common.cuh"
#include "launchers.cuh"
#include <cstdlib>
#include <algorithm>
#include <type_traits>

namespace ircur {

// ------------------------------------------------------------------- prep
constexpr int kTT = 32;  // transpose tile

template <typename T>
__global__ void __launch_bounds__(256) prep_transpose_kernel(const T* __restrict__ D, int64_t ldd,
                                                             int64_t nloc, int64_t n2, T* __restrict__ Dt,
                                                             int64_t ldt, unsigned long long* maxbits,
                                                             int* nonfinite) {
  __shared__ T tile[kTT][kTT + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int64_t cb = (int64_t)blockIdx.x * kTT, rb = (int64_t)blockIdx.y * kTT;
  double mx = 0.0;
  int bad = 0;
#pragma unroll
  for (int k = 0; k < kTT; k += 8) {
    const int64_t r = rb + ty + k, c = cb + tx;
    T v = T(0);
    if (r < nloc && c < n2) {
      v = __ldcs(D + r * ldd + c);
      const double av = fabs((double)v);
      if (!isfinite(av)) bad = 1; else mx = fmax(mx, av);
    }
    tile[ty + k][tx] = v;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kTT; k += 8) {
    const int64_t c = cb + ty + k, r = rb + tx;
    if (r < nloc && c < n2) __stcs(Dt + c * ldt + r, tile[tx][ty + k]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if (tx == 0) {
    if (mx > 0.0) atomicMax(maxbits, dbits(mx));
    if (bad) atomicOr(nonfinite, 1);
  }
}

template <typename T>
__device__ __forceinline__ void prep_scan_kernel_body(const T* __restrict__ D, int64_t ldd, int64_t nloc, int64_t n2, unsigned long long* maxbits, int* nonfinite, int64_t bx, int64_t nbx) {
  double mx = 0.0;
  int bad = 0;
  const int64_t total = nloc * n2;
  const int64_t stride = nbx * blockDim.x;
  for (int64_t e = bx * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t r = e / n2, c = e - r * n2;
    const double av = fabs((double)__ldcs(D + r * ldd + c));
    if (!isfinite(av)) bad = 1; else mx = fmax(mx, av);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (mx > 0.0) atomicMax(maxbits, dbits(mx));
    if (bad) atomicOr(nonfinite, 1);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) prep_scan_kernel(const T* __restrict__ D, int64_t ldd, int64_t nloc, int64_t n2, unsigned long long* maxbits, int* nonfinite) {
  prep_scan_kernel_body(D, ldd, nloc, n2, maxbits, nonfinite, blockIdx.x, gridDim.x);
}

// contiguous rows, 16-byte vector loads (ldd*sizeof(T) % 16 == 0, aligned base)
template <typename T>
__device__ __forceinline__ void prep_scan_vec_kernel_body(const T* __restrict__ D, int64_t ldd, int64_t nloc, int64_t n2, unsigned long long* maxbits, int* nonfinite, int64_t bx, int64_t nbx) {
  constexpr int VW = 16 / sizeof(T);
  using V4 = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  T mx = T(0);
  int bad = 0;
  const int64_t vpr = n2 / VW;  // full vectors per row
  const int64_t total = nloc * vpr;
  const int64_t stride = nbx * blockDim.x;
  constexpr int UN = 4;  // independent 16-byte loads in flight per thread
  int64_t e = bx * blockDim.x + threadIdx.x;
  if (ldd == n2) {  // dense rows: treat D as one flat vector array
    const V4* Dv = reinterpret_cast<const V4*>(D);
    for (; e + (UN - 1) * stride < total; e += UN * stride) {
      V4 v[UN];
#pragma unroll
      for (int u = 0; u < UN; ++u) v[u] = __ldcs(Dv + e + u * stride);
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        const T* pv = reinterpret_cast<const T*>(&v[u]);
#pragma unroll
        for (int w = 0; w < VW; ++w) {
          const T av = fabs(pv[w]);
          bad |= !isfinite(av);
          mx = fmax(mx, av);
        }
      }
    }
  }
  for (; e < total; e += stride) {
    const int64_t r = e / vpr, cv = e - r * vpr;
    const V4 v = __ldcs(reinterpret_cast<const V4*>(D + r * ldd) + cv);
    const T* pv = reinterpret_cast<const T*>(&v);
#pragma unroll
    for (int u = 0; u < VW; ++u) {
      const T av = fabs(pv[u]);
      bad |= !isfinite(av);
      mx = fmax(mx, av);
    }
  }
  // row tails
  const int64_t tail = n2 - vpr * VW;
  if (tail > 0) {
    for (int64_t e = bx * blockDim.x + threadIdx.x; e < nloc * tail; e += stride) {
      const int64_t r = e / tail, c = vpr * VW + (e - r * tail);
      const T av = fabs(D[r * ldd + c]);
      bad |= !isfinite(av);
      mx = fmax(mx, av);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (mx > 0.0) atomicMax(maxbits, dbits(mx));
    if (bad) atomicOr(nonfinite, 1);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) prep_scan_vec_kernel(const T* __restrict__ D, int64_t ldd, int64_t nloc, int64_t n2, unsigned long long* maxbits, int* nonfinite) {
  prep_scan_vec_kernel_body(D, ldd, nloc, n2, maxbits, nonfinite, blockIdx.x, gridDim.x);
}

// Persistent 64x64-tile transpose fused with the finite/max scan.  Each CTA
// walks tiles t = blockIdx.x + i*gridDim.x; `col_major_order` chooses whether
// consecutive tiles share a column band (writes of concurrently running CTAs
// land in the same 64 rows of Dt) or a row band (reads share 64 rows of D).
constexpr int kPT = 64;
template <typename T>
__device__ __forceinline__ void prep_transpose64_kernel_body(const T* __restrict__ D, int64_t ldd, int64_t nloc, int64_t n2, T* __restrict__ Dt, int64_t ldt, unsigned long long* maxbits, int* nonfinite, int col_major_order, int64_t bx, int64_t nbx) {
  __shared__ T tile[kPT][kPT + 1];
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
  constexpr int VW = 16 / sizeof(T);                      // elements per 16-byte vector
  constexpr int TPR = kPT / VW;                            // threads per 64-element row segment
  constexpr int RPI = 256 / TPR;                           // rows per vector pass
  const int vx = threadIdx.x % TPR, vy = threadIdx.x / TPR;
  using V4 = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  const bool vec_ok = ((ldd * (int64_t)sizeof(T)) % 16 == 0) && ((ldt * (int64_t)sizeof(T)) % 16 == 0) &&
                      ((uintptr_t)D % 16 == 0) && ((uintptr_t)Dt % 16 == 0);
  const int64_t tr = (nloc + kPT - 1) / kPT, tcn = (n2 + kPT - 1) / kPT;
  const int64_t ntiles = tr * tcn;
  T mx = T(0);
  int bad = 0;
  for (int64_t t = bx; t < ntiles; t += nbx) {
    int64_t br, bc;
    if (col_major_order) { bc = t / tr; br = t - bc * tr; } else { br = t / tcn; bc = t - br * tcn; }
    const int64_t rb = br * kPT, cb = bc * kPT;
    const bool full = (rb + kPT <= nloc) && (cb + kPT <= n2);
    if (full && vec_ok) {
      V4 v[kPT / RPI];
#pragma unroll
      for (int k = 0; k < kPT / RPI; ++k)
        v[k] = __ldcs(reinterpret_cast<const V4*>(D + (rb + vy + k * RPI) * ldd + cb) + vx);
#pragma unroll
      for (int k = 0; k < kPT / RPI; ++k) {
        const T* pv = reinterpret_cast<const T*>(&v[k]);
#pragma unroll
        for (int u = 0; u < VW; ++u) {
          const T av = fabs(pv[u]);
          bad |= !isfinite(av);
          mx = fmax(mx, av);
          tile[vy + k * RPI][vx * VW + u] = pv[u];
        }
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kPT / RPI; ++k) {
        const int c = vy + k * RPI;  // Dt row (= D column) within the tile
        V4 o;
        T* po = reinterpret_cast<T*>(&o);
#pragma unroll
        for (int u = 0; u < VW; ++u) po[u] = tile[vx * VW + u][c];
        __stcs(reinterpret_cast<V4*>(Dt + (cb + c) * ldt + rb) + vx, o);
      }
    } else {
#pragma unroll 4
      for (int k = 0; k < kPT; k += 4) {
        const int64_t r = rb + ty + k, c = cb + tx;
        T v = T(0);
        if (r < nloc && c < n2) {
          v = __ldcs(D + r * ldd + c);
          const T av = fabs(v);
          bad |= !isfinite(av);
          mx = fmax(mx, av);
        }
        tile[ty + k][tx] = v;
      }
      __syncthreads();
#pragma unroll 4
      for (int k = 0; k < kPT; k += 4) {
        const int64_t c = cb + ty + k, r = rb + tx;
        if (r < nloc && c < n2) __stcs(Dt + c * ldt + r, tile[tx][ty + k]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (mx > 0.0) atomicMax(maxbits, dbits(mx));
    if (bad) atomicOr(nonfinite, 1);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) prep_transpose64_kernel(const T* __restrict__ D, int64_t ldd, int64_t nloc, int64_t n2, T* __restrict__ Dt, int64_t ldt, unsigned long long* maxbits, int* nonfinite, int col_major_order) {
  prep_transpose64_kernel_body(D, ldd, nloc, n2, Dt, ldt, maxbits, nonfinite, col_major_order, blockIdx.x, gridDim.x);
}

template <typename T>
cudaError_t launch_prep(const T* D, int64_t ldd, int64_t nloc, int64_t n2, T* Dt, int64_t ldt,
                        unsigned long long* maxbits, int* nonfinite, int num_sms, cudaStream_t st) {
  if (nloc == 0 || n2 == 0) return cudaSuccess;
  if (Dt) {
    static const int mode = [] {
      const char* m = std::getenv("IRCUR_TRANSPOSE");
      return m ? std::atoi(m) : 1;
    }();
    if (mode == 0) {
      dim3 grid((unsigned)((n2 + kTT - 1) / kTT), (unsigned)((nloc + kTT - 1) / kTT));
      prep_transpose_kernel<T><<<grid, 256, 0, st>>>(D, ldd, nloc, n2, Dt, ldt, maxbits, nonfinite);
    } else {
      const int64_t ntiles = ((nloc + kPT - 1) / kPT) * ((n2 + kPT - 1) / kPT);
      const int64_t cap = (int64_t)num_sms * 8;
      const unsigned blocks = (unsigned)(ntiles < cap ? ntiles : cap);
      prep_transpose64_kernel<T><<<blocks, 256, 0, st>>>(D, ldd, nloc, n2, Dt, ldt, maxbits, nonfinite,
                                                         mode == 2 ? 0 : 1);
    }
  } else {
    const int64_t total = nloc * n2;
    int64_t want = (total + 256 * 8 - 1) / (256 * 8);
    const int64_t cap = (int64_t)num_sms * 8;
    const unsigned blocks = (unsigned)(want < cap ? (want < 1 ? 1 : want) : cap);
    const bool vec = ((ldd * (int64_t)sizeof(T)) % 16 == 0) && ((uintptr_t)D % 16 == 0);
    if (vec)
      prep_scan_vec_kernel<T><<<blocks, 256, 0, st>>>(D, ldd, nloc, n2, maxbits, nonfinite);
    else
      prep_scan_kernel<T><<<blocks, 256, 0, st>>>(D, ldd, nloc, n2, maxbits, nonfinite);
  }
  return cudaGetLastError();
}

// Sampled column-major copy: the same full read of D (finite flag, max|D|)
// but only the columns with colsel[c] >= 0 are written, to line colsel[c] of
// Dt.  The host selects the union of the column index sets the iterations
// will use (about 20% of D at n = 1e5), so the per-solve pass moves ~1.2x
// |D| instead of the 2x |D| of a full transpose.
template <typename T, int TR, int TC, bool NM>
__device__ __forceinline__ void prep_select_kernel_body(const T* __restrict__ D, int64_t ldd, int64_t nloc, int64_t n2, const int* __restrict__ colsel, T* __restrict__ Dt, int64_t ldt, unsigned long long* maxbits, int* nonfinite, int64_t bx, int64_t nbx) {
  // Each thread owns one 16-byte column group of a 64 x 64 tile in KR rows.
  // The next tile's vectors and column map are loaded before the current
  // tile is processed (register double buffering).  Selected columns are
  // staged in a compact, double-buffered shared buffer (slot = rank of the
  // column among the tile's selected columns, from a 16-lane shuffle scan
  // that every warp computes identically) and written out as 16-byte
  // vectors: one barrier per tile.
  constexpr int VW = 16 / sizeof(T);   // elements per vector
  constexpr int TPR = TC / VW;         // threads per TC-element row segment (one warp at most)
  constexpr int RPI = 256 / TPR;       // rows per pass
  constexpr int KR = TR / RPI;         // rows per thread
  constexpr int SL = TR + VW;          // staged column length (16-byte aligned rows)
  constexpr int CPW = TR / VW;         // vectors per staged column
  constexpr int NB = 2 * TC * SL * sizeof(T) <= 40 * 1024 ? 2 : 1;  // staging buffers (two when they fit 48 KB static)
  static_assert(TPR <= 32 && KR >= 1 && RPI * KR == TR, "tile shape");
  __shared__ __align__(16) T sbuf[NB][TC][SL];
  __shared__ int sdst[NB][TC];
  using V4 = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  using I4 = typename std::conditional<sizeof(T) == 4, int4, int2>::type;
  const int vx = threadIdx.x % TPR, vy = threadIdx.x / TPR;
  const int lane = threadIdx.x & 31;
  const bool vec_ok = ((ldd * (int64_t)sizeof(T)) % 16 == 0) && ((ldt * (int64_t)sizeof(T)) % 16 == 0) &&
                      ((uintptr_t)D % 16 == 0) && ((uintptr_t)Dt % 16 == 0) && (n2 % VW == 0);
  const int64_t tr = (nloc + TR - 1) / TR, tcn = (n2 + TC - 1) / TC;
  const int64_t ntiles = tr * tcn;
  T mx = T(0);
  int bad = 0;
  // fp32: max of |x| over the bit patterns (|x| >= +inf's pattern flags NaN/Inf),
  // or (NM) a NaN-propagating float max of |x|: one FMNMX per element
  uint32_t mbits = 0u;
  float fm = 0.f;
  // tile coordinates advanced incrementally (no 64-bit divisions in the loop)
  const int64_t grid = nbx;
  const int64_t gbr = grid / tcn, gbc = grid - gbr * tcn;
  auto advance = [&](int64_t& br, int64_t& bc) {
    br += gbr;
    bc += gbc;
    if (bc >= tcn) { bc -= tcn; ++br; }
  };
  auto full_tile = [&](int64_t br, int64_t bc) {
    return vec_ok && (br * TR + TR <= nloc) && (bc * TC + TC <= n2);
  };
  V4 nv[KR];
  I4 ncs;
  auto load = [&](int64_t br, int64_t bc) {
    const int64_t rb = br * TR, cb = bc * TC;
#pragma unroll
    for (int k = 0; k < KR; ++k) nv[k] = __ldcs(reinterpret_cast<const V4*>(D + (rb + vy + k * RPI) * ldd + cb) + vx);
    ncs = __ldg(reinterpret_cast<const I4*>(colsel + cb) + vx);
  };
  int64_t t = bx;
  int64_t br = t / tcn, bc = t - br * tcn;
  if (t < ntiles && full_tile(br, bc)) load(br, bc);
  int b = 0;
  for (; t < ntiles; t += grid, b = (b + 1) % NB) {
    const int64_t rb = br * TR, cb = bc * TC;
    int64_t nbr = br, nbc = bc;
    advance(nbr, nbc);
    const bool next_full = t + grid < ntiles && full_tile(nbr, nbc);
    if (full_tile(br, bc)) {
      V4 v[KR];
#pragma unroll
      for (int k = 0; k < KR; ++k) v[k] = nv[k];
      const I4 cs = ncs;
      if (next_full) load(nbr, nbc);
      const int* csp = reinterpret_cast<const int*>(&cs);
      int mine = 0;
#pragma unroll
      for (int u = 0; u < VW; ++u) mine += csp[u] >= 0;
      // exclusive scan of `mine` over the TPR lanes of this row segment
      int incl = mine;
#pragma unroll
      for (int o = 1; o < TPR; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o, TPR);
        if ((lane % TPR) >= o) incl += y;
      }
      const int total = __shfl_sync(0xffffffffu, incl, TPR - 1, TPR);
      int slot = incl - mine;
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        const T* pv = reinterpret_cast<const T*>(&v[k]);
        if constexpr (sizeof(T) == 4) {
#pragma unroll
          for (int u = 0; u < VW; ++u) {
            if constexpr (NM) {
              asm("max.NaN.f32 %0, %0, %1;" : "+f"(fm) : "f"(fabsf((float)pv[u])));
            } else {
              mbits = max(mbits, __float_as_uint(pv[u]) & 0x7fffffffu);
            }
          }
        } else {
#pragma unroll
          for (int u = 0; u < VW; ++u) {
            const T av = fabs(pv[u]);
            bad |= !isfinite(av);
            mx = fmax(mx, av);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < VW; ++u) {
        if (csp[u] >= 0) {
#pragma unroll
          for (int k = 0; k < KR; ++k) sbuf[b][slot][vy + k * RPI] = reinterpret_cast<const T*>(&v[k])[u];
          if (vy == 0) sdst[b][slot] = csp[u];
          ++slot;
        }
      }
      __syncthreads();
      for (int w = threadIdx.x; w < total * CPW; w += 256) {
        const int k = w / CPW, x = w - k * CPW;
        __stcs(reinterpret_cast<V4*>(Dt + (int64_t)sdst[b][k] * ldt + rb) + x,
               *reinterpret_cast<const V4*>(&sbuf[b][k][x * VW]));
      }
      if (NB == 1) __syncthreads();
    } else {
      // edge or unaligned tile: element-wise (each thread: one column, TR/(256/TC) rows)
      for (int e = threadIdx.x; e < TR * TC; e += 256) {
        const int kk = e / TC, tx = e - kk * TC;
        const int64_t c = cb + tx, r = rb + kk;
        if (r < nloc && c < n2) {
          const int d = colsel[c];
          const T val = __ldcs(D + r * ldd + c);
          const T av = fabs(val);
          bad |= !isfinite(av);
          mx = fmax(mx, av);
          if (d >= 0) Dt[(int64_t)d * ldt + r] = val;
        }
      }
      if (next_full) load(nbr, nbc);
      __syncthreads();  // keeps the staging-buffer reuse distance of two barriers
    }
    br = nbr;
    bc = nbc;
  }
  if constexpr (sizeof(T) == 4) {
    if constexpr (NM) {
      const bool fin = fm <= 3.402823466e38f;  // false for NaN and +inf
      bad |= !fin;
      mx = fmax(mx, fin ? fm : 0.f);
    } else {
      bad |= mbits >= 0x7f800000u;
      mx = fmax(mx, __uint_as_float(mbits < 0x7f800000u ? mbits : 0u));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (mx > 0.0) atomicMax(maxbits, dbits(mx));
    if (bad) atomicOr(nonfinite, 1);
  }
}

template <typename T, int TR, int TC, bool NM>
__global__ void __launch_bounds__(256) prep_select_kernel(const T* __restrict__ D, int64_t ldd, int64_t nloc, int64_t n2, const int* __restrict__ colsel, T* __restrict__ Dt, int64_t ldt, unsigned long long* maxbits, int* nonfinite) {
  prep_select_kernel_body<T, TR, TC, NM>(D, ldd, nloc, n2, colsel, Dt, ldt, maxbits, nonfinite, blockIdx.x, gridDim.x);
}

template <typename T>
cudaError_t launch_prep_select(const T* D, int64_t ldd, int64_t nloc, int64_t n2, const int* colsel, T* Dt,
                               int64_t ldt, unsigned long long* maxbits, int* nonfinite, int num_sms,
                               cudaStream_t st) {
  if (nloc == 0 || n2 == 0) return cudaSuccess;
  static const int shape = [] {  // tile shape (tuning knob): 0 = 64 x 64, 1 = 32 x 128, 2 = 64 x 128 rows x columns
    const char* e = std::getenv("IRCUR_PREP_SHAPE");
    // fp32 at cfg5 (sampled copy, same box): 8.33 ms (64 x 128: 512-byte row runs read, 256-byte
    // column runs written) vs 8.45 ms (32 x 128) vs 8.7 ms (64 x 64)
    return e ? std::atoi(e) : 2;
  }();
  const bool wide = sizeof(T) == 4 && shape >= 1;
  const int tr = wide && shape == 1 ? 32 : kPT, tc = wide ? 128 : kPT;
  const int64_t ntiles = ((nloc + tr - 1) / tr) * ((n2 + tc - 1) / tc);
  // persistent grid: every CTA resident (the loop strides over the tiles)
  auto grid_for = [&](auto kern) {
    static const int per_sm = [&] {  // once per kernel, thread-safe
      int v = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, 256, 0) != cudaSuccess || v < 1) v = 4;
      return v;
    }();
    const int64_t cap = (int64_t)num_sms * per_sm;
    return (unsigned)(ntiles < cap ? ntiles : cap);
  };
  static const int nanmax = [] {  // NaN-propagating float max (one FMNMX per element) vs the bit-pattern max
    const char* e = std::getenv("IRCUR_PREP_NANMAX");
    return e ? std::atoi(e) : 1;  // measured 8.11 vs 8.15 ms at cfg5 (same box)
  }();
  if constexpr (sizeof(T) == 4) {
    if (wide && shape == 2) {
      auto kern = prep_select_kernel<T, 64, 128, true>;
      kern<<<grid_for(kern), 256, 0, st>>>(D, ldd, nloc, n2, colsel, Dt, ldt, maxbits, nonfinite);
      return cudaGetLastError();
    }
    if (wide) {
      auto kern = nanmax ? prep_select_kernel<T, 32, 128, true> : prep_select_kernel<T, 32, 128, false>;
      kern<<<grid_for(kern), 256, 0, st>>>(D, ldd, nloc, n2, colsel, Dt, ldt, maxbits, nonfinite);
      return cudaGetLastError();
    }
  }
  auto kern = prep_select_kernel<T, kPT, kPT, false>;
  kern<<<grid_for(kern), 256, 0, st>>>(D, ldd, nloc, n2, colsel, Dt, ldt, maxbits, nonfinite);
  return cudaGetLastError();
}

// -------------------------------------------------------------- slab norms
// partials[blockIdx.x] = sum of squares of this CTA's share; rows part uses
// blocks [0, nb_rows), cols part blocks [nb_rows, nb_rows + nb_cols).
// Sum of squares of the line segment p[0, len) (contiguous), this thread's share.
// 16-byte vector loads on the aligned body, four in flight per thread.
template <typename T>
__device__ __forceinline__ double seg_sq(const T* __restrict__ p, int64_t len) {
  constexpr int V = 16 / sizeof(T);
  using VT = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  double acc = 0.0;
  int64_t head = (int64_t)((16 - ((uintptr_t)p & 15)) & 15) / sizeof(T);
  if (((uintptr_t)p % sizeof(T)) != 0) head = len;  // unaligned element type: scalar only
  head = head < len ? head : len;
  if ((int64_t)threadIdx.x < head) {
    const double v = (double)p[threadIdx.x];
    acc = fma(v, v, acc);
  }
  const VT* q = reinterpret_cast<const VT*>(p + head);
  const int64_t nv = (len - head) / V;
  int64_t i = threadIdx.x;
  for (; i + 3 * 256 < nv; i += 4 * 256) {
    VT a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = __ldg(q + i + u * 256);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const T* e = reinterpret_cast<const T*>(&a[u]);
#pragma unroll
      for (int w = 0; w < V; ++w) acc = fma((double)e[w], (double)e[w], acc);
    }
  }
  for (; i < nv; i += 256) {
    const VT a = __ldg(q + i);
    const T* e = reinterpret_cast<const T*>(&a);
#pragma unroll
    for (int w = 0; w < V; ++w) acc = fma((double)e[w], (double)e[w], acc);
  }
  const int64_t t0 = head + nv * V;
  if (t0 + (int64_t)threadIdx.x < len) {
    const double v = (double)p[t0 + threadIdx.x];
    acc = fma(v, v, acc);
  }
  return acc;
}

// ||D(I,:)||_F^2 (blocks [0, nb_rows)) and ||D(:,J)||_F^2 (the rest), one
// partial per block (fixed work split: deterministic).  Work unit = one line
// segment of kSlabSeg elements: a sampled row of D, or a column line of the
// column-major copy Dt when it holds D(:,J).
constexpr int64_t kSlabSeg = 8192;

template <typename T>
__device__ __forceinline__ void slab_sq_kernel_body(const T* D, int64_t ldd, int64_t row0, int64_t nloc, int64_t n2, const int* I, int mI, const int* J, int nJ, int nb_rows, double* partials, const T* Dt, int64_t ldt, const int* Jline, int64_t bx, int64_t nbx) {
  __shared__ double sh[8];
  double acc = 0.0;
  if ((int)bx < nb_rows) {
    const int64_t segs = (n2 + kSlabSeg - 1) / kSlabSeg, units = (int64_t)mI * segs;
    for (int64_t u = bx; u < units; u += nb_rows) {
      const int64_t k = u / segs, s = (u - k * segs) * kSlabSeg;
      const int64_t len = n2 - s < kSlabSeg ? n2 - s : kSlabSeg;
      acc += seg_sq(D + ((int64_t)I[k] - row0) * ldd + s, len);
    }
  } else {
    const int nb_cols = (int)nbx - nb_rows;
    const int cb = (int)bx - nb_rows;
    if (Dt) {  // the column-major copy holds D(:,J): contiguous lines
      const int64_t segs = (nloc + kSlabSeg - 1) / kSlabSeg, units = (int64_t)nJ * segs;
      for (int64_t u = cb; u < units; u += nb_cols) {
        const int64_t k = u / segs, s = (u - k * segs) * kSlabSeg;
        const int64_t len = nloc - s < kSlabSeg ? nloc - s : kSlabSeg;
        acc += seg_sq(Dt + (int64_t)Jline[k] * ldt + s, len);
      }
    } else {  // strided gather D(x, J[k]): one row x per step, threads along J
      for (int64_t x = cb; x < nloc; x += nb_cols) {
        const T* row = D + x * ldd;
        for (int k = threadIdx.x; k < nJ; k += 256) {
          const double v = (double)row[J[k]];
          acc = fma(v, v, acc);
        }
      }
    }
  }
  const double s = block_sum<256>(acc, sh);
  if (threadIdx.x == 0) partials[bx] = s;
}

template <typename T>
__global__ void __launch_bounds__(256) slab_sq_kernel(const T* D, int64_t ldd, int64_t row0, int64_t nloc, int64_t n2, const int* I, int mI, const int* J, int nJ, int nb_rows, double* partials, const T* Dt, int64_t ldt, const int* Jline) {
  slab_sq_kernel_body(D, ldd, row0, nloc, n2, I, mI, J, nJ, nb_rows, partials, Dt, ldt, Jline, blockIdx.x, gridDim.x);
}

template <typename T>
cudaError_t launch_slab_sq(const T* D, int64_t ldd, int64_t row0, int64_t nloc, int64_t n2,
                           const int* I, int mI, const int* J, int nJ, int nb_rows, int nb_cols,
                           double* partials, const T* Dt, int64_t ldt, const int* Jline, cudaStream_t st) {
  slab_sq_kernel<T><<<nb_rows + nb_cols, 256, 0, st>>>(D, ldd, row0, nloc, n2, I, mI, J, nJ, nb_rows,
                                                       partials, Dt, ldt, Jline);
  return cudaGetLastError();
}

// --------------------------------------------------------------- generator
// numpy PCG64 (XSL-RR 128/64): state' = state * M + inc; out = rotr(hi^lo, state'>>122)
__device__ __forceinline__ u128 mul128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}
__device__ __forceinline__ u128 add128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}
__device__ __constant__ u128 kPcgMult = {4865540595714422341ull, 2549297995355413924ull};

// advance the LCG by `delta` steps (Brown's algorithm, O(log delta))
__device__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mult = {1ull, 0ull}, acc_plus = {0ull, 0ull};
  u128 cur_mult = kPcgMult, cur_plus = inc;
  while (delta > 0) {
    if (delta & 1ull) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, u128{1ull, 0ull}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  return add128(mul128(acc_mult, state), acc_plus);
}
__device__ __forceinline__ uint64_t pcg_next(u128& st, u128 inc) {
  st = add128(mul128(st, kPcgMult), inc);
  const uint64_t x = st.hi ^ st.lo;
  const unsigned rot = (unsigned)(st.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
__device__ __forceinline__ double pcg_double(u128& st, u128 inc) {
  return (double)(pcg_next(st, inc) >> 11) * (1.0 / 9007199254740992.0);
}

constexpr int kGenNT = 256;
constexpr int kGenPer = 16;  // consecutive cells per thread

// L_ij accumulated exactly as the numpy restatement: W[:,0]*V[:,0], then
// + W[:,t]*V[:,t] (separate multiply and add, no FMA).
__device__ __forceinline__ double gen_L(const double* W, const double* V, int rank, int64_t i, int64_t j) {
  double l = __dmul_rn(W[i * rank], V[j * rank]);
  for (int t = 1; t < rank; ++t) l = __dadd_rn(l, __dmul_rn(W[i * rank + t], V[j * rank + t]));
  return l;
}

__global__ void __launch_bounds__(kGenNT) gen_kernel(GenArgs a) {
  __shared__ double shm[kGenNT / 32];
  __shared__ long long shq[kGenNT / 32];
  const int64_t cells = a.nrows * a.n2;
  const int64_t first = ((int64_t)blockIdx.x * kGenNT + threadIdx.x) * kGenPer;
  double mx = 0.0;
  long long q = 0;
  if (first < cells) {
    const int64_t gfirst = a.row0 * a.n2 + first;  // global row-major cell id
    const int64_t total = a.n1 * a.n2;
    u128 sm = a.st0, sv = a.st0;
    if (!a.stats_only) {
      sm = pcg_advance(a.st0, a.inc, (uint64_t)gfirst);
      sv = pcg_advance(a.st0, a.inc, (uint64_t)(total + gfirst));
    }
    const double A = a.amp_a;
    const double span = A - (-A);
    const int64_t last = min(cells, first + kGenPer);
    for (int64_t e = first; e < last; ++e) {
      const int64_t il = e / a.n2, j = e - il * a.n2;
      const double l = gen_L(a.W, a.V, a.rank, a.row0 + il, j);
      if (a.stats_only) {
        const double al = fabs(l);
        mx = fmax(mx, al);
        q += (long long)rint(al * 16777216.0);
      } else {
        const double um = pcg_double(sm, a.inc);
        const double uv = pcg_double(sv, a.inc);
        const double s = (um < a.alpha) ? __dadd_rn(-A, __dmul_rn(span, uv)) : 0.0;
        const double d = __dadd_rn(l, s);
        if (a.dtype == 0)
          reinterpret_cast<float*>(a.D)[il * a.ldd + j] = (float)d;
        else
          reinterpret_cast<double*>(a.D)[il * a.ldd + j] = d;
      }
    }
  }
  if (a.stats_only) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      q += __shfl_xor_sync(0xffffffffu, q, o);
    }
    if ((threadIdx.x & 31) == 0) {
      shm[threadIdx.x >> 5] = mx;
      shq[threadIdx.x >> 5] = q;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double m2 = 0.0;
      long long q2 = 0;
      for (int i = 0; i < kGenNT / 32; ++i) {
        m2 = fmax(m2, shm[i]);
        q2 += shq[i];
      }
      a.blk_max[blockIdx.x] = m2;
      a.blk_qsum[blockIdx.x] = q2;
    }
  }
}

cudaError_t launch_gen(const GenArgs& a, int64_t* nblocks_out, cudaStream_t st) {
  const int64_t cells = a.nrows * a.n2;
  const int64_t nb = (cells + (int64_t)kGenNT * kGenPer - 1) / ((int64_t)kGenNT * kGenPer);
  if (nblocks_out) *nblocks_out = nb;
  if (nb == 0) return cudaSuccess;
  gen_kernel<<<(unsigned)nb, kGenNT, 0, st>>>(a);
  return cudaGetLastError();
}
int64_t gen_blocks(int64_t nrows, int64_t n2) {
  const int64_t cells = nrows * n2;
  return (cells + (int64_t)kGenNT * kGenPer - 1) / ((int64_t)kGenNT * kGenPer);
}

// ------------------------------------------------- batched prep (ircur_batch_prepare_many)
// Every problem's prep pass, slab norms and result gather in one launch each
// (grid.y = problem): the same per-problem bodies as the single-problem
// launches, so max|D|, the non-finite flag, the column copy and the slab
// partials are those of each problem's own pass (the partials use the
// problem's own block split, and the gather adds them in the host's order).
__global__ void prep_batch_init_kernel(const PrepBatchArg* __restrict__ as, int n) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) {
    *as[p].maxbits = 0ull;
    *as[p].nonfinite = 0;
  }
}

template <typename T, int MODE>
__global__ void __launch_bounds__(256) prep_batched_kernel(const PrepBatchArg* __restrict__ as) {
  const PrepBatchArg& a = as[blockIdx.y];
  if (a.mode != MODE || a.nloc == 0 || a.n2 == 0) return;
  const T* D = static_cast<const T*>(a.D);
  if constexpr (MODE == 0) {
    const bool vec = ((a.ldd * (int64_t)sizeof(T)) % 16 == 0) && ((uintptr_t)D % 16 == 0);
    if (vec)
      prep_scan_vec_kernel_body<T>(D, a.ldd, a.nloc, a.n2, a.maxbits, a.nonfinite, blockIdx.x, gridDim.x);
    else
      prep_scan_kernel_body<T>(D, a.ldd, a.nloc, a.n2, a.maxbits, a.nonfinite, blockIdx.x, gridDim.x);
  } else if constexpr (MODE == 1) {
    prep_transpose64_kernel_body<T>(D, a.ldd, a.nloc, a.n2, static_cast<T*>(a.Dt), a.ldt, a.maxbits, a.nonfinite,
                                    1, blockIdx.x, gridDim.x);
  } else if constexpr (sizeof(T) == 4) {
    prep_select_kernel_body<T, 64, 128, true>(D, a.ldd, a.nloc, a.n2, a.colsel, static_cast<T*>(a.Dt), a.ldt,
                                              a.maxbits, a.nonfinite, blockIdx.x, gridDim.x);
  } else {
    prep_select_kernel_body<T, kPT, kPT, false>(D, a.ldd, a.nloc, a.n2, a.colsel, static_cast<T*>(a.Dt), a.ldt,
                                                a.maxbits, a.nonfinite, blockIdx.x, gridDim.x);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) slab_batched_kernel(const PrepBatchArg* __restrict__ as) {
  const PrepBatchArg& a = as[blockIdx.y];
  const int nb = a.nb_rows + a.nb_cols;
  if ((int)blockIdx.x >= nb) return;
  slab_sq_kernel_body<T>(static_cast<const T*>(a.D), a.ldd, a.row0, a.nloc, a.n2, a.I, a.mI, a.J, a.nJ, a.nb_rows,
                         a.partials, a.use_dt ? static_cast<const T*>(a.Dt) : nullptr, a.ldt, a.Jline, blockIdx.x,
                         nb);
}

// res[4 p ..]: max|D| (the maxbits pattern), non-finite flag, row-slab and
// column-slab sums of squares (partials added in order, as ircur_slab_sqnorms)
__global__ void prep_batch_gather_kernel(const PrepBatchArg* __restrict__ as, int n, double* __restrict__ res) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const PrepBatchArg& a = as[p];
  res[4 * (size_t)p] = __longlong_as_double((long long)*a.maxbits);
  res[4 * (size_t)p + 1] = (double)*a.nonfinite;
  double x = 0.0, y = 0.0;
  for (int i = 0; i < a.nb_rows; ++i) x += a.partials[i];
  for (int i = 0; i < a.nb_cols; ++i) y += a.partials[a.nb_rows + i];
  res[4 * (size_t)p + 2] = x;
  res[4 * (size_t)p + 3] = y;
}

template <typename T>
cudaError_t launch_prep_batched(const PrepBatchArg* d_args, const PrepBatchArg* h_args, int n, double* d_res,
                                cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n > 65535) return cudaErrorInvalidValue;
  constexpr int kTilesPerCta = 16;  // each CTA strides over ~16 of its problem's tiles
  int64_t want[3] = {0, 0, 0};
  int max_slab = 0;
  for (int p = 0; p < n; ++p) {
    const PrepBatchArg& a = h_args[p];
    if (a.mode < 0 || a.mode > 2) return cudaErrorInvalidValue;
    int64_t tiles;
    if (a.mode == 0) {
      tiles = (a.nloc * a.n2 + 256 * (16 / (int64_t)sizeof(T)) - 1) / (256 * (16 / (int64_t)sizeof(T)));
    } else if (a.mode == 1) {
      tiles = ((a.nloc + kPT - 1) / kPT) * ((a.n2 + kPT - 1) / kPT);
    } else {
      const int64_t tr = kPT, tc = sizeof(T) == 4 ? 128 : kPT;  // (the default shapes of launch_prep_select)
      tiles = ((a.nloc + tr - 1) / tr) * ((a.n2 + tc - 1) / tc);
    }
    want[a.mode] = std::max(want[a.mode], (tiles + kTilesPerCta - 1) / kTilesPerCta);
    max_slab = std::max(max_slab, a.nb_rows + a.nb_cols);
  }
  prep_batch_init_kernel<<<(n + 127) / 128, 128, 0, st>>>(d_args, n);
  if (want[0] > 0) prep_batched_kernel<T, 0><<<dim3((unsigned)std::min<int64_t>(want[0], 1 << 20), n), 256, 0, st>>>(d_args);
  if (want[1] > 0) prep_batched_kernel<T, 1><<<dim3((unsigned)std::min<int64_t>(want[1], 1 << 20), n), 256, 0, st>>>(d_args);
  if (want[2] > 0) prep_batched_kernel<T, 2><<<dim3((unsigned)std::min<int64_t>(want[2], 1 << 20), n), 256, 0, st>>>(d_args);
  if (max_slab > 0) slab_batched_kernel<T><<<dim3((unsigned)max_slab, n), 256, 0, st>>>(d_args);
  prep_batch_gather_kernel<<<(n + 127) / 128, 128, 0, st>>>(d_args, n, d_res);
  return cudaGetLastError();
}

// ------------------------------------------------------ column gather
// Columns cols[0, ncols) of the row-major D into lines [slot0, slot0 + ncols)
// of the column-major copy (extend_cover: the loop ran past the sets the prep
// pass covered).  64 x 32 tiles through shared memory: the reads are one
// 32-byte sector per element (strided columns), the writes 256-byte runs.
constexpr int kGcRows = 64, kGcCols = 32;
template <typename T>
__global__ void __launch_bounds__(256) gather_cols_kernel(const T* __restrict__ D, int64_t ldd, int64_t nloc,
                                                          const int* __restrict__ cols, int ncols,
                                                          T* __restrict__ Dt, int64_t ldt, int64_t slot0) {
  __shared__ T tile[kGcRows][kGcCols + 1];
  const int64_t r0 = (int64_t)blockIdx.x * kGcRows;
  const int c0 = blockIdx.y * kGcCols;
  const int tid = threadIdx.x;
  {
    const int cc = tid & (kGcCols - 1);
    const int64_t col = c0 + cc < ncols ? cols[c0 + cc] : -1;
#pragma unroll
    for (int rr = tid / kGcCols; rr < kGcRows; rr += 256 / kGcCols)
      tile[rr][cc] = (col >= 0 && r0 + rr < nloc) ? D[(r0 + rr) * ldd + col] : T(0);
  }
  __syncthreads();
  {
    const int rr = tid & (kGcRows - 1);
#pragma unroll
    for (int cc = tid / kGcRows; cc < kGcCols; cc += 256 / kGcRows)
      if (c0 + cc < ncols && r0 + rr < nloc) Dt[(slot0 + c0 + cc) * ldt + r0 + rr] = tile[rr][cc];
  }
}

template <typename T>
cudaError_t launch_gather_cols(const T* D, int64_t ldd, int64_t nloc, const int* cols, int ncols, T* Dt,
                               int64_t ldt, int64_t slot0, cudaStream_t st) {
  if (ncols <= 0 || nloc <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((nloc + kGcRows - 1) / kGcRows), (unsigned)((ncols + kGcCols - 1) / kGcCols));
  gather_cols_kernel<T><<<grid, 256, 0, st>>>(D, ldd, nloc, cols, ncols, Dt, ldt, slot0);
  return cudaGetLastError();
}

#define IRCUR_PREP_INST(T)                                                                       \
  template cudaError_t launch_prep<T>(const T*, int64_t, int64_t, int64_t, T*, int64_t,          \
                                      unsigned long long*, int*, int, cudaStream_t);              \
  template cudaError_t launch_prep_select<T>(const T*, int64_t, int64_t, int64_t, const int*, T*,  \
                                             int64_t, unsigned long long*, int*, int, cudaStream_t); \
  template cudaError_t launch_slab_sq<T>(const T*, int64_t, int64_t, int64_t, int64_t, const int*, \
                                         int, const int*, int, int, int, double*, const T*, int64_t, \
                                         const int*, cudaStream_t);                                      \
  template cudaError_t launch_prep_batched<T>(const PrepBatchArg*, const PrepBatchArg*, int, double*, cudaStream_t); \
  template cudaError_t launch_gather_cols<T>(const T*, int64_t, int64_t, const int*, int, T*, int64_t, int64_t, cudaStream_t);
IRCUR_PREP_INST(float)
IRCUR_PREP_INST(double)

}  // namespace ircur
