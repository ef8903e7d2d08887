// Background / foreground frames of the video pipeline on the device
// (reference: cli.py:217-230 run_video, mio.py:177-187 matrix_to_frames).
//
// For frames [t0, t0 + nt) (columns of D, pixels as rows, pixel (x, y) at row
// y + x * height): low = L(:, t) = P Q(:, t) (the solver's factors), resid =
// |D(:, t) - low|, peak_t = max over pixels (0 -> 1), fg = resid * 255 /
// peak_t; both low and fg are rounded to the nearest integer, clamped to
// [0, 255] and written as uint8 frames (t, y, x).  Pass 1 finds the peaks
// (max is order independent, so the float atomics are deterministic); pass 2
// writes the frames.  Arithmetic in fp64 like the reference.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ircur_b200.h"

namespace ircur {

constexpr int kVFT = 32;  // frames per CTA tile (threads along frames: coalesced D reads)
constexpr int kVRows = 8; // pixel rows per CTA tile

template <typename T>
__device__ __forceinline__ double low_entry(const T* Pt, int64_t ldp, const T* Q, int64_t ldq, int r, int64_t i,
                                            int64_t t) {
  double l = (double)Pt[i] * (double)Q[t];
  for (int k = 1; k < r; ++k) l = fma((double)Pt[k * ldp + i], (double)Q[k * ldq + t], l);
  return l;
}

template <typename T>
__global__ void __launch_bounds__(256) video_peak_kernel(const T* Pt, int64_t ldp, const T* Q, int64_t ldq,
                                                         const T* D, int64_t ldd, int64_t n1, int64_t t0, int nt,
                                                         int r, unsigned long long* peaks) {
  const int tf = threadIdx.x & (kVFT - 1), tr = threadIdx.x / kVFT;
  const int64_t t = (int64_t)blockIdx.x * kVFT + tf;
  double mx = 0.0;
  if (t < nt) {
    for (int64_t i = (int64_t)blockIdx.y * kVRows + tr; i < n1; i += (int64_t)gridDim.y * kVRows) {
      const double low = low_entry(Pt, ldp, Q, ldq, r, i, t0 + t);
      mx = fmax(mx, fabs((double)D[i * ldd + t0 + t] - low));
    }
    atomicMax(peaks + t, (unsigned long long)__double_as_longlong(mx));  // mx >= 0: bit order == value order
  }
}

__device__ __forceinline__ uint8_t to_pixel(double v) {
  v = rint(v);
  v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
  return (uint8_t)v;
}

template <typename T>
__global__ void __launch_bounds__(256) video_frames_kernel(const T* Pt, int64_t ldp, const T* Q, int64_t ldq,
                                                           const T* D, int64_t ldd, int64_t n1, int height,
                                                           int width, int64_t t0, int nt, int r,
                                                           const unsigned long long* peaks, uint8_t* bg,
                                                           uint8_t* fg) {
  const int tf = threadIdx.x & (kVFT - 1), tr = threadIdx.x / kVFT;
  const int64_t t = (int64_t)blockIdx.x * kVFT + tf;
  if (t >= nt) return;
  double pk = __longlong_as_double((long long)peaks[t]);
  if (pk == 0.0) pk = 1.0;
  const double scale = 255.0 / pk;
  const int64_t fsz = (int64_t)height * width;
  for (int64_t i = (int64_t)blockIdx.y * kVRows + tr; i < n1; i += (int64_t)gridDim.y * kVRows) {
    const double low = low_entry(Pt, ldp, Q, ldq, r, i, t0 + t);
    const double resid = fabs((double)D[i * ldd + t0 + t] - low);
    const int64_t x = i / height, y = i - x * height;  // row = y + x * height
    const int64_t o = t * fsz + y * width + x;
    bg[o] = to_pixel(low);
    fg[o] = to_pixel(resid * scale);
  }
}

}  // namespace ircur

using namespace ircur;

extern "C" int ircur_video_frames(const void* Pt, int64_t ldp, const void* Q, int64_t ldq, const void* D, int64_t ldd,
                                  int dtype, int64_t n1, int height, int width, int64_t t0, int nt, int rank,
                                  unsigned long long* peaks, uint8_t* bg, uint8_t* fg, void* stream) {
  if (!Pt || !Q || !D || !peaks || !bg || !fg || rank < 1 || nt < 0 || height < 1 || width < 1 ||
      (int64_t)height * width != n1)
    return IRCUR_EINVAL;
  if (nt == 0) return IRCUR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(peaks, 0, (size_t)nt * sizeof(unsigned long long), st) != cudaSuccess) return IRCUR_ECUDA;
  const int64_t gy = (n1 + kVRows - 1) / kVRows;
  dim3 grid((unsigned)((nt + kVFT - 1) / kVFT), (unsigned)(gy < 4096 ? gy : 4096));
  if (dtype == IRCUR_F32) {
    video_peak_kernel<float><<<grid, 256, 0, st>>>((const float*)Pt, ldp, (const float*)Q, ldq, (const float*)D, ldd,
                                                   n1, t0, nt, rank, peaks);
    video_frames_kernel<float><<<grid, 256, 0, st>>>((const float*)Pt, ldp, (const float*)Q, ldq, (const float*)D,
                                                     ldd, n1, height, width, t0, nt, rank, peaks, bg, fg);
  } else if (dtype == IRCUR_F64) {
    video_peak_kernel<double><<<grid, 256, 0, st>>>((const double*)Pt, ldp, (const double*)Q, ldq, (const double*)D,
                                                    ldd, n1, t0, nt, rank, peaks);
    video_frames_kernel<double><<<grid, 256, 0, st>>>((const double*)Pt, ldp, (const double*)Q, ldq,
                                                      (const double*)D, ldd, n1, height, width, t0, nt, rank, peaks,
                                                      bg, fg);
  } else {
    return IRCUR_EINVAL;
  }
  return cudaGetLastError() == cudaSuccess ? IRCUR_OK : IRCUR_ECUDA;
}
