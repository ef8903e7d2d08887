// BIN matrix I/O to and from device memory (reference: mio.py:66-121).
//
// The reference's binary format stores rows x cols float64 values in
// column-major order after a 12-byte header.  The solver wants D row-major
// in HBM (possibly a row shard), so file column blocks are staged on the
// device and transposed here, with the finiteness check the reference's
// reader performs (first non-finite value in file order -> its flat index,
// from which the host reports the byte offset like mio.py:116-119).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ircur_b200.h"

namespace ircur {

constexpr int kTT2 = 32;

// src: column-major block, `nr` rows (leading dimension ldsrc) x `nc`
// columns (fp64); dst: row-major, columns [0, nc) of rows [0, nr) at ld ldd.
// first_bad: atomicMin of (global flat file index) of non-finite values.
template <typename O>
__global__ void __launch_bounds__(256) colmajor_to_rowmajor_kernel(const double* __restrict__ src, int64_t ldsrc,
                                                                   int64_t nr, int64_t nc, O* __restrict__ dst,
                                                                   int64_t ldd, int64_t file_rows, int64_t row0,
                                                                   int64_t col0, unsigned long long* first_bad) {
  __shared__ double tile[kTT2][kTT2 + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int64_t rb = (int64_t)blockIdx.x * kTT2, cb = (int64_t)blockIdx.y * kTT2;
#pragma unroll
  for (int k = 0; k < kTT2; k += 8) {
    const int64_t c = cb + ty + k, r = rb + tx;  // coalesced along rows of the column-major source
    double v = 0.0;
    if (r < nr && c < nc) {
      v = src[c * ldsrc + r];
      if (!isfinite(v)) atomicMin(first_bad, (unsigned long long)((col0 + c) * file_rows + row0 + r));
    }
    tile[ty + k][tx] = v;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kTT2; k += 8) {
    const int64_t r = rb + ty + k, c = cb + tx;  // coalesced along columns of the row-major target
    if (r < nr && c < nc) dst[r * ldd + c] = (O)tile[tx][ty + k];
  }
}

// src: row-major (rows [0, nr), columns [0, nc), ld lds) -> dst column-major fp64 (ld nr)
template <typename I>
__global__ void __launch_bounds__(256) rowmajor_to_colmajor_kernel(const I* __restrict__ src, int64_t lds, int64_t nr,
                                                                   int64_t nc, double* __restrict__ dst) {
  __shared__ double tile[kTT2][kTT2 + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t rb = (int64_t)blockIdx.x * kTT2, cb = (int64_t)blockIdx.y * kTT2;
#pragma unroll
  for (int k = 0; k < kTT2; k += 8) {
    const int64_t r = rb + ty + k, c = cb + tx;
    tile[ty + k][tx] = (r < nr && c < nc) ? (double)src[r * lds + c] : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kTT2; k += 8) {
    const int64_t c = cb + ty + k, r = rb + tx;
    if (r < nr && c < nc) dst[c * nr + r] = tile[tx][ty + k];
  }
}

}  // namespace ircur

using namespace ircur;

extern "C" int ircur_bin_block_to_rowmajor(const double* src, int64_t ldsrc, int64_t nr, int64_t nc, void* dst,
                                           int64_t ldd, int dst_dtype, int64_t file_rows, int64_t row0,
                                           int64_t col0, unsigned long long* first_bad, void* stream) {
  if (!src || !dst || !first_bad || nr < 0 || nc < 0 || ldsrc < nr || ldd < nc) return IRCUR_EINVAL;
  if (nr == 0 || nc == 0) return IRCUR_OK;
  dim3 grid((unsigned)((nr + kTT2 - 1) / kTT2), (unsigned)((nc + kTT2 - 1) / kTT2));
  cudaStream_t st = (cudaStream_t)stream;
  if (dst_dtype == IRCUR_F64)
    colmajor_to_rowmajor_kernel<double><<<grid, 256, 0, st>>>(src, ldsrc, nr, nc, (double*)dst, ldd, file_rows, row0,
                                                              col0, first_bad);
  else if (dst_dtype == IRCUR_F32)
    colmajor_to_rowmajor_kernel<float><<<grid, 256, 0, st>>>(src, ldsrc, nr, nc, (float*)dst, ldd, file_rows, row0,
                                                             col0, first_bad);
  else
    return IRCUR_EINVAL;
  return cudaGetLastError() == cudaSuccess ? IRCUR_OK : IRCUR_ECUDA;
}

extern "C" int ircur_rowmajor_to_bin_block(const void* src, int64_t lds, int src_dtype, int64_t nr, int64_t nc,
                                           double* dst, void* stream) {
  if (!src || !dst || nr < 0 || nc < 0 || lds < nc) return IRCUR_EINVAL;
  if (nr == 0 || nc == 0) return IRCUR_OK;
  dim3 grid((unsigned)((nr + kTT2 - 1) / kTT2), (unsigned)((nc + kTT2 - 1) / kTT2));
  cudaStream_t st = (cudaStream_t)stream;
  if (src_dtype == IRCUR_F64)
    rowmajor_to_colmajor_kernel<double><<<grid, 256, 0, st>>>((const double*)src, lds, nr, nc, dst);
  else if (src_dtype == IRCUR_F32)
    rowmajor_to_colmajor_kernel<float><<<grid, 256, 0, st>>>((const float*)src, lds, nr, nc, dst);
  else
    return IRCUR_EINVAL;
  return cudaGetLastError() == cudaSuccess ? IRCUR_OK : IRCUR_ECUDA;
}
