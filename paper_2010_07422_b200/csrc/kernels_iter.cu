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
__global__ void __launch_bounds__(256) core_kernel(CoreArgs<T> a) {
  if (*a.done) return;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int total = a.mI * a.nJ;
  if (idx >= total) return;
  const int k1 = idx / a.nJ, k2 = idx - k1 * a.nJ;
  const int64_t il = (int64_t)a.I[k1] - a.row0;
  const int j = a.J[k2];
  T pa[R], qb[R];
#pragma unroll
  for (int t = 0; t < R; ++t) {
    pa[t] = a.Pt[t * a.ldp + il];
    qb[t] = a.Qt[t * a.ldq + j];
  }
  if (k2 == 0) {
#pragma unroll
    for (int t = 0; t < R; ++t) a.PoldI[(int64_t)k1 * R + t] = pa[t];
  }
  if (k1 == 0) {
#pragma unroll
    for (int t = 0; t < R; ++t) a.QoldJ[(int64_t)k2 * R + t] = qb[t];
  }
  const T l = lowrank_entry<T, R>(pa, qb);
  const T d = a.D[il * a.ldd + j];
  T s;
  const T c = keep_value(d, l, a.zt, s);
  a.U[(int64_t)k1 * a.ldu + k2] = (double)c;
}

// ---------------------------------------------------------------- strips
constexpr int kStripNT = 256;
constexpr int kStripNW = kStripNT / 32;
constexpr int kStripTX = 64;       // positions per CTA (2 per lane)
constexpr int kStripLPT = 16;      // lines per thread (register-resident c values)
constexpr int kStripLPC = kStripNW * kStripLPT;  // lines per CTA

template <typename T, int R>
struct StripSmem {
  static constexpr int RP = ((R * (int)sizeof(T) + 15) / 16) * 16 / (int)sizeof(T);
  static constexpr size_t lvec = (size_t)kStripLPC * 3 * RP * sizeof(T);
  static constexpr size_t red = (size_t)kStripNW * R * kStripTX * sizeof(T);
  static constexpr size_t part = (size_t)R * kStripTX * sizeof(T);
  static constexpr size_t fnew = part;
  static constexpr size_t dred = 2 * kStripNW * sizeof(double);
  static constexpr size_t lidx = kStripLPC * sizeof(int);
  static constexpr size_t bytes = lvec + red + part + fnew + dred + lidx;
};

template <typename T>
__device__ __forceinline__ Pair<T> load_pair(const T* src, int64_t base, int x, int64_t ps,
                                             bool vec, bool v0, bool v1) {
  Pair<T> d;
  if (vec && v1) {
    if constexpr (sizeof(T) == 4) {
      d.v = __ldg(reinterpret_cast<const float2*>(src + base + x));
    } else {
      d.v = __ldg(reinterpret_cast<const double2*>(src + base + x));
    }
  } else {
    d.v.x = v0 ? __ldg(src + base + (int64_t)x * ps) : T(0);
    d.v.y = v1 ? __ldg(src + base + (int64_t)(x + 1) * ps) : T(0);
  }
  return d;
}

template <typename T, int R>
__global__ void __launch_bounds__(kStripNT, (sizeof(T) == 4 ? 2 : 1))
strips_kernel(const __grid_constant__ StripsArgs<T> a) {
  if (*a.done) return;  // uniform for the whole grid (flag written only by finalize)
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int cluster_id = blockIdx.x / CS;
  const int which = cluster_id < a.s[0].tiles ? 0 : 1;
  const StripDesc<T>& s = a.s[which];
  const int tile = which == 0 ? cluster_id : cluster_id - a.s[0].tiles;
  const int x0 = tile * kStripTX;
  const int per = (s.nk + CS - 1) / CS;
  const int kb = rank * per;
  const int nmy = max(0, min(s.nk, kb + per) - kb);

  using SM = StripSmem<T, R>;
  constexpr int RP = SM::RP;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* lvec = reinterpret_cast<T*>(smraw);
  T* red = reinterpret_cast<T*>(smraw + SM::lvec);
  T* part = reinterpret_cast<T*>(smraw + SM::lvec + SM::red);
  T* fnew = reinterpret_cast<T*>(smraw + SM::lvec + SM::red + SM::part);
  double* dred = reinterpret_cast<double*>(smraw + SM::lvec + SM::red + SM::part + SM::fnew);

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int xa = x0 + 2 * lane;
  const bool v0 = xa < s.npos, v1 = xa + 1 < s.npos;
  const bool vec = s.vec_ok != 0;
  // Issue every strip load of this thread first (all lines in flight at
  // once: memory-level parallelism = lines per thread), then stage the small
  // per-line vectors while the DRAM requests are outstanding.
  Pair<T> cv[kStripLPT];  // holds d, then c = d - s
  if (nmy > 0) {
    const int kl_last = nmy - 1;
#pragma unroll
    for (int j = 0; j < kStripLPT; ++j) {
      const int kl = min(w + kStripNW * j, kl_last);
      const int64_t base = (int64_t)(__ldg(s.lines + kb + kl) - s.line_off) * s.line_stride;
      cv[j] = load_pair<T>(s.src, base, xa, s.pos_stride, vec, v0, v1);
    }
  }
  for (int e = tid; e < nmy * 3 * R; e += kStripNT) {
    const int kl = e / (3 * R);
    const int rem = e - kl * 3 * R;
    const int vv = rem / R;
    const int t = rem - vv * R;
    const T* sv = vv == 0 ? s.lineA : (vv == 1 ? s.lineW : s.lineRes);
    lvec[(kl * 3 + vv) * RP + t] = sv[(int64_t)(kb + kl) * R + t];
  }
  Pair<T> b[R];
#pragma unroll
  for (int t = 0; t < R; ++t) {
    b[t].v.x = v0 ? s.Bold[t * s.ldb + xa] : T(0);
    b[t].v.y = v1 ? s.Bold[t * s.ldb + xa + 1] : T(0);
  }
  __syncthreads();

  const T zt = a.zt;
  Pair<T> acc[R];
#pragma unroll
  for (int t = 0; t < R; ++t) acc[t] = Pair<T>::splat(T(0));
  T den = T(0);
#pragma unroll
  for (int j = 0; j < kStripLPT; ++j) {
    const int kl = w + kStripNW * j;
    if (kl >= nmy) cv[j] = Pair<T>::splat(T(0));
    if (kl < nmy) {
      const Pair<T> d = cv[j];
      const T* av = lvec + (kl * 3) * RP;
      Pair<T> l = pmul(Pair<T>::splat(av[0]), b[0]);
#pragma unroll
      for (int t = 1; t < R; ++t) l = pfma(Pair<T>::splat(av[t]), b[t], l);
      T s0, s1;
      cv[j].v.x = keep_value(d.v.x, l.v.x, zt, s0);
      cv[j].v.y = keep_value(d.v.y, l.v.y, zt, s1);
      den = fma_rn(d.v.x, d.v.x, den);
      den = fma_rn(d.v.y, d.v.y, den);
      const T* wv = av + RP;
#pragma unroll
      for (int t = 0; t < R; ++t) acc[t] = pfma(Pair<T>::splat(wv[t]), cv[j], acc[t]);
    }
  }
  // cross-warp reduction (fixed order) -> this CTA's partial factor
#pragma unroll
  for (int t = 0; t < R; ++t) {
    red[(w * R + t) * kStripTX + 2 * lane] = acc[t].v.x;
    red[(w * R + t) * kStripTX + 2 * lane + 1] = acc[t].v.y;
  }
  __syncthreads();
  for (int o = tid; o < R * kStripTX; o += kStripNT) {
    T sum = red[o];
#pragma unroll
    for (int ww = 1; ww < kStripNW; ++ww) sum += red[ww * R * kStripTX + o];
    part[o] = sum;
  }
  // cluster reduction over the CTAs that split the lines (fixed rank order;
  // every CTA computes the identical sum)
  cl.sync();
  for (int o = tid; o < R * kStripTX; o += kStripNT) {
    T sum = *cl.map_shared_rank(part + o, 0);
    for (int q = 1; q < CS; ++q) sum += *cl.map_shared_rank(part + o, q);
    fnew[o] = sum;
  }
  __syncthreads();
  // positions in the other index set take the factor computed from the core
  // (Q(:,J) = W^T U, P(I,:) = U V Sigma^+), so both strips and the next
  // iteration see one value for the I x J block.
  if (s.nother > 0) {
    const int e0 = lower_bound_i32(s.other, s.nother, x0 + s.other_off);
    const int e1 = lower_bound_i32(s.other, s.nother, x0 + kStripTX + s.other_off);
    for (int e = e0 + tid; e < e1; e += kStripNT) {
      const int x = s.other[e] - s.other_off - x0;
#pragma unroll
      for (int t = 0; t < R; ++t) fnew[t * kStripTX + x] = s.otherF[(int64_t)e * R + t];
    }
  }
  cl.sync();  // peers finished reading `part`; fnew complete
  if (rank == 0) {
    for (int o = tid; o < R * kStripTX; o += kStripNT) {
      const int t = o / kStripTX, x = o - t * kStripTX;
      if (x0 + x < s.npos) s.Fnew[t * s.ldf + x0 + x] = fnew[o];
    }
  }
  // pass 2: stopping residual on the register-resident strip values
  Pair<T> f[R];
#pragma unroll
  for (int t = 0; t < R; ++t) {
    f[t].v.x = fnew[t * kStripTX + 2 * lane];
    f[t].v.y = fnew[t * kStripTX + 2 * lane + 1];
  }
  T res = T(0);
#pragma unroll
  for (int j = 0; j < kStripLPT; ++j) {
    const int kl = w + kStripNW * j;
    if (kl < nmy) {
      const T* rv = lvec + (kl * 3 + 2) * RP;
      Pair<T> l = pmul(Pair<T>::splat(rv[0]), f[0]);
#pragma unroll
      for (int t = 1; t < R; ++t) l = pfma(Pair<T>::splat(rv[t]), f[t], l);
      const T r0 = sub_rn(cv[j].v.x, l.v.x);
      const T r1 = sub_rn(cv[j].v.y, l.v.y);
      res = fma_rn(r0, r0, res);
      res = fma_rn(r1, r1, res);
    }
  }
  const double dsum = block_sum<kStripNT>((double)den, dred);
  const double rsum = block_sum<kStripNT>((double)res, dred + kStripNW);
  if (tid == 0) {
    a.partials[2 * blockIdx.x] = dsum;
    a.partials[2 * blockIdx.x + 1] = rsum;
  }
}

// ------------------------------------------------------------- finalize
constexpr int kFinNT = 512;

__global__ void __launch_bounds__(kFinNT) finalize_kernel(FinalizeArgs a) {
  if (*a.done) return;
  __shared__ double sh[4][kFinNT / 32];
  const int tid = threadIdx.x;
  // deterministic: each thread sums a fixed strided subset (loads unrolled,
  // adds in order), then a fixed butterfly per warp and a fixed warp order.
  double v[4] = {0, 0, 0, 0};
#pragma unroll 4
  for (int c = tid; c < a.ncta_rows; c += kFinNT) {
    const double2 p = *reinterpret_cast<const double2*>(a.partials + 2 * c);
    v[0] += p.x;
    v[1] += p.y;
  }
#pragma unroll 4
  for (int c = tid; c < a.ncta_cols; c += kFinNT) {
    const double2 p = *reinterpret_cast<const double2*>(a.partials + 2 * (a.ncta_rows + c));
    v[2] += p.x;
    v[3] += p.y;
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
    if (a.host_iters) {
      *a.host_iters = a.k + 1;
      if (fin) *a.host_done = 1;
      __threadfence_system();
    }
  }
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
  for (int rr = 0; rr < nrows; ++rr) {
    O* out = L + (xr0 + rr) * ldl + y0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (y0 + u < n2) out[u] = (O)lowrank_entry<T, R>(ps[rr], q[u]);
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

template <typename T>
size_t strips_smem_bytes(int R) {
  size_t b = 0;
  IRCUR_DISPATCH_RANK(R, RR, b = StripSmem<T, RR>::bytes);
  return b;
}

template <typename T, int R>
static cudaError_t launch_strips_r(const StripsArgs<T>& a, int cs, cudaStream_t st) {
  const size_t smem = StripSmem<T, R>::bytes;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(strips_kernel<T, R>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute(strips_kernel<T, R>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr_done = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((a.s[0].tiles + a.s[1].tiles) * cs), 1, 1);
  cfg.blockDim = dim3(kStripNT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, strips_kernel<T, R>, a);
}

template <typename T>
cudaError_t launch_strips(const StripsArgs<T>& a, int R, int cs, cudaStream_t st) {
  if (a.s[0].tiles + a.s[1].tiles == 0) return cudaSuccess;
  cudaError_t e = cudaErrorInvalidValue;
  IRCUR_DISPATCH_RANK(R, RR, e = launch_strips_r<T, RR>(a, cs, st));
  return e;
}

int strips_lines_per_cta() { return kStripLPC; }
int strips_tx() { return kStripTX; }

cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t st) {
  finalize_kernel<<<1, kFinNT, 0, st>>>(a);
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
  template size_t strips_smem_bytes<T>(int);                                               \
  template cudaError_t launch_strips<T>(const StripsArgs<T>&, int, int, cudaStream_t);     \
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
