// Fused row + column strip kernel of the IRCUR hot path (sm_100a).
//
// One pass over the sampled strips per iteration:
//   Phase I   s = T_zeta(d - L_k)            (solver.py:375-377, strict |x| > zeta)
//   Phase II  c = d - s  (R = D(I,:) - S, C = D(:,J) - S)   (solver.py:380-382)
//   factor    Fnew(:,x) = sum_k W_k c_k(x)   (Q_{k+1} = W_r^T R, P_{k+1} = C V_r Sigma^+)
//   residual  sum (c - <Res_k, Fnew(:,x)>)^2 and sum d^2   (e_k, solver.py:393-400)
//
// Persistent CTAs (or thread-block clusters that split the sampled lines)
// walk 64-position tiles of both strips.  Every line segment of a tile (256 B
// fp32 / 512 B fp64) is fetched with a TMA bulk copy (cp.async.bulk) into a
// double-buffered shared-memory stage completed on an mbarrier, so the next
// tile streams from HBM while the current one is computed.  Tile values are
// thresholded in place in shared memory, reduced per tile (warps, then
// cluster CTAs over DSMEM, fixed order) and re-read for the residual.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>

#include "kernels_iter.cuh"
#include "launchers.cuh"

namespace cg = cooperative_groups;

namespace ircur {

constexpr int kSNT = 512;
constexpr int kSNW = kSNT / 32;
constexpr int kSTX = 64;  // positions per tile (2 per lane)
// lines processed together per warp (independent chains); fewer for wide
// (fp64 / large-rank) register footprints so nothing spills at 128 regs
template <typename T, int R>
__host__ __device__ constexpr int group_lines() { return (sizeof(T) == 8 && R > 5) ? 1 : ((sizeof(T) == 8 || R > 12) ? 2 : 4); }

struct StripsLayout {
  int RP;
  size_t seg, bars, stage, lptr, lvec, lidx, red, part, fnew, dred, total;
};

__host__ __device__ inline size_t align128(size_t x) { return (x + 127) & ~size_t(127); }

__host__ __device__ inline StripsLayout strips_layout(int maxl, int R, int esz) {
  StripsLayout L;
  L.RP = ((R * esz + 15) / 16) * 16 / esz;
  L.seg = (size_t)kSTX * esz;
  size_t off = 0;
  L.bars = off; off += 128;
  // per buffer: maxl line segments, the R rows of the old factor, then the
  // tile's 64 entries of the override map (ints)
  L.stage = off; off = align128(off + 2 * (size_t)(maxl + R + 1) * L.seg);
  L.lptr = off; off = align128(off + 2 * (size_t)(maxl + R) * sizeof(void*));
  L.lvec = off; off = align128(off + (size_t)maxl * 3 * L.RP * esz);
  L.lidx = off; off = align128(off + 2 * (size_t)maxl * sizeof(int));
  L.red = off; off = align128(off + (size_t)kSNW * R * L.seg);
  L.part = off; off = align128(off + 2 * (size_t)R * L.seg);
  L.fnew = off; off = align128(off + (size_t)R * L.seg);
  L.dred = off; off = align128(off + 4 * kSNW * sizeof(double));
  L.total = off;
  return L;
}

// ---- PTX helpers: mbarrier + TMA bulk copy -------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// cp.async (LDGSTS): 16-byte chunk with zero-fill beyond src_bytes, or one element
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* dst, const T* src, bool ok) {
  if constexpr (sizeof(T) == 4)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 4 : 0)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <typename T>
__device__ __forceinline__ Pair<T> lds_pair(const T* p) {
  Pair<T> v;
  if constexpr (sizeof(T) == 4) v.v = *reinterpret_cast<const float2*>(p);
  else v.v = *reinterpret_cast<const double2*>(p);
  return v;
}
template <typename T>
__device__ __forceinline__ void sts_pair(T* p, Pair<T> v) {
  if constexpr (sizeof(T) == 4) *reinterpret_cast<float2*>(p) = v.v;
  else *reinterpret_cast<double2*>(p) = v.v;
}

template <typename T, int R>
__global__ void __launch_bounds__(kSNT, 1) strips_kernel(const __grid_constant__ StripsArgs<T> a) {
  if (*a.done) return;  // uniform for the whole grid (flag written only by finalize)
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int ncl = gridDim.x / CS;
  const int cid = blockIdx.x / CS;
  const StripsLayout L = strips_layout(a.maxl, R, (int)sizeof(T));
  const int RP = L.RP;
  const int maxl = a.maxl;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bars);
  T* stage = reinterpret_cast<T*>(sm + L.stage);
  const T** lptr = reinterpret_cast<const T**>(sm + L.lptr);  // [2][maxl + R] segment sources
  T* lvec = reinterpret_cast<T*>(sm + L.lvec);
  int* lidx = reinterpret_cast<int*>(sm + L.lidx);
  T* red = reinterpret_cast<T*>(sm + L.red);
  T* part = reinterpret_cast<T*>(sm + L.part);
  T* fnew = reinterpret_cast<T*>(sm + L.fnew);
  double* dred = reinterpret_cast<double*>(sm + L.dred);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int tiles0 = a.s[0].tiles;
  const int total = tiles0 + a.s[1].tiles;
  const uint32_t seg = (uint32_t)L.seg;

  int kb[2], nmy[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int per = (a.s[q].nk + CS - 1) / CS;
    kb[q] = rank * per;
    nmy[q] = max(0, min(a.s[q].nk, kb[q] + per) - kb[q]);
  }
  for (int e = tid; e < nmy[0]; e += kSNT) lidx[e] = a.s[0].lines[kb[0] + e] - a.s[0].line_off;
  for (int e = tid; e < nmy[1]; e += kSNT) lidx[maxl + e] = a.s[1].lines[kb[1] + e] - a.s[1].line_off;
#pragma unroll
  for (int q = 0; q < 2; ++q) {  // line sources of the bulk path: my lines, then the factor rows
    const StripDesc<T>& s = a.s[q];
    if (!s.bulk_ok) continue;
    for (int e = tid; e < nmy[q] + R; e += kSNT)
      lptr[q * (maxl + R) + e] = e < nmy[q] ? s.src + (int64_t)(s.lines[kb[q] + e] - s.line_off) * s.line_stride
                                            : s.Bold + (int64_t)(e - nmy[q]) * s.ldb;
  }
  (void)bars; (void)seg;
  __syncthreads();

  auto tile_of = [&](int i, int& q, int& x0) -> bool {
    const int t = cid + i * ncl;
    if (t >= total) return false;
    q = t < tiles0 ? 0 : 1;
    x0 = (t - (q ? tiles0 : 0)) * kSTX;
    return true;
  };
  // every thread issues its share of the asynchronous copies (cp.async) of
  // tile i (the CTA's line segments + the R rows of the old factor) into
  // stage st, then commits one group (possibly empty: uniform group count).
  auto issue = [&](int i, int st) {
    int q, x0;
    if (tile_of(i, q, x0)) {
      const StripDesc<T>& s = a.s[q];
      const int* li = lidx + q * maxl;
      T* stg = stage + (size_t)st * (maxl + R + 1) * kSTX;
      T* bsg = stg + (size_t)maxl * kSTX;
      const int nl = nmy[q];
      if (tid < kSTX / 4) {  // override map of the tile: 16 x 16-byte chunks of ints
        const int pos = x0 + 4 * tid;
        const int rem = s.npos - pos;
        const int bytes = rem >= 4 ? 16 : (rem > 0 ? 4 * rem : 0);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         smem_u32(reinterpret_cast<int*>(stg + (size_t)(maxl + R) * kSTX) + 4 * tid)),
                     "l"(s.omap + (bytes ? pos : x0)), "r"(bytes)
                     : "memory");
      }
      if (s.bulk_ok) {
        // lane -> fixed 16-byte chunk of a segment, LPP segments per pass;
        // segment v < nl is line v, v >= nl the factor row v - nl
        constexpr int EPC = 16 / (int)sizeof(T);  // elements per 16-byte chunk
        constexpr int CPL = kSTX / EPC;           // chunks per line segment
        constexpr int LPP = kSNT / CPL;           // segments per pass
        const int ch = tid % CPL;
        const T* const* lp = lptr + q * (maxl + R);
        const uint32_t sb = smem_u32(stg) + ch * 16;
        const int nv = nl + R;
        if (x0 + kSTX <= s.npos) {
          for (int v = tid / CPL; v < nv; v += LPP) {
            const int dl = v < nl ? v : maxl + (v - nl);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sb + dl * kSTX * (int)sizeof(T)),
                         "l"(lp[v] + x0 + ch * EPC)
                         : "memory");
          }
        } else {
          const int pos = x0 + ch * EPC;
          const int rem = s.npos - pos;
          const int bytes = rem >= EPC ? 16 : (rem > 0 ? rem * (int)sizeof(T) : 0);
          const int sp = bytes ? pos : x0;
          for (int v = tid / CPL; v < nv; v += LPP) {
            const int dl = v < nl ? v : maxl + (v - nl);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sb + dl * kSTX * (int)sizeof(T)),
                         "l"(lp[v] + sp), "r"(bytes)
                         : "memory");
          }
        }
      } else {
        const int nel = (nl + R) * kSTX;
        for (int e = tid; e < nel; e += kSNT) {
          const int ln = e / kSTX, x = e - ln * kSTX;
          const int pos = x0 + x;
          const bool ok = pos < s.npos;
          if (ln < nl)
            cp_async_elem(stg + (size_t)ln * kSTX + x,
                          s.src + (int64_t)li[ln] * s.line_stride + (int64_t)(ok ? pos : 0) * s.pos_stride, ok);
          else
            cp_async_elem(bsg + (size_t)(ln - nl) * kSTX + x, s.Bold + (int64_t)(ln - nl) * s.ldb + (ok ? pos : 0),
                          ok);
        }
      }
    }
    cp_async_commit();
  };
  issue(0, 0);
  issue(1, 1);

  int cur_strip = -1;
  double den_acc0 = 0.0, res_acc0 = 0.0, den_acc1 = 0.0, res_acc1 = 0.0;
  const T zt = a.zt;
  const bool rec = a.dbg && blockIdx.x == 0 && tid == 0;
  long long tpc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tq = clock64();
#define SPH(k) do { if (rec) { const long long _t = clock64(); tpc[k] += _t - tq; tq = _t; } } while (0)
  for (int i = 0;; ++i) {
    int q, x0;
    if (!tile_of(i, q, x0)) break;
    const int st = i & 1;
    const StripDesc<T>& s = a.s[q];
    const int nl = nmy[q];
    T* stg = stage + (size_t)st * (maxl + R + 1) * kSTX;
    T* bsg = stg + (size_t)maxl * kSTX;
    const int* omt = reinterpret_cast<const int*>(stg + (size_t)(maxl + R) * kSTX);  // override map of the tile
    if (q != cur_strip) {
      // per-line vectors of this strip (my lines): A | W | Res, padded to RP
      for (int e = tid; e < nl * 3 * R; e += kSNT) {
        const int kl = e / (3 * R);
        const int rem = e - kl * 3 * R;
        const int vv = rem / R;
        const int t = rem - vv * R;
        const T* sv = vv == 0 ? s.lineA : (vv == 1 ? s.lineW : s.lineRes);
        lvec[(kl * 3 + vv) * RP + t] = sv[(int64_t)(kb[q] + kl) * R + t];
      }
      cur_strip = q;
      __syncthreads();
    }
    SPH(6);
    cp_async_wait1();  // this thread's copies of tile i have landed
    __syncthreads();   // ... and everybody else's
    SPH(0);

    // ---- pass 1: Phase I/II in place + factor partials
    const int mode = s.mode;  // uniform per tile (and per cluster)
    const bool accum = mode != kStripFinish;
    Pair<T> b[R];
#pragma unroll
    for (int t = 0; t < R; ++t) b[t] = lds_pair(bsg + t * kSTX + 2 * lane);
    Pair<T> acc[R];
#pragma unroll
    for (int t = 0; t < R; ++t) acc[t] = Pair<T>::splat(T(0));
    Pair<T> den = Pair<T>::splat(T(0));
    const int pe = 2 * lane;
    // lines in groups of kG with interleaved (independent) rank-r chains
    constexpr int kG = group_lines<T, R>();
    int kl = w;
    for (; kl + (kG - 1) * kSNW < nl; kl += kG * kSNW) {
      Pair<T> d[kG], l[kG], c[kG];
      const T* av[kG];
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        av[g] = lvec + ((kl + g * kSNW) * 3) * RP;
        d[g] = lds_pair(stg + (size_t)(kl + g * kSNW) * kSTX + pe);
      }
#pragma unroll
      for (int g = 0; g < kG; ++g) l[g] = pmul(Pair<T>::splat(av[g][0]), b[0]);
#pragma unroll
      for (int t = 1; t < R; ++t)
#pragma unroll
        for (int g = 0; g < kG; ++g) l[g] = pfma(Pair<T>::splat(av[g][t]), b[t], l[g]);
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        c[g] = keep_pair(d[g], l[g], zt);
        den = pfma(d[g], d[g], den);
        sts_pair(stg + (size_t)(kl + g * kSNW) * kSTX + pe, c[g]);
      }
      if (accum) {
#pragma unroll
        for (int t = 0; t < R; ++t)
#pragma unroll
          for (int g = 0; g < kG; ++g) acc[t] = pfma(Pair<T>::splat(av[g][RP + t]), c[g], acc[t]);
      }
    }
    for (; kl < nl; kl += kSNW) {
      T* cell = stg + (size_t)kl * kSTX + pe;
      const Pair<T> d = lds_pair(cell);
      const T* av = lvec + (kl * 3) * RP;
      Pair<T> l = pmul(Pair<T>::splat(av[0]), b[0]);
#pragma unroll
      for (int t = 1; t < R; ++t) l = pfma(Pair<T>::splat(av[t]), b[t], l);
      const Pair<T> c = keep_pair(d, l, zt);
      den = pfma(d, d, den);
      sts_pair(cell, c);
      if (accum) {
        const T* wv = av + RP;
#pragma unroll
        for (int t = 0; t < R; ++t) acc[t] = pfma(Pair<T>::splat(wv[t]), c, acc[t]);
      }
    }
    SPH(1);
    if (accum) {
      const double dsum = (double)den.v.x + (double)den.v.y;
      if (q == 0) den_acc0 += dsum; else den_acc1 += dsum;
#pragma unroll
      for (int t = 0; t < R; ++t) sts_pair(red + ((size_t)w * R + t) * kSTX + pe, acc[t]);
      __syncthreads();
      // Positions of the other index set take the factor computed from the
      // core (Q(:,J) = W^T U, P(I,:) = U V Sigma^+): one value for the I x J
      // block.  Applied where each output is produced (not in kStripPartial).
      const bool ovr = mode != kStripPartial;
      T* pbuf = part + (size_t)(i & 1) * R * kSTX;
      for (int o = tid; o < R * kSTX; o += kSNT) {
        T sum = red[o];
#pragma unroll
        for (int ww = 1; ww < kSNW; ++ww) sum += red[(size_t)ww * R * kSTX + o];
        if (CS > 1) {
          pbuf[o] = sum;
        } else {
          const int t = o / kSTX, x = o - t * kSTX;
          const int e = (ovr && x0 + x < s.npos) ? omt[x] : -1;
          fnew[o] = e >= 0 ? s.otherF[(int64_t)e * R + t] : sum;
        }
      }
      if (CS > 1) {
        cl.sync();
        for (int o = tid; o < R * kSTX; o += kSNT) {
          T sum = *cl.map_shared_rank(pbuf + o, 0);
          for (int qq = 1; qq < CS; ++qq) sum += *cl.map_shared_rank(pbuf + o, qq);
          const int t = o / kSTX, x = o - t * kSTX;
          const int e = (ovr && x0 + x < s.npos) ? omt[x] : -1;
          fnew[o] = e >= 0 ? s.otherF[(int64_t)e * R + t] : sum;
        }
      }
    } else {  // kStripFinish: the factor sums were all-reduced across the row shards
      for (int o = tid; o < R * kSTX; o += kSNT) {
        const int t = o / kSTX, x = o - t * kSTX;
        const int e = x0 + x < s.npos ? omt[x] : -1;
        fnew[o] = e >= 0 ? s.otherF[(int64_t)e * R + t]
                         : (x0 + x < s.npos ? s.Fsrc[(int64_t)t * s.ldfs + x0 + x] : T(0));
      }
    }
    __syncthreads();
    SPH(2);
    for (int o = tid; o < R * kSTX; o += kSNT) {
      const int t = o / kSTX, x = o - t * kSTX;
      if ((t % CS) == rank && x0 + x < s.npos) s.Fnew[(int64_t)t * s.ldf + x0 + x] = fnew[o];
    }
    if (mode == kStripPartial) {  // residual after the all-reduce (kStripFinish launch)
      __syncthreads();
      issue(i + 2, st);
      continue;
    }
    SPH(3);
    // ---- pass 2: stopping residual on the thresholded tile
    Pair<T> f[R];
#pragma unroll
    for (int t = 0; t < R; ++t) f[t] = lds_pair(fnew + t * kSTX + pe);
    Pair<T> res = Pair<T>::splat(T(0));
    kl = w;
    for (; kl + (kG - 1) * kSNW < nl; kl += kG * kSNW) {
      Pair<T> c[kG], l[kG];
      const T* rv[kG];
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        rv[g] = lvec + ((kl + g * kSNW) * 3 + 2) * RP;
        c[g] = lds_pair(stg + (size_t)(kl + g * kSNW) * kSTX + pe);
      }
#pragma unroll
      for (int g = 0; g < kG; ++g) l[g] = pmul(Pair<T>::splat(rv[g][0]), f[0]);
#pragma unroll
      for (int t = 1; t < R; ++t)
#pragma unroll
        for (int g = 0; g < kG; ++g) l[g] = pfma(Pair<T>::splat(rv[g][t]), f[t], l[g]);
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        const Pair<T> rr = psub(c[g], l[g]);
        res = pfma(rr, rr, res);
      }
    }
    for (; kl < nl; kl += kSNW) {
      const Pair<T> c = lds_pair(stg + (size_t)kl * kSTX + pe);
      const T* rv = lvec + (kl * 3 + 2) * RP;
      Pair<T> l = pmul(Pair<T>::splat(rv[0]), f[0]);
#pragma unroll
      for (int t = 1; t < R; ++t) l = pfma(Pair<T>::splat(rv[t]), f[t], l);
      const Pair<T> rr = psub(c, l);
      res = pfma(rr, rr, res);
    }
    const double rsum = (double)res.v.x + (double)res.v.y;
    if (q == 0) res_acc0 += rsum; else res_acc1 += rsum;
    SPH(4);
    __syncthreads();  // stage st, fnew, red are free again
    issue(i + 2, st);
    SPH(5);
  }
  if (rec)
    for (int k = 0; k < 8; ++k) a.dbg[k] += tpc[k];
#undef SPH
  cp_async_wait0();
  const double d0 = block_sum<kSNT>(den_acc0, dred);
  const double r0 = block_sum<kSNT>(res_acc0, dred + kSNW);
  const double d1 = block_sum<kSNT>(den_acc1, dred + 2 * kSNW);
  const double r1 = block_sum<kSNT>(res_acc1, dred + 3 * kSNW);
  if (tid == 0) {
    double4 p;
    p.x = d0; p.y = r0; p.z = d1; p.w = r1;
    *reinterpret_cast<double4*>(a.partials + 4 * blockIdx.x) = p;
  }
  if (CS > 1) cl.sync();  // peers may still read this CTA's `part`
}

// ------------------------------------------------------------------ launch
template <typename T>
size_t strips_smem_bytes(int maxl, int R) {
  return strips_layout(maxl, R, (int)sizeof(T)).total;
}

// smallest cluster size whose per-CTA line share fits in shared memory
template <typename T>
int strips_pick_cluster(int nk_max, int R) {
  for (int cs = 1; cs <= 16; ++cs) {
    const int maxl = (nk_max + cs - 1) / cs;
    if (strips_smem_bytes<T>(maxl, R) <= (size_t)227 * 1024) return cs;
  }
  return -1;
}

template <typename T, int R>
static cudaError_t launch_strips_r(const StripsArgs<T>& a, int cs, int num_sms, cudaStream_t st) {
  const size_t smem = strips_smem_bytes<T>(a.maxl, R);
  static std::atomic<unsigned long long> devs{0};  // per device (several host threads may launch)
  const cudaError_t fattr = smem_attr_once(devs, strips_kernel<T, R>, 227 * 1024, true);
  if (fattr != cudaSuccess) return fattr;
  const int tiles = a.s[0].tiles + a.s[1].tiles;
  const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(2, (size_t)(227 * 1024) / (smem + 1024)));
  int ncl = std::max(1, std::min(tiles, num_sms * per_sm / cs));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ncl * cs), 1, 1);
  cfg.blockDim = dim3(kSNT, 1, 1);
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

// read per launch (cheap), so tests can switch kernels within one process
static int strips_version() {
  const char* e = std::getenv("IRCUR_STRIPS_VER");
  if (!e) e = std::getenv("IRCUR_STRIPS_V1") ? "1" : nullptr;
  return e ? std::atoi(e) : 3;
}

std::atomic<int> g_last_strips_kernel{0};  // diagnostics: 1, 2, 3 or 5 (ircur_debug_counter 2)

bool strips6_selected(const StripsArgs<float>& a, int R) {
  return strips_version() >= 6 && strips6_supported(a, R);
}

bool strips5_selected(const StripsArgs<float>& a, int R) {
  return strips_version() == 5 && strips5_supported(a, R);
}

bool strips3_selected(const StripsArgs<float>& a, int R) {
  const bool aligned = (a.s[0].tiles == 0 || a.s[0].bulk_ok) && (a.s[1].tiles == 0 || a.s[1].bulk_ok);
  const int maxl = a.s[0].nk > a.s[1].nk ? a.s[0].nk : a.s[1].nk;
  return strips_version() >= 3 && !strips_tc_selected(a, R) && aligned &&
         strips3_smem_bytes(maxl, R) <= (size_t)227 * 1024;
}

template <typename T>
cudaError_t launch_strips(const StripsArgs<T>& a, int R, int cs, int num_sms, int* ncta_out,
                          cudaStream_t st) {
  const int tiles = a.s[0].tiles + a.s[1].tiles;
  if (ncta_out) *ncta_out = 0;
  if (tiles == 0) return cudaSuccess;
  if constexpr (sizeof(T) == 4) {
    // fp32: the 64-position single-stage kernel, else the two-group
    // 32-position kernel, else this cluster kernel.  IRCUR_STRIPS_VER=5 adds
    // the tensor-core kernel in front (measured no faster at cfg5 and slower
    // on the small configs, so it is opt-in); 1|2 cap the choice (A/B).
    const int ver = strips_version();
    const bool aligned = (a.s[0].tiles == 0 || a.s[0].bulk_ok) && (a.s[1].tiles == 0 || a.s[1].bulk_ok);
    if (ver >= 6) {
      const cudaError_t e = launch_strips6(a, R, num_sms, ncta_out, st);
      if (e != cudaErrorNotSupported) {
        g_last_strips_kernel = 6;
        return e;
      }
    }
    if (ver == 5) {
      const cudaError_t e = launch_strips5(a, R, num_sms, ncta_out, st);
      if (e != cudaErrorNotSupported) {
        g_last_strips_kernel = 5;
        return e;
      }
    }
    if (ver >= 3 && aligned) {
      const cudaError_t e = launch_strips3(a, R, num_sms, ncta_out, st);
      if (e != cudaErrorNotSupported) {
        g_last_strips_kernel = 3;
        return e;
      }
    }
    if (ver >= 2 && aligned) {
      const cudaError_t e = launch_strips2(a, R, num_sms, ncta_out, st);
      if (e != cudaErrorNotSupported) {
        g_last_strips_kernel = 2;
        return e;
      }
    }
  }
  cudaError_t e = cudaErrorInvalidValue;
  g_last_strips_kernel = 1;
  IRCUR_DISPATCH_RANK(R, RR, e = launch_strips_r<T, RR>(a, cs, num_sms, st));
  if (ncta_out) {
    const size_t smem = strips_smem_bytes<T>(a.maxl, R);
    const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(2, (size_t)(227 * 1024) / (smem + 1024)));
    *ncta_out = std::max(1, std::min(tiles, num_sms * per_sm / cs)) * cs;
  }
  return e;
}

int strips_tx() { return kSTX; }

template size_t strips_smem_bytes<float>(int, int);
template size_t strips_smem_bytes<double>(int, int);
template int strips_pick_cluster<float>(int, int);
template int strips_pick_cluster<double>(int, int);
template cudaError_t launch_strips<float>(const StripsArgs<float>&, int, int, int, int*, cudaStream_t);
template cudaError_t launch_strips<double>(const StripsArgs<double>&, int, int, int, int*, cudaStream_t);

}  // namespace ircur
