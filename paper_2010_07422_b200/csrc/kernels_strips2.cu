// Fused row + column strip kernel, fp32 variant for sm_100a (see
// kernels_strips.cu for the per-entry semantics: Phase I/II, factor sums,
// overrides, stopping residual; solver.py:375-400).
//
// Layout: one persistent 512-thread CTA per SM made of TWO independent
// groups of 8 warps.  Each group owns a single-buffered shared stage
// holding every sampled line of a 32-position tile (no cluster split), and
// walks its own tiles with its own named barriers, so while one group is
// in a barrier/reduction phase the other keeps the FMA pipe busy.  Within a
// group, lane = position and each warp takes PAIRS of lines, packed into
// the two halves of FFMA2 (the per-pair line vectors A | W | Res are
// interleaved in shared memory, shared by both groups).  The per-tile
// factor sums are reduced over the 8 warps of the group in a fixed order.
#include <cuda_runtime.h>

#include "kernels_iter.cuh"
#include "launchers.cuh"

namespace ircur {

constexpr int kS2Groups = 2;
constexpr int kS2GW = 8;                  // warps per group
constexpr int kS2GT = kS2GW * 32;         // threads per group
constexpr int kS2NT = kS2Groups * kS2GT;  // threads per CTA
constexpr int kS2TX = 32;                 // positions per tile (one per lane)

struct Strips2Layout {
  int RP, maxp;
  size_t lvec, stage, bst, omt, lptr, red, fnew, dred, total;
};

__host__ __device__ inline size_t al128(size_t x) { return (x + 127) & ~size_t(127); }

// maxl: most lines of either strip (every line of a tile is resident)
__host__ __device__ inline Strips2Layout strips2_layout(int maxl, int R) {
  Strips2Layout L;
  L.RP = R + (R & 1);        // even: the float2 pairs of t, t+1 load as 16 bytes
  L.maxp = (maxl + 1) / 2;   // line pairs
  size_t off = 0;
  L.lvec = off; off = al128(off + (size_t)L.maxp * 3 * L.RP * sizeof(float2));
  L.stage = off; off = al128(off + (size_t)kS2Groups * 2 * L.maxp * kS2TX * sizeof(float));
  L.bst = off; off = al128(off + (size_t)kS2Groups * R * kS2TX * sizeof(float));
  L.omt = off; off = al128(off + (size_t)kS2Groups * kS2TX * sizeof(int));
  L.lptr = off; off = al128(off + (size_t)2 * (2 * L.maxp + R) * sizeof(void*));
  L.red = off; off = al128(off + (size_t)kS2Groups * kS2GW * R * kS2TX * sizeof(float));
  L.fnew = off; off = al128(off + (size_t)kS2Groups * R * kS2TX * sizeof(float));
  L.dred = off; off = al128(off + 4 * (kS2NT / 32) * sizeof(double));
  L.total = off;
  return L;
}

__device__ __forceinline__ void group_sync(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "n"(kS2GT) : "memory");
}
__device__ __forceinline__ uint32_t s2_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int R>
__global__ void __launch_bounds__(kS2NT, 1) strips2_kernel(const __grid_constant__ StripsArgs<float> a) {
  if (*a.done) return;
  const Strips2Layout L = strips2_layout(a.maxl, R);
  constexpr int RPc = R + (R & 1);
  extern __shared__ __align__(128) unsigned char sm[];
  float2* lvec = reinterpret_cast<float2*>(sm + L.lvec);
  const float** lptr = reinterpret_cast<const float**>(sm + L.lptr);
  double* dred = reinterpret_cast<double*>(sm + L.dred);
  const int tid = threadIdx.x, g = tid / kS2GT, gt = tid % kS2GT, lane = tid & 31, wg = gt >> 5;
  float* stage = reinterpret_cast<float*>(sm + L.stage) + (size_t)g * 2 * L.maxp * kS2TX;
  float* bst = reinterpret_cast<float*>(sm + L.bst) + (size_t)g * R * kS2TX;
  int* omt = reinterpret_cast<int*>(sm + L.omt) + (size_t)g * kS2TX;
  float* red = reinterpret_cast<float*>(sm + L.red) + (size_t)g * kS2GW * R * kS2TX;
  float* fnew = reinterpret_cast<float*>(sm + L.fnew) + (size_t)g * R * kS2TX;
  const float zt = a.zt;

#pragma unroll
  for (int q = 0; q < 2; ++q) {  // segment sources: lines, then the R rows of the old factor
    const StripDesc<float>& s = a.s[q];
    float const** lp = lptr + q * (2 * L.maxp + R);
    for (int e = tid; e < s.nk + R; e += kS2NT)
      lp[e] = e < s.nk ? s.src + (int64_t)(s.lines[e] - s.line_off) * s.line_stride : s.Bold + (int64_t)(e - s.nk) * s.ldb;
  }
  double den_acc[2] = {0.0, 0.0}, res_acc[2] = {0.0, 0.0};
  const int tiles0 = a.s[0].tiles;
  const bool rec = a.dbg && blockIdx.x == 0 && tid == 0;
  long long tpc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tq = clock64();
#define SPH(k) do { if (rec) { const long long _t = clock64(); tpc[k] += _t - tq; tq = _t; } } while (0)
  for (int q = 0; q < 2; ++q) {
    const StripDesc<float>& s = a.s[q];
    const int nl = s.nk, np = (nl + 1) / 2, nl2 = 2 * np;
    const int mode = s.mode;
    // per-pair line vectors of this strip: (A | W | Res)[t] for lines 2kp, 2kp+1
    __syncthreads();  // the other group may still read the previous strip's vectors
    for (int e = tid; e < np * 3 * RPc; e += kS2NT) {
      const int kp = e / (3 * RPc), rem = e - kp * 3 * RPc, v = rem / RPc, t = rem - v * RPc;
      const float* sv = v == 0 ? s.lineA : (v == 1 ? s.lineW : s.lineRes);
      const int k0 = 2 * kp, k1 = k0 + 1;
      float2 val = make_float2(0.f, 0.f);
      if (t < R) {
        val.x = sv[(int64_t)k0 * R + t];
        if (k1 < nl) val.y = sv[(int64_t)k1 * R + t];
      }
      lvec[e] = val;
    }
    __syncthreads();
    if (s.tiles == 0) continue;
    // this CTA's tiles of strip q, alternating between the two groups
    const int t_lo = q == 0 ? 0 : tiles0, t_hi = t_lo + s.tiles;
    int i0 = (t_lo - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    if ((int)blockIdx.x >= t_lo) i0 = 0;
    const float* const* lp = lptr + q * (2 * L.maxp + R);
    for (int i = i0 + g;; i += kS2Groups) {
      const int t = (int)blockIdx.x + i * (int)gridDim.x;
      if (t >= t_hi) break;
      const int x0 = (t - t_lo) * kS2TX;
      SPH(6);
      // ---- stage the tile: 8 x 16-byte chunks per 128-byte line segment
      {
        const int ch = gt & 7;
        const int pos = x0 + ch * 4;
        const int rem = s.npos - pos;
        const int bytes = rem >= 4 ? 16 : (rem > 0 ? rem * 4 : 0);
        const int sp = bytes ? pos : x0;
        for (int v = gt >> 3; v < nl2 + R; v += kS2GT / 8) {
          float* dst = v < nl2 ? stage + (size_t)v * kS2TX : bst + (size_t)(v - nl2) * kS2TX;
          const float* src = v < nl ? lp[v] : (v < nl2 ? lp[0] : lp[nl + (v - nl2)]);
          const int b = v < nl || v >= nl2 ? bytes : 0;  // the padding line of an odd count reads zeros
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s2_smem(dst + ch * 4)),
                       "l"(src + sp), "r"(b)
                       : "memory");
        }
        if (gt < 8) {
          const int ob = rem >= 4 ? 16 : (rem > 0 ? rem * 4 : 0);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s2_smem(omt + ch * 4)),
                       "l"(s.omap + (ob ? pos : x0)), "r"(ob)
                       : "memory");
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
      }
      group_sync(g);
      SPH(0);
      float b[R];
#pragma unroll
      for (int tt = 0; tt < R; ++tt) b[tt] = bst[tt * kS2TX + lane];
      // ---- pass 1: Phase I/II in place (pairs of lines per FFMA2) + factor partials
      Pair<float> acc[R];
#pragma unroll
      for (int tt = 0; tt < R; ++tt) acc[tt] = Pair<float>::splat(0.f);
      Pair<float> den = Pair<float>::splat(0.f);
      const bool accum = mode != kStripFinish;
      // two line pairs per step (independent FFMA2 chains), then a tail pair
      int kp = wg;
      for (; kp + kS2GW < np; kp += 2 * kS2GW) {
        const float2* va0 = lvec + (size_t)kp * 3 * RPc;
        const float2* va1 = lvec + (size_t)(kp + kS2GW) * 3 * RPc;
        float* c00 = stage + (size_t)(2 * kp) * kS2TX + lane;
        float* c10 = stage + (size_t)(2 * (kp + kS2GW)) * kS2TX + lane;
        Pair<float> d0, d1, l0, l1;
        d0.v = make_float2(c00[0], c00[kS2TX]);
        d1.v = make_float2(c10[0], c10[kS2TX]);
        l0.v = __fmul2_rn(va0[0], make_float2(b[0], b[0]));
        l1.v = __fmul2_rn(va1[0], make_float2(b[0], b[0]));
#pragma unroll
        for (int tt = 1; tt < R; ++tt) {
          l0.v = __ffma2_rn(va0[tt], make_float2(b[tt], b[tt]), l0.v);
          l1.v = __ffma2_rn(va1[tt], make_float2(b[tt], b[tt]), l1.v);
        }
        const Pair<float> c0 = keep_pair(d0, l0, zt);
        const Pair<float> c1 = keep_pair(d1, l1, zt);
        den = pfma(d0, d0, den);
        den = pfma(d1, d1, den);
        c00[0] = c0.v.x;
        c00[kS2TX] = c0.v.y;
        c10[0] = c1.v.x;
        c10[kS2TX] = c1.v.y;
        if (accum) {
          const float2* vw0 = va0 + RPc;
          const float2* vw1 = va1 + RPc;
#pragma unroll
          for (int tt = 0; tt < R; ++tt) {
            acc[tt].v = __ffma2_rn(vw0[tt], c0.v, acc[tt].v);
            acc[tt].v = __ffma2_rn(vw1[tt], c1.v, acc[tt].v);
          }
        }
      }
      if (kp < np) {
        const float2* va = lvec + (size_t)kp * 3 * RPc;
        float* c0 = stage + (size_t)(2 * kp) * kS2TX + lane;
        Pair<float> d;
        d.v = make_float2(c0[0], c0[kS2TX]);
        Pair<float> l;
        l.v = __fmul2_rn(va[0], make_float2(b[0], b[0]));
#pragma unroll
        for (int tt = 1; tt < R; ++tt) l.v = __ffma2_rn(va[tt], make_float2(b[tt], b[tt]), l.v);
        const Pair<float> c = keep_pair(d, l, zt);
        den = pfma(d, d, den);
        c0[0] = c.v.x;
        c0[kS2TX] = c.v.y;
        if (accum) {
          const float2* vw = va + RPc;
#pragma unroll
          for (int tt = 0; tt < R; ++tt) acc[tt].v = __ffma2_rn(vw[tt], c.v, acc[tt].v);
        }
      }
      SPH(1);
      if (accum) {
        den_acc[q] += (double)den.v.x + (double)den.v.y;
#pragma unroll
        for (int tt = 0; tt < R; ++tt) red[(wg * R + tt) * kS2TX + lane] = acc[tt].v.x + acc[tt].v.y;
      }
      group_sync(g);
      SPH(2);
      // ---- factor sums over the group's warps (fixed order) + overrides
      const bool ovr = mode != kStripPartial;
      for (int o = gt; o < R * kS2TX; o += kS2GT) {
        const int tt = o / kS2TX, x = o - tt * kS2TX;
        const int e = (ovr && x0 + x < s.npos) ? omt[x] : -1;
        float v;
        if (e >= 0) {
          v = s.otherF[(int64_t)e * R + tt];
        } else if (accum) {
          v = red[tt * kS2TX + x];
#pragma unroll
          for (int w = 1; w < kS2GW; ++w) v += red[(w * R + tt) * kS2TX + x];
        } else {
          v = x0 + x < s.npos ? s.Fsrc[(int64_t)tt * s.ldfs + x0 + x] : 0.f;
        }
        fnew[o] = v;
        if (x0 + x < s.npos) s.Fnew[(int64_t)tt * s.ldf + x0 + x] = v;
      }
      group_sync(g);
      SPH(3);
      if (mode != kStripPartial) {
        // ---- pass 2: stopping residual on the thresholded tile
        float f[R];
#pragma unroll
        for (int tt = 0; tt < R; ++tt) f[tt] = fnew[tt * kS2TX + lane];
        Pair<float> res = Pair<float>::splat(0.f);
        int kq = wg;
        for (; kq + kS2GW < np; kq += 2 * kS2GW) {
          const float2* vr0 = lvec + (size_t)kq * 3 * RPc + 2 * RPc;
          const float2* vr1 = lvec + (size_t)(kq + kS2GW) * 3 * RPc + 2 * RPc;
          const float* c00 = stage + (size_t)(2 * kq) * kS2TX + lane;
          const float* c10 = stage + (size_t)(2 * (kq + kS2GW)) * kS2TX + lane;
          Pair<float> c0, c1, l0, l1;
          c0.v = make_float2(c00[0], c00[kS2TX]);
          c1.v = make_float2(c10[0], c10[kS2TX]);
          l0.v = __fmul2_rn(vr0[0], make_float2(f[0], f[0]));
          l1.v = __fmul2_rn(vr1[0], make_float2(f[0], f[0]));
#pragma unroll
          for (int tt = 1; tt < R; ++tt) {
            l0.v = __ffma2_rn(vr0[tt], make_float2(f[tt], f[tt]), l0.v);
            l1.v = __ffma2_rn(vr1[tt], make_float2(f[tt], f[tt]), l1.v);
          }
          const Pair<float> r0 = psub(c0, l0);
          const Pair<float> r1 = psub(c1, l1);
          res = pfma(r0, r0, res);
          res = pfma(r1, r1, res);
        }
        if (kq < np) {
          const float2* vr = lvec + (size_t)kq * 3 * RPc + 2 * RPc;
          const float* c0 = stage + (size_t)(2 * kq) * kS2TX + lane;
          Pair<float> c;
          c.v = make_float2(c0[0], c0[kS2TX]);
          Pair<float> l;
          l.v = __fmul2_rn(vr[0], make_float2(f[0], f[0]));
#pragma unroll
          for (int tt = 1; tt < R; ++tt) l.v = __ffma2_rn(vr[tt], make_float2(f[tt], f[tt]), l.v);
          const Pair<float> rr = psub(c, l);
          res = pfma(rr, rr, res);
        }
        res_acc[q] += (double)res.v.x + (double)res.v.y;
      }
      SPH(4);
      group_sync(g);  // stage, fnew, red free for the group's next tile
      SPH(5);
    }
  }
  if (rec)
    for (int k = 0; k < 8; ++k) a.dbg[k] += tpc[k];
#undef SPH
  __syncthreads();
  const double d0 = block_sum<kS2NT>(den_acc[0], dred);
  const double r0 = block_sum<kS2NT>(res_acc[0], dred + kS2NT / 32);
  const double d1 = block_sum<kS2NT>(den_acc[1], dred + 2 * (kS2NT / 32));
  const double r1 = block_sum<kS2NT>(res_acc[1], dred + 3 * (kS2NT / 32));
  if (tid == 0) {
    double4 p;
    p.x = d0; p.y = r0; p.z = d1; p.w = r1;
    *reinterpret_cast<double4*>(a.partials + 4 * blockIdx.x) = p;
  }
}

size_t strips2_smem_bytes(int maxl, int R) { return strips2_layout(maxl, R).total; }

// fp32 only; maxl = most lines of either strip.  Returns cudaErrorNotSupported
// when the lines do not fit (the caller then uses the cluster kernel).
cudaError_t launch_strips2(const StripsArgs<float>& a0, int R, int num_sms, int* ncta_out, cudaStream_t st) {
  StripsArgs<float> a = a0;
  a.maxl = a.s[0].nk > a.s[1].nk ? a.s[0].nk : a.s[1].nk;
  for (int q = 0; q < 2; ++q)  // the caller counts tiles of the 64-position kernel
    if (a.s[q].tiles > 0) a.s[q].tiles = (a.s[q].npos + kS2TX - 1) / kS2TX;
  const size_t smem = strips2_smem_bytes(a.maxl, R);
  if (smem > (size_t)227 * 1024) return cudaErrorNotSupported;
  if (ncta_out) *ncta_out = 0;
  const int tiles = a.s[0].tiles + a.s[1].tiles;
  if (tiles == 0) return cudaSuccess;
  cudaError_t e = cudaErrorInvalidValue;
  IRCUR_DISPATCH_RANK(R, RR, {
    static std::atomic<unsigned long long> devs{0};  // once per device
    const cudaError_t attr = smem_attr_once(devs, strips2_kernel<RR>, 227 * 1024);
    if (attr != cudaSuccess) return attr;
    strips2_kernel<RR><<<num_sms, kS2NT, smem, st>>>(a);
    e = cudaGetLastError();
  });
  if (ncta_out) *ncta_out = num_sms;
  return e;
}

}  // namespace ircur
