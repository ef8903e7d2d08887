// Hybrid FFMA / warp-level tensor-core strip kernel (fp32 data, sm_100a).
//
// Same per-entry semantics as kernels_strips3.cu (Phase I/II, the new factor
// with the core overrides, the stopping residual; solver.py:375-400).  The
// work of one 8-line block of a 32-position tile is split over two pipes:
//
//   l = <P(line,:), Q(:,pos)>   FFMA2 chains (mul, then fma in t order: the
//                               core kernel's chain, bit for bit)
//   c = d - T_zeta(d - l)       Phase I/II in registers
//   F[pos, t] += c . W'         MMA2 on the tensor cores (mma.sync tf32, K = 8 lines)
//   r = c - F'.Res'^T           MMA3 on the tensor cores (K = 32), onto c
//
// fp32 accuracy from tf32 operands by a 3-term split, x = x_hi + x_lo with
// x_hi = x & 0xffffe000 (exact), a.b ~ a_hi b_hi + a_lo b_hi + a_hi b_lo.  For
// MMA3 the three terms of each t are laid along K (<= 30 of 32 slots); for
// MMA2 the split is laid along N: c_hi x [W_hi | W_lo | t8/t9] and
// c_lo x [W_hi | t8/t9] (5 n-tiles).
//
// Fragment bookkeeping (m16n8k8, g = lane / 4, c = lane % 4).  A warp owns
// 8-line blocks, both 16-position m-tiles of the tile.  Row g of m-tile mt is
// position 4g + 2mt, row g + 8 is 4g + 2mt + 1, so a lane's four positions are
// contiguous (one 16-byte shared load per line) and pair up for FFMA2.  A lane
// evaluates lines 8b + 2c and 8b + 2c + 1 at its four positions -- exactly its
// part of MMA2's A fragment once K index c is read as line 8b + 2c and c + 4
// as line 8b + 2c + 1 (W' rows permuted to match) -- and MMA3's accumulator
// (column n = line 8b + n) holds the same entries.  So the thresholded
// entries go from Phase I/II into MMA2 and, via the stage, back into MMA3's
// accumulator without any shuffle.
//
// Per tile: pass 1 (l, Phase I/II, c written back over d in the stage, MMA2
// partials), a fixed-order reduction of the warps' partials with the override
// of the other index set, then pass 2 (MMA3 accumulated onto c, the squared
// residual).  D tiles are double-buffered with cp.async: tile i + 1 loads
// while tile i is computed.  The I x J entries of c are taken from the core U
// (the strips' factors are the tensor cores' sums, which the sampled-factor
// kernel of the overlapped loop does not reproduce bit for bit; patched into
// the stage before pass 2, as pass 1's factor sums at those positions are
// replaced by the override), so on the intersection the strips hold the core's values, as _sync_intersection makes
// them in the reference (solver.py:216-221).  den and the residual are reduced
// per tile, so e_k does not depend on the grid size.
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels_iter.cuh"
#include "launchers.cuh"
#include "umma.cuh"

namespace ircur {

namespace s6 {
constexpr int TP = 32;         // positions per tile
constexpr int RMAX = 10;       // 3 r <= 32 K slots
constexpr int LMAX = 512;      // lines per strip

constexpr int PS = 12;         // floats per line of P and Res (t 0..9, 2 zeros)
constexpr int WS = 20;         // floats per line of W: (hi, lo) of t 0..7, then hi8 lo8 hi9 lo9

struct Layout {
  int nl8;
  size_t stage, stage_bytes, bq, om, pv, rv, wv, lidx, red, fsm, a3, dred, bars, total;
};
__host__ __device__ inline size_t al(size_t x) { return (x + 127) & ~size_t(127); }
template <int NW>
__host__ __device__ inline Layout layout(int maxl) {
  Layout L;
  L.nl8 = (maxl + 7) & ~7;
  size_t off = 0;
  // per stage: D [nl8][32] (16-byte chunks swizzled), Q rows [RMAX][32], omap [32]
  L.bq = (size_t)L.nl8 * TP * 4;
  L.om = L.bq + (size_t)RMAX * TP * 4;
  L.stage_bytes = al(L.om + TP * 4);
  L.stage = off; off += 2 * L.stage_bytes;
  L.pv = off; off = al(off + (size_t)L.nl8 * PS * 4);
  L.rv = off; off = al(off + (size_t)L.nl8 * PS * 4);
  L.wv = off; off = al(off + (size_t)L.nl8 * WS * 4);
  L.lidx = off; off = al(off + (size_t)2 * L.nl8 * 4);
  L.red = off; off = al(off + (size_t)NW * RMAX * TP * 4);
  L.fsm = off; off = al(off + (size_t)RMAX * TP * 4);
  L.a3 = off; off = al(off + (size_t)32 * 32 * 4);
  L.dred = off; off = al(off + (size_t)2 * NW * 2 * 8);
  L.bars = off; off = al(off + 4 * 8);
  L.total = off;
  return L;
}
}  // namespace s6

__device__ __forceinline__ float s6_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
__device__ __forceinline__ float s6_lo(float x) { return __fsub_rn(x, s6_hi(x)); }
__device__ __forceinline__ uint32_t s6_u(float x) { return __float_as_uint(x); }
// the same tf32 value in a different register: the tensor core reads only the
// top 19 bits of an fp32 container, so setting bit 0 leaves the operand
// unchanged, but the compiler cannot merge the two copies (which would cost a
// register move to rebuild each HMMA operand group)
__device__ __forceinline__ uint32_t s6_twin(uint32_t x) { return x | 1u; }

__device__ __forceinline__ void s6_mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void s6_cp16(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes)
               : "memory");
}

// The K-slot table of the K = r products (MMA1: A = Q at positions, B = P of
// lines; MMA3: A = F, B = Res).  Lane c owns K slots j = 2s + h (k-step s, half
// h: K index c + 4h + 8s).  Slots 0-2 carry t = 2c, 3-5 t = 2c + 1 as the terms
// (hi.hi, lo.hi, hi.lo); slots 6 and 7 share t = 8, 9 among lanes c = 0..2
// (c = 3: zero).  Each lane reads 4 values per operand: t = 2c, 2c + 1, t6, t7.
struct S6Slots {
  int t6, t7;
  bool z67;               // c == 3: slots 6, 7 are zero
  bool a6lo, a7lo, b6lo, b7lo;
  int r6, r7;             // columns of slots 6, 7 in a zero-padded line record (PS floats; 11 is zero)
  uint32_t m6, m7;        // ~0 where the B piece of slot 6 / 7 is the lo part
};
__device__ __forceinline__ S6Slots s6_slots(int c) {
  S6Slots s;
  s.t6 = c == 2 ? 9 : 8;
  s.t7 = c == 0 ? 8 : 9;
  s.z67 = c == 3;
  s.a6lo = c == 2; s.a7lo = c == 0;
  s.b6lo = c == 1; s.b7lo = c == 2;
  s.r6 = s.z67 ? 11 : s.t6;
  s.r7 = s.z67 ? 11 : s.t7;
  s.m6 = s.b6lo ? 0xffffffffu : 0u;
  s.m7 = s.b7lo ? 0xffffffffu : 0u;
  return s;
}
// the 8 slot values of the A side (positions) from its 4 source values
__device__ __forceinline__ void s6_aslots(const S6Slots& S, float va, float vb, float v6, float v7, float neg,
                                          float (&o)[8]) {
  o[0] = neg * s6_hi(va); o[1] = neg * s6_lo(va); o[2] = __uint_as_float(s6_twin(s6_u(o[0])));
  o[3] = neg * s6_hi(vb); o[4] = neg * s6_lo(vb); o[5] = __uint_as_float(s6_twin(s6_u(o[3])));
  o[6] = S.z67 ? 0.f : neg * (S.a6lo ? s6_lo(v6) : s6_hi(v6));
  o[7] = S.z67 ? 0.f : neg * (S.a7lo ? s6_lo(v7) : s6_hi(v7));
}
// B side from a line record rl (PS floats, zero beyond R): branch-free (the
// lane's slot-6/7 columns and pieces are per-lane constants, applied by masks)
__device__ __forceinline__ void s6_bslots(const S6Slots& S, const float* rl, int c, uint32_t (&o)[8]) {
  const float2 vab = *reinterpret_cast<const float2*>(rl + 2 * c);
  const float v6 = rl[S.r6], v7 = rl[S.r7];
  const float ha = s6_hi(vab.x), hb = s6_hi(vab.y), h6 = s6_hi(v6), h7 = s6_hi(v7);
  o[0] = s6_u(ha); o[1] = s6_twin(o[0]); o[2] = s6_u(__fsub_rn(vab.x, ha));
  o[3] = s6_u(hb); o[4] = s6_twin(o[3]); o[5] = s6_u(__fsub_rn(vab.y, hb));
  const uint32_t l6 = s6_u(__fsub_rn(v6, h6)), l7 = s6_u(__fsub_rn(v7, h7));
  o[6] = (l6 & S.m6) | (s6_u(h6) & ~S.m6);
  o[7] = (l7 & S.m7) | (s6_u(h7) & ~S.m7);
}

// NW = 8 (or 12) compute warps (whole warpgroups) plus one producer warpgroup that
// issues every tile's copies: a warp issuing cp.async blocks until the SM's
// copy queue drains (measured: ~20% of the compute warps' time when they
// issued the next tile's copies themselves), so only the producers wait on
// it.  One warp alone issues too slowly (1.0 TB/s for these 128-byte
// segments, tools/micro/strip_fill.cu; 128 threads: 3.3 TB/s)..
template <int NW, int R>
__global__ void __launch_bounds__((NW + 4) * 32, 1) strips6_kernel(const __grid_constant__ StripsArgs<float> a) {
  using namespace s6;
  static_assert(NW % 4 == 0, "compute warps: whole warpgroups");
  constexpr int NT = NW * 32;        // compute threads
  constexpr int NTA = NT + 128;      // + the producer warpgroup
  if (*a.done) return;
  const int maxl = a.s[0].nk > a.s[1].nk ? a.s[0].nk : a.s[1].nk;
  const Layout Ly = layout<NW>(maxl);
  const int nl8 = Ly.nl8;
  extern __shared__ __align__(128) unsigned char sm[];
  float* Pv = reinterpret_cast<float*>(sm + Ly.pv);
  float* Rv = reinterpret_cast<float*>(sm + Ly.rv);
  float* Wv = reinterpret_cast<float*>(sm + Ly.wv);
  int* lidx = reinterpret_cast<int*>(sm + Ly.lidx);
  float* red = reinterpret_cast<float*>(sm + Ly.red);
  float* fsm = reinterpret_cast<float*>(sm + Ly.fsm);
  double* dred = reinterpret_cast<double*>(sm + Ly.dred);
  float4* a3s = reinterpret_cast<float4*>(sm + Ly.a3);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + Ly.bars);  // [2]: tile landed in stage b
  uint64_t* empty = full + 2;                                    // [2]: stage b consumed
  auto stageD = [&](int b) { return reinterpret_cast<float*>(sm + Ly.stage + (size_t)b * Ly.stage_bytes); };
  auto stageQ = [&](int b) { return reinterpret_cast<float*>(sm + Ly.stage + (size_t)b * Ly.stage_bytes + Ly.bq); };
  auto stageO = [&](int b) { return reinterpret_cast<int*>(sm + Ly.stage + (size_t)b * Ly.stage_bytes + Ly.om); };

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, c = lane & 3;
  const S6Slots S = s6_slots(c);
  const int tiles0 = a.s[0].tiles, total = tiles0 + a.s[1].tiles;
  const int bx = (int)blockIdx.x, nbx = (int)gridDim.x;
  const int ntl = bx < total ? (total - 1 - bx) / nbx + 1 : 0;
  auto tile_of = [&](int i) { return bx + i * nbx; };

  // line ids of both strips (relative to line_off); zero Q rows >= R of both stages, fsm
  for (int e = tid; e < 2 * nl8; e += NTA) {
    const int q = e >= nl8, L = e - q * nl8;
    const StripDesc<float>& s = a.s[q];
    lidx[e] = (s.tiles > 0 && L < s.nk) ? s.lines[L] - s.line_off : 0;
  }
  for (int e = tid; e < 2 * RMAX * TP; e += NTA) {
    const int b = e / (RMAX * TP), o = e - b * RMAX * TP;
    if (o >= R * TP) stageQ(b)[o] = 0.f;
  }
  for (int e = tid; e < RMAX * TP; e += NTA) fsm[e] = 0.f;
  if (tid == 0) {
    umma::bar_init(&full[0], 128);
    umma::bar_init(&full[1], 128);
    umma::bar_init(&empty[0], NW);
    umma::bar_init(&empty[1], NW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // the line vectors of strip q (zero beyond nk and t >= R)
  auto load_strip = [&](int q) {
    const StripDesc<float>& s = a.s[q];
    for (int e = tid; e < nl8 * PS; e += NT) {
      const int L = e / PS, t = e - L * PS;
      const bool ok = L < s.nk && t < R;
      Pv[e] = ok ? s.lineA[(int64_t)L * R + t] : 0.f;
      Rv[e] = ok ? s.lineRes[(int64_t)L * R + t] : 0.f;
    }
    for (int e = tid; e < nl8 * WS; e += NT) {  // W' pieces: (hi, lo) of t 0..7, then hi8 lo8 hi9 lo9
      const int L = e / WS, k = e - L * WS;
      const int t = k < 16 ? k >> 1 : 8 + ((k - 16) >> 1);
      const bool lo = k & 1;
      const float x = (L < s.nk && t < R) ? s.lineW[(int64_t)L * R + t] : 0.f;
      Wv[e] = lo ? s6_lo(x) : s6_hi(x);
    }
  };
  auto cbar = [] { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); };  // compute warps only
  __syncthreads();  // lidx, barriers

  if (w >= NW) {
    // ================= producers: tile i into stage i & 1 once the tile two back left it
    const int pt = tid - NT, ch = pt & 7;
    for (int i = 0; i < ntl; ++i) {
      const int t = tile_of(i), b = i & 1;
      if (i >= 2) umma::bar_wait(&empty[b], (uint32_t)(((i - 2) >> 1) & 1));
      const int q = t < tiles0 ? 0 : 1;
      const StripDesc<float>& s = a.s[q];
      const int x0 = (t - (q ? tiles0 : 0)) * TP;
      float* D = stageD(b);
      const int* li = lidx + q * nl8;
      const int pos = x0 + 4 * ch, rem = s.npos - pos;
      const uint32_t bytes = rem >= 4 ? 16u : (rem > 0 ? 4u * rem : 0u);
      const float* src = s.src + (bytes ? pos : x0);
      const int ls = (int)s.line_stride;  // (strips6_supported: < 2^31)
      for (int L = pt >> 3; L < s.nk; L += 16)
        s6_cp16(D + L * TP + 4 * (ch ^ (L & 6)), src + (long long)li[L] * ls, bytes);
      for (int tt = pt >> 3; tt < R; tt += 16)
        s6_cp16(stageQ(b) + tt * TP + 4 * ch, s.Bold + (int64_t)tt * s.ldb + (bytes ? pos : x0), bytes);
      if (pt < 8) s6_cp16(stageO(b) + 4 * ch, s.omap + (bytes ? pos : x0), bytes);
      umma::cp_async_arrive(&full[b]);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }

  const bool rec = a.dbg && bx == 0 && tid == 0;
  long long tpc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tq = clock64();
#define S6PH(k) do { if (rec) { const long long _t = clock64(); tpc[k] += _t - tq; tq = _t; } } while (0)
  int cur = -1;
  int pad_pending = 3;  // stages whose rows [nk, nl8) must be zeroed before their next tile (bit b)
  Pair<float> den2 = Pair<float>::splat(0.f), res2 = Pair<float>::splat(0.f);
  for (int i = 0; i < ntl; ++i) {
    const int t = tile_of(i), b = i & 1;
    const int q = t < tiles0 ? 0 : 1;
    const StripDesc<float>& s = a.s[q];
    const int x0 = (t - (q ? tiles0 : 0)) * TP;
    const int nk = s.nk, nb = (nk + 7) >> 3;
    S6PH(7);
    if (q != cur) {  // new strip: every compute warp is done with the previous tile
      cbar();
      load_strip(q);
      if (cur >= 0) pad_pending = 3;
      cur = q;
      cbar();
    }
    umma::bar_wait(&full[b], (uint32_t)((i >> 1) & 1));  // tile i landed
    if (pad_pending & (1 << b)) {  // (the producer never writes these rows of this strip)
      float* Dz = stageD(b);
      for (int e = tid; e < (nl8 - nk) * TP; e += NT) Dz[nk * TP + e] = 0.f;
      pad_pending &= ~(1 << b);
      cbar();
    }
    S6PH(0);
    S6PH(1);
    float* D = stageD(b);
    const float* Qs = stageQ(b);
    const int* Om = stageO(b);
    // per tile: override indices at this lane's four positions; the old
    // factor at them as FFMA2 pairs (positions 4g, 4g + 1 | 4g + 2, 4g + 3)
    // I x J entries of c: the core's values (solver.py:216-221), fetched now
    // (latency under pass 1) and written into the stage after it.  Pass 1
    // needs none of them: the factor at these positions is the override.
    const int om_l = x0 + lane < s.npos ? Om[lane] : -1;
    const unsigned omask = __ballot_sync(0xffffffffu, om_l >= 0);  // (the same in every warp)
    const int n_items = __popc(omask) * nk;
    float upre[2];
    int uoff[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int item = tid + k * NT;
      uoff[k] = -1;
      if (item < n_items) {
        const int which = item / nk, L = item - which * nk;
        unsigned m = omask;
        for (int z = 0; z < which; ++z) m &= m - 1;
        const int pos = __ffs(m) - 1, e = Om[pos];
        upre[k] = (float)s.U[(int64_t)L * s.u_ls + (int64_t)e * s.u_ps];
        uoff[k] = L * TP + 4 * ((pos >> 2) ^ (L & 6)) + (pos & 3);
      }
    }
    float2 qp[R][2];
#pragma unroll
    for (int tt = 0; tt < R; ++tt) {
      const float4 v = *reinterpret_cast<const float4*>(Qs + tt * TP + 4 * g);
      qp[tt][0] = make_float2(v.x, v.y);
      qp[tt][1] = make_float2(v.z, v.w);
    }
    // ---- pass 1: l (FFMA2), Phase I/II (solver.py:375-382), c over d, MMA2 partials
    float acc[2][5][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int n = 0; n < 5; ++n)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[mt][n][j] = 0.f;
    const uint32_t n4mask = (g & 1) ? 0u : 0xffffffffu, wxmask = g < 4 ? 0xffffffffu : 0u;
    for (int blk = w; blk < nb; blk += NW) {
      const int L0 = 8 * blk + 2 * c;
      // W' fragments, lines L0 and L0 + 1 at column g: [W_hi | W_lo | hi8 lo8 hi9 lo9] and [W_hi | hi8 0 hi9 0]
      uint32_t bw[5][2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float* wl = Wv + (L0 + h) * WS;
        const float2 whl = *reinterpret_cast<const float2*>(wl + 2 * g);
        const uint32_t wx = s6_u(wl[16 + (g & 3)]) & wxmask;  // (zero for g >= 4)
        bw[0][h] = s6_u(whl.x);
        bw[1][h] = s6_u(whl.y);
        bw[2][h] = wx;
        bw[3][h] = bw[0][h];
        bw[4][h] = wx & n4mask;
      }
      const int sw = L0 & 6;
      float* d0p = D + L0 * TP + 4 * (g ^ sw);
      float* d1p = d0p + TP;
      const float4 dv0 = *reinterpret_cast<const float4*>(d0p);
      const float4 dv1 = *reinterpret_cast<const float4*>(d1p);
      Pair<float> dd[2][2];  // [line h][m-tile]
      dd[0][0].v = make_float2(dv0.x, dv0.y); dd[0][1].v = make_float2(dv0.z, dv0.w);
      dd[1][0].v = make_float2(dv1.x, dv1.y); dd[1][1].v = make_float2(dv1.z, dv1.w);
      // l = <P(line, :), Q(:, pos)>: the core kernel's chain (lowrank_entry), two positions per FFMA2
      Pair<float> ll[2][2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float* pl = Pv + (L0 + h) * PS;
        float pv[PS];
#pragma unroll
        for (int k4 = 0; k4 < (R + 3) / 4; ++k4) {
          const float4 v = *reinterpret_cast<const float4*>(pl + 4 * k4);
          pv[4 * k4] = v.x; pv[4 * k4 + 1] = v.y; pv[4 * k4 + 2] = v.z; pv[4 * k4 + 3] = v.w;
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          ll[h][mt].v = __fmul2_rn(make_float2(pv[0], pv[0]), qp[0][mt]);
#pragma unroll
          for (int tt = 1; tt < R; ++tt) ll[h][mt].v = __ffma2_rn(make_float2(pv[tt], pv[tt]), qp[tt][mt], ll[h][mt].v);
        }
      }
      Pair<float> ee[2][2];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          ee[h][mt] = keep_pair(dd[h][mt], ll[h][mt], a.zt);
          den2 = pfma(dd[h][mt], dd[h][mt], den2);
        }
      // MMA2, A fragment of m-tile mt: (row g, K c) = (p, L0), (g + 8, c) = (p + 1, L0), (g, c + 4) = (p, L0 + 1), ..
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        Pair<float> h0, h1;
        h0.v = make_float2(s6_hi(ee[0][mt].v.x), s6_hi(ee[0][mt].v.y));
        h1.v = make_float2(s6_hi(ee[1][mt].v.x), s6_hi(ee[1][mt].v.y));
        const Pair<float> l0 = psub(ee[0][mt], h0), l1 = psub(ee[1][mt], h1);
        const uint32_t ah[4] = {s6_u(h0.v.x), s6_u(h0.v.y), s6_u(h1.v.x), s6_u(h1.v.y)};
        const uint32_t al[4] = {s6_u(l0.v.x), s6_u(l0.v.y), s6_u(l1.v.x), s6_u(l1.v.y)};
        s6_mma(acc[mt][0], ah, bw[0][0], bw[0][1]);
        s6_mma(acc[mt][1], ah, bw[1][0], bw[1][1]);
        s6_mma(acc[mt][2], ah, bw[2][0], bw[2][1]);
        s6_mma(acc[mt][3], al, bw[3][0], bw[3][1]);
        s6_mma(acc[mt][4], al, bw[4][0], bw[4][1]);
      }
      *reinterpret_cast<float4*>(d0p) = make_float4(ee[0][0].v.x, ee[0][0].v.y, ee[0][1].v.x, ee[0][1].v.y);
      *reinterpret_cast<float4*>(d1p) = make_float4(ee[1][0].v.x, ee[1][0].v.y, ee[1][1].v.x, ee[1][1].v.y);
    }
    S6PH(2);
    // ---- this warp's factor partials: F(p, t) = (hi.hi + lo.hi) + hi.lo
    {
      float* rw = red + (size_t)w * RMAX * TP;
      float fa[4], fb[4], fx[4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
        for (int r8 = 0; r8 < 2; ++r8) {
          const int j0 = 2 * r8;  // accumulator entries of row g (+8): columns 2c, 2c + 1
          fa[2 * mt + r8] = __fadd_rn(__fadd_rn(acc[mt][0][j0], acc[mt][3][j0]), acc[mt][1][j0]);
          fb[2 * mt + r8] = __fadd_rn(__fadd_rn(acc[mt][0][j0 + 1], acc[mt][3][j0 + 1]), acc[mt][1][j0 + 1]);
          fx[2 * mt + r8] = __fadd_rn(__fadd_rn(acc[mt][2][j0], acc[mt][4][j0]), acc[mt][2][j0 + 1]);
        }
      }
      *reinterpret_cast<float4*>(rw + (2 * c) * TP + 4 * g) = make_float4(fa[0], fa[1], fa[2], fa[3]);
      *reinterpret_cast<float4*>(rw + (2 * c + 1) * TP + 4 * g) = make_float4(fb[0], fb[1], fb[2], fb[3]);
      if (c < 2) *reinterpret_cast<float4*>(rw + (8 + c) * TP + 4 * g) = make_float4(fx[0], fx[1], fx[2], fx[3]);
    }
    cbar();  // (B)
    S6PH(3);
    if (i > 0 && tid == 0) {  // per-tile sums of tile i - 1 (warps in order; all wrote them before (B))
      const int tp = tile_of(i - 1), qp = tp < tiles0 ? 0 : 1;
      const double* dr = dred + ((i - 1) & 1) * NW * 2;
      double sd = 0.0, sr = 0.0;
      for (int ww = 0; ww < NW; ++ww) {
        sd += dr[2 * ww];
        sr += dr[2 * ww + 1];
      }
      double* pr = a.partials + 4 * (size_t)tp;
      pr[qp ? 2 : 0] = sd; pr[qp ? 3 : 1] = sr; pr[qp ? 0 : 2] = 0.0; pr[qp ? 1 : 3] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (uoff[k] >= 0) D[uoff[k]] = upre[k];
    for (int item = tid + 2 * NT; item < n_items; item += NT) {  // (more than 2 I x J positions in the tile: rare)
      const int which = item / nk, L = item - which * nk;
      unsigned m = omask;
      for (int z = 0; z < which; ++z) m &= m - 1;
      const int pos = __ffs(m) - 1, e = Om[pos];
      D[L * TP + 4 * ((pos >> 2) ^ (L & 6)) + (pos & 3)] = (float)s.U[(int64_t)L * s.u_ls + (int64_t)e * s.u_ps];
    }
    // ---- factor sums over the warps (fixed order), override, new factor
    for (int o = tid; o < R * TP; o += NT) {
      const int tt = o >> 5, pos = o & 31;
      const int x = x0 + pos;
      float v = red[tt * TP + pos];
#pragma unroll 4
      for (int ww = 1; ww < NW; ++ww) v = __fadd_rn(v, red[((size_t)ww * RMAX + tt) * TP + pos]);
      if (x < s.npos) {
        const int e = Om[pos];
        if (e >= 0) v = s.otherF[(int64_t)e * R + tt];
        s.Fnew[(int64_t)tt * s.ldf + x] = v;
      } else {
        v = 0.f;
      }
      fsm[tt * TP + pos] = v;
    }
    cbar();  // (C)
    S6PH(4);
    // MMA3 A fragments -F' of every lane, built once per tile: float4 k of
    // lane ln holds (mt, st) = (k >> 2, k & 3), entries j = 0..3
    for (int e = tid; e < 32 * 8; e += NT) {
      const int ln = e & 31, k = e >> 5;
      const int gg = ln >> 2, cc = ln & 3, mt = k >> 2, st = k & 3;
      const S6Slots S2 = s6_slots(cc);
      float o4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int p = 4 * gg + 2 * mt + (j & 1), slot = 2 * st + (j >> 1);
        const int tt = slot < 3 ? 2 * cc : (slot < 6 ? 2 * cc + 1 : (slot == 6 ? S2.t6 : S2.t7));
        const float f = fsm[tt * TP + p];
        const int term = slot < 6 ? slot % 3 : -1;  // 0 hi, 1 lo, 2 hi twin
        float v;
        if (term == 0) v = -s6_hi(f);
        else if (term == 1) v = -s6_lo(f);
        else if (term == 2) v = __uint_as_float(s6_twin(s6_u(-s6_hi(f))));
        else if (S2.z67) v = 0.f;
        else v = -((slot == 6 ? S2.a6lo : S2.a7lo) ? s6_lo(f) : s6_hi(f));
        o4[j] = v;
      }
      a3s[k * 32 + ln] = make_float4(o4[0], o4[1], o4[2], o4[3]);
    }
    cbar();  // (D)
    S6PH(5);
    // ---- pass 2: r = c - F'.Res'^T (MMA3 accumulated onto c), squared residual (solver.py:393-400)
    uint32_t A3[2][4][4];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 v = a3s[k * 32 + lane];
      A3[k >> 2][k & 3][0] = s6_u(v.x); A3[k >> 2][k & 3][1] = s6_u(v.y);
      A3[k >> 2][k & 3][2] = s6_u(v.z); A3[k >> 2][k & 3][3] = s6_u(v.w);
    }
    for (int blk = w; blk < nb; blk += NW) {
      const int L0 = 8 * blk + 2 * c, Lg = 8 * blk + g;
      uint32_t B3[8];
      s6_bslots(S, Rv + Lg * PS, c, B3);
      const int sw = L0 & 6;
      const float4 cv0 = *reinterpret_cast<const float4*>(D + L0 * TP + 4 * (g ^ sw));
      const float4 cv1 = *reinterpret_cast<const float4*>(D + (L0 + 1) * TP + 4 * (g ^ sw));
      float r[2][4] = {{cv0.x, cv1.x, cv0.y, cv1.y}, {cv0.z, cv1.z, cv0.w, cv1.w}};
#pragma unroll
      for (int st = 0; st < 4; ++st)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) s6_mma(r[mt], A3[mt][st], B3[2 * st], B3[2 * st + 1]);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        Pair<float> x0p, x1p;
        x0p.v = make_float2(r[mt][0], r[mt][1]);
        x1p.v = make_float2(r[mt][2], r[mt][3]);
        res2 = pfma(x0p, x0p, res2);
        res2 = pfma(x1p, x1p, res2);
      }
    }
    S6PH(6);
    {  // this warp's sums of tile i (read by thread 0 after the next barrier)
      const double dw = warp_sum((double)den2.v.x + (double)den2.v.y);
      const double rw2 = warp_sum((double)res2.v.x + (double)res2.v.y);
      if (lane == 0) {
        dred[(i & 1) * NW * 2 + 2 * w] = dw;
        dred[(i & 1) * NW * 2 + 2 * w + 1] = rw2;
      }
      den2 = Pair<float>::splat(0.f);
      res2 = Pair<float>::splat(0.f);
    }
    __syncwarp();
    if (lane == 0) umma::bar_arrive(&empty[b]);  // this warp is done with stage b
  }
  if (ntl > 0) {
    cbar();
    if (tid == 0) {
      const int i = ntl - 1;
      const int tp = tile_of(i), qp = tp < tiles0 ? 0 : 1;
      const double* dr = dred + (i & 1) * NW * 2;
      double sd = 0.0, sr = 0.0;
      for (int ww = 0; ww < NW; ++ww) {
        sd += dr[2 * ww];
        sr += dr[2 * ww + 1];
      }
      double* pr = a.partials + 4 * (size_t)tp;
      pr[qp ? 2 : 0] = sd; pr[qp ? 3 : 1] = sr; pr[qp ? 0 : 2] = 0.0; pr[qp ? 1 : 3] = 0.0;
    }
  }
  if (rec)
    for (int k = 0; k < 8; ++k) a.dbg[k] += tpc[k];
#undef S6PH
}

bool strips6_supported(const StripsArgs<float>& a, int R) {
  if (R > s6::RMAX || !a.tc_ok) return false;
  int maxl = 0;
  for (int q = 0; q < 2; ++q) {
    const StripDesc<float>& s = a.s[q];
    if (s.tiles == 0) continue;
    if (!s.bulk_ok || s.mode != kStripFull || s.pos_stride != 1 || !s.U) return false;
    if (s.nk > s6::LMAX || s.line_stride >= ((int64_t)1 << 31)) return false;
    if (((uintptr_t)s.Bold & 15) || (s.ldb & 3) || ((uintptr_t)s.omap & 15)) return false;
    maxl = s.nk > maxl ? s.nk : maxl;
  }
  return s6::layout<12>(maxl).total <= (size_t)227 * 1024;  // (the larger of the two layouts)
}

size_t strips6_smem_bytes(int maxl) { return s6::layout<12>(maxl).total; }

template <int NW, int R>
static cudaError_t launch_s6(const StripsArgs<float>& a, int grid, size_t smem, cudaStream_t st) {
  static std::atomic<unsigned long long> devs{0};
  const cudaError_t attr = smem_attr_once(devs, strips6_kernel<NW, R>, 227 * 1024);
  if (attr != cudaSuccess) return attr;
  strips6_kernel<NW, R><<<grid, (NW + 4) * 32, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_strips6(const StripsArgs<float>& a0, int R, int num_sms, int* ncta_out, cudaStream_t st) {
  using namespace s6;
  if (ncta_out) *ncta_out = 0;
  if (!strips6_supported(a0, R)) return cudaErrorNotSupported;
  StripsArgs<float> a = a0;
  for (int q = 0; q < 2; ++q)
    if (a.s[q].tiles > 0) a.s[q].tiles = (a.s[q].npos + TP - 1) / TP;
  const int tiles = a.s[0].tiles + a.s[1].tiles;
  if (tiles == 0) return cudaSuccess;
  const int maxl = a.s[0].nk > a.s[1].nk ? a.s[0].nk : a.s[1].nk;
  const int grid = tiles < num_sms ? tiles : num_sms;
  cudaError_t e = cudaErrorNotSupported;
  const char* nwe = std::getenv("IRCUR_S6_NW");  // A/B: 8 (default, measured faster) or 12 compute warps
  if (!nwe || std::atoi(nwe) != 12) {
    IRCUR_DISPATCH_RANK(R, RR, if constexpr (RR <= RMAX) e = launch_s6<8, RR>(a, grid, layout<8>(maxl).total, st));
  } else {
    IRCUR_DISPATCH_RANK(R, RR, if constexpr (RR <= RMAX) e = launch_s6<12, RR>(a, grid, layout<12>(maxl).total, st));
  }
  if (e == cudaSuccess && ncta_out) *ncta_out = tiles;  // partial slots: one per tile
  return e;
}

}  // namespace ircur
