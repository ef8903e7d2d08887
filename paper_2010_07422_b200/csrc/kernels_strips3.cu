// Fused row + column strip kernel, fp32, 64-position tiles (sm_100a).
//
// Same per-entry semantics as kernels_strips.cu / kernels_strips2.cu
// (Phase I/II, factor sums with the core overrides, stopping residual;
// solver.py:375-400).  What bounds those kernels is shared-memory wavefronts,
// dominated by the per-line vectors A | W | Res that every warp broadcasts
// for each line it processes (LDS.128 broadcast = 2 wavefronts, 8 bytes
// each).  Here each lane owns TWO adjacent positions (2 lane and 2 lane + 1 of
// a 64-position tile, packed in FFMA2 pairs), so every line-vector load feeds
// 2x the entries of kernels_strips2.cu and every stage access is one 8-byte
// load or store.  The price is shared memory: all sampled lines of a
// 64-position tile are resident in ONE single-buffered stage per CTA (16 warps
// on the same tile), filled in two halves with cp.async.
//
// Two instantiations:
//   TC = false  pass 2 (the stopping residual) as FFMA2 chains; the next
//               tile's halves are issued as pass 2 frees them.
//   TC = true   pass 2 on the tensor cores: the thresholded tile moves to TMEM
//               (tcgen05.st) and tcgen05.mma kind::tf32 accumulates
//               -Res' F'^T onto it, with Res' in TMEM and F' in shared memory,
//               both split exactly into three tf32 pieces; the next tile's
//               fill is issued under the MMAs.  Taken for row strips of at
//               least 32768 positions.
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels_iter.cuh"
#include "launchers.cuh"
#include "umma.cuh"

namespace ircur {

constexpr int kS3NT = 512;
constexpr int kS3NW = kS3NT / 32;
constexpr int kS3TX = 64;  // positions per tile (2 lane, 2 lane + 1 per lane)

// Tensor-core residual (TC): pass 2, r = c - <Res_line, Fnew(:, x)>, runs as
// tcgen05 tf32 MMAs with the lines on the TMEM lanes (M = 128 lines per
// block, N = 64 positions).  A = Res' lives in TMEM (written once per strip),
// B = F' is a 16 KB K-major SW128 operand in shared memory.
// Both are split exactly into three tf32 pieces (x = hi + mid + lo, 11 + 11 +
// 2 bits), and the six products whose weight is above 2^-31 are laid along
// K = 6 R <= 64, so the product is exact to fp32 round-off and the fp32
// accumulator is the only rounding.  The stage rows are padded to 68 floats:
// a thread then reads its own line's 64 entries with conflict-free LDS.128.
constexpr int kS3K = 64;       // K of the residual MMA (6 R <= 64)
constexpr int kS3SXtc = 68;    // padded stage row (floats) of the TC layout
// TMEM columns for lines in up to nb 128-line blocks: Res' in [0, 64 nb), the
// residual accumulator in [cols / 2, cols / 2 + 64 nb).  Up to 256 lines need
// 256 columns, so two CTAs of the batched kernel can share an SM.
__host__ __device__ inline int strips3_tmem_cols(int maxl) { return maxl <= 128 ? 128 : (maxl <= 256 ? 256 : 512); }

struct Strips3Layout {
  int RP, maxp, SX, nvec;
  size_t fop, lvec, stage, bst, omt, lptr, red, fnew, dred, bars, total;
};

__host__ __device__ inline size_t al3(size_t x) { return (x + 127) & ~size_t(127); }

__host__ __device__ inline Strips3Layout strips3_layout(int maxl, int R, bool tc = false) {
  Strips3Layout L;
  L.RP = R + (R & 1);
  L.maxp = (maxl + 1) / 2;
  L.SX = tc ? kS3SXtc : kS3TX;
  L.nvec = tc ? 2 : 3;  // A | W (| Res: the FFMA residual only)
  size_t off = 0;
  if (tc) { L.fop = off; off = al3(off + (size_t)kS3TX * kS3K * sizeof(float)); }  // F' (1 KB atoms)
  L.lvec = off; off = al3(off + (size_t)L.maxp * L.nvec * L.RP * sizeof(float2));
  L.stage = off; off = al3(off + (size_t)2 * L.maxp * L.SX * sizeof(float));
  L.bst = off; off = al3(off + (size_t)R * kS3TX * sizeof(float));
  L.omt = off; off = al3(off + (size_t)kS3TX * sizeof(int));
  L.lptr = off; off = al3(off + (size_t)2 * (2 * L.maxp + R) * sizeof(void*));
  L.red = off; off = al3(off + (size_t)kS3NW * R * kS3TX * sizeof(float));
  L.fnew = off;
  if (!tc) off = al3(off + (size_t)R * kS3TX * sizeof(float));  // (TC: the sums go straight into F')
  L.dred = off; off = al3(off + 4 * kS3NW * sizeof(double));
  L.bars = off; off = al3(off + 64);
  L.total = off;
  return L;
}

__device__ __forceinline__ uint32_t s3_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// byte offset of element (row, k) of the F' operand: K-major, 128-byte
// swizzle, 64 rows (positions) x K = 64 as two K atoms of 32 (8 KB each)
__device__ __forceinline__ uint32_t s3_fop(int row, int k) {
  return (uint32_t)((k >> 5) * (kS3TX * 128) + (row >> 3) * 1024 + (row & 7) * 128 +
                    (((((k & 31) >> 2) ^ (row & 7)) & 7) << 4) + (k & 3) * 4);
}
// exact three-way tf32 split: x = hi + mid + lo (11 + 11 + 2 significant bits)
__device__ __forceinline__ void s3_split(float x, float& hi, float& mid, float& lo) {
  hi = umma::tf32_hi(x);
  const float m1 = __fsub_rn(x, hi);
  mid = umma::tf32_hi(m1);
  lo = __fsub_rn(m1, mid);
}

template <int R, bool TC>
__device__ __forceinline__ void strips3_body(const StripsArgs<float>& a, int bx, int nbx) {
  static_assert(!TC || 6 * R <= kS3K, "the residual MMA lays six products along K = 64");
  if (*a.done) return;
  const Strips3Layout L = strips3_layout(a.maxl, R, TC);
  constexpr int RPc = R + (R & 1);
  constexpr int NV = TC ? 2 : 3;
  constexpr int SX = TC ? kS3SXtc : kS3TX;
  extern __shared__ __align__(1024) unsigned char sm[];
  float2* lvec = reinterpret_cast<float2*>(sm + L.lvec);
  float* stage = reinterpret_cast<float*>(sm + L.stage);
  float* bst = reinterpret_cast<float*>(sm + L.bst);
  int* omt = reinterpret_cast<int*>(sm + L.omt);
  const float** lptr = reinterpret_cast<const float**>(sm + L.lptr);
  float* red = reinterpret_cast<float*>(sm + L.red);
  float* fnew = reinterpret_cast<float*>(sm + L.fnew);
  double* dred = reinterpret_cast<double*>(sm + L.dred);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bars);  // TC: one per 128-line block
  uint32_t* tbase = reinterpret_cast<uint32_t*>(sm + L.bars + 32);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const float zt = a.zt;
  const bool rec = a.dbg && bx == 0 && tid == 0;
  long long tpc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tq = clock64();
#define SPH(k) do { if (rec) { const long long _t = clock64(); tpc[k] += _t - tq; tq = _t; } } while (0)

  const int tmem_d = strips3_tmem_cols(a.maxl) / 2;  // first column of the residual accumulator
  uint32_t T = 0;       // TMEM base
  uint32_t mma_n = 0;   // residual MMAs issued so far (mbarrier phase)
  unsigned char* fop = sm + L.fop;
  if constexpr (TC) {
    for (int e = tid; e < kS3TX * kS3K / 4; e += kS3NT)  // (the K padding past 6 R stays zero)
      reinterpret_cast<float4*>(fop)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (w == 0) umma::tmem_alloc(tbase, (uint32_t)strips3_tmem_cols(a.maxl));
    if (tid == 0) {
#pragma unroll
      for (int b = 0; b < 4; ++b) umma::bar_init(bars + b, 1);
      umma::bar_init_fence();
    }
    umma::fence_before();
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {  // segment sources: lines, then the R rows of the old factor
    const StripDesc<float>& s = a.s[q];
    float const** lp = lptr + q * (2 * L.maxp + R);
    for (int e = tid; e < s.nk + R; e += kS3NT)
      lp[e] = e < s.nk ? s.src + (int64_t)(s.lines[e] - s.line_off) * s.line_stride : s.Bold + (int64_t)(e - s.nk) * s.ldb;
  }
  const int tiles0 = a.s[0].tiles;
  const int total = tiles0 + a.s[1].tiles;
  __syncthreads();
  if constexpr (TC) {
    umma::fence_after();
    T = *tbase;
  }
  // The stage is filled in two halves by line pairs: A = pairs [0, npA) with
  // the old factor's rows and the override map, B = the rest.  FFMA residual:
  // A of the next tile is issued once pass 2 is done with A of this one, and
  // B once pass 2 is done with B, so the fills overlap pass 2 (B) and pass 1
  // (A) instead of stalling the CTA.  TC residual: the thresholded tile moves
  // to TMEM right after pass 1, which frees the stage; both halves are issued
  // then.  Each warp still walks its line pairs in ascending order, so
  // the factor sums are those of a single pass.
  auto halves = [&](int t, int& np, int& npA) {
    const int q = t < tiles0 ? 0 : 1;
    np = (a.s[q].nk + 1) / 2;
    npA = (np + 1) / 2;
  };
  auto issue_half = [&](int t, int h) {
    const int q = t < tiles0 ? 0 : 1;
    const StripDesc<float>& s = a.s[q];
    const int nl = s.nk;
    int np, npA;
    halves(t, np, npA);
    const int nl2 = 2 * np;
    const int x0 = (t - (q ? tiles0 : 0)) * kS3TX;
    const float* const* lp = lptr + q * (2 * L.maxp + R);
    const int ch = tid & 15;
    const int pos = x0 + ch * 4;
    const int rem = s.npos - pos;
    const int bytes = rem >= 4 ? 16 : (rem > 0 ? rem * 4 : 0);
    const int sp = bytes ? pos : x0;
    const int v0 = h ? 2 * npA : 0, v1 = h ? nl2 : 2 * npA + R;  // (half A: + the R rows, mapped past nl2)
    for (int u = v0 + (tid >> 4); u < v1; u += kS3NT / 16) {
      const int v = (!h && u >= 2 * npA) ? nl2 + (u - 2 * npA) : u;
      float* dst = v < nl2 ? stage + (size_t)v * SX : bst + (size_t)(v - nl2) * kS3TX;
      const float* src = v < nl ? lp[v] : (v < nl2 ? lp[0] : lp[nl + (v - nl2)]);
      const int bb = v < nl || v >= nl2 ? bytes : 0;  // the padding line of an odd count reads zeros
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s3_smem(dst + ch * 4)), "l"(src + sp),
                   "r"(bb)
                   : "memory");
    }
    if (!h && tid < 16) {
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s3_smem(omt + ch * 4)),
                   "l"(s.omap + sp), "r"(bytes)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (bx < total) {
    issue_half(bx, 0);
    issue_half(bx, 1);
  }
  int cur = -1;
  for (int t = bx; t < total; t += nbx) {
    const int q = t < tiles0 ? 0 : 1;
    const StripDesc<float>& s = a.s[q];
    const int nl = s.nk, np = (nl + 1) / 2;
    const int npA = (np + 1) / 2;
    const int mode = s.mode;
    const int x0 = (t - (q ? tiles0 : 0)) * kS3TX;
    const int tn = t + nbx;
    const bool next = tn < total;
    const bool same_next = next && ((tn < tiles0) == (t < tiles0));  // the next tile's halves line up with these
    if (q != cur) {  // per-pair line vectors of this strip: (A | W | Res)[t] for lines 2kp, 2kp+1
#pragma unroll 4  // (independent global loads: batch them)
      for (int e = tid; e < np * NV * RPc; e += kS3NT) {
        const int kp = e / (NV * RPc), rem = e - kp * NV * RPc, v = rem / RPc, tt = rem - v * RPc;
        const float* sv = v == 0 ? s.lineA : (v == 1 ? s.lineW : s.lineRes);
        const int k0 = 2 * kp, k1 = k0 + 1;
        float2 val = make_float2(0.f, 0.f);
        if (tt < R) {
          val.x = sv[(int64_t)k0 * R + tt];
          if (k1 < nl) val.y = sv[(int64_t)k1 * R + tt];
        }
        lvec[e] = val;
      }
      if constexpr (TC) {
        // Res' of this strip into TMEM: line 128 b + 32 (w & 3) + lane of block
        // b = w >> 2 is lane 32 (w & 3) + lane, columns [64 b, 64 b + 64):
        // [hi | hi | mid | mid | hi | lo] against F' = [hi | mid | hi | mid | lo | hi]
        // (every residual MMA of the previous strip completed before the
        // barrier that closed its last tile)
        const int line = 128 * (w >> 2) + 32 * (w & 3) + lane;
        const bool live = mode != kStripPartial && line < nl;
        const uint32_t ta = T + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)(kS3K * (w >> 2));
        float rr[R];  // this line's Res row (loaded once)
#pragma unroll
        for (int tt = 0; tt < R; ++tt) rr[tt] = live ? s.lineRes[(int64_t)line * R + tt] : 0.f;
#pragma unroll
        for (int c = 0; c < kS3K / 16; ++c) {  // 16 columns at a time (registers)
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int k = 16 * c + j, part = k / R, tt = k - part * R;  // compile-time after unrolling
            float val = 0.f;
            if (part < 6) {
              float hi, mid, lo;
              s3_split(rr[tt], hi, mid, lo);
              val = (part == 0 || part == 1 || part == 4) ? hi : (part == 5 ? lo : mid);
            }
            v[j] = val;
          }
          umma::st16(ta + 16 * c, v);
        }
        umma::st_wait();
        umma::fence_before();
      }
      cur = q;
    }
    SPH(6);
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // half A of this tile (B may be in flight)
    __syncthreads();
    SPH(0);
    Pair<float> b[R];
#pragma unroll
    for (int tt = 0; tt < R; ++tt) b[tt].v = reinterpret_cast<const float2*>(bst + tt * kS3TX)[lane];
    // ---- pass 1: Phase I/II in place + factor partials (positions 2 lane, 2 lane + 1 per FFMA2)
    Pair<float> acc[R];
#pragma unroll
    for (int tt = 0; tt < R; ++tt) acc[tt] = Pair<float>::splat(0.f);
    Pair<float> den = Pair<float>::splat(0.f);
    const bool accum = mode != kStripFinish;
    auto pass1 = [&](int k_lo, int k_hi) {
      for (int kp = w + ((k_lo > w ? k_lo - w : 0) + kS3NW - 1) / kS3NW * kS3NW; kp < k_hi; kp += kS3NW) {
        const float2* va = lvec + (size_t)kp * NV * RPc;
        float2* c0 = reinterpret_cast<float2*>(stage + (size_t)(2 * kp) * SX) + lane;
        float2* c1 = c0 + SX / 2;
        Pair<float> d0, d1;
        d0.v = *c0;
        d1.v = *c1;
        float2 av = va[0];
        Pair<float> l0, l1;
        l0.v = __fmul2_rn(make_float2(av.x, av.x), b[0].v);
        l1.v = __fmul2_rn(make_float2(av.y, av.y), b[0].v);
#pragma unroll
        for (int tt = 1; tt < R; ++tt) {
          av = va[tt];
          l0.v = __ffma2_rn(make_float2(av.x, av.x), b[tt].v, l0.v);
          l1.v = __ffma2_rn(make_float2(av.y, av.y), b[tt].v, l1.v);
        }
        const Pair<float> e0 = keep_pair(d0, l0, zt);
        const Pair<float> e1 = keep_pair(d1, l1, zt);
        den = pfma(d0, d0, den);
        den = pfma(d1, d1, den);
        *c0 = e0.v;
        *c1 = e1.v;
        if (accum) {
          const float2* vw = va + RPc;
#pragma unroll
          for (int tt = 0; tt < R; ++tt) {
            const float2 wv = vw[tt];
            acc[tt].v = __ffma2_rn(make_float2(wv.x, wv.x), e0.v, acc[tt].v);
            acc[tt].v = __ffma2_rn(make_float2(wv.y, wv.y), e1.v, acc[tt].v);
          }
        }
      }
    };
    pass1(0, npA);
    asm volatile("cp.async.wait_group 0;" ::: "memory");  // half B
    __syncthreads();
    pass1(npA, np);
    SPH(1);
    const double den_t = accum ? (double)den.v.x + (double)den.v.y : 0.0;
    double res_t = 0.0;
    if (accum) {
#pragma unroll
      for (int tt = 0; tt < R; ++tt) {
        reinterpret_cast<float2*>(red + (w * R + tt) * kS3TX)[lane] = acc[tt].v;
      }
    }
    __syncthreads();
    SPH(2);
    const bool ovr = mode != kStripPartial;
    if constexpr (TC) {
      // The thresholded tile moves to TMEM as the residual accumulator: the
      // thread of line 128 b + 32 (w & 3) + lane stores its 64 entries to lane
      // 32 (w & 3) + lane, columns [256 + 64 b, + 64).  The MMAs then subtract
      // Res' F'^T from it: the large hi*hi products come first, so only the
      // first accumulations round at the magnitude of c.  With c in TMEM the
      // stage is free once the factor sums are done, and the next tile's fill
      // runs under the MMAs and the residual.
      const int bk = w >> 2, line = 128 * bk + 32 * (w & 3) + lane;
      if (mode != kStripPartial && 128 * bk < nl) {
        const uint32_t ta = T + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)(tmem_d + kS3TX * bk);
        const float4* crow = reinterpret_cast<const float4*>(stage + (size_t)(line < nl ? line : 0) * SX);
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          float v[16];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 c = crow[4 * c4 + j];
            v[4 * j] = c.x;
            v[4 * j + 1] = c.y;
            v[4 * j + 2] = c.z;
            v[4 * j + 3] = c.w;
          }
          umma::st16(ta + 16 * c4, v);
        }
        umma::st_wait();
      }
    }
    // ---- factor sums over the 16 warps (fixed order) + overrides
    for (int o = tid; o < R * kS3TX; o += kS3NT) {
      const int tt = o / kS3TX, x = o - tt * kS3TX;
      const int e = (ovr && x0 + x < s.npos) ? omt[x] : -1;
      float v;
      if (e >= 0) {
        v = s.otherF[(int64_t)e * R + tt];
      } else if (accum) {
        v = red[tt * kS3TX + x];
#pragma unroll
        for (int ww = 1; ww < kS3NW; ++ww) v += red[(ww * R + tt) * kS3TX + x];
      } else {
        v = x0 + x < s.npos ? s.Fsrc[(int64_t)tt * s.ldfs + x0 + x] : 0.f;
      }
      if constexpr (TC) {  // -F' = -[hi | mid | hi | mid | lo | hi] (the MMAs accumulate -Res' F'^T onto c)
        float hi, mid, lo;
        s3_split(-v, hi, mid, lo);
        *reinterpret_cast<float*>(fop + s3_fop(x, tt)) = hi;
        *reinterpret_cast<float*>(fop + s3_fop(x, R + tt)) = mid;
        *reinterpret_cast<float*>(fop + s3_fop(x, 2 * R + tt)) = hi;
        *reinterpret_cast<float*>(fop + s3_fop(x, 3 * R + tt)) = mid;
        *reinterpret_cast<float*>(fop + s3_fop(x, 4 * R + tt)) = lo;
        *reinterpret_cast<float*>(fop + s3_fop(x, 5 * R + tt)) = hi;
      } else {
        fnew[o] = v;
      }
      if (x0 + x < s.npos) s.Fnew[(int64_t)tt * s.ldf + x0 + x] = v;
    }
    if constexpr (TC) {
      umma::fence_async_smem();
      umma::fence_before();
    }
    __syncthreads();  // (stage, bst and omt are consumed: the next tile's fill may land)
    SPH(3);
    Pair<float> res = Pair<float>::splat(0.f);
    if constexpr (TC) {
      // ---- pass 2 on the tensor core: r = c - Res' F'^T per 128-line block,
      // each block's MMAs issued by lane 0 of its first warp
      const int bk = w >> 2;
      const bool mine = mode != kStripPartial && 128 * bk < nl;
      if (mine && (w & 3) == 0 && lane == 0) {
        umma::fence_after();
        const uint32_t idesc = umma::idesc_tf32(128, kS3TX, 0, 0);
        const uint32_t fb = umma::smem_u32(fop);
#pragma unroll
        for (int j = 0; j < kS3K / 8; ++j)
          umma::mma_ts(T + tmem_d + kS3TX * bk, T + kS3K * bk + 8 * j,
                       umma::smem_desc(fb + (j >> 2) * (kS3TX * 128) + (j & 3) * 32, 16, 1024, umma::kSwizzle128),
                       idesc, true);
        umma::commit(bars + bk);
      }
      __syncwarp();
      if (next) {
        issue_half(tn, 0);
        issue_half(tn, 1);
      }
      if (mine) {
        umma::bar_wait(bars + bk, mma_n & 1);
        ++mma_n;
        umma::fence_after();
        const int line = 128 * bk + 32 * (w & 3) + lane;
        const uint32_t ta = T + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)(tmem_d + kS3TX * bk);
#pragma unroll
        for (int hx = 0; hx < 4; ++hx) {
          float p[16];
          umma::ld16(ta + 16 * hx, p);
          umma::ld_wait();
          if (line < nl) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              Pair<float> r0;
              r0.v = make_float2(p[2 * j], p[2 * j + 1]);
              res = pfma(r0, r0, res);
            }
          }
        }
        umma::fence_before();
        res_t = (double)res.v.x + (double)res.v.y;
      }
    } else {
    Pair<float> f[R];
    if (mode != kStripPartial) {
#pragma unroll
      for (int tt = 0; tt < R; ++tt) f[tt].v = reinterpret_cast<const float2*>(fnew + tt * kS3TX)[lane];
    }
    // ---- pass 2: stopping residual on the thresholded tile
    auto pass2 = [&](int k_lo, int k_hi) {
      for (int kp = w + ((k_lo > w ? k_lo - w : 0) + kS3NW - 1) / kS3NW * kS3NW; kp < k_hi; kp += kS3NW) {
        const float2* vr = lvec + (size_t)kp * 3 * RPc + 2 * RPc;
        const float2* c0 = reinterpret_cast<const float2*>(stage + (size_t)(2 * kp) * kS3TX) + lane;
        const float2* c1 = c0 + kS3TX / 2;
        Pair<float> e0, e1;
        e0.v = *c0;
        e1.v = *c1;
        float2 rv = vr[0];
        Pair<float> l0, l1;
        l0.v = __fmul2_rn(make_float2(rv.x, rv.x), f[0].v);
        l1.v = __fmul2_rn(make_float2(rv.y, rv.y), f[0].v);
#pragma unroll
        for (int tt = 1; tt < R; ++tt) {
          rv = vr[tt];
          l0.v = __ffma2_rn(make_float2(rv.x, rv.x), f[tt].v, l0.v);
          l1.v = __ffma2_rn(make_float2(rv.y, rv.y), f[tt].v, l1.v);
        }
        const Pair<float> r0 = psub(e0, l0);
        const Pair<float> r1 = psub(e1, l1);
        res = pfma(r0, r0, res);
        res = pfma(r1, r1, res);
      }
    };
    if (mode != kStripPartial) pass2(0, npA);
    if (same_next) {  // half A of this tile is free
      __syncthreads();
      issue_half(tn, 0);
    }
    if (mode != kStripPartial) {
      pass2(npA, np);
      res_t = (double)res.v.x + (double)res.v.y;
    }
    }
    SPH(4);
    {  // per-tile sums (warps in order): e_k does not depend on the grid size
      const double dw = warp_sum(den_t), rw = warp_sum(res_t);
      if (lane == 0) {
        dred[2 * w] = dw;
        dred[2 * w + 1] = rw;
      }
    }
    __syncthreads();  // stage, fnew, red free for the next tile
    if (!TC && next) {
      if (!same_next) issue_half(tn, 0);  // (issued above unless the strip changes)
      issue_half(tn, 1);
    }
    if (w == 0) {  // fixed xor tree over the 16 warps' sums
      double sd = lane < kS3NW ? dred[2 * lane] : 0.0, sr = lane < kS3NW ? dred[2 * lane + 1] : 0.0;
#pragma unroll
      for (int o = kS3NW / 2; o > 0; o >>= 1) {
        sd += __shfl_xor_sync(0xffffffffu, sd, o);
        sr += __shfl_xor_sync(0xffffffffu, sr, o);
      }
      if (lane == 0) {
        double* pr = a.partials + 4 * (size_t)t;
        pr[q ? 2 : 0] = sd;
        pr[q ? 3 : 1] = sr;
        pr[q ? 0 : 2] = 0.0;
        pr[q ? 1 : 3] = 0.0;
      }
    }
    SPH(5);
  }
  if constexpr (TC) {
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    if (w == 0) umma::tmem_free(T, (uint32_t)strips3_tmem_cols(a.maxl));
  }
  if (rec)
    for (int k = 0; k < 8; ++k) a.dbg[k] += tpc[k];
#undef SPH
}

template <int R, bool TC>
__global__ void __launch_bounds__(kS3NT, 1) strips3_kernel(const __grid_constant__ StripsArgs<float> a) {
  strips3_body<R, TC>(a, (int)blockIdx.x, (int)gridDim.x);
}
// batched problems: problem blockIdx.y, its tiles over blockIdx.x
template <int R, bool TC>
__global__ void __launch_bounds__(kS3NT, R <= 6 ? 2 : 1) strips3_kernel_batched(const StripsArgs<float>* __restrict__ as) {
  strips3_body<R, TC>(as[blockIdx.y], (int)blockIdx.x, (int)gridDim.x);
}

size_t strips3_smem_bytes(int maxl, int R) { return strips3_layout(maxl, R).total; }

// The tensor-core residual is the default where it applies (R <= 10, at most
// 512 lines per strip, the padded stage fits) and pays: its per-tile MMA
// round trip needs several tiles per CTA to amortise, so it is taken for row
// strips of at least 32768 positions (measured: cfg5 263 -> 244 us per launch,
// n = 10^4 and smaller 10-15% slower).  The rule depends on the row strip's
// width only, which row sharding and batching do not change, so a problem
// gets the same residual arithmetic on every path.  IRCUR_S3_TC=0 keeps the
// FFMA residual, =2 forces the tensor-core one wherever it fits (A/B runs, tests).
constexpr int kS3TcMinPos = 32768;
std::atomic<int> g_last_strips3_tc{0};
static int strips3_tc_knob() {  // read per launch (tests switch it)
  const char* e = std::getenv("IRCUR_S3_TC");
  return e && e[0] >= '0' && e[0] <= '2' ? e[0] - '0' : 1;
}
bool strips3_uses_tc(int maxl, int R, int row_positions) {
  const int knob = strips3_tc_knob();
  return knob != 0 && (knob == 2 || row_positions >= kS3TcMinPos) && 6 * R <= kS3K && maxl <= 512 &&
         strips3_layout(maxl, R, true).total <= (size_t)227 * 1024;
}

// n problems, ctas CTAs each (the tiles of a problem stride over them).  The
// arguments' tile counts are those of strips3 (64-position tiles) and maxl
// the largest line count over the problems (the smem layout).
template <int RR>
static cudaError_t strips3_launch_batched_one(const StripsArgs<float>* d_args, int n, int ctas, bool tc, size_t smem,
                                              cudaStream_t st) {
  if constexpr (6 * RR <= kS3K) {
    if (tc) {
      static std::atomic<unsigned long long> devs{0};
      const cudaError_t attr = smem_attr_once(devs, strips3_kernel_batched<RR, true>, 227 * 1024);
      if (attr != cudaSuccess) return attr;
      strips3_kernel_batched<RR, true><<<dim3((unsigned)ctas, (unsigned)n), kS3NT, smem, st>>>(d_args);
      return cudaGetLastError();
    }
  }
  static std::atomic<unsigned long long> devs{0};
  const cudaError_t attr = smem_attr_once(devs, strips3_kernel_batched<RR, false>, 227 * 1024);
  if (attr != cudaSuccess) return attr;
  strips3_kernel_batched<RR, false><<<dim3((unsigned)ctas, (unsigned)n), kS3NT, smem, st>>>(d_args);
  return cudaGetLastError();
}

cudaError_t launch_strips3_batched(const StripsArgs<float>* d_args, int n, int ctas, int maxl, int R,
                                   int min_row_positions, cudaStream_t st) {
  if (n <= 0 || ctas <= 0) return cudaSuccess;
  if (strips3_layout(maxl, R).total > (size_t)227 * 1024) return cudaErrorNotSupported;
  // the same residual arithmetic as a problem's own solve (launch_strips3 makes the same choice)
  const bool tc = strips3_uses_tc(maxl, R, min_row_positions);
  const size_t smem = strips3_layout(maxl, R, tc).total;
  cudaError_t e = cudaErrorInvalidValue;
  IRCUR_DISPATCH_RANK(R, RR, { e = strips3_launch_batched_one<RR>(d_args, n, ctas, tc, smem, st); });
  g_last_strips3_tc = tc ? 1 : 0;
  return e;
}

// one rank's launch: the tensor-core residual where it applies, else the FFMA one
template <int RR>
static cudaError_t strips3_launch_one(const StripsArgs<float>& a, bool tc, int grid, size_t smem, cudaStream_t st) {
  if constexpr (6 * RR <= kS3K) {
    if (tc) {
      static std::atomic<unsigned long long> devs{0};  // once per device
      const cudaError_t attr = smem_attr_once(devs, strips3_kernel<RR, true>, 227 * 1024);
      if (attr != cudaSuccess) return attr;
      strips3_kernel<RR, true><<<grid, kS3NT, smem, st>>>(a);
      return cudaGetLastError();
    }
  }
  static std::atomic<unsigned long long> devs{0};  // once per device
  const cudaError_t attr = smem_attr_once(devs, strips3_kernel<RR, false>, 227 * 1024);
  if (attr != cudaSuccess) return attr;
  strips3_kernel<RR, false><<<grid, kS3NT, smem, st>>>(a);
  return cudaGetLastError();
}

// cudaErrorNotSupported when the sampled lines do not fit the stage
cudaError_t launch_strips3(const StripsArgs<float>& a0, int R, int num_sms, int* ncta_out, cudaStream_t st) {
  StripsArgs<float> a = a0;
  a.maxl = a.s[0].nk > a.s[1].nk ? a.s[0].nk : a.s[1].nk;
  for (int q = 0; q < 2; ++q)  // the caller counts tiles of the 64-position cluster kernel (same width)
    if (a.s[q].tiles > 0) a.s[q].tiles = (a.s[q].npos + kS3TX - 1) / kS3TX;
  const bool tc = strips3_uses_tc(a.maxl, R, a.s[0].tiles > 0 ? a.s[0].npos : a.s[1].npos);
  const size_t smem = strips3_layout(a.maxl, R, tc).total;
  if (smem > (size_t)227 * 1024) return cudaErrorNotSupported;
  if (ncta_out) *ncta_out = 0;
  const int tiles = a.s[0].tiles + a.s[1].tiles;
  if (tiles == 0) return cudaSuccess;
  // persistent grid, but no idle CTAs: small problems solved side by side
  // (solve_batch) then leave the other SMs to their neighbours' kernels
  const int grid = tiles < num_sms ? tiles : num_sms;
  cudaError_t e = cudaErrorInvalidValue;
  IRCUR_DISPATCH_RANK(R, RR, { e = strips3_launch_one<RR>(a, tc, grid, smem, st); });
  g_last_strips3_tc = tc ? 1 : 0;
  if (ncta_out) *ncta_out = tiles;  // partial slots: one per tile
  return e;
}

}  // namespace ircur
