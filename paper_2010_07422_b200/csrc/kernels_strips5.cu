// Tensor-core strip kernel (fp32 data; sm_100a tcgen05, kind::tf32).
//
// Same per-entry semantics as kernels_strips3.cu (Phase I/II, the new factor
// with the core overrides, the stopping residual; solver.py:375-400), with the
// three rank-r contractions of a tile on the tensor cores instead of FFMA
// chains.  A tile is 128 positions x all sampled lines of one strip; the
// lines are split over a 4-CTA cluster (<= 128 lines per CTA):
//
//   MMA1  L^T[pos, line]  = B'[pos, k]   . A'[line, k]^T        (K = 32)
//   MMA2  F^T[pos, t]     = c[pos, line] . W'[line, t]           (K = lines)
//   MMA3  Lnew^T[pos, line] = F'[pos, k] . Res'[line, k]^T       (K = 32)
//
// fp32 accuracy from tf32 operands by a 3-term split (the tensor core reads
// the top 10 mantissa bits of an fp32 container, i.e. truncates; measured by
// tools/micro/umma_probe.cu): x = x_hi + x_lo exactly, and
//   a.b ~ a_hi b_hi + a_lo b_hi + a_hi b_lo.
// For the K = r products the split is concatenated along K: B' = [B | B | B_lo]
// against A' = [A_hi | A_lo | A_hi] (3r <= 32).  For MMA2, c (its fp32 value,
// read as c_hi) times [W_hi | W_lo] (N = 32) plus c_lo times W_hi (N = 16).
//
// TMEM (lane = position, 512 columns), two tile slots by tile parity:
//   TL[2] [0,256)   L, then c in place (Phase I/II in registers: l -> c), then
//                   the residual r = c - Lnew: MMA3 accumulates -F'.Res'^T
//                   onto c
//   TC    [256,384) c_lo (MMA2 A operand)
//   TB[2] [384,448) B' (MMA1 A operand), then -F' (MMA3 A operand)
//   TF    [448,480) F^T partial sums (MMA2 accumulator: cols 0-15 hi, 16-31 lo)
// Software pipeline (per CTA, tile t): Phase I/II of t, then the residual of
// t - 1, then -- by the four warps of line group 0 -- B' of t + 1 (so MMA1 of
// t + 1 runs while they finish t) and the factor epilogue of t, while the other
// warps go on to Phase I/II of t + 1.  The epilogue sums the four CTAs' F^T
// partials in rank order: each CTA owns 32 positions, receives the partials
// of its positions from every rank (distributed shared memory stores +
// cluster-scope mbarriers), applies the override of the other index set,
// writes the new factor, and sends the final values to every rank, so all
// four hold the same bits.  D tiles are double-buffered with cp.async (tile
// t + 2 loads once Phase I/II of t is done).  The I x J entries of c are taken
// from the core U (the core kernel's values), so the strips agree with U bit
// for bit on the intersection, as _sync_intersection makes them in the
// reference (solver.py:216-221).
//
// den and the residual are reduced per tile and written per (tile, rank), so
// e_k does not depend on the grid size.
#include <cuda_runtime.h>

#include "kernels_iter.cuh"
#include "launchers.cuh"
#include "umma.cuh"

namespace ircur {

namespace s5 {
constexpr int CS = 4;          // CTAs per cluster
constexpr int TP = 128;        // positions per tile (MMA M, TMEM lanes)
constexpr int ML = 128;        // lines per CTA (MMA N of the K = r products)
constexpr int NW = 16;         // elementwise warps
constexpr int NT = (NW + 1) * 32;
constexpr int KC = 32;         // concatenated K of the r-products
constexpr int RMAX = 10;       // 3 r <= KC
// TMEM columns
constexpr uint32_t TL0 = 0, TC = 256, TB0 = 384, TF = 448, TCOLS = 512;
// shared memory (offsets from a 1 KB aligned base)
constexpr size_t D_BYTES = (size_t)ML * TP * 4;             // one D tile: [line][pos]
constexpr size_t O_D = 0;                                   // 2 D tiles
constexpr size_t O_BST = O_D + 2 * D_BYTES;                 // 2 x Bold staging [RMAX][TP]
constexpr size_t BST_BYTES = (size_t)RMAX * TP * 4;
constexpr size_t O_OM = O_BST + 2 * BST_BYTES;              // 2 x omap [TP]
constexpr size_t O_AOP = (O_OM + 2 * TP * 4 + 1023) & ~(size_t)1023;  // A' [ML][KC] K-major SW128
constexpr size_t O_ROP = O_AOP + (size_t)ML * KC * 4;       // Res'
constexpr size_t O_WOP = O_ROP + (size_t)ML * KC * 4;       // W'  [32 rows][ML lines] K-major SW128
constexpr int XF = 12;                                      // floats per position in the exchange (R <= 10, 16 B multiple)
constexpr size_t O_XIN = O_WOP + (size_t)32 * ML * 4;       // [2][CS src][32 own pos][XF] partials received
constexpr size_t O_XOUT = O_XIN + (size_t)2 * CS * 32 * XF * 4;  // [2][TP][XF] final factor values
constexpr size_t O_WS = O_XOUT + (size_t)2 * TP * XF * 4;  // per-warp (den, res) doubles
constexpr size_t O_LOFF = O_WS + (size_t)NW * 2 * 8;        // line offsets (int64) [2 strips][ML]
constexpr size_t O_BAR = O_LOFF + (size_t)2 * ML * 8;
constexpr int NBAR = 2 + 3 + 4 + 2 + 4;  // full[2], lfull ffull bfull, cready[4], bready fready, xin[2] xout[2]
constexpr size_t O_TBASE = O_BAR + NBAR * 8;
constexpr size_t SMEM = O_TBASE + 16 + 1024;                // + alignment slack
}  // namespace s5

__device__ __forceinline__ float s5_lo(float x) { return __fsub_rn(x, umma::tf32_hi(x)); }

// byte offset of element (row, k) in a K-major 128B-swizzled operand whose
// rows are 128 bytes (32 fp32 along K), 8-row atoms of 1 KB
__device__ __forceinline__ uint32_t s5_kmaj(int row, int k) {
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((((k >> 2) ^ (row & 7)) & 7) << 4) + (k & 3) * 4);
}
// W' (32 rows t' x ML lines along K): K atoms of 32 lines, 4 KB each
__device__ __forceinline__ uint32_t s5_wop(int tp, int line) {
  return (uint32_t)((line >> 5) * 4096) + s5_kmaj(tp, line & 31);
}

__device__ __forceinline__ void s5_ld32(uint32_t taddr, float* v) {
  umma::ld16(taddr, v);
  umma::ld16(taddr + 16, v + 16);
}
__device__ __forceinline__ void s5_st32(uint32_t taddr, const float* v) {
  umma::st16(taddr, v);
  umma::st16(taddr + 16, v + 16);
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t n_clusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
// 4 floats of a peer CTA's shared memory (the loads of a cluster_sync_all()
// protected buffer need no ordering among themselves: no memory clobber)
__device__ __forceinline__ float4 ld_cluster_v4(uint32_t local_saddr, uint32_t rank) {
  uint32_t remote;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_saddr), "r"(rank));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(remote));
  return v;
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ void st_cluster_v4(uint32_t local_saddr, uint32_t rank, float4 v) {
  uint32_t remote;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_saddr), "r"(rank));
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(remote), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
// arrive on a peer's (or this CTA's) mbarrier, releasing this thread's prior
// shared::cluster stores at cluster scope
__device__ __forceinline__ void arrive_cluster(uint64_t* local_bar, uint32_t rank) {
  uint32_t remote;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(umma::smem_u32(local_bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(umma::smem_u32(b)), "r"(parity)
        : "memory");
}

template <int R>
__global__ void __launch_bounds__(s5::NT, 1) strips5_kernel(const __grid_constant__ StripsArgs<float> a) {
  using namespace s5;
  if (*a.done) return;  // (stream-ordered: uniform across the cluster)
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = sm_raw + ((1024 - (umma::smem_u32(sm_raw) & 1023)) & 1023);
  float* Dt = reinterpret_cast<float*>(sm + O_D);
  float* Bst = reinterpret_cast<float*>(sm + O_BST);
  int* Om = reinterpret_cast<int*>(sm + O_OM);
  unsigned char* Aop = sm + O_AOP;
  unsigned char* Rop = sm + O_ROP;
  unsigned char* Wop = sm + O_WOP;
  float* Xin = reinterpret_cast<float*>(sm + O_XIN);
  float* Xout = reinterpret_cast<float*>(sm + O_XOUT);
  double* Ws = reinterpret_cast<double*>(sm + O_WS);
  int64_t* loff = reinterpret_cast<int64_t*>(sm + O_LOFF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + O_BAR);
  uint64_t* full = bars;          // [2] D tile landed (cp.async, 512 arrivals)
  uint64_t* lfull = bars + 2;     // MMA1 done
  uint64_t* ffull = bars + 3;     // MMA2 done
  uint64_t* bfull = bars + 4;     // MMA3 done
  uint64_t* cready = bars + 5;    // [4] c / c_lo of line group g in TMEM
  uint64_t* bready = bars + 9;    // B' in TMEM
  uint64_t* fready = bars + 10;   // -F' in TMEM
  uint64_t* xin = bars + 11;      // [2] partials of my positions from all ranks
  uint64_t* xout = bars + 13;     // [2] final values from all owners
  uint32_t* tbase = reinterpret_cast<uint32_t*>(sm + O_TBASE);

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t rank = cluster_rank();
  const int cid = (int)cluster_id_x(), ncl = (int)n_clusters_x();
  const bool issuer_warp = w == NW;
  if (issuer_warp) umma::tmem_alloc(tbase, TCOLS);
  if (tid == 0) {
    umma::bar_init(&full[0], NW * 32);
    umma::bar_init(&full[1], NW * 32);
    umma::bar_init(lfull, 1);
    umma::bar_init(ffull, 1);
    umma::bar_init(bfull, 1);
    for (int g = 0; g < 4; ++g) umma::bar_init(&cready[g], 4);
    umma::bar_init(bready, 4);
    umma::bar_init(fready, 4);
    for (int k = 0; k < 2; ++k) {
      umma::bar_init(&xin[k], CS * 32);
      umma::bar_init(&xout[k], CS * 32);
    }
    umma::bar_init_fence();
  }
  for (int e = tid; e < 2 * ML; e += NT) {  // element offsets of this CTA's line segments, both strips
    const int q = e / ML, li = e - q * ML;
    const StripDesc<float>& s = a.s[q];
    const int nk = s.nk, h = (nk + CS - 1) / CS, l0 = (int)rank * h;
    loff[e] = (s.tiles > 0 && li < h && l0 + li < nk) ? (int64_t)(s.lines[l0 + li] - s.line_off) * s.line_stride : 0;
  }
  umma::fence_before();
  __syncthreads();
  cluster_sync_all();  // every CTA's barriers are initialised before any remote arrive
  umma::fence_after();
  const uint32_t T = *tbase;

  const int tiles0 = a.s[0].tiles, total = tiles0 + a.s[1].tiles;
  auto strip_of = [&](int t) { return t < tiles0 ? 0 : 1; };
  // this CTA's lines of strip q: [l0, l0 + hl)
  auto line_range = [&](int q, int& l0, int& hl) {
    const int nk = a.s[q].nk;
    const int h = (nk + CS - 1) / CS;
    l0 = (int)rank * h;
    hl = nk - l0 < h ? nk - l0 : h;
    if (hl < 0) hl = 0;
  };
  // ---- cp.async loads of tile t into buffer b (elementwise warps)
  auto issue_loads = [&](int t, int b) {
    const int q = strip_of(t);
    const StripDesc<float>& s = a.s[q];
    const int x0 = (t - (q ? tiles0 : 0)) * TP;
    int l0, hl;
    line_range(q, l0, hl);
    float* dst = Dt + (size_t)b * ML * TP;
    const int nch = hl * (TP / 4);
    for (int e = tid; e < nch; e += NW * 32) {
      const int li = e >> 5, ch = e & 31;
      const int pos = x0 + ch * 4;
      const int rem = s.npos - pos;
      const int bytes = rem >= 4 ? 16 : (rem > 0 ? rem * 4 : 0);
      umma::cp_async16(dst + (size_t)li * TP + ch * 4, s.src + loff[q * ML + li] + (bytes ? pos : x0),
                       (uint32_t)bytes);
    }
    float* bdst = Bst + (size_t)b * RMAX * TP;
    for (int e = tid; e < R * (TP / 4); e += NW * 32) {
      const int tt = e >> 5, ch = e & 31;
      const int pos = x0 + ch * 4;
      const int rem = s.npos - pos;
      const int bytes = rem >= 4 ? 16 : (rem > 0 ? rem * 4 : 0);
      umma::cp_async16(bdst + (size_t)tt * TP + ch * 4, s.Bold + (int64_t)tt * s.ldb + (bytes ? pos : x0),
                       (uint32_t)bytes);
    }
    if (tid < TP / 4) {
      const int pos = x0 + tid * 4;
      const int rem = s.npos - pos;
      const int bytes = rem >= 4 ? 16 : (rem > 0 ? rem * 4 : 0);
      umma::cp_async16(Om + b * TP + tid * 4, s.omap + (bytes ? pos : x0), (uint32_t)bytes);
    }
    umma::cp_async_arrive(&full[b]);
  };
  // ---- per-strip operands: A', Res' (K-major rows [x_hi | x_lo | x_hi | 0]) and W'
  auto build_strip_ops = [&](int q) {
    const StripDesc<float>& s = a.s[q];
    int l0, hl;
    line_range(q, l0, hl);
    for (int e = tid; e < ML * KC; e += NW * 32) {
      const int li = e / KC, k = e - li * KC;
      float va = 0.f, vr = 0.f;
      if (li < hl && k < 3 * R) {
        const int tt = k % R, part = k / R;  // 0: hi, 1: lo, 2: hi
        const float xa = s.lineA[(int64_t)(l0 + li) * R + tt];
        const float xr = s.lineRes[(int64_t)(l0 + li) * R + tt];
        va = part == 1 ? s5_lo(xa) : umma::tf32_hi(xa);
        vr = part == 1 ? s5_lo(xr) : umma::tf32_hi(xr);
      }
      *reinterpret_cast<float*>(Aop + s5_kmaj(li, k)) = va;
      *reinterpret_cast<float*>(Rop + s5_kmaj(li, k)) = vr;
    }
    for (int e = tid; e < 32 * ML; e += NW * 32) {
      const int tp = e / ML, li = e - tp * ML;
      const int tt = tp & 15;
      float v = 0.f;
      if (li < hl && tt < R) {
        const float x = s.lineW[(int64_t)(l0 + li) * R + tt];
        v = tp < 16 ? umma::tf32_hi(x) : s5_lo(x);
      }
      *reinterpret_cast<float*>(Wop + s5_wop(tp, li)) = v;
    }
    umma::fence_async_smem();
  };

  const uint32_t idesc_r = umma::idesc_tf32(128, ML, 0, 0);
  const uint32_t idesc_f32 = umma::idesc_tf32(128, 32, 0, 0);
  const uint32_t idesc_f16 = umma::idesc_tf32(128, 16, 0, 0);
  const uint32_t a_op = umma::smem_u32(Aop), r_op = umma::smem_u32(Rop), w_op = umma::smem_u32(Wop);
  auto TL = [&](int i) { return TL0 + 128u * (uint32_t)(i & 1); };
  auto TB = [&](int i) { return TB0 + 32u * (uint32_t)(i & 1); };

  if (issuer_warp) {
    // ================= MMA issue (one thread), in tile order
    if (lane == 0) {
      int i = 0;
      for (int t = cid; t < total; t += ncl, ++i) {
        const uint32_t ph = (uint32_t)(i & 1);
        const int q = strip_of(t);
        int l0, hl;
        line_range(q, l0, hl);
        const int ng = (hl + 31) / 32;
        const bool fresh = i == 0 || strip_of(t - ncl) != q;
        const bool next_same = t + ncl < total && strip_of(t + ncl) == q;
        if (fresh) {  // MMA1 of t (otherwise issued during tile t - 1)
          umma::bar_wait(bready, ph);
          umma::fence_after();
          for (int k = 0; k < KC / 8; ++k)
            umma::mma_ts(T + TL(i), T + TB(i) + 8 * k, umma::smem_desc(a_op + 32 * k, 16, 1024, umma::kSwizzle128),
                         idesc_r, k > 0);
          umma::commit(lfull);
        }
        for (int g = 0; g < ng; ++g) {  // MMA2: F^T = c . [W_hi | W_lo] + c_lo . W_hi
          umma::bar_wait(&cready[g], ph);
          umma::fence_after();
          for (int k = 0; k < 4; ++k) {
            const uint64_t wd = umma::smem_desc(w_op + g * 4096 + 32 * k, 16, 1024, umma::kSwizzle128);
            umma::mma_ts(T + TF, T + TL(i) + 32 * g + 8 * k, wd, idesc_f32, (g | k) > 0);
            umma::mma_ts(T + TF, T + TC + 32 * g + 8 * k, wd, idesc_f16, true);
          }
        }
        umma::commit(ffull);
        if (next_same) {  // MMA1 of t + 1 into the other slot
          umma::bar_wait(bready, ph ^ 1u);
          umma::fence_after();
          for (int k = 0; k < KC / 8; ++k)
            umma::mma_ts(T + TL(i + 1), T + TB(i + 1) + 8 * k,
                         umma::smem_desc(a_op + 32 * k, 16, 1024, umma::kSwizzle128), idesc_r, k > 0);
          umma::commit(lfull);
        }
        // MMA3: r = c - F'.Res'^T accumulated onto c (F' stored negated)
        umma::bar_wait(fready, ph);
        umma::fence_after();
        for (int k = 0; k < KC / 8; ++k)
          umma::mma_ts(T + TL(i), T + TB(i) + 8 * k, umma::smem_desc(r_op + 32 * k, 16, 1024, umma::kSwizzle128),
                       idesc_r, true);
        umma::commit(bfull);
      }
    }
    __syncwarp();
  } else {
    // ================= elementwise warps
    const int q_ = w & 3, g_ = w >> 2;  // position quadrant (TMEM lanes), line group (TMEM columns)
    const int p = 32 * q_ + lane;        // position in the tile
    const uint32_t lane_off = (uint32_t)(32 * q_) << 16;
    // optional per-phase clock64 totals of thread 0 (ircur_set_profiling)
    const bool rec = a.dbg && blockIdx.x == 0 && tid == 0;
    long long tpc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tq = clock64();
#define S5PH(k) do { if (rec) { const long long _t = clock64(); tpc[k] += _t - tq; tq = _t; } } while (0)
    // B' = [B | B | B_lo | 0] of tile t (buffer b) into TB(i), group-0 warps
    auto build_bprime = [&](int i, int b) {
      const float* Bb = Bst + (size_t)b * RMAX * TP;
      float v[KC];
#pragma unroll
      for (int k = 0; k < KC; ++k) v[k] = 0.f;
#pragma unroll
      for (int tt = 0; tt < R; ++tt) {
        const float x = Bb[tt * TP + p];
        v[tt] = x;
        v[R + tt] = x;
        v[2 * R + tt] = s5_lo(x);
      }
      s5_st32(T + lane_off + TB(i), v);
      umma::st_wait();
      umma::fence_before();
      __syncwarp();
      if (lane == 0) umma::bar_arrive(bready);
    };
    // residual of tile i (TL(i) holds r after MMA3) and its per-tile sums
    float den_prev = 0.f;
    int t_prev = -1, q_prev = 0;
    auto phase_b = [&](int i, int t, int q, float den) {
      float res = 0.f;
      umma::bar_wait(bfull, (uint32_t)(i & 1));
      umma::fence_after();
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        float r[16];
        umma::ld16(T + lane_off + TL(i) + 32 * g_ + 16 * hh, r);
        umma::ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) res = __fmaf_rn(r[j], r[j], res);
      }
      umma::fence_before();
      const double dd = warp_sum((double)den), rd = warp_sum((double)res);
      if (lane == 0) {
        Ws[2 * w] = dd;
        Ws[2 * w + 1] = rd;
      }
      named_bar(1, NW * 32);  // all elementwise warps: residual of tile t done
      if (tid == 0) {
        double sd = 0.0, sr = 0.0;
        for (int ww = 0; ww < NW; ++ww) {
          sd += Ws[2 * ww];
          sr += Ws[2 * ww + 1];
        }
        double4 pr;
        pr.x = q ? 0.0 : sd;
        pr.y = q ? 0.0 : sr;
        pr.z = q ? sd : 0.0;
        pr.w = q ? sr : 0.0;
        *reinterpret_cast<double4*>(a.partials + 4 * ((size_t)t * CS + rank)) = pr;
      }
      named_bar(2, NW * 32);  // Ws read before the next tile's sums
    };

    if (cid < total) issue_loads(cid, 0);
    if (cid + ncl < total) issue_loads(cid + ncl, 1);
    int cur = -1;
    int i = 0;
    for (int t = cid; t < total; t += ncl, ++i) {
      const int b = i & 1;
      const uint32_t ph = (uint32_t)(i & 1);
      const int q = strip_of(t);
      const StripDesc<float>& s = a.s[q];
      const int x0 = (t - (q ? tiles0 : 0)) * TP;
      int l0, hl;
      line_range(q, l0, hl);
      const bool fresh = q != cur;
      const bool next_same = t + ncl < total && strip_of(t + ncl) == q;
      S5PH(7);
      if (fresh) {
        if (t_prev >= 0) {  // drain the previous strip's last tile before its operands are replaced
          phase_b(i - 1, t_prev, q_prev, den_prev);
          t_prev = -1;
        }
        build_strip_ops(q);
        named_bar(1, NW * 32);
        cur = q;
        umma::bar_wait(&full[b], (uint32_t)((i >> 1) & 1));
        if (g_ == 0) build_bprime(i, b);
      } else {
        umma::bar_wait(&full[b], (uint32_t)((i >> 1) & 1));
      }
      S5PH(0);
      const float* Db = Dt + (size_t)b * ML * TP;
      const bool inpos = x0 + p < s.npos;
      const int om = inpos ? Om[b * TP + p] : -1;
      // ---- Phase I/II (solver.py:375-382): l -> c in TMEM, c_lo beside it
      float den = 0.f;
      umma::bar_wait(lfull, ph);
      umma::fence_after();
      S5PH(1);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {  // 16 lines at a time (register pressure)
        const int c0 = 32 * g_ + 16 * hh;
        float l[16];
        umma::ld16(T + lane_off + TL(i) + c0, l);
        umma::ld_wait();
        float c[16], cl[16];
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          const int li = c0 + j;
          Pair<float> d, lp;
          d.v = make_float2(li < hl ? Db[(size_t)li * TP + p] : 0.f, li + 1 < hl ? Db[(size_t)(li + 1) * TP + p] : 0.f);
          lp.v = make_float2(l[j], l[j + 1]);
          const Pair<float> e = keep_pair(d, lp, a.zt);
          c[j] = li < hl ? e.v.x : 0.f;
          c[j + 1] = li + 1 < hl ? e.v.y : 0.f;
          den = __fmaf_rn(d.v.x, d.v.x, den);
          den = __fmaf_rn(d.v.y, d.v.y, den);
        }
        if (om >= 0) {  // I x J entries: the core's values (U = (D - S)(I, J))
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int li = c0 + j;
            if (li < hl) c[j] = (float)s.U[(int64_t)(l0 + li) * s.u_ls + (int64_t)om * s.u_ps];
          }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) cl[j] = s5_lo(c[j]);
        umma::st16(T + lane_off + TL(i) + c0, c);
        umma::st16(T + lane_off + TC + c0, cl);
      }
      umma::st_wait();
      umma::fence_before();
      __syncwarp();
      if (lane == 0) umma::bar_arrive(&cready[g_]);
      S5PH(2);
      // ---- residual of the previous tile (same strip)
      if (t_prev >= 0) phase_b(i - 1, t_prev, q_prev, den_prev);
      S5PH(3);
      // D buffer b is free once every warp is past Phase I/II of t (the
      // residual's barrier, or this one): tile t + 2 loads into it
      if (t_prev < 0) named_bar(1, NW * 32);
      if (t + 2 * ncl < total) issue_loads(t + 2 * ncl, b);
      if (g_ == 0) {
        // B' of the next tile (same strip): its MMA1 runs during this epilogue
        if (next_same) {
          umma::bar_wait(&full[b ^ 1], (uint32_t)(((i + 1) >> 1) & 1));
          build_bprime(i + 1, b ^ 1);
        }
        S5PH(4);
        // ---- factor epilogue: partials -> owner rank -> sum, override, write -> all ranks
        umma::bar_wait(ffull, ph);
        umma::fence_after();
        float v[32];
        s5_ld32(T + lane_off + TF, v);
        umma::ld_wait();
        float pf[XF];
#pragma unroll
        for (int k = 0; k < XF; ++k) pf[k] = (k < R && hl > 0) ? __fadd_rn(v[k], v[16 + k]) : 0.f;
        // my partial of position p -> rank q_ (the owner of positions 32 q_ ..), slot [rank]
        float* xin_slot = Xin + (((size_t)b * CS + rank) * 32 + lane) * XF;
#pragma unroll
        for (int k = 0; k < XF; k += 4)
          st_cluster_v4(umma::smem_u32(xin_slot + k), (uint32_t)q_, make_float4(pf[k], pf[k + 1], pf[k + 2], pf[k + 3]));
        arrive_cluster(&xin[b], (uint32_t)q_);
        S5PH(5);
        const uint32_t xph = (uint32_t)((i >> 1) & 1);  // xin/xout[b] complete every other tile
        if (q_ == (int)rank) {  // owner: the four partials in rank order, override, write, broadcast
          wait_cluster(&xin[b], xph);
          float f[XF];
#pragma unroll
          for (int k = 0; k < XF; ++k) f[k] = Xin[(((size_t)b * CS + 0) * 32 + lane) * XF + k];
#pragma unroll
          for (int rr = 1; rr < CS; ++rr)
#pragma unroll
            for (int k = 0; k < XF; ++k) f[k] = __fadd_rn(f[k], Xin[(((size_t)b * CS + rr) * 32 + lane) * XF + k]);
          if (om >= 0) {
#pragma unroll
            for (int k = 0; k < R; ++k) f[k] = s.otherF[(int64_t)om * R + k];
          }
          if (inpos) {
#pragma unroll
            for (int k = 0; k < R; ++k) s.Fnew[(int64_t)k * s.ldf + x0 + p] = f[k];
          }
          float* xo = Xout + ((size_t)b * TP + p) * XF;
          for (uint32_t rr = 0; rr < CS; ++rr) {
#pragma unroll
            for (int k = 0; k < XF; k += 4)
              st_cluster_v4(umma::smem_u32(xo + k), rr, make_float4(f[k], f[k + 1], f[k + 2], f[k + 3]));
            arrive_cluster(&xout[b], rr);
          }
        }
        // final values of my positions (owner rank q_) -> -F' = -[F | F | F_lo | 0]
        wait_cluster(&xout[b], xph);
        S5PH(6);
        {
          const float* xo = Xout + ((size_t)b * TP + p) * XF;
          float nv[KC];
#pragma unroll
          for (int k = 0; k < KC; ++k) nv[k] = 0.f;
#pragma unroll
          for (int tt = 0; tt < R; ++tt) {
            const float f = xo[tt];
            nv[tt] = -f;
            nv[R + tt] = -f;
            nv[2 * R + tt] = -s5_lo(f);
          }
          s5_st32(T + lane_off + TB(i), nv);
          umma::st_wait();
          umma::fence_before();
          __syncwarp();
          if (lane == 0) umma::bar_arrive(fready);
        }
      }
      den_prev = den;
      t_prev = t;
      q_prev = q;
    }
    if (t_prev >= 0) phase_b(i - 1, t_prev, q_prev, den_prev);
    if (rec)
      for (int k = 0; k < 8; ++k) a.dbg[k] += tpc[k];
#undef S5PH
  }
  __syncwarp();
  // no CTA leaves while a peer may still store into its shared memory or arrive on its barriers
  cluster_sync_all();
  umma::fence_after();
  if (issuer_warp) umma::tmem_free(T, TCOLS);
}

bool strips5_supported(const StripsArgs<float>& a, int R) {
  if (R > s5::RMAX) return false;
  for (int q = 0; q < 2; ++q) {
    const StripDesc<float>& s = a.s[q];
    if (s.tiles == 0) continue;
    if (!s.bulk_ok || s.mode != kStripFull || s.pos_stride != 1 || !s.U) return false;
    if (s.nk > s5::CS * s5::ML) return false;
    if (((uintptr_t)s.Bold & 15) || (s.ldb & 3) || ((uintptr_t)s.omap & 15)) return false;
  }
  return true;
}

cudaError_t launch_strips5(const StripsArgs<float>& a0, int R, int num_sms, int* ncta_out, cudaStream_t st) {
  using namespace s5;
  if (ncta_out) *ncta_out = 0;
  if (!strips5_supported(a0, R)) return cudaErrorNotSupported;
  StripsArgs<float> a = a0;
  for (int q = 0; q < 2; ++q)
    if (a.s[q].tiles > 0) a.s[q].tiles = (a.s[q].npos + TP - 1) / TP;
  const int tiles = a.s[0].tiles + a.s[1].tiles;
  if (tiles == 0) return cudaSuccess;
  const int ncl = std::max(1, std::min(tiles, num_sms / CS));
  cudaError_t e = cudaErrorInvalidValue;
  auto launch = [&](auto kern) {
    static std::atomic<unsigned long long> devs{0};  // once per device (per rank instantiation)
    (void)devs;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(ncl * CS), 1, 1);
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = CS;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
  };
  static std::atomic<unsigned long long> devs[RMAX + 1];
  switch (R) {
#define S5_CASE(RR)                                                                           \
  case RR: {                                                                                  \
    const cudaError_t attr = smem_attr_once(devs[RR], strips5_kernel<RR>, (int)SMEM);         \
    if (attr != cudaSuccess) return attr;                                                     \
    e = launch(strips5_kernel<RR>);                                                           \
  } break;
    S5_CASE(1) S5_CASE(2) S5_CASE(3) S5_CASE(4) S5_CASE(5) S5_CASE(6) S5_CASE(7) S5_CASE(8) S5_CASE(9) S5_CASE(10)
#undef S5_CASE
    default: return cudaErrorNotSupported;
  }
  if (e == cudaSuccess && ncta_out) *ncta_out = tiles * CS;  // partial slots: one per (tile, rank)
  return e;
}

}  // namespace ircur
