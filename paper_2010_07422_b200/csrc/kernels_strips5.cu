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

#ifndef S5_MMA3_FIRST
#define S5_MMA3_FIRST 0  // issuer polling order: MMA3 before MMA1 / MMA2
#endif
#ifndef S5_PROF_EPI
#define S5_PROF_EPI 0  // 1: the per-phase clock totals follow epilogue warp 0 instead of elementwise thread 0
#endif

namespace ircur {

namespace s5 {
constexpr int CS = 4;          // CTAs per cluster
constexpr int TP = 128;        // positions per tile (MMA M, TMEM lanes)
constexpr int ML = 128;        // TMEM columns / operand rows for the lines of one CTA
constexpr int HMAX = 116;      // lines per CTA (<= 464 sampled lines per strip)
constexpr int NEW = 16;        // elementwise warps: 4 per lane quadrant, 32 lines each
constexpr int NEP = 4;         // epilogue warps: one per lane quadrant
constexpr int NT = (NEW + NEP + 1) * 32;  // + the MMA-issuing warp
constexpr int KC = 32;         // concatenated K of the r-products
constexpr int RMAX = 10;       // 3 r <= KC
// TMEM columns (512): two slots by tile parity
constexpr uint32_t TL0 = 0, TC = 256, TB0 = 384, TF0 = 448, TCOLS = 512;
// shared memory (offsets from a 1 KB aligned base)
constexpr size_t D_BYTES = (size_t)HMAX * TP * 4;           // one D tile: [line][pos]
constexpr size_t O_D = 0;                                   // 2 D tiles
constexpr size_t O_AOP = (O_D + 2 * D_BYTES + 1023) & ~(size_t)1023;  // A' [ML][KC] K-major SW128
constexpr size_t O_ROP = O_AOP + (size_t)ML * KC * 4;       // Res'
constexpr size_t O_WOP = O_ROP + (size_t)ML * KC * 4;       // W'  [32 rows][ML lines] K-major SW128
constexpr size_t O_BP = O_WOP + (size_t)32 * ML * 4;        // B' [TP][KC] K-major SW128 (MMA1 A operand)
constexpr size_t O_BST = O_BP + (size_t)TP * KC * 4;        // 2 x Bold staging [RMAX][TP] (cp.async)
constexpr size_t O_OM = O_BST + 2 * (size_t)RMAX * TP * 4;  // 2 x omap [TP]
constexpr int XF = 12;                                      // floats per position in the exchange (R <= 10)
constexpr size_t O_XIN = O_OM + 2 * TP * 4;                 // [2][CS src][32 own pos][XF] partials received
constexpr size_t O_XOUT = O_XIN + (size_t)2 * CS * 32 * XF * 4;  // [2][TP][XF] final factor values
constexpr size_t O_WS = O_XOUT + (size_t)2 * TP * XF * 4;  // per-warp den (elementwise) / res (epilogue)
constexpr size_t O_LOFF = O_WS + (size_t)NEW * 2 * 8;       // line offsets (int64) [2 strips][ML]
constexpr size_t O_BAR = O_LOFF + (size_t)2 * ML * 8;
// per tile parity: full lfull ffull bfull bready fready rdone xin xout cready[4]; + opsready
constexpr int NB_PER = 13;
constexpr int NBAR = 2 * NB_PER + 1;
constexpr size_t O_TBASE = O_BAR + NBAR * 8;
constexpr size_t SMEM = O_TBASE + 16 + 1024;                // + alignment slack
static_assert(SMEM <= 227 * 1024, "strips5 shared memory");
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
// arrive without release semantics: a preceding fence_cluster() orders all of
// this thread's earlier stores (one fence for several destinations)
__device__ __forceinline__ void arrive_cluster_relaxed(uint64_t* local_bar, uint32_t rank) {
  uint32_t remote;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(umma::smem_u32(local_bar)), "r"(rank));
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void fence_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
// 16 bytes into a peer's (or this CTA's) shared memory; the bytes complete
// the transaction count of the peer's mbarrier (no fence, no separate arrive)
__device__ __forceinline__ void st_async_v4(uint32_t local_saddr, uint64_t* local_bar, uint32_t rank, float4 v) {
  uint32_t ra, rb;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_saddr), "r"(rank));
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(umma::smem_u32(local_bar)), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(ra),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(rb)
               : "memory");
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
  unsigned char* Aop = sm + O_AOP;
  unsigned char* Rop = sm + O_ROP;
  unsigned char* Wop = sm + O_WOP;
  unsigned char* Bp = sm + O_BP;
  float* Bst = reinterpret_cast<float*>(sm + O_BST);
  int* Om = reinterpret_cast<int*>(sm + O_OM);
  float* Xin = reinterpret_cast<float*>(sm + O_XIN);
  float* Xout = reinterpret_cast<float*>(sm + O_XOUT);
  double* Ws = reinterpret_cast<double*>(sm + O_WS);
  int64_t* loff = reinterpret_cast<int64_t*>(sm + O_LOFF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + O_BAR);
  // barriers of tile parity b: bar(b, k)
  auto bar = [&](int b, int k) { return bars + b * NB_PER + k; };
  constexpr int kFull = 0, kL = 1, kF = 2, kB = 3, kBready = 4, kFready = 5, kRdone = 6, kXin = 7, kXout = 8,
                kC = 9;  // kC + g: cready of line group g
  uint64_t* opsready = bars + 2 * NB_PER;
  uint32_t* tbase = reinterpret_cast<uint32_t*>(sm + O_TBASE);

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t rank = cluster_rank();
  const int cid = (int)cluster_id_x(), ncl = (int)n_clusters_x();
  const bool issuer_warp = w == NEW + NEP;
  if (issuer_warp) umma::tmem_alloc(tbase, TCOLS);
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      umma::bar_init(bar(b, kFull), NEW * 32);
      umma::bar_init(bar(b, kL), 1);
      umma::bar_init(bar(b, kF), 1);
      umma::bar_init(bar(b, kB), 1);
      umma::bar_init(bar(b, kBready), 4);
      umma::bar_init(bar(b, kFready), 4);
      umma::bar_init(bar(b, kRdone), NEP);
      umma::bar_init(bar(b, kXin), 1);   // armed by the owner warp: expect 4 ranks x 32 positions
      umma::bar_init(bar(b, kXout), 4);  // armed by each epilogue warp: its 32 positions
      for (int g = 0; g < 4; ++g) umma::bar_init(bar(b, kC + g), 4);
    }
    umma::bar_init(opsready, 1);
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
  const int ntl = cid < total ? (total - 1 - cid) / ncl + 1 : 0;  // this cluster's tiles
  auto tile_of = [&](int i) { return cid + i * ncl; };
  auto strip_of = [&](int t) { return t < tiles0 ? 0 : 1; };
  auto fresh_at = [&](int i) { return i == 0 || strip_of(tile_of(i)) != strip_of(tile_of(i - 1)); };
  auto line_range = [&](int q, int& l0, int& hl) {  // this CTA's lines of strip q: [l0, l0 + hl)
    const int nk = a.s[q].nk;
    const int h = (nk + CS - 1) / CS;
    l0 = (int)rank * h;
    hl = nk - l0 < h ? nk - l0 : h;
    if (hl < 0) hl = 0;
  };
  auto TL = [&](int i) { return TL0 + 128u * (uint32_t)(i & 1); };
  auto TB = [&](int i) { return TB0 + 32u * (uint32_t)(i & 1); };
  auto TF = [&](int i) { return TF0 + 32u * (uint32_t)(i & 1); };
  auto xph = [&](int i) { return (uint32_t)((i >> 1) & 1); };  // phase parity of tile i's barriers

  if (issuer_warp) {
    // ================= MMA issue (one thread): three in-order streams, polled
    //   MMA1(n1): B' built, TL slot free (residual of n1 - 2 read)
    //   MMA2(n2): line groups of c / c_lo written, after MMA1(n2), TF slot read (MMA3(n2 - 2) issued)
    //   MMA3(n3): -F' written, after MMA2(n3)
    if (lane == 0) {
      const uint32_t idesc_r = umma::idesc_tf32(128, ML, 0, 0);
      const uint32_t idesc_f32 = umma::idesc_tf32(128, 32, 0, 0);
      const uint32_t idesc_f16 = umma::idesc_tf32(128, 16, 0, 0);
      const uint32_t a_op = umma::smem_u32(Aop), r_op = umma::smem_u32(Rop), w_op = umma::smem_u32(Wop);
      const uint32_t bp0 = umma::smem_u32(Bp);
      int n1 = 0, n2 = 0, g2 = 0, n3 = 0, nfresh = 0;
      while (n3 < ntl) {
#if S5_MMA3_FIRST
        // MMA3 first: it is on the epilogue's path (the tensor pipe runs in issue order)
        if (n3 < n2 && umma::bar_try(bar(n3 & 1, kFready), xph(n3))) {
          umma::fence_after();
          const uint32_t r_base = r_op;
          for (int k = 0; k < KC / 8; ++k)  // r = c - F'.Res'^T accumulated onto c (F' stored negated)
            umma::mma_ts(T + TL(n3), T + TB(n3) + 8 * k, umma::smem_desc(r_base + 32 * k, 16, 1024, umma::kSwizzle128),
                         idesc_r, true);
          umma::commit(bar(n3 & 1, kB));
          ++n3;
          continue;
        }

#endif
        if (n1 < ntl && umma::bar_try(bar(n1 & 1, kBready), xph(n1)) &&
            (n1 < 2 || umma::bar_try(bar(n1 & 1, kRdone), xph(n1 - 2))) &&
            (!fresh_at(n1) || umma::bar_try(opsready, (uint32_t)(nfresh & 1)))) {
          if (fresh_at(n1)) ++nfresh;
          umma::fence_after();
          const uint32_t bpa = bp0;
          for (int k = 0; k < KC / 8; ++k)
            umma::mma_ss(T + TL(n1), umma::smem_desc(bpa + 32 * k, 16, 1024, umma::kSwizzle128),
                         umma::smem_desc(a_op + 32 * k, 16, 1024, umma::kSwizzle128), idesc_r, k > 0);
          umma::commit(bar(n1 & 1, kL));
          ++n1;
          continue;
        }
        if (n2 < n1 && n2 < n3 + 2) {
          int l0, hl;
          line_range(strip_of(tile_of(n2)), l0, hl);
          const int ng = (hl + 31) / 32;
          if (g2 < ng && umma::bar_try(bar(n2 & 1, kC + g2), xph(n2))) {
            umma::fence_after();
            for (int k = 0; k < 4; ++k) {
              const uint64_t wd = umma::smem_desc(w_op + g2 * 4096 + 32 * k, 16, 1024, umma::kSwizzle128);
              umma::mma_ts(T + TF(n2), T + TL(n2) + 32 * g2 + 8 * k, wd, idesc_f32, (g2 | k) > 0);
              umma::mma_ts(T + TF(n2), T + TC + 32 * g2 + 8 * k, wd, idesc_f16, true);
            }
            ++g2;
          }
          if (g2 >= ng) {
            umma::commit(bar(n2 & 1, kF));
            ++n2;
            g2 = 0;
            continue;
          }
        }
#if !S5_MMA3_FIRST
        if (n3 < n2 && umma::bar_try(bar(n3 & 1, kFready), xph(n3))) {
          umma::fence_after();
          const uint32_t r_base = r_op;
          for (int k = 0; k < KC / 8; ++k)  // r = c - F'.Res'^T accumulated onto c (F' stored negated)
            umma::mma_ts(T + TL(n3), T + TB(n3) + 8 * k, umma::smem_desc(r_base + 32 * k, 16, 1024, umma::kSwizzle128),
                         idesc_r, true);
          umma::commit(bar(n3 & 1, kB));
          ++n3;
          continue;
        }

#endif
      }
    }
    __syncwarp();
  } else if (w < NEW) {
    // ================= elementwise warps: loads, Phase I/II, residual
    const int q_ = w & 3, g_ = w >> 2;  // lane quadrant, line group (TMEM columns 32 g_ ..)
    const int p = 32 * q_ + lane;
    const uint32_t lane_off = (uint32_t)(32 * q_) << 16;
    const int et = tid;  // 0 .. NEW * 32 - 1
    const bool rec = a.dbg && blockIdx.x == 0 && tid == 0 && !S5_PROF_EPI;
    long long tpc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tq = clock64();
#define S5PH(k) do { if (rec) { const long long _t = clock64(); tpc[k] += _t - tq; tq = _t; } } while (0)
    // tile i into buffer i & 1: 16-byte cp.async per chunk, every elementwise
    // thread arrives on the buffer's barrier when its copies land.  (1-D bulk
    // copies of the 512-byte line segments were measured slower: the copy
    // engine takes ~70 cycles per copy, ~7 bytes/cycle per SM.)
    auto issue_loads = [&](int i) {
      const int t = tile_of(i), b = i & 1;
      const int q = strip_of(t);
      const StripDesc<float>& s = a.s[q];
      const int x0 = (t - (q ? tiles0 : 0)) * TP;
      int l0, hl;
      line_range(q, l0, hl);
      float* dst = Dt + (size_t)b * HMAX * TP;
      if (x0 + TP <= s.npos) {  // whole tile: fixed chunk per thread, lines 16 apart
        const int ch = et & 31;
        const float* src0 = s.src + x0 + ch * 4;
        float* dst0 = dst + ch * 4;
        for (int li = et >> 5; li < hl; li += NEW)
          umma::cp_async16(dst0 + (size_t)li * TP, src0 + loff[q * ML + li], 16u);
      } else {
        const int nch = hl * (TP / 4);
        for (int e = et; e < nch; e += NEW * 32) {
          const int li = e >> 5, ch = e & 31;
          const int pos = x0 + ch * 4;
          const int rem = s.npos - pos;
          const int bytes = rem >= 4 ? 16 : (rem > 0 ? rem * 4 : 0);
          umma::cp_async16(dst + (size_t)li * TP + ch * 4, s.src + loff[q * ML + li] + (bytes ? pos : x0),
                           (uint32_t)bytes);
        }
      }
      if (et < R * (TP / 4)) {  // the old factor's rows at these positions (for B')
        const int tt = et >> 5, ch = et & 31;
        const int pos = x0 + ch * 4;
        const int rem = s.npos - pos;
        const int bytes = rem >= 4 ? 16 : (rem > 0 ? rem * 4 : 0);
        umma::cp_async16(Bst + ((size_t)b * RMAX + tt) * TP + ch * 4, s.Bold + (int64_t)tt * s.ldb + (bytes ? pos : x0),
                         (uint32_t)bytes);
      } else if (et >= 480 && et < 480 + TP / 4) {
        const int c4 = et - 480;
        const int pos = x0 + c4 * 4;
        const int rem = s.npos - pos;
        const int bytes = rem >= 4 ? 16 : (rem > 0 ? rem * 4 : 0);
        umma::cp_async16(Om + b * TP + c4 * 4, s.omap + (bytes ? pos : x0), (uint32_t)bytes);
      }
      umma::cp_async_arrive(bar(b, kFull));
    };
    auto build_strip_ops = [&](int q) {  // A', Res' rows [x_hi | x_lo | x_hi | 0]; W' [W_hi ; W_lo]
      const StripDesc<float>& s = a.s[q];
      int l0, hl;
      line_range(q, l0, hl);
      for (int e = et; e < ML * KC; e += NEW * 32) {
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
      for (int e = et; e < 32 * ML; e += NEW * 32) {
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
    // B' = [B | B | B_lo | 0] of tile j (K-major SW128 row p), group-0 warps.
    // The slot is free: MMA1(j - 1) completed before Phase I/II of j - 1.
    auto build_bprime = [&](int j) {
      const int bj = j & 1;
      umma::bar_wait(bar(bj, kFull), xph(j));  // Bold rows of tile j landed
      const float* Bb = Bst + (size_t)bj * RMAX * TP;
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
#pragma unroll
      for (int c4 = 0; c4 < KC / 4; ++c4)
        *reinterpret_cast<float4*>(Bp + s5_kmaj(p, 4 * c4)) =
            make_float4(v[4 * c4], v[4 * c4 + 1], v[4 * c4 + 2], v[4 * c4 + 3]);
      umma::fence_async_smem();
      __syncwarp();
      if (lane == 0) umma::bar_arrive(bar(bj, kBready));
    };

    if (ntl > 0) issue_loads(0);
    if (ntl > 1) issue_loads(1);
    if (ntl > 0 && g_ == 0) build_bprime(0);
    int cur = -1;
    for (int i = 0; i < ntl; ++i) {
      const int t = tile_of(i), b = i & 1;
      const int q = strip_of(t);
      const StripDesc<float>& s = a.s[q];
      const int x0 = (t - (q ? tiles0 : 0)) * TP;
      int l0, hl;
      line_range(q, l0, hl);
      S5PH(7);
      if (q != cur) {  // new strip: once every MMA of the previous one completed, its operands
        if (i > 0) umma::bar_wait(bar((i - 1) & 1, kB), xph(i - 1));
        build_strip_ops(q);
        named_bar(1, NEW * 32);
        if (tid == 0) umma::bar_arrive(opsready);
        cur = q;
      }
      umma::bar_wait(bar(b, kFull), xph(i));
      S5PH(0);
      const float* Db = Dt + (size_t)b * HMAX * TP;
      // ---- Phase I/II (solver.py:375-382): l -> c in TMEM, c_lo beside it
      float den = 0.f;
      umma::bar_wait(bar(b, kL), xph(i));
      umma::fence_after();
      S5PH(1);
      {
        const int g = g_;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {  // 16 lines at a time (register pressure)
          const int c0 = 32 * g + 16 * hh;
          float l[16];
          umma::ld16(T + lane_off + TL(i) + c0, l);
          umma::ld_wait();
          float c[16], cl[16];
          if (hh == 0 && i > 0) umma::bar_wait(bar((i - 1) & 1, kF), xph(i - 1));  // MMA2(i - 1) read c_lo
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            const int li = c0 + j;
            Pair<float> d, lp;
            d.v = make_float2(li < hl ? Db[(size_t)li * TP + p] : 0.f,
                              li + 1 < hl ? Db[(size_t)(li + 1) * TP + p] : 0.f);
            lp.v = make_float2(l[j], l[j + 1]);
            const Pair<float> e = keep_pair(d, lp, a.zt);
            c[j] = li < hl ? e.v.x : 0.f;
            c[j + 1] = li + 1 < hl ? e.v.y : 0.f;
            den = __fmaf_rn(d.v.x, d.v.x, den);
            den = __fmaf_rn(d.v.y, d.v.y, den);
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) cl[j] = s5_lo(c[j]);
          umma::st16(T + lane_off + TL(i) + c0, c);
          umma::st16(T + lane_off + TC + c0, cl);
        }
        umma::st_wait();
        umma::fence_before();
        __syncwarp();
        if (lane == 0) umma::bar_arrive(bar(b, kC + g));
      }
      S5PH(2);
      // ---- den of tile i (per tile, warps in order); the barrier also frees D buffer b
      {
        const double dd = warp_sum((double)den);
        if (lane == 0) Ws[w] = dd;
        named_bar(1, NEW * 32);
        if (tid == 0) {
          double sd = 0.0;
          for (int ww = 0; ww < NEW; ++ww) sd += Ws[ww];
          double* pr = a.partials + 4 * ((size_t)t * CS + rank);
          pr[q ? 2 : 0] = sd;
          pr[q ? 0 : 2] = 0.0;
        }
      }
      S5PH(3);
      if (g_ == 0 && i + 1 < ntl) build_bprime(i + 1);  // (after thread 0 read Ws: MMA1(i + 1) gates the others)
      if (i + 2 < ntl) issue_loads(i + 2);
      S5PH(4);
    }
    if (rec)
      for (int k = 0; k < 8; ++k) a.dbg[k] += tpc[k];
#undef S5PH
  } else {
    // ================= epilogue warps (one per lane quadrant): B' of the next
    // tile, then the factor epilogue of this one
    const int q_ = w & 3;
    const int p = 32 * q_ + lane;
    const uint32_t lane_off = (uint32_t)(32 * q_) << 16;
    const bool rec = a.dbg && blockIdx.x == 0 && tid == NEW * 32 && S5_PROF_EPI;
    long long tpc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tq = clock64();
#define S5PE(k) do { if (rec) { const long long _t = clock64(); tpc[k] += _t - tq; tq = _t; } } while (0)
    constexpr uint32_t kXinBytes = CS * 32 * XF * 4, kXoutBytes = 32 * XF * 4;
    if (lane == 0)
      for (int bb = 0; bb < 2 && bb < ntl; ++bb) {
        if (q_ == (int)rank) umma::arrive_expect_tx(bar(bb, kXin), kXinBytes);
        umma::arrive_expect_tx(bar(bb, kXout), kXoutBytes);
      }
    double* Wse = Ws + NEW;  // epilogue warps' per-tile residual sums
    for (int i = 0; i < ntl; ++i) {
      const int t = tile_of(i), b = i & 1;
      const int q = strip_of(t);
      const StripDesc<float>& s = a.s[q];
      const int x0 = (t - (q ? tiles0 : 0)) * TP;
      const bool inpos = x0 + p < s.npos;
      int l0, hl;
      line_range(q, l0, hl);
      S5PE(7);
      // ---- factor epilogue: partials -> owner rank -> sum, override, write -> all ranks
      const int om = inpos ? s.omap[x0 + p] : -1;
      umma::bar_wait(bar(b, kF), xph(i));
      umma::fence_after();
      S5PE(1);
      float v[32];
      s5_ld32(T + lane_off + TF(i), v);
      umma::ld_wait();
      umma::fence_before();
      float pf[XF];
#pragma unroll
      for (int k = 0; k < XF; ++k) pf[k] = (k < R && hl > 0) ? __fadd_rn(v[k], v[16 + k]) : 0.f;
      float* xin_slot = Xin + (((size_t)b * CS + rank) * 32 + lane) * XF;
#pragma unroll
      for (int k = 0; k < XF; k += 4)
        st_async_v4(umma::smem_u32(xin_slot + k), bar(b, kXin), (uint32_t)q_,
                    make_float4(pf[k], pf[k + 1], pf[k + 2], pf[k + 3]));
      S5PE(2);
      if (q_ == (int)rank) {  // owner of positions 32 q_ ..: the four partials in rank order
        wait_cluster(bar(b, kXin), xph(i));
        S5PE(3);
        float f[XF];
        {
          float4 xv[CS][XF / 4];
#pragma unroll
          for (int rr = 0; rr < CS; ++rr)
#pragma unroll
            for (int k4 = 0; k4 < XF / 4; ++k4)
              xv[rr][k4] = *reinterpret_cast<const float4*>(Xin + (((size_t)b * CS + rr) * 32 + lane) * XF + 4 * k4);
#pragma unroll
          for (int k4 = 0; k4 < XF / 4; ++k4) {
            f[4 * k4] = xv[0][k4].x; f[4 * k4 + 1] = xv[0][k4].y; f[4 * k4 + 2] = xv[0][k4].z; f[4 * k4 + 3] = xv[0][k4].w;
          }
#pragma unroll
          for (int rr = 1; rr < CS; ++rr)  // rank order: ((P0 + P1) + P2) + P3
#pragma unroll
            for (int k4 = 0; k4 < XF / 4; ++k4) {
              f[4 * k4] = __fadd_rn(f[4 * k4], xv[rr][k4].x);
              f[4 * k4 + 1] = __fadd_rn(f[4 * k4 + 1], xv[rr][k4].y);
              f[4 * k4 + 2] = __fadd_rn(f[4 * k4 + 2], xv[rr][k4].z);
              f[4 * k4 + 3] = __fadd_rn(f[4 * k4 + 3], xv[rr][k4].w);
            }
        }
        __syncwarp();
        if (lane == 0 && i + 2 < ntl) umma::arrive_expect_tx(bar(b, kXin), kXinBytes);  // tile i + 2
        if (om >= 0) {
#pragma unroll
          for (int k = 0; k < R; ++k) f[k] = s.otherF[(int64_t)om * R + k];
        }
        float* xo = Xout + ((size_t)b * TP + p) * XF;
        for (uint32_t rr = 0; rr < CS; ++rr) {
#pragma unroll
          for (int k = 0; k < XF; k += 4)
            st_async_v4(umma::smem_u32(xo + k), bar(b, kXout), rr, make_float4(f[k], f[k + 1], f[k + 2], f[k + 3]));
        }
      }
      S5PE(4);
      wait_cluster(bar(b, kXout), xph(i));
      S5PE(5);
      // -F' = -[F | F | F_lo | 0] into TB(i), once MMA3(i - 2) read the slot
      if (i >= 2) umma::bar_wait(bar(b, kB), xph(i - 2));
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
        __syncwarp();
        if (lane == 0 && i + 2 < ntl) umma::arrive_expect_tx(bar(b, kXout), kXoutBytes);  // tile i + 2
        s5_st32(T + lane_off + TB(i), nv);
        umma::st_wait();
        umma::fence_before();
        __syncwarp();
        if (lane == 0) umma::bar_arrive(bar(b, kFready));
        if (q_ == (int)rank && inpos) {  // the new factor at the positions this rank owns
#pragma unroll
          for (int k = 0; k < R; ++k) s.Fnew[(int64_t)k * s.ldf + x0 + p] = xo[k];
        }
      }
      S5PE(6);
      // ---- residual r = c - Lnew of position p over this CTA's lines (solver.py:393-400)
      umma::bar_wait(bar(b, kB), xph(i));
      umma::fence_after();
      S5PE(0);
      float res = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < ML; c0 += 32) {
        if (c0 < hl) {
          float r[32];
          s5_ld32(T + lane_off + TL(i) + c0, r);
          umma::ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) res = __fmaf_rn(r[j], r[j], res);
        }
      }
      umma::fence_before();
      __syncwarp();
      if (lane == 0) umma::bar_arrive(bar(b, kRdone));  // TL(i) may be overwritten (MMA1 of i + 2)
      const double rd = warp_sum((double)res);
      if (lane == 0) Wse[q_] = rd;
      named_bar(3, NEP * 32);
      if (q_ == 0 && lane == 0) {
        const double sr = ((Wse[0] + Wse[1]) + Wse[2]) + Wse[3];
        double* pr = a.partials + 4 * ((size_t)t * CS + rank);
        pr[q ? 3 : 1] = sr;
        pr[q ? 1 : 3] = 0.0;
      }
      named_bar(4, NEP * 32);  // Wse read before the next tile's sums
    }
    if (rec)
      for (int k = 0; k < 8; ++k) a.dbg[k] += tpc[k];
#undef S5PE
  }
  __syncwarp();
  // no CTA leaves while a peer may still store into its shared memory or arrive on its barriers
  cluster_sync_all();
  umma::fence_after();
  if (issuer_warp) umma::tmem_free(T, TCOLS);
}

bool strips5_supported(const StripsArgs<float>& a, int R) {
  if (R > s5::RMAX || !a.tc_ok) return false;
  for (int q = 0; q < 2; ++q) {
    const StripDesc<float>& s = a.s[q];
    if (s.tiles == 0) continue;
    if (!s.bulk_ok || s.mode != kStripFull || s.pos_stride != 1 || !s.U) return false;
    if (s.nk > s5::CS * s5::HMAX) return false;
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
  // clusters: as many as fit at once beside whatever else holds SMs (the
  // overlapped loop leaves num_sms < the device's SMs for the SVD cluster);
  // 4-CTA clusters need 4 free SMs of one GPC, so the count is the device's
  // maximum of co-resident clusters less the GPC share the other work takes
  int dev = 0, dev_sms = num_sms;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, dev);
  static int max_active[64] = {0};
  int& mac = max_active[dev & 63];
  if (mac == 0) {
    cudaLaunchConfig_t qc = {};
    qc.gridDim = dim3((unsigned)(CS * (dev_sms / CS)), 1, 1);
    qc.blockDim = dim3(NT, 1, 1);
    qc.dynamicSmemBytes = SMEM;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = CS;
    qa[0].val.clusterDim.y = 1;
    qa[0].val.clusterDim.z = 1;
    qc.attrs = qa;
    qc.numAttrs = 1;
    static std::atomic<unsigned long long> qdevs{0};
    smem_attr_once(qdevs, strips5_kernel<1>, (int)SMEM);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, strips5_kernel<1>, &qc) != cudaSuccess || n <= 0) n = dev_sms / (CS + 1);
    cudaGetLastError();
    mac = n;
  }
  int ncl_cap = mac;
  if (num_sms < dev_sms) ncl_cap -= (dev_sms - num_sms + CS - 1) / CS + 1;
  if (const char* e = std::getenv("IRCUR_S5_CLUSTERS")) ncl_cap = std::atoi(e);  // tuning knob
  const int ncl = std::max(1, std::min(tiles, ncl_cap));
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
