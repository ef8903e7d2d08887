// Host-side index draws of the reference, bit for bit (sampling.py:93-104).
//
// The reference draws I = unique(gen.integers(0, n1, m1)) then
// J = unique(gen.integers(0, n2, m2)) from one numpy Generator (PCG64) —
// before the loop and again at the top of every resampled iteration
// (solver.py:325-329, 362-364).  numpy's integers() for a range below 2^32
// is bounded 32-bit Lemire rejection on the bit generator's next_uint32,
// which splits each 64-bit PCG64 output into two 32-bit halves (low half
// first, the high half kept for the next call: the `has_uint32/uinteger`
// fields of the PCG64 state).  This reproduces that stream from the state
// numpy reports, and replaces np.unique's sort with a bitmap over [0, n)
// (dense draws) or an LSD radix sort (sparse draws).
// Checked against numpy in tests/test_host_logic.py.
#include <stdint.h>

#include <cstring>
#include <algorithm>
#include <cstdlib>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/ircur_b200.h"

namespace {

struct Pcg64 {
  unsigned __int128 state, inc;
  int has32;
  uint32_t u32;
  int64_t words = 0;  // 32-bit words handed out

  uint64_t next64() {
    const unsigned __int128 mult = ((unsigned __int128)2549297995355413924ull << 64) | 4865540595714422341ull;
    state = state * mult + inc;
    const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    const unsigned rot = (unsigned)(hi >> 58);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  uint32_t next32() {
    ++words;
    if (has32) {
      has32 = 0;
      return u32;
    }
    const uint64_t v = next64();
    has32 = 1;
    u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  // state after k more LCG steps (jump-ahead by squaring)
  void advance(uint64_t k) {
    const unsigned __int128 mult = ((unsigned __int128)2549297995355413924ull << 64) | 4865540595714422341ull;
    unsigned __int128 am = 1, ap = 0, cm = mult, cp = inc;
    while (k) {
      if (k & 1) {
        am *= cm;
        ap = ap * cm + cp;
      }
      cp = (cm + 1) * cp;
      cm *= cm;
      k >>= 1;
    }
    state = am * state + ap;
  }
  // the generator `w` 32-bit words after this one (this one unchanged)
  Pcg64 seek(int64_t w) const {
    Pcg64 g = *this;
    g.words = 0;
    if (w == 0) return g;
    if (g.has32) {  // the first word is the buffered high half
      g.has32 = 0;
      --w;
    }
    g.advance((uint64_t)(w / 2));
    if (w & 1) {
      const uint64_t v = g.next64();
      g.has32 = 1;
      g.u32 = (uint32_t)(v >> 32);
    }
    g.words = 0;
    return g;
  }
  // numpy's buffered_bounded_lemire_uint32: uniform on [0, rng]
  uint32_t bounded(uint32_t rng) {
    const uint32_t excl = rng + 1u;
    uint64_t m = (uint64_t)next32() * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t thr = (uint32_t)(0xFFFFFFFFu - rng) % excl;
      while (left < thr) {
        m = (uint64_t)next32() * excl;
        left = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
};

// Scratch of one draw_unique call.
struct Scratch {
  std::vector<uint64_t> bits;  // bitmap over [0, n) (dense draws)
  std::vector<uint32_t> a, b;  // radix-sort buffers (sparse draws)
  std::vector<uint32_t> hist;
};

// unique(integers(0, n, m)) into out (sorted); returns the count.  Sparse
// draws (the bitmap scan would touch mostly empty words, one unpredictable
// branch each) are LSD radix sorted instead, with at most 11-bit digits,
// and deduplicated in one pass.
int draw_unique(Pcg64& g, int64_t n, int m, Scratch& sc, int64_t* out) {
  if (n == 1) {  // rng == 0: numpy fills zeros without drawing
    out[0] = 0;
    return 1;
  }
  const uint32_t rng = (uint32_t)(n - 1);
  const int64_t nw = (n + 63) >> 6;
  const int nbits = 64 - __builtin_clzll((uint64_t)rng);
  const int passes = (nbits + 10) / 11;
  const int dbits = (nbits + passes - 1) / passes;
  if ((int64_t)passes * (2 * (int64_t)m + (1 << dbits)) < 2 * nw) {  // sort cheaper than the scan
    uint32_t* a = sc.a.data();
    uint32_t* b = sc.b.data();
    for (int i = 0; i < m; ++i) a[i] = rng == 0xFFFFFFFFu ? g.next32() : g.bounded(rng);
    const uint32_t nb = 1u << dbits, mask = nb - 1;
    uint32_t* h = sc.hist.data();
    for (int p = 0, sh = 0; p < passes; ++p, sh += dbits) {
      std::memset(h, 0, nb * sizeof(uint32_t));
      for (int i = 0; i < m; ++i) ++h[(a[i] >> sh) & mask];
      uint32_t run = 0;
      for (uint32_t d = 0; d < nb; ++d) {
        const uint32_t c = h[d];
        h[d] = run;
        run += c;
      }
      for (int i = 0; i < m; ++i) b[h[(a[i] >> sh) & mask]++] = a[i];
      std::swap(a, b);
    }
    int cnt = 0;
    uint32_t prev = 0;
    for (int i = 0; i < m; ++i) {
      const uint32_t v = a[i];
      out[cnt] = v;
      cnt += (cnt == 0) | (v != prev);
      prev = v;
    }
    return cnt;
  }
  std::vector<uint64_t>& bits = sc.bits;
  if ((int64_t)bits.size() < nw) bits.assign((size_t)nw, 0ull);
  for (int i = 0; i < m; ++i) {
    const uint32_t v = rng == 0xFFFFFFFFu ? g.next32() : g.bounded(rng);
    bits[v >> 6] |= 1ull << (v & 63);
  }
  int cnt = 0;
  for (int64_t w = 0; w < nw; ++w) {
    uint64_t bw = bits[w];
    if (!bw) continue;
    bits[w] = 0;
    while (bw) {
      out[cnt++] = (w << 6) + __builtin_ctzll(bw);
      bw &= bw - 1;
    }
  }
  return cnt;
}

// Threads for n_sets draws: ~6 sets (~30 us) per thread at least; env
// IRCUR_DRAW_THREADS overrides (1 = sequential).
thread_local int tls_draw_threads = 0;  // ircur::set_draw_threads_for_thread

int draw_threads(int n_sets) {
  if (tls_draw_threads > 0) return std::max(1, std::min(tls_draw_threads, n_sets));
  static const int forced = [] {
    const char* e = std::getenv("IRCUR_DRAW_THREADS");
    return e ? std::atoi(e) : 0;
  }();
  int hw = (int)std::thread::hardware_concurrency();
  hw = hw < 1 ? 1 : (hw > 8 ? 8 : hw);
  int n = forced > 0 ? forced : std::min(hw, n_sets / 6);
  return std::max(1, std::min(n, n_sets));
}

}  // namespace

namespace ircur {
// callers that already run one problem per thread (ircur_batch_prepare_many)
// draw each problem's sets on the calling thread
void set_draw_threads_for_thread(int n) { tls_draw_threads = n; }
}  // namespace ircur

extern "C" int ircur_draw_index_sets(const uint64_t* pcg, int64_t n1, int64_t n2, int m_rows, int m_cols,
                                     int n_sets, int64_t* rows, int32_t* row_counts, int64_t* cols,
                                     int32_t* col_counts, uint64_t* pcg_out) {
  if (!pcg || !rows || !cols || !row_counts || !col_counts || n_sets < 1 || m_rows < 1 || m_cols < 1 ||
      n1 < 1 || n2 < 1 || n1 > 0x100000000ll || n2 > 0x100000000ll)
    return IRCUR_EINVAL;
  Pcg64 g0;
  g0.state = ((unsigned __int128)pcg[1] << 64) | pcg[0];
  g0.inc = ((unsigned __int128)pcg[3] << 64) | pcg[2];
  g0.has32 = (int)pcg[4];
  g0.u32 = (uint32_t)pcg[5];
  // Sets are drawn in chunks on several threads.  Chunk c starts at the
  // stream position it would have without Lemire rejections (one word per
  // draw, numpy draws nothing for n == 1); a rejection (probability
  // ~ (2^32 mod n) / 2^32 per draw) shifts every later chunk, which is then
  // redrawn from its true start.  The result is the sequential one.
  const int64_t per_set = (n1 > 1 ? m_rows : 0) + (n2 > 1 ? m_cols : 0);
  int nth = draw_threads(n_sets);
  const int per = (n_sets + nth - 1) / nth;
  nth = (n_sets + per - 1) / per;
  std::vector<int64_t> start(nth), used(nth, -1), want(nth);
  std::vector<Pcg64> end(nth);
  auto run_chunk = [&](int c) {
    Pcg64 g = g0.seek(start[c]);
    Scratch sc;
    const int mm = m_rows > m_cols ? m_rows : m_cols;
    sc.a.resize(mm);
    sc.b.resize(mm);
    sc.hist.resize(1u << 11);
    for (int s = c * per; s < std::min(n_sets, (c + 1) * per); ++s) {
      row_counts[s] = draw_unique(g, n1, m_rows, sc, rows + (size_t)s * m_rows);
      col_counts[s] = draw_unique(g, n2, m_cols, sc, cols + (size_t)s * m_cols);
    }
    used[c] = g.words;
    end[c] = g;
  };
  for (int c = 0; c < nth; ++c) start[c] = (int64_t)c * per * per_set;
  std::vector<int> todo(nth);
  for (int c = 0; c < nth; ++c) todo[c] = c;
  while (!todo.empty()) {
    if (todo.size() == 1) {
      run_chunk(todo[0]);
    } else {
      std::vector<std::thread> pool;
      for (size_t i = 1; i < todo.size(); ++i) pool.emplace_back(run_chunk, todo[i]);
      run_chunk(todo[0]);
      for (auto& t : pool) t.join();
    }
    todo.clear();
    int64_t pos = 0;
    for (int c = 0; c < nth; ++c) {
      if (start[c] != pos) {  // drawn from the wrong position: redo from the true one
        start[c] = pos;
        todo.push_back(c);
      }
      pos += used[c];  // (a redone chunk's length is re-checked on the next round)
    }
  }
  Pcg64 g = end[nth - 1];
  if (pcg_out) {
    pcg_out[0] = (uint64_t)g.state;
    pcg_out[1] = (uint64_t)(g.state >> 64);
    pcg_out[2] = (uint64_t)g.inc;
    pcg_out[3] = (uint64_t)(g.inc >> 64);
    pcg_out[4] = (uint64_t)g.has32;
    pcg_out[5] = (uint64_t)g.u32;
  }
  return IRCUR_OK;
}
