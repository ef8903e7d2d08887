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
// numpy reports, and replaces np.unique's sort with a bitmap over [0, n).
// Checked against numpy in tests/test_host_logic.py.
#include <stdint.h>

#include <cstring>
#include <string>
#include <vector>

#include "../../include/ircur_b200.h"

namespace {

struct Pcg64 {
  unsigned __int128 state, inc;
  int has32;
  uint32_t u32;

  uint64_t next64() {
    const unsigned __int128 mult = ((unsigned __int128)2549297995355413924ull << 64) | 4865540595714422341ull;
    state = state * mult + inc;
    const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    const unsigned rot = (unsigned)(hi >> 58);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  uint32_t next32() {
    if (has32) {
      has32 = 0;
      return u32;
    }
    const uint64_t v = next64();
    has32 = 1;
    u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
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

// unique(integers(0, n, m)) into out (sorted); returns the count
int draw_unique(Pcg64& g, int64_t n, int m, std::vector<uint64_t>& bits, int64_t* out) {
  if (n == 1) {  // rng == 0: numpy fills zeros without drawing
    out[0] = 0;
    return 1;
  }
  const uint32_t rng = (uint32_t)(n - 1);
  for (int i = 0; i < m; ++i) {
    const uint32_t v = rng == 0xFFFFFFFFu ? g.next32() : g.bounded(rng);
    bits[v >> 6] |= 1ull << (v & 63);
  }
  int cnt = 0;
  const int64_t nw = (n + 63) >> 6;
  for (int64_t w = 0; w < nw; ++w) {
    uint64_t b = bits[w];
    if (!b) continue;
    bits[w] = 0;
    while (b) {
      out[cnt++] = (w << 6) + __builtin_ctzll(b);
      b &= b - 1;
    }
  }
  return cnt;
}

}  // namespace

extern "C" int ircur_draw_index_sets(const uint64_t* pcg, int64_t n1, int64_t n2, int m_rows, int m_cols,
                                     int n_sets, int64_t* rows, int32_t* row_counts, int64_t* cols,
                                     int32_t* col_counts, uint64_t* pcg_out) {
  if (!pcg || !rows || !cols || !row_counts || !col_counts || n_sets < 1 || m_rows < 1 || m_cols < 1 ||
      n1 < 1 || n2 < 1 || n1 > 0x100000000ll || n2 > 0x100000000ll)
    return IRCUR_EINVAL;
  Pcg64 g;
  g.state = ((unsigned __int128)pcg[1] << 64) | pcg[0];
  g.inc = ((unsigned __int128)pcg[3] << 64) | pcg[2];
  g.has32 = (int)pcg[4];
  g.u32 = (uint32_t)pcg[5];
  std::vector<uint64_t> b1((size_t)((n1 + 63) >> 6), 0ull), b2((size_t)((n2 + 63) >> 6), 0ull);
  for (int s = 0; s < n_sets; ++s) {
    row_counts[s] = draw_unique(g, n1, m_rows, b1, rows + (size_t)s * m_rows);
    col_counts[s] = draw_unique(g, n2, m_cols, b2, cols + (size_t)s * m_cols);
  }
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
