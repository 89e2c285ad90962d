// SWAR threshold/pack helpers shared by threshold.cu, pipe.cu and cluster.cu.
//   mtb bit       = g > median                         threshold.py:42-45
//   exclusion bit = |g - median| > tol  (no wrap)       threshold.py:48-56
#pragma once

#include "common.cuh"

namespace mtb {

// Per-level threshold constants of the VABSDIFF4 / carry-majority form.
struct ThConst {
  uint32_t med;     // median replicated in 4 bytes (VABSDIFF4 operand)
  uint32_t ym;      // (255 - median) replicated: x > median <=> x + ym carries out of the byte
  uint32_t yml;     // ym & 0x7f7f7f7f
  int med_lo;       // median <= 127 (ym bit 7 set): carry = (x | s) bit 7, else (x & s) bit 7
};

// Generic form (any median, any tolerance): full majority for both carries.
__device__ __forceinline__ void th_word(const uint32_t (&g)[8], const ThConst& c, uint32_t yt, uint32_t ytl,
                                        int valid, uint32_t& mw, uint32_t& ew) {
  constexpr uint32_t H = 0x80808080u, L7 = 0x7f7f7f7fu;
  uint32_t m = 0, e = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t x = g[k];
    const uint32_t s = (x & L7) + c.yml;
    const uint32_t gm = ((x & c.ym) | (x & s) | (c.ym & s)) & H;
    uint32_t d;
    asm("vabsdiff4.u32.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(c.med), "r"(0u));
    const uint32_t sd = (d & L7) + ytl;
    const uint32_t ge = ((d & yt) | (d & sd) | (yt & sd)) & H;
    m = (((gm * 0x00204081u) >> (28 - 4 * k)) & (0xfu << (4 * k))) | m;
    e = (((ge * 0x00204081u) >> (28 - 4 * k)) & (0xfu << (4 * k))) | e;
  }
  const uint32_t keep = valid >= 32 ? 0xffffffffu : (valid <= 0 ? 0u : ((1u << valid) - 1u));
  mw = m & keep;
  ew = e & keep;
}


// Bits of 32 gray pixels (8 words) -> MTB word and exclusion word.
//   mtb  : g > med               — byte carry-out of g + (255 - med), MAJ(x7, ym7, s7)
//   excl : |g - med| > tol       — d = VABSDIFF4(g, med); carry-out of d + (255 - tol)
// With the per-level bit 7 of the addend known, MAJ is one LOP3 that also
// masks bit 7; the four flags of a word are gathered by one multiply.
// MED_LO: bit 7 of (255 - median) is set, so the MTB carry MAJ(x7, 1, s7)
// is (x | s) bit 7 — one LOP3 with the mask; else MAJ(x7, 0, s7) = x & s.
// The exclusion compare assumes tol <= 127 (the carry is (d | sd) bit 7);
// larger tolerances take the generic majority form.
template <bool MED_LO, bool TOL_LO>
__device__ __forceinline__ void th_word_t(const uint32_t (&g)[8], const ThConst& c, uint32_t yt, uint32_t ytl,
                                          int valid, uint32_t& mw, uint32_t& ew) {
  constexpr uint32_t H = 0x80808080u, L7 = 0x7f7f7f7fu;
  // Gather: umulhi(flags, magic << 4) puts the 4 byte flags (bits 7,15,23,31)
  // in bits 0..3 of the high word (other terms land below bit 32 or at >= bit
  // 40); a funnel shift (nib:acc) >> 4 pushes them in from the top and drops
  // the garbage, so after 8 words word k's flags sit at bits 4k..4k+3.  One
  // FMA-pipe and one ALU-pipe op per word and map.
  // Two words per funnel shift: the odd word's nibble is gathered 4 bits
  // higher (magic << 8) and added by the IMAD.HI of the even word.
  constexpr uint32_t M4 = 0x00204081u << 4, M8 = 0x00204081u << 8;
  uint32_t m = 0, e = 0, pm = 0, pe = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t x = g[k];
    const uint32_t s = (x & L7) + c.yml;
    const uint32_t gm = MED_LO ? ((x | s) & H) : (x & s & H);       // byte carry-out of x + (255 - med)
    uint32_t d;
    asm("vabsdiff4.u32.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(c.med), "r"(0u));
    const uint32_t sd = (d & L7) + ytl;
    const uint32_t ge = TOL_LO ? ((d | sd) & H) : (((d & yt) | (d & sd) | (yt & sd)) & H);   // |x - med| > tol
    if ((k & 1) == 0) {
      pm = gm;
      pe = ge;
    } else {
      m = __funnelshift_r(m, __umulhi(pm, M4) + __umulhi(gm, M8), 8);
      e = __funnelshift_r(e, __umulhi(pe, M4) + __umulhi(ge, M8), 8);
    }
  }
  const uint32_t keep = valid >= 32 ? 0xffffffffu : (valid <= 0 ? 0u : ((1u << valid) - 1u));
  mw = m & keep;
  ew = e & keep;
}

}  // namespace mtb
