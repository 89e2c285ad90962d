// SWAR threshold/pack helpers shared by threshold.cu and pipe.cu.
//   mtb bit       = g > median                         threshold.py:42-45
//   exclusion bit = |g - median| > tol  (no wrap)       threshold.py:48-56
#pragma once

#include "common.cuh"

namespace mtb {

// SWAR "x > c" for the four bytes of x at once (c a per-level constant):
// x > c  <=>  x + (255 - c) carries out of the byte.  With xl = x & 0x7f7f7f7f
// and yl = (255 - c) & 0x7f7f7f7f replicated, s = xl + yl never carries across
// bytes, and the byte carry-out is MAJ(x7, y7, s7) — one LOP3.  Result: bit 7
// of each byte (other bits are junk).
struct GtConst {
  uint32_t y;    // (255 - c) replicated in all four bytes
  uint32_t yl;   // y & 0x7f7f7f7f
};
__device__ __forceinline__ GtConst gt_const(int c) {
  c = c < 0 ? 0 : (c > 255 ? 255 : c);
  const uint32_t y = (uint32_t)(255 - c) * 0x01010101u;
  return {y, y & 0x7f7f7f7fu};
}
__device__ __forceinline__ uint32_t gt_bytes(uint32_t x, uint32_t xl, GtConst k) {
  const uint32_t s = xl + k.yl;
  return (x & k.y) | (x & s) | (k.y & s);  // majority -> one LOP3
}
// Bits 7,15,23,31 of m (others zero) -> bits 0..3 of the result, in order.
__device__ __forceinline__ uint32_t gather_msb(uint32_t m) { return (m * 0x00204081u) >> 28; }

// pack32 in SWAR form (about 4 instructions per pixel).  Bit-identical to
// pack32 for 0 <= median <= 255 and tol >= 0.
__device__ __forceinline__ void pack32_swar(const uint32_t (&g)[8], int valid, GtConst kmed, GtConst khi,
                                            GtConst klo, uint32_t lomask, uint32_t& mtb, uint32_t& eb) {
  constexpr uint32_t H = 0x80808080u;
  uint32_t m = 0, e = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t x = g[k], xl = x & 0x7f7f7f7fu;
    const uint32_t gm = gt_bytes(x, xl, kmed) & H;
    const uint32_t gh = gt_bytes(x, xl, khi) & H;
    const uint32_t gl = gt_bytes(x, xl, klo);                 // x > lo - 1, i.e. x >= lo
    const uint32_t ge = gh | (~gl & lomask);                  // x > hi  or  x < lo
    m |= gather_msb(gm) << (4 * k);
    e |= gather_msb(ge) << (4 * k);
  }
  const uint32_t keep = valid >= 32 ? 0xffffffffu : (valid <= 0 ? 0u : ((1u << valid) - 1u));
  mtb = m & keep;
  eb = e & keep;
}

}  // namespace mtb
