// K1 tile machinery shared by the stand-alone pyramid kernel (k1_rgb.cu) and
// the fused pipeline (pipe.cu): TMA/mbarrier helpers, L2-policy stores, the
// dp4a gray/box arithmetic and the per-thread 8x8 block of one 32x256 tile.
// Semantics: image.py:58-68 (gray), pyramid.py:17-62 (levels),
// threshold.py:25-28 (histograms); see k1_rgb.cu for the design notes.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace mtb {

constexpr int kK1Groups = 4;
constexpr int kK1GroupThreads = 128;
constexpr int kK1Threads = kK1Groups * kK1GroupThreads;
constexpr int kK1Stages = 2;
constexpr int kK1TileRows = 32;
constexpr int kK1TilePx = 256;
constexpr int kK1RowBytes = 3 * kK1TilePx;                 // 768
constexpr int kK1TileBytes = kK1TileRows * kK1RowBytes;    // 24 KB
constexpr int kHistStrideK1 = 32;   // must equal kHistStride in pyramid.cu

struct K1Args {
  const uint8_t* rgb;
  int64_t rgb_pitch, rgb_img_stride;
  int w, h;
  uint8_t* gray;
  int64_t gray_img_stride;
  int off[6], pitch[6];     // within-image byte offsets (image gray arena < 2 GB)
  int lw[6], lh[6];
  int nl;                 // levels produced (1..6)
  uint32_t* hist;         // histograms [img][level][bin * hist_bin]
  int64_t hist_img_stride;
  int hist_bin;           // u32 stride between bins (32: spread, 1: dense)
  int tiles_x, tiles_y;   // ceil(w/256) x ceil(h/32)
  int n_img;              // images of this launch (tiles are numbered image-major)
  int keep_gray;          // store gray with L2::evict_last (else evict_normal)
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// TMA 3-D tile copy (box 192 u32 x 32 rows x 1 image) -> this CTA's smem.
__device__ __forceinline__ void tma_tile(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                         unsigned long long* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_addr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void group_bar(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(kK1GroupThreads) : "memory");
}
// One histogram increment at a shared address (ATOMS.POPC.INC).
__device__ __forceinline__ void hinc(uint32_t addr) { asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory"); }

// Gray stores with an L2 policy (evict_last when a threshold pass follows).
__device__ __forceinline__ void st_gray8(uint8_t* p, uint32_t a, uint32_t b, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(a), "r"(b), "l"(policy) : "memory");
}
__device__ __forceinline__ void st_gray4(uint8_t* p, uint32_t a, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(a), "l"(policy) : "memory");
}
__device__ __forceinline__ void st_gray2(uint8_t* p, uint32_t a, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.u16 [%0], %1, %2;" ::"l"(p), "h"((unsigned short)a), "l"(policy) : "memory");
}
__device__ __forceinline__ void st_gray1(uint8_t* p, uint32_t a, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.u8 [%0], %1, %2;" ::"l"(p), "h"((unsigned short)a), "l"(policy) : "memory");
}

// Four gray values (dp4a sums, gray = byte 1) of the 4 pixels in words w0..w2
// ([R0 G0 B0 R1] [G1 B1 R2 G2] [B2 R3 G3 B3]); returns the packed gray word.
__device__ __forceinline__ uint32_t gray4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t (&s)[4]) {
  s[0] = __dp4a(w0, 0x0013B736u, 0u);
  s[1] = __dp4a(w1, 0x000013B7u, __dp4a(w0, 0x36000000u, 0u));
  s[2] = __dp4a(w2, 0x00000013u, __dp4a(w1, 0xB7360000u, 0u));
  s[3] = __dp4a(w2, 0x13B73600u, 0u);
  const uint32_t g01 = __byte_perm(s[0], s[1], 0x0051);
  const uint32_t g23 = __byte_perm(s[2], s[3], 0x0051);
  return __byte_perm(g01, g23, 0x5410);
}
// 2x2 box sum + 2 of the byte pair `pair` (0: bytes 0-1, 1: bytes 2-3) of a
// word of the upper row u and of the lower row d: (a+b+c+d+2), < 1024.  The
// average is sum >> 2 and its histogram byte offset is sum & 0x3fc.
__device__ __forceinline__ uint32_t box_sum(uint32_t u, uint32_t d, int pair) {
  const uint32_t w = pair ? 0x01010000u : 0x00000101u;
  return __dp4a(u, w, __dp4a(d, w, 2u));
}

// One 32x256 tile of one group; this thread's 8x8 block starts at tile row
// 8*wg, tile column 8*lane.  v = its RGB bytes (row r: words v[r][0..2]).
template <bool FULL>
__device__ __forceinline__ void k1_block(const K1Args& a, uint8_t* gray, const uint2 (&v)[8][3], int tx, int ty,
                                         int wg, int lane, uint32_t hb, uint64_t policy, uint8_t* l3_slot) {
  const int x0 = tx * kK1TilePx + 8 * lane;
  const int y0 = ty * kK1TileRows + 8 * wg;
  // ---- level 0 (8 rows x 8 px) and level 1 (4 rows x 4 px) ---------------
  uint32_t l1[4];
  {
    uint8_t* p0 = gray + (a.off[0] + y0 * a.pitch[0] + x0);
    uint8_t* p1 = gray + (a.off[1] + (y0 >> 1) * a.pitch[1] + (x0 >> 1));
    const bool col0 = FULL || x0 < a.pitch[0];
    const int nv0 = FULL ? 8 : min(8, max(0, a.w - x0));
    const int x1 = x0 >> 1;
    const int nv1 = FULL ? 4 : min(4, max(0, a.lw[1] - x1));
#pragma unroll
    for (int rp = 0; rp < 4; ++rp) {
      uint32_t gw[2][2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = 2 * rp + j;
        const bool row_ok = FULL || (y0 + r < a.h);
        uint32_t sa[4], sb[4];
        gw[j][0] = gray4(v[r][0].x, v[r][0].y, v[r][1].x, sa);
        gw[j][1] = gray4(v[r][1].y, v[r][2].x, v[r][2].y, sb);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (FULL || (row_ok && i < nv0)) hinc(hb | ((sa[i] >> 6) & 0x3fcu));
          if (FULL || (row_ok && 4 + i < nv0)) hinc(hb | ((sb[i] >> 6) & 0x3fcu));
        }
        if (row_ok && col0) st_gray8(p0 + r * a.pitch[0], gw[j][0], gw[j][1], policy);
      }
      if (a.nl >= 2) {
        const uint32_t s0 = box_sum(gw[0][0], gw[1][0], 0), s1 = box_sum(gw[0][0], gw[1][0], 1);
        const uint32_t s2 = box_sum(gw[0][1], gw[1][1], 0), s3 = box_sum(gw[0][1], gw[1][1], 1);
        const uint32_t hb1 = hb + 1024;
        const bool row_ok = FULL || ((y0 >> 1) + rp < a.lh[1]);
        if (FULL || (row_ok && 0 < nv1)) hinc(hb1 | (s0 & 0x3fcu));
        if (FULL || (row_ok && 1 < nv1)) hinc(hb1 | (s1 & 0x3fcu));
        if (FULL || (row_ok && 2 < nv1)) hinc(hb1 | (s2 & 0x3fcu));
        if (FULL || (row_ok && 3 < nv1)) hinc(hb1 | (s3 & 0x3fcu));
        const uint32_t x01 = (s0 + (s1 << 16)) >> 2, x23 = (s2 + (s3 << 16)) >> 2;
        l1[rp] = __byte_perm(x01, x23, 0x6420);
        if (row_ok && (FULL || x1 < a.pitch[1])) st_gray4(p1 + rp * a.pitch[1], l1[rp], policy);
      }
    }
  }
  if (a.nl < 3) return;
  // ---- level 2 (2 rows x 2 px) --------------------------------------------
  uint32_t l2[2];
  {
    const int x2 = x0 >> 2, y2 = y0 >> 2;
    const int nv2 = FULL ? 2 : min(2, max(0, a.lw[2] - x2));
    uint8_t* p2 = gray + (a.off[2] + y2 * a.pitch[2] + x2);
    const uint32_t hb2 = hb + 2048;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const uint32_t s0 = box_sum(l1[2 * r], l1[2 * r + 1], 0), s1 = box_sum(l1[2 * r], l1[2 * r + 1], 1);
      const bool row_ok = FULL || (y2 + r < a.lh[2]);
      if (FULL || (row_ok && 0 < nv2)) hinc(hb2 | (s0 & 0x3fcu));
      if (FULL || (row_ok && 1 < nv2)) hinc(hb2 | (s1 & 0x3fcu));
      l2[r] = ((s0 >> 2) & 0xffu) | ((s1 << 6) & 0xff00u);
      if (row_ok && (FULL || x2 < a.pitch[2])) st_gray2(p2 + r * a.pitch[2], l2[r], policy);
    }
  }
  if (a.nl < 4) return;
  // ---- level 3 (1 px) -----------------------------------------------------
  {
    const int x3 = x0 >> 3, y3 = y0 >> 3;
    const uint32_t s = box_sum(l2[0], l2[1], 0);
    const uint32_t v3 = s >> 2;
    *l3_slot = (uint8_t)v3;
    if (FULL || (x3 < a.lw[3] && y3 < a.lh[3])) {
      hinc((hb + 3072) | (s & 0x3fcu));
      st_gray1(gray + (a.off[3] + y3 * a.pitch[3] + x3), v3, policy);
    }
  }
}

// Levels 4 (2 x 16 px) and 5 (1 x 8 px) of tile (tx, ty) from its level-3
// values l3[4][32]; executed by one whole warp.
__device__ __forceinline__ void k1_levels45(const K1Args& a, uint8_t* gray, const uint8_t (*l3)[32], int tx, int ty,
                                            int lane, uint32_t hb, bool full, uint64_t policy) {
  const int r = lane >> 4, c = lane & 15;
  const uint32_t v4 = (l3[2 * r][2 * c] + l3[2 * r][2 * c + 1] + l3[2 * r + 1][2 * c] + l3[2 * r + 1][2 * c + 1] + 2u) >> 2;
  {
    const int y = ty * 2 + r, x = tx * 16 + c;
    if (full || (y < a.lh[4] && x < a.lw[4])) {
      st_gray1(gray + (a.off[4] + y * a.pitch[4] + x), v4, policy);
      hinc((hb + 4096) | (v4 << 2));
    }
  }
  if (a.nl < 6) return;
  const int c5 = lane & 7;
  const uint32_t q0 = __shfl_sync(0xffffffffu, v4, 2 * c5), q1 = __shfl_sync(0xffffffffu, v4, 2 * c5 + 1);
  const uint32_t q2 = __shfl_sync(0xffffffffu, v4, 16 + 2 * c5), q3 = __shfl_sync(0xffffffffu, v4, 17 + 2 * c5);
  if (lane < 8) {
    const uint32_t v5 = (q0 + q1 + q2 + q3 + 2u) >> 2;
    const int y = ty, x = tx * 8 + lane;
    if (full || (y < a.lh[5] && x < a.lw[5])) {
      st_gray1(gray + (a.off[5] + y * a.pitch[5] + x), v5, policy);
      hinc((hb + 5120) | (v5 << 2));
    }
  }
}


// ---------------------------------------------------------------------------
// Tile-major gray layout (the fused pipeline's private L2-resident slots):
// tile t = ty * tiles_x + tx owns kTileGrayBytes contiguous bytes holding its
// levels 0..5 as dense row-major blocks with compile-time row strides, so
// every gray store is [base + immediate].
// L0 32x256, L1 16x128, L2 8x64, L3 4x32, L4 2x16, L5 1x8
__host__ __device__ constexpr int tm_off(int k) {
  return k == 0 ? 0 : k == 1 ? 8192 : k == 2 ? 10240 : k == 3 ? 10752 : k == 4 ? 10880 : 10912;
}
__host__ __device__ constexpr int tm_pitch(int k) { return 256 >> k; }
constexpr int kTileGrayBytes = 11008;                                // 86 x 128 B

// Tile-major gray stores with an L2::evict_last policy (the gray is read
// back one launch later).
__device__ __forceinline__ void st8(uint8_t* p, uint32_t a, uint32_t b, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(a), "r"(b), "l"(pol) : "memory");
}

// Shared-memory variant of st8 (SMEM tile-major slots, csrc/cluster.cu).
__device__ __forceinline__ void sts8(uint8_t* p, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(smem_addr(p)), "r"(a), "r"(b) : "memory");
}

// k1_block for the tile-major layout: `tg` = this tile's gray region (global,
// or shared memory when SMEM; l3_slot is unused then: level 3 is read back
// from tg).
template <bool FULL, bool SMEM = false>
__device__ __forceinline__ void k1_block_tm(const K1Args& a, uint8_t* tg, const uint2 (&v)[8][3], int tx, int ty,
                                            int wg, int lane, uint32_t hb, uint8_t* l3_slot, uint64_t gpol) {
  const int x0 = tx * kK1TilePx + 8 * lane;
  const int y0 = ty * kK1TileRows + 8 * wg;
  uint32_t l1[4];
  {
    uint8_t* p0 = tg + tm_off(0) + (8 * wg) * tm_pitch(0) + 8 * lane;
    const int nv0 = FULL ? 8 : min(8, max(0, a.w - x0));
    const int nv1 = FULL ? 4 : min(4, max(0, a.lw[1] - (x0 >> 1)));
#pragma unroll
    for (int rp = 0; rp < 4; ++rp) {
      uint32_t gw[2][2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = 2 * rp + j;
        const bool row_ok = FULL || (y0 + r < a.h);
        uint32_t sa[4], sb[4];
        gw[j][0] = gray4(v[r][0].x, v[r][0].y, v[r][1].x, sa);
        gw[j][1] = gray4(v[r][1].y, v[r][2].x, v[r][2].y, sb);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (FULL || (row_ok && i < nv0)) hinc(hb | ((sa[i] >> 6) & 0x3fcu));
          if (FULL || (row_ok && 4 + i < nv0)) hinc(hb | ((sb[i] >> 6) & 0x3fcu));
        }
        if constexpr (SMEM)
          sts8(p0 + r * tm_pitch(0), gw[j][0], gw[j][1]);
        else
          st8(p0 + r * tm_pitch(0), gw[j][0], gw[j][1], gpol);
      }
      if (a.nl >= 2) {
        const uint32_t s0 = box_sum(gw[0][0], gw[1][0], 0), s1 = box_sum(gw[0][0], gw[1][0], 1);
        const uint32_t s2 = box_sum(gw[0][1], gw[1][1], 0), s3 = box_sum(gw[0][1], gw[1][1], 1);
        const uint32_t hb1 = hb + 1024;
        const bool row_ok = FULL || ((y0 >> 1) + rp < a.lh[1]);
        if (FULL || (row_ok && 0 < nv1)) hinc(hb1 | (s0 & 0x3fcu));
        if (FULL || (row_ok && 1 < nv1)) hinc(hb1 | (s1 & 0x3fcu));
        if (FULL || (row_ok && 2 < nv1)) hinc(hb1 | (s2 & 0x3fcu));
        if (FULL || (row_ok && 3 < nv1)) hinc(hb1 | (s3 & 0x3fcu));
        const uint32_t x01 = (s0 + (s1 << 16)) >> 2, x23 = (s2 + (s3 << 16)) >> 2;
        l1[rp] = __byte_perm(x01, x23, 0x6420);
        if constexpr (SMEM)   // (the global layout re-derives level 1 from level 0 in K3)
          *reinterpret_cast<uint32_t*>(tg + tm_off(1) + (4 * wg + rp) * tm_pitch(1) + 4 * lane) = l1[rp];
      }
    }
  }
  if (a.nl < 3) return;
  uint32_t l2[2];
  {
    const int x2 = x0 >> 2, y2 = y0 >> 2;
    const int nv2 = FULL ? 2 : min(2, max(0, a.lw[2] - x2));
    uint8_t* p2 = tg + tm_off(2) + (2 * wg) * tm_pitch(2) + 2 * lane;
    const uint32_t hb2 = hb + 2048;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const uint32_t s0 = box_sum(l1[2 * r], l1[2 * r + 1], 0), s1 = box_sum(l1[2 * r], l1[2 * r + 1], 1);
      const bool row_ok = FULL || (y2 + r < a.lh[2]);
      if (FULL || (row_ok && 0 < nv2)) hinc(hb2 | (s0 & 0x3fcu));
      if (FULL || (row_ok && 1 < nv2)) hinc(hb2 | (s1 & 0x3fcu));
      l2[r] = ((s0 >> 2) & 0xffu) | ((s1 << 6) & 0xff00u);
      *reinterpret_cast<unsigned short*>(p2 + r * tm_pitch(2)) = (unsigned short)l2[r];
    }
  }
  if (a.nl < 4) return;
  {
    const int x3 = x0 >> 3, y3 = y0 >> 3;
    const uint32_t s = box_sum(l2[0], l2[1], 0);
    const uint32_t v3 = s >> 2;
    if constexpr (!SMEM) *l3_slot = (uint8_t)v3;
    tg[tm_off(3) + wg * tm_pitch(3) + lane] = (uint8_t)v3;
    if (FULL || (x3 < a.lw[3] && y3 < a.lh[3])) hinc((hb + 3072) | (s & 0x3fcu));
  }
}

// Levels 4 (2 x 16) and 5 (1 x 8) of one tile, tile-major stores; one warp.
__device__ __forceinline__ void k1_levels45_tm(const K1Args& a, uint8_t* tg, const uint8_t (*l3)[32], int tx, int ty,
                                               int lane, uint32_t hb, bool full) {
  const int r = lane >> 4, c = lane & 15;
  const uint32_t v4 = (l3[2 * r][2 * c] + l3[2 * r][2 * c + 1] + l3[2 * r + 1][2 * c] + l3[2 * r + 1][2 * c + 1] + 2u) >> 2;
  tg[tm_off(4) + r * tm_pitch(4) + c] = (uint8_t)v4;
  if (full || (ty * 2 + r < a.lh[4] && tx * 16 + c < a.lw[4])) hinc((hb + 4096) | (v4 << 2));
  if (a.nl < 6) return;
  const int c5 = lane & 7;
  const uint32_t q0 = __shfl_sync(0xffffffffu, v4, 2 * c5), q1 = __shfl_sync(0xffffffffu, v4, 2 * c5 + 1);
  const uint32_t q2 = __shfl_sync(0xffffffffu, v4, 16 + 2 * c5), q3 = __shfl_sync(0xffffffffu, v4, 17 + 2 * c5);
  if (lane < 8) {
    const uint32_t v5 = (q0 + q1 + q2 + q3 + 2u) >> 2;
    tg[tm_off(5) + lane] = (uint8_t)v5;
    if (full || (ty < a.lh[5] && tx * 8 + lane < a.lw[5])) hinc((hb + 5120) | (v5 << 2));
  }
}

}  // namespace mtb
