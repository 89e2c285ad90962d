// K1 (fast path): RGB8 -> gray -> 2x box pyramid (levels 0..5) -> per-level
// 256-bin histograms, one streaming pass over the RGB input.
//
// Reference semantics are those listed in pyramid.cu (image.py:58-68,
// pyramid.py:17-62, threshold.py:25-28).  This kernel is the roofline kernel
// of the whole path: it reads every RGB byte exactly once.  Design (sm_100a):
//
//  * One 512-thread CTA per SM, persistent over a contiguous band of the
//    32x256-pixel tiles of one image.  Four independent 128-thread groups
//    each own one tile at a time and synchronise only on their own named
//    barrier; each group streams its tiles through a 2-stage ring with ONE
//    TMA tensor copy per tile (24 KB, L2 evict-first: RGB is read once).
//  * A thread owns an 8x8 pixel block: it pulls its 192 RGB bytes into
//    registers first (24 conflict-free LDS.64), the group barrier frees the
//    ring stage and the refill is issued before any arithmetic, so each TMA
//    has a whole tile of work (about 2 tile-times) to land.
//  * Gray via IDP.4A: 4 pixels (12 bytes = 3 words) cost 6 dp4a + 3 byte
//    permutes.  Levels 1-3 of the block are thread-local (4x4, 2x2, 1x1;
//    box sums by dp4a), levels 4-5 of the tile by one rotating warp from a
//    128-byte level-3 buffer.
//  * Histograms: shared-memory atomics (ATOMS.POPC.INC aggregates equal bins
//    in a warp).  Each level's 1 KB histogram sits at a 1 KB-aligned shared
//    address, so a bin address is ONE LOP3 (base | (sum >> 6 & 0x3fc)) after
//    the shift.  CTA histograms are reduced across a thread-block cluster
//    through DSMEM, then one global RED per nonzero bin per cluster into a
//    128-B-strided ("spread") histogram.
//  * Gray levels are stored with an optional L2::evict_last policy so a
//    threshold pass that follows closely re-reads them from L2.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace cg = cooperative_groups;

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
  uint32_t* hist;         // spread histograms [img][level][bin * 32]
  int64_t hist_img_stride;
  int tiles_x, tiles_y;   // ceil(w/256) x ceil(h/32)
  int n_img;              // images of this launch (tiles are numbered image-major)
  int keep_gray;          // store gray with L2::evict_last (else evict_normal)
  int probe;              // diagnostics (MTB_K1_PROBE): 1 = stream tiles only, 2 = compute only (no TMA)
};

struct K1Smem {
  uint32_t hist[kK1Groups][6][256];                    // first: 1 KB-aligned levels, one set per group
  uint8_t rgb[kK1Groups][kK1Stages][kK1TileBytes];     // TMA rings
  uint8_t l3[kK1Groups][2][4][32];                     // level-3 tile values, by tile parity
  unsigned long long full[kK1Groups][kK1Stages];       // mbarriers of the ring stages
};
constexpr int kK1SmemBytes = (int)sizeof(K1Smem) + 1024;  // + alignment slack

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
#ifndef K1_EXP_NO_HIST
__device__ __forceinline__ void hinc(uint32_t addr) { asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory"); }
#else
__device__ __forceinline__ void hinc(uint32_t addr) { asm volatile("" ::"r"(addr)); }
#endif

// Gray stores with an L2 policy (evict_last when a threshold pass follows).
__device__ __forceinline__ void st_gray8(uint8_t* p, uint32_t a, uint32_t b, uint64_t policy) {
#ifdef K1_EXP_NO_STORE
  asm volatile("" ::"l"(p), "r"(a), "r"(b)); return;
#endif
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

__global__ void __launch_bounds__(kK1Threads, 1) k1_rgb_pyramid_kernel(K1Args a, const __grid_constant__ CUtensorMap rgb_map) {
  extern __shared__ __align__(128) uint8_t k1_smem_raw[];
  const uint32_t raw = smem_addr(k1_smem_raw);
  K1Smem& S = *reinterpret_cast<K1Smem*>(k1_smem_raw + ((1024u - (raw & 1023u)) & 1023u));

  const int tid = threadIdx.x;
  const int g = tid >> 7;             // group
  const int t = tid & 127;            // thread in group
  const int lane = tid & 31;
  const int wg = t >> 5;              // warp in group: tile rows 8wg..8wg+7
  // This group's histograms: level k at hb + 1024 k (1 KB aligned, so a bin
  // address is hb_k | 4*bin).
  uint32_t* gh_s = &S.hist[g][0][0];
  const uint32_t hb = smem_addr(gh_s);

  for (int i = t; i < 6 * 256; i += kK1GroupThreads) gh_s[i] = 0;
  if (t == 0) {
    for (int s = 0; s < kK1Stages; ++s) mbar_init(&S.full[g][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  uint64_t pol_first, pol_gray;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
  if (a.keep_gray)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_gray));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_gray));

  // Tiles are numbered image-major over the whole launch; this CTA owns a
  // contiguous range and its group g every 4th tile of it.
  const int tiles_img = a.tiles_x * a.tiles_y;
  const int64_t ntiles = (int64_t)tiles_img * a.n_img;
  const int t_begin = (int)((int64_t)blockIdx.x * ntiles / gridDim.x);
  const int t_end = (int)((int64_t)(blockIdx.x + 1) * ntiles / gridDim.x);

  auto coords = [&](int tile, int& img, int& ty, int& tx) {
    img = tile / tiles_img;
    const int r = tile - img * tiles_img;
    ty = r / a.tiles_x;
    tx = r - ty * a.tiles_x;
  };
  auto issue = [&](int tile, int stage) {
    int img, ty, tx;
    coords(tile, img, ty, tx);
    mbar_expect_tx(&S.full[g][stage], kK1TileBytes);
    tma_tile(S.rgb[g][stage], &rgb_map, (kK1RowBytes / 4) * tx, kK1TileRows * ty, img, &S.full[g][stage], pol_first);
  };
  // Flush this group's histograms of image `img` to the global spread
  // histograms and zero them (called by the whole group after a group barrier).
  auto flush = [&](int img) {
    uint32_t* gh = a.hist + img * a.hist_img_stride;
    for (int i = t; i < a.nl * 256; i += kK1GroupThreads) {
      const uint32_t c = gh_s[i];
      if (c) {
        atomicAdd(&gh[(int64_t)i * kHistStrideK1], c);
        gh_s[i] = 0;
      }
    }
  };
  if (t == 0 && a.probe != 2) {
    for (int s = 0; s < kK1Stages; ++s)
      if (t_begin + g + kK1Groups * s < t_end) issue(t_begin + g + kK1Groups * s, s);
  }

  int k = 0, pimg = -1, ptx = 0, pty = 0;
  bool pfull = true;
  uint8_t* gray = a.gray;
  for (int tile = t_begin + g; tile < t_end; tile += kK1Groups, ++k) {
    const int stage = k % kK1Stages;
    int img, ty, tx;
    coords(tile, img, ty, tx);
    const bool full = (ty * kK1TileRows + kK1TileRows <= a.h) && (tx * kK1TilePx + kK1TilePx <= a.w);
    // Pull this thread's 8x8-pixel RGB block into registers.
    uint2 v[8][3];
    if (a.probe != 2) mbar_wait(&S.full[g][stage], (uint32_t)(k / kK1Stages) & 1u);
    {
      const uint8_t* src = S.rgb[g][stage] + (8 * wg) * kK1RowBytes + 24 * lane;
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) v[r][c] = *reinterpret_cast<const uint2*>(src + r * kK1RowBytes + 8 * c);
    }
    group_bar(g);  // stage consumed by all 128 threads; l3 of tile k-1 complete
    if (t == 0 && a.probe != 2 && tile + kK1Groups * kK1Stages < t_end) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(tile + kK1Groups * kK1Stages, stage);
    }
    if (a.probe == 1) continue;
    if (k > 0 && a.nl >= 5 && wg == ((k - 1) & 3))
      k1_levels45(a, gray, S.l3[g][(k - 1) & 1], ptx, pty, lane, hb, pfull, pol_gray);
    if (img != pimg) {
      // First tile of a new image: the previous image's counts are complete
      // in this group (its level-4/5 tail was just done above).
      if (pimg >= 0) {
        group_bar(g);
        flush(pimg);
        group_bar(g);
      }
      gray = a.gray + img * a.gray_img_stride;
    }
    uint8_t* l3_slot = &S.l3[g][k & 1][wg][lane];
    if (full)
      k1_block<true>(a, gray, v, tx, ty, wg, lane, hb, pol_gray, l3_slot);
    else
      k1_block<false>(a, gray, v, tx, ty, wg, lane, hb, pol_gray, l3_slot);
    pimg = img;
    ptx = tx;
    pty = ty;
    pfull = full;
  }
  group_bar(g);
  if (a.probe != 1 && k > 0) {
    if (a.nl >= 5 && wg == ((k - 1) & 3)) k1_levels45(a, gray, S.l3[g][(k - 1) & 1], ptx, pty, lane, hb, pfull, pol_gray);
    group_bar(g);
    flush(pimg);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool k1_rgb_supported(int w, int64_t rgb_pitch, int64_t rgb_img_stride, const void* rgb) {
  return (3 * (int64_t)w) % 4 == 0 && (rgb_pitch & 15) == 0 && (rgb_img_stride & 15) == 0 &&
         ((uintptr_t)rgb & 15) == 0 && encode_tiled() != nullptr;
}

static int g_keep_gray = 0;   // set by mtb_set_gray_policy (capi.cu)
void k1_set_keep_gray(int v) { g_keep_gray = v; }

// Levels 0..min(n,6)-1 of n_img images in ONE persistent launch (one CTA per
// SM over the image-major tile sequence).
int launch_k1_rgb(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride, int n_img, const Plan& p,
                  uint8_t* gray, uint32_t* spread_hist, int64_t hist_img_stride, cudaStream_t st) {
  K1Args a{};
  a.rgb_pitch = rgb_pitch;
  a.rgb_img_stride = rgb_img_stride;
  a.w = p.lv[0].w;
  a.h = p.lv[0].h;
  a.gray_img_stride = p.gray_img_bytes;
  if (p.gray_img_bytes >= ((int64_t)1 << 31)) {
    set_error("k1: gray arena of one image exceeds 2 GB");
    return MTB_EINVAL;
  }
  a.nl = p.n < 6 ? p.n : 6;
  for (int k = 0; k < 6; ++k) {
    const int l = k < p.n ? k : p.n - 1;
    a.off[k] = (int)p.lv[l].gray_off;
    a.pitch[k] = (int)p.lv[l].gray_pitch;
    a.lw[k] = k < p.n ? p.lv[k].w : 0;
    a.lh[k] = k < p.n ? p.lv[k].h : 0;
  }
  a.hist_img_stride = hist_img_stride;
  a.keep_gray = g_keep_gray;
  {
    const char* pr = getenv("MTB_K1_PROBE");
    a.probe = pr ? atoi(pr) : 0;
  }
  a.tiles_x = (a.w + kK1TilePx - 1) / kK1TilePx;   // edge tiles included: TMA zero-fills outside the image
  a.tiles_y = (a.h + kK1TileRows - 1) / kK1TileRows;
  a.n_img = n_img;
  const int64_t ntiles = (int64_t)a.tiles_x * a.tiles_y * n_img;
  if (ntiles == 0) return MTB_OK;
  if (ntiles >= ((int64_t)1 << 31)) {
    set_error("k1: too many tiles in one launch");
    return MTB_EINVAL;
  }
  static bool attr_done = false;
  if (!attr_done) {
    MTB_CUDA(cudaFuncSetAttribute(k1_rgb_pyramid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kK1SmemBytes));
    attr_done = true;
  }
  int x = num_sms();
  if (x > (ntiles + kK1Groups - 1) / kK1Groups) x = (int)((ntiles + kK1Groups - 1) / kK1Groups);
  if (x < 1) x = 1;
  a.rgb = rgb;
  a.gray = gray;
  a.hist = spread_hist;
  CUtensorMap map;
  {
    const cuuint64_t dims[3] = {(cuuint64_t)(3 * (int64_t)a.w / 4), (cuuint64_t)a.h, (cuuint64_t)n_img};
    const cuuint64_t strides[2] = {(cuuint64_t)rgb_pitch, (cuuint64_t)rgb_img_stride};
    const cuuint32_t box[3] = {kK1RowBytes / 4, kK1TileRows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode_tiled()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, (void*)rgb, dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed for the RGB batch");
      return MTB_ECUDA;
    }
  }
  k1_rgb_pyramid_kernel<<<x, kK1Threads, kK1SmemBytes, st>>>(a, map);
  return check_launch("k1_rgb_pyramid_kernel");
}

}  // namespace mtb
