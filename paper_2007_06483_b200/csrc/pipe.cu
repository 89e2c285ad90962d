// The fused alignment pipeline: preprocess (K1 + medians + K3) and the
// coarse-to-fine search (K4) of a whole batch of exposure pairs, software-
// pipelined over persistent launches of B images each (B = 2 up to 64 MB of
// gray per image) so the gray pyramids stay in L2 as far as they fit.
//
// Reference path (bit-exact): pipeline.py:80-90 -> build_mtb_pyramid
// (image.py:58-68, pyramid.py:17-62, threshold.py:25-88) -> find_offset
// (search.py:53-95, kernels/_native.pyx:73-111).
//
// Launch j (one 512-thread CTA per SM; programmatic dependent launch, and
// every cross-launch dependency is an acquire/release flag, never a grid
// wait):
//   * warps 0-11 (3 groups of 4): K1 of images jB .. jB+B-1 — TMA tile
//     copies into a 2-stage ring per group, gray + levels 1-5 + per-image
//     histograms, gray stored tile-major into ring slot i % 3B (levels 0, 2-5;
//     level 1 is re-derived by K3); the CTA flushes its histograms and the
//     last CTA of an image publishes its medians (med_ready flag); then they
//     join the aux queue.
//   * warps 12-15 from the start, 0-11 once their tiles run out: this CTA's
//     static slice of the aux queue — search tiles of every (pair, level) due
//     in this launch (each waits for the previous level's decided flag; a
//     CTA's partial counts of an item are flushed when its last tile of the
//     item is done, the last CTA applies the search.py:67 key), then K3 of
//     the B images of launch j-1: levels 3 and 2 (gathered pieces), level 0
//     half tiles (one 4 KB TMA bulk copy each, level 1 derived from the staged
//     rows), levels 4-5, row padding; consumed gray lines are discarded.
//   * the CTA's end adds itself to each K3 image's done count (gates the
//     gray slot's reuse three launches on and the pair's first search level).
// HBM traffic per image is the RGB read, the packed maps and whatever gray
// the L2 cannot hold (measured in DESIGN.md 4.3).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

// Level-0 gray is stored with L2::evict_last (no persisting set-aside: it
// measured slower); the RGB stream is evict_first.
#include "k1_tile.cuh"
#include "swar.cuh"

namespace mtb {

constexpr int kPipeMaxLevels = 6;
constexpr int kPipeMaxItems = 96;
constexpr int kPipeImgs = 2;                  // images per launch (K1 part and K3 part)
constexpr int kPipeThreads = 512;     // 12 K1 warps + 4 aux warps
constexpr int kPipeCtasPerSm = 1;
constexpr int kPipeWarps = kPipeThreads / 32;
constexpr int kK3Units = 4;                     // K3 task = 4 x 32 bitmap words = 4 KB of gray
constexpr int kK3Words = 32 * kK3Units;
constexpr int kK3Bytes = 32 * kK3Words;
constexpr int kSRows = 8;                       // search tile: 8 output rows x 32 words

struct PipeItem {
  int pair;      // index into acc/errs/done
  int ref, tgt;  // image indices
  int level;
  int tile0;     // first search warp-tile of this item in this launch
};

struct PipeArgs {
  K1Args g;                          // K1 geometry; g.gray = slot base, g.gray_img_stride = slot stride
  int n;                             // pyramid levels (<= 6)
  int tol;
  int nw32[kPipeMaxLevels];          // u32 words per packed row
  int64_t bit_off32[kPipeMaxLevels]; // u32 word offset of level k in an image's map arena
  int th_units0[kPipeMaxLevels + 1]; // prefix of threshold units (rows x 32-word chunks) per level
  int th_cpr[kPipeMaxLevels];        // 32-word chunks per row
  uint32_t tx_magic;                 // t / tiles_x == umulhi(t, tx_magic) (tiles_x > 1)
  int th_pad_words;                  // levels 0..3 row-padding words not covered by tiles
  uint32_t* mtb;                     // map arenas, u32 view; image stride bit_img_words32
  uint32_t* excl;
  int64_t bit_img_words32;
  int32_t* medians;                  // [img][n]
  int32_t* acc;                      // [P][n][2]
  unsigned long long* errs;          // [P][n][9]
  uint32_t* done;                    // [P][n]
  uint32_t* ctr;                     // [launch] K1 tile counters (zeroed)
  uint32_t* med_ready;               // [img] 1 once the image's medians (and all its gray) are published
  uint32_t* k3_done;                 // [img] CTAs that finished thresholding the image
  const uint32_t* img_ready;         // [img] nonzero once the image's RGB is in HBM (streamed input), or null
  uint32_t* decided;                 // [P][n] 1 once the (pair, level) offset is published
  int n_launch;
  int j;                             // this launch's index
  int k1_img0, k1_cnt;               // images k1_img0 .. +k1_cnt-1 of the K1 part (k1_cnt may be 0)
  int gray_slots;                    // gray ring slots in use: 3 x images per launch
  uint8_t* k1_gray[kPipeImgs];       // ring slot of each K1 image of this launch (host-computed: no
  const uint8_t* th_gray[kPipeImgs]; //   integer modulo per tile / task), and of each K3 image
  int th_img0, th_cnt;               // images of the K3 part
  int n_items;
  int search_tiles;
  PipeItem items[kPipeMaxItems];
};

// Per-level threshold constants (threshold.py:42-56), in shared memory.

// Warp roles: warps 0..7 = two K1 groups streaming image j (never wait on
// earlier launches: the gray ring has 3 slots), warps 8..15 = the aux warps
// (K3 + search) which wait for launch j-1.
constexpr int kPK1Groups = 3;
constexpr int kPK1Warps = 4 * kPK1Groups;
constexpr int kPAuxWarps = kPipeWarps - kPK1Warps;
constexpr int kPStages = 2;
constexpr int kPGraySlots = 3 * kPipeImgs;    // gray ring capacity: written, being read, lagging readers
                                              // (3 x images per launch slots in use)
constexpr int kAuxPhases = 7;     // aux task phases: K3 levels 0..3, levels 4..5, padding, search

// Per-aux-warp staging of one search warp-tile: 8 output rows x 32 words of
// the reference maps, 10 source rows x 35 words of the target maps.
struct SearchStage {
  uint32_t a[kSRows][32], ea[kSRows][32];
  uint32_t b[kSRows + 2][36], eb[kSRows + 2][36];
};

struct PipeSmem {
  uint32_t hist[kPipeImgs][6][256];                       // per K1 image; 1 KB-aligned levels (k1_tile.cuh)
  uint8_t rgb[kPK1Groups][kPStages][kK1TileBytes];
  uint8_t abuf[kPAuxWarps > 0 ? kPAuxWarps : 1][2][kK3Bytes];                  // aux warps: K3 double buffer / search staging
  uint8_t l3[kPK1Groups][2][4][32];
  unsigned long long full[kPK1Groups][kPStages];
  int tile_of[kPK1Groups][kPStages];                      // tile in each ring stage (-1: no more)
  unsigned long long kbar[kPipeWarps][2];                 // per-warp K3 staging mbarriers
  ThConst th[kPipeImgs][kPipeMaxLevels];                 // threshold constants of the K3 images
  int pt1[kAuxPhases];                                    // one image's task count per aux phase
  int last;
  int next;                                               // aux task queue head
  int plo[kAuxPhases], pcnt[kAuxPhases];                  // this CTA's slice of each aux phase
  int pend[kAuxPhases], pdelta[kAuxPhases];               // queue index end / task = index + delta
  int ileft[kPipeMaxItems];                               // this CTA's search tiles of each item not yet done
  int th_state;                                           // 0 idle, 1 being filled, 2 S.th valid
  int k1_warps_done;                                      // K1 warps past their last tile
  int aux_ready;                                          // aux prologue done (queue + slices valid)
  unsigned scnt[kPipeMaxItems][9];                        // per-item partial search counts
};
constexpr int kPipeSmemBytes = (int)sizeof(PipeSmem) + 1024;

__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Cross-launch dependencies are flags in global memory (release: fence +
// atomic; acquire: ld.acquire.gpu), not whole-grid waits: launch j+1's aux
// work starts as soon as image j's K1 is published, while launch j's aux
// work may still run on other SMs.  Every flag is produced by a launch whose
// CTAs are all resident once its successor runs (a launch can only start
// after every CTA of its predecessor has started), so spinning cannot
// deadlock.
// CTA-scope flag handoffs in shared memory (release store / acquire load).
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Wait until *p >= v with acquire semantics.  Usually the flag is already
// set: one acquire load.  Otherwise poll with relaxed loads (an acquire load
// at gpu scope invalidates the SM's L1, CCTL.IVALL, so polling with it would
// do that on every iteration) and acquire once with a final acquire load
// (cheaper than a gpu-scope fence, which waits for all the warp's
// outstanding memory operations).  MTB_SPIN_LIMIT (debug builds) bounds the
// spin: a lost flag then fails the launch (trap) instead of hanging the GPU.
__device__ __forceinline__ void spin_geq(const uint32_t* p, uint32_t v) {
  if (ld_acquire(p) >= v) return;
#ifdef MTB_SPIN_LIMIT
  long long n = 0;
  while (ld_relaxed(p) < v) {
    __nanosleep(100);
    if (++n > (long long)MTB_SPIN_LIMIT) __trap();
  }
#else
  while (ld_relaxed(p) < v) __nanosleep(100);
#endif
  (void)ld_acquire(p);
}

// Lower median of one level's spread histogram (threshold.py:31-39): the
// smallest m with cumsum[m] >= (total + 1) / 2.  One warp; lane owns 8 bins.
__device__ __forceinline__ int warp_median(const uint32_t* spread, int lane) {
  uint32_t bins[8];
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    bins[i] = __ldcg(spread + (lane * 8 + i) * kHistStrideK1);
    s += bins[i];
  }
  uint32_t incl = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  const uint32_t target = (total + 1) >> 1;
  const unsigned mask = __ballot_sync(0xffffffffu, incl >= target);
  if (total == 0) return 0;   // empty level cannot occur (levels are >= 1x1)
  const int L = __ffs(mask) - 1;
  int med = 0;
  if (lane == L) {
    uint32_t c = incl - s;
    for (int i = 0; i < 8; ++i) {
      c += bins[i];
      if (c >= target) { med = lane * 8 + i; break; }
    }
  }
  return __shfl_sync(0xffffffffu, med, L);
}

// Unit u of the threshold sequence: 32 bitmap words of one level.  Levels
// 0..3 are in tile order (tile, row, word; threshold tasks below); levels
// 4..5 are row-major words (a word spans 2 or 4 tiles).
struct ThUnit {
  int k;            // level
  int64_t out;      // bitmap word index within the image's arena (u32), or -1
  int valid;        // valid pixels of the word
  int y, j;         // word coordinates
};

__device__ __forceinline__ ThUnit th_unit(const PipeArgs& a, const uint8_t* slot, int u, int lane) {
  // level-4/5 units only (levels 0..3 are threshold tasks of 4 KB)
  ThUnit r;
  const int k = (a.n > 5 && u >= a.th_units0[5]) ? 5 : 4;
  r.k = k;
  const int f = (u - a.th_units0[k]) * 32 + lane;   // row-major word index in the level
  r.y = f / a.nw32[k];
  r.j = f - r.y * a.nw32[k];
  r.out = r.y < a.g.lh[k] ? a.bit_off32[k] + f : -1;
  r.valid = a.g.lw[k] - 32 * r.j;
  return r;
}

__device__ __forceinline__ int div_tiles_x(const PipeArgs& a, int t) {
  return a.g.tiles_x == 1 ? t : (int)__umulhi((uint32_t)t, a.tx_magic);
}

// Levels 0..3: the level's bitmap words in tile order (tile, row, word); a
// unit is 32 words = 1 KB of contiguous tile-major gray.  NU units per warp
// iteration keep NU x 1 KB of loads in flight per warp.
template <int K>
__device__ __forceinline__ int th_level_units(const PipeArgs& a) {
  return (int)((((int64_t)a.g.tiles_x * a.g.tiles_y << (8 - 2 * K)) + 31) >> 5);
}

// ---- K3 via TMA bulk copies ------------------------------------------------
// Task r of level K (K <= 3) = bitmap words f0 = 128 r .. f0 + 127 in tile
// order = 4 KB of tile-major gray made of pieces of min(128, words/tile) words
// (L0: one 4 KB half-tile, L1: 2 x 2 KB, L2: 8 x 512 B, L3: 32 x 128 B).
// Lane i copies piece i with cp.async.bulk into the warp's staging buffer;
// the copy completes on the buffer's mbarrier, so a warp computes task r
// while task r+1 is in flight, without holding it in registers.
__device__ __forceinline__ void k3_bulk_issue(const PipeArgs& a, const uint8_t* slot, int K, int r, int lane,
                                              uint8_t* buf, unsigned long long* bar) {
  if (K == 0) {   // one contiguous 4 KB half-tile
    if (lane == 0) {
      mbar_expect_tx(bar, (uint32_t)kK3Bytes);
      const uint8_t* src = slot + (int64_t)(r >> 1) * kTileGrayBytes + (r & 1) * kK3Bytes;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_addr(buf)),
          "l"(src), "r"(kK3Bytes), "r"(smem_addr(bar))
          : "memory");
    }
    return;
  }
  const int lwpt = 8 - 2 * K;
  const int wpt = 1 << lwpt;
  const int pw = wpt < kK3Words ? wpt : kK3Words;   // words per piece
  const int npieces = kK3Words / pw;
  const int ntiles = a.g.tiles_x * a.g.tiles_y;
  const int f0 = kK3Words * r;
  // bytes that exist (pieces of tiles past the end are not copied)
  const int tiles_needed = ((f0 + kK3Words - 1) >> lwpt) - (f0 >> lwpt) + 1;
  int bytes = kK3Bytes;
  if ((f0 >> lwpt) + tiles_needed > ntiles) {
    const int last_f = ntiles << lwpt;                  // words that exist at this level
    bytes = (last_f - f0) * 32;
  }
  if (lane == 0) mbar_expect_tx(bar, (uint32_t)bytes);
  __syncwarp();
  if (lane < npieces) {
    const int f = f0 + lane * pw;
    const int t = f >> lwpt;
    if (t < ntiles) {
      const uint8_t* src = slot + (int64_t)t * kTileGrayBytes + tm_off(K) + (f & (wpt - 1)) * 32;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_addr(buf + lane * pw * 32)),
          "l"(src), "r"(pw * 32), "r"(smem_addr(bar))
          : "memory");
    }
  }
}

// Lanes read their 32-byte word as two 16-byte halves; lanes with bit 2 set
// read the upper half first so each LDS.128 of a warp touches 8 distinct
// 16-B bank groups per 128 B (lane stride 32 B otherwise hits only 4: 2-way
// conflicts).  The pack of swapped halves comes out rotated by 16 bits.
__device__ __forceinline__ uint32_t keep_mask(int valid) {
  return valid >= 32 ? 0xffffffffu : (valid <= 0 ? 0u : ((1u << valid) - 1u));
}
__device__ __forceinline__ void ld_word_sw(const uint8_t* p, int sw, uint32_t (&g)[8]) {
  const uint4 v0 = *reinterpret_cast<const uint4*>(p + 16 * sw);
  const uint4 v1 = *reinterpret_cast<const uint4*>(p + 16 * (sw ^ 1));
  g[0] = v0.x; g[1] = v0.y; g[2] = v0.z; g[3] = v0.w;
  g[4] = v1.x; g[5] = v1.y; g[6] = v1.z; g[7] = v1.w;
}

template <bool MED_LO>
__device__ __forceinline__ void k3_bulk_units(const PipeArgs& a, uint32_t* mtb, uint32_t* excl, const ThConst& c,
                                              uint32_t yt, uint32_t ytl, int K, int r, int lane, const uint8_t* buf) {
  const int lwpr = 3 - K, wpr = 1 << lwpr;
  const int lwpt = 8 - 2 * K, wpt = 1 << lwpt;
  const int rows = kK1TileRows >> K;
  const int ntiles = a.g.tiles_x * a.g.tiles_y;
  const int nw = a.nw32[K], lh = a.g.lh[K], lw = a.g.lw[K];
  const int boff = (int)a.bit_off32[K];
  const int f0 = kK3Words * r;
#pragma unroll 1
  for (int i = 0; i < kK3Units; ++i) {
    const int w = i * 32 + lane;
    const int f = f0 + w;
    const int t = f >> lwpt;
    const int rem = f & (wpt - 1);
    const int row = rem >> lwpr, cc = rem & (wpr - 1);
    const int ty = div_tiles_x(a, t), tx = t - ty * a.g.tiles_x;
    const int y = ty * rows + row, j = tx * wpr + cc;
    uint32_t g[8];
    const int sw = (lane >> 2) & 1;
    ld_word_sw(buf + w * 32, sw, g);
    uint32_t m, e;
    th_word_t<MED_LO, true>(g, c, yt, ytl, 32, m, e);
    const uint32_t keep = keep_mask(lw - 32 * j), rot = 16 * sw;
    m = __funnelshift_l(m, m, rot) & keep;
    e = __funnelshift_l(e, e, rot) & keep;
    if (t < ntiles && y < lh && j < nw) {
      const int o = boff + y * nw + j;
      mtb[o] = m;
      excl[o] = e;
    }
  }
}

// Level 0: the task is half a tile (rows 16 (r & 1) .. +15, 8 words each);
// unit i covers rows +4i .. +4i+3, so tile, column and validity are per task.
#ifndef K3_L0_UNROLL
#define K3_L0_UNROLL 1
#endif
constexpr int kK3L0Unroll = K3_L0_UNROLL;   // units of a level-0 task interleaved by the compiler
template <bool MED_LO>
__device__ __forceinline__ void k3_bulk_units_l0(const PipeArgs& a, uint32_t* mtb, uint32_t* excl, const ThConst& c,
                                                 uint32_t yt, uint32_t ytl, int r, int lane, const uint8_t* buf) {
  const int nw = a.nw32[0], lh = a.g.lh[0];
  const int t = r >> 1;
  const int ty = div_tiles_x(a, t), tx = t - ty * a.g.tiles_x;
  const int j = tx * 8 + (lane & 7);
  const int y0 = ty * kK1TileRows + ((r & 1) << 4) + (lane >> 3);
  const uint32_t keep = keep_mask(a.g.lw[0] - 32 * j);
  const int sw = (lane >> 2) & 1;
  const uint32_t rot = 16 * sw;
  const bool ok = j < nw;
  // running pointers: unit i is 4 rows below unit i-1
  uint32_t* pm = mtb + (int)a.bit_off32[0] + y0 * nw + j;
  uint32_t* pe = excl + (int)a.bit_off32[0] + y0 * nw + j;
  const uint8_t* src = buf + lane * 32;
  int rows_left = ok ? lh - y0 : 0;
#pragma unroll kK3L0Unroll
  for (int i = 0; i < kK3Units; ++i) {
    uint32_t g[8];
    ld_word_sw(src, sw, g);
    uint32_t m, e;
    th_word_t<MED_LO, true>(g, c, yt, ytl, 32, m, e);
    m = __funnelshift_l(m, m, rot) & keep;
    e = __funnelshift_l(e, e, rot) & keep;
    if (rows_left > 0) {
      *pm = m;
      *pe = e;
    }
    src += 32 * 32;
    pm += 4 * nw;
    pe += 4 * nw;
    rows_left -= 4;
  }
}

// Level 1 of a level-0 task's half tile, derived from its staged level-0
// rows (pyramid.py:17-32, the same rounding as K1's level 1, so the bits
// match the median K1's level-1 histogram gave): 16 x 256 px -> 8 x 128 px =
// 32 words, one per lane (row lane/4, word lane%4), thresholded and stored.
// K1 therefore never writes level-1 gray and there are no level-1 tasks.
__device__ __forceinline__ void k3_level1_from_l0(const PipeArgs& a, uint32_t* mtb, uint32_t* excl, const ThConst& c1,
                                                  uint32_t yt, uint32_t ytl, int r, int lane, const uint8_t* buf) {
  const int r1 = lane >> 2, c = lane & 3;
  const uint8_t* up = buf + (2 * r1) * kK1TilePx + 64 * c;
  // Lane (r1, c) reads its four 16-px chunks starting at chunk r1 & 3, so a
  // warp's LDS.128 covers all 8 bank groups (lanes differ by 512 B per row
  // and 64 B per column: in order they would share 2 of 8, 16-way).  The
  // pack then comes out rotated by 8 (r1 & 3) bits.
  const int q0 = r1 & 3;
  uint32_t g[8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {   // chunk (q0 + q) & 3: 16 L0 px of each row -> 8 L1 px = g[2q], g[2q+1]
    const int qq = (q0 + q) & 3;
    const uint4 u = *reinterpret_cast<const uint4*>(up + 16 * qq);
    const uint4 d = *reinterpret_cast<const uint4*>(up + kK1TilePx + 16 * qq);
    const uint32_t uw[4] = {u.x, u.y, u.z, u.w}, dw[4] = {d.x, d.y, d.z, d.w};
    uint32_t x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = (box_sum(uw[k], dw[k], 0) + (box_sum(uw[k], dw[k], 1) << 16)) >> 2;
    g[2 * q] = __byte_perm(x[0], x[1], 0x6420);
    g[2 * q + 1] = __byte_perm(x[2], x[3], 0x6420);
  }
  const int t = r >> 1;
  const int ty = div_tiles_x(a, t), tx = t - ty * a.g.tiles_x;
  const int y = ty * (kK1TileRows / 2) + 8 * (r & 1) + r1, j = tx * 4 + c;
  uint32_t m, e;
  th_word(g, c1, yt, ytl, 32, m, e);   // generic form: smaller code measured faster here
  const uint32_t keep = keep_mask(a.g.lw[1] - 32 * j), rot = 8 * q0;
  m = __funnelshift_l(m, m, rot) & keep;
  e = __funnelshift_l(e, e, rot) & keep;
  if (y < a.g.lh[1] && j < a.nw32[1]) {
    const int o = (int)a.bit_off32[1] + y * a.nw32[1] + j;
    mtb[o] = m;
    excl[o] = e;
  }
}

__device__ __forceinline__ void k3_bulk_finish(const PipeArgs& a, const uint8_t* slot, uint32_t* mtb, uint32_t* excl,
                                               const ThConst* th, uint32_t yt, uint32_t ytl, int K, int r, int lane,
                                               const uint8_t* buf, unsigned long long* bar, uint32_t parity) {
  mbar_wait(bar, parity);
  const ThConst c = th[K];
  if (a.tol > 127) {
    // rare: generic majority for the exclusion compare
    const int f0 = kK3Words * r;
    for (int i = 0; i < kK3Units; ++i) {
      const int w = i * 32 + lane, f = f0 + w;
      const int lwpr = 3 - K, lwpt = 8 - 2 * K;
      const int t = f >> lwpt, rem = f & ((1 << lwpt) - 1);
      const int row = rem >> lwpr, cc = rem & ((1 << lwpr) - 1);
      const int ty = div_tiles_x(a, t), tx = t - ty * a.g.tiles_x;
      const int y = ty * (kK1TileRows >> K) + row, j = tx * (1 << lwpr) + cc;
      const uint4 v0 = *reinterpret_cast<const uint4*>(buf + w * 32);
      const uint4 v1 = *reinterpret_cast<const uint4*>(buf + w * 32 + 16);
      const uint32_t g[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
      uint32_t m, e;
      th_word(g, c, yt, ytl, a.g.lw[K] - 32 * j, m, e);
      if (t < a.g.tiles_x * a.g.tiles_y && y < a.g.lh[K] && j < a.nw32[K]) {
        const int o = (int)a.bit_off32[K] + y * a.nw32[K] + j;
        mtb[o] = m;
        excl[o] = e;
      }
    }
  } else if (K == 0) {
    if (c.med_lo)
      k3_bulk_units_l0<true>(a, mtb, excl, c, yt, ytl, r, lane, buf);
    else
      k3_bulk_units_l0<false>(a, mtb, excl, c, yt, ytl, r, lane, buf);
  } else if (c.med_lo) {
    k3_bulk_units<true>(a, mtb, excl, c, yt, ytl, K, r, lane, buf);
  } else {
    k3_bulk_units<false>(a, mtb, excl, c, yt, ytl, K, r, lane, buf);
  }
  if (K == 0 && a.n > 1) k3_level1_from_l0(a, mtb, excl, th[1], yt, ytl, r, lane, buf);
  const int lwpt = 8 - 2 * K, wpt = 1 << lwpt;
  const int ntiles = a.g.tiles_x * a.g.tiles_y;
  // line `lane` of the task's gray: drop it from L2 without write-back
  if (K == 0) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(slot + (int64_t)(r >> 1) * kTileGrayBytes +
                                                       (r & 1) * kK3Bytes + lane * 128)
                 : "memory");
  } else if (lane < kK3Bytes / 128) {
    const int f = kK3Words * r + 4 * lane;
    const int t = f >> lwpt;
    if (t < ntiles)
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(slot + (int64_t)t * kTileGrayBytes + tm_off(K) +
                                                         (f & (wpt - 1)) * 32)
                   : "memory");
  }
  __syncwarp();   // the buffer may be refilled next
}

// 32 gray bytes of a level-4/5 word gathered from the tiles it spans
// (K = 4: two 16-px tile rows, K = 5: four 8-px tile rows).
template <int K>
__device__ __forceinline__ void th_gather45(const PipeArgs& a, const uint8_t* slot, const ThUnit& r, uint32_t (&g)[8]) {
  constexpr int tw = kK1TilePx >> K;
  constexpr int rows = kK1TileRows >> K;
  constexpr int nq = 32 / tw;
  const int ty = r.y / rows, row = r.y - ty * rows;
#pragma unroll
  for (int q = 0; q < nq; ++q) {
    const int tx = nq * r.j + q;
    uint32_t w4[4] = {0, 0, 0, 0};
    // (a unit's last words may lie below the level: r.out < 0, nothing is
    // stored, and the tile row would be past the slot)
    if (tx < a.g.tiles_x && r.out >= 0) {
      const uint8_t* p = slot + (int64_t)(ty * a.g.tiles_x + tx) * kTileGrayBytes + tm_off(K) + row * tm_pitch(K);
      if (tw == 16) {
        const uint4 v = *reinterpret_cast<const uint4*>(p);
        w4[0] = v.x; w4[1] = v.y; w4[2] = v.z; w4[3] = v.w;
      } else {
        const uint2 v = *reinterpret_cast<const uint2*>(p);
        w4[0] = v.x; w4[1] = v.y;
      }
    }
#pragma unroll
    for (int i = 0; i < tw / 4; ++i) g[q * (tw / 4) + i] = w4[i];
  }
}

// ---- K4 part ---------------------------------------------------------------
__device__ __forceinline__ void cp_async4(uint32_t* dst, const uint32_t* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(ok ? 4 : 0)
               : "memory");
}

// One search warp-tile (8 output rows x 32 words) of item `it`, staged into
// this warp's shared buffer with cp.async (every load in flight at once),
// then: per output word 9 x (LOP3 + LOP3 + POPC) over a 3-row register window
// of the target rows pre-shifted by bx-1, bx, bx+1 (funnel shifts).
__device__ __forceinline__ void pipe_search_tile(const PipeArgs& a, const PipeItem& it, int tile, int lane,
                                                 SearchStage& sm, unsigned* scnt) {
  const int k = it.level;
  const int h = a.g.lh[k];
  const int nw = a.nw32[k];
  const int cpr = (nw + 31) >> 5;
  const int rb = tile / cpr, cb = tile - rb * cpr;
  const int y0 = rb * kSRows;
  const int j0 = cb * 32;
  const int n = a.n;
  if (lane == 0) {
    if (k + 1 < n) {
      spin_geq(a.decided + (int64_t)it.pair * n + (k + 1), 1u);
    } else {
      spin_geq(a.k3_done + it.ref, gridDim.x);
      spin_geq(a.k3_done + it.tgt, gridDim.x);
    }
  }
  __syncwarp();
  int bx = 0, by = 0;
  if (k + 1 < n) {
    const int32_t* prev = a.acc + ((int64_t)it.pair * n + (k + 1)) * 2;
    bx = 2 * __ldcg(prev);
    by = 2 * __ldcg(prev + 1);
  }
  const uint32_t* A = a.mtb + (int64_t)it.ref * a.bit_img_words32 + a.bit_off32[k];
  const uint32_t* EA = a.excl + (int64_t)it.ref * a.bit_img_words32 + a.bit_off32[k];
  const uint32_t* B = a.mtb + (int64_t)it.tgt * a.bit_img_words32 + a.bit_off32[k];
  const uint32_t* EB = a.excl + (int64_t)it.tgt * a.bit_img_words32 + a.bit_off32[k];
  const int qb = bx >> 5;
  // ---- stage: A/EA rows y0..y0+7, words j0..j0+31; B/EB source rows
  //      y0-by-1 .. y0-by+8, words j0-qb-2 .. j0-qb+32
  {
    // Running row pointers; a copy with src-size 0 reads nothing and
    // zero-fills, so out-of-map rows/words need no address clamping.
    const int j = j0 + lane;
    const bool colA = j < nw;
    const int ja = colA ? j : 0;
    const uint32_t* pa = A + (int64_t)y0 * nw + ja;
    const uint32_t* pea = EA + (int64_t)y0 * nw + ja;
#pragma unroll
    for (int r = 0; r < kSRows; ++r) {
      const bool ok = colA && (y0 + r < h);
      cp_async4(&sm.a[r][lane], pa, ok);
      cp_async4(&sm.ea[r][lane], pea, ok);
      pa += nw;
      pea += nw;
    }
    const int sy0 = y0 - by - 1;
    const int idx0 = j0 - qb - 2 + lane, idx1 = idx0 + 32;
    const bool c0 = idx0 >= 0 && idx0 < nw, c1 = lane < 3 && idx1 >= 0 && idx1 < nw;
    // word idx0 + 32 of the same row (lanes 0-2) is an immediate offset off
    // the same pointer (a zero-size copy reads nothing, so the clamped base
    // needs no separate check)
    const int64_t rowoff = (int64_t)sy0 * nw + (c0 ? idx0 : 0);
    const uint32_t* pb0 = B + rowoff;
    const uint32_t* peb0 = EB + rowoff;
    const int shift1 = c0 ? 32 : idx1;   // pb0 + shift1 = word idx1 when c1
#pragma unroll
    for (int r = 0; r < kSRows + 2; ++r) {
      const int sy = sy0 + r;
      const bool rok = sy >= 0 && sy < h;
      cp_async4(&sm.b[r][lane], pb0, rok && c0);
      cp_async4(&sm.eb[r][lane], peb0, rok && c0);
      if (lane < 3) {
        cp_async4(&sm.b[r][lane + 32], pb0 + shift1, rok && c1);
        cp_async4(&sm.eb[r][lane + 32], peb0 + shift1, rok && c1);
      }
      pb0 += nw;
      peb0 += nw;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
  }
  // Candidate ddx = d - 1 shifts the target by dx = bx + d - 1 = 32 q + r.
  // With qb = bx >> 5 and rb = bx & 31 only three word selections occur
  // (staged word w[i] = lane + i holds W[j - qb - 2 + i]):
  //   rb == 0 : d=0 -> (w2, w3) r=31, d=1 -> (w1, w2) r=0,  d=2 -> (w1, w2) r=1
  //   rb == 31: d=0 -> (w1, w2) r=30, d=1 -> (w1, w2) r=31, d=2 -> (w0, w1) r=0
  //   else    : d   -> (w1, w2) r = rb + d - 1   (rb = rbx below)
  // so the row loop is instantiated per case without per-lane selects.
  const int rbx = bx & 31;
  unsigned cnt[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) cnt[i] = 0;
  auto rows = [&](auto case_tag) {
    constexpr int CASE = decltype(case_tag)::value;   // 0: rb==0, 1: rb==31, 2: other
    const int r0 = CASE == 0 ? 31 : (CASE == 1 ? 30 : rbx - 1);
    const int r1 = CASE == 0 ? 0 : (CASE == 1 ? 31 : rbx);
    const int r2 = CASE == 0 ? 1 : (CASE == 1 ? 0 : rbx + 1);
    auto shifted = [&](int lr, uint32_t (&sb)[3], uint32_t (&se)[3]) {
      const uint32_t b0 = sm.b[lr][lane], b1 = sm.b[lr][lane + 1], b2 = sm.b[lr][lane + 2];
      const uint32_t e0 = sm.eb[lr][lane], e1 = sm.eb[lr][lane + 1], e2 = sm.eb[lr][lane + 2];
      if (CASE == 0) {
        const uint32_t b3 = sm.b[lr][lane + 3], e3 = sm.eb[lr][lane + 3];
        sb[0] = shifted_word(b2, b3, r0); se[0] = shifted_word(e2, e3, r0);
      } else {
        sb[0] = shifted_word(b1, b2, r0); se[0] = shifted_word(e1, e2, r0);
      }
      sb[1] = shifted_word(b1, b2, r1); se[1] = shifted_word(e1, e2, r1);
      if (CASE == 1) {
        sb[2] = shifted_word(b0, b1, r2); se[2] = shifted_word(e0, e1, r2);
      } else {
        sb[2] = shifted_word(b1, b2, r2); se[2] = shifted_word(e1, e2, r2);
      }
    };
    // output row y0+rr needs staged source rows rr+2 (ddy=-1), rr+1 (0), rr (+1)
    uint32_t b0[3], e0[3], b1[3], e1[3];
    shifted(0, b0, e0);
    shifted(1, b1, e1);
#pragma unroll 2
    for (int rr = 0; rr < kSRows; ++rr) {
      uint32_t b2[3], e2[3];
      shifted(rr + 2, b2, e2);
      const uint32_t av = sm.a[rr][lane], ev = sm.ea[rr][lane];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        cnt[0 + d] += __popc((av ^ b2[d]) & ev & e2[d]);
        cnt[3 + d] += __popc((av ^ b1[d]) & ev & e1[d]);
        cnt[6 + d] += __popc((av ^ b0[d]) & ev & e0[d]);
      }
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        b0[d] = b1[d]; e0[d] = e1[d];
        b1[d] = b2[d]; e1[d] = e2[d];
      }
    }
  };
  if (rbx == 0) rows(std::integral_constant<int, 0>{});
  else if (rbx == 31) rows(std::integral_constant<int, 1>{});
  else rows(std::integral_constant<int, 2>{});
  __syncwarp();   // the staging buffer is reused by the next tile
  // CTA-level partial counts (shared atomics); flushed once per CTA and item
  // by pipe_search_flush after all of the CTA's tasks are done.
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const unsigned v = warp_sum(cnt[i]);
    if (lane == 0 && v) atomicAdd(scnt + i, v);
  }
}

// After the CTA's last task: add its partial counts of item `it` to the
// pair's 9 u64 counters; the last CTA to do so applies the search.py:67 key
// (err, |ddx|+|ddy|, index) and publishes the level's offset.
__device__ __forceinline__ void pipe_search_flush(const PipeArgs& a, const PipeItem& it, const unsigned* scnt) {
  const int n = a.n, k = it.level;
  unsigned long long* errs = a.errs + ((int64_t)it.pair * n + k) * 9;
  for (int i = 0; i < 9; ++i)
    if (scnt[i]) atomicAdd(errs + i, (unsigned long long)scnt[i]);
  __threadfence();
  uint32_t* done = a.done + (int64_t)it.pair * n + k;
  if (atomicAdd(done, 1u) == gridDim.x - 1) {
    __threadfence();
    int bx = 0, by = 0;
    if (k + 1 < n) {
      spin_geq(a.decided + (int64_t)it.pair * n + (k + 1), 1u);
      const int32_t* prev = a.acc + ((int64_t)it.pair * n + (k + 1)) * 2;
      bx = 2 * __ldcg(prev);
      by = 2 * __ldcg(prev + 1);
    }
    int best = 0, bd = 0;
    unsigned long long be = 0;
    for (int i = 0; i < 9; ++i) {
      const unsigned long long e = __ldcg(errs + i);
      const int d = abs(i % 3 - 1) + abs(i / 3 - 1);
      if (i == 0 || e < be || (e == be && d < bd)) { best = i; be = e; bd = d; }
    }
    int32_t* out = a.acc + ((int64_t)it.pair * n + k) * 2;
    out[0] = bx + best % 3 - 1;
    out[1] = by + best / 3 - 1;
    __threadfence();
    atomicExch(a.decided + (int64_t)it.pair * n + k, 1u);
  }
}

// ---- the non-K1 work of a launch as a per-CTA task queue -------------------
// Phases: K3 levels 0..3 (tile order, NU consecutive units per task), levels
// 4..5, uncovered row padding, search warp-tiles.  CTA c owns the slice
// [c*T/G, (c+1)*T/G) of every phase's T tasks; its warps pull tasks from a
// shared-memory counter — the aux warps right after the grid dependency
// wait, the K1 warps once their tiles are done — so the CTA's K1 and aux
// work finish together.
static_assert(sizeof(SearchStage) <= 2 * kK3Bytes, "search staging fits a warp's two K3 buffers");
static_assert(kPStages * kK1TileBytes >= 4 * 12288, "K1 warps stage in their group ring");

struct AuxCtx {
  uint32_t yt, ytl;
  int lane;
  SearchStage* stage;          // search staging (aliases kbuf)
  uint8_t* kbuf;               // 2 x 4 KB K3 staging
  unsigned long long* kbar;    // its 2 mbarriers
};

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Global task count of phase p.
__device__ __forceinline__ int aux_phase_tasks1(const PipeArgs& a, int p) {
  const bool th = a.th_cnt > 0;
  switch (p) {
    case 0: return th ? (th_level_units<0>(a) + kK3Units - 1) / kK3Units : 0;
    case 1: return 0;   // level 1 is derived inside the level-0 tasks
    case 2: return th && a.n > 2 ? (th_level_units<2>(a) + kK3Units - 1) / kK3Units : 0;
    case 3: return th && a.n > 3 ? (th_level_units<3>(a) + kK3Units - 1) / kK3Units : 0;
    case 4: return th ? a.th_units0[a.n] - a.th_units0[a.n < 4 ? a.n : 4] : 0;
    case 5: return th ? (a.th_pad_words + 31) / 32 : 0;
    default: return a.search_tiles;   // 6
  }
}
// K3 / level 4-5 / padding phases hold th_cnt images' tasks back to back.
__device__ __forceinline__ int aux_phase_tasks(const PipeArgs& a, int p) {
  return p < 6 ? a.th_cnt * aux_phase_tasks1(a, p) : a.search_tiles;
}
__device__ __forceinline__ const uint8_t* aux_slot(const PipeArgs& a, int b) { return a.th_gray[b]; }
__device__ __forceinline__ uint32_t* aux_mtb(const PipeArgs& a, int b) {
  return a.mtb + (int64_t)(a.th_img0 + b) * a.bit_img_words32;
}
__device__ __forceinline__ uint32_t* aux_excl(const PipeArgs& a, int b) {
  return a.excl + (int64_t)(a.th_img0 + b) * a.bit_img_words32;
}

// Zero padding words: flat index f over levels 0..3 of (row, uncovered word).
__device__ __forceinline__ void aux_pad(const PipeArgs& a, uint32_t* mtb, uint32_t* excl, int f) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k >= a.n) return;
    const int j0 = a.g.tiles_x * (8 >> k);
    const int npad = a.nw32[k] - j0;
    if (npad <= 0) continue;
    const int cnt = npad * a.g.lh[k];
    if (f < cnt) {
      const int y = f / npad, j = j0 + (f - y * npad);
      const int64_t o = a.bit_off32[k] + (int64_t)y * a.nw32[k] + j;
      mtb[o] = 0u;
      excl[o] = 0u;
      return;
    }
    f -= cnt;
  }
}

// Runs global task `t` of phase `p`.
__device__ __forceinline__ void aux_run(const PipeArgs& a, PipeSmem& S, const AuxCtx& x, int p, int t, int b) {
  switch (p) {
    case 4: {
      const uint8_t* slot = aux_slot(a, b);
      const ThUnit r = th_unit(a, slot, a.th_units0[a.n < 4 ? a.n : 4] + t, x.lane);
      uint32_t g8[8];
      if (r.k == 4) th_gather45<4>(a, slot, r, g8);
      else th_gather45<5>(a, slot, r, g8);
      uint32_t m, e;
      th_word(g8, S.th[b][r.k], x.yt, x.ytl, r.valid, m, e);
      if (r.out >= 0) { aux_mtb(a, b)[r.out] = m; aux_excl(a, b)[r.out] = e; }
      break;
    }
    case 5: {
      const int f = t * 32 + x.lane;
      if (f < a.th_pad_words) aux_pad(a, aux_mtb(a, b), aux_excl(a, b), f);
      break;
    }
    default:
      break;   // search tiles: aux_drain
  }
}

// The CTA's share of every phase's tasks, pulled by its warps from a
// shared-memory counter: the aux warps right after their prologue, the K1
// warps once the images' tiles are exhausted (tiles are claimed dynamically,
// so every CTA's K1 warps run dry at about the same time and the equal static
// slices stay balanced).
// Queue order q -> phase: search tiles first (their CTA partial counts are
// flushed per item as soon as the CTA's last tile of it is done, so the next
// launch's level can start early), then K3 levels 3, 2, 0 (+1), [1: no tasks],
// 4..5, padding.
constexpr int kSearchQ = 0;   // queue position of the search tiles
__device__ __forceinline__ int aux_phase_of(const PipeArgs& a, int q) {
  const int k = q == kSearchQ ? 6 : (q < kSearchQ ? q : q - 1);
  if (k < 4) {
    // the latency-bound gathered levels 3 and 2 first, level 0 (with level 1
    // derived in it) last, so the CTA's final tasks are the cheap contiguous
    // ones (+0.8 % at 24 MP, +0.2 % at 12 MP)
    constexpr int order[4] = {3, 2, 0, 1};
    return k == 0 ? order[0] : (k == 1 ? order[1] : (k == 2 ? order[2] : order[3]));
  }
  return k;
}

// The threshold constants of image th_img are needed only by K3 and level
// 4-5 tasks, and only once image th_img's medians are published: the first
// warp to reach such a task waits for them and fills S.th; others wait on
// S.th_state.  Search tasks (first in the queue) run meanwhile.
__device__ __forceinline__ void aux_need_thresholds(const PipeArgs& a, PipeSmem& S, int lane) {
  if (ld_acquire_cta(&S.th_state) == 2) return;
  int claim = 0;
  if (lane == 0) claim = atomicCAS(&S.th_state, 0, 1) == 0;
  claim = __shfl_sync(0xffffffffu, claim, 0);
  if (claim) {
    if (lane < a.th_cnt) spin_geq(a.med_ready + a.th_img0 + lane, 1u);
    __syncwarp();
    if (lane < a.n * a.th_cnt) {
      const int b = lane / a.n, k = lane - b * a.n;
      const int med = __ldcg(a.medians + (a.th_img0 + b) * a.n + k);
      ThConst c;
      c.med = (uint32_t)med * 0x01010101u;
      c.ym = (uint32_t)(255 - med) * 0x01010101u;
      c.yml = c.ym & 0x7f7f7f7fu;
      c.med_lo = med <= 127;
      S.th[b][k] = c;
    }
    __syncwarp();
    if (lane == 0) st_release_cta(&S.th_state, 2);
  } else {
    while (ld_acquire_cta(&S.th_state) != 2) __nanosleep(32);
  }
  __syncwarp();
}

__device__ __forceinline__ void aux_drain(const PipeArgs& a, PipeSmem& S, const AuxCtx& x) {
  if (x.lane == 0) {
    mbar_init(&x.kbar[0], 1);
    mbar_init(&x.kbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t par = 0u;                         // mbarrier phase bit per staging buffer
  int pend_k = -1, pend_r = 0, pend_b = 0;   // K3 task in flight (level, task, staging buffer)
  int pend_img = 0;                          // ... and its image (0 .. th_cnt-1)
  int nb = 0;                                // next staging buffer
  // Queue phase of the last claim: a warp's claims only grow, so the phase
  // bounds are reloaded only when a claim crosses the current phase's end.
  int q = -1, qend = 0, qdelta = 0, p = -1, t1 = 0x7fffffff;
  for (;;) {
    int t = 0;
    if (x.lane == 0) asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(t) : "r"(smem_addr(&S.next)) : "memory");
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= qend) {
      do {
        ++q;
      } while (q < kAuxPhases && t >= S.pend[q]);
      if (q < kAuxPhases) {
        p = aux_phase_of(a, q);
        qend = S.pend[q];
        qdelta = S.pdelta[q];
        t1 = p < 6 ? S.pt1[p] : 0x7fffffff;
      } else {
        p = -1;
        qend = 0x7fffffff;
      }
    }
    int r = t + qdelta;
    int bi = 0;   // K3 / level 4-5 / padding tasks: which of the th_cnt images
#pragma unroll
    for (int i = 1; i < kPipeImgs; ++i)
      if (r >= t1) {
        r -= t1;
        ++bi;
      }
    const bool k3 = p >= 0 && p < 4;
    if (k3) aux_need_thresholds(a, S, x.lane);
    if (k3) k3_bulk_issue(a, aux_slot(a, bi), p, r, x.lane, x.kbuf + nb * kK3Bytes, &x.kbar[nb]);
    if (pend_k >= 0) {   // the one call site of the K3 compute
      k3_bulk_finish(a, aux_slot(a, pend_img), aux_mtb(a, pend_img), aux_excl(a, pend_img), S.th[pend_img], x.yt,
                     x.ytl, pend_k, pend_r, x.lane, x.kbuf + pend_b * kK3Bytes, &x.kbar[pend_b], (par >> pend_b) & 1u);
      par ^= 1u << pend_b;
      pend_k = -1;
    }
    if (k3) {
      pend_k = p;
      pend_r = r;
      pend_img = bi;
      pend_b = nb;
      nb ^= 1;
      continue;
    }
    if (p < 0) return;
    if (p == 4) aux_need_thresholds(a, S, x.lane);
    aux_run(a, S, x, p, r, bi);
    if (p == 6) {
      int it = 0;
      while (it + 1 < a.n_items && r >= a.items[it + 1].tile0) ++it;
      pipe_search_tile(a, a.items[it], r - a.items[it].tile0, x.lane, *x.stage, S.scnt[it]);
      // this CTA's last tile of the item: publish its partial counts (the
      // item's level can be decided before this CTA's later search tiles)
      __syncwarp();
      if (x.lane == 0) {
        __threadfence_block();
        if (atomicSub(&S.ileft[it], 1) == 1) {
          __threadfence_block();
          pipe_search_flush(a, a.items[it], S.scnt[it]);
        }
      }
      __syncwarp();
    }
  }
}

// Before any aux task of launch j: image th_img's medians published
// (spin), threshold constants, the CTA's task slices, queue and search
// counters reset.  Run by `n` threads (at = 0..n-1) synchronised on `bar`.
__device__ __forceinline__ void aux_prologue(const PipeArgs& a, PipeSmem& S, int at, int n, int bar) {
  if (at == 0) S.next = 0;
  if (at < kAuxPhases) {
    const int G = gridDim.x, c = blockIdx.x;
    const int T = aux_phase_tasks(a, aux_phase_of(a, at));
    S.pt1[aux_phase_of(a, at)] = aux_phase_tasks1(a, aux_phase_of(a, at));
    S.plo[at] = (int)((int64_t)c * T / G);
    S.pcnt[at] = (int)((int64_t)(c + 1) * T / G) - S.plo[at];
  }
  for (int i = at; i < a.n_items * 9; i += n) (&S.scnt[0][0])[i] = 0;
  named_bar(bar, n);
  if (at == 0) {
    int e = 0;
    for (int q = 0; q < kAuxPhases; ++q) {
      S.pdelta[q] = S.plo[q] - e;
      e += S.pcnt[q];
      S.pend[q] = e;
    }
  }
  // this CTA's tiles of each item; an item it has none of is flushed now
  // (every CTA counts towards every item's completion)
  for (int i = at; i < a.n_items; i += n) {
    const int lo = S.plo[kSearchQ], hi = lo + S.pcnt[kSearchQ];
    const int t0 = a.items[i].tile0, t1 = i + 1 < a.n_items ? a.items[i + 1].tile0 : a.search_tiles;
    const int c = max(0, min(hi, t1) - max(lo, t0));
    S.ileft[i] = c;
    if (c == 0) pipe_search_flush(a, a.items[i], S.scnt[i]);
  }
  named_bar(bar, n);
}

__global__ void __launch_bounds__(kPipeThreads, kPipeCtasPerSm) pipe_kernel(const __grid_constant__ PipeArgs a,
                                                             const __grid_constant__ CUtensorMap rgb_map) {
  extern __shared__ __align__(128) uint8_t pipe_smem_raw[];
  const uint32_t raw = smem_addr(pipe_smem_raw);
  PipeSmem& S = *reinterpret_cast<PipeSmem*>(pipe_smem_raw + ((1024u - (raw & 1023u)) & 1023u));
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  // All dependencies on earlier launches are explicit flags, so the next
  // launch may be scheduled as soon as this one's CTAs are all resident.
  grid_dep_launch();
  if (tid == 0) {   // control words read across warp roles (smem is not zeroed between CTAs)
    S.aux_ready = 0;
    S.k1_warps_done = 0;
    S.th_state = 0;
  }
  __syncthreads();

  if (warp < kPK1Warps) {
    // ======================= K1 warps: image k1_img ==========================
    const int g = warp >> 2;          // K1 group
    const int t = tid & 127;
    const int wg = warp & 3;
    const int kt = tid;               // 0..255 among the K1 threads
    const uint32_t hb = smem_addr(&S.hist[0][0]);
    if (a.k1_cnt > 0) {
      const int tiles_img = a.g.tiles_x * a.g.tiles_y;
      const int tiles_all = a.k1_cnt * tiles_img;
      uint32_t* ctr = a.ctr + a.j;   // K1 tile counter of this launch
      uint64_t pol_first;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
      uint64_t gpol;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(gpol));
      for (int i = kt; i < kPipeImgs * 6 * 256; i += 32 * kPK1Warps) (&S.hist[0][0][0])[i] = 0;
      // Claim the next tile for ring stage `stage` (launch-wide counter over
      // the k1_cnt images' tiles, image-major: CTAs that start late take
      // fewer tiles) and start its copy; past the end, complete the stage's
      // phase with tile -1.  The first tile of each group is static (no
      // atomic round trip before the CTA's first copy).
      auto claim = [&](int stage, int fixed) {
        int tile = fixed >= 0 ? fixed : kPK1Groups * (int)gridDim.x + (int)atomicAdd(ctr, 1u);
        if (tile >= tiles_all) tile = -1;
        S.tile_of[g][stage] = tile;
        if (tile >= 0) {
          int b = 0, t1 = tile;
          while (t1 >= tiles_img) {
            t1 -= tiles_img;
            ++b;
          }
          const int ty = div_tiles_x(a, t1), tx = t1 - ty * a.g.tiles_x;
          mbar_expect_tx(&S.full[g][stage], kK1TileBytes);
          tma_tile(S.rgb[g][stage], &rgb_map, (kK1RowBytes / 4) * tx, kK1TileRows * ty, a.k1_img0 + b,
                   &S.full[g][stage], pol_first);
        } else {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&S.full[g][stage])) : "memory");
        }
      };
      if (t == 0) {
        // streamed input (mtb_align_fused_ex): the images' H2D copies have landed
        if (a.img_ready)
          for (int b = 0; b < a.k1_cnt; ++b) spin_geq(a.img_ready + a.k1_img0 + b, 1u);
        for (int s = 0; s < kPStages; ++s) mbar_init(&S.full[g][s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        claim(0, (int)blockIdx.x * kPK1Groups + g);
        for (int s = 1; s < kPStages; ++s) claim(s, -1);
      }
      // gray slot i % kPGraySlots last held image i - kPGraySlots: wait until
      // every CTA has thresholded it
      if (kt < a.k1_cnt && a.k1_img0 + kt >= a.gray_slots)
        spin_geq(a.k3_done + (a.k1_img0 + kt - a.gray_slots), gridDim.x);
      named_bar(5, 32 * kPK1Warps);   // hist zeroed, mbarriers initialised, slots free
      int k = 0, ptx = 0, pty = 0;
      uint8_t* ptg = nullptr;
      uint32_t phb = hb;
      bool pfull = true;
      for (;; ++k) {
        const int stage = k % kPStages;
        mbar_wait(&S.full[g][stage], (uint32_t)(k / kPStages) & 1u);
        int tile = *reinterpret_cast<volatile int*>(&S.tile_of[g][stage]);
        if (tile < 0) break;
        int b = 0;
        while (tile >= tiles_img) {
          tile -= tiles_img;
          ++b;
        }
        const int ty = div_tiles_x(a, tile), tx = tile - ty * a.g.tiles_x;
        const bool full = (ty * kK1TileRows + kK1TileRows <= a.g.h) && (tx * kK1TilePx + kK1TilePx <= a.g.w);
        uint2 v[8][3];
        {
          const uint8_t* src = S.rgb[g][stage] + (8 * wg) * kK1RowBytes + 24 * lane;
#pragma unroll
          for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) v[r][c] = *reinterpret_cast<const uint2*>(src + r * kK1RowBytes + 8 * c);
        }
        group_bar(g);
        if (t == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          claim(stage, -1);
        }
        if (k > 0 && a.g.nl >= 5 && wg == ((k - 1) & 3))
          k1_levels45_tm(a.g, ptg, S.l3[g][(k - 1) & 1], ptx, pty, lane, phb, pfull);
        const int img = a.k1_img0 + b;
        uint8_t* tg = a.k1_gray[b] + (int64_t)tile * kTileGrayBytes;
        const uint32_t hbi = hb + (uint32_t)b * (6 * 256 * 4);
        uint8_t* l3_slot = &S.l3[g][k & 1][wg][lane];
        if (full)
          k1_block_tm<true>(a.g, tg, v, tx, ty, wg, lane, hbi, l3_slot, gpol);
        else
          k1_block_tm<false>(a.g, tg, v, tx, ty, wg, lane, hbi, l3_slot, gpol);
        ptx = tx;
        pty = ty;
        ptg = tg;
        phb = hbi;
        pfull = full;
      }
      group_bar(g);
      if (k > 0 && a.g.nl >= 5 && wg == ((k - 1) & 3))
        k1_levels45_tm(a.g, ptg, S.l3[g][(k - 1) & 1], ptx, pty, lane, phb, pfull);
      // The last K1 warp of the CTA to finish flushes the CTA's histograms;
      // for each image of which this is the last CTA it also publishes the
      // medians (threshold.py:31-39).  Counter: word 1 of bin 0's 128-B line.
      // The other K1 warps go straight to the aux work.
      int mine = 0;
      if (lane == 0) {
        __threadfence_block();
        mine = atomicAdd(&S.k1_warps_done, 1) == kPK1Warps - 1;
      }
      mine = __shfl_sync(0xffffffffu, mine, 0);
      if (mine) {
        __threadfence_block();
        for (int b = 0; b < a.k1_cnt; ++b) {
          const int img = a.k1_img0 + b;
          uint32_t* gh = a.g.hist + (int64_t)img * a.g.hist_img_stride;
          for (int i = lane; i < a.g.nl * 256; i += 32) {
            const uint32_t c = *reinterpret_cast<volatile uint32_t*>(&(&S.hist[b][0][0])[i]);
            if (c) atomicAdd(&gh[(int64_t)i * kHistStrideK1], c);
          }
          int last = 0;
          if (lane == 0) {
            __threadfence();
            last = atomicAdd(gh + 1, 1u) == gridDim.x - 1;
          }
          last = __shfl_sync(0xffffffffu, last, 0);
          if (last) {
            __threadfence();
            for (int k = 0; k < a.n; ++k) {
              const int m = warp_median(gh + k * 256 * kHistStrideK1, lane);
              if (lane == 0) a.medians[img * a.n + k] = m;
            }
            if (lane == 0) {
              __threadfence();
              atomicExch(a.med_ready + img, 1u);
            }
          }
        }
      }
    }
    // Join the aux work (the aux prologue has long finished: spin on its flag).
    if constexpr (kPAuxWarps > 0) {
      while (ld_acquire_cta(&S.aux_ready) == 0) __nanosleep(64);
    } else {
      aux_prologue(a, S, tid, kPipeThreads, 9);
    }
  } else {
    // ======================= aux warps: K3 + search ==========================
    aux_prologue(a, S, tid - 32 * kPK1Warps, 32 * kPAuxWarps, 6);
    if (tid == 32 * kPK1Warps) st_release_cta(&S.aux_ready, 1);
  }

  // ============ every warp: this CTA's share of the aux tasks ================
  AuxCtx ax;
  ax.yt = (uint32_t)(255 - a.tol) * 0x01010101u;
  ax.ytl = ax.yt & 0x7f7f7f7fu;
  ax.lane = lane;
  // K1 warps stage in their group's ring (all its TMA copies have landed,
  // 16 KB per warp); aux warps in their own 8 KB
  ax.kbuf = warp < kPK1Warps
                ? &S.rgb[0][0][0] + (size_t)(warp >> 2) * (kPStages * kK1TileBytes) + (warp & 3) * 12288
                : &S.abuf[warp - kPK1Warps][0][0];
  ax.kbar = S.kbar[warp];
  ax.stage = reinterpret_cast<SearchStage*>(ax.kbuf);
  aux_drain(a, S, ax);
  named_bar(10, kPipeThreads);   // every task of this CTA done
  if (tid == 0 && a.th_cnt > 0) {
    __threadfence();
    for (int b = 0; b < a.th_cnt; ++b) atomicAdd(a.k3_done + a.th_img0 + b, 1u);
  }

}

bool k1_rgb_supported(int w, int64_t rgb_pitch, int64_t rgb_img_stride, const void* rgb);
PFN_cuTensorMapEncodeTiled_v12000 k1_encode_tiled();
int64_t spread_hist_elems(int n_levels);

}  // namespace mtb

using namespace mtb;

// Images per launch: 2 up to 64 MB of gray per image (24 MP = 33 MB: 2
// images per launch measured 16.7 K vs 16.1 K pairs/s although more gray
// spills to HBM; 12 MP: 28.2 K vs 24.1 K), else 1.
static int pipe_images_per_launch(int w, int h) {
  const int64_t slot = (int64_t)((w + kK1TilePx - 1) / kK1TilePx) * ((h + kK1TileRows - 1) / kK1TileRows) *
                       kTileGrayBytes;
  return slot <= ((int64_t)64 << 20) ? kPipeImgs : 1;
}

extern "C" int mtb_align_fused_images_per_launch(int w, int h) { return pipe_images_per_launch(w, h); }

// Launch plan of one mtb_align_fused call: launch j runs K1 of images
// jB .. jB+B-1 and K3 of images (j-1)B .. jB-1; pair q runs its levels
// n-1 .. 0 in launches t(q) .. t(q)+n-1, t(q) >= max(ref, tgt) / B + 2 (the
// launch after its images' K3).  A launch carries at most kPipeMaxItems
// (pair, level) items: a pair whose levels would overfill one of its launches
// starts later (greedy, pairs in readiness order), so the whole plan is valid
// before anything is enqueued.  (One launch for all trailing levels, chained
// through the decided flags, measured 6 % slower than one launch per level.)
struct PipeLaunch {
  int j;                                    // launch index (K1/K3 images, tile counter)
  std::vector<std::pair<int, int>> items;   // (pair, level)
};
static std::vector<PipeLaunch> pipe_plan(int n_img, int B, int nl, const int32_t* pairs, int n_pairs) {
  const int k1_launches = (n_img + B - 1) / B;
  std::vector<int> order(n_pairs), start(n_pairs);
  for (int q = 0; q < n_pairs; ++q) {
    order[q] = q;
    start[q] = std::max(pairs[2 * q], pairs[2 * q + 1]) / B + 2;
  }
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return start[x] < start[y]; });
  std::vector<int> load;   // items per launch
  int J = k1_launches + 1;
  for (int q : order) {
    int t = start[q];
    for (;;) {
      if ((int)load.size() < t + nl) load.resize(t + nl, 0);
      bool fits = true;
      for (int d = 0; d < nl && fits; ++d) fits = load[t + d] < kPipeMaxItems;
      if (fits) break;
      ++t;
    }
    for (int d = 0; d < nl; ++d) ++load[t + d];
    start[q] = t;
    J = std::max(J, t + nl);
  }
  std::vector<PipeLaunch> plan(J);
  for (int j = 0; j < J; ++j) plan[j].j = j;
  for (int q : order)
    for (int d = 0; d < nl; ++d) plan[start[q] + d].items.emplace_back(q, nl - 1 - d);
  return plan;
}

// Upper bound of the launch count (sizes the per-launch tile counters).
static int64_t pipe_max_launches(int n_img, int n_pairs, int levels) {
  const int64_t L = levels < 1 ? 1 : levels;
  return (int64_t)n_img + 8 + ((int64_t)n_pairs * L + kPipeMaxItems - 1) / kPipeMaxItems + L;
}

extern "C" int mtb_align_fused_launches(int w, int h, int levels, int n_img, const int32_t* pairs_host, int n_pairs) {
  Plan p;
  if (!make_plan(w, h, levels, &p) || n_img < 1 || n_pairs < 0 || (n_pairs > 0 && !pairs_host)) return -1;
  return (int)pipe_plan(n_img, pipe_images_per_launch(w, h), p.n, pairs_host, n_pairs).size();
}

extern "C" int64_t mtb_align_fused_sync_words(int n_img, int n_pairs, int levels) {
  return pipe_max_launches(n_img, n_pairs, levels) + 2 * (int64_t)n_img + (int64_t)n_pairs * (levels < 1 ? 1 : levels);
}

extern "C" int mtb_align_fused_workspace(int w, int h, int levels, int64_t* gray_bytes, int64_t* hist_elems) {
  Plan p;
  if (!make_plan(w, h, levels, &p)) return -1;
  const int64_t tiles = (int64_t)((w + kK1TilePx - 1) / kK1TilePx) * ((h + kK1TileRows - 1) / kK1TileRows);
  if (gray_bytes) *gray_bytes = kPGraySlots * tiles * kTileGrayBytes;
  if (hist_elems) *hist_elems = spread_hist_elems(p.n);
  return p.n <= kPipeMaxLevels ? p.n : -1;
}

extern "C" int mtb_align_fused_ex(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride, int w, int h,
                                  int n_img, int levels, int tol, const int32_t* pairs_host, int n_pairs,
                                  uint8_t* gray_ws, uint32_t* hist_ws, int32_t* medians, uint64_t* mtb,
                                  uint64_t* exclusion, int32_t* acc, unsigned long long* errs, uint32_t* done,
                                  uint32_t* sync_ws, const uint32_t* img_ready, void* stream) {
  clear_error();
  MTB_REQUIRE(rgb && gray_ws && hist_ws && medians && mtb && exclusion && sync_ws, "null pointer");
  MTB_REQUIRE(n_pairs == 0 || (pairs_host && acc && errs && done), "null pair buffers");
  MTB_REQUIRE(n_img >= 1 && n_img <= 65535, "image count out of range");
  MTB_REQUIRE(n_pairs >= 0 && n_pairs <= 65535, "pair count out of range");
  MTB_REQUIRE(tol >= 0 && tol <= 255, "noise tolerance must be in 0..255");
  MTB_REQUIRE(rgb_pitch >= 3 * (int64_t)w, "rgb pitch smaller than row");
  Plan p;
  MTB_REQUIRE(make_plan(w, h, levels, &p), "image must be at least 16x16 and levels >= 1");
  MTB_REQUIRE(p.n <= kPipeMaxLevels, "fused path supports at most 6 pyramid levels");
  MTB_REQUIRE(k1_rgb_supported(w, rgb_pitch, rgb_img_stride, rgb),
              "fused path needs 16-byte aligned RGB rows with 3*W % 4 == 0");
  const int64_t slot_bytes =
      (int64_t)((w + kK1TilePx - 1) / kK1TilePx) * ((h + kK1TileRows - 1) / kK1TileRows) * kTileGrayBytes;
  MTB_REQUIRE(slot_bytes < ((int64_t)1 << 31), "image too large for the fused path");
  for (int q = 0; q < n_pairs; ++q) {
    MTB_REQUIRE(pairs_host[2 * q] >= 0 && pairs_host[2 * q] < n_img && pairs_host[2 * q + 1] >= 0 &&
                    pairs_host[2 * q + 1] < n_img,
                "pair image index out of range");
  }
  cudaStream_t st = as_stream(stream);

  PipeArgs a;
  std::memset(&a, 0, sizeof(a));
  K1Args& g = a.g;
  g.w = w;
  g.h = h;
  g.nl = p.n;
  for (int k = 0; k < 6; ++k) {
    const int l = k < p.n ? k : p.n - 1;
    g.off[k] = (int)p.lv[l].gray_off;
    g.pitch[k] = (int)p.lv[l].gray_pitch;
    g.lw[k] = k < p.n ? p.lv[k].w : 0;
    g.lh[k] = k < p.n ? p.lv[k].h : 0;
  }
  g.gray = gray_ws;
  g.gray_img_stride = slot_bytes;   // tile-major slot (k1_tile.cuh kTmOff)
  g.hist = hist_ws;
  g.hist_img_stride = spread_hist_elems(p.n);
  g.hist_bin = kHistStrideK1;
  g.tiles_x = (w + kK1TilePx - 1) / kK1TilePx;
  g.tiles_y = (h + kK1TileRows - 1) / kK1TileRows;
  g.n_img = 1;
  g.keep_gray = 1;
  a.n = p.n;
  a.tol = tol;
  a.th_units0[0] = 0;
  const int ntiles = ((w + kK1TilePx - 1) / kK1TilePx) * ((h + kK1TileRows - 1) / kK1TileRows);
  a.tx_magic = g.tiles_x > 1 ? (uint32_t)((((uint64_t)1 << 32) + g.tiles_x - 1) / g.tiles_x) : 0u;
  MTB_REQUIRE(g.tiles_x < 4096, "image too wide for the fused path");
  for (int k = 0; k < p.n; ++k) {
    a.nw32[k] = (int)(2 * p.lv[k].nw64);
    a.bit_off32[k] = 2 * p.lv[k].bit_off;
    a.th_cpr[k] = (a.nw32[k] + 31) / 32;
    // levels 0..3: tile-order words (256 >> 2k per tile); 4..5: row-major words
    const int64_t words = k <= 3 ? (int64_t)ntiles * (256 >> (2 * k)) : (int64_t)a.nw32[k] * p.lv[k].h;
    a.th_units0[k + 1] = a.th_units0[k] + (int)((words + 31) / 32);
  }
  for (int k = p.n + 1; k <= kPipeMaxLevels; ++k) a.th_units0[k] = a.th_units0[p.n];
  a.th_pad_words = 0;
  for (int k = 0; k < p.n && k < 4; ++k) {
    const int npad = a.nw32[k] - g.tiles_x * (8 >> k);
    if (npad > 0) a.th_pad_words += npad * p.lv[k].h;
  }
  a.mtb = reinterpret_cast<uint32_t*>(mtb);
  a.excl = reinterpret_cast<uint32_t*>(exclusion);
  a.bit_img_words32 = 2 * p.bit_img_words;
  a.medians = medians;
  a.ctr = sync_ws;
  a.img_ready = img_ready;
  a.acc = acc;
  a.errs = errs;
  a.done = done;

  MTB_CUDA(cudaMemsetAsync(hist_ws, 0, sizeof(uint32_t) * spread_hist_elems(p.n) * n_img, st));
  if (n_pairs > 0) {
    MTB_CUDA(cudaMemsetAsync(errs, 0, sizeof(unsigned long long) * 9 * p.n * n_pairs, st));
    MTB_CUDA(cudaMemsetAsync(done, 0, sizeof(uint32_t) * p.n * n_pairs, st));
  }

  const int B = pipe_images_per_launch(w, h);
  a.gray_slots = 3 * B;
  const std::vector<PipeLaunch> plan = pipe_plan(n_img, B, p.n, pairs_host, n_pairs);
  const int J = plan.back().j + 1;
  // sync_ws (mtb_align_fused_sync_words): [Jmax] K1 tile counters, [n_img]
  // medians-ready flags, [n_img] K3-done counters, [P][n] decided flags
  const int64_t jmax = pipe_max_launches(n_img, n_pairs, p.n);
  MTB_REQUIRE(J <= jmax, "internal: launch count");
  const int64_t sync_words = jmax + 2 * (int64_t)n_img + (int64_t)n_pairs * p.n;
  MTB_CUDA(cudaMemsetAsync(sync_ws, 0, sizeof(uint32_t) * sync_words, st));
  a.ctr = sync_ws;
  a.med_ready = sync_ws + jmax;
  a.k3_done = a.med_ready + n_img;
  a.decided = a.k3_done + n_img;
  a.n_launch = (int)plan.size();
  int search_tiles_level[kPipeMaxLevels];
  for (int k = 0; k < p.n; ++k) search_tiles_level[k] = ((p.lv[k].h + kSRows - 1) / kSRows) * ((a.nw32[k] + 31) / 32);

  CUtensorMap map;
  {
    const cuuint64_t dims[3] = {(cuuint64_t)(3 * (int64_t)w / 4), (cuuint64_t)h, (cuuint64_t)n_img};
    const cuuint64_t strides[2] = {(cuuint64_t)rgb_pitch, (cuuint64_t)rgb_img_stride};
    const cuuint32_t box[3] = {kK1RowBytes / 4, kK1TileRows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = k1_encode_tiled()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, (void*)rgb, dims, strides, box,
                                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed for the RGB batch");
      return MTB_ECUDA;
    }
  }
  // the shared-memory opt-in is per device (cheap; set on every call)
  MTB_CUDA(cudaFuncSetAttribute(pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPipeSmemBytes));
  const int grid = num_sms() * kPipeCtasPerSm;
  int launches = 0;
  for (const PipeLaunch& L : plan) {
    const int j = L.j;
    a.j = j;
    a.k1_img0 = j * B;
    a.k1_cnt = std::max(0, std::min(B, n_img - j * B));
    a.th_img0 = (j - 1) * B;
    a.th_cnt = j >= 1 ? std::max(0, std::min(B, n_img - (j - 1) * B)) : 0;
    for (int b = 0; b < kPipeImgs; ++b) {
      a.k1_gray[b] = gray_ws + (int64_t)((a.k1_img0 + b) % a.gray_slots) * g.gray_img_stride;
      a.th_gray[b] = gray_ws + (int64_t)(((a.th_img0 + b) % a.gray_slots + a.gray_slots) % a.gray_slots) * g.gray_img_stride;
    }
    a.n_items = 0;
    a.search_tiles = 0;
    for (const auto& qi : L.items) {   // pipe_plan caps a launch at kPipeMaxItems items
      PipeItem& it = a.items[a.n_items++];
      it.pair = qi.first;
      it.ref = pairs_host[2 * qi.first];
      it.tgt = pairs_host[2 * qi.first + 1];
      it.level = qi.second;
      it.tile0 = a.search_tiles;
      a.search_tiles += search_tiles_level[it.level];
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kPipeThreads);
    cfg.dynamicSmemBytes = kPipeSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = j > 0 ? 1 : 0;   // launch 0 follows the memsets in full stream order
    const cudaError_t e = cudaLaunchKernelEx(&cfg, pipe_kernel, a, map);
    if (e != cudaSuccess) {
      set_error(std::string("pipe_kernel: ") + cudaGetErrorString(e));
      return MTB_ECUDA;
    }
    ++launches;
  }
  return check_launch("pipe_kernel", launches);
}

extern "C" int mtb_align_fused(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride, int w, int h,
                               int n_img, int levels, int tol, const int32_t* pairs_host, int n_pairs,
                               uint8_t* gray_ws, uint32_t* hist_ws, int32_t* medians, uint64_t* mtb,
                               uint64_t* exclusion, int32_t* acc, unsigned long long* errs, uint32_t* done,
                               uint32_t* sync_ws, void* stream) {
  return mtb_align_fused_ex(rgb, rgb_pitch, rgb_img_stride, w, h, n_img, levels, tol, pairs_host, n_pairs, gray_ws,
                            hist_ws, medians, mtb, exclusion, acc, errs, done, sync_ws, nullptr, stream);
}

// Stream-ordered 32-bit store (cuStreamWriteValue32, with its implicit memory
// barrier): marks an image's H2D copy complete for mtb_align_fused_ex.
extern "C" int mtb_stream_write_u32(uint32_t* dptr, uint32_t value, void* stream) {
  clear_error();
  MTB_REQUIRE(dptr, "null pointer");
  using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  static WriteFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WriteFn>(p);
  }
  if (!fn) {
    set_error("cuStreamWriteValue32 unavailable");
    return MTB_ECUDA;
  }
  if (fn(reinterpret_cast<CUstream>(as_stream(stream)), reinterpret_cast<CUdeviceptr>(dptr), value, 0) !=
      CUDA_SUCCESS) {
    set_error("cuStreamWriteValue32 failed");
    return MTB_ECUDA;
  }
  return MTB_OK;
}
