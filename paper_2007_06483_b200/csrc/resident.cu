// The SMEM-resident fused alignment kernel: preprocess (K1 + medians + K3)
// and the coarse-to-fine search (K4) of a whole batch of exposure pairs in
// ONE persistent launch, with every image's gray pyramid held in shared
// memory between its histogram pass and its threshold pass (SURVEY.md §7
// hard part 1, option 1), so gray never reaches L2 or HBM.
//
// Reference path (bit-exact): pipeline.py:80-90 -> build_mtb_pyramid
// (image.py:58-68, pyramid.py:17-62, threshold.py:25-88) -> find_offset
// (search.py:53-95, kernels/_native.pyx:73-111).
//
// Geometry.  An image is cut into jobs of 32 rows x 64 px (job-major order
// jy * jobs_x + jx).  CTA c (one per SM, 512 threads) owns the same
// contiguous range of jobs [c*T/G, (c+1)*T/G) of every image, and job j of
// its range lives in shared-memory slot j (2736 B: levels 0..5 of the job,
// tile-major).  A 24 MP image is 11,750 jobs = at most 80 per SM = 219 KB.
//
// Warp roles.
//   * K1 warps (16 - kRSearchWarps): claim jobs of the CTA's sequence
//     (image s, job j) through a shared counter.  Job (s, j): issue the 8x8
//     px RGB block loads of every lane (24 x LDG.64, L2 evict_first: 6 KB
//     per warp in flight, so the register file is the staging buffer), then
//     threshold image s-1's job j out of slot j (K3: MTB + exclusion words of
//     levels 0..5 -> the packed map arenas), then build image s's gray,
//     levels 1..5 and histograms into slot j (K1).  The warp that completes
//     the CTA's last K1 job of image s flushes the CTA histogram (one RED per
//     nonzero bin) and arrives on the image's counter; the K3 of image s
//     starts once every CTA has arrived (the median needs the whole image:
//     threshold.py:31-39) and each CTA derives the medians itself.
//   * search warps: pull search tasks (pair, level, 32 rows x 32 words)
//     from a global queue; the task that completes a (pair, level) applies
//     the search.py:67 key and appends the next finer level to the queue;
//     the CTA that completes an image's maps appends level n-1 of the pairs
//     that became ready.  K1 warps join them once their jobs run out.
//
// HBM traffic per image: the RGB read once (72 MB at 24 MP) plus the packed
// maps (8 MB written, read back by the search from L2).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "k1_tile.cuh"   // gray4, box_sum
#include "common.cuh"

namespace mtb {

constexpr int kRThreads = 512;
constexpr int kRWarps = kRThreads / 32;
#ifndef RES_SEARCH_WARPS
#define RES_SEARCH_WARPS 2
#endif
constexpr int kRSearchWarps = RES_SEARCH_WARPS;
constexpr int kRK1Warps = kRWarps - kRSearchWarps;
constexpr int kJobRows = 32, kJobPx = 64;
constexpr int kSlotBytes = 2224;          // L0 2048 + L2 128 + L3 32 + L4 8 + L5 2 (level 1 is derived in K3)
constexpr int kStageBytes = kJobRows * 3 * kJobPx;   // one job's RGB: 32 rows x 192 B (TMA box 48 u32 x 32 rows)
constexpr int kRMaxStages = 8;
constexpr int kRMaxLevels = 6;
constexpr int kRSearchRows = 32;          // search task: 32 output rows x 32 words
constexpr int kRSmemLimit = 232448;       // opt-in dynamic + static shared memory per CTA on sm_100
constexpr int kRMaxPairsPerUpload = 1536;

__host__ __device__ constexpr int slot_off(int k) {
  return k == 0 ? 0 : k == 2 ? 2048 : k == 3 ? 2176 : k == 4 ? 2208 : 2216;
}
// Level 0: row i (0..31) of 64 px, 16-B chunk q (0..3), XOR-swizzled so the
// K3 reads (lane = row, 16 B per lane) and the K1 stores are bank-conflict free.
__device__ __forceinline__ int l0_addr(int row, int q) { return row * 64 + 16 * (q ^ (((row >> 1) ^ (row >> 3)) & 3)); }

struct ResArgs {
  const uint8_t* rgb;
  int64_t rgb_pitch, rgb_img_stride;
  int w, h, n, tol;
  int lw[kRMaxLevels], lh[kRMaxLevels], nw32[kRMaxLevels];
  int64_t bit_off32[kRMaxLevels];
  int64_t bit_img_words32;
  int jobs_x, jobs;                 // per image
  int n_img;
  uint32_t* mtb;
  uint32_t* excl;
  uint32_t* part;                   // [2][G][6 * 256] partial histograms of each CTA (image parity)
  uint32_t* tot;                    // [2][6 * 256] summed histograms
  uint32_t* arrive2;                // [n_img] CTAs that summed their bins of the image
  int32_t* medians;                 // [img][n]
  int n_pairs;
  const int32_t* pairs;             // device [P][2] (ref, tgt)
  const int32_t* ready_pairs;       // device: pair indices sorted by max(ref, tgt)
  const int32_t* ready_start;       // device [n_img + 1]: first ready_pairs index with max >= img
  int32_t* acc;                     // [P][n][2]
  unsigned long long* errs;         // [P][n][9]
  uint32_t* done;                   // [P][n] finished search tasks
  uint32_t* arrive;                 // [n_img] CTAs that flushed their histograms of the image
  uint32_t* k3done;                 // [n_img] CTAs that wrote their maps of the image
  uint32_t* qitem;                  // [P * n] search queue: 0 = empty, else pair * 8 + level + 1
  uint32_t* qclaim;                 // [P * n] claimed tasks of each queue entry
  uint32_t* qtail;                  // entries appended
  uint32_t* medflag;                // [G][32] per-CTA line: [0] images flushed, [1] images with medians, [2..7] medians
  const uint32_t* img_ready;        // [n_img] nonzero once the image's RGB is in HBM (streamed input), or null
  int tasks[kRMaxLevels], strips[kRMaxLevels];
  int stages;                       // TMA ring depth
#ifdef RES_EXP_TRACE   // experiment builds only: [n_img][G][4] %globaltimer stamps
  unsigned long long* trace;
#endif
};

#ifdef RES_EXP_TRACE
__device__ __forceinline__ void rtrace(const ResArgs& a, int s, int what) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  a.trace[((int64_t)s * gridDim.x + blockIdx.x) * 8 + what] = t;
}
#define RTRACE(a, s, w) rtrace(a, s, w)
#else
#define RTRACE(a, s, w)
#endif

// Threshold constants of one level (threshold.py:42-56).
struct RTh {
  uint32_t med, ym, yml;
  int med_lo;
};

struct ResShared {
  unsigned long long full[kRMaxStages];   // TMA ring: job RGB landed
  int stage_job[kRMaxStages];             // job whose copy was issued into each stage
  RTh th[2][kRMaxLevels];  // threshold constants of images s (parity s & 1)
  int medtag[2];           // s + 1 once th[s & 1] holds image s's constants
  int medclaim[2];         // s + 1 once a warp computes them
  int k1cnt[2], k3cnt[2];  // K1 / K3 jobs finished of image s (parity s & 1)
  int claim;               // job sequence counter
  int ready_img;           // streamed input: images known to be in HBM
  int stages;              // TMA ring depth
};

// ---- memory-model helpers ---------------------------------------------------
// Spins poll with relaxed loads (L2, no L1 invalidation) and acquire once the
// condition holds: an acquire load at gpu scope invalidates the SM's L1
// (CCTL.IVALL), which would throw away the K1 warps' RGB lines on every poll.
__device__ __forceinline__ uint32_t r_ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void r_fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void r_spin_geq(const uint32_t* p, uint32_t v, int ns) {
  while (r_ld_relaxed(p) < v) __nanosleep(ns);
  r_fence_acquire();
}
__device__ __forceinline__ int r_ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
  return v;
}
__device__ __forceinline__ void r_st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t r_ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t r_atom_add_acqrel(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void r_st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void r_st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// CTA-scope counter bump that publishes the warp's prior writes (shared and
// global) to the warp that observes the final count.
__device__ __forceinline__ int r_smem_add_acqrel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_addr(p)), "r"(v)
               : "memory");
  return old;
}
// ---- K1: gray, levels 1..5, histograms of one job (one warp) --------------
// The job's RGB (32 rows x 192 B) lands in a shared-memory stage by one TMA
// tile copy; lane (r = lane >> 3, c = lane & 7) copies its 8x8 px block
// (v[i][0..2] = the 24 B of block row i) to registers and the stage is
// refilled with a later job's tile right away.
__device__ __forceinline__ void stage_to_regs(const uint8_t* stage, int lane, uint2 (&v)[8][3]) {
  const uint8_t* src = stage + (8 * (lane >> 3)) * (3 * kJobPx) + 24 * (lane & 7);
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) v[i][k] = *reinterpret_cast<const uint2*>(src + i * (3 * kJobPx) + 8 * k);
}

// Histogram increment at shared address `addr` (ATOMS.POPC.INC); the level
// histograms are 1 KB-aligned, so bin b of level k is hb + 1024 k | 4 b.
__device__ __forceinline__ void hadd(uint32_t addr) { asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory"); }

// Level 0 gray into the slot (swizzled rows); level 1 only feeds the
// histogram and level 2 (K3 re-derives it from level 0); levels 2..5 into
// the slot.
template <bool FULL>
__device__ __forceinline__ void res_k1(const ResArgs& a, const uint2 (&v)[8][3], int jx, int jy, int lane,
                                       uint8_t* slot, uint32_t hb) {
  const int r = lane >> 3, c = lane & 7;
  const int x0 = jx * kJobPx + 8 * c, y0 = jy * kJobRows + 8 * r;
  const int nv0 = FULL ? 8 : min(8, max(0, a.w - x0));
  const int nv1 = FULL ? 4 : min(4, max(0, a.lw[1] - (x0 >> 1)));
  uint32_t l1[4];
#pragma unroll
  for (int rp = 0; rp < 4; ++rp) {
    uint32_t gw[2][2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int i = 2 * rp + j;
      const bool row_ok = FULL || (y0 + i < a.h);
      uint32_t sa[4], sb[4];
      gw[j][0] = gray4(v[i][0].x, v[i][0].y, v[i][1].x, sa);
      gw[j][1] = gray4(v[i][1].y, v[i][2].x, v[i][2].y, sb);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (FULL || (row_ok && q < nv0)) hadd(hb | ((sa[q] >> 6) & 0x3fcu));
        if (FULL || (row_ok && 4 + q < nv0)) hadd(hb | ((sb[q] >> 6) & 0x3fcu));
      }
      const int row = 8 * r + i;
      *reinterpret_cast<uint2*>(slot + l0_addr(row, c >> 1) + 8 * (c & 1)) = make_uint2(gw[j][0], gw[j][1]);
    }
    if (a.n >= 2) {
      const uint32_t s0 = box_sum(gw[0][0], gw[1][0], 0), s1 = box_sum(gw[0][0], gw[1][0], 1);
      const uint32_t s2 = box_sum(gw[0][1], gw[1][1], 0), s3 = box_sum(gw[0][1], gw[1][1], 1);
      const bool row_ok = FULL || ((y0 >> 1) + rp < a.lh[1]);
      if (FULL || (row_ok && 0 < nv1)) hadd((hb + 1024) | (s0 & 0x3fcu));
      if (FULL || (row_ok && 1 < nv1)) hadd((hb + 1024) | (s1 & 0x3fcu));
      if (FULL || (row_ok && 2 < nv1)) hadd((hb + 1024) | (s2 & 0x3fcu));
      if (FULL || (row_ok && 3 < nv1)) hadd((hb + 1024) | (s3 & 0x3fcu));
      const uint32_t x01 = (s0 + (s1 << 16)) >> 2, x23 = (s2 + (s3 << 16)) >> 2;
      l1[rp] = __byte_perm(x01, x23, 0x6420);
    }
  }
  if (a.n < 3) return;
  uint32_t l2[2];
  {
    const int x2 = x0 >> 2, y2 = y0 >> 2;
    const int nv2 = FULL ? 2 : min(2, max(0, a.lw[2] - x2));
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint32_t s0 = box_sum(l1[2 * q], l1[2 * q + 1], 0), s1 = box_sum(l1[2 * q], l1[2 * q + 1], 1);
      const bool row_ok = FULL || (y2 + q < a.lh[2]);
      if (FULL || (row_ok && 0 < nv2)) hadd((hb + 2048) | (s0 & 0x3fcu));
      if (FULL || (row_ok && 1 < nv2)) hadd((hb + 2048) | (s1 & 0x3fcu));
      l2[q] = ((s0 >> 2) & 0xffu) | ((s1 << 6) & 0xff00u);
      *reinterpret_cast<unsigned short*>(slot + slot_off(2) + (2 * r + q) * 16 + 2 * c) = (unsigned short)l2[q];
    }
  }
  if (a.n < 4) return;
  uint32_t v3;
  {
    const uint32_t s = box_sum(l2[0], l2[1], 0);
    v3 = s >> 2;
    if (FULL || ((x0 >> 3) < a.lw[3] && (y0 >> 3) < a.lh[3])) hadd((hb + 3072) | (s & 0x3fcu));
    slot[slot_off(3) + r * 8 + c] = (uint8_t)v3;
  }
  if (a.n < 5) return;
  // level 4: 2x2 level-3 px of lanes (r, c), (r, c^1), (r^1, c), (r^1, c^1)
  uint32_t t4 = v3 + __shfl_xor_sync(0xffffffffu, v3, 1);
  t4 += __shfl_xor_sync(0xffffffffu, t4, 8);
  const uint32_t v4 = (t4 + 2u) >> 2;
  if ((lane & 9) == 0) {
    const int x4 = jx * 4 + (c >> 1), y4 = jy * 2 + (r >> 1);
    if (FULL || (x4 < a.lw[4] && y4 < a.lh[4])) hadd((hb + 4096) | (v4 << 2));
    slot[slot_off(4) + (r >> 1) * 4 + (c >> 1)] = (uint8_t)v4;
  }
  if (a.n < 6) return;
  // level 5: level-4 px live at lanes (r even, c even); pairs c^2 and r^2
  uint32_t t5 = v4 + __shfl_xor_sync(0xffffffffu, v4, 2);
  t5 += __shfl_xor_sync(0xffffffffu, t5, 16);
  const uint32_t v5 = (t5 + 2u) >> 2;
  if ((lane & 0x1b) == 0) {   // r in {0}, c in {0, 4}
    const int x5 = jx * 2 + (c >> 2), y5 = jy;
    if (FULL || (x5 < a.lw[5] && y5 < a.lh[5])) hadd((hb + 5120) | (v5 << 2));
    slot[slot_off(5) + (c >> 2)] = (uint8_t)v5;
  }
}

// Zero the map words of image `img` that K3 ORs into (levels 4..5: a word
// spans 8 / 16 jobs; its owner job, jx % 2^(k-1) == 0, clears it) and the
// row-padding words past the last job column (levels 1..5), for this job's
// rows.  Runs in K1(img); K3(img) starts only after the image's barrier.
__device__ __forceinline__ void res_zero_words(const ResArgs& a, int img, int jx, int jy, int lane) {
  uint32_t* mtb = a.mtb + (int64_t)img * a.bit_img_words32;
  uint32_t* excl = a.excl + (int64_t)img * a.bit_img_words32;
  if (lane < 3) {   // levels 4 (2 rows) and 5 (1 row): OR targets
    const int k = lane < 2 ? 4 : 5;
    const int row = lane < 2 ? lane : 0;
    if (k < a.n && (jx & ((1 << (k - 1)) - 1)) == 0) {
      const int y = ((jy * kJobRows) >> k) + row;
      if (y < a.lh[k]) {
        const int64_t o = a.bit_off32[k] + (int64_t)y * a.nw32[k] + (jx >> (k - 1));
        mtb[o] = 0u;
        excl[o] = 0u;
      }
    }
  }
  if (jx == a.jobs_x - 1) {
    // (level, row) combos of this job at levels 1..5: 16 + 8 + 4 + 2 + 1
    for (int f = lane; f < 31; f += 32) {
      const int k = f < 16 ? 1 : f < 24 ? 2 : f < 28 ? 3 : f < 30 ? 4 : 5;
      const int row = f - (k == 1 ? 0 : k == 2 ? 16 : k == 3 ? 24 : k == 4 ? 28 : 30);
      if (k >= a.n) continue;
      const int y = ((jy * kJobRows) >> k) + row;
      if (y >= a.lh[k]) continue;
      const int first = ((a.jobs_x - 1) >> (k - 1)) + 1;
      for (int j = first; j < a.nw32[k]; ++j) {
        const int64_t o = a.bit_off32[k] + (int64_t)y * a.nw32[k] + j;
        mtb[o] = 0u;
        excl[o] = 0u;
      }
    }
  }
}

// ---- K3: MTB + exclusion words of one job out of its slot -------------------
// Carry trick of pipe.cu th_word_t: g > med <=> byte carry-out of g + (255 -
// med); |g - med| > tol <=> carry-out of VABSDIFF4(g, med) + (255 - tol).
template <bool MED_LO>
__device__ __forceinline__ void res_th_word_fast(const uint32_t (&g)[8], const RTh& c, uint32_t ytl, int valid,
                                                 uint32_t& mw, uint32_t& ew) {
  constexpr uint32_t H = 0x80808080u, L7 = 0x7f7f7f7fu;
  constexpr uint32_t M4 = 0x00204081u << 4, M8 = 0x00204081u << 8;
  uint32_t m = 0, e = 0, pm = 0, pe = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t x = g[k];
    const uint32_t s = (x & L7) + c.yml;
    const uint32_t gm = MED_LO ? ((x | s) & H) : (x & s & H);
    uint32_t d;
    asm("vabsdiff4.u32.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(c.med), "r"(0u));
    const uint32_t sd = (d & L7) + ytl;
    const uint32_t ge = (d | sd) & H;   // tol <= 127
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
// Generic form (any median, any tolerance; per-lane constants).
__device__ __forceinline__ void res_th_word(const uint32_t (&g)[8], const RTh& c, uint32_t yt, uint32_t ytl,
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
    m |= ((gm * 0x00204081u) >> (28 - 4 * k)) & (0xfu << (4 * k));
    e |= ((ge * 0x00204081u) >> (28 - 4 * k)) & (0xfu << (4 * k));
  }
  const uint32_t keep = valid >= 32 ? 0xffffffffu : (valid <= 0 ? 0u : ((1u << valid) - 1u));
  mw = m & keep;
  ew = e & keep;
}

__device__ __forceinline__ void res_k3(const ResArgs& a, const RTh* th, uint32_t yt, uint32_t ytl, int img, int jx,
                                       int jy, int lane, const uint8_t* slot) {
  uint32_t* mtb = a.mtb + (int64_t)img * a.bit_img_words32;
  uint32_t* excl = a.excl + (int64_t)img * a.bit_img_words32;
  // ---- level 0: lane = job row, two words (px 0..31, 32..63)
  {
    const int y = jy * kJobRows + lane;
    const uint4 q0 = *reinterpret_cast<const uint4*>(slot + l0_addr(lane, 0));
    const uint4 q1 = *reinterpret_cast<const uint4*>(slot + l0_addr(lane, 1));
    const uint4 q2 = *reinterpret_cast<const uint4*>(slot + l0_addr(lane, 2));
    const uint4 q3 = *reinterpret_cast<const uint4*>(slot + l0_addr(lane, 3));
    const uint32_t g0[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
    const uint32_t g1[8] = {q2.x, q2.y, q2.z, q2.w, q3.x, q3.y, q3.z, q3.w};
    const int valid = a.w - jx * kJobPx;
    uint32_t m0, e0, m1, e1;
    const RTh c = th[0];
    if (a.tol > 127) {
      res_th_word(g0, c, yt, ytl, valid, m0, e0);
      res_th_word(g1, c, yt, ytl, valid - 32, m1, e1);
    } else if (c.med_lo) {
      res_th_word_fast<true>(g0, c, ytl, valid, m0, e0);
      res_th_word_fast<true>(g1, c, ytl, valid - 32, m1, e1);
    } else {
      res_th_word_fast<false>(g0, c, ytl, valid, m0, e0);
      res_th_word_fast<false>(g1, c, ytl, valid - 32, m1, e1);
    }
    if (y < a.h) {
      const int64_t o = a.bit_off32[0] + (int64_t)y * a.nw32[0] + 2 * jx;
      *reinterpret_cast<uint2*>(mtb + o) = make_uint2(m0, m1);
      *reinterpret_cast<uint2*>(excl + o) = make_uint2(e0, e1);
    }
  }
  if (a.n < 2) return;
  // ---- level 1, derived from the slot's level 0 (pyramid.py:17-32, the same
  //      nested rounding as K1): lane = (level-1 row lane >> 1, half lane & 1),
  //      16 px from 2 x 32 level-0 px; the two halves of a word meet by shuffle
  {
    const int r1 = lane >> 1, hf = lane & 1;
    const uint4 u0 = *reinterpret_cast<const uint4*>(slot + l0_addr(2 * r1, 2 * hf));
    const uint4 u1 = *reinterpret_cast<const uint4*>(slot + l0_addr(2 * r1, 2 * hf + 1));
    const uint4 d0 = *reinterpret_cast<const uint4*>(slot + l0_addr(2 * r1 + 1, 2 * hf));
    const uint4 d1 = *reinterpret_cast<const uint4*>(slot + l0_addr(2 * r1 + 1, 2 * hf + 1));
    const uint32_t uw[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
    const uint32_t dw[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
    uint32_t g[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const uint32_t xa = (box_sum(uw[2 * m], dw[2 * m], 0) + (box_sum(uw[2 * m], dw[2 * m], 1) << 16)) >> 2;
      const uint32_t xb = (box_sum(uw[2 * m + 1], dw[2 * m + 1], 0) + (box_sum(uw[2 * m + 1], dw[2 * m + 1], 1) << 16)) >> 2;
      g[m] = __byte_perm(xa, xb, 0x6420);
    }
    const int valid = min(16, a.lw[1] - (jx * (kJobPx / 2) + 16 * hf));
    uint32_t m, e;
    res_th_word(g, th[1], yt, ytl, valid, m, e);
    const uint32_t mo = __shfl_xor_sync(0xffffffffu, m, 1), eo = __shfl_xor_sync(0xffffffffu, e, 1);
    const int y = jy * (kJobRows / 2) + r1;
    if (hf == 0 && y < a.lh[1]) {
      const int64_t o = a.bit_off32[1] + (int64_t)y * a.nw32[1] + jx;
      mtb[o] = m | (mo << 16);
      excl[o] = e | (eo << 16);
    }
  }
  if (a.n < 3) return;
  // ---- levels 2..5 (OR-ed into words shared with neighbouring jobs): lanes
  //      0-7 level-2 rows (16 px), 8-11 level 3 (8 px), 12-13 level 4, 14 level 5
  const int k = lane < 8 ? 2 : lane < 12 ? 3 : lane < 14 ? 4 : lane < 15 ? 5 : 0;
  const int row = lane - (k == 2 ? 0 : k == 3 ? 8 : k == 4 ? 12 : 14);
  if (k == 0 || k >= a.n) return;
  const int y = ((jy * kJobRows) >> k) + row;
  if (y >= a.lh[k]) return;
  uint32_t g[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (k == 2) {
    const uint4 q0 = *reinterpret_cast<const uint4*>(slot + slot_off(2) + row * 16);
    g[0] = q0.x; g[1] = q0.y; g[2] = q0.z; g[3] = q0.w;
  } else if (k == 3) {
    const uint2 q0 = *reinterpret_cast<const uint2*>(slot + slot_off(3) + row * 8);
    g[0] = q0.x; g[1] = q0.y;
  } else if (k == 4) {
    g[0] = *reinterpret_cast<const uint32_t*>(slot + slot_off(4) + row * 4);
  } else {
    g[0] = *reinterpret_cast<const unsigned short*>(slot + slot_off(5));
  }
  const int npx = kJobPx >> k;                     // px of this level in the job's row
  const int valid = min(npx, a.lw[k] - ((jx * kJobPx) >> k));
  uint32_t m, e;
  res_th_word(g, th[k], yt, ytl, valid, m, e);
  const int64_t o = a.bit_off32[k] + (int64_t)y * a.nw32[k] + (jx >> (k - 1));
  const int part = jx & ((1 << (k - 1)) - 1);     // this job's part of the word
  if (k <= 3) {
    // levels 2 / 3: the job owns a half word / a byte of it (plain stores);
    // the last job of a row also clears the parts of the word no job covers
    const bool last = jx == a.jobs_x - 1;
    if (k == 2) {
      unsigned short* pm = reinterpret_cast<unsigned short*>(mtb + o) + part;
      unsigned short* pe = reinterpret_cast<unsigned short*>(excl + o) + part;
      pm[0] = (unsigned short)m;
      pe[0] = (unsigned short)e;
      if (last && part == 0) {
        pm[1] = 0;
        pe[1] = 0;
      }
    } else {
      uint8_t* pm = reinterpret_cast<uint8_t*>(mtb + o);
      uint8_t* pe = reinterpret_cast<uint8_t*>(excl + o);
      pm[part] = (uint8_t)m;
      pe[part] = (uint8_t)e;
      if (last)
        for (int b = part + 1; b < 4; ++b) {
          pm[b] = 0;
          pe[b] = 0;
        }
    }
  } else {
    // levels 4 / 5: 4 / 2 bits per job, OR-ed into words cleared in K1
    const int sh = npx * part;
    if (m) atomicOr(mtb + o, m << sh);
    if (e) atomicOr(excl + o, e << sh);
  }
}

// Lower median of one level's histogram (threshold.py:31-39): the smallest m
// with cumsum[m] >= (total + 1) / 2.  One warp; lane owns bins 8 lane .. +7.
__device__ __forceinline__ int res_warp_median(const uint32_t (&bins)[8], int lane) {
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += bins[i];
  uint32_t incl = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  const uint32_t target = (total + 1) >> 1;
  const unsigned mask = __ballot_sync(0xffffffffu, incl >= target);
  if (total == 0) return 0;
  const int L = __ffs(mask) - 1;
  int med = 0;
  if (lane == L) {
    uint32_t cacc = incl - s;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      cacc += bins[i];
      if (cacc >= target && med == 0 && cacc - bins[i] < target) med = lane * 8 + i;
    }
  }
  return __shfl_sync(0xffffffffu, med, L);
}

// Histogram reduction without atomics (same-line REDs from 148 CTAs queue at
// the L2 slice for tens of microseconds, and the median is on the critical
// path here):
//   1. the CTA that finishes its K1 jobs of image s stores its partial
//      histograms (plain coalesced stores) into part[s & 1][cta], arrives on
//      arrive[s]; the last to arrive raises every CTA's flag word 0;
//   2. each CTA sums its ~10 bins over all partials into tot[s & 1], arrives
//      on arrive2[s]; the last derives the n medians (threshold.py:31-39),
//      writes them into every CTA's line (words 2..7) and raises word 1.
// Per-CTA 128-B flag lines: no hot spot for the 148 pollers.
__device__ __forceinline__ uint32_t* part_hist(const ResArgs& a, int s, int c) {
  return a.part + ((int64_t)(s & 1) * gridDim.x + c) * (kRMaxLevels * 256);
}

__device__ __noinline__ void res_flush_hist(const ResArgs& a, int s, int lane, uint32_t hb) {
  uint4* sh = reinterpret_cast<uint4*>(__cvta_shared_to_generic(hb));
  uint4* dst = reinterpret_cast<uint4*>(part_hist(a, s, blockIdx.x));
  for (int i = lane; i < a.n * 64; i += 32) {
    dst[i] = sh[i];
    sh[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  __syncwarp();
  int last = 0;
  if (lane == 0) {
    __threadfence();
    last = r_atom_add_acqrel(a.arrive + s, 1u) == gridDim.x - 1;
    RTRACE(a, s, 1);
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();
  for (int c = lane; c < (int)gridDim.x; c += 32) r_st_relaxed(a.medflag + (int64_t)c * 32, (uint32_t)s + 1u);
}

// Phase 2 (the claimer warp of each CTA): this CTA's bins of the total, then
// the medians (the last CTA).  Returns after the CTA's line holds them.
__device__ __noinline__ void res_reduce_hist(const ResArgs& a, int s, int lane) {
  const int G = gridDim.x, c = blockIdx.x;
  uint32_t* line = a.medflag + (int64_t)c * 32;
  if (lane == 0) {
    while (r_ld_relaxed(line) < (uint32_t)s + 1u) __nanosleep(64);
    RTRACE(a, s, 6);
    r_fence_acquire();
  }
  __syncwarp();
  const int nb = a.n * 256;
  const int b0 = (int)((int64_t)c * nb / G), b1 = (int)((int64_t)(c + 1) * nb / G);
  uint32_t* tot = a.tot + (int64_t)(s & 1) * (kRMaxLevels * 256);
  for (int b = b0; b < b1; ++b) {
    uint32_t v = 0;
    for (int cc = lane; cc < G; cc += 32) v += __ldcg(part_hist(a, s, cc) + b);
    v = warp_sum(v);
    if (lane == 0) tot[b] = v;
  }
  __syncwarp();
  int last = 0;
  if (lane == 0) {
    __threadfence();
    last = r_atom_add_acqrel(a.arrive2 + s, 1u) == (uint32_t)G - 1;
    RTRACE(a, s, 4);
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (last) {
    uint32_t bins[kRMaxLevels][8];
#pragma unroll
    for (int k = 0; k < kRMaxLevels; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) bins[k][i] = k < a.n ? __ldcg(tot + k * 256 + lane * 8 + i) : 0u;
    int meds = 0;   // lane k holds level k's median
#pragma unroll
    for (int k = 0; k < kRMaxLevels; ++k) {
      if (k >= a.n) break;
      const int med = res_warp_median(bins[k], lane);
      if (lane == k) meds = med;
    }
    if (lane < a.n) a.medians[(int64_t)s * a.n + lane] = meds;
    uint32_t mk[kRMaxLevels];
#pragma unroll
    for (int k = 0; k < kRMaxLevels; ++k) mk[k] = (uint32_t)__shfl_sync(0xffffffffu, meds, k);
    for (int cc = lane; cc < G; cc += 32)
#pragma unroll
      for (int k = 0; k < kRMaxLevels; ++k)
        if (k < a.n) a.medflag[(int64_t)cc * 32 + 2 + k] = mk[k];
    __syncwarp();
    __threadfence();
    for (int cc = lane; cc < G; cc += 32) r_st_relaxed(a.medflag + (int64_t)cc * 32 + 1, (uint32_t)s + 1u);
    if (lane == 0) RTRACE(a, s, 5);
  }
  if (lane == 0) {
    while (r_ld_relaxed(line + 1) < (uint32_t)s + 1u) __nanosleep(64);
    r_fence_acquire();
  }
  __syncwarp();
}

// Threshold constants of image s in shared memory: the first warp that needs
// them waits for the CTA's flag (every CTA has flushed image s), sums the
// histogram copies and derives all n medians (threshold.py:31-39); it also
// clears this CTA's share of ring slot s + 2 (image s - 2's, read by every
// CTA before image s could complete).
__device__ __forceinline__ const RTh* res_need_medians(const ResArgs& a, ResShared& S, int s, int lane) {
  const int par = s & 1;
  const int want = s + 1, prev = s >= 2 ? s - 1 : 0;   // claims of one parity go s-2 -> s
  for (;;) {
    // role (decided by lane 0, warp-uniform): 2 = constants ready, 1 = this
    // warp computes them, 0 = wait (claimed elsewhere, or image s-2 unclaimed)
    int role = 0;
    if (lane == 0) {
      if (r_ld_acquire_cta(&S.medtag[par]) == want) {
        role = 2;
      } else {
        const int cur = *reinterpret_cast<volatile int*>(&S.medclaim[par]);
        if (cur == prev && atomicCAS(&S.medclaim[par], prev, want) == prev) role = 1;
      }
    }
    role = __shfl_sync(0xffffffffu, role, 0);
    if (role == 2) break;
    if (role == 1) {
      res_reduce_hist(a, s, lane);
      if (lane < a.n) {
        const int med = (int)__ldcg(a.medflag + (int64_t)blockIdx.x * 32 + 2 + lane);
        RTh c;
        c.med = (uint32_t)med * 0x01010101u;
        c.ym = (uint32_t)(255 - med) * 0x01010101u;
        c.yml = c.ym & 0x7f7f7f7fu;
        c.med_lo = med <= 127;
        S.th[par][lane] = c;
      }
      __syncwarp();
      if (lane == 0) {
        RTRACE(a, s, 2);
        r_st_release_cta(&S.medtag[par], want);
      }
      __syncwarp();
      break;
    }
    __nanosleep(128);
  }
  __syncwarp();
  return S.th[par];
}

// ---- K4: one search task = 32 output rows x 32 words of one (pair, level) ---
// Candidate i = (ddy + 1) * 3 + (ddx + 1) counts
//   popc((A ^ B_shift) & EA & EB_shift) over the task's words, with B the
// target map translated by (bx + ddx, by + ddy) (kernels/_native.pyx:73-111).
// Lane = output word j; staged words w_i = W[j - qb - 2 + i] (i = 0..3) of a
// source row come from one coalesced row load plus three edge words, spread
// by shuffles; the 3-row window slides down the task.
// Raw loads of one output row: the target source row's word jb + lane
// (+ edge words jb + 32 + lane, lanes 0..2) of both target maps, and the
// reference words of the output row.
struct RawRow {
  uint32_t u, u2, ue, ue2, a, ea;
};

__device__ __forceinline__ RawRow raw_row(const uint32_t* A, const uint32_t* EA, const uint32_t* B,
                                          const uint32_t* EB, int y, int s, int y1, int lh, int nw, int jb, int j,
                                          int lane) {
  RawRow r;
  const bool yok = y < y1;
  const bool rok = yok && s >= 0 && s < lh;
  const int64_t ro = (int64_t)(rok ? s : 0) * nw;
  const int j0 = jb + lane, j1 = j0 + 32;
  const bool c0 = rok && j0 >= 0 && j0 < nw;
  const bool c1 = rok && lane < 3 && j1 >= 0 && j1 < nw;
  r.u = c0 ? __ldcg(B + ro + j0) : 0u;
  r.ue = c0 ? __ldcg(EB + ro + j0) : 0u;
  r.u2 = c1 ? __ldcg(B + ro + j1) : 0u;
  r.ue2 = c1 ? __ldcg(EB + ro + j1) : 0u;
  const bool aok = yok && j < nw;
  const int64_t ao = (int64_t)(aok ? y : 0) * nw + (aok ? j : 0);
  r.a = aok ? __ldcg(A + ao) : 0u;
  r.ea = aok ? __ldcg(EA + ao) : 0u;
  return r;
}

// The three candidate words (ddx = -1, 0, +1) of a source row, both maps.
// CASE 0: rbx == 0 (staged words w1, w2, w3), 1: rbx == 31 (w0, w1, w2),
// 2: other (w1, w2); staged word w_i = W[j - qb - 2 + i] comes from lane + i.
template <int CASE>
__device__ __forceinline__ void shifted3(const RawRow& r, int rbx, int lane, uint32_t (&sb)[3], uint32_t (&se)[3]) {
  auto word = [&](uint32_t x, uint32_t x2, int i) {
    const uint32_t p = __shfl_sync(0xffffffffu, x, (lane + i) & 31);
    const uint32_t q = __shfl_sync(0xffffffffu, x2, (lane + i) & 31);
    return lane + i < 32 ? p : q;
  };
  const uint32_t b1 = word(r.u, r.u2, 1), b2 = word(r.u, r.u2, 2);
  const uint32_t e1 = word(r.ue, r.ue2, 1), e2 = word(r.ue, r.ue2, 2);
  if (CASE == 0) {
    const uint32_t b3 = word(r.u, r.u2, 3), e3 = word(r.ue, r.ue2, 3);
    sb[0] = shifted_word(b2, b3, 31); se[0] = shifted_word(e2, e3, 31);
    sb[1] = shifted_word(b1, b2, 0); se[1] = shifted_word(e1, e2, 0);
    sb[2] = shifted_word(b1, b2, 1); se[2] = shifted_word(e1, e2, 1);
  } else if (CASE == 1) {
    sb[0] = shifted_word(b1, b2, 30); se[0] = shifted_word(e1, e2, 30);
    sb[1] = shifted_word(b1, b2, 31); se[1] = shifted_word(e1, e2, 31);
    sb[2] = shifted_word(r.u, b1, 0); se[2] = shifted_word(r.ue, e1, 0);
  } else {
    sb[0] = shifted_word(b1, b2, rbx - 1); se[0] = shifted_word(e1, e2, rbx - 1);
    sb[1] = shifted_word(b1, b2, rbx); se[1] = shifted_word(e1, e2, rbx);
    sb[2] = shifted_word(b1, b2, rbx + 1); se[2] = shifted_word(e1, e2, rbx + 1);
  }
}

// Output rows y0..y1-1: row y needs source rows y - by + 1 (ddy = -1),
// y - by (0), y - by - 1 (+1); a 3-row window of shifted words slides down.
// Loads run kRPre rows ahead (two register blocks) so the L2 latency is
// covered by the compare work of the block before.
constexpr int kRPre = 4;
template <int CASE>
__device__ __forceinline__ void res_search_rows(const uint32_t* A, const uint32_t* EA, const uint32_t* B,
                                                const uint32_t* EB, int y0, int y1, int by, int rbx, int lh, int nw,
                                                int jb, int j, int lane, unsigned (&cnt)[9]) {
  uint32_t b0[3], e0[3], b1[3], e1[3];
  {
    const RawRow r0 = raw_row(A, EA, B, EB, y0, y0 - by - 1, y1, lh, nw, jb, j, lane);
    const RawRow r1 = raw_row(A, EA, B, EB, y0, y0 - by, y1, lh, nw, jb, j, lane);
    shifted3<CASE>(r0, rbx, lane, b0, e0);
    shifted3<CASE>(r1, rbx, lane, b1, e1);
  }
  RawRow cur[kRPre];
#pragma unroll
  for (int i = 0; i < kRPre; ++i) cur[i] = raw_row(A, EA, B, EB, y0 + i, y0 + i - by + 1, y1, lh, nw, jb, j, lane);
#pragma unroll 1
  for (int yb = y0; yb < y1; yb += kRPre) {
    RawRow nxt[kRPre];
#pragma unroll
    for (int i = 0; i < kRPre; ++i) {
      const int y = yb + kRPre + i;
      nxt[i] = raw_row(A, EA, B, EB, y, y - by + 1, y1, lh, nw, jb, j, lane);
    }
#pragma unroll
    for (int i = 0; i < kRPre; ++i) {
      if (yb + i >= y1) break;
      uint32_t b2[3], e2[3];
      shifted3<CASE>(cur[i], rbx, lane, b2, e2);
      const uint32_t av = cur[i].a, ev = cur[i].ea;
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
#pragma unroll
    for (int i = 0; i < kRPre; ++i) cur[i] = nxt[i];
  }
}

__device__ __forceinline__ void res_append(const ResArgs& a, uint32_t code) {
  const uint32_t pos = atomicAdd(a.qtail, 1u);
  r_st_release(a.qitem + pos, code);
}

__device__ __forceinline__ void res_search_task(const ResArgs& a, int p, int k, int task, int lane) {
  const int n = a.n;
  const int nw = a.nw32[k], lh = a.lh[k];
  const int strips = a.strips[k];
  const int rb = task / strips, cs = task - rb * strips;
  const int y0 = rb * kRSearchRows, y1 = min(y0 + kRSearchRows, lh);
  const int j = cs * 32 + lane;
  int bx = 0, by = 0;
  if (k + 1 < n) {
    const int32_t* prev = a.acc + ((int64_t)p * n + (k + 1)) * 2;
    bx = 2 * __ldcg(prev);
    by = 2 * __ldcg(prev + 1);
  }
  const int ref = __ldg(a.pairs + 2 * p), tgt = __ldg(a.pairs + 2 * p + 1);
  const uint32_t* A = a.mtb + (int64_t)ref * a.bit_img_words32 + a.bit_off32[k];
  const uint32_t* EA = a.excl + (int64_t)ref * a.bit_img_words32 + a.bit_off32[k];
  const uint32_t* B = a.mtb + (int64_t)tgt * a.bit_img_words32 + a.bit_off32[k];
  const uint32_t* EB = a.excl + (int64_t)tgt * a.bit_img_words32 + a.bit_off32[k];
  const int qb = bx >> 5, rbx = bx & 31;
  const int jb = cs * 32 - qb - 2;   // lane's staged word 0 = W[j - qb - 2]
  unsigned cnt[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) cnt[i] = 0;
  if (rbx == 0)
    res_search_rows<0>(A, EA, B, EB, y0, y1, by, rbx, lh, nw, jb, j, lane, cnt);
  else if (rbx == 31)
    res_search_rows<1>(A, EA, B, EB, y0, y1, by, rbx, lh, nw, jb, j, lane, cnt);
  else
    res_search_rows<2>(A, EA, B, EB, y0, y1, by, rbx, lh, nw, jb, j, lane, cnt);
  unsigned long long* errs = a.errs + ((int64_t)p * n + k) * 9;
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const unsigned v = warp_sum(cnt[i]);
    if (lane == i && v) atomicAdd(errs + i, (unsigned long long)v);
  }
  __syncwarp();
  int last = 0;
  if (lane == 0) {
    __threadfence();
    last = atomicAdd(a.done + (int64_t)p * n + k, 1u) == (unsigned)a.tasks[k] - 1;
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  // the level's last task: search.py:67 key (err, |ddx| + |ddy|, index)
  if (lane == 0) {
    __threadfence();
    int best = 0, bd = 0;
    unsigned long long be = 0;
    for (int i = 0; i < 9; ++i) {
      const unsigned long long e = __ldcg(errs + i);
      const int d = abs(i % 3 - 1) + abs(i / 3 - 1);
      if (i == 0 || e < be || (e == be && d < bd)) {
        best = i;
        be = e;
        bd = d;
      }
    }
    int32_t* out = a.acc + ((int64_t)p * n + k) * 2;
    out[0] = bx + best % 3 - 1;
    out[1] = by + best / 3 - 1;
    if (k > 0) {
      __threadfence();
      res_append(a, (uint32_t)(p * 8 + (k - 1)) + 1u);
    }
  }
  __syncwarp();
}

// Search worker loop: take tasks from the global queue in append order until
// all P x n entries are appended and fully claimed.
__device__ __forceinline__ void res_search_loop(const ResArgs& a, int lane) {
#ifdef RES_EXP_NO_SEARCH   // experiment builds only (tools/build_exp.sh): preprocess alone
  return;
#endif
  const int total = a.n_pairs * a.n;
  int head = 0;
  while (head < total) {
    uint32_t it = 0;
    if (lane == 0) {
      it = r_ld_relaxed(a.qitem + head);
      if (it) r_fence_acquire();
    }
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it == 0) {
      __nanosleep(512);
      continue;
    }
    const int p = (int)((it - 1) >> 3), k = (int)((it - 1) & 7);
    int t = 0;
    if (lane == 0) t = (int)atomicAdd(a.qclaim + head, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= a.tasks[k]) {
      ++head;
      continue;
    }
    res_search_task(a, p, k, t, lane);
  }
}

__global__ void __launch_bounds__(kRThreads, 1) res_kernel(const __grid_constant__ ResArgs a,
                                                             const __grid_constant__ CUtensorMap rgb_map) {
  extern __shared__ __align__(1024) uint8_t res_dyn[];   // [stages][kStageBytes] then [nc][kSlotBytes]
  __shared__ __align__(1024) uint32_t s_hist[6][256];   // this CTA's histograms of the image in K1
  __shared__ ResShared S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, c = blockIdx.x;
  const int j0 = (int)((int64_t)c * a.jobs / G);
  const int nc = (int)((int64_t)(c + 1) * a.jobs / G) - j0;   // jobs (= slots) of this CTA per image
  const int nst = a.stages;
  const int n_img = a.n_img;
  uint8_t* stages = res_dyn;
  uint8_t* slots = res_dyn + (size_t)nst * kStageBytes;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  // TMA tile copy of job q's RGB (q = s * nc + jl) into stage q % nst; one lane.
  auto issue = [&](int q) {
    const int s = q / nc, jl = q - s * nc;
    if (s >= n_img) return;
    if (a.img_ready && *reinterpret_cast<volatile int*>(&S.ready_img) < s) {   // streamed input: H2D landed
      r_spin_geq(a.img_ready + s, 1u, 128);
      atomicMax(&S.ready_img, s);
    }
    const int job = j0 + jl, jy = job / a.jobs_x, jx = job - jy * a.jobs_x;
    const int st = q % nst;
    *reinterpret_cast<volatile int*>(&S.stage_job[st]) = q;
    mbar_expect_tx(&S.full[st], (uint32_t)kStageBytes);
    tma_tile(stages + (size_t)st * kStageBytes, &rgb_map, (3 * kJobPx / 4) * jx, kJobRows * jy, s, &S.full[st], pol);
  };
  for (int i = tid; i < 6 * 256; i += kRThreads) (&s_hist[0][0])[i] = 0u;
  if (tid < 2) {
    S.medtag[tid] = 0;
    S.medclaim[tid] = 0;
    S.k1cnt[tid] = 0;
    S.k3cnt[tid] = 0;
  }
  if (tid == 0) {
    S.claim = 0;
    S.ready_img = a.img_ready ? -1 : 0x7fffffff;
    for (int st = 0; st < nst; ++st) {
      mbar_init(&S.full[st], 1);
      S.stage_job[st] = -1;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (nc > 0)
      for (int q = 0; q < nst; ++q) issue(q);
  }
  __syncthreads();
  if (warp >= kRK1Warps || nc == 0) {
    res_search_loop(a, lane);
    return;
  }
  const uint32_t yt = (uint32_t)(255 - a.tol) * 0x01010101u, ytl = yt & 0x7f7f7f7fu;
  const uint32_t hb = smem_addr(&s_hist[0][0]);
  // Job sequence of this CTA: q = s * nc + jl for images s = 0..n_img-1, then
  // the drain (s = n_img: K3 of the last image only).
  for (;;) {
    int q = 0;
    if (lane == 0) q = atomicAdd(&S.claim, 1);
    q = __shfl_sync(0xffffffffu, q, 0);
    const int s = q / nc, jl = q - s * nc;
    if (s > n_img) break;
    const int job = j0 + jl;
#ifdef RES_EXP_TRACE
    if (jl == 0 && lane == 0 && s < n_img) rtrace(a, s, 0);
#endif
    const int jy = job / a.jobs_x, jx = job - jy * a.jobs_x;
    const bool full = (jx + 1) * kJobPx <= a.w && (jy + 1) * kJobRows <= a.h;
    uint8_t* slot = slots + (size_t)jl * kSlotBytes;
    uint2 v[8][3];
    if (s < n_img) {
      // this job's RGB: wait for its stage, copy the block to registers,
      // refill the stage with job q + nst
      const int st = q % nst;
      if (lane == 0)
        while (*reinterpret_cast<volatile int*>(&S.stage_job[st]) != q) __nanosleep(20);
      __syncwarp();
      mbar_wait(&S.full[st], (uint32_t)(q / nst) & 1u);
      stage_to_regs(stages + (size_t)st * kStageBytes, lane, v);
      __syncwarp();
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(q + nst);
      }
    }
    if (s > 0) {
      // K3 of image s-1 out of this slot
      const RTh* th = res_need_medians(a, S, s - 1, lane);
      res_k3(a, th, yt, ytl, s - 1, jx, jy, lane, slot);
      __syncwarp();
      int last = 0;
      if (lane == 0) last = r_smem_add_acqrel(&S.k3cnt[(s - 1) & 1], 1) == nc - 1;
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last && lane == 0) {
        S.k3cnt[(s - 1) & 1] = 0;
        RTRACE(a, s - 1, 3);
        __threadfence();
        if (r_atom_add_acqrel(a.k3done + (s - 1), 1u) == (uint32_t)G - 1) {
          // every CTA wrote image s-1's maps: level n-1 of the pairs it completes
          const int p0 = __ldg(a.ready_start + (s - 1)), p1 = __ldg(a.ready_start + s);
          for (int qq = p0; qq < p1; ++qq) res_append(a, (uint32_t)(__ldg(a.ready_pairs + qq) * 8 + (a.n - 1)) + 1u);
        }
      }
    }
    if (s == n_img) continue;   // drain job: K3 only
    if (full)
      res_k1<true>(a, v, jx, jy, lane, slot, hb);
    else
      res_k1<false>(a, v, jx, jy, lane, slot, hb);
    res_zero_words(a, s, jx, jy, lane);
    __syncwarp();
    int last = 0;
    if (lane == 0) last = r_smem_add_acqrel(&S.k1cnt[s & 1], 1) == nc - 1;
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      if (lane == 0) S.k1cnt[s & 1] = 0;
      res_flush_hist(a, s, lane, hb);
    }
  }
  res_search_loop(a, lane);
}

// Uploads host tables through kernel parameters (graph-capturable, no
// pageable memcpy): dst[off + i] = v[i], i < n.
struct ResUpload {
  int32_t v[2 * kRMaxPairsPerUpload];
};
__global__ void res_upload_kernel(int32_t* dst, int n, const __grid_constant__ ResUpload u) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = u.v[i];
}

PFN_cuTensorMapEncodeTiled_v12000 k1_encode_tiled();

}  // namespace mtb

using namespace mtb;

static int res_jobs(int w, int h) { return ((w + kJobPx - 1) / kJobPx) * ((h + kJobRows - 1) / kJobRows); }

// Largest per-CTA job count the shared-memory slots hold.
// Static shared memory of res_kernel (histograms + control) and the stage
// ring depth that fits beside nc slots (0 if fewer than 3 stages fit).
static int res_static_smem() { return 8 * 1024; }   // s_hist (6 KB, 1 KB-aligned) + ResShared, rounded up
static int res_stages(int nc) {
  const int room = kRSmemLimit - res_static_smem() - nc * kSlotBytes;
  const int st = room / kStageBytes;
  return st < 3 ? 0 : std::min(st, kRMaxStages);
}

extern "C" int mtb_resident_supported(int w, int h, int levels, int64_t rgb_pitch, int64_t rgb_img_stride) {
  Plan p;
  if (!make_plan(w, h, levels, &p) || p.n > kRMaxLevels) return 0;
  // TMA: 16-B aligned rows and image strides; whole 16-px groups per row
  if (w % 16 != 0 || rgb_pitch % 16 != 0 || rgb_img_stride % 16 != 0 || rgb_pitch < 3 * (int64_t)w) return 0;
  if (k1_encode_tiled() == nullptr) return 0;
  const int jobs = res_jobs(w, h);
  const int per = (jobs + num_sms() - 1) / num_sms();
  return res_stages(per) > 0 ? 1 : 0;
}

extern "C" int64_t mtb_resident_sync_words(int n_img, int n_pairs, int levels) {
  const int64_t L = levels < 1 ? 1 : (levels > kRMaxLevels ? kRMaxLevels : levels);
  // part [2][G][1536]; tot [2][1536]; arrive, arrive2, k3done [n_img]; qitem, qclaim [P*L];
  // qtail (+pad 31); medflag [G][32]; pairs [2P]; ready_pairs [P]; ready_start [n_img+1]
  return 2 * (int64_t)num_sms() * 1536 + 2 * 1536 + 3 * (int64_t)n_img + 2 * (int64_t)n_pairs * L + 32 +
         32 * (int64_t)num_sms() + 3 * (int64_t)n_pairs + n_img + 1;
}

static int res_upload(int32_t* dst, const std::vector<int32_t>& v, cudaStream_t st) {
  ResUpload u;
  for (size_t off = 0; off < v.size(); off += 2 * kRMaxPairsPerUpload) {
    const int cnt = (int)std::min<size_t>(2 * kRMaxPairsPerUpload, v.size() - off);
    std::memcpy(u.v, v.data() + off, sizeof(int32_t) * cnt);
    res_upload_kernel<<<1, 256, 0, st>>>(dst + off, cnt, u);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_error(std::string("res_upload_kernel: ") + cudaGetErrorString(e));
      return MTB_ECUDA;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  return MTB_OK;
}

// The resident path of mtb_align_fused_ex (the caller validated arguments).
int mtb_resident_run(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride, int w, int h, int n_img,
                     int levels, int tol, const int32_t* pairs_host, int n_pairs, uint32_t* hist_ws,
                     int32_t* medians, uint64_t* mtb, uint64_t* exclusion, int32_t* acc, unsigned long long* errs,
                     uint32_t* done, uint32_t* sync_ws, const uint32_t* img_ready, void* stream) {
  Plan p;
  MTB_REQUIRE(make_plan(w, h, levels, &p), "image must be at least 16x16 and levels >= 1");
  cudaStream_t st = as_stream(stream);
  ResArgs a;
  std::memset(&a, 0, sizeof(a));
  a.rgb = rgb;
  a.rgb_pitch = rgb_pitch;
  a.rgb_img_stride = rgb_img_stride;
  a.w = w;
  a.h = h;
  a.n = p.n;
  a.tol = tol;
  for (int k = 0; k < kRMaxLevels; ++k) {
    a.lw[k] = k < p.n ? p.lv[k].w : 0;
    a.lh[k] = k < p.n ? p.lv[k].h : 0;
    a.nw32[k] = k < p.n ? (int)(2 * p.lv[k].nw64) : 0;
    a.bit_off32[k] = k < p.n ? 2 * p.lv[k].bit_off : 0;
    a.strips[k] = k < p.n ? (a.nw32[k] + 31) / 32 : 1;
    a.tasks[k] = k < p.n ? a.strips[k] * ((a.lh[k] + kRSearchRows - 1) / kRSearchRows) : 0;
  }
  a.bit_img_words32 = 2 * p.bit_img_words;
  a.jobs_x = (w + kJobPx - 1) / kJobPx;
  a.jobs = res_jobs(w, h);
  a.n_img = n_img;
  a.mtb = reinterpret_cast<uint32_t*>(mtb);
  a.excl = reinterpret_cast<uint32_t*>(exclusion);
  a.medians = medians;
  a.n_pairs = n_pairs;
  a.acc = acc;
  a.errs = errs;
  a.done = done;
  a.img_ready = img_ready;
  // sync_ws layout (mtb_resident_sync_words)
  uint32_t* w32 = sync_ws;
  a.part = w32;
  a.tot = a.part + 2 * (int64_t)num_sms() * 1536;
  a.arrive = a.tot + 2 * 1536;
  a.arrive2 = a.arrive + n_img;
  a.k3done = a.arrive2 + n_img;
  a.qitem = a.k3done + n_img;
  a.qclaim = a.qitem + (int64_t)n_pairs * p.n;
  a.qtail = a.qclaim + (int64_t)n_pairs * p.n;
  a.medflag = a.qtail + 32;
  int32_t* tab = reinterpret_cast<int32_t*>(a.medflag + 32 * (int64_t)num_sms());
  const int64_t zero_words = (int64_t)(tab - reinterpret_cast<int32_t*>(sync_ws));
  int32_t* d_pairs = tab;
  int32_t* d_ready = d_pairs + 2 * (int64_t)n_pairs;
  int32_t* d_start = d_ready + n_pairs;
  a.pairs = d_pairs;
  a.ready_pairs = d_ready;
  a.ready_start = d_start;
  // host tables: pairs sorted by the image whose maps complete them
  std::vector<int32_t> tbl;
  tbl.reserve(3 * (size_t)n_pairs + n_img + 1);
  for (int q = 0; q < 2 * n_pairs; ++q) tbl.push_back(pairs_host[q]);
  std::vector<int32_t> order(n_pairs);
  for (int q = 0; q < n_pairs; ++q) order[q] = q;
  auto mx = [&](int q) { return std::max(pairs_host[2 * q], pairs_host[2 * q + 1]); };
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return mx(x) < mx(y); });
  for (int q = 0; q < n_pairs; ++q) tbl.push_back(order[q]);
  {
    int q = 0;
    for (int s = 0; s <= n_img; ++s) {
      while (q < n_pairs && mx(order[q]) < s) ++q;
      tbl.push_back(q);
    }
  }
  if (n_pairs > 0) {
    MTB_CUDA(cudaMemsetAsync(errs, 0, sizeof(unsigned long long) * 9 * p.n * n_pairs, st));
    MTB_CUDA(cudaMemsetAsync(done, 0, sizeof(uint32_t) * p.n * n_pairs, st));
  }
  MTB_CUDA(cudaMemsetAsync(sync_ws, 0, sizeof(uint32_t) * zero_words, st));
  int rc = res_upload(tab, tbl, st);
  if (rc != MTB_OK) return rc;

  const int grid = std::min(num_sms(), a.jobs);   // every CTA owns >= 1 job (the barrier counts CTAs)
  const int nc = (a.jobs + grid - 1) / grid;
  a.stages = res_stages(nc);
  MTB_REQUIRE(a.stages > 0, "image too large for the resident path");
  const int smem = a.stages * kStageBytes + nc * kSlotBytes;
  CUtensorMap map;
  {
    const cuuint64_t dims[3] = {(cuuint64_t)(3 * (int64_t)w / 4), (cuuint64_t)h, (cuuint64_t)n_img};
    const cuuint64_t strides[2] = {(cuuint64_t)rgb_pitch, (cuuint64_t)rgb_img_stride};
    const cuuint32_t box[3] = {3 * kJobPx / 4, kJobRows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = k1_encode_tiled()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, (void*)rgb, dims, strides, box,
                                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed for the RGB batch");
      return MTB_ECUDA;
    }
  }
  MTB_CUDA(cudaFuncSetAttribute(res_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kRThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;   // every CTA co-resident: the per-image barrier spins
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#ifdef RES_EXP_TRACE
  const char* tpath = getenv("MTB_RES_TRACE");
  const size_t tbytes = sizeof(unsigned long long) * 8 * (size_t)n_img * grid;
  a.trace = nullptr;
  if (tpath) {
    MTB_CUDA(cudaMalloc(&a.trace, tbytes));
    MTB_CUDA(cudaMemsetAsync(a.trace, 0, tbytes, st));
  }
#endif
  const cudaError_t e = cudaLaunchKernelEx(&cfg, res_kernel, a, map);
  if (e != cudaSuccess) {
    set_error(std::string("res_kernel: ") + cudaGetErrorString(e));
    return MTB_ECUDA;
  }
#ifdef RES_EXP_TRACE
  if (tpath) {
    std::vector<unsigned long long> h(tbytes / 8);
    MTB_CUDA(cudaStreamSynchronize(st));
    MTB_CUDA(cudaMemcpy(h.data(), a.trace, tbytes, cudaMemcpyDeviceToHost));
    cudaFree(a.trace);
    FILE* f = fopen(tpath, "wb");
    if (f) {
      const int hdr[2] = {n_img, grid};
      fwrite(hdr, sizeof(int), 2, f);
      fwrite(h.data(), 1, tbytes, f);
      fclose(f);
    }
  }
#endif
  return check_launch("res_kernel", 1);
}
