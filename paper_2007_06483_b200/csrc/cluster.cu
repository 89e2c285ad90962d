// Small-image preprocess in ONE launch with the gray pyramid kept on chip:
// RGB8 -> gray -> 2x box pyramid -> per-level histograms -> medians ->
// MTB / exclusion bitmaps.  The gray pyramid of one image lives in the
// shared memory of a thread-block cluster (C CTAs, DSMEM) and never touches
// HBM, so the path moves the compulsory bytes only: RGB in, bitmaps out.
//
// Reference semantics (bit-exact, as the staged kernels): image.py:58-68
// (gray), pyramid.py:17-62 (levels), threshold.py:25-56 (histogram, lower
// median, MTB and exclusion bits), bitmap.py:32-40 (LSB-first packing).
//
// Design (sm_100a):
//  * One CTA per SM, clusters of C CTAs, persistent over images: cluster q
//    handles images q, q + nq, ...; CTA rank r owns the contiguous range of
//    32x256 tiles [r T / C, (r+1) T / C) of each image (T tiles per image).
//  * Phase A (per image): G groups of 128 threads stream their tiles with one
//    TMA 3-D copy each (1 ring stage per group, 24 KB; the refill is issued as
//    soon as the group has pulled the tile into registers, and the last tile
//    of an image prefetches the group's first tile of the next image, so the
//    loads run under phases B and C).  Gray levels 0..3 go to a tile-major
//    shared slot (k1_block_tm<SMEM>), histograms to shared memory
//    (ATOMS.POPC.INC); levels 4-5 per tile from level 3, one warp per tile,
//    into a small double-buffered array that peers read through DSMEM.
//  * Phase B: every CTA pushes its nonzero bins into the cluster's
//    distributed sum (bin i lives in CTA i % C, slot i / C; RED over DSMEM;
//    triple-buffered by image so no second barrier is needed), one cluster
//    barrier (release / acquire), gather of the summed histograms, warp-scan
//    lower median per level (as hist_median_kernel).
//  * Phase C: thresholds from the shared gray, deferred into the NEXT
//    image's phase A: just before a group overwrites a tile slot with the
//    next image, it packs the slot's words of the previous image (levels
//    0..3, 340 words per tile, specialised VABSDIFF4 / carry forms), so the
//    pack runs under that tile's TMA latency; the words of levels 4..5 (a
//    word spans 2 or 4 tiles, possibly of different CTAs) are spread over the
//    cluster and read the tiles' level-4/5 bytes through DSMEM.  The last
//    image of a cluster is packed after the loop.
// HBM traffic per image = RGB (3 W H) + bitmaps (2 bits per pyramid pixel,
// packed), against + 2 x gray (4/3 W H each way) for the staged kernels.
// Measured: the kernel is instruction-bound; it beats the
// staged kernels 1.3-1.7x while an image fits 1-2 CTAs (<= 0.4 MP) and
// loses at 4-16 CTAs (cluster barrier and fewer co-resident clusters), so
// the engine dispatches it for the small shapes only.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "k1_tile.cuh"
#include "swar.cuh"

namespace cg = cooperative_groups;

namespace mtb {

PFN_cuTensorMapEncodeTiled_v12000 k1_encode_tiled();   // k1_rgb.cu
bool k1_rgb_supported(int w, int64_t rgb_pitch, int64_t rgb_img_stride, const void* rgb);

constexpr int kCmSlotBytes = tm_off(4);   // tile-major levels 0..3 of one tile (10880 B)
constexpr int kCmL45Bytes = 48;           // level 4 (2 x 16 B) + level 5 (8 B) of one tile, 16-B padded
constexpr int kCmWords03 = 256 + 64 + 16 + 4;   // bitmap words of levels 0..3 in one tile
constexpr int kCmSmemMax = 232448 - 1024;       // opt-in maximum minus the 1 KB alignment slack

struct CmArgs {
  K1Args k;               // geometry: w, h, lw, lh, nl, tiles_x, tiles_y (gray/off/pitch unused)
  int T;                  // tiles per image
  int C;                  // cluster size
  int G;                  // streaming groups of 128 threads (blockDim = 128 G)
  int tpc;                // tile slots per CTA
  int n_img, nq;          // images; clusters in the grid
  int tol;
  int sum_slice;          // ceil(nl * 256 / C): bins per CTA in the distributed sum
  int nw32[6], bit_off32[6];
  int64_t bit_img_words32;
  uint32_t* mtb;
  uint32_t* excl;
  int32_t* medians;       // [img][nl]
  uint32_t* hist_out;     // [img][nl][256] or null
  int off_sum, off_rgb, off_gray, off_l45, off_th, off_bar;   // shared-memory layout (bytes)
};

struct CmLayout {
  int off_sum, off_rgb, off_gray, off_l45, off_th, off_bar, bytes;
};
// hist [6][256] u32 at 0 (1 KB-aligned levels), summed histograms tot [6][256]
// at 6 KB, then the distributed-sum slices, the TMA stages, the gray slots,
// the level-4/5 double buffer, threshold constants and mbarriers.
static CmLayout cm_layout(int nl, int C, int G, int tpc) {
  CmLayout L;
  const int slice = (nl * 256 + C - 1) / C;
  L.off_sum = 12288;
  L.off_rgb = (int)round_up(L.off_sum + 3 * slice * 4, 128);
  L.off_gray = L.off_rgb + G * kK1TileBytes;
  L.off_l45 = L.off_gray + tpc * kCmSlotBytes;
  L.off_th = L.off_l45 + 2 * tpc * kCmL45Bytes;
  L.off_bar = L.off_th + 12 * (int)sizeof(ThConst);
  L.bytes = (int)round_up(L.off_bar + 8 * G, 128);
  return L;
}

#ifdef CM_TRACE
// Experiment builds only (tools/build_exp.sh NAME -DCM_TRACE): %globaltimer at
// the phase boundaries of the first 8 images of the first 256 CTAs.
__device__ unsigned long long g_cm_trace[256][8][6];
__device__ __forceinline__ void cm_mark(int j, int p) {
  if (threadIdx.x == 0 && blockIdx.x < 256 && j < 8) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_cm_trace[blockIdx.x][j][p] = t;
  }
}
#else
__device__ __forceinline__ void cm_mark(int, int) {}
#endif

__device__ __forceinline__ uint32_t* cm_remote(cg::cluster_group& cl, uint32_t* p, int rank) {
  return cl.map_shared_rank(p, (unsigned)rank);
}

// Word f (0..339) of one tile's levels 0..3 in tile-major order -> level,
// row, column.  The slot holds these words contiguously: word f is the 32
// gray bytes at slot + 32 f.
__device__ __forceinline__ void cm_word(int f, int& k, int& row, int& col) {
  if (f < 256) {
    k = 0; row = f >> 3; col = f & 7;
  } else if (f < 320) {
    f -= 256; k = 1; row = f >> 2; col = f & 3;
  } else if (f < 336) {
    f -= 320; k = 2; row = f >> 1; col = f & 1;
  } else {
    k = 3; row = f - 336; col = 0;
  }
}

// Threshold + pack of one 32-pixel word with the level's constants, in the
// specialised carry forms (MED_LO per level, TOL_LO = tol <= 127).
__device__ __forceinline__ void cm_th(const uint32_t (&g)[8], const ThConst& c, bool tol_lo, uint32_t yt,
                                      uint32_t ytl, int valid, uint32_t& m, uint32_t& e) {
  if (c.med_lo) {
    if (tol_lo) th_word_t<true, true>(g, c, yt, ytl, valid, m, e);
    else th_word_t<true, false>(g, c, yt, ytl, valid, m, e);
  } else {
    if (tol_lo) th_word_t<false, true>(g, c, yt, ytl, valid, m, e);
    else th_word_t<false, false>(g, c, yt, ytl, valid, m, e);
  }
}

struct CmOut {
  uint32_t* mtb;
  uint32_t* excl;
  const ThConst* th;   // the image's per-level constants
  bool tol_lo;
  uint32_t yt, ytl;
};

// Levels 0..3 of one tile slot: words t, t + nt, ... of the slot.  Lanes read
// their word's two 16-B halves in swizzled order ((lane >> 2) & 1), so each
// LDS.128 of a warp covers 8 distinct 16-B bank groups per 128 B.  The owner
// of a row's last tile also writes the row's zero padding words.
__device__ __forceinline__ void cm_threshold_slot(const CmArgs& a, const uint8_t* slot, int tile, const CmOut& o,
                                                  int t, int nthreads, int lane) {
  const int nl = a.k.nl;
  const int nw = nl >= 4 ? 340 : nl == 3 ? 336 : nl == 2 ? 320 : 256;
  const int ty = tile / a.k.tiles_x, tx = tile - ty * a.k.tiles_x;
  const int sw = (lane >> 2) & 1;
  for (int f = t; f < nw; f += nthreads) {
    int k, row, col;
    cm_word(f, k, row, col);
    const uint4* p = reinterpret_cast<const uint4*>(slot + 32 * f);
    uint4 u0 = p[sw], u1 = p[sw ^ 1];
    if (sw) {
      const uint4 x = u0;
      u0 = u1;
      u1 = x;
    }
    const int y = ty * (kK1TileRows >> k) + row, jw = tx * (8 >> k) + col;
    if (y < a.k.lh[k] && jw < a.nw32[k]) {
      const uint32_t g[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
      uint32_t m, e;
      cm_th(g, o.th[k], o.tol_lo, o.yt, o.ytl, a.k.lw[k] - 32 * jw, m, e);
      const int64_t w = a.bit_off32[k] + (int64_t)y * a.nw32[k] + jw;
      o.mtb[w] = m;
      o.excl[w] = e;
    }
  }
  if (tx == a.k.tiles_x - 1) {
    for (int e = t; e < 60; e += nthreads) {   // (level, row) pairs of levels 0..3: 32 + 16 + 8 + 4
      const int k = e < 32 ? 0 : e < 48 ? 1 : e < 56 ? 2 : 3;
      const int row = e - (k == 0 ? 0 : k == 1 ? 32 : k == 2 ? 48 : 56);
      const int y = ty * (kK1TileRows >> k) + row;
      if (k >= nl || y >= a.k.lh[k]) continue;
      for (int jw = a.k.tiles_x * (8 >> k); jw < a.nw32[k]; ++jw) {
        o.mtb[a.bit_off32[k] + (int64_t)y * a.nw32[k] + jw] = 0u;
        o.excl[a.bit_off32[k] + (int64_t)y * a.nw32[k] + jw] = 0u;
      }
    }
  }
}

// Levels 4..5: row-major words (a word spans 2 or 4 tiles, possibly of
// different CTAs) spread over the cluster; tile bytes read through DSMEM from
// the owners' level-4/5 buffers of the image (l45b = this CTA's copy).
__device__ __forceinline__ void cm_threshold_l45(const CmArgs& a, cg::cluster_group& cl, uint8_t* l45b,
                                                 const CmOut& o, int r, int tid, int nthr) {
  const int C = a.C, T = a.T, tx_n = a.k.tiles_x;
  for (int k = 4; k < a.k.nl; ++k) {
    const int words = a.nw32[k] * a.k.lh[k];
    const int span = k == 4 ? 2 : 4;   // tiles per word
    for (int f = r * nthr + tid; f < words; f += C * nthr) {
      const int y = f / a.nw32[k], jw = f - y * a.nw32[k];
      const int ty = k == 4 ? y >> 1 : y;
      const int boff = k == 4 ? (y & 1) * 16 : 32;
      uint32_t g[8];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        if (s >= span) break;
        const int tx = jw * span + s;
        uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0;
        if (tx < tx_n) {
          const int tile = ty * tx_n + tx;
          const int owner = (int)(((int64_t)(tile + 1) * C - 1) / T);
          const int slot = tile - (int)((int64_t)owner * T / C);
          uint32_t* lp = reinterpret_cast<uint32_t*>(l45b + slot * kCmL45Bytes + boff);
          const uint32_t* rp = cm_remote(cl, lp, owner);
          if (k == 4) {
            const uint4 u = *reinterpret_cast<const uint4*>(rp);
            w0 = u.x; w1 = u.y; w2 = u.z; w3 = u.w;
          } else {
            const uint2 u = *reinterpret_cast<const uint2*>(rp);
            w0 = u.x; w1 = u.y;
          }
        }
        if (k == 4) {
          g[4 * s] = w0; g[4 * s + 1] = w1; g[4 * s + 2] = w2; g[4 * s + 3] = w3;
        } else {
          g[2 * s] = w0; g[2 * s + 1] = w1;
        }
      }
      uint32_t m, e;
      cm_th(g, o.th[k], o.tol_lo, o.yt, o.ytl, a.k.lw[k] - 32 * jw, m, e);
      const int64_t w = a.bit_off32[k] + (int64_t)y * a.nw32[k] + jw;
      o.mtb[w] = m;
      o.excl[w] = e;
    }
  }
}

__global__ void __launch_bounds__(512, 1) cluster_maps_kernel(CmArgs a, const __grid_constant__ CUtensorMap rgb_map) {
  extern __shared__ __align__(128) uint8_t cm_raw[];
  const uint32_t raw = smem_addr(cm_raw);
  uint8_t* base = cm_raw + ((1024u - (raw & 1023u)) & 1023u);
  uint32_t* hist = reinterpret_cast<uint32_t*>(base);
  uint32_t* tot = reinterpret_cast<uint32_t*>(base + 6144);
  uint32_t* sum = reinterpret_cast<uint32_t*>(base + a.off_sum);
  uint8_t* rgb = base + a.off_rgb;
  uint8_t* gray = base + a.off_gray;
  uint8_t* l45 = base + a.off_l45;
  ThConst* th = reinterpret_cast<ThConst*>(base + a.off_th);   // [image parity][level]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(base + a.off_bar);

  cg::cluster_group cl = cg::this_cluster();
  const int C = a.C, G = a.G, T = a.T, nl = a.k.nl, tx_n = a.k.tiles_x;
  const int r = (int)cl.block_rank();
  const int q = (int)(blockIdx.x / C);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int g = tid >> 7, t = tid & 127, lane = tid & 31, wg = t >> 5, warp = tid >> 5, nwarps = nthr >> 5;
  const int t0 = (int)((int64_t)r * T / C);
  const int nt = (int)((int64_t)(r + 1) * T / C) - t0;
  const int nbins = nl * 256;
  const uint32_t hb = smem_addr(hist);
  CmOut po;   // outputs and constants of the previous image (thresholded during this image's phase A)
  po.tol_lo = a.tol <= 127;
  po.yt = (uint32_t)(255 - a.tol) * 0x01010101u;
  po.ytl = po.yt & 0x7f7f7f7fu;

  for (int i = tid; i < 6 * 256; i += nthr) hist[i] = 0;
  for (int i = tid; i < 3 * a.sum_slice; i += nthr) sum[i] = 0;
  if (tid < G) mbar_init(&full[tid], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  cl.sync();   // every CTA's sum slices are zero before any peer pushes into them

  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](int img, int i) {   // local tile i of image img -> group g's stage
    const int tile = t0 + i;
    const int ty = tile / tx_n, tx = tile - ty * tx_n;
    mbar_expect_tx(&full[g], kK1TileBytes);
    tma_tile(rgb + g * kK1TileBytes, &rgb_map, (kK1RowBytes / 4) * tx, kK1TileRows * ty, img, &full[g], pol);
  };
  if (t == 0 && g < nt && q < a.n_img) issue(q, g);

  uint32_t par = 0;
  int j = 0;
  for (int img = q; img < a.n_img; ++j, img += a.nq) {
    const int nimg = img + a.nq;
    uint8_t* l45b = l45 + (j & 1) * a.tpc * kCmL45Bytes;
    if (j > 0)   // previous image's levels 4..5 (its level-4/5 buffers stay valid until this image's barrier)
      cm_threshold_l45(a, cl, l45 + ((j - 1) & 1) * a.tpc * kCmL45Bytes, po, r, tid, nthr);
    cm_mark(j, 0);
    // ---- A: levels 0..3 of the owned tiles (TMA -> registers -> shared); the
    // previous image's words of a slot are thresholded just before the slot is
    // overwritten, under this tile's TMA latency ------------------------------
    for (int i = g; i < nt; i += G) {
      const int tile = t0 + i;
      const int ty = tile / tx_n, tx = tile - ty * tx_n;
      const bool fl = (ty * kK1TileRows + kK1TileRows <= a.k.h) && (tx * kK1TilePx + kK1TilePx <= a.k.w);
      uint8_t* tg = gray + i * kCmSlotBytes;
      if (j > 0) cm_threshold_slot(a, tg, tile, po, t, kK1GroupThreads, lane);
      uint2 v[8][3];
      mbar_wait(&full[g], par);
      par ^= 1u;
      {
        const uint8_t* src = rgb + g * kK1TileBytes + (8 * wg) * kK1RowBytes + 24 * lane;
#pragma unroll
        for (int rr = 0; rr < 8; ++rr)
#pragma unroll
          for (int c = 0; c < 3; ++c) v[rr][c] = *reinterpret_cast<const uint2*>(src + rr * kK1RowBytes + 8 * c);
      }
      group_bar(g);   // stage consumed and the slot's previous words read by the whole group
      if (t == 0) {
        if (i + G < nt) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(img, i + G);
        } else if (nimg < a.n_img) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(nimg, g);   // this group's first tile of the next image
        }
      }
      if (fl)
        k1_block_tm<true, true>(a.k, tg, v, tx, ty, wg, lane, hb, nullptr, 0);
      else
        k1_block_tm<false, true>(a.k, tg, v, tx, ty, wg, lane, hb, nullptr, 0);
    }
    cm_mark(j, 1);
    __syncthreads();
    // ---- A': levels 4 and 5 of each owned tile from its level 3 (one warp per tile) ----
    if (nl >= 5) {
      for (int i = warp; i < nt; i += nwarps) {
        const int tile = t0 + i;
        const int ty = tile / tx_n, tx = tile - ty * tx_n;
        const uint8_t* l3 = gray + i * kCmSlotBytes + tm_off(3);
        uint8_t* o = l45b + i * kCmL45Bytes;
        const int rr = lane >> 4, c = lane & 15;
        const uint32_t v4 = (l3[(2 * rr) * 32 + 2 * c] + l3[(2 * rr) * 32 + 2 * c + 1] + l3[(2 * rr + 1) * 32 + 2 * c] +
                             l3[(2 * rr + 1) * 32 + 2 * c + 1] + 2u) >> 2;
        o[rr * 16 + c] = (uint8_t)v4;
        if (ty * 2 + rr < a.k.lh[4] && tx * 16 + c < a.k.lw[4]) hinc((hb + 4096) | (v4 << 2));
        if (nl >= 6) {
          const int c5 = lane & 7;
          const uint32_t q0 = __shfl_sync(0xffffffffu, v4, 2 * c5), q1 = __shfl_sync(0xffffffffu, v4, 2 * c5 + 1);
          const uint32_t q2 = __shfl_sync(0xffffffffu, v4, 16 + 2 * c5), q3 = __shfl_sync(0xffffffffu, v4, 17 + 2 * c5);
          if (lane < 8) {
            const uint32_t v5 = (q0 + q1 + q2 + q3 + 2u) >> 2;
            o[32 + lane] = (uint8_t)v5;
            if (ty < a.k.lh[5] && tx * 8 + lane < a.k.lw[5]) hinc((hb + 5120) | (v5 << 2));
          }
        }
      }
    }
    __syncthreads();
    cm_mark(j, 2);
    // ---- B: cluster-wide histograms and medians ------------------------------
    uint32_t* sj = sum + (j % 3) * a.sum_slice;
    for (int i = tid; i < nbins; i += nthr) {
      const uint32_t c = hist[i];
      if (c) {
        hist[i] = 0;
        atomicAdd(cm_remote(cl, sj + i / C, i % C), c);
      }
    }
    cl.sync();   // arrive.release / wait.acquire: all pushes (and level-4/5 bytes) visible
    cm_mark(j, 3);
    for (int i = tid; i < nbins; i += nthr) tot[i] = *cm_remote(cl, sj + i / C, i % C);
    {
      // the slice of image j+2 (= j-1 mod 3): every peer read it before this barrier
      uint32_t* sz = sum + ((j + 2) % 3) * a.sum_slice;
      for (int i = tid; i < a.sum_slice; i += nthr) sz[i] = 0;
    }
    __syncthreads();
    ThConst* thj = th + (j & 1) * 6;
    if (warp < nl) {
      const uint32_t* src = tot + warp * 256;
      uint32_t bins[8];
      uint32_t s = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        bins[i] = src[lane * 8 + i];
        s += bins[i];
      }
      if (r == 0 && a.hist_out) {
        uint32_t* dst = a.hist_out + ((int64_t)img * nl + warp) * 256;
#pragma unroll
        for (int i = 0; i < 8; ++i) dst[lane * 8 + i] = bins[i];
      }
      uint32_t incl = s;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t target = (total >> 1) + (total & 1u);   // (total + 1) / 2 without overflow
      const unsigned mask = __ballot_sync(0xffffffffu, incl >= target);
      int med = -1;
      if (total > 0) {
        const int L = __ffs(mask) - 1;
        if (lane == L) {
          uint32_t c = incl - s;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            c += bins[i];
            if (c >= target) {
              med = lane * 8 + i;
              break;
            }
          }
        }
        med = __shfl_sync(0xffffffffu, med, L);
      }
      if (lane == 0) {
        if (r == 0) a.medians[(int64_t)img * nl + warp] = med;
        ThConst c;
        c.med = (uint32_t)med * 0x01010101u;
        c.ym = (uint32_t)(255 - med) * 0x01010101u;
        c.yml = c.ym & 0x7f7f7f7fu;
        c.med_lo = med <= 127;
        thj[warp] = c;
      }
    }
    __syncthreads();
    cm_mark(j, 4);
    po.mtb = a.mtb + (int64_t)img * a.bit_img_words32;
    po.excl = a.excl + (int64_t)img * a.bit_img_words32;
    po.th = thj;
    cm_mark(j, 5);
  }
  // ---- C of the cluster's last image: all threads ----------------------------
  if (j > 0) {
    for (int i = 0; i < nt; ++i) cm_threshold_slot(a, gray + i * kCmSlotBytes, t0 + i, po, tid, nthr, lane);
    cm_threshold_l45(a, cl, l45 + ((j - 1) & 1) * a.tpc * kCmL45Bytes, po, r, tid, nthr);
  }
  cl.sync();   // no CTA leaves while a peer may still read its shared memory
}

// Cluster shape for a plan: the smallest cluster whose CTAs can each hold
// their share of the image's tiles next to G streaming stages (G = 4, else
// 3 or 2), and that the device can co-schedule.  MTB_CM_CLUSTER /
// MTB_CM_GROUPS force a shape (experiments).
struct CmShape {
  int C, G, tpc, nq_max;
  CmLayout L;
};

static int cm_max_clusters(int C, int G, int smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int>, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  const auto key = std::make_tuple(dev, C, G, smem);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  int n = 0;
  if (cudaFuncSetAttribute(cluster_maps_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess &&
      cudaFuncSetAttribute(cluster_maps_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)C);
    cfg.blockDim = dim3((unsigned)(128 * G));
    cfg.dynamicSmemBytes = (size_t)smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&n, cluster_maps_kernel, &cfg) != cudaSuccess) n = 0;
  }
  cudaGetLastError();
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = n;
  return n;
}

static bool cm_shape(const Plan& p, CmShape* out) {
  if (p.n > 6) return false;
  const int tiles_x = (p.lv[0].w + kK1TilePx - 1) / kK1TilePx, tiles_y = (p.lv[0].h + kK1TileRows - 1) / kK1TileRows;
  const int64_t T = (int64_t)tiles_x * tiles_y;
  const char* ec = std::getenv("MTB_CM_CLUSTER");
  const char* eg = std::getenv("MTB_CM_GROUPS");
  const int fc = ec ? std::atoi(ec) : 0, fg = eg ? std::atoi(eg) : 0;
  for (int C = 1; C <= 16; C *= 2) {
    if (fc && C != fc) continue;
    const int tpc = (int)((T + C - 1) / C);
    for (int G = 4; G >= 2; --G) {
      if (fg && G != fg) continue;
      const CmLayout L = cm_layout(p.n, C, G, tpc);
      if (L.bytes > kCmSmemMax) continue;
      const int nq = cm_max_clusters(C, G, L.bytes + 1024);
      if (nq < 1) continue;
      *out = CmShape{C, G, tpc, nq, L};
      return true;
    }
  }
  return false;
}


int launch_cluster_maps(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride, int n_img, const Plan& p,
                        int tol, uint32_t* hist_out, int32_t* medians, uint64_t* mtb, uint64_t* excl,
                        cudaStream_t st) {
  CmShape s;
  if (!cm_shape(p, &s)) {
    set_error("preprocess_maps: image too large for one cluster's shared memory (or more than 6 levels)");
    return MTB_EINVAL;
  }
  CmArgs a{};
  a.k.w = p.lv[0].w;
  a.k.h = p.lv[0].h;
  a.k.nl = p.n;
  for (int k = 0; k < 6; ++k) {
    a.k.lw[k] = k < p.n ? p.lv[k].w : 0;
    a.k.lh[k] = k < p.n ? p.lv[k].h : 0;
    a.nw32[k] = k < p.n ? (int)(2 * p.lv[k].nw64) : 0;
    a.bit_off32[k] = k < p.n ? (int)(2 * p.lv[k].bit_off) : 0;
  }
  a.k.tiles_x = (a.k.w + kK1TilePx - 1) / kK1TilePx;
  a.k.tiles_y = (a.k.h + kK1TileRows - 1) / kK1TileRows;
  a.T = a.k.tiles_x * a.k.tiles_y;
  a.C = s.C;
  a.G = s.G;
  a.tpc = s.tpc;
  a.n_img = n_img;
  a.nq = n_img < s.nq_max ? n_img : s.nq_max;
  a.tol = tol;
  a.sum_slice = (p.n * 256 + s.C - 1) / s.C;
  a.bit_img_words32 = 2 * p.bit_img_words;
  a.mtb = reinterpret_cast<uint32_t*>(mtb);
  a.excl = reinterpret_cast<uint32_t*>(excl);
  a.medians = medians;
  a.hist_out = hist_out;
  a.off_sum = s.L.off_sum;
  a.off_rgb = s.L.off_rgb;
  a.off_gray = s.L.off_gray;
  a.off_l45 = s.L.off_l45;
  a.off_th = s.L.off_th;
  a.off_bar = s.L.off_bar;
  const int smem = s.L.bytes + 1024;
  MTB_CUDA(cudaFuncSetAttribute(cluster_maps_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  MTB_CUDA(cudaFuncSetAttribute(cluster_maps_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CUtensorMap map;
  {
    const cuuint64_t dims[3] = {(cuuint64_t)(3 * (int64_t)a.k.w / 4), (cuuint64_t)a.k.h, (cuuint64_t)n_img};
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
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(a.nq * s.C));
  cfg.blockDim = dim3((unsigned)(128 * s.G));
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)s.C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  MTB_CUDA(cudaLaunchKernelEx(&cfg, cluster_maps_kernel, a, map));
  return check_launch("cluster_maps_kernel");
}

}  // namespace mtb

using namespace mtb;

extern "C" int mtb_preprocess_maps_shape(int w, int h, int levels, int* shape) {
  clear_error();
  CmShape s;
  Plan p;
  if ((3 * (int64_t)w) % 4 != 0 || !make_plan(w, h, levels, &p) || !cm_shape(p, &s)) return 0;
  if (shape) {
    shape[0] = s.C;
    shape[1] = s.G;
    shape[2] = s.tpc;
    shape[3] = s.nq_max;
  }
  return s.C;
}

extern "C" int mtb_preprocess_maps_cluster(int w, int h, int levels) {
  return mtb_preprocess_maps_shape(w, h, levels, nullptr);
}

#ifdef CM_TRACE
extern "C" int mtb_cm_trace(unsigned long long* host) {
  MTB_CUDA(cudaMemcpyFromSymbol(host, g_cm_trace, sizeof(g_cm_trace)));
  return MTB_OK;
}
#endif

extern "C" int mtb_preprocess_maps(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride, int w, int h,
                                   int n_img, int levels, int tol, uint32_t* hist_out, int32_t* medians,
                                   uint64_t* mtb, uint64_t* exclusion, void* stream) {
  clear_error();
  MTB_REQUIRE(tol >= 0 && tol <= 255, "noise tolerance must be in 0..255");
  MTB_REQUIRE(rgb && medians && mtb && exclusion, "null pointer");
  MTB_REQUIRE(n_img >= 1 && n_img <= 65535, "image count out of range");
  MTB_REQUIRE(rgb_pitch >= 3 * (int64_t)w, "rgb pitch smaller than row");
  Plan p;
  MTB_REQUIRE(make_plan(w, h, levels, &p), "image must be at least 16x16 and levels >= 1");
  MTB_REQUIRE(k1_rgb_supported(w, rgb_pitch, rgb_img_stride, rgb),
              "preprocess_maps needs 3*W % 4 == 0 and 16-byte aligned rows and images");
  return launch_cluster_maps(rgb, rgb_pitch, rgb_img_stride, n_img, p, tol, hist_out, medians, mtb, exclusion,
                             as_stream(stream));
}
