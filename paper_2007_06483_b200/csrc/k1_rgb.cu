// K1 (fast path): RGB8 -> gray -> 2x box pyramid (levels 0..5) -> per-level
// 256-bin histograms, one streaming pass over the RGB input.
//
// Reference semantics are those listed in pyramid.cu (image.py:58-68,
// pyramid.py:17-62, threshold.py:25-28).  This kernel is the roofline kernel
// of the whole path: it reads every RGB byte exactly once.  Design (sm_100a):
//
//  * One 1024-thread CTA per SM, persistent over a contiguous band of the
//    interior 32x128-pixel tiles of one image (edge tiles go to the generic
//    kernel in pyramid.cu).  Eight independent 128-thread groups each own one
//    tile at a time and synchronise only on their own named barrier.
//  * Each thread owns a 32-pixel row segment (96 RGB bytes).  The bytes of its
//    NEXT tile are fetched with cp.async (LDGSTS, 16 B each, L2 evict-first
//    policy) into the thread's own shared-memory slot right after it has
//    pulled the current ones into registers, so the copy has a whole tile of
//    work to land and no register holds in-flight data (32 warps/SM fit).
//  * Gray via IDP.4A: pixel groups of 4 (12 bytes = 3 words) need 6 dp4a and
//    3 byte-permutes; no byte extraction.
//  * Levels 1-2 by all threads with SIMD pair sums in 16-bit lanes;
//    levels 3-5 by one warp per tile (rotating) with warp syncs only.
//  * Histograms: shared-memory atomics (ATOMS.POPC.INC aggregates equal
//    addresses in a warp), reduced across a thread-block cluster through
//    distributed shared memory, then one global RED per nonzero bin per
//    cluster into a 128-B-strided ("spread") histogram.
//  * Gray levels are stored with an L2::evict_last policy: the threshold pass
//    re-reads them right after, ideally from L2.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace mtb {

constexpr int kK1Groups = 8;
constexpr int kK1GroupThreads = 128;
constexpr int kK1Threads = kK1Groups * kK1GroupThreads;
constexpr int kHistStrideK1 = 32;   // must equal kHistStride in pyramid.cu

struct K1Args {
  const uint8_t* rgb;
  int64_t rgb_pitch, rgb_img_stride;
  int w, h;
  uint8_t* gray;
  int64_t gray_img_stride;
  int64_t off[6], pitch[6];
  int lw[6], lh[6];
  int nl;                 // levels produced (1..6)
  uint32_t* hist;         // spread histograms [img][level][bin * 32]
  int64_t hist_img_stride;
  int tiles_x, tiles_y;   // ceil(w/128) x ceil(h/32)
  int cluster;            // CTAs per cluster (1, 2, 4)
  int probe;              // diagnostics only (MTB_K1_PROBE): 1 = stream tiles, skip all compute
};

constexpr int kTileRgbBytes = 32 * 384;   // one 32x128 tile of RGB8

struct alignas(128) GroupSmem {
  uint8_t rgb[2][kTileRgbBytes];  // TMA ring: two tiles in flight per group
  uint8_t l3[2][4 * 16];          // level-3 values, double-buffered by tile parity
  uint8_t l4[2 * 8];
  unsigned long long full[2];     // mbarriers of the two ring stages
};

struct K1Smem {
  GroupSmem grp[kK1Groups];
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
// TMA 3-D tile copy (box 96 u32 x 32 rows x 1 image) -> this CTA's smem.
__device__ __forceinline__ void tma_tile(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar))
      : "memory");
}
// Bulk (TMA engine) copy of `bytes` contiguous bytes global -> this CTA's smem,
// completing on `bar` (tx count).
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ uint4 ld_stream16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void group_bar(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(kK1GroupThreads) : "memory");
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

// Two 2x2 box averages from one word of each of two rows (4 source pixels
// per word): avg of bytes 0-1 in byte 0, avg of bytes 2-3 in byte 2.
__device__ __forceinline__ uint32_t box2(uint32_t u, uint32_t d) {
  const uint32_t s = (u & 0x00FF00FFu) + ((u >> 8) & 0x00FF00FFu) + (d & 0x00FF00FFu) + ((d >> 8) & 0x00FF00FFu) +
                     0x00020002u;
  return s >> 2;
}
// 2x2 box sum + 2 of the byte pair `pair` (0: bytes 0-1, 1: bytes 2-3) of a
// word of the upper row u and of the lower row d: (a+b+c+d+2), < 1024.  The
// average is sum >> 2 and its histogram byte offset is sum & 0x3fc.
__device__ __forceinline__ uint32_t box_sum(uint32_t u, uint32_t d, int pair) {
  const uint32_t w = pair ? 0x01010000u : 0x00000101u;
  return __dp4a(u, w, __dp4a(d, w, 2u));
}
// Four box sums -> four packed average bytes.
__device__ __forceinline__ uint32_t pack_sums(uint32_t s0, uint32_t s1, uint32_t s2, uint32_t s3) {
  const uint32_t x01 = (s0 + (s1 << 16)) >> 2, x23 = (s2 + (s3 << 16)) >> 2;
  return __byte_perm(x01, x23, 0x6420);
}
// Increment the counter at byte offset `off` of the (static) histogram array;
// written as plain C++ on the array so the base folds into the ATOMS address.
__device__ __forceinline__ void hist_inc(uint32_t* hist, uint32_t off) { atomicAdd(&hist[off >> 2], 1u); }
// Pack the two results of two box2 words into 4 consecutive bytes.
__device__ __forceinline__ uint32_t pack_box(uint32_t q0, uint32_t q1) { return __byte_perm(q0, q1, 0x6420); }

// Thread layout inside a 128-thread group (one 32x128 tile): thread = (ry, cx)
// owns level-0 rows 2ry, 2ry+1 and columns 16cx .. 16cx+15 (ry 0..15, cx 0..7);
// lane = (ry & 3) * 8 + cx, warp-in-group = ry >> 2.  Level 1 is computed in
// registers, level 2 with one shuffle (partner ry^1 = lane^8), level 3 with
// another (partner ry^2 = lane^16); levels 4-5 (which span warps) go through a
// 64-byte shared buffer and one named barrier per tile.
// CLUSTER: reduce histograms across a thread-block cluster through DSMEM.  A
// separate instantiation, because cluster-capable code addresses its own
// shared memory through the CTA's cluster window (an extra add per access).
template <bool CLUSTER>
__global__ void __launch_bounds__(kK1Threads, 1) k1_rgb_pyramid_kernel(K1Args a, const __grid_constant__ CUtensorMap rgb_map) {
  extern __shared__ __align__(128) uint8_t k1_smem_raw[];
  K1Smem& SM = *reinterpret_cast<K1Smem*>(k1_smem_raw);
  __shared__ uint32_t s_hist[6 * 256];   // static: its base folds into the ATOMS immediate

  const int tid = threadIdx.x;
  const int g = tid >> 7;             // group
  const int t = tid & 127;            // thread in group
  const int lane = tid & 31;
  const int wig = t >> 5;             // warp in group
  const int cx = lane & 7;
  const int ry = (wig << 2) | (lane >> 3);
  const int img = blockIdx.y;
  GroupSmem& S = SM.grp[g];

  for (int i = tid; i < 6 * 256; i += kK1Threads) s_hist[i] = 0;
  if (t == 0) {
    mbar_init(&S.full[0], 1);
    mbar_init(&S.full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const uint8_t* rgb = a.rgb + img * a.rgb_img_stride;
  uint8_t* gray = a.gray + img * a.gray_img_stride;

  const int ntiles = a.tiles_x * a.tiles_y;
  const int t_begin = (int)((int64_t)blockIdx.x * ntiles / gridDim.x);
  const int t_end = (int)((int64_t)(blockIdx.x + 1) * ntiles / gridDim.x);

  // One thread per group streams tiles into the group's 2-stage ring with a
  // single TMA tensor copy each (box = the tile's 32 rows x 384 bytes).
  auto issue = [&](int tile, int stage) {
    if (t == 0) {
      const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
      mbar_expect_tx(&S.full[stage], kTileRgbBytes);
      tma_tile(S.rgb[stage], &rgb_map, 96 * tx, 32 * ty, img, &S.full[stage]);
    }
  };
  if (t_begin + g < t_end) issue(t_begin + g, 0);
  if (t_begin + g + kK1Groups < t_end) issue(t_begin + g + kK1Groups, 1);

  int iter = 0;
  int ty = (t_begin + g) / a.tiles_x, tx = (t_begin + g) - ty * a.tiles_x;
  for (int tile = t_begin + g; tile < t_end; tile += kK1Groups, ++iter) {
    if (iter) {  // advance (ty, tx) by kK1Groups tiles without a division
      tx += kK1Groups;
      while (tx >= a.tiles_x) { tx -= a.tiles_x; ++ty; }
    }
    const int y0 = ty * 32 + 2 * ry, x0 = tx * 128 + 16 * cx;
    const int stage = iter & 1;
    // Interior tiles need no bounds checks; edge tiles (TMA zero-fills what
    // lies outside the image) mask their histogram counts and row stores.
    const bool full = (ty * 32 + 32 <= a.h) && (tx * 128 + 128 <= a.w);

    auto body = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      // ---- level 0: 2 rows x 16 pixels ------------------------------------
      uint32_t gw[2][4];
      {
        mbar_wait(&S.full[stage], (iter >> 1) & 1);
        const uint8_t* p0 = S.rgb[stage] + (2 * ry) * 384 + 48 * cx;
        const uint8_t* p1 = p0 + 384;
        const uint4 q0 = *reinterpret_cast<const uint4*>(p0), q1 = *reinterpret_cast<const uint4*>(p0 + 16),
                    q2 = *reinterpret_cast<const uint4*>(p0 + 32);
        const uint4 q3 = *reinterpret_cast<const uint4*>(p1), q4 = *reinterpret_cast<const uint4*>(p1 + 16),
                    q5 = *reinterpret_cast<const uint4*>(p1 + 32);
        const uint32_t wv[2][12] = {{q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, q2.y, q2.z, q2.w},
                                    {q3.x, q3.y, q3.z, q3.w, q4.x, q4.y, q4.z, q4.w, q5.x, q5.y, q5.z, q5.w}};
        const int nvx = FULL ? 16 : min(16, max(0, a.w - x0));
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const bool row_ok = FULL || (y0 + j < a.h);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint32_t s4[4];
            gw[j][k] = gray4(wv[j][3 * k], wv[j][3 * k + 1], wv[j][3 * k + 2], s4);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              // 256 bins: byte offset 4*(s>>8).  (A 16K-sub-bin variant with a
              // one-op address measured slower: fewer equal addresses per warp
              // for ATOMS.POPC.INC to aggregate.)
              if (FULL) {
                hist_inc(s_hist, (s4[i] >> 6) & 0x3fcu);
              } else if (row_ok && 4 * k + i < nvx) {
                hist_inc(s_hist, (s4[i] >> 6) & 0x3fcu);
              }
            }
          }
          if (row_ok)
            *reinterpret_cast<uint4*>(gray + a.off[0] + (int64_t)(y0 + j) * a.pitch[0] + x0) =
                make_uint4(gw[j][0], gw[j][1], gw[j][2], gw[j][3]);
        }
      }
      if (a.nl < 2) return;

      // ---- level 1: 1 row x 8 pixels, in registers ------------------------
      uint32_t l1[2];
      {
        uint32_t sm[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) sm[i] = box_sum(gw[0][i >> 1], gw[1][i >> 1], i & 1);
        l1[0] = pack_sums(sm[0], sm[1], sm[2], sm[3]);
        l1[1] = pack_sums(sm[4], sm[5], sm[6], sm[7]);
        const int y = ty * 16 + ry, x = tx * 64 + 8 * cx;
        if (FULL || y < a.lh[1]) {
          *reinterpret_cast<uint2*>(gray + a.off[1] + (int64_t)y * a.pitch[1] + x) = make_uint2(l1[0], l1[1]);
          const int nv = FULL ? 8 : min(8, max(0, a.lw[1] - x));
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (FULL || i < nv) hist_inc(s_hist + 256, sm[i] & 0x3fcu);
          }
        }
      }
      if (a.nl < 3) return;

      // ---- level 2: partner ry^1 (lane^8); even-ry thread emits 4 pixels --
      uint32_t l2 = 0;
      {
        const uint32_t o0 = __shfl_xor_sync(0xffffffffu, l1[0], 8);
        const uint32_t o1 = __shfl_xor_sync(0xffffffffu, l1[1], 8);
        if ((ry & 1) == 0) {
          const uint32_t s0 = box_sum(l1[0], o0, 0), s1 = box_sum(l1[0], o0, 1);
          const uint32_t s2 = box_sum(l1[1], o1, 0), s3 = box_sum(l1[1], o1, 1);
          l2 = pack_sums(s0, s1, s2, s3);
          const int y = ty * 8 + (ry >> 1), x = tx * 32 + 4 * cx;
          if (FULL || y < a.lh[2]) {
            *reinterpret_cast<uint32_t*>(gray + a.off[2] + (int64_t)y * a.pitch[2] + x) = l2;
            const int nv = FULL ? 4 : min(4, max(0, a.lw[2] - x));
            if (FULL || 0 < nv) hist_inc(s_hist + 512, s0 & 0x3fcu);
            if (FULL || 1 < nv) hist_inc(s_hist + 512, s1 & 0x3fcu);
            if (FULL || 2 < nv) hist_inc(s_hist + 512, s2 & 0x3fcu);
            if (FULL || 3 < nv) hist_inc(s_hist + 512, s3 & 0x3fcu);
          }
        }
      }
      if (a.nl < 4) return;

      // ---- level 3: partner ry^2 (lane^16); ry%4==0 thread emits 2 pixels -
      {
        const uint32_t o = __shfl_xor_sync(0xffffffffu, l2, 16);
        if ((ry & 3) == 0) {
          const uint32_t s0 = box_sum(l2, o, 0), s1 = box_sum(l2, o, 1);
          const uint32_t v0 = s0 >> 2, v1 = s1 >> 2;
          const uint16_t pk = (uint16_t)(v0 | (v1 << 8));
          const int r3 = ry >> 2;  // 0..3
          *reinterpret_cast<uint16_t*>(&S.l3[iter & 1][r3 * 16 + 2 * cx]) = pk;
          const int y = ty * 4 + r3, x = tx * 16 + 2 * cx;
          if (FULL || y < a.lh[3]) {
            *reinterpret_cast<uint16_t*>(gray + a.off[3] + (int64_t)y * a.pitch[3] + x) = pk;
            if (FULL || x < a.lw[3]) hist_inc(s_hist + 768, s0 & 0x3fcu);
            if (FULL || x + 1 < a.lw[3]) hist_inc(s_hist + 768, s1 & 0x3fcu);
          }
        }
      }
    };
    if (a.probe) {
      mbar_wait(&S.full[stage], (iter >> 1) & 1);
    } else if (full) {
      body(std::true_type{});
    } else {
      body(std::false_type{});
    }

    group_bar(g);  // every thread has consumed ring stage `stage` (and written l3)
    if (tile + 2 * kK1Groups < t_end) {
      if (t == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(tile + 2 * kK1Groups, stage);
    }
    if (a.nl < 5) continue;

    // ---- levels 4..5: one warp of the group (rotating) --------------------
    if (wig == (iter & 3)) {
      const uint8_t* l3 = S.l3[iter & 1];
      if (lane < 16) {  // level 4: 2 x 8
        const int r = lane >> 3, c = lane & 7;
        const uint8_t* sp = l3 + (2 * r) * 16 + 2 * c;
        const uint32_t v = (sp[0] + sp[1] + sp[16] + sp[17] + 2u) >> 2;
        S.l4[r * 8 + c] = (uint8_t)v;
        const int y = ty * 2 + r, x = tx * 8 + c;
        if (full || (y < a.lh[4] && x < a.lw[4])) {
          gray[a.off[4] + (int64_t)y * a.pitch[4] + x] = (uint8_t)v;
          atomicAdd(&s_hist[1024 + v], 1u);
        }
      }
      __syncwarp();
      if (a.nl > 5 && lane < 4) {  // level 5: 1 x 4
        const uint8_t* sp = S.l4 + 2 * lane;
        const uint32_t v = (sp[0] + sp[1] + sp[8] + sp[9] + 2u) >> 2;
        const int y = ty, x = tx * 4 + lane;
        if (full || (y < a.lh[5] && x < a.lw[5])) {
          gray[a.off[5] + (int64_t)y * a.pitch[5] + x] = (uint8_t)v;
          atomicAdd(&s_hist[1280 + v], 1u);
        }
      }
      __syncwarp();
    }
  }

  // ---- histogram reduction: CTA -> cluster leader (DSMEM) -> global -------
  __syncthreads();

  uint32_t* gh = a.hist + img * a.hist_img_stride;
  const int nbins = a.nl * 256;
  if constexpr (CLUSTER) {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    if (cl.block_rank() != 0) {
      uint32_t* dst = cl.map_shared_rank(s_hist, 0);
      for (int i = tid; i < nbins; i += kK1Threads) {
        const uint32_t v = s_hist[i];
        if (v) atomicAdd(&dst[i], v);
      }
    }
    cl.sync();
    if (cl.block_rank() != 0) return;
  }
  for (int i = tid; i < nbins; i += kK1Threads) {
    const uint32_t v = s_hist[i];
    if (v) atomicAdd(&gh[(int64_t)i * kHistStrideK1], v);
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

// Levels 0..min(n,6)-1 of the interior tiles of n_img images (chunks of <= 4
// images per launch so every launch fills the GPU with one CTA per SM).
int launch_k1_rgb(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride, int n_img, const Plan& p,
                  uint8_t* gray, uint32_t* spread_hist, int64_t hist_img_stride, cudaStream_t st) {
  K1Args a{};
  a.rgb_pitch = rgb_pitch;
  a.rgb_img_stride = rgb_img_stride;
  a.w = p.lv[0].w;
  a.h = p.lv[0].h;
  a.gray_img_stride = p.gray_img_bytes;
  a.nl = p.n < 6 ? p.n : 6;
  for (int k = 0; k < 6; ++k) {
    const int l = k < p.n ? k : p.n - 1;
    a.off[k] = p.lv[l].gray_off;
    a.pitch[k] = p.lv[l].gray_pitch;
    a.lw[k] = k < p.n ? p.lv[k].w : 0;
    a.lh[k] = k < p.n ? p.lv[k].h : 0;
  }
  a.hist_img_stride = hist_img_stride;
  {
    const char* pr = getenv("MTB_K1_PROBE");
    a.probe = pr ? atoi(pr) : 0;
  }
  a.tiles_x = (a.w + 127) / 128;   // edge tiles included: TMA zero-fills outside the image
  a.tiles_y = (a.h + 31) / 32;
  const int ntiles = a.tiles_x * a.tiles_y;
  if (ntiles == 0) return MTB_OK;
  static bool attr_done = false;
  const int smem = (int)sizeof(K1Smem);
  if (!attr_done) {
    MTB_CUDA(cudaFuncSetAttribute(k1_rgb_pyramid_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    MTB_CUDA(cudaFuncSetAttribute(k1_rgb_pyramid_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_done = true;
  }
  const int sms = num_sms();
  int launches = 0;
  for (int i0 = 0; i0 < n_img; i0 += 4) {
    const int c = n_img - i0 < 4 ? n_img - i0 : 4;
    int x = sms / c;
    if (x > (ntiles + kK1Groups - 1) / kK1Groups) x = (ntiles + kK1Groups - 1) / kK1Groups;
    if (x < 1) x = 1;
    int cl = 1;
    if (x % 4 == 0) cl = 4;
    else if (x % 2 == 0) cl = 2;
    a.cluster = cl;
    a.rgb = rgb + i0 * rgb_img_stride;
    a.gray = gray + i0 * p.gray_img_bytes;
    CUtensorMap map;
    {
      const cuuint64_t dims[3] = {(cuuint64_t)(3 * (int64_t)a.w / 4), (cuuint64_t)a.h, (cuuint64_t)c};
      const cuuint64_t strides[2] = {(cuuint64_t)rgb_pitch, (cuuint64_t)rgb_img_stride};
      const cuuint32_t box[3] = {96, 32, 1};
      const cuuint32_t estr[3] = {1, 1, 1};
      const CUresult r = encode_tiled()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, (void*)a.rgb, dims, strides, box,
                                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed for the RGB batch");
        return MTB_ECUDA;
      }
    }
    a.hist = spread_hist + i0 * hist_img_stride;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)x, (unsigned)c);
    cfg.blockDim = dim3(kK1Threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = cl > 1 ? 1 : 0;
    const cudaError_t e = cl > 1 ? cudaLaunchKernelEx(&cfg, k1_rgb_pyramid_kernel<true>, a, map)
                                 : cudaLaunchKernelEx(&cfg, k1_rgb_pyramid_kernel<false>, a, map);
    if (e != cudaSuccess) {
      set_error(std::string("k1_rgb_pyramid_kernel: ") + cudaGetErrorString(e));
      return MTB_ECUDA;
    }
    ++launches;
  }
  return check_launch("k1_rgb_pyramid_kernel", launches);
}

}  // namespace mtb
