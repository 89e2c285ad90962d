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

#include "k1_tile.cuh"

namespace cg = cooperative_groups;

namespace mtb {

struct K1Smem {
  uint32_t hist[kK1Groups][6][256];                    // first: 1 KB-aligned levels, one set per group
  uint8_t rgb[kK1Groups][kK1Stages][kK1TileBytes];     // TMA rings
  uint8_t l3[kK1Groups][2][4][32];                     // level-3 tile values, by tile parity
  unsigned long long full[kK1Groups][kK1Stages];       // mbarriers of the ring stages
};
constexpr int kK1SmemBytes = (int)sizeof(K1Smem) + 1024;  // + alignment slack

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
        atomicAdd(&gh[(int64_t)i * a.hist_bin], c);
        gh_s[i] = 0;
      }
    }
  };
  if (t == 0) {
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
    mbar_wait(&S.full[g][stage], (uint32_t)(k / kK1Stages) & 1u);
    {
      const uint8_t* src = S.rgb[g][stage] + (8 * wg) * kK1RowBytes + 24 * lane;
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) v[r][c] = *reinterpret_cast<const uint2*>(src + r * kK1RowBytes + 8 * c);
    }
    group_bar(g);  // stage consumed by all 128 threads; l3 of tile k-1 complete
    if (t == 0 && tile + kK1Groups * kK1Stages < t_end) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(tile + kK1Groups * kK1Stages, stage);
    }
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
  if (k > 0) {
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

PFN_cuTensorMapEncodeTiled_v12000 k1_encode_tiled() { return encode_tiled(); }

bool k1_rgb_supported(int w, int64_t rgb_pitch, int64_t rgb_img_stride, const void* rgb) {
  return (3 * (int64_t)w) % 4 == 0 && (rgb_pitch & 15) == 0 && (rgb_img_stride & 15) == 0 &&
         ((uintptr_t)rgb & 15) == 0 && encode_tiled() != nullptr;
}

static int g_keep_gray = 0;   // set by mtb_set_gray_policy (capi.cu)
void k1_set_keep_gray(int v) { g_keep_gray = v; }

// Levels 0..min(n,6)-1 of n_img images in ONE persistent launch (one CTA per
// SM over the image-major tile sequence).
int launch_k1_rgb(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride, int n_img, const Plan& p,
                  uint8_t* gray, uint32_t* spread_hist, int64_t hist_img_stride, int hist_bin, cudaStream_t st) {
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
  a.hist_bin = hist_bin;
  a.keep_gray = g_keep_gray;
  a.tiles_x = (a.w + kK1TilePx - 1) / kK1TilePx;   // edge tiles included: TMA zero-fills outside the image
  a.tiles_y = (a.h + kK1TileRows - 1) / kK1TileRows;
  a.n_img = n_img;
  const int64_t ntiles = (int64_t)a.tiles_x * a.tiles_y * n_img;
  if (ntiles == 0) return MTB_OK;
  if (ntiles >= ((int64_t)1 << 31)) {
    set_error("k1: too many tiles in one launch");
    return MTB_EINVAL;
  }
  // the shared-memory opt-in is per device (cheap; set on every call)
  MTB_CUDA(cudaFuncSetAttribute(k1_rgb_pyramid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kK1SmemBytes));
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
