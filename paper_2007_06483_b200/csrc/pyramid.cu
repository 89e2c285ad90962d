// K1: RGB8 -> gray -> 2x box pyramid -> per-level 256-bin histograms, fused,
// plus the reference-granularity primitives to_grayscale / downsample_half /
// histogram.
//
// Reference semantics (bit-exact):
//   gray   = (54 R + 183 G + 19 B) >> 8                       image.py:17-19,58-68
//   down   = (a + b + c + d + 2) >> 2 over aligned 2x2 blocks,
//            dims floor-halved, trailing odd row/col dropped    pyramid.py:17-32
//   levels = min(requested, max_levels(w, h))                  pyramid.py:35-62
//   hist   = 256-bin counts per level                          threshold.py:25-28
//
// Tiling: a level-s tile is 32 rows x 128 columns.  Level s+t pixel (x, y)
// depends only on the level-s block [x*2^t, (x+1)*2^t) x [y*2^t, (y+1)*2^t),
// so with 32-row/128-col tiles aligned to the image origin, levels s..s+5 are
// tile-local and no halo is needed.  Level s+t pixel (x, y) exists iff
// x < (w >> t) and y < (h >> t) (floor halving), which is exactly the set of
// tile pixels whose full 2^t x 2^t source block lies inside the image.
#include "common.cuh"

namespace mtb {

constexpr int kTileRows = 32;
constexpr int kTileCols = 128;
constexpr int kTileLevels = 6;        // levels produced per tile pass (t = 0..5)
constexpr int kPyrThreads = 256;      // 16 level-s pixels per thread
constexpr int kHistStride = 32;       // u32 stride between global bins (one 128-B line each)

struct PyrArgs {
  const uint8_t* src;
  int64_t src_pitch;
  int64_t src_img_stride;
  int src_w, src_h;                   // dims of the source level s
  uint8_t* gray;                      // gray arena base (image 0)
  int64_t gray_img_stride;
  int64_t off[kTileLevels];           // arena offsets of levels s..s+5
  int64_t pitch[kTileLevels];
  int w[kTileLevels], h[kTileLevels];
  int nl;                             // tile levels produced (t = 0..nl-1), 1..6
  uint32_t* hist;                     // [img][level][bin] * hist_bin (spread: kHistStride, dense: 1)
  int64_t hist_img_stride;            // u32 elements
  int hist_bin;                       // u32 stride between global bins
  int hist_level0;                    // global level index of t = 0
  int tiles_x, tiles_y;
  int edge_only;                      // 1: only the partial right column / bottom row tiles
};

__device__ __forceinline__ uint4 ld_stream16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t avg4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return (a + b + c + d + 2u) >> 2;
}

// Gray value of the pixel whose R byte is byte `o` of the 12-word run `w`.
template <int O>
__device__ __forceinline__ uint32_t gray_at(const uint32_t (&w)[12]) {
  constexpr int a = O >> 2, s = O & 3;
  constexpr uint32_t sel = (s) | ((s + 1) << 4) | ((s + 2) << 8) | ((s + 3) << 12);
  const uint32_t hi = (a + 1 < 12) ? w[(a + 1 < 12) ? a + 1 : 11] : 0u;
  const uint32_t px = __byte_perm(w[a], hi, sel);       // bytes R, G, B, x
  return __dp4a(px, 0x0013B736u, 0u) >> 8;              // 54 R + 183 G + 19 B (x weight 0)
}

// RGB_SRC: level s = 0 comes from RGB8 and is itself stored + histogrammed.
// Otherwise the source is an existing gray level whose histogram is done.
template <bool RGB_SRC>
__global__ void __launch_bounds__(kPyrThreads)
pyramid_tiles_kernel(PyrArgs a) {
  __shared__ __align__(16) uint8_t s_lv[4096 + 1024 + 256 + 64 + 16 + 16];
  __shared__ uint32_t s_hist[kTileLevels * 256];
  constexpr int kLvOff[kTileLevels] = {0, 4096, 5120, 5376, 5440, 5456};

  const int tid = threadIdx.x;
  const int img = blockIdx.y;
  for (int i = tid; i < kTileLevels * 256; i += kPyrThreads) s_hist[i] = 0;

  const uint8_t* src = a.src + img * a.src_img_stride;
  uint8_t* gray = a.gray + img * a.gray_img_stride;
  const bool vec_ok = RGB_SRC ? ((a.src_pitch & 15) == 0 && ((uintptr_t)a.src & 15) == 0 &&
                                 (a.src_img_stride & 15) == 0)
                              : ((a.src_pitch & 15) == 0 && ((uintptr_t)a.src & 15) == 0 &&
                                 (a.src_img_stride & 15) == 0);
  const int ntiles = a.tiles_x * a.tiles_y;
  __syncthreads();

  // Edge mode: tiles of the partial right column (if w % 128) then of the
  // partial bottom row (if h % 32), the ones the interior kernel skips.
  const bool col_part = (a.src_w % kTileCols) != 0, row_part = (a.src_h % kTileRows) != 0;
  const int n_col = col_part ? a.tiles_y : 0;
  const int n_row = row_part ? a.tiles_x - (col_part ? 1 : 0) : 0;
  const int n_work = a.edge_only ? n_col + n_row : ntiles;
  for (int tile = blockIdx.x; tile < n_work; tile += gridDim.x) {
    int ty, tx;
    if (!a.edge_only) {
      ty = tile / a.tiles_x;
      tx = tile - ty * a.tiles_x;
    } else if (tile < n_col) {
      ty = tile;
      tx = a.tiles_x - 1;
    } else {
      ty = a.tiles_y - 1;
      tx = tile - n_col;
    }

    // ---- level s (t = 0): 16 pixels per thread -------------------------
    {
      const int r = tid >> 3, c = (tid & 7) << 4;
      const int y = ty * kTileRows + r;
      const int x0 = tx * kTileCols + c;
      uint32_t g[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) g[i] = 0;
      if (y < a.src_h && x0 < a.src_w) {
        const uint8_t* row = src + (int64_t)y * a.src_pitch;
        const bool full = x0 + 16 <= a.src_w;
        if (RGB_SRC) {
          if (full && vec_ok) {
            uint32_t w[12];
            const uint4 v0 = ld_stream16(row + 3 * (int64_t)x0);
            const uint4 v1 = ld_stream16(row + 3 * (int64_t)x0 + 16);
            const uint4 v2 = ld_stream16(row + 3 * (int64_t)x0 + 32);
            w[0] = v0.x; w[1] = v0.y; w[2] = v0.z; w[3] = v0.w;
            w[4] = v1.x; w[5] = v1.y; w[6] = v1.z; w[7] = v1.w;
            w[8] = v2.x; w[9] = v2.y; w[10] = v2.z; w[11] = v2.w;
            g[0] = gray_at<0>(w);   g[1] = gray_at<3>(w);   g[2] = gray_at<6>(w);
            g[3] = gray_at<9>(w);   g[4] = gray_at<12>(w);  g[5] = gray_at<15>(w);
            g[6] = gray_at<18>(w);  g[7] = gray_at<21>(w);  g[8] = gray_at<24>(w);
            g[9] = gray_at<27>(w);  g[10] = gray_at<30>(w); g[11] = gray_at<33>(w);
            g[12] = gray_at<36>(w); g[13] = gray_at<39>(w); g[14] = gray_at<42>(w);
            g[15] = gray_at<45>(w);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              if (x0 + i < a.src_w) {
                const uint8_t* p = row + 3 * (int64_t)(x0 + i);
                g[i] = (54u * p[0] + 183u * p[1] + 19u * p[2]) >> 8;
              }
            }
          }
        } else {
          if (full && vec_ok) {
            const uint4 v = ld_stream16(row + x0);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 16; ++i) g[i] = (w[i >> 2] >> (8 * (i & 3))) & 0xffu;
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (x0 + i < a.src_w) g[i] = row[x0 + i];
          }
        }
      }
      uint4 packed;
      packed.x = g[0] | (g[1] << 8) | (g[2] << 16) | (g[3] << 24);
      packed.y = g[4] | (g[5] << 8) | (g[6] << 16) | (g[7] << 24);
      packed.z = g[8] | (g[9] << 8) | (g[10] << 16) | (g[11] << 24);
      packed.w = g[12] | (g[13] << 8) | (g[14] << 16) | (g[15] << 24);
      *reinterpret_cast<uint4*>(s_lv + r * kTileCols + c) = packed;
      if (RGB_SRC) {
        if (y < a.h[0] && x0 < a.pitch[0])
          *reinterpret_cast<uint4*>(gray + a.off[0] + (int64_t)y * a.pitch[0] + x0) = packed;
        if (y < a.h[0]) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (x0 + i < a.w[0]) atomicAdd(&s_hist[g[i]], 1u);
        }
      }
    }
    __syncthreads();

    // ---- level s+1: 16 x 64, 4 pixels per thread ------------------------
    if (a.nl > 1) {
      const int r = tid >> 4, c = (tid & 15) << 2;
      const uint8_t* s0 = s_lv + (2 * r) * kTileCols + 2 * c;
      const uint2 u = *reinterpret_cast<const uint2*>(s0);
      const uint2 d = *reinterpret_cast<const uint2*>(s0 + kTileCols);
      uint32_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t uw = (k < 2) ? u.x : u.y, dw = (k < 2) ? d.x : d.y;
        const int sh = 16 * (k & 1);
        o[k] = avg4((uw >> sh) & 0xff, (uw >> (sh + 8)) & 0xff, (dw >> sh) & 0xff, (dw >> (sh + 8)) & 0xff);
      }
      const uint32_t packed = o[0] | (o[1] << 8) | (o[2] << 16) | (o[3] << 24);
      *reinterpret_cast<uint32_t*>(s_lv + kLvOff[1] + r * 64 + c) = packed;
      const int y = ty * (kTileRows >> 1) + r, x0 = tx * (kTileCols >> 1) + c;
      if (y < a.h[1]) {
        if (x0 < a.pitch[1])
          *reinterpret_cast<uint32_t*>(gray + a.off[1] + (int64_t)y * a.pitch[1] + x0) = packed;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (x0 + k < a.w[1]) atomicAdd(&s_hist[256 + o[k]], 1u);
      }
    }
    __syncthreads();

    // ---- levels s+2 .. s+nl-1: one pixel per thread ---------------------
#pragma unroll
    for (int t = 2; t < kTileLevels; ++t) {
      if (t < a.nl) {
        const int rows = kTileRows >> t, cols = kTileCols >> t;
        if (tid < rows * cols) {
          const int r = tid / cols, c = tid - r * cols;
          const uint8_t* sp = s_lv + kLvOff[t - 1] + (2 * r) * (2 * cols) + 2 * c;
          const uint32_t v = avg4(sp[0], sp[1], sp[2 * cols], sp[2 * cols + 1]);
          s_lv[kLvOff[t] + r * cols + c] = (uint8_t)v;
          const int y = ty * rows + r, x = tx * cols + c;
          if (y < a.h[t]) {
            if (x < a.pitch[t]) gray[a.off[t] + (int64_t)y * a.pitch[t] + x] = (uint8_t)v;
            if (x < a.w[t]) atomicAdd(&s_hist[t * 256 + v], 1u);
          }
        }
      }
      __syncthreads();
    }
  }

  // ---- flush the CTA's histograms (skip empty bins) -----------------------
  const int t0 = RGB_SRC ? 0 : 1;
  uint32_t* gh = a.hist + img * a.hist_img_stride;
  for (int i = t0 * 256 + tid; i < a.nl * 256; i += kPyrThreads) {
    const uint32_t v = s_hist[i];
    if (v) atomicAdd(&gh[(int64_t)(a.hist_level0 * 256 + i) * a.hist_bin], v);
  }
}

// Gather the spread histogram into dense u32 [img][level][256] and take the
// lower median of each (threshold.py:31-39): one warp per (image, level).
__global__ void hist_median_kernel(const uint32_t* __restrict__ spread, int64_t spread_img_stride, int bin,
                                   int n_levels, uint32_t* __restrict__ dense,
                                   int32_t* __restrict__ medians) {
  const int lane = threadIdx.x & 31;
  const int level = threadIdx.x >> 5;
  const int img = blockIdx.x;
  if (level >= n_levels) return;
  const uint32_t* base = spread + img * spread_img_stride;
  if (bin == 0) bin = base[spread_img_stride - 1] ? 1 : kHistStride;   // layout marker (hist_prepare)
  const uint32_t* src = base + (int64_t)level * 256 * bin;
  uint32_t bins[8];
  unsigned long long s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    bins[i] = src[(int64_t)(lane * 8 + i) * bin];
    s += bins[i];
  }
  if (dense) {
    uint32_t* dst = dense + ((int64_t)img * n_levels + level) * 256;
#pragma unroll
    for (int i = 0; i < 8; ++i) dst[lane * 8 + i] = bins[i];
  }
  unsigned long long incl = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  const unsigned long long total = __shfl_sync(0xffffffffu, incl, 31);
  const unsigned long long target = (total + 1) >> 1;
  const unsigned mask = __ballot_sync(0xffffffffu, incl >= target);
  int med = -1;
  if (total > 0) {
    const int L = __ffs(mask) - 1;
    if (lane == L) {
      unsigned long long c = incl - s;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        c += bins[i];
        if (c >= target) { med = lane * 8 + i; break; }
      }
    }
    med = __shfl_sync(0xffffffffu, med, L);
  }
  if (lane == 0) medians[img * n_levels + level] = med;
}

// ------------------------------------------------------------ primitives --

__global__ void gray_kernel(const uint8_t* __restrict__ rgb, int64_t rgb_pitch, int64_t rgb_img_stride,
                            int w, int h, uint8_t* __restrict__ gray, int64_t gray_pitch,
                            int64_t gray_img_stride) {
  const int img = blockIdx.y;
  const int64_t n = (int64_t)w * h;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / w), x = (int)(i - (int64_t)y * w);
    const uint8_t* p = rgb + img * rgb_img_stride + y * rgb_pitch + 3 * (int64_t)x;
    gray[img * gray_img_stride + y * gray_pitch + x] = (uint8_t)((54u * p[0] + 183u * p[1] + 19u * p[2]) >> 8);
  }
}

__global__ void downsample_kernel(const uint8_t* __restrict__ src, int64_t src_pitch, int w2, int h2,
                                  uint8_t* __restrict__ dst, int64_t dst_pitch) {
  const int64_t n = (int64_t)w2 * h2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / w2), x = (int)(i - (int64_t)y * w2);
    const uint8_t* p = src + (2 * (int64_t)y) * src_pitch + 2 * x;
    dst[y * dst_pitch + x] = (uint8_t)avg4(p[0], p[1], p[src_pitch], p[src_pitch + 1]);
  }
}

__global__ void histogram_kernel(const uint8_t* __restrict__ gray, int64_t pitch, int w, int h,
                                 unsigned long long* __restrict__ hist) {
  __shared__ uint32_t s[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const int64_t n = (int64_t)w * h;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / w), x = (int)(i - (int64_t)y * w);
    atomicAdd(&s[gray[y * pitch + x]], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (s[i]) atomicAdd(&hist[i], (unsigned long long)s[i]);
}

__global__ void median64_kernel(const unsigned long long* __restrict__ hist, int n_hist,
                                int32_t* __restrict__ medians) {
  const int lane = threadIdx.x & 31;
  const int hidx = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (hidx >= n_hist) return;
  const unsigned long long* src = hist + (int64_t)hidx * 256;
  unsigned long long bins[8], s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) { bins[i] = src[lane * 8 + i]; s += bins[i]; }
  unsigned long long incl = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  const unsigned long long total = __shfl_sync(0xffffffffu, incl, 31);
  const unsigned long long target = (total + 1) >> 1;
  const unsigned mask = __ballot_sync(0xffffffffu, incl >= target);
  int med = -1;
  if (total > 0) {
    const int L = __ffs(mask) - 1;
    if (lane == L) {
      unsigned long long c = incl - s;
      for (int i = 0; i < 8; ++i) { c += bins[i]; if (c >= target) { med = lane * 8 + i; break; } }
    }
    med = __shfl_sync(0xffffffffu, med, L);
  }
  if (lane == 0) medians[hidx] = med;
}

// -------------------------------------------------------------- launchers --

// Spread-histogram workspace needed by launch_pyramid (u32 elements / image).
int64_t spread_hist_elems(int n_levels) { return (int64_t)n_levels * 256 * kHistStride; }

// Bin stride of the staged histograms of one K1 launch: spread (one 128-B
// line per bin) when many CTAs flush into one image's histogram, dense when
// each CTA's tile range covers >= 2 whole images (the flushes of an image
// then come from a handful of CTAs; the memset and the median pass touch
// 32x less: ~200 MB less per 1024 small images).  Each image's workspace
// region keeps the spread size; its LAST word records the layout (nonzero:
// dense; in the spread layout it is an unused word of the last bin's line),
// so mtb_threshold_levels reads the histograms right whatever call filled them.
int hist_bin_for(const Plan& p, int n_img) {
  const int64_t tiles = (int64_t)((p.lv[0].w + 255) / 256) * ((p.lv[0].h + 31) / 32);
  return (int64_t)n_img * tiles >= 2 * tiles * num_sms() ? 1 : kHistStride;
}

// Zeroes the histogram workspace of n_img images for a K1 launch with this
// bin stride and writes the per-image layout marker.
int hist_prepare(uint32_t* hist_ws, const Plan& p, int n_img, int hist_bin, cudaStream_t st) {
  const int64_t region = spread_hist_elems(p.n);
  if (hist_bin == kHistStride) {
    MTB_CUDA(cudaMemsetAsync(hist_ws, 0, sizeof(uint32_t) * region * n_img, st));
  } else {
    const size_t pitch = sizeof(uint32_t) * region;
    MTB_CUDA(cudaMemset2DAsync(hist_ws, pitch, 0, sizeof(uint32_t) * (size_t)p.n * 256 * hist_bin, n_img, st));
    MTB_CUDA(cudaMemset2DAsync(hist_ws + region - 1, pitch, 1, sizeof(uint32_t), n_img, st));
  }
  return MTB_OK;
}

// Builds gray levels 0..n-1 (plan p) and their spread histograms for n_img
// images.  Level 0 comes from RGB; deeper levels are produced 6 per pass.
int launch_k1_rgb(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride, int n_img, const Plan& p,
                  uint8_t* gray, uint32_t* spread_hist, int64_t hist_img_stride, int hist_bin, cudaStream_t st);
bool k1_rgb_supported(int w, int64_t rgb_pitch, int64_t rgb_img_stride, const void* rgb);

// Builds gray levels 0..n-1 (plan p) and their spread histograms for n_img
// images: levels 0..5 by the fused RGB kernel (k1_rgb.cu), deeper levels by
// tile passes over the deepest level produced so far (6 levels per pass).
int launch_pyramid(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride, int n_img,
                   const Plan& p, uint8_t* gray, uint32_t* spread_hist, int hist_bin, cudaStream_t st) {
  const int64_t hist_img = spread_hist_elems(p.n);   // per-image region; dense bins use its start
  // Interior tiles: the fast kernel (needs 16-B aligned RGB rows).  Edge
  // tiles (and every tile when rows are unaligned): the generic kernel.
  const bool vec_ok = k1_rgb_supported(p.lv[0].w, rgb_pitch, rgb_img_stride, rgb);
  int launches = 0;
  if (vec_ok) {
    int rc = launch_k1_rgb(rgb, rgb_pitch, rgb_img_stride, n_img, p, gray, spread_hist, hist_img, hist_bin, st);
    if (rc) return rc;
  }
  {
    PyrArgs a{};
    a.src = rgb;
    a.src_pitch = rgb_pitch;
    a.src_img_stride = rgb_img_stride;
    a.src_w = p.lv[0].w;
    a.src_h = p.lv[0].h;
    a.gray = gray;
    a.gray_img_stride = p.gray_img_bytes;
    a.nl = p.n < kTileLevels ? p.n : kTileLevels;
    for (int t = 0; t < kTileLevels; ++t) {
      const int l = t < p.n ? t : p.n - 1;
      a.off[t] = p.lv[l].gray_off;
      a.pitch[t] = t < p.n ? p.lv[l].gray_pitch : 0;
      a.w[t] = t < p.n ? p.lv[l].w : 0;
      a.h[t] = t < p.n ? p.lv[l].h : 0;
    }
    a.hist = spread_hist;
    a.hist_img_stride = hist_img;
    a.hist_bin = hist_bin;
    a.hist_level0 = 0;
    a.tiles_x = (int)((a.src_w + kTileCols - 1) / kTileCols);
    a.tiles_y = (int)((a.src_h + kTileRows - 1) / kTileRows);
    a.edge_only = 0;
    // The TMA kernel covers every tile (edges included); the generic kernel
    // only runs when the RGB rows do not allow the tensor map.
    const int64_t ntiles = vec_ok ? 0 : (int64_t)a.tiles_x * a.tiles_y;
    if (ntiles > 0) {
      int64_t per_img = (int64_t)num_sms() * 4 / (n_img > 0 ? n_img : 1);
      if (per_img < 1) per_img = 1;
      if (per_img > ntiles) per_img = ntiles;
      pyramid_tiles_kernel<true><<<dim3((unsigned)per_img, (unsigned)n_img), kPyrThreads, 0, st>>>(a);
      ++launches;
    }
  }
  int s = 5;
  while (s < p.n - 1) {
    PyrArgs a{};
    a.src = gray + p.lv[s].gray_off;
    a.src_pitch = p.lv[s].gray_pitch;
    a.src_img_stride = p.gray_img_bytes;
    a.src_w = p.lv[s].w;
    a.src_h = p.lv[s].h;
    a.gray = gray;
    a.gray_img_stride = p.gray_img_bytes;
    a.nl = p.n - s < kTileLevels ? p.n - s : kTileLevels;
    for (int t = 0; t < kTileLevels; ++t) {
      const int l = s + t < p.n ? s + t : p.n - 1;
      a.off[t] = p.lv[l].gray_off;
      a.pitch[t] = s + t < p.n ? p.lv[l].gray_pitch : 0;
      a.w[t] = s + t < p.n ? p.lv[l].w : 0;
      a.h[t] = s + t < p.n ? p.lv[l].h : 0;
    }
    a.hist = spread_hist;
    a.hist_img_stride = hist_img;
    a.hist_bin = hist_bin;
    a.hist_level0 = s;
    a.tiles_x = (int)((a.src_w + kTileCols - 1) / kTileCols);
    a.tiles_y = (int)((a.src_h + kTileRows - 1) / kTileRows);
    a.edge_only = 0;
    const int64_t ntiles = (int64_t)a.tiles_x * a.tiles_y;
    int64_t per_img = (int64_t)num_sms() * 4 / (n_img > 0 ? n_img : 1);
    if (per_img < 1) per_img = 1;
    if (per_img > ntiles) per_img = ntiles;
    pyramid_tiles_kernel<false><<<dim3((unsigned)per_img, (unsigned)n_img), kPyrThreads, 0, st>>>(a);
    ++launches;
    s += a.nl - 1;
  }
  return launches ? check_launch("pyramid_tiles_kernel", launches) : MTB_OK;
}

// hist_bin 0: per image, from the layout marker hist_prepare left in the
// region's last word (the split entry points cannot know the layout the
// pyramid call chose).
int launch_hist_median(const uint32_t* spread_hist, int n_img, int n_levels, int hist_bin, uint32_t* dense,
                       int32_t* medians, cudaStream_t st) {
  hist_median_kernel<<<n_img, 32 * n_levels, 0, st>>>(spread_hist, spread_hist_elems(n_levels), hist_bin,
                                                      n_levels, dense, medians);
  return check_launch("hist_median_kernel");
}

}  // namespace mtb

using namespace mtb;

extern "C" int mtb_to_grayscale(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride, int w, int h,
                                int n_img, uint8_t* gray, int64_t gray_pitch, int64_t gray_img_stride,
                                void* stream) {
  clear_error();
  MTB_REQUIRE(rgb && gray, "null pointer");
  MTB_REQUIRE(w >= 1 && h >= 1 && n_img >= 1, "image dimensions must be at least 1x1");
  MTB_REQUIRE(rgb_pitch >= 3 * (int64_t)w && gray_pitch >= w, "pitch smaller than row");
  dim3 grid(grid_cap((int64_t)w * h, 256), n_img);
  gray_kernel<<<grid, 256, 0, as_stream(stream)>>>(rgb, rgb_pitch, rgb_img_stride, w, h, gray, gray_pitch,
                                                   gray_img_stride);
  return check_launch("gray_kernel");
}

extern "C" int mtb_downsample_half(const uint8_t* src, int64_t src_pitch, int w, int h, uint8_t* dst,
                                   int64_t dst_pitch, void* stream) {
  clear_error();
  MTB_REQUIRE(src && dst, "null pointer");
  MTB_REQUIRE(w >= 2 && h >= 2, "cannot downsample; need at least 2x2");
  MTB_REQUIRE(src_pitch >= w && dst_pitch >= w / 2, "pitch smaller than row");
  const int w2 = w / 2, h2 = h / 2;
  downsample_kernel<<<grid_cap((int64_t)w2 * h2, 256), 256, 0, as_stream(stream)>>>(src, src_pitch, w2, h2, dst,
                                                                                    dst_pitch);
  return check_launch("downsample_kernel");
}

extern "C" int mtb_histogram(const uint8_t* gray, int64_t pitch, int w, int h, unsigned long long* hist,
                             void* stream) {
  clear_error();
  MTB_REQUIRE(gray && hist, "null pointer");
  MTB_REQUIRE(w >= 1 && h >= 1, "image dimensions must be at least 1x1");
  MTB_CUDA(cudaMemsetAsync(hist, 0, 256 * sizeof(unsigned long long), as_stream(stream)));
  histogram_kernel<<<grid_cap((int64_t)w * h, 256, 2), 256, 0, as_stream(stream)>>>(gray, pitch, w, h, hist);
  return check_launch("histogram_kernel");
}

extern "C" int mtb_median_from_histogram(const unsigned long long* hist, int n_hist, int32_t* medians,
                                         void* stream) {
  clear_error();
  MTB_REQUIRE(hist && medians, "null pointer");
  MTB_REQUIRE(n_hist >= 1, "need at least one histogram");
  const int per_block = 4;
  median64_kernel<<<(n_hist + per_block - 1) / per_block, 32 * per_block, 0, as_stream(stream)>>>(hist, n_hist,
                                                                                                   medians);
  return check_launch("median64_kernel");
}
