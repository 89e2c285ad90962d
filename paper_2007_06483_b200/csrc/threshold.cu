// K3: threshold + bit-pack (MTB and exclusion bitmaps) for every pyramid
// level, plus bitmap utilities (pack a bool mask, unpack, popcount) and the
// tone LUT used by the on-device stack generator.
//
// Reference semantics (bit-exact):
//   mtb bit       = g > median                         threshold.py:42-45
//   exclusion bit = |g - median| > tol  (no wrap)       threshold.py:48-56
//   packing       = LSB-first, ceil(W/64) u64 per row,
//                   zero padding bits                   bitmap.py:32-40
// A u32 word j of a packed row holds pixels 32j..32j+31 (bit x&31); the row
// pitch is 2*ceil(W/64) u32 words, byte-identical to the reference's u64 rows.
#include "swar.cuh"

namespace mtb {

struct ThreshLevel {
  int w, h;
  int64_t gray_off, gray_pitch;  // bytes (pitch is a multiple of 128)
  int64_t bit_off;               // u64 words
  int nw32;                      // u32 words per packed row
  int chunks;                    // wide level (nw32 >= 32): 1 (one warp item per row); 0: narrow
  uint32_t magic;                // narrow level: ceil(2^32 / nw32) (row = umulhi(word, magic))
  int item_begin;                // first warp item of this level (levels concatenated)
};

struct ThreshArgs {
  const uint8_t* gray;
  int64_t gray_img_stride;
  const int32_t* medians;        // [img][n]
  int tol;
  int n;
  ThreshLevel lv[kMaxLevels];
  int items;                     // warp items per image: sum over levels of h * chunks
  uint32_t* mtb;                 // bitmap arena (u32 view), image stride bit_img_words*2
  uint32_t* excl;
  int64_t bit_img_words32;
  int discard;                   // drop the consumed gray lines from L2 (no write-back)
};

// Bits of one 32-pixel word from 32 gray bytes (pixels beyond `valid` are 0).
__device__ __forceinline__ void pack32(const uint32_t (&g)[8], int valid, int med, int tol,
                                       uint32_t& mtb, uint32_t& eb) {
  const int hi = med + tol, lo = med - tol;
  uint32_t m = 0, e = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int v = (g[i >> 2] >> (8 * (i & 3))) & 0xff;
    m |= (uint32_t)(v > med) << i;
    e |= (uint32_t)((v > hi) | (v < lo)) << i;
  }
  const uint32_t keep = valid >= 32 ? 0xffffffffu : (valid <= 0 ? 0u : ((1u << valid) - 1u));
  mtb = m & keep;
  eb = e & keep;
}

// A warp item = one row of a wide level (>= 32 words per row; lane j packs
// words j, j + 32, ...), or 32 consecutive words of a narrow level's
// row-major word sequence (several rows, so no lane idles); the items of all
// levels are concatenated and the warps of an image's CTAs stride over them.  The per-level compare
// constants are built once per CTA in shared memory and the pack is the
// VABSDIFF4 / carry-majority form of the fused pipeline (th_word_t, about 7
// instructions per 4 pixels), so an item costs little beyond its bytes.
#ifndef TH_MIN_BLOCKS
#define TH_MIN_BLOCKS 8
#endif
__global__ void __launch_bounds__(256, TH_MIN_BLOCKS) threshold_levels_kernel(ThreshArgs a) {
  __shared__ ThConst s_th[kMaxLevels];
  const int img = blockIdx.y;
  if (threadIdx.x < a.n) {
    const int med = a.medians[img * a.n + threadIdx.x];
    ThConst c;
    c.med = (uint32_t)med * 0x01010101u;
    c.ym = (uint32_t)(255 - med) * 0x01010101u;
    c.yml = c.ym & 0x7f7f7f7fu;
    c.med_lo = med <= 127;
    s_th[threadIdx.x] = c;
  }
  __syncthreads();
  const bool tol_lo = a.tol <= 127;
  const uint32_t yt = (uint32_t)(255 - a.tol) * 0x01010101u, ytl = yt & 0x7f7f7f7fu;
  const int lane = threadIdx.x & 31;
  const uint8_t* gray = a.gray + img * a.gray_img_stride;
  uint32_t* mtb = a.mtb + img * a.bit_img_words32;
  uint32_t* excl = a.excl + img * a.bit_img_words32;
  const int wpc = blockDim.x >> 5;
  const int stride = gridDim.x * wpc;
  int k = 0;
  // One word: pack + store (word j of row y of level L; x0 = 32 j < w known).
  auto word = [&](const ThreshLevel& L, int y, int j, bool in_px) {
    uint32_t mw = 0, ew = 0;
    if (in_px) {
      // gray pitch is a multiple of 128 bytes: these 32 bytes are in-bounds and aligned.
      const uint8_t* src = gray + L.gray_off + (int64_t)y * L.gray_pitch + 32 * j;
      const uint4* p = reinterpret_cast<const uint4*>(src);
      const uint4 v0 = __ldcs(p), v1 = __ldcs(p + 1);
      const uint32_t g[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
      const ThConst c = s_th[k];
      const int valid = L.w - 32 * j;
      if (c.med_lo) {
        if (tol_lo) th_word_t<true, true>(g, c, yt, ytl, valid, mw, ew);
        else th_word_t<true, false>(g, c, yt, ytl, valid, mw, ew);
      } else {
        if (tol_lo) th_word_t<false, true>(g, c, yt, ytl, valid, mw, ew);
        else th_word_t<false, false>(g, c, yt, ytl, valid, mw, ew);
      }
      if (a.discard && L.chunks) {
        // wide level: words j..j+3 share one 128-B line and are lanes of this
        // warp; drop the line from L2 (no write-back) once all of them read it
        // (narrow levels keep theirs: a row's line may span two items).
        __syncwarp(__activemask());
        if ((j & 3) == 0) asm volatile("discard.global.L2 [%0], 128;" ::"l"(src) : "memory");
      }
    }
    const int64_t o = 2 * L.bit_off + (int64_t)y * L.nw32 + j;
    mtb[o] = mw;
    excl[o] = ew;
  };
  for (int it = blockIdx.x * wpc + (threadIdx.x >> 5); it < a.items; it += stride) {
    while (k + 1 < a.n && it >= a.lv[k + 1].item_begin) ++k;   // items only increase
    const ThreshLevel& L = a.lv[k];
    const int rem = it - L.item_begin;
    int y, j, jend;
    if (L.chunks) {          // wide: an item is one row, lane j packs words j, j + 32, ...
      y = rem;
      j = lane;
      jend = L.nw32;
    } else {                 // narrow: an item is 32 consecutive words of the level (several rows)
      const int f = rem * 32 + lane;
      y = (int)__umulhi((uint32_t)f, L.magic);
      j = f - y * L.nw32;
      jend = y < L.h ? j + 1 : j;
    }
#pragma unroll 1
    for (; j < jend; j += 32) word(L, y, j, 32 * j < L.w);
  }
}

// Single image of arbitrary pitch/alignment (the make_mtb / make_exclusion API).
__global__ void threshold_image_kernel(const uint8_t* __restrict__ gray, int64_t pitch, int w, int h, int med,
                                       int tol, uint32_t* __restrict__ mtb, uint32_t* __restrict__ excl) {
  const int nw32 = 2 * (int)((w + 63) / 64);
  const int64_t n = (int64_t)nw32 * h;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / nw32), j = (int)(i - (int64_t)y * nw32);
    const int x0 = 32 * j;
    uint32_t g[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int valid = w - x0;
    for (int b = 0; b < 32 && b < valid; ++b) g[b >> 2] |= (uint32_t)gray[y * pitch + x0 + b] << (8 * (b & 3));
    uint32_t mw, ew;
    pack32(g, valid, med, tol, mw, ew);
    if (mtb) mtb[i] = mw;
    if (excl) excl[i] = ew;
  }
}

__global__ void pack_mask_kernel(const uint8_t* __restrict__ mask, int64_t pitch, int w, int h,
                                 uint32_t* __restrict__ words) {
  const int nw32 = 2 * (int)((w + 63) / 64);
  const int64_t n = (int64_t)nw32 * h;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / nw32), j = (int)(i - (int64_t)y * nw32);
    const int x0 = 32 * j;
    uint32_t v = 0;
    for (int b = 0; b < 32 && x0 + b < w; ++b) v |= (uint32_t)(mask[y * pitch + x0 + b] != 0) << b;
    words[i] = v;
  }
}

__global__ void unpack_kernel(const uint32_t* __restrict__ words, int nw32, int w, int h, uint8_t* __restrict__ out,
                              int64_t pitch, uint8_t on) {
  const int64_t n = (int64_t)w * h;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / w), x = (int)(i - (int64_t)y * w);
    const uint32_t bit = (words[(int64_t)y * nw32 + (x >> 5)] >> (x & 31)) & 1u;
    out[y * pitch + x] = bit ? on : 0;
  }
}

__global__ void popcount_kernel(const uint32_t* __restrict__ words, int64_t n, unsigned long long* out) {
  unsigned c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += __popc(words[i]);
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

__global__ void count_nonzero_kernel(const uint8_t* __restrict__ cells, int64_t h, int64_t w, int64_t pitch,
                                     unsigned long long* out) {
  unsigned c = 0;
  const int64_t n = h * w;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = i / w, x = i - y * w;
    c += cells[y * pitch + x] != 0;
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

__global__ void lut_kernel(const uint8_t* __restrict__ in, const uint8_t* __restrict__ lut, int64_t n,
                           uint8_t* __restrict__ out) {
  __shared__ uint8_t s[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s[i] = lut[i];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = s[in[i]];
}

int launch_threshold_levels(const uint8_t* gray, const Plan& p, int n_img, const int32_t* medians, int tol,
                            uint64_t* mtb, uint64_t* excl, int discard, cudaStream_t st) {
  ThreshArgs a{};
  a.gray = gray;
  a.gray_img_stride = p.gray_img_bytes;
  a.medians = medians;
  a.tol = tol;
  a.n = p.n;
  int items = 0;
  for (int k = 0; k < p.n; ++k) {
    ThreshLevel& L = a.lv[k];
    L.w = p.lv[k].w;
    L.h = p.lv[k].h;
    L.gray_off = p.lv[k].gray_off;
    L.gray_pitch = p.lv[k].gray_pitch;
    L.bit_off = p.lv[k].bit_off;
    L.nw32 = (int)(2 * p.lv[k].nw64);
    L.chunks = L.nw32 >= 32 ? 1 : 0;
    L.magic = (uint32_t)((((uint64_t)1 << 32) + L.nw32 - 1) / L.nw32);   // exact for f < 2^32 / nw32
    L.item_begin = items;
    items += L.chunks ? L.h : (L.h * L.nw32 + 31) / 32;
  }
  a.items = items;
  a.mtb = reinterpret_cast<uint32_t*>(mtb);
  a.excl = reinterpret_cast<uint32_t*>(excl);
  a.bit_img_words32 = 2 * p.bit_img_words;
  a.discard = discard;
  int64_t per_img = (int64_t)num_sms() * 8 / (n_img > 0 ? n_img : 1);
  if (per_img < 1) per_img = 1;
  const int64_t need = (items + 7) / 8;   // 8 warps (items) per CTA
  if (per_img > need) per_img = need;
  threshold_levels_kernel<<<dim3((unsigned)per_img, (unsigned)n_img), 256, 0, st>>>(a);
  return check_launch("threshold_levels_kernel");
}

}  // namespace mtb

using namespace mtb;

extern "C" int mtb_threshold_pack(const uint8_t* gray, int64_t pitch, int w, int h, int median, int tol,
                                  uint64_t* mtb, uint64_t* exclusion, void* stream) {
  clear_error();
  MTB_REQUIRE(gray, "null gray pointer");
  MTB_REQUIRE(w >= 1 && h >= 1, "image dimensions must be at least 1x1");
  MTB_REQUIRE(pitch >= w, "pitch smaller than row");
  if (!mtb && !exclusion) return MTB_OK;
  const int64_t n = 2 * ((w + 63) / 64) * (int64_t)h;
  threshold_image_kernel<<<grid_cap(n, 256), 256, 0, as_stream(stream)>>>(
      gray, pitch, w, h, median, tol, reinterpret_cast<uint32_t*>(mtb), reinterpret_cast<uint32_t*>(exclusion));
  return check_launch("threshold_image_kernel");
}

extern "C" int mtb_pack_mask(const uint8_t* mask, int64_t pitch, int w, int h, uint64_t* words, void* stream) {
  clear_error();
  MTB_REQUIRE(mask && words, "null pointer");
  MTB_REQUIRE(w >= 1 && h >= 1, "mask dimensions must be at least 1x1");
  const int64_t n = 2 * ((w + 63) / 64) * (int64_t)h;
  pack_mask_kernel<<<grid_cap(n, 256), 256, 0, as_stream(stream)>>>(mask, pitch, w, h,
                                                                   reinterpret_cast<uint32_t*>(words));
  return check_launch("pack_mask_kernel");
}

extern "C" int mtb_unpack_bits(const uint64_t* words, int64_t nwords64, int w, int h, uint8_t* cells,
                               int64_t cell_pitch, int on_value, void* stream) {
  clear_error();
  MTB_REQUIRE(words && cells, "null pointer");
  MTB_REQUIRE(w >= 1 && h >= 1, "bitmap dimensions must be at least 1x1");
  MTB_REQUIRE(nwords64 * 64 >= w, "row word count too small for width");
  unpack_kernel<<<grid_cap((int64_t)w * h, 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const uint32_t*>(words), (int)(2 * nwords64), w, h, cells, cell_pitch, (uint8_t)on_value);
  return check_launch("unpack_kernel");
}

extern "C" int mtb_count_ones_packed(const uint64_t* words, int64_t h, int64_t nwords64, unsigned long long* out,
                                     void* stream) {
  clear_error();
  MTB_REQUIRE(out, "null output pointer");
  MTB_REQUIRE(h >= 0 && nwords64 >= 0, "negative dimensions");
  MTB_CUDA(cudaMemsetAsync(out, 0, sizeof(unsigned long long), as_stream(stream)));
  const int64_t n = 2 * h * nwords64;
  if (n == 0) return MTB_OK;
  MTB_REQUIRE(words, "null words pointer");
  popcount_kernel<<<grid_cap(n, 256, 4), 256, 0, as_stream(stream)>>>(reinterpret_cast<const uint32_t*>(words), n,
                                                                     out);
  return check_launch("popcount_kernel");
}

extern "C" int mtb_count_ones_bytemap(const uint8_t* cells, int64_t h, int64_t w, int64_t pitch,
                                      unsigned long long* out, void* stream) {
  clear_error();
  MTB_REQUIRE(out, "null output pointer");
  MTB_REQUIRE(h >= 0 && w >= 0 && pitch >= w, "bad dimensions");
  MTB_CUDA(cudaMemsetAsync(out, 0, sizeof(unsigned long long), as_stream(stream)));
  if (h * w == 0) return MTB_OK;
  MTB_REQUIRE(cells, "null cells pointer");
  count_nonzero_kernel<<<grid_cap(h * w, 256, 4), 256, 0, as_stream(stream)>>>(cells, h, w, pitch, out);
  return check_launch("count_nonzero_kernel");
}

extern "C" int mtb_apply_lut(const uint8_t* in, const uint8_t* lut, int64_t n, uint8_t* out, void* stream) {
  clear_error();
  MTB_REQUIRE(in && lut && out, "null pointer");
  if (n <= 0) return MTB_OK;
  lut_kernel<<<grid_cap(n, 256), 256, 0, as_stream(stream)>>>(in, lut, n, out);
  return check_launch("lut_kernel");
}
