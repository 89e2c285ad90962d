// K5: whole-pixel translation with fill (shift_rgb / shift_gray).
//
// Reference semantics (image.py:71-106): out(x, y) = in(x - dx, y - dy) when
// 0 <= x - dx < w and 0 <= y - dy < h, otherwise the fill value.
#include "common.cuh"

namespace mtb {

// Four output pixels (12 bytes) per thread; offsets per image from device memory.
__global__ void __launch_bounds__(256)
shift_rgb_kernel(const uint8_t* __restrict__ in, int64_t in_pitch, int64_t in_img_stride, int w, int h,
                 const int32_t* __restrict__ offsets, uint32_t fill, uint8_t* __restrict__ out, int64_t out_pitch,
                 int64_t out_img_stride, bool aligned) {
  const int img = blockIdx.y;
  const int dx = offsets[2 * img], dy = offsets[2 * img + 1];
  const uint8_t* src = in + img * in_img_stride;
  uint8_t* dst = out + img * out_img_stride;
  const int groups = (w + 3) / 4;
  const int64_t n = (int64_t)groups * h;
  const uint8_t f0 = fill & 0xff, f1 = (fill >> 8) & 0xff, f2 = (fill >> 16) & 0xff;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / groups);
    const int x0 = 4 * (int)(i - (int64_t)y * groups);
    const int sy = y - dy;
    const bool row_ok = sy >= 0 && sy < h;
    uint8_t b[12];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int sx = x0 + k - dx;
      if (row_ok && sx >= 0 && sx < w) {
        const uint8_t* p = src + (int64_t)sy * in_pitch + 3 * (int64_t)sx;
        b[3 * k] = p[0]; b[3 * k + 1] = p[1]; b[3 * k + 2] = p[2];
      } else {
        b[3 * k] = f0; b[3 * k + 1] = f1; b[3 * k + 2] = f2;
      }
    }
    uint8_t* q = dst + (int64_t)y * out_pitch + 3 * (int64_t)x0;
    if (aligned && x0 + 4 <= w) {
      uint32_t* q4 = reinterpret_cast<uint32_t*>(q);
#pragma unroll
      for (int k = 0; k < 3; ++k)
        q4[k] = b[4 * k] | (b[4 * k + 1] << 8) | (b[4 * k + 2] << 16) | ((uint32_t)b[4 * k + 3] << 24);
    } else {
      for (int k = 0; k < 4 && x0 + k < w; ++k) {
        q[3 * k] = b[3 * k]; q[3 * k + 1] = b[3 * k + 1]; q[3 * k + 2] = b[3 * k + 2];
      }
    }
  }
}

// 16 px (48 B) per thread: interior chunks read the 64-B aligned superset of
// their source bytes with four 16-B loads and rebuild the 12 output words by
// byte funnels (PRMT), then write three 16-B stores; chunks touching the
// image border (or a fill region) take the per-pixel path.  Needs 16-B
// aligned output rows.
template <int Q>   // Q = (source byte offset >> 2) & 3
__device__ __forceinline__ void funnel12(const uint32_t (&w)[16], uint32_t sel, uint32_t (&o)[12]) {
#pragma unroll
  for (int k = 0; k < 12; ++k) o[k] = __byte_perm(w[Q + k], w[Q + k + 1], sel);
}

__global__ void __launch_bounds__(256)
shift_rgb16_kernel(const uint8_t* __restrict__ in, int64_t in_pitch, int64_t in_img_stride, int w, int h,
                   const int32_t* __restrict__ offsets, uint32_t fill, uint8_t* __restrict__ out, int64_t out_pitch,
                   int64_t out_img_stride) {
  const int img = blockIdx.y;
  const int dx = offsets[2 * img], dy = offsets[2 * img + 1];
  const uint8_t* src = in + img * in_img_stride;
  uint8_t* dst = out + img * out_img_stride;
  const int chunks = (w + 15) / 16;
  const int64_t n = (int64_t)chunks * h;
  const uint8_t f0 = fill & 0xff, f1 = (fill >> 8) & 0xff, f2 = (fill >> 16) & 0xff;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / chunks);
    const int x0 = 16 * (int)(i - (int64_t)y * chunks);
    const int sy = y - dy, sx0 = x0 - dx;
    uint8_t* q = dst + (int64_t)y * out_pitch + 3 * (int64_t)x0;
    if (sy >= 0 && sy < h && sx0 >= 0 && sx0 + 16 <= w && x0 + 16 <= w) {
      const uint8_t* a = src + (int64_t)sy * in_pitch + 3 * (int64_t)sx0;
      const uintptr_t s = (uintptr_t)a & 15;
      const uint4* a16 = reinterpret_cast<const uint4*>(a - s);
      uint32_t wv[16];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const uint4 v = __ldcs(a16 + c);
        wv[4 * c] = v.x; wv[4 * c + 1] = v.y; wv[4 * c + 2] = v.z; wv[4 * c + 3] = v.w;
      }
      uint4 v3 = make_uint4(0, 0, 0, 0);
      if (s) v3 = __ldcs(a16 + 3);   // bytes past the source chunk only when unaligned
      wv[12] = v3.x; wv[13] = v3.y; wv[14] = v3.z; wv[15] = v3.w;
      const uint32_t sel = 0x3210u + 0x1111u * (uint32_t)(s & 3);
      uint32_t o[12];
      switch (s >> 2) {
        case 0: funnel12<0>(wv, sel, o); break;
        case 1: funnel12<1>(wv, sel, o); break;
        case 2: funnel12<2>(wv, sel, o); break;
        default: funnel12<3>(wv, sel, o); break;
      }
      uint4* q16 = reinterpret_cast<uint4*>(q);
      __stcs(q16, make_uint4(o[0], o[1], o[2], o[3]));
      __stcs(q16 + 1, make_uint4(o[4], o[5], o[6], o[7]));
      __stcs(q16 + 2, make_uint4(o[8], o[9], o[10], o[11]));
    } else {
      for (int k = 0; k < 16 && x0 + k < w; ++k) {
        const int sx = sx0 + k;
        if (sy >= 0 && sy < h && sx >= 0 && sx < w) {
          const uint8_t* p = src + (int64_t)sy * in_pitch + 3 * (int64_t)sx;
          q[3 * k] = p[0]; q[3 * k + 1] = p[1]; q[3 * k + 2] = p[2];
        } else {
          q[3 * k] = f0; q[3 * k + 1] = f1; q[3 * k + 2] = f2;
        }
      }
    }
  }
}

__global__ void shift_gray_kernel(const uint8_t* __restrict__ in, int64_t in_pitch, int w, int h, int dx, int dy,
                                  uint8_t fill, uint8_t* __restrict__ out, int64_t out_pitch) {
  const int64_t n = (int64_t)w * h;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / w), x = (int)(i - (int64_t)y * w);
    const int sx = x - dx, sy = y - dy;
    out[y * out_pitch + x] = (sx >= 0 && sx < w && sy >= 0 && sy < h) ? in[(int64_t)sy * in_pitch + sx] : fill;
  }
}

}  // namespace mtb

using namespace mtb;

extern "C" int mtb_shift_rgb(const uint8_t* in, int64_t in_pitch, int64_t in_img_stride, int w, int h, int n_img,
                             const int32_t* offsets, int fill_r, int fill_g, int fill_b, uint8_t* out,
                             int64_t out_pitch, int64_t out_img_stride, void* stream) {
  clear_error();
  MTB_REQUIRE(in && out && offsets, "null pointer");
  MTB_REQUIRE(w >= 1 && h >= 1 && n_img >= 1, "image dimensions must be at least 1x1");
  MTB_REQUIRE(in_pitch >= 3 * (int64_t)w && out_pitch >= 3 * (int64_t)w, "pitch smaller than row");
  const uint32_t fill = (uint32_t)(fill_r & 0xff) | ((uint32_t)(fill_g & 0xff) << 8) | ((uint32_t)(fill_b & 0xff) << 16);
  const bool aligned = ((uintptr_t)out & 3) == 0 && (out_pitch & 3) == 0 && (out_img_stride & 3) == 0;
  if (((uintptr_t)out & 15) == 0 && (out_pitch & 15) == 0 && (out_img_stride & 15) == 0) {
    const int64_t n16 = (int64_t)((w + 15) / 16) * h;
    int64_t per = (int64_t)num_sms() * 8 / n_img;
    if (per < 1) per = 1;
    if (per > (n16 + 255) / 256) per = (n16 + 255) / 256;
    shift_rgb16_kernel<<<dim3((unsigned)per, n_img), 256, 0, as_stream(stream)>>>(
        in, in_pitch, in_img_stride, w, h, offsets, fill, out, out_pitch, out_img_stride);
    return check_launch("shift_rgb16_kernel");
  }
  const int64_t n = (int64_t)((w + 3) / 4) * h;
  int64_t per_img = (int64_t)num_sms() * 8 / n_img;
  if (per_img < 1) per_img = 1;
  if (per_img > (n + 255) / 256) per_img = (n + 255) / 256;
  shift_rgb_kernel<<<dim3((unsigned)per_img, n_img), 256, 0, as_stream(stream)>>>(
      in, in_pitch, in_img_stride, w, h, offsets, fill, out, out_pitch, out_img_stride, aligned);
  return check_launch("shift_rgb_kernel");
}

extern "C" int mtb_shift_gray(const uint8_t* in, int64_t in_pitch, int w, int h, int dx, int dy, int fill,
                              uint8_t* out, int64_t out_pitch, void* stream) {
  clear_error();
  MTB_REQUIRE(in && out, "null pointer");
  MTB_REQUIRE(w >= 1 && h >= 1, "image dimensions must be at least 1x1");
  shift_gray_kernel<<<grid_cap((int64_t)w * h, 256), 256, 0, as_stream(stream)>>>(in, in_pitch, w, h, dx, dy,
                                                                                  (uint8_t)fill, out, out_pitch);
  return check_launch("shift_gray_kernel");
}
