// C-ABI plumbing: error state, launch accounting, pyramid planning and the
// fused preprocess entry point (pipeline.py:80-85 on the device).
#include <cstring>

#include "common.cuh"

namespace mtb {

static thread_local std::string t_last_error;
std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { t_last_error = msg; }
void clear_error() { t_last_error.clear(); }

int check_launch(const char* what, int n_launches) {
  g_launches.fetch_add((uint64_t)n_launches, std::memory_order_relaxed);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return MTB_ECUDA;
  }
  return MTB_OK;
}

// SM count of the CURRENT device, cached per device ordinal.
static std::atomic<int> g_sms[64];
int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int v = g_sms[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
      cudaGetLastError();
      v = 148;
    }
    g_sms[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

bool make_plan(int w, int h, int requested, Plan* p) {
  int n;
  if (requested < 0) {
    // Exact level count for a row shard of a larger image (the level count
    // was decided on the full image): every level must keep >= 1 row/column.
    n = -requested;
    if (n > kMaxLevels || (w >> (n - 1)) < 1 || (h >> (n - 1)) < 1) return false;
  } else {
    if (requested < 1 || w < kMinLevelSize || h < kMinLevelSize) return false;
    const int ml = max_levels(w, h);
    n = requested < ml ? requested : ml;
    if (n > kMaxLevels) return false;
  }
  std::memset(p, 0, sizeof(*p));
  p->n = n;
  int64_t goff = 0, boff = 0;
  for (int k = 0; k < n; ++k) {
    LevelGeom& L = p->lv[k];
    L.w = w >> k;
    L.h = h >> k;
    L.gray_pitch = round_up(L.w, 128);
    L.gray_off = goff;
    goff = round_up(goff + L.gray_pitch * L.h, 256);
    L.nw64 = (L.w + 63) / 64;
    L.bit_off = boff;
    boff = round_up(boff + L.nw64 * L.h, 32);
  }
  p->gray_img_bytes = goff;
  p->bit_img_words = boff;
  return true;
}

// Defined in pyramid.cu / threshold.cu.
int64_t spread_hist_elems(int n_levels);
int hist_bin_for(const Plan& p, int n_img);
int hist_prepare(uint32_t* hist_ws, const Plan& p, int n_img, int hist_bin, cudaStream_t st);
int launch_pyramid(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride, int n_img, const Plan& p,
                   uint8_t* gray, uint32_t* spread_hist, int hist_bin, cudaStream_t st);
int launch_hist_median(const uint32_t* spread_hist, int n_img, int n_levels, int hist_bin, uint32_t* dense,
                       int32_t* medians, cudaStream_t st);
int launch_threshold_levels(const uint8_t* gray, const Plan& p, int n_img, const int32_t* medians, int tol,
                            uint64_t* mtb, uint64_t* excl, int discard, cudaStream_t st);

}  // namespace mtb

using namespace mtb;

extern "C" const char* mtb_last_error(void) { return t_last_error.c_str(); }
extern "C" int mtb_abi_version(void) { return 1; }
extern "C" uint64_t mtb_launch_count(void) { return g_launches.load(); }

extern "C" int mtb_plan_levels(int w, int h, int requested, int64_t* geom, int64_t* sizes) {
  Plan p;
  if (!make_plan(w, h, requested, &p)) return -1;
  if (geom) {
    for (int k = 0; k < kMaxLevels; ++k) {
      int64_t* g = geom + 6 * k;
      if (k < p.n) {
        g[0] = p.lv[k].w;
        g[1] = p.lv[k].h;
        g[2] = p.lv[k].gray_pitch;
        g[3] = p.lv[k].gray_off;
        g[4] = p.lv[k].nw64;
        g[5] = p.lv[k].bit_off;
      } else {
        for (int i = 0; i < 6; ++i) g[i] = 0;
      }
    }
  }
  if (sizes) {
    sizes[0] = p.gray_img_bytes;
    sizes[1] = p.bit_img_words;
    sizes[2] = spread_hist_elems(p.n);
  }
  return p.n;
}

extern "C" int mtb_pyramid_hist(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride, int w, int h,
                                int n_img, int levels, uint8_t* gray, uint32_t* hist_ws, void* stream) {
  clear_error();
  MTB_REQUIRE(rgb && gray && hist_ws, "null pointer");
  MTB_REQUIRE(n_img >= 1 && n_img <= 65535, "image count out of range");
  MTB_REQUIRE(rgb_pitch >= 3 * (int64_t)w, "rgb pitch smaller than row");
  MTB_REQUIRE((int64_t)w * h < (int64_t)4294967295LL, "image too large for 32-bit histograms");
  Plan p;
  MTB_REQUIRE(make_plan(w, h, levels, &p), "image must be at least 16x16 and levels >= 1");
  cudaStream_t st = as_stream(stream);
  const int bin = hist_bin_for(p, n_img);
  int rc = hist_prepare(hist_ws, p, n_img, bin, st);
  if (rc) return rc;
  return launch_pyramid(rgb, rgb_pitch, rgb_img_stride, n_img, p, gray, hist_ws, bin, st);
}

extern "C" int mtb_threshold_levels(const uint8_t* gray, const uint32_t* hist_ws, int w, int h, int n_img,
                                    int levels, int tol, uint32_t* hist_out, int32_t* medians, uint64_t* mtb,
                                    uint64_t* exclusion, int discard_gray, void* stream) {
  clear_error();
  MTB_REQUIRE(gray && hist_ws && medians && mtb && exclusion, "null pointer");
  MTB_REQUIRE(n_img >= 1 && n_img <= 65535, "image count out of range");
  MTB_REQUIRE(tol >= 0 && tol <= 255, "noise tolerance must be in 0..255");
  Plan p;
  MTB_REQUIRE(make_plan(w, h, levels, &p), "image must be at least 16x16 and levels >= 1");
  cudaStream_t st = as_stream(stream);
  int rc = launch_hist_median(hist_ws, n_img, p.n, 0, hist_out, medians, st);   // layout from the marker
  if (rc) return rc;
  return launch_threshold_levels(gray, p, n_img, medians, tol, mtb, exclusion, discard_gray, st);
}

extern "C" int mtb_preprocess(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride, int w, int h,
                              int n_img, int levels, int tol, uint8_t* gray, uint32_t* hist_ws, uint32_t* hist_out,
                              int32_t* medians, uint64_t* mtb, uint64_t* exclusion, void* stream) {
  clear_error();
  MTB_REQUIRE(tol >= 0 && tol <= 255, "noise tolerance must be in 0..255");
  MTB_REQUIRE(rgb && gray && hist_ws && medians && mtb && exclusion, "null pointer");
  MTB_REQUIRE(n_img >= 1 && n_img <= 65535, "image count out of range");
  MTB_REQUIRE(rgb_pitch >= 3 * (int64_t)w, "rgb pitch smaller than row");
  MTB_REQUIRE((int64_t)w * h < (int64_t)4294967295LL, "image too large for 32-bit histograms");
  Plan p;
  MTB_REQUIRE(make_plan(w, h, levels, &p), "image must be at least 16x16 and levels >= 1");
  cudaStream_t st = as_stream(stream);
  const int bin = hist_bin_for(p, n_img);
  int rc = hist_prepare(hist_ws, p, n_img, bin, st);
  if (rc) return rc;
  rc = launch_pyramid(rgb, rgb_pitch, rgb_img_stride, n_img, p, gray, hist_ws, bin, st);
  if (rc) return rc;
  rc = launch_hist_median(hist_ws, n_img, p.n, bin, hist_out, medians, st);
  if (rc) return rc;
  return launch_threshold_levels(gray, p, n_img, medians, tol, mtb, exclusion, 0, st);
}

extern "C" int mtb_threshold_levels_medians(const uint8_t* gray, int w, int h, int n_img, int levels, int tol,
                                            const int32_t* medians, uint64_t* mtb, uint64_t* exclusion,
                                            int discard_gray, void* stream) {
  clear_error();
  MTB_REQUIRE(gray && medians && mtb && exclusion, "null pointer");
  MTB_REQUIRE(n_img >= 1 && n_img <= 65535, "image count out of range");
  MTB_REQUIRE(tol >= 0 && tol <= 255, "noise tolerance must be in 0..255");
  Plan p;
  MTB_REQUIRE(make_plan(w, h, levels, &p), "invalid level plan");
  return launch_threshold_levels(gray, p, n_img, medians, tol, mtb, exclusion, discard_gray, as_stream(stream));
}
