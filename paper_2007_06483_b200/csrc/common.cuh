// Shared helpers for the sm_100a MTB engine: error state, launch accounting,
// pyramid planning, bit tricks.  See include/mtbalign_b200.h for the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/mtbalign_b200.h"

namespace mtb {

// ---------------------------------------------------------------- errors --
void set_error(const std::string& msg);
void clear_error();
extern std::atomic<uint64_t> g_launches;

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Call after every launch: counts it and converts a launch failure into MTB_ECUDA.
int check_launch(const char* what, int n_launches = 1);

#define MTB_REQUIRE(cond, msg)              \
  do {                                      \
    if (!(cond)) {                          \
      ::mtb::set_error(std::string(msg));   \
      return MTB_EINVAL;                    \
    }                                       \
  } while (0)

#define MTB_CUDA(call)                                                          \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess) {                                                    \
      ::mtb::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));     \
      return MTB_ECUDA;                                                         \
    }                                                                           \
  } while (0)

// SM count of the current device (cached; 148 on B200).
int num_sms();

// Grid size for a grid-stride loop over n items: enough CTAs to cover n,
// capped at `waves` CTAs per SM.
inline int grid_cap(int64_t n, int threads, int waves = 8) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * waves;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

// --------------------------------------------------------------- planning --
// pyramid.py:14 MIN_LEVEL_SIZE, pyramid.py:35-42 max_levels.
constexpr int kMinLevelSize = 16;
constexpr int kMaxLevels = MTB_MAX_LEVELS;

struct LevelGeom {
  int w, h;
  int64_t gray_pitch;   // bytes, multiple of 128 (one L2 line; a u32 bitmap word = 32 aligned bytes)
  int64_t gray_off;     // bytes from the image's gray arena base, 256-aligned
  int64_t nw64;         // ceil(w/64) u64 words per packed row (bitmap.py:35)
  int64_t bit_off;      // u64 words from the image's bitmap arena base, 32-word aligned
};

struct Plan {
  int n;
  LevelGeom lv[kMaxLevels];
  int64_t gray_img_bytes;   // per-image gray arena, 256-aligned
  int64_t bit_img_words;    // per-image bitmap arena (one map), multiple of 32 words
};

inline int max_levels(int w, int h) {
  int n = 0;
  while (w >= kMinLevelSize && h >= kMinLevelSize) {
    ++n;
    w /= 2;
    h /= 2;
  }
  return n;
}

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// Returns false on invalid input (pyramid.py:52-56 ValueErrors).
bool make_plan(int w, int h, int requested, Plan* p);

// ------------------------------------------------------------ device bits --
__device__ __forceinline__ unsigned warp_sum(unsigned v) { return __reduce_add_sync(0xffffffffu, v); }

// Word j (32-bit) of a packed row after translating content by `dx` pixels
// toward higher x, given the two source words W[j-q-1] (lo) and W[j-q] (hi)
// where q = dx >> 5 (floor) and r = dx & 31.  Mirrors _word_shifted_pos/_neg
// (kernels/_native.pyx:50-70) for both signs at once.
__device__ __forceinline__ uint32_t shifted_word(uint32_t lo, uint32_t hi, int r) {
  return __funnelshift_l(lo, hi, r);
}

}  // namespace mtb
