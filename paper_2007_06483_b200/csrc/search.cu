// K4: the shifted XOR/AND/popcount error test and the coarse-to-fine level
// search, on packed bitmaps.
//
// Reference semantics (bit-exact):
//   err(dx, dy) = sum over the row overlap 0 <= y-dy < h of
//                 popcount((A[y] ^ S(B[y-dy], dx)) & EA[y] & S(EB[y-dy], dx))
//   where S shifts a packed row toward higher x by dx bits with zero fill
//   (kernels/_native.pyx:50-111, fallback.py:24-81, conftest.py:14-24).
//   search_level: 9 candidates base + (ddx, ddy), (ddy, ddx) row-major over
//   {-1,0,1}^2, winner minimises (err, |ddx|+|ddy|, index)   search.py:20-23,53-71
//   find_offset: deepest level first, base = 2 * previous   search.py:74-95
#include <type_traits>

#include "common.cuh"

namespace mtb {

// 4-byte global -> shared copy, zero-filled when !ok (src is not read then).
__device__ __forceinline__ void cp_async4(uint32_t* dst, const uint32_t* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(ok ? 4 : 0)
               : "memory");
}

// CW-word (16 or 8 byte) global -> shared copy of `bytes` leading bytes, zero-filled.
template <int CW>
__device__ __forceinline__ void cp_async_n(uint32_t* dst, const uint32_t* src, int bytes) {
  if constexpr (CW == 4)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes)
                 : "memory");
}

// Word idx of a packed row (u32 view), zero outside [0, nw32).
__device__ __forceinline__ uint32_t row_word(const uint32_t* row, int64_t idx, int nw32) {
  return (idx >= 0 && idx < nw32) ? __ldg(row + idx) : 0u;
}

// ----------------------------------------------------- generic K-candidate --
// errs[k] += shifted_error(a, ea, b, eb, offsets[k]); one grid.y slice per k.
__global__ void __launch_bounds__(256)
shifted_error_multi_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ ea,
                           const uint32_t* __restrict__ b, const uint32_t* __restrict__ eb, int64_t h, int nw32,
                           const int32_t* __restrict__ offsets, int64_t dx0, int64_t dy0,
                           unsigned long long* __restrict__ errs) {
  // offsets == nullptr: a single candidate (dx0, dy0) passed by value.
  const int k = blockIdx.y;
  const int64_t dx = offsets ? (int64_t)offsets[2 * k] : dx0;
  const int64_t dy = offsets ? (int64_t)offsets[2 * k + 1] : dy0;
  const int64_t y0 = dy > 0 ? dy : 0;
  const int64_t y1 = h + (dy < 0 ? dy : 0);
  unsigned c = 0;
  if (y1 > y0) {
    const int64_t q = dx >> 5;  // floor division (arithmetic shift)
    const int r = (int)(dx & 31);
    const int64_t n = (y1 - y0) * nw32;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t yy = i / nw32;
      const int j = (int)(i - yy * nw32);
      const int64_t y = y0 + yy, sy = y - dy;
      const uint32_t* brow = b + sy * nw32;
      const uint32_t* erow = eb + sy * nw32;
      const uint32_t bs = shifted_word(row_word(brow, j - q - 1, nw32), row_word(brow, j - q, nw32), r);
      const uint32_t es = shifted_word(row_word(erow, j - q - 1, nw32), row_word(erow, j - q, nw32), r);
      c += __popc((__ldg(a + y * nw32 + j) ^ bs) & __ldg(ea + y * nw32 + j) & es);
    }
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&errs[k], (unsigned long long)c);
}

__global__ void shifted_error_bytemap_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ ea,
                                             const uint8_t* __restrict__ b, const uint8_t* __restrict__ eb,
                                             int64_t h, int64_t w, int64_t pitch, int64_t dx, int64_t dy,
                                             unsigned long long* out) {
  const int64_t x0 = dx > 0 ? dx : 0, x1 = w + (dx < 0 ? dx : 0);
  const int64_t y0 = dy > 0 ? dy : 0, y1 = h + (dy < 0 ? dy : 0);
  unsigned c = 0;
  if (x1 > x0 && y1 > y0) {
    const int64_t ow = x1 - x0, n = ow * (y1 - y0);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t y = y0 + i / ow, x = x0 + i % ow;
      const int64_t s = (y - dy) * pitch + (x - dx), d = y * pitch + x;
      c += ((a[d] ^ b[s]) & ea[d] & eb[s]) != 0;
    }
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

// The search.py:67 key, on (err, |ddx|+|ddy|, index).
__device__ __forceinline__ bool key_less(unsigned long long e, int d, int i, unsigned long long be, int bd, int bi) {
  if (e != be) return e < be;
  if (d != bd) return d < bd;
  return i < bi;
}

__global__ void select_candidate_kernel(const unsigned long long* errs, const int32_t* offsets, int k, int bdx,
                                        int bdy, int32_t* chosen) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int best = 0;
  unsigned long long be = errs[0];
  int bd = abs(offsets[0] - bdx) + abs(offsets[1] - bdy);
  for (int i = 1; i < k; ++i) {
    const unsigned long long e = errs[i];
    const int d = abs(offsets[2 * i] - bdx) + abs(offsets[2 * i + 1] - bdy);
    if (key_less(e, d, i, be, bd, best)) { best = i; be = e; bd = d; }
  }
  chosen[0] = offsets[2 * best];
  chosen[1] = offsets[2 * best + 1];
  chosen[2] = best;
}

// ----------------------------------------------------------- level search --
// One CTA = one tile of 64 output rows x 32 words (1024 pixels) of one pair's
// level.  The reference maps A/EA of the tile and the target maps B/EB of the
// tile plus its halo (rows -1..+1 around the base dy, words -2..+1 around the
// base dx) are staged in shared memory with coalesced loads issued all at
// once; then each warp slides down 8 output rows keeping the three source
// rows it needs, each pre-shifted by bx-1, bx, bx+1 (funnel shifts), in
// registers.  Per output word: 9 x (2 LOP3 + POPC).  CTA partials go to the
// pair's 9 u64 counters; the last CTA of the pair picks the winner with the
// search.py:67 key and publishes it for the next level.
constexpr int kSTRows = 64;          // output rows per tile
constexpr int kSTWords = 32;         // output words per tile
constexpr int kSTWarps = 8;          // 8 rows per warp
constexpr int kSTThreads = kSTWarps * 32;
constexpr int kSTBRows = kSTRows + 2;
// target rows staged: the tile's 32 words plus halo (2 left, 1 right) = 35,
// from an origin up to 3 words further left (16-B aligned copies): 40 words
constexpr int kSTBPitch = 40;

struct LevelSearchArgs {
  const uint64_t* const* maps;   // [P][4] {ref.mtb, ref.excl, tgt.mtb, tgt.excl}
  int w, h, nw32;                // h = rows of the whole level (image coordinates)
  // Row windows (row sharding): the reference maps hold image rows
  // [a_row0, a_row0 + a_rows), the target maps rows [b_row0, b_row0 + b_rows)
  // (own rows plus halo).  Unsharded: a_row0 = b_row0 = 0, a_rows = b_rows = h.
  int a_row0, a_rows, b_row0, b_rows;
  int decide;                    // 1: last CTA applies the search.py:67 key; 0: counts only
  const int32_t* prev;           // previous (coarser) level's chosen offset, or nullptr
  int64_t prev_stride;
  const int32_t* base;           // explicit base [P][2] when prev == nullptr (may be nullptr)
  int32_t* acc;
  int64_t acc_stride;
  unsigned long long* errs;
  int64_t errs_stride;
  uint32_t* done;
  int64_t done_stride;
  int tiles_x;                   // ceil(nw32 / 32)
  // Segmented target (row sharding, SEG kernels): the reference words come
  // from a_m / a_e (rows [a_row0, a_row0 + a_rows)), the target rows from up
  // to three buffers, segment s holding image rows [seg_row0[s], +seg_rows[s])
  // (previous shard's halo, own rows, next shard's halo): no concatenation.
  const uint32_t* a_m;
  const uint32_t* a_e;
  const uint32_t* seg_m[3];
  const uint32_t* seg_e[3];
  int seg_row0[3], seg_rows[3];
};

struct __align__(16) SearchSmem {
  uint32_t a[kSTRows][kSTWords];
  uint32_t ea[kSTRows][kSTWords];
  uint32_t b[kSTBRows][kSTBPitch];
  uint32_t eb[kSTBRows][kSTBPitch];
  unsigned part[kSTWarps][9];
  int last;
};

// One 64 x 32-word tile of pair p's level (base offset bx, by): returns, for
// threads 0..8, the tile's error count of candidate tid (0 for the others).
template <bool SEG>
__device__ __forceinline__ unsigned long long search_tile(const LevelSearchArgs& a, SearchSmem& S, int p, int tile,
                                                          int bx, int by) {
  const int tid = threadIdx.x, lane = tid & 31, wi = tid >> 5;
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int ly0 = ty * kSTRows, j0 = tx * kSTWords;   // local (reference-window) row of the tile
  const int y0 = a.a_row0 + ly0;                       // image row of the tile
  const uint32_t* A = SEG ? a.a_m : reinterpret_cast<const uint32_t*>(a.maps[4 * p + 0]);
  const uint32_t* EA = SEG ? a.a_e : reinterpret_cast<const uint32_t*>(a.maps[4 * p + 1]);
  const uint32_t* B = SEG ? nullptr : reinterpret_cast<const uint32_t*>(a.maps[4 * p + 2]);
  const uint32_t* EB = SEG ? nullptr : reinterpret_cast<const uint32_t*>(a.maps[4 * p + 3]);

  const int qb = bx >> 5;
  const int sy0 = y0 - by - 1;           // first staged source row
  const int64_t sj0 = (int64_t)j0 - qb - 2;  // first staged source word

  // ---- stage: global -> shared by cp.async (zero-filled outside the maps),
  // all copies in flight together, in chunks of CW words: 16 B when rows are
  // 16-byte multiples (nw32 % 4 == 0), else 8 B (rows are whole u64 words).
  // The target halo is staged from the CW-aligned word at or left of sj0
  // (staged column `mis` holds word sj0); partial edge chunks go word by word. ----
  int mis = 0;
  auto b_row = [&](int64_t y, const uint32_t*& pm, const uint32_t*& pe) {
    pm = nullptr;
    pe = nullptr;
    if (y >= 0 && y < a.h) {
      if (SEG) {
#pragma unroll
        for (int sg = 0; sg < 3; ++sg)
          if (a.seg_m[sg] && y >= a.seg_row0[sg] && y < (int64_t)a.seg_row0[sg] + a.seg_rows[sg]) {
            pm = a.seg_m[sg] + (y - a.seg_row0[sg]) * a.nw32;
            pe = a.seg_e[sg] + (y - a.seg_row0[sg]) * a.nw32;
          }
      } else if (y >= a.b_row0 && y < a.b_row0 + a.b_rows) {
        pm = B + (y - a.b_row0) * a.nw32;
        pe = EB + (y - a.b_row0) * a.nw32;
      }
    }
  };
  auto stage = [&](auto cw_tag) {
    constexpr int CW = decltype(cw_tag)::value;   // words per copy: 4 or 2
    constexpr int CA = kSTWords / CW;               // chunks per reference row
#pragma unroll
    for (int k = 0; k < kSTRows * CA / kSTThreads; ++k) {
      const int c = tid + kSTThreads * k, r = c / CA, q = c - r * CA;
      const int ly = ly0 + r, w = j0 + CW * q;
      const int nb = ly < a.a_rows ? max(0, min(4 * CW, 4 * (a.nw32 - w))) : 0;
      const int64_t o = nb ? (int64_t)ly * a.nw32 + w : 0;
      cp_async_n<CW>(&S.a[r][CW * q], A + o, nb);
      cp_async_n<CW>(&S.ea[r][CW * q], EA + o, nb);
    }
    const int64_t bw0 = sj0 & ~(int64_t)(CW - 1);
    mis = (int)(sj0 - bw0);
    constexpr int CB = kSTBPitch / CW;   // chunks per staged target row
    for (int c = tid; c < kSTBRows * CB; c += kSTThreads) {
      const int r = c / CB, q = c - r * CB;
      const uint32_t* pm;
      const uint32_t* pe;
      b_row((int64_t)sy0 + r, pm, pe);
      const int64_t w = bw0 + CW * q;
      if (pm && w >= 0 && w + CW <= a.nw32) {
        cp_async_n<CW>(&S.b[r][CW * q], pm + w, 4 * CW);
        cp_async_n<CW>(&S.eb[r][CW * q], pe + w, 4 * CW);
      } else if (!pm || w + CW <= 0 || w >= a.nw32) {
        cp_async_n<CW>(&S.b[r][CW * q], A, 0);
        cp_async_n<CW>(&S.eb[r][CW * q], A, 0);
      } else {
#pragma unroll
        for (int i = 0; i < CW; ++i) {
          const bool ok = w + i >= 0 && w + i < a.nw32;
          cp_async4(&S.b[r][CW * q + i], ok ? pm + w + i : A, ok);
          cp_async4(&S.eb[r][CW * q + i], ok ? pe + w + i : A, ok);
        }
      }
    }
  };
  if ((a.nw32 & 3) == 0)
    stage(std::integral_constant<int, 4>{});
  else
    stage(std::integral_constant<int, 2>{});
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();

  // ---- compute: warp wi -> output rows 8wi .. 8wi+7, lane -> word ----
  // Candidate dx = bx - 1, bx, bx + 1 reads staged words (lane + 1, lane + 2)
  // funnel-shifted by (dx & 31), except dx = bx - 1 when bx & 31 == 0 (words
  // lane + 2, lane + 3) and dx = bx + 1 when bx & 31 == 31 (lane, lane + 1):
  // three compile-time cases (CTA-uniform), no per-word selects.
  unsigned cnt[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) cnt[i] = 0;
  const int rbeg = wi * (kSTRows / kSTWarps);
  const int rbx = bx & 31;
  const int lm = lane + mis;   // staged column of source word j0 + lane - qb - 2
  auto rows = [&](auto case_tag) {
    constexpr int CASE = decltype(case_tag)::value;   // 0: rbx == 0, 1: rbx == 31, 2: other
    const int r0 = CASE == 0 ? 31 : (CASE == 1 ? 30 : rbx - 1);
    const int r1 = CASE == 0 ? 0 : (CASE == 1 ? 31 : rbx);
    const int r2 = CASE == 0 ? 1 : (CASE == 1 ? 0 : rbx + 1);
    auto shifted_row = [&](int lb, uint32_t (&sb)[3], uint32_t (&se)[3]) {
      const uint32_t w0 = S.b[lb][lm], w1 = S.b[lb][lm + 1], w2 = S.b[lb][lm + 2];
      const uint32_t v0 = S.eb[lb][lm], v1 = S.eb[lb][lm + 1], v2 = S.eb[lb][lm + 2];
      if (CASE == 0) {
        const uint32_t w3 = S.b[lb][lm + 3], v3 = S.eb[lb][lm + 3];
        sb[0] = shifted_word(w2, w3, r0); se[0] = shifted_word(v2, v3, r0);
      } else {
        sb[0] = shifted_word(w1, w2, r0); se[0] = shifted_word(v1, v2, r0);
      }
      sb[1] = shifted_word(w1, w2, r1); se[1] = shifted_word(v1, v2, r1);
      if (CASE == 1) {
        sb[2] = shifted_word(w0, w1, r2); se[2] = shifted_word(v0, v1, r2);
      } else {
        sb[2] = shifted_word(w1, w2, r2); se[2] = shifted_word(v1, v2, r2);
      }
    };
    // output local row rr needs source local rows rr (ddy=+1), rr+1 (ddy=0), rr+2 (ddy=-1)
    uint32_t b0[3], e0[3], b1[3], e1[3];
    shifted_row(rbeg, b0, e0);
    shifted_row(rbeg + 1, b1, e1);
#pragma unroll
    for (int k = 0; k < kSTRows / kSTWarps; ++k) {
      const int rr = rbeg + k;
      uint32_t b2[3], e2[3];
      shifted_row(rr + 2, b2, e2);
      const uint32_t av = S.a[rr][lane], ev = S.ea[rr][lane];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        cnt[0 + d] += __popc((av ^ b2[d]) & ev & e2[d]);  // ddy = -1
        cnt[3 + d] += __popc((av ^ b1[d]) & ev & e1[d]);  // ddy =  0
        cnt[6 + d] += __popc((av ^ b0[d]) & ev & e0[d]);  // ddy = +1
      }
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        b0[d] = b1[d]; e0[d] = e1[d];
        b1[d] = b2[d]; e1[d] = e2[d];
      }
    }
  };
  if (ly0 + rbeg < a.a_rows) {
    if (rbx == 0) rows(std::integral_constant<int, 0>{});
    else if (rbx == 31) rows(std::integral_constant<int, 1>{});
    else rows(std::integral_constant<int, 2>{});
  }
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const unsigned v = warp_sum(cnt[i]);
    if (lane == 0) S.part[wi][i] = v;
  }
  __syncthreads();
  unsigned long long v = 0;
  if (tid < 9) {
#pragma unroll
    for (int k = 0; k < kSTWarps; ++k) v += S.part[k][tid];
  }
  return v;
}

template <bool SEG>
__global__ void __launch_bounds__(kSTThreads)
level_search_kernel(LevelSearchArgs a) {
  __shared__ SearchSmem S;
  const int p = blockIdx.y;
  const int tid = threadIdx.x;
  int bx = 0, by = 0;
  if (a.prev) {
    bx = 2 * a.prev[p * a.prev_stride];
    by = 2 * a.prev[p * a.prev_stride + 1];
  } else if (a.base) {
    bx = a.base[2 * p];
    by = a.base[2 * p + 1];
  }
  const unsigned long long v = search_tile<SEG>(a, S, p, blockIdx.x, bx, by);
  unsigned long long* errs = a.errs + p * a.errs_stride;
  if (tid < 9 && v) atomicAdd(&errs[tid], v);
  if (!a.decide) return;
  __threadfence();
  __syncthreads();
  if (tid == 0) S.last = (atomicAdd(&a.done[p * a.done_stride], 1u) == gridDim.x - 1);
  __syncthreads();
  if (S.last && tid == 0) {
    __threadfence();
    int best = 0;
    unsigned long long be = 0;
    int bd = 0;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      const unsigned long long e = *((volatile unsigned long long*)&errs[i]);
      const int d = abs(i % 3 - 1) + abs(i / 3 - 1);
      if (i == 0 || key_less(e, d, i, be, bd, best)) { best = i; be = e; bd = d; }
    }
    a.acc[p * a.acc_stride] = bx + best % 3 - 1;
    a.acc[p * a.acc_stride + 1] = by + best / 3 - 1;
  }
}

// The coarse levels of find_offset for one pair per CTA (search.py:74-95):
// levels n-1 .. k_lo, each a loop over its few tiles, the decision kept on
// chip and fed to the next level as its base; replaces one launch (and one
// grid of a handful of CTAs per pair) per coarse level.
struct PairSearchArgs {
  const uint64_t* const* maps;   // table [level][P][4]
  int w[kMaxLevels], h[kMaxLevels], nw32[kMaxLevels];
  int n_levels, k_lo, P;
  const int32_t* base;           // [P][2] or nullptr
  int32_t* acc;                  // [P][n][2]
  unsigned long long* errs;      // [P][n][9]
};

__global__ void __launch_bounds__(kSTThreads, 3) pair_search_kernel(PairSearchArgs pa) {
  __shared__ SearchSmem S;
  __shared__ unsigned long long s_e[9];
  __shared__ int s_b[2];
  const int p = blockIdx.x, tid = threadIdx.x, n = pa.n_levels;
  int bx = pa.base ? pa.base[2 * p] : 0, by = pa.base ? pa.base[2 * p + 1] : 0;
  for (int k = n - 1; k >= pa.k_lo; --k) {
    LevelSearchArgs a{};
    a.maps = pa.maps + (int64_t)k * pa.P * 4;
    a.w = pa.w[k];
    a.h = pa.h[k];
    a.nw32 = pa.nw32[k];
    a.a_rows = a.b_rows = a.h;
    a.tiles_x = (a.nw32 + kSTWords - 1) / kSTWords;
    const int tiles = a.tiles_x * ((a.h + kSTRows - 1) / kSTRows);
    unsigned long long tot = 0;
    for (int t = 0; t < tiles; ++t) tot += search_tile<false>(a, S, p, t, bx, by);
    if (tid < 9) {
      s_e[tid] = tot;
      pa.errs[((int64_t)p * n + k) * 9 + tid] = tot;
    }
    __syncthreads();
    if (tid == 0) {
      int best = 0;
      unsigned long long be = 0;
      int bd = 0;
#pragma unroll
      for (int i = 0; i < 9; ++i) {
        const int d = abs(i % 3 - 1) + abs(i / 3 - 1);
        if (i == 0 || key_less(s_e[i], d, i, be, bd, best)) { best = i; be = s_e[i]; bd = d; }
      }
      s_b[0] = bx + best % 3 - 1;
      s_b[1] = by + best / 3 - 1;
      pa.acc[((int64_t)p * n + k) * 2] = s_b[0];
      pa.acc[((int64_t)p * n + k) * 2 + 1] = s_b[1];
    }
    __syncthreads();
    bx = 2 * s_b[0];
    by = 2 * s_b[1];
  }
}

// The search.py:67 decision for P pairs from already-summed error counts
// (row-sharded search: counts are all-reduced across ranks first).
__global__ void decide_level_kernel(const unsigned long long* __restrict__ errs, int64_t errs_stride,
                                    const int32_t* __restrict__ prev, int64_t prev_stride,
                                    const int32_t* __restrict__ base, int32_t* __restrict__ acc, int64_t acc_stride,
                                    int P) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int bx = 0, by = 0;
  if (prev) {
    bx = 2 * prev[p * prev_stride];
    by = 2 * prev[p * prev_stride + 1];
  } else if (base) {
    bx = base[2 * p];
    by = base[2 * p + 1];
  }
  const unsigned long long* e = errs + p * errs_stride;
  int best = 0;
  unsigned long long be = 0;
  int bd = 0;
  for (int i = 0; i < 9; ++i) {
    const int d = abs(i % 3 - 1) + abs(i / 3 - 1);
    if (i == 0 || key_less(e[i], d, i, be, bd, best)) { best = i; be = e[i]; bd = d; }
  }
  acc[p * acc_stride] = bx + best % 3 - 1;
  acc[p * acc_stride + 1] = by + best / 3 - 1;
}

}  // namespace mtb

using namespace mtb;

extern "C" int mtb_shifted_error_packed(const uint64_t* a, const uint64_t* ea, const uint64_t* b, const uint64_t* eb,
                                        int64_t h, int64_t nwords64, int64_t dx, int64_t dy, unsigned long long* out,
                                        void* stream) {
  clear_error();
  MTB_REQUIRE(out, "null output pointer");
  MTB_REQUIRE(h >= 0 && nwords64 >= 0, "negative dimensions");
  MTB_CUDA(cudaMemsetAsync(out, 0, sizeof(unsigned long long), as_stream(stream)));
  if (h == 0 || nwords64 == 0) return MTB_OK;
  MTB_REQUIRE(a && ea && b && eb, "null bitmap pointer");
  MTB_REQUIRE(nwords64 < (1 << 25), "row too wide");
  const int64_t n = 2 * nwords64 * h;
  shifted_error_multi_kernel<<<dim3(grid_cap(n, 256), 1), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const uint32_t*>(a), reinterpret_cast<const uint32_t*>(ea),
      reinterpret_cast<const uint32_t*>(b), reinterpret_cast<const uint32_t*>(eb), h, (int)(2 * nwords64), nullptr,
      dx, dy, out);
  return check_launch("shifted_error_multi_kernel");
}

extern "C" int mtb_shifted_error_multi(const uint64_t* a, const uint64_t* ea, const uint64_t* b, const uint64_t* eb,
                                       int64_t h, int64_t nwords64, const int32_t* offsets, int k,
                                       unsigned long long* errs, void* stream) {
  clear_error();
  MTB_REQUIRE(errs && offsets, "null pointer");
  MTB_REQUIRE(k >= 1 && k <= 65535, "candidate count out of range");
  MTB_REQUIRE(h >= 0 && nwords64 >= 0, "negative dimensions");
  MTB_CUDA(cudaMemsetAsync(errs, 0, sizeof(unsigned long long) * k, as_stream(stream)));
  if (h == 0 || nwords64 == 0) return MTB_OK;
  MTB_REQUIRE(a && ea && b && eb, "null bitmap pointer");
  const int64_t n = 2 * nwords64 * h;
  int g = grid_cap(n, 256);
  if (k > 1) {
    g = (int)((int64_t)num_sms() * 8 / k);
    if (g < 1) g = 1;
    const int64_t need = (n + 255) / 256;
    if (g > need) g = (int)need;
  }
  shifted_error_multi_kernel<<<dim3(g, k), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const uint32_t*>(a), reinterpret_cast<const uint32_t*>(ea),
      reinterpret_cast<const uint32_t*>(b), reinterpret_cast<const uint32_t*>(eb), h, (int)(2 * nwords64), offsets,
      0, 0, errs);
  return check_launch("shifted_error_multi_kernel");
}

extern "C" int mtb_shifted_error_bytemap(const uint8_t* a, const uint8_t* ea, const uint8_t* b, const uint8_t* eb,
                                         int64_t h, int64_t w, int64_t pitch, int64_t dx, int64_t dy,
                                         unsigned long long* out, void* stream) {
  clear_error();
  MTB_REQUIRE(out, "null output pointer");
  MTB_REQUIRE(h >= 0 && w >= 0 && pitch >= w, "bad dimensions");
  MTB_CUDA(cudaMemsetAsync(out, 0, sizeof(unsigned long long), as_stream(stream)));
  if (h * w == 0) return MTB_OK;
  MTB_REQUIRE(a && ea && b && eb, "null bitmap pointer");
  shifted_error_bytemap_kernel<<<grid_cap(h * w, 256), 256, 0, as_stream(stream)>>>(a, ea, b, eb, h, w, pitch, dx, dy,
                                                                                   out);
  return check_launch("shifted_error_bytemap_kernel");
}

extern "C" int mtb_select_candidate(const unsigned long long* errs, const int32_t* offsets, int k, int base_dx,
                                    int base_dy, int32_t* chosen, void* stream) {
  clear_error();
  MTB_REQUIRE(errs && offsets && chosen, "null pointer");
  MTB_REQUIRE(k >= 1, "need at least one candidate");
  select_candidate_kernel<<<1, 32, 0, as_stream(stream)>>>(errs, offsets, k, base_dx, base_dy, chosen);
  return check_launch("select_candidate_kernel");
}

extern "C" int mtb_find_offset_batch(const uint64_t* const* maps, const int32_t* dims, int n_levels, int P,
                                     const int32_t* base, int32_t* acc, unsigned long long* errs, uint32_t* done,
                                     void* stream) {
  clear_error();
  MTB_REQUIRE(maps && dims && acc && errs && done, "null pointer");
  MTB_REQUIRE(n_levels >= 1 && n_levels <= MTB_MAX_LEVELS, "level count out of range");
  MTB_REQUIRE(P >= 1 && P <= 65535, "pair count out of range");
  for (int k = 0; k < n_levels; ++k) {
    MTB_REQUIRE(dims[3 * k] >= 1 && dims[3 * k + 1] >= 1, "level dimensions must be positive");
    MTB_REQUIRE((int64_t)dims[3 * k + 2] * 64 >= dims[3 * k], "row word count too small for width");
  }
  cudaStream_t st = as_stream(stream);
  MTB_CUDA(cudaMemsetAsync(errs, 0, sizeof(unsigned long long) * 9 * n_levels * P, st));
  MTB_CUDA(cudaMemsetAsync(done, 0, sizeof(uint32_t) * n_levels * P, st));
  int launches = 0;
  // Coarse levels with few tiles: one CTA per pair runs them back to back
  // (pair_search_kernel); with few pairs only the single-tile levels, so the
  // serial per-pair loop never replaces a wide grid.
  const int max_tiles = P >= 64 ? 8 : 2;
  int k_lo = n_levels;
  while (k_lo > 0) {
    const int k = k_lo - 1;
    const int nw32 = 2 * dims[3 * k + 2];
    const int tiles = ((nw32 + kSTWords - 1) / kSTWords) * ((dims[3 * k + 1] + kSTRows - 1) / kSTRows);
    if (tiles > max_tiles) break;
    k_lo = k;
  }
  if (k_lo < n_levels) {
    PairSearchArgs pa{};
    pa.maps = maps;
    for (int k = 0; k < n_levels; ++k) {
      pa.w[k] = dims[3 * k];
      pa.h[k] = dims[3 * k + 1];
      pa.nw32[k] = 2 * dims[3 * k + 2];
    }
    pa.n_levels = n_levels;
    pa.k_lo = k_lo;
    pa.P = P;
    pa.base = base;
    pa.acc = acc;
    pa.errs = errs;
    pair_search_kernel<<<P, kSTThreads, 0, st>>>(pa);
    ++launches;
  }
  for (int k = k_lo - 1; k >= 0; --k) {
    LevelSearchArgs a{};
    a.maps = maps + (int64_t)k * P * 4;
    a.w = dims[3 * k];
    a.h = dims[3 * k + 1];
    a.nw32 = 2 * dims[3 * k + 2];
    a.prev = (k == n_levels - 1) ? nullptr : acc + 2 * (k + 1);
    a.prev_stride = 2 * n_levels;
    a.base = base;
    a.acc = acc + 2 * k;
    a.acc_stride = 2 * n_levels;
    a.errs = errs + 9 * k;
    a.errs_stride = 9 * n_levels;
    a.done = done + k;
    a.done_stride = n_levels;
    a.a_row0 = 0;
    a.a_rows = a.h;
    a.b_row0 = 0;
    a.b_rows = a.h;
    a.decide = 1;
    a.tiles_x = (a.nw32 + kSTWords - 1) / kSTWords;
    const int tiles_y = (a.h + kSTRows - 1) / kSTRows;
    level_search_kernel<false><<<dim3(a.tiles_x * tiles_y, P), kSTThreads, 0, st>>>(a);
    ++launches;
  }
  return check_launch("level_search_kernel", launches);
}

extern "C" int mtb_search_level_rows(const uint64_t* const* maps, int w, int h, int64_t nwords64, int a_row0,
                                     int a_rows, int b_row0, int b_rows, int P, const int32_t* prev,
                                     int64_t prev_stride, const int32_t* base, unsigned long long* errs,
                                     int64_t errs_stride, void* stream) {
  clear_error();
  MTB_REQUIRE(maps && errs, "null pointer");
  MTB_REQUIRE(P >= 1 && P <= 65535, "pair count out of range");
  MTB_REQUIRE(w >= 1 && h >= 1 && nwords64 * 64 >= w, "bad level dimensions");
  MTB_REQUIRE(a_rows >= 0 && b_rows >= 0 && a_row0 >= 0 && a_row0 + a_rows <= h, "bad row windows");
  cudaStream_t st = as_stream(stream);
  for (int p = 0; p < P; ++p)
    MTB_CUDA(cudaMemsetAsync(errs + p * errs_stride, 0, 9 * sizeof(unsigned long long), st));
  if (a_rows == 0) return MTB_OK;
  LevelSearchArgs a{};
  a.maps = maps;
  a.w = w;
  a.h = h;
  a.nw32 = (int)(2 * nwords64);
  a.prev = prev;
  a.prev_stride = prev_stride;
  a.base = base;
  a.errs = errs;
  a.errs_stride = errs_stride;
  a.a_row0 = a_row0;
  a.a_rows = a_rows;
  a.b_row0 = b_row0;
  a.b_rows = b_rows;
  a.decide = 0;
  a.tiles_x = (a.nw32 + kSTWords - 1) / kSTWords;
  const int tiles_y = (a_rows + kSTRows - 1) / kSTRows;
  level_search_kernel<false><<<dim3(a.tiles_x * tiles_y, P), kSTThreads, 0, st>>>(a);
  return check_launch("level_search_kernel");
}

extern "C" int mtb_search_level_rows3(const uint64_t* a_mtb, const uint64_t* a_excl, int a_row0, int a_rows,
                                      const uint64_t* const* seg, const int* seg_row0, const int* seg_rows, int w,
                                      int h, int64_t nwords64, const int32_t* prev, const int32_t* base,
                                      unsigned long long* errs, void* stream) {
  clear_error();
  MTB_REQUIRE(a_mtb && a_excl && seg && seg_row0 && seg_rows && errs, "null pointer");
  MTB_REQUIRE(w >= 1 && h >= 1 && nwords64 * 64 >= w, "bad level dimensions");
  MTB_REQUIRE(a_rows >= 0 && a_row0 >= 0 && a_row0 + a_rows <= h, "bad row windows");
  cudaStream_t st = as_stream(stream);
  MTB_CUDA(cudaMemsetAsync(errs, 0, 9 * sizeof(unsigned long long), st));
  if (a_rows == 0) return MTB_OK;
  LevelSearchArgs a{};
  a.w = w;
  a.h = h;
  a.nw32 = (int)(2 * nwords64);
  a.prev = prev;
  a.base = base;
  a.errs = errs;
  a.a_row0 = a_row0;
  a.a_rows = a_rows;
  a.a_m = reinterpret_cast<const uint32_t*>(a_mtb);
  a.a_e = reinterpret_cast<const uint32_t*>(a_excl);
  for (int s = 0; s < 3; ++s) {
    const bool on = seg[2 * s] && seg[2 * s + 1] && seg_rows[s] > 0;
    MTB_REQUIRE(!on || seg_row0[s] >= -(1 << 30), "bad segment");
    a.seg_m[s] = on ? reinterpret_cast<const uint32_t*>(seg[2 * s]) : nullptr;
    a.seg_e[s] = on ? reinterpret_cast<const uint32_t*>(seg[2 * s + 1]) : nullptr;
    a.seg_row0[s] = on ? seg_row0[s] : 0;
    a.seg_rows[s] = on ? seg_rows[s] : 0;
  }
  a.decide = 0;
  a.tiles_x = (a.nw32 + kSTWords - 1) / kSTWords;
  const int tiles_y = (a_rows + kSTRows - 1) / kSTRows;
  level_search_kernel<true><<<dim3(a.tiles_x * tiles_y, 1), kSTThreads, 0, st>>>(a);
  return check_launch("level_search_kernel");
}

extern "C" int mtb_decide_level(const unsigned long long* errs, int64_t errs_stride, const int32_t* prev,
                                int64_t prev_stride, const int32_t* base, int32_t* acc, int64_t acc_stride, int P,
                                void* stream) {
  clear_error();
  MTB_REQUIRE(errs && acc, "null pointer");
  MTB_REQUIRE(P >= 1, "pair count out of range");
  decide_level_kernel<<<(P + 127) / 128, 128, 0, as_stream(stream)>>>(errs, errs_stride, prev, prev_stride, base, acc,
                                                                    acc_stride, P);
  return check_launch("decide_level_kernel");
}
