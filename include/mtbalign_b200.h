/*
 * mtbalign_b200.h — C ABI of the B200 (sm_100a) MTB alignment engine.
 *
 * This is the drop-in boundary for the reference package `mtbalign` 0.1.0
 * (/root/reference/pkg).  The reference's operator boundary is its kernel
 * engine module (pkg/src/mtbalign/kernels/__init__.py:16-61), whose compiled
 * engine exports four functions (kernels/_native.pyx:32,41,73,114).  Those four
 * are re-declared first, with the same argument meaning, as device-pointer
 * entry points.  Below them are the level-granular and fused entry points that
 * the host mirror (paper_2007_06483_b200/*.py) uses so the coarse-to-fine
 * search never round-trips to the host.
 *
 * Conventions (all functions):
 *   - every pointer argument is a DEVICE pointer unless marked [host];
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *   - launches are asynchronous; results are valid once `stream` completes;
 *   - return value: MTB_OK (0) on success, MTB_EINVAL for argument errors,
 *     MTB_ECUDA for CUDA launch/runtime errors; mtb_last_error() returns a
 *     thread-local, NUL-terminated description of the last failure;
 *   - no C++ exception crosses this boundary;
 *   - packed bitmaps use the reference layout exactly (bitmap.py:32-40):
 *     per row ceil(W/64) little-endian u64 words, pixel x at bit x&63 of word
 *     x>>6, padding bits zero.  Kernels address them as u32 words (pixel x at
 *     bit x&31 of word x>>5, 2*ceil(W/64) words per row), which is the same
 *     memory on a little-endian device.
 *   - all arithmetic is integer and bit-exact against the CPU reference.
 */
#ifndef MTBALIGN_B200_H
#define MTBALIGN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MTB_OK 0
#define MTB_EINVAL 1
#define MTB_ECUDA 2

/* Largest pyramid depth the planner accepts (the CLI caps at 10, cli.py:36). */
#define MTB_MAX_LEVELS 16

/* ------------------------------------------------------------------------ */
/* Library / error state                                                     */
/* ------------------------------------------------------------------------ */

/* Last error message of the calling thread ("" if none). */
const char* mtb_last_error(void);
/* ABI version, bumped on any signature change (currently 1). */
int mtb_abi_version(void);
/* Number of kernels this library launched in-process (all entry points). */
uint64_t mtb_launch_count(void);

/* ------------------------------------------------------------------------ */
/* 1. Engine contract — replaces kernels/_native.pyx (and fallback.py twins) */
/* ------------------------------------------------------------------------ */

/* Replaces count_ones_packed (kernels/_native.pyx:41-47; fallback.py:19-21).
 * words: h rows x nwords64 u64 words.  *out = total popcount. */
int mtb_count_ones_packed(const uint64_t* words, int64_t h, int64_t nwords64,
                          unsigned long long* out, void* stream);

/* Replaces count_ones_bytemap (kernels/_native.pyx:32-38; fallback.py:15-16).
 * cells: h x w u8, row pitch `pitch` bytes.  *out = number of nonzero cells. */
int mtb_count_ones_bytemap(const uint8_t* cells, int64_t h, int64_t w, int64_t pitch,
                           unsigned long long* out, void* stream);

/* Replaces shifted_error_packed (kernels/_native.pyx:73-111; fallback.py:67-81).
 * *out = sum over the row overlap of popcount((a ^ shift(b,dx)) & ea & shift(eb,dx))
 * with rows of b/eb read at y-dy; out-of-range source bits are zero. */
int mtb_shifted_error_packed(const uint64_t* a, const uint64_t* ea,
                             const uint64_t* b, const uint64_t* eb,
                             int64_t h, int64_t nwords64, int64_t dx, int64_t dy,
                             unsigned long long* out, void* stream);

/* Replaces shifted_error_bytemap (kernels/_native.pyx:114-132; fallback.py:53-64).
 * Cells are 0 or 255 (any nonzero counts as set). */
int mtb_shifted_error_bytemap(const uint8_t* a, const uint8_t* ea,
                              const uint8_t* b, const uint8_t* eb,
                              int64_t h, int64_t w, int64_t pitch, int64_t dx, int64_t dy,
                              unsigned long long* out, void* stream);

/* ------------------------------------------------------------------------ */
/* 2. Primitive operators (one reference function each)                      */
/* ------------------------------------------------------------------------ */

/* to_grayscale (image.py:58-68): gray = (54R + 183G + 19B) >> 8.
 * rgb: n_img images of h rows, row pitch rgb_pitch bytes, image stride
 * rgb_img_stride bytes; gray likewise with gray_pitch / gray_img_stride. */
int mtb_to_grayscale(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride,
                     int w, int h, int n_img,
                     uint8_t* gray, int64_t gray_pitch, int64_t gray_img_stride,
                     void* stream);

/* downsample_half (pyramid.py:17-32): out = (2x2 block sum + 2) >> 2,
 * out dims (w/2, h/2) floor; requires w >= 2 and h >= 2. */
int mtb_downsample_half(const uint8_t* src, int64_t src_pitch, int w, int h,
                        uint8_t* dst, int64_t dst_pitch, void* stream);

/* histogram (threshold.py:25-28): hist[256] (u64) = bin counts of the image.
 * Overwrites hist. */
int mtb_histogram(const uint8_t* gray, int64_t pitch, int w, int h,
                  unsigned long long* hist, void* stream);

/* median_from_histogram (threshold.py:31-39), batched: for each of n_hist
 * 256-bin u64 histograms write the lower median (smallest m with
 * cumsum[m] >= (total+1)/2), or -1 when the histogram is empty. */
int mtb_median_from_histogram(const unsigned long long* hist, int n_hist,
                              int32_t* medians, void* stream);

/* make_mtb / make_exclusion (threshold.py:42-56) fused with the packer
 * (_pack_rows, bitmap.py:32-40): mtb bit = g > median, exclusion bit =
 * |g - median| > tol.  Either output may be NULL.  Outputs are h x nwords64
 * u64 words with nwords64 = ceil(w/64). */
int mtb_threshold_pack(const uint8_t* gray, int64_t pitch, int w, int h,
                       int median, int tol,
                       uint64_t* mtb, uint64_t* exclusion, void* stream);

/* Bitmap.from_bool packed branch (bitmap.py:59-72 -> _pack_rows :32-40):
 * bit = (mask byte != 0). */
int mtb_pack_mask(const uint8_t* mask, int64_t pitch, int w, int h,
                  uint64_t* words, void* stream);

/* _unpack_rows (bitmap.py:43-45) and the bytemap branch of from_bool
 * (bitmap.py:67-68): cells[y][x] = bit ? on_value : 0. */
int mtb_unpack_bits(const uint64_t* words, int64_t nwords64, int w, int h,
                    uint8_t* cells, int64_t cell_pitch, int on_value, void* stream);

/* shift_rgb (image.py:82-93), batched: out_i(x,y) = in_i(x-dx_i, y-dy_i) when in
 * bounds else fill.  offsets: n_img x {dx, dy} int32 (device). */
int mtb_shift_rgb(const uint8_t* in, int64_t in_pitch, int64_t in_img_stride,
                  int w, int h, int n_img, const int32_t* offsets,
                  int fill_r, int fill_g, int fill_b,
                  uint8_t* out, int64_t out_pitch, int64_t out_img_stride, void* stream);

/* shift_gray (image.py:96-106): single image, host offset. */
int mtb_shift_gray(const uint8_t* in, int64_t in_pitch, int w, int h,
                   int dx, int dy, int fill,
                   uint8_t* out, int64_t out_pitch, void* stream);

/* apply a 256-entry u8 lookup table (synth.py:25-33 apply_tone), n bytes. */
int mtb_apply_lut(const uint8_t* in, const uint8_t* lut, int64_t n, uint8_t* out, void* stream);

/* Evaluate K candidate offsets (offsets: K x {dx, dy} int32, device) of the
 * packed error test; errs[k] = shifted_error(a, ea, b, eb, offsets[k]).
 * This is the inner loop of search_level (search.py:63-70) and of
 * brute_force_offset (search.py:110-118). */
int mtb_shifted_error_multi(const uint64_t* a, const uint64_t* ea,
                            const uint64_t* b, const uint64_t* eb,
                            int64_t h, int64_t nwords64,
                            const int32_t* offsets, int k,
                            unsigned long long* errs, void* stream);

/* The tie-break of search.py:67-70 / :114-117 on the device: choose the
 * candidate minimising (err, |dx-base_dx| + |dy-base_dy|, index); writes
 * chosen[0..1] = offset and chosen[2] = index. */
int mtb_select_candidate(const unsigned long long* errs, const int32_t* offsets, int k,
                         int base_dx, int base_dy, int32_t* chosen, void* stream);

/* ------------------------------------------------------------------------ */
/* 3. Fused, level-granular hot path                                         */
/* ------------------------------------------------------------------------ */

/* Pyramid plan (pyramid.py:35-62): level count n = min(requested, max_levels)
 * and the device arena geometry used by mtb_preprocess.  geom [host] receives
 * MTB_MAX_LEVELS x 6 int64: {w, h, gray_pitch, gray_offset, nwords64,
 * bitmap_offset_words}; sizes [host] receives {gray_image_bytes,
 * bitmap_image_words, hist_workspace_u32_per_image}.  Returns n (>= 1), or -1
 * on invalid input (image smaller than 16x16, requested < 1).
 * requested < 0 plans EXACTLY -requested levels without the 16x16 clamp: a
 * row shard of a larger image whose level count was fixed on the full image
 * (every level must keep >= 1 row).  The fused entry points below accept the
 * same negative `levels`. */
int mtb_plan_levels(int w, int h, int requested, int64_t* geom, int64_t* sizes);

/* to_grayscale -> build_pyramid -> build_mtb_pyramid for a batch of images
 * (pipeline.py:80-85; image.py:58-68, pyramid.py:45-62, threshold.py:25-88),
 * fused: one RGB pass builds gray level 0, levels 1..n-1 and the per-level
 * 256-bin histograms; medians are taken on device; one pass thresholds and
 * bit-packs every level.
 *   rgb        n_img x h x (row pitch rgb_pitch) interleaved RGB8
 *   gray       workspace, n_img x gray_image_bytes (from mtb_plan_levels)
 *   hist_ws    workspace, n_img x hist_workspace_u32_per_image u32 (zeroed here)
 *   hist_out   optional out (may be NULL), n_img x n x 256 u32 histograms
 *   medians    out, n_img x n int32
 *   mtb, exclusion  out, n_img x bitmap_image_words u64 (arena of mtb_plan_levels)
 */
int mtb_preprocess(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride,
                   int w, int h, int n_img, int levels, int tol,
                   uint8_t* gray, uint32_t* hist_ws, uint32_t* hist_out, int32_t* medians,
                   uint64_t* mtb, uint64_t* exclusion, void* stream);

/* The two halves of mtb_preprocess, for per-stage timing (pipeline.py:77-85):
 * mtb_pyramid_hist = gray + pyramid + spread histograms (zeroes hist_ws);
 * mtb_threshold_levels = medians + threshold/pack of every level; with
 * discard_gray != 0 the gray lines it consumed are dropped from L2 without
 * write-back (discard.global.L2), leaving the gray workspace undefined. */
int mtb_pyramid_hist(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride,
                     int w, int h, int n_img, int levels,
                     uint8_t* gray, uint32_t* hist_ws, void* stream);
int mtb_threshold_levels(const uint8_t* gray, const uint32_t* hist_ws, int w, int h, int n_img,
                         int levels, int tol, uint32_t* hist_out, int32_t* medians,
                         uint64_t* mtb, uint64_t* exclusion, int discard_gray, void* stream);

/* mtb_preprocess for small images without a gray arena (csrc/cluster.cu): the
 * gray pyramid of each image is held in the shared memory of a thread-block
 * cluster, so HBM sees only the RGB read and the bitmap writes.  Same outputs
 * (medians [img][n], optional dense histograms [img][n][256], packed maps) as
 * mtb_preprocess.  Needs n <= 6 levels, 3*w % 4 == 0, 16-byte aligned rows and
 * images, and an image whose tiles fit one cluster (about 1.5 MP); otherwise
 * MTB_EINVAL.  mtb_preprocess_maps_cluster returns the cluster size it would
 * use on the current device (0 = geometry not supported). */
int mtb_preprocess_maps(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride,
                        int w, int h, int n_img, int levels, int tol,
                        uint32_t* hist_out, int32_t* medians, uint64_t* mtb, uint64_t* exclusion, void* stream);
int mtb_preprocess_maps_cluster(int w, int h, int levels);
/* The full launch shape: shape[4] = {cluster size, streaming groups of 128
 * threads, tile slots per CTA, clusters the device co-schedules}; returns the
 * cluster size (0 = not supported). */
int mtb_preprocess_maps_shape(int w, int h, int levels, int* shape);

/* Coarse-to-fine search (find_offset, search.py:74-95; per level
 * search_level, search.py:53-71) for P pairs at once, all levels on device.
 *   maps     device table, n_levels x P x 4 pointers {ref.mtb, ref.excl,
 *            tgt.mtb, tgt.excl} to each level's packed words
 *   dims     [host] n_levels x 3 int32 {w, h, nwords64}; index 0 = full res
 *   base     optional device P x 2 int32 base offset for the deepest level
 *            (NULL = (0,0), as find_offset)
 *   acc      out, P x n_levels x 2 int32: chosen offset per level (index = level)
 *   errs     out, P x n_levels x 9 u64: the 9 candidate errors per level in
 *            NEIGHBORHOOD order (search.py:23); index = level
 *   done     workspace, P x n_levels u32 (zeroed by this call)
 * The final offset of pair p is acc[p][0]. */
int mtb_find_offset_batch(const uint64_t* const* maps, const int32_t* dims, int n_levels, int P,
                          const int32_t* base, int32_t* acc, unsigned long long* errs,
                          uint32_t* done, void* stream);

/* ------------------------------------------------------------------------ */
/* 4. Row-sharded search (one gigapixel pair over several GPUs)  */
/* ------------------------------------------------------------------------ */

/* One level of search_level (search.py:53-71) over a window of rows: the
 * reference maps hold image rows [a_row0, a_row0+a_rows) of the level, the
 * target maps rows [b_row0, b_row0+b_rows) (the shard's rows plus halo);
 * rows outside [0, h) or outside the target window contribute 0.  Writes the
 * 9 partial counts per pair to errs (P x errs_stride u64, zeroed here) and
 * does NOT decide: the caller sums the counts across shards (NCCL
 * all-reduce) and calls mtb_decide_level.  Base offsets come from prev
 * (2 * previous level's choice) or base (deepest level) or (0,0). */
int mtb_search_level_rows(const uint64_t* const* maps, int w, int h, int64_t nwords64,
                          int a_row0, int a_rows, int b_row0, int b_rows, int P,
                          const int32_t* prev, int64_t prev_stride, const int32_t* base,
                          unsigned long long* errs, int64_t errs_stride, void* stream);

/* mtb_search_level_rows for ONE pair with the target window in up to three
 * separate buffers (row sharding without concatenating the halos): the
 * reference maps a_mtb / a_excl hold rows [a_row0, a_row0+a_rows); segment s
 * (s = 0..2: previous shard's halo, own rows, next shard's halo) holds target
 * rows [seg_row0[s], seg_row0[s]+seg_rows[s]) in seg[2s] (MTB) / seg[2s+1]
 * (exclusion), device pointers passed by value (a NULL pair or 0 rows = no
 * segment).  Rows in no segment, or outside [0, h), contribute 0.  Replaces
 * the reference's b[y - dy] row reads (kernels/_native.pyx:93-95) for a
 * shard.  Writes 9 partial counts to errs (zeroed here); no decision. */
int mtb_search_level_rows3(const uint64_t* a_mtb, const uint64_t* a_excl, int a_row0, int a_rows,
                           const uint64_t* const* seg, const int* seg_row0, const int* seg_rows, int w, int h,
                           int64_t nwords64, const int32_t* prev, const int32_t* base, unsigned long long* errs,
                           void* stream);

/* Threshold + pack every level with GIVEN medians (n_img x n int32): the
 * row-sharded flow all-reduces the histograms first, so every shard
 * thresholds with the medians of the whole image (threshold.py:80-88). */
int mtb_threshold_levels_medians(const uint8_t* gray, int w, int h, int n_img, int levels, int tol,
                                 const int32_t* medians, uint64_t* mtb, uint64_t* exclusion,
                                 int discard_gray, void* stream);

/* The search.py:67 key over summed counts: acc[p] = chosen offset. */
int mtb_decide_level(const unsigned long long* errs, int64_t errs_stride,
                     const int32_t* prev, int64_t prev_stride, const int32_t* base,
                     int32_t* acc, int64_t acc_stride, int P, void* stream);

/* ------------------------------------------------------------------------ */
/* 4. Fused pipeline — preprocess + find_offset of a whole batch            */
/* ------------------------------------------------------------------------ */

/* Workspace of mtb_align_fused for W x H images: *gray_bytes = the tile-major
 * gray ring (3 image slots, kept L2-resident), *hist_elems = spread-histogram
 * u32 per image.  Returns the level count, or -1 when the geometry needs the
 * staged entry points (more than 6 levels). */
int mtb_align_fused_workspace(int w, int h, int levels, int64_t* gray_bytes, int64_t* hist_elems);

/* u32 words of the sync_ws scratch of mtb_align_fused: per-launch tile
 * counters, per-image medians-ready flags and threshold-done counters, and
 * per-(pair, level) decided flags (zeroed by the call). */
int64_t mtb_align_fused_sync_words(int n_img, int n_pairs, int levels);

/* Images per launch B of the fused pipeline for W x H images (2 when two
 * images' gray pyramids fit L2 alongside two being read, else 1; env
 * MTB_PIPE_IMGS overrides): launch j runs K1 of images
 * jB .. jB+B-1 and K3 of the B images before them; pair (r, t) runs its
 * levels in launches max(r, t)/B + 2 ... + levels - 1. */
int mtb_align_fused_images_per_launch(int w, int h);

/* Number of pipe_kernel launches mtb_align_fused makes for this batch, or -1
 * on invalid arguments. */
int mtb_align_fused_launches(int w, int h, int levels, int n_img, const int32_t* pairs_host, int n_pairs);

/* pipeline.py:80-90 (to_grayscale -> build_pyramid -> build_mtb_pyramid for
 * every image) followed by find_offset (search.py:74-95) for every pair in
 * pairs_host [host, n_pairs x (ref, tgt)], as one software-pipelined
 * sequence of n_img + 1 + levels launches (one image per launch, K1 / K3 /
 * search of different images overlapped, gray never written to HBM).
 * rgb: n_img images, 16-B aligned rows with 3*W % 16 == 0.  Outputs have the
 * layouts of mtb_preprocess (medians, packed maps) and mtb_find_offset_batch
 * (acc [P][n][2], errs [P][n][9], done [P][n] scratch).  Bit-identical to the
 * staged entry points. */
int mtb_align_fused(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride, int w, int h, int n_img,
                    int levels, int tol, const int32_t* pairs_host, int n_pairs, uint8_t* gray_ws,
                    uint32_t* hist_ws, int32_t* medians, uint64_t* mtb, uint64_t* exclusion, int32_t* acc,
                    unsigned long long* errs, uint32_t* done, uint32_t* sync_ws, void* stream);

/* 5. Ingest (decode_image imageio.py:82-94 -> pinned host ->
 * H2D overlapped with K1).  mtb_align_fused with streamed input: the RGB
 * batch may still be arriving; K1 of image i starts once img_ready[i] != 0.
 * The caller zeroes img_ready before the call (stream-ordered before it) and
 * sets each flag after that image's H2D copy with mtb_stream_write_u32 on the
 * copy stream; img_ready = NULL is mtb_align_fused. */
int mtb_align_fused_ex(const uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_img_stride, int w, int h, int n_img,
                       int levels, int tol, const int32_t* pairs_host, int n_pairs, uint8_t* gray_ws,
                       uint32_t* hist_ws, int32_t* medians, uint64_t* mtb, uint64_t* exclusion, int32_t* acc,
                       unsigned long long* errs, uint32_t* done, uint32_t* sync_ws, const uint32_t* img_ready,
                       void* stream);

/* Stream-ordered store of `value` to device word dptr (cuStreamWriteValue32
 * with its implicit memory barrier: every earlier operation of the stream,
 * e.g. an H2D copy, is visible first). */
int mtb_stream_write_u32(uint32_t* dptr, uint32_t value, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MTBALIGN_B200_H */
