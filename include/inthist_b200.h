/*
 * inthist_b200.h -- C ABI of the B200 integral-histogram engine.
 *
 * The reference `inthist` (arXiv 1711.01919 CPU restatement) exposes its hot
 * path as Python module functions; no FFI exists upstream.  Each entry point
 * below replaces the compute body of one reference function (paths relative
 * to the reference package pkg/src/inthist/):
 *
 *   ih_integral_histogram   <- strategies.py:219-229 compute() and the four
 *                              strategies it dispatches to: compute_sequential
 *                              :109-115, compute_crossweave :129-150,
 *                              compute_sts :162-169, compute_wavefront :172-216
 *                              (all bit-identical), plus the
 *                              binning BinSpec.bin_image core.py:94-96.
 *   ih_region_histograms    <- core.py:179-195 region_histogram (batched).
 *   ih_window_counts        <- likelihood.py:34-52 window_counts.
 *   ih_likelihood_map       <- likelihood.py:55-77 likelihood_map (fused).
 *   ih_wavefront            <- strategies.py:172-216 compute_wavefront with a
 *                              trace: the tiled wavefront as scheduled.
 *   ih_scan_u64             <- scan.py:33-76 inclusive/exclusive/blocked_scan.
 *   ih_scan_axis_u32        <- scan.py:79-92 scan_rows / scan_cols.
 *   ih_transpose            <- scan.py:95-103 transpose.
 *
 * Conventions (all entry points):
 *   - stream-ordered and asynchronous: work is enqueued on `stream`; nothing
 *     synchronises the host; no allocation (the caller owns every buffer,
 *     including the workspace); no global state except the optional
 *     row-segment hint table of ih_plan_hint.
 *   - all pointers except `lut256` are DEVICE pointers; sizes in elements
 *     unless suffixed _bytes.
 *   - argument validation mirrors the reference's exception order; every
 *     status maps 1:1 onto a reference exception class (errors.py:4-29).
 *   - no CPU fallback: a missing/failed CUDA device yields IH_ERR_CUDA.
 *
 * Layout: the integral-histogram tensor is bin-major (bins, H, W) uint32,
 * C-contiguous, exactly as IntegralHistogram.counts (core.py:106-116).  A
 * batch of frames is (frames, slab_bins, H, W).
 */
#ifndef INTHIST_B200_H
#define INTHIST_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    IH_OK = 0,
    IH_ERR_SHAPE = 1,     /* errors.py:16 ShapeError     */
    IH_ERR_CAPACITY = 2,  /* errors.py:8  CapacityError  */
    IH_ERR_PARAM = 3,     /* errors.py:20 ParameterError */
    IH_ERR_BOUNDS = 4,    /* errors.py:12 BoundsError    */
    IH_ERR_CUDA = 5       /* RuntimeError (device/launch failure) */
} ih_status;

/* Kernel family used by ih_integral_histogram.  Results are bit-identical
 * for every choice (the reference's contract). */
typedef enum {
    IH_KERNEL_AUTO = 0,         /* single-pass scan (column-tiled beyond 2048 columns) */
    IH_KERNEL_SINGLE_PASS = 1,  /* K2: fused bin + 2D scan, each output byte written once */
    IH_KERNEL_CROSSWEAVE = 2    /* K1 + K1b: fused bin/row scan, then column scan (CW-B) */
} ih_kernel;

/* Workspace bytes ih_integral_histogram needs for this problem (0 is a valid
 * answer).  `slab_bins` = bin_hi - bin_lo. */
size_t ih_workspace_bytes(int64_t frames, int64_t height, int64_t width,
                          int32_t slab_bins, int32_t kernel);

/* Integral histograms of `frames` 8-bit images, bins [bin_lo, bin_hi) only.
 *
 *   img           device, frame f row r at img + f*frame_stride + r*img_pitch
 *   lut256        HOST pointer, 256 entries, each < bins (BinSpec.table)
 *   bins          total bin count of the spec, 1..256 (core.py:72-73)
 *   bin_lo/hi     the slab this call produces (bin sharding; 0/bins = all)
 *   out           device, (frames, bin_hi-bin_lo, height, width) uint32,
 *                 16-byte aligned when width % 4 == 0 (4-byte otherwise)
 *   workspace     device scratch of >= ih_workspace_bytes(...) bytes,
 *                 16-byte aligned.  Contents need no initialisation.
 *
 * Errors, in the reference's order (strategies.py:131-132, core.py:53-57):
 *   IH_ERR_SHAPE     frames/height/width < 1, bins outside 1..256, LUT entry
 *                    >= bins, bad slab, null pointers
 *   IH_ERR_CAPACITY  width*height > 2^32-1
 *   IH_ERR_PARAM     img_pitch < width, frame_stride < height*img_pitch,
 *                    workspace too small, unknown kernel, misaligned out or
 *                    workspace (checked before any launch)
 *   IH_ERR_CUDA      launch failure */
ih_status ih_integral_histogram(const uint8_t *img, int64_t frames, int64_t height,
                                int64_t width, int64_t img_pitch, int64_t frame_stride,
                                const uint8_t *lut256, int32_t bins, int32_t bin_lo,
                                int32_t bin_hi, uint32_t *out, void *workspace,
                                size_t workspace_bytes, int32_t kernel, void *stream);

/* The two phases of ih_integral_histogram, exported separately so callers
 * (bench.py) can time the dominant kernel alone with events on `stream`.
 * ih_integral_histogram == ih_ih_prepare + ih_ih_scan. */
ih_status ih_ih_prepare(const uint8_t *img, int64_t frames, int64_t height, int64_t width,
                        int64_t img_pitch, int64_t frame_stride, const uint8_t *lut256,
                        int32_t bins, int32_t bin_lo, int32_t bin_hi, void *workspace,
                        size_t workspace_bytes, int32_t kernel, void *stream);
ih_status ih_ih_scan(const uint8_t *img, int64_t frames, int64_t height, int64_t width,
                     int64_t img_pitch, int64_t frame_stride, const uint8_t *lut256,
                     int32_t bins, int32_t bin_lo, int32_t bin_hi, uint32_t *out,
                     void *workspace, size_t workspace_bytes, int32_t kernel, void *stream);

/* The execution plan ih_integral_histogram would use for this problem
 * (diagnostics and benchmark bookkeeping; no device work).  `aligned16` says
 * whether image rows are 16-byte aligned (the TMA path).  On return:
 *   info[0] kernel family used (ih_kernel)   info[1] kernel launches per call
 *   info[2] row segments per frame           info[3] rows per segment
 *   info[4] 128-column chunks per lane       info[5] rows per barrier batch
 *   info[6] warps per CTA                    info[7] workspace bytes needed
 *   info[8] column tiles per row             info[9] tile width (columns)
 *   info[10] resident scan CTAs (SMs x CTAs/SM)  info[11] scan CTAs per row segment
 *   info[12] big segments (the rest are tail segments)  info[13] tail segment rows
 *   info[14] segment carries: 0 none, 1 count table (prepass kernels), 2 look-back,
 *            3 cluster (DSMEM), 4 in-kernel (K2s: one launch, small images)
 *   info[15] bins per scan CTA (1, 2: rows packed into the spare bytes; 4)
 * (`info` holds 16 entries; ABI 1.7, 15 before.)  Same shape/parameter errors as ih_integral_histogram. */
ih_status ih_plan_describe(int64_t frames, int64_t height, int64_t width, int32_t slab_bins,
                           int32_t kernel, int32_t aligned16, int64_t *info);

/* Row-segment hint for one problem shape (frames, height, width, slab bins):
 * ih_integral_histogram then splits each frame into `nseg` row segments
 * instead of its heuristic choice; with tail_pct > 0 the last ~tail_pct % of
 * the rows become short segments of 1/tail_div the height (0: 4), which the
 * segment-major scan grid runs last.  flags bit 0: carry the segments through
 * a thread-block cluster (the <= 16 segments of a strip exchange their column
 * counts in distributed shared memory: one launch, no prepass; taken when the
 * plan allows it -- no column tiles, H < 65536); bit 1: the K2s one-launch
 * kernel (in-kernel carries; W <= 2048, 16-byte aligned rows, H < 65536);
 * bit 2: skewed segments -- tail_pct is then the percent of segments that
 * are dispatched first and tail_div (> 100) their size ratio x 100 to the
 * rest, so the older CTA of a co-resident pair (favoured by the warp
 * scheduler) does proportionally more rows; bit 3 / bit 4: bin pairs (two
 * rows per packed word, each CTA writing 2 bin planes) / bin quads.  Results are identical for
 * every choice; only speed changes.  nseg = 0 removes the hint.  A small
 * process-wide table guarded by a mutex; device.autotune() fills it. */
ih_status ih_plan_hint(int64_t frames, int64_t height, int64_t width, int32_t slab_bins,
                       int32_t nseg, int32_t tail_pct, int32_t tail_div, int32_t flags);

/* Batched four-corner region queries (core.py:179-195).
 *   t        device (nb, height, width) uint32 integral histogram (a slab is fine)
 *   regions  device (Q, 4) int32 rows (r0, c0, r1, c1), inclusive (core.py:131-158)
 *   out      device (Q, nb) uint64
 * IH_ERR_BOUNDS if any region is degenerate or outside the tensor is NOT
 * detectable without a sync: the caller validates (the Python layer does,
 * for host and device regions, core.py:142/:158 order).  The kernel never
 * reads outside the tensor: a degenerate or out-of-range region yields a
 * row of zeros. */
ih_status ih_region_histograms(const uint32_t *t, int32_t nb, int64_t height, int64_t width,
                               const int32_t *regions, int64_t q, uint64_t *out, void *stream);

/* Every h x w window's counts (likelihood.py:34-52).
 *   out  device (nb, height-h+1, width-w+1) int64, 8-byte aligned (16-byte
 *        aligned takes the paired 16-byte-store kernel; otherwise 8-byte stores)
 * IH_ERR_PARAM if h < 1 or w < 1; IH_ERR_BOUNDS if h > height or w > width
 * (likelihood.py:36-41 order); IH_ERR_PARAM if out is not 8-byte aligned. */
ih_status ih_window_counts(const uint32_t *t, int32_t nb, int64_t height, int64_t width,
                           int32_t h, int32_t w, int64_t *out, void *stream);

/* Sliding-window likelihood map (likelihood.py:55-77), fused: for every
 * h x w placement, sum over bins of metric(template_b, count_b / (h*w)),
 * clipped to [0, 1]; only the map is written.
 *   template_host  HOST pointer, nb doubles (a normalized histogram)
 *   metric         IH_METRIC_INTERSECTION (sum min) or IH_METRIC_BHATTACHARYYA (sum sqrt(p q))
 *   out            device (height-h+1, width-w+1) float64
 * IH_ERR_SHAPE nb outside 1..256; IH_ERR_PARAM bad metric / h,w < 1;
 * IH_ERR_BOUNDS window larger than the image (likelihood.py:64-69 order). */
typedef enum { IH_METRIC_INTERSECTION = 0, IH_METRIC_BHATTACHARYYA = 1 } ih_metric;
ih_status ih_likelihood_map(const uint32_t *t, int32_t nb, int64_t height, int64_t width,
                            int32_t h, int32_t w, const double *template_host, int32_t metric,
                            double *out, void *stream);

/* The same map through a per-(bin, count) metric table held in `workspace`
 * (device, >= ih_likelihood_workspace_bytes(nb, h, w) bytes, 8-byte aligned):
 * every window count lies in [0, h*w], so each term is computed once and the
 * map kernel only gathers -- bit-identical to ih_likelihood_map.  With a
 * smaller (or null) workspace it computes the terms directly. */
size_t ih_likelihood_workspace_bytes(int32_t nb, int32_t h, int32_t w);
ih_status ih_likelihood_map_ws(const uint32_t *t, int32_t nb, int64_t height, int64_t width,
                               int32_t h, int32_t w, const double *template_host, int32_t metric,
                               double *out, void *workspace, size_t workspace_bytes,
                               void *stream);

/* --- Scan building blocks (reference scan.py:33-103), K6 kernels ----------
 * Device pointers, asynchronous on `stream`; not on the integral-histogram
 * path (K2 fuses its scans).
 *
 * ih_scan_u64: out[i] = in[0] + ... + in[i]  (exclusive = 0; scan.py:33-36)
 *              out[i] = in[0] + ... + in[i-1] (exclusive = 1; scan.py:39-44)
 * over n u64 elements, summed mod 2^64 like numpy's uint64 cumsum, stored as
 * u32.  If any stored prefix exceeds 2^32-1 the kernels set *overflow to 1
 * (it is cleared first; NULL skips the check) -- the caller raises the
 * reference's ScanOverflowError after synchronising (scan.py:27-30).  The
 * result equals the reference's blocked_scan for every block length
 * (scan.py:47-76), whose three phases these kernels are.
 * `workspace` (device, >= ih_scan_workspace_bytes(n), 8-byte aligned) holds
 * the per-tile totals.  IH_ERR_PARAM: n < 0, null pointers, short workspace. */
size_t ih_scan_workspace_bytes(int64_t n);
ih_status ih_scan_u64(const uint64_t *in, int64_t n, uint32_t *out, int32_t exclusive,
                      uint32_t *overflow, void *workspace, size_t workspace_bytes,
                      void *stream);

/* Inclusive u32 (wrapping) scan along the middle axis of a contiguous
 * (outer, n, inner) array (numpy cumsum(dtype=uint32) semantics, scan.py:79-92):
 * scan_rows of an (R, C) plane is (R, C, 1), scan_cols is (1, R, C).
 * elem_bytes: 1 (u8 input) or 4 (u32 input); out is u32, same extents and
 * not overlapping `in`.  IH_ERR_PARAM on bad extents / element size. */
ih_status ih_scan_axis_u32(const void *in, int32_t elem_bytes, int64_t outer, int64_t n,
                           int64_t inner, uint32_t *out, void *stream);

/* out (cols x rows) = in (rows x cols)^T for elem_bytes in {1, 2, 4, 8, 16}
 * (scan.py:95-103; the reference's cache-blocking tile is a host concern).
 * IH_ERR_PARAM on bad extents / element size. */
ih_status ih_transpose(const void *in, int64_t rows, int64_t cols, int32_t elem_bytes,
                       void *out, void *stream);

/* Debug: when set, k2_scan writes {start ns, prologue-done ns, end ns, SM id}
 * (4 u64) per CTA into the device buffer (grids of at most `ctas` CTAs).
 * NULL turns it off.  Not for production use (adds a barrier per CTA). */
/* The wavefront tiled scan (WF-TiS) as actually scheduled, with its event
 * trace (replaces the compute body of compute_wavefront(..., trace=list),
 * strategies.py:172-216; the throughput path is ih_integral_histogram).
 * t x t tiles run in dependency order: tile (i, j) starts only after (i-1, j)
 * and (i, j-1) have finished.  Output: the full (bins, height, width) tensor,
 * bit-identical to ih_integral_histogram, and
 *   events   device, (ceil(H/t) * ceil(W/t), 2) uint32: per tile (row-major
 *            tile index i*nj + j) the global sequence numbers of its "start"
 *            and "finish" events (0, 1, 2, ... in the order they happened).
 * workspace: >= ih_wavefront_workspace_bytes(height, width, tile) bytes.
 * Errors: IH_ERR_PARAM for tile < 1 (first, strategies.py:185-186), then as
 * ih_integral_histogram with frames = 1 and the full bin range. */
size_t ih_wavefront_workspace_bytes(int64_t height, int64_t width, int32_t tile);
ih_status ih_wavefront(const uint8_t *img, int64_t height, int64_t width, int64_t img_pitch,
                       const uint8_t *lut256, int32_t bins, int32_t tile, uint32_t *out,
                       uint32_t *events, void *workspace, size_t workspace_bytes, void *stream);

void ih_debug_trace(void *device_buffer, size_t ctas);

/* Human-readable status name. */
const char *ih_status_string(ih_status s);

/* Last CUDA error string recorded by a failing call on this thread. */
const char *ih_last_error(void);

/* ABI version: (major << 16) | minor. */
int32_t ih_abi_version(void);

/* Page-locked host buffer for D2H of large results (cudaHostAlloc), owned by
 * the caller and released with ih_host_free -- unlike a caching host
 * allocator, the pages go back to the OS when the result is dropped.  NULL on
 * failure (no device, or the pages cannot be locked).  No reference
 * counterpart: the reference keeps its tensor in host memory
 * (IntegralHistogram.counts, core.py:106-116). */
void *ih_host_alloc(size_t bytes);
void ih_host_free(void *p);

#ifdef __cplusplus
}
#endif
#endif /* INTHIST_B200_H */
