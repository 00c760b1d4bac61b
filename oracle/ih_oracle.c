/*
 * ih_oracle.c -- CPU restatement of the reference `inthist` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * kernels and the timed CPU baseline of `bench.py --impl reference`.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load it.  The product path (paper_1711_01919_b200) never links or
 * calls it and has no CPU fallback.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to the reference package, pkg/src/inthist/).
 *
 * Parity is pinned: tests/test_oracle.py checks these routines against the
 * golden crc32 vectors produced by running the reference itself
 * (tests/golden/make_golden.py) and against SURVEY.md Appendix A.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <zlib.h>
#include <pthread.h>
#include <unistd.h>

/* core.py:94-96  BinSpec.bin_image: table[pixels] (256-entry u8 LUT). */
void iho_bin_image(const uint8_t *img, int64_t H, int64_t W, int64_t pitch,
                   const uint8_t *lut, uint8_t *binned) {
    for (int64_t r = 0; r < H; ++r)
        for (int64_t c = 0; c < W; ++c)
            binned[r * W + c] = lut[img[r * pitch + c]];
}

/* strategies.py:86-106  _propagate: fused recursion over [r0,r1)x[c0,c1),
 * all bins:  out[b,r,c] = out[b,r-1,c] + out[b,r,c-1] - out[b,r-1,c-1] + (bin==b)
 * with out-of-range neighbours reading as zero.  The reference accumulates in
 * u64 (numba promotion) and truncates on the u32 store; every true value is
 * <= W*H <= 2^32-1 (core.py:53-57), so u32 modular arithmetic is identical. */
void iho_propagate(const uint8_t *binned, int64_t H, int64_t W, int32_t bins,
                   uint32_t *out, int64_t r0, int64_t r1, int64_t c0, int64_t c1) {
    for (int32_t b = 0; b < bins; ++b) {
        uint32_t *plane = out + (int64_t)b * H * W;
        for (int64_t r = r0; r < r1; ++r) {
            for (int64_t c = c0; c < c1; ++c) {
                uint64_t v = (binned[r * W + c] == (uint8_t)b) ? 1u : 0u;
                if (r > 0) v += plane[(r - 1) * W + c];
                if (c > 0) {
                    v += plane[r * W + c - 1];
                    if (r > 0) v -= plane[(r - 1) * W + c - 1];
                }
                plane[r * W + c] = (uint32_t)v;
            }
        }
    }
}

/* strategies.py:109-115  compute_sequential: bin, zero, propagate whole image.
 * `out` is (bins, H, W) u32, C-contiguous (core.py:106-116). */
void iho_compute_sequential(const uint8_t *img, int64_t H, int64_t W, int64_t pitch,
                            const uint8_t *lut, int32_t bins, uint32_t *out) {
    uint8_t *binned = (uint8_t *)malloc((size_t)(H * W));
    iho_bin_image(img, H, W, pitch, lut, binned);
    memset(out, 0, (size_t)bins * (size_t)H * (size_t)W * sizeof(uint32_t));
    iho_propagate(binned, H, W, bins, out, 0, H, 0, W);
    free(binned);
}

struct cw_task {
    const uint8_t *binned;
    uint32_t *out;
    int64_t H, W;
    int32_t bins;
    int phase;          /* 1 = row scans, 2 = column scans */
    int64_t lo, hi;     /* task range [lo, hi) of the flattened (bin x band) list */
    int64_t nbands, band;
};

static void *cw_worker(void *arg) {
    struct cw_task *t = (struct cw_task *)arg;
    const int64_t H = t->H, W = t->W;
    for (int64_t k = t->lo; k < t->hi; ++k) {
        if (t->phase == 1) {            /* task = (bin, row) */
            int32_t b = (int32_t)(k / H);
            int64_t r = k % H;
            const uint8_t *src = t->binned + r * W;
            uint32_t *dst = t->out + ((int64_t)b * H + r) * W;
            uint32_t run = 0;
            for (int64_t c = 0; c < W; ++c) {
                run += (src[c] == (uint8_t)b);
                dst[c] = run;
            }
        } else {                        /* task = (bin, column band) */
            int32_t b = (int32_t)(k / t->nbands);
            int64_t j = k % t->nbands;
            uint32_t *plane = t->out + (int64_t)b * H * W;
            int64_t c0 = j * t->band, c1 = c0 + t->band < W ? c0 + t->band : W;
            for (int64_t r = 1; r < H; ++r) {
                uint32_t *row = plane + r * W;
                const uint32_t *above = plane + (r - 1) * W;
                for (int64_t c = c0; c < c1; ++c) row[c] += above[c];
            }
        }
    }
    return NULL;
}

static void cw_run_phase(struct cw_task *proto, int64_t ntasks, int nthreads) {
    if (nthreads > 256) nthreads = 256;
    if (nthreads > ntasks) nthreads = (int)(ntasks > 0 ? ntasks : 1);
    pthread_t th[256];
    struct cw_task tasks[256];
    int64_t step = (ntasks + nthreads - 1) / nthreads;
    for (int i = 0; i < nthreads; ++i) {
        tasks[i] = *proto;
        tasks[i].lo = i * step < ntasks ? i * step : ntasks;
        tasks[i].hi = (i + 1) * step < ntasks ? (i + 1) * step : ntasks;
        if (nthreads == 1) cw_worker(&tasks[i]);
        else pthread_create(&th[i], NULL, cw_worker, &tasks[i]);
    }
    if (nthreads > 1)
        for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);  /* the barrier */
}

int iho_max_threads(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

/* strategies.py:129-150  compute_crossweave (CW-B), threaded.
 * Phase 1 (_cw_rows :118-121): per (bin, row) out = (binned == b), then an
 * inclusive scan along the row (scan.py:76-81).  Barrier (thread join; the
 * reference's _run_tasks :68-76).
 * Phase 2 (_cw_cols :124-126): per (bin, column band) inclusive scan down the
 * columns (scan.py:84-89), walking rows so the inner loop is contiguous.
 * workers = 0 means all online CPUs (resolve_workers :62-65).  Output is
 * independent of the worker count (integer addition is associative). */
void iho_compute_crossweave(const uint8_t *img, int64_t H, int64_t W, int64_t pitch,
                            const uint8_t *lut, int32_t bins, uint32_t *out,
                            int32_t workers) {
    int nthreads = workers > 0 ? workers : iho_max_threads();
    uint8_t *binned = (uint8_t *)malloc((size_t)(H * W));
    iho_bin_image(img, H, W, pitch, lut, binned);
    struct cw_task proto = {binned, out, H, W, bins, 1, 0, 0, 0, 256};
    cw_run_phase(&proto, (int64_t)bins * H, nthreads);
    proto.phase = 2;
    proto.nbands = (W + proto.band - 1) / proto.band;
    cw_run_phase(&proto, (int64_t)bins * proto.nbands, nthreads);
    free(binned);
}

/* streaming.py:123-155  compute_streamed restricted to one-bin chunks with
 * full-height strips: produce bin plane `b` row by row with a vertical carry
 * and feed it to crc32 -- the per-plane checksum of SURVEY.md Appendix A,
 * computable in O(W) memory for tensors that do not fit in host RAM.
 * Returns crc32 of plane b as little-endian u32 (bench.py:65-66 convention).
 * `crc_in` allows chaining planes into the whole-tensor crc. */
uint32_t iho_plane_crc32(const uint8_t *img, int64_t H, int64_t W, int64_t pitch,
                         const uint8_t *lut, int32_t b, uint32_t crc_in) {
    uint32_t *acc = (uint32_t *)calloc((size_t)W, sizeof(uint32_t));
    uLong crc = crc_in;
    for (int64_t r = 0; r < H; ++r) {
        const uint8_t *src = img + r * pitch;
        uint32_t run = 0;
        for (int64_t c = 0; c < W; ++c) {
            run += (lut[src[c]] == (uint8_t)b);
            acc[c] += run;
        }
        crc = crc32(crc, (const Bytef *)acc, (uInt)(W * 4)); /* x86: LE */
    }
    free(acc);
    return (uint32_t)crc;
}

/* zlib crc32 over a buffer (bench.py:65-66 tensor_checksum), chainable. */
uint32_t iho_crc32(const void *data, uint64_t nbytes, uint32_t crc_in) {
    uLong crc = crc_in;
    const Bytef *p = (const Bytef *)data;
    while (nbytes > 0) {
        uInt chunk = nbytes > (1u << 30) ? (1u << 30) : (uInt)nbytes;
        crc = crc32(crc, p, chunk);
        p += chunk;
        nbytes -= chunk;
    }
    return (uint32_t)crc;
}

/* core.py:179-195  region_histogram: inclusive rectangle (core.py:131-158),
 * four corner reads per bin combined in int64, corners with r<0 or c<0 read
 * as zero, result cast to u64.  regions: (Q,4) int32 rows r0,c0,r1,c1.
 * out: (Q, bins) u64.  Bounds are validated by the caller (core.py:156-158). */
void iho_region_histograms(const uint32_t *t, int32_t bins, int64_t H, int64_t W,
                           const int32_t *regions, int64_t Q, uint64_t *out) {
    for (int64_t q = 0; q < Q; ++q) {
        int64_t r0 = regions[4 * q + 0], c0 = regions[4 * q + 1];
        int64_t r1 = regions[4 * q + 2], c1 = regions[4 * q + 3];
        for (int32_t b = 0; b < bins; ++b) {
            const uint32_t *p = t + (int64_t)b * H * W;
            int64_t a = (int64_t)p[r1 * W + c1];
            int64_t up = r0 > 0 ? (int64_t)p[(r0 - 1) * W + c1] : 0;
            int64_t lf = c0 > 0 ? (int64_t)p[r1 * W + c0 - 1] : 0;
            int64_t ul = (r0 > 0 && c0 > 0) ? (int64_t)p[(r0 - 1) * W + c0 - 1] : 0;
            out[q * bins + b] = (uint64_t)(a - up - lf + ul);
        }
    }
}

/* likelihood.py:34-52  window_counts: (bins, H-h+1, W-w+1) int64 counts of
 * every h x w window; the top row / left column of placements skip the
 * out-of-range corner terms (:44-51). */
void iho_window_counts(const uint32_t *t, int32_t bins, int64_t H, int64_t W,
                       int64_t h, int64_t w, int64_t *out) {
    int64_t R = H - h + 1, C = W - w + 1;
    for (int32_t b = 0; b < bins; ++b) {
        const uint32_t *p = t + (int64_t)b * H * W;
        int64_t *o = out + (int64_t)b * R * C;
        for (int64_t i = 0; i < R; ++i) {
            for (int64_t j = 0; j < C; ++j) {
                int64_t v = (int64_t)p[(i + h - 1) * W + (j + w - 1)];
                if (i > 0) v -= (int64_t)p[(i - 1) * W + (j + w - 1)];
                if (j > 0) v -= (int64_t)p[(i + h - 1) * W + (j - 1)];
                if (i > 0 && j > 0) v += (int64_t)p[(i - 1) * W + (j - 1)];
                o[i * C + j] = v;
            }
        }
    }
}

