// ih_single_pass.cu -- K2: the single-pass integral-histogram scan (sm_100a).
//
// Replaces the reference's four CPU strategies (strategies.py:109-229):
// sequential recursion, cross-weave (CW-B), scan-transpose-scan (CW-STS) and
// the wavefront tiled scan (WF-TiS).  Every output element is computed in
// registers and written to HBM exactly once.
//
// Decomposition:
//   CTA  = (bin group g of 4 bins, row segment s, frame f), full image width.
//   warp = CPL consecutive 128-column chunks of that width.
//   lane = 4 consecutive columns per chunk; registers hold the vertical
//          accumulator acc[chunk][col][bin] = H_b(r, c) of the current row.
// Per row: packed one-hot (4 bins in the 4 bytes of a u32, via a 257-entry
// smem table), 3 in-lane adds, one 5-step warp shuffle scan on packed bytes
// (4 bins at once), cross-warp exclusive prefix through smem (one barrier per
// batch of R rows, double-buffered), then acc += row prefix (IADD3) and a
// 16-byte streaming store per (lane, bin).
//
// Carries between row segments (reduce-then-scan, SURVEY.md 7.4 option B):
//   k2_colcounts : per (segment, column, bin) pixel counts     (reads image)
//   k2_colprefix : exclusive prefix of those over segments     (tiny table)
//   k2_scan      : initial acc(c) = full-width row scan of that prefix, which
//                  equals H_b(r_s - 1, c) -- the last row of the segment above.
// With one segment per frame (large batches) only k2_scan runs.
#include "ih_kernels.cuh"

namespace ih {

// ---------------------------------------------------------------------------
// k2_colcounts: ws[f][s][b][c] = #{ r in segment s : Q(I(r,c)) = b }, for the
// 64-bin slab `blockIdx.z % nslab64` of the padded bin range, s < nseg-1.
// CTA = 128 threads = one 128-column chunk; thread t owns column t (no atomics:
// hist[b][t] is private to t, bank = t mod 32, conflict-free).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k2_colcounts(const uint8_t* __restrict__ img,
                                                     int64_t H, int64_t W, int64_t pitch,
                                                     int64_t fstride, RelLut lut, int S,
                                                     int nseg, int nbp, int64_t Wp,
                                                     int nslab64, uint32_t* __restrict__ ws) {
  __shared__ uint32_t hist[64][kChunk];
  __shared__ uint8_t slut[256];
  const int t = threadIdx.x;
  const int64_t c = (int64_t)blockIdx.x * kChunk + t;
  const int s = blockIdx.y;
  const int slab = blockIdx.z % nslab64;
  const int64_t f = blockIdx.z / nslab64;
  for (int v = t; v < 256; v += 128) slut[v] = lut.rel[v];
#pragma unroll 8
  for (int b = 0; b < 64; ++b) hist[b][t] = 0;
  __syncthreads();
  const uint8_t* base = img + f * fstride;
  const int64_t r0 = (int64_t)s * S;
  const int64_t r1 = (r0 + S < H ? r0 + S : H);
  const uint32_t lo = (uint32_t)slab * 64u;
  if (c < W) {
    int64_t r = r0;
    for (; r + 8 <= r1; r += 8) {
      uint8_t p[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) p[k] = __ldg(base + (r + k) * pitch + c);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        uint32_t d = (uint32_t)slut[p[k]] - lo;
        if (d < 64u) hist[d][t] += 1u;
      }
    }
    for (; r < r1; ++r) {
      uint32_t d = (uint32_t)slut[__ldg(base + r * pitch + c)] - lo;
      if (d < 64u) hist[d][t] += 1u;
    }
  }
  // (no barrier needed: every thread reads back only its own column)
  const int nbs = min(64, nbp - slab * 64);
  uint32_t* dst = ws + ((f * nseg + s) * (int64_t)nbp + lo) * Wp + c;
  for (int b = 0; b < nbs; ++b) dst[(int64_t)b * Wp] = hist[b][t];
}

// ---------------------------------------------------------------------------
// k2_colprefix: in place, ws[f][s][b][c] <- sum_{s' < s} counts[f][s'][b][c]
// (exclusive prefix over segments; slot nseg-1 is never read as a count).
// Thread per (f, b, c); loads of the nseg-1 slots are independent.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k2_colprefix(uint32_t* __restrict__ ws, int64_t frames,
                                                     int nseg, int nbp, int64_t Wp) {
  const int64_t plane = (int64_t)nbp * Wp;
  const int64_t total = frames * plane;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = i / plane, rem = i % plane;
    uint32_t* p = ws + f * nseg * plane + rem;
    uint32_t run = 0;
    int s = 0;
    for (; s + 4 <= nseg - 1; s += 4) {
      uint32_t v0 = p[(s + 0) * plane], v1 = p[(s + 1) * plane];
      uint32_t v2 = p[(s + 2) * plane], v3 = p[(s + 3) * plane];
      p[(s + 0) * plane] = run; run += v0;
      p[(s + 1) * plane] = run; run += v1;
      p[(s + 2) * plane] = run; run += v2;
      p[(s + 3) * plane] = run; run += v3;
    }
    for (; s < nseg - 1; ++s) {
      uint32_t v = p[s * plane];
      p[s * plane] = run;
      run += v;
    }
    p[(int64_t)(nseg - 1) * plane] = run;
  }
}

// ---------------------------------------------------------------------------
// k2_scan: the single pass.  Template parameters:
//   CPL  chunks per lane (warp covers CPL*128 columns)
//   R    rows per barrier batch
//   VEC  W % 4 == 0 (16-byte output stores legal)
//   TMA  image rows 16-byte aligned: rows are staged into a shared-memory ring
//        by cp.async.bulk (TMA bulk copies, mbarrier completion), NST batches
//        ahead of the consumers; otherwise lanes load pixels with LDG.
// ---------------------------------------------------------------------------
struct ScanArgs {
  const uint8_t* img;
  int64_t H, W, pitch, fstride;
  int nb;          // slab bins (bin_hi - bin_lo)
  int nbp;         // padded to a multiple of 4
  int S, nseg;     // segment rows, segments per frame
  int64_t Wp;      // padded width (multiple of 128) = row stride of the smem ring
  uint32_t row_bytes;      // bytes copied per row by TMA = round_up(W, 16)
  const uint32_t* colpre;  // ws (nseg > 1) or nullptr
  uint32_t* out;
};

template <int R>
struct Ring {
  static constexpr int kStages = R >= 4 ? 2 : (R == 2 ? 4 : 8);  // 8 rows in flight
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA 1D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void tma_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Inclusive warp scan with the lane predicate folded into the shuffle
// (shfl.sync.up returns p = source lane valid) -> SHFL + predicated IADD.
__device__ __forceinline__ uint32_t warp_scan_pred(uint32_t x) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    asm volatile(
        "{\n\t.reg .b32 y;\n\t.reg .pred p;\n\t"
        "shfl.sync.up.b32 y|p, %0, %1, 0, -1;\n\t"
        "@p add.u32 %0, %0, y;\n\t}"
        : "+r"(x)
        : "r"(d));
  }
  return x;
}

template <int CPL, int R, bool VEC, bool TMA>
__global__ void __launch_bounds__(512) k2_scan(ScanArgs a, RelLut lut) {
  constexpr int NST = Ring<R>::kStages;
  __shared__ uint32_t oh[kOneHotEntries];
  __shared__ uint4 tot[2][R][32];
  __shared__ __align__(8) uint64_t full_bar[NST];
  extern __shared__ __align__(128) uint8_t ring[];  // [NST][R][Wp] image rows (TMA)

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int g = blockIdx.x;
  const int s = blockIdx.y;
  const int64_t f = blockIdx.z;
  const int64_t H = a.H, W = a.W;
  const uint8_t* img = a.img + f * a.fstride;
  const int64_t rs = (int64_t)s * a.S;
  const int64_t re = (rs + a.S < H ? rs + a.S : H);
  const int nbatch = (int)((re - rs + R - 1) / R);

  build_onehot(oh, lut, g);
  if (TMA && threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) mbar_init(&full_bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }

  // lane columns: c0[k] + j, j = 0..3
  int c0[CPL];
  uint32_t inval[CPL][4];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    c0[k] = (warp * CPL + k) * kChunk + lane * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j) inval[k][j] = (c0[k] + j < W) ? 0u : 256u;
  }

  // output: bin i of this group at plane0 + i * plane_stride (bins >= nb masked)
  const int64_t plane_elems = H * W;
  uint32_t* plane0 = a.out + (f * a.nb + (int64_t)g * kGroup) * plane_elems;
  const int nbins_here = min(kGroup, a.nb - g * kGroup);

  uint32_t acc[CPL][4][kGroup];
#pragma unroll
  for (int k = 0; k < CPL; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < kGroup; ++i) acc[k][j][i] = 0u;

  __syncthreads();  // oh[] and barriers ready

  auto issue = [&](int b) {  // producer: thread 0 only
    const int stage = b % NST;
    const int64_t r0 = rs + (int64_t)b * R;
    const int rows = (int)(re - r0 < R ? re - r0 : R);
    mbar_expect_tx(&full_bar[stage], (uint32_t)rows * a.row_bytes);
    for (int rr = 0; rr < rows; ++rr)
      tma_row(ring + ((size_t)stage * R + rr) * a.Wp, img + (r0 + rr) * a.pitch, a.row_bytes,
              &full_bar[stage]);
  };
  if (TMA && threadIdx.x == 0)
    for (int b = 0; b < NST && b < nbatch; ++b) issue(b);

  // ---- segment carry: acc(c) = sum_{c' <= c} colpre[f][s][b][c'] = H_b(r_s - 1, c)
  if (s > 0) {
    const int64_t plane_sz = (int64_t)a.nbp * a.Wp;
    const uint32_t* cp = a.colpre + (f * a.nseg + s) * plane_sz + (int64_t)g * kGroup * a.Wp;
    uint32_t run[kGroup] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      uint32_t lt[kGroup];
#pragma unroll
      for (int i = 0; i < kGroup; ++i) {
        const uint4 v = *reinterpret_cast<const uint4*>(cp + i * a.Wp + c0[k]);
        acc[k][0][i] = v.x;
        acc[k][1][i] = v.x + v.y;
        acc[k][2][i] = v.x + v.y + v.z;
        acc[k][3][i] = v.x + v.y + v.z + v.w;
        lt[i] = acc[k][3][i];
      }
#pragma unroll
      for (int i = 0; i < kGroup; ++i) {
        const uint32_t x = warp_scan_pred(lt[i]);
        const uint32_t ex = x - lt[i] + run[i];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[k][j][i] += ex;
        run[i] += __shfl_sync(kFull, x, 31);
      }
    }
    if (lane == 0) tot[0][0][warp] = make_uint4(run[0], run[1], run[2], run[3]);
    __syncthreads();
    const uint4 t = lane < warp ? tot[0][0][lane] : make_uint4(0u, 0u, 0u, 0u);
    const uint32_t wp[4] = {__reduce_add_sync(kFull, t.x), __reduce_add_sync(kFull, t.y),
                            __reduce_add_sync(kFull, t.z), __reduce_add_sync(kFull, t.w)};
#pragma unroll
    for (int k = 0; k < CPL; ++k)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < kGroup; ++i) acc[k][j][i] += wp[i];
    __syncthreads();  // tot[0] is reused by the first batch
  }

  int64_t row_off = rs * W;  // element offset of the current row within a plane
  for (int b = 0; b < nbatch; ++b) {
    const int buf = b & 1;
    const int64_t r0 = rs + (int64_t)b * R;
    const int rows = (int)(re - r0 < R ? re - r0 : R);
    const int stage = b % NST;
    if (TMA) mbar_wait(&full_bar[stage], (uint32_t)((b / NST) & 1));

    uint32_t v[R][CPL][4];  // packed in-chunk inclusive row prefix, 4 bins per word
    uint32_t ct[R][CPL];    // packed chunk totals
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        uint32_t o[4] = {0u, 0u, 0u, 0u};
        if (rr < rows) {
          if (TMA) {
            const uint32_t px = *reinterpret_cast<const uint32_t*>(
                ring + ((size_t)stage * R + rr) * a.Wp + c0[k]);
#pragma unroll
            for (int j = 0; j < 4; ++j) o[j] = oh[((px >> (8 * j)) & 0xffu) | inval[k][j]];
          } else {
            load_onehot4<false>(img + (r0 + rr) * a.pitch, c0[k], W, oh, inval[k], o);
          }
        }
        const uint32_t l1 = o[0] + o[1];
        const uint32_t l2 = l1 + o[2];
        const uint32_t l3 = l2 + o[3];
        const uint32_t x = warp_scan_pred(l3);
        const uint32_t ex = x - l3;
        v[rr][k][0] = o[0] + ex;
        v[rr][k][1] = l1 + ex;
        v[rr][k][2] = l2 + ex;
        v[rr][k][3] = x;
        ct[rr][k] = __shfl_sync(kFull, x, 31);
      }
      if (lane == 0) {
        uint32_t w4[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int k = 0; k < CPL; ++k)
#pragma unroll
          for (int i = 0; i < kGroup; ++i) w4[i] += byte_of(ct[rr][k], i);
        tot[buf][rr][warp] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
      }
    }
    __syncthreads();  // totals visible; every warp is done reading ring stage `stage`
    if (TMA && threadIdx.x == 0 && b + NST < nbatch) issue(b + NST);
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const uint4 t = lane < warp ? tot[buf][rr][lane] : make_uint4(0u, 0u, 0u, 0u);
      uint32_t run[kGroup] = {__reduce_add_sync(kFull, t.x), __reduce_add_sync(kFull, t.y),
                              __reduce_add_sync(kFull, t.z), __reduce_add_sync(kFull, t.w)};
      if (rr < rows) {
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int i = 0; i < kGroup; ++i) acc[k][j][i] += run[i] + byte_of(v[rr][k][j], i);
#pragma unroll
          for (int i = 0; i < kGroup; ++i) run[i] += byte_of(ct[rr][k], i);
          const int c = c0[k];
          if (c < W) {
            uint32_t* p = plane0 + row_off + c;
#pragma unroll
            for (int i = 0; i < kGroup; ++i) {
              if (i < nbins_here) {
                if (VEC) {
                  st_stream_v4(p, acc[k][0][i], acc[k][1][i], acc[k][2][i], acc[k][3][i]);
                } else {
#pragma unroll
                  for (int j = 0; j < 4; ++j)
                    if (c + j < W) st_stream(p + j, acc[k][j][i]);
                }
              }
              p += plane_elems;
            }
          }
        }
        row_off += W;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K1 / K1b: the cross-weave (CW-B) analog, strategies.py:118-150.
// k1_rowscan: out[b][r][c] = #{c' <= c : Q(I(r,c')) = b}   (fused bin + row scan)
//   CTA = 8 warps = 8 rows of one frame for one bin group; the warp walks the
//   row chunk by chunk carrying the running count (no width limit).
// k1b_colscan: in place, out[b][r][c] += out[b][r-1][c]     (column scan)
// ---------------------------------------------------------------------------
template <bool VEC, bool ALIGNED>
__global__ void __launch_bounds__(256) k1_rowscan(const uint8_t* __restrict__ imgs, int64_t H,
                                                   int64_t W, int64_t pitch, int64_t fstride,
                                                   int nb, RelLut lut, uint32_t* __restrict__ out) {
  __shared__ uint32_t oh[kOneHotEntries];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int g = blockIdx.x;
  const int64_t r = (int64_t)blockIdx.y * 8 + warp;
  const int64_t f = blockIdx.z;
  build_onehot(oh, lut, g);
  __syncthreads();
  if (r >= H) return;
  const uint8_t* row = imgs + f * fstride + r * pitch;
  uint32_t* dst[kGroup];
  bool ok[kGroup];
#pragma unroll
  for (int i = 0; i < kGroup; ++i) {
    const int b = g * kGroup + i;
    ok[i] = b < nb;
    dst[i] = out + ((f * nb + (ok[i] ? b : 0)) * H + r) * W;
  }
  uint32_t run[kGroup] = {0u, 0u, 0u, 0u};
  for (int64_t cb = 0; cb < W; cb += kChunk) {
    const int64_t c = cb + lane * 4;
    uint32_t inval[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) inval[j] = (c + j < W) ? 0u : 256u;
    uint32_t o[4];
    load_onehot4<ALIGNED>(row, c, W, oh, inval, o);
    const uint32_t l1 = o[0] + o[1], l2 = l1 + o[2], l3 = l2 + o[3];
    const uint32_t x = warp_incl_scan(l3, lane);
    const uint32_t ex = x - l3;
    const uint32_t v[4] = {o[0] + ex, l1 + ex, l2 + ex, x};
    const uint32_t tot = __shfl_sync(kFull, x, 31);
    if (c < W) {
#pragma unroll
      for (int i = 0; i < kGroup; ++i) {
        if (!ok[i]) continue;
        const uint32_t e0 = run[i] + byte_of(v[0], i), e1 = run[i] + byte_of(v[1], i);
        const uint32_t e2 = run[i] + byte_of(v[2], i), e3 = run[i] + byte_of(v[3], i);
        if (VEC) {
          *reinterpret_cast<uint4*>(dst[i] + c) = make_uint4(e0, e1, e2, e3);
        } else {
          const uint32_t e[4] = {e0, e1, e2, e3};
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (c + j < W) dst[i][c + j] = e[j];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kGroup; ++i) run[i] += byte_of(tot, i);
  }
}

// Thread per (plane, 4-column quad) (VEC) or (plane, column); walks all rows.
template <bool VEC>
__global__ void __launch_bounds__(256) k1b_colscan(uint32_t* __restrict__ out, int64_t planes,
                                                    int64_t H, int64_t W) {
  const int64_t per = VEC ? W / 4 : W;
  const int64_t total = planes * per;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / per, q = i % per;
    uint32_t* col = out + p * H * W + (VEC ? q * 4 : q);
    if (VEC) {
      uint4 acc = *reinterpret_cast<uint4*>(col);
      int64_t r = 1;
      for (; r + 4 <= H; r += 4) {
        uint4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = *reinterpret_cast<uint4*>(col + (r + k) * W);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          acc.x += v[k].x; acc.y += v[k].y; acc.z += v[k].z; acc.w += v[k].w;
          *reinterpret_cast<uint4*>(col + (r + k) * W) = acc;
        }
      }
      for (; r < H; ++r) {
        uint4 v = *reinterpret_cast<uint4*>(col + r * W);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        *reinterpret_cast<uint4*>(col + r * W) = acc;
      }
    } else {
      uint32_t acc = col[0];
      for (int64_t r = 1; r < H; ++r) {
        acc += col[r * W];
        col[r * W] = acc;
      }
    }
  }
}

}  // namespace ih
