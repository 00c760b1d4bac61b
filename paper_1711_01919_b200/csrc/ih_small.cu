// ih_small.cu -- K2s: one-launch single pass for images that cannot fill the
// GPU with (frames x bin groups) CTAs (sm_100a).
//
// Same output as k2_scan (strategies.py:86-115 _propagate / compute_sequential,
// the reference's contract SPEC.md:286).  For a single 512x512 frame the
// count-table path needs three dependent launches (count, prefix, scan) whose
// latencies dominate a ~5 us problem.  K2s does the row-segment carries inside
// the scan kernel itself:
//
//   CTA  = (frame f, segment s of S rows, bin group g of 4 bins), linear
//          block index in (f, s, g) order, so a CTA only ever waits on tiles
//          with a lower index, which the in-order block dispatch has started
//          before it (forward progress without a co-residency assumption).
//   NWG  warp-groups per CTA (4 for W <= 512, 2 for W <= 1024, 1 up to 2048);
//          warp-group k owns the k-th quarter/half of the segment's rows, one
//          warp per 128-column chunk.
//   1. TMA bulk copies stage all S image rows in shared memory (one mbarrier
//      per warp-group, so each group starts as soon as its rows land).
//   2. Every warp-group counts its rows per column for the 4 bins (packed
//      16-bit lanes: bins 0/2 in one word, 1/3 in the other); the CTA's
//      aggregate (2 words per column) is published to the workspace with a
//      release flag.
//   3. The CTA waits for the flags of segments s' < s of its (f, g) and sums
//      their aggregates (split over the warp-groups, L2 loads all in flight);
//      warp-group k adds the counts of groups k' < k from shared memory.  That
//      is the column-count vector of all rows above the group's first row.
//   4. Row-scan of that vector = H_b(r0 - 1, c); then the usual packed
//      one-hot row scan per row (warp shuffles on 4 bins at once, cross-warp
//      prefix through shared memory behind a named per-group barrier) and
//      16-byte streaming stores: every output byte is written once.
//
// The aggregate reads are quadratic in the segment count (segment s reads s
// vectors of 8*W bytes), which is why K2s is only planned when a single wave
// of CTAs covers the whole problem (small W*H*frames*bins).
#include "ih_kernels.cuh"

namespace ih {

struct SmallArgs {
  const uint8_t* img;
  int64_t H, W, pitch, fstride;
  int nb;           // slab bins
  int ngroups;      // bin groups of 4
  int nseg;         // segments per frame
  int S;            // rows per segment (the last one may be shorter)
  int Sk;           // rows per warp-group = ceil(S / NWG)
  int wpg;          // warps per warp-group (= 128-column chunks)
  int TWp;          // wpg * 128: aggregate / count vector stride
  int RS;           // shared-memory stride of the staged image rows (pitch or TWp)
  int contig;       // 1: a warp-group's rows are one bulk copy (RS == pitch)
  uint32_t row_bytes;  // TMA bytes per image row = round_up(W, 16) (contig == 0)
  uint32_t* flags;     // per tile: 1 once its aggregate is published (zeroed per launch)
  uint32_t* agg;       // per tile [2][TWp] u32 column counts, 16-bit lanes
  uint32_t* out;
  unsigned long long* trace;  // debug (ih_debug_trace): per CTA {start, carries done, end, smid},
                              // then per CTA {rows landed, published, flags seen, -}
};

__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void add4(uint4& a, const uint4& b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  a.w += b.w;
}

// Steps 4a/4b of one warp-group: row-scan of the column-count vector (e4/o4:
// bins 0/2 and 1/3 in 16-bit lanes, all rows above r0) into H_b(r0 - 1, c),
// then the packed one-hot scan of the group's `nrows` staged rows and the
// 16-byte streaming stores.
template <int NWG, bool VEC>
__device__ __forceinline__ void scan_rows_small(const SmallArgs& a, const uint32_t* oh,
                                                uint4 (*tot)[4][NWG][16 / NWG],
                                                const uint8_t* myrows, const uint32_t inval[4],
                                                const uint32_t e4[4], const uint32_t o4[4],
                                                int64_t f, int g, int64_t r0, int nrows, int wg,
                                                int w, int lane, int cl) {
  constexpr int R = 4;
  uint32_t acc[4][4];  // [column j][bin i]
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    acc[j][0] = e4[j] & 0xffffu;
    acc[j][1] = o4[j] & 0xffffu;
    acc[j][2] = e4[j] >> 16;
    acc[j][3] = o4[j] >> 16;
  }
  const int gthreads = a.wpg * 32;
  const int barid = 1 + wg;  // named barrier of this warp-group (0 = __syncthreads)

  // ---- 4a. row-scan of the column counts: acc(c) <- sum_{c' <= c} = H_b(r0 - 1, c)
  if (r0 > 0) {
    uint32_t lt[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[1][i] += acc[0][i];
      acc[2][i] += acc[1][i];
      acc[3][i] += acc[2][i];
      lt[i] = acc[3][i];
    }
    uint32_t run[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t x = warp_scan_pred(lt[i]);
      const uint32_t ex = x - lt[i];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j][i] += ex;
      run[i] = __shfl_sync(kFull, x, 31);
    }
    if (lane == 0) tot[0][0][wg][w] = make_uint4(run[0], run[1], run[2], run[3]);
    named_bar(barid, gthreads);
    const uint4 tw = lane < w ? tot[0][0][wg][lane] : make_uint4(0u, 0u, 0u, 0u);
    const uint32_t wp[4] = {__reduce_add_sync(kFull, tw.x), __reduce_add_sync(kFull, tw.y),
                            __reduce_add_sync(kFull, tw.z), __reduce_add_sync(kFull, tw.w)};
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[j][i] += wp[i];
    named_bar(barid, gthreads);  // tot[0] is reused by the first batch
  }

  // ---- 4b. the scan of this group's rows
  const int64_t H = a.H, W = a.W;
  const int64_t plane = H * W;
  const int nbins_here = min(kGroup, a.nb - g * kGroup);
  const bool colok = cl < W;
  uint32_t* prow = a.out + (f * a.nb + (int64_t)g * kGroup) * plane + r0 * W + cl;
  const int nbatch = (nrows + R - 1) / R;
  for (int b = 0; b < nbatch; ++b) {
    const int buf = b & 1;
    const int rows = min(R, nrows - b * R);
    uint32_t v[R][4], ct[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      uint32_t o[4] = {0u, 0u, 0u, 0u};
      if (rr < rows) {
        const uint32_t px =
            *reinterpret_cast<const uint32_t*>(myrows + (size_t)(b * R + rr) * a.RS);
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = oh[((px >> (8 * j)) & 0xffu) | inval[j]];
      }
      const uint32_t l1 = o[0] + o[1], l2 = l1 + o[2], l3 = l2 + o[3];
      const uint32_t x = warp_scan_pred(l3);
      const uint32_t ex = x - l3;
      v[rr][0] = o[0] + ex;
      v[rr][1] = l1 + ex;
      v[rr][2] = l2 + ex;
      v[rr][3] = x;
      ct[rr] = __shfl_sync(kFull, x, 31);
      if (lane == 0)
        tot[buf][rr][wg][w] = make_uint4(byte_of(ct[rr], 0), byte_of(ct[rr], 1),
                                         byte_of(ct[rr], 2), byte_of(ct[rr], 3));
    }
    named_bar(barid, gthreads);  // double-buffered totals: one barrier per batch
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      if (rr >= rows) break;
      const uint4 tw = lane < w ? tot[buf][rr][wg][lane] : make_uint4(0u, 0u, 0u, 0u);
      const uint32_t run[4] = {__reduce_add_sync(kFull, tw.x), __reduce_add_sync(kFull, tw.y),
                               __reduce_add_sync(kFull, tw.z), __reduce_add_sync(kFull, tw.w)};
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[j][i] += run[i] + byte_of(v[rr][j], i);
      if (colok) {
        uint32_t* p = prow;
#pragma unroll
        for (int i = 0; i < kGroup; ++i, p += plane) {
          if (i >= nbins_here) break;
          if (VEC) {
            st_stream_v4(p, acc[0][i], acc[1][i], acc[2][i], acc[3][i]);
          } else {
            const uint32_t al = (uint32_t)reinterpret_cast<uintptr_t>(p) & 15u;
            if (!inval[3] && al == 0u) {
              st_stream_v4(p, acc[0][i], acc[1][i], acc[2][i], acc[3][i]);
            } else if (!inval[3] && (al & 7u) == 0u) {
              st_stream_v2(p, acc[0][i], acc[1][i]);
              st_stream_v2(p + 2, acc[2][i], acc[3][i]);
            } else if (!inval[3]) {
              st_stream(p, acc[0][i]);
              st_stream_v2(p + 1, acc[1][i], acc[2][i]);
              st_stream(p + 3, acc[3][i]);
            } else {
#pragma unroll
              for (int j = 0; j < 4; ++j)
                if (!inval[j]) st_stream(p + j, acc[j][i]);
            }
          }
        }
      }
      prow += W;
    }
  }
}

// 1-D grid in (f, s, g) order; aggregates and release/acquire flags in the
// workspace (the flags are zeroed per call by a memset).  Tried and removed:
// the segments of a (frame, group) as one thread-block cluster exchanging the
// aggregates through DSMEM (no workspace, no memset) -- 16-CTA clusters of
// one-CTA-per-SM blocks could not be co-resident on B200 at all, and 9-CTA
// clusters ran in two waves of GPC placements (512x512x64 bins 36.6 vs 25.0
// us, profiles/r02d/k2s_modes.txt).
template <int NWG, bool VEC>
__global__ void __launch_bounds__(512, 1) k2_small(SmallArgs a, RelLut lut) {
  constexpr int R = 4;                // rows per cross-warp batch
  constexpr int MAXW = 16 / NWG;      // warps per group
  __shared__ uint32_t oh[kOneHotEntries];
  __shared__ uint4 tot[2][R][NWG][MAXW];
  __shared__ __align__(8) uint64_t full_bar[NWG];
  extern __shared__ __align__(128) uint8_t smem[];
  // smem: image rows [S x RS + slack] | cnt [NWG][2][TWp] | psum [NWG][2][TWp]
  const size_t ring_bytes = ((size_t)a.S * a.RS + a.TWp + 15) / 16 * 16;
  uint8_t* ring = smem;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + ring_bytes);
  uint32_t* psum = cnt + (size_t)NWG * 2 * a.TWp;

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wg = warp / a.wpg;        // warp-group
  const int w = warp - wg * a.wpg;    // warp inside the group
  const int64_t H = a.H, W = a.W;
  const unsigned long long t_start = a.trace ? globaltimer() : 0ull;

  // Tile = blockIdx.x in (f, s, g) order: CTAs are dispatched in index order,
  // so every tile a CTA waits on (same f and g, lower s) started before it --
  // the assumption CUB's decoupled look-back makes; no co-residency needed.
  const uint32_t t = blockIdx.x;
  const int g = (int)(t % (uint32_t)a.ngroups);
  const int s = (int)((t / (uint32_t)a.ngroups) % (uint32_t)a.nseg);
  const int64_t f = (int64_t)(t / ((uint32_t)a.ngroups * (uint32_t)a.nseg));
  const int64_t rs = (int64_t)s * a.S, re = min(rs + a.S, H);
  if (threadIdx.x == 0) {  // stage the segment's rows: one barrier per warp-group
    for (int k = 0; k < NWG; ++k) mbar_init(&full_bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint8_t* img = a.img + f * a.fstride;
    for (int k = 0; k < NWG; ++k) {
      const int64_t k0 = min(rs + (int64_t)k * a.Sk, re), k1 = min(k0 + a.Sk, re);
      if (k1 <= k0) continue;
      if (a.contig) {  // rows k0..k1-1 are contiguous: one bulk copy
        mbar_expect_tx(&full_bar[k], (uint32_t)((k1 - k0) * a.pitch));
        tma_row(ring + (size_t)(k0 - rs) * a.RS, img + k0 * a.pitch, (uint32_t)((k1 - k0) * a.pitch),
                &full_bar[k]);
      } else {
        mbar_expect_tx(&full_bar[k], (uint32_t)(k1 - k0) * a.row_bytes);
        for (int64_t r = k0; r < k1; ++r)
          tma_row(ring + (size_t)(r - rs) * a.RS, img + r * a.pitch, a.row_bytes, &full_bar[k]);
      }
    }
  }
  build_onehot(oh, lut, g);  // overlaps the row copies
  __syncthreads();  // table and mbarrier inits visible
  const int64_t r0 = min(rs + (int64_t)wg * a.Sk, re), r1 = min(r0 + a.Sk, re);
  const int nrows = (int)(r1 - r0);
  const int cl = w * kChunk + lane * 4;  // this lane's first column
  uint32_t inval[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) inval[j] = (cl + j < W) ? 0u : 256u;
  const uint8_t* myrows = ring + (size_t)(r0 - rs) * a.RS + cl;

  // ---- 2. column counts of this group's rows, 16-bit lanes
  if (nrows > 0) mbar_wait(&full_bar[wg], 0u);
  unsigned long long* ph = a.trace ? a.trace + 4 * ((size_t)gridDim.x + blockIdx.x) : nullptr;
  if (ph && threadIdx.x == 0) ph[0] = globaltimer();  // phases: rows landed
  uint32_t ce[4] = {0u, 0u, 0u, 0u}, co[4] = {0u, 0u, 0u, 0u};
  for (int rr = 0; rr < nrows; ++rr) {
    const uint32_t px = *reinterpret_cast<const uint32_t*>(myrows + (size_t)rr * a.RS);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t o = oh[((px >> (8 * j)) & 0xffu) | inval[j]];
      ce[j] += o & 0x00ff00ffu;
      co[j] += (o >> 8) & 0x00ff00ffu;
    }
  }
  uint32_t* mycnt = cnt + (size_t)wg * 2 * a.TWp;
  *reinterpret_cast<uint4*>(mycnt + cl) = make_uint4(ce[0], ce[1], ce[2], ce[3]);
  *reinterpret_cast<uint4*>(mycnt + a.TWp + cl) = make_uint4(co[0], co[1], co[2], co[3]);
  __syncthreads();

  // ---- the CTA aggregate (sum over the warp-groups; the frame's last
  // segment has no reader)
  const size_t vec = (size_t)2 * a.TWp;  // u32 per aggregate
  const size_t tbase = ((size_t)f * a.ngroups + g) * a.nseg;  // tile index of segment 0
  const int nthr = blockDim.x;
  if (s + 1 < a.nseg) {
    uint32_t* dst = a.agg + (tbase + s) * vec;
    for (int i = threadIdx.x * 4; i < (int)vec; i += nthr * 4) {
      uint4 x = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int k = 0; k < NWG; ++k) add4(x, *reinterpret_cast<const uint4*>(cnt + (size_t)k * vec + i));
      __stcg(reinterpret_cast<uint4*>(dst + i), x);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release_gpu(a.flags + tbase + s, 1u);
  }
  if (ph && threadIdx.x == 0) ph[1] = globaltimer();  // aggregate published

  // ---- 3. wait for the segments above, sum their aggregates
  if (s > 0) {
    for (int sp = threadIdx.x; sp < s; sp += nthr)
      while (ld_acquire_gpu(a.flags + tbase + sp) == 0u) __nanosleep(32);
    __syncthreads();
    if (ph && threadIdx.x == 0) ph[2] = globaltimer();  // predecessors' flags seen
    // warp-group k sums segments sp = k, k + NWG, ... (4 in flight)
    uint4 pe = make_uint4(0u, 0u, 0u, 0u), po = make_uint4(0u, 0u, 0u, 0u);
    for (int sp = wg; sp < s; sp += 4 * NWG) {
      uint4 e[4], o[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = sp + u * NWG;
        e[u] = o[u] = make_uint4(0u, 0u, 0u, 0u);
        if (q < s) {
          const uint32_t* src = a.agg + (tbase + q) * vec;
          e[u] = __ldcg(reinterpret_cast<const uint4*>(src + cl));
          o[u] = __ldcg(reinterpret_cast<const uint4*>(src + a.TWp + cl));
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        add4(pe, e[u]);
        add4(po, o[u]);
      }
    }
    uint32_t* myps = psum + (size_t)wg * vec;
    *reinterpret_cast<uint4*>(myps + cl) = pe;
    *reinterpret_cast<uint4*>(myps + a.TWp + cl) = po;
  }
  __syncthreads();

  // ---- column counts of every row above r0: segments above + groups above
  uint32_t e4[4] = {0u, 0u, 0u, 0u}, o4[4] = {0u, 0u, 0u, 0u};
  for (int k = 0; k < NWG; ++k) {
    if (s > 0) {
      const uint4 x = *reinterpret_cast<const uint4*>(psum + (size_t)k * vec + cl);
      const uint4 y = *reinterpret_cast<const uint4*>(psum + (size_t)k * vec + a.TWp + cl);
      e4[0] += x.x; e4[1] += x.y; e4[2] += x.z; e4[3] += x.w;
      o4[0] += y.x; o4[1] += y.y; o4[2] += y.z; o4[3] += y.w;
    }
    if (k < wg) {
      const uint4 x = *reinterpret_cast<const uint4*>(cnt + (size_t)k * vec + cl);
      const uint4 y = *reinterpret_cast<const uint4*>(cnt + (size_t)k * vec + a.TWp + cl);
      e4[0] += x.x; e4[1] += x.y; e4[2] += x.z; e4[3] += x.w;
      o4[0] += y.x; o4[1] += y.y; o4[2] += y.z; o4[3] += y.w;
    }
  }
  const size_t cta = blockIdx.x;
  if (a.trace && threadIdx.x == 0) {  // debug timeline (uniform branch)
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    a.trace[4 * cta + 0] = t_start;
    a.trace[4 * cta + 1] = globaltimer();
    a.trace[4 * cta + 3] = smid;
  }
  if (nrows > 0) scan_rows_small<NWG, VEC>(a, oh, tot, myrows, inval, e4, o4, f, g, r0, nrows, wg, w, lane, cl);
  if (a.trace && lane == 0 && w == 0)  // each group's end; the last one wins
    atomicMax(a.trace + 4 * cta + 2, globaltimer());
}

}  // namespace ih
