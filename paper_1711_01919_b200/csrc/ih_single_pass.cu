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
// k2_colcounts: ws[f][s][b][c] = #{ r in segment s : Q(I(r,c)) = b } (u16) for the
// 32-bin slab `blockIdx.z % nslab` of the padded bin range, segments s < nseg-1.
// CTA = 8 warps on the same 128-column chunk, each warp counting a contiguous
// eighth of the segment's rows (lane = 4 columns, one 32-bit pixel load per
// row, 8 rows of loads in flight).  Every warp owns a private 16-bit
// histogram [bin][k][lane] in shared memory (bank = lane: conflict-free, no
// atomics); the 8 histograms are summed once at the end.  Segment rows are
// < 65536 (host-enforced).  Pixels past the right edge map to LUT entry 256+.
// ---------------------------------------------------------------------------
constexpr int kCountSlab = 32;
constexpr int kCountRows = kCountSlab + 1;  // + a dummy row for "no bin in this slab"
// shared bytes of one warp's private histogram
constexpr size_t kCountWarpSmem = (size_t)kCountRows * 4 * 32 * sizeof(uint16_t);

// NW warps per CTA (2, 4 or 8): fewer for short segments, where zeroing and
// summing the private histograms would otherwise dominate
template <bool ALIGNED, int kCountWarps>
__global__ void __launch_bounds__(kCountWarps * 32) k2_colcounts(
    const uint8_t* __restrict__ img, int64_t H, int64_t W, int64_t pitch, int64_t fstride,
    RelLut lut, Segs sg, int nseg, int nbp, int64_t Wp, int nslab, uint16_t* __restrict__ ws,
    uint32_t* __restrict__ ctot) {
  extern __shared__ __align__(16) uint16_t chist[];  // [warp][bin row][k][lane]
  __shared__ uint16_t sofs[512];  // pixel -> byte offset of its bin row (dummy row if none)
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * kChunk + 4 * lane;
  const int s = blockIdx.y;
  const int slab = blockIdx.z % nslab;
  const int64_t f = blockIdx.z / nslab;
  const uint32_t lo = (uint32_t)slab * kCountSlab;
  constexpr uint32_t kRowBytes = 4 * 32 * sizeof(uint16_t);  // one bin row: [k][lane]
  griddep_launch_dependents();
  for (int v = threadIdx.x; v < 512; v += blockDim.x) {
    const uint32_t d = v < 256 ? (uint32_t)lut.rel[v] - lo : 0xffffffffu;
    sofs[v] = (uint16_t)((d < (uint32_t)kCountSlab ? d : (uint32_t)kCountSlab) * kRowBytes);
  }
  {
    uint4* z = reinterpret_cast<uint4*>(chist);
    for (int i = threadIdx.x; i < (int)(kCountWarps * kCountWarpSmem / 16); i += blockDim.x)
      z[i] = make_uint4(0, 0, 0, 0);
  }
  uint32_t inval[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) inval[k] = (c + k < W) ? 0u : 256u;
  __syncthreads();
  // this lane's counters: byte base + bin-row offset + k * 64
  char* hbase = reinterpret_cast<char*>(chist + (size_t)warp * kCountRows * 4 * 32 + lane);
  const uint8_t* base = img + f * fstride;
  const int64_t seg0 = sg.start(s);
  const int64_t seg1 = min(sg.start(s + 1), H);
  const int64_t per = (seg1 - seg0 + kCountWarps - 1) / kCountWarps;
  const int64_t r0 = seg0 + warp * per;
  const int64_t r1 = (r0 + per < seg1 ? r0 + per : seg1);
  auto load_px = [&](int64_t r) -> uint32_t {
    const uint8_t* row = base + r * pitch + c;
    if (ALIGNED) return __ldg(reinterpret_cast<const uint32_t*>(row));
    uint32_t px = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (c + k < W) px |= (uint32_t)__ldg(row + k) << (8 * k);
    return px;
  };
  auto count4 = [&](uint32_t px) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint16_t* h = reinterpret_cast<uint16_t*>(
          hbase + sofs[((px >> (8 * k)) & 0xffu) | inval[k]] + k * 32 * sizeof(uint16_t));
      *h += 1;
    }
  };
  if (c < W && r0 < r1) {
    // software pipeline: the next 8 rows' loads are in flight while counting
    constexpr int U = 8;
    uint32_t cur[U], nxt[U];
#pragma unroll
    for (int i = 0; i < U; ++i) cur[i] = r0 + i < r1 ? load_px(r0 + i) : 0u;
    for (int64_t r = r0; r < r1; r += U) {
#pragma unroll
      for (int i = 0; i < U; ++i) nxt[i] = r + U + i < r1 ? load_px(r + U + i) : 0u;
#pragma unroll
      for (int i = 0; i < U; ++i)
        if (r + i < r1) count4(cur[i]);
#pragma unroll
      for (int i = 0; i < U; ++i) cur[i] = nxt[i];
    }
  }
  __syncthreads();
  griddep_wait();  // PDL: complete only after the predecessor (transitivity)
  // sum the 8 private histograms; item = (bin, lane) -> 4 columns, one 8-byte store
  const int nbs = min(kCountSlab, nbp - (int)lo);
  uint16_t* dst = ws + ((f * nseg + s) * (int64_t)nbp + lo) * Wp + (int64_t)blockIdx.x * kChunk;
  for (int e = threadIdx.x; e < nbs * 32; e += blockDim.x) {
    const int l = e & 31, b = e >> 5;
    uint32_t sum[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int w = 0; w < kCountWarps; ++w)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        sum[k] += chist[(size_t)w * kCountRows * 4 * 32 + (b * 4 + k) * 32 + l];
    *reinterpret_cast<uint2*>(dst + (int64_t)b * Wp + 4 * l) =
        make_uint2(sum[0] | (sum[1] << 16), sum[2] | (sum[3] << 16));
    if (ctot) {  // column-tiled scans: the chunk's total per bin (warp-uniform b)
      const uint32_t t = __reduce_add_sync(kFull, sum[0] + sum[1] + sum[2] + sum[3]);
      if (l == 0) ctot[((f * nseg + s) * (int64_t)gridDim.x + blockIdx.x) * nbp + lo + b] = t;
    }
  }
}

// ---------------------------------------------------------------------------
// k2_colcounts_all: the same table for ALL slab bins in one pass (one read and
// one count per pixel instead of one per 32-bin slab).  CTA = (128-column
// chunk, segment, frame); NW warps stride the segment's rows (8 rows of loads
// in flight per warp) and count into ONE shared histogram with 32-bit shared
// atomics.  Word (b, h, lane) packs the 16-bit counts of columns 4*lane+2h
// (low half) and 4*lane+2h+1 (high half): increments are 1 << 16*(k&1), and
// the bank is the lane, so a warp's atomics never conflict.  Counts per
// segment are < 65536 (host-enforced), so halves never carry.  The dump is
// directly the u16x4 layout of the table.  Pixels outside the slab add into a
// discard row, so the per-pixel add is unconditional (no branch), and rows
// are addressed by stepping one pointer.  (Tried: counting 1- to 8-bin slabs
// in registers through a one-hot u64 table -- 64-bit shared loads made it
// 15-55 % slower than these shared adds; software-pipelining the row loads:
// neutral.  The kernel is bound by the shared-memory pipe -- the LUT lookup
// with ~3-way bank conflicts plus the add -- at ~6 pixels per clock per SM,
// and runs mostly under the previous call's scan via PDL.)
// ---------------------------------------------------------------------------
// Shared-memory add without a return value, as PTX: atomicAdd(.., 1) would be
// turned into warp-aggregated ATOMS.POPC.INC with a match loop per pixel.
__device__ __forceinline__ void red_shared_add(uint32_t saddr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}

// The last n < U rows of a count loop (rows p, p + rstep, ...): loads for
// binary sub-batches of n (U/2, ..., 2, 1 rows, warp-uniform branches) are
// all issued before any row is counted -- one load latency, and unlike one
// predicated U-row batch, no predicated-off counting work for short tails.
template <int U, typename Load, typename Use>
__device__ __forceinline__ void tail_rows(int n, const uint8_t* p, int64_t rstep, Load load,
                                          Use use) {
  uint32_t px[U];
  int at = 0;
#pragma unroll
  for (int b = U / 2; b >= 1; b >>= 1)
    if (n & b) {
#pragma unroll
      for (int i = 0; i < b; ++i) px[(U - 2 * b) + i] = load(p + (int64_t)(at + i) * rstep);
      at += b;
    }
#pragma unroll
  for (int b = U / 2; b >= 1; b >>= 1)
    if (n & b) {
#pragma unroll
      for (int i = 0; i < b; ++i) use(px[(U - 2 * b) + i]);
    }
}

template <bool ALIGNED, int U>
__global__ void __launch_bounds__(256) k2_colcounts_all(
    const uint8_t* __restrict__ img, int64_t H, int64_t W, int64_t pitch, int64_t fstride,
    RelLut lut, Segs sg, int nseg, int nbp, int64_t Wp, int cw, uint16_t* __restrict__ ws,
    uint32_t* __restrict__ ctot) {
  // [cw][nbp + 1][2][32]: one table per column chunk of the CTA, row nbp = discard
  extern __shared__ __align__(16) uint32_t hist2[];
  __shared__ uint32_t sw[512];  // pixel (| 256 past the edge) -> word offset of its bin row
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  // warp -> (column chunk wc of the CTA's cw, row phase of 8 / cw): whole
  // chunks per warp keep 8 rows of loads in flight even on short segments
  const int lg = __ffs(cw) - 1, wc = warp & (cw - 1), rs = 8 >> lg, phase = warp >> lg;  // cw = 2^lg
  const int64_t nch = Wp / kChunk;
  const int64_t c = ((int64_t)blockIdx.x * cw + wc) * kChunk + 4 * lane;
  const int s = blockIdx.y;
  const int64_t f = blockIdx.z;
  const int tw = (nbp + 1) * 64;  // words per chunk table
  griddep_launch_dependents();
  for (int v = threadIdx.x; v < 512; v += blockDim.x) {
    const uint32_t b = v < 256 ? (uint32_t)lut.rel[v] : 0xffffffffu;
    sw[v] = (b < (uint32_t)nbp ? b : (uint32_t)nbp) * 64u;  // outside the slab: discard row
  }
  {
    uint4* z = reinterpret_cast<uint4*>(hist2);
    for (int i = threadIdx.x; i < cw * tw / 4; i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
  }
  uint32_t inval[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) inval[k] = (c + k < W) ? 0u : 256u;
  __syncthreads();
  const uint32_t hs = (uint32_t)__cvta_generic_to_shared(hist2 + wc * tw + lane);
  const uint8_t* base = img + f * fstride;
  const int64_t seg0 = sg.start(s);
  const int64_t seg1 = min(sg.start(s + 1), H);
  auto load_px = [&](const uint8_t* row) -> uint32_t {
    if (ALIGNED) return __ldg(reinterpret_cast<const uint32_t*>(row));
    uint32_t px = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (c + k < W) px |= (uint32_t)__ldg(row + k) << (8 * k);
    return px;
  };
  auto count4 = [&](uint32_t px) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t v = ((px >> (8 * k)) & 0xffu) | inval[k];
      red_shared_add(hs + 4 * (sw[v] + (k >> 1) * 32), 1u << (16 * (k & 1)));
    }
  };
  if (c < W) {
    // rows seg0 + phase + i*rs; 8 rows of loads in flight per warp, addressed
    // by stepping one row pointer (no 64-bit multiply per load); a 32-bit row
    // count (segments are < 65536 rows)
    const int64_t rstep = (int64_t)rs * pitch;
    const int nrows = (int)(seg1 - seg0);
    const int mine = nrows > phase ? (nrows - phase + rs - 1) / rs : 0;
    const uint8_t* p = base + (seg0 + phase) * pitch + c;
    for (int it = 0; it < mine / U; ++it, p += U * rstep) {
      uint32_t px[U];
#pragma unroll
      for (int i = 0; i < U; ++i) px[i] = load_px(p + i * rstep);
#pragma unroll
      for (int i = 0; i < U; ++i) count4(px[i]);
    }
    // the last < U rows: all loads in flight at once (a row-at-a-time loop
    // serialises on the load latency), without predicated-off work
    tail_rows<U>(mine % U, p, rstep, load_px, count4);
  }
  __syncthreads();
  griddep_wait();  // PDL: complete only after the predecessor (transitivity)
  for (int k = 0; k < cw; ++k) {
    const int64_t ch = (int64_t)blockIdx.x * cw + k;
    if (ch >= nch) break;
    const uint32_t* h = hist2 + k * tw;
    uint16_t* dst = ws + ((f * nseg + s) * (int64_t)nbp) * Wp + ch * kChunk;
    for (int e = threadIdx.x; e < nbp * 32; e += blockDim.x) {  // warp-uniform bin b
      const int l = e & 31, b = e >> 5;
      const uint32_t w0 = h[(b * 2) * 32 + l], w1 = h[(b * 2 + 1) * 32 + l];
      *reinterpret_cast<uint2*>(dst + (int64_t)b * Wp + 4 * l) = make_uint2(w0, w1);
      if (ctot) {  // column-tiled scans: the chunk's total per bin
        const uint32_t sum = __reduce_add_sync(kFull, (w0 & 0xffffu) + (w0 >> 16) + (w1 & 0xffffu) + (w1 >> 16));
        if (l == 0) ctot[((f * nseg + s) * nch + ch) * nbp + b] = sum;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k2_colcounts_g1: the same table for slabs of ONE packed group (<= 4 bins,
// e.g. B = 1 / 2 / 4): counting in registers instead of shared atomics.  A
// lane's 4 columns take one one-hot word per pixel (the scan's packed-byte
// table: one byte per bin of the group), added byte-wise into 4 registers and
// widened into 16-bit lanes every 248 rows.  Warps map to (column chunk, row
// phase) as in k2_colcounts_all; the row phases of a chunk are summed through
// shared memory and dumped as the u16 table rows of the slab's <= 4 bins.
// (Slower, profiles/r02l/: a warp-shuffle bin lookup, 81 -> 91 us on HD x 64
// x 1 bin; a conflict-free lane-replicated 32 KB table, 61 -> 77 us.)  Same output as k2_colcounts_all (no
// column tiles).
// ---------------------------------------------------------------------------
template <bool ALIGNED, int U>
__global__ void __launch_bounds__(256) k2_colcounts_g1(
    const uint8_t* __restrict__ img, int64_t H, int64_t W, int64_t pitch, int64_t fstride,
    RelLut lut, Segs sg, int nseg, int nbp, int64_t Wp, int cw, uint16_t* __restrict__ ws) {
  __shared__ uint32_t oh[kOneHotEntries];
  __shared__ uint4 part[8][2][32];  // [warp][bins 0/2 | 1/3][lane] 16-bit lanes, 4 columns
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int lg = __ffs(cw) - 1, wc = warp & (cw - 1), rs = 8 >> lg, phase = warp >> lg;  // cw = 2^lg
  const int64_t nch = Wp / kChunk;
  const int64_t c = ((int64_t)blockIdx.x * cw + wc) * kChunk + 4 * lane;
  const int s = blockIdx.y;
  const int64_t f = blockIdx.z;
  griddep_launch_dependents();
  build_onehot(oh, lut, 0);
  uint32_t inval[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) inval[k] = (c + k < W) ? 0u : 256u;
  __syncthreads();
  const int64_t seg0 = sg.start(s);
  const int64_t seg1 = min(sg.start(s + 1), H);
  uint32_t ce[4] = {0u, 0u, 0u, 0u}, co[4] = {0u, 0u, 0u, 0u};
  if (c < W) {
    // this warp's rows: seg0 + phase + rs i (32-bit counters: segments are
    // < 65536 rows), pointer-stepped
    const int nrows = (int)(seg1 - seg0);
    int left = nrows > phase ? (nrows - phase + rs - 1) / rs : 0;
    const uint8_t* q = img + f * fstride + (seg0 + phase) * pitch + c;
    const int64_t rstep = rs * pitch;
    auto load_px = [&](const uint8_t* row) -> uint32_t {
      if (ALIGNED) return __ldg(reinterpret_cast<const uint32_t*>(row));
      uint32_t px = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (c + k < W) px |= (uint32_t)__ldg(row + k) << (8 * k);
      return px;
    };
    auto add4 = [&](uint32_t px, uint32_t acc[4]) {
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] += oh[((px >> (8 * k)) & 0xffu) | inval[k]];
    };
    while (left > 0) {
      // byte-packed counts: <= 248 rows (31 x 8) per flush into 16-bit lanes
      const int chunk = left < 248 ? left : 248;
      uint32_t acc[4] = {0u, 0u, 0u, 0u};
      for (int it = 0; it < chunk / U; ++it) {
        uint32_t px[U];
#pragma unroll
        for (int i = 0; i < U; ++i) px[i] = load_px(q + i * rstep);
#pragma unroll
        for (int i = 0; i < U; ++i) add4(px[i], acc);
        q += U * rstep;
      }
      const int rem = chunk % U;  // all loads in flight at once (tail_rows)
      tail_rows<U>(rem, q, rstep, load_px, [&](uint32_t px) { add4(px, acc); });
      q += rem * rstep;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        ce[k] += acc[k] & 0x00ff00ffu;
        co[k] += (acc[k] >> 8) & 0x00ff00ffu;
      }
      left -= chunk;
    }
  }
  part[warp][0][lane] = make_uint4(ce[0], ce[1], ce[2], ce[3]);
  part[warp][1][lane] = make_uint4(co[0], co[1], co[2], co[3]);
  __syncthreads();
  griddep_wait();  // PDL: complete only after the predecessor (transitivity)
  for (int e = threadIdx.x; e < cw * 64; e += blockDim.x) {  // (chunk k, half h: bins h / h + 2)
    const int l = e & 31, h = (e >> 5) & 1, k = e >> 6;
    const int64_t ch = (int64_t)blockIdx.x * cw + k;
    if (ch >= nch) break;
    uint4 t = make_uint4(0u, 0u, 0u, 0u);
    for (int r = 0; r < rs; ++r) {
      const uint4 x = part[r * cw + k][h][l];
      t.x += x.x; t.y += x.y; t.z += x.z; t.w += x.w;
    }
    uint16_t* dst = ws + ((f * nseg + s) * (int64_t)nbp) * Wp + ch * kChunk + 4 * l;
    // 16-bit lanes: low half = bin h, high half = bin h + 2
    if (h < nbp)
      *reinterpret_cast<uint2*>(dst + (int64_t)h * Wp) =
          make_uint2(__byte_perm(t.x, t.y, 0x5410), __byte_perm(t.z, t.w, 0x5410));
    if (h + 2 < nbp)
      *reinterpret_cast<uint2*>(dst + (int64_t)(h + 2) * Wp) =
          make_uint2(__byte_perm(t.x, t.y, 0x7632), __byte_perm(t.z, t.w, 0x7632));
  }
}

// ---------------------------------------------------------------------------
// k2_colprefix: in place, ws[f][s][b][c] <- sum_{s' < s} counts[f][s'][b][c]
// (u16; only used when H <= 65535 so every prefix fits).  Thread per
// (f, b, 4 columns); loads are issued 8 segments at a time before any store.
// Slot nseg-1 holds no count on entry.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint2 add_u16x4(uint2 a, uint2 b) {  // lanes never carry (< 65536)
  return make_uint2(a.x + b.x, a.y + b.y);
}

// Two-level: 8 lanes per 4-column quad, lane t owning a run of segment slots;
// run totals are exclusive-scanned with 3 shuffles inside the 8-lane group, so
// every load is issued up front (no chain of round trips over the segments).
constexpr int kPrefixLanes = 8;
constexpr int kPrefixRegs = 8;  // slots per lane held in registers (nseg <= 64)

__global__ void __launch_bounds__(256) k2_colprefix(uint16_t* __restrict__ ws, int64_t frames,
                                                     int nseg, int nbp, int64_t Wp) {
  const int64_t plane = (int64_t)nbp * Wp;  // elements per segment slot
  const int64_t quads = plane / 4;
  const int64_t groups = frames * quads;
  const int sub = threadIdx.x & (kPrefixLanes - 1);
  const int per = (nseg + kPrefixLanes - 1) / kPrefixLanes;  // slots per lane
  const int j0 = sub * per, j1 = min(nseg, j0 + per);
  griddep_launch_dependents();
  griddep_wait();  // PDL: the count table is complete
  for (int64_t gi = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kPrefixLanes; ;
       gi += (int64_t)gridDim.x * blockDim.x / kPrefixLanes) {
    // all 8 lanes of a group iterate together (the shuffles need them)
    const bool live = gi < groups;
    if (__all_sync(kFull, !live)) break;
    const int64_t f = live ? gi / quads : 0, q = live ? gi % quads : 0;
    uint2* p = reinterpret_cast<uint2*>(ws + f * nseg * plane) + q;
    if (per <= kPrefixRegs) {  // <= 64 segments: every load of the run in flight at once
      uint2 v[kPrefixRegs];
      uint2 tot = make_uint2(0u, 0u);
#pragma unroll
      for (int i = 0; i < kPrefixRegs; ++i) {
        const int j = j0 + i;
        v[i] = live && j < j1 && j < nseg - 1 ? p[(int64_t)j * quads] : make_uint2(0u, 0u);
        tot = add_u16x4(tot, v[i]);
      }
      uint2 inc = tot;
#pragma unroll
      for (int d = 1; d < kPrefixLanes; d <<= 1) {
        const uint32_t x = __shfl_up_sync(kFull, inc.x, d, kPrefixLanes);
        const uint32_t y = __shfl_up_sync(kFull, inc.y, d, kPrefixLanes);
        if (sub >= d) inc = add_u16x4(inc, make_uint2(x, y));
      }
      uint2 run = make_uint2(inc.x - tot.x, inc.y - tot.y);
#pragma unroll
      for (int i = 0; i < kPrefixRegs; ++i) {
        const int j = j0 + i;
        if (live && j < j1) {
          p[(int64_t)j * quads] = run;
          run = add_u16x4(run, v[i]);
        }
      }
      continue;
    }
    uint2 tot = make_uint2(0u, 0u);
    for (int j = j0; j < j1 && j < nseg - 1; ++j)
      if (live) tot = add_u16x4(tot, p[(int64_t)j * quads]);
    // exclusive scan of the run totals across the 8 lanes of this group
    uint2 inc = tot;
#pragma unroll
    for (int d = 1; d < kPrefixLanes; d <<= 1) {
      const uint32_t x = __shfl_up_sync(kFull, inc.x, d, kPrefixLanes);
      const uint32_t y = __shfl_up_sync(kFull, inc.y, d, kPrefixLanes);
      if (sub >= d) inc = add_u16x4(inc, make_uint2(x, y));
    }
    uint2 run = make_uint2(inc.x - tot.x, inc.y - tot.y);  // lanes never borrow (< 65536)
    if (live) {
      for (int j = j0; j < j1; ++j) {
        const uint2 v = j < nseg - 1 ? p[(int64_t)j * quads] : make_uint2(0u, 0u);
        p[(int64_t)j * quads] = run;
        run = add_u16x4(run, v);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k2_rowleft: column-tile row carries for the COLT scan.
//   lc[f][t][r][b] = #{ c < (t+1)*TW : Q(I(r,c)) = b },  t < T-1, b < nbp  (u32)
// i.e. H_b restricted to row r at the last column left of tile t+1.  Warp per row walking the row left to right (one 32-bit
// pixel load per lane per 128-column chunk, 16 chunks of loads in flight)
// into a warp-private shared histogram; the histogram is cumulative, so at
// each tile boundary it is dumped as is (coalesced, one u32 per bin).
// ---------------------------------------------------------------------------
constexpr int kRowLeftWarps = 8;

template <bool ALIGNED>
__global__ void __launch_bounds__(kRowLeftWarps * 32) k2_rowleft(
    const uint8_t* __restrict__ img, int64_t H, int64_t W, int64_t pitch, int64_t fstride,
    RelLut lut, int nbp, int T, int TW, uint32_t* __restrict__ lc) {
  __shared__ uint32_t hist[kRowLeftWarps][256];
  __shared__ uint8_t rel[256];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  griddep_launch_dependents();
  for (int v = threadIdx.x; v < 256; v += blockDim.x) rel[v] = lut.rel[v];
  for (int v = lane; v < 256; v += 32) hist[warp][v] = 0u;
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * kRowLeftWarps + warp;
  const int64_t f = blockIdx.y;
  if (r >= H) return;
  const uint8_t* row = img + f * fstride + r * pitch;
  uint32_t* h = hist[warp];
  auto load_px = [&](int64_t c) -> uint32_t {  // columns < (T-1)*TW < W: always in range
    if (ALIGNED) return __ldg(reinterpret_cast<const uint32_t*>(row + c));
    uint32_t px = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) px |= (uint32_t)__ldg(row + c + k) << (8 * k);
    return px;
  };
  auto count4 = [&](uint32_t px) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      // rel = 0xff marks "outside the slab" unless the slab has 256 bins (then
      // it is bin 255); either way only bins < nbp are counted (a marker pixel
      // with nbp == 256 lands in padding bin 255, which is never stored)
      const uint32_t b = rel[(px >> (8 * k)) & 0xffu];
      if (b < (uint32_t)nbp) atomicAdd(&h[b], 1u);
    }
  };
  const int cpt = TW / kChunk;  // chunks per tile
  constexpr int U = 16;
  for (int t = 0; t + 1 < T; ++t) {
    const int64_t cb = (int64_t)t * TW + 4 * lane;
    for (int k0 = 0; k0 < cpt; k0 += U) {
      uint32_t px[U];
#pragma unroll
      for (int u = 0; u < U; ++u) px[u] = k0 + u < cpt ? load_px(cb + (int64_t)(k0 + u) * kChunk) : 0u;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (k0 + u < cpt) count4(px[u]);
    }
    __syncwarp();
    uint32_t* dst = lc + (((f * (T - 1) + t) * H) + r) * (int64_t)nbp;
    for (int b = lane; b < nbp; b += 32) dst[b] = h[b];
    __syncwarp();
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
//   COLT column tiles: the CTA covers columns [t*TW, (t+1)*TW) of the row;
//        rows get the counts left of the tile from k2_rowleft, the segment
//        carry adds the count kernel's chunk totals left of the tile, segments above.
// ---------------------------------------------------------------------------
struct ScanArgs {
  const uint8_t* img;
  int64_t H, W, pitch, fstride;
  int nb;          // slab bins (bin_hi - bin_lo)
  int nbp;         // padded to a multiple of 4
  Segs sg;         // row segmentation
  int nseg;        // segments per frame
  int64_t Wp;      // padded width = T * TW (row stride of the carry tables)
  int T;           // column tiles per row (COLT kernels; 1 otherwise)
  int TW;          // tile width = warps * CPL * 128 = row stride of the smem ring
  uint32_t row_bytes;      // bytes copied per row by TMA = round_up(W, 16) (T == 1)
  const uint32_t* rowleft; // COLT: (frames, T-1, H, nbp) u32 row counts left of tile t+1
  const uint32_t* chunktot; // COLT: (frames, nseg, Wp/128, nbp) u32 per-chunk totals of the count table
  const uint16_t* colpre;  // CARRY_TABLE: (frames, nseg, nbp, Wp) u16 column counts or prefixes
  int table_is_prefix;     // 1: slot s holds sum_{s'<s} counts (k2_colprefix ran); 0: raw counts
  uint32_t* lb_ticket;     // CARRY_LOOKBACK: tile ticket counter (zeroed per launch)
  uint32_t* lb_flags;      //   per-tile status: 0, kFlagAgg, kFlagIncl (zeroed per launch)
  uint32_t* lb_agg;        //   per-tile column counts      (ntiles, 4, Wp) u32
  uint32_t* lb_incl;       //   per-tile inclusive prefixes (ntiles, 4, Wp) u32
  uint32_t* out;
  unsigned long long* trace;  // debug (ih_debug_trace): per CTA {start, prologue done, end, smid}
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t smem_u32_any(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// Row-segment carry schemes of k2_scan.
enum Carry { CARRY_NONE = 0, CARRY_TABLE = 1, CARRY_LOOKBACK = 2, CARRY_CLUSTER = 3 };

// Thread-block-cluster helpers (CARRY_CLUSTER): the segments of one strip form
// one cluster; counts are exchanged through distributed shared memory.
__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// load a u32 from the same shared-memory offset in cluster CTA `rank`
__device__ __forceinline__ uint32_t ld_dsmem(const uint32_t* local, uint32_t rank) {
  uint32_t remote, v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32_any(local)), "r"(rank));
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(remote) : "memory");
  return v;
}
constexpr uint32_t kFlagAgg = 1u, kFlagIncl = 2u;

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

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

// MAXT: launch bound -- 512 (<= 16 warps, up to 128 registers) or 1024
// (<= 32 warps at <= 64 registers: full SM occupancy from one CTA).
// COLT kernels must keep two 16-warp CTAs per SM (<= 64 registers).
// STG (experimental, IH_STAGED_STORES=1): output rows are staged in shared
// memory ([R][4 bins][TW] u32 after the input ring) and written by TMA bulk
// copies of whole plane rows (one per bin and row) instead of per-lane stores.
//
// KB (bins per group, 4/2/1): for B <= 2 the byte lanes of a word carry KR = 4/KB
// ROWS of KB bins instead of one row of 4 bins, so a warp scan serves KR rows
// and no lane is wasted on empty bins.
template <int CPL, int R, bool VEC, bool TMA, int CARRY, int MAXT, bool COLT, bool STG = false,
          int KB = kGroup>
__global__ void __launch_bounds__(MAXT, COLT ? 2 : 0) k2_scan(ScanArgs a, RelLut lut) {
  constexpr int NST = Ring<R>::kStages;
  constexpr int KR = kGroup / KB;  // rows packed per word
  constexpr int NP = R / KR;       // packed passes per batch
  static_assert(KB == 4 || KB == 2 || KB == 1, "bins per group");
  static_assert(R % KR == 0, "a batch holds whole packed passes");
  static_assert(KB == 4 || (!COLT && !STG && CARRY != CARRY_LOOKBACK && CARRY != CARRY_CLUSTER),
                "row packing: plain or table carries, no column tiles");
  static_assert(!STG || (TMA && VEC && !COLT && CPL == 1), "staged stores: TMA, VEC, CPL 1");
  static_assert(!(COLT && CARRY == CARRY_LOOKBACK), "column tiles use table carries");
  static_assert(!(COLT && CARRY == CARRY_CLUSTER), "column tiles use table carries");
  constexpr bool CL = CARRY == CARRY_CLUSTER;
  // CARRY_CLUSTER: this CTA's per-column segment counts, [word][thread]
  // (word = (k*4 + j)*2 + {0: bins 0/2, 1: bins 1/3}, 16-bit lanes)
  __shared__ uint32_t ccnt[CL && CPL == 1 ? 8 * 512 : 1];
  __shared__ uint32_t oh[kOneHotEntries];
  __shared__ uint4 tot[2][R][32];
  __shared__ uint4 sleft[2][COLT ? R : 1];  // COLT: per-row counts left of the tile
  __shared__ uint4 sls[COLT ? 32 : 1];      // COLT: per-warp carry parts left of the tile
  __shared__ __align__(8) uint64_t full_bar[NST];
  __shared__ uint32_t s_tile, s_flag;
  extern __shared__ __align__(128) uint8_t ring[];  // [NST][R][Wp] image rows (TMA)

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t H = a.H, W = a.W;
  const unsigned long long t_start = a.trace ? globaltimer() : 0ull;

  // Tile (frame f, bin group g, segment s).  With look-back carries the tile
  // comes from an atomic ticket, so every tile a CTA waits on has already
  // started (forward progress); segments of one (f, g) chain are adjacent.
  int g, s, t = 0;
  int64_t f;
  if (CARRY == CARRY_LOOKBACK) {
    if (threadIdx.x == 0) s_tile = atomicAdd(a.lb_ticket, 1u);
    __syncthreads();
    const uint32_t t = s_tile;
    s = (int)(t % (uint32_t)a.nseg);
    g = (int)((t / (uint32_t)a.nseg) % (uint32_t)gridDim.x);
    f = (int64_t)(t / ((uint32_t)a.nseg * gridDim.x));
  } else {
    if (COLT) {
      g = (int)(blockIdx.x / (unsigned)a.T);
      t = (int)(blockIdx.x % (unsigned)a.T);
    } else {
      g = blockIdx.x;
    }
    // segment-major grid: every frame's segment 0 first, the (short) tail
    // segments last
    s = blockIdx.z;
    f = blockIdx.y;
  }
  const uint8_t* img = a.img + f * a.fstride;
  const int64_t ct = COLT ? (int64_t)t * a.TW : 0;  // first column of the tile
  // TMA bytes per row: the tile's columns rounded up to 16 (inside the pitched row)
  const uint32_t row_bytes =
      COLT ? (uint32_t)min((int64_t)a.TW, (W - ct + 15) / 16 * 16) : a.row_bytes;
  const int64_t rs = a.sg.start(s);
  const int64_t re = min(a.sg.start(s + 1), H);
  const int nbatch = (int)((re - rs + R - 1) / R);
  // look-back: segments other than the last count their rows first (pass 0)
  const bool count_pass = (CARRY == CARRY_LOOKBACK || CL) && s + 1 < a.nseg;
  const int nb_count = count_pass ? nbatch : 0;
  const int nb_total = nb_count + nbatch;

  // ring batch b -> first row (pass 0 = counting, pass 1 = scan)
  auto batch_row0 = [&](int b) { return rs + (int64_t)(b < nb_count ? b : b - nb_count) * R; };
  auto issue = [&](int b) {  // producer: thread 0 only
    const int stage = b % NST;
    const int64_t r0 = batch_row0(b);
    const int rows = (int)(re - r0 < R ? re - r0 : R);
    mbar_expect_tx(&full_bar[stage], (uint32_t)rows * row_bytes);
    for (int rr = 0; rr < rows; ++rr)
      tma_row(ring + ((size_t)stage * R + rr) * a.TW, img + (r0 + rr) * a.pitch + ct, row_bytes,
              &full_bar[stage]);
  };
  // start the image stream first: the ring fill overlaps the table build below
  // (nobody waits on a barrier before the __syncthreads that follows)
  if (TMA && threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) mbar_init(&full_bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int b = 0; b < NST && b < nb_total; ++b) issue(b);
  }
  build_onehot_kb<KB>(oh, lut, g);

  // lane columns: ct + cl[k] + j, j = 0..3 (cl = column inside the tile)
  int cl[CPL];
  uint32_t inval[CPL][4];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    cl[k] = (warp * CPL + k) * kChunk + lane * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j) inval[k][j] = (ct + cl[k] + j < W) ? 0u : 256u;
  }

  // PDL: everything above touches only the image (never written by the
  // prepare kernels) and shared memory; the carry tables are read below
  griddep_wait();

  // output: bin i of this group at plane0 + i * plane_stride (bins >= nb masked)
  const int64_t plane_elems = H * W;
  bool colok[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) colok[k] = ct + cl[k] < W;
  uint32_t* plane0 = a.out + (f * a.nb + (int64_t)g * KB) * plane_elems;
  const int nbins_here = min(KB, a.nb - g * KB);

  uint32_t acc[CPL][4][KB];
#pragma unroll
  for (int k = 0; k < CPL; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < KB; ++i) acc[k][j][i] = 0u;

  // table carries: sum the count slots above this segment (independent global
  // loads, issued before the first barrier so they overlap the table build)
  if (CARRY == CARRY_TABLE && s > 0) {
    const int64_t plane_sz = (int64_t)a.nbp * a.Wp;
    const uint16_t* cp = a.colpre + (f * a.nseg) * plane_sz + (int64_t)g * KB * a.Wp;
    if constexpr (COLT) if (t > 0) {
      // the carry also counts the pixels above the segment and left of the
      // tile: the count kernel's per-chunk totals, segments s' < s, chunks
      // left of the tile (spread over the CTA, reduced through sls[])
      const int nch = (int)(a.Wp / kChunk), left = (int)(ct / kChunk);
      uint4 part = make_uint4(0u, 0u, 0u, 0u);
      const uint32_t* tt = a.chunktot + (f * a.nseg) * nch * a.nbp + g * KB;
      for (int e = threadIdx.x; e < s * left; e += blockDim.x) {
        const int sp = e / left, x = e - sp * left;
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(tt + ((int64_t)sp * nch + x) * a.nbp));
        part.x += v.x;
        part.y += v.y;
        part.z += v.z;
        part.w += v.w;
      }
      part.x = __reduce_add_sync(kFull, part.x);
      part.y = __reduce_add_sync(kFull, part.y);
      part.z = __reduce_add_sync(kFull, part.z);
      part.w = __reduce_add_sync(kFull, part.w);
      if (lane == 0) sls[warp] = part;
    }
    // prefix table: one slot; raw counts: sum slots 0..s-1 here (L2-resident),
    // U slots' loads in flight at a time (register budget bounds U)
    constexpr int U = CPL >= 4 ? 1 : 4;
    const int sp0 = a.table_is_prefix ? s : 0;
    const int sp1 = a.table_is_prefix ? s + 1 : s;
    for (int sp = sp0; sp < sp1; sp += U) {
      uint2 v[U][CPL][KB];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < CPL; ++k)
#pragma unroll
          for (int i = 0; i < KB; ++i)
            v[u][k][i] = sp + u < sp1 ? *reinterpret_cast<const uint2*>(
                                            cp + (sp + u) * plane_sz + i * a.Wp + ct + cl[k])
                                      : make_uint2(0u, 0u);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < CPL; ++k)
#pragma unroll
          for (int i = 0; i < KB; ++i) {
            acc[k][0][i] += v[u][k][i].x & 0xffffu;
            acc[k][1][i] += v[u][k][i].x >> 16;
            acc[k][2][i] += v[u][k][i].y & 0xffffu;
            acc[k][3][i] += v[u][k][i].y >> 16;
          }
    }

  }

  // COLT: row counts left of the tile (k2_rowleft), prefetched one batch ahead
  // by lanes 0..R-1 of warp 0 and handed to the CTA through sleft[]
  const uint32_t* lrow = nullptr;
  uint4 lnext = make_uint4(0u, 0u, 0u, 0u);
  if (COLT && t > 0) {
    lrow = a.rowleft + ((f * (a.T - 1) + (t - 1)) * H) * a.nbp + g * KB;
    if (warp == 0 && lane < R && rs + lane < re)
      lnext = __ldg(reinterpret_cast<const uint4*>(lrow + (rs + lane) * a.nbp));
  }

  __syncthreads();  // oh[] and barriers ready
  const unsigned long long t_ready = a.trace ? globaltimer() : 0ull;

  // 4 one-hot words of lane columns cl[k]..+3 for row rr of ring batch b
  auto onehot4 = [&](int b, int rr, int k, uint32_t o[4]) {
    if (TMA) {
      const int stage = b % NST;
      const uint32_t px = *reinterpret_cast<const uint32_t*>(
          ring + ((size_t)stage * R + rr) * a.TW + cl[k]);
#pragma unroll
      for (int j = 0; j < 4; ++j) o[j] = oh[((px >> (8 * j)) & 0xffu) | inval[k][j]];
    } else {
      load_onehot4<false>(img + (batch_row0(b) + rr) * a.pitch, ct + cl[k], W, oh, inval[k], o);
    }
  };

  if constexpr (CL) {
    // ---- pass 0 (all but the last segment): per-column counts of this
    // segment's rows, 4 bins in two words of 16-bit lanes, into ccnt[]
    if (count_pass) {
      uint32_t ce[CPL][4], co[CPL][4];
#pragma unroll
      for (int k = 0; k < CPL; ++k)
#pragma unroll
        for (int j = 0; j < 4; ++j) ce[k][j] = co[k][j] = 0u;
      for (int b = 0; b < nb_count; ++b) {
        const int rows = (int)(re - batch_row0(b) < R ? re - batch_row0(b) : R);
        if (TMA) mbar_wait(&full_bar[b % NST], (uint32_t)((b / NST) & 1));
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          if (rr < rows) {
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              uint32_t o[4];
              onehot4(b, rr, k, o);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                ce[k][j] += o[j] & 0x00ff00ffu;
                co[k][j] += (o[j] >> 8) & 0x00ff00ffu;
              }
            }
          }
        }
        __syncthreads();  // ring stage consumed
        if (TMA && threadIdx.x == 0 && b + NST < nb_total) issue(b + NST);
      }
#pragma unroll
      for (int k = 0; k < CPL; ++k)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          ccnt[((k * 4 + j) * 2 + 0) * blockDim.x + threadIdx.x] = ce[k][j];
          ccnt[((k * 4 + j) * 2 + 1) * blockDim.x + threadIdx.x] = co[k][j];
        }
    }
    cluster_arrive_release();  // counts visible cluster-wide
    cluster_wait_acquire();
    // ---- carry: sum the counts of the cluster's segments above (DSMEM reads;
    // cluster rank = segment, every column sum < 65536 since H < 65536)
    for (int sp = 0; sp < s; ++sp) {
#pragma unroll
      for (int k = 0; k < CPL; ++k)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t e = ld_dsmem(&ccnt[((k * 4 + j) * 2 + 0) * blockDim.x + threadIdx.x], sp);
          const uint32_t o = ld_dsmem(&ccnt[((k * 4 + j) * 2 + 1) * blockDim.x + threadIdx.x], sp);
          acc[k][j][0] += e & 0xffffu;
          acc[k][j][1] += o & 0xffffu;
          acc[k][j][2] += e >> 16;
          acc[k][j][3] += o >> 16;
        }
    }
    cluster_arrive_release();  // done reading the others' ccnt (waited at exit)
  }

  if constexpr (CARRY == CARRY_LOOKBACK) {
    const int64_t ntile_vec = (int64_t)KB * a.Wp;  // u32 per published vector
    const uint32_t tile = s_tile;
    uint32_t* flags = a.lb_flags;
    uint32_t* agg = a.lb_agg;
    uint32_t* incl = a.lb_incl;
    // ---- pass 0: per-column counts of this segment's rows for the 4 bins,
    // 16-bit lanes (bins 0/2 in ce, 1/3 in co); segments are < 65536 rows.
    if (count_pass) {
      uint32_t ce[CPL][4], co[CPL][4];
#pragma unroll
      for (int k = 0; k < CPL; ++k)
#pragma unroll
        for (int j = 0; j < 4; ++j) ce[k][j] = co[k][j] = 0u;
      for (int b = 0; b < nb_count; ++b) {
        const int rows = (int)(re - batch_row0(b) < R ? re - batch_row0(b) : R);
        if (TMA) mbar_wait(&full_bar[b % NST], (uint32_t)((b / NST) & 1));
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          if (rr < rows) {
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              uint32_t o[4];
              onehot4(b, rr, k, o);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                ce[k][j] += o[j] & 0x00ff00ffu;
                co[k][j] += (o[j] >> 8) & 0x00ff00ffu;
              }
            }
          }
        }
        __syncthreads();  // ring stage consumed
        if (TMA && threadIdx.x == 0 && b + NST < nb_total) issue(b + NST);
      }
      // publish the aggregate: agg[tile][i][c]
      uint32_t* dst = agg + (int64_t)tile * ntile_vec;
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        uint32_t cnt[KB][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          cnt[0][j] = ce[k][j] & 0xffffu;
          cnt[1][j] = co[k][j] & 0xffffu;
          cnt[2][j] = ce[k][j] >> 16;
          cnt[3][j] = co[k][j] >> 16;
        }
#pragma unroll
        for (int i = 0; i < KB; ++i)
          __stcg(reinterpret_cast<uint4*>(dst + i * a.Wp + cl[k]),
                 make_uint4(cnt[i][0], cnt[i][1], cnt[i][2], cnt[i][3]));
        if (s == 0) {  // segment 0: its aggregate is its inclusive prefix
#pragma unroll
          for (int i = 0; i < KB; ++i)
            __stcg(reinterpret_cast<uint4*>(incl + (int64_t)tile * ntile_vec + i * a.Wp + cl[k]),
                   make_uint4(cnt[i][0], cnt[i][1], cnt[i][2], cnt[i][3]));
        }
      }
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) st_release_gpu(flags + tile, s == 0 ? kFlagIncl : kFlagAgg);
    }
    // ---- look-back: acc = sum over segments s' < s of their column counts
    if (s > 0) {
      for (int sp = s - 1; sp >= 0; --sp) {
        const uint32_t pt = tile - (uint32_t)(s - sp);
        if (threadIdx.x == 0) {
          uint32_t v;
          while ((v = ld_acquire_gpu(flags + pt)) == 0u) __nanosleep(64);
          s_flag = v;
        }
        __syncthreads();
        const uint32_t v = s_flag;
        const uint32_t* src = (v == kFlagIncl ? incl : agg) + (int64_t)pt * ntile_vec;
#pragma unroll
        for (int k = 0; k < CPL; ++k)
#pragma unroll
          for (int i = 0; i < KB; ++i) {
            const uint4 x = __ldcg(reinterpret_cast<const uint4*>(src + i * a.Wp + cl[k]));
            acc[k][0][i] += x.x;
            acc[k][1][i] += x.y;
            acc[k][2][i] += x.z;
            acc[k][3][i] += x.w;
          }
        __syncthreads();  // s_flag reuse
        if (v == kFlagIncl) break;
      }
      if (count_pass) {  // inclusive = exclusive + own aggregate
        const uint32_t* own = agg + (int64_t)tile * ntile_vec;
        uint32_t* dst = incl + (int64_t)tile * ntile_vec;
#pragma unroll
        for (int k = 0; k < CPL; ++k)
#pragma unroll
          for (int i = 0; i < KB; ++i) {
            const uint4 x = __ldcg(reinterpret_cast<const uint4*>(own + i * a.Wp + cl[k]));
            __stcg(reinterpret_cast<uint4*>(dst + i * a.Wp + cl[k]),
                   make_uint4(acc[k][0][i] + x.x, acc[k][1][i] + x.y, acc[k][2][i] + x.z,
                              acc[k][3][i] + x.w));
          }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) st_release_gpu(flags + tile, kFlagIncl);
      }
    }
  }

  // ---- segment carry: acc(c) <- sum_{c' <= c} acc(c') = H_b(r_s - 1, c)
  if (CARRY != CARRY_NONE && s > 0) {
    uint32_t run[KB] = {};
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      uint32_t lt[KB];
#pragma unroll
      for (int i = 0; i < KB; ++i) {
        acc[k][1][i] += acc[k][0][i];
        acc[k][2][i] += acc[k][1][i];
        acc[k][3][i] += acc[k][2][i];
        lt[i] = acc[k][3][i];
      }
#pragma unroll
      for (int i = 0; i < KB; ++i) {
        const uint32_t x = warp_scan_pred(lt[i]);
        const uint32_t ex = x - lt[i] + run[i];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[k][j][i] += ex;
        run[i] += __shfl_sync(kFull, x, 31);
      }
    }
    if (lane == 0) {
      uint32_t r4[kGroup] = {};
#pragma unroll
      for (int i = 0; i < KB; ++i) r4[i] = run[i];
      tot[0][0][warp] = make_uint4(r4[0], r4[1], r4[2], r4[3]);
    }
    __syncthreads();
    const uint4 tw = lane < warp ? tot[0][0][lane] : make_uint4(0u, 0u, 0u, 0u);
    uint32_t wp[4] = {__reduce_add_sync(kFull, tw.x), __reduce_add_sync(kFull, tw.y),
                      __reduce_add_sync(kFull, tw.z), __reduce_add_sync(kFull, tw.w)};
    if (COLT && t > 0) {
      const uint4 x = lane < (int)(blockDim.x >> 5) ? sls[lane] : make_uint4(0u, 0u, 0u, 0u);
      wp[0] += __reduce_add_sync(kFull, x.x);
      wp[1] += __reduce_add_sync(kFull, x.y);
      wp[2] += __reduce_add_sync(kFull, x.z);
      wp[3] += __reduce_add_sync(kFull, x.w);
    }
#pragma unroll
    for (int k = 0; k < CPL; ++k)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < KB; ++i) acc[k][j][i] += wp[i];
    __syncthreads();  // tot[0] is reused by the first batch
  }

  // ---- pass 1: the scan
  // per-chunk pointer to this lane's 4 columns of the current row in bin 0's
  // plane; bin i is `i * plane_elems` further.  Stepped by W per row.
  uint32_t* prow[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) prow[k] = plane0 + rs * W + ct + cl[k];
  const bool full_group = nbins_here == KB;
  uint32_t* stage = STG ? reinterpret_cast<uint32_t*>(ring + (size_t)NST * R * a.TW) : nullptr;
  for (int b = nb_count; b < nb_total; ++b) {
    const int bi = b - nb_count;
    const int buf = bi & 1;
    const int64_t r0 = rs + (int64_t)bi * R;
    const int rows = (int)(re - r0 < R ? re - r0 : R);
    if (TMA) mbar_wait(&full_bar[b % NST], (uint32_t)((b / NST) & 1));

    uint32_t v[NP][CPL][4];  // packed in-chunk inclusive row prefix: byte q*KB+i = row q, bin i
    uint32_t ct[NP][CPL];    // packed chunk totals
#pragma unroll
    for (int rr = 0; rr < NP; ++rr) {  // packed pass rr: rows rr*KR .. rr*KR+KR-1
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        uint32_t o[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int q = 0; q < KR; ++q) {
          if (rr * KR + q < rows) {
            uint32_t oq[4];
            onehot4(b, rr * KR + q, k, oq);
#pragma unroll
            for (int j = 0; j < 4; ++j) o[j] += oq[j] << (8 * KB * q);
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
    if (COLT && t > 0 && warp == 0 && lane < R) {
      sleft[buf][lane] = lnext;
      const int64_t rn = r0 + R + lane;
      lnext = rn < re ? __ldg(reinterpret_cast<const uint4*>(lrow + rn * a.nbp))
                      : make_uint4(0u, 0u, 0u, 0u);
    }
    if (STG && threadIdx.x == 0)  // last batch's bulk stores have read the stage buffer
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();  // totals visible; every warp is done reading the ring stage
    if (TMA && threadIdx.x == 0 && b + NST < nb_total) issue(b + NST);
#pragma unroll
    for (int pp = 0; pp < NP; ++pp) {
      const uint4 tw = lane < warp ? tot[buf][pp][lane] : make_uint4(0u, 0u, 0u, 0u);
      uint32_t run4[kGroup] = {__reduce_add_sync(kFull, tw.x), __reduce_add_sync(kFull, tw.y),
                               __reduce_add_sync(kFull, tw.z), __reduce_add_sync(kFull, tw.w)};
      if (COLT && t > 0) {
        const uint4 L = sleft[buf][pp];
        run4[0] += L.x;
        run4[1] += L.y;
        run4[2] += L.z;
        run4[3] += L.w;
      }
#pragma unroll
      for (int q = 0; q < KR; ++q) {
      const int rr = pp * KR + q;  // the row of this batch
      uint32_t* run = run4 + q * KB;  // this row's byte lanes
      if (rr < rows) {
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int i = 0; i < KB; ++i) acc[k][j][i] += run[i] + byte_of(v[pp][k][j], q * KB + i);
#pragma unroll
          for (int i = 0; i < KB; ++i) run[i] += byte_of(ct[pp][k], q * KB + i);
          if (STG) {
            uint32_t* sp = stage + (size_t)rr * KB * a.TW + cl[k];
#pragma unroll
            for (int i = 0; i < KB; ++i)
              *reinterpret_cast<uint4*>(sp + (size_t)i * a.TW) =
                  make_uint4(acc[k][0][i], acc[k][1][i], acc[k][2][i], acc[k][3][i]);
          } else if (colok[k]) {
            uint32_t* p = prow[k];
            if (VEC && full_group) {
#pragma unroll
              for (int i = 0; i < KB; ++i, p += plane_elems)
                st_stream_v4(p, acc[k][0][i], acc[k][1][i], acc[k][2][i], acc[k][3][i]);
            } else {
#pragma unroll
              for (int i = 0; i < KB; ++i, p += plane_elems) {
                if (i < nbins_here) {
                  if (VEC) {
                    st_stream_v4(p, acc[k][0][i], acc[k][1][i], acc[k][2][i], acc[k][3][i]);
                  } else {
                    // W % 4 != 0: rows start at varying 4-byte offsets; use the
                    // widest store this row's alignment allows (warp-uniform:
                    // lanes are 16 bytes apart)
                    const uint32_t al = (uint32_t)reinterpret_cast<uintptr_t>(p) & 15u;
                    if (al == 0u && !inval[k][3]) {
                      st_stream_v4(p, acc[k][0][i], acc[k][1][i], acc[k][2][i], acc[k][3][i]);
                    } else if ((al & 7u) == 0u && !inval[k][3]) {
                      st_stream_v2(p, acc[k][0][i], acc[k][1][i]);
                      st_stream_v2(p + 2, acc[k][2][i], acc[k][3][i]);
                    } else if (!inval[k][3]) {  // odd word offset: 4 + 8 + 4 bytes
                      st_stream(p, acc[k][0][i]);
                      st_stream_v2(p + 1, acc[k][1][i], acc[k][2][i]);
                      st_stream(p + 3, acc[k][3][i]);
                    } else {
#pragma unroll
                      for (int j = 0; j < 4; ++j)
                        if (!inval[k][j]) st_stream(p + j, acc[k][j][i]);
                    }
                  }
                }
              }
            }
          }
          prow[k] += W;
        }
      }
      }  // q
    }
    if (STG) {  // the batch's rows are staged: bulk-copy whole plane rows out
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int rr = 0; rr < rows; ++rr)
          for (int i = 0; i < nbins_here; ++i) {
            uint32_t* dst = plane0 + (int64_t)i * plane_elems + (r0 + rr) * W;
            asm volatile(
                "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                "r"(smem_u32(stage + ((size_t)rr * KB + i) * a.TW)), "r"((uint32_t)(W * 4))
                : "memory");
          }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
  }
  if (STG && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (CL) cluster_wait_acquire();  // no CTA leaves while a neighbour may read its ccnt[]
  if (a.trace) {  // debug timeline (uniform branch)
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
      const size_t cta = blockIdx.x + (size_t)gridDim.x * (blockIdx.y + (size_t)gridDim.y * blockIdx.z);
      a.trace[4 * cta + 0] = t_start;
      a.trace[4 * cta + 1] = t_ready;
      a.trace[4 * cta + 2] = globaltimer();
      a.trace[4 * cta + 3] = smid;
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
