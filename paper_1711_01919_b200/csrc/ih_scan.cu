// ih_scan.cu -- K6: the scan module's building blocks as device kernels
// (reference pkg/src/inthist/scan.py:33-103).  Not on the integral-histogram
// path (K2 fuses its scans); these back the public scan helpers.
//
// k6_block_totals / k6_scan_totals / k6_scan_apply
//   1-D inclusive / exclusive scan of u64 elements into u32 outputs with the
//   reference's overflow guard (scan.py:27-30): sums accumulate in u64 (mod
//   2^64, like numpy's uint64 cumsum) and any output prefix above 2^32-1 sets
//   a device flag.  Reduce-then-scan in three launches -- per-tile totals, an
//   exclusive scan of the totals, per-tile scans plus the tile offset: the
//   same three-phase organisation as the reference's blocked_scan
//   (scan.py:47-76), with a 2048-element tile.
// k6_scan_inner / k6_scan_strided
//   u32 (wrapping) inclusive scan along one axis of an (outer, n, inner)
//   array: inner == 1 is scan_rows (warp per row, 512 elements per step,
//   carried), inner > 1 is scan_cols (32 columns x 32 row segments per CTA,
//   reduce-then-scan through shared memory).  numpy's cumsum(dtype=uint32) semantics
//   (scan.py:79-92).
// k6_transpose
//   32x32 shared-memory tiles with one padding column (conflict-free column
//   reads), for 1/2/4/8/16-byte elements (scan.py:95-103).
#pragma once
#include <cstdint>

#include "ih_kernels.cuh"

namespace ih {

constexpr int kScanThreads = 256;
constexpr int kScanPerThread = 8;
constexpr int kScanTile = kScanThreads * kScanPerThread;  // 2048 elements per CTA

__device__ __forceinline__ uint64_t shfl_up_u64(uint64_t x, int d) {
  const uint32_t lo = __shfl_up_sync(kFull, (uint32_t)x, d);
  const uint32_t hi = __shfl_up_sync(kFull, (uint32_t)(x >> 32), d);
  return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t x, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t y = shfl_up_u64(x, d);
    if (lane >= d) x += y;
  }
  return x;
}

// Exclusive block-wide prefix of one u64 per thread (256 threads); returns the
// block total through *total.
__device__ __forceinline__ uint64_t block_excl_scan_u64(uint64_t x, uint64_t* total) {
  __shared__ uint64_t warp_tot[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t incl = warp_incl_scan_u64(x, lane);
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  uint64_t before = 0, all = 0;
#pragma unroll
  for (int i = 0; i < kScanThreads / 32; ++i) {
    const uint64_t t = warp_tot[i];
    if (i < warp) before += t;
    all += t;
  }
  *total = all;
  return before + incl - x;
}

// Loads this thread's 8 consecutive elements of the tile (zeros past n).
template <bool V2>
__device__ __forceinline__ void load8_u64(const uint64_t* __restrict__ in, int64_t n, int64_t i0,
                                          uint64_t v[kScanPerThread]) {
  if (V2 && i0 + kScanPerThread <= n) {
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(in + i0);
#pragma unroll
    for (int j = 0; j < kScanPerThread / 2; ++j) {
      const ulonglong2 q = __ldg(p + j);
      v[2 * j] = q.x;
      v[2 * j + 1] = q.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kScanPerThread; ++j) v[j] = i0 + j < n ? __ldg(in + i0 + j) : 0ull;
  }
}

template <bool V2>
__global__ void __launch_bounds__(kScanThreads) k6_block_totals(const uint64_t* __restrict__ in,
                                                                int64_t n,
                                                                uint64_t* __restrict__ totals) {
  const int64_t i0 = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanPerThread;
  uint64_t v[kScanPerThread];
  load8_u64<V2>(in, n, i0, v);
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanPerThread; ++j) s += v[j];
  uint64_t total;
  block_excl_scan_u64(s, &total);
  if (threadIdx.x == 0) totals[blockIdx.x] = total;
}

// One CTA: exclusive scan of the tile totals in place (carried over chunks of
// 256), and the overflow flag cleared for k6_scan_apply.
__global__ void __launch_bounds__(kScanThreads) k6_scan_totals(uint64_t* __restrict__ totals,
                                                               int64_t nt,
                                                               uint32_t* __restrict__ flag) {
  if (threadIdx.x == 0 && flag) *flag = 0u;
  uint64_t carry = 0;
  for (int64_t b = 0; b < nt; b += kScanThreads) {
    const int64_t i = b + threadIdx.x;
    const uint64_t x = i < nt ? totals[i] : 0ull;
    uint64_t total;
    const uint64_t ex = block_excl_scan_u64(x, &total);
    if (i < nt) totals[i] = carry + ex;
    carry += total;
    __syncthreads();  // warp_tot reuse
  }
}

template <bool V2, bool V4OUT>
__global__ void __launch_bounds__(kScanThreads) k6_scan_apply(const uint64_t* __restrict__ in,
                                                              int64_t n,
                                                              const uint64_t* __restrict__ offsets,
                                                              int exclusive,
                                                              uint32_t* __restrict__ out,
                                                              uint32_t* __restrict__ flag) {
  const int64_t i0 = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanPerThread;
  uint64_t v[kScanPerThread];
  load8_u64<V2>(in, n, i0, v);
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanPerThread; ++j) s += v[j];
  uint64_t total;
  uint64_t run = offsets[blockIdx.x] + block_excl_scan_u64(s, &total);
  uint32_t o[kScanPerThread];
  bool over = false;
#pragma unroll
  for (int j = 0; j < kScanPerThread; ++j) {
    const uint64_t incl = run + v[j];
    const uint64_t val = exclusive ? run : incl;
    over |= (i0 + j < n) && (val >> 32) != 0;
    o[j] = (uint32_t)val;
    run = incl;
  }
  if (V4OUT && i0 + kScanPerThread <= n) {
    uint4* p = reinterpret_cast<uint4*>(out + i0);
    p[0] = make_uint4(o[0], o[1], o[2], o[3]);
    p[1] = make_uint4(o[4], o[5], o[6], o[7]);
  } else {
#pragma unroll
    for (int j = 0; j < kScanPerThread; ++j)
      if (i0 + j < n) out[i0 + j] = o[j];
  }
  if (__syncthreads_or(over) && threadIdx.x == 0 && flag) atomicOr(flag, 1u);
}

// Four consecutive elements as u32 (one 16-byte / 4-byte load when VEC).
template <typename T, bool VEC>
__device__ __forceinline__ void load4(const T* __restrict__ p, int64_t c, int64_t n,
                                      uint32_t x[4]) {
  if (VEC && c + 4 <= n) {
    if constexpr (sizeof(T) == 4) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(p + c));
      x[0] = q.x, x[1] = q.y, x[2] = q.z, x[3] = q.w;
    } else {
      const uint32_t q = __ldg(reinterpret_cast<const uint32_t*>(p + c));
#pragma unroll
      for (int j = 0; j < 4; ++j) x[j] = (q >> (8 * j)) & 0xffu;
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) x[j] = c + j < n ? (uint32_t)__ldg(p + c + j) : 0u;
}

// scan_rows: one warp per (outer) row of n contiguous elements; each step
// loads kU chunks of 128 (all loads issued before the dependent scans), then
// scans them in order carrying the running total.  VEC (rows 16-byte aligned,
// n % 4 == 0): one vector load and one 16-byte store per lane per chunk.
template <typename T, bool VEC>
__global__ void __launch_bounds__(256) k6_scan_inner(const T* __restrict__ in, int64_t rows,
                                                     int64_t n, uint32_t* __restrict__ out) {
  constexpr int kU = 2;
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const T* src = in + r * n;
  uint32_t* dst = out + r * n;
  uint32_t carry = 0;
  for (int64_t cb = 0; cb < n; cb += 128 * kU) {
    uint32_t x[kU][4];
#pragma unroll
    for (int u = 0; u < kU; ++u) load4<T, VEC>(src, cb + u * 128 + lane * 4, n, x[u]);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t c = cb + u * 128 + lane * 4;
      const uint32_t l1 = x[u][0] + x[u][1], l2 = l1 + x[u][2], l3 = l2 + x[u][3];
      const uint32_t incl = warp_incl_scan(l3, lane);
      const uint32_t ex = carry + incl - l3;
      if (VEC && c + 4 <= n) {
        *reinterpret_cast<uint4*>(dst + c) = make_uint4(ex + x[u][0], ex + l1, ex + l2, ex + l3);
      } else {
        const uint32_t y[4] = {ex + x[u][0], ex + l1, ex + l2, ex + l3};
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (c + j < n) dst[c + j] = y[j];
      }
      carry += __shfl_sync(kFull, incl, 31);
    }
  }
}

// scan_cols (and any middle axis): CTA = 32 adjacent columns x 32 row
// segments (warp = one segment of 32 columns, coalesced).  Each thread sums
// its segment, the segment offsets come from a shared-memory table, then the
// thread rescans its segment with the offset (two reads, one write).
template <typename T>
__global__ void __launch_bounds__(1024) k6_scan_strided(const T* __restrict__ in, int64_t outer,
                                                        int64_t n, int64_t inner,
                                                        uint32_t* __restrict__ out) {
  __shared__ uint32_t part[32][33];
  const int tx = threadIdx.x & 31, seg = threadIdx.x >> 5;
  const int64_t col = (int64_t)blockIdx.x * 32 + tx;
  const int64_t len = (n + 31) / 32;
  const int64_t r0 = seg * len, r1 = r0 + len < n ? r0 + len : n;
  for (int64_t o = blockIdx.y; o < outer; o += gridDim.y) {
    const T* src = in + o * n * inner + col;
    uint32_t* dst = out + o * n * inner + col;
    const bool live = col < inner;
    uint32_t sum = 0;
    if (live) {
      int64_t r = r0;
      for (; r + 4 <= r1; r += 4) {
        uint32_t x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = (uint32_t)__ldg(src + (r + j) * inner);
        sum += (x[0] + x[1]) + (x[2] + x[3]);
      }
      for (; r < r1; ++r) sum += (uint32_t)__ldg(src + r * inner);
    }
    part[seg][tx] = sum;
    __syncthreads();
    uint32_t run = 0;
    for (int s = 0; s < seg; ++s) run += part[s][tx];
    if (live) {
      int64_t r = r0;
      for (; r + 4 <= r1; r += 4) {
        uint32_t x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = (uint32_t)__ldg(src + (r + j) * inner);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          run += x[j];
          dst[(r + j) * inner] = run;
        }
      }
      for (; r < r1; ++r) {
        run += (uint32_t)__ldg(src + r * inner);
        dst[r * inner] = run;
      }
    }
    __syncthreads();  // part reuse
  }
}

// out (cols x rows) = in (rows x cols)^T; 32x32 tile per CTA, 32x8 threads.
template <typename T>
__global__ void __launch_bounds__(256) k6_transpose(const T* __restrict__ in, int64_t rows,
                                                    int64_t cols, T* __restrict__ out) {
  __shared__ T tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int64_t r0 = (int64_t)blockIdx.y * 32; r0 < rows; r0 += (int64_t)gridDim.y * 32) {
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
      const int64_t r = r0 + ty + k, c = c0 + tx;
      if (r < rows && c < cols) tile[ty + k][tx] = in[r * cols + c];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
      const int64_t c = c0 + ty + k, r = r0 + tx;  // output row c, column r
      if (c < cols && r < rows) out[c * rows + r] = tile[tx][ty + k];
    }
    __syncthreads();  // tile reuse by the next row band
  }
}

}  // namespace ih
