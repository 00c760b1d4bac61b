// ih_wavefront.cu -- K7: the wavefront tiled scan (WF-TiS) run as scheduled
// on the device, with a recorded event trace.
//
// Reference: compute_wavefront, strategies.py:172-216.  The image is cut into
// t x t tiles; tile (i, j) may start only after (i-1, j) and (i, j-1) have
// finished; each tile runs the fused recursion `_propagate` (strategies.py:
// 86-106) over all bins, reading the finished neighbours' border values.
// `trace` receives ("start"|"finish", i, j) events in the order they happened
// (strategies.py:194-208 appends them under a lock).
//
// The throughput path (K2, ih_single_pass.cu) replaces the wavefront with
// row-segment carries and has no tiles.  This kernel exists for callers that
// ask for the schedule itself: it executes the real dependency-driven
// wavefront and records the order of events with a global sequence counter
// (one atomicAdd per event, the device analog of the reference's lock).
//
//   * One CTA per tile.  Tiles are claimed through an atomic ticket in
//     anti-diagonal order, so every tile a CTA waits on was claimed earlier
//     by a running CTA (forward progress without co-residency assumptions).
//   * Thread 0 spins on the two predecessor flags (ld.acquire.gpu), takes the
//     "start" sequence number, and releases the CTA with a barrier.
//   * Warp w computes bins w, w + nwarps, ...: per tile row, a warp scan over
//     32-column pieces gives the in-tile row prefix; with
//       H(r, c) = H(r-1, c) + rowpref(r, c0..c) + [H(r, c0-1) - H(r-1, c0-1)]
//     every value depends only on the tile above / left / above-left (read
//     with ld.global.cg: written by other SMs) and this tile's previous row.
//   * __threadfence + barrier, then "finish" sequence number and
//     st.release.gpu of the tile flag.
// u32 modular arithmetic is exact: every count is <= W*H <= 2^32-1.
#include "ih_kernels.cuh"

namespace ih {

constexpr int kWfWarps = 8;

struct WfArgs {
  const uint8_t* img;
  int64_t H, W, pitch;
  int nb;            // bins
  int tile;          // t
  int64_t ni, nj;    // tile grid
  uint32_t* ticket;  // claim counter (zeroed by the host per launch)
  uint32_t* seq;     // event sequence counter (zeroed per launch)
  uint32_t* flags;   // per tile: 1 = finished (zeroed per launch)
  uint32_t* ev;      // per tile: {start seq, finish seq}
  uint32_t* out;     // (nb, H, W)
};

__device__ __forceinline__ uint32_t wf_ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wf_st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(kWfWarps * 32) k7_wavefront(WfArgs a, RelLut lut) {
  __shared__ uint8_t rel[256];
  __shared__ int64_t s_ij[2];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  for (int v = threadIdx.x; v < 256; v += blockDim.x) rel[v] = lut.rel[v];
  if (threadIdx.x == 0) {
    // ticket k -> the k-th tile in anti-diagonal order (diagonal d holds the
    // tiles i + j = d, i ascending: strategies.py:210-211)
    int64_t k = atomicAdd(a.ticket, 1u);
    int64_t d = 0;
    for (;; ++d) {
      const int64_t ilo = d - a.nj + 1 > 0 ? d - a.nj + 1 : 0;
      const int64_t ihi = d < a.ni - 1 ? d : a.ni - 1;
      const int64_t n = ihi - ilo + 1;
      if (k < n) {
        s_ij[0] = ilo + k;
        s_ij[1] = d - (ilo + k);
        break;
      }
      k -= n;
    }
    const int64_t i = s_ij[0], j = s_ij[1];
    if (i > 0)
      while (wf_ld_acquire(a.flags + (i - 1) * a.nj + j) == 0u) __nanosleep(32);
    if (j > 0)
      while (wf_ld_acquire(a.flags + i * a.nj + j - 1) == 0u) __nanosleep(32);
    a.ev[2 * (i * a.nj + j)] = atomicAdd(a.seq, 1u);  // "start"
  }
  __syncthreads();
  const int64_t i = s_ij[0], j = s_ij[1];
  const int64_t r0 = i * a.tile, r1 = min(r0 + a.tile, a.H);
  const int64_t c0 = j * a.tile, c1 = min(c0 + a.tile, a.W);
  const int64_t plane = a.H * a.W;
  for (int b = warp; b < a.nb; b += kWfWarps) {
    uint32_t* P = a.out + (int64_t)b * plane;
    for (int64_t r = r0; r < r1; ++r) {
      // left border difference H(r, c0-1) - H(r-1, c0-1) (0 at the image edge)
      uint32_t run = 0u;
      if (c0 > 0) {
        run = __ldcg(P + r * a.W + c0 - 1);
        if (r > 0) run -= __ldcg(P + (r - 1) * a.W + c0 - 1);
      }
      const uint8_t* row = a.img + r * a.pitch;
      for (int64_t cb = c0; cb < c1; cb += 32) {
        const int64_t c = cb + lane;
        const bool in = c < c1;
        const uint32_t hit = in && rel[row[in ? c : c0]] == (uint32_t)b ? 1u : 0u;
        uint32_t x = hit;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, x, d);
          if (lane >= d) x += y;
        }
        if (in) {
          // the row above: another tile's bottom row (r == r0) or this lane's
          // own store of the previous row
          const uint32_t up = r > 0 ? __ldcg(P + (r - 1) * a.W + c) : 0u;
          __stcg(P + r * a.W + c, up + run + x);
        }
        run += __shfl_sync(kFull, x, 31);
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    a.ev[2 * (i * a.nj + j) + 1] = atomicAdd(a.seq, 1u);  // "finish"
    __threadfence();
    wf_st_release(a.flags + i * a.nj + j, 1u);
  }
}

}  // namespace ih
