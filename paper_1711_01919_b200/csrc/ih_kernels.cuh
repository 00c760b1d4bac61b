// ih_kernels.cuh -- sm_100a kernels of the B200 integral-histogram engine.
//
// Reference algorithm (pkg/src/inthist/, read-only reference):
//   H_b(r,c) = #{ (r',c') : r'<=r, c'<=c, Q(I(r',c')) = b }    (core.py:1-7, :106-128)
// computed by the reference with four CPU strategies (strategies.py:86-229).
// All kernels below produce the identical bin-major (B,H,W) uint32 tensor.
//
// Notation used throughout:
//   chunk   = 128 consecutive columns = one warp-wide row piece, 4 pixels/lane
//   group   = 4 consecutive bins of the slab, packed one byte per bin in a u32
//   segment = S consecutive rows handled by one CTA of the single-pass kernel
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ih {

constexpr int kChunk = 128;       // columns per warp chunk
constexpr int kGroup = 4;         // bins per packed group
constexpr unsigned kFull = 0xffffffffu;

// Row segmentation of a frame: `nbig` segments of S rows, then segments of S2
// rows (S2 <= S: the short "tail" segments run last in the scan grid, which
// shortens the end of the last wave).  Uniform when nbig == nseg.
struct Segs {
  int S, nbig, S2;
  __host__ __device__ int64_t start(int64_t s) const {
    return s < nbig ? s * S : (int64_t)nbig * S + (s - nbig) * S2;
  }
};

// Per-call binning table: relative bin (lut[v] - bin_lo) or 0xFF when the
// bin lies outside the slab [bin_lo, bin_hi).  Passed by value (kernel param).
struct alignas(16) RelLut {  // 16-byte aligned: kernels copy it out as words
  uint8_t rel[256];
};

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t byte_of(uint32_t v, int i) {
  return __byte_perm(v, 0u, 0x4440u | (uint32_t)i);
}

// Inclusive warp scan; with packed operands every byte lane scans
// independently as long as no byte exceeds 255 (callers guarantee <=128).
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, x, d);
    if (lane >= d) x += y;
  }
  return x;
}

// Programmatic dependent launch (PDL).  A kernel launched with programmatic
// stream serialization may start while its predecessor in the stream still
// runs; griddep_wait() blocks until that predecessor has completed and its
// writes are visible (a no-op without the launch attribute).  Kernels of the
// prepare chain call griddep_launch_dependents() once they are running so the
// next kernel's prologue (TMA ring fill, one-hot table) overlaps their tail.
// Every PDL-launched kernel waits before it completes, so completion stays
// transitive along the chain.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Streaming (evict-first) 16-byte / 4-byte global stores: every output byte
// is written exactly once and never re-read by the producing kernel.
#ifndef IH_STORE_HINT
#define IH_STORE_HINT ".cs"
#endif
__device__ __forceinline__ void st_stream_v4(uint32_t* p, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.global" IH_STORE_HINT ".v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b),
               "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ void st_stream_v2(uint32_t* p, uint32_t a, uint32_t b) {
  asm volatile("st.global" IH_STORE_HINT ".v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(b)
               : "memory");
}
__device__ __forceinline__ void st_stream(uint32_t* p, uint32_t a) {
  asm volatile("st.global" IH_STORE_HINT ".u32 [%0], %1;" ::"l"(p), "r"(a) : "memory");
}

// Build the packed one-hot table of one bin group in shared memory:
// oh[v] = 1 << 8*(rel(v) - 4g) when rel(v) is in the group, else 0;
// oh[256..511] = 0 are the "column beyond the image edge" entries, indexed as
// (pixel | 256) so the edge mask costs one OR.
constexpr int kOneHotEntries = 512;
__device__ __forceinline__ void build_onehot(uint32_t* oh, const RelLut& lut, int g) {
  for (int v = threadIdx.x; v < kOneHotEntries; v += blockDim.x) {
    uint32_t word = 0;
    if (v < 256) {
      uint32_t d = (uint32_t)lut.rel[v] - (uint32_t)(g * kGroup);
      if (d < (uint32_t)kGroup) word = 1u << (8u * d);
    }
    oh[v] = word;
  }
}

// The same for a group of KB (1, 2 or 4) bins: byte d of the word counts bin
// g*KB + d (the row-packed K2 variants put further rows in the higher bytes).
template <int KB>
__device__ __forceinline__ void build_onehot_kb(uint32_t* oh, const RelLut& lut, int g) {
  for (int v = threadIdx.x; v < kOneHotEntries; v += blockDim.x) {
    uint32_t word = 0;
    if (v < 256) {
      uint32_t d = (uint32_t)lut.rel[v] - (uint32_t)(g * KB);
      if (d < (uint32_t)KB) word = 1u << (8u * d);
    }
    oh[v] = word;
  }
}

// Load the 4 pixels of one lane in one chunk row and return their 4 one-hot
// words through the table.  `inval` has bit 8 set for pixel slots at or
// beyond the right image edge (they map to oh[256 + byte] == 0).
template <bool ALIGNED>
__device__ __forceinline__ void load_onehot4(const uint8_t* row, int64_t c, int64_t W,
                                             const uint32_t* oh, const uint32_t inval[4],
                                             uint32_t out[4]) {
  uint32_t px = 0;
  if (c < W) {
    if (ALIGNED) {
      px = __ldg(reinterpret_cast<const uint32_t*>(row + c));
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (c + j < W) px |= (uint32_t)__ldg(row + c + j) << (8 * j);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) out[j] = oh[((px >> (8 * j)) & 0xffu) | inval[j]];
}

}  // namespace ih
