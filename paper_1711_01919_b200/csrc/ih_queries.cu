// ih_queries.cu -- K3 batched region histograms and K4 window counts (sm_100a).
//
// K3 replaces core.py:179-195 region_histogram (one region per call there,
// a batch of Q regions here); K4 replaces likelihood.py:34-52 window_counts.
// Both are four-corner inclusion-exclusion over the bin-major (nb, H, W) u32
// tensor, computed in int64 exactly like the reference (core.py:184-194).
#include "ih_kernels.cuh"

namespace ih {

// Thread per (query, bin); bin fastest so the (Q, nb) u64 output is coalesced.
__global__ void __launch_bounds__(256) k3_region_histograms(const uint32_t* __restrict__ t, int nb,
                                                             int64_t H, int64_t W,
                                                             const int4* __restrict__ regions,
                                                             int64_t Q,
                                                             unsigned long long* __restrict__ out) {
  const int64_t total = Q * nb;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = i / nb;
    const int b = (int)(i % nb);
    const int4 rg = __ldg(regions + q);  // r0, c0, r1, c1 (inclusive)
    const uint32_t* p = t + (int64_t)b * H * W;
    const int64_t r0 = rg.x, c0 = rg.y, r1 = rg.z, c1 = rg.w;
    int64_t v = (int64_t)__ldg(p + r1 * W + c1);
    if (r0 > 0) v -= (int64_t)__ldg(p + (r0 - 1) * W + c1);
    if (c0 > 0) v -= (int64_t)__ldg(p + r1 * W + (c0 - 1));
    if (r0 > 0 && c0 > 0) v += (int64_t)__ldg(p + (r0 - 1) * W + (c0 - 1));
    out[i] = (unsigned long long)v;
  }
}

// Thread per output element (b, i, j), j fastest: the four corner rows are
// read coalesced; corners above row 0 / left of column 0 are zero
// (likelihood.py:44-51).
__global__ void __launch_bounds__(256) k4_window_counts(const uint32_t* __restrict__ t, int nb,
                                                         int64_t H, int64_t W, int h, int w,
                                                         long long* __restrict__ out) {
  const int64_t R = H - h + 1, C = W - w + 1;
  const int64_t total = (int64_t)nb * R * C;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = idx / (R * C);
    const int64_t rem = idx % (R * C);
    const int64_t i = rem / C, j = rem % C;
    const uint32_t* p = t + b * H * W;
    const int64_t rb = i + h - 1, cr = j + w - 1;
    long long v = (long long)__ldg(p + rb * W + cr);
    if (i > 0) v -= (long long)__ldg(p + (i - 1) * W + cr);
    if (j > 0) v -= (long long)__ldg(p + rb * W + (j - 1));
    if (i > 0 && j > 0) v += (long long)__ldg(p + (i - 1) * W + (j - 1));
    out[idx] = v;
  }
}

}  // namespace ih
