// Write-bandwidth probe: which store patterns reach the ~7.5 TB/s write-only
// ceiling (memset) on B200, versus the K2 output pattern (CTA = 4 bin planes x
// a segment of rows x full width, 16-byte evict-first stores).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda.h>

__device__ __forceinline__ void st_cs(uint32_t* p, uint32_t a) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %1, %1, %1};" ::"l"(p), "r"(a) : "memory");
}
__device__ __forceinline__ void st_wb(uint32_t* p, uint32_t a) {
  asm volatile("st.global.v4.u32 [%0], {%1, %1, %1, %1};" ::"l"(p), "r"(a) : "memory");
}

__device__ __forceinline__ void st_v8(uint32_t* p, uint32_t a) {
  asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(a) : "memory");
}
__global__ void linear_v8(uint32_t* out, size_t n32) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n32; i += (size_t)gridDim.x * blockDim.x)
    st_v8(out + 8 * i, 7u);
}
// K2-like with 32-byte stores: lane owns 8 columns of NP planes
template <int NP>
__global__ void k2like_v8(uint32_t* out, int H, int W, int nb, int S) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = blockIdx.x, s = blockIdx.y, f = blockIdx.z;
  const int64_t plane = (int64_t)H * W;
  const int c = warp * 256 + lane * 8;
  if (c >= W) return;
  uint32_t* base = out + ((int64_t)f * nb + g * NP) * plane + c;
  const int r0 = s * S, r1 = min(r0 + S, H);
  for (int r = r0; r < r1; ++r) {
#pragma unroll
    for (int i = 0; i < NP; ++i) st_v8(base + i * plane + (int64_t)r * W, r);
  }
}
// TMA bulk store: each CTA stages one row of NP planes in smem and bulk-copies
// them out (thread 0 issues, bulk_group completion), double-buffered.
template <int NP>
__global__ void k2like_tma(uint32_t* out, int H, int W, int nb, int S) {
  extern __shared__ __align__(128) uint32_t srow[];  // [2][NP][W]
  const int g = blockIdx.x, s = blockIdx.y, f = blockIdx.z;
  const int64_t plane = (int64_t)H * W;
  uint32_t* base = out + ((int64_t)f * nb + g * NP) * plane;
  const int r0 = s * S, r1 = min(r0 + S, H);
  for (int r = r0; r < r1; ++r) {
    uint32_t* buf = srow + ((r - r0) & 1) * NP * W;
    if (threadIdx.x == 0)  // the buffer written 2 rows ago must have been read by the TMA
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    for (int i = threadIdx.x * 4; i < NP * W; i += blockDim.x * 4)
      *reinterpret_cast<uint4*>(buf + i) = make_uint4(r, r, r, r);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < NP; ++i)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(base + i * plane + (int64_t)r * W),
                     "r"((uint32_t)__cvta_generic_to_shared(buf + i * W)), "r"((uint32_t)(W * 4)) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// per-warp TMA bulk stores: each warp stages its 128 columns of NP planes for a
// row (512 B per plane) and lane 0 bulk-copies them; NB buffers per warp
template <int NP, int NB>
__global__ void k2like_tma_warp(uint32_t* out, int H, int W, int nb, int S) {
  extern __shared__ __align__(128) uint32_t sw[];  // [warp][NB][NP][128]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = blockIdx.x, s = blockIdx.y, f = blockIdx.z;
  const int64_t plane = (int64_t)H * W;
  uint32_t* base = out + ((int64_t)f * nb + g * NP) * plane + warp * 128;
  uint32_t* mine = sw + warp * NB * NP * 128;
  const int r0 = s * S, r1 = min(r0 + S, H);
  for (int r = r0; r < r1; ++r) {
    uint32_t* buf = mine + ((r - r0) % NB) * NP * 128;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NB - 1) : "memory");
    __syncwarp();
#pragma unroll
    for (int i = 0; i < NP; ++i) *reinterpret_cast<uint4*>(buf + i * 128 + lane * 4) = make_uint4(r, r, r, r);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < NP; ++i)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" ::"l"(base + i * plane + (int64_t)r * W),
                     "r"((uint32_t)__cvta_generic_to_shared(buf + i * 128)) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// K2-like, batches of RB rows written plane by plane (bin-outer, row-inner)
template <int NP, int RB>
__global__ void k2like_planeorder(uint32_t* out, int H, int W, int nb, int S) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = blockIdx.x, s = blockIdx.y, f = blockIdx.z;
  const int64_t plane = (int64_t)H * W;
  uint32_t* base = out + ((int64_t)f * nb + g * NP) * plane + warp * 128 + lane * 4;
  const int r0 = s * S, r1 = min(r0 + S, H);
  for (int r = r0; r < r1; r += RB) {
#pragma unroll
    for (int i = 0; i < NP; ++i)
#pragma unroll
      for (int rr = 0; rr < RB; ++rr)
        if (r + rr < r1) st_cs(base + i * plane + (int64_t)(r + rr) * W, r);
  }
}


// 2-D tensor-map TMA stores (cp.async.bulk.tensor -> UTMASTG): the output is
// viewed as a [F*nb*H][W] u32 matrix; a CTA stages R rows of its NP planes in
// shared memory as [plane][box][R][BOXW] tiles (box width <= 256 elements)
// and thread 0 stores each tile with one tensor copy, NBUF-buffered.
template <int NP, int R, int BOXW, int NBUF>
__global__ void k2like_tmap(const __grid_constant__ CUtensorMap tm, int H, int W, int nb, int S) {
  extern __shared__ __align__(1024) uint32_t st[];  // [NBUF][NP][nbox][TS]
  constexpr int TS = (R * BOXW + 31) / 32 * 32;    // tile stride: 128-byte aligned tiles
  const int g = blockIdx.x, s = blockIdx.y, f = blockIdx.z;
  const int nbox = W / BOXW, per = NP * nbox * TS;
  const int r0 = s * S, r1 = min(r0 + S, H);
  for (int r = r0, k = 0; r < r1; r += R, ++k) {
    uint32_t* buf = st + (k % NBUF) * per;
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NBUF - 1) : "memory");
    __syncthreads();
    for (int i = threadIdx.x * 4; i < per; i += blockDim.x * 4)
      *reinterpret_cast<uint4*>(buf + i) = make_uint4(r, r, r, r);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < NP; ++i)
        for (int bx = 0; bx < nbox; ++bx) {
          const int y = (int)(((int64_t)f * nb + g * NP + i) * H + r), x = bx * BOXW;
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tm),
              "r"(x), "r"(y), "r"((uint32_t)__cvta_generic_to_shared(buf + (i * nbox + bx) * TS))
              : "memory");
        }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <bool CS>
__global__ void linear(uint32_t* out, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    CS ? st_cs(out + 4 * i, 7u) : st_wb(out + 4 * i, 7u);
}

// K2-like: grid (groups, segments, frames); 15 warps x 128 columns; per row,
// each lane stores 16 B into each of NP planes (bins) of its group.
template <bool CS, int NP>
__global__ void k2like(uint32_t* out, int H, int W, int nb, int S) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = blockIdx.x, s = blockIdx.y, f = blockIdx.z;
  const int64_t plane = (int64_t)H * W;
  uint32_t* base = out + ((int64_t)f * nb + g * NP) * plane + warp * 128 + lane * 4;
  const int r0 = s * S, r1 = min(r0 + S, H);
  for (int r = r0; r < r1; ++r) {
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      uint32_t* p = base + i * plane + (int64_t)r * W;
      CS ? st_cs(p, r) : st_wb(p, r);
    }
  }
}

int main(int argc, char** argv) {
  const int H = 1080, W = 1920, nb = 32, F = 64;
  const size_t elems = (size_t)F * nb * H * W;
  uint32_t* out;
  cudaMalloc(&out, elems * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    printf("{\"probe\": \"%s\", \"ms\": %.4f, \"gbs\": %.1f}\n", name, ms, elems * 4 / ms / 1e6);
  };
  timeit("memset", [&] { cudaMemsetAsync(out, 0, elems * 4); });
  // 2-D tensor-map TMA stores of staged [R x 240] tiles, against K2's 16-byte
  // stores and 1-D bulk row copies above (same grid and segments)
  {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)F * nb * H};
    cuuint64_t strides[1] = {(cuuint64_t)W * 4};
    cuuint32_t box[2] = {240, 1}, estr[2] = {1, 1};
    auto enc = [&](int rows) {
      box[1] = rows;
      CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, out, dims, strides, box, estr,
                                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS) printf("{\"error\": \"cuTensorMapEncodeTiled %d\"}\n", (int)cr);
    };
    for (int nseg : {5, 9}) {
      const int S = (H + nseg - 1) / nseg;
      char nm[64];
      enc(1);
      {
        const int sm = 2 * 4 * 8 * 256 * 4;
        cudaFuncSetAttribute(k2like_tmap<4, 1, 240, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        snprintf(nm, sizeof nm, "k2like_tmap2d_np4_r1_nbuf2_nseg%d", nseg);
        timeit(nm, [&] { k2like_tmap<4, 1, 240, 2><<<dim3(nb / 4, nseg, F), 480, sm>>>(tm, H, W, nb, S); });
      }
      enc(2);
      {
        const int sm = 2 * 2 * 2 * W * 4;
        cudaFuncSetAttribute(k2like_tmap<2, 2, 240, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        snprintf(nm, sizeof nm, "k2like_tmap2d_np2_r2_nbuf2_nseg%d", nseg);
        timeit(nm, [&] { k2like_tmap<2, 2, 240, 2><<<dim3(nb / 2, nseg, F), 480, sm>>>(tm, H, W, nb, S); });
      }
      enc(4);
      {
        const int sm = 4 * 4 * W * 4;
        cudaFuncSetAttribute(k2like_tmap<4, 4, 240, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        snprintf(nm, sizeof nm, "k2like_tmap2d_np4_r4_nbuf1_nseg%d", nseg);
        timeit(nm, [&] { k2like_tmap<4, 4, 240, 1><<<dim3(nb / 4, nseg, F), 480, sm>>>(tm, H, W, nb, S); });
      }
      // K2's own pattern for comparison in the same run
      snprintf(nm, sizeof nm, "k2like_cs_np4_nseg%d_ref", nseg);
      timeit(nm, [&] { k2like<true, 4><<<dim3(nb / 4, nseg, F), 480>>>(out, H, W, nb, S); });
      snprintf(nm, sizeof nm, "k2like_tma_np4_nseg%d_ref", nseg);
      cudaFuncSetAttribute(k2like_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 4 * W * 4);
      timeit(nm, [&] { k2like_tma<4><<<dim3(nb / 4, nseg, F), 480, 2 * 4 * W * 4>>>(out, H, W, nb, S); });
    }
  }
  if (argc > 1) {  // "tmap": only the tensor-map section
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
  }
  timeit("linear_cs", [&] { linear<true><<<148 * 8, 256>>>(out, elems / 4); });
  timeit("linear_wb", [&] { linear<false><<<148 * 8, 256>>>(out, elems / 4); });
  timeit("linear_v8", [&] { linear_v8<<<148 * 8, 256>>>(out, elems / 8); });
  for (int nseg : {5, 9}) {
    const int S = (H + nseg - 1) / nseg;
    char nm[64];
    snprintf(nm, sizeof nm, "k2like_v8_np4_nseg%d", nseg);
    timeit(nm, [&] { k2like_v8<4><<<dim3(nb / 4, nseg, F), 256>>>(out, H, W, nb, S); });
    snprintf(nm, sizeof nm, "k2like_tma_np4_nseg%d", nseg);
    cudaFuncSetAttribute(k2like_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 4 * W * 4);
    timeit(nm, [&] { k2like_tma<4><<<dim3(nb / 4, nseg, F), 480, 2 * 4 * W * 4>>>(out, H, W, nb, S); });
  }
  for (int nseg : {5, 9}) {
    const int S = (H + nseg - 1) / nseg;
    char nm[64];
    snprintf(nm, sizeof nm, "k2like_tmawarp_nb2_nseg%d", nseg);
    cudaFuncSetAttribute(k2like_tma_warp<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 15 * 2 * 4 * 512);
    timeit(nm, [&] { k2like_tma_warp<4, 2><<<dim3(nb / 4, nseg, F), 480, 15 * 2 * 4 * 512>>>(out, H, W, nb, S); });
    snprintf(nm, sizeof nm, "k2like_tmawarp_nb4_nseg%d", nseg);
    cudaFuncSetAttribute(k2like_tma_warp<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 15 * 4 * 4 * 512);
    timeit(nm, [&] { k2like_tma_warp<4, 4><<<dim3(nb / 4, nseg, F), 480, 15 * 4 * 4 * 512>>>(out, H, W, nb, S); });
  }
  for (int nseg : {5, 9}) {
    const int S = (H + nseg - 1) / nseg;
    char nm[64];
    snprintf(nm, sizeof nm, "k2like_planeorder_rb4_nseg%d", nseg);
    timeit(nm, [&] { k2like_planeorder<4, 4><<<dim3(nb / 4, nseg, F), 480>>>(out, H, W, nb, S); });
    snprintf(nm, sizeof nm, "k2like_planeorder_rb8_nseg%d", nseg);
    timeit(nm, [&] { k2like_planeorder<4, 8><<<dim3(nb / 4, nseg, F), 480>>>(out, H, W, nb, S); });
  }
  for (int nseg : {3, 5, 9}) {
    const int S = (H + nseg - 1) / nseg;
    char nm[64];
    snprintf(nm, sizeof nm, "k2like_cs_np4_nseg%d", nseg);
    timeit(nm, [&] { k2like<true, 4><<<dim3(nb / 4, nseg, F), 480>>>(out, H, W, nb, S); });
    snprintf(nm, sizeof nm, "k2like_wb_np4_nseg%d", nseg);
    timeit(nm, [&] { k2like<false, 4><<<dim3(nb / 4, nseg, F), 480>>>(out, H, W, nb, S); });
    snprintf(nm, sizeof nm, "k2like_cs_np1_nseg%d", nseg);
    timeit(nm, [&] { k2like<true, 1><<<dim3(nb, nseg, F), 480>>>(out, H, W, nb, S); });
  }
  // occupancy-matched to k2_scan (2 CTAs of 15 warps per SM): a dummy dynamic
  // shared-memory request of 100 KB per CTA
  cudaFuncSetAttribute(k2like<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 << 10);
  cudaFuncSetAttribute(k2like_planeorder<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 << 10);
  cudaFuncSetAttribute(k2like_planeorder<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 << 10);
  cudaFuncSetAttribute(k2like<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 << 10);
  for (int nseg : {5, 9}) {
    const int S = (H + nseg - 1) / nseg;
    char nm[64];
    snprintf(nm, sizeof nm, "occ2_k2like_cs_np4_nseg%d", nseg);
    timeit(nm, [&] { k2like<true, 4><<<dim3(nb / 4, nseg, F), 480, 100 << 10>>>(out, H, W, nb, S); });
    snprintf(nm, sizeof nm, "occ2_planeorder_rb2_nseg%d", nseg);
    timeit(nm, [&] { k2like_planeorder<4, 2><<<dim3(nb / 4, nseg, F), 480, 100 << 10>>>(out, H, W, nb, S); });
    snprintf(nm, sizeof nm, "occ2_planeorder_rb4_nseg%d", nseg);
    timeit(nm, [&] { k2like_planeorder<4, 4><<<dim3(nb / 4, nseg, F), 480, 100 << 10>>>(out, H, W, nb, S); });
    snprintf(nm, sizeof nm, "occ2_k2like_cs_np1_nseg%d", nseg);
    timeit(nm, [&] { k2like<true, 1><<<dim3(nb, nseg, F), 480, 100 << 10>>>(out, H, W, nb, S); });
  }
  // lone CTAs: one 480-thread CTA per SM (148 CTAs, a 100 KB dummy smem request
  // keeps a second one off the SM) writing K2's store pattern: the per-SM
  // store rate a single k2_scan CTA could reach if it did nothing else
  {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(k2like<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
    for (int smem_kb : {200, 100}) {  // 200 KB: one CTA per SM; 100 KB: two
      const int nseg = (sms + 7) / 8;  // 8 groups x nseg segments ~ one CTA per SM
      const int S = (H + nseg - 1) / nseg;
      char nm[64];
      snprintf(nm, sizeof nm, "lone_k2like_np4_smem%dKB_ctas%d", smem_kb, 8 * nseg);
      timeit(nm, [&] { k2like<true, 4><<<dim3(nb / 4, nseg, 1), 480, (size_t)smem_kb << 10>>>(out, H, W, nb, S); });
    }
    // the same lone CTAs with 32-byte stores (240 threads: 8 columns per lane)
    // and with whole-row TMA bulk stores staged in shared memory
    const int nseg = (sms + 7) / 8;
    const int S = (H + nseg - 1) / nseg;
    cudaFuncSetAttribute(k2like_v8<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
    timeit("lone_k2like_v8_np4", [&] { k2like_v8<4><<<dim3(nb / 4, nseg, 1), 256, 200 << 10>>>(out, H, W, nb, S); });
    cudaFuncSetAttribute(k2like_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
    timeit("lone_k2like_tma_np4", [&] { k2like_tma<4><<<dim3(nb / 4, nseg, 1), 480, 200 << 10>>>(out, H, W, nb, S); });
    const double lone_bytes = (double)nb * H * W * 4;
    printf("{\"note\": \"lone_* lines write one frame (%.0f MB): GB/s = that / ms; the gbs field assumes the whole buffer\"}\n", lone_bytes / 1e6);
  }
  // cfg1 shape (512 x 512 x 32 bins, one frame, 33.5 MB): pure stores with
  // the K2 pattern, timed as 20 back-to-back launches rotating over 8 output
  // buffers (268 MB > L2, like bench.py --workload 512) and over one buffer
  // (L2-resident, like scripts/graph_time.py)
  {
    const int h = 512, w = 512, b = 32;
    const size_t one = (size_t)b * h * w;
    for (int nbuf : {1, 8}) {
      for (int nseg : {8, 16, 32, 64}) {
        const int S = (h + nseg - 1) / nseg;
        const int wpc = w / 128;  // warps per CTA
        cudaEventRecord(e0);
        for (int i = 0; i < 20; ++i)
          k2like<true, 4><<<dim3(b / 4, nseg, 1), wpc * 32>>>(out + (i % nbuf) * one, h, w, b, S);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"probe\": \"cfg1_k2like_np4_nseg%d_bufs%d\", \"us_per_launch\": %.2f, \"gbs\": %.1f}\n",
               nseg, nbuf, ms * 1000 / 20, one * 4 * 20 / ms / 1e6);
      }
    }
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) cudaMemsetAsync(out + (i % 8) * one, 0, one * 4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"probe\": \"cfg1_memset_bufs8\", \"us_per_launch\": %.2f}\n", ms * 1000 / 20);
  }

  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
