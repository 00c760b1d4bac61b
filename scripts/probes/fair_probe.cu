// Fairness probe: do two co-resident 15-warp CTAs progress equally (they do
// not: the older CTA is favoured), and do the two halves of ONE 30-warp CTA
// (named barriers per half) progress equally?  Each unit of work = R-row
// batches of 4-plane 16-byte stores with a barrier per batch, like k2_scan.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void st_cs(uint32_t* p, uint32_t a) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %1, %1, %1};" ::"l"(p), "r"(a) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// unit u: planes 4u..4u+3, rows [0, S) of an H x W plane set
__device__ void do_unit(uint32_t* out, int u, int S, int W, int64_t plane, int lt, int bar, int nthr) {
  const int lane = lt & 31, warp = lt >> 5;
  uint32_t* base = out + (int64_t)u * 4 * plane + warp * 128 + lane * 4;
  uint32_t x = u;
  for (int r = 0; r < S; r += 4) {
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      // a little ALU work per row, like the scan
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) x += __shfl_up_sync(0xffffffffu, x, d);
#pragma unroll
      for (int i = 0; i < 4; ++i) st_cs(base + i * plane + (int64_t)(r + rr) * W, x + i);
    }
    if (bar == 0) __syncthreads(); else named_sync(bar, nthr);
  }
}

__global__ void __launch_bounds__(480) two_ctas(uint32_t* out, int S, int W, int64_t plane, unsigned long long* tr) {
  const unsigned long long t0 = gt();
  do_unit(out, blockIdx.x, S, W, plane, threadIdx.x, 0, 480);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    tr[3 * blockIdx.x] = t0; tr[3 * blockIdx.x + 1] = gt(); tr[3 * blockIdx.x + 2] = smid;
  }
}
__global__ void __launch_bounds__(960) one_cta_two_halves(uint32_t* out, int S, int W, int64_t plane, unsigned long long* tr) {
  const int half = threadIdx.x / 480, lt = threadIdx.x % 480;
  const int u = 2 * blockIdx.x + half;
  const unsigned long long t0 = gt();
  do_unit(out, u, S, W, plane, lt, 1 + half, 480);
  named_sync(1 + half, 480);
  if (lt == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    tr[3 * u] = t0; tr[3 * u + 1] = gt(); tr[3 * u + 2] = smid;
  }
}

int main() {
  const int W = 1920, S = 240, units = 296;  // one wave of 2 x 148 units
  const int64_t plane = (int64_t)S * W;
  uint32_t* out;
  unsigned long long* tr;
  cudaMalloc(&out, (size_t)units * 4 * plane * 4);
  cudaMalloc(&tr, units * 3 * 8);
  unsigned long long h[units * 3];
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      if (mode == 0) two_ctas<<<units, 480>>>(out, S, W, plane, tr);
      else one_cta_two_halves<<<units / 2, 960>>>(out, S, W, plane, tr);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, tr, sizeof h, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, tmax = 0;
    for (int i = 0; i < units; ++i) { if (h[3 * i] < t0) t0 = h[3 * i]; if (h[3 * i + 1] > tmax) tmax = h[3 * i + 1]; }
    double lmin = 1e30, lmax = 0, lsum = 0;
    for (int i = 0; i < units; ++i) { double l = (h[3 * i + 1] - h[3 * i]) / 1e3; lmin = l < lmin ? l : lmin; lmax = l > lmax ? l : lmax; lsum += l; }
    printf("{\"mode\": \"%s\", \"span_us\": %.1f, \"life_min\": %.1f, \"life_mean\": %.1f, \"life_max\": %.1f, \"gbs\": %.1f}\n",
           mode == 0 ? "two_ctas_per_sm" : "one_cta_two_halves", (tmax - t0) / 1e3, lmin, lsum / units, lmax,
           (double)units * 4 * plane * 4 / ((tmax - t0) / 1e9) / 1e9);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
