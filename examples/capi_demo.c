/*
 * capi_demo.c -- the C ABI (include/inthist_b200.h) from plain C, no Python,
 * no torch: what a non-Python host (a cgo / JNI / N-API binding, or a C++
 * service) does.  Computes the integral histogram of a synthetic 1920x1080
 * frame with 32 uniform bins, checks the invariant sum_b H_b(H-1, W-1) = H*W,
 * answers one region query and prints a crc-free digest.
 *
 *   make -C examples && ./examples/capi_demo
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "../include/inthist_b200.h"

#define CHECK_CUDA(x)                                                              \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
      return 1;                                                                    \
    }                                                                              \
  } while (0)
#define CHECK_IH(x)                                                                \
  do {                                                                             \
    ih_status s_ = (x);                                                            \
    if (s_ != IH_OK) {                                                             \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, ih_status_string(s_), \
              ih_last_error());                                                    \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

int main(void) {
  const int64_t H = 1080, W = 1920, pitch = 1920;
  const int32_t bins = 32;
  uint8_t lut[256];
  for (int v = 0; v < 256; ++v) lut[v] = (uint8_t)((v * bins) >> 8); /* BinSpec.uniform */

  uint8_t* h_img = (uint8_t*)malloc((size_t)H * W);
  uint32_t x = 12345u;
  for (int64_t i = 0; i < H * W; ++i) { /* xorshift pixels */
    x ^= x << 13; x ^= x >> 17; x ^= x << 5;
    h_img[i] = (uint8_t)x;
  }
  uint8_t* d_img;
  uint32_t* d_out;
  CHECK_CUDA(cudaMalloc((void**)&d_img, (size_t)H * pitch));
  CHECK_CUDA(cudaMalloc((void**)&d_out, (size_t)bins * H * W * sizeof(uint32_t)));
  CHECK_CUDA(cudaMemcpy(d_img, h_img, (size_t)H * W, cudaMemcpyHostToDevice));

  const size_t ws_bytes = ih_workspace_bytes(1, H, W, bins, IH_KERNEL_AUTO);
  void* d_ws = NULL;
  if (ws_bytes) CHECK_CUDA(cudaMalloc(&d_ws, ws_bytes));
  cudaStream_t stream;
  CHECK_CUDA(cudaStreamCreate(&stream));

  CHECK_IH(ih_integral_histogram(d_img, 1, H, W, pitch, H * pitch, lut, bins, 0, bins, d_out,
                                 d_ws, ws_bytes, IH_KERNEL_AUTO, (void*)stream));

  /* one region query: the whole image -> per-bin totals (u64) */
  int32_t h_reg[4] = {0, 0, (int32_t)H - 1, (int32_t)W - 1};
  int32_t* d_reg;
  uint64_t* d_hist;
  CHECK_CUDA(cudaMalloc((void**)&d_reg, 16));
  CHECK_CUDA(cudaMalloc((void**)&d_hist, bins * sizeof(uint64_t)));
  CHECK_CUDA(cudaMemcpy(d_reg, h_reg, 16, cudaMemcpyHostToDevice));
  CHECK_IH(ih_region_histograms(d_out, bins, H, W, d_reg, 1, d_hist, (void*)stream));
  uint64_t h_hist[32];
  CHECK_CUDA(cudaMemcpyAsync(h_hist, d_hist, sizeof h_hist, cudaMemcpyDeviceToHost, stream));
  CHECK_CUDA(cudaStreamSynchronize(stream));

  /* host recount of the bin totals */
  uint64_t want[32] = {0};
  for (int64_t i = 0; i < H * W; ++i) want[lut[h_img[i]]]++;
  uint64_t total = 0;
  for (int b = 0; b < bins; ++b) {
    if (h_hist[b] != want[b]) {
      fprintf(stderr, "bin %d: %llu != %llu\n", b, (unsigned long long)h_hist[b],
              (unsigned long long)want[b]);
      return 1;
    }
    total += h_hist[b];
  }
  if (total != (uint64_t)(H * W)) return 1;
  printf("capi_demo ok: %lldx%lld x%d bins, abi %d.%d, workspace %zu bytes, total %llu\n",
         (long long)W, (long long)H, bins, ih_abi_version() >> 16, ih_abi_version() & 0xffff,
         ws_bytes, (unsigned long long)total);
  cudaFree(d_img); cudaFree(d_out); cudaFree(d_ws); cudaFree(d_reg); cudaFree(d_hist);
  cudaStreamDestroy(stream);
  free(h_img);
  return 0;
}
