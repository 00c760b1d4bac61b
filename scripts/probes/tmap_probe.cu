// Minimal 2-D tensor-map TMA store check: one CTA stores a [rows x boxw] u32
// tile from shared memory; the host checks the values.  Usage: tmap_probe BOXW ROWS
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include <cuda.h>

__global__ void store_tile(const __grid_constant__ CUtensorMap tm, int boxw, int rows) {
  extern __shared__ __align__(1024) uint32_t tile[];
  for (int i = threadIdx.x; i < boxw * rows; i += blockDim.x) tile[i] = 1000000u + i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tm),
                 "r"(boxw), "r"(1), "r"((uint32_t)__cvta_generic_to_shared(tile))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main(int argc, char** argv) {
  const int boxw = argc > 1 ? atoi(argv[1]) : 32, rows = argc > 2 ? atoi(argv[2]) : 1;
  const int W = 1920, H = 64;
  uint32_t* out;
  cudaMalloc(&out, (size_t)W * H * 4);
  cudaMemset(out, 0, (size_t)W * H * 4);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
  cuuint64_t strides[1] = {(cuuint64_t)W * 4};
  cuuint32_t box[2] = {(cuuint32_t)boxw, (cuuint32_t)rows}, estr[2] = {1, 1};
  CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, out, dims, strides, box, estr,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode boxw=%d rows=%d -> %d\n", boxw, rows, (int)cr);
  cudaFuncSetAttribute(store_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
  store_tile<<<1, 128, 64 << 10>>>(tm, boxw, rows);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel -> %s\n", cudaGetErrorString(e));
  std::vector<uint32_t> h((size_t)W * H);
  cudaMemcpy(h.data(), out, h.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < boxw; ++c)
      if (h[(size_t)(1 + r) * W + boxw + c] != 1000000u + r * boxw + c) ++bad;
  printf("mismatches %d of %d\n", bad, rows * boxw);
  return 0;
}
