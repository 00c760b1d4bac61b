// Random-gather ceiling probe for K3 (batched region histograms).
//
// K3 on the 8192^2 x 256 tensor (68.7 GB) with Q = 65,536 regions issues
// Q * 256 * 4 = 67.1 M isolated 4-byte reads.  This probe times the same
// number of 4-byte reads over the same footprint with patterns of decreasing
// structure, so K3's time can be stated as a fraction of what random reads
// of that footprint can do on this B200:
//   k3like_u{4,8}   K3's own access structure (warp per region, lanes over
//                   bins, 4 corners per plane), U bins of loads in flight
//   rand_{hint}_u{U} uniformly random 4-byte addresses over the footprint,
//                   U loads in flight per thread, L2 fetch-size hint
//                   none / 64B / 128B / 256B
// Output: one JSON line per probe (ms, reads/s, 64-byte-granule GB/s).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t mix(uint64_t x) {  // splitmix64
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

template <int HINT>
__device__ __forceinline__ uint32_t ld(const uint32_t* p) {
  uint32_t v;
  if (HINT == 64)
    asm volatile("ld.global.nc.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p));
  else if (HINT == 128)
    asm volatile("ld.global.nc.L2::128B.u32 %0, [%1];" : "=r"(v) : "l"(p));
  else if (HINT == 256)
    asm volatile("ld.global.nc.L2::256B.u32 %0, [%1];" : "=r"(v) : "l"(p));
  else
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// uniformly random reads: thread i does `per` reads, U in flight
template <int HINT, int U>
__global__ void __launch_bounds__(256) rand_reads(const uint32_t* t, uint64_t n_elems, int64_t total,
                                                  int per, uint32_t* sink) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (int k = 0; k < per; k += U) {
    uint32_t v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = tid * per + k + u;
      v[u] = i < total ? ld<HINT>(t + mix((uint64_t)i) % n_elems) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// K3's structure: warp per region, lanes over bins, 4 corners per plane
template <int U>
__global__ void __launch_bounds__(256) k3like(const uint32_t* t, int nb, int64_t H, int64_t W,
                                              const int4* regs, int64_t Q, unsigned long long* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t plane = H * W;
  for (int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < Q; q += warps) {
    const int4 rg = regs[q];
    const int64_t r0 = rg.x, c0 = rg.y, r1 = rg.z, c1 = rg.w;
    const bool top = r0 > 0, left = c0 > 0;
    const int64_t o11 = r1 * W + c1, o01 = top ? (r0 - 1) * W + c1 : 0;
    const int64_t o10 = left ? r1 * W + (c0 - 1) : 0, o00 = top && left ? (r0 - 1) * W + (c0 - 1) : 0;
    for (int b0 = 0; b0 < nb; b0 += 32 * U) {
      uint32_t v[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t* p = t + (int64_t)(b0 + u * 32 + lane) * plane;
        v[u][0] = ld<64>(p + o11);
        v[u][1] = top ? ld<64>(p + o01) : 0u;
        v[u][2] = left ? ld<64>(p + o10) : 0u;
        v[u][3] = top && left ? ld<64>(p + o00) : 0u;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        out[q * nb + b0 + u * 32 + lane] =
            (unsigned long long)((int64_t)v[u][0] - v[u][1] - v[u][2] + (int64_t)v[u][3]);
    }
  }
}

__global__ void make_regions(int4* regs, int64_t Q, int H, int W) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= Q) return;
  const uint64_t a = mix(4 * q), b = mix(4 * q + 1), c = mix(4 * q + 2), d = mix(4 * q + 3);
  int ra = (int)(a % H), rb = (int)(b % H), ca = (int)(c % W), cb = (int)(d % W);
  regs[q] = make_int4(min(ra, rb), min(ca, cb), max(ra, rb), max(ca, cb));
}

int main() {
  const int64_t H = 8192, W = 8192, NB = 256, Q = 65536;
  const uint64_t n = (uint64_t)NB * H * W;  // 68.7 GB of u32
  uint32_t* t = nullptr;
  if (cudaMalloc(&t, n * 4) != cudaSuccess) {
    printf("{\"error\": \"cudaMalloc %.1f GB failed\"}\n", n * 4 / 1e9);
    return 1;
  }
  cudaMemset(t, 1, n * 4);
  int4* regs;
  unsigned long long* out;
  uint32_t* sink;
  cudaMalloc(&regs, Q * sizeof(int4));
  cudaMalloc(&out, Q * NB * 8);
  cudaMalloc(&sink, 4);
  make_regions<<<(Q + 255) / 256, 256>>>(regs, Q, (int)H, (int)W);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int64_t reads = Q * NB * 4;
  auto time = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    const int reps = 10;
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("{\"probe\": \"%s\", \"ms\": %.4f, \"Greads_s\": %.2f, \"gbs_64B\": %.1f, \"err\": \"%s\"}\n",
           name, ms, reads / ms / 1e6, reads * 64.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
  };
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cps : {16, 64}) {
    char nm[64];
    snprintf(nm, sizeof nm, "k3like_u4_cps%d", cps);
    time(nm, [&] { k3like<4><<<(unsigned)std::min<int64_t>(Q / 8, (int64_t)sms * cps), 256>>>(t, (int)NB, H, W, regs, Q, out); });
    snprintf(nm, sizeof nm, "k3like_u8_cps%d", cps);
    time(nm, [&] { k3like<8><<<(unsigned)std::min<int64_t>(Q / 8, (int64_t)sms * cps), 256>>>(t, (int)NB, H, W, regs, Q, out); });
  }
  // uniformly random: `per` reads per thread over a grid of sms * 8 CTAs x 256 threads
  const int64_t threads = (int64_t)sms * 8 * 256;
  const int per = (int)((reads + threads - 1) / threads);
  const unsigned blocks = (unsigned)(sms * 8);
  time("rand_none_u16", [&] { rand_reads<0, 16><<<blocks, 256>>>(t, n, reads, per, sink); });
  time("rand_64B_u4", [&] { rand_reads<64, 4><<<blocks, 256>>>(t, n, reads, per, sink); });
  time("rand_64B_u16", [&] { rand_reads<64, 16><<<blocks, 256>>>(t, n, reads, per, sink); });
  time("rand_64B_u32", [&] { rand_reads<64, 32><<<blocks, 256>>>(t, n, reads, per, sink); });
  time("rand_128B_u16", [&] { rand_reads<128, 16><<<blocks, 256>>>(t, n, reads, per, sink); });
  time("rand_256B_u16", [&] { rand_reads<256, 16><<<blocks, 256>>>(t, n, reads, per, sink); });
  // random reads confined to a 32-plane slab (one 8-way shard, 8.6 GB)
  time("rand_64B_u16_slab32", [&] { rand_reads<64, 16><<<blocks, 256>>>(t, n / 8, reads, per, sink); });
  return 0;
}
