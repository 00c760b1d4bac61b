// ih_queries.cu -- K3 batched region histograms and K4 window counts (sm_100a).
//
// K3 replaces core.py:179-195 region_histogram (one region per call there,
// a batch of Q regions here); K4 replaces likelihood.py:34-52 window_counts.
// Both are four-corner inclusion-exclusion over the bin-major (nb, H, W) u32
// tensor, computed in int64 exactly like the reference (core.py:184-194).
#include "ih_kernels.cuh"

namespace ih {

// A 32-bit read-only load whose L2 miss fetches 64 bytes from DRAM (instead
// of the default 128): K3's corner reads are isolated, so half of a 128-byte
// fetch is waste.  Measured (ncu, 65,536 regions x 32 bins): DRAM reads
// 1.06 -> 0.53 GB per launch, time unchanged at 0.19 ms -- the gathers are
// bound by request rate / latency, not by DRAM bandwidth.
__device__ __forceinline__ uint32_t ldg_l2_64(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// K3: one warp per query (grid-stride over queries), lanes over bins: the
// (Q, nb) u64 output row of a query is written coalesced, and each lane keeps
// 4 corners x 4 bins = 16 independent gathers in flight (the reads are random
// by nature: 4 corners per bin plane, planes H*W*4 bytes apart).
__global__ void __launch_bounds__(256) k3_region_histograms(const uint32_t* __restrict__ t, int nb,
                                                             int64_t H, int64_t W,
                                                             const int4* __restrict__ regions,
                                                             int64_t Q,
                                                             unsigned long long* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t plane = H * W;
  for (int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < Q;
       q += warps) {
    const int4 rg = __ldg(regions + q);  // r0, c0, r1, c1 (inclusive), warp-uniform
    const int64_t r0 = rg.x, c0 = rg.y, r1 = rg.z, c1 = rg.w;
    unsigned long long* orow = out + q * nb;
    if (r0 < 0 || c0 < 0 || r0 > r1 || c0 > c1 || r1 >= H || c1 >= W) {
      // invalid region (the Python layer raises BoundsError before launch;
      // a C caller gets zeros, never an out-of-bounds read)
      for (int b = lane; b < nb; b += 32) orow[b] = 0ull;
      continue;
    }
    const bool top = r0 > 0, left = c0 > 0;
    const int64_t o11 = r1 * W + c1;
    const int64_t o01 = top ? (r0 - 1) * W + c1 : 0;
    const int64_t o10 = left ? r1 * W + (c0 - 1) : 0;
    const int64_t o00 = top && left ? (r0 - 1) * W + (c0 - 1) : 0;
    for (int b0 = 0; b0 < nb; b0 += 128) {
      uint32_t v[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int b = b0 + u * 32 + lane;
        const uint32_t* p = t + (int64_t)(b < nb ? b : 0) * plane;
        v[u][0] = b < nb ? ldg_l2_64(p + o11) : 0u;
        v[u][1] = b < nb && top ? ldg_l2_64(p + o01) : 0u;
        v[u][2] = b < nb && left ? ldg_l2_64(p + o10) : 0u;
        v[u][3] = b < nb && top && left ? ldg_l2_64(p + o00) : 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int b = b0 + u * 32 + lane;
        if (b < nb)
          orow[b] = (unsigned long long)((int64_t)v[u][0] - (int64_t)v[u][1] - (int64_t)v[u][2] +
                                         (int64_t)v[u][3]);
      }
    }
  }
}

// K4: grid (column blocks, output rows, bins); thread per output element, two
// per thread (j and j + blockDim.x).  The four corner rows are read coalesced;
// corners above row 0 / left of column 0 are zero (likelihood.py:44-51).
__global__ void __launch_bounds__(256) k4_window_counts(const uint32_t* __restrict__ t, int nb,
                                                         int64_t H, int64_t W, int h, int w,
                                                         long long* __restrict__ out) {
  const int64_t R = H - h + 1, C = W - w + 1;
  const int64_t b = blockIdx.z;
  const uint32_t* p = t + b * H * W;
  for (int64_t i = blockIdx.y; i < R; i += gridDim.y) {
    const uint32_t* bot = p + (i + h - 1) * W;
    const uint32_t* topr = p + (i - 1) * W;  // used only when i > 0
    long long* orow = out + (b * R + i) * C;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int64_t j = ((int64_t)blockIdx.x * 2 + half) * blockDim.x + threadIdx.x;
      if (j >= C) continue;
      long long v = (long long)__ldg(bot + j + w - 1);
      if (j > 0) v -= (long long)__ldg(bot + j - 1);
      if (i > 0) {
        v -= (long long)__ldg(topr + j + w - 1);
        if (j > 0) v += (long long)__ldg(topr + j - 1);
      }
      __stcs(orow + j, v);
    }
  }
}

// K4 (ILP): as k4_window_counts with U outputs per thread (columns j + u*256),
// all 4U corner loads issued before the first store: the corner reads are L2
// hits, so memory-level parallelism per thread decides the throughput.
template <int U, int MINB>
__global__ void __launch_bounds__(256, MINB) k4_window_counts_ilp(const uint32_t* __restrict__ t, int nb,
                                                             int64_t H, int64_t W, int h, int w,
                                                             long long* __restrict__ out) {
  const int64_t R = H - h + 1, C = W - w + 1;
  const int64_t b = blockIdx.z;
  const uint32_t* p = t + b * H * W;
  for (int64_t i = blockIdx.y; i < R; i += gridDim.y) {
    const uint32_t* bot = p + (i + h - 1) * W;
    const uint32_t* topr = p + (i - 1) * W;  // used only when i > 0
    long long* orow = out + (b * R + i) * C;
    uint32_t a[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = ((int64_t)blockIdx.x * U + u) * blockDim.x + threadIdx.x;
      const bool ok = j < C;
      a[u][0] = ok ? __ldg(bot + j + w - 1) : 0u;
      a[u][1] = ok && j > 0 ? __ldg(bot + j - 1) : 0u;
      a[u][2] = ok && i > 0 ? __ldg(topr + j + w - 1) : 0u;
      a[u][3] = ok && i > 0 && j > 0 ? __ldg(topr + j - 1) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = ((int64_t)blockIdx.x * U + u) * blockDim.x + threadIdx.x;
      // the window count is exact in u32 (0 <= n <= h*w < 2^32): modular
      // arithmetic, then a zero-extending store
      if (j < C) __stcs(orow + j, (long long)(a[u][0] - a[u][1] - a[u][2] + a[u][3]));
    }
  }
}

// K4 (pairs): like k4_window_counts_ilp, but a thread forms two adjacent
// outputs per step and writes them with one 16-byte streaming store.  The pair
// start is shifted by the parity of the row's first element index, so every
// pair store is 16-byte aligned for any output width; column 0 of an odd-based
// row is stored alone.
template <int U>
__global__ void __launch_bounds__(256, 6) k4_window_counts_pairs(const uint32_t* __restrict__ t,
                                                                  int nb, int64_t H, int64_t W,
                                                                  int h, int w,
                                                                  long long* __restrict__ out) {
  const int64_t R = H - h + 1, C = W - w + 1;
  const int64_t b = blockIdx.z;
  const uint32_t* p = t + b * H * W;
  for (int64_t i = blockIdx.y; i < R; i += gridDim.y) {
    const uint32_t* bot = p + (i + h - 1) * W;
    const uint32_t* topr = p + (i - 1) * W;  // used only when i > 0
    const int64_t rowbase = (b * R + i) * C;
    long long* orow = out + rowbase;
    const int off = (int)(rowbase & 1);  // pairs start at odd columns when rowbase is odd
    auto count = [&](int64_t j) -> uint32_t {
      const uint32_t a11 = __ldg(bot + j + w - 1);
      const uint32_t a10 = j > 0 ? __ldg(bot + j - 1) : 0u;
      const uint32_t a01 = i > 0 ? __ldg(topr + j + w - 1) : 0u;
      const uint32_t a00 = i > 0 && j > 0 ? __ldg(topr + j - 1) : 0u;
      return a11 - a10 - a01 + a00;  // exact in u32
    };
    uint32_t n[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t js = 2 * (((int64_t)blockIdx.x * U + u) * blockDim.x + threadIdx.x) + off;
      n[u][0] = js < C ? count(js) : 0u;
      n[u][1] = js + 1 < C ? count(js + 1) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t js = 2 * (((int64_t)blockIdx.x * U + u) * blockDim.x + threadIdx.x) + off;
      if (js + 1 < C)
        __stcs(reinterpret_cast<longlong2*>(orow + js),
               make_longlong2((long long)n[u][0], (long long)n[u][1]));
      else if (js < C)
        __stcs(orow + js, (long long)n[u][0]);
    }
    if (off && blockIdx.x == 0 && threadIdx.x == 0) __stcs(orow, (long long)count(0));
  }
}

// K4 (quads, the default for 16-byte aligned tensor rows): a thread forms 4
// adjacent outputs j = q..q+3 (q % 4 == 0) of one row.  Their left corners
// are columns q-1..q+2 (a 16-byte load at q plus one word at q-1) and their
// right corners columns q+w-1..q+w+2, taken from one or two aligned 16-byte
// loads at the word offset M = (w - 1) % 4 (a template parameter: no per-row
// select).  8 loads per 4 outputs instead of 16 scalar corner loads -- the
// pairs kernel executed 59 instructions per output and was issue bound
// (profiles/r02c/k4_pairs_summary.json).  Stores: two 16-byte pairs, or a
// word + pair + word when the output row starts at an odd element.  Threads
// whose loads would pass the row end take the scalar corner path.
__device__ __forceinline__ uint4 ldg4(const uint32_t* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}
template <int M>
__device__ __forceinline__ void pick4(const uint4& a, const uint4& b, uint32_t r[4]) {
  const uint32_t v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) r[k] = v[M + k];
}

// One row's 4 outputs (see k4_window_counts_quads): corner loads issued by
// load(), differences and stores by finish(), so a thread can keep several
// rows' loads in flight.
template <int M>
struct K4Quad {
  uint4 lb, rb0, rb1, lt, rt0, rt1;
  uint32_t lbm, ltm;
  __device__ __forceinline__ void load(const uint32_t* bot, const uint32_t* top, int64_t q,
                                       int64_t a0) {
    lb = ldg4(bot + q);
    lbm = q > 0 ? __ldg(bot + q - 1) : 0u;
    rb0 = ldg4(bot + a0);
    rb1 = M ? ldg4(bot + a0 + 4) : make_uint4(0u, 0u, 0u, 0u);
    if (top) {
      lt = ldg4(top + q);
      ltm = q > 0 ? __ldg(top + q - 1) : 0u;
      rt0 = ldg4(top + a0);
      rt1 = M ? ldg4(top + a0 + 4) : make_uint4(0u, 0u, 0u, 0u);
    } else {
      lt = rt0 = rt1 = make_uint4(0u, 0u, 0u, 0u);
      ltm = 0u;
    }
  }
  __device__ __forceinline__ void finish(long long* o) const {
    uint32_t rb[4], rt[4], n[4];
    pick4<M>(rb0, rb1, rb);
    pick4<M>(rt0, rt1, rt);
    // exact in u32: each difference is a window count
    n[0] = (rb[0] - lbm) - (rt[0] - ltm);
    n[1] = (rb[1] - lb.x) - (rt[1] - lt.x);
    n[2] = (rb[2] - lb.y) - (rt[2] - lt.y);
    n[3] = (rb[3] - lb.z) - (rt[3] - lt.z);
    if ((((uintptr_t)o) & 15) == 0) {
      __stcs(reinterpret_cast<longlong2*>(o), make_longlong2(n[0], n[1]));
      __stcs(reinterpret_cast<longlong2*>(o + 2), make_longlong2(n[2], n[3]));
    } else {
      __stcs(o, (long long)n[0]);
      __stcs(reinterpret_cast<longlong2*>(o + 1), make_longlong2(n[1], n[2]));
      __stcs(o + 3, (long long)n[3]);
    }
  }
};

template <int M>
__global__ void __launch_bounds__(256) k4_window_counts_quads(const uint32_t* __restrict__ t,
                                                                int nb, int64_t H, int64_t W,
                                                                int h, int w,
                                                                long long* __restrict__ out) {
  const int64_t R = H - h + 1, C = W - w + 1;
  const int64_t b = blockIdx.z;
  const uint32_t* p = t + b * H * W;
  const int64_t q = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (q >= C) return;
  const int64_t a0 = q + w - 1 - M;  // 16-byte aligned base of the right corners
  const bool fast = q + 4 <= C && a0 + (M ? 8 : 4) <= W;
  const int64_t ry = gridDim.y;
  if (fast) {
    // one row per step (two rows i, i + ry per step keep more loads in flight
    // but were 0.146 -> 0.201 ms: 64 registers, half the CTAs, and twice the
    // tensor rows live in L2 at a time; profiles/r02l/k4_sweep.jsonl)
    for (int64_t i = blockIdx.y; i < R; i += ry) {
      K4Quad<M> x;
      x.load(p + (i + h - 1) * W, i > 0 ? p + (i - 1) * W : nullptr, q, a0);
      x.finish(out + (b * R + i) * C + q);
    }
    return;
  }
  for (int64_t i = blockIdx.y; i < R; i += ry) {
    const uint32_t* bot = p + (i + h - 1) * W;
    const uint32_t* top = p + (i - 1) * W;  // used only when i > 0
    long long* orow = out + (b * R + i) * C;
    for (int k = 0; k < 4 && q + k < C; ++k) {
      const int64_t j = q + k;
      const uint32_t a11 = __ldg(bot + j + w - 1);
      const uint32_t a10 = j > 0 ? __ldg(bot + j - 1) : 0u;
      const uint32_t a01 = i > 0 ? __ldg(top + j + w - 1) : 0u;
      const uint32_t a00 = i > 0 && j > 0 ? __ldg(top + j - 1) : 0u;
      __stcs(orow + j, (long long)(a11 - a10 - a01 + a00));
    }
  }
}

// Row-difference staging for K4 (the "vs" variant).  For output
// row i the window count at column j is
//     V[j + w - 1] - V[j - 1],   V(c) = T(i + h - 1, c) - T(i - 1, c)
// (V(-1) = 0, T(-1, .) = 0).  V(c) counts the pixels of rows (i-1, i+h-1] in
// columns [0, c], so 0 <= V <= h*(c+1) <= H*W <= 2^32-1: exact in u32, and the
// difference of two V values is the exact (non-negative) window count.  A CTA
// stages V for its column block once per (row, bin) with two coalesced row
// reads instead of four corner gathers per output, then every thread forms 4
// consecutive outputs from shared memory.
//   CTA = (column block of CW = 4*blockDim outputs, output rows i (grid-stride)).
//   smem: V for columns j0-1 .. j0+CW+w-2, i.e. CW + w u32 (x2 buffers in K5).
__device__ __forceinline__ void stage_v(uint32_t* V, const uint32_t* bot, const uint32_t* top,
                                        int64_t j0, int span) {
  for (int k = threadIdx.x; k < span; k += blockDim.x) {
    const int64_t c = j0 - 1 + k;
    uint32_t v = 0u;
    if (c >= 0) v = __ldg(bot + c) - (top ? __ldg(top + c) : 0u);
    V[k] = v;
  }
}

// K4 (staged): grid (column blocks, rows, bins); int64 out, 16-byte streaming
// stores when the output row length C is even (every row start 16-B aligned).
__global__ void __launch_bounds__(256) k4_window_counts_vs(const uint32_t* __restrict__ t, int nb,
                                                            int64_t H, int64_t W, int h, int w,
                                                            long long* __restrict__ out) {
  extern __shared__ uint32_t V[];
  const int64_t R = H - h + 1, C = W - w + 1;
  const int CW = 4 * blockDim.x;
  const int64_t j0 = (int64_t)blockIdx.x * CW;
  const int ncols = (int)min((int64_t)CW, C - j0);
  const int span = ncols + w;
  const int64_t b = blockIdx.z;
  const uint32_t* p = t + b * H * W;
  const bool vec = (C & 1) == 0;
  for (int64_t i = blockIdx.y; i < R; i += gridDim.y) {
    stage_v(V, p + (i + h - 1) * W, i > 0 ? p + (i - 1) * W : nullptr, j0, span);
    __syncthreads();
    const int q = 4 * threadIdx.x;
    if (q < ncols) {
      long long o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) o[e] = q + e < ncols ? (long long)(V[q + e + w] - V[q + e]) : 0;
      long long* dst = out + (b * R + i) * C + j0 + q;
      if (vec && q + 4 <= ncols) {
        __stcs(reinterpret_cast<longlong2*>(dst), make_longlong2(o[0], o[1]));
        __stcs(reinterpret_cast<longlong2*>(dst) + 1, make_longlong2(o[2], o[3]));
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (q + e < ncols) __stcs(dst + e, o[e]);
      }
    }
    __syncthreads();  // V is rewritten for the next row
  }
}

// K5: fused likelihood map (likelihood.py:55-77).  One thread per window
// placement (i, j), j fastest: for every bin b, the window count from four
// corner reads, q = count / (h*w) (a true division, as numpy does), the metric
// term min(t_b, q) or sqrt(t_b * q), accumulated over b = 0..nb-1 in order
// (numpy's axis-0 reduction order), then clipped to [0, 1].  Only the
// (H-h+1, W-w+1) float64 map is written: the (nb, ...) int64 counts of K4 never
// exist.  The template rides in the kernel parameters (<= 256 doubles).
struct Template {
  double t[256];
};

template <bool INTERSECTION>
__global__ void __launch_bounds__(256) k5_likelihood_map(const uint32_t* __restrict__ t, int nb,
                                                          int64_t H, int64_t W, int h, int w,
                                                          Template tpl, double* __restrict__ out) {
  const int64_t R = H - h + 1, C = W - w + 1;
  const double area = (double)h * (double)w;
  const int64_t plane = H * W;
  for (int64_t i = blockIdx.y; i < R; i += gridDim.y) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= C) continue;
    const int64_t o11 = (i + h - 1) * W + (j + w - 1);
    const int64_t o01 = (i - 1) * W + (j + w - 1);
    const int64_t o10 = (i + h - 1) * W + (j - 1);
    const int64_t o00 = (i - 1) * W + (j - 1);
    double acc = 0.0;
    constexpr int U = 8;  // bins per step: 32 independent corner loads in flight
    for (int b0 = 0; b0 < nb; b0 += U) {
      long long v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int b = b0 + u < nb ? b0 + u : nb - 1;
        const uint32_t* p = t + (int64_t)b * plane;
        const uint32_t a11 = __ldg(p + o11);
        const uint32_t a10 = j > 0 ? __ldg(p + o10) : 0u;
        const uint32_t a01 = i > 0 ? __ldg(p + o01) : 0u;
        const uint32_t a00 = i > 0 && j > 0 ? __ldg(p + o00) : 0u;
        v[u] = (long long)a11 - (long long)a10 - (long long)a01 + (long long)a00;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {  // the sum over bins stays in order b = 0..nb-1
        if (b0 + u < nb) {
          const double q = (double)v[u] / area;
          const double tb = tpl.t[b0 + u];
          acc += INTERSECTION ? fmin(tb, q) : sqrt(tb * q);
        }
      }
    }
    out[i * C + j] = fmin(fmax(acc, 0.0), 1.0);
  }
}

// K5 with a metric table.  Every window count n lies in [0, h*w], so the
// per-(bin, n) term M[b][n] = min(t_b, n/(h*w)) or sqrt(t_b * (n/(h*w))) is
// computed once (k5_metric_table, the exact expressions of k5_likelihood_map)
// and the map kernel only gathers: 4 corner reads, one table read (the bin's
// slice is L1/L2-resident while the CTA's threads walk that bin) and an add,
// in bin order -- bit-identical to k5_likelihood_map, without its per-element
// FP64 division and square root.
template <bool INTERSECTION>
__global__ void __launch_bounds__(256) k5_metric_table(Template tpl, int nb, int64_t area,
                                                        double* __restrict__ M) {
  const int64_t n1 = area + 1;
  const int64_t total = (int64_t)nb * n1;
  const double a = (double)area;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(e / n1);
    const int64_t n = e - b * n1;
    const double q = (double)(long long)n / a;
    const double tb = tpl.t[b];
    M[e] = INTERSECTION ? fmin(tb, q) : sqrt(tb * q);
  }
}

__global__ void __launch_bounds__(256) k5_likelihood_map_tab(const uint32_t* __restrict__ t, int nb,
                                                              int64_t H, int64_t W, int h, int w,
                                                              const double* __restrict__ M,
                                                              double* __restrict__ out) {
  const int64_t R = H - h + 1, C = W - w + 1;
  const int64_t n1 = (int64_t)h * w + 1;
  const int64_t plane = H * W;
  for (int64_t i = blockIdx.y; i < R; i += gridDim.y) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= C) continue;
    const int64_t o11 = (i + h - 1) * W + (j + w - 1);
    const int64_t o01 = (i - 1) * W + (j + w - 1);
    const int64_t o10 = (i + h - 1) * W + (j - 1);
    const int64_t o00 = (i - 1) * W + (j - 1);
    double acc = 0.0;
    constexpr int U = 8;  // bins per step: 32 corner loads, then 8 table loads in flight
    for (int b0 = 0; b0 < nb; b0 += U) {
      uint32_t n[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int b = b0 + u < nb ? b0 + u : nb - 1;
        const uint32_t* p = t + (int64_t)b * plane;
        const uint32_t a11 = __ldg(p + o11);
        const uint32_t a10 = j > 0 ? __ldg(p + o10) : 0u;
        const uint32_t a01 = i > 0 ? __ldg(p + o01) : 0u;
        const uint32_t a00 = i > 0 && j > 0 ? __ldg(p + o00) : 0u;
        n[u] = a11 - a10 - a01 + a00;  // exact window count in [0, h*w]
      }
      double m[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int b = b0 + u < nb ? b0 + u : nb - 1;
        m[u] = __ldg(M + (int64_t)b * n1 + n[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)  // the sum over bins stays in order b = 0..nb-1
        if (b0 + u < nb) acc += m[u];
    }
    out[i * C + j] = fmin(fmax(acc, 0.0), 1.0);
  }
}

// K5 (table, P placements per thread, 32 apart): each bin's four corner
// pointers serve P placements (loads at +0, +32, ...): a P-th of the address
// arithmetic per placement, and every warp load is one coalesced run.  Same
// terms, same bin order: bit-identical to k5_likelihood_map / _tab.
template <int P, int UB = (P >= 4 ? 2 : 4)>
__global__ void __launch_bounds__(256) k5_likelihood_map_tabp(const uint32_t* __restrict__ t, int nb,
                                                               int64_t H, int64_t W, int h, int w,
                                                               const double* __restrict__ M,
                                                               double* __restrict__ out) {
  const int64_t R = H - h + 1, C = W - w + 1;
  const int64_t n1 = (int64_t)h * w + 1;
  const int64_t plane = H * W;
  for (int64_t i = blockIdx.y; i < R; i += gridDim.y) {
    // a warp covers 32*P consecutive placements, lane l taking l, l+32, ...:
    // every corner load and output store of the warp is one coalesced run
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t j = (g >> 5) * (32 * P) + (g & 31);
    if (j >= C) continue;
    const int64_t o11 = (i + h - 1) * W + (j + w - 1);
    const int64_t o01 = (i - 1) * W + (j + w - 1);
    const int64_t o10 = (i + h - 1) * W + (j - 1);
    const int64_t o00 = (i - 1) * W + (j - 1);
    bool ok[P];
#pragma unroll
    for (int q = 0; q < P; ++q) ok[q] = j + 32 * q < C;
    double acc[P];
#pragma unroll
    for (int q = 0; q < P; ++q) acc[q] = 0.0;
    constexpr int U = UB;  // bins per step
    if (i > 0 && j > 0 && j + 32 * (P - 1) < C) {
      // interior placements (all but the first row / column and a ragged
      // tail): no predicates, the four corner pointers and the table row step
      // by one plane / one table row per bin -- the general path below spends
      // most of its issue slots on 64-bit address arithmetic and predicates
      const uint32_t* p11 = t + o11;
      const uint32_t* p10 = t + o10;
      const uint32_t* p01 = t + o01;
      const uint32_t* p00 = t + o00;
      const double* Mb = M;
      int b = 0;
      for (; b + U <= nb; b += U) {
        uint32_t n[U][P];
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int q = 0; q < P; ++q)
            n[u][q] = __ldg(p11 + 32 * q) - __ldg(p10 + 32 * q) - __ldg(p01 + 32 * q) + __ldg(p00 + 32 * q);
          p11 += plane, p10 += plane, p01 += plane, p00 += plane;
        }
        double m[U][P];
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int q = 0; q < P; ++q) m[u][q] = __ldg(Mb + n[u][q]);
          Mb += n1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)  // bin order b = 0..nb-1
#pragma unroll
          for (int q = 0; q < P; ++q) acc[q] += m[u][q];
      }
      for (; b < nb; ++b) {
#pragma unroll
        for (int q = 0; q < P; ++q) {
          const uint32_t c = __ldg(p11 + 32 * q) - __ldg(p10 + 32 * q) - __ldg(p01 + 32 * q) + __ldg(p00 + 32 * q);
          acc[q] += __ldg(Mb + c);
        }
        p11 += plane, p10 += plane, p01 += plane, p00 += plane;
        Mb += n1;
      }
#pragma unroll
      for (int q = 0; q < P; ++q) out[i * C + j + 32 * q] = fmin(fmax(acc[q], 0.0), 1.0);
      continue;
    }
    for (int b0 = 0; b0 < nb; b0 += U) {
      uint32_t n[U][P];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int b = b0 + u < nb ? b0 + u : nb - 1;
        const uint32_t* p = t + (int64_t)b * plane;
        const uint32_t* p11 = p + o11;
        const uint32_t* p10 = p + o10;
        const uint32_t* p01 = p + o01;
        const uint32_t* p00 = p + o00;
#pragma unroll
        for (int q = 0; q < P; ++q) {
          const bool left = j + 32 * q > 0;
          const uint32_t a11 = ok[q] ? __ldg(p11 + 32 * q) : 0u;
          const uint32_t a10 = ok[q] && left ? __ldg(p10 + 32 * q) : 0u;
          const uint32_t a01 = ok[q] && i > 0 ? __ldg(p01 + 32 * q) : 0u;
          const uint32_t a00 = ok[q] && i > 0 && left ? __ldg(p00 + 32 * q) : 0u;
          n[u][q] = a11 - a10 - a01 + a00;  // exact window count
        }
      }
      double m[U][P];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int b = b0 + u < nb ? b0 + u : nb - 1;
        const double* Mb = M + (int64_t)b * n1;
#pragma unroll
        for (int q = 0; q < P; ++q) m[u][q] = ok[q] ? __ldg(Mb + n[u][q]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)  // the sum over bins stays in order b = 0..nb-1
        if (b0 + u < nb) {
#pragma unroll
          for (int q = 0; q < P; ++q) acc[q] += m[u][q];
        }
    }
#pragma unroll
    for (int q = 0; q < P; ++q)
      if (ok[q]) out[i * C + j + 32 * q] = fmin(fmax(acc[q], 0.0), 1.0);
  }
}

// K5 (table) over chains of output rows h apart: output row r reads tensor
// rows r - 1 and r + h - 1, so rows r and r + h share row r + h - 1.  A
// thread takes K output rows i0 + h*k (k < K) of P placements (32 apart, as
// _tabp) and, per bin, the horizontal differences
//     D_k = T(row_k, j + w - 1) - T(row_k, j - 1),  row_k = i0 - 1 + h*k
// of K + 1 tensor rows (2 loads each); window count n_k = D_{k+1} - D_k
// (exact in u32).  2P(K+1) corner loads per bin instead of 4PK.  Same terms,
// same bin order: bit-identical to _tabp.
template <int K, int P>
__global__ void __launch_bounds__(256) k5_likelihood_map_chain(const uint32_t* __restrict__ t,
                                                                int nb, int64_t H, int64_t W,
                                                                int h, int w,
                                                                const double* __restrict__ M,
                                                                double* __restrict__ out) {
  const int64_t R = H - h + 1, C = W - w + 1;
  const int64_t n1 = (int64_t)h * w + 1;
  const int64_t plane = H * W;
  const int64_t blocks_per_i0 = (R + (int64_t)h * K - 1) / ((int64_t)h * K);
  const int64_t nchains = blocks_per_i0 * h;
  for (int64_t y = blockIdx.y; y < nchains; y += gridDim.y) {
    const int64_t i0 = (y % h) + (int64_t)h * K * (y / h);  // first output row of the chain
    if (i0 >= R) continue;
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t j = (g >> 5) * (32 * P) + (g & 31);
    if (j >= C) continue;
    bool ok[P];
#pragma unroll
    for (int q = 0; q < P; ++q) ok[q] = j + 32 * q < C;
    int nrows = 0;  // valid output rows of this chain
#pragma unroll
    for (int k = 0; k < K; ++k) nrows += i0 + (int64_t)h * k < R;
    double acc[K][P];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int q = 0; q < P; ++q) acc[k][q] = 0.0;
    const double* Mb = M;
    for (int b = 0; b < nb; ++b, Mb += n1) {
      const uint32_t* p = t + (int64_t)b * plane;
      uint32_t D[K + 1][P];
#pragma unroll
      for (int k = 0; k <= K; ++k) {
        const int64_t row = i0 - 1 + (int64_t)h * k;
        const bool rv = row >= 0 && k <= nrows;  // row K only if it bounds a valid output
        const uint32_t* pr = p + row * W;
#pragma unroll
        for (int q = 0; q < P; ++q) {
          const int64_t jj = j + 32 * q;
          const uint32_t right = rv && ok[q] ? __ldg(pr + jj + w - 1) : 0u;
          const uint32_t left = rv && ok[q] && jj > 0 ? __ldg(pr + jj - 1) : 0u;
          D[k][q] = right - left;
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int q = 0; q < P; ++q)
          if (k < nrows && ok[q]) acc[k][q] += __ldg(Mb + (D[k + 1][q] - D[k][q]));
    }
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int q = 0; q < P; ++q)
        if (k < nrows && ok[q]) out[(i0 + (int64_t)h * k) * C + j + 32 * q] = fmin(fmax(acc[k][q], 0.0), 1.0);
  }
}

}  // namespace ih
