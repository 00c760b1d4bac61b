// ih_capi.cu -- the extern "C" boundary (include/inthist_b200.h).
//
// Host-side planning, validation (reference exception order) and launches.
// Unity build: the kernel translation units are included here so the shared
// library is a single nvcc invocation.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unistd.h>

#include <mutex>
#include <unordered_map>
#include <utility>

#include "../../include/inthist_b200.h"
#include "ih_kernels.cuh"
#include "ih_queries.cu"
#include "ih_scan.cu"
#include "ih_single_pass.cu"
#include "ih_small.cu"
#include "ih_wavefront.cu"

namespace {

thread_local char g_last_error[512] = "";

ih_status cuda_fail(const char* where) {
  cudaError_t e = cudaGetLastError();
  snprintf(g_last_error, sizeof g_last_error, "%s: %s", where, cudaGetErrorString(e));
  return IH_ERR_CUDA;
}

ih_status fail(ih_status s, const char* msg) {
  snprintf(g_last_error, sizeof g_last_error, "%s", msg);
  return s;
}

int64_t env_int(const char* name, int64_t dflt) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  return strtoll(v, nullptr, 10);
}

// SMs of the current device (cudaDevAttrMultiProcessorCount, cached per
// device): the wave planner and the grid caps use the real count, so MIG
// slices, green contexts and other SKUs plan for what they have.  148 (B200)
// only when no device is present (ih_workspace_bytes on a CPU host).
int device_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return 148;
  }
  if (cache[dev] > 0) return cache[dev];
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) {
    cudaGetLastError();
    return 148;
  }
  cache[dev] = n;
  return n;
}

// The IH_* tuning knobs are read from the environment (tests and A/B scripts
// set them per call).  One pass over environ fingerprints them; plans and the
// per-call knobs are cached under that fingerprint, so a steady stream of
// calls costs a hash lookup instead of ~15 getenv and an occupancy query.
uint64_t knob_fingerprint() {
  uint64_t h = 1469598103934665603ull;
  for (char** e = environ; e && *e; ++e) {
    const char* s = *e;
    if (s[0] != 'I' || s[1] != 'H' || s[2] != '_') continue;
    for (; *s; ++s) h = (h ^ (uint8_t)*s) * 1099511628211ull;
    h = (h ^ 0x1f) * 1099511628211ull;
  }
  return h;
}

// Row-segment hints (ih_plan_hint): measured segment counts per problem shape,
// set by an autotuner; consulted by plan_k2 before its own heuristic.
struct PlanHint {
  int64_t frames, H, W;
  int32_t nb, nseg, tail_pct, tail_div, flags;
};
constexpr int32_t kHintCluster = 1;  // ih_plan_hint flags: cluster (DSMEM) carries
constexpr int32_t kHintSmall = 2;    // ih_plan_hint flags: K2s one-launch path
constexpr int32_t kHintSkew = 4;     // ih_plan_hint flags: skewed segments (tail_pct = % of
                                     // big segments, tail_div = size ratio x 100)
constexpr int32_t kHintKb2 = 8;      // ih_plan_hint flags: bin pairs (2 rows per packed word)
constexpr int32_t kHintKb4 = 16;     // ih_plan_hint flags: bin quads (the 4-bin group kernel)
constexpr int kMaxHints = 64;
PlanHint g_hints[kMaxHints];
int g_nhints = 0;
uint32_t g_hint_gen = 0;  // bumped by ih_plan_hint: invalidates cached plans
std::mutex g_hint_mu;

unsigned long long* g_trace = nullptr;  // ih_debug_trace
size_t g_trace_ctas = 0;

int32_t hint_lookup(int64_t frames, int64_t H, int64_t W, int32_t nb, int32_t* tail_pct,
                    int32_t* tail_div, int32_t* flags) {
  std::lock_guard<std::mutex> lock(g_hint_mu);
  for (int i = 0; i < g_nhints; ++i)
    if (g_hints[i].frames == frames && g_hints[i].H == H && g_hints[i].W == W && g_hints[i].nb == nb) {
      *tail_pct = g_hints[i].tail_pct;
      *tail_div = g_hints[i].tail_div;
      *flags = g_hints[i].flags;
      return g_hints[i].nseg;
    }
  return 0;
}

// Launch with programmatic stream serialization when `pdl` (see ih_kernels.cuh
// griddep_wait): only for a kernel whose stream predecessor is a kernel this
// same call launched, so user work before the call is always fully ordered.
template <typename... KArgs, typename... Args>
cudaError_t launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                   bool pdl, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------ planning
struct K2Plan {
  int cpl = 0;       // chunks per lane; 0 = width unsupported by K2
  int nwarps = 0;    // warps per CTA
  int R = 4;         // rows per barrier batch
  int ngroups = 0;   // bin groups of 4
  int nbp = 0;       // padded slab bins
  int nseg = 1;      // row segments per frame
  int S = 0;         // rows per (big) segment
  int nbig = 1;      // big segments; the rest are tail segments of S2 rows
  int S2 = 0;
  int64_t Wp = 0;    // padded width = T * TW
  int T = 1;         // column tiles (colt)
  int TW = 0;        // tile width = nwarps * cpl * 128
  bool colt = false; // column-tiled instantiation (W > 2048 unless IH_NO_COLTILE)
  bool staged = false;  // experimental TMA bulk-store epilogue (IH_STAGED_STORES)
  int kb = 4;           // bins per group: 4, or 1/2 with 4/2 rows packed per word (B <= 2)
  int slots = 0;     // resident CTAs of the scan kernel (SMs x CTAs per SM)
  int64_t units = 0; // scan CTAs per row segment (frames x bin groups x tiles)
  int carry = 0;     // ih::Carry: NONE (nseg == 1), TABLE or LOOKBACK
  bool big = false;  // 1024-thread instantiation (up to 32 warps, <= 64 registers)
  bool vec = true;   // W % 4 == 0
  bool tma = true;   // 16-byte aligned rows
  bool small = false;  // K2s: one launch, in-kernel segment carries (ih_small.cu)
  int nwg = 1;         // K2s warp-groups per CTA
  int Sk = 0;          // K2s rows per warp-group
};

// Opt a kernel into `bytes` of dynamic shared memory.  Static + dynamic
// shared memory above 48 KB needs the attribute, so it is set for any
// non-zero request (once per kernel and size: cached).
bool set_dyn_smem(const void* fn, size_t bytes) {
  // the attribute is per device: cache by (kernel, current device)
  static std::mutex mu;
  static std::unordered_map<uint64_t, size_t> done;
  if (bytes == 0) return true;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  const uint64_t key = (uint64_t)(uintptr_t)fn * 64u + (uint64_t)dev;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return true;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) !=
      cudaSuccess)
    return false;
  done[key] = bytes;
  return true;
}

using K2Fn = void (*)(ih::ScanArgs, ih::RelLut);

ih::Segs segs(const K2Plan& p) { return ih::Segs{p.S, p.nbig, p.S2}; }

template <int CPL, int R, bool VEC, bool TMA, int MAXT>
K2Fn pick_carry(int carry, bool colt) {
  if constexpr (CPL == 1 && MAXT == 512) {  // column tiles: CPL 1, table carries
    if (colt)
      return carry == ih::CARRY_TABLE ? ih::k2_scan<CPL, R, VEC, TMA, ih::CARRY_TABLE, MAXT, true>
             : carry == ih::CARRY_NONE ? ih::k2_scan<CPL, R, VEC, TMA, ih::CARRY_NONE, MAXT, true>
                                       : nullptr;
  }
  if (colt) return nullptr;
  switch (carry) {
    case ih::CARRY_CLUSTER:
      if constexpr (MAXT == 512 && CPL == 1)
        return ih::k2_scan<CPL, R, VEC, TMA, ih::CARRY_CLUSTER, MAXT, false>;
      return nullptr;
    case ih::CARRY_TABLE: return ih::k2_scan<CPL, R, VEC, TMA, ih::CARRY_TABLE, MAXT, false>;
    case ih::CARRY_LOOKBACK: return ih::k2_scan<CPL, R, VEC, TMA, ih::CARRY_LOOKBACK, MAXT, false>;
    default: return ih::k2_scan<CPL, R, VEC, TMA, ih::CARRY_NONE, MAXT, false>;
  }
}
template <int R>
K2Fn pick_staged(int carry) {
  return carry == ih::CARRY_TABLE ? ih::k2_scan<1, R, true, true, ih::CARRY_TABLE, 512, false, true>
                                  : ih::k2_scan<1, R, true, true, ih::CARRY_NONE, 512, false, true>;
}

template <int KB, bool VEC, bool TMA>
K2Fn pick_rowpack_c(int carry) {
  return carry == ih::CARRY_TABLE
             ? ih::k2_scan<1, 4, VEC, TMA, ih::CARRY_TABLE, 512, false, false, KB>
             : ih::k2_scan<1, 4, VEC, TMA, ih::CARRY_NONE, 512, false, false, KB>;
}
template <int KB>
K2Fn pick_rowpack(const K2Plan& p) {
  if (p.vec && p.tma) return pick_rowpack_c<KB, true, true>(p.carry);
  if (p.vec) return pick_rowpack_c<KB, true, false>(p.carry);
  if (p.tma) return pick_rowpack_c<KB, false, true>(p.carry);
  return pick_rowpack_c<KB, false, false>(p.carry);
}

template <int CPL, int R>
K2Fn pick_vt(const K2Plan& p) {
  if constexpr (CPL == 1 && R <= 2) {
    if (p.staged) return pick_staged<R>(p.carry);
  }
  if constexpr (CPL == 1 && R == 4) {
    if (p.kb == 1) return pick_rowpack<1>(p);
    if (p.kb == 2) return pick_rowpack<2>(p);
  }
  if constexpr (CPL == 1) {  // 1024-thread variants: CPL 1, aligned fast path only
    if (p.big) return pick_carry<CPL, R, true, true, 1024>(p.carry, false);
  } else {
    if (p.big) return nullptr;
  }
  if (p.vec && p.tma) return pick_carry<CPL, R, true, true, 512>(p.carry, p.colt);
  if (p.vec) return pick_carry<CPL, R, true, false, 512>(p.carry, p.colt);
  if (p.tma) return pick_carry<CPL, R, false, true, 512>(p.carry, p.colt);
  return pick_carry<CPL, R, false, false, 512>(p.carry, p.colt);
}
// The instantiated (CPL, R) pairs; plan_k2 only produces these.
K2Fn pick_k2(const K2Plan& p) {
  switch (p.cpl * 10 + p.R) {
    case 11: return pick_vt<1, 1>(p);
    case 12: return pick_vt<1, 2>(p);
    case 14: return pick_vt<1, 4>(p);
    case 21: return pick_vt<2, 1>(p);
    case 22: return pick_vt<2, 2>(p);
    case 41: return pick_vt<4, 1>(p);
    default: return nullptr;
  }
}
size_t k2_ring_smem(const K2Plan& p) {
  if (!p.tma) return 0;
  const int nst = p.R >= 4 ? 2 : (p.R == 2 ? 4 : 8);  // ih::Ring<R>::kStages
  const size_t stage = p.staged ? (size_t)p.R * ih::kGroup * p.TW * sizeof(uint32_t) : 0;
  return (size_t)nst * p.R * p.TW + stage;
}

// Resident CTAs per SM for the plan's kernel (occupancy API); a register-based
// estimate when no device is present (ih_workspace_bytes on a CPU host).
int ctas_per_sm(const K2Plan& p) {
  K2Fn fn = pick_k2(p);
  const size_t smem = k2_ring_smem(p);
  int n = 0;
  if (fn && set_dyn_smem((const void*)fn, smem) &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, p.nwarps * 32, smem) == cudaSuccess &&
      n > 0)
    return n;
  cudaGetLastError();  // clear a sticky "no device" error
  const int regs = p.cpl == 1 ? 56 : p.cpl == 2 ? (p.big ? 64 : 96) : 128;
  n = 65536 / (regs * p.nwarps * 32);
  return n < 1 ? 1 : n;
}

// ---- K2s (ih_small.cu): one launch with in-kernel segment carries
using KSFn = void (*)(ih::SmallArgs, ih::RelLut);
KSFn pick_small(const K2Plan& p) {
  switch (p.nwg) {
    case 4: return p.vec ? ih::k2_small<4, true> : ih::k2_small<4, false>;
    case 2: return p.vec ? ih::k2_small<2, true> : ih::k2_small<2, false>;
    default: return p.vec ? ih::k2_small<1, true> : ih::k2_small<1, false>;
  }
}
// staged rows: one bulk copy per warp-group when the rows are contiguous in
// a pitch of at most twice the vector width (the smem row stride is then the
// pitch); otherwise one copy per row at stride TW
bool small_contig(const K2Plan& p, int64_t pitch) { return pitch <= 2 * (int64_t)p.TW; }
size_t small_ring_bytes(const K2Plan& p, int64_t pitch) {
  const int64_t rs = small_contig(p, pitch) ? pitch : p.TW;
  return ((size_t)p.S * rs + p.TW + 15) / 16 * 16;
}
size_t small_smem(const K2Plan& p, int64_t pitch) {  // rows | cnt | psum
  return small_ring_bytes(p, pitch) + (size_t)2 * p.nwg * 2 * p.TW * sizeof(uint32_t);
}
int small_ctas_per_sm(const K2Plan& p) {
  KSFn fn = pick_small(p);
  const size_t smem = small_smem(p, 2 * (int64_t)p.TW);  // the larger staging layout
  int n = 0;
  if (set_dyn_smem((const void*)fn, smem) &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, p.nwarps * 32, smem) == cudaSuccess &&
      n > 0)
    return n;
  cudaGetLastError();
  return 1;
}
// Plan K2s when one wave of CTAs covers the problem with >= 2 segments per
// frame: W <= 2048 (one 128-column chunk per warp, <= 16 warps), 16-byte
// aligned rows (TMA), H <= 65535 (16-bit count lanes).  `force`: hint flag /
// IH_SMALL=1; automatically only for frames x bin groups <= 4 -- the
// measured cases where one launch beats the count-table path (512x512x16
// bins 16.3 vs 21.4 us graph-timed; with 8+ groups the table path's
// 3 launches win, e.g. 512x512x32 16.8 vs 18.6 us: profiles/r02d/).
bool plan_small(K2Plan& p, int64_t frames, int64_t H, int64_t W, int nb, bool force,
                int64_t want_nseg) {
  const int64_t nch = (W + ih::kChunk - 1) / ih::kChunk;
  if (!p.tma || H > 65535 || nch > 16 || frames > 65535) return false;
  K2Plan q = p;
  q.small = true;
  q.cpl = 1;
  q.colt = false;
  q.big = false;
  q.staged = false;
  q.kb = ih::kGroup;
  q.R = 4;
  q.T = 1;
  q.nwg = nch <= 4 ? 4 : nch <= 8 ? 2 : 1;
  const int wpg = (int)nch;
  q.TW = wpg * ih::kChunk;
  q.Wp = q.TW;
  q.nwarps = q.nwg * wpg;
  q.ngroups = (nb + ih::kGroup - 1) / ih::kGroup;
  q.nbp = q.ngroups * ih::kGroup;
  const int64_t units = frames * q.ngroups;
  if (!force && units > 4) return false;
  const int64_t sms = device_sms();
  // segment count for one wave; the shared-memory size depends on S, so
  // settle the occupancy in two rounds
  int64_t nseg = sms / units;
  for (int it = 0; it < 2; ++it) {
    if (nseg < 1) nseg = 1;
    if (nseg > H) nseg = H;
    q.S = (int)((H + nseg - 1) / nseg);
    q.slots = (int)(sms * small_ctas_per_sm(q));
    nseg = q.slots / units;
  }
  // >= one 4-row batch per warp-group (unless forced)
  const int64_t max_seg = force ? H : H / (4 * q.nwg);
  if (nseg > max_seg) nseg = max_seg;
  if (nseg < 2 && !force) return false;  // frames x groups already fill a wave
  if (force && want_nseg > 0) nseg = want_nseg < H ? want_nseg : H;  // hint / IH_NSEG
  if (nseg < 1) nseg = 1;
  q.S = (int)((H + nseg - 1) / nseg);
  q.nseg = (int)((H + q.S - 1) / q.S);
  q.Sk = (q.S + q.nwg - 1) / q.nwg;
  q.nbig = q.nseg;
  q.S2 = q.S;
  q.units = units;
  q.carry = ih::CARRY_NONE;
  if (small_smem(q, 2 * (int64_t)q.TW) > 200 * 1024) return false;
  p = q;
  return true;
}

K2Plan plan_k2_uncached(int64_t frames, int64_t H, int64_t W, int nb, bool vec, bool tma) {
  K2Plan p;
  p.vec = vec;
  p.tma = tma;
  const int64_t nchunks = (W + ih::kChunk - 1) / ih::kChunk;
  int64_t tile_chunks = env_int("IH_TILE_CHUNKS", 16);  // max chunks per column tile
  if (tile_chunks < 1 || tile_chunks > 16) tile_chunks = 16;
  if (nchunks > tile_chunks && env_int("IH_NO_COLTILE", 0) == 0) {
    // W > 2048: column tiles of <= 16 chunks (CPL 1), as even as possible
    p.colt = true;
    p.cpl = 1;
    p.T = (int)((nchunks + tile_chunks - 1) / tile_chunks);
  } else if (vec && tma && env_int("IH_NO_BIG", 0) == 0 && nchunks > 16 && nchunks <= 32) {
    // W in (2048, 4096]: one 1024-thread CTA per SM, CPL 1 at <= 64 registers
    p.big = true;
    p.cpl = 1;
  } else if (nchunks <= 16) {  // at most 16 warps per CTA (<= 128 registers)
    p.cpl = 1;
  } else if (nchunks <= 32) {
    p.cpl = 2;
  } else if (nchunks <= 64) {
    p.cpl = 4;
  } else {
    return p;  // cpl = 0: use the cross-weave kernels
  }
  const int64_t tchunks = (nchunks + p.T - 1) / p.T;  // chunks per column tile
  p.nwarps = (int)((tchunks + p.cpl - 1) / p.cpl);
  p.TW = p.nwarps * p.cpl * ih::kChunk;
  p.Wp = (int64_t)p.T * p.TW;
  // rows per barrier batch: tuned on B200 (scripts/sweep*.py, profiles/); the
  // caps keep the accumulators + batch state inside the register budget
  p.R = p.cpl == 1 ? 4 : p.cpl == 2 ? 2 : 1;
  const int64_t r_env = env_int("IH_ROWS_PER_BATCH", 0);
  if (r_env == 1 || r_env == 2 || r_env == 4) p.R = (int)r_env;
  const int rmax = p.cpl == 1 ? 4 : p.cpl == 2 ? 2 : 1;
  if (p.R > rmax) p.R = rmax;
  // experimental staged stores: full-width HD-type kernel, R <= 2 (smem)
  p.staged = env_int("IH_STAGED_STORES", 0) != 0 && !p.colt && !p.big && p.cpl == 1 && vec && tma;
  if (p.staged && p.R > 2) p.R = 2;
  {  // row packing for 1- and 2-bin slabs (plain / table carries, no column tiles)
    int32_t tp = 0, td = 0, fl = 0;
    hint_lookup(frames, H, W, nb, &tp, &td, &fl);
    const bool rowpack_ok = !p.colt && !p.big && p.cpl == 1 && !p.staged &&
                            env_int("IH_NO_ROWPACK", 0) == 0 && env_int("IH_CARRY_LOOKBACK", 0) == 0 &&
                            env_int("IH_CARRY_CLUSTER", 0) == 0 && !(fl & kHintCluster);
    p.kb = rowpack_ok && nb <= 2 ? nb : ih::kGroup;
    // bin pairs with two rows per packed word for >= 24 bins on rows wider
    // than 512 with aligned stores and >= 256 bin pairs over the frames: each CTA
    // then writes 2 bin planes instead of 4 for the same scan work per
    // output, a store pattern HBM drains faster (round-2 A/B, profiles/r02k/:
    // HD x 64 bench step 0.979 -> 0.983-0.991, its 4-GPU share 0.947 ->
    // 0.983; 1600x900x64 graph-timed 0.915 -> 0.953; loses for 512-wide
    // rows, < 24 bins, odd widths and the 8-frame share, 0.944 -> 0.926).
    // IH_KB=1/2/4 or the plan-hint flags (autotuner) choose explicitly.
    const int64_t kb_env = env_int("IH_KB", (fl & kHintKb2) ? 2 : (fl & kHintKb4) ? 4 : 0);
    if (rowpack_ok && kb_env == 0 && nb >= 24 && nchunks > 4 && vec &&
        frames * ((nb + 1) / 2) >= 256)
      p.kb = 2;
    if (rowpack_ok && (kb_env == 1 || kb_env == 2 || kb_env == 4)) p.kb = (int)kb_env;
    if (p.kb < ih::kGroup) p.R = 4;
  }
  p.ngroups = (nb + p.kb - 1) / p.kb;
  p.nbp = p.ngroups * p.kb;
  p.carry = ih::CARRY_TABLE;  // for the occupancy query; fixed up below
  // Row segments (measured, scripts/sweep2.py -> profiles/r01_sweep_*.jsonl):
  // every CTA does the same work, so the CTA count should be a whole number
  // of "waves" of resident CTAs; ~4 waves when frames x groups fill at least a
  // quarter wave, ~2 waves (8 for the 1024-thread variant) otherwise.  If
  // the minimum segment height caps the count, snap down to whole waves.
  // Each segment costs a u16 count slot of 1/(2S) of the output (mostly L2).
  const int64_t slots = (int64_t)device_sms() * ctas_per_sm(p);
  const int64_t units = frames * p.ngroups * p.T;
  // 32-row minimum segments; 16 for short images, 8 up to 512 rows (single
  // 512^2 x 32 frame: 24.0 -> 18.7 -> 16.7 us/call graph-timed; 384^2 17.7 ->
  // 13.9; 600 / 768 rows are faster at 16, profiles/r01i/min_segment_rows.txt)
  const int64_t min_rows =
      env_int("IH_MIN_SEG_ROWS", H >= 256 && H <= 512 ? 8 : H > 512 && H <= 768 ? 16 : 32);
  const int64_t max_seg = (H + min_rows - 1) / min_rows;
  const bool many = units * 4 >= slots;  // >= a quarter wave without segments
  double waves = many ? 4.0 : (p.big ? 8.0 : 2.0);
  const int64_t w_env = env_int("IH_TARGET_WAVES_X10", 0);
  if (w_env > 0) waves = w_env / 10.0;
  const double raw = waves * (double)slots / (double)units;
  int64_t nseg;
  if (raw <= (double)max_seg && (slots == device_sms() || (p.colt && !many))) {
    // one CTA per SM, or few waves of column tiles: a partial last wave idles
    // whole SMs for a CTA's lifetime; pick the count in [raw/2, 2*raw] that
    // leaves the fewest idle slots (ties: fewer segments)
    int64_t best = 1;
    double best_idle = 2.0;
    const int64_t lo = (int64_t)(raw / 2) > 1 ? (int64_t)(raw / 2) : 1;
    const int64_t hi = (int64_t)(2 * raw) < max_seg ? (int64_t)(2 * raw) : max_seg;
    for (int64_t n = lo; n <= hi; ++n) {
      const double w = (double)(units * n) / (double)slots;
      const double idle = ((double)(int64_t)(w + 0.999999) - w) / (double)(int64_t)(w + 0.999999);
      if (idle < best_idle - 0.02) {
        best_idle = idle;
        best = n;
      }
    }
    nseg = best;
  } else if (raw <= (double)max_seg && !many && env_int("IH_FEW_UNITS_V1", 0) == 0) {
    // few frames x groups, several CTAs per SM: the fewest segments (>= raw/2,
    // i.e. >= about one wave) whose last wave is >= 95 % full -- every extra
    // segment costs a prologue and a carry slot, and a partly filled last
    // wave leaves its slots idle (round 2 sweep, profiles/r02h/: HD x 4
    // 19 -> 9 segments 0.735 -> 0.867 of HBM, 512^2 x 8 frames 40 -> 20)
    const int64_t lo = (int64_t)(raw / 2) > 1 ? (int64_t)(raw / 2) : 1;
    nseg = (int64_t)(raw + 0.5);
    for (int64_t n = lo; n <= max_seg && n <= (int64_t)(2 * raw) + 1; ++n) {
      const double w = (double)(units * n) / (double)slots;
      const double full = w / (double)(int64_t)(w + 0.999999);
      if (full >= 0.95) {
        nseg = n;
        break;
      }
    }
  } else if (raw <= (double)max_seg) {
    nseg = many ? (int64_t)(raw + 0.999) : (int64_t)(raw + 0.5);
  } else {
    const int64_t whole = max_seg * units / slots;  // whole waves that fit under the cap
    nseg = whole >= 1 ? whole * slots / units : max_seg;
  }
  if (nseg > max_seg) nseg = max_seg;
  if (nseg > 65535) nseg = 65535;
  if (nseg < 1) nseg = 1;
  p.slots = (int)slots;
  p.units = units;
  int32_t hinted_tail_pct = 0, hinted_tail_div = 0, hinted_flags = 0;
  const int32_t hinted =
      hint_lookup(frames, H, W, nb, &hinted_tail_pct, &hinted_tail_div, &hinted_flags);
  if (hinted > 0) nseg = hinted < H ? hinted : H;
  const int64_t forced = env_int("IH_NSEG", 0);
  if (forced > 0) nseg = forced < H ? forced : H;
  // u16 count tables: a segment has < 65536 rows; images taller than 65535
  // rows cannot use u16 prefixes, so the scan sums count slots (O(nseg^2)):
  // keep nseg small there
  if (H > 65535 && nseg > 64) nseg = 64;
  p.S = (int)((H + nseg - 1) / nseg);
  if (nseg > 1 && p.S > 65535) p.S = 65535;
  p.nseg = (int)((H + p.S - 1) / p.S);
  p.nbig = p.nseg;
  p.S2 = p.S;
  // skewed segments (IH_SKEW_X100 / hint flag kHintSkew): the first ~pct %
  // of the segments (dispatched first: the older CTA of each co-resident
  // pair, which the warp scheduler favours) get rows in the ratio skew/100
  // to the rest, so both CTAs of an SM finish together.  Measured on a
  // one-wave 4K x 16-bin grid: lower-index CTAs end at ~73 us, the younger
  // ones at ~90 us for equal work (profiles/r02e/tail_order.jsonl).
  const bool skew_hint = (hinted_flags & kHintSkew) != 0;
  const int64_t skew = env_int("IH_SKEW_X100", skew_hint ? hinted_tail_div : 0);
  const int64_t skew_pct = env_int("IH_SKEW_PCT", skew_hint ? hinted_tail_pct : 50);
  bool skewed = false;
  if (skew > 100 && skew <= 400 && skew_pct > 0 && skew_pct < 100 && p.nseg >= 2 && H <= 65535) {
    const int64_t n = p.nseg;
    int64_t nbig = (n * skew_pct + 50) / 100;
    if (nbig < 1) nbig = 1;
    if (nbig >= n) nbig = n - 1;
    // S * (nbig + (n - nbig) * 100 / skew) >= H
    const double denom = (double)nbig + (double)(n - nbig) * 100.0 / (double)skew;
    int64_t S = (int64_t)((double)H / denom) + 1;
    int64_t S2 = S * 100 / skew;
    if (S2 >= 1 && nbig * S < H && S < 65536) {
      const int64_t rem = H - nbig * S;
      p.S = (int)S;
      p.nbig = (int)nbig;
      p.S2 = (int)S2;
      p.nseg = (int)(nbig + (rem + S2 - 1) / S2);
      skewed = true;
    }
  }
  // tail split (IH_TAIL_PCT / hint): the last ~pct % of the rows become
  // segments of S/div rows, dispatched last (segment-major scan grid)
  int64_t tail_pct = skewed || skew_hint ? 0 : env_int("IH_TAIL_PCT", hinted_tail_pct);
  int64_t tail_div = env_int("IH_TAIL_DIV", hinted_tail_div > 0 ? hinted_tail_div : 4);
  if (tail_pct > 0 && tail_pct < 100 && tail_div > 1 && p.nseg > 1 && H <= 65535) {
    const int64_t s2 = (p.S + tail_div - 1) / tail_div;
    const int64_t tail_rows = H * tail_pct / 100;
    int64_t nbig = (H - tail_rows + p.S - 1) / p.S;  // big segments cover the rest
    if (nbig < 1) nbig = 1;
    if (nbig * p.S < H && s2 >= 8) {
      const int64_t rem = H - nbig * p.S;
      p.nbig = (int)nbig;
      p.S2 = (int)s2;
      p.nseg = (int)(nbig + (rem + s2 - 1) / s2);
    }
  }
  // cluster carries: the segments of a strip are one thread-block cluster
  // (<= 16 CTAs) exchanging counts through distributed shared memory -- one
  // launch, no prepass; CPL-1 512-thread kernels without column tiles, H < 65536
  const bool cluster_ok =
      !p.colt && !p.big && p.cpl == 1 && p.kb == ih::kGroup && p.nseg <= 16 && H <= 65535;
  const bool want_cluster = env_int("IH_CARRY_CLUSTER", (hinted_flags & kHintCluster) ? 1 : 0) != 0;
  if (p.nseg <= 1) p.carry = ih::CARRY_NONE;
  else if (want_cluster && cluster_ok) p.carry = ih::CARRY_CLUSTER;
  else if (p.colt) p.carry = ih::CARRY_TABLE;
  else p.carry = env_int("IH_CARRY_LOOKBACK", 0) ? ih::CARRY_LOOKBACK : ih::CARRY_TABLE;
  if (p.carry == ih::CARRY_LOOKBACK || p.carry == ih::CARRY_CLUSTER) p.staged = false;
  // K2s for images that one wave of CTAs covers: automatic unless a knob or a
  // hint chose the segmentation / carry scheme; IH_SMALL=1 or the hint flag
  // force it where it applies, IH_SMALL=0 disables it
  const int64_t small_env = env_int("IH_SMALL", -1);
  const bool auto_mode = hinted <= 0 && forced <= 0 && env_int("IH_TAIL_PCT", 0) == 0 &&
                         env_int("IH_SKEW_X100", 0) == 0 &&
                         !want_cluster && env_int("IH_CARRY_LOOKBACK", 0) == 0 &&
                         env_int("IH_STAGED_STORES", 0) == 0 && env_int("IH_COLCOUNTS_SLAB", 0) == 0 &&
                         env_int("IH_MIN_SEG_ROWS", 0) == 0 && env_int("IH_TARGET_WAVES_X10", 0) == 0;
  const bool force_small = small_env == 1 || (hinted_flags & kHintSmall);
  if (small_env != 0 && (force_small || auto_mode) && p.cpl == 1 && !p.colt)
    plan_small(p, frames, H, W, nb, force_small, forced > 0 ? forced : hinted);
  return p;
}

// Plan cache: (knob fingerprint, hint generation, device, shape, alignment).
struct PlanKey {
  uint64_t fp;
  uint32_t gen;
  int dev;
  int64_t frames, H, W;
  int nb;
  bool vec, tma;
  bool operator==(const PlanKey& o) const {
    return fp == o.fp && gen == o.gen && dev == o.dev && frames == o.frames && H == o.H &&
           W == o.W && nb == o.nb && vec == o.vec && tma == o.tma;
  }
};
struct PlanKeyHash {
  size_t operator()(const PlanKey& k) const {
    uint64_t h = k.fp ^ ((uint64_t)k.gen << 32) ^ (uint64_t)(uint32_t)k.dev;
    for (int64_t v : {k.frames, k.H, k.W, (int64_t)k.nb * 4 + k.vec * 2 + k.tma})
      h = (h ^ (uint64_t)v) * 1099511628211ull;
    return (size_t)h;
  }
};

K2Plan plan_k2(int64_t frames, int64_t H, int64_t W, int nb, bool vec, bool tma, uint64_t fp) {
  static std::mutex mu;
  static std::unordered_map<PlanKey, K2Plan, PlanKeyHash> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    dev = -1;
  }
  uint32_t gen;
  {
    std::lock_guard<std::mutex> lock(g_hint_mu);
    gen = g_hint_gen;
  }
  const PlanKey key{fp, gen, dev, frames, H, W, nb, vec, tma};
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  const K2Plan p = plan_k2_uncached(frames, H, W, nb, vec, tma);
  std::lock_guard<std::mutex> lock(mu);
  if (cache.size() >= 4096) cache.clear();
  cache.emplace(key, p);
  return p;
}
K2Plan plan_k2(int64_t frames, int64_t H, int64_t W, int nb, bool vec, bool tma) {
  return plan_k2(frames, H, W, nb, vec, tma, knob_fingerprint());
}

// Per-call knobs, re-read only when the IH_* environment changes.
struct Knobs {
  uint64_t fp = 0;
  bool valid = false;
  bool no_pdl = false, no_tma = false, colcounts_slab = false;
  int64_t table_sum_max = 24;
};
const Knobs& knobs() {
  thread_local Knobs k;
  const uint64_t fp = knob_fingerprint();
  if (!k.valid || k.fp != fp) {
    k.fp = fp;
    k.valid = true;
    k.no_pdl = env_int("IH_NO_PDL", 0) != 0;
    k.no_tma = env_int("IH_NO_TMA", 0) != 0;
    k.colcounts_slab = env_int("IH_COLCOUNTS_SLAB", 0) != 0;
    k.table_sum_max = env_int("IH_TABLE_SUM_MAX", 24);
  }
  return k;
}

int resolve_kernel(int kernel, const K2Plan& p) {
  if (kernel == IH_KERNEL_AUTO) return p.cpl ? IH_KERNEL_SINGLE_PASS : IH_KERNEL_CROSSWEAVE;
  return kernel;
}

// CARRY_TABLE with up to 24 segments skips k2_colprefix: the scan CTA of
// segment s sums the s count slots above it (L2-resident, 4 slots in flight).
// u16 prefixes need H <= 65535; taller images always sum counts in the scan.
bool table_prefix_h(const K2Plan& p, int64_t H) {
  return H <= 65535 && p.nseg > knobs().table_sum_max;
}

// Workspace layouts.
//   CARRY_TABLE:    (frames, nseg, nbp, Wp) u16 column counts (or prefixes).
//   CARRY_LOOKBACK: [ticket | pad 16 B][flags: ntiles u32, 16 B padded]
//                   [agg: ntiles x 4 x Wp u32][incl: ntiles x 4 x Wp u32]
int64_t lb_tiles(int64_t frames, const K2Plan& p) { return frames * p.ngroups * p.nseg; }
size_t lb_header_bytes(int64_t frames, const K2Plan& p) {
  return 16 + (size_t)((lb_tiles(frames, p) * 4 + 15) / 16 * 16);
}
//   column tiles:   [CARRY_TABLE table, 256 B aligned][rowleft: (frames, T-1, H, nbp) u32]
//                   [chunktot: (frames, nseg, Wp/128, nbp) u32 per-chunk table totals, nseg > 1]
size_t k2_table_bytes(int64_t frames, const K2Plan& p) {
  if (p.carry != ih::CARRY_TABLE) return 0;
  return ((size_t)frames * p.nseg * p.nbp * p.Wp * sizeof(uint16_t) + 255) / 256 * 256;
}
size_t k2_rowleft_bytes(int64_t frames, int64_t H, const K2Plan& p) {
  if (!p.colt || p.T < 2) return 0;
  return (size_t)frames * (p.T - 1) * H * p.nbp * sizeof(uint32_t);
}
size_t k2_chunktot_bytes(int64_t frames, const K2Plan& p) {
  if (!p.colt || p.T < 2 || p.carry != ih::CARRY_TABLE) return 0;
  return (size_t)frames * p.nseg * (p.Wp / ih::kChunk) * p.nbp * sizeof(uint32_t);
}
//   K2s (small):    [pad 16 B][flags: tiles u32, 16 B padded]
//                   [aggregates: tiles x 2 x TW u32], tiles = frames x groups x nseg
int64_t small_tiles(int64_t frames, const K2Plan& p) { return frames * p.ngroups * p.nseg; }
size_t small_header_bytes(int64_t frames, const K2Plan& p) {
  return 16 + (size_t)((small_tiles(frames, p) * 4 + 15) / 16 * 16);
}
size_t k2_ws_bytes(int64_t frames, int64_t H, const K2Plan& p) {
  if (p.small)
    return small_header_bytes(frames, p) +
           (size_t)small_tiles(frames, p) * 2 * p.TW * sizeof(uint32_t);
  if (p.colt)
    return k2_table_bytes(frames, p) + k2_rowleft_bytes(frames, H, p) + k2_chunktot_bytes(frames, p);
  if (p.carry == ih::CARRY_TABLE) return (size_t)frames * p.nseg * p.nbp * p.Wp * sizeof(uint16_t);
  if (p.carry == ih::CARRY_LOOKBACK)
    return lb_header_bytes(frames, p) +
           2 * (size_t)lb_tiles(frames, p) * ih::kGroup * p.Wp * sizeof(uint32_t);
  return 0;
}

struct Call {
  const uint8_t* img;
  int64_t frames, H, W, pitch, fstride;
  ih::RelLut lut;
  int nb;
  int kernel;
  K2Plan plan;
  cudaStream_t stream;
  mutable int launched = 0;  // kernels this call has launched (PDL eligibility)
  bool pdl_ok = false;       // PDL allowed (IH_NO_PDL unset)
  bool pdl() const { return pdl_ok && launched > 0; }
};

// Validation in the reference's order: shape (core.py:28-36, :72-79),
// capacity (core.py:53-57), then parameters.
ih_status validate(const uint8_t* img, int64_t frames, int64_t H, int64_t W, int64_t pitch,
                   int64_t fstride, const uint8_t* lut256, int32_t bins, int32_t bin_lo,
                   int32_t bin_hi, int32_t kernel, Call* c) {
  if (frames < 1 || H < 1 || W < 1) return fail(IH_ERR_SHAPE, "image must be a non-empty 2D array");
  if (bins < 1 || bins > 256) return fail(IH_ERR_SHAPE, "bin count must be in [1, 256]");
  if (!lut256) return fail(IH_ERR_SHAPE, "lookup table must have exactly 256 entries");
  for (int v = 0; v < 256; ++v)
    if (lut256[v] >= bins) return fail(IH_ERR_SHAPE, "lookup table entries must lie in [0, bins)");
  if (bin_lo < 0 || bin_hi > bins || bin_lo >= bin_hi)
    return fail(IH_ERR_SHAPE, "bin slab must satisfy 0 <= bin_lo < bin_hi <= bins");
  if ((uint64_t)W * (uint64_t)H > 0xffffffffull)
    return fail(IH_ERR_CAPACITY, "image exceeds the 32-bit count range");
  if (!img) return fail(IH_ERR_PARAM, "null image pointer");
  if (pitch < W) return fail(IH_ERR_PARAM, "img_pitch < width");
  if (frames > 1 && fstride < H * pitch) return fail(IH_ERR_PARAM, "frame_stride < height*img_pitch");
  if (frames > 65535) return fail(IH_ERR_PARAM, "at most 65535 frames per call");
  if (kernel < IH_KERNEL_AUTO || kernel > IH_KERNEL_CROSSWEAVE)
    return fail(IH_ERR_PARAM, "unknown kernel");
  const Knobs& kn = knobs();
  c->img = img;
  c->pdl_ok = !kn.no_pdl;
  c->frames = frames;
  c->H = H;
  c->W = W;
  c->pitch = pitch;
  c->fstride = frames > 1 ? fstride : H * pitch;
  c->nb = bin_hi - bin_lo;
  for (int v = 0; v < 256; ++v) {
    const int rel = (int)lut256[v] - bin_lo;
    c->lut.rel[v] = (rel >= 0 && rel < c->nb) ? (uint8_t)rel : (uint8_t)0xff;
  }
  // TMA bulk copies need 16-byte aligned rows; a row copy reads round_up(W, 16)
  // bytes, which stays inside the pitched row because pitch % 16 == 0.
  const bool tma = (uintptr_t)img % 16 == 0 && pitch % 16 == 0 && c->fstride % 16 == 0 &&
                   !kn.no_tma;
  c->plan = plan_k2(frames, H, W, c->nb, W % 4 == 0, tma, kn.fp);
  c->kernel = resolve_kernel(kernel, c->plan);
  if (c->kernel == IH_KERNEL_SINGLE_PASS && c->plan.cpl == 0)
    return fail(IH_ERR_PARAM, "single-pass kernel without column tiles supports width <= 8192; use crossweave");
  return IH_OK;
}

bool aligned_rows(const Call& c) {
  return ((uintptr_t)c.img % 4 == 0) && (c.pitch % 4 == 0) && (c.fstride % 4 == 0);
}


ih_status launch_colprefix(const Call& c, void* ws);

ih_status launch_prepare(const Call& c, void* ws, size_t ws_bytes) {
  if (c.kernel != IH_KERNEL_SINGLE_PASS) return IH_OK;
  const K2Plan& p = c.plan;
  const size_t need = k2_ws_bytes(c.frames, c.H, p);
  if (need == 0) return IH_OK;
  if (ws_bytes < need || !ws)
    return fail(IH_ERR_PARAM, "workspace too small (see ih_workspace_bytes)");
  if (p.small) {  // K2s: reset the aggregate flags
    if (cudaMemsetAsync(ws, 0, small_header_bytes(c.frames, p), c.stream) != cudaSuccess)
      return cuda_fail("K2s flag reset");
    return IH_OK;
  }
  if (p.colt && p.T > 1) {  // row counts left of each tile boundary
    uint32_t* lc = (uint32_t*)((uint8_t*)ws + k2_table_bytes(c.frames, p));
    dim3 grid((unsigned)((c.H + ih::kRowLeftWarps - 1) / ih::kRowLeftWarps), (unsigned)c.frames);
    if (launch(aligned_rows(c) ? ih::k2_rowleft<true> : ih::k2_rowleft<false>, grid,
               dim3(ih::kRowLeftWarps * 32), 0, c.stream, c.pdl(), c.img, c.H, c.W, c.pitch,
               c.fstride, c.lut, p.nbp, p.T, p.TW, lc) != cudaSuccess)
      return cuda_fail("k2_rowleft");
    ++c.launched;
  }
  if (p.carry == ih::CARRY_NONE) return IH_OK;
  if (p.carry == ih::CARRY_LOOKBACK) {  // reset the ticket and the tile flags
    if (cudaMemsetAsync(ws, 0, lb_header_bytes(c.frames, p), c.stream) != cudaSuccess)
      return cuda_fail("look-back flag reset");
    return IH_OK;
  }
  const bool al = aligned_rows(c);
  uint32_t* ctot = k2_chunktot_bytes(c.frames, p)
                       ? (uint32_t*)((uint8_t*)ws + k2_table_bytes(c.frames, p) +
                                     k2_rowleft_bytes(c.frames, c.H, p))
                       : nullptr;
  // column chunks per count CTA (one per warp, the other warps split the rows):
  // the largest power of two <= 8 chunks of the row whose per-chunk shared
  // tables stay <= 40 KB and whose grid still has >= 8 CTAs per SM (HD x 64 x
  // 1 bin, 20 segments: 8 chunks per CTA, 81 -> 61 us; one 4K frame of 16 bins
  // over 37 segments needs 1: 4 CTAs over 36 x 30 chunks under-fill the SMs).
  // IH_COUNT_CW forces 1/2/4/8.
  const int64_t nch = p.Wp / ih::kChunk;
  // (rows of loads in flight per warp: 8; 16 measured no faster, profiles/r02l/)
  auto count_cw = [&](size_t table_bytes) {
    const int64_t rows_of_ctas = (int64_t)(p.nseg - 1) * c.frames;
    int cw = 8;
    while (cw > 1 && (cw > nch || (size_t)cw * table_bytes > (40u << 10) ||
                      (nch + cw - 1) / cw * rows_of_ctas < 8 * (int64_t)device_sms()))
      cw >>= 1;
    const int64_t force = env_int("IH_COUNT_CW", 0);
    if (force == 1 || force == 2 || force == 4 || force == 8) cw = (int)force;
    // a forced width still has to fit the per-CTA shared tables (256 bins:
    // 66 KB per chunk; the opt-in maximum is 227 KB)
    while (cw > 1 && (size_t)cw * table_bytes > (200u << 10)) cw >>= 1;
    return cw;
  };
  if (p.nbp <= ih::kGroup && !p.colt && env_int("IH_COLCOUNTS_G1", 1) != 0 &&
      !knobs().colcounts_slab) {  // one group of <= 4 bins: counts in registers
    const int cw = count_cw(0);
    dim3 grid((unsigned)((nch + cw - 1) / cw), (unsigned)(p.nseg - 1), (unsigned)c.frames);
    auto kern = al ? ih::k2_colcounts_g1<true, 8> : ih::k2_colcounts_g1<false, 8>;
    if (launch(kern, grid, dim3(256), 0, c.stream, c.pdl(), c.img, c.H, c.W, c.pitch, c.fstride,
               c.lut, segs(p), p.nseg, p.nbp, p.Wp, cw, (uint16_t*)ws) != cudaSuccess)
      return cuda_fail("k2_colcounts_g1");
    ++c.launched;
    return launch_colprefix(c, ws);
  }
  if (!knobs().colcounts_slab) {  // all bins in one pass (shared atomics)
    const size_t table = (size_t)(p.nbp + 1) * 64 * sizeof(uint32_t);
    const int cw = count_cw(table);
    dim3 grid((unsigned)((nch + cw - 1) / cw), (unsigned)(p.nseg - 1), (unsigned)c.frames);
    auto kern = al ? ih::k2_colcounts_all<true, 8> : ih::k2_colcounts_all<false, 8>;
    const size_t smem = cw * table;
    if (!set_dyn_smem((const void*)kern, smem))
      return cuda_fail("k2_colcounts_all smem attribute");
    if (launch(kern, grid, dim3(256), smem, c.stream, c.pdl(), c.img, c.H, c.W, c.pitch,
               c.fstride, c.lut, segs(p), p.nseg, p.nbp, p.Wp, cw, (uint16_t*)ws, ctot) != cudaSuccess)
      return cuda_fail("k2_colcounts_all");
    ++c.launched;
    return launch_colprefix(c, ws);
  }
  const int nslab = (p.nbp + ih::kCountSlab - 1) / ih::kCountSlab;
  dim3 grid((unsigned)(p.Wp / ih::kChunk), (unsigned)(p.nseg - 1), (unsigned)(c.frames * nslab));
  // warps per colcounts CTA: ~48+ rows per warp, 2..8 warps
  const int nw = p.S >= 384 ? 8 : p.S >= 192 ? 4 : 2;
  auto kern = al ? (nw == 8 ? ih::k2_colcounts<true, 8>
                            : nw == 4 ? ih::k2_colcounts<true, 4> : ih::k2_colcounts<true, 2>)
                 : (nw == 8 ? ih::k2_colcounts<false, 8>
                            : nw == 4 ? ih::k2_colcounts<false, 4> : ih::k2_colcounts<false, 2>);
  const size_t smem = nw * ih::kCountWarpSmem;
  if (!set_dyn_smem((const void*)kern, smem))
    return cuda_fail("k2_colcounts smem attribute");
  if (launch(kern, grid, dim3(nw * 32), smem, c.stream, c.pdl(), c.img, c.H, c.W, c.pitch,
             c.fstride, c.lut, segs(p), p.nseg, p.nbp, p.Wp, nslab, (uint16_t*)ws, ctot) != cudaSuccess)
    return cuda_fail("k2_colcounts");
  ++c.launched;
  return launch_colprefix(c, ws);
}

ih_status launch_colprefix(const Call& c, void* ws) {
  const K2Plan& p = c.plan;
  if (!table_prefix_h(p, c.H)) return IH_OK;  // the scan kernel sums the count slots
  const int64_t total = c.frames * p.nbp * p.Wp / 4 * ih::kPrefixLanes;  // 8 lanes per quad
  int64_t blocks = (total + 255) / 256;
  if (blocks > device_sms() * 16) blocks = device_sms() * 16;
  if (launch(ih::k2_colprefix, dim3((unsigned)blocks), dim3(256), 0, c.stream, c.pdl(),
             (uint16_t*)ws, c.frames, p.nseg, p.nbp, p.Wp) != cudaSuccess)
    return cuda_fail("k2_colprefix");
  ++c.launched;
  return IH_OK;
}

ih_status launch_k2(const Call& c, const ih::ScanArgs& a, dim3 grid, int threads) {
  K2Fn fn = pick_k2(c.plan);
  if (!fn) return fail(IH_ERR_PARAM, "internal: no K2 instantiation for plan");
  const size_t smem = k2_ring_smem(c.plan);
  if (!set_dyn_smem((const void*)fn, smem))
    return cuda_fail("k2_scan smem attribute");
  // look-back carries read flags a memset just reset: never PDL there
  const bool pdl = c.pdl() && c.plan.carry != ih::CARRY_LOOKBACK;
  if (c.plan.carry == ih::CARRY_CLUSTER) {  // cluster = the segments of one strip
    if (c.plan.nseg > 8 &&
        cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
      return cuda_fail("k2_scan cluster size attribute");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = (unsigned)c.plan.nseg;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, fn, a, c.lut) != cudaSuccess) return cuda_fail("k2_scan (cluster)");
  } else if (launch(fn, grid, dim3(threads), smem, c.stream, pdl, a, c.lut) != cudaSuccess) {
    return cuda_fail("k2_scan");
  }
  ++c.launched;
  return IH_OK;
}

ih_status launch_scan(const Call& c, uint32_t* out, void* ws, size_t ws_bytes) {
  if (!out) return fail(IH_ERR_PARAM, "null output pointer");
  if (c.kernel == IH_KERNEL_CROSSWEAVE) {
    const int ngroups = (c.nb + ih::kGroup - 1) / ih::kGroup;
    dim3 grid((unsigned)ngroups, (unsigned)((c.H + 7) / 8), (unsigned)c.frames);
    if (grid.y > 65535) return fail(IH_ERR_PARAM, "crossweave kernel supports height <= 524280");
    const bool vec = (c.W % 4) == 0, al = aligned_rows(c);
    if (vec && al) ih::k1_rowscan<true, true><<<grid, 256, 0, c.stream>>>(c.img, c.H, c.W, c.pitch, c.fstride, c.nb, c.lut, out);
    else if (vec) ih::k1_rowscan<true, false><<<grid, 256, 0, c.stream>>>(c.img, c.H, c.W, c.pitch, c.fstride, c.nb, c.lut, out);
    else if (al) ih::k1_rowscan<false, true><<<grid, 256, 0, c.stream>>>(c.img, c.H, c.W, c.pitch, c.fstride, c.nb, c.lut, out);
    else ih::k1_rowscan<false, false><<<grid, 256, 0, c.stream>>>(c.img, c.H, c.W, c.pitch, c.fstride, c.nb, c.lut, out);
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k1_rowscan");
    const int64_t planes = c.frames * c.nb;
    const int64_t per = vec ? c.W / 4 : c.W;
    int64_t blocks = (planes * per + 255) / 256;
    if (blocks > device_sms() * 32) blocks = device_sms() * 32;
    if (c.H > 1) {
      if (vec) ih::k1b_colscan<true><<<(unsigned)blocks, 256, 0, c.stream>>>(out, planes, c.H, c.W);
      else ih::k1b_colscan<false><<<(unsigned)blocks, 256, 0, c.stream>>>(out, planes, c.H, c.W);
      if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k1b_colscan");
    }
    return IH_OK;
  }
  const K2Plan& p = c.plan;
  if (k2_ws_bytes(c.frames, c.H, p) > 0 && (ws_bytes < k2_ws_bytes(c.frames, c.H, p) || !ws))
    return fail(IH_ERR_PARAM, "workspace too small (see ih_workspace_bytes)");
  if (p.small) {
    ih::SmallArgs a;
    a.img = c.img;
    a.H = c.H;
    a.W = c.W;
    a.pitch = c.pitch;
    a.fstride = c.fstride;
    a.nb = c.nb;
    a.ngroups = p.ngroups;
    a.nseg = p.nseg;
    a.S = p.S;
    a.Sk = p.Sk;
    a.wpg = p.nwarps / p.nwg;
    a.TWp = p.TW;
    a.contig = small_contig(p, c.pitch) ? 1 : 0;
    a.RS = a.contig ? (int)c.pitch : p.TW;
    a.row_bytes = (uint32_t)((c.W + 15) / 16 * 16);
    uint8_t* base = (uint8_t*)ws;
    a.flags = (uint32_t*)(base + 16);
    a.agg = (uint32_t*)(base + small_header_bytes(c.frames, p));
    a.out = out;
    const int64_t tiles = small_tiles(c.frames, p);
    a.trace = (g_trace && 2 * (size_t)tiles <= g_trace_ctas) ? g_trace : nullptr;
    KSFn fn = pick_small(p);
    const size_t smem = small_smem(p, c.pitch);
    if (!set_dyn_smem((const void*)fn, smem)) return cuda_fail("k2_small smem attribute");
    // after the flag memset: no PDL
    if (launch(fn, dim3((unsigned)tiles), dim3(p.nwarps * 32), smem, c.stream, false, a, c.lut) !=
        cudaSuccess)
      return cuda_fail("k2_small");
    ++c.launched;
    return IH_OK;
  }
  ih::ScanArgs a;
  a.img = c.img;
  a.H = c.H;
  a.W = c.W;
  a.pitch = c.pitch;
  a.fstride = c.fstride;
  a.nb = c.nb;
  a.nbp = p.nbp;
  a.sg = segs(p);
  a.nseg = p.nseg;
  a.Wp = p.Wp;
  a.T = p.T;
  a.TW = p.TW;
  a.row_bytes = (uint32_t)((c.W + 15) / 16 * 16);
  a.rowleft = p.colt && p.T > 1 ? (const uint32_t*)((const uint8_t*)ws + k2_table_bytes(c.frames, p))
                                : nullptr;
  a.chunktot = k2_chunktot_bytes(c.frames, p)
                   ? (const uint32_t*)((const uint8_t*)a.rowleft + k2_rowleft_bytes(c.frames, c.H, p))
                   : nullptr;
  a.colpre = p.carry == ih::CARRY_TABLE ? (const uint16_t*)ws : nullptr;
  a.table_is_prefix = table_prefix_h(p, c.H) ? 1 : 0;
  a.lb_ticket = a.lb_flags = a.lb_agg = a.lb_incl = nullptr;
  if (p.carry == ih::CARRY_LOOKBACK) {
    uint8_t* base = (uint8_t*)ws;
    a.lb_ticket = (uint32_t*)base;
    a.lb_flags = (uint32_t*)(base + 16);
    a.lb_agg = (uint32_t*)(base + lb_header_bytes(c.frames, p));
    a.lb_incl = a.lb_agg + lb_tiles(c.frames, p) * ih::kGroup * p.Wp;
  }
  a.out = out;
  // segment-major: (units, frames, segments); look-back decodes its own ticket
  dim3 grid((unsigned)(p.ngroups * p.T), (unsigned)c.frames, (unsigned)p.nseg);
  if (p.carry == ih::CARRY_LOOKBACK)
    grid = dim3((unsigned)(p.ngroups * p.T), (unsigned)p.nseg, (unsigned)c.frames);
  a.trace = (g_trace && (size_t)grid.x * grid.y * grid.z <= g_trace_ctas) ? g_trace : nullptr;
  const int threads = p.nwarps * 32;
  return launch_k2(c, a, grid, threads);
}

}  // namespace

extern "C" {

size_t ih_workspace_bytes(int64_t frames, int64_t height, int64_t width, int32_t slab_bins,
                          int32_t kernel) {
  if (frames < 1 || height < 1 || width < 1 || slab_bins < 1) return 0;
  // the plan depends on the input alignment (1024-thread variants need the TMA
  // path); size the workspace for either
  size_t n = 0;
  const uint64_t fp = knob_fingerprint();
  for (int variant = 0; variant < 4; ++variant) {
    K2Plan p = plan_k2(frames, height, width, slab_bins, width % 4 == 0 && (variant & 1),
                       (variant & 2) != 0, fp);
    if (resolve_kernel(kernel, p) != IH_KERNEL_SINGLE_PASS || p.cpl == 0) continue;
    const size_t b = k2_ws_bytes(frames, height, p);
    if (b > n) n = b;
  }
  return n;
}

// Buffer alignment the kernels rely on: 16-byte output stores when every row
// starts 16-byte aligned (width % 4 == 0), 4-byte elements otherwise; uint4
// workspace slots.  Checked before any launch: a misaligned vector store
// would fault and poison the caller's CUDA context.
ih_status check_buffers(const Call& c, const void* out, bool need_out, const void* ws) {
  if (need_out) {
    if (!out) return fail(IH_ERR_PARAM, "null output pointer");
    const uintptr_t a = c.W % 4 == 0 ? 15u : 3u;
    if ((uintptr_t)out & a)
      return fail(IH_ERR_PARAM, c.W % 4 == 0 ? "out must be 16-byte aligned when width % 4 == 0"
                                             : "out must be 4-byte aligned");
  }
  if (ws && ((uintptr_t)ws & 15)) return fail(IH_ERR_PARAM, "workspace must be 16-byte aligned");
  return IH_OK;
}

ih_status ih_ih_prepare(const uint8_t* img, int64_t frames, int64_t height, int64_t width,
                        int64_t img_pitch, int64_t frame_stride, const uint8_t* lut256,
                        int32_t bins, int32_t bin_lo, int32_t bin_hi, void* workspace,
                        size_t workspace_bytes, int32_t kernel, void* stream) {
  Call c;
  ih_status st = validate(img, frames, height, width, img_pitch, frame_stride, lut256, bins,
                          bin_lo, bin_hi, kernel, &c);
  if (st != IH_OK) return st;
  st = check_buffers(c, nullptr, false, workspace);
  if (st != IH_OK) return st;
  c.stream = (cudaStream_t)stream;
  return launch_prepare(c, workspace, workspace_bytes);
}

ih_status ih_ih_scan(const uint8_t* img, int64_t frames, int64_t height, int64_t width,
                     int64_t img_pitch, int64_t frame_stride, const uint8_t* lut256, int32_t bins,
                     int32_t bin_lo, int32_t bin_hi, uint32_t* out, void* workspace,
                     size_t workspace_bytes, int32_t kernel, void* stream) {
  Call c;
  ih_status st = validate(img, frames, height, width, img_pitch, frame_stride, lut256, bins,
                          bin_lo, bin_hi, kernel, &c);
  if (st != IH_OK) return st;
  st = check_buffers(c, out, true, workspace);
  if (st != IH_OK) return st;
  c.stream = (cudaStream_t)stream;
  return launch_scan(c, out, workspace, workspace_bytes);
}

ih_status ih_integral_histogram(const uint8_t* img, int64_t frames, int64_t height, int64_t width,
                                int64_t img_pitch, int64_t frame_stride, const uint8_t* lut256,
                                int32_t bins, int32_t bin_lo, int32_t bin_hi, uint32_t* out,
                                void* workspace, size_t workspace_bytes, int32_t kernel,
                                void* stream) {
  Call c;
  ih_status st = validate(img, frames, height, width, img_pitch, frame_stride, lut256, bins,
                          bin_lo, bin_hi, kernel, &c);
  if (st != IH_OK) return st;
  st = check_buffers(c, out, true, workspace);
  if (st != IH_OK) return st;
  c.stream = (cudaStream_t)stream;
  st = launch_prepare(c, workspace, workspace_bytes);
  if (st != IH_OK) return st;
  return launch_scan(c, out, workspace, workspace_bytes);
}

ih_status ih_region_histograms(const uint32_t* t, int32_t nb, int64_t height, int64_t width,
                               const int32_t* regions, int64_t q, uint64_t* out, void* stream) {
  if (nb < 1 || height < 1 || width < 1) return fail(IH_ERR_SHAPE, "tensor must be non-empty");
  if (q < 0) return fail(IH_ERR_PARAM, "negative query count");
  if (q == 0) return IH_OK;
  if (!t || !regions || !out) return fail(IH_ERR_PARAM, "null pointer");
  if ((uintptr_t)regions % 16 != 0) return fail(IH_ERR_PARAM, "regions must be 16-byte aligned");
  int64_t blocks = (q + 7) / 8;  // 8 warps per CTA, one query per warp
  if (blocks > device_sms() * 64) blocks = device_sms() * 64;
  ih::k3_region_histograms<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      t, nb, height, width, reinterpret_cast<const int4*>(regions), q,
      reinterpret_cast<unsigned long long*>(out));
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k3_region_histograms");
  return IH_OK;
}

ih_status ih_window_counts(const uint32_t* t, int32_t nb, int64_t height, int64_t width, int32_t h,
                           int32_t w, int64_t* out, void* stream) {
  if (h < 1 || w < 1) return fail(IH_ERR_PARAM, "window extents must be >= 1");
  if (h > height || w > width) return fail(IH_ERR_BOUNDS, "window exceeds image");
  if (nb < 1) return fail(IH_ERR_SHAPE, "tensor must be non-empty");
  if (!t || !out) return fail(IH_ERR_PARAM, "null pointer");
  if (nb > 65535) return fail(IH_ERR_PARAM, "too many bins");
  const int64_t R = height - h + 1, C = width - w + 1;
  const int threads = C >= 1024 ? 256 : (int)((C + 127) / 128 * 32);
  const size_t smem = (size_t)(4 * threads + w) * sizeof(uint32_t);
  // IH_K4_MODE 3: pairs of adjacent outputs per 16-byte store;
  // 1: 4 strided outputs per thread; 0: the two-output kernel; 2: staged row
  // differences (while CW + w u32 fit in shared memory)
  // mode 3's 16-byte pair stores need a 16-byte aligned `out`; int64 views
  // at odd element offsets take the 8-byte-store kernel (mode 1)
  // mode 4 (default where it applies): 4 adjacent outputs per thread from
  // 16-byte corner loads -- needs 16-byte aligned tensor rows (W % 4 == 0)
  // and a 16-byte aligned `out`; otherwise mode 3
  int64_t k4mode = env_int("IH_K4_MODE", 4);
  if (k4mode == 4 && (width % 4 != 0 || ((uintptr_t)t & 15) || ((uintptr_t)out & 15))) k4mode = 3;
  // modes 2 and 3 store 16-byte pairs: an `out` 8 bytes past a 16-byte
  // boundary takes the 8-byte-store kernel
  if ((k4mode == 2 || k4mode == 3) && ((uintptr_t)out & 15)) k4mode = 1;
  if ((uintptr_t)out & 7) return fail(IH_ERR_PARAM, "out must be 8-byte aligned");
  if (k4mode == 4) {
    const int64_t cb = (C + 4 * 256 - 1) / (4 * 256);
    int64_t ry = (int64_t)device_sms() * env_int("IH_K4_CTAS_PER_SM", 256) / (cb * nb);
    ry = ry < 1 ? 1 : ry > R ? R : ry > 65535 ? 65535 : ry;
    dim3 grid((unsigned)cb, (unsigned)ry, (unsigned)nb);
    const int m = (w - 1) & 3;
    auto k = m == 0 ? ih::k4_window_counts_quads<0> : m == 1 ? ih::k4_window_counts_quads<1>
           : m == 2 ? ih::k4_window_counts_quads<2> : ih::k4_window_counts_quads<3>;
    k<<<grid, 256, 0, (cudaStream_t)stream>>>(t, nb, height, width, h, w,
                                             reinterpret_cast<long long*>(out));
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k4_window_counts_quads");
    return IH_OK;
  }
  if (k4mode == 3) {  // two adjacent outputs per 16-byte store
    const int U = env_int("IH_K4_PAIRS_U", 2) == 4 ? 4 : env_int("IH_K4_PAIRS_U", 2) == 1 ? 1 : 2;
    const int64_t cb = (C + 1 + 2 * 256 * U - 1) / (2 * 256 * U);  // U pairs per thread
    // grid-strided rows, ~256 CTAs' worth per SM (measured best: HD x32 64x64
    // windows 0.164 -> 0.148 ms vs mode 1; profiles/r01f/queries_k4_pairs.jsonl)
    int64_t ry = (int64_t)device_sms() * env_int("IH_K4_CTAS_PER_SM", 256) / (cb * nb);
    ry = ry < 1 ? 1 : ry > R ? R : ry > 65535 ? 65535 : ry;
    dim3 grid((unsigned)cb, (unsigned)ry, (unsigned)nb);
    auto k = U == 4 ? ih::k4_window_counts_pairs<4> : U == 1 ? ih::k4_window_counts_pairs<1>
                                                            : ih::k4_window_counts_pairs<2>;
    k<<<grid, 256, 0, (cudaStream_t)stream>>>(t, nb, height, width, h, w,
                                             reinterpret_cast<long long*>(out));
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k4_window_counts_pairs");
    return IH_OK;
  }
  if (k4mode == 1) {
    // rows are grid-strided over ~64 CTAs per SM in total, so each CTA walks
    // several rows (one-row CTAs: 0.52 of HBM, 148*64 CTAs: 0.59, HD x32;
    // with u32 window arithmetic and <= 40 registers: 0.70)
    const int64_t cb = (C + 1023) / 1024;
    int64_t ry = (int64_t)device_sms() * 64 / (cb * nb);
    ry = ry < 1 ? 1 : ry > R ? R : ry > 65535 ? 65535 : ry;
    ry = env_int("IH_K4_ROWS_GRID", ry);
    dim3 grid((unsigned)cb, (unsigned)ry, (unsigned)nb);
    // IH_K4_VARIANT = U*10 + min CTAs/SM (A/B; 46 measured best, profiles/r01f/queries_k4_variants.jsonl)
    const int64_t v = env_int("IH_K4_VARIANT", 46);
    auto k = v == 48 ? ih::k4_window_counts_ilp<4, 8> : v == 28 ? ih::k4_window_counts_ilp<2, 8>
           : v == 86 ? ih::k4_window_counts_ilp<8, 6> : v == 84 ? ih::k4_window_counts_ilp<8, 4>
                     : ih::k4_window_counts_ilp<4, 6>;
    const int U = v / 10 == 2 ? 2 : v / 10 == 8 ? 8 : 4;
    grid.x = (unsigned)((C + 256 * U - 1) / (256 * U));
    k<<<grid, 256, 0, (cudaStream_t)stream>>>(t, nb, height, width, h, w,
                                            reinterpret_cast<long long*>(out));
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k4_window_counts_ilp");
    return IH_OK;
  }
  if (smem <= 160 * 1024 && k4mode == 2) {
    auto k = ih::k4_window_counts_vs;
    if (!set_dyn_smem((const void*)k, smem))
      return cuda_fail("k4 smem attribute");
    const int64_t cblocks = (C + 4 * threads - 1) / (4 * threads);
    dim3 grid((unsigned)cblocks, (unsigned)(R < 65535 ? R : 65535), (unsigned)nb);
    k<<<grid, threads, smem, (cudaStream_t)stream>>>(t, nb, height, width, h, w,
                                                     reinterpret_cast<long long*>(out));
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k4_window_counts_vs");
    return IH_OK;
  }
  dim3 grid((unsigned)((C + 511) / 512), (unsigned)(R < 65535 ? R : 65535), (unsigned)nb);
  ih::k4_window_counts<<<grid, 256, 0, (cudaStream_t)stream>>>(
      t, nb, height, width, h, w, reinterpret_cast<long long*>(out));
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k4_window_counts");
  return IH_OK;
}

ih_status ih_plan_describe(int64_t frames, int64_t height, int64_t width, int32_t slab_bins,
                           int32_t kernel, int32_t aligned16, int64_t* info) {
  if (frames < 1 || height < 1 || width < 1) return fail(IH_ERR_SHAPE, "image must be non-empty");
  if (slab_bins < 1 || slab_bins > 256) return fail(IH_ERR_SHAPE, "bin count must be in [1, 256]");
  if ((uint64_t)width * (uint64_t)height > 0xffffffffull)
    return fail(IH_ERR_CAPACITY, "image exceeds the 32-bit count range");
  if (kernel < IH_KERNEL_AUTO || kernel > IH_KERNEL_CROSSWEAVE)
    return fail(IH_ERR_PARAM, "unknown kernel");
  if (!info) return fail(IH_ERR_PARAM, "null info pointer");
  const bool tma = aligned16 != 0 && !knobs().no_tma;
  K2Plan p = plan_k2(frames, height, width, slab_bins, width % 4 == 0, tma);
  const int k = resolve_kernel(kernel, p);
  for (int i = 0; i < 16; ++i) info[i] = 0;
  info[0] = k;
  if (k == IH_KERNEL_CROSSWEAVE) {
    info[1] = height > 1 ? 2 : 1;
    return IH_OK;
  }
  if (p.cpl == 0) return fail(IH_ERR_PARAM, "single-pass kernel supports width <= 8192");
  int launches = 1;  // K2s: one kernel (after a memset of its flags)
  if (p.carry == ih::CARRY_TABLE) launches += table_prefix_h(p, height) ? 2 : 1;
  if (p.colt && p.T > 1) launches += 1;  // k2_rowleft
  info[1] = launches;
  info[2] = p.nseg;
  info[3] = p.S;
  info[4] = p.cpl;
  info[5] = p.R;
  info[6] = p.nwarps;
  info[7] = (int64_t)k2_ws_bytes(frames, height, p);
  info[8] = p.T;
  info[9] = p.TW;
  info[10] = p.slots;
  info[11] = p.units;
  info[12] = p.nbig;
  info[13] = p.S2;
  info[14] = p.small ? 4 : p.carry;  // ih::Carry, 4 = K2s in-kernel carries
  info[15] = p.kb;
  return IH_OK;
}

size_t ih_likelihood_workspace_bytes(int32_t nb, int32_t h, int32_t w) {
  if (nb < 1 || nb > 256 || h < 1 || w < 1) return 0;
  const uint64_t bytes = (uint64_t)nb * ((uint64_t)h * (uint64_t)w + 1) * sizeof(double);
  return bytes <= (512ull << 20) ? (size_t)bytes : 0;  // no table for huge windows
}

ih_status ih_likelihood_map(const uint32_t* t, int32_t nb, int64_t height, int64_t width,
                            int32_t h, int32_t w, const double* template_host, int32_t metric,
                            double* out, void* stream) {
  return ih_likelihood_map_ws(t, nb, height, width, h, w, template_host, metric, out, nullptr, 0,
                              stream);
}

ih_status ih_likelihood_map_ws(const uint32_t* t, int32_t nb, int64_t height, int64_t width,
                               int32_t h, int32_t w, const double* template_host, int32_t metric,
                               double* out, void* workspace, size_t workspace_bytes,
                               void* stream) {
  if (nb < 1 || nb > 256) return fail(IH_ERR_SHAPE, "bin count must be in [1, 256]");
  if (!template_host) return fail(IH_ERR_SHAPE, "null template");
  if (metric != IH_METRIC_INTERSECTION && metric != IH_METRIC_BHATTACHARYYA)
    return fail(IH_ERR_PARAM, "unknown metric");
  if (h < 1 || w < 1) return fail(IH_ERR_PARAM, "window extents must be >= 1");
  if (h > height || w > width) return fail(IH_ERR_BOUNDS, "window exceeds image");
  if (!t || !out) return fail(IH_ERR_PARAM, "null pointer");
  ih::Template tpl;
  for (int b = 0; b < 256; ++b) tpl.t[b] = b < nb ? template_host[b] : 0.0;
  const int64_t R = height - h + 1, C = width - w + 1;
  const size_t tab = ih_likelihood_workspace_bytes(nb, h, w);
  if (tab && workspace && workspace_bytes >= tab && env_int("IH_K5_DIRECT", 0) == 0) {
    double* M = (double*)workspace;
    const int64_t total = (int64_t)nb * ((int64_t)h * w + 1);
    int64_t blocks = (total + 255) / 256;
    if (blocks > device_sms() * 16) blocks = device_sms() * 16;
    if (metric == IH_METRIC_INTERSECTION)
      ih::k5_metric_table<true><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
          tpl, nb, (int64_t)h * w, M);
    else
      ih::k5_metric_table<false><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
          tpl, nb, (int64_t)h * w, M);
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k5_metric_table");
    const int64_t P = env_int("IH_K5_PAIRS", 2);  // placements per thread (32 apart)
    // output rows h apart per thread (2: HD x32 64x64 0.1003 -> 0.0992 ms,
    // 8x8 0.1068 -> 0.0981; 4 / 8 spill: profiles/r02h/k5_chain.jsonl)
    const int64_t KC = env_int("IH_K5_CHAIN", 2);
    if ((KC == 2 || KC == 4 || KC == 8) && (P == 2 || P == 4)) {
      const int64_t nchains = (R + (int64_t)h * KC - 1) / ((int64_t)h * KC) * h;
      dim3 grid((unsigned)((C + 256 * P - 1) / (256 * P)), (unsigned)(nchains < 65535 ? nchains : 65535));
      auto k = KC == 2 ? (P == 4 ? ih::k5_likelihood_map_chain<2, 4> : ih::k5_likelihood_map_chain<2, 2>)
             : KC == 4 ? (P == 4 ? ih::k5_likelihood_map_chain<4, 4> : ih::k5_likelihood_map_chain<4, 2>)
                       : ih::k5_likelihood_map_chain<8, 2>;  // (K = 8 only with P = 2)
      k<<<grid, 256, 0, (cudaStream_t)stream>>>(t, nb, height, width, h, w, M, out);
      if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k5_likelihood_map_chain");
      return IH_OK;
    }
    if (P == 2 || P == 4) {
      dim3 grid((unsigned)((C + 256 * P - 1) / (256 * P)), (unsigned)(R < 65535 ? R : 65535));
      // bins per step (P = 2): 2 -> 48 registers, the best occupancy / MLP
      // balance (HD x32 64x64: U 2 / 4 / 8 = 0.0996 / 0.108 / 0.101 ms)
      const int64_t ub = env_int("IH_K5_U", 2);
      auto k = P == 4 ? ih::k5_likelihood_map_tabp<4>
             : ub == 8 ? ih::k5_likelihood_map_tabp<2, 8>
             : ub == 2 ? ih::k5_likelihood_map_tabp<2, 2> : ih::k5_likelihood_map_tabp<2, 4>;
      k<<<grid, 256, 0, (cudaStream_t)stream>>>(t, nb, height, width, h, w, M, out);
      if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k5_likelihood_map_tabp");
      return IH_OK;
    }
    dim3 grid((unsigned)((C + 255) / 256), (unsigned)(R < 65535 ? R : 65535));
    ih::k5_likelihood_map_tab<<<grid, 256, 0, (cudaStream_t)stream>>>(t, nb, height, width, h, w,
                                                                      M, out);
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k5_likelihood_map_tab");
    return IH_OK;
  }
  // one row per CTA: K5 is FP64-issue bound (a true division and a sqrt per
  // placement and bin) and wants every warp slot filled
  dim3 grid((unsigned)((C + 255) / 256), (unsigned)(R < 65535 ? R : 65535));
  if (metric == IH_METRIC_INTERSECTION)
    ih::k5_likelihood_map<true><<<grid, 256, 0, (cudaStream_t)stream>>>(t, nb, height, width, h,
                                                                        w, tpl, out);
  else
    ih::k5_likelihood_map<false><<<grid, 256, 0, (cudaStream_t)stream>>>(t, nb, height, width,
                                                                         h, w, tpl, out);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k5_likelihood_map");
  return IH_OK;
}

ih_status ih_plan_hint(int64_t frames, int64_t height, int64_t width, int32_t slab_bins,
                       int32_t nseg, int32_t tail_pct, int32_t tail_div, int32_t flags) {
  if (frames < 1 || height < 1 || width < 1) return fail(IH_ERR_SHAPE, "image must be non-empty");
  if (slab_bins < 1 || slab_bins > 256) return fail(IH_ERR_SHAPE, "bin count must be in [1, 256]");
  if (nseg < 0) return fail(IH_ERR_PARAM, "negative segment count");
  if (tail_pct < 0 || tail_pct >= 100 || tail_div < 0)
    return fail(IH_ERR_PARAM, "tail split must satisfy 0 <= pct < 100, div >= 0");
  std::lock_guard<std::mutex> lock(g_hint_mu);
  for (int i = 0; i < g_nhints; ++i) {
    PlanHint& h = g_hints[i];
    if (h.frames == frames && h.H == height && h.W == width && h.nb == slab_bins) {
      if (nseg > 0) {
        h.nseg = nseg;
        h.tail_pct = tail_pct;
        h.tail_div = tail_div;
        h.flags = flags;
      } else {
        h = g_hints[--g_nhints];
      }
      ++g_hint_gen;
      return IH_OK;
    }
  }
  if (nseg == 0) return IH_OK;
  ++g_hint_gen;
  if (g_nhints == kMaxHints) g_nhints = 0;  // a small cache: start over when full
  g_hints[g_nhints++] = PlanHint{frames, height, width, slab_bins, nseg, tail_pct, tail_div, flags};
  return IH_OK;
}

size_t ih_scan_workspace_bytes(int64_t n) {
  const int64_t tiles = n > 0 ? (n + ih::kScanTile - 1) / ih::kScanTile : 0;
  return (size_t)(tiles > 0 ? tiles : 1) * sizeof(uint64_t);
}

ih_status ih_scan_u64(const uint64_t* in, int64_t n, uint32_t* out, int32_t exclusive,
                      uint32_t* overflow, void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 0) return fail(IH_ERR_PARAM, "n must be >= 0");
  if (n == 0) return IH_OK;
  if (!in || !out || !workspace) return fail(IH_ERR_PARAM, "null pointer");
  if (workspace_bytes < ih_scan_workspace_bytes(n) || ((uintptr_t)workspace & 7))
    return fail(IH_ERR_PARAM, "scan workspace too small or misaligned");
  const int64_t tiles = (n + ih::kScanTile - 1) / ih::kScanTile;
  if (tiles > 0x7fffffffLL) return fail(IH_ERR_PARAM, "n too large");
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t* totals = static_cast<uint64_t*>(workspace);
  const bool v2 = ((uintptr_t)in & 15) == 0, v4 = ((uintptr_t)out & 15) == 0;
  const dim3 grid((unsigned)tiles);
  if (v2)
    ih::k6_block_totals<true><<<grid, ih::kScanThreads, 0, s>>>(in, n, totals);
  else
    ih::k6_block_totals<false><<<grid, ih::kScanThreads, 0, s>>>(in, n, totals);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k6_block_totals");
  ih::k6_scan_totals<<<1, ih::kScanThreads, 0, s>>>(totals, tiles, overflow);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k6_scan_totals");
  auto k = v2 ? (v4 ? ih::k6_scan_apply<true, true> : ih::k6_scan_apply<true, false>)
              : (v4 ? ih::k6_scan_apply<false, true> : ih::k6_scan_apply<false, false>);
  k<<<grid, ih::kScanThreads, 0, s>>>(in, n, totals, exclusive ? 1 : 0, out, overflow);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k6_scan_apply");
  return IH_OK;
}

ih_status ih_scan_axis_u32(const void* in, int32_t elem_bytes, int64_t outer, int64_t n,
                           int64_t inner, uint32_t* out, void* stream) {
  if (outer < 0 || n < 0 || inner < 0) return fail(IH_ERR_PARAM, "extents must be >= 0");
  if (elem_bytes != 1 && elem_bytes != 4) return fail(IH_ERR_PARAM, "elem_bytes must be 1 or 4");
  if (outer == 0 || n == 0 || inner == 0) return IH_OK;
  if (!in || !out) return fail(IH_ERR_PARAM, "null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  if (inner == 1) {
    const int64_t blocks = (outer + 7) / 8;
    if (blocks > 0x7fffffffLL) return fail(IH_ERR_PARAM, "too many rows");
    // vector path: every row start 16-byte aligned (u32) / 4-byte aligned (u8)
    const bool vec = n % 4 == 0 && ((uintptr_t)in % (elem_bytes * 4)) == 0 &&
                     ((uintptr_t)out & 15) == 0;
    const unsigned g = (unsigned)blocks;
    if (elem_bytes == 1) {
      auto k = vec ? ih::k6_scan_inner<uint8_t, true> : ih::k6_scan_inner<uint8_t, false>;
      k<<<g, 256, 0, s>>>(static_cast<const uint8_t*>(in), outer, n, out);
    } else {
      auto k = vec ? ih::k6_scan_inner<uint32_t, true> : ih::k6_scan_inner<uint32_t, false>;
      k<<<g, 256, 0, s>>>(static_cast<const uint32_t*>(in), outer, n, out);
    }
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k6_scan_inner");
    return IH_OK;
  }
  const int64_t bx = (inner + 31) / 32;
  if (bx > 0x7fffffffLL) return fail(IH_ERR_PARAM, "too many columns");
  const dim3 grid((unsigned)bx, (unsigned)(outer < 65535 ? outer : 65535));
  if (elem_bytes == 1)
    ih::k6_scan_strided<uint8_t><<<grid, 1024, 0, s>>>(static_cast<const uint8_t*>(in), outer, n,
                                                       inner, out);
  else
    ih::k6_scan_strided<uint32_t><<<grid, 1024, 0, s>>>(static_cast<const uint32_t*>(in), outer,
                                                        n, inner, out);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k6_scan_strided");
  return IH_OK;
}

ih_status ih_transpose(const void* in, int64_t rows, int64_t cols, int32_t elem_bytes, void* out,
                       void* stream) {
  if (rows < 0 || cols < 0) return fail(IH_ERR_PARAM, "extents must be >= 0");
  if (rows == 0 || cols == 0) return IH_OK;
  if (!in || !out) return fail(IH_ERR_PARAM, "null pointer");
  const int64_t bx = (cols + 31) / 32, by = (rows + 31) / 32;
  if (bx > 0x7fffffffLL) return fail(IH_ERR_PARAM, "too many columns");
  const dim3 grid((unsigned)bx, (unsigned)(by < 65535 ? by : 65535));
  cudaStream_t s = (cudaStream_t)stream;
  switch (elem_bytes) {
    case 1: ih::k6_transpose<uint8_t><<<grid, 256, 0, s>>>((const uint8_t*)in, rows, cols, (uint8_t*)out); break;
    case 2: ih::k6_transpose<uint16_t><<<grid, 256, 0, s>>>((const uint16_t*)in, rows, cols, (uint16_t*)out); break;
    case 4: ih::k6_transpose<uint32_t><<<grid, 256, 0, s>>>((const uint32_t*)in, rows, cols, (uint32_t*)out); break;
    case 8: ih::k6_transpose<uint64_t><<<grid, 256, 0, s>>>((const uint64_t*)in, rows, cols, (uint64_t*)out); break;
    case 16:
      if (((uintptr_t)in | (uintptr_t)out) & 15) return fail(IH_ERR_PARAM, "16-byte elements need 16-byte alignment");
      ih::k6_transpose<uint4><<<grid, 256, 0, s>>>((const uint4*)in, rows, cols, (uint4*)out);
      break;
    default: return fail(IH_ERR_PARAM, "elem_bytes must be 1, 2, 4, 8 or 16");
  }
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k6_transpose");
  return IH_OK;
}

size_t ih_wavefront_workspace_bytes(int64_t height, int64_t width, int32_t tile) {
  if (height < 1 || width < 1 || tile < 1) return 0;
  const int64_t ntiles = ((height + tile - 1) / tile) * ((width + tile - 1) / tile);
  return 16 + (size_t)(ntiles * 4 + 15) / 16 * 16;
}

ih_status ih_wavefront(const uint8_t* img, int64_t height, int64_t width, int64_t img_pitch,
                       const uint8_t* lut256, int32_t bins, int32_t tile, uint32_t* out,
                       uint32_t* events, void* workspace, size_t workspace_bytes, void* stream) {
  if (tile < 1) return fail(IH_ERR_PARAM, "tile must be >= 1");  // strategies.py:185-186
  Call c;
  ih_status st = validate(img, 1, height, width, img_pitch, height * img_pitch, lut256, bins, 0,
                          bins, IH_KERNEL_AUTO, &c);
  if (st != IH_OK) return st;
  if (!out || !events) return fail(IH_ERR_PARAM, "null pointer");
  const int64_t ni = (height + tile - 1) / tile, nj = (width + tile - 1) / tile;
  if (ni * nj > 0x7fffffffLL) return fail(IH_ERR_PARAM, "too many tiles");
  const size_t need = ih_wavefront_workspace_bytes(height, width, tile);
  if (!workspace || workspace_bytes < need)
    return fail(IH_ERR_PARAM, "workspace too small (see ih_wavefront_workspace_bytes)");
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(workspace, 0, need, s) != cudaSuccess) return cuda_fail("wavefront reset");
  ih::WfArgs a;
  a.img = img;
  a.H = height;
  a.W = width;
  a.pitch = img_pitch;
  a.nb = bins;
  a.tile = tile;
  a.ni = ni;
  a.nj = nj;
  a.ticket = (uint32_t*)workspace;
  a.seq = a.ticket + 1;
  a.flags = (uint32_t*)((uint8_t*)workspace + 16);
  a.ev = events;
  a.out = out;
  ih::k7_wavefront<<<(unsigned)(ni * nj), ih::kWfWarps * 32, 0, s>>>(a, c.lut);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k7_wavefront");
  return IH_OK;
}

void ih_debug_trace(void* device_buffer, size_t ctas) {
  g_trace = (unsigned long long*)device_buffer;
  g_trace_ctas = device_buffer ? ctas : 0;
}

const char* ih_status_string(ih_status s) {
  switch (s) {
    case IH_OK: return "IH_OK";
    case IH_ERR_SHAPE: return "IH_ERR_SHAPE";
    case IH_ERR_CAPACITY: return "IH_ERR_CAPACITY";
    case IH_ERR_PARAM: return "IH_ERR_PARAM";
    case IH_ERR_BOUNDS: return "IH_ERR_BOUNDS";
    case IH_ERR_CUDA: return "IH_ERR_CUDA";
  }
  return "IH_ERR_UNKNOWN";
}

const char* ih_last_error(void) { return g_last_error; }

int32_t ih_abi_version(void) { return (1 << 16) | 7; }

void* ih_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (bytes == 0 || cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void ih_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"
