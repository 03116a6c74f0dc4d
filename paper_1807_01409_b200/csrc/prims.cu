// Device primitives: exclusive scan, stable LSD radix sort, compaction.
#include <cuda_runtime.h>

#include <algorithm>
#include <utility>
#include <cstdlib>

#include "prims.cuh"

namespace tidq {
namespace prims {

namespace {

// Chained kernels (the radix passes up -> scan -> down per digit, the
// exclusive scan's reduce -> sums -> down) run as programmatic dependent
// launches: each kernel waits for its predecessor's
// memory at the top and lets its successor be scheduled at once, so the
// launch latency of the next kernel overlaps this one.
__device__ __forceinline__ void rdx_pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
void rdx_launch(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t stream,
                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TIDQ_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}


constexpr int kT = 256;        // threads per block
constexpr int kItems = 8;      // items per thread
constexpr int kTileN = kT * kItems;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// inclusive block scan of one uint64 per thread; returns inclusive value,
// writes the block total to *total (shared)
__device__ __forceinline__ uint64_t block_inclusive_scan(uint64_t x, uint64_t* warp_tot,
                                                         uint64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    uint64_t w = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += y;
    }
    if (lane < nw) warp_tot[lane] = w;
    if (lane == nw - 1) *total = w;
  }
  __syncthreads();
  if (warp > 0) x += warp_tot[warp - 1];
  return x;
}

template <class Tin>
__global__ void __launch_bounds__(kT) scan_reduce_kernel(const Tin* __restrict__ in, uint64_t n,
                                                         uint64_t* __restrict__ sums) {
  __shared__ uint64_t wt[kT / 32];
  __shared__ uint64_t tot;
  rdx_pdl_enter();
  const uint64_t lo = uint64_t(blockIdx.x) * kTileN;
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t k = lo + uint64_t(i) * kT + threadIdx.x;
    if (k < n) s += uint64_t(in[k]);
  }
  block_inclusive_scan(s, wt, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// single block: exclusive scan of the block sums in place, total -> sums[nb]
__global__ void __launch_bounds__(1024) scan_sums_kernel(uint64_t* sums, uint64_t nb) {
  __shared__ uint64_t wt[32];
  __shared__ uint64_t tot;
  rdx_pdl_enter();
  uint64_t carry = 0;
  for (uint64_t lo = 0; lo < nb; lo += blockDim.x) {
    const uint64_t k = lo + threadIdx.x;
    const uint64_t x = k < nb ? sums[k] : 0;
    const uint64_t inc = block_inclusive_scan(x, wt, &tot);
    if (k < nb) sums[k] = carry + inc - x;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[nb] = carry;
}

template <class Tin>
__global__ void __launch_bounds__(kT) scan_down_kernel(const Tin* __restrict__ in, uint64_t n,
                                                       const uint64_t* __restrict__ base,
                                                       uint64_t* __restrict__ out) {
  __shared__ uint64_t tile[kTileN];
  __shared__ uint64_t wt[kT / 32];
  __shared__ uint64_t tot;
  rdx_pdl_enter();
  const uint64_t lo = uint64_t(blockIdx.x) * kTileN;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t k = lo + uint64_t(i) * kT + threadIdx.x;
    tile[i * kT + threadIdx.x] = k < n ? uint64_t(in[k]) : 0;
  }
  __syncthreads();
  uint64_t v[kItems];
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    v[i] = tile[threadIdx.x * kItems + i];
    s += v[i];
  }
  const uint64_t inc = block_inclusive_scan(s, wt, &tot);
  uint64_t run = base[blockIdx.x] + inc - s;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    tile[threadIdx.x * kItems + i] = run;
    run += v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t k = lo + uint64_t(i) * kT + threadIdx.x;
    if (k < n) out[k] = tile[i * kT + threadIdx.x];
  }
}

template <class Tin>
uint64_t scan_impl(Ctx* c, const Tin* in, uint64_t* out, uint64_t n, bool sync = true) {
  if (n == 0) return 0;
  const uint64_t nb = (n + kTileN - 1) / kTileN;
  DevBuf sums(c, (nb + 1) * 8);
  rdx_launch(scan_reduce_kernel<Tin>, unsigned(nb), kT, 0, c->stream, in, n, sums.as<uint64_t>());
  rdx_launch(scan_sums_kernel, 1, 1024, 0, c->stream, sums.as<uint64_t>(), nb);
  rdx_launch(scan_down_kernel<Tin>, unsigned(nb), kT, 0, c->stream, in, n, (const uint64_t*)sums.as<uint64_t>(),
             out);
  c->count_launch(3);
  TIDQ_CUDA(cudaGetLastError());
  if (!sync) return 0;
  uint64_t* h = static_cast<uint64_t*>(c->pinned_small);
  TIDQ_CUDA(cudaMemcpyAsync(h, sums.as<uint64_t>() + nb, 8, cudaMemcpyDeviceToHost, c->stream));
  TIDQ_CUDA(cudaStreamSynchronize(c->stream));
  return h[0];
}

// ---- radix sort ----------------------------------------------------------------
// Stable LSD radix sort of (key, value) pairs.  Digit width D in {8, 9, 10}
// is chosen per sort so that ceil(bits / D) passes cover only the key's
// significant bits (26-bit term IDs: 3 passes of 9 bits).  Three kernels per
// pass: up-sweep (per-tile digit counts + global digit totals), a per-digit
// scan (one CTA per digit turns counts into global output offsets), and a
// down-sweep that ranks the tile stably (per-warp peer groups from shared
// atomicOr digit masks + per-warp digit counters), stages it digit-sorted in
// shared memory and writes
// every digit run contiguously (coalesced).  Passes whose digit is constant
// over all keys are skipped.
constexpr int kRT = 256;                // threads per radix CTA

constexpr int kRWarps = kRT / 32;
// IT keys per thread: 16 (4096-key tiles) for large sorts; 8 (2048-key tiles,
// twice the CTAs, half the serial ranking chain per CTA) below 16 M keys.

// Per-warp private histograms (summed per CTA at the end) keep lanes of
// different warps off the same shared-memory counters.
template <class K, int D, int IT>
__global__ void __launch_bounds__(kRT) radix_up_kernel(const K* __restrict__ keys, uint64_t n,
                                                       int shift, uint32_t* __restrict__ counts,
                                                       uint32_t* __restrict__ totals,
                                                       uint32_t n_tiles) {
  constexpr int R = 1 << D;
  __shared__ uint32_t h[kRWarps][R];
  rdx_pdl_enter();
  for (int i = threadIdx.x; i < kRWarps * R; i += kRT) (&h[0][0])[i] = 0;
  __syncthreads();
  uint32_t* my = h[threadIdx.x >> 5];
  const uint64_t lo = uint64_t(blockIdx.x) * (kRT * IT);
  K k[IT];
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const uint64_t j = lo + uint64_t(i) * kRT + threadIdx.x;
    k[i] = j < n ? __ldg(keys + j) : K(0);
  }
#pragma unroll
  for (int i = 0; i < IT; ++i)
    if (lo + uint64_t(i) * kRT + threadIdx.x < n) atomicAdd(&my[uint32_t(k[i] >> shift) & (R - 1)], 1u);
  __syncthreads();
  for (int d = threadIdx.x; d < R; d += kRT) {
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < kRWarps; ++w) c += h[w][d];
    counts[size_t(d) * n_tiles + blockIdx.x] = c;
    if (c) atomicAdd(totals + d, c);
  }
}

// CTA d: global start of digit d (sum of lower digits' totals) + exclusive
// scan of digit d's per-tile counts, in place.
__global__ void __launch_bounds__(1024) radix_scan_kernel(uint32_t* __restrict__ counts,
                                                          const uint32_t* __restrict__ totals,
                                                          uint32_t n_tiles) {
  __shared__ uint32_t wt[32];
  __shared__ uint32_t s_base;
  rdx_pdl_enter();
  const int d = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    uint32_t a = 0;
    for (int j = lane; j < d; j += 32) a += totals[j];
    a = __reduce_add_sync(0xffffffffu, a);
    if (lane == 0) s_base = a;
  }
  __syncthreads();
  uint32_t carry = s_base;
  uint32_t* row = counts + size_t(d) * n_tiles;
  for (uint32_t lo = 0; lo < n_tiles; lo += blockDim.x) {
    const uint32_t j = lo + threadIdx.x;
    const uint32_t x = j < n_tiles ? row[j] : 0;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wt[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = wt[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      wt[lane] = w;
    }
    __syncthreads();
    if (j < n_tiles) row[j] = carry + (warp ? wt[warp - 1] : 0) + inc - x;
    carry += wt[31];
    __syncthreads();
  }
}

// dynamic smem: wcnt[kRWarps][R] u32 | dstart[R] u32 | keys[(kRT * IT)] K | vals[(kRT * IT)] u32 | wmask[kRWarps][R]
template <class K, int D, int IT>
constexpr size_t radix_down_smem() {  // + the per-warp peer masks
  return size_t(2 * kRWarps + 1) * (1 << D) * 4 + (sizeof(K) + 4) * kRT * IT;
}

// 16 keys per thread: 3 CTAs per SM for 32-bit keys (80 registers, no
// spills), 1.5x the warps of the 128-register build, which ncu showed
// latency-bound at 24 % warp occupancy; 64-bit keys and 10-bit digits keep 2
// CTAs (at 80 registers they spill).  8 keys per thread: 4 CTAs.
template <class K, int D, int IT>
__global__ void __launch_bounds__(kRT, IT <= 8 ? 4 : (sizeof(K) == 4 && D <= 9 ? 3 : 2)) radix_down_kernel(const K* __restrict__ kin,
                                                         const uint32_t* __restrict__ vin,
                                                         K* __restrict__ kout,
                                                         uint32_t* __restrict__ vout, uint64_t n,
                                                         int shift,
                                                         const uint32_t* __restrict__ offs,
                                                         uint32_t n_tiles) {
  constexpr int R = 1 << D;
  extern __shared__ __align__(16) unsigned char rsm[];
  uint32_t* wcnt = reinterpret_cast<uint32_t*>(rsm);  // [kRWarps][R]
  uint32_t* dstart = wcnt + kRWarps * R;              // [R]
  K* skeys = reinterpret_cast<K*>(dstart + R);
  uint32_t* svals = reinterpret_cast<uint32_t*>(skeys + (kRT * IT));
  uint32_t* wmask = svals + kRT * IT;                 // [kRWarps][R] peer masks
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  rdx_pdl_enter();
  for (int i = threadIdx.x; i < kRWarps * R; i += kRT) {
    wcnt[i] = 0;
    wmask[i] = 0;
  }
  __syncthreads();
  const uint64_t t0 = uint64_t(blockIdx.x) * (kRT * IT);
  const uint64_t lo = t0 + uint64_t(warp) * (32 * IT);
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  K key[IT];
  uint32_t val[IT];
  uint32_t rank[IT];
#pragma unroll
  for (int r = 0; r < IT; ++r) {
    const uint64_t k = lo + uint64_t(r) * 32 + lane;
    const bool valid = k < n;
    key[r] = valid ? kin[k] : K(0);
    val[r] = valid ? vin[k] : 0u;
  }
  uint32_t* my = wcnt + warp * R;
  // Peer groups by shared-memory atomicOr of the lane bits into a per-warp
  // digit mask, cleared by the group's leader: measured faster than
  // __match_any_sync (5.5 M 28-bit keys 0.298 -> 0.258 ms, 20 M 1.27 -> 1.01
  // ms, tools/sort_bench.py; C4 joins 3-7 % faster)
  uint32_t* wm = wmask + warp * R;
#pragma unroll
  for (int r = 0; r < IT; ++r) {
    const bool valid = lo + uint64_t(r) * 32 + lane < n;
    const int d = int(uint32_t(key[r] >> shift) & (R - 1));
    if (valid) atomicOr(&wm[d], 1u << lane);
    __syncwarp();
    const uint32_t peers = valid ? wm[d] : (1u << lane);
    const uint32_t base = valid ? my[d] : 0u;
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) {
      my[d] = base + __popc(peers);
      wm[d] = 0;
    }
    __syncwarp();
    rank[r] = base + __popc(peers & lt);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < R; d += kRT) {  // exclusive over warps; digit tile totals
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kRWarps; ++w) {
      const uint32_t x = wcnt[w * R + d];
      wcnt[w * R + d] = run;
      run += x;
    }
    dstart[d] = run;
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the R digit totals, R/32 per lane
    constexpr int PL = R / 32;
    uint32_t v[PL];
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < PL; ++j) {
      v[j] = dstart[lane * PL + j];
      s += v[j];
    }
    uint32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    uint32_t run = inc - s;
#pragma unroll
    for (int j = 0; j < PL; ++j) {
      dstart[lane * PL + j] = run;
      run += v[j];
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < IT; ++r) {
    if (lo + uint64_t(r) * 32 + lane >= n) continue;
    const int d = int(uint32_t(key[r] >> shift) & (R - 1));
    const uint32_t lp = dstart[d] + my[d] + rank[r];
    skeys[lp] = key[r];
    svals[lp] = val[r];
  }
  // the tile's global digit offsets minus their local starts, staged once in
  // shared memory (wcnt is free now): one global load per digit instead of
  // one dependent global load per element in the scatter below
  __syncthreads();  // every warp is done reading its counters (my[])
  uint32_t* sbase = wcnt;
  for (int d = threadIdx.x; d < R; d += kRT) sbase[d] = offs[size_t(d) * n_tiles + blockIdx.x] - dstart[d];
  __syncthreads();
  const uint32_t tile_n = uint32_t(n - t0 < uint64_t((kRT * IT)) ? n - t0 : uint64_t((kRT * IT)));
  for (uint32_t i = threadIdx.x; i < tile_n; i += kRT) {
    const K k = skeys[i];
    const int d = int(uint32_t(k >> shift) & (R - 1));
    const uint32_t dst = sbase[d] + i;
    kout[dst] = k;
    vout[dst] = svals[i];
  }
}

template <class K, int D, int IT>
void radix_passes(Ctx* c, K*& ka, K*& kb, uint32_t*& va, uint32_t*& vb, uint64_t n, int passes) {
  constexpr int R = 1 << D;
  const uint32_t n_tiles = uint32_t((n + (kRT * IT) - 1) / (kRT * IT));
  // digit totals: one zeroed slice per pass (one memset for the sort)
  DevBuf cnt(c, size_t(n_tiles) * R * 4), tot(c, size_t(passes) * R * 4);
  constexpr size_t smem = radix_down_smem<K, D, IT>();
  auto down = radix_down_kernel<K, D, IT>;
  ensure_dyn_smem(reinterpret_cast<const void*>(down), c->device, int(smem));
  TIDQ_CUDA(cudaMemsetAsync(tot.ptr, 0, size_t(passes) * R * 4, c->stream));
  for (int p = 0; p < passes; ++p) {
    const int shift = D * p;
    uint32_t* tp = tot.as<uint32_t>() + size_t(p) * R;
    rdx_launch(radix_up_kernel<K, D, IT>, n_tiles, kRT, 0, c->stream, (const K*)ka, n, shift,
               cnt.as<uint32_t>(), tp, n_tiles);
    c->count_launch();
    // No host round trip per pass (it cost a stream drain per pass: 140 us
    // per pass on 6 M keys): passes cover only the significant bits of the
    // max key, and a pass whose digit is constant is a correct (stable)
    // identity scatter.
    rdx_launch(radix_scan_kernel, R, 1024, 0, c->stream, cnt.as<uint32_t>(), (const uint32_t*)tp, n_tiles);
    rdx_launch(down, n_tiles, kRT, smem, c->stream, (const K*)ka, (const uint32_t*)va, kb, vb, n, shift,
               (const uint32_t*)cnt.as<uint32_t>(), n_tiles);
    c->count_launch(2);
    TIDQ_CUDA(cudaGetLastError());
    std::swap(ka, kb);
    std::swap(va, vb);
  }
}

// ---- onesweep radix sort ---------------------------------------------------------
// One histogram pass over the keys counts the 8-bit digits of EVERY pass at
// once; then each pass is ONE kernel: a CTA takes the next tile index from an
// atomic counter (so every lower tile is already running), ranks its 4096
// (u32) / 2048 (u64) keys stably as the LSD down-sweep does, publishes its
// per-digit counts, and finds its global digit offsets with a decoupled
// look-back over the lower tiles' published counts (one thread per digit; a
// status word = 2 flag bits | 30-bit count: aggregate or inclusive prefix).
// Per pass the keys are read once and written once: no up-sweep re-read, no
// per-digit scan kernel, no per-tile count array.
constexpr int kOsMaxPasses = 8;
constexpr uint32_t kOsFlagA = 1u << 30, kOsFlagP = 2u << 30, kOsVal = (1u << 30) - 1;

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// hist[p][256] += digit counts of pass p over all keys (per-warp shared
// histograms: skewed high digits do not serialise a CTA on one counter)
template <class K>
__global__ void __launch_bounds__(kRT) os_hist_kernel(const K* __restrict__ keys, uint64_t n, int passes,
                                                      uint32_t* __restrict__ hist) {
  extern __shared__ uint32_t oh[];  // [kRWarps][passes][256]
  rdx_pdl_enter();
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kRWarps * passes * 256; i += kRT) oh[i] = 0;
  __syncthreads();
  uint32_t* my = oh + warp * passes * 256;
  constexpr int kU = 4;
  const uint64_t stride = uint64_t(gridDim.x) * kRT * kU;
  for (uint64_t b = uint64_t(blockIdx.x) * kRT * kU; b < n; b += stride) {
    K k[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t j = b + uint64_t(u) * kRT + threadIdx.x;
      k[u] = j < n ? __ldg(keys + j) : K(0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (b + uint64_t(u) * kRT + threadIdx.x >= n) continue;
      for (int p = 0; p < passes; ++p) atomicAdd(&my[p * 256 + (uint32_t(k[u] >> (8 * p)) & 255u)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += kRT) {
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < kRWarps; ++w) c += oh[w * passes * 256 + i];
    if (c) atomicAdd(hist + i, c);
  }
}

template <class K, int IT>
constexpr size_t os_pass_smem() {
  return size_t(kRWarps) * 256 * 4 + 3 * 256 * 4 + (sizeof(K) + 4) * kRT * IT + size_t(kRWarps) * 256 * 4;
}

template <class K, int IT>
__global__ void __launch_bounds__(kRT, sizeof(K) == 4 ? 3 : 2) os_pass_kernel(
    const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout, uint32_t* __restrict__ vout,
    uint64_t n, int shift, const uint32_t* __restrict__ hist, uint32_t* __restrict__ status,
    uint32_t* __restrict__ tile_ctr) {
  static_assert(kRT == 256, "one look-back thread per digit");
  constexpr int R = 256, TILE = kRT * IT;
  extern __shared__ __align__(16) unsigned char osm[];
  uint32_t* wcnt = reinterpret_cast<uint32_t*>(osm);  // [kRWarps][R]
  uint32_t* dstart = wcnt + kRWarps * R;              // [R] tile-local digit starts
  uint32_t* gstart = dstart + R;                      // [R] global digit starts (this pass)
  uint32_t* sbase = gstart + R;                       // [R] global offset - local start
  K* skeys = reinterpret_cast<K*>(sbase + R);
  uint32_t* svals = reinterpret_cast<uint32_t*>(skeys + TILE);
  uint32_t* wmask = svals + TILE;  // [kRWarps][R] peer masks
  __shared__ uint32_t s_tile, s_wsum[kRWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  rdx_pdl_enter();
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (int i = threadIdx.x; i < kRWarps * R; i += kRT) {
    wcnt[i] = 0;
    wmask[i] = 0;
  }
  {  // exclusive scan of this pass's 256 digit totals -> global digit starts
    const uint32_t h = hist[threadIdx.x];
    uint32_t inc = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_wsum[warp] = inc;
    __syncthreads();
    uint32_t pre = 0;
#pragma unroll
    for (int w = 0; w < kRWarps; ++w) pre += w < warp ? s_wsum[w] : 0u;
    gstart[threadIdx.x] = pre + inc - h;
  }
  const uint32_t tile = s_tile;
  const uint64_t t0 = uint64_t(tile) * TILE;
  const uint64_t lo = t0 + uint64_t(warp) * (32 * IT);
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  K key[IT];
  uint32_t val[IT];
  uint32_t rank[IT];
#pragma unroll
  for (int r = 0; r < IT; ++r) {
    const uint64_t k = lo + uint64_t(r) * 32 + lane;
    const bool valid = k < n;
    key[r] = valid ? kin[k] : K(0);
    val[r] = valid ? vin[k] : 0u;
  }
  uint32_t* my = wcnt + warp * R;
  // peer groups by shared atomicOr masks (the LSD down-sweep's measured
  // winner over __match_any_sync), cleared by each group's leader
  uint32_t* wm = wmask + warp * R;
#pragma unroll
  for (int r = 0; r < IT; ++r) {
    const bool valid = lo + uint64_t(r) * 32 + lane < n;
    const int d = int(uint32_t(key[r] >> shift) & (R - 1));
    if (valid) atomicOr(&wm[d], 1u << lane);
    __syncwarp();
    const uint32_t peers = valid ? wm[d] : (1u << lane);
    const uint32_t base = valid ? my[d] : 0u;
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) {
      my[d] = base + __popc(peers);
      wm[d] = 0;
    }
    __syncwarp();
    rank[r] = base + __popc(peers & lt);
  }
  __syncthreads();
  const int d0 = threadIdx.x;  // this thread's digit: counts over warps, publish, look back
  uint32_t cnt = 0;
#pragma unroll
  for (int w = 0; w < kRWarps; ++w) {
    const uint32_t x = wcnt[w * R + d0];
    wcnt[w * R + d0] = cnt;
    cnt += x;
  }
  uint32_t* st = status + size_t(tile) * R + d0;
  if (tile == 0) {
    st_relaxed(st, kOsFlagP | cnt);
    sbase[d0] = gstart[d0];
  } else {
    st_relaxed(st, kOsFlagA | cnt);
    uint32_t excl = 0;
    const uint32_t* q = st - R;
    while (true) {
      uint32_t s;
      do {
        s = ld_relaxed(q);
      } while (!(s & (kOsFlagA | kOsFlagP)));
      excl += s & kOsVal;
      if (s & kOsFlagP) break;
      q -= R;
    }
    st_relaxed(st, kOsFlagP | (excl + cnt));
    sbase[d0] = gstart[d0] + excl;
  }
  dstart[d0] = cnt;
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the tile's digit totals, 8 per lane
    uint32_t v[8];
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      v[j] = dstart[lane * 8 + j];
      s += v[j];
    }
    uint32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    uint32_t run = inc - s;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      dstart[lane * 8 + j] = run;
      sbase[lane * 8 + j] -= run;
      run += v[j];
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < IT; ++r) {
    if (lo + uint64_t(r) * 32 + lane >= n) continue;
    const int d = int(uint32_t(key[r] >> shift) & (R - 1));
    const uint32_t lp = dstart[d] + my[d] + rank[r];
    skeys[lp] = key[r];
    svals[lp] = val[r];
  }
  __syncthreads();
  const uint32_t tile_n = uint32_t(n - t0 < uint64_t(TILE) ? n - t0 : uint64_t(TILE));
  for (uint32_t i = threadIdx.x; i < tile_n; i += kRT) {
    const K k = skeys[i];
    const uint32_t dst = sbase[uint32_t(k >> shift) & (R - 1)] + i;
    kout[dst] = k;
    vout[dst] = svals[i];
  }
}

template <class K, int IT>
void onesweep_passes(Ctx* c, K*& ka, K*& kb, uint32_t*& va, uint32_t*& vb, uint64_t n, int passes) {
  constexpr int TILE = kRT * IT;
  const uint64_t n_tiles = (n + TILE - 1) / TILE;
  // one zeroed block: [passes][256] histograms | [passes] tile counters | [passes][n_tiles][256] status
  const size_t words = size_t(passes) * 256 + passes + size_t(passes) * n_tiles * 256;
  DevBuf scratch(c, words * 4);
  uint32_t* hist = scratch.as<uint32_t>();
  uint32_t* ctr = hist + passes * 256;
  uint32_t* status = ctr + passes;
  TIDQ_CUDA(cudaMemsetAsync(scratch.ptr, 0, words * 4, c->stream));
  const size_t hsm = size_t(kRWarps) * passes * 256 * 4;
  auto hk = os_hist_kernel<K>;
  ensure_dyn_smem(reinterpret_cast<const void*>(hk), c->device, int(hsm));
  const unsigned hgrid = unsigned(std::min<uint64_t>((n + kRT * 4 - 1) / (kRT * 4), uint64_t(c->sm_count) * 4));
  rdx_launch(hk, hgrid, kRT, hsm, c->stream, (const K*)ka, n, passes, hist);
  constexpr size_t smem = os_pass_smem<K, IT>();
  auto pk = os_pass_kernel<K, IT>;
  ensure_dyn_smem(reinterpret_cast<const void*>(pk), c->device, int(smem));
  for (int p = 0; p < passes; ++p) {
    rdx_launch(pk, unsigned(n_tiles), kRT, smem, c->stream, (const K*)ka, (const uint32_t*)va, kb, vb, n, 8 * p,
               (const uint32_t*)(hist + p * 256), status + size_t(p) * n_tiles * 256, ctr + p);
    TIDQ_CUDA(cudaGetLastError());
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  c->count_launch(1 + passes);
}

// Which passes sort n keys of kbytes bytes: with the atomicOr peer masks
// onesweep measured faster than the LSD passes for 32-bit keys from ~1 M on
// (28 bits: 3.4 M 0.164 vs 0.170 ms, 5.5 M 0.228 vs 0.253, 20 M 0.74 vs
// 1.22), equal at 0.5 M, and slower for 64-bit keys (65 M by 16 bits: 2.31
// vs 1.72 ms; tools/sort_bench.py, profiles/r02_sort_bench*.jsonl).  Env TIDQ_RADIX =
// lsd | onesweep forces one (A/B and tests); n must stay below 2^30 (30-bit
// look-back counts).
bool use_onesweep(uint64_t n, size_t kbytes) {
  if (n >= (1ull << 30)) return false;
  const char* e = std::getenv("TIDQ_RADIX");
  if (e && e[0] == 'l') return false;
  if (e && e[0] == 'o') return true;
  return kbytes == 4 && n >= (1ull << 20);
}

// Digit width: 8-bit digits write 16-key runs per digit and tile
// (coalesced) and win below ~16 M keys even with one more pass (6 M keys,
// 28 bits: 4 x 8 bits 313 us vs 3 x 10 bits 379 us); above, fewer passes
// win (65 M 52-bit keys: 6 x 9 bits 5.1 ms vs 7 x 8 bits 6.6 ms).
// Onesweep always uses 8-bit digits.
void radix_plan(uint64_t n, int bits, size_t kbytes, int& passes, int& dbits) {
  passes = (n <= (1ull << 24) || use_onesweep(n, kbytes)) ? (bits + 7) / 8 : (bits + 9) / 10;
  dbits = std::max(8, (bits + passes - 1) / passes);  // 8, 9 or 10
}

template <class K>
void radix_impl(Ctx* c, K* keys, uint32_t* vals, uint64_t n, int bits) {
  if (n <= 1 || bits <= 0) return;
  TIDQ_REQUIRE(n < (1ull << 32), TIDQ_E_INVALID, "radix sort above 2^32 keys");
  int passes, dbits;
  radix_plan(n, bits, sizeof(K), passes, dbits);
  DevBuf k2(c, n * sizeof(K)), v2(c, n * 4);
  K* ka = keys;
  K* kb = k2.as<K>();
  uint32_t* va = vals;
  uint32_t* vb = v2.as<uint32_t>();
  const int np = (bits + dbits - 1) / dbits;
  if (dbits == 8 && np <= kOsMaxPasses && use_onesweep(n, sizeof(K))) {
    if constexpr (sizeof(K) == 4)
      onesweep_passes<K, 16>(c, ka, kb, va, vb, n, np);
    else
      onesweep_passes<K, 8>(c, ka, kb, va, vb, n, np);
  } else if (n <= (1ull << 24)) {
    if (dbits == 8)
      radix_passes<K, 8, 8>(c, ka, kb, va, vb, n, np);
    else if (dbits == 9)
      radix_passes<K, 9, 8>(c, ka, kb, va, vb, n, np);
    else
      radix_passes<K, 10, 8>(c, ka, kb, va, vb, n, np);
  } else {
    // 64-bit keys with 8-bit digits: 8 keys per thread (4 CTAs per SM) beat
    // 16 (2 CTAs per SM) — C3 DISTINCT ?s ?o UNION x4 partition sort, 65 M
    // keys: 5.40 -> 5.08 ms per query; with 9-bit digits the 4-key runs per
    // digit lose (8.04 -> 8.79 ms at 93 M keys)
    if (dbits == 8 && sizeof(K) == 8)
      radix_passes<K, 8, 8>(c, ka, kb, va, vb, n, np);
    else if (dbits == 8)
      radix_passes<K, 8, 16>(c, ka, kb, va, vb, n, np);
    else if (dbits == 9)
      radix_passes<K, 9, 16>(c, ka, kb, va, vb, n, np);
    else
      radix_passes<K, 10, 16>(c, ka, kb, va, vb, n, np);
  }
  if (ka != keys) {
    TIDQ_CUDA(cudaMemcpyAsync(keys, ka, n * sizeof(K), cudaMemcpyDeviceToDevice, c->stream));
    TIDQ_CUDA(cudaMemcpyAsync(vals, va, n * 4, cudaMemcpyDeviceToDevice, c->stream));
  }
}

// Elementwise kernels: a CTA owns kEW consecutive elements, every thread
// kEI independent items (coalesced, in flight together); no grid-stride loops.
constexpr int kEWT = 256;
constexpr int kEI = 4;
constexpr int kEW = kEWT * kEI;

inline unsigned ew_grid(uint64_t n) { return unsigned((n + kEW - 1) / kEW); }

__global__ void __launch_bounds__(kEWT) max_kernel(const uint32_t* __restrict__ x, uint64_t n,
                                                   uint32_t* out) {
  __shared__ uint32_t wmax[kEWT / 32];
  const uint64_t base = uint64_t(blockIdx.x) * kEW * 4;  // 4 elements per item (uint4)
  uint32_t m = 0;
  if (base + kEW * 4 <= n && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    uint4 v[kEI];
#pragma unroll
    for (int j = 0; j < kEI; ++j)
      v[j] = __ldg(reinterpret_cast<const uint4*>(x + base) + j * kEWT + threadIdx.x);
#pragma unroll
    for (int j = 0; j < kEI; ++j) m = max(m, max(max(v[j].x, v[j].y), max(v[j].z, v[j].w)));
  } else {
    for (uint64_t i = base + threadIdx.x; i < n && i < base + kEW * 4; i += kEWT) m = max(m, x[i]);
  }
  // one atomic per CTA (a per-warp atomicMax on one address serialised:
  // 189 us for 69 M keys)
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < kEWT / 32 ? wmax[threadIdx.x] : 0u;
    m = __reduce_max_sync(0xffffffffu, m);
    if (threadIdx.x == 0 && m) atomicMax(out, m);
  }
}

__global__ void __launch_bounds__(kEWT) iota_kernel(uint32_t* out, uint64_t n) {
  rdx_pdl_enter();
  const uint64_t base = uint64_t(blockIdx.x) * kEW;
#pragma unroll
  for (int j = 0; j < kEI; ++j) {
    const uint64_t i = base + j * kEWT + threadIdx.x;
    if (i < n) out[i] = uint32_t(i);
  }
}

__global__ void __launch_bounds__(kEWT) gather_kernel(const uint32_t* __restrict__ src,
                                                      const uint32_t* __restrict__ idx,
                                                      uint32_t* __restrict__ out, uint64_t n) {
  const uint64_t base = uint64_t(blockIdx.x) * kEW;
  uint32_t v[kEI];
#pragma unroll
  for (int j = 0; j < kEI; ++j) {
    const uint64_t i = base + j * kEWT + threadIdx.x;
    v[j] = i < n ? ld_gather(src + __ldg(idx + i)) : 0u;
  }
#pragma unroll
  for (int j = 0; j < kEI; ++j) {
    const uint64_t i = base + j * kEWT + threadIdx.x;
    if (i < n) out[i] = v[j];
  }
}

struct ColPtrs {
  const uint32_t* in[8];
  uint32_t* out[8];
};

// ---- bitmap row selection ----------------------------------------------------
// A warp owns 32 keep-words (1024 rows).  count: rows kept per warp.  write:
// for each word, lanes test their row's bit, ballot ranks them, and the kept
// rows of every column are copied to out[base + rank] (coalesced both ways).
constexpr int kSelWarps = 8;

__global__ void __launch_bounds__(kSelWarps * 32) select_count_kernel(const uint32_t* __restrict__ words,
                                                                      uint64_t n_words,
                                                                      uint32_t* __restrict__ counts) {
  rdx_pdl_enter();
  const uint64_t w = blockIdx.x * uint64_t(kSelWarps) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const uint64_t k = w * 32 + lane;
  const uint32_t c = __reduce_add_sync(0xffffffffu, k < n_words ? __popc(words[k]) : 0u);
  if (lane == 0 && w * 32 < n_words) counts[w] = c;
}

__global__ void __launch_bounds__(kSelWarps * 32) select_write_kernel(const uint32_t* __restrict__ words,
                                                                      uint64_t n_rows,
                                                                      const uint64_t* __restrict__ offs,
                                                                      int n_cols, const __grid_constant__ ColPtrs cp) {
  rdx_pdl_enter();
  const uint64_t w = blockIdx.x * uint64_t(kSelWarps) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const uint64_t n_words = (n_rows + 31) / 32;
  if (w * 32 >= n_words) return;
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  const uint32_t my_word = (w * 32 + lane < n_words) ? words[w * 32 + lane] : 0u;
  // Per column, 8 words at a time: the kept values of 8 x 32 rows are loaded
  // together, then stored (one word at a time the outputs' possible aliasing
  // of the inputs chained a load round trip per word: 32 per warp).
  constexpr int kB = 8;
  const uint64_t pos0 = offs[w];
  for (int k = 0; k < n_cols; ++k) {
    const uint32_t* __restrict__ in = cp.in[k];
    uint32_t* out = cp.out[k];
    uint64_t pos = pos0;
#pragma unroll 1
    for (int j0 = 0; j0 < 32; j0 += kB) {
      uint32_t wd[kB], v[kB];
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        wd[i] = __shfl_sync(0xffffffffu, my_word, j0 + i);
        const uint64_t row = (w * 32 + j0 + i) * 32 + lane;
        v[i] = (wd[i] >> lane) & 1u ? __ldg(in + row) : 0u;
      }
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        if ((wd[i] >> lane) & 1u) out[pos + __popc(wd[i] & lt)] = v[i];
        pos += __popc(wd[i]);
      }
    }
  }
}

}  // namespace

uint64_t exclusive_scan(Ctx* c, const uint32_t* in, uint64_t* out, uint64_t n) {
  return scan_impl<uint32_t>(c, in, out, n);
}
uint64_t exclusive_scan(Ctx* c, const uint64_t* in, uint64_t* out, uint64_t n) {
  return scan_impl<uint64_t>(c, in, out, n);
}
void exclusive_scan_async(Ctx* c, const uint32_t* in, uint64_t* out, uint64_t n) {
  scan_impl<uint32_t>(c, in, out, n, false);
}

void radix_sort_pairs(Ctx* c, uint32_t* keys, uint32_t* vals, uint64_t n, int bits) {
  radix_impl<uint32_t>(c, keys, vals, n, std::min(bits, 32));
}
int radix_sorted_bits(uint64_t n, int bits) {  // (the 64-bit partition sort's digits)
  int passes, dbits;
  radix_plan(n, bits, 8, passes, dbits);
  return passes * dbits;
}

void radix_sort_pairs(Ctx* c, uint64_t* keys, uint32_t* vals, uint64_t n, int bits) {
  radix_impl<uint64_t>(c, keys, vals, n, std::min(bits, 64));
}

uint32_t max_u32(Ctx* c, const uint32_t* x, uint64_t n) {
  if (n == 0) return 0;
  DevBuf m(c, 4);
  TIDQ_CUDA(cudaMemsetAsync(m.ptr, 0, 4, c->stream));
  max_kernel<<<unsigned((n + kEW * 4 - 1) / (kEW * 4)), kEWT, 0, c->stream>>>(x, n, m.as<uint32_t>());
  c->count_launch();
  uint32_t* h = static_cast<uint32_t*>(c->pinned_small);
  TIDQ_CUDA(cudaMemcpyAsync(h, m.ptr, 4, cudaMemcpyDeviceToHost, c->stream));
  TIDQ_CUDA(cudaStreamSynchronize(c->stream));
  return h[0];
}

void max_u32_multi(Ctx* c, int k, const uint32_t* const* x, const uint64_t* n, uint32_t* out) {
  TIDQ_REQUIRE(k >= 1 && k <= 8, TIDQ_E_INVALID, "max_u32_multi: 1..8 columns");
  DevBuf m(c, 4 * 8);
  TIDQ_CUDA(cudaMemsetAsync(m.ptr, 0, 4 * k, c->stream));
  for (int i = 0; i < k; ++i) {
    if (!n[i]) continue;
    max_kernel<<<unsigned((n[i] + kEW * 4 - 1) / (kEW * 4)), kEWT, 0, c->stream>>>(x[i], n[i],
                                                                                   m.as<uint32_t>() + i);
    c->count_launch();
  }
  uint32_t* h = static_cast<uint32_t*>(c->pinned_small);
  TIDQ_CUDA(cudaMemcpyAsync(h, m.ptr, 4 * k, cudaMemcpyDeviceToHost, c->stream));
  TIDQ_CUDA(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < k; ++i) out[i] = h[i];
}

void iota(Ctx* c, uint32_t* out, uint64_t n) {
  if (!n) return;
  rdx_launch(iota_kernel, ew_grid(n), kEWT, 0, c->stream, out, n);
  c->count_launch();
}

void gather_u32(Ctx* c, const uint32_t* src, const uint32_t* idx, uint32_t* out, uint64_t n) {
  if (!n) return;
  gather_kernel<<<ew_grid(n), kEWT, 0, c->stream>>>(src, idx, out, n);
  c->count_launch();
}

uint64_t select_count(Ctx* c, const uint32_t* words, uint64_t n_rows, DevBuf& offs) {
  const uint64_t n_words = (n_rows + 31) / 32;
  const uint64_t n_warps = (n_words + 31) / 32;
  offs = DevBuf(c, (n_warps + 1) * 8);
  if (!n_words) return 0;
  DevBuf counts(c, n_warps * 4);
  rdx_launch(select_count_kernel, unsigned((n_warps + kSelWarps - 1) / kSelWarps), kSelWarps * 32, 0, c->stream, 
      words, n_words, counts.as<uint32_t>());
  c->count_launch();
  return exclusive_scan(c, counts.as<uint32_t>(), offs.as<uint64_t>(), n_warps);
}

void select_count_async(Ctx* c, const uint32_t* words, uint64_t n_rows, DevBuf& offs) {
  const uint64_t n_words = (n_rows + 31) / 32;
  const uint64_t n_warps = (n_words + 31) / 32;
  offs = DevBuf(c, (n_warps + 1) * 8);
  DevBuf counts(c, (n_warps + 1) * 4);
  TIDQ_CUDA(cudaMemsetAsync(counts.as<uint32_t>() + n_warps, 0, 4, c->stream));
  if (n_words) {
    rdx_launch(select_count_kernel, unsigned((n_warps + kSelWarps - 1) / kSelWarps), kSelWarps * 32, 0, c->stream, 
        words, n_words, counts.as<uint32_t>());
    c->count_launch();
  }
  exclusive_scan_async(c, counts.as<uint32_t>(), offs.as<uint64_t>(), n_warps + 1);  // offs[n_warps] = total
}

void select_write(Ctx* c, const uint32_t* words, uint64_t n_rows, const DevBuf& offs, int n_cols,
                  const uint32_t* const* in, uint32_t* const* out) {
  const uint64_t n_words = (n_rows + 31) / 32;
  const uint64_t n_warps = (n_words + 31) / 32;
  if (!n_words || !n_cols) return;
  for (int lo = 0; lo < n_cols; lo += 8) {
    ColPtrs cp{};
    const int k = std::min(8, n_cols - lo);
    for (int i = 0; i < k; ++i) {
      cp.in[i] = in[lo + i];
      cp.out[i] = out[lo + i];
    }
    rdx_launch(select_write_kernel, unsigned((n_warps + kSelWarps - 1) / kSelWarps), kSelWarps * 32, 0, c->stream, 
        words, n_rows, offs.as<uint64_t>(), k, cp);
    c->count_launch();
  }
  TIDQ_CUDA(cudaGetLastError());
}

}  // namespace prims
}  // namespace tidq
