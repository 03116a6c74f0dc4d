// Device primitives: exclusive scan, stable LSD radix sort, compaction.
#include <cuda_runtime.h>

#include <algorithm>

#include "prims.cuh"

namespace tidq {
namespace prims {

namespace {

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
  scan_reduce_kernel<Tin><<<unsigned(nb), kT, 0, c->stream>>>(in, n, sums.as<uint64_t>());
  scan_sums_kernel<<<1, 1024, 0, c->stream>>>(sums.as<uint64_t>(), nb);
  scan_down_kernel<Tin><<<unsigned(nb), kT, 0, c->stream>>>(in, n, sums.as<uint64_t>(), out);
  c->count_launch(3);
  TIDQ_CUDA(cudaGetLastError());
  if (!sync) return 0;
  uint64_t* h = static_cast<uint64_t*>(c->pinned_small);
  TIDQ_CUDA(cudaMemcpyAsync(h, sums.as<uint64_t>() + nb, 8, cudaMemcpyDeviceToHost, c->stream));
  TIDQ_CUDA(cudaStreamSynchronize(c->stream));
  return h[0];
}

// ---- radix sort ----------------------------------------------------------------

template <class K>
__global__ void __launch_bounds__(kT) radix_hist_kernel(const K* __restrict__ keys, uint64_t n,
                                                        int shift, uint32_t* __restrict__ hist,
                                                        uint32_t n_tiles) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t lo = uint64_t(blockIdx.x) * kTileN;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t k = lo + uint64_t(i) * kT + threadIdx.x;
    if (k < n) atomicAdd(&h[uint32_t(keys[k] >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[size_t(threadIdx.x) * n_tiles + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter: warp w owns tile items [w*256, (w+1)*256) in 8 rounds of 32;
// ranks within the warp come from __match_any_sync peer groups and per-warp
// digit counters; a per-digit scan over the 8 warps orders warps.
template <class K>
__global__ void __launch_bounds__(kT) radix_scatter_kernel(const K* __restrict__ kin,
                                                           const uint32_t* __restrict__ vin,
                                                           K* __restrict__ kout,
                                                           uint32_t* __restrict__ vout, uint64_t n,
                                                           int shift,
                                                           const uint64_t* __restrict__ offs,
                                                           uint32_t n_tiles) {
  __shared__ uint32_t wcnt[kT / 32][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (kT / 32) * 256; i += kT) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const uint64_t lo = uint64_t(blockIdx.x) * kTileN + uint64_t(warp) * (32 * kItems);
  const uint32_t lt = lanemask_lt();
  K key[kItems];
  uint32_t val[kItems];
  uint32_t rank[kItems];
  int dig[kItems];
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const uint64_t k = lo + uint64_t(r) * 32 + lane;
    const bool valid = k < n;
    key[r] = valid ? kin[k] : K(0);
    val[r] = valid ? vin[k] : 0u;
    const int d = valid ? int(uint32_t(key[r] >> shift) & 255u) : 256 + lane;
    dig[r] = d;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t base = 0;
    if (valid) base = wcnt[warp][d];
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) wcnt[warp][d] = base + __popc(peers);
    __syncwarp();
    rank[r] = base + __popc(peers & lt);
  }
  __syncthreads();
  {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) {
      const uint32_t x = wcnt[w][threadIdx.x];
      wcnt[w][threadIdx.x] = run;
      run += x;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const int d = dig[r];
    if (d < 256) {
      const uint64_t pos = offs[size_t(d) * n_tiles + blockIdx.x] + wcnt[warp][d] + rank[r];
      kout[pos] = key[r];
      vout[pos] = val[r];
    }
  }
}

template <class K>
void radix_impl(Ctx* c, K* keys, uint32_t* vals, uint64_t n, int bits) {
  if (n <= 1 || bits <= 0) return;
  const uint32_t n_tiles = uint32_t((n + kTileN - 1) / kTileN);
  const int passes = (bits + 7) / 8;
  DevBuf k2(c, n * sizeof(K)), v2(c, n * 4);
  DevBuf hist(c, size_t(n_tiles) * 256 * 4), offs(c, size_t(n_tiles) * 256 * 8);
  K* ka = keys;
  K* kb = k2.as<K>();
  uint32_t* va = vals;
  uint32_t* vb = v2.as<uint32_t>();
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    radix_hist_kernel<K><<<n_tiles, kT, 0, c->stream>>>(ka, n, shift, hist.as<uint32_t>(), n_tiles);
    c->count_launch();
    exclusive_scan(c, hist.as<uint32_t>(), offs.as<uint64_t>(), uint64_t(n_tiles) * 256);
    radix_scatter_kernel<K><<<n_tiles, kT, 0, c->stream>>>(ka, va, kb, vb, n, shift,
                                                           offs.as<uint64_t>(), n_tiles);
    c->count_launch();
    TIDQ_CUDA(cudaGetLastError());
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  if (ka != keys) {
    TIDQ_CUDA(cudaMemcpyAsync(keys, ka, n * sizeof(K), cudaMemcpyDeviceToDevice, c->stream));
    TIDQ_CUDA(cudaMemcpyAsync(vals, va, n * 4, cudaMemcpyDeviceToDevice, c->stream));
  }
}

__global__ void max_kernel(const uint32_t* __restrict__ x, uint64_t n, uint32_t* out) {
  uint32_t m = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    m = max(m, x[i]);
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void iota_kernel(uint32_t* out, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = uint32_t(i);
}

__global__ void gather_kernel(const uint32_t* __restrict__ src, const uint32_t* __restrict__ idx,
                              uint32_t* __restrict__ out, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = src[idx[i]];
}

struct ColPtrs {
  const uint32_t* in[8];
  uint32_t* out[8];
};

__global__ void compact_kernel(const uint32_t* __restrict__ flags,
                               const uint64_t* __restrict__ offs, uint64_t n, int n_cols,
                               ColPtrs cp) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (flags[i]) {
      const uint64_t o = offs[i];
      for (int k = 0; k < n_cols; ++k) cp.out[k][o] = cp.in[k][i];
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
void radix_sort_pairs(Ctx* c, uint64_t* keys, uint32_t* vals, uint64_t n, int bits) {
  radix_impl<uint64_t>(c, keys, vals, n, std::min(bits, 64));
}

uint32_t max_u32(Ctx* c, const uint32_t* x, uint64_t n) {
  if (n == 0) return 0;
  DevBuf m(c, 4);
  TIDQ_CUDA(cudaMemsetAsync(m.ptr, 0, 4, c->stream));
  max_kernel<<<grid_for(c, n, 256), 256, 0, c->stream>>>(x, n, m.as<uint32_t>());
  c->count_launch();
  uint32_t* h = static_cast<uint32_t*>(c->pinned_small);
  TIDQ_CUDA(cudaMemcpyAsync(h, m.ptr, 4, cudaMemcpyDeviceToHost, c->stream));
  TIDQ_CUDA(cudaStreamSynchronize(c->stream));
  return h[0];
}

void iota(Ctx* c, uint32_t* out, uint64_t n) {
  if (!n) return;
  iota_kernel<<<grid_for(c, n, 256), 256, 0, c->stream>>>(out, n);
  c->count_launch();
}

void gather_u32(Ctx* c, const uint32_t* src, const uint32_t* idx, uint32_t* out, uint64_t n) {
  if (!n) return;
  gather_kernel<<<grid_for(c, n, 256), 256, 0, c->stream>>>(src, idx, out, n);
  c->count_launch();
}

uint64_t compact_offsets(Ctx* c, const uint32_t* flags, uint64_t* offsets, uint64_t n) {
  return exclusive_scan(c, flags, offsets, n);
}

void compact_cols(Ctx* c, const uint32_t* flags, const uint64_t* offsets, uint64_t n, int n_cols,
                  const uint32_t* const* in, uint32_t* const* out) {
  if (!n || !n_cols) return;
  for (int lo = 0; lo < n_cols; lo += 8) {
    ColPtrs cp{};
    const int k = std::min(8, n_cols - lo);
    for (int i = 0; i < k; ++i) {
      cp.in[i] = in[lo + i];
      cp.out[i] = out[lo + i];
    }
    compact_kernel<<<grid_for(c, n, 256), 256, 0, c->stream>>>(flags, offsets, n, k, cp);
    c->count_launch();
  }
  TIDQ_CUDA(cudaGetLastError());
}

}  // namespace prims
}  // namespace tidq
