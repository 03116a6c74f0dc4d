// Store kernels: AoS -> SoA transpose (upload path), the counter-based
// synthetic generator and row gather (kernel.py:257-266).
#include <cuda_runtime.h>

#include <memory>

#include "internal.cuh"

namespace tidq {

// Four triples per thread: three 16-B loads of AoS, one 16-B store per column.
__global__ void __launch_bounds__(256) transpose_aos_kernel(const uint4* __restrict__ aos,
                                                            uint64_t n4, uint4* __restrict__ s,
                                                            uint4* __restrict__ p,
                                                            uint4* __restrict__ o) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n4;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint4 a = __ldcs(aos + 3 * i);
    const uint4 b = __ldcs(aos + 3 * i + 1);
    const uint4 c = __ldcs(aos + 3 * i + 2);
    // a = s0 p0 o0 s1 | b = p1 o1 s2 p2 | c = o2 s3 p3 o3
    s[i] = make_uint4(a.x, a.w, b.z, c.y);
    p[i] = make_uint4(a.y, b.x, b.w, c.z);
    o[i] = make_uint4(a.z, b.y, c.x, c.w);
  }
}

__global__ void transpose_tail_kernel(const uint32_t* __restrict__ aos, uint64_t lo, uint64_t n,
                                      uint32_t* s, uint32_t* p, uint32_t* o) {
  const uint64_t i = lo + threadIdx.x;
  if (i < n) {
    s[i] = aos[3 * i];
    p[i] = aos[3 * i + 1];
    o[i] = aos[3 * i + 2];
  }
}

void launch_transpose_aos(Ctx* c, const uint32_t* aos, uint64_t n, uint32_t* s, uint32_t* p,
                          uint32_t* o, cudaStream_t stream) {
  const uint64_t n4 = n / 4;
  if (n4) {
    const int grid = int(std::min<uint64_t>((n4 + 255) / 256, uint64_t(c->sm_count) * 8));
    transpose_aos_kernel<<<grid, 256, 0, stream>>>(reinterpret_cast<const uint4*>(aos), n4,
                                                   reinterpret_cast<uint4*>(s),
                                                   reinterpret_cast<uint4*>(p),
                                                   reinterpret_cast<uint4*>(o));
    c->count_launch();
  }
  if (n % 4) {
    transpose_tail_kernel<<<1, 32, 0, stream>>>(aos, n4 * 4, n, s, p, o);
    c->count_launch();
  }
  TIDQ_CUDA(cudaGetLastError());
}

// ---- synthetic generator ----------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// first r in [0, n) with h < cdf[r]  (cdf ascending, cdf[n-1] = 2^64-1)
__device__ __forceinline__ uint32_t zipf_rank(const uint64_t* __restrict__ cdf, uint32_t n,
                                              uint64_t h) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (h < __ldg(cdf + mid))
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo < n ? lo : n - 1;
}

__global__ void __launch_bounds__(256) generate_kernel(tidq_synth_params prm,
                                                       const uint64_t* __restrict__ cdf,
                                                       uint32_t* __restrict__ s,
                                                       uint32_t* __restrict__ p,
                                                       uint32_t* __restrict__ o) {
  const uint64_t salt = prm.seed * 0xD1B54A32D192ED03ull;
  const uint32_t ent0 = prm.n_p + 1;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < prm.n_triples;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t g = (prm.base_index + i) << 2;
    const uint64_t h0 = splitmix64((g | 0) ^ salt);
    const uint64_t h1 = splitmix64((g | 1) ^ salt);
    const uint64_t h2 = splitmix64((g | 2) ^ salt);
    s[i] = ent0 + uint32_t(((h0 >> 32) * uint64_t(prm.n_e)) >> 32);
    p[i] = 1 + zipf_rank(cdf, prm.n_p, h1);
    o[i] = ent0 + uint32_t(((h2 >> 32) * uint64_t(prm.n_e)) >> 32);
  }
}

void launch_generate(Ctx* c, const tidq_synth_params& prm, const uint64_t* cdf_dev, uint32_t* s,
                     uint32_t* p, uint32_t* o, cudaStream_t stream) {
  if (prm.n_triples == 0) return;
  const int grid =
      int(std::min<uint64_t>((prm.n_triples + 255) / 256, uint64_t(c->sm_count) * 16));
  generate_kernel<<<grid, 256, 0, stream>>>(prm, cdf_dev, s, p, o);
  c->count_launch();
  TIDQ_CUDA(cudaGetLastError());
}

// ---- gather ------------------------------------------------------------------
__global__ void gather_rows_kernel(const uint32_t* __restrict__ s, const uint32_t* __restrict__ p,
                                   const uint32_t* __restrict__ o, const int64_t* __restrict__ idx,
                                   uint64_t n, uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const int64_t k = idx[i];
    out[3 * i] = s[k];
    out[3 * i + 1] = p[k];
    out[3 * i + 2] = o[k];
  }
}

}  // namespace tidq

using namespace tidq;

extern "C" int tidq_store_gather(tidq_store* st, const int64_t* local_idx, uint64_t n,
                                 uint32_t* aos_out) {
  return guarded([&] {
    TIDQ_REQUIRE(st && ((local_idx && aos_out) || n == 0), TIDQ_E_INVALID, "null argument");
    if (n == 0) return;
    Ctx* c = st->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    for (uint64_t i = 0; i < n; ++i)
      TIDQ_REQUIRE(local_idx[i] >= 0 && uint64_t(local_idx[i]) < st->n, TIDQ_E_INVALID,
                   "gather index out of range");
    DevBuf didx(c, n * 8), dout(c, n * 12);
    TIDQ_CUDA(cudaMemcpyAsync(didx.ptr, local_idx, n * 8, cudaMemcpyHostToDevice, c->stream));
    const int grid = int(std::min<uint64_t>((n + 255) / 256, uint64_t(c->sm_count) * 8));
    gather_rows_kernel<<<grid, 256, 0, c->stream>>>(st->s.as<uint32_t>(), st->p.as<uint32_t>(),
                                                    st->o.as<uint32_t>(), didx.as<int64_t>(), n,
                                                    dout.as<uint32_t>());
    c->count_launch();
    TIDQ_CUDA(cudaGetLastError());
    TIDQ_CUDA(cudaMemcpyAsync(aos_out, dout.ptr, n * 12, cudaMemcpyDeviceToHost, c->stream));
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
  });
}

namespace tidq {
struct GatherCols {
  int n;
  const uint32_t* src[3];
  uint32_t* dst[3];
};

__global__ void __launch_bounds__(256) gather_cols_kernel(const uint32_t* __restrict__ idx, uint64_t n,
                                                          const __grid_constant__ GatherCols gc) {
  const uint64_t base = uint64_t(blockIdx.x) * 1024;
  uint32_t r[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint64_t i = base + j * 256 + threadIdx.x;
    r[j] = i < n ? __ldg(idx + i) : 0u;
  }
  for (int k = 0; k < gc.n; ++k) {
    uint32_t v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = base + j * 256 + threadIdx.x < n ? ld_gather(gc.src[k] + r[j]) : 0u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t i = base + j * 256 + threadIdx.x;
      if (i < n) gc.dst[k][i] = v[j];
    }
  }
}
// Several patterns' deferred columns in one pass, each through its own
// index column: every index load of a thread's rows, then every gather, are
// in flight together (one launch instead of one per pattern)
constexpr int kGatherMax = 8;
struct GatherColsM {
  int n;
  const uint32_t* idx[kGatherMax];
  const uint32_t* src[kGatherMax];
  uint32_t* dst[kGatherMax];
};

__global__ void __launch_bounds__(256) gather_cols_multi_kernel(uint64_t n, const __grid_constant__ GatherColsM gc) {
  const uint64_t base = uint64_t(blockIdx.x) * 1024;
  uint32_t r[kGatherMax][4];
#pragma unroll
  for (int k = 0; k < kGatherMax; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t i = base + j * 256 + threadIdx.x;
      r[k][j] = k < gc.n && i < n ? __ldg(gc.idx[k] + i) : 0u;
    }
#pragma unroll
  for (int k = 0; k < kGatherMax; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t i = base + j * 256 + threadIdx.x;
      if (k < gc.n && i < n) r[k][j] = ld_gather(gc.src[k] + r[k][j]);
    }
#pragma unroll
  for (int k = 0; k < kGatherMax; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t i = base + j * 256 + threadIdx.x;
      if (k < gc.n && i < n) gc.dst[k][i] = r[k][j];
    }
}
}  // namespace tidq

extern "C" int tidq_store_gather_cols_multi(tidq_store* st, tidq_table* t, int32_t n_out, const int32_t* spec,
                                            const int32_t* idx_cols, tidq_table** out) {
  return guarded([&] {
    TIDQ_REQUIRE(st && t && out && spec && idx_cols && n_out >= 1 && n_out <= 16, TIDQ_E_INVALID, "bad argument");
    Ctx* c = st->ctx;
    TIDQ_REQUIRE(t->ctx == c, TIDQ_E_INVALID, "table and store on different contexts");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    const uint64_t n = t->n_rows();
    const uint32_t* cols[3] = {st->s.as<uint32_t>(), st->p.as<uint32_t>(), st->o.as<uint32_t>()};
    auto o = std::make_unique<tidq_table>();
    o->ctx = c;
    o->set_rows(n);
    o->capacity = n;
    o->cols.resize(n_out);
    GatherColsM gc{};
    std::vector<int> used(t->cols.size(), 0);
    for (int k = 0; k < n_out; ++k) {
      if (spec[k] >= 0) {
        TIDQ_REQUIRE(spec[k] < int32_t(t->cols.size()), TIDQ_E_INVALID, "column out of range");
        ++used[spec[k]];
      } else {
        TIDQ_REQUIRE(spec[k] >= -3, TIDQ_E_INVALID, "slot must be 0, 1 or 2");
        TIDQ_REQUIRE(gc.n < kGatherMax, TIDQ_E_INVALID, "at most 8 gathered columns");
        const int ic = idx_cols[k];
        TIDQ_REQUIRE(ic >= 0 && ic < int32_t(t->cols.size()) && t->cols[ic].dtype == TIDQ_U32, TIDQ_E_INVALID,
                     "index column must be a uint32 column of the table");
        Column& col = o->cols[k];
        col.dtype = TIDQ_U32;
        col.buf = DevBuf(c, std::max<uint64_t>(n, 1) * 4);
        gc.idx[gc.n] = t->cols[ic].buf.as<uint32_t>();
        gc.src[gc.n] = cols[-1 - spec[k]];
        gc.dst[gc.n] = col.buf.as<uint32_t>();
        ++gc.n;
      }
    }
    if (n && gc.n) {  // gather before any index column is moved out
      gather_cols_multi_kernel<<<unsigned((n + 1023) / 1024), 256, 0, c->stream>>>(n, gc);
      c->count_launch();
      TIDQ_CUDA(cudaGetLastError());
    }
    for (int k = 0; k < n_out; ++k) {
      if (spec[k] < 0) continue;
      Column& src = t->cols[spec[k]];
      Column& dst = o->cols[k];
      dst.dtype = src.dtype;
      if (--used[spec[k]] == 0 && src.buf.ptr) {
        dst.buf = std::move(src.buf);  // last use: move
      } else {
        dst.buf = DevBuf(c, std::max<uint64_t>(n, 1) * Column::width(src.dtype));
        if (n) TIDQ_CUDA(cudaMemcpyAsync(dst.buf.ptr, src.buf.ptr, n * Column::width(src.dtype),
                                         cudaMemcpyDeviceToDevice, c->stream));
      }
    }
    *out = o.release();  // stream-ordered: no wait
  });
}

extern "C" int tidq_store_gather_cols(tidq_store* st, tidq_table* t, int32_t idx_col, int32_t n_out,
                                      const int32_t* spec, tidq_table** out) {
  return guarded([&] {
    TIDQ_REQUIRE(st && t && out && spec && n_out >= 1 && n_out <= 16, TIDQ_E_INVALID, "bad argument");
    TIDQ_REQUIRE(idx_col >= 0 && idx_col < int32_t(t->cols.size()) && t->cols[idx_col].dtype == TIDQ_U32,
                 TIDQ_E_INVALID, "index column must be uint32");
    Ctx* c = st->ctx;
    TIDQ_REQUIRE(t->ctx == c, TIDQ_E_INVALID, "table and store on different contexts");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    const uint64_t n = t->n_rows();
    const uint32_t* cols[3] = {st->s.as<uint32_t>(), st->p.as<uint32_t>(), st->o.as<uint32_t>()};
    auto o = std::make_unique<tidq_table>();
    o->ctx = c;
    o->set_rows(n);
    o->capacity = n;
    o->cols.resize(n_out);
    GatherCols gc{};
    std::vector<int> used(t->cols.size(), 0);
    for (int k = 0; k < n_out; ++k) {
      if (spec[k] >= 0) {
        TIDQ_REQUIRE(spec[k] < int32_t(t->cols.size()), TIDQ_E_INVALID, "column out of range");
        ++used[spec[k]];
      } else {
        TIDQ_REQUIRE(spec[k] >= -3, TIDQ_E_INVALID, "slot must be 0, 1 or 2");
        TIDQ_REQUIRE(gc.n < 3, TIDQ_E_INVALID, "at most 3 gathered columns");
        Column& col = o->cols[k];
        col.dtype = TIDQ_U32;
        col.buf = DevBuf(c, std::max<uint64_t>(n, 1) * 4);
        gc.src[gc.n] = cols[-1 - spec[k]];
        gc.dst[gc.n] = col.buf.as<uint32_t>();
        ++gc.n;
      }
    }
    if (n && gc.n) {  // gather before any index column is moved out
      gather_cols_kernel<<<unsigned((n + 1023) / 1024), 256, 0, c->stream>>>(
          t->cols[idx_col].buf.as<uint32_t>(), n, gc);
      c->count_launch();
      TIDQ_CUDA(cudaGetLastError());
    }
    for (int k = 0; k < n_out; ++k) {
      if (spec[k] < 0) continue;
      Column& src = t->cols[spec[k]];
      Column& dst = o->cols[k];
      dst.dtype = src.dtype;
      if (--used[spec[k]] == 0 && src.buf.ptr) {
        dst.buf = std::move(src.buf);  // last use: move
      } else {
        dst.buf = DevBuf(c, std::max<uint64_t>(n, 1) * Column::width(src.dtype));
        if (n) TIDQ_CUDA(cudaMemcpyAsync(dst.buf.ptr, src.buf.ptr, n * Column::width(src.dtype),
                                         cudaMemcpyDeviceToDevice, c->stream));
      }
    }
    *out = o.release();  // stream-ordered: no wait
  });
}

// ---- predicate histogram (capacity hints for ?P? scans) -----------------------
namespace tidq {

// counts[p] for p <= max_id; a per-CTA shared histogram when it fits, else
// global atomics aggregated per warp with __match_any_sync (Zipf-hot ids).
__global__ void __launch_bounds__(256) pred_hist_smem_kernel(const uint32_t* __restrict__ p,
                                                             uint64_t n, uint32_t max_id,
                                                             unsigned long long* __restrict__ out) {
  extern __shared__ uint32_t h[];
  for (uint32_t i = threadIdx.x; i <= max_id; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t v = p[i];
    if (v <= max_id) atomicAdd(&h[v], 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i <= max_id; i += blockDim.x)
    if (h[i]) atomicAdd(out + i, (unsigned long long)h[i]);
}

__global__ void __launch_bounds__(256) pred_hist_global_kernel(const uint32_t* __restrict__ p,
                                                               uint64_t n, uint32_t max_id,
                                                               unsigned long long* __restrict__ out) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t base = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) & ~31ull; base < n;
       base += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = base + lane;
    const uint32_t v = i < n ? p[i] : 0xffffffffu;
    const bool ok = i < n && v <= max_id;
    const uint32_t peers = __match_any_sync(0xffffffffu, ok ? v : 0xffffffffu);
    if (ok && lane == uint32_t(__ffs(peers) - 1)) atomicAdd(out + v, (unsigned long long)__popc(peers));
  }
}

}  // namespace tidq

extern "C" int tidq_store_pred_hist(tidq_store* st, uint32_t max_id, uint64_t* counts_out) {
  return guarded([&] {
    TIDQ_REQUIRE(st && counts_out, TIDQ_E_INVALID, "null argument");
    TIDQ_REQUIRE(max_id < (1u << 28), TIDQ_E_INVALID, "max_id too large for a dense histogram");
    Ctx* c = st->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    const size_t bins = size_t(max_id) + 1;
    DevBuf d(c, bins * 8);
    TIDQ_CUDA(cudaMemsetAsync(d.ptr, 0, bins * 8, c->stream));
    if (st->n) {
      const int grid = int(std::min<uint64_t>((st->n + 255) / 256, uint64_t(c->sm_count) * 4));
      if (bins * 4 <= 96 * 1024) {
        ensure_dyn_smem(reinterpret_cast<const void*>(pred_hist_smem_kernel), c->device, 96 * 1024);
        pred_hist_smem_kernel<<<grid, 256, bins * 4, c->stream>>>(
            st->p.as<uint32_t>(), st->n, max_id, d.as<unsigned long long>());
      } else {
        pred_hist_global_kernel<<<grid, 256, 0, c->stream>>>(st->p.as<uint32_t>(), st->n, max_id,
                                                             d.as<unsigned long long>());
      }
      c->count_launch();
      TIDQ_CUDA(cudaGetLastError());
    }
    TIDQ_CUDA(cudaMemcpyAsync(counts_out, d.ptr, bins * 8, cudaMemcpyDeviceToHost, c->stream));
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
  });
}

// ---- predicate-code column ------------------------------------------------------
// A dictionary-coded copy of the predicate column: code = rank of the
// predicate ID among the store's distinct predicate IDs.  RDF stores have few
// distinct predicates (10^4 in the synthetic configs), so a 16-bit code
// halves the bytes the scan's mark streams for the usual ?s P ?o keys; the
// uint32 columns stay (every gather, projection and download reads them).
namespace tidq {

// Codes are rank + kPcodeBase: every code is then a normal, finite fp16
// bit pattern, so the multi-stream mark can compare two codes per
// instruction on the half-precision pipe (setp.eq.f16x2) exactly; 0xFFFF
// (no predicate) is a NaN and equals nothing.
__global__ void __launch_bounds__(256) pcode_lut_kernel(const uint32_t* __restrict__ pvals, uint32_t n_vals,
                                                        uint16_t* __restrict__ lut) {
  const uint32_t i = blockIdx.x * 256 + threadIdx.x;
  if (i < n_vals) lut[pvals[i]] = uint16_t(i + kPcodeBase);
}

// p16[i] = lut[p[i]] over the padded column (padding p = 0 -> 0xFFFF unless 0 is a predicate)
__global__ void __launch_bounds__(256) pcode_map_kernel(const uint32_t* __restrict__ p, uint64_t n,
                                                        const uint16_t* __restrict__ lut, uint32_t lut_n,
                                                        uint16_t* __restrict__ out) {
  const uint64_t i0 = (uint64_t(blockIdx.x) * 256 + threadIdx.x) * 4;
  if (i0 >= n) return;
  const uint4 v = *reinterpret_cast<const uint4*>(p + i0);  // n is a multiple of the scan tile
  auto code = [&](uint32_t x) -> uint32_t { return x < lut_n ? lut[x] : 0xFFFFu; };
  *reinterpret_cast<uint2*>(out + i0) =
      make_uint2(code(v.x) | (code(v.y) << 16), code(v.z) | (code(v.w) << 16));
}

}  // namespace tidq

extern "C" int tidq_store_pcodes(tidq_store* st, const uint32_t* pvals, uint32_t n_vals) {
  return guarded([&] {
    TIDQ_REQUIRE(st && (pvals || !n_vals), TIDQ_E_INVALID, "null argument");
    TIDQ_REQUIRE(n_vals <= kPcodeMax, TIDQ_E_INVALID, "more than 30000 distinct predicates");
    for (uint32_t i = 1; i < n_vals; ++i)
      TIDQ_REQUIRE(pvals[i - 1] < pvals[i], TIDQ_E_INVALID, "pvals must ascend strictly");
    TIDQ_REQUIRE(!n_vals || pvals[n_vals - 1] < (1u << 28), TIDQ_E_INVALID, "predicate IDs above 2^28");
    Ctx* c = st->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    st->p16.reset();
    st->pvals.clear();
    if (!n_vals) return;
    const uint32_t lut_n = pvals[n_vals - 1] + 1;
    DevBuf dv(c, size_t(n_vals) * 4), lut(c, size_t(lut_n) * 2);
    TIDQ_CUDA(cudaMemcpyAsync(dv.ptr, pvals, size_t(n_vals) * 4, cudaMemcpyHostToDevice, c->stream));
    TIDQ_CUDA(cudaMemsetAsync(lut.ptr, 0xFF, size_t(lut_n) * 2, c->stream));
    pcode_lut_kernel<<<(n_vals + 255) / 256, 256, 0, c->stream>>>(dv.as<uint32_t>(), n_vals, lut.as<uint16_t>());
    DevBuf p16(c, std::max<uint64_t>(st->padded, 1) * 2);
    if (st->padded)
      pcode_map_kernel<<<unsigned((st->padded / 4 + 255) / 256), 256, 0, c->stream>>>(
          st->p.as<uint32_t>(), st->padded, lut.as<uint16_t>(), lut_n, p16.as<uint16_t>());
    c->count_launch(2);
    TIDQ_CUDA(cudaGetLastError());
    st->p16 = std::move(p16);  // stream-ordered: the next scan on this stream sees it
    st->pvals.assign(pvals, pvals + n_vals);
  });
}

// ---- interleaved (s, o) column ---------------------------------------------------
namespace tidq {
__global__ void __launch_bounds__(256) so_build_kernel(const uint32_t* __restrict__ s, const uint32_t* __restrict__ o,
                                                       uint64_t n, uint2* __restrict__ so) {
  const uint64_t i0 = (uint64_t(blockIdx.x) * 256 + threadIdx.x) * 4;
  if (i0 >= n) return;
  const uint4 a = *reinterpret_cast<const uint4*>(s + i0);  // n: a multiple of the scan tile
  const uint4 b = *reinterpret_cast<const uint4*>(o + i0);
  uint4* d = reinterpret_cast<uint4*>(so + i0);
  d[0] = make_uint4(a.x, b.x, a.y, b.y);
  d[1] = make_uint4(a.z, b.z, a.w, b.w);
}
}  // namespace tidq

extern "C" int tidq_store_so(tidq_store* st, int32_t enable) {
  return guarded([&] {
    TIDQ_REQUIRE(st, TIDQ_E_INVALID, "null store");
    Ctx* c = st->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    st->so.reset();
    if (!enable) return;
    DevBuf so(c, std::max<uint64_t>(st->padded, 1) * 8);
    if (st->padded)
      so_build_kernel<<<unsigned((st->padded / 4 + 255) / 256), 256, 0, c->stream>>>(
          st->s.as<uint32_t>(), st->o.as<uint32_t>(), st->padded, so.as<uint2>());
    c->count_launch();
    TIDQ_CUDA(cudaGetLastError());
    st->so = std::move(so);  // stream-ordered
  });
}
