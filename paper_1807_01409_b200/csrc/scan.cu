// The TripleID pattern scan (reference kernel.py:148-227 search_chunk /
// search_multi, query_ops.py:263-295 scan_patterns with the pattern_table
// repeated-variable mask query_ops.py:210-229 and the FILTER of
// query_ops.py:241-252 fused as an epilogue predicate).
//
// One pass over the resident SoA columns:
//   * each CTA owns one tile of kTile consecutive triples; only the columns a
//     key binds are streamed (128-bit, L1::no_allocate);
//   * every key is tested per triple in registers -> 32-bit mark set;
//   * each output stream (a key, or the union of keys for search_multi)
//     selects triples by its mark bits, then applies its epilogue
//     predicates (slot equalities, FILTER bitmaps);
//   * order-preserving compaction: ballots give the rank inside a 128-triple
//     warp chunk, a 32-entry chunk scan gives the rank inside the tile, and a
//     decoupled look-back over the tiles gives the global offset, so every
//     stream comes out in ascending triple order in ONE read of the data;
//   * free columns the outputs need are gathered only for 4-triple vectors
//     that contain a candidate hit.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <memory>

#include "internal.cuh"

namespace tidq {
namespace scan {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kRounds = 8;
constexpr int kVec = 4;
constexpr int kTile = kThreads * kRounds * kVec;  // 4096 triples
constexpr int kChunks = kRounds * kWarps;         // 32 warp chunks per tile
static_assert(kTile == int(kScanTile), "tile size mismatch with store padding");
static_assert(kChunks == 32, "chunk scan assumes one warp");

enum : uint32_t { kFlagInvalid = 0, kFlagAggregate = 1, kFlagPrefix = 2 };

struct StreamP {
  uint32_t select;
  uint32_t eq_flags;
  int32_t n_out;
  int32_t out_kind[TIDQ_MAX_OUT];
  void* out_ptr[TIDQ_MAX_OUT];
  int32_t answer_key;
  int32_t n_filters;
  int32_t filter_slot[TIDQ_MAX_FILTERS];
  const uint32_t* filter_words[TIDQ_MAX_FILTERS];
  uint64_t filter_nbits[TIDQ_MAX_FILTERS];
  uint64_t capacity;
};

struct Params {
  const uint32_t* col[3];
  uint64_t n;
  uint64_t base;
  uint32_t n_tiles;
  uint32_t sample_stride;
  int32_t n_keys;
  int32_t n_streams;
  uint32_t load_mask;  // bit k: column k is read for every triple
  uint32_t late_mask;  // bit k: column k is gathered for candidate vectors
  uint32_t cand_mask;  // union of stream selects
  uint32_t key[TIDQ_MAX_KEYS][3];
  uint32_t key_bound[TIDQ_MAX_KEYS];  // bit k: slot k bound
  StreamP streams[TIDQ_MAX_STREAMS];
  uint32_t* flags;    // [n_tiles]
  uint32_t* agg;      // [n_tiles][n_streams]
  uint64_t* incl;     // [n_tiles][n_streams]
  uint64_t* counts;   // [n_streams]
};

__device__ __forceinline__ uint4 ld_stream(const uint32_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t pick(const uint32_t (&v)[3][kRounds][kVec], int slot, int r,
                                         int c) {
  return slot == 0 ? v[0][r][c] : (slot == 1 ? v[1][r][c] : v[2][r][c]);
}

__device__ __forceinline__ bool bitmap_test(const uint32_t* words, uint64_t nbits, uint32_t id) {
  return uint64_t(id) < nbits && ((__ldg(words + (id >> 5)) >> (id & 31)) & 1u);
}

// Dynamic shared memory layout: nib[n_streams][kThreads] (uint16) then
// cnt[n_streams][kChunks] (uint32), total[n_streams], base[n_streams].
template <bool kCountOnly>
__global__ void __launch_bounds__(kThreads) scan_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int S = P.n_streams;
  uint64_t* s_base = reinterpret_cast<uint64_t*>(smem);
  uint32_t* s_total = reinterpret_cast<uint32_t*>(s_base + TIDQ_MAX_STREAMS);
  uint32_t* s_cnt = s_total + TIDQ_MAX_STREAMS;                 // [S][kChunks]
  uint16_t* s_nib = reinterpret_cast<uint16_t*>(s_cnt + S * kChunks);  // [S][kThreads]

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const uint32_t tile = kCountOnly ? blockIdx.x * P.sample_stride : blockIdx.x;
  const uint64_t t0 = uint64_t(tile) * kTile;

  // ---- load the bound columns ------------------------------------------------
  uint32_t v[3][kRounds][kVec];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (P.load_mask & (1u << k)) {
      const uint32_t* src = P.col[k] + t0;
#pragma unroll
      for (int r = 0; r < kRounds; ++r) {
        const uint4 x = ld_stream(src + (size_t(r) * kThreads + tid) * kVec);
        v[k][r][0] = x.x;
        v[k][r][1] = x.y;
        v[k][r][2] = x.z;
        v[k][r][3] = x.w;
      }
    } else {
#pragma unroll
      for (int r = 0; r < kRounds; ++r)
#pragma unroll
        for (int c = 0; c < kVec; ++c) v[k][r][c] = 0;
    }
  }

  // ---- match: mark set per triple ---------------------------------------------
  uint32_t mark[kRounds][kVec];
#pragma unroll
  for (int r = 0; r < kRounds; ++r)
#pragma unroll
    for (int c = 0; c < kVec; ++c) mark[r][c] = 0;
#pragma unroll 1
  for (int q = 0; q < P.n_keys; ++q) {
    const uint32_t b = P.key_bound[q];
    const uint32_t k0 = P.key[q][0], k1 = P.key[q][1], k2 = P.key[q][2];
    const uint32_t bit = 1u << q;
#pragma unroll
    for (int r = 0; r < kRounds; ++r)
#pragma unroll
      for (int c = 0; c < kVec; ++c) {
        const bool ok = (!(b & 1u) || v[0][r][c] == k0) && (!(b & 2u) || v[1][r][c] == k1) &&
                        (!(b & 4u) || v[2][r][c] == k2);
        mark[r][c] |= ok ? bit : 0u;
      }
  }
  if (t0 + kTile > P.n) {  // partial last tile: drop padding triples
#pragma unroll
    for (int r = 0; r < kRounds; ++r)
#pragma unroll
      for (int c = 0; c < kVec; ++c)
        if (t0 + (uint64_t(r) * kThreads + tid) * kVec + c >= P.n) mark[r][c] = 0;
  }

  // ---- gather the free columns for vectors holding a candidate -------------------
  if (P.late_mask) {
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      const uint32_t any =
          (mark[r][0] | mark[r][1] | mark[r][2] | mark[r][3]) & P.cand_mask;
      if (any) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          if (P.late_mask & (1u << k)) {
            const uint4 x = ld_stream(P.col[k] + t0 + (size_t(r) * kThreads + tid) * kVec);
            v[k][r][0] = x.x;
            v[k][r][1] = x.y;
            v[k][r][2] = x.z;
            v[k][r][3] = x.w;
          }
        }
      }
    }
  }

  // ---- per stream: predicates -> hit nibbles -> warp-chunk counts ----------------
#pragma unroll 1
  for (int s = 0; s < S; ++s) {
    const StreamP& st = P.streams[s];
    const uint32_t sel = st.select;
    const uint32_t eqf = st.eq_flags;
    const int nf = st.n_filters;
    uint32_t nibs = 0;
#pragma unroll
    for (int r = 0; r < kRounds; ++r)
#pragma unroll
      for (int c = 0; c < kVec; ++c) {
        bool hit = (mark[r][c] & sel) != 0;
        if (eqf) {
          hit = hit && (!(eqf & TIDQ_EQ_SP) || v[0][r][c] == v[1][r][c]) &&
                (!(eqf & TIDQ_EQ_SO) || v[0][r][c] == v[2][r][c]) &&
                (!(eqf & TIDQ_EQ_PO) || v[1][r][c] == v[2][r][c]);
        }
        if (hit && nf) {
          for (int f = 0; f < nf; ++f)
            hit = hit && bitmap_test(st.filter_words[f], st.filter_nbits[f],
                                     pick(v, st.filter_slot[f], r, c));
        }
        nibs |= uint32_t(hit) << (r * kVec + c);
      }
    if (!kCountOnly) s_nib[s * kThreads + tid] = uint16_t(nibs);
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      const uint32_t cnt = __reduce_add_sync(0xffffffffu, __popc((nibs >> (r * kVec)) & 0xFu));
      if (lane == 0) s_cnt[s * kChunks + r * kWarps + warp] = cnt;
    }
  }
  __syncthreads();

  // ---- chunk scan: exclusive chunk offsets + tile totals ------------------------
  for (int s = warp; s < S; s += kWarps) {
    const uint32_t x = s_cnt[s * kChunks + lane];
    uint32_t inc = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += y;
    }
    s_cnt[s * kChunks + lane] = inc - x;
    if (lane == 31) s_total[s] = inc;
  }
  __syncthreads();

  if (kCountOnly) {
    if (tid < S) atomicAdd(reinterpret_cast<unsigned long long*>(P.counts + tid),
                           (unsigned long long)s_total[tid]);
    return;
  }

  // ---- decoupled look-back: global offset of this tile for every stream ----------
  if (warp == 0) {
    uint64_t excl = 0;  // lane s accumulates stream s
    if (tile == 0) {
      if (lane == 0) {
        for (int s = 0; s < S; ++s) P.incl[s] = s_total[s];
        __threadfence();
        st_release(P.flags, kFlagPrefix);
      }
    } else {
      if (lane == 0) {
        for (int s = 0; s < S; ++s) P.agg[size_t(tile) * S + s] = s_total[s];
        __threadfence();
        st_release(P.flags + tile, kFlagAggregate);
      }
      int64_t pred = int64_t(tile) - 1;
      while (true) {
        const int64_t t = pred - lane;
        uint32_t f = kFlagPrefix;
        if (t >= 0) {
          do {
            f = ld_acquire(P.flags + t);
          } while (f == kFlagInvalid);
        }
        const uint32_t pm = __ballot_sync(0xffffffffu, f == kFlagPrefix);
        const int stop = pm ? __ffs(pm) - 1 : 31;
        __threadfence();
        if (lane < S) {
          for (int w = 0; w <= stop; ++w) {
            const size_t tt = size_t(pred - w);
            excl += (pm && w == stop) ? ld_relaxed_u64(P.incl + tt * S + lane)
                                      : uint64_t(ld_relaxed_u32(P.agg + tt * S + lane));
          }
        }
        if (pm) break;
        pred -= 32;
      }
      if (lane < S) s_base[lane] = excl;
      __syncwarp();
      if (lane == 0) {
        for (int s = 0; s < S; ++s) P.incl[size_t(tile) * S + s] = s_base[s] + s_total[s];
        __threadfence();
        st_release(P.flags + tile, kFlagPrefix);
      }
    }
    if (tile == 0 && lane < S) s_base[lane] = 0;
    if (tile == P.n_tiles - 1 && lane < S) P.counts[lane] = excl + s_total[lane];
  }
  __syncthreads();

  // ---- write: rank = tile base + chunk offset + lanes before + within thread -------
  const uint32_t lt = lanemask_lt();
#pragma unroll 1
  for (int s = 0; s < S; ++s) {
    const StreamP& st = P.streams[s];
    const uint32_t nibs = s_nib[s * kThreads + tid];
    const uint64_t base = s_base[s];
    const uint64_t cap = st.capacity;
    const int n_out = st.n_out;
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      const uint32_t nib = (nibs >> (r * kVec)) & 0xFu;
      const uint32_t b0 = __ballot_sync(0xffffffffu, nib & 1u);
      const uint32_t b1 = __ballot_sync(0xffffffffu, nib & 2u);
      const uint32_t b2 = __ballot_sync(0xffffffffu, nib & 4u);
      const uint32_t b3 = __ballot_sync(0xffffffffu, nib & 8u);
      if (!nib) continue;
      uint64_t pos = base + s_cnt[s * kChunks + r * kWarps + warp] + __popc(b0 & lt) +
                     __popc(b1 & lt) + __popc(b2 & lt) + __popc(b3 & lt);
#pragma unroll
      for (int c = 0; c < kVec; ++c) {
        if (!(nib & (1u << c))) continue;
        if (pos < cap) {
          for (int k = 0; k < n_out; ++k) {
            const int kind = st.out_kind[k];
            void* dst = st.out_ptr[k];
            if (kind <= TIDQ_OUT_O) {
              static_cast<uint32_t*>(dst)[pos] = pick(v, kind, r, c);
            } else if (kind == TIDQ_OUT_INDEX) {
              static_cast<int64_t*>(dst)[pos] =
                  int64_t(P.base + t0 + (uint64_t(r) * kThreads + tid) * kVec + c);
            } else if (kind == TIDQ_OUT_MARKS) {
              static_cast<uint32_t*>(dst)[pos] = mark[r][c];
            } else {  // TIDQ_OUT_ANSWER
              const int q = st.answer_key;
              const uint32_t a = (v[0][r][c] == P.key[q][0] ? 4u : 0u) |
                                 (v[1][r][c] == P.key[q][1] ? 2u : 0u) |
                                 (v[2][r][c] == P.key[q][2] ? 1u : 0u);
              static_cast<uint8_t*>(dst)[pos] = uint8_t(a);
            }
          }
        }
        ++pos;
      }
    }
  }
}

// Algorithmic bytes of one scan launch: every bound
// column read once (4 B/triple); per emitted row and output field, the write
// plus, for a free column, its read.  FILTER bitmap lookups are not counted.
uint64_t algorithmic_bytes(const Params& P, const uint64_t* counts) {
  uint64_t b = 4ull * P.n * uint64_t(__builtin_popcount(P.load_mask));
  for (int s = 0; s < P.n_streams; ++s) {
    const StreamP& st = P.streams[s];
    uint64_t per_row = 0;
    for (int k = 0; k < st.n_out; ++k) {
      const int kind = st.out_kind[k];
      if (kind <= TIDQ_OUT_O) per_row += (P.load_mask >> kind & 1) ? 4 : 8;
      else if (kind == TIDQ_OUT_INDEX) per_row += 8;
      else if (kind == TIDQ_OUT_MARKS) per_row += 4;
      else per_row += 1 + 4 * (3 - __builtin_popcount(P.load_mask));
    }
    b += per_row * counts[s];
  }
  return b;
}

size_t smem_bytes(int S) {
  return TIDQ_MAX_STREAMS * 8 + TIDQ_MAX_STREAMS * 4 + size_t(S) * kChunks * 4 +
         size_t(S) * kThreads * 2;
}

}  // namespace scan

// Host side of one scan: validate the spec, derive column masks, size the
// outputs (sampled estimate), run the single-pass kernel, retry exactly on
// capacity overflow, and hand back one table per stream.
void run_scan(tidq_store* st, const tidq_scan_spec& spec, tidq_table** out) {
  using namespace scan;
  Ctx* c = st->ctx;
  TIDQ_REQUIRE(spec.n_keys >= 1 && spec.n_keys <= TIDQ_MAX_KEYS, TIDQ_E_TOO_MANY_KEYS,
               std::to_string(spec.n_keys) + " keys; supported range is 1.." +
                   std::to_string(TIDQ_MAX_KEYS));
  TIDQ_REQUIRE(spec.n_streams >= 1 && spec.n_streams <= TIDQ_MAX_STREAMS, TIDQ_E_INVALID,
               "n_streams must be in 1..32");
  const int S = spec.n_streams;
  auto P = std::make_unique<Params>();
  std::memset(P.get(), 0, sizeof(Params));
  P->col[0] = st->s.as<uint32_t>();
  P->col[1] = st->p.as<uint32_t>();
  P->col[2] = st->o.as<uint32_t>();
  P->n = st->n;
  P->base = st->base;
  P->n_keys = spec.n_keys;
  P->n_streams = S;
  uint32_t load = 0, need = 0, cand = 0;
  const uint32_t all_keys = spec.n_keys == 32 ? 0xffffffffu : ((1u << spec.n_keys) - 1);
  for (int q = 0; q < spec.n_keys; ++q) {
    uint32_t b = 0;
    for (int k = 0; k < 3; ++k) {
      P->key[q][k] = spec.keys[q][k];
      if (spec.keys[q][k]) b |= 1u << k;
    }
    P->key_bound[q] = b;
    load |= b;
  }
  for (int s = 0; s < S; ++s) {
    const tidq_stream_spec& ss = spec.streams[s];
    StreamP& sp = P->streams[s];
    TIDQ_REQUIRE((ss.select & ~all_keys) == 0 && ss.select != 0, TIDQ_E_INVALID,
                 "stream select must name keys of this scan");
    TIDQ_REQUIRE(ss.n_out >= 0 && ss.n_out <= TIDQ_MAX_OUT, TIDQ_E_INVALID, "bad n_out");
    TIDQ_REQUIRE(ss.n_filters >= 0 && ss.n_filters <= TIDQ_MAX_FILTERS, TIDQ_E_INVALID,
                 "bad n_filters");
    sp.select = ss.select;
    sp.eq_flags = ss.eq_flags & 7u;
    cand |= ss.select;
    if (sp.eq_flags & TIDQ_EQ_SP) need |= 3u;
    if (sp.eq_flags & TIDQ_EQ_SO) need |= 5u;
    if (sp.eq_flags & TIDQ_EQ_PO) need |= 6u;
    sp.n_out = ss.n_out;
    for (int k = 0; k < ss.n_out; ++k) {
      const int kind = ss.out[k];
      TIDQ_REQUIRE(kind >= TIDQ_OUT_S && kind <= TIDQ_OUT_ANSWER, TIDQ_E_INVALID,
                   "bad output kind");
      sp.out_kind[k] = kind;
      if (kind <= TIDQ_OUT_O) need |= 1u << kind;
      if (kind == TIDQ_OUT_ANSWER) {
        TIDQ_REQUIRE(ss.answer_key >= 0 && ss.answer_key < spec.n_keys, TIDQ_E_INVALID,
                     "bad answer_key");
        need |= 7u;
      }
    }
    sp.answer_key = ss.answer_key;
    sp.n_filters = ss.n_filters;
    for (int f = 0; f < ss.n_filters; ++f) {
      TIDQ_REQUIRE(ss.filter[f] && ss.filter_slot[f] >= 0 && ss.filter_slot[f] < 3,
                   TIDQ_E_INVALID, "bad filter");
      sp.filter_slot[f] = ss.filter_slot[f];
      sp.filter_words[f] = ss.filter[f]->words.as<uint32_t>();
      sp.filter_nbits[f] = ss.filter[f]->n_bits;
      need |= 1u << ss.filter_slot[f];
    }
  }
  P->load_mask = load;
  P->late_mask = need & ~load;
  P->cand_mask = cand;

  const uint64_t n_tiles = std::max<uint64_t>((st->n + kTile - 1) / kTile, 1);
  TIDQ_REQUIRE(n_tiles < (1ull << 31), TIDQ_E_INVALID, "store too large for one scan");
  P->n_tiles = uint32_t(n_tiles);
  const size_t smem = smem_bytes(S);

  // scratch: counts[S] | flags[n_tiles] | agg[n_tiles*S] | incl[n_tiles*S]
  const size_t counts_b = round_up(size_t(S) * 8, 256);
  const size_t flags_b = round_up(n_tiles * 4, 256);
  const size_t agg_b = round_up(n_tiles * S * 4, 256);
  const size_t incl_b = round_up(n_tiles * S * 8, 256);
  const size_t scratch = counts_b + flags_b + agg_b + incl_b;
  if (c->lookback.bytes < scratch) c->lookback = DevBuf(c, scratch);
  char* base = c->lookback.as<char>();
  P->counts = reinterpret_cast<uint64_t*>(base);
  P->flags = reinterpret_cast<uint32_t*>(base + counts_b);
  P->agg = reinterpret_cast<uint32_t*>(base + counts_b + flags_b);
  P->incl = reinterpret_cast<uint64_t*>(base + counts_b + flags_b + agg_b);
  uint64_t* host_counts = static_cast<uint64_t*>(c->pinned_small);

  // ---- capacity: hint, else a sampled count (1 of every `stride` tiles) ----
  std::vector<uint64_t> cap(S, 0);
  bool need_estimate = false;
  for (int s = 0; s < S; ++s) {
    cap[s] = spec.streams[s].capacity_hint;
    if (!cap[s]) need_estimate = true;
  }
  if (need_estimate) {
    const uint32_t stride = uint32_t(std::max<uint64_t>(1, n_tiles / 256));
    const uint32_t sampled = uint32_t((n_tiles + stride - 1) / stride);
    P->sample_stride = stride;
    TIDQ_CUDA(cudaMemsetAsync(P->counts, 0, size_t(S) * 8, c->stream));
    scan_kernel<true><<<sampled, kThreads, smem, c->stream>>>(*P);
    c->count_launch();
    TIDQ_CUDA(cudaGetLastError());
    TIDQ_CUDA(cudaMemcpyAsync(host_counts, P->counts, size_t(S) * 8, cudaMemcpyDeviceToHost,
                              c->stream));
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    for (int s = 0; s < S; ++s) {
      if (cap[s]) continue;
      if (stride == 1) {
        cap[s] = host_counts[s];  // sampled every tile: exact
      } else {
        const double est = double(host_counts[s]) * double(n_tiles) / double(sampled);
        const double slack = 8.0 * std::sqrt(est * stride) + 2.0 * kTile * stride;
        cap[s] = uint64_t(std::min<double>(double(st->n), est * 1.25 + slack));
      }
    }
  }

  std::vector<std::unique_ptr<tidq_table>> tables(S);
  auto allocate = [&](int s, uint64_t capacity) {
    auto t = std::make_unique<tidq_table>();
    t->ctx = c;
    t->capacity = capacity;
    const tidq_stream_spec& ss = spec.streams[s];
    for (int k = 0; k < ss.n_out; ++k) {
      Column col;
      const int kind = ss.out[k];
      col.dtype = kind == TIDQ_OUT_INDEX ? TIDQ_I64 : kind == TIDQ_OUT_ANSWER ? TIDQ_U8 : TIDQ_U32;
      col.buf = DevBuf(c, std::max<uint64_t>(capacity, 1) * Column::width(col.dtype));
      P->streams[s].out_ptr[k] = col.buf.ptr;
      t->cols.push_back(std::move(col));
    }
    P->streams[s].capacity = capacity;
    tables[s] = std::move(t);
  };
  for (int s = 0; s < S; ++s) allocate(s, cap[s]);

  for (int attempt = 0; attempt < 2; ++attempt) {
    TIDQ_CUDA(cudaMemsetAsync(P->flags, 0, n_tiles * 4, c->stream));
    cudaEvent_t ev = c->prof_begin(c->stream);
    scan_kernel<false><<<uint32_t(n_tiles), kThreads, smem, c->stream>>>(*P);
    c->count_launch();
    TIDQ_CUDA(cudaGetLastError());
    c->prof_end("scan", ev, c->stream, 0);
    TIDQ_CUDA(cudaMemcpyAsync(host_counts, P->counts, size_t(S) * 8, cudaMemcpyDeviceToHost,
                              c->stream));
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    if (ev) c->prof["scan"].bytes += algorithmic_bytes(*P, host_counts);
    bool overflow = false;
    for (int s = 0; s < S; ++s)
      if (host_counts[s] > tables[s]->capacity) overflow = true;
    if (!overflow) break;
    TIDQ_REQUIRE(attempt == 0, TIDQ_E_CUDA, "scan overflow after exact resize");
    std::vector<uint64_t> exact(host_counts, host_counts + S);
    for (int s = 0; s < S; ++s) allocate(s, exact[s]);
  }
  for (int s = 0; s < S; ++s) {
    tables[s]->n_rows = host_counts[s];
    out[s] = tables[s].release();
  }
}

}  // namespace tidq

using namespace tidq;

extern "C" int tidq_scan(tidq_store* st, const tidq_scan_spec* spec, tidq_table** out_tables) {
  return guarded([&] {
    TIDQ_REQUIRE(st && spec && out_tables, TIDQ_E_INVALID, "null argument");
    Ctx* c = st->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    run_scan(st, *spec, out_tables);
  });
}

extern "C" int tidq_scan_host(tidq_ctx* ctx, const uint32_t* aos, uint64_t n_triples,
                              uint64_t base_index, const tidq_scan_spec* spec,
                              tidq_table** out_tables) {
  tidq_store* st = nullptr;
  int rc = tidq_store_upload(ctx, aos, n_triples, base_index, &st);
  if (rc != TIDQ_OK) return rc;
  rc = tidq_scan(st, spec, out_tables);
  const int rc2 = tidq_store_free(st);
  return rc != TIDQ_OK ? rc : rc2;
}
