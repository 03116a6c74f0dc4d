// The TripleID pattern scan (reference kernel.py:148-227 search_chunk /
// search_multi, query_ops.py:263-295 scan_patterns with the pattern_table
// repeated-variable mask query_ops.py:210-229 and the FILTER of
// query_ops.py:241-252 fused as an epilogue predicate).
//
// One pass over the resident SoA columns (HBM-bound; no tensor cores):
//   * a CTA takes the next tile of kTile consecutive triples (dynamic tile
//     id, so predecessors are always running or done); only the columns the
//     keys bind are streamed, with 128-bit L1::no_allocate loads, all rounds
//     issued back to back (32 triples / 128 B in flight per thread and column);
//   * keys are tested in registers -> hit bits (single key) or a 32-bit mark
//     set per triple (multi key, kept in shared memory);
//   * each output stream (a key, or the union of keys for search_multi)
//     selects triples by its mark bits and, in the general variant, applies
//     its epilogue predicates (repeated-variable equalities, FILTER bitmaps);
//   * order-preserving compaction: ballots rank a hit inside its 128-triple
//     warp chunk, a 32-entry scan ranks the chunk inside the tile, and a
//     decoupled look-back over packed 64-bit (flag|count) status words — one
//     per (tile, stream), so no fences are needed — gives the tile's global
//     offset; every stream comes out in ascending triple order from ONE read;
//   * free columns the outputs need are prefetched into L2 for hit vectors
//     before the look-back and gathered (one 128-bit load per hit vector) in
//     the write phase.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <memory>

#include "internal.cuh"
#include "pscan.cuh"

namespace tidq {
namespace scan {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kRounds = 8;
constexpr int kVec = 4;
constexpr int kTile = kThreads * kRounds * kVec;  // 4096 triples
constexpr int kChunks = kRounds * kWarps;         // 32 warp chunks per tile
static_assert(int(kScanTile) % kTile == 0, "store padding must cover whole tiles");
static_assert(kChunks == 32, "chunk scan assumes one warp");

constexpr uint64_t kFlagA = 1ull << 62;  // aggregate of this tile only
constexpr uint64_t kFlagP = 2ull << 62;  // inclusive prefix through this tile
constexpr uint64_t kValMask = (1ull << 62) - 1;

// resolved output field kinds
enum : int32_t { kFieldCol = 0, kFieldConst = 1, kFieldIndex = 2, kFieldMarks = 3, kFieldAnswer = 4 };

struct Field {
  int32_t kind;
  int32_t slot;       // kFieldCol: column 0/1/2
  uint32_t constant;  // kFieldConst
  void* ptr;
};

struct StreamP {
  uint32_t select;
  uint32_t eq_flags;
  int32_t n_out;
  int32_t answer_key;
  Field out[TIDQ_MAX_OUT];
  int32_t n_filters;
  int32_t filter_slot[TIDQ_MAX_FILTERS];
  const uint32_t* filter_words[TIDQ_MAX_FILTERS];
  uint64_t filter_nbits[TIDQ_MAX_FILTERS];
  uint64_t capacity;
  uint32_t prefetch_mask;  // columns gathered by this stream's outputs
};

struct Params {
  const uint32_t* col[3];
  const uint32_t* bcol[3];  // bound columns in load order
  int32_t bslot[3];         // slot of bound column b
  uint64_t n;
  uint64_t base;
  uint32_t n_tiles;
  uint32_t sample_stride;
  int32_t n_keys;
  int32_t n_streams;
  uint32_t key[TIDQ_MAX_KEYS][3];
  uint32_t kb_mask[TIDQ_MAX_KEYS];  // bit b: key q compares bound column b
  uint32_t kv[TIDQ_MAX_KEYS][3];    // key q's value for bound column b
  StreamP streams[TIDQ_MAX_STREAMS];
  uint32_t* tile_counter;
  uint64_t* status;  // [n_tiles][n_streams] packed flag|value
  uint64_t* counts;  // [n_streams]
};

__device__ __forceinline__ uint4 ld_stream(const uint32_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t comp(const uint4& v, int c) {
  return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}

__device__ __forceinline__ bool bitmap_test(const uint32_t* words, uint64_t nbits, uint32_t id) {
  return uint64_t(id) < nbits && ((__ldg(words + (id >> 5)) >> (id & 31)) & 1u);
}

struct alignas(16) Smem {
  uint64_t excl[TIDQ_MAX_STREAMS];
  uint32_t total[TIDQ_MAX_STREAMS];
  uint32_t tile;
};

// dynamic smem after Smem: cnt[S][kChunks] u32, nib[S][kThreads] u32,
// marks[kTile] u32 (multi-key only)
template <int NB, bool kSingle, bool kGeneral, bool kCountOnly>
__global__ void __launch_bounds__(kThreads, 4) scan_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int S = P.n_streams;
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem_raw + sizeof(Smem));
  uint32_t* s_nib = s_cnt + S * kChunks;
  uint32_t* s_marks = s_nib + S * kThreads;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  uint32_t tile;
  if (kCountOnly) {
    tile = blockIdx.x * P.sample_stride;
  } else {
    if (tid == 0) sm.tile = atomicAdd(P.tile_counter, 1u);
    if (tid < TIDQ_MAX_STREAMS) sm.excl[tid] = 0;
    __syncthreads();
    tile = sm.tile;
  }
  const uint64_t t0 = uint64_t(tile) * kTile;
  const bool partial = t0 + kTile > P.n;

  // ---- stream the bound columns: all rounds in flight -------------------------
  uint4 x[NB > 0 ? NB : 1][kRounds];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const uint32_t* src = P.bcol[b] + t0 + size_t(tid) * kVec;
#pragma unroll
    for (int r = 0; r < kRounds; ++r) x[b][r] = ld_stream(src + size_t(r) * kThreads * kVec);
  }

  // ---- match ----------------------------------------------------------------------
  uint32_t hb = 0;  // kSingle: bit r*4+c = key 0 accepts triple (r, c)
  if (kSingle) {
    uint32_t kv[NB > 0 ? NB : 1];
#pragma unroll
    for (int b = 0; b < NB; ++b) kv[b] = P.kv[0][b];
#pragma unroll
    for (int r = 0; r < kRounds; ++r)
#pragma unroll
      for (int c = 0; c < kVec; ++c) {
        bool ok = true;
#pragma unroll
        for (int b = 0; b < NB; ++b) ok = ok && comp(x[b][r], c) == kv[b];
        hb |= uint32_t(ok) << (r * kVec + c);
      }
    if (partial) {
#pragma unroll
      for (int r = 0; r < kRounds; ++r)
#pragma unroll
        for (int c = 0; c < kVec; ++c)
          if (t0 + (uint64_t(r) * kThreads + tid) * kVec + c >= P.n) hb &= ~(1u << (r * kVec + c));
    }
  } else {
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      uint32_t m[kVec] = {0u, 0u, 0u, 0u};
#pragma unroll 1
      for (int q = 0; q < P.n_keys; ++q) {
        const uint32_t kb = P.kb_mask[q];
#pragma unroll
        for (int c = 0; c < kVec; ++c) {
          bool ok = true;
#pragma unroll
          for (int b = 0; b < NB; ++b)
            ok = ok && (!(kb & (1u << b)) || comp(x[b][r], c) == P.kv[q][b]);
          m[c] |= uint32_t(ok) << q;
        }
      }
      const int el = (r * kThreads + tid) * kVec;
      uint4 mv = make_uint4(m[0], m[1], m[2], m[3]);
      if (partial) {
        if (t0 + el + 0 >= P.n) mv.x = 0;
        if (t0 + el + 1 >= P.n) mv.y = 0;
        if (t0 + el + 2 >= P.n) mv.z = 0;
        if (t0 + el + 3 >= P.n) mv.w = 0;
      }
      *reinterpret_cast<uint4*>(s_marks + el) = mv;
    }
    __syncwarp();  // each thread only reads back its own marks
  }

  // ---- per stream: hit bits (+ epilogue predicates) and warp-chunk counts ------------
#pragma unroll 1
  for (int s = 0; s < S; ++s) {
    const StreamP& st = P.streams[s];
    const uint32_t sel = st.select;
    uint32_t nibs = 0;
#pragma unroll 1
    for (int r = 0; r < kRounds; ++r) {
      const int el = (r * kThreads + tid) * kVec;
      uint32_t nib;
      if (kSingle) {
        nib = (hb >> (r * kVec)) & 0xFu;
      } else {
        const uint4 mv = *reinterpret_cast<const uint4*>(s_marks + el);
        nib = ((mv.x & sel) ? 1u : 0u) | ((mv.y & sel) ? 2u : 0u) | ((mv.z & sel) ? 4u : 0u) |
              ((mv.w & sel) ? 8u : 0u);
      }
      if (kGeneral && nib && (st.eq_flags || st.n_filters)) {
#pragma unroll
        for (int c = 0; c < kVec; ++c) {
          if (!(nib & (1u << c))) continue;
          const uint64_t e = t0 + el + c;
          const uint32_t vs = __ldg(P.col[0] + e), vp = __ldg(P.col[1] + e), vo = __ldg(P.col[2] + e);
          bool ok = (!(st.eq_flags & TIDQ_EQ_SP) || vs == vp) &&
                    (!(st.eq_flags & TIDQ_EQ_SO) || vs == vo) &&
                    (!(st.eq_flags & TIDQ_EQ_PO) || vp == vo);
          for (int f = 0; ok && f < st.n_filters; ++f) {
            const int sl = st.filter_slot[f];
            ok = bitmap_test(st.filter_words[f], st.filter_nbits[f], sl == 0 ? vs : (sl == 1 ? vp : vo));
          }
          if (!ok) nib &= ~(1u << c);
        }
      }
      if (!kCountOnly && nib && st.prefetch_mask) {
#pragma unroll
        for (int k = 0; k < 3; ++k)
          if (st.prefetch_mask & (1u << k)) prefetch_l2(P.col[k] + t0 + el);
      }
      nibs |= nib << (r * kVec);
      const uint32_t cnt = __reduce_add_sync(0xffffffffu, __popc(nib));
      if (lane == 0) s_cnt[s * kChunks + r * kWarps + warp] = cnt;
    }
    if (!kCountOnly) s_nib[s * kThreads + tid] = nibs;
  }
  __syncthreads();

  // ---- chunk scan: exclusive chunk offsets + tile totals -----------------------------
  for (int s = warp; s < S; s += kWarps) {
    const uint32_t v = s_cnt[s * kChunks + lane];
    uint32_t inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += y;
    }
    s_cnt[s * kChunks + lane] = inc - v;
    if (lane == 31) sm.total[s] = inc;
  }
  __syncthreads();

  if (kCountOnly) {
    if (tid < S)
      atomicAdd(reinterpret_cast<unsigned long long*>(P.counts + tid),
                (unsigned long long)sm.total[tid]);
    return;
  }

  // ---- decoupled look-back (warp 0): lane = (window slot w, stream s) --------------
  if (warp == 0) {
    uint64_t* status = P.status;
    const int W = 32 / S;  // tiles examined per stream per step
    const int my_s = lane % S;
    const int my_w = lane / S;
    const bool valid = my_w < W;
    if (lane < S)
      st_relaxed(status + size_t(tile) * S + lane, (tile == 0 ? kFlagP : kFlagA) | sm.total[lane]);
    if (tile > 0) {
      uint32_t smask = 0;  // lanes of my stream
      for (int w = 0; w < W; ++w) smask |= 1u << (w * S + my_s);
      const uint32_t all_streams = S == 32 ? 0xffffffffu : ((1u << S) - 1);
      uint32_t done = 0;  // bit s: stream s resolved
      int64_t pred = int64_t(tile) - 1;
      while (true) {
        const int64_t t = pred - my_w;
        const bool mine_open = valid && !((done >> my_s) & 1u);
        uint64_t v = kFlagP;  // before tile 0: prefix 0
        if (mine_open && t >= 0) {
          do {
            v = ld_relaxed(status + size_t(t) * S + my_s);
          } while ((v >> 62) == 0);
        }
        const uint32_t pm = __ballot_sync(0xffffffffu, mine_open && (v >> 62) == 2);
        const uint32_t mine = pm & smask;
        const int stop_lane = mine ? __ffs(mine) - 1 : 32;
        const uint64_t add = (mine_open && lane <= stop_lane) ? (v & kValMask) : 0;
        if (add)
          atomicAdd(reinterpret_cast<unsigned long long*>(&sm.excl[my_s]), (unsigned long long)add);
        // lane s (window slot 0 of stream s) reports whether stream s resolved
        const uint32_t found = __ballot_sync(0xffffffffu, mine_open && mine != 0 && my_w == 0);
        done |= found & all_streams;
        if ((done & all_streams) == all_streams) break;
        pred -= W;
      }
      __syncwarp();
      if (lane < S)
        st_relaxed(status + size_t(tile) * S + lane, kFlagP | (sm.excl[lane] + sm.total[lane]));
    }
    __syncwarp();
    if (tile == P.n_tiles - 1 && lane < S) P.counts[lane] = sm.excl[lane] + sm.total[lane];
  }
  __syncthreads();

  // ---- write: rank = tile base + chunk offset + lanes before + within thread ---------
  const uint32_t lt = lanemask_lt();
#pragma unroll 1
  for (int s = 0; s < S; ++s) {
    const StreamP& st = P.streams[s];
    const uint32_t nibs = s_nib[s * kThreads + tid];
    const uint64_t base = sm.excl[s];
    const uint64_t cap = st.capacity;
    const int n_out = st.n_out;
    const uint32_t pf = st.prefetch_mask;
#pragma unroll 2
    for (int r = 0; r < kRounds; ++r) {
      const uint32_t nib = (nibs >> (r * kVec)) & 0xFu;
      const uint32_t b0 = __ballot_sync(0xffffffffu, nib & 1u);
      const uint32_t b1 = __ballot_sync(0xffffffffu, nib & 2u);
      const uint32_t b2 = __ballot_sync(0xffffffffu, nib & 4u);
      const uint32_t b3 = __ballot_sync(0xffffffffu, nib & 8u);
      if (!nib) continue;
      const int el = (r * kThreads + tid) * kVec;
      uint64_t pos = base + s_cnt[s * kChunks + r * kWarps + warp] + __popc(b0 & lt) +
                     __popc(b1 & lt) + __popc(b2 & lt) + __popc(b3 & lt);
      // gather: one 128-bit load per needed column for this hit vector
      uint4 g[3];
#pragma unroll
      for (int k = 0; k < 3; ++k)
        g[k] = (pf & (1u << k)) ? *reinterpret_cast<const uint4*>(P.col[k] + t0 + el)
                                : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int c = 0; c < kVec; ++c) {
        if (!(nib & (1u << c))) continue;
        if (pos < cap) {
          for (int k = 0; k < n_out; ++k) {
            const Field& f = st.out[k];
            switch (f.kind) {
              case kFieldCol:
                static_cast<uint32_t*>(f.ptr)[pos] = comp(g[f.slot], c);
                break;
              case kFieldConst:
                static_cast<uint32_t*>(f.ptr)[pos] = f.constant;
                break;
              case kFieldIndex:
                static_cast<int64_t*>(f.ptr)[pos] = int64_t(P.base + t0 + el + c);
                break;
              case kFieldMarks:
                static_cast<uint32_t*>(f.ptr)[pos] = kSingle ? 1u : s_marks[el + c];
                break;
              default: {  // answer code vs keys[answer_key]
                const int q = st.answer_key;
                const uint32_t a = (comp(g[0], c) == P.key[q][0] ? 4u : 0u) |
                                   (comp(g[1], c) == P.key[q][1] ? 2u : 0u) |
                                   (comp(g[2], c) == P.key[q][2] ? 1u : 0u);
                static_cast<uint8_t*>(f.ptr)[pos] = uint8_t(a);
              }
            }
          }
        }
        ++pos;
      }
    }
  }
}

using KernelFn = void (*)(Params);

template <int NB>
KernelFn pick_kernel(bool single, bool general, bool count_only) {
  if (count_only) {
    if (single) return general ? scan_kernel<NB, true, true, true> : scan_kernel<NB, true, false, true>;
    return general ? scan_kernel<NB, false, true, true> : scan_kernel<NB, false, false, true>;
  }
  if (single) return general ? scan_kernel<NB, true, true, false> : scan_kernel<NB, true, false, false>;
  return general ? scan_kernel<NB, false, true, false> : scan_kernel<NB, false, false, false>;
}

KernelFn select_kernel(int nb, bool single, bool general, bool count_only) {
  switch (nb) {
    case 0: return pick_kernel<0>(single, general, count_only);
    case 1: return pick_kernel<1>(single, general, count_only);
    case 2: return pick_kernel<2>(single, general, count_only);
    default: return pick_kernel<3>(single, general, count_only);
  }
}

size_t smem_bytes(int S, bool single) {
  return sizeof(Smem) + size_t(S) * kChunks * 4 + size_t(S) * kThreads * 4 +
         (single ? 0 : size_t(kTile) * 4);
}

// Algorithmic bytes of one scan launch: every bound
// column read once (4 B/triple); per emitted row and output field, the write
// plus, for a gathered free column, its 4-byte read.  FILTER bitmap lookups
// and the L2-resident look-back state are not counted.
uint64_t algorithmic_bytes(const Params& P, int nb, const uint64_t* counts) {
  uint64_t b = 4ull * P.n * uint64_t(nb);
  for (int s = 0; s < P.n_streams; ++s) {
    const StreamP& st = P.streams[s];
    uint64_t per_row = 0;
    for (int k = 0; k < st.n_out; ++k) {
      switch (st.out[k].kind) {
        case kFieldCol: per_row += 8; break;
        case kFieldConst: per_row += 4; break;
        case kFieldIndex: per_row += 8; break;
        case kFieldMarks: per_row += 4; break;
        default: per_row += 1 + 4ull * (3 - nb); break;
      }
    }
    b += per_row * counts[s];
  }
  return b;
}

}  // namespace scan

// Host side of one scan: validate the spec, resolve bound columns and output
// fields, size the outputs (hint or sampled estimate), run the single-pass
// kernel, retry exactly on capacity overflow, hand back one table per stream.
void run_scan(tidq_store* st, const tidq_scan_spec& spec, tidq_table** out) {
  using namespace scan;
  Ctx* c = st->ctx;
  TIDQ_REQUIRE(spec.n_keys >= 1 && spec.n_keys <= TIDQ_MAX_KEYS, TIDQ_E_TOO_MANY_KEYS,
               std::to_string(spec.n_keys) + " keys; supported range is 1.." +
                   std::to_string(TIDQ_MAX_KEYS));
  TIDQ_REQUIRE(spec.n_streams >= 1 && spec.n_streams <= TIDQ_MAX_STREAMS, TIDQ_E_INVALID,
               "n_streams must be in 1..32");
  const int S = spec.n_streams;
  const int K = spec.n_keys;
  auto P = std::make_unique<Params>();
  std::memset(P.get(), 0, sizeof(Params));
  P->col[0] = st->s.as<uint32_t>();
  P->col[1] = st->p.as<uint32_t>();
  P->col[2] = st->o.as<uint32_t>();
  P->n = st->n;
  P->base = st->base;
  P->n_keys = K;
  P->n_streams = S;
  uint32_t load = 0;
  for (int q = 0; q < K; ++q)
    for (int k = 0; k < 3; ++k)
      if (spec.keys[q][k]) load |= 1u << k;
  int nb = 0;
  for (int k = 0; k < 3; ++k)
    if (load & (1u << k)) {
      P->bcol[nb] = P->col[k];
      P->bslot[nb] = k;
      ++nb;
    }
  for (int q = 0; q < K; ++q) {
    for (int k = 0; k < 3; ++k) P->key[q][k] = spec.keys[q][k];
    for (int b = 0; b < nb; ++b) {
      const uint32_t v = spec.keys[q][P->bslot[b]];
      if (v) P->kb_mask[q] |= 1u << b;
      P->kv[q][b] = v;
    }
  }
  const bool single = K == 1;
  bool general = false;
  const uint32_t all_keys = K == 32 ? 0xffffffffu : ((1u << K) - 1);
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
    const bool one_key = __builtin_popcount(ss.select) == 1;
    const int q1 = one_key ? __builtin_ctz(ss.select) : -1;
    sp.n_out = ss.n_out;
    for (int k = 0; k < ss.n_out; ++k) {
      const int kind = ss.out[k];
      Field& f = sp.out[k];
      if (kind >= TIDQ_OUT_S && kind <= TIDQ_OUT_O) {
        if (one_key && spec.keys[q1][kind]) {  // bound by the stream's key: a constant
          f.kind = kFieldConst;
          f.constant = spec.keys[q1][kind];
        } else {
          f.kind = kFieldCol;
          f.slot = kind;
          sp.prefetch_mask |= 1u << kind;
        }
      } else if (kind == TIDQ_OUT_INDEX) {
        f.kind = kFieldIndex;
      } else if (kind == TIDQ_OUT_MARKS) {
        f.kind = kFieldMarks;
      } else if (kind == TIDQ_OUT_ANSWER) {
        TIDQ_REQUIRE(ss.answer_key >= 0 && ss.answer_key < K, TIDQ_E_INVALID, "bad answer_key");
        f.kind = kFieldAnswer;
        sp.prefetch_mask |= 7u;
      } else {
        throw Error(TIDQ_E_INVALID, "bad output kind");
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
    }
    if (sp.eq_flags || sp.n_filters) general = true;
  }

  const uint64_t n_tiles = std::max<uint64_t>((st->n + kTile - 1) / kTile, 1);
  TIDQ_REQUIRE(n_tiles < (1ull << 31), TIDQ_E_INVALID, "store too large for one scan");
  P->n_tiles = uint32_t(n_tiles);
  const size_t smem = smem_bytes(S, single);
  KernelFn kmain = select_kernel(nb, single, general, false);
  KernelFn kcount = select_kernel(nb, single, general, true);

  // scratch: counts[S] | tile counter | status[n_tiles*S]
  const size_t counts_b = 512;  // counts[<=32] at 0, tile counter at 256, status at 512
  const size_t status_b = round_up(n_tiles * S * 8, 256);
  const size_t scratch = counts_b + status_b;
  if (c->lookback.bytes < scratch) c->lookback = DevBuf(c, scratch);
  char* sbase = c->lookback.as<char>();
  P->counts = reinterpret_cast<uint64_t*>(sbase);
  P->tile_counter = reinterpret_cast<uint32_t*>(sbase + 256);
  P->status = reinterpret_cast<uint64_t*>(sbase + counts_b);
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
    kcount<<<sampled, kThreads, smem, c->stream>>>(*P);
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
      P->streams[s].out[k].ptr = col.buf.ptr;
      t->cols.push_back(std::move(col));
    }
    P->streams[s].capacity = capacity;
    tables[s] = std::move(t);
  };
  for (int s = 0; s < S; ++s) allocate(s, cap[s]);

  // ---- the persistent warp-specialised kernel takes the hot shapes ----------
  bool use_p = nb >= 1 && S <= pscan::kMaxS && !general;
  for (int s = 0; s < S && use_p; ++s)
    for (int k = 0; k < P->streams[s].n_out; ++k)
      if (P->streams[s].out[k].kind > kFieldIndex) use_p = false;
  if (const char* env = std::getenv("TIDQ_SCAN_KERNEL")) use_p = use_p && std::string(env) != "v2";
  const int s_eff = S <= 1 ? 1 : (S <= 2 ? 2 : 4);
  const uint32_t pn_tiles = uint32_t(std::max<uint64_t>((st->n + pscan::kTile - 1) / pscan::kTile, 1));
  const int stages = nb == 1 ? 6 : 3 - (nb == 3 ? 1 : 0);
  auto pp = std::make_unique<pscan::Params>();
  auto launch_p = [&]() {
    std::memset(pp.get(), 0, sizeof(pscan::Params));
    for (int k = 0; k < 3; ++k) pp->col[k] = P->col[k];
    for (int b = 0; b < nb; ++b) pp->bcol[b] = P->bcol[b];
    pp->n = P->n;
    pp->base = P->base;
    pp->n_tiles = pn_tiles;
    pp->n_keys = K;
    pp->n_streams = s_eff;
    pp->stages = stages;
    for (int q = 0; q < K; ++q) {
      pp->kb_mask[q] = P->kb_mask[q];
      for (int b = 0; b < 3; ++b) pp->kv[q][b] = P->kv[q][b];
    }
    for (int s = 0; s < S; ++s) {
      const StreamP& a = P->streams[s];
      pscan::StreamP& b = pp->streams[s];
      b.select = a.select;
      b.n_out = a.n_out;
      b.capacity = a.capacity;
      b.gather_mask = a.prefetch_mask;
      for (int k = 0; k < a.n_out; ++k) {
        b.out[k].kind = a.out[k].kind;  // kFieldCol/Const/Index share values
        b.out[k].slot = a.out[k].slot;
        b.out[k].constant = a.out[k].constant;
        b.out[k].ptr = a.out[k].ptr;
      }
    }
    pp->tile_counter = P->tile_counter;
    pp->status = P->status;
    pp->counts = P->counts;
    const size_t psmem = pscan::smem_bytes(nb, stages);
    auto fn = nb == 1 ? (K == 1 ? pscan::pscan_kernel<1, true> : pscan::pscan_kernel<1, false>)
            : nb == 2 ? (K == 1 ? pscan::pscan_kernel<2, true> : pscan::pscan_kernel<2, false>)
                      : (K == 1 ? pscan::pscan_kernel<3, true> : pscan::pscan_kernel<3, false>);
    TIDQ_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, int(psmem)));
    const unsigned grid = unsigned(std::min<uint64_t>(pn_tiles, uint64_t(c->sm_count)));
    fn<<<grid, pscan::kThreads, psmem, c->stream>>>(*pp);
  };

  for (int attempt = 0; attempt < 2; ++attempt) {
    TIDQ_CUDA(cudaMemsetAsync(sbase, 0, counts_b + n_tiles * S * 8, c->stream));
    cudaEvent_t ev = c->prof_begin(c->stream);
    if (use_p)
      launch_p();
    else
      kmain<<<uint32_t(n_tiles), kThreads, smem, c->stream>>>(*P);
    c->count_launch();
    TIDQ_CUDA(cudaGetLastError());
    c->prof_end("scan", ev, c->stream, 0);
    TIDQ_CUDA(cudaMemcpyAsync(host_counts, P->counts, size_t(S) * 8, cudaMemcpyDeviceToHost,
                              c->stream));
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    if (ev) c->prof["scan"].bytes += algorithmic_bytes(*P, nb, host_counts);
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
