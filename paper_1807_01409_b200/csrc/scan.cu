// The TripleID pattern scan (reference kernel.py:148-227 search_chunk /
// search_multi, query_ops.py:263-295 scan_patterns with the pattern_table
// repeated-variable mask query_ops.py:210-229 and the FILTER of
// query_ops.py:241-252 fused as an epilogue predicate).
//
// HBM-bound integer streaming; no tensor cores.  Two embarrassingly parallel
// passes, no inter-CTA waiting anywhere:
//
//   mark  one CTA per 4096-triple tile streams ONLY the columns the keys bind
//         (128-bit L1::no_allocate loads, 32 triples / 128 B in flight per
//         thread and column), tests every key in registers, applies the
//         stream epilogue predicates, and writes per stream a hit bitmap
//         (1 bit per triple, one 32-bit word per thread: N/8 bytes), the
//         tile's hit count, and adds it to its 64-tile super-tile sum;
//   (host) reads the few super-tile sums -> exact output sizes and the
//         super-tile offsets (no device-wide scan pass);
//   emit  one warp per work item (a tile with hits, or a quarter of a dense
//         tile), persistent grid over the item list mark appended: item
//         offset = super-tile offset + counts of the preceding tiles of its
//         super-tile (one warp reduction) + hits of the tile's earlier rounds;
//         the warp builds the ascending hit list from the bitmap, gathers the
//         free columns with L2-only sector loads and writes each stream's rows.
//
// Extra traffic over a single pass is the bitmap write+read (N/8 bytes per
// stream, 3% of a 4-byte column); every stream comes out in ascending triple
// order, bit-identical to the reference's np.nonzero compaction.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <memory>

#include "internal.cuh"
#include "prims.cuh"

namespace tidq {
namespace scan {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kRounds = 8;
constexpr int kVec = 4;
constexpr int kTile = kThreads * kRounds * kVec;  // 4096 triples
constexpr int kChunks = kRounds * kWarps;         // 32 warp chunks of 128 triples
constexpr int kSuper = 64;                        // tiles per super-tile
constexpr int kSparseMax = 1024;                  // hits per tile one emit warp handles
constexpr int kEmitWarps = 8;                     // warps (tiles) per sparse-emit CTA
static_assert(int(kScanTile) % kTile == 0, "store padding must cover whole tiles");
static_assert(kChunks == 32, "chunk scan assumes one warp");

// resolved output field kinds
enum : int32_t { kFieldCol = 0, kFieldConst = 1, kFieldLocal = 2, kFieldIndex = 3, kFieldMarks = 4,
                 kFieldAnswer = 5 };  // kinds <= kFieldLocal are 32-bit "simple" fields

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
  uint32_t gather_mask;  // columns the emit pass stages for hit vectors
  uint32_t use_so;       // s and o both gathered: one 8-byte load from P.so
  uint32_t epi_mask;     // columns the mark epilogue predicates read
  uint32_t post;         // predicates evaluated by emit (keep flags), not by mark
  uint8_t* keep;         // post: per output row, 1 = predicates hold
  uint32_t* key_bm;      // optional: emit sets bit v of every row's value in key_bm_slot
  uint64_t key_bm_bits;
  int32_t key_bm_slot;
};

struct Params {
  const uint32_t* col[3];
  const uint32_t* bcol[3];  // bound columns in load order
  int32_t bslot[3];         // slot of bound column b
  uint64_t n;
  uint64_t base;
  uint32_t n_tiles;
  uint32_t n_super;
  int32_t n_keys;
  int32_t n_streams;
  uint32_t key[TIDQ_MAX_KEYS][3];
  uint32_t kb_mask[TIDQ_MAX_KEYS];  // bit b: key q compares bound column b
  uint32_t kv[TIDQ_MAX_KEYS][3];    // key q's value for bound column b
  StreamP streams[TIDQ_MAX_STREAMS];
  uint32_t* bitmap;            // [S][n_tiles][kThreads] hit bits
  uint32_t* counts;            // [S][n_tiles] hits per tile
  uint32_t* super_sum;         // [S][n_super] hits per super-tile (zero before mark)
  const uint64_t* super_off;   // [S][n_super] exclusive offsets (from the host)
  uint64_t* host_total[TIDQ_MAX_STREAMS];  // pinned slots the offsets kernel writes (async)
  uint32_t lookup_min, lookup_range;  // mark_lookup_kernel: stream key values - lookup_min
  uint32_t emit_group;         // tiles per emit-warp group (<= 32)
  uint32_t emit_split;         // 1: one warp per (group, stream); 0: a warp emits all streams
  uint32_t concat;             // TIDQ_SCAN_CONCAT: every stream writes one shared table
  uint32_t* write_counts;      // optional [n] counters: +1 per triple slot mark writes
  const uint16_t* p16;         // predicate codes (bound column 0 = p, kv[.][0] are codes) or null
  const uint2* so;             // interleaved (s, o) pairs or null
};

// write_counts instrumentation (reference kernel.py:153,172-173,221-222):
// each mark thread adds 1 to the counter of every triple slot whose mark
// bits it wrote, so a test can assert the slots are covered exactly once.
__device__ __forceinline__ void count_writes(const Params& P, uint64_t t0, int tid, uint32_t valid) {
  if (!P.write_counts) return;
#pragma unroll 1
  for (int r = 0; r < kRounds; ++r)
#pragma unroll
    for (int c = 0; c < kVec; ++c)
      if ((valid >> (r * kVec + c)) & 1u) atomicAdd(P.write_counts + t0 + (uint64_t(r) * kThreads + tid) * kVec + c, 1u);
}

// Programmatic dependent launch: a dependent grid is scheduled while its
// predecessor drains and waits here until the predecessor has completed.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint4 ld_stream(const uint32_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// 4 predicate codes (16-bit) of one round, widened to the uint4 the
// compare loops read
__device__ __forceinline__ uint4 ld_stream16(const uint16_t* p) {
  uint32_t a, b;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "l"(p));
  return make_uint4(a & 0xFFFFu, a >> 16, b & 0xFFFFu, b >> 16);
}

// the kRounds loads of bound column b for thread tid of the tile at t0: the
// 16-bit predicate codes when the pass binds only the predicate (P.p16),
// else the uint32 column
__device__ __forceinline__ void load_bound(const Params& P, int b, uint64_t t0, int tid, uint4 (&x)[kRounds]) {
  if (b == 0 && P.p16) {
    const uint16_t* src = P.p16 + t0 + size_t(tid) * kVec;
#pragma unroll
    for (int r = 0; r < kRounds; ++r) x[r] = ld_stream16(src + size_t(r) * kThreads * kVec);
  } else {
    const uint32_t* src = P.bcol[b] + t0 + size_t(tid) * kVec;
#pragma unroll
    for (int r = 0; r < kRounds; ++r) x[r] = ld_stream(src + size_t(r) * kThreads * kVec);
  }
}

__device__ __forceinline__ uint32_t comp(const uint4& v, int c) {
  return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}

__device__ __forceinline__ bool bitmap_test(const uint32_t* words, uint64_t nbits, uint32_t id) {
  return uint64_t(id) < nbits && ((__ldg(words + (id >> 5)) >> (id & 31)) & 1u);
}

// Stream epilogue predicates of one accepted triple: the repeated-variable
// equalities of pattern_table (query_ops.py:220-225) and the FILTER bitmap
// tests (query_ops.py:241-252).
__device__ __forceinline__ bool epilogue_ok(const StreamP& st, uint32_t vs, uint32_t vp, uint32_t vo) {
  bool ok = (!(st.eq_flags & TIDQ_EQ_SP) || vs == vp) && (!(st.eq_flags & TIDQ_EQ_SO) || vs == vo) &&
            (!(st.eq_flags & TIDQ_EQ_PO) || vp == vo);
  for (int f = 0; ok && f < st.n_filters; ++f) {
    const int sl = st.filter_slot[f];
    ok = bitmap_test(st.filter_words[f], st.filter_nbits[f], sl == 0 ? vs : (sl == 1 ? vp : vo));
  }
  return ok;
}

// ------------------------------------------------------------------------ mark
// dynamic smem: marks[kTile] u32 (multi-key only)
template <int NB, bool kSingle, bool kGeneral>
__global__ void __launch_bounds__(kThreads) mark_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(16) uint32_t s_marks[];
  __shared__ uint32_t s_count[TIDQ_MAX_STREAMS];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int S = P.n_streams;
  const uint32_t tile = blockIdx.x;
  const uint64_t t0 = uint64_t(tile) * kTile;
  const bool partial = t0 + kTile > P.n;
  if (tid < TIDQ_MAX_STREAMS) s_count[tid] = 0;

  uint4 x[NB > 0 ? NB : 1][kRounds];
#pragma unroll
  for (int b = 0; b < NB; ++b) load_bound(P, b, t0, tid, x[b]);
  // PDL: the store columns are read-only, so the loads above may overlap the
  // previous scan's emit; scratch (bitmaps, counts, sums) is written below,
  // after that scan has completed
  pdl_wait();

  uint32_t valid = 0xffffffffu;
  if (partial) {
    valid = 0;
#pragma unroll
    for (int r = 0; r < kRounds; ++r)
#pragma unroll
      for (int c = 0; c < kVec; ++c)
        valid |= uint32_t(t0 + (uint64_t(r) * kThreads + tid) * kVec + c < P.n) << (r * kVec + c);
  }

  uint32_t hb = 0;  // kSingle: bit r*4+c = key 0 accepts triple (r, c)
  if (kSingle) {
    const uint32_t kb0 = 0xffffffffu;  // every loaded column is bound by the key
#pragma unroll
    for (int r = 0; r < kRounds; ++r)
#pragma unroll
      for (int c = 0; c < kVec; ++c) {
        bool ok = true;
#pragma unroll
        for (int b = 0; b < NB; ++b) ok = ok && (!((kb0 >> b) & 1u) || comp(x[b][r], c) == P.kv[0][b]);
        hb |= uint32_t(ok) << (r * kVec + c);
      }
    hb &= valid;
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
      const uint32_t vb = valid >> (r * kVec);
      *reinterpret_cast<uint4*>(s_marks + (r * kThreads + tid) * kVec) =
          make_uint4(vb & 1u ? m[0] : 0u, vb & 2u ? m[1] : 0u, vb & 4u ? m[2] : 0u,
                     vb & 8u ? m[3] : 0u);
    }
  }
  __syncthreads();  // s_count zeroed (each thread reads back only its own marks)

  const size_t words = size_t(P.n_tiles) * kThreads;
#pragma unroll 1
  for (int s = 0; s < S; ++s) {
    const StreamP& st = P.streams[s];
    uint32_t bits = 0;
    if (kSingle) {
      bits = hb;
    } else {
      const uint32_t sel = st.select;
#pragma unroll 1
      for (int r = 0; r < kRounds; ++r) {
        const uint4 mv = *reinterpret_cast<const uint4*>(s_marks + (r * kThreads + tid) * kVec);
        bits |= (((mv.x & sel) ? 1u : 0u) | ((mv.y & sel) ? 2u : 0u) | ((mv.z & sel) ? 4u : 0u) |
                 ((mv.w & sel) ? 8u : 0u))
                << (r * kVec);
      }
    }
    if (kGeneral && bits && !st.post && (st.eq_flags || st.n_filters)) {
      {  // gather just the predicate columns of each hit (streaming them with
         // the keys measured slower: 1.74 vs 0.91 ms on C4 star x2 FILTER)
        uint32_t rest = bits;
        const uint32_t em = st.epi_mask;
        while (rest) {
          const int i = __ffs(rest) - 1;
          rest &= rest - 1;
          const uint64_t e = t0 + (uint64_t(i >> 2) * kThreads + tid) * kVec + (i & 3);
          const uint32_t v0 = (em & 1u) ? ld_gather(P.col[0] + e) : 0u;
          const uint32_t v1 = (em & 2u) ? ld_gather(P.col[1] + e) : 0u;
          const uint32_t v2 = (em & 4u) ? ld_gather(P.col[2] + e) : 0u;
          if (!epilogue_ok(st, v0, v1, v2)) bits &= ~(1u << i);
        }
      }
    }
    P.bitmap[s * words + size_t(tile) * kThreads + tid] = bits;
    const uint32_t c = __reduce_add_sync(0xffffffffu, __popc(bits));
    if (lane == 0 && c) atomicAdd(&s_count[s], c);
  }
  __syncthreads();
  if (tid < S) {
    const uint32_t c = s_count[tid];
    P.counts[size_t(tid) * P.n_tiles + tile] = c;
    if (c) atomicAdd(P.super_sum + size_t(tid) * P.n_super + tile / kSuper, c);
  }
  count_writes(P, t0, tid, valid);
  pdl_launch_dependents();
}

// mark, one key on the predicate-code column, no epilogue (the ?s P ?o
// scan): the 16-bit codes stay packed (two per register) and are compared in
// place; TPC consecutive tiles per CTA with all their loads issued at once
// (TPC = 2 / 4, i.e. the uint32 scan's bytes in flight per thread, measured
// no faster than 1: the code column streams at ~5.2 TB/s either way).
template <int TPC>
__global__ void __launch_bounds__(kThreads) mark_p16_kernel(const __grid_constant__ Params P) {
  __shared__ uint32_t s_count[TPC][TIDQ_MAX_STREAMS];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int S = P.n_streams;
  uint2 raw[TPC][kRounds];
#pragma unroll
  for (int h = 0; h < TPC; ++h) {
    const uint32_t tile = blockIdx.x * TPC + h;
    const uint16_t* src = P.p16 + uint64_t(tile) * kTile + size_t(tid) * kVec;
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      if (tile < P.n_tiles)
        asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                     : "=r"(raw[h][r].x), "=r"(raw[h][r].y)
                     : "l"(src + size_t(r) * kThreads * kVec));
      else
        raw[h][r] = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
    }
  }
  if (tid < TIDQ_MAX_STREAMS)
#pragma unroll
    for (int h = 0; h < TPC; ++h) s_count[h][tid] = 0;
  pdl_wait();  // scratch is written only after the previous scan
  const uint32_t kv = P.kv[0][0];
  const size_t words = size_t(P.n_tiles) * kThreads;
  __syncthreads();  // s_count zeroed
#pragma unroll
  for (int h = 0; h < TPC; ++h) {
    const uint32_t tile = blockIdx.x * TPC + h;
    if (tile >= P.n_tiles) break;  // CTA-uniform
    const uint64_t t0 = uint64_t(tile) * kTile;
    uint32_t hb = 0;
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      const uint2 v = raw[h][r];
      hb |= (uint32_t((v.x & 0xFFFFu) == kv) | (uint32_t((v.x >> 16) == kv) << 1) |
             (uint32_t((v.y & 0xFFFFu) == kv) << 2) | (uint32_t((v.y >> 16) == kv) << 3))
            << (r * kVec);
    }
    uint32_t valid = 0xffffffffu;
    if (t0 + kTile > P.n) {
      valid = 0;
#pragma unroll
      for (int r = 0; r < kRounds; ++r)
#pragma unroll
        for (int c = 0; c < kVec; ++c)
          valid |= uint32_t(t0 + (uint64_t(r) * kThreads + tid) * kVec + c < P.n) << (r * kVec + c);
    }
    hb &= valid;
    const uint32_t cw = __reduce_add_sync(0xffffffffu, __popc(hb));
    for (int s = 0; s < S; ++s) {
      P.bitmap[s * words + size_t(tile) * kThreads + tid] = hb;
      if (lane == 0 && cw) atomicAdd(&s_count[h][s], cw);
    }
    count_writes(P, t0, tid, valid);
  }
  __syncthreads();
#pragma unroll
  for (int h = 0; h < TPC; ++h) {
    const uint32_t tile = blockIdx.x * TPC + h;
    if (tid < S && tile < P.n_tiles) {
      const uint32_t c = s_count[h][tid];
      P.counts[size_t(tid) * P.n_tiles + tile] = c;
      if (c) atomicAdd(P.super_sum + size_t(tid) * P.n_super + tile / kSuper, c);
    }
  }
  pdl_launch_dependents();
}

// ------------------------------------------------------------------------ emit
// One warp per (stream, group of emit_group consecutive tiles), grid-stride.
// Lane t < emit_group reads tile t's hit count, a ballot names the tiles with
// hits, and the warp emits them one after another: a tile with at most
// kSparseMax hits is one work unit (rounds 0..8); a denser tile is four units
// of two rounds each (elements [1024 q, 1024 (q + 1))), so a unit never holds
// more than kSparseMax hits.  Sparse groups of up to kBatchMaxGroup tiles are
// one batched unit.  Per unit and stream the warp reads the tile's 128 bitmap
// words (4 per lane), computes the unit's output offset (super-tile offset +
// counts of the preceding tiles of its super-tile + hits of the tile's
// earlier rounds), builds the unit-local ascending hit list in shared memory
// (a whole tile: three packed warp scans, list_hits_all; otherwise one scan
// per round, list_hits), then gathers the free columns of 4 hits per lane at
// a time (L2-only sector loads, all in flight together) and writes rows
// base+k, coalesced across lanes.

// The 16-bit round masks of a lane's 4 bitmap words: m_r = nibble r of x, y,
// z, w (x lowest).  The even/odd nibbles of x|y and z|w are first paired
// into bytes, then each round is one byte permute (8 PRMT + 8 LOP instead of
// ~90 shift/mask instructions per tile).
struct RoundMasks {
  uint32_t e, o, e2, o2;
  __device__ __forceinline__ explicit RoundMasks(const uint4& w4)
      : e((w4.x & 0x0F0F0F0Fu) | ((w4.y << 4) & 0xF0F0F0F0u)),
        o(((w4.x >> 4) & 0x0F0F0F0Fu) | (w4.y & 0xF0F0F0F0u)),
        e2((w4.z & 0x0F0F0F0Fu) | ((w4.w << 4) & 0xF0F0F0F0u)),
        o2(((w4.z >> 4) & 0x0F0F0F0Fu) | (w4.w & 0xF0F0F0F0u)) {}
  __device__ __forceinline__ uint32_t operator()(int r) const {
    const uint32_t k = uint32_t(r >> 1);
    return __byte_perm(r & 1 ? o : e, r & 1 ? o2 : e2, k | ((k + 4) << 4)) & 0xFFFFu;
  }
};

// Append the hits of rounds [r_lo, r_hi) of a tile's bitmap (4 words per
// lane in w4) to the warp's list at `run`, in ascending element order:
// entry = (tag << 12) | element.  Returns the new run.
__device__ __forceinline__ uint32_t list_hits(const uint4& w4, int r_lo, int r_hi, uint32_t tag,
                                              uint16_t* list, uint32_t run, int lane) {
  const RoundMasks rm(w4);
  // (unrolled twice, not fully: the call sites' full copies made the emit
  // 11.5 K instructions and ncu showed 21 % of its warp stalls waiting on
  // instruction fetch; 5.8 K now — C2 sweep -2.5 %, C5 star / chain x3
  // -3.5 / -2.7 %, C3 neutral; fully rolled cost C3 UNION 2 %)
#pragma unroll 2
  for (int r = r_lo; r < r_hi; ++r) {
    uint32_t m = rm(r);
    if (!__any_sync(0xffffffffu, m)) continue;  // an empty round (sparse tiles: most of them)
    const uint32_t cnt = __popc(m);
    uint32_t inc = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += y;
    }
    uint32_t pos = run + inc - cnt;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      list[pos++] = uint16_t((tag << 12) | (((r * kThreads + 4 * lane + (b >> 2)) << 2) | (b & 3)));
    }
    run += __shfl_sync(0xffffffffu, inc, 31);
  }
  return run;
}

// list_hits over all kRounds rounds with three packed warp scans instead of
// one per round: the per-lane round counts (<= 16) sit in 10-bit fields,
// three rounds per word, and the warp-wide prefix of every round comes out
// of the same shuffles.
__device__ __forceinline__ uint32_t list_hits_all(const uint4& w4, uint32_t tag, uint16_t* list, uint32_t run,
                                                  int lane) {
  uint32_t m[kRounds];
  uint32_t pk[3] = {0u, 0u, 0u};
  const RoundMasks rm(w4);
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    m[r] = rm(r);
    pk[r / 3] += uint32_t(__popc(m[r])) << (10 * (r % 3));
  }
  uint32_t inc[3] = {pk[0], pk[1], pk[2]};
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc[j], d);
      if (lane >= d) inc[j] += y;
    }
  }
  uint32_t tot[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) tot[j] = __shfl_sync(0xffffffffu, inc[j], 31);
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const int j = r / 3, sh = 10 * (r % 3);
    uint32_t pos = run + (((inc[j] - pk[j]) >> sh) & 0x3FFu);
    uint32_t mm = m[r];
    while (mm) {
      const int b = __ffs(mm) - 1;
      mm &= mm - 1;
      list[pos++] = uint16_t((tag << 12) | (((r * kThreads + 4 * lane + (b >> 2)) << 2) | (b & 3)));
    }
    run += (tot[j] >> sh) & 0x3FFu;
  }
  return run;
}

// Rows base + k for the c listed hits (entry = (tag << 12) | element; the
// triple is t0 + tag * kTile + element): gathers of the free columns, 4 hits
// per lane in flight, coalesced row writes.
template <bool kSimple>
__device__ __forceinline__ void write_rows(const Params& P, const StreamP& st, const uint16_t* list,
                                           uint32_t c, uint64_t base, uint64_t t0, int lane) {
  const int nf = st.n_out;
  const uint32_t gm = st.gather_mask;
  int kind[TIDQ_MAX_OUT], slot[TIDQ_MAX_OUT];
  uint32_t cst[TIDQ_MAX_OUT];
  void* optr[TIDQ_MAX_OUT];
#pragma unroll
  for (int f = 0; f < TIDQ_MAX_OUT; ++f) {
    kind[f] = f < nf ? st.out[f].kind : kFieldConst;
    slot[f] = f < nf ? st.out[f].slot : 0;
    cst[f] = f < nf ? st.out[f].constant : 0u;
    optr[f] = f < nf ? st.out[f].ptr : nullptr;
  }
  constexpr int kPer = 4;  // hits per lane with loads in flight together
  for (uint32_t k0 = 0; k0 < c; k0 += 32 * kPer) {
    uint32_t e[kPer], v[kPer][3];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const uint32_t k = k0 + i * 32 + lane;
      const uint32_t x = k < c ? list[k] : 0u;
      e[i] = (x >> 12) * kTile + (x & 0xFFFu);
      if (st.use_so) {
        const uint2 so = k < c ? ld_gather(P.so + t0 + e[i]) : make_uint2(0u, 0u);
        v[i][0] = so.x;
        v[i][2] = so.y;
        v[i][1] = (k < c && (gm & 2u)) ? ld_gather(P.col[1] + t0 + e[i]) : 0u;
      } else {
#pragma unroll
        for (int q = 0; q < 3; ++q)
          v[i][q] = (k < c && (gm & (1u << q))) ? ld_gather(P.col[q] + t0 + e[i]) : 0u;
      }
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const uint32_t k = k0 + i * 32 + lane;
      if (k >= c) continue;
      const uint64_t p = base + k;
      if (p >= st.capacity) continue;
      if (st.key_bm) {  // a join's key set, built while the row is in registers
        const uint32_t kv = st.key_bm_slot == 0 ? v[i][0] : (st.key_bm_slot == 1 ? v[i][1] : v[i][2]);
        if (kv < st.key_bm_bits && (!st.post || epilogue_ok(st, v[i][0], v[i][1], v[i][2])))
          atomicOr(st.key_bm + (kv >> 5), 1u << (kv & 31));
      }
#pragma unroll
      for (int f = 0; f < TIDQ_MAX_OUT; ++f) {
        if (f >= nf) break;
        if (kSimple || kind[f] <= kFieldLocal) {
          static_cast<uint32_t*>(optr[f])[p] =
              kind[f] == kFieldConst   ? cst[f]
              : kind[f] == kFieldLocal ? uint32_t(t0 + e[i])
                                       : (slot[f] == 0 ? v[i][0] : (slot[f] == 1 ? v[i][1] : v[i][2]));
          if (f == 0 && st.post) st.keep[p] = uint8_t(epilogue_ok(st, v[i][0], v[i][1], v[i][2]));
        } else if (kind[f] == kFieldIndex) {
          static_cast<int64_t*>(optr[f])[p] = int64_t(P.base + t0 + e[i]);
        } else if (kind[f] == kFieldMarks) {  // re-test every key on the gathered values
          uint32_t m = 0;
          for (int q = 0; q < P.n_keys; ++q) {
            const bool ok = (!P.key[q][0] || v[i][0] == P.key[q][0]) &&
                            (!P.key[q][1] || v[i][1] == P.key[q][1]) &&
                            (!P.key[q][2] || v[i][2] == P.key[q][2]);
            m |= uint32_t(ok) << q;
          }
          static_cast<uint32_t*>(optr[f])[p] = m;
        } else {  // answer code vs keys[answer_key] (kernel.py:67-74)
          const int q = st.answer_key;
          static_cast<uint8_t*>(optr[f])[p] = uint8_t((v[i][0] == P.key[q][0] ? 4u : 0u) |
                                                      (v[i][1] == P.key[q][1] ? 2u : 0u) |
                                                      (v[i][2] == P.key[q][2] ? 1u : 0u));
        }
      }
    }
  }
}

constexpr uint32_t kBatchMaxGroup = 8;  // tiles per batched group (registers: 8 x uint4)

template <bool kSimple>
__global__ void __launch_bounds__(kEmitWarps * 32, 4) emit_kernel(const __grid_constant__ Params P) {
  __shared__ uint16_t s_list[kEmitWarps][kSparseMax];
  pdl_wait();  // offsets (and mark) are complete
  pdl_launch_dependents();  // the next scan's mark may start loading as this grid drains
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const size_t words = size_t(P.n_tiles) * kThreads;
  const uint32_t G = P.emit_group;
  const uint32_t n_groups = (P.n_tiles + G - 1) / G;
  uint16_t* list = s_list[warp];
  // (group, stream) pairs, tile-major: the warps emitting the streams of one
  // tile run together and share its gathered s/p/o lines in L2
  const uint32_t SW = P.emit_split ? uint32_t(P.n_streams) : 1u;  // work items per group
  const uint32_t n_work = n_groups * SW;
  for (uint32_t wk = blockIdx.x * kEmitWarps + warp; wk < n_work; wk += gridDim.x * kEmitWarps) {
  const uint32_t g = wk / SW;
  const int s_lo = P.emit_split ? int(wk - g * SW) : 0;
  const int s_hi = P.emit_split ? s_lo + 1 : P.n_streams;
  uint32_t tcl = 0;
  if (lane < G && g * G + lane < P.n_tiles)
    for (int s = s_lo; s < s_hi; ++s) tcl = max(tcl, P.counts[size_t(s) * P.n_tiles + g * G + lane]);
  const uint32_t has = __ballot_sync(0xffffffffu, tcl != 0);
  const uint32_t dense = __ballot_sync(0xffffffffu, tcl > kSparseMax);
  if (!has) continue;
  // ---- batched group: the group's tiles (one super-tile, one stream) have
  // at most kSparseMax hits together; every bitmap load is issued at once and
  // one list / one gather pass covers the whole group
  if (G > 1 && G <= kBatchMaxGroup && s_hi == s_lo + 1 &&
      __reduce_add_sync(0xffffffffu, lane < G ? tcl : 0u) <= kSparseMax) {
    const int s = s_lo;
    const StreamP& st = P.streams[s];
    const uint32_t tile0 = g * G;
    uint4 w4[kBatchMaxGroup];
#pragma unroll
    for (uint32_t j = 0; j < kBatchMaxGroup; ++j)
      w4[j] = ((has >> j) & 1u)
                  ? *reinterpret_cast<const uint4*>(P.bitmap + s * words + size_t(tile0 + j) * kThreads + 4 * lane)
                  : make_uint4(0, 0, 0, 0);
    // group offset: super-tile offset + counts of the preceding tiles in it
    const uint32_t sb = tile0 / kSuper;
    const uint32_t first = sb * kSuper;
    uint32_t a = 0;
    if (first + lane < tile0) a += P.counts[size_t(s) * P.n_tiles + first + lane];
    if (first + 32 + lane < tile0) a += P.counts[size_t(s) * P.n_tiles + first + 32 + lane];
    const uint64_t base = P.super_off[size_t(s) * P.n_super + sb] + __reduce_add_sync(0xffffffffu, a);
    uint32_t run = 0;
#pragma unroll
    for (uint32_t j = 0; j < kBatchMaxGroup; ++j)
      if ((has >> j) & 1u) run = list_hits(w4[j], 0, kRounds, j, list, run, lane);
    __syncwarp();
    write_rows<kSimple>(P, st, list, run, base, uint64_t(tile0) * kTile, lane);
    __syncwarp();  // the list is reused by the next work item
    continue;
  }
  for (uint32_t rest = has; rest; rest &= rest - 1) {
  const int t = __ffs(rest) - 1;
  const uint32_t tile = g * G + t;
  const int n_units = (dense >> t) & 1u ? 4 : 1;
  for (int u = 0; u < n_units; ++u) {
    const int r_lo = n_units == 1 ? 0 : 2 * u;
    const int r_hi = n_units == 1 ? kRounds : r_lo + 2;
    const uint64_t t0 = uint64_t(tile) * kTile;
    for (int s = s_lo; s < s_hi; ++s) {
      if (P.counts[size_t(s) * P.n_tiles + tile] == 0) continue;  // warp-uniform
      const StreamP& st = P.streams[s];
      const uint4 w4 = *reinterpret_cast<const uint4*>(P.bitmap + s * words + size_t(tile) * kThreads + 4 * lane);
      // tile offset: super-tile offset + counts of the preceding tiles in it
      const uint32_t sb = tile / kSuper;
      const uint32_t first = sb * kSuper;
      uint32_t a = 0;
      if (first + lane < tile) a += P.counts[size_t(s) * P.n_tiles + first + lane];
      if (first + 32 + lane < tile) a += P.counts[size_t(s) * P.n_tiles + first + 32 + lane];
      // hits of this tile in rounds before r_lo (quarter items)
      const uint32_t pre_mask = (1u << (r_lo * kVec)) - 1u;
      a += __popc(w4.x & pre_mask) + __popc(w4.y & pre_mask) + __popc(w4.z & pre_mask) +
           __popc(w4.w & pre_mask);
      const uint64_t base = P.super_off[size_t(s) * P.n_super + sb] + __reduce_add_sync(0xffffffffu, a);
      const uint32_t c = n_units == 1 ? list_hits_all(w4, 0, list, 0, lane)
                                      : list_hits(w4, r_lo, r_hi, 0, list, 0, lane);
      __syncwarp();
      write_rows<kSimple>(P, st, list, c, base, t0, lane);
      __syncwarp();  // the list is reused by the next stream / unit
    }
  }
  }
  }
}

// ---- post-filter compaction ----------------------------------------------------
// Dense predicate streams are marked without their predicates (the fast mark
// kernels) and the emit, which gathers the predicate columns with the row
// anyway, writes a keep flag per row; this compacts the rows in order.
// Rows beyond the stream's device-side total are ignored, so the launch is
// sized from the capacity and nothing waits for the host.
constexpr int kPfT = 256, kPfI = 4, kPfBlk = kPfT * kPfI;

__global__ void __launch_bounds__(kPfT) postfilter_count_kernel(const uint8_t* __restrict__ keep,
                                                                const uint64_t* __restrict__ total,
                                                                uint32_t* __restrict__ bcount,
                                                                unsigned long long* __restrict__ kept) {
  const uint64_t n = *total;
  const uint64_t base = uint64_t(blockIdx.x) * kPfBlk;
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < kPfI; ++j) {
    const uint64_t r = base + j * kPfT + threadIdx.x;
    c += r < n ? keep[r] : 0u;
  }
  __shared__ uint32_t w[kPfT / 32];
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x < 32) {
    c = threadIdx.x < kPfT / 32 ? w[threadIdx.x] : 0u;
    c = __reduce_add_sync(0xffffffffu, c);
    if (threadIdx.x == 0) {
      bcount[blockIdx.x] = c;
      if (c) atomicAdd(kept, (unsigned long long)c);
    }
  }
}

struct PostCols {
  int n;
  const uint32_t* in[TIDQ_MAX_OUT];
  uint32_t* out[TIDQ_MAX_OUT];
};

__global__ void __launch_bounds__(kPfT) postfilter_write_kernel(const uint8_t* __restrict__ keep,
                                                                const uint64_t* __restrict__ total,
                                                                const uint64_t* __restrict__ boffs,
                                                                const __grid_constant__ PostCols pc) {
  __shared__ uint32_t wbase[kPfBlk / 32];
  const uint64_t n = *total;
  const uint64_t base = uint64_t(blockIdx.x) * kPfBlk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  // rows base + j*kPfT + tid: warp (j, warp) owns 32 consecutive rows
  uint32_t ball[kPfI];
#pragma unroll
  for (int j = 0; j < kPfI; ++j) {
    const uint64_t r = base + j * kPfT + threadIdx.x;
    ball[j] = __ballot_sync(0xffffffffu, r < n && keep[r]);
    if (lane == 0) wbase[j * (kPfT / 32) + warp] = __popc(ball[j]);
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the 32 warp-row counts, in row order
    const uint32_t v = wbase[lane];
    uint32_t inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += y;
    }
    wbase[lane] = inc - v;
  }
  __syncthreads();
  const uint64_t b0 = boffs[blockIdx.x];
  uint64_t dst[kPfI];
#pragma unroll
  for (int j = 0; j < kPfI; ++j) dst[j] = b0 + wbase[j * (kPfT / 32) + warp] + __popc(ball[j] & lt);
  // per column: the kept rows' loads in flight together, then the stores
  for (int k = 0; k < pc.n; ++k) {
    uint32_t v[kPfI];
#pragma unroll
    for (int j = 0; j < kPfI; ++j)
      v[j] = (ball[j] >> lane) & 1u ? pc.in[k][base + j * kPfT + threadIdx.x] : 0u;
#pragma unroll
    for (int j = 0; j < kPfI; ++j)
      if ((ball[j] >> lane) & 1u) pc.out[k][dst[j]] = v[j];
  }
}

// Device-side super-tile offsets (hint mode: no host round trip between the
// passes): block s scans stream s's super-tile sums; totals[s] = its rows.
__global__ void __launch_bounds__(1024) super_offsets_kernel(const __grid_constant__ Params P,
                                                             uint64_t* soff, uint64_t* totals) {
  __shared__ uint64_t wt[32];
  pdl_wait();  // mark's counts are complete
  pdl_launch_dependents();
  // TIDQ_SCAN_CONCAT: one block runs the streams in order and carries the
  // offsets across them, so stream s's rows land after stream s-1's in one
  // shared output table
  const int s_lo = P.concat ? 0 : blockIdx.x, s_hi = P.concat ? P.n_streams : blockIdx.x + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t carry = 0;
  for (int s = s_lo; s < s_hi; ++s) {
    uint32_t* in = P.super_sum + size_t(s) * P.n_super;
    const uint64_t start = carry;
    for (uint32_t lo = 0; lo < P.n_super; lo += blockDim.x) {
      const uint32_t j = lo + threadIdx.x;
      const uint64_t x = j < P.n_super ? in[j] : 0;
      if (j < P.n_super) in[j] = 0;  // leave the sums zeroed for the next scan
      uint64_t inc = x;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += y;
      }
      if (lane == 31) wt[warp] = inc;
      __syncthreads();
      if (warp == 0) {
        uint64_t w = wt[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint64_t y = __shfl_up_sync(0xffffffffu, w, d);
          if (lane >= d) w += y;
        }
        wt[lane] = w;
      }
      __syncthreads();
      const uint64_t before = warp ? wt[warp - 1] : 0;
      if (j < P.n_super) soff[size_t(s) * P.n_super + j] = carry + before + inc - x;
      carry += wt[31];
      __syncthreads();
    }
    if (threadIdx.x == 0) totals[s] = carry - start;
  }
  if (threadIdx.x == 0 && P.host_total[s_lo])
    *(volatile uint64_t*)P.host_total[s_lo] = carry;  // mapped pinned memory
}

// mark, UNION fast path: one bound column, every stream selects exactly one
// key (e.g. a UNION of ?P? patterns) and no epilogue predicates — each
// stream's hit bits are built in registers straight from the streamed column.
// Templated on the stream count so only S compares per element are issued.
constexpr int kMulti1Max = 8;

template <int SS>  // SS = 0: runtime stream count, SS-wide loops for SS > 0
__global__ void __launch_bounds__(kThreads) mark_multi1_kernel(const __grid_constant__ Params P) {
  constexpr int SU = SS ? SS : kMulti1Max;
  const int S = SS ? SS : P.n_streams;
  __shared__ uint32_t s_count[kMulti1Max];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const uint32_t tile = blockIdx.x;
  const uint64_t t0 = uint64_t(tile) * kTile;
  if (tid < kMulti1Max) s_count[tid] = 0;
  uint4 x[kRounds];
  load_bound(P, 0, t0, tid, x);
  pdl_wait();  // as in mark_kernel: scratch is written only after the previous scan
  uint32_t valid = 0xffffffffu;
  if (t0 + kTile > P.n) {
    valid = 0;
#pragma unroll
    for (int r = 0; r < kRounds; ++r)
#pragma unroll
      for (int c = 0; c < kVec; ++c)
        valid |= uint32_t(t0 + (uint64_t(r) * kThreads + tid) * kVec + c < P.n) << (r * kVec + c);
  }
  uint32_t kv[SU], bits[SU];
#pragma unroll
  for (int s = 0; s < SU; ++s) {
    kv[s] = s < S ? P.kv[__ffs(P.streams[s].select) - 1][0] : 0u;
    bits[s] = 0;
  }
#pragma unroll
  for (int r = 0; r < kRounds; ++r)
#pragma unroll
    for (int c = 0; c < kVec; ++c) {
      const uint32_t v = comp(x[r], c);
#pragma unroll
      for (int s = 0; s < SU; ++s) bits[s] |= uint32_t(v == kv[s]) << (r * kVec + c);
    }
  __syncthreads();
  const size_t words = size_t(P.n_tiles) * kThreads;
#pragma unroll
  for (int s = 0; s < SU; ++s) {
    if (s >= S) break;
    const uint32_t b = bits[s] & valid;
    P.bitmap[s * words + size_t(tile) * kThreads + tid] = b;
    const uint32_t cnt = __reduce_add_sync(0xffffffffu, __popc(b));
    if (lane == 0 && cnt) atomicAdd(&s_count[s], cnt);
  }
  __syncthreads();
  if (tid < S) {
    const uint32_t cnt = s_count[tid];
    P.counts[size_t(tid) * P.n_tiles + tile] = cnt;
    if (cnt) atomicAdd(P.super_sum + size_t(tid) * P.n_super + tile / kSuper, cnt);
  }
  count_writes(P, t0, tid, valid);
  pdl_launch_dependents();
}


// mark, UNION of SS <= 3 one-column keys on the predicate-code column: the
// codes stay packed two per register and each register is compared with a
// stream's code on the half-precision pipe (setp.eq.f16x2: two predicates
// per instruction, exact for the normal fp16 patterns the codes are), the
// bits inserted by predicated ORs.  The integer compare-per-element kernel
// is ALU-bound here (ncu: 86 % SM throughput at 3 streams).
template <int SS>
__global__ void __launch_bounds__(kThreads) mark_multi1_p16_kernel(const __grid_constant__ Params P) {
  __shared__ uint32_t s_count[SS];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const uint32_t tile = blockIdx.x;
  const uint64_t t0 = uint64_t(tile) * kTile;
  if (tid < SS) s_count[tid] = 0;
  uint32_t xa[kRounds], xb[kRounds];
  const uint16_t* src = P.p16 + t0 + size_t(tid) * kVec;
#pragma unroll
  for (int r = 0; r < kRounds; ++r)
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(xa[r]), "=r"(xb[r])
                 : "l"(src + size_t(r) * kThreads * kVec));
  pdl_wait();  // as in mark_kernel: scratch is written only after the previous scan
  uint32_t valid = 0xffffffffu;
  if (t0 + kTile > P.n) {
    valid = 0;
#pragma unroll
    for (int r = 0; r < kRounds; ++r)
#pragma unroll
      for (int c = 0; c < kVec; ++c)
        valid |= uint32_t(t0 + (uint64_t(r) * kThreads + tid) * kVec + c < P.n) << (r * kVec + c);
  }
  uint32_t kk[SS], bits[SS];
#pragma unroll
  for (int s = 0; s < SS; ++s) {
    const uint32_t kv = P.kv[__ffs(P.streams[s].select) - 1][0];
    kk[s] = kv | (kv << 16);
    bits[s] = 0;
  }
#pragma unroll
  for (int r = 0; r < kRounds; ++r)
#pragma unroll
    for (int s = 0; s < SS; ++s) {
      const uint32_t m0 = 1u << (r * kVec), m1 = 2u << (r * kVec), m2 = 4u << (r * kVec), m3 = 8u << (r * kVec);
      asm("{\n .reg .pred a, b, c, d;\n"
          " setp.eq.f16x2 a|b, %1, %3;\n"
          " setp.eq.f16x2 c|d, %2, %3;\n"
          " @a or.b32 %0, %0, %4;\n @b or.b32 %0, %0, %5;\n"
          " @c or.b32 %0, %0, %6;\n @d or.b32 %0, %0, %7;\n}"
          : "+r"(bits[s])
          : "r"(xa[r]), "r"(xb[r]), "r"(kk[s]), "r"(m0), "r"(m1), "r"(m2), "r"(m3));
    }
  __syncthreads();
  const size_t words = size_t(P.n_tiles) * kThreads;
#pragma unroll
  for (int s = 0; s < SS; ++s) {
    const uint32_t b = bits[s] & valid;
    P.bitmap[s * words + size_t(tile) * kThreads + tid] = b;
    const uint32_t cnt = __reduce_add_sync(0xffffffffu, __popc(b));
    if (lane == 0 && cnt) atomicAdd(&s_count[s], cnt);
  }
  __syncthreads();
  if (tid < SS) {
    const uint32_t cnt = s_count[tid];
    P.counts[size_t(tid) * P.n_tiles + tile] = cnt;
    if (cnt) atomicAdd(P.super_sum + size_t(tid) * P.n_super + tile / kSuper, cnt);
  }
  count_writes(P, t0, tid, valid);
  pdl_launch_dependents();
}

// mark, UNION of one-column keys with DISTINCT values in a narrow range
// (kmin + [0, range), range <= kLookupMax): a shared table maps value - kmin
// to 1 + the stream selecting it, so each element costs one lookup and one
// bit insert into its stream's word (shared, thread-private) instead of one
// compare per stream.  ncu showed the compare-per-stream kernel ALU-bound
// (92.5 % ALU pipe, 30 instructions per element at 8 streams).
constexpr int kLookupMax = 1024;

__global__ void __launch_bounds__(kThreads) mark_lookup_kernel(const __grid_constant__ Params P) {
  __shared__ uint8_t tab[kLookupMax];
  __shared__ uint32_t sw[TIDQ_MAX_STREAMS][kThreads];
  __shared__ uint32_t s_count[TIDQ_MAX_STREAMS];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int S = P.n_streams;
  const uint32_t tile = blockIdx.x;
  const uint64_t t0 = uint64_t(tile) * kTile;
  uint4 x[kRounds];
  load_bound(P, 0, t0, tid, x);
  const uint32_t kmin = P.lookup_min, range = P.lookup_range;
  for (uint32_t i = tid; i < range; i += kThreads) tab[i] = 0;
  if (tid < TIDQ_MAX_STREAMS) s_count[tid] = 0;
  for (int s = 0; s < S; ++s) sw[s][tid] = 0;
  __syncthreads();
  if (tid < S) tab[P.kv[__ffs(P.streams[tid].select) - 1][0] - kmin] = uint8_t(tid + 1);
  pdl_wait();  // as in mark_kernel: scratch is written only after the previous scan
  __syncthreads();
  uint32_t valid = 0xffffffffu;
  if (t0 + kTile > P.n) {
    valid = 0;
#pragma unroll
    for (int r = 0; r < kRounds; ++r)
#pragma unroll
      for (int c = 0; c < kVec; ++c)
        valid |= uint32_t(t0 + (uint64_t(r) * kThreads + tid) * kVec + c < P.n) << (r * kVec + c);
  }
#pragma unroll
  for (int r = 0; r < kRounds; ++r)
#pragma unroll
    for (int c = 0; c < kVec; ++c) {
      const uint32_t d = comp(x[r], c) - kmin;
      if (d < range) {
        const uint32_t id = tab[d];
        if (id) sw[id - 1][tid] |= 1u << (r * kVec + c);
      }
    }
  const size_t words = size_t(P.n_tiles) * kThreads;
  for (int s = 0; s < S; ++s) {
    const uint32_t b = sw[s][tid] & valid;
    P.bitmap[s * words + size_t(tile) * kThreads + tid] = b;
    const uint32_t cnt = __reduce_add_sync(0xffffffffu, __popc(b));
    if (lane == 0 && cnt) atomicAdd(&s_count[s], cnt);
  }
  __syncthreads();
  if (tid < S) {
    const uint32_t cnt = s_count[tid];
    P.counts[size_t(tid) * P.n_tiles + tile] = cnt;
    if (cnt) atomicAdd(P.super_sum + size_t(tid) * P.n_super + tile / kSuper, cnt);
  }
  count_writes(P, t0, tid, valid);
  pdl_launch_dependents();
}

using MarkFn = void (*)(Params);

template <int NB>
MarkFn pick_mark(bool single, bool general) {
  if (single) return general ? mark_kernel<NB, true, true> : mark_kernel<NB, true, false>;
  return general ? mark_kernel<NB, false, true> : mark_kernel<NB, false, false>;
}

// Measured (C3/C4, 500M triples): the S-specialised kernel streams at copy
// bandwidth for S <= 3 (46 registers); from S = 4 it holds 69-73 registers
// and the runtime-S kernel (45 registers, 8-wide compare loop) is 2x faster.
MarkFn select_multi1(int S) {
  switch (S) {
    case 1: return mark_multi1_kernel<1>;
    case 2: return mark_multi1_kernel<2>;
    case 3: return mark_multi1_kernel<3>;
    default: return mark_multi1_kernel<0>;
  }
}

MarkFn select_mark(int nb, bool single, bool general) {
  switch (nb) {
    case 0: return pick_mark<0>(single, general);
    case 1: return pick_mark<1>(single, general);
    case 2: return pick_mark<2>(single, general);
    default: return pick_mark<3>(single, general);
  }
}

// Algorithmic bytes of one scan: every bound column
// read once (4 B/triple; 2 B for the predicate-code column); per emitted row
// and output field, the write plus, for a gathered free column, its 4-byte
// read.  FILTER bitmap lookups and the hit-bitmap round trip (N/8 B per
// stream) are not counted.
uint64_t algorithmic_bytes(const Params& P, int nb, const uint64_t* counts) {
  uint64_t b = (P.p16 ? 2ull : 4ull) * P.n * uint64_t(nb);
  for (int s = 0; s < P.n_streams; ++s) {
    const StreamP& st = P.streams[s];
    uint64_t per_row = 0;
    for (int k = 0; k < st.n_out; ++k) {
      switch (st.out[k].kind) {
        case kFieldCol: per_row += 8; break;
        case kFieldConst: per_row += 4; break;
        case kFieldLocal: per_row += 4; break;
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
// fields, run mark -> (host super-tile offsets) -> emit, and hand back one
// exact table per stream.
// Launch with programmatic stream serialization: the grid may be scheduled
// before its predecessor on the stream completes (it griddepcontrol.waits).
template <class... KArgs, class... Args>
static void launch_pdl(void (*kernel)(KArgs...), uint32_t grid, uint32_t block, size_t smem,
                       cudaStream_t stream, Args&&... args) {
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

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
struct HostTrace {
  bool on = getenv("TIDQ_HOST_TRACE") != nullptr;
  double acc[8] = {0};
  int calls = 0;
};
static HostTrace g_trace;

void run_scan(tidq_store* st, const tidq_scan_spec& spec, tidq_table** out) {
  using namespace scan;
  Ctx* c = st->ctx;
  double tt[8] = {now_us()};
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
  // predicate codes: a pass whose only bound column is p streams the store's
  // 16-bit code column; key values become codes (absent predicate: 0xFFFF,
  // which no triple carries)
  int p_bytes = 4;
  const char* p16_env = getenv("TIDQ_P16");
  if (st->p16.ptr && nb == 1 && P->bslot[0] == 1 && !(p16_env && p16_env[0] == '0')) {
    P->p16 = st->p16.as<uint16_t>();
    p_bytes = 2;
    for (int q = 0; q < K; ++q) {
      if (!(P->kb_mask[q] & 1u)) continue;
      auto it = std::lower_bound(st->pvals.begin(), st->pvals.end(), P->kv[q][0]);
      P->kv[q][0] = (it != st->pvals.end() && *it == P->kv[q][0])
                        ? uint32_t(it - st->pvals.begin()) + kPcodeBase : 0xFFFFu;
    }
  }
  const bool single = K == 1;
  bool general = false;
  bool simple = true;
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
          sp.gather_mask |= 1u << kind;
        }
      } else if (kind == TIDQ_OUT_LOCAL) {
        TIDQ_REQUIRE(st->n <= (1ull << 32), TIDQ_E_INVALID, "local indices need a store below 2^32 triples");
        f.kind = kFieldLocal;
      } else if (kind == TIDQ_OUT_INDEX) {
        f.kind = kFieldIndex;
        simple = false;
      } else if (kind == TIDQ_OUT_MARKS) {
        f.kind = kFieldMarks;
        sp.gather_mask |= load;  // marks are re-tested on the bound values
        simple = false;
      } else if (kind == TIDQ_OUT_ANSWER) {
        TIDQ_REQUIRE(ss.answer_key >= 0 && ss.answer_key < K, TIDQ_E_INVALID, "bad answer_key");
        f.kind = kFieldAnswer;
        sp.gather_mask |= 7u;
        simple = false;
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
    if (ss.key_bitmap) {
      TIDQ_REQUIRE(ss.key_bitmap_slot >= 0 && ss.key_bitmap_slot < 3, TIDQ_E_INVALID, "bad key_bitmap_slot");
      sp.key_bm = ss.key_bitmap->words.as<uint32_t>();
      sp.key_bm_bits = ss.key_bitmap->n_bits;
      sp.key_bm_slot = ss.key_bitmap_slot;
      sp.gather_mask |= 1u << ss.key_bitmap_slot;  // a variable slot: gathered
    }
    if (sp.eq_flags & TIDQ_EQ_SP) sp.epi_mask |= 3u;
    if (sp.eq_flags & TIDQ_EQ_SO) sp.epi_mask |= 5u;
    if (sp.eq_flags & TIDQ_EQ_PO) sp.epi_mask |= 6u;
    for (int f = 0; f < sp.n_filters; ++f) sp.epi_mask |= 1u << sp.filter_slot[f];
    if (sp.eq_flags || sp.n_filters) general = true;
  }
  const int nkb = nb;  // columns some key binds (the algorithmic read set)

  const uint64_t n_tiles = std::max<uint64_t>((st->n + kTile - 1) / kTile, 1);
  TIDQ_REQUIRE(n_tiles < (1ull << 31), TIDQ_E_INVALID, "store too large for one scan");
  const uint64_t n_super = (n_tiles + kSuper - 1) / kSuper;
  P->n_tiles = uint32_t(n_tiles);
  P->n_super = uint32_t(n_super);
  const uint64_t n_counts = uint64_t(S) * n_tiles;

  // scratch: bitmap | counts | super offsets | stream totals, and the
  // super-tile sums in their own buffer that is all zero between scans (the
  // consumer of the sums re-zeroes them; a failed scan leaves it dirty)
  const size_t bitmap_b = round_up(n_counts * kThreads * 4, 256);
  const size_t counts_b = round_up(n_counts * 4, 256);
  const size_t soff_b = round_up(S * n_super * 8, 256);
  const size_t totals_b = round_up(8 * TIDQ_MAX_STREAMS, 256);
  const size_t need = bitmap_b + counts_b + soff_b + totals_b;
  if (c->lookback.bytes < need) c->lookback = DevBuf(c, need);
  char* sbase = c->lookback.as<char>();
  P->bitmap = reinterpret_cast<uint32_t*>(sbase);
  P->counts = reinterpret_cast<uint32_t*>(sbase + bitmap_b);
  uint64_t* soff_dev = reinterpret_cast<uint64_t*>(sbase + bitmap_b + counts_b);
  uint64_t* totals_dev = reinterpret_cast<uint64_t*>(sbase + bitmap_b + counts_b + soff_b);
  P->super_off = soff_dev;
  const size_t ssum_used = size_t(S) * n_super * 4;
  if (c->ssum.bytes < ssum_used) {
    c->ssum = DevBuf(c, round_up(ssum_used, 1 << 16));
    c->ssum_clean = false;
  }
  if (!c->ssum_clean) TIDQ_CUDA(cudaMemsetAsync(c->ssum.ptr, 0, c->ssum.bytes, c->stream));
  c->ssum_clean = false;  // until this scan's consumer has re-zeroed it
  P->super_sum = c->ssum.as<uint32_t>();
  const size_t hs = round_up(ssum_used, 8) + S * n_super * 8;
  char* hbuf = c->pinned_scratch(hs);
  uint32_t* ssum_h = reinterpret_cast<uint32_t*>(hbuf);
  uint64_t* soff_h = reinterpret_cast<uint64_t*>(hbuf + round_up(ssum_used, 8));

  // ---- output allocation (exact, or from capacity hints) ----
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
  bool hinted = true;
  for (int s = 0; s < S; ++s) hinted = hinted && spec.streams[s].capacity_hint > 0;
  // TIDQ_SCAN_CONCAT: all streams write one table (stream order = row
  // order), a UNION of single-pattern branches without the concatenation
  const bool concat = spec.flags & TIDQ_SCAN_CONCAT;
  auto share_outputs = [&](uint64_t capacity) {  // table 0's columns for every stream
    allocate(0, capacity);
    for (int s = 1; s < S; ++s) {
      for (int k = 0; k < P->streams[s].n_out; ++k) P->streams[s].out[k].ptr = P->streams[0].out[k].ptr;
      P->streams[s].capacity = capacity;
    }
  };
  if (concat) {
    TIDQ_REQUIRE(hinted, TIDQ_E_INVALID, "TIDQ_SCAN_CONCAT needs a capacity hint on every stream");
    for (int s = 1; s < S; ++s) {
      TIDQ_REQUIRE(spec.streams[s].n_out == spec.streams[0].n_out, TIDQ_E_INVALID,
                   "TIDQ_SCAN_CONCAT streams must have the same outputs");
      for (int k = 0; k < spec.streams[s].n_out; ++k) {
        auto width = [](int kind) { return kind == TIDQ_OUT_INDEX ? 8 : kind == TIDQ_OUT_ANSWER ? 1 : 4; };
        TIDQ_REQUIRE(width(spec.streams[s].out[k]) == width(spec.streams[0].out[k]), TIDQ_E_INVALID,
                     "TIDQ_SCAN_CONCAT streams must have the same output types");
      }
    }
    P->concat = 1;
    for (int s = 1; s < S; ++s) allocate(s, 0);  // the empty tables of streams 1..S-1
    uint64_t cap = 0;
    for (int s = 0; s < S; ++s) cap += std::min<uint64_t>(spec.streams[s].capacity_hint, st->n);
    share_outputs(cap);
  } else if (hinted) {
    for (int s = 0; s < S; ++s) allocate(s, std::min<uint64_t>(spec.streams[s].capacity_hint, st->n));
  }

  // Post-filter: a predicate stream whose pre-predicate hits are dense (>= 1
  // per 64 triples: most 128-B lines of the predicate column would be
  // gathered by mark AND again by emit) is marked without its predicates and
  // filtered by the emit + a compaction.  Needs guaranteed capacity bounds.
  std::vector<DevBuf> keep_flags(S);
  bool any_post = false;
  if (hinted && simple && !concat && (spec.flags & TIDQ_SCAN_ASYNC)) {
    for (int s = 0; s < S; ++s) {
      StreamP& sp = P->streams[s];
      if (!(sp.eq_flags || sp.n_filters) || sp.n_out == 0 || spec.streams[s].capacity_hint * 64 < st->n)
        continue;
      sp.post = 1;
      sp.gather_mask |= sp.epi_mask;
      keep_flags[s] = DevBuf(c, std::max<uint64_t>(tables[s]->capacity, 1));
      sp.keep = keep_flags[s].as<uint8_t>();
      any_post = true;
    }
    if (any_post) {
      general = false;
      for (int s = 0; s < S; ++s)
        general = general || (!P->streams[s].post && (P->streams[s].eq_flags || P->streams[s].n_filters));
    }
  }
  // interleaved (s, o) gathers for streams that need both
  const char* so_env = getenv("TIDQ_SO");
  if (st->so.ptr && !(so_env && so_env[0] == '0')) {
    P->so = st->so.as<uint2>();
    for (int s = 0; s < S; ++s) P->streams[s].use_so = (P->streams[s].gather_mask & 5u) == 5u;
  }
  // device pointer to each stream's final row count
  std::vector<const uint64_t*> count_src(S);
  for (int s = 0; s < S; ++s) count_src[s] = totals_dev + s;
  std::vector<DevBuf> post_scratch;
  auto postfilter = [&]() {
    for (int s = 0; s < S; ++s) {
      StreamP& sp = P->streams[s];
      if (!sp.post) continue;
      const uint64_t cap = std::max<uint64_t>(tables[s]->capacity, 1);
      const uint64_t nb = (cap + kPfBlk - 1) / kPfBlk;
      DevBuf bcount(c, nb * 4), boffs(c, nb * 8), kept(c, 8);
      TIDQ_CUDA(cudaMemsetAsync(kept.ptr, 0, 8, c->stream));
      postfilter_count_kernel<<<unsigned(nb), kPfT, 0, c->stream>>>(
          sp.keep, totals_dev + s, bcount.as<uint32_t>(), kept.as<unsigned long long>());
      prims::exclusive_scan_async(c, bcount.as<uint32_t>(), boffs.as<uint64_t>(), nb);
      PostCols pc{};
      pc.n = sp.n_out;
      std::vector<DevBuf> fresh(sp.n_out);
      for (int k = 0; k < sp.n_out; ++k) {
        fresh[k] = DevBuf(c, cap * 4);
        pc.in[k] = tables[s]->cols[k].buf.as<uint32_t>();
        pc.out[k] = fresh[k].as<uint32_t>();
      }
      postfilter_write_kernel<<<unsigned(nb), kPfT, 0, c->stream>>>(sp.keep, totals_dev + s,
                                                                    boffs.as<uint64_t>(), pc);
      c->count_launch(2);
      TIDQ_CUDA(cudaGetLastError());
      for (int k = 0; k < sp.n_out; ++k) tables[s]->cols[k].buf = std::move(fresh[k]);
      count_src[s] = kept.as<uint64_t>();
      post_scratch.push_back(std::move(kept));  // read by the count copy below
    }
  };

  // emit grid: one warp per group of emit_group tiles
  auto launch_emit = [&](uint64_t max_hits) {
    // group size from the hit density: dense scans want one warp per tile
    // (or pair), sparse ones a coalesced count check over many tiles per warp
    // one warp per (tile group, stream): measured faster than one warp
    // emitting every stream of its tiles (C3 UNION x4: 1.94 vs 2.25 ms)
    P->emit_split = 1;
    const double per_tile = double(max_hits) / double(n_tiles) / double(S);
    // (tiles of 4096: >= 8 hits per tile -> a warp per tile (gather-bound:
    // more warps win, C2 rank 10: 50 vs 54 us); fewer -> groups
    // of 8 tiles emitted as one batch (kBatchMaxGroup) when their hits fit one
    // list; very sparse -> 32 tiles per coalesced count check)
    static const double dense_thr = [] {  // TIDQ_EMIT_DENSE: A/B knob for the threshold
      const char* e = getenv("TIDQ_EMIT_DENSE");
      return e ? atof(e) : 8.0;
    }();
    P->emit_group = per_tile >= dense_thr ? 1u : per_tile >= 1.0 / 32 ? 8u : 32u;
    // multi-stream scans of moderate density (every stream <= batch_max hits
    // per tile: 8 tiles' hits fit one list): one batched unit per 8 tiles and
    // stream amortises the unit setup (offsets, list scans, row-writer setup)
    // that the issue-bound emit spends most of its instructions on
    // (the largest G in {8, 4, 2} whose G tiles of the densest stream fit
    // ~90 % of the unit list; TIDQ_EMIT_BATCH_CAP: A/B knob, 0: off)
    const char* bm_env = getenv("TIDQ_EMIT_BATCH_CAP");
    const double batch_cap = bm_env ? atof(bm_env) : 920.0;
    // (not with post-filtered streams: C4 FILTER queries measured 2-5 % slower)
    const char* s1_env = getenv("TIDQ_EMIT_BATCH_S1");  // A/B knob: single-stream scans too
    const int min_s = s1_env && s1_env[0] == '1' ? 1 : 2;
    if (S >= min_s && P->emit_group == 1 && batch_cap > 0 && !any_post) {
      double mx = 0;
      for (int s = 0; s < S; ++s)
        mx = std::max(mx, double(concat ? std::min<uint64_t>(spec.streams[s].capacity_hint, st->n)
                                        : P->streams[s].capacity) / double(n_tiles));
      for (uint32_t g = kBatchMaxGroup; g >= 2; g /= 2)
        if (g * mx <= batch_cap) {
          P->emit_group = g;
          break;
        }
    }
    const uint64_t groups = (n_tiles + P->emit_group - 1) / P->emit_group * uint64_t(P->emit_split ? S : 1);
    const uint32_t grid = uint32_t(std::max<uint64_t>(1, (groups + kEmitWarps - 1) / kEmitWarps));
    auto emit = simple ? emit_kernel<true> : emit_kernel<false>;
    launch_pdl(emit, grid, kEmitWarps * 32, 0, c->stream, *P);
    c->count_launch();
    TIDQ_CUDA(cudaGetLastError());
  };

  tt[1] = now_us();
  // ---- pass 1: mark + count ----
  MarkFn mark = select_mark(nb, single, general);
  size_t mark_smem = single ? 0 : size_t(kTile) * 4;
  bool multi1 = !single && !general && nb == 1 && S <= kMulti1Max;
  for (int s = 0; s < S && multi1; ++s)
    multi1 = __builtin_popcount(P->streams[s].select) == 1 &&
             P->kb_mask[__builtin_ctz(P->streams[s].select)] == 1u;  // key binds the column
  if (multi1) {
    mark = select_multi1(S);
    mark_smem = 0;
  }
  // the predicate-code column: fp16x2 compares for up to kF16Max one-column
  // streams (TIDQ_MARK_F16=0: the integer kernels; TIDQ_MARK_F16_MAX: A/B of
  // the stream count up to which it replaces the lookup kernel)
  const char* h_env = getenv("TIDQ_MARK_F16");
  const char* hm_env = getenv("TIDQ_MARK_F16_MAX");
  const int f16_max = std::min(hm_env ? atoi(hm_env) : 8, 8);
  bool f16 = P->p16 && !single && !general && nb == 1 && S <= f16_max && !(h_env && h_env[0] == '0');
  for (int s = 0; s < S && f16; ++s)
    f16 = __builtin_popcount(P->streams[s].select) == 1 && P->kb_mask[__builtin_ctz(P->streams[s].select)] == 1u;
  if (f16) {
    static const MarkFn f16k[8] = {mark_multi1_p16_kernel<1>, mark_multi1_p16_kernel<2>, mark_multi1_p16_kernel<3>,
                                   mark_multi1_p16_kernel<4>, mark_multi1_p16_kernel<5>, mark_multi1_p16_kernel<6>,
                                   mark_multi1_p16_kernel<7>, mark_multi1_p16_kernel<8>};
    mark = f16k[S - 1];
    mark_smem = 0;
    multi1 = true;  // (not the lookup kernel below)
  }
  // one-column UNIONs of >= 4 streams with distinct keys in a narrow range:
  // the lookup kernel (one shared-table lookup per element, not one compare
  // per stream)
  const char* lk_env = getenv("TIDQ_LOOKUP_MIN_S");  // A/B knob
  const int lookup_min_s = lk_env ? atoi(lk_env) : 4;
  bool lookup = !single && !general && nb == 1 && S >= lookup_min_s && !f16;
  for (int s = 0; s < S && lookup; ++s)
    lookup = __builtin_popcount(P->streams[s].select) == 1 &&
             P->kb_mask[__builtin_ctz(P->streams[s].select)] == 1u;
  if (lookup) {
    uint32_t kmin = 0xffffffffu, kmax = 0;
    std::vector<uint32_t> kvs;
    for (int s = 0; s < S; ++s) {
      const uint32_t v = P->kv[__builtin_ctz(P->streams[s].select)][0];
      kmin = std::min(kmin, v);
      kmax = std::max(kmax, v);
      kvs.push_back(v);
    }
    std::sort(kvs.begin(), kvs.end());
    lookup = uint64_t(kmax) - kmin < uint64_t(kLookupMax) &&
             std::adjacent_find(kvs.begin(), kvs.end()) == kvs.end();
    if (lookup) {
      P->lookup_min = kmin;
      P->lookup_range = kmax - kmin + 1;
      mark = mark_lookup_kernel;
      mark_smem = 0;
    }
  }
  DevBuf wcount;  // write_counts instrumentation: the caller's counters, in and out
  if (spec.write_counts && st->n) {
    wcount = DevBuf(c, st->n * 4);
    TIDQ_CUDA(cudaMemcpyAsync(wcount.ptr, spec.write_counts, st->n * 4, cudaMemcpyHostToDevice, c->stream));
    P->write_counts = wcount.as<uint32_t>();
  }
  cudaEvent_t ev = c->prof_begin(c->stream);
  cudaEvent_t evm = c->prof_begin(c->stream);
  uint32_t mark_grid = uint32_t(n_tiles);
  if (P->p16 && single && !general && !multi1 && !lookup) {  // ?s P ?o on the code column
    constexpr int kTpc = 1;  // 2 / 4 tiles per CTA measured no faster (C2 mark 38.4 / 40.2 vs 37.8 us)
    mark = mark_p16_kernel<kTpc>;
    mark_smem = 0;
    mark_grid = uint32_t((n_tiles + kTpc - 1) / kTpc);
  }
  launch_pdl(mark, mark_grid, kThreads, mark_smem, c->stream, *P);
  c->count_launch();
  // the mark pass alone: 4 B per triple and bound column
  c->prof_end("scan.mark", evm, c->stream, uint64_t(p_bytes) * st->n * uint64_t(nkb));
  TIDQ_CUDA(cudaGetLastError());
  std::vector<uint64_t> counts(S, 0);
  if (hinted) {
    // ---- hint mode: offsets on the device, emit immediately, one sync ----
    // TIDQ_SCAN_ASYNC: the hints are guaranteed bounds (no overflow to
    // re-emit), so return once queued; each table's count is written by the
    // offsets kernel straight into a pinned slot (post-filtered streams: a
    // copy of the kept count) and read on first use.  (Profiling runs
    // synchronously: it needs counts.)
    const bool async = (spec.flags & TIDQ_SCAN_ASYNC) && !ev && !wcount.ptr && int(c->free_row_slots.size()) >= S;
    std::vector<int> slots;
    if (async)
      for (int s = 0; s < S; ++s) {
        slots.push_back(c->free_row_slots.back());
        c->free_row_slots.pop_back();
        if (!P->streams[s].post && !(concat && s)) P->host_total[s] = c->row_slots + slots[s];
      }
    launch_pdl(super_offsets_kernel, concat ? 1 : S, 1024, 0, c->stream, *P, soff_dev, totals_dev);
    c->count_launch();
    uint64_t hint_hits = 0;
    for (int s = 0; s < S; ++s) hint_hits += P->streams[s].capacity;
    if (concat) hint_hits = P->streams[0].capacity;
    launch_emit(hint_hits);
    if (any_post) postfilter();
    tt[2] = now_us();
    c->prof_end("scan", ev, c->stream, 0, 0);
    if (async) {
      for (int s = 0; s < S; ++s) {
        if (P->streams[s].post)
          TIDQ_CUDA(cudaMemcpyAsync(c->row_slots + slots[s], count_src[s], 8, cudaMemcpyDeviceToHost, c->stream));
        if (concat && s) {
          tables[s]->set_rows(0);
          c->free_row_slots.push_back(slots[s]);
        } else {
          tables[s]->defer_rows(slots[s]);
        }
        out[s] = tables[s].release();
      }
      c->ssum_clean = true;  // the offsets kernel re-zeroes the sums in stream order
      if (g_trace.on) {
        g_trace.acc[4] += tt[1] - tt[0];
        g_trace.acc[5] += tt[2] - tt[1];
        g_trace.acc[6] += now_us() - tt[2];
        if (++g_trace.calls % 100 == 0) {
          fprintf(stderr, "[tidq host] per async scan: setup %.1f us, launches %.1f us, tail %.1f us\n",
                  g_trace.acc[4] / 100, g_trace.acc[5] / 100, g_trace.acc[6] / 100);
          for (double& x : g_trace.acc) x = 0;
        }
      }
      return;
    }
    uint64_t* th = reinterpret_cast<uint64_t*>(hbuf);
    if (any_post) {
      for (int s = 0; s < S; ++s)
        TIDQ_CUDA(cudaMemcpyAsync(th + s, count_src[s], 8, cudaMemcpyDeviceToHost, c->stream));
    } else {
      TIDQ_CUDA(cudaMemcpyAsync(th, totals_dev, S * 8, cudaMemcpyDeviceToHost, c->stream));
    }
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    tt[3] = now_us();
    bool overflow = false;
    for (int s = 0; s < S; ++s) {
      counts[s] = th[s];
      if (counts[s] > tables[s]->capacity) overflow = true;
    }
    if (concat) {  // everything is table 0's
      uint64_t total = 0;
      for (int s = 0; s < S; ++s) total += counts[s], counts[s] = 0;
      counts[0] = total;
      overflow = total > tables[0]->capacity;
      if (overflow) {
        share_outputs(total);  // the offsets already include the stream bases
        launch_emit(total);
      }
    } else if (overflow) {  // a hint was too small: re-emit those streams exactly
      uint64_t total = 0;
      for (int s = 0; s < S; ++s) {
        if (counts[s] > tables[s]->capacity) allocate(s, counts[s]);
        total += counts[s];
      }
      launch_emit(total);
    }
  } else {
    c->prof_end("scan", ev, c->stream, 0, 0);
    TIDQ_CUDA(cudaMemcpyAsync(ssum_h, P->super_sum, ssum_used, cudaMemcpyDeviceToHost, c->stream));
    TIDQ_CUDA(cudaMemsetAsync(P->super_sum, 0, ssum_used, c->stream));
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    for (int s = 0; s < S; ++s) {
      uint64_t run = 0;
      for (uint64_t j = 0; j < n_super; ++j) {
        soff_h[s * n_super + j] = run;
        run += ssum_h[s * n_super + j];
      }
      counts[s] = run;
    }
    for (int s = 0; s < S; ++s) allocate(s, counts[s]);
    uint64_t total = 0;
    for (int s = 0; s < S; ++s) total += counts[s];
    if (total) {
      TIDQ_CUDA(cudaMemcpyAsync(soff_dev, soff_h, S * n_super * 8, cudaMemcpyHostToDevice, c->stream));
      cudaEvent_t ev2 = c->prof_begin(c->stream);
      launch_emit(total);
      c->prof_end("scan", ev2, c->stream, 0, 0);
    }
  }
  if (ev) {
    auto& kp = c->prof["scan"];
    kp.launches += 1;
    kp.bytes += algorithmic_bytes(*P, nkb, counts.data());
  }
  if (wcount.ptr)
    TIDQ_CUDA(cudaMemcpyAsync(spec.write_counts, wcount.ptr, st->n * 4, cudaMemcpyDeviceToHost, c->stream));
  TIDQ_CUDA(cudaStreamSynchronize(c->stream));
  c->ssum_clean = true;
  for (int s = 0; s < S; ++s) {
    tables[s]->set_rows(counts[s]);
    out[s] = tables[s].release();
  }
  if (g_trace.on) {
    tt[4] = now_us();
    g_trace.acc[0] += tt[1] - tt[0];
    if (tt[2] > 0) {
      g_trace.acc[1] += tt[2] - tt[1];
      g_trace.acc[2] += tt[3] - tt[2];
      g_trace.acc[3] += tt[4] - tt[3];
    }
    if (++g_trace.calls % 100 == 0) {
      fprintf(stderr, "[tidq host] per scan: setup %.1f us, launches %.1f us, sync wait %.1f us, tail %.1f us\n",
              g_trace.acc[0] / 100, g_trace.acc[1] / 100, g_trace.acc[2] / 100, g_trace.acc[3] / 100);
      for (double& x : g_trace.acc) x = 0;
    }
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
