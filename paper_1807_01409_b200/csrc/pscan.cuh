// Persistent, warp-specialised pattern scan for sm_100a (the hot path of
// tidq_scan: streams whose outputs are columns / constants / indices and no
// epilogue predicates).  One CTA per SM runs a four-role pipeline over
// 8192-triple tiles:
//
//   warp 0   producer   grabs the next tile id (atomic counter, so tiles are
//                       handed out in order to running CTAs) and streams the
//                       bound columns of that tile into a shared-memory ring
//                       with cp.async.bulk (TMA) + mbarrier complete_tx;
//   warps 2-9 matchers  test the keys on the staged tile, build per-stream hit
//                       bits, rank hits inside 128-triple warp chunks, scan
//                       the 64 chunks, publish the tile aggregate, and
//                       prefetch the gathered columns of hit vectors into L2;
//   warp 1   look-back  resolves the tile's global offset CONCURRENTLY with
//                       the matchers (it only needs predecessors), examining
//                       up to 128 predecessor tiles per L2 round trip over
//                       packed 64-bit (flag|count) status words, then
//                       publishes the inclusive prefix;
//   warps 10-13 writers gather the free columns (L2 hits) and write every
//                       stream's rows at their final, order-preserving place.
//
// Roles hand tiles to each other through mbarriers (full/empty for the TMA
// ring; started/counted/based/freed for a ring of metadata slots), so the
// HBM stream never waits for a look-back or a gather.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace tidq {
namespace pscan {

constexpr int kTile = 8192;
constexpr int kMatchWarps = 8;
constexpr int kMatchThreads = kMatchWarps * 32;  // 256
constexpr int kWriteWarps = 4;
constexpr int kRounds = kTile / (kMatchThreads * 4);  // 8 uint4 per matcher thread
constexpr int kChunks = kRounds * kMatchWarps;        // 64 chunks of 128 triples
constexpr int kMaxS = 4;
constexpr int kSlots = 4;
constexpr int kMaxStages = 8;
constexpr int kColBytes = kTile * 4;  // 32 KiB per column per tile
constexpr int kThreads = 32 * (2 + kMatchWarps + kWriteWarps);  // 448
static_assert(kRounds == 8, "layout assumes 8 rounds");

constexpr uint64_t kFlagA = 1ull << 62;
constexpr uint64_t kFlagP = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

enum : int32_t { kFieldCol = 0, kFieldConst = 1, kFieldIndex = 2 };

struct Field {
  int32_t kind;
  int32_t slot;
  uint32_t constant;
  void* ptr;
};

struct StreamP {
  uint32_t select;
  int32_t n_out;
  Field out[4];
  uint64_t capacity;
  uint32_t gather_mask;
};

struct Params {
  const uint32_t* col[3];
  const uint32_t* bcol[3];
  uint64_t n;
  uint64_t base;
  uint32_t n_tiles;
  int32_t n_keys;
  int32_t n_streams;  // power of two <= kMaxS (padding streams select nothing)
  int32_t stages;
  uint32_t kb_mask[32];
  uint32_t kv[32][3];
  StreamP streams[kMaxS];
  uint32_t* tile_counter;
  uint64_t* status;
  uint64_t* counts;
};

struct Slot {
  uint32_t tile;
  uint32_t total[kMaxS];
  uint64_t base[kMaxS];
  uint32_t cnt[kMaxS][kChunks];
  uint32_t nib[kMaxS][kMatchThreads];
};

struct alignas(16) Ctrl {
  uint64_t full[kMaxStages];
  uint64_t empty[kMaxStages];
  uint64_t started[kSlots];
  uint64_t counted[kSlots];
  uint64_t based[kSlots];
  uint64_t freed[kSlots];
  uint32_t stage_tile[kMaxStages];
};

__host__ __device__ constexpr size_t ring_offset() {
  return (sizeof(Ctrl) + kSlots * sizeof(Slot) + 127) / 128 * 128;
}

inline size_t smem_bytes(int nb, int stages) { return ring_offset() + size_t(stages) * nb * kColBytes; }

// ---- PTX helpers ------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile(
      "{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile(
      "{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void match_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint4 ld_nc(const uint32_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t lane_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ uint32_t comp4(const uint4& v, int c) {
  return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}

// ---- the kernel ---------------------------------------------------------------------
template <int NB, bool kSingle>
__global__ void __launch_bounds__(kThreads, 1) pscan_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(128) unsigned char sm[];
  Ctrl& ct = *reinterpret_cast<Ctrl*>(sm);
  Slot* slots = reinterpret_cast<Slot*>(sm + sizeof(Ctrl));
  unsigned char* ring = sm + ring_offset();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int D = P.stages;
  const int S = P.n_streams;

  if (threadIdx.x == 0) {
    for (int i = 0; i < D; ++i) {
      mbar_init(&ct.full[i], 1);
      mbar_init(&ct.empty[i], kMatchWarps);
    }
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&ct.started[i], 1);
      mbar_init(&ct.counted[i], 1);
      mbar_init(&ct.based[i], 1);
      mbar_init(&ct.freed[i], kWriteWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ===================== producer =====================
    if (lane != 0) return;
    for (uint32_t k = 0;; ++k) {
      const int st = int(k % D);
      if (k >= uint32_t(D)) mbar_wait(&ct.empty[st], ((k / D) & 1u) ^ 1u);
      const uint32_t tile = atomicAdd(P.tile_counter, 1u);
      ct.stage_tile[st] = tile;
      if (tile < P.n_tiles) {
        mbar_arrive_tx(&ct.full[st], uint32_t(NB) * kColBytes);
#pragma unroll
        for (int b = 0; b < NB; ++b)
          tma_load(ring + (size_t(st) * NB + b) * kColBytes, P.bcol[b] + size_t(tile) * kTile,
                   kColBytes, &ct.full[st]);
      } else {
        mbar_arrive(&ct.full[st]);
        return;
      }
    }
  } else if (warp >= 2 && warp < 2 + kMatchWarps) {
    // ===================== matchers =====================
    const int mt = threadIdx.x - 64;
    const int mw = mt >> 5;
    for (uint32_t k = 0;; ++k) {
      const int st = int(k % D);
      mbar_wait(&ct.full[st], (k / D) & 1u);
      const uint32_t tile = ct.stage_tile[st];
      const int sl = int(k % kSlots);
      Slot& slot = slots[sl];
      if (k >= uint32_t(kSlots)) mbar_wait(&ct.freed[sl], ((k / kSlots) & 1u) ^ 1u);
      if (tile >= P.n_tiles) {
        if (mt == 0) {
          slot.tile = tile;
          mbar_arrive(&ct.started[sl]);
          mbar_arrive(&ct.counted[sl]);
        }
        return;
      }
      uint4 x[NB][kRounds];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const uint4* src = reinterpret_cast<const uint4*>(ring + (size_t(st) * NB + b) * kColBytes);
#pragma unroll
        for (int r = 0; r < kRounds; ++r) x[b][r] = src[r * kMatchThreads + mt];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ct.empty[st]);  // stage may be refilled
      if (mt == 0) {
        slot.tile = tile;
        mbar_arrive(&ct.started[sl]);  // look-back can start now
      }
      const uint64_t t0 = uint64_t(tile) * kTile;
      const bool partial = t0 + kTile > P.n;
      // ---- keys -> per-stream hit bits (bit r*4+c) ----
      uint32_t hits[kMaxS] = {0u, 0u, 0u, 0u};
      if (kSingle) {
        uint32_t hb = 0;
#pragma unroll
        for (int r = 0; r < kRounds; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            bool ok = true;
#pragma unroll
            for (int b = 0; b < NB; ++b) ok = ok && comp4(x[b][r], c) == P.kv[0][b];
            hb |= uint32_t(ok) << (r * 4 + c);
          }
#pragma unroll
        for (int s = 0; s < kMaxS; ++s)
          if (s < S && P.streams[s].select) hits[s] = hb;
      } else {
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
          uint32_t m[4] = {0u, 0u, 0u, 0u};
#pragma unroll 1
          for (int q = 0; q < P.n_keys; ++q) {
            const uint32_t kb = P.kb_mask[q];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              bool ok = true;
#pragma unroll
              for (int b = 0; b < NB; ++b)
                ok = ok && (!(kb & (1u << b)) || comp4(x[b][r], c) == P.kv[q][b]);
              m[c] |= uint32_t(ok) << q;
            }
          }
#pragma unroll
          for (int s = 0; s < kMaxS; ++s) {
            const uint32_t sel = s < S ? P.streams[s].select : 0u;
#pragma unroll
            for (int c = 0; c < 4; ++c) hits[s] |= uint32_t((m[c] & sel) != 0) << (r * 4 + c);
          }
        }
      }
      if (partial) {
        uint32_t valid = 0;
#pragma unroll
        for (int r = 0; r < kRounds; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            valid |= uint32_t(t0 + (uint64_t(r) * kMatchThreads + mt) * 4 + c < P.n) << (r * 4 + c);
#pragma unroll
        for (int s = 0; s < kMaxS; ++s) hits[s] &= valid;
      }
      // ---- counts per warp chunk, L2 prefetch of gathered columns ----
#pragma unroll
      for (int s = 0; s < kMaxS; ++s) {
        if (s >= S) break;
        slot.nib[s][mt] = hits[s];
        const uint32_t gm = P.streams[s].gather_mask;
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
          const uint32_t nib = (hits[s] >> (r * 4)) & 0xFu;
          const uint32_t cnt = __reduce_add_sync(0xffffffffu, __popc(nib));
          if (lane == 0) slot.cnt[s][r * kMatchWarps + mw] = cnt;
          if (nib && gm) {
            const size_t e = size_t(t0) + (size_t(r) * kMatchThreads + mt) * 4;
#pragma unroll
            for (int kc = 0; kc < 3; ++kc)
              if (gm & (1u << kc)) asm volatile("prefetch.global.L2 [%0];" ::"l"(P.col[kc] + e));
          }
        }
      }
      match_bar();
      // ---- chunk scan: 64 chunks per stream, one warp per stream ----
      if (mw < S) {
        const int s = mw;
        const uint32_t a = slot.cnt[s][2 * lane], b = slot.cnt[s][2 * lane + 1];
        const uint32_t pair = a + b;
        uint32_t inc = pair;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
          if (lane >= d) inc += y;
        }
        const uint32_t ex = inc - pair;
        slot.cnt[s][2 * lane] = ex;
        slot.cnt[s][2 * lane + 1] = ex + a;
        if (lane == 31) slot.total[s] = inc;
      }
      match_bar();
      if (mt == 0) {
        for (int s = 0; s < S; ++s)
          st_relaxed(P.status + size_t(tile) * S + s, (tile == 0 ? kFlagP : kFlagA) | slot.total[s]);
        mbar_arrive(&ct.counted[sl]);
      }
    }
  } else if (warp == 1) {
    // ===================== look-back =====================
    const int W = 32 / S;
    const int my_s = lane & (S - 1);
    const int my_w = lane / S;
    uint32_t smask = 0;
    for (int w = 0; w < W; ++w) smask |= 1u << (w * S + my_s);
    for (uint32_t k = 0;; ++k) {
      const int sl = int(k % kSlots);
      Slot& slot = slots[sl];
      const uint32_t par = (k / kSlots) & 1u;
      mbar_wait(&ct.started[sl], par);
      const uint32_t tile = slot.tile;
      if (tile >= P.n_tiles) {
        if (lane == 0) mbar_arrive(&ct.based[sl]);
        return;
      }
      uint64_t acc = 0;
      if (tile > 0) {
        bool open = true;
        int64_t pred = int64_t(tile) - 1;
        while (true) {
          uint64_t v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int64_t t = pred - (my_w * 4 + j);
            v[j] = (open && t >= 0) ? ld_relaxed(P.status + size_t(t) * S + my_s) : kFlagP;
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int64_t t = pred - (my_w * 4 + j);
            while ((v[j] >> 62) == 0 && open && t >= 0) v[j] = ld_relaxed(P.status + size_t(t) * S + my_s);
          }
          int jp = 4;
#pragma unroll
          for (int j = 3; j >= 0; --j)
            if ((v[j] >> 62) == 2) jp = j;
          const uint32_t has = __ballot_sync(0xffffffffu, open && jp < 4);
          const uint32_t mine = has & smask;
          const int stop_w = mine ? (__ffs(mine) - 1) / S : W;
          if (open) {
            if (my_w < stop_w) {
#pragma unroll
              for (int j = 0; j < 4; ++j) acc += v[j] & kValMask;
            } else if (my_w == stop_w) {
#pragma unroll
              for (int j = 0; j < 4; ++j)
                if (j <= jp) acc += v[j] & kValMask;
            }
          }
          if (mine) open = false;
          if (!__ballot_sync(0xffffffffu, open)) break;
          pred -= 4 * W;
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1)
          if (off >= S) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      }
      mbar_wait(&ct.counted[sl], par);
      if (lane < S) {
        const uint64_t tot = slot.total[lane];
        st_relaxed(P.status + size_t(tile) * S + lane, kFlagP | (acc + tot));
        slot.base[lane] = acc;
        if (tile == P.n_tiles - 1) P.counts[lane] = acc + tot;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ct.based[sl]);
    }
  } else {
    // ===================== writers =====================
    const int ww = warp - 2 - kMatchWarps;
    const uint32_t lt = lane_lt();
    for (uint32_t k = 0;; ++k) {
      const int sl = int(k % kSlots);
      Slot& slot = slots[sl];
      mbar_wait(&ct.based[sl], (k / kSlots) & 1u);
      const uint32_t tile = slot.tile;
      if (tile >= P.n_tiles) return;
      const uint64_t t0 = uint64_t(tile) * kTile;
      for (int s = 0; s < S; ++s) {
        const StreamP& st = P.streams[s];
        if (!st.select) continue;
        const uint64_t base = slot.base[s];
        const uint32_t gm = st.gather_mask;
        const int n_out = st.n_out;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          const int mw = ww * 2 + h;
          const int mt = mw * 32 + lane;
          const uint32_t hits = slot.nib[s][mt];
          // gather all rounds first (loads in flight together), then write
          constexpr int kBatch = 4;  // rounds whose gathers are in flight together
#pragma unroll 1
          for (int r0 = 0; r0 < kRounds; r0 += kBatch) {
          uint4 g[kBatch][3];
          uint64_t pos[kBatch];
#pragma unroll
          for (int i = 0; i < kBatch; ++i) {
            const int r = r0 + i;
            const uint32_t nib = (hits >> (r * 4)) & 0xFu;
            const uint32_t b0 = __ballot_sync(0xffffffffu, nib & 1u);
            const uint32_t b1 = __ballot_sync(0xffffffffu, nib & 2u);
            const uint32_t b2 = __ballot_sync(0xffffffffu, nib & 4u);
            const uint32_t b3 = __ballot_sync(0xffffffffu, nib & 8u);
            pos[i] = base + slot.cnt[s][r * kMatchWarps + mw] + __popc(b0 & lt) + __popc(b1 & lt) +
                     __popc(b2 & lt) + __popc(b3 & lt);
            const size_t e = size_t(t0) + (size_t(r) * kMatchThreads + mt) * 4;
#pragma unroll
            for (int kc = 0; kc < 3; ++kc)
              g[i][kc] = (nib && (gm & (1u << kc))) ? ld_nc(P.col[kc] + e) : make_uint4(0, 0, 0, 0);
          }
#pragma unroll
          for (int i = 0; i < kBatch; ++i) {
            const int r = r0 + i;
            const uint32_t nib = (hits >> (r * 4)) & 0xFu;
            if (!nib) continue;
            uint64_t p = pos[i];
            const uint64_t e = t0 + (uint64_t(r) * kMatchThreads + mt) * 4;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              if (!(nib & (1u << c))) continue;
              if (p < st.capacity) {
                for (int f = 0; f < n_out; ++f) {
                  const Field& fd = st.out[f];
                  if (fd.kind == kFieldCol)
                    static_cast<uint32_t*>(fd.ptr)[p] =
                        comp4(fd.slot == 0 ? g[i][0] : (fd.slot == 1 ? g[i][1] : g[i][2]), c);
                  else if (fd.kind == kFieldConst)
                    static_cast<uint32_t*>(fd.ptr)[p] = fd.constant;
                  else
                    static_cast<int64_t*>(fd.ptr)[p] = int64_t(P.base + e + c);
                }
              }
              ++p;
            }
          }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ct.freed[sl]);
    }
  }
}

}  // namespace pscan
}  // namespace tidq
