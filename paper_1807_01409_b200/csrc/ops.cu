// Table operators of the query path (reference query_ops.py):
//   UNION concat with UNBOUND = 0            query_ops.py:359-376
//   FILTER by accepted-ID bitmap             query_ops.py:241-252
//   DISTINCT, first occurrence kept          query_ops.py:379-399
//   equi-join step of join_group             query_ops.py:144-177, 316-341
// All device-side; the host only sequences calls and reads counts.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <memory>
#include <vector>

#include "internal.cuh"
#include "prims.cuh"

namespace tidq {
namespace {

using prims::grid_for;

std::unique_ptr<tidq_table> make_table(Ctx* c, uint64_t n, int n_cols, int32_t dtype = TIDQ_U32) {
  auto t = std::make_unique<tidq_table>();
  t->ctx = c;
  t->set_rows(n);
  t->capacity = n;
  for (int k = 0; k < n_cols; ++k) {
    Column col;
    col.dtype = dtype;
    col.buf = DevBuf(c, std::max<uint64_t>(n, 1) * Column::width(dtype));
    t->cols.push_back(std::move(col));
  }
  return t;
}

const uint32_t* col_u32(const tidq_table* t, int k) {
  TIDQ_REQUIRE(k >= 0 && k < int(t->cols.size()), TIDQ_E_INVALID, "column out of range");
  TIDQ_REQUIRE(t->cols[k].dtype == TIDQ_U32, TIDQ_E_INVALID, "column is not uint32");
  return t->cols[k].buf.as<uint32_t>();
}

constexpr int kT = 256;          // threads per CTA of the elementwise kernels
constexpr int kI = 4;            // items per thread
constexpr int kBlk = kT * kI;    // rows per CTA (a multiple of 32: warps own whole keep words)

inline unsigned blk_grid(uint64_t n) { return unsigned((n + kBlk - 1) / kBlk); }

// keep word of rows whose `col` ID has its bit set in the FILTER bitmap
__global__ void __launch_bounds__(kT) bitmap_keep_kernel(const uint32_t* __restrict__ col, uint64_t n,
                                                         const uint32_t* __restrict__ words,
                                                         uint64_t nbits, uint32_t* __restrict__ keep,
                                                         uint32_t* __restrict__ setbm) {
  // setbm (optional): the key set of the KEPT rows, built on the way (the
  // two-sided semi-join's second bitmap: keys(this side) AND the other set)
  pdl_chain_enter();
  const uint64_t base = uint64_t(blockIdx.x) * kBlk;
  uint32_t id[kI];
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t i = base + j * kT + threadIdx.x;
    id[j] = i < n ? __ldg(col + i) : 0xffffffffu;
  }
  bool ok[kI];
#pragma unroll
  for (int j = 0; j < kI; ++j)  // all bitmap probes in flight before any store
    ok[j] = base + j * kT + threadIdx.x < n && uint64_t(id[j]) < nbits &&
            ((__ldg(words + (id[j] >> 5)) >> (id[j] & 31)) & 1u);
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t i = base + j * kT + threadIdx.x;
    if (setbm && ok[j]) atomicOr(setbm + (id[j] >> 5), 1u << (id[j] & 31));
    const uint32_t w = __ballot_sync(0xffffffffu, ok[j]);
    if ((threadIdx.x & 31) == 0 && i < n + 31) keep[i >> 5] = w;
  }
}

// keep word over SORTED positions: i is a run head (first of equal keys)
template <class K>
__global__ void __launch_bounds__(kT) sorted_heads_kernel(const K* __restrict__ keys, uint64_t n,
                                                          uint32_t* __restrict__ keep) {
  const uint64_t base = uint64_t(blockIdx.x) * kBlk;
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t i = base + j * kT + threadIdx.x;
    const bool head = i < n && (i == 0 || __ldg(keys + i) != __ldg(keys + i - 1));
    const uint32_t w = __ballot_sync(0xffffffffu, head);
    if ((threadIdx.x & 31) == 0 && i < n + 31) keep[i >> 5] = w;
  }
}

// DISTINCT with packed keys: mark the ORIGINAL row of every run head in a
// row bitmap (L2-resident atomics), so the kept rows come out in
// first-occurrence order (stable sort: a run's head is its smallest row).
template <class K>
__global__ void __launch_bounds__(kT) head_rows_kernel(const K* __restrict__ keys,
                                                       const uint32_t* __restrict__ perm, uint64_t n,
                                                       uint32_t* __restrict__ keep_rows) {
  const uint64_t base = uint64_t(blockIdx.x) * kBlk;
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t i = base + j * kT + threadIdx.x;
    if (i < n && (i == 0 || __ldg(keys + i) != __ldg(keys + i - 1))) {
      const uint32_t r = __ldg(perm + i);
      atomicOr(keep_rows + (r >> 5), 1u << (r & 31));
    }
  }
}

// same for more than two projected columns: compare whole rows through perm
struct RowCols {
  const uint32_t* c[8];
};

__global__ void __launch_bounds__(kT) head_rows_cols_kernel(const uint32_t* __restrict__ perm, uint64_t n,
                                                            int n_cols, const __grid_constant__ RowCols rc,
                                                            uint32_t* __restrict__ keep_rows) {
  const uint64_t base = uint64_t(blockIdx.x) * kBlk;
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t i = base + j * kT + threadIdx.x;
    if (i >= n) continue;
    const uint32_t r = __ldg(perm + i);
    bool head = i == 0;
    if (!head) {
      const uint32_t q = __ldg(perm + i - 1);
      for (int k = 0; k < n_cols && !head; ++k) head = ld_gather(rc.c[k] + r) != ld_gather(rc.c[k] + q);
    }
    if (head) atomicOr(keep_rows + (r >> 5), 1u << (r & 31));
  }
}

__global__ void __launch_bounds__(kT) pack2_kernel(const uint32_t* __restrict__ hi,
                                                   const uint32_t* __restrict__ lo,
                                                   const uint32_t* __restrict__ perm, uint64_t n,
                                                   int shift, uint64_t* __restrict__ out) {
  const uint64_t base = uint64_t(blockIdx.x) * kBlk;
  uint64_t v[kI];
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t i = base + j * kT + threadIdx.x;
    const uint32_t r = i < n ? (perm ? __ldg(perm + i) : uint32_t(i)) : 0u;
    v[j] = i < n ? (uint64_t(ld_gather(hi + r)) << shift) | uint64_t(ld_gather(lo + r)) : 0ull;
  }
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t i = base + j * kT + threadIdx.x;
    if (i < n) out[i] = v[j];
  }
}

__device__ __forceinline__ uint64_t lower_bound(const uint32_t* a, uint64_t lo, uint64_t hi, uint32_t k) {
  while (lo < hi) {
    const uint64_t m = (lo + hi) >> 1;
    if (__ldg(a + m) < k) lo = m + 1; else hi = m;
  }
  return lo;
}

__device__ __forceinline__ uint64_t upper_bound(const uint32_t* a, uint64_t lo, uint64_t hi, uint32_t k) {
  while (lo < hi) {
    const uint64_t m = (lo + hi) >> 1;
    if (__ldg(a + m) <= k) lo = m + 1; else hi = m;
  }
  return lo;
}

// equal_range of every sorted left key in the sorted right keys; a CTA first
// narrows the right range to [lower(first key), upper(last key)) of its rows
// and, when that range is short (the usual case: both sides sorted over the
// same key space), stages it in shared memory for the per-row searches.
constexpr int kEqStage = 4096;

__device__ __forceinline__ uint32_t lower_bound_s(const uint32_t* a, uint32_t lo, uint32_t hi, uint32_t k) {
  while (lo < hi) {
    const uint32_t m = (lo + hi) >> 1;
    if (a[m] < k) lo = m + 1; else hi = m;
  }
  return lo;
}

__device__ __forceinline__ uint32_t upper_bound_s(const uint32_t* a, uint32_t lo, uint32_t hi, uint32_t k) {
  while (lo < hi) {
    const uint32_t m = (lo + hi) >> 1;
    if (a[m] <= k) lo = m + 1; else hi = m;
  }
  return lo;
}

__global__ void __launch_bounds__(kT) equal_range_kernel(const uint32_t* __restrict__ ls, uint64_t nl,
                                                         const uint32_t* __restrict__ rs, uint64_t nr,
                                                         uint64_t* __restrict__ start,
                                                         uint64_t* __restrict__ cnt) {
  pdl_chain_enter();
  __shared__ uint64_t s_lo, s_hi;
  __shared__ uint32_t s_r[kEqStage];
  const uint64_t base = uint64_t(blockIdx.x) * kBlk;
  const uint64_t last = min(nl, base + kBlk) - 1;
  if (threadIdx.x == 0) s_lo = lower_bound(rs, 0, nr, __ldg(ls + base));
  if (threadIdx.x == 32) s_hi = upper_bound(rs, 0, nr, __ldg(ls + last));
  __syncthreads();
  const uint64_t blo = s_lo, bhi = s_hi;
  const bool staged = bhi - blo <= kEqStage;
  if (staged) {
    for (uint64_t i = blo + threadIdx.x; i < bhi; i += kT) s_r[i - blo] = __ldg(rs + i);
    __syncthreads();
  }
  const uint32_t span = uint32_t(staged ? bhi - blo : 0);
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t i = base + j * kT + threadIdx.x;
    if (i >= nl) continue;
    const uint32_t k = __ldg(ls + i);
    uint64_t a, b;
    if (staged) {
      const uint32_t la = lower_bound_s(s_r, 0, span, k);
      a = blo + la;
      b = blo + upper_bound_s(s_r, la, span, k);
    } else {
      a = lower_bound(rs, blo, bhi, k);
      b = upper_bound(rs, a, bhi, k);
    }
    start[i] = a;
    cnt[i] = b - a;
  }
}

struct JoinOut {
  int n_out;
  uint32_t key_mask;  // bit k: output k is the join key column (written from the sorted keys)
  uint32_t direct_mask;  // bit k: output k is the value its side's sort carried (no gather)
  int side[8];
  const uint32_t* src[8];
  uint32_t* dst[8];
  int n_eq;
  const uint32_t* eq_l[4];
  const uint32_t* eq_r[4];
  int64_t* pair_l;  // optional int64 pair outputs (merge_join drop-in)
  int64_t* pair_r;
};

// Load-balanced expansion: output p belongs to the left row i with
// offs[i] <= p < offs[i+1] and to right row ro[start[i] + p - offs[i]];
// order = (key, left row, right row).  A CTA owns kBlk consecutive outputs and
// narrows the left-row search to the rows covering them.  With equality
// pairs, a keep word per 32 outputs is produced by ballot.
//
// The kI outputs of a thread are resolved in phases — row searches, then
// every (l, r) load, then per output column all kI gathers before any store —
// so the loads of different outputs overlap instead of each output's chain
// (search -> l/r -> value -> store) waiting on the previous one's stores
// (which the compiler must assume may alias the inputs).  An output column
// that is the join key comes from the sorted key array (coalesced) instead of
// a random gather: the key of every pair is ls[i].
constexpr int kExStage = 2048;

__global__ void __launch_bounds__(kT) expand_kernel(const uint64_t* __restrict__ offs, uint64_t nl,
                                                    const uint64_t* __restrict__ start,
                                                    const uint32_t* __restrict__ lo,
                                                    const uint32_t* __restrict__ ro,
                                                    const uint32_t* __restrict__ lkeys, uint64_t total,
                                                    JoinOut jo, uint32_t* __restrict__ keep) {
  pdl_chain_enter();
  __shared__ uint64_t s_a, s_b;
  __shared__ uint64_t s_offs[kExStage];
  const uint64_t base = uint64_t(blockIdx.x) * kBlk;
  const uint64_t lastp = min(total, base + kBlk) - 1;
  // last i with offs[i] <= p  ==  upper_bound(offs, p) - 1
  if (threadIdx.x == 0) {
    uint64_t a = 0, b = nl;
    while (b - a > 1) {
      const uint64_t m = (a + b) >> 1;
      if (__ldg(offs + m) <= base) a = m; else b = m;
    }
    s_a = a;
  }
  if (threadIdx.x == 32) {
    uint64_t a = 0, b = nl;
    while (b - a > 1) {
      const uint64_t m = (a + b) >> 1;
      if (__ldg(offs + m) <= lastp) a = m; else b = m;
    }
    s_b = a + 1;
  }
  __syncthreads();
  const uint64_t ra = s_a, rb = s_b;
  // the rows covering this CTA's outputs: offsets staged in shared memory
  const bool staged = rb - ra <= kExStage;
  if (staged) {
    for (uint64_t i = ra + threadIdx.x; i < rb; i += kT) s_offs[i - ra] = __ldg(offs + i);
    __syncthreads();
  }
  uint64_t row[kI];
  uint32_t l[kI], r[kI];
#pragma unroll
  for (int j = 0; j < kI; ++j) {  // phase 1: the left row of each output
    const uint64_t p = base + j * kT + threadIdx.x;
    uint64_t a = ra;
    if (p < total) {
      if (staged) {
        uint32_t x = 0, y = uint32_t(rb - ra);
        while (y - x > 1) {
          const uint32_t m = (x + y) >> 1;
          if (s_offs[m] <= p) x = m; else y = m;
        }
        a = ra + x;
      } else {
        uint64_t b = rb;
        while (b - a > 1) {
          const uint64_t m = (a + b) >> 1;
          if (__ldg(offs + m) <= p) a = m; else b = m;
        }
      }
    }
    row[j] = a;
  }
#pragma unroll
  for (int j = 0; j < kI; ++j) {  // phase 2: (l, r) of every output, loads in flight together
    const uint64_t p = base + j * kT + threadIdx.x;
    const uint64_t a = row[j];
    if (p < total) {
      const uint64_t oa = staged ? s_offs[a - ra] : __ldg(offs + a);
      l[j] = __ldg(lo + a);
      r[j] = ld_gather(ro + __ldg(start + a) + (p - oa));
    } else {
      l[j] = r[j] = 0;
    }
  }
  for (int k = 0; k < jo.n_out; ++k) {  // phase 3: per column, kI gathers, then kI stores
    const uint32_t* src = jo.src[k];
    const bool side = jo.side[k] != 0;
    const bool key = (jo.key_mask >> k) & 1u;
    const bool direct = (jo.direct_mask >> k) & 1u;
    uint32_t v[kI];
#pragma unroll
    for (int j = 0; j < kI; ++j) {
      const uint64_t p = base + j * kT + threadIdx.x;
      v[j] = p >= total ? 0u
             : key      ? __ldg(lkeys + row[j])
             : direct   ? (side ? r[j] : l[j])
                        : ld_gather(src + (side ? r[j] : l[j]));
    }
#pragma unroll
    for (int j = 0; j < kI; ++j) {
      const uint64_t p = base + j * kT + threadIdx.x;
      if (p < total) jo.dst[k][p] = v[j];
    }
  }
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t p = base + j * kT + threadIdx.x;
    bool ok = p < total;
    if (ok && jo.pair_l) {
      jo.pair_l[p] = l[j];
      jo.pair_r[p] = r[j];
    }
    for (int e = 0; ok && e < jo.n_eq; ++e) ok = ld_gather(jo.eq_l[e] + l[j]) == ld_gather(jo.eq_r[e] + r[j]);
    if (keep) {
      const uint32_t w = __ballot_sync(0xffffffffu, ok);
      if ((threadIdx.x & 31) == 0 && p < total + 31) keep[p >> 5] = w;
    }
  }
}

// Sort a key column stably, carrying row ids: out keys sorted, out ids = perm.
// `mx`: a bound on the keys (the caller's key bound or measured maximum) —
// no max pass and host round trip of its own.
// `sorted`: the column already ascends (the stable sort would be the identity).
void sort_column(Ctx* c, const uint32_t* col, uint64_t n, uint32_t mx, DevBuf& keys, DevBuf& ids,
                 bool sorted = false) {
  keys = DevBuf(c, std::max<uint64_t>(n, 1) * 4);
  ids = DevBuf(c, std::max<uint64_t>(n, 1) * 4);
  if (!n) return;
  TIDQ_CUDA(cudaMemcpyAsync(keys.ptr, col, n * 4, cudaMemcpyDeviceToDevice, c->stream));
  prims::iota(c, ids.as<uint32_t>(), n);
  if (!sorted) prims::radix_sort_pairs(c, keys.as<uint32_t>(), ids.as<uint32_t>(), n, prims::bits_for(mx));
}

// ---- semi-join reduction ------------------------------------------------------
// Before the sort-merge, each side keeps only the rows whose key occurs on the
// other side: a key bitmap (1 bit per ID value, L2-resident at these ID
// ranges: 2^26 IDs = 8 MB) is built from each side with fire-and-forget
// atomicOr, the other side tests it and compacts (keys, row ids) in row
// order.  Pair order is unchanged: the dropped rows have no partner, and the
// kept rows keep their relative order and original row ids.
__global__ void __launch_bounds__(kT) key_bitmap_kernel(const uint32_t* __restrict__ keys, uint64_t n,
                                                        uint32_t* __restrict__ bm) {
  pdl_chain_enter();
  const uint64_t base = uint64_t(blockIdx.x) * kBlk;
  uint32_t k[kI];
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t i = base + j * kT + threadIdx.x;
    k[j] = i < n ? __ldg(keys + i) : 0u;
  }
#pragma unroll
  for (int j = 0; j < kI; ++j)
    if (base + j * kT + threadIdx.x < n) atomicOr(bm + (k[j] >> 5), 1u << (k[j] & 31));
}

// out = (a ? a : all ones) & b, word-wise
__global__ void __launch_bounds__(256) bitmap_and_kernel(const uint32_t* __restrict__ a,
                                                         const uint32_t* __restrict__ b, uint64_t words,
                                                         uint32_t* __restrict__ out) {
  pdl_chain_enter();
  const uint64_t base = uint64_t(blockIdx.x) * 1024;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint64_t i = base + j * 256 + threadIdx.x;
    if (i < words) out[i] = (a ? a[i] : 0xffffffffu) & b[i];
  }
}

// kept (key, row id) of the rows whose keep bit is set, in row order
__global__ void __launch_bounds__(256) semi_write_kernel(const uint32_t* __restrict__ words, uint64_t n_rows,
                                                         const uint64_t* __restrict__ offs,
                                                         const uint32_t* __restrict__ keys,
                                                         uint32_t* __restrict__ kout,
                                                         uint32_t* __restrict__ iout,
                                                         const uint32_t* __restrict__ idsrc) {
  pdl_chain_enter();
  const uint64_t w = blockIdx.x * 8ull + (threadIdx.x >> 5);  // a warp owns 32 words = 1024 rows
  const int lane = threadIdx.x & 31;
  const uint64_t n_words = (n_rows + 31) / 32;
  if (w * 32 >= n_words) return;
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  const uint32_t my_word = (w * 32 + lane < n_words) ? words[w * 32 + lane] : 0u;
  uint64_t pos = offs[w];
  // 8 keep words' kept keys loaded together, then stored (as select_write)
#pragma unroll 1
  for (int j0 = 0; j0 < 32; j0 += 8) {
    uint32_t wd[8], v[8], id[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      wd[i] = __shfl_sync(0xffffffffu, my_word, j0 + i);
      const uint32_t row = uint32_t((w * 32 + j0 + i) * 32 + lane);
      const bool k = (wd[i] >> lane) & 1u;
      v[i] = k ? __ldg(keys + row) : 0u;
      id[i] = idsrc ? (k ? __ldg(idsrc + row) : 0u) : row;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if ((wd[i] >> lane) & 1u) {
        const uint64_t dst = pos + __popc(wd[i] & lt);
        kout[dst] = v[i];
        iout[dst] = id[i];
      }
      pos += __popc(wd[i]);
    }
  }
}

struct SemiSide {
  DevBuf keys, ids;  // kept keys and their row ids (row order)
  uint64_t n = 0;
};

// rows of `key` (n rows) whose key bit is set in `bm` (nbits bits)
// rows of `key` (n rows) whose key bit is set in `bm` (nbits bits): keep
// bitmap + per-warp offsets, total left on the device (semi_finish writes)
struct SemiPending {
  DevBuf keep, offs;
  uint64_t n = 0;
};

void semi_count(Ctx* c, const uint32_t* key, uint64_t n, const uint32_t* bm, uint64_t nbits, SemiPending& sp,
                uint32_t* setbm = nullptr) {
  sp.n = n;
  sp.keep = DevBuf(c, ((n + kBlk - 1) / kBlk) * kBlk / 8 + 4);
  if (n) {
    pdl_chain_launch(bitmap_keep_kernel, blk_grid(n), kT, 0, c->stream, key, n, bm, nbits, sp.keep.as<uint32_t>(),
                     setbm);
    c->count_launch();
  }
  prims::select_count_async(c, sp.keep.as<uint32_t>(), n, sp.offs);
}

// idsrc: carry this column's value of each kept row instead of its row id
// (a side whose only output column it is: the join writes it straight from
// the sorted pairs instead of gathering it by row id)
void semi_finish(Ctx* c, const uint32_t* key, SemiPending& sp, uint64_t kept, SemiSide& out,
                 const uint32_t* idsrc = nullptr) {
  out.n = kept;
  out.keys = DevBuf(c, std::max<uint64_t>(kept, 1) * 4);
  out.ids = DevBuf(c, std::max<uint64_t>(kept, 1) * 4);
  if (kept) {
    const uint64_t n_warps = ((sp.n + 31) / 32 + 31) / 32;
    pdl_chain_launch(semi_write_kernel, unsigned((n_warps + 7) / 8), 256, 0, c->stream, 
        sp.keep.as<uint32_t>(), sp.n, sp.offs.as<uint64_t>(), key, out.keys.as<uint32_t>(),
        out.ids.as<uint32_t>(), idsrc);
    c->count_launch();
  }
  TIDQ_CUDA(cudaGetLastError());
}

// max of two columns, one host synchronisation
void max2(Ctx* c, const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb, uint32_t& ma, uint32_t& mb) {
  uint32_t m[2];
  const uint32_t* cols[2] = {a, b};
  const uint64_t ns[2] = {na, nb};
  prims::max_u32_multi(c, 2, cols, ns, m);
  ma = m[0];
  mb = m[1];
}

// Sort-merge join core: both sides sorted (stable), per-left-row match ranges,
// exclusive scan of the match counts = the pair count (checked against the
// row cap before any output is written).
struct JoinPlan {
  DevBuf ls, lo, rs, ro, start, cnt, offs;
  uint64_t nl = 0, total = 0;
  bool lcarry = false, rcarry = false;  // lo / ro hold a payload column's values, not row ids
};

constexpr uint64_t kSemiMinRows = 1u << 16;      // below: sort directly
constexpr uint64_t kSemiMaxBits = 1ull << 31;    // key bitmaps up to 256 MB each

// Work queued while a SideStream is active goes to the context's side stream
// (c->stream is switched; allocations and frees follow it, so the
// stream-ordered pool orders them), ordered after everything queued before;
// back() returns to the main stream, join() makes the main stream wait for
// the side work.
struct SideStream {
  Ctx* c;
  cudaStream_t main;
  bool on = true, joined = false;
  explicit SideStream(Ctx* cc) : c(cc), main(cc->stream) {
    TIDQ_CUDA(cudaEventRecord(c->ev_fork, main));
    TIDQ_CUDA(cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
    c->stream = c->side_stream;
  }
  void back() {
    if (!on) return;
    TIDQ_CUDA(cudaEventRecord(c->ev_join, c->side_stream));
    c->stream = main;
    on = false;
  }
  void join() {
    back();
    TIDQ_CUDA(cudaStreamWaitEvent(main, c->ev_join, 0));
    joined = true;
  }
  ~SideStream() {  // (an exception inside: still back on, and ordered after, the side work)
    if (joined) return;
    if (on) {
      cudaEventRecord(c->ev_join, c->side_stream);
      c->stream = main;
    }
    cudaStreamWaitEvent(main, c->ev_join, 0);
  }
};

bool side_sorts() {
  static const bool on = [] {  // A/B knob: TIDQ_SIDE_SORT=0 sorts the two sides one after the other
    const char* e = getenv("TIDQ_SIDE_SORT");
    return !(e && e[0] == '0');
  }();
  return on;
}

void join_prepare(Ctx* c, const uint32_t* lkey, uint64_t nl, const uint32_t* rkey, uint64_t nr,
                  JoinPlan& jp, bool reduced = false, uint64_t key_bound = 0,
                  const tidq_bitmap* lbm_in = nullptr, const tidq_bitmap* rbm_in = nullptr,
                  bool lsorted = false, bool rsorted = false,
                  const uint32_t* lcarry = nullptr, const uint32_t* rcarry = nullptr) {
  // (l/rsorted: that side's keys already ascend — e.g. the previous join's
  // output in a star — and its sort is skipped; the semi-join filter keeps
  // row order, so a filtered sorted side stays sorted)
  phase_mark(c, nullptr);
  uint32_t ml = 0, mr = 0;
  if (key_bound) {  // caller's bound on every key (e.g. the store's largest ID + 1): no max pass
    ml = mr = uint32_t(std::min<uint64_t>(key_bound - 1, 0xffffffffull));
  } else if (nl && nr) {
    max2(c, lkey, nl, rkey, nr, ml, mr);
  }
  phase_mark(c, "semi.max");
  const uint64_t nbits = uint64_t(std::max(ml, mr)) + 1;
  if (!reduced && nl && nr && nl + nr >= kSemiMinRows && nbits <= kSemiMaxBits) {
    const uint64_t words = (nbits + 31) / 32;
    // key sets of both sides: given (e.g. built by the scan's emit; a
    // superset only filters less) or built here
    DevBuf bml, bmr;
    const uint32_t* wl = lbm_in && lbm_in->n_bits >= nbits ? lbm_in->words.as<uint32_t>() : nullptr;
    const uint32_t* wr = rbm_in && rbm_in->n_bits >= nbits ? rbm_in->words.as<uint32_t>() : nullptr;
    SemiPending pl, pr;  // both sides counted, one host round trip for both totals
    SemiSide L, R;
    phase_mark(c, "semi.bitmaps");
    if (wl && wr) {
      semi_count(c, lkey, nl, wr, nbits, pl);
      semi_count(c, rkey, nr, wl, nbits, pr);
    } else {
      // one key set suffices: side A's set (given, else built from the
      // smaller side) filters side B, which builds the set of its KEPT keys
      // on the way (keys(B) AND keys(A)); that set then filters A — the same
      // two kept row sets as two full key sets, without the atomics of B's
      // full set (C5 star x3 first join: the 40.8 M-row side's)
      const bool a_left = wl ? true : wr ? false : nl <= nr;
      const uint32_t* wa = a_left ? wl : wr;
      DevBuf& ba = a_left ? bml : bmr;
      DevBuf& bk = a_left ? bmr : bml;
      if (!wa) {
        ba = DevBuf(c, words * 4);
        TIDQ_CUDA(cudaMemsetAsync(ba.ptr, 0, words * 4, c->stream));
        pdl_chain_launch(key_bitmap_kernel, blk_grid(a_left ? nl : nr), kT, 0, c->stream, a_left ? lkey : rkey,
                         a_left ? nl : nr, ba.as<uint32_t>());
        c->count_launch();
        wa = ba.as<uint32_t>();
      }
      bk = DevBuf(c, words * 4);
      TIDQ_CUDA(cudaMemsetAsync(bk.ptr, 0, words * 4, c->stream));
      if (a_left) {
        semi_count(c, rkey, nr, wa, nbits, pr, bk.as<uint32_t>());
        semi_count(c, lkey, nl, bk.as<uint32_t>(), nbits, pl);
      } else {
        semi_count(c, lkey, nl, wa, nbits, pl, bk.as<uint32_t>());
        semi_count(c, rkey, nr, bk.as<uint32_t>(), nbits, pr);
      }
    }
    uint64_t* h = static_cast<uint64_t*>(c->pinned_small);
    TIDQ_CUDA(cudaMemcpyAsync(h, pl.offs.as<uint64_t>() + ((nl + 1023) / 1024), 8, cudaMemcpyDeviceToHost,
                              c->stream));
    TIDQ_CUDA(cudaMemcpyAsync(h + 1, pr.offs.as<uint64_t>() + ((nr + 1023) / 1024), 8, cudaMemcpyDeviceToHost,
                              c->stream));
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    const uint64_t kl = h[0], kr = h[1];
    const int bits = prims::bits_for(std::min(ml, mr));  // kept keys occur on both sides
    jp.lcarry = lcarry != nullptr;
    jp.rcarry = rcarry != nullptr;
    const bool sort_l = kl > 1 && !lsorted, sort_r = kr > 1 && !rsorted;
    if (sort_l && sort_r && side_sorts()) {
      // the two sides' compaction + sort are independent and each is
      // latency-bound at low occupancy (ncu: 34 % warps active in a sort
      // pass): the right side's run on the side stream while the left
      // side's run here
      SideStream side(c);
      semi_finish(c, rkey, pr, kr, R, rcarry);
      prims::radix_sort_pairs(c, R.keys.as<uint32_t>(), R.ids.as<uint32_t>(), R.n, bits);
      side.back();
      semi_finish(c, lkey, pl, kl, L, lcarry);
      prims::radix_sort_pairs(c, L.keys.as<uint32_t>(), L.ids.as<uint32_t>(), L.n, bits);
      side.join();
      phase_mark(c, "semi.filter+sort_both");
      jp.nl = L.n;
      jp.ls = std::move(L.keys);
      jp.lo = std::move(L.ids);
      jp.rs = std::move(R.keys);
      jp.ro = std::move(R.ids);
    } else {
      semi_finish(c, lkey, pl, kl, L, lcarry);
      semi_finish(c, rkey, pr, kr, R, rcarry);
      phase_mark(c, "semi.filter");
      jp.nl = L.n;
      jp.ls = std::move(L.keys);
      jp.lo = std::move(L.ids);
      jp.rs = std::move(R.keys);
      jp.ro = std::move(R.ids);
      if (L.n > 1 && !lsorted) prims::radix_sort_pairs(c, jp.ls.as<uint32_t>(), jp.lo.as<uint32_t>(), L.n, bits);
      phase_mark(c, "sort_left");
      if (R.n > 1 && !rsorted) prims::radix_sort_pairs(c, jp.rs.as<uint32_t>(), jp.ro.as<uint32_t>(), R.n, bits);
      phase_mark(c, "sort_right");
    }
    nl = L.n;
    nr = R.n;
  } else {
    jp.nl = nl;
    sort_column(c, lkey, nl, ml, jp.ls, jp.lo, lsorted);
    phase_mark(c, "sort_left");
    sort_column(c, rkey, nr, mr, jp.rs, jp.ro, rsorted);
    phase_mark(c, "sort_right");
  }
  jp.start = DevBuf(c, std::max<uint64_t>(nl, 1) * 8);
  jp.cnt = DevBuf(c, std::max<uint64_t>(nl, 1) * 8);
  jp.offs = DevBuf(c, (nl + 1) * 8);
  if (nl == 0 || nr == 0) {
    jp.total = 0;
    return;
  }
  pdl_chain_launch(equal_range_kernel, blk_grid(nl), kT, 0, c->stream, jp.ls.as<uint32_t>(), nl, jp.rs.as<uint32_t>(),
                                                          nr, jp.start.as<uint64_t>(), jp.cnt.as<uint64_t>());
  c->count_launch();
  TIDQ_CUDA(cudaGetLastError());
  phase_mark(c, "equal_range");
  jp.total = prims::exclusive_scan(c, jp.cnt.as<uint64_t>(), jp.offs.as<uint64_t>(), nl);
  phase_mark(c, "count_scan");
}

void join_expand(Ctx* c, JoinPlan& jp, JoinOut& jo, uint32_t* keep) {
  if (!jp.total) return;
  pdl_chain_launch(expand_kernel, blk_grid(jp.total), kT, 0, c->stream,
      jp.offs.as<uint64_t>(), jp.nl, jp.start.as<uint64_t>(), jp.lo.as<uint32_t>(),
      jp.ro.as<uint32_t>(), jp.ls.as<uint32_t>(), jp.total, jo, keep);
  c->count_launch();
  TIDQ_CUDA(cudaGetLastError());
}

// rows of `in` whose bit is set in `keep` (n_rows bits) -> new table
std::unique_ptr<tidq_table> select_rows(Ctx* c, const uint32_t* keep, uint64_t n_rows,
                                        const std::vector<const uint32_t*>& in) {
  DevBuf offs;
  const uint64_t kept = prims::select_count(c, keep, n_rows, offs);
  auto t = make_table(c, kept, int(in.size()));
  std::vector<uint32_t*> o(in.size());
  for (size_t k = 0; k < in.size(); ++k) o[k] = t->cols[k].buf.as<uint32_t>();
  if (kept) prims::select_write(c, keep, n_rows, offs, int(in.size()), in.data(), o.data());
  return t;
}

// ---- DISTINCT by first-occurrence table -----------------------------------------
// project_distinct keeps, per distinct projected row, its FIRST occurrence
// (query_ops.py:393-398).  When the projected row packs into <= 28 bits and
// the key range is not much larger than the row count, the first occurrence
// is the minimum row index per key, recorded with atomicMin in a table
// indexed by the key; a second pass marks rows whose index is their key's
// minimum and the order-preserving compaction emits them.  Two streaming
// passes + one random access per row instead of an LSD sort of (key, row)
// pairs (C3 DISTINCT ?s UNION x4, 65 M rows: 2.2 vs 2.75 ms).  Duplicates
// inside a warp are resolved with match_any (the leader is the lowest row),
// and a plain load of the current minimum skips atomics that cannot win, so
// hot keys do not serialise on one address.  (An open-addressing table for
// wider keys measured slower than the sort: 11-13 vs 7.9 ms on 93 M rows.)
struct DistinctKeys {
  const uint32_t* hi;  // null for one column
  const uint32_t* lo;
  int lo_bits;
};

__device__ __forceinline__ uint32_t dkey(const DistinctKeys& dk, uint64_t r) {
  const uint32_t lo = __ldg(dk.lo + r);
  return dk.hi ? (__ldg(dk.hi + r) << dk.lo_bits) | lo : lo;
}

__global__ void __launch_bounds__(kT) distinct_insert_kernel(DistinctKeys dk, uint64_t n, uint32_t k_lo,
                                                             uint32_t k_hi, uint32_t* __restrict__ minrow) {
  const uint64_t base = uint64_t(blockIdx.x) * kBlk;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t r = base + j * kT + threadIdx.x;
    const bool valid = r < n;
    uint32_t k = valid ? dkey(dk, r) : 0xffffffffu;  // keys are < 2^28
    if (k < k_lo || k >= k_hi) k = 0xffffffffu;     // another pass's key range
    const uint32_t peers = __match_any_sync(0xffffffffu, k);
    if (k != 0xffffffffu && lane == __ffs(peers) - 1 && *(volatile uint32_t*)(minrow + k) > uint32_t(r))
      atomicMin(minrow + k, uint32_t(r));
  }
}

__global__ void __launch_bounds__(kT) distinct_keep_kernel(DistinctKeys dk, uint64_t n, uint32_t k_lo,
                                                           uint32_t k_hi, bool accumulate,
                                                           const uint32_t* __restrict__ minrow,
                                                           uint32_t* __restrict__ keep) {
  const uint64_t base = uint64_t(blockIdx.x) * kBlk;
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t r = base + j * kT + threadIdx.x;
    const uint32_t k = r < n ? dkey(dk, r) : 0xffffffffu;
    const bool head = k >= k_lo && k < k_hi && ld_gather(minrow + k) == uint32_t(r);
    const uint32_t w = __ballot_sync(0xffffffffu, head);
    if ((threadIdx.x & 31) == 0 && r < n + 31) keep[r >> 5] = accumulate ? keep[r >> 5] | w : w;
  }
}

// One pass per key range instead of insert + keep: the keep bitmap starts
// with every row set and each row that cannot be its key's first occurrence
// clears its bit — a lower row of the same key in its warp, a smaller
// minimum already in the table, or a smaller row returned by its atomicMin —
// and a row whose atomicMin displaced a larger minimum clears that row's bit.
// A row survives iff no smaller row of its key exists, whatever the order the
// atomics land in; the table lookup of the separate keep pass disappears.
// The loads of every row's key, of the table minima and the atomicMins are
// each issued for all of a thread's rows before any result is used (the
// chain key -> minimum -> atomic per row is latency-bound otherwise).
constexpr int kClaimI = 8;  // rows per thread
constexpr int kClaimBlk = kT * kClaimI;

template <bool kClaimMatch>
__global__ void __launch_bounds__(kT) distinct_claim_kernel(DistinctKeys dk, uint64_t n, uint32_t k_lo,
                                                            uint32_t k_hi, uint32_t* __restrict__ minrow,
                                                            uint32_t* __restrict__ keep) {
  const uint64_t base = uint64_t(blockIdx.x) * kClaimBlk;
  const int lane = threadIdx.x & 31;
  uint32_t k[kClaimI], cur[kClaimI];
  bool lead[kClaimI];
#pragma unroll
  for (int j = 0; j < kClaimI; ++j) {
    const uint64_t r = base + j * kT + threadIdx.x;  // a warp's 32 rows: one keep word
    k[j] = r < n ? dkey(dk, r) : 0xffffffffu;        // keys are < 2^28
    if (k[j] < k_lo || k[j] >= k_hi) k[j] = 0xffffffffu;  // another pass's key range
  }
  static_assert(kClaimI <= 8, "");
#pragma unroll
  for (int j = 0; j < kClaimI; ++j) {
    if (kClaimMatch) {  // lanes of one key: the lowest claims for the warp
      const uint32_t peers = __match_any_sync(0xffffffffu, k[j]);
      lead[j] = k[j] != 0xffffffffu && lane == __ffs(peers) - 1;
    } else {  // every row claims for itself (the atomics order a warp's repeats)
      lead[j] = k[j] != 0xffffffffu;
    }
  }
#pragma unroll
  for (int j = 0; j < kClaimI; ++j) cur[j] = lead[j] ? __ldcg(minrow + k[j]) : 0u;
#pragma unroll
  for (int j = 0; j < kClaimI; ++j) {
    const uint32_t r = uint32_t(base + j * kT + threadIdx.x);
    if (lead[j] && cur[j] > r) cur[j] = atomicMin(minrow + k[j], r);  // the minimum before this row's
  }
#pragma unroll
  for (int j = 0; j < kClaimI; ++j) {
    const uint32_t r = uint32_t(base + j * kT + threadIdx.x);
    // not first: a lower row of this warp has the key, or the table held a smaller row
    const bool dup = k[j] != 0xffffffffu && (!lead[j] || cur[j] < r);
    if (lead[j] && cur[j] > r && cur[j] != 0xffffffffu)
      atomicAnd(keep + (cur[j] >> 5), ~(1u << (cur[j] & 31)));  // displaced: not the first
    const uint32_t w = __ballot_sync(0xffffffffu, dup);
    if (lane == 0 && w) atomicAnd(keep + (r >> 5), ~w);
  }
}

constexpr int kDirectMaxBits = 28;  // table up to 2^28 x 4 B = 1 GiB

// Fills `keep` (row bitmap) for DISTINCT over <= 2 columns whose packed key
// is narrow; returns false when the caller must sort instead.
// `mx`: the columns' maxima (one batched max pass for both DISTINCT paths).
bool distinct_by_table(Ctx* c, const std::vector<const uint32_t*>& src, uint64_t n, const uint32_t* mx,
                       uint32_t* keep) {
  const int nc = int(src.size());
  if (nc > 2 || n == 0) return false;
  DistinctKeys dk{};
  int bits;
  if (nc == 1) {
    dk.lo = src[0];
    bits = prims::bits_for(mx[0]);
  } else {
    dk.hi = src[0];
    dk.lo = src[1];
    dk.lo_bits = std::max(1, prims::bits_for(mx[1]));
    bits = dk.lo_bits + prims::bits_for(mx[0]);
  }
  if (bits > kDirectMaxBits || (1ull << bits) > 4 * n + (1u << 20)) return false;
  phase_mark(c, "distinct.max");
  // one slot per possible key (the largest key + 1)
  const uint64_t slots = nc == 1 ? uint64_t(mx[0]) + 1 : ((uint64_t(mx[0]) + 1) << dk.lo_bits);
  DevBuf minrow(c, slots * 4);
  TIDQ_CUDA(cudaMemsetAsync(minrow.ptr, 0xff, slots * 4, c->stream));
  // Key-range passes: a table larger than the L2 takes its random atomics
  // and reads from DRAM (C3 DISTINCT ?s UNION x4: 50 M slots = 200 MB, 65 M
  // rows); passes over L2-sized key ranges re-read the (streamed) key column
  // but keep the table accesses in L2.  Measured on C3 DISTINCT ?s UNION
  // x4 / x8 with insert + keep passes: one pass 3.84 / 5.49 ms; 2 passes of
  // 100 MB 3.28 / 4.76; 3 of 67 MB 3.44 / 5.01; 5 of 40 MB 3.73 / 5.41
  // (re-reads dominate).  With one claim pass per range (ncu: a 100 MB range
  // hits L2 for only half its sectors, 1.0 GB DRAM read per pass) 3 ranges of
  // 67 MB win: 2.27 / 3.29 (2 ranges) -> 2.22 / 3.19 ms; 4-6 ranges lose.
  static const uint64_t pass_slots = [] {
    const char* e = getenv("TIDQ_DISTINCT_PASS_MB");  // (0: one pass)
    return (e ? uint64_t(atoll(e)) : uint64_t(70)) << 18;  // MB of 4-byte slots
  }();
  const uint64_t passes = pass_slots ? (slots + pass_slots - 1) / pass_slots : 1;
  const uint64_t span = (slots + passes - 1) / passes;
  static const bool claim = [] {  // A/B knob: TIDQ_DISTINCT_CLAIM=0 = insert pass + keep pass
    const char* e = getenv("TIDQ_DISTINCT_CLAIM");
    return !(e && e[0] == '0');
  }();
  if (claim) {  // every row kept until shown not to be first
    TIDQ_CUDA(cudaMemsetAsync(keep, 0xff, n / 8, c->stream));
    if (n % 8) TIDQ_CUDA(cudaMemsetAsync(reinterpret_cast<uint8_t*>(keep) + n / 8, (1 << (n % 8)) - 1, 1, c->stream));
  }
  for (uint64_t q = 0; q < passes; ++q) {
    const uint32_t lo = uint32_t(q * span), hi = uint32_t(std::min(slots, (q + 1) * span));
    if (claim) {
      // (no match_any dedup of a warp's equal keys first: the plain load of
      // the minimum already keeps later warps' atomics off hot keys, and the
      // match measured slower, x8 3.36 vs 3.29 ms)
      static const bool match = [] {  // A/B knob: TIDQ_CLAIM_MATCH=1 = warp dedup by match_any first
        const char* e = getenv("TIDQ_CLAIM_MATCH");
        return e && e[0] == '1';
      }();
      (match ? distinct_claim_kernel<true> : distinct_claim_kernel<false>)
          <<<unsigned((n + kClaimBlk - 1) / kClaimBlk), kT, 0, c->stream>>>(dk, n, lo, hi, minrow.as<uint32_t>(),
                                                                            keep);
      c->count_launch();
      continue;
    }
    distinct_insert_kernel<<<blk_grid(n), kT, 0, c->stream>>>(dk, n, lo, hi, minrow.as<uint32_t>());
    distinct_keep_kernel<<<blk_grid(n), kT, 0, c->stream>>>(dk, n, lo, hi, q > 0, minrow.as<uint32_t>(), keep);
    c->count_launch(2);
  }
  TIDQ_CUDA(cudaGetLastError());
  phase_mark(c, "distinct.direct");
  return true;
}

// ---- DISTINCT by hash partition (wide keys) ---------------------------------------
// Two projected columns packed into one 64-bit key: the key goes through a
// bijective 64-bit mix (so mixed keys are equal iff rows are equal), the
// (mixed key, row) pairs are radix-partitioned on the low `pbits` bits of the
// mix (2 passes instead of the 6-pass LSD sort of the whole 52-bit key), and
// one CTA per partition builds a shared-memory hash table mixed key -> minimum
// row and flags each key's first row (byte flags, L2-resident).  Duplicates
// share a partition, so the partition minimum is the global first
// occurrence; the order-preserving compaction follows.  A partition above the
// table capacity (one key repeated thousands of times) sends the DISTINCT to
// the sort path.  (A one-pass counting scatter — global histogram + atomic
// partition cursors — measured 2.5 ms against 1.9 ms for the two radix
// passes on 65 M rows: 65 K hot counters serialise in L2.)
constexpr int kDpSlots = 4096;           // shared table slots per partition CTA
constexpr int kDpCap = kDpSlots / 2;     // rows per partition (load factor <= 1/2)
constexpr int kDpT = 512;

__device__ __forceinline__ uint64_t mix64(uint64_t k) {  // invertible (splitmix64 finaliser)
  k = (k ^ (k >> 30)) * 0xBF58476D1CE4E5B9ull;
  k = (k ^ (k >> 27)) * 0x94D049BB133111EBull;
  return k ^ (k >> 31);
}

__global__ void __launch_bounds__(kT) dp_mix_kernel(const uint32_t* __restrict__ hi,
                                                    const uint32_t* __restrict__ lo, int lo_bits,
                                                    uint64_t n, uint64_t* __restrict__ key,
                                                    uint32_t* __restrict__ row) {
  const uint64_t base = uint64_t(blockIdx.x) * kBlk;
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t r = base + j * kT + threadIdx.x;
    if (r < n) {
      key[r] = mix64((uint64_t(__ldg(hi + r)) << lo_bits) | __ldg(lo + r));
      row[r] = uint32_t(r);
    }
  }
}

constexpr size_t kDpDedupSmem = size_t(kDpSlots) * 12;

// Partition starts from the sorted keys: row i starts every partition in
// (part(i-1), part(i)]; start[np] = n.
__global__ void __launch_bounds__(kT) dp_bounds_kernel(const uint64_t* __restrict__ key, uint64_t n,
                                                       uint64_t mask, uint32_t* __restrict__ start) {
  const uint64_t base = uint64_t(blockIdx.x) * kBlk;
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t i = base + j * kT + threadIdx.x;
    if (i > n) continue;
    const uint64_t cur = i < n ? (__ldg(key + i) & mask) : mask + 1;
    const uint64_t prev = i == 0 ? ~0ull : (__ldg(key + i - 1) & mask);
    for (uint64_t p = prev + 1; p <= cur; ++p) start[p] = uint32_t(i);  // prev = ~0: from 0
  }
}

// One CTA per partition p = [start[p], start[p+1]) of the rows sorted by
// p = key & mask.  Every thread loads its (<= kDpR) rows once, up front, and
// keeps them (key, row, slot) in registers across both phases.  The shared
// table is sized to the partition (2x its rows, a power of two); a partition
// above kDpCap rows raises *overflow and leaves its flags unset.
constexpr int kDpR = kDpCap / kDpT;  // rows per thread

// The same starts by one binary search per partition (lower bound of p in
// the sorted key & mask): np + 1 threads of ~log2(n) dependent loads whose
// upper levels are shared in L2, instead of a pass over every key
__global__ void __launch_bounds__(256) dp_starts_kernel(const uint64_t* __restrict__ key, uint64_t n,
                                                        uint64_t mask, uint64_t np, uint32_t* __restrict__ start) {
  const uint64_t p = uint64_t(blockIdx.x) * 256 + threadIdx.x;
  if (p > np) return;
  uint64_t lo = 0, hi = n;
  if (p == np) lo = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if ((__ldg(key + mid) & mask) < p)
      lo = mid + 1;
    else
      hi = mid;
  }
  start[p] = uint32_t(lo);
}

__global__ void __launch_bounds__(kDpT) dp_dedup_kernel(const uint64_t* __restrict__ key,
                                                        const uint32_t* __restrict__ row,
                                                        const uint32_t* __restrict__ start,
                                                        uint8_t* __restrict__ flag,
                                                        uint32_t* __restrict__ overflow,
                                                        uint32_t* __restrict__ keepw, int clear_dups) {
  extern __shared__ __align__(16) unsigned char dsm[];  // tkey | tmin
  unsigned long long* tkey = reinterpret_cast<unsigned long long*>(dsm);
  uint32_t* tmin = reinterpret_cast<uint32_t*>(tkey + kDpSlots);
  const uint64_t p = blockIdx.x;
  const uint64_t b0 = start[p];
  const uint64_t mrows = start[p + 1] - b0;
  if (mrows == 0) return;
  if (mrows > uint64_t(kDpCap)) {
    if (threadIdx.x == 0) atomicExch(overflow, 1u);
    return;
  }
  const uint32_t m = uint32_t(mrows);
  unsigned long long k[kDpR];
  uint32_t r[kDpR], h[kDpR];
#pragma unroll
  for (int j = 0; j < kDpR; ++j) {
    const uint32_t i = threadIdx.x + j * kDpT;
    k[j] = i < m ? __ldg(key + b0 + i) : 0ull;
    r[j] = i < m ? __ldg(row + b0 + i) : 0u;
  }
  uint32_t slots = 64;
  while (slots < 2 * m) slots <<= 1;
  // the empty marker is a value no key of this partition can take: its low
  // bit differs from the partition index's
  const unsigned long long empty = (unsigned long long)((p + 1) & 1);
  for (uint32_t i = threadIdx.x; i < slots; i += kDpT) {
    tkey[i] = empty;
    tmin[i] = 0xffffffffu;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kDpR; ++j) {
    if (threadIdx.x + j * kDpT >= m) break;
    uint32_t x = uint32_t(k[j] >> 40) & (slots - 1);  // bits above the partition bits
    while (true) {
      const unsigned long long cur = tkey[x];
      if (cur == k[j]) break;
      if (cur == empty) {
        const unsigned long long prev = atomicCAS(&tkey[x], empty, k[j]);
        if (prev == empty || prev == k[j]) break;
      }
      x = (x + 1) & (slots - 1);
    }
    h[j] = x;
    atomicMin(&tmin[x], r[j]);
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kDpR; ++j) {
    if (threadIdx.x + j * kDpT >= m) break;
    const bool first = tmin[h[j]] == r[j];
    if (keepw && clear_dups) {  // keep bitmap preset to every row: clear the repeats (few)
      if (!first) atomicAnd(keepw + (r[j] >> 5), ~(1u << (r[j] & 31)));
    } else if (first) {
      if (keepw)  // the row-order keep bitmap directly (L2-resident bits, no byte flags)
        atomicOr(keepw + (r[j] >> 5), 1u << (r[j] & 31));
      else
        flag[r[j]] = 1;
    }
  }
}

// keep word per 32 rows from byte flags
__global__ void __launch_bounds__(kT) flags_to_words_kernel(const uint8_t* __restrict__ flag, uint64_t n,
                                                            uint32_t* __restrict__ keep) {
  const uint64_t base = uint64_t(blockIdx.x) * kBlk;
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t r = base + j * kT + threadIdx.x;
    const uint32_t w = __ballot_sync(0xffffffffu, r < n && flag[r]);
    if ((threadIdx.x & 31) == 0 && r < n + 31) keep[r >> 5] = w;
  }
}

// partition sort + dedup of m (mixed key, row) pairs: flag[row] = 1 for each
// key's minimum row; false when a key repeats beyond a partition's table
bool dp_dedup_pairs(Ctx* c, DevBuf& key, DevBuf& row, uint64_t m, uint8_t* flag, uint32_t* keepw = nullptr,
                    bool clear_dups = false) {
  if (!m) return true;
  int pbits = 1;
  // <= 3/4 kDpCap rows per partition on average (Poisson tails stay far below
  // kDpCap): 93 M rows -> 16 bits, two 8-bit radix passes instead of two 9-bit
  while (pbits < 24 && (m >> pbits) > uint64_t(kDpCap) * 3 / 4) ++pbits;
  pbits = prims::radix_sorted_bits(m, pbits);  // partitions = the bits the sort groups by
  if (pbits > 26) return false;
  const uint64_t np = 1ull << pbits;
  DevBuf overflow(c, 4), start(c, (np + 1) * 4);
  prims::radix_sort_pairs(c, key.as<uint64_t>(), row.as<uint32_t>(), m, pbits);  // by the low pbits
  phase_mark(c, "distinct.partition_sort");
  ensure_dyn_smem(reinterpret_cast<const void*>(dp_dedup_kernel), c->device, int(kDpDedupSmem));
  TIDQ_CUDA(cudaMemsetAsync(overflow.ptr, 0, 4, c->stream));
  static const bool bsearch = [] {  // A/B knob: TIDQ_DP_BSEARCH=0 = the pass over every key
    const char* e = getenv("TIDQ_DP_BSEARCH");
    return !(e && e[0] == '0');
  }();
  if (bsearch)
    dp_starts_kernel<<<unsigned((np + 1 + 255) / 256), 256, 0, c->stream>>>(key.as<uint64_t>(), m, np - 1, np,
                                                                           start.as<uint32_t>());
  else
    dp_bounds_kernel<<<blk_grid(m + 1), kT, 0, c->stream>>>(key.as<uint64_t>(), m, np - 1, start.as<uint32_t>());
  dp_dedup_kernel<<<unsigned(np), kDpT, kDpDedupSmem, c->stream>>>(
      key.as<uint64_t>(), row.as<uint32_t>(), start.as<uint32_t>(), flag, overflow.as<uint32_t>(), keepw,
      int(clear_dups));
  c->count_launch(2);
  uint32_t* h = static_cast<uint32_t*>(c->pinned_small);
  TIDQ_CUDA(cudaMemcpyAsync(h, overflow.ptr, 4, cudaMemcpyDeviceToHost, c->stream));
  TIDQ_CUDA(cudaStreamSynchronize(c->stream));
  return h[0] == 0;  // else a key repeated more often than a partition table holds: sort instead
}

// (A candidate filter in front — every pair hashed into an L2-resident bit
// table with atomicOr, only rows whose slot was hit twice partitioned —
// measured slower on C3 DISTINCT ?s ?o UNION x8: 7.09 vs 6.70 ms; 93 M
// returning atomics took 1.4 ms and the candidates' append 2.2 ms.)
bool distinct_by_partition(Ctx* c, const std::vector<const uint32_t*>& src, uint64_t n, uint32_t* keep) {
  if (src.size() != 2 || n < (1u << 16) || n >= (1ull << 32)) return false;
  DevBuf key(c, n * 8), row(c, n * 4);
  // (hi << 32) | lo: unique for any two 32-bit values, so no max pass is needed
  dp_mix_kernel<<<blk_grid(n), kT, 0, c->stream>>>(src[0], src[1], 32, n, key.as<uint64_t>(), row.as<uint32_t>());
  c->count_launch();
  const char* kb_env = getenv("TIDQ_DP_KEEPBITS");  // A/B knob: 0 = byte flags + flags_to_words
  if (!(kb_env && kb_env[0] == '0')) {
    // first occurrences set their bits in the (zeroed) keep bitmap directly,
    // or (default) every row's bit is preset and the repeats clear theirs:
    // distinct pairs are the common case, so far fewer atomics
    const char* cd_env = getenv("TIDQ_DP_CLEARDUPS");  // A/B knob: 0 = set the first occurrences
    const bool clear_dups = !(cd_env && cd_env[0] == '0');
    if (clear_dups) {
      TIDQ_CUDA(cudaMemsetAsync(keep, 0xff, n / 8, c->stream));
      if (n % 8) TIDQ_CUDA(cudaMemsetAsync(reinterpret_cast<uint8_t*>(keep) + n / 8, (1 << (n % 8)) - 1, 1, c->stream));
    }
    if (!dp_dedup_pairs(c, key, row, n, nullptr, keep, clear_dups)) {
      const size_t keep_b = ((n + kBlk - 1) / kBlk) * kBlk / 8 + 4;
      TIDQ_CUDA(cudaMemsetAsync(keep, 0, keep_b, c->stream));  // the sort path rebuilds it
      return false;
    }
    phase_mark(c, "distinct.partition_dedup");
    return true;
  }
  DevBuf flag(c, n);
  TIDQ_CUDA(cudaMemsetAsync(flag.ptr, 0, n, c->stream));
  if (!dp_dedup_pairs(c, key, row, n, flag.as<uint8_t>())) return false;
  flags_to_words_kernel<<<blk_grid(n), kT, 0, c->stream>>>(flag.as<uint8_t>(), n, keep);
  c->count_launch();
  TIDQ_CUDA(cudaGetLastError());
  phase_mark(c, "distinct.partition_dedup");
  return true;
}

}  // namespace
}  // namespace tidq

using namespace tidq;

extern "C" {

int tidq_table_concat(tidq_ctx* ctx, int32_t n_tables, tidq_table* const* tables,
                      int32_t n_out_cols, const int32_t* src_cols, tidq_table** out) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx && out && n_tables >= 0 && n_out_cols >= 0, TIDQ_E_INVALID, "bad argument");
    TIDQ_REQUIRE(n_tables == 0 || (tables && (src_cols || n_out_cols == 0)), TIDQ_E_INVALID,
                 "null tables");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx);
    uint64_t n = 0;
    for (int i = 0; i < n_tables; ++i) n += tables[i]->n_rows();
    auto t = make_table(ctx, n, n_out_cols);
    for (int k = 0; k < n_out_cols; ++k) {
      uint64_t at = 0;
      char* dst = t->cols[k].buf.as<char>();
      for (int i = 0; i < n_tables; ++i) {
        const uint64_t m = tables[i]->n_rows();
        if (!m) continue;
        const int src = src_cols[size_t(i) * n_out_cols + k];
        if (src < 0) {
          TIDQ_CUDA(cudaMemsetAsync(dst + at * 4, 0, m * 4, ctx->stream));  // UNBOUND
        } else {
          TIDQ_CUDA(cudaMemcpyAsync(dst + at * 4, col_u32(tables[i], src), m * 4,
                                    cudaMemcpyDeviceToDevice, ctx->stream));
        }
        at += m;
      }
    }
    TIDQ_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = t.release();
  });
}

int tidq_table_project(tidq_table* tb, int32_t n_cols, const int32_t* cols, tidq_table** out) {
  return guarded([&] {
    TIDQ_REQUIRE(tb && out && n_cols >= 0 && (cols || !n_cols), TIDQ_E_INVALID, "bad argument");
    Ctx* c = tb->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    auto t = make_table(c, tb->n_rows(), n_cols);
    for (int k = 0; k < n_cols; ++k)
      if (tb->n_rows())
        TIDQ_CUDA(cudaMemcpyAsync(t->cols[k].buf.ptr, col_u32(tb, cols[k]), tb->n_rows() * 4,
                                  cudaMemcpyDeviceToDevice, c->stream));
    // stream-ordered: the table's row count is known, nothing to wait for
    *out = t.release();
  });
}

int tidq_table_filter_bitmap(tidq_table* tb, int32_t col, const tidq_bitmap* bm, tidq_table** out) {
  return guarded([&] {
    TIDQ_REQUIRE(tb && bm && out, TIDQ_E_INVALID, "null argument");
    Ctx* c = tb->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    const uint64_t n = tb->n_rows();
    const int nc = int(tb->cols.size());
    const uint32_t* key = col_u32(tb, col);
    DevBuf keep(c, ((n + kBlk - 1) / kBlk) * kBlk / 8 + 4);
    if (n) {
      pdl_chain_launch(bitmap_keep_kernel, blk_grid(n), kT, 0, c->stream, key, n, bm->words.as<uint32_t>(), bm->n_bits,
                                                              keep.as<uint32_t>(), (uint32_t*)nullptr);
      c->count_launch();
    }
    std::vector<const uint32_t*> in(nc);
    for (int k = 0; k < nc; ++k) in[k] = col_u32(tb, k);
    auto t = select_rows(c, keep.as<uint32_t>(), n, in);
    // stream-ordered: the table's row count is known, nothing to wait for
    *out = t.release();
  });
}

int tidq_table_unique_col(tidq_table* tb, int32_t col, tidq_table** out) {
  return guarded([&] {
    TIDQ_REQUIRE(tb && out, TIDQ_E_INVALID, "null argument");
    Ctx* c = tb->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    const uint64_t n = tb->n_rows();
    DevBuf keys, ids;
    sort_column(c, col_u32(tb, col), n, n ? prims::max_u32(c, col_u32(tb, col), n) : 0u, keys, ids);
    DevBuf keep(c, ((n + kBlk - 1) / kBlk) * kBlk / 8 + 4);
    if (n) {
      sorted_heads_kernel<uint32_t><<<blk_grid(n), kT, 0, c->stream>>>(keys.as<uint32_t>(), n,
                                                                       keep.as<uint32_t>());
      c->count_launch();
    }
    auto t = select_rows(c, keep.as<uint32_t>(), n, {keys.as<uint32_t>()});
    // stream-ordered: the table's row count is known, nothing to wait for
    *out = t.release();
  });
}

// DISTINCT over `cols`: stable LSD sort of row ids by the projected columns
// (two columns per 64-bit radix key holding only their significant bits, last
// columns first); run heads mark their ORIGINAL row in a row bitmap; an
// order-preserving bitmap selection then yields exactly the reference's
// first-occurrence order (query_ops.py:393-398).
int tidq_distinct(tidq_table* tb, int32_t n_cols, const int32_t* cols, tidq_table** out) {
  return tidq_distinct_bound(tb, n_cols, cols, 0, out);
}

int tidq_distinct_bound(tidq_table* tb, int32_t n_cols, const int32_t* cols, uint64_t key_bound,
                        tidq_table** out) {
  return guarded([&] {
    TIDQ_REQUIRE(tb && out && n_cols >= 1 && cols, TIDQ_E_INVALID, "distinct needs columns");
    Ctx* c = tb->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    const uint64_t n = tb->n_rows();
    TIDQ_REQUIRE(n < (1ull << 32), TIDQ_E_INVALID, "distinct input above 2^32 rows");
    cudaEvent_t ev = c->prof_begin(c->stream);
    std::vector<const uint32_t*> src(n_cols);
    for (int k = 0; k < n_cols; ++k) src[k] = col_u32(tb, cols[k]);
    const size_t keep_b = ((n + kBlk - 1) / kBlk) * kBlk / 8 + 4;
    DevBuf keep(c, keep_b);
    TIDQ_CUDA(cudaMemsetAsync(keep.ptr, 0, keep_b, c->stream));
    phase_mark(c, nullptr);
    uint32_t mx[2] = {0, 0};
    if (n && n_cols <= 2 && key_bound) {  // the caller's bound (e.g. the store's largest ID + 1): no max pass
      mx[0] = mx[1] = uint32_t(std::min<uint64_t>(key_bound - 1, 0xffffffffull));
    } else if (n && n_cols <= 2) {
      const uint64_t ns[2] = {n, n};
      prims::max_u32_multi(c, n_cols, src.data(), ns, mx);
    }
    if (n && n_cols <= 2 && (distinct_by_table(c, src, n, mx, keep.as<uint32_t>()) ||
                             distinct_by_partition(c, src, n, keep.as<uint32_t>()))) {
      // keep bitmap filled by the first-occurrence table / hash partitions
    } else if (n) {
      DevBuf perm(c, n * 4), k64, k32;
      prims::iota(c, perm.as<uint32_t>(), n);
      int j = n_cols - 1;
      bool first = true;
      int last_kind = 0;  // 1: sorted k32, 2: sorted k64
      while (j >= 0) {
        if (j >= 1) {
          if (!k64.ptr) k64 = DevBuf(c, n * 8);
          const uint32_t mx_hi = prims::max_u32(c, src[j - 1], n);
          const int lo_bits = std::max(1, prims::bits_for(prims::max_u32(c, src[j], n)));
          // (hi << lo_bits) | lo orders pairs like (hi, lo): only the significant bits are sorted
          pack2_kernel<<<blk_grid(n), kT, 0, c->stream>>>(src[j - 1], src[j],
                                                           first ? nullptr : perm.as<uint32_t>(), n,
                                                           lo_bits, k64.as<uint64_t>());
          c->count_launch();
          phase_mark(c, "distinct.pack");
          prims::radix_sort_pairs(c, k64.as<uint64_t>(), perm.as<uint32_t>(), n,
                                  lo_bits + prims::bits_for(mx_hi));
          phase_mark(c, "distinct.sort64");
          j -= 2;
          last_kind = 2;
        } else {
          if (!k32.ptr) k32 = DevBuf(c, n * 4);
          const uint32_t mx = prims::max_u32(c, src[0], n);
          if (first) {
            TIDQ_CUDA(cudaMemcpyAsync(k32.ptr, src[0], n * 4, cudaMemcpyDeviceToDevice, c->stream));
          } else {
            prims::gather_u32(c, src[0], perm.as<uint32_t>(), k32.as<uint32_t>(), n);
          }
          phase_mark(c, "distinct.prep32");
          prims::radix_sort_pairs(c, k32.as<uint32_t>(), perm.as<uint32_t>(), n, prims::bits_for(mx));
          phase_mark(c, "distinct.sort32");
          j -= 1;
          last_kind = 1;
        }
        first = false;
      }
      if (n_cols <= 2) {  // the last sort key holds the whole row: compare adjacent keys
        if (last_kind == 2)
          head_rows_kernel<uint64_t><<<blk_grid(n), kT, 0, c->stream>>>(k64.as<uint64_t>(),
                                                                         perm.as<uint32_t>(), n,
                                                                         keep.as<uint32_t>());
        else
          head_rows_kernel<uint32_t><<<blk_grid(n), kT, 0, c->stream>>>(k32.as<uint32_t>(),
                                                                         perm.as<uint32_t>(), n,
                                                                         keep.as<uint32_t>());
      } else {
        // a row heads a run when it differs from its predecessor in ANY
        // column: the flags of 8-column batches are OR-ed into one bitmap
        for (int lo = 0; lo < n_cols; lo += 8) {
          RowCols rc{};
          const int nb = std::min(8, n_cols - lo);
          for (int k = 0; k < nb; ++k) rc.c[k] = src[lo + k];
          head_rows_cols_kernel<<<blk_grid(n), kT, 0, c->stream>>>(perm.as<uint32_t>(), n, nb, rc,
                                                                   keep.as<uint32_t>());
          if (lo + 8 < n_cols) c->count_launch();
        }
      }
      c->count_launch();
      TIDQ_CUDA(cudaGetLastError());
    }
    phase_mark(c, "distinct.heads");
    auto t = select_rows(c, keep.as<uint32_t>(), n, src);
    // stream-ordered: the table's row count is known, nothing to wait for
    phase_mark(c, "distinct.select");
    phase_report("tidq_distinct");
    // SURVEY 8(d) DISTINCT bytes: w*M + w*U (w = projected row bytes)
    c->prof_end("distinct", ev, c->stream, 4ull * n_cols * (n + t->n_rows()));
    *out = t.release();
  });
}

int tidq_join(tidq_table* left, int32_t lkey, tidq_table* right, int32_t rkey, int32_t n_out,
              const tidq_colref* out_cols, int32_t n_eq, const int32_t* eq_pairs, int64_t row_cap,
              int32_t algo, uint64_t key_bound, const tidq_bitmap* lkeys_bm, const tidq_bitmap* rkeys_bm,
              tidq_table** out, uint64_t* n_pairs) {
  return guarded([&] {
    TIDQ_REQUIRE(left && right && out && left->ctx == right->ctx, TIDQ_E_INVALID, "bad tables");
    TIDQ_REQUIRE(n_out >= 0 && (out_cols || !n_out), TIDQ_E_INVALID, "bad outputs");
    TIDQ_REQUIRE(n_eq >= 0 && n_eq <= 4 && (eq_pairs || !n_eq), TIDQ_E_INVALID, "bad eq pairs");
    Ctx* c = left->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    cudaEvent_t ev = c->prof_begin(c->stream);
    JoinPlan jp;
    // a side with exactly one non-key output column (and no equality pairs)
    // carries that column's values through the semi-join and sort in place
    // of its row ids: the expansion then writes it from the sorted pairs
    // instead of a random gather per output row
    int lpc = -1, rpc = -1;
    bool lmany = false, rmany = false;
    const char* cv_env = getenv("TIDQ_JOIN_CARRY");  // A/B knob (0: gather by row id)
    const bool carry_ok = n_eq == 0 && !(cv_env && cv_env[0] == '0');
    for (int k = 0; k < n_out && carry_ok; ++k) {
      const int side = out_cols[k].side, col = out_cols[k].col;
      if (col == (side ? rkey : lkey)) continue;
      int& pc = side ? rpc : lpc;
      bool& many = side ? rmany : lmany;
      if (pc >= 0 && pc != col) many = true;
      pc = col;
    }
    const uint32_t* lcarry = carry_ok && lpc >= 0 && !lmany ? col_u32(left, lpc) : nullptr;
    const uint32_t* rcarry = carry_ok && rpc >= 0 && !rmany ? col_u32(right, rpc) : nullptr;
    join_prepare(c, col_u32(left, lkey), left->n_rows(), col_u32(right, rkey), right->n_rows(), jp,
                 (algo & TIDQ_JOIN_REDUCED) != 0, key_bound, lkeys_bm, rkeys_bm, left->sorted_by == lkey,
                 right->sorted_by == rkey, lcarry, rcarry);
    if (n_pairs) *n_pairs = jp.total;
    if (row_cap >= 0 && jp.total > uint64_t(row_cap))
      throw Error(TIDQ_E_ROW_CAP, "join produced " + std::to_string(jp.total) +
                                      " rows, cap is " + std::to_string(row_cap));
    auto t = make_table(c, jp.total, n_out);
    DevBuf keep;
    if (n_eq) keep = DevBuf(c, ((jp.total + kBlk - 1) / kBlk) * kBlk / 8 + 4);
    phase_mark(c, "alloc_out");
    // the expansion writes up to 8 output columns per launch; the equality
    // keep bitmap comes from the first launch (a launch without outputs when
    // the join has none)
    for (int lo = 0; lo == 0 || lo < n_out; lo += 8) {
      JoinOut jo{};
      jo.n_out = std::min(8, n_out - lo);
      for (int k = 0; k < jo.n_out; ++k) {
        jo.side[k] = out_cols[lo + k].side;
        jo.src[k] = col_u32(out_cols[lo + k].side ? right : left, out_cols[lo + k].col);
        jo.dst[k] = t->cols[lo + k].buf.as<uint32_t>();
        if (out_cols[lo + k].col == (out_cols[lo + k].side ? rkey : lkey)) jo.key_mask |= 1u << k;
        else if (out_cols[lo + k].side ? jp.rcarry : jp.lcarry) jo.direct_mask |= 1u << k;
      }
      jo.n_eq = lo == 0 ? n_eq : 0;
      for (int e = 0; e < jo.n_eq; ++e) {
        jo.eq_l[e] = col_u32(left, eq_pairs[2 * e]);
        jo.eq_r[e] = col_u32(right, eq_pairs[2 * e + 1]);
      }
      join_expand(c, jp, jo, lo == 0 && n_eq ? keep.as<uint32_t>() : nullptr);
    }
    phase_mark(c, "expand");
    if (n_eq && jp.total) {
      std::vector<const uint32_t*> in(n_out);
      for (int k = 0; k < n_out; ++k) in[k] = t->cols[k].buf.as<uint32_t>();
      t = select_rows(c, keep.as<uint32_t>(), jp.total, in);
    }
    // rows come out in key order (key asc, left row asc, right row asc)
    for (int k = 0; k < n_out && t->sorted_by < 0; ++k)
      if (out_cols[k].col == (out_cols[k].side ? rkey : lkey)) t->sorted_by = k;
    // stream-ordered: the table's row count is known, nothing to wait for
    phase_mark(c, "eq_select");
    phase_report("tidq_join");
    // SURVEY 8(d) join bytes: both sides' rows (build + probe) + the output rows
    c->prof_end("join", ev, c->stream,
                4ull * (left->cols.size() * left->n_rows() + right->cols.size() * right->n_rows() +
                        uint64_t(n_out) * t->n_rows()));
    *out = t.release();
  });
}

int tidq_tables_semijoin(int32_t n_tables, tidq_table* const* tables, const int32_t* key_cols,
                         uint64_t n_bits, tidq_table** out) {
  return guarded([&] {
    TIDQ_REQUIRE(n_tables >= 2 && n_tables <= 32 && tables && key_cols && out, TIDQ_E_INVALID,
                 "semijoin needs 2..32 tables");
    Ctx* c = tables[0]->ctx;
    for (int i = 0; i < n_tables; ++i)
      TIDQ_REQUIRE(tables[i] && tables[i]->ctx == c, TIDQ_E_INVALID, "tables on different contexts");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    std::vector<const uint32_t*> keys(n_tables);
    std::vector<uint64_t> ns(n_tables);
    for (int i = 0; i < n_tables; ++i) {
      keys[i] = col_u32(tables[i], key_cols[i]);
      ns[i] = tables[i]->n_rows();
    }
    uint64_t nbits = n_bits;
    if (nbits == 0) {
      uint32_t mx = 0;
      for (int lo = 0; lo < n_tables; lo += 8) {  // batched maxima, one sync per 8 columns
        uint32_t m[8];
        const int k = std::min(8, n_tables - lo);
        prims::max_u32_multi(c, k, keys.data() + lo, ns.data() + lo, m);
        for (int i = 0; i < k; ++i) mx = std::max(mx, m[i]);
      }
      nbits = uint64_t(mx) + 1;
    }
    TIDQ_REQUIRE(nbits <= (1ull << 32), TIDQ_E_INVALID, "n_bits above 2^32");
    const uint64_t words = (nbits + 31) / 32;
    // bitmap i: the keys of table i
    std::vector<DevBuf> bm(n_tables);
    for (int i = 0; i < n_tables; ++i) {
      bm[i] = DevBuf(c, words * 4);
      TIDQ_CUDA(cudaMemsetAsync(bm[i].ptr, 0, words * 4, c->stream));
      if (ns[i]) {
        pdl_chain_launch(key_bitmap_kernel, blk_grid(ns[i]), kT, 0, c->stream, keys[i], ns[i], bm[i].as<uint32_t>());
        c->count_launch();
      }
    }
    for (int i = 0; i < n_tables; ++i)
      for (const auto& col : tables[i]->cols)
        TIDQ_REQUIRE(col.dtype == TIDQ_U32, TIDQ_E_INVALID, "semijoin tables must be uint32");
    // AND of the other tables' bitmaps, per table (n >= 3: prefix/suffix ANDs)
    std::vector<DevBuf> keep(n_tables), offs(n_tables);
    for (int i = 0; i < n_tables; ++i) {
      DevBuf andm;
      const uint32_t* test = nullptr;
      if (n_tables == 2) {
        test = bm[1 - i].as<uint32_t>();
      } else {
        andm = DevBuf(c, words * 4);
        bool first = true;
        for (int j = 0; j < n_tables; ++j) {
          if (j == i) continue;
          pdl_chain_launch(bitmap_and_kernel, unsigned((words + 1023) / 1024), 256, 0, c->stream, 
              first ? nullptr : andm.as<uint32_t>(), bm[j].as<uint32_t>(), words, andm.as<uint32_t>());
          first = false;
        }
        c->count_launch(n_tables - 1);
        test = andm.as<uint32_t>();
      }
      keep[i] = DevBuf(c, ((ns[i] + kBlk - 1) / kBlk) * kBlk / 8 + 4);
      if (ns[i]) {
        pdl_chain_launch(bitmap_keep_kernel, blk_grid(ns[i]), kT, 0, c->stream, keys[i], ns[i], test, nbits,
                                                                   keep[i].as<uint32_t>(), (uint32_t*)nullptr);
        c->count_launch();
      }
      prims::select_count_async(c, keep[i].as<uint32_t>(), ns[i], offs[i]);
    }
    // every table's kept count in ONE host round trip, then the compactions
    uint64_t* h = static_cast<uint64_t*>(c->pinned_small);
    for (int i = 0; i < n_tables; ++i)
      TIDQ_CUDA(cudaMemcpyAsync(h + i, offs[i].as<uint64_t>() + (ns[i] + 1023) / 1024, 8,
                                cudaMemcpyDeviceToHost, c->stream));
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    std::vector<uint64_t> kept(h, h + n_tables);
    for (int i = 0; i < n_tables; ++i) {
      std::vector<const uint32_t*> in(tables[i]->cols.size());
      for (size_t k = 0; k < in.size(); ++k) in[k] = tables[i]->cols[k].buf.as<uint32_t>();
      auto t = make_table(c, kept[i], int(in.size()));
      std::vector<uint32_t*> o(in.size());
      for (size_t k = 0; k < in.size(); ++k) o[k] = t->cols[k].buf.as<uint32_t>();
      if (kept[i]) prims::select_write(c, keep[i].as<uint32_t>(), ns[i], offs[i], int(in.size()), in.data(), o.data());
      out[i] = t.release();
    }
    // stream-ordered: the table's row count is known, nothing to wait for
  });
}

// BindingRelation.prepare_for_join (query_ops.py:110-118): np.argsort(key,
// kind="stable") -> the device's stable LSD radix sort carrying row ids.
int tidq_argsort_u32(tidq_ctx* ctx, const uint32_t* keys, uint64_t n, uint32_t* sorted_out,
                     uint32_t* perm_out) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx && (keys || !n) && (sorted_out || !n) && (perm_out || !n), TIDQ_E_INVALID,
                 "null argument");
    TIDQ_REQUIRE(n < (1ull << 32), TIDQ_E_INVALID, "argsort input above 2^32 keys");
    if (!n) return;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx);
    DevBuf in(ctx, n * 4), k, ids;
    TIDQ_CUDA(cudaMemcpyAsync(in.ptr, keys, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    const uint32_t mx = prims::max_u32(ctx, in.as<uint32_t>(), n);
    sort_column(ctx, in.as<uint32_t>(), n, mx, k, ids);
    TIDQ_CUDA(cudaMemcpyAsync(sorted_out, k.ptr, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    TIDQ_CUDA(cudaMemcpyAsync(perm_out, ids.ptr, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    TIDQ_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int tidq_debug_radix_sort(tidq_ctx* ctx, int32_t key_bytes, void* keys, uint32_t* vals, uint64_t n,
                          int32_t bits, int32_t reps, double* ms_per_sort) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx && (keys || !n) && (vals || !n), TIDQ_E_INVALID, "null argument");
    TIDQ_REQUIRE(key_bytes == 4 || key_bytes == 8, TIDQ_E_INVALID, "key_bytes must be 4 or 8");
    TIDQ_REQUIRE(bits >= 0 && bits <= 8 * key_bytes, TIDQ_E_INVALID, "bits out of range");
    TIDQ_REQUIRE(n < (1ull << 32), TIDQ_E_INVALID, "radix sort above 2^32 keys");
    if (ms_per_sort) *ms_per_sort = 0;
    if (!n) return;
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx);
    const size_t kb = n * size_t(key_bytes), vb = n * 4;
    DevBuf k0(ctx, kb), v0(ctx, vb), k(ctx, kb), v(ctx, vb);
    TIDQ_CUDA(cudaMemcpyAsync(k0.ptr, keys, kb, cudaMemcpyHostToDevice, ctx->stream));
    TIDQ_CUDA(cudaMemcpyAsync(v0.ptr, vals, vb, cudaMemcpyHostToDevice, ctx->stream));
    auto run = [&] {
      if (key_bytes == 4)
        prims::radix_sort_pairs(ctx, k.as<uint32_t>(), v.as<uint32_t>(), n, bits);
      else
        prims::radix_sort_pairs(ctx, k.as<uint64_t>(), v.as<uint32_t>(), n, bits);
    };
    cudaEvent_t ev[2];
    TIDQ_CUDA(cudaEventCreate(&ev[0]));
    TIDQ_CUDA(cudaEventCreate(&ev[1]));
    double total = 0;
    for (int r = reps > 0 ? -1 : 0; r < std::max(reps, 1); ++r) {  // r = -1: untimed warm-up
      TIDQ_CUDA(cudaMemcpyAsync(k.ptr, k0.ptr, kb, cudaMemcpyDeviceToDevice, ctx->stream));
      TIDQ_CUDA(cudaMemcpyAsync(v.ptr, v0.ptr, vb, cudaMemcpyDeviceToDevice, ctx->stream));
      TIDQ_CUDA(cudaEventRecord(ev[0], ctx->stream));
      run();
      TIDQ_CUDA(cudaEventRecord(ev[1], ctx->stream));
      TIDQ_CUDA(cudaEventSynchronize(ev[1]));
      float ms = 0;
      TIDQ_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
      if (r >= 0) total += ms;
    }
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    if (ms_per_sort && reps > 0) *ms_per_sort = total / reps;
    TIDQ_CUDA(cudaMemcpyAsync(keys, k.ptr, kb, cudaMemcpyDeviceToHost, ctx->stream));
    TIDQ_CUDA(cudaMemcpyAsync(vals, v.ptr, vb, cudaMemcpyDeviceToHost, ctx->stream));
    TIDQ_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int tidq_merge_join_pairs(tidq_ctx* ctx, const uint32_t* lkeys, uint64_t nl, const uint32_t* rkeys,
                          uint64_t nr, tidq_table** out) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx && out && (lkeys || !nl) && (rkeys || !nr), TIDQ_E_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx);
    DevBuf l(ctx, std::max<uint64_t>(nl, 1) * 4), r(ctx, std::max<uint64_t>(nr, 1) * 4);
    if (nl) TIDQ_CUDA(cudaMemcpyAsync(l.ptr, lkeys, nl * 4, cudaMemcpyHostToDevice, ctx->stream));
    if (nr) TIDQ_CUDA(cudaMemcpyAsync(r.ptr, rkeys, nr * 4, cudaMemcpyHostToDevice, ctx->stream));
    JoinPlan jp;
    join_prepare(ctx, l.as<uint32_t>(), nl, r.as<uint32_t>(), nr, jp);
    auto t = make_table(ctx, jp.total, 2, TIDQ_I64);
    JoinOut jo{};
    jo.pair_l = t->cols[0].buf.as<int64_t>();
    jo.pair_r = t->cols[1].buf.as<int64_t>();
    join_expand(ctx, jp, jo, nullptr);
    TIDQ_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = t.release();
  });
}

}  // extern "C"
