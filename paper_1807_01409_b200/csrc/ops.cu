// Table operators of the query path (reference query_ops.py):
//   UNION concat with UNBOUND = 0            query_ops.py:359-376
//   FILTER by accepted-ID bitmap             query_ops.py:241-252
//   DISTINCT, first occurrence kept          query_ops.py:379-399
//   equi-join step of join_group             query_ops.py:144-177, 316-341
// All device-side; the host only sequences calls and reads counts.
#include <cuda_runtime.h>

#include <algorithm>
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
  t->n_rows = n;
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

__global__ void bitmap_flags_kernel(const uint32_t* __restrict__ col, uint64_t n,
                                    const uint32_t* __restrict__ words, uint64_t nbits,
                                    uint32_t* __restrict__ flags) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t id = col[i];
    flags[i] = (uint64_t(id) < nbits && ((__ldg(words + (id >> 5)) >> (id & 31)) & 1u)) ? 1u : 0u;
  }
}

// flags[i] = 1 iff sorted row i differs from row i-1 (rows compared through perm)
struct RowCols {
  const uint32_t* c[8];
};

__global__ void head_flags_kernel(const uint32_t* __restrict__ perm, uint64_t n, int n_cols,
                                  RowCols rc, uint32_t* __restrict__ keep_by_row) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t r = perm[i];
    bool head = i == 0;
    if (!head) {
      const uint32_t q = perm[i - 1];
      for (int k = 0; k < n_cols && !head; ++k) head = rc.c[k][r] != rc.c[k][q];
    }
    keep_by_row[r] = head ? 1u : 0u;
  }
}

__global__ void pack2_kernel(const uint32_t* __restrict__ hi, const uint32_t* __restrict__ lo,
                             const uint32_t* __restrict__ perm, uint64_t n, int shift,
                             uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t r = perm ? perm[i] : uint32_t(i);
    out[i] = (uint64_t(hi[r]) << shift) | uint64_t(lo[r]);
  }
}

__global__ void adjacent_unique_flags_kernel(const uint32_t* __restrict__ keys, uint64_t n,
                                             uint32_t* __restrict__ flags) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

// equal_range of every sorted left key in the sorted right keys
__global__ void equal_range_kernel(const uint32_t* __restrict__ ls, uint64_t nl,
                                   const uint32_t* __restrict__ rs, uint64_t nr,
                                   uint64_t* __restrict__ start, uint64_t* __restrict__ cnt) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nl;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t k = ls[i];
    uint64_t lo = 0, hi = nr;
    while (lo < hi) {
      const uint64_t m = (lo + hi) >> 1;
      if (rs[m] < k) lo = m + 1; else hi = m;
    }
    const uint64_t a = lo;
    hi = nr;
    while (lo < hi) {
      const uint64_t m = (lo + hi) >> 1;
      if (rs[m] <= k) lo = m + 1; else hi = m;
    }
    start[i] = a;
    cnt[i] = lo - a;
  }
}

struct JoinOut {
  int n_out;
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
// offs[i] <= p < offs[i+1] (binary search), and to right row
// ro[start[i] + p - offs[i]].  Output order = (key, left row, right row).
__global__ void expand_kernel(const uint64_t* __restrict__ offs, uint64_t nl,
                              const uint64_t* __restrict__ start, const uint32_t* __restrict__ lo,
                              const uint32_t* __restrict__ ro, uint64_t total, JoinOut jo,
                              uint32_t* __restrict__ keep) {
  for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < total;
       p += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t a = 0, b = nl;  // last i with offs[i] <= p
    while (b - a > 1) {
      const uint64_t m = (a + b) >> 1;
      if (offs[m] <= p) a = m; else b = m;
    }
    const uint32_t l = lo[a];
    const uint32_t r = ro[start[a] + (p - offs[a])];
    for (int k = 0; k < jo.n_out; ++k) jo.dst[k][p] = jo.src[k][jo.side[k] ? r : l];
    if (jo.pair_l) {
      jo.pair_l[p] = l;
      jo.pair_r[p] = r;
    }
    if (keep) {
      bool ok = true;
      for (int e = 0; e < jo.n_eq; ++e) ok = ok && jo.eq_l[e][l] == jo.eq_r[e][r];
      keep[p] = ok ? 1u : 0u;
    }
  }
}

// Sort a key column stably, carrying row ids: out keys sorted, out ids = perm.
void sort_column(Ctx* c, const uint32_t* col, uint64_t n, DevBuf& keys, DevBuf& ids) {
  keys = DevBuf(c, std::max<uint64_t>(n, 1) * 4);
  ids = DevBuf(c, std::max<uint64_t>(n, 1) * 4);
  if (!n) return;
  TIDQ_CUDA(cudaMemcpyAsync(keys.ptr, col, n * 4, cudaMemcpyDeviceToDevice, c->stream));
  prims::iota(c, ids.as<uint32_t>(), n);
  const uint32_t mx = prims::max_u32(c, col, n);
  prims::radix_sort_pairs(c, keys.as<uint32_t>(), ids.as<uint32_t>(), n, prims::bits_for(mx));
}

// Sort-merge join core.  Returns the pair count (before the equality mask).
// Fills `jo` outputs when `write`; `keep` (if non-null) gets eq flags.
struct JoinPlan {
  DevBuf ls, lo, rs, ro, start, cnt, offs;
  uint64_t nl = 0, total = 0;
};

void join_prepare(Ctx* c, const uint32_t* lkey, uint64_t nl, const uint32_t* rkey, uint64_t nr,
                  JoinPlan& jp) {
  jp.nl = nl;
  sort_column(c, lkey, nl, jp.ls, jp.lo);
  sort_column(c, rkey, nr, jp.rs, jp.ro);
  jp.start = DevBuf(c, std::max<uint64_t>(nl, 1) * 8);
  jp.cnt = DevBuf(c, std::max<uint64_t>(nl, 1) * 8);
  jp.offs = DevBuf(c, (nl + 1) * 8);
  if (nl == 0 || nr == 0) {
    jp.total = 0;
    return;
  }
  equal_range_kernel<<<grid_for(c, nl, 256), 256, 0, c->stream>>>(
      jp.ls.as<uint32_t>(), nl, jp.rs.as<uint32_t>(), nr, jp.start.as<uint64_t>(),
      jp.cnt.as<uint64_t>());
  c->count_launch();
  TIDQ_CUDA(cudaGetLastError());
  jp.total = prims::exclusive_scan(c, jp.cnt.as<uint64_t>(), jp.offs.as<uint64_t>(), nl);
}

void join_expand(Ctx* c, JoinPlan& jp, JoinOut& jo, uint32_t* keep) {
  if (!jp.total) return;
  expand_kernel<<<grid_for(c, jp.total, 256, 16), 256, 0, c->stream>>>(
      jp.offs.as<uint64_t>(), jp.nl, jp.start.as<uint64_t>(), jp.lo.as<uint32_t>(),
      jp.ro.as<uint32_t>(), jp.total, jo, keep);
  c->count_launch();
  TIDQ_CUDA(cudaGetLastError());
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
    for (int i = 0; i < n_tables; ++i) n += tables[i]->n_rows;
    auto t = make_table(ctx, n, n_out_cols);
    for (int k = 0; k < n_out_cols; ++k) {
      uint64_t at = 0;
      char* dst = t->cols[k].buf.as<char>();
      for (int i = 0; i < n_tables; ++i) {
        const uint64_t m = tables[i]->n_rows;
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
    auto t = make_table(c, tb->n_rows, n_cols);
    for (int k = 0; k < n_cols; ++k)
      if (tb->n_rows)
        TIDQ_CUDA(cudaMemcpyAsync(t->cols[k].buf.ptr, col_u32(tb, cols[k]), tb->n_rows * 4,
                                  cudaMemcpyDeviceToDevice, c->stream));
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    *out = t.release();
  });
}

int tidq_table_filter_bitmap(tidq_table* tb, int32_t col, const tidq_bitmap* bm, tidq_table** out) {
  return guarded([&] {
    TIDQ_REQUIRE(tb && bm && out, TIDQ_E_INVALID, "null argument");
    Ctx* c = tb->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    const uint64_t n = tb->n_rows;
    const int nc = int(tb->cols.size());
    const uint32_t* key = col_u32(tb, col);
    DevBuf flags(c, std::max<uint64_t>(n, 1) * 4), offs(c, (n + 1) * 8);
    uint64_t kept = 0;
    if (n) {
      bitmap_flags_kernel<<<grid_for(c, n, 256), 256, 0, c->stream>>>(
          key, n, bm->words.as<uint32_t>(), bm->n_bits, flags.as<uint32_t>());
      c->count_launch();
      kept = prims::compact_offsets(c, flags.as<uint32_t>(), offs.as<uint64_t>(), n);
    }
    auto t = make_table(c, kept, nc);
    std::vector<const uint32_t*> in(nc);
    std::vector<uint32_t*> o(nc);
    for (int k = 0; k < nc; ++k) {
      in[k] = col_u32(tb, k);
      o[k] = t->cols[k].buf.as<uint32_t>();
    }
    prims::compact_cols(c, flags.as<uint32_t>(), offs.as<uint64_t>(), n, nc, in.data(), o.data());
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    *out = t.release();
  });
}

int tidq_table_unique_col(tidq_table* tb, int32_t col, tidq_table** out) {
  return guarded([&] {
    TIDQ_REQUIRE(tb && out, TIDQ_E_INVALID, "null argument");
    Ctx* c = tb->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    const uint64_t n = tb->n_rows;
    DevBuf keys, ids;
    sort_column(c, col_u32(tb, col), n, keys, ids);
    DevBuf flags(c, std::max<uint64_t>(n, 1) * 4), offs(c, (n + 1) * 8);
    uint64_t u = 0;
    if (n) {
      adjacent_unique_flags_kernel<<<grid_for(c, n, 256), 256, 0, c->stream>>>(
          keys.as<uint32_t>(), n, flags.as<uint32_t>());
      c->count_launch();
      u = prims::compact_offsets(c, flags.as<uint32_t>(), offs.as<uint64_t>(), n);
    }
    auto t = make_table(c, u, 1);
    const uint32_t* in[1] = {keys.as<uint32_t>()};
    uint32_t* o[1] = {t->cols[0].buf.as<uint32_t>()};
    prims::compact_cols(c, flags.as<uint32_t>(), offs.as<uint64_t>(), n, 1, in, o);
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    *out = t.release();
  });
}

// DISTINCT over `cols`: stable LSD sort of row ids by the projected columns
// (two columns per 64-bit radix key, last columns first), run heads flagged
// at their ORIGINAL row, then an order-preserving compaction — so the output
// is exactly the reference's first-occurrence order (query_ops.py:393-398).
int tidq_distinct(tidq_table* tb, int32_t n_cols, const int32_t* cols, tidq_table** out) {
  return guarded([&] {
    TIDQ_REQUIRE(tb && out && n_cols >= 1 && n_cols <= 8 && cols, TIDQ_E_INVALID,
                 "distinct needs 1..8 columns");
    Ctx* c = tb->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    const uint64_t n = tb->n_rows;
    TIDQ_REQUIRE(n < (1ull << 32), TIDQ_E_INVALID, "distinct input above 2^32 rows");
    std::vector<const uint32_t*> src(n_cols);
    for (int k = 0; k < n_cols; ++k) src[k] = col_u32(tb, cols[k]);
    DevBuf perm(c, std::max<uint64_t>(n, 1) * 4);
    DevBuf flags(c, std::max<uint64_t>(n, 1) * 4), offs(c, (n + 1) * 8);
    uint64_t u = 0;
    if (n) {
      prims::iota(c, perm.as<uint32_t>(), n);
      DevBuf k64(c, n * 8), k32(c, n * 4);
      // column groups from the last: pairs (hi=c[j-1], lo=c[j]) or a single c[0]
      int j = n_cols - 1;
      bool first = true;
      while (j >= 0) {
        if (j >= 1) {
          const uint32_t mx_hi = prims::max_u32(c, src[j - 1], n);
          const int lo_bits = std::max(1, prims::bits_for(prims::max_u32(c, src[j], n)));
          // (hi << lo_bits) | lo orders pairs like (hi, lo): only the significant bits are sorted
          pack2_kernel<<<grid_for(c, n, 256), 256, 0, c->stream>>>(
              src[j - 1], src[j], first ? nullptr : perm.as<uint32_t>(), n, lo_bits,
              k64.as<uint64_t>());
          c->count_launch();
          prims::radix_sort_pairs(c, k64.as<uint64_t>(), perm.as<uint32_t>(), n,
                                  lo_bits + prims::bits_for(mx_hi));
          j -= 2;
        } else {
          const uint32_t mx = prims::max_u32(c, src[0], n);
          if (first) {
            TIDQ_CUDA(cudaMemcpyAsync(k32.ptr, src[0], n * 4, cudaMemcpyDeviceToDevice, c->stream));
          } else {
            prims::gather_u32(c, src[0], perm.as<uint32_t>(), k32.as<uint32_t>(), n);
          }
          prims::radix_sort_pairs(c, k32.as<uint32_t>(), perm.as<uint32_t>(), n,
                                  prims::bits_for(mx));
          j -= 1;
        }
        first = false;
      }
      RowCols rc{};
      for (int k = 0; k < n_cols; ++k) rc.c[k] = src[k];
      head_flags_kernel<<<grid_for(c, n, 256), 256, 0, c->stream>>>(perm.as<uint32_t>(), n, n_cols,
                                                                    rc, flags.as<uint32_t>());
      c->count_launch();
      u = prims::compact_offsets(c, flags.as<uint32_t>(), offs.as<uint64_t>(), n);
    }
    auto t = make_table(c, u, n_cols);
    std::vector<uint32_t*> o(n_cols);
    for (int k = 0; k < n_cols; ++k) o[k] = t->cols[k].buf.as<uint32_t>();
    prims::compact_cols(c, flags.as<uint32_t>(), offs.as<uint64_t>(), n, n_cols, src.data(),
                        o.data());
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    *out = t.release();
  });
}

int tidq_join(tidq_table* left, int32_t lkey, tidq_table* right, int32_t rkey, int32_t n_out,
              const tidq_colref* out_cols, int32_t n_eq, const int32_t* eq_pairs, int64_t row_cap,
              int32_t algo, tidq_table** out, uint64_t* n_pairs) {
  return guarded([&] {
    TIDQ_REQUIRE(left && right && out && left->ctx == right->ctx, TIDQ_E_INVALID, "bad tables");
    TIDQ_REQUIRE(n_out >= 0 && n_out <= 8 && (out_cols || !n_out), TIDQ_E_INVALID, "bad outputs");
    TIDQ_REQUIRE(n_eq >= 0 && n_eq <= 4 && (eq_pairs || !n_eq), TIDQ_E_INVALID, "bad eq pairs");
    (void)algo;
    Ctx* c = left->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    JoinPlan jp;
    join_prepare(c, col_u32(left, lkey), left->n_rows, col_u32(right, rkey), right->n_rows, jp);
    if (n_pairs) *n_pairs = jp.total;
    if (row_cap >= 0 && jp.total > uint64_t(row_cap))
      throw Error(TIDQ_E_ROW_CAP, "join produced " + std::to_string(jp.total) +
                                      " rows, cap is " + std::to_string(row_cap));
    JoinOut jo{};
    jo.n_out = n_out;
    auto t = make_table(c, jp.total, n_out);
    for (int k = 0; k < n_out; ++k) {
      jo.side[k] = out_cols[k].side;
      jo.src[k] = col_u32(out_cols[k].side ? right : left, out_cols[k].col);
      jo.dst[k] = t->cols[k].buf.as<uint32_t>();
    }
    jo.n_eq = n_eq;
    for (int e = 0; e < n_eq; ++e) {
      jo.eq_l[e] = col_u32(left, eq_pairs[2 * e]);
      jo.eq_r[e] = col_u32(right, eq_pairs[2 * e + 1]);
    }
    DevBuf keep;
    if (n_eq) keep = DevBuf(c, std::max<uint64_t>(jp.total, 1) * 4);
    join_expand(c, jp, jo, n_eq ? keep.as<uint32_t>() : nullptr);
    if (n_eq && jp.total) {
      DevBuf offs(c, (jp.total + 1) * 8);
      const uint64_t kept = prims::compact_offsets(c, keep.as<uint32_t>(), offs.as<uint64_t>(),
                                                   jp.total);
      auto t2 = make_table(c, kept, n_out);
      std::vector<const uint32_t*> in(n_out);
      std::vector<uint32_t*> o(n_out);
      for (int k = 0; k < n_out; ++k) {
        in[k] = t->cols[k].buf.as<uint32_t>();
        o[k] = t2->cols[k].buf.as<uint32_t>();
      }
      prims::compact_cols(c, keep.as<uint32_t>(), offs.as<uint64_t>(), jp.total, n_out, in.data(),
                          o.data());
      t = std::move(t2);
    }
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    *out = t.release();
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
