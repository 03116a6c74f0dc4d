// Multi-GPU exchange of binding tables: one process per GPU,
// a libtidq-owned NCCL communicator over NVLink/NVSwitch.
//
//   tidq_table_partition  rows grouped by destination rank
//                         dest = hash(key columns) % nranks (stable, radix on dest)
//   tidq_table_alltoallv  variable-size all-to-all: per-peer counts first
//                         (one 8-byte send/recv per peer), then every column
//                         with grouped ncclSend/ncclRecv straight from/to HBM
//   tidq_table_allgather  every rank's rows, in rank order (small build sides,
//                         final result collection)
//
// The hash is the one distributed.py documents (and its numpy twin in the
// tests uses): h = 0; for each key column v: h = (h ^ v) * 0x9E3779B97F4A7C15
// (mod 2^64); dest = (h >> 32) % nranks.
#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "internal.cuh"
#include "prims.cuh"

#ifdef TIDQ_HAVE_NCCL
#include <nccl.h>
#endif

struct tidq_comm {
  tidq_ctx* ctx = nullptr;
  int nranks = 1;
  int rank = 0;
  // exchange accounting (tidq_comm_stats): payload bytes this rank sent to
  // other ranks and the device time of the payload exchanges
  uint64_t bytes_out = 0;
  double exchange_ms = 0;
#ifdef TIDQ_HAVE_NCCL
  ncclComm_t nccl = nullptr;
#endif
};

namespace tidq {
namespace {

constexpr int kT = 256;
constexpr int kI = 4;
constexpr int kBlk = kT * kI;

struct KeyCols {
  const uint32_t* c[4];
  int n;
};

__global__ void __launch_bounds__(kT) dest_kernel(KeyCols kc, uint64_t n, uint32_t nranks,
                                                  uint32_t* __restrict__ dest) {
  const uint64_t base = uint64_t(blockIdx.x) * kBlk;
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t i = base + j * kT + threadIdx.x;
    if (i >= n) continue;
    uint64_t h = 0;
    for (int k = 0; k < kc.n; ++k) h = (h ^ uint64_t(__ldg(kc.c[k] + i))) * 0x9E3779B97F4A7C15ull;
    dest[i] = uint32_t((h >> 32) % nranks);
  }
}

__global__ void __launch_bounds__(kT) dest_count_kernel(const uint32_t* __restrict__ dest, uint64_t n,
                                                        unsigned long long* __restrict__ counts) {
  __shared__ unsigned long long h[1024];
  for (int i = threadIdx.x; i < 1024; i += kT) h[i] = 0;
  __syncthreads();
  const uint64_t base = uint64_t(blockIdx.x) * kBlk;
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const uint64_t i = base + j * kT + threadIdx.x;
    if (i < n) atomicAdd(&h[dest[i] & 1023], 1ull);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 1024; i += kT)
    if (h[i]) atomicAdd(counts + i, h[i]);
}

#ifdef TIDQ_HAVE_NCCL
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(TIDQ_E_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}
#endif

}  // namespace
}  // namespace tidq

using namespace tidq;

extern "C" {

int tidq_comm_unique_id(uint8_t* id_out) {
  return guarded([&] {
    TIDQ_REQUIRE(id_out, TIDQ_E_INVALID, "null output");
#ifdef TIDQ_HAVE_NCCL
    ncclUniqueId id;
    nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
#else
    throw Error(TIDQ_E_UNSUPPORTED, "libtidq was built without NCCL");
#endif
  });
}

int tidq_comm_create(tidq_ctx* ctx, const uint8_t* id, int32_t nranks, int32_t rank, tidq_comm** out) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx && id && out && nranks >= 1 && rank >= 0 && rank < nranks, TIDQ_E_INVALID,
                 "bad communicator arguments");
#ifdef TIDQ_HAVE_NCCL
    DeviceGuard g(ctx);
    auto cm = std::make_unique<tidq_comm>();
    cm->ctx = ctx;
    cm->nranks = nranks;
    cm->rank = rank;
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    nccl_check(ncclCommInitRank(&cm->nccl, nranks, uid, rank), "ncclCommInitRank");
    *out = cm.release();
#else
    (void)id;
    throw Error(TIDQ_E_UNSUPPORTED, "libtidq was built without NCCL");
#endif
  });
}

int tidq_comm_destroy(tidq_comm* comm) {
  return guarded([&] {
    if (!comm) return;
#ifdef TIDQ_HAVE_NCCL
    if (comm->nccl) ncclCommDestroy(comm->nccl);
#endif
    delete comm;
  });
}

int tidq_table_partition(tidq_table* t, int32_t n_key_cols, const int32_t* key_cols, int32_t nranks,
                         tidq_table** out, uint64_t* counts) {
  return guarded([&] {
    TIDQ_REQUIRE(t && out && counts && key_cols && n_key_cols >= 1 && n_key_cols <= 4 && nranks >= 1 &&
                     nranks <= 1024,
                 TIDQ_E_INVALID, "bad partition arguments");
    Ctx* c = t->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    const uint64_t n = t->n_rows();
    TIDQ_REQUIRE(n < (1ull << 32), TIDQ_E_INVALID, "partition input above 2^32 rows");
    KeyCols kc{};
    kc.n = n_key_cols;
    for (int k = 0; k < n_key_cols; ++k) {
      TIDQ_REQUIRE(key_cols[k] >= 0 && key_cols[k] < int(t->cols.size()) && t->cols[key_cols[k]].dtype == TIDQ_U32,
                   TIDQ_E_INVALID, "bad key column");
      kc.c[k] = t->cols[key_cols[k]].buf.as<uint32_t>();
    }
    auto o = std::make_unique<tidq_table>();
    o->ctx = c;
    o->set_rows(n);
    o->capacity = n;
    DevBuf dest(c, std::max<uint64_t>(n, 1) * 4), perm(c, std::max<uint64_t>(n, 1) * 4);
    DevBuf dcounts(c, 1024 * 8);
    TIDQ_CUDA(cudaMemsetAsync(dcounts.ptr, 0, 1024 * 8, c->stream));
    if (n) {
      const unsigned grid = unsigned((n + kBlk - 1) / kBlk);
      dest_kernel<<<grid, kT, 0, c->stream>>>(kc, n, uint32_t(nranks), dest.as<uint32_t>());
      dest_count_kernel<<<grid, kT, 0, c->stream>>>(dest.as<uint32_t>(), n,
                                                    dcounts.as<unsigned long long>());
      c->count_launch(2);
      prims::iota(c, perm.as<uint32_t>(), n);
      if (nranks > 1)
        prims::radix_sort_pairs(c, dest.as<uint32_t>(), perm.as<uint32_t>(), n, prims::bits_for(nranks - 1));
    }
    for (auto& col : t->cols) {
      Column oc;
      oc.dtype = col.dtype;
      oc.buf = DevBuf(c, std::max<uint64_t>(n, 1) * Column::width(col.dtype));
      TIDQ_REQUIRE(col.dtype == TIDQ_U32, TIDQ_E_INVALID, "partition supports uint32 columns");
      if (n) prims::gather_u32(c, col.buf.as<uint32_t>(), perm.as<uint32_t>(), oc.buf.as<uint32_t>(), n);
      o->cols.push_back(std::move(oc));
    }
    TIDQ_CUDA(cudaMemcpyAsync(counts, dcounts.ptr, size_t(nranks) * 8, cudaMemcpyDeviceToHost, c->stream));
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    *out = o.release();
  });
}

int tidq_table_alltoallv(tidq_comm* comm, tidq_table* t, const uint64_t* send_counts, tidq_table** out,
                         uint64_t* recv_counts) {
  return guarded([&] {
    TIDQ_REQUIRE(comm && t && out && send_counts, TIDQ_E_INVALID, "null argument");
#ifdef TIDQ_HAVE_NCCL
    Ctx* c = comm->ctx;
    TIDQ_REQUIRE(t->ctx == c, TIDQ_E_INVALID, "table and communicator on different devices");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    const int R = comm->nranks;
    uint64_t total_send = 0;
    for (int r = 0; r < R; ++r) total_send += send_counts[r];
    TIDQ_REQUIRE(total_send == t->n_rows(), TIDQ_E_INVALID, "send counts do not add up to the table");
    // 1. exchange the per-peer row counts
    DevBuf sc(c, size_t(R) * 8), rc(c, size_t(R) * 8);
    TIDQ_CUDA(cudaMemcpyAsync(sc.ptr, send_counts, size_t(R) * 8, cudaMemcpyHostToDevice, c->stream));
    nccl_check(ncclGroupStart(), "ncclGroupStart");
    for (int r = 0; r < R; ++r) {
      nccl_check(ncclSend(sc.as<uint64_t>() + r, 1, ncclUint64, r, comm->nccl, c->stream), "ncclSend");
      nccl_check(ncclRecv(rc.as<uint64_t>() + r, 1, ncclUint64, r, comm->nccl, c->stream), "ncclRecv");
    }
    nccl_check(ncclGroupEnd(), "ncclGroupEnd");
    std::vector<uint64_t> rcnt(R);
    TIDQ_CUDA(cudaMemcpyAsync(rcnt.data(), rc.ptr, size_t(R) * 8, cudaMemcpyDeviceToHost, c->stream));
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    uint64_t total_recv = 0;
    for (int r = 0; r < R; ++r) total_recv += rcnt[r];
    if (recv_counts)
      for (int r = 0; r < R; ++r) recv_counts[r] = rcnt[r];
    // 2. every column: grouped send/recv, received rows in source-rank order
    cudaEvent_t e0, e1;
    TIDQ_CUDA(cudaEventCreate(&e0));
    TIDQ_CUDA(cudaEventCreate(&e1));
    TIDQ_CUDA(cudaEventRecord(e0, c->stream));
    auto o = std::make_unique<tidq_table>();
    o->ctx = c;
    o->set_rows(total_recv);
    o->capacity = total_recv;
    for (auto& col : t->cols) {
      Column oc;
      oc.dtype = col.dtype;
      const size_t w = Column::width(col.dtype);
      oc.buf = DevBuf(c, std::max<uint64_t>(total_recv, 1) * w);
      nccl_check(ncclGroupStart(), "ncclGroupStart");
      uint64_t so = 0, ro = 0;
      for (int r = 0; r < R; ++r) {
        if (send_counts[r])
          nccl_check(ncclSend(col.buf.as<char>() + so * w, send_counts[r] * w, ncclUint8, r, comm->nccl,
                              c->stream), "ncclSend");
        if (rcnt[r])
          nccl_check(ncclRecv(oc.buf.as<char>() + ro * w, rcnt[r] * w, ncclUint8, r, comm->nccl, c->stream),
                     "ncclRecv");
        if (r != comm->rank) comm->bytes_out += send_counts[r] * w;
        so += send_counts[r];
        ro += rcnt[r];
      }
      nccl_check(ncclGroupEnd(), "ncclGroupEnd");
      o->cols.push_back(std::move(oc));
    }
    TIDQ_CUDA(cudaEventRecord(e1, c->stream));
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    float ms = 0;
    TIDQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    comm->exchange_ms += ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *out = o.release();
#else
    (void)recv_counts;
    throw Error(TIDQ_E_UNSUPPORTED, "libtidq was built without NCCL");
#endif
  });
}

int tidq_comm_stats(tidq_comm* comm, int32_t reset, uint64_t* bytes_out, double* exchange_ms) {
  return guarded([&] {
    TIDQ_REQUIRE(comm && bytes_out && exchange_ms, TIDQ_E_INVALID, "null argument");
    *bytes_out = comm->bytes_out;
    *exchange_ms = comm->exchange_ms;
    if (reset) {
      comm->bytes_out = 0;
      comm->exchange_ms = 0;
    }
  });
}

int tidq_comm_allreduce_u64(tidq_comm* comm, const uint64_t* in, uint64_t* out, int32_t n) {
  return guarded([&] {
    TIDQ_REQUIRE(comm && in && out && n >= 1 && n <= 512, TIDQ_E_INVALID, "bad allreduce arguments");
#ifdef TIDQ_HAVE_NCCL
    Ctx* c = comm->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    DevBuf d(c, size_t(n) * 8);
    TIDQ_CUDA(cudaMemcpyAsync(d.ptr, in, size_t(n) * 8, cudaMemcpyHostToDevice, c->stream));
    nccl_check(ncclAllReduce(d.ptr, d.ptr, size_t(n), ncclUint64, ncclSum, comm->nccl, c->stream),
               "ncclAllReduce");
    TIDQ_CUDA(cudaMemcpyAsync(out, d.ptr, size_t(n) * 8, cudaMemcpyDeviceToHost, c->stream));
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
#else
    throw Error(TIDQ_E_UNSUPPORTED, "libtidq was built without NCCL");
#endif
  });
}

int tidq_table_allgather(tidq_comm* comm, tidq_table* t, tidq_table** out) {
  return guarded([&] {
    TIDQ_REQUIRE(comm && t && out, TIDQ_E_INVALID, "null argument");
#ifdef TIDQ_HAVE_NCCL
    Ctx* c = comm->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    const int R = comm->nranks;
    DevBuf n_dev(c, 8), all_dev(c, size_t(R) * 8);
    const uint64_t mine = t->n_rows();
    TIDQ_CUDA(cudaMemcpyAsync(n_dev.ptr, &mine, 8, cudaMemcpyHostToDevice, c->stream));
    nccl_check(ncclAllGather(n_dev.ptr, all_dev.ptr, 1, ncclUint64, comm->nccl, c->stream), "ncclAllGather");
    std::vector<uint64_t> cnt(R);
    TIDQ_CUDA(cudaMemcpyAsync(cnt.data(), all_dev.ptr, size_t(R) * 8, cudaMemcpyDeviceToHost, c->stream));
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    uint64_t total = 0;
    for (int r = 0; r < R; ++r) total += cnt[r];
    auto o = std::make_unique<tidq_table>();
    o->ctx = c;
    o->set_rows(total);
    o->capacity = total;
    for (auto& col : t->cols) {
      Column oc;
      oc.dtype = col.dtype;
      const size_t w = Column::width(col.dtype);
      oc.buf = DevBuf(c, std::max<uint64_t>(total, 1) * w);
      // variable sizes: every rank broadcasts its slice (grouped)
      nccl_check(ncclGroupStart(), "ncclGroupStart");
      uint64_t at = 0;
      for (int r = 0; r < R; ++r) {
        if (cnt[r])
          nccl_check(ncclBroadcast(r == comm->rank ? col.buf.ptr : oc.buf.as<char>() + at * w,
                                   oc.buf.as<char>() + at * w, cnt[r] * w, ncclUint8, r, comm->nccl,
                                   c->stream),
                     "ncclBroadcast");
        at += cnt[r];
      }
      nccl_check(ncclGroupEnd(), "ncclGroupEnd");
      o->cols.push_back(std::move(oc));
    }
    TIDQ_CUDA(cudaStreamSynchronize(c->stream));
    *out = o.release();
#else
    throw Error(TIDQ_E_UNSUPPORTED, "libtidq was built without NCCL");
#endif
  });
}

}  // extern "C"
