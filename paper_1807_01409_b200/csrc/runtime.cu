// libtidq runtime: contexts, pool-backed device buffers, resident SoA stores,
// device tables, FILTER bitmaps.  ABI entry points wrap their bodies in
// tidq::guarded() so failures become status codes + tidq_last_error().
#include <cuda_runtime.h>
#include <cerrno>
#include <thread>
#include <atomic>
#include <unistd.h>
#include <sys/stat.h>
#include <fcntl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <memory>
#include <string>

#include "internal.cuh"
#include "prims.cuh"

namespace tidq {

namespace {
struct PhaseTrace {
  bool on = getenv("TIDQ_PHASE_TRACE") != nullptr;
  std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
  std::vector<std::pair<std::string, double>> acc, gacc;
  cudaEvent_t ev_last = nullptr;
};
PhaseTrace& phase_trace() {
  static PhaseTrace t;
  return t;
}
}  // namespace

void ensure_dyn_smem(const void* kernel, int device, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  std::lock_guard<std::mutex> lk(mu);
  int& have = done[{kernel, device}];
  if (have >= bytes) return;
  TIDQ_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  have = bytes;
}

void phase_mark(Ctx* c, const char* name) {
  PhaseTrace& t = phase_trace();
  if (!t.on) return;
  double gus = 0;
  if (c) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, c->stream);
    cudaStreamSynchronize(c->stream);
    if (t.ev_last) {
      float ms = 0;
      cudaEventElapsedTime(&ms, t.ev_last, e);
      gus = ms * 1e3;
      cudaEventDestroy(t.ev_last);
    }
    t.ev_last = e;
  }
  const auto now = std::chrono::steady_clock::now();
  const double us = std::chrono::duration<double, std::micro>(now - t.last).count();
  t.last = now;
  if (!name) return;
  for (size_t i = 0; i < t.acc.size(); ++i)
    if (t.acc[i].first == name) {
      t.acc[i].second += us;
      t.gacc[i].second += gus;
      return;
    }
  t.acc.emplace_back(name, us);
  t.gacc.emplace_back(name, gus);
}

void phase_report(const char* what) {
  PhaseTrace& t = phase_trace();
  if (!t.on) return;
  fprintf(stderr, "[tidq phases] %s:", what);
  for (size_t i = 0; i < t.acc.size(); ++i)
    fprintf(stderr, " %s=%.0f/%.0fus", t.acc[i].first.c_str(), t.acc[i].second, t.gacc[i].second);
  fprintf(stderr, " (wall/stream)\n");
  t.acc.clear();
  t.gacc.clear();
}


static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }

DevBuf::DevBuf(Ctx* c, size_t b) : ctx(c), bytes(b) {
  if (b == 0) return;
  // Stream-ordered allocation from the ctx pool (release threshold = max, so
  // steady-state queries do not hit cudaMalloc).
  cudaError_t e = cudaMallocFromPoolAsync(&ptr, b, c->pool, c->stream);
  if (e != cudaSuccess) {
    ptr = nullptr;
    cudaGetLastError();
    throw Error(TIDQ_E_NOMEM, "device allocation of " + std::to_string(b) +
                                  " bytes failed: " + cudaGetErrorString(e));
  }
}

DevBuf& DevBuf::operator=(DevBuf&& o) noexcept {
  if (this != &o) {
    reset();
    ptr = o.ptr;
    bytes = o.bytes;
    ctx = o.ctx;
    o.ptr = nullptr;
    o.bytes = 0;
  }
  return *this;
}

void DevBuf::reset() {
  if (ptr && ctx) cudaFreeAsync(ptr, ctx->stream);
  ptr = nullptr;
  bytes = 0;
}

DevBuf::~DevBuf() { reset(); }

static void sync(Ctx* c) { TIDQ_CUDA(cudaStreamSynchronize(c->stream)); }

// Upload an AoS host array into SoA device columns in pipelined slabs:
// H2D on the copy stream into one of two staging slabs while the compute
// stream transposes the previous slab (reference layout: store.py:61-79).
// Pipelined AoS -> SoA ingest through page-locked slabs (8 Mi triples = 96
// MiB): `fill(dst, lo, cnt)` writes triples [lo, lo+cnt) into a host slab
// (parallel memcpy from pageable memory, parallel pread from a file) while
// the previous slab's H2D copy (copy stream) and transpose (compute stream)
// run.  Returns false when fill failed.
template <class Fill>
static bool ingest_slabs(Ctx* c, uint64_t n, uint32_t* s, uint32_t* p, uint32_t* o, Fill&& fill) {
  const uint64_t slab = 8ull << 20;
  const size_t slab_bytes = slab * 12;
  for (auto& b : c->staging)
    if (b.bytes < slab_bytes) b = DevBuf(c, slab_bytes);
  for (int i = 0; i < 2; ++i)
    if (!c->pinned_slab[i]) TIDQ_CUDA(cudaMallocHost(&c->pinned_slab[i], slab_bytes));
  cudaEvent_t copied[2], done[2];
  for (int i = 0; i < 2; ++i) {
    TIDQ_CUDA(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
    TIDQ_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    TIDQ_CUDA(cudaEventRecord(done[i], c->stream));
    TIDQ_CUDA(cudaEventRecord(copied[i], c->copy_stream));
  }
  bool ok = true;
  uint64_t k = 0;
  for (uint64_t lo = 0; lo < n; lo += slab, ++k) {
    const int b = int(k & 1);
    const uint64_t cnt = std::min(slab, n - lo);
    TIDQ_CUDA(cudaEventSynchronize(copied[b]));  // the H2D that last read this host slab
    char* dst = static_cast<char*>(c->pinned_slab[b]);
    if (!fill(dst, lo, cnt)) {
      ok = false;
      break;
    }
    TIDQ_CUDA(cudaStreamWaitEvent(c->copy_stream, done[b], 0));
    TIDQ_CUDA(cudaMemcpyAsync(c->staging[b].ptr, dst, cnt * 12, cudaMemcpyHostToDevice, c->copy_stream));
    TIDQ_CUDA(cudaEventRecord(copied[b], c->copy_stream));
    TIDQ_CUDA(cudaStreamWaitEvent(c->stream, copied[b], 0));
    launch_transpose_aos(c, c->staging[b].as<uint32_t>(), cnt, s + lo, p + lo, o + lo, c->stream);
    TIDQ_CUDA(cudaEventRecord(done[b], c->stream));
  }
  sync(c);
  TIDQ_CUDA(cudaStreamSynchronize(c->copy_stream));
  for (int i = 0; i < 2; ++i) {
    cudaEventDestroy(copied[i]);
    cudaEventDestroy(done[i]);
  }
  return ok;
}

// Run f(t, lo, len) over [0, bytes) split across up to 8 host threads.
template <class F>
static bool parallel_bytes(size_t bytes, F&& f) {
  const int n_threads = int(std::max(1u, std::min(8u, std::thread::hardware_concurrency())));
  const size_t part = (bytes + n_threads - 1) / n_threads;
  std::atomic<bool> ok{true};
  std::vector<std::thread> th;
  for (int t = 0; t < n_threads; ++t) {
    const size_t a0 = size_t(t) * part;
    if (a0 >= bytes) break;
    const size_t len = std::min(part, bytes - a0);
    th.emplace_back([&, a0, len] {
      if (!f(a0, len)) ok = false;
    });
  }
  for (auto& t : th) t.join();
  return ok;
}

static bool host_pinned(const void* ptr) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

static void upload_aos(Ctx* c, const uint32_t* aos, uint64_t n, uint32_t* s, uint32_t* p,
                       uint32_t* o) {
  if (n == 0) return;
  if (!host_pinned(aos)) {
    // pageable: parallel memcpy into the page-locked slabs (a pageable
    // cudaMemcpy runs at ~11 GB/s through the driver's bounce buffer)
    const char* src = reinterpret_cast<const char*>(aos);
    ingest_slabs(c, n, s, p, o, [&](char* dst, uint64_t lo, uint64_t cnt) {
      return parallel_bytes(cnt * 12, [&](size_t a0, size_t len) {
        memcpy(dst + a0, src + lo * 12 + a0, len);
        return true;
      });
    });
    return;
  }
  // Staged through device slabs on a copy stream, transposed on the compute
  // stream: 55 GB/s from pinned memory (= the PCIe copy ceiling measured with
  // torch); a zero-copy transpose reading mapped host memory reached 41 GB/s.
  const uint64_t slab = 8ull << 20;  // triples per slab (96 MiB of AoS)
  const uint64_t slab_bytes = slab * 12;
  for (auto& b : c->staging)
    if (b.bytes < slab_bytes) b = DevBuf(c, slab_bytes);
  cudaEvent_t copied[2], done[2];
  for (int i = 0; i < 2; ++i) {
    TIDQ_CUDA(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
    TIDQ_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
  }
  // staging buffers were allocated on the compute stream; order the copy
  // stream after that allocation.
  TIDQ_CUDA(cudaEventRecord(done[0], c->stream));
  TIDQ_CUDA(cudaEventRecord(done[1], c->stream));
  uint64_t k = 0;
  for (uint64_t lo = 0; lo < n; lo += slab, ++k) {
    const int b = int(k & 1);
    const uint64_t cnt = std::min(slab, n - lo);
    TIDQ_CUDA(cudaStreamWaitEvent(c->copy_stream, done[b], 0));
    TIDQ_CUDA(cudaMemcpyAsync(c->staging[b].ptr, aos + lo * 3, cnt * 12, cudaMemcpyHostToDevice,
                              c->copy_stream));
    TIDQ_CUDA(cudaEventRecord(copied[b], c->copy_stream));
    TIDQ_CUDA(cudaStreamWaitEvent(c->stream, copied[b], 0));
    launch_transpose_aos(c, c->staging[b].as<uint32_t>(), cnt, s + lo, p + lo, o + lo, c->stream);
    TIDQ_CUDA(cudaEventRecord(done[b], c->stream));
  }
  sync(c);
  for (int i = 0; i < 2; ++i) {
    cudaEventDestroy(copied[i]);
    cudaEventDestroy(done[i]);
  }
}

static tidq_store* new_store(Ctx* c, uint64_t n, uint64_t base) {
  auto st = std::make_unique<tidq_store>();
  st->ctx = c;
  st->n = n;
  st->base = base;
  st->padded = round_up(std::max<uint64_t>(n, 1), kScanTile);
  const size_t bytes = st->padded * 4;
  st->s = DevBuf(c, bytes);
  st->p = DevBuf(c, bytes);
  st->o = DevBuf(c, bytes);
  // zero the padding tail so vector loads past n read defined values
  const size_t tail = (st->padded - n) * 4;
  if (tail) {
    TIDQ_CUDA(cudaMemsetAsync(st->s.as<uint32_t>() + n, 0, tail, c->stream));
    TIDQ_CUDA(cudaMemsetAsync(st->p.as<uint32_t>() + n, 0, tail, c->stream));
    TIDQ_CUDA(cudaMemsetAsync(st->o.as<uint32_t>() + n, 0, tail, c->stream));
  }
  return st.release();
}

}  // namespace tidq

using namespace tidq;

extern "C" {

int tidq_abi_version(void) { return TIDQ_ABI_VERSION; }

const char* tidq_last_error(void) { return g_last_error.c_str(); }

int tidq_device_count(int* n) {
  return guarded([&] {
    TIDQ_REQUIRE(n, TIDQ_E_INVALID, "null output");
    cudaError_t e = cudaGetDeviceCount(n);
    if (e != cudaSuccess) {
      cudaGetLastError();
      *n = 0;
    }
  });
}

int tidq_ctx_create(int device, tidq_ctx** out) {
  return guarded([&] {
    TIDQ_REQUIRE(out, TIDQ_E_INVALID, "null output");
    int count = 0;
    TIDQ_CUDA(cudaGetDeviceCount(&count));
    TIDQ_REQUIRE(device >= 0 && device < count, TIDQ_E_INVALID,
                 "device " + std::to_string(device) + " out of range (" +
                     std::to_string(count) + " visible)");
    auto c = std::make_unique<tidq_ctx>();
    c->device = device;
    TIDQ_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    TIDQ_CUDA(cudaGetDeviceProperties(&prop, device));
    TIDQ_REQUIRE(prop.major >= 10, TIDQ_E_UNSUPPORTED,
                 std::string("libtidq is built for sm_100a; device is ") + prop.name);
    c->sm_count = prop.multiProcessorCount;
    TIDQ_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    TIDQ_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    TIDQ_CUDA(cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking));
    TIDQ_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    TIDQ_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    TIDQ_CUDA(cudaDeviceGetDefaultMemPool(&c->pool, device));
    uint64_t threshold = UINT64_MAX;
    TIDQ_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    TIDQ_CUDA(cudaMallocHost(&c->pinned_small, 4096));
    TIDQ_CUDA(cudaMallocHost(reinterpret_cast<void**>(&c->row_slots), sizeof(uint64_t) * tidq_ctx::kRowSlots));
    for (int i = tidq_ctx::kRowSlots - 1; i >= 0; --i) c->free_row_slots.push_back(i);
    *out = c.release();
  });
}

}  // extern "C"

// Deferred row counts: the count was queued as a D2H copy into a pinned slot
// on the ctx stream; the first use waits for the stream and reads it.
uint64_t tidq_table::n_rows() {
  if (pending_slot_ >= 0) {
    TIDQ_CUDA(cudaStreamSynchronize(ctx->stream));
    rows_ = ctx->row_slots[pending_slot_];
    ctx->free_row_slots.push_back(pending_slot_);
    pending_slot_ = -1;
  }
  return rows_;
}

tidq_table::~tidq_table() {
  if (pending_slot_ >= 0) {  // the copy into the slot must land before reuse
    cudaStreamSynchronize(ctx->stream);
    ctx->free_row_slots.push_back(pending_slot_);
  }
}

extern "C" {

int tidq_ctx_mem_info(tidq_ctx* ctx, uint64_t* free_bytes, uint64_t* total_bytes) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx && free_bytes && total_bytes, TIDQ_E_INVALID, "null argument");
    DeviceGuard g(ctx);
    size_t f = 0, t = 0;
    TIDQ_CUDA(cudaMemGetInfo(&f, &t));
    *free_bytes = f;
    *total_bytes = t;
  });
}

int tidq_ctx_trim(tidq_ctx* ctx) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx, TIDQ_E_INVALID, "null ctx");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx);
    TIDQ_CUDA(cudaStreamSynchronize(ctx->stream));
    TIDQ_CUDA(cudaMemPoolTrimTo(ctx->pool, 0));
  });
}

int tidq_ctx_destroy(tidq_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->lookback.reset();
    ctx->ssum.reset();
    ctx->staging[0].reset();
    ctx->staging[1].reset();
    cudaStreamSynchronize(ctx->stream);
    if (ctx->pinned_small) cudaFreeHost(ctx->pinned_small);
    if (ctx->row_slots) cudaFreeHost(ctx->row_slots);
    if (ctx->host_scratch) cudaFreeHost(ctx->host_scratch);
    for (void* p : ctx->pinned_slab)
      if (p) cudaFreeHost(p);
    cudaStreamSynchronize(ctx->side_stream);
    cudaEventDestroy(ctx->ev_fork);
    cudaEventDestroy(ctx->ev_join);
    cudaStreamDestroy(ctx->side_stream);
    cudaStreamDestroy(ctx->copy_stream);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

int tidq_ctx_sync(tidq_ctx* ctx) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx, TIDQ_E_INVALID, "null ctx");
    DeviceGuard g(ctx);
    sync(ctx);
  });
}

int tidq_ctx_launches(tidq_ctx* ctx, uint64_t* n) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx && n, TIDQ_E_INVALID, "null argument");
    *n = ctx->launches;
  });
}

int tidq_host_alloc(uint64_t bytes, void** out) {
  return guarded([&] {
    TIDQ_REQUIRE(out, TIDQ_E_INVALID, "null output");
    *out = nullptr;
    if (bytes) TIDQ_CUDA(cudaMallocHost(out, bytes));
  });
}

int tidq_host_free(void* p) {
  return guarded([&] {
    if (p) TIDQ_CUDA(cudaFreeHost(p));
  });
}

// ---- store ---------------------------------------------------------------

int tidq_store_upload(tidq_ctx* ctx, const uint32_t* aos, uint64_t n_triples,
                      uint64_t base_index, tidq_store** out) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx && out, TIDQ_E_INVALID, "null argument");
    TIDQ_REQUIRE(aos || n_triples == 0, TIDQ_E_INVALID, "null triple data");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx);
    std::unique_ptr<tidq_store> st(new_store(ctx, n_triples, base_index));
    upload_aos(ctx, aos, n_triples, st->s.as<uint32_t>(), st->p.as<uint32_t>(),
               st->o.as<uint32_t>());
    sync(ctx);
    *out = st.release();
  });
}

// ---- .tid ingest ---------------------------------------------------------------
// Host threads pread slab k+1 into one page-locked buffer while slab k's H2D
// copy and transpose run from the other (ingest_slabs).
int tidq_store_load_tid(tidq_ctx* ctx, const char* path, uint64_t base_index, tidq_store** out) {
  return tidq_store_load_tid_range(ctx, path, 0, UINT64_MAX, base_index, out);
}

// Rows [row_lo, row_lo + row_count) of a .tid file (clamped to the file's
// count) -> a resident store whose global indices start at base_index +
// row_lo: the row-sharded load of a multi-GPU store (rank g loads its
// contiguous range), restating read_chunks' base-index iteration
// (store.py:121-146) for an arbitrary range.
int tidq_store_load_tid_range(tidq_ctx* ctx, const char* path, uint64_t row_lo, uint64_t row_count,
                              uint64_t base_index, tidq_store** out) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx && path && out, TIDQ_E_INVALID, "null argument");
    const int fd = open(path, O_RDONLY);
    TIDQ_REQUIRE(fd >= 0, TIDQ_E_IO, std::string(path) + ": " + strerror(errno));
    struct FdGuard {
      int fd;
      ~FdGuard() { close(fd); }
    } fg{fd};
    struct stat sb;
    TIDQ_REQUIRE(fstat(fd, &sb) == 0, TIDQ_E_IO, std::string(path) + ": " + strerror(errno));
    unsigned char hdr[16];
    const ssize_t hn = pread(fd, hdr, 16, 0);
    TIDQ_REQUIRE(hn == 16, TIDQ_E_TRUNCATED, std::string(path) + ": header shorter than 16 bytes");
    TIDQ_REQUIRE(memcmp(hdr, "TID1", 4) == 0, TIDQ_E_BAD_MAGIC, std::string(path) + ": bad magic");
    uint32_t version;
    uint64_t count;
    memcpy(&version, hdr + 4, 4);
    memcpy(&count, hdr + 8, 8);
    TIDQ_REQUIRE(version == 1, TIDQ_E_BAD_VERSION,
                 std::string(path) + ": version " + std::to_string(version) + ", expected 1");
    const uint64_t avail = sb.st_size > 16 ? uint64_t(sb.st_size - 16) / 12 : 0;
    TIDQ_REQUIRE(avail >= count, TIDQ_E_TRUNCATED,
                 std::string(path) + ": header declares " + std::to_string(count) +
                     " triples, data ends at triple " + std::to_string(avail));
    TIDQ_REQUIRE(row_lo <= count, TIDQ_E_INVALID,
                 std::string(path) + ": row range starts at " + std::to_string(row_lo) + " beyond " +
                     std::to_string(count) + " triples");
    const uint64_t first = row_lo;
    count = std::min(row_count, count - row_lo);
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx);
    std::unique_ptr<tidq_store> st(new_store(ctx, count, base_index + first));
    if (count) {
      const bool ok = ingest_slabs(
          ctx, count, st->s.as<uint32_t>(), st->p.as<uint32_t>(), st->o.as<uint32_t>(),
          [&](char* dst, uint64_t lo, uint64_t cnt) {
            return parallel_bytes(cnt * 12, [&](size_t a0, size_t len) {
              size_t got = 0;
              while (got < len) {
                const ssize_t r =
                    pread(fd, dst + a0 + got, len - got, off_t(16 + (first + lo) * 12 + a0 + got));
                if (r <= 0) return false;
                got += size_t(r);
              }
              return true;
            });
          });
      TIDQ_REQUIRE(ok, TIDQ_E_TRUNCATED, std::string(path) + ": read failed before triple " +
                                             std::to_string(first + count));
    }
    sync(ctx);
    *out = st.release();
  });
}

int tidq_store_generate(tidq_ctx* ctx, const tidq_synth_params* prm, const uint64_t* zipf_cdf,
                        tidq_store** out) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx && prm && out && zipf_cdf, TIDQ_E_INVALID, "null argument");
    TIDQ_REQUIRE(prm->n_p >= 1 && prm->n_e >= 1, TIDQ_E_INVALID, "n_p and n_e must be >= 1");
    TIDQ_REQUIRE(uint64_t(prm->n_p) + prm->n_e < 0xFFFFFFFFull, TIDQ_E_INVALID,
                 "ID space exceeds 32 bits");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx);
    std::unique_ptr<tidq_store> st(new_store(ctx, prm->n_triples, prm->base_index));
    DevBuf cdf(ctx, size_t(prm->n_p) * 8);
    TIDQ_CUDA(cudaMemcpyAsync(cdf.ptr, zipf_cdf, size_t(prm->n_p) * 8, cudaMemcpyHostToDevice,
                              ctx->stream));
    launch_generate(ctx, *prm, cdf.as<uint64_t>(), st->s.as<uint32_t>(), st->p.as<uint32_t>(),
                    st->o.as<uint32_t>(), ctx->stream);
    cdf.reset();
    sync(ctx);
    *out = st.release();
  });
}

int tidq_store_info(const tidq_store* st, uint64_t* n_triples, uint64_t* base_index) {
  return guarded([&] {
    TIDQ_REQUIRE(st, TIDQ_E_INVALID, "null store");
    if (n_triples) *n_triples = st->n;
    if (base_index) *base_index = st->base;
  });
}

int tidq_store_download(tidq_store* st, uint64_t lo, uint64_t n, uint32_t* aos_out) {
  return guarded([&] {
    TIDQ_REQUIRE(st && (aos_out || n == 0), TIDQ_E_INVALID, "null argument");
    TIDQ_REQUIRE(lo + n <= st->n, TIDQ_E_INVALID, "row range out of bounds");
    if (n == 0) return;
    Ctx* c = st->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    std::vector<uint32_t> tmp(n);
    const uint32_t* cols[3] = {st->s.as<uint32_t>(), st->p.as<uint32_t>(), st->o.as<uint32_t>()};
    for (int k = 0; k < 3; ++k) {
      TIDQ_CUDA(cudaMemcpyAsync(tmp.data(), cols[k] + lo, n * 4, cudaMemcpyDeviceToHost, c->stream));
      sync(c);
      for (uint64_t i = 0; i < n; ++i) aos_out[i * 3 + k] = tmp[i];
    }
  });
}

int tidq_store_col_max(tidq_store* st, int32_t col, uint32_t* out) {
  return guarded([&] {
    TIDQ_REQUIRE(st && out && col >= 0 && col < 3, TIDQ_E_INVALID, "bad argument");
    Ctx* c = st->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    const DevBuf& b = col == 0 ? st->s : (col == 1 ? st->p : st->o);
    *out = prims::max_u32(c, b.as<uint32_t>(), st->n);
  });
}

int tidq_store_free(tidq_store* st) {
  return guarded([&] {
    if (!st) return;
    Ctx* c = st->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    delete st;
    sync(c);
  });
}

// ---- tables --------------------------------------------------------------

int tidq_table_info(const tidq_table* t, uint64_t* n_rows, int32_t* n_cols) {
  return guarded([&] {
    TIDQ_REQUIRE(t, TIDQ_E_INVALID, "null table");
    if (n_rows) {
      std::lock_guard<std::mutex> lk(t->ctx->mu);
      DeviceGuard g(t->ctx);
      *n_rows = const_cast<tidq_table*>(t)->n_rows();
    }
    if (n_cols) *n_cols = int32_t(t->cols.size());
  });
}

int tidq_table_ncols(const tidq_table* t, int32_t* n_cols) {
  return guarded([&] {
    TIDQ_REQUIRE(t && n_cols, TIDQ_E_INVALID, "null argument");
    *n_cols = int32_t(t->cols.size());
  });
}

int tidq_table_col_dtype(const tidq_table* t, int32_t col, int32_t* dtype) {
  return guarded([&] {
    TIDQ_REQUIRE(t && dtype, TIDQ_E_INVALID, "null argument");
    TIDQ_REQUIRE(col >= 0 && col < int32_t(t->cols.size()), TIDQ_E_INVALID, "column out of range");
    *dtype = t->cols[col].dtype;
  });
}

int tidq_table_download_col(tidq_table* t, int32_t col, void* host_out) {
  return guarded([&] {
    TIDQ_REQUIRE(t, TIDQ_E_INVALID, "null table");
    TIDQ_REQUIRE(col >= 0 && col < int32_t(t->cols.size()), TIDQ_E_INVALID, "column out of range");
    Ctx* c = t->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    if (t->n_rows() == 0) return;
    TIDQ_REQUIRE(host_out, TIDQ_E_INVALID, "null output");
    const Column& k = t->cols[col];
    TIDQ_CUDA(cudaMemcpyAsync(host_out, k.buf.ptr, t->n_rows() * Column::width(k.dtype),
                              cudaMemcpyDeviceToHost, c->stream));
    sync(c);
  });
}

int tidq_table_upload_u32(tidq_ctx* ctx, int32_t n_cols, const uint32_t* const* cols,
                          uint64_t n_rows, tidq_table** out) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx && out && n_cols >= 0, TIDQ_E_INVALID, "bad argument");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx);
    auto t = std::make_unique<tidq_table>();
    t->ctx = ctx;
    t->set_rows(n_rows);
    t->capacity = n_rows;
    for (int32_t k = 0; k < n_cols; ++k) {
      Column col;
      col.dtype = TIDQ_U32;
      col.buf = DevBuf(ctx, n_rows * 4);
      if (n_rows) {
        TIDQ_REQUIRE(cols && cols[k], TIDQ_E_INVALID, "null column");
        TIDQ_CUDA(cudaMemcpyAsync(col.buf.ptr, cols[k], n_rows * 4, cudaMemcpyHostToDevice,
                                  ctx->stream));
      }
      t->cols.push_back(std::move(col));
    }
    sync(ctx);
    *out = t.release();
  });
}

int tidq_table_free(tidq_table* t) {
  return guarded([&] {
    if (!t) return;
    Ctx* c = t->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    delete t;
  });
}

// ---- FILTER bitmaps ------------------------------------------------------

int tidq_bitmap_upload(tidq_ctx* ctx, const uint32_t* words, uint64_t n_bits, tidq_bitmap** out) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx && out && (words || n_bits == 0), TIDQ_E_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx);
    auto b = std::make_unique<tidq_bitmap>();
    b->ctx = ctx;
    b->n_bits = n_bits;
    const uint64_t n_words = (n_bits + 31) / 32;
    b->words = DevBuf(ctx, std::max<uint64_t>(n_words, 1) * 4);
    if (n_words)
      TIDQ_CUDA(cudaMemcpyAsync(b->words.ptr, words, n_words * 4, cudaMemcpyHostToDevice,
                                ctx->stream));
    sync(ctx);
    *out = b.release();
  });
}

int tidq_bitmap_create(tidq_ctx* ctx, uint64_t n_bits, tidq_bitmap** out) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx && out, TIDQ_E_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx);
    auto b = std::make_unique<tidq_bitmap>();
    b->ctx = ctx;
    b->n_bits = n_bits;
    const uint64_t n_words = std::max<uint64_t>((n_bits + 31) / 32, 1);
    b->words = DevBuf(ctx, n_words * 4);
    TIDQ_CUDA(cudaMemsetAsync(b->words.ptr, 0, n_words * 4, ctx->stream));  // stream-ordered
    *out = b.release();
  });
}

int tidq_bitmap_free(tidq_bitmap* b) {
  return guarded([&] {
    if (!b) return;
    Ctx* c = b->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c);
    delete b;
  });
}

}  // extern "C"

// ---- timing / profiling ----------------------------------------------------

cudaEvent_t tidq_ctx::prof_begin(cudaStream_t s) {
  if (!profiling) return nullptr;
  cudaEvent_t e = take_event();
  TIDQ_CUDA(cudaEventRecord(e, s));
  return e;
}

void tidq_ctx::prof_end(const char* name, cudaEvent_t begin, cudaStream_t s, uint64_t algo_bytes,
                        uint64_t launches) {
  if (!begin) return;
  cudaEvent_t e = take_event();
  TIDQ_CUDA(cudaEventRecord(e, s));
  KernelProf& kp = prof[name];
  kp.events.emplace_back(begin, e);
  kp.launches += launches;
  kp.bytes += algo_bytes;
}

static void resolve_prof(tidq_ctx* c) {
  for (auto& kv : c->prof) {
    auto& kp = kv.second;
    if (kp.events.empty()) continue;
    TIDQ_CUDA(cudaEventSynchronize(kp.events.back().second));
    for (auto& ev : kp.events) {
      float ms = 0;
      TIDQ_CUDA(cudaEventElapsedTime(&ms, ev.first, ev.second));
      kp.ms += ms;
      c->event_pool.push_back(ev.first);
      c->event_pool.push_back(ev.second);
    }
    kp.events.clear();
  }
}

extern "C" {

int tidq_timer_begin(tidq_ctx* ctx) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx, TIDQ_E_INVALID, "null ctx");
    DeviceGuard g(ctx);
    for (auto& e : ctx->timer)
      if (!e) TIDQ_CUDA(cudaEventCreate(&e));
    TIDQ_CUDA(cudaEventRecord(ctx->timer[0], ctx->stream));
  });
}

int tidq_timer_end(tidq_ctx* ctx, double* ms) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx && ms && ctx->timer[0], TIDQ_E_INVALID, "timer not started");
    DeviceGuard g(ctx);
    TIDQ_CUDA(cudaEventRecord(ctx->timer[1], ctx->stream));
    TIDQ_CUDA(cudaEventSynchronize(ctx->timer[1]));
    float f = 0;
    TIDQ_CUDA(cudaEventElapsedTime(&f, ctx->timer[0], ctx->timer[1]));
    *ms = f;
  });
}

int tidq_profile_enable(tidq_ctx* ctx, int on) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx, TIDQ_E_INVALID, "null ctx");
    ctx->profiling = on != 0;
  });
}

int tidq_profile_read(tidq_ctx* ctx, const char* kernel, double* total_ms, uint64_t* launches,
                      uint64_t* algo_bytes) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx && kernel, TIDQ_E_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx);
    resolve_prof(ctx);
    auto it = ctx->prof.find(kernel);
    const bool have = it != ctx->prof.end();
    if (total_ms) *total_ms = have ? it->second.ms : 0.0;
    if (launches) *launches = have ? it->second.launches : 0;
    if (algo_bytes) *algo_bytes = have ? it->second.bytes : 0;
  });
}

int tidq_profile_reset(tidq_ctx* ctx) {
  return guarded([&] {
    TIDQ_REQUIRE(ctx, TIDQ_E_INVALID, "null ctx");
    std::lock_guard<std::mutex> lk(ctx->mu);
    DeviceGuard g(ctx);
    resolve_prof(ctx);
    ctx->prof.clear();
  });
}

}  // extern "C"
