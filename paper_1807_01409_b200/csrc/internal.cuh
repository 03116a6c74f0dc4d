// Internal runtime types of libtidq: device context, resident store, device
// tables and the error plumbing that turns CUDA failures into ABI status codes.
#pragma once

#include <cuda_runtime.h>
#include <utility>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tidq.h"

namespace tidq {

// ---- errors ---------------------------------------------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

#define TIDQ_CUDA(call)                                                           \
  do {                                                                            \
    cudaError_t _e = (call);                                                      \
    if (_e != cudaSuccess) {                                                      \
      throw ::tidq::Error(_e == cudaErrorMemoryAllocation ? TIDQ_E_NOMEM          \
                                                          : TIDQ_E_CUDA,          \
                          std::string(#call) + ": " + cudaGetErrorString(_e));    \
    }                                                                             \
  } while (0)

#define TIDQ_REQUIRE(cond, code, msg)                  \
  do {                                                 \
    if (!(cond)) throw ::tidq::Error((code), (msg));   \
  } while (0)

// Wrap an ABI entry point body: exceptions -> status + thread-local message.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return TIDQ_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return TIDQ_E_NOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return TIDQ_E_CUDA;
  }
}

}  // namespace tidq

struct tidq_ctx;

namespace tidq {
using Ctx = ::tidq_ctx;

// ---- device buffer (stream-ordered pool allocation) -------------------------

struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  Ctx* ctx = nullptr;
  DevBuf() = default;
  DevBuf(Ctx* c, size_t b);
  ~DevBuf();
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
  DevBuf& operator=(DevBuf&& o) noexcept;
  void reset();
  template <class T>
  T* as() const { return static_cast<T*>(ptr); }
};

}  // namespace tidq

// ---- opaque handle definitions (global namespace, as declared in tidq.h) ---
struct tidq_ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;   // compute stream
  cudaStream_t copy_stream = nullptr;
  // second compute stream: independent halves of an operator (the two join
  // sides' sorts) run on it concurrently, forked / joined by the events
  cudaStream_t side_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaMemPool_t pool = nullptr;
  std::mutex mu;
  uint64_t launches = 0;
  // scratch reused across scans (grown on demand)
  tidq::DevBuf lookback;           // scan bitmaps, tile counts, offsets
  tidq::DevBuf ssum;               // scan super-tile sums: all zero between scans
  bool ssum_clean = false;
  tidq::DevBuf staging[2];         // H2D slabs for upload
  void* pinned_slab[2] = {nullptr, nullptr};  // page-locked read slabs (.tid ingest)
  void* pinned_small = nullptr;    // 4 KiB pinned scratch for counts
  // pinned slots receiving the row counts of deferred (TIDQ_SCAN_ASYNC) tables
  static constexpr int kRowSlots = 4096;
  uint64_t* row_slots = nullptr;
  std::vector<int> free_row_slots;
  char* host_scratch = nullptr;    // pinned: super-tile sums / offsets of a scan
  size_t host_scratch_bytes = 0;
  char* pinned_scratch(size_t bytes) {
    if (bytes > host_scratch_bytes) {
      if (host_scratch) cudaFreeHost(host_scratch);
      host_scratch = nullptr;
      host_scratch_bytes = 0;
      if (cudaMallocHost(reinterpret_cast<void**>(&host_scratch), bytes) != cudaSuccess)
        throw tidq::Error(TIDQ_E_NOMEM, "pinned host allocation failed");
      host_scratch_bytes = bytes;
    }
    return host_scratch;
  }
  void count_launch(uint64_t n = 1) { launches += n; }
  // device timers and per-kernel profiling (events on the launching stream)
  cudaEvent_t timer[2] = {nullptr, nullptr};
  bool profiling = false;
  struct KernelProf {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
    double ms = 0;           // resolved time
    uint64_t launches = 0;
    uint64_t bytes = 0;      // algorithmic bytes
  };
  std::map<std::string, KernelProf> prof;
  std::vector<cudaEvent_t> event_pool;  // recycled profiling events
  cudaEvent_t take_event() {
    if (!event_pool.empty()) {
      cudaEvent_t e = event_pool.back();
      event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) throw tidq::Error(TIDQ_E_CUDA, "cudaEventCreate failed");
    return e;
  }
  // bracket a launch: returns true when profiling (caller records end)
  cudaEvent_t prof_begin(cudaStream_t s);
  void prof_end(const char* name, cudaEvent_t begin, cudaStream_t s, uint64_t algo_bytes,
                uint64_t launches = 1);
};

namespace tidq {

// Make ctx current on the calling thread.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(Ctx* c) {
    cudaGetDevice(&prev);
    if (prev != c->device) TIDQ_CUDA(cudaSetDevice(c->device));
  }
  ~DeviceGuard() {}
};

struct Column {
  DevBuf buf;
  int32_t dtype = TIDQ_U32;
  static size_t width(int32_t dt) { return dt == TIDQ_I64 ? 8 : dt == TIDQ_U8 ? 1 : 4; }
};

}  // namespace tidq

struct tidq_store {
  tidq_ctx* ctx = nullptr;
  uint64_t n = 0;        // triples
  uint64_t base = 0;     // global index of triple 0
  uint64_t padded = 0;   // column length (multiple of the scan tile)
  tidq::DevBuf s, p, o;  // SoA columns, zero padded
  // optional predicate-code column: p16[i] = index of p[i] in pvals (the
  // store's distinct predicate IDs, ascending, <= 65535 of them); the scan's
  // mark streams it (2 B per triple) when a pass binds only the predicate
  tidq::DevBuf p16;             // code = rank + kPcodeBase (fp16-normal bit patterns)
  std::vector<uint32_t> pvals;
  // optional interleaved (s, o) pairs: a hit whose row needs both is ONE
  // 8-byte gather, and 16 pairs share a 128-B line (vs 32 values of each of
  // two columns), so sparse emits touch fewer DRAM lines
  tidq::DevBuf so;
};

struct tidq_table {
  tidq_ctx* ctx = nullptr;
  uint64_t capacity = 0;
  std::vector<tidq::Column> cols;
  int32_t sorted_by = -1;  // a column the rows ascend by (a sort-merge join's key), -1: unknown
  // Row count; a TIDQ_SCAN_ASYNC result holds a pinned slot the count is
  // copied into by the stream and resolves (waits) on first use.
  uint64_t n_rows();
  void set_rows(uint64_t n) { rows_ = n; }
  void defer_rows(int slot) { pending_slot_ = slot; }
  bool pending() const { return pending_slot_ >= 0; }
  ~tidq_table();

 private:
  uint64_t rows_ = 0;
  int pending_slot_ = -1;
};

struct tidq_bitmap {
  tidq_ctx* ctx = nullptr;
  uint64_t n_bits = 0;
  tidq::DevBuf words;
};

namespace tidq {
constexpr uint32_t kPcodeBase = 0x400;  // predicate code = rank + base (see store.cu)
constexpr uint32_t kPcodeMax = 30000;   // distinct predicates a code column holds
// kernels (defined in the .cu files)
void launch_transpose_aos(Ctx* c, const uint32_t* aos, uint64_t n, uint32_t* s, uint32_t* p,
                          uint32_t* o, cudaStream_t stream);
void launch_generate(Ctx* c, const tidq_synth_params& prm, const uint64_t* cdf_dev,
                     uint32_t* s, uint32_t* p, uint32_t* o, cudaStream_t stream);
void run_scan(tidq_store* st, const tidq_scan_spec& spec, tidq_table** out);
constexpr uint64_t kScanTile = 8192;  // store padding: a multiple of every scan tile
inline uint64_t round_up(uint64_t x, uint64_t m) { return (x + m - 1) / m * m; }
}  // namespace tidq

namespace tidq {
// Random 4-byte gathers of single-use data: cache in L2 only (no L1 line
// allocation).  DRAM traffic per gather stays ~110 B at 1 % selectivity
// (ncu, profiles/): HBM fetches whole lines for scattered sectors, and
// cudaLimitMaxL2FetchGranularity = 32 did not change it.
__device__ __forceinline__ uint32_t ld_gather(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint2 ld_gather(const uint2* p) {
  uint2 v;
  asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ld_gather(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

// Programmatic dependent launch for chains of table-operator kernels: a
// kernel launched with pdl_chain_launch calls pdl_chain_enter() first (wait
// for the predecessor grid's memory, then release its own successor), so
// back-to-back launches overlap their launch latency.  After a memset or
// copy the dependency is the ordinary full one.
__device__ __forceinline__ void pdl_chain_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
void pdl_chain_launch(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t stream,
                      Args&&... args) {
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
}  // namespace tidq

namespace tidq {
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute is per device, and a process may hold contexts on several.
void ensure_dyn_smem(const void* kernel, int device, int bytes);
// Diagnostic phase timer (env TIDQ_PHASE_TRACE=1): synchronises the ctx
// stream and charges the wall time since the previous mark to `name`;
// phase_report prints and clears the totals.  A no-op when disabled.
void phase_mark(Ctx* c, const char* name);
void phase_report(const char* what);
}  // namespace tidq
