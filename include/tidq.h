/*
 * tidq.h — C ABI of libtidq.so, the B200 (sm_100a) TripleID-Q query path.
 *
 * The reference (`/root/reference/pkg/src/tripleid`, pure Python + numpy) has
 * no FFI: its operator API *is* the Python module surface.  Every entry point
 * below is what a ctypes binding of that surface needs; each cites the
 * reference function it replaces.  The Python mirror in
 * `paper_1807_01409_b200/` binds exactly these symbols.
 *
 * Conventions
 *  - Every call returns an int status: TIDQ_OK (0) or a negative TIDQ_E_*.
 *    The message of the last failure on the calling thread is returned by
 *    tidq_last_error().  No C++ exception ever crosses this boundary.
 *  - Host buffers passed in are BORROWED for the duration of the call.
 *    Device objects (ctx, store, table, bitmap) are owned by opaque handles
 *    and released with the matching *_free / *_destroy call.
 *  - All calls are synchronous on return (stream-ordered per ctx) and
 *    serialised per ctx by an internal mutex.  Calls on different ctx
 *    handles may run concurrently.
 *  - Term IDs are uint32 and 0 is the wildcard, never stored
 *    (reference store.py:28, store.py:89-93, dictionary.py:25).
 */
#ifndef TIDQ_H
#define TIDQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TIDQ_ABI_VERSION 1

/* ---- status codes ------------------------------------------------------ */
#define TIDQ_OK 0
#define TIDQ_E_INVALID (-1)      /* bad argument            -> ValueError            */
#define TIDQ_E_CUDA (-2)         /* CUDA runtime failure     -> RuntimeError          */
#define TIDQ_E_NOMEM (-3)        /* device/host allocation   -> MemoryError           */
#define TIDQ_E_TOO_MANY_KEYS (-4)/* k outside 1..32          -> TooManySubqueries     */
#define TIDQ_E_ROW_CAP (-5)      /* join above row cap       -> ResourceLimit         */
#define TIDQ_E_NCCL (-6)         /* NCCL failure             -> RuntimeError          */
#define TIDQ_E_UNSUPPORTED (-7)  /* feature not built in     -> NotImplementedError   */
#define TIDQ_E_IO (-8)           /* file open/read failure   -> OSError               */
#define TIDQ_E_BAD_MAGIC (-9)    /* .tid magic != "TID1"     -> BadMagic              */
#define TIDQ_E_BAD_VERSION (-10) /* .tid version != 1        -> BadVersion            */
#define TIDQ_E_TRUNCATED (-11)   /* .tid shorter than header -> TruncatedFile         */
#define TIDQ_E_PARSE (-12)       /* malformed N-Triples line -> ParseError (strict)   */

/* kernel.py:33 MAX_SUBQUERIES */
#define TIDQ_MAX_KEYS 32
#define TIDQ_MAX_STREAMS 32
#define TIDQ_MAX_OUT 4
#define TIDQ_MAX_FILTERS 2

typedef struct tidq_ctx tidq_ctx;       /* one CUDA device + stream + pool    */
typedef struct tidq_store tidq_store;   /* resident SoA s/p/o columns (HBM)   */
typedef struct tidq_table tidq_table;   /* device columns of equal length     */
typedef struct tidq_bitmap tidq_bitmap; /* device bitset over term IDs        */

/* ---- runtime ----------------------------------------------------------- */
int tidq_abi_version(void);
const char* tidq_last_error(void);
int tidq_device_count(int* n);
int tidq_ctx_create(int device, tidq_ctx** out);
/* free / total device memory of the ctx's device (cudaMemGetInfo) */
int tidq_ctx_mem_info(tidq_ctx* ctx, uint64_t* free_bytes, uint64_t* total_bytes);
/* Return the context's unused pooled device memory to the driver (waits for
 * the ctx stream).  The pool keeps freed memory for reuse (no cudaMalloc on
 * the query path); a caller switching between working sets of very
 * different sizes trims between them. */
int tidq_ctx_trim(tidq_ctx* ctx);
int tidq_ctx_destroy(tidq_ctx* ctx);
int tidq_ctx_sync(tidq_ctx* ctx);
/* number of libtidq kernels launched on this ctx so far (evidence counter) */
int tidq_ctx_launches(tidq_ctx* ctx, uint64_t* n);
/* pinned host memory for H2D/D2H at full PCIe rate (bench e2e inputs) */
int tidq_host_alloc(uint64_t bytes, void** out);
int tidq_host_free(void* p);

/* device-side timing on the ctx stream (CUDA events; never wall clock) */
int tidq_timer_begin(tidq_ctx* ctx);
int tidq_timer_end(tidq_ctx* ctx, double* ms); /* synchronises the ctx stream */
/* Per-kernel accounting for the roofline: while enabled, every launch of the
 * named hot kernel ("scan", ...) is bracketed by events on its own stream and
 * its ALGORITHMIC bytes are accumulated. */
int tidq_profile_enable(tidq_ctx* ctx, int on);
int tidq_profile_read(tidq_ctx* ctx, const char* kernel, double* total_ms, uint64_t* launches,
                      uint64_t* algo_bytes);
int tidq_profile_reset(tidq_ctx* ctx);

/* ---- store (reference store.py) ---------------------------------------- */
/* TripleChunk(data, base_index) -> resident SoA.  `aos` is the flat
 * [s0,p0,o0,s1,...] uint32 array of store.py:61-79; copied H2D in pipelined
 * slabs and transposed on the device into three 16-B aligned columns. */
int tidq_store_upload(tidq_ctx* ctx, const uint32_t* aos, uint64_t n_triples,
                      uint64_t base_index, tidq_store** out);

/* Late materialisation: a new table whose column k is, for spec[k] >= 0,
 * column spec[k] of `t` (moved out of `t`, which is left without those
 * columns), and for spec[k] = -1 - slot, the store column `slot` (0=s 1=p
 * 2=o) gathered at the uint32 local triple indices in column `idx_col` of `t`.
 * Used by query_ops' semi-join-reduced scan. */
int tidq_store_gather_cols(tidq_store* st, tidq_table* t, int32_t idx_col, int32_t n_out,
                           const int32_t* spec, tidq_table** out);
/* tidq_store_gather_cols with an index column per gathered output: spec[k] <
 * 0 gathers store slot -1-spec[k] at the local triple indices of column
 * idx_cols[k] (several patterns' deferred variables in one pass, <= 8
 * gathered outputs); spec[k] >= 0 takes table column spec[k]. */
int tidq_store_gather_cols_multi(tidq_store* st, tidq_table* t, int32_t n_out, const int32_t* spec,
                                 const int32_t* idx_cols, tidq_table** out);

/* A whole .tid file (store.py:1-10: 16-B header "<4sIQ" = "TID1", 1, count,
 * then count x 3 little-endian uint32) -> resident SoA, without a Python
 * round trip: parallel pread into page-locked double buffers, H2D on the copy
 * stream, AoS->SoA transpose on the compute stream.  Replaces the
 * read_chunks + per-chunk upload path of store.py:107-153 for stores that fit
 * in HBM (chunk-invariant results).  Errors match read_header /
 * read_chunks: TIDQ_E_BAD_MAGIC, TIDQ_E_BAD_VERSION, TIDQ_E_TRUNCATED. */
int tidq_store_load_tid(tidq_ctx* ctx, const char* path, uint64_t base_index, tidq_store** out);
/* Rows [row_lo, row_lo + row_count) of a .tid file (row_count clamped to the
 * file; UINT64_MAX = to the end), global indices base_index + row_lo ...:
 * the row-sharded load of one rank's contiguous range.  Replaces the
 * base-index iteration of read_chunks (reference store.py:121-146) for an
 * arbitrary row range.  Header errors as tidq_store_load_tid; row_lo beyond
 * the file's count -> TIDQ_E_INVALID. */
int tidq_store_load_tid_range(tidq_ctx* ctx, const char* path, uint64_t row_lo, uint64_t row_count,
                              uint64_t base_index, tidq_store** out);

/* Counter-based synthetic store, generated on the device.
 * Triple i (global index base_index+i):
 *   h_j = splitmix64(((i<<2)|j) ^ (seed*0xD1B54A32D192ED03)), j=0,1,2
 *   p   = 1 + first r with h_1 < zipf_cdf[r]
 *   s   = n_p + 1 + (((h_0>>32) * n_e) >> 32)
 *   o   = n_p + 1 + (((h_2>>32) * n_e) >> 32)                           */
typedef struct {
  uint64_t n_triples;   /* triples in this store (shard)               */
  uint64_t base_index;  /* global index of the first triple            */
  uint64_t seed;
  uint32_t n_p;         /* predicates: IDs 1..n_p                       */
  uint32_t n_e;         /* entities:   IDs n_p+1..n_p+n_e               */
} tidq_synth_params;
int tidq_store_generate(tidq_ctx* ctx, const tidq_synth_params* params,
                        const uint64_t* zipf_cdf /* n_p entries, host */,
                        tidq_store** out);
int tidq_store_info(const tidq_store* st, uint64_t* n_triples, uint64_t* base_index);
/* copy rows [lo, lo+n) back as AoS (tests, gather_rows) */
int tidq_store_download(tidq_store* st, uint64_t lo, uint64_t n, uint32_t* aos_out);
/* rows at local indices (int64, any order) -> AoS; kernel.py:257-266 gather_rows */
int tidq_store_gather(tidq_store* st, const int64_t* local_idx, uint64_t n, uint32_t* aos_out);
/* max ID of one column (0=s 1=p 2=o); 0 for an empty store */
int tidq_store_col_max(tidq_store* st, int32_t col, uint32_t* out);
/* counts[p] for p in [0, max_id] over the predicate column: exact output
 * sizes (capacity hints) for ?P? keys, so a scan needs no mid-pass host sync */
int tidq_store_pred_hist(tidq_store* st, uint32_t max_id, uint64_t* counts_out);
/* Predicate-code column (a B200 layout choice; no reference counterpart):
 * pvals = the store's distinct predicate IDs, strictly ascending, at most
 * 30000 of them, each below 2^28.  Builds a 16-bit column of each triple's
 * predicate rank, which the scan's mark then streams instead of the uint32
 * predicate column whenever a pass binds only the predicate (env TIDQ_P16=0
 * disables it).  n_vals = 0 drops the column.  Results are unchanged. */
int tidq_store_pcodes(tidq_store* st, const uint32_t* pvals, uint32_t n_vals);
/* Interleaved (subject, object) pair column (a B200 layout choice; no
 * reference counterpart): 8 B per triple more HBM; the scan's emit then reads
 * a row that needs both ?s and ?o with one 8-byte gather (env TIDQ_SO=0
 * disables its use).  enable = 0 drops it.  Results are unchanged. */
int tidq_store_so(tidq_store* st, int32_t enable);
int tidq_store_free(tidq_store* st);

/* ---- scan (reference kernel.py search_chunk / search_multi,
 *            query_ops.py scan_patterns + pattern_table + apply_filter) ---- */
/* Output field kinds of one stream */
#define TIDQ_OUT_S 0       /* uint32 subject of the triple               */
#define TIDQ_OUT_P 1       /* uint32 predicate                           */
#define TIDQ_OUT_O 2       /* uint32 object                              */
#define TIDQ_OUT_INDEX 3   /* int64 global triple index (base_index + i) */
#define TIDQ_OUT_MARKS 4   /* uint32 mark set, bit q = key q accepts     */
#define TIDQ_OUT_ANSWER 5  /* uint8 answer code vs keys[answer_key]      */
#define TIDQ_OUT_LOCAL 6   /* uint32 triple index within the store (i)   */

/* repeated-variable equalities (query_ops.py:220-225) */
#define TIDQ_EQ_SP 1u
#define TIDQ_EQ_SO 2u
#define TIDQ_EQ_PO 4u

typedef struct {
  uint32_t select;      /* element belongs to the stream iff marks & select != 0 */
  uint32_t eq_flags;    /* TIDQ_EQ_* slot equalities the row must satisfy        */
  int32_t n_out;        /* output fields, <= TIDQ_MAX_OUT                        */
  int32_t out[TIDQ_MAX_OUT];
  int32_t answer_key;   /* key index for TIDQ_OUT_ANSWER                          */
  int32_t n_filters;    /* FILTER regex(str(?v)) as accepted-ID bitmaps           */
  int32_t filter_slot[TIDQ_MAX_FILTERS];            /* 0=s 1=p 2=o               */
  const tidq_bitmap* filter[TIDQ_MAX_FILTERS];
  uint64_t capacity_hint; /* 0: library estimates; overflow is retried exactly  */
  tidq_bitmap* key_bitmap; /* optional: the emit ORs in the bit of every row's   */
  int32_t key_bitmap_slot; /* value in this slot (0=s 1=p 2=o): a join's key set */
} tidq_stream_spec;

typedef struct {
  int32_t n_keys;                       /* 1..32 (kernel.py:196-197)    */
  uint32_t keys[TIDQ_MAX_KEYS][3];      /* (s,p,o), 0 = free            */
  int32_t n_streams;                    /* 1..32                        */
  tidq_stream_spec streams[TIDQ_MAX_STREAMS];
  uint32_t flags;                       /* TIDQ_SCAN_*                  */
  uint32_t* write_counts;               /* optional HOST array of n_triples counters: the
                                           mark pass adds 1 to every triple slot it writes
                                           (the reference's write_counts instrumentation,
                                           kernel.py:153,172-173,221-222: disjointness) */
} tidq_scan_spec;

/* Every stream's capacity_hint is a guaranteed upper bound of its row count
 * (e.g. the store's predicate histogram for keys that bind the predicate):
 * tidq_scan returns as soon as the work is queued, without waiting for the
 * device.  The tables' row counts are resolved on first use (tidq_table_info,
 * any operator taking the table, download, free), which waits for the scan.
 * Consecutive queries therefore queue back to back on the ctx stream. */
#define TIDQ_SCAN_ASYNC 1u
/* All streams write ONE table, stream 0's rows first, then stream 1's, ...
 * (each in ascending triple order): out_tables[0] holds the rows of every
 * stream, out_tables[1..] are empty.  The streams must have the same output
 * types and every stream a capacity_hint.  This is the UNION of
 * single-pattern branches (query_ops.py:359-376) without a concatenation
 * pass; no predicate is deferred to a post-filter. */
#define TIDQ_SCAN_CONCAT 2u

/* One pass over the store: every key tested per triple, each stream
 * compacted in ascending triple order (order-preserving, deterministic).
 * out_tables[i] receives stream i's table; its columns are the stream's
 * output fields in order. */
int tidq_scan(tidq_store* st, const tidq_scan_spec* spec, tidq_table** out_tables);

/* Operator-compatible host-buffer scan (kernel.py:148-227): uploads the AoS
 * chunk, scans, downloads.  Two-step: the call returns counts and a table
 * handle; download with tidq_table_download_col, then free. */
int tidq_scan_host(tidq_ctx* ctx, const uint32_t* aos, uint64_t n_triples,
                   uint64_t base_index, const tidq_scan_spec* spec,
                   tidq_table** out_tables);

/* ---- tables (reference query_ops.py BindingTable / pair arrays) -------- */
#define TIDQ_U32 0
#define TIDQ_I64 1
#define TIDQ_U8 2
int tidq_table_info(const tidq_table* t, uint64_t* n_rows, int32_t* n_cols);
/* column count only: never waits for a deferred row count (TIDQ_SCAN_ASYNC) */
int tidq_table_ncols(const tidq_table* t, int32_t* n_cols);
int tidq_table_col_dtype(const tidq_table* t, int32_t col, int32_t* dtype);
int tidq_table_download_col(tidq_table* t, int32_t col, void* host_out);
/* n_cols uint32 host columns of n rows -> device table */
int tidq_table_upload_u32(tidq_ctx* ctx, int32_t n_cols, const uint32_t* const* cols,
                          uint64_t n_rows, tidq_table** out);
int tidq_table_free(tidq_table* t);

/* ---- table operators (reference query_ops.py) ---------------------------- */
/* UNION (query_ops.py:359-376): rows of the tables in order; output column k
 * of table i is its column src_cols[i*n_out_cols+k], or UNBOUND (0) if -1. */
int tidq_table_concat(tidq_ctx* ctx, int32_t n_tables, tidq_table* const* tables,
                      int32_t n_out_cols, const int32_t* src_cols, tidq_table** out);
/* column subset copy (projection, query_ops.py:386-390) */
int tidq_table_project(tidq_table* t, int32_t n_cols, const int32_t* cols, tidq_table** out);
/* rows whose `col` ID has its bit set in the bitmap, order kept (the isin of
 * apply_filter, query_ops.py:251-252) */
int tidq_table_filter_bitmap(tidq_table* t, int32_t col, const tidq_bitmap* b, tidq_table** out);
/* ascending distinct values of one column (np.unique of apply_filter,
 * query_ops.py:247) -> one-column table */
int tidq_table_unique_col(tidq_table* t, int32_t col, tidq_table** out);
/* DISTINCT over `cols` keeping the first occurrence of each row, in
 * first-occurrence order (query_ops.py:391-399) */
int tidq_distinct(tidq_table* t, int32_t n_cols, const int32_t* cols, tidq_table** out);
/* tidq_distinct with a bound on every value of the columns (> each value, e.g.
 * the store's largest term ID + 1), which replaces the max pass and its host
 * round trip; 0: measured as tidq_distinct does. */
int tidq_distinct_bound(tidq_table* t, int32_t n_cols, const int32_t* cols, uint64_t key_bound,
                        tidq_table** out);

/* One join step of join_group (query_ops.py:316-341): pairs of rows with
 * left[lkey] == right[rkey] in merge_join order (key, left row, right row —
 * query_ops.py:144-177); ResourceLimit (TIDQ_E_ROW_CAP) if the pair count
 * exceeds row_cap (row_cap < 0: no cap); output columns gathered from either
 * side; rows failing any eq pair (left col == right col) dropped. */
typedef struct {
  int32_t side; /* 0 = left, 1 = right */
  int32_t col;
} tidq_colref;
/* tidq_join `algo` flags */
#define TIDQ_JOIN_REDUCED 1  /* inputs already semi-join reduced: skip the key-bitmap pre-filter */
int tidq_join(tidq_table* left, int32_t lkey, tidq_table* right, int32_t rkey, int32_t n_out,
              const tidq_colref* out_cols, int32_t n_eq, const int32_t* eq_pairs /* [n_eq][2] */,
              int64_t row_cap, int32_t algo /* TIDQ_JOIN_* flags, 0 = default */,
              uint64_t key_bound /* > every key (e.g. store max ID + 1), 0 = computed */,
              const tidq_bitmap* lkeys_bm, const tidq_bitmap* rkeys_bm /* optional key sets of
              the two sides (a superset is fine: e.g. built by the scan), key_bound bits */,
              tidq_table** out, uint64_t* n_pairs);
/* merge_join drop-in (query_ops.py:144-177): host key vectors -> table of two
 * int64 columns (l, r) in (key, l, r) order */
/* Semi-join reduction on one join variable: tables[i] keeps the rows whose
 * key (uint32 column key_cols[i]) occurs in EVERY other table's key column;
 * row order is kept.  A row without a partner in some table that binds the
 * variable cannot appear in the join of all of them (query_ops.py:298-342
 * joins every pattern of a group), so the join result is unchanged.
 * out[i] receives the reduced table i. */
int tidq_tables_semijoin(int32_t n_tables, tidq_table* const* tables, const int32_t* key_cols,
                         uint64_t n_bits /* > every key; 0: computed */, tidq_table** out);

/* BindingRelation.prepare_for_join (query_ops.py:110-118): stable argsort of
 * n uint32 keys (np.argsort(kind="stable")); host in, host out. */
int tidq_argsort_u32(tidq_ctx* ctx, const uint32_t* keys, uint64_t n, uint32_t* sorted_out,
                     uint32_t* perm_out);

/* Diagnostics (tests, tools/sort_bench.py; replaces no reference interface):
 * stable radix sort of n host (key, value) pairs by the low `bits` key bits
 * (key_bytes 4 or 8; sorted in place, host in / host out) with the active
 * implementation (onesweep; env TIDQ_RADIX=lsd: the three-kernel LSD passes).
 * reps > 0 also times reps device sorts of the same input (CUDA events around
 * each sort, input restored outside them) -> *ms_per_sort. */
int tidq_debug_radix_sort(tidq_ctx* ctx, int32_t key_bytes, void* keys, uint32_t* vals, uint64_t n,
                          int32_t bits, int32_t reps, double* ms_per_sort);

/* merge_join (query_ops.py:144-177): (l, r) int64 pairs in (key, l, r) order. */
int tidq_merge_join_pairs(tidq_ctx* ctx, const uint32_t* lkeys, uint64_t nl, const uint32_t* rkeys,
                          uint64_t nr, tidq_table** out);

/* ---- multi-GPU exchange (the paper's multi-GPU/MPI plan,
 *      PAPER.md:494-495) — one process per GPU, NCCL over NVLink ---------- */
typedef struct tidq_comm tidq_comm;
#define TIDQ_COMM_ID_BYTES 128
/* rank 0 creates the id and hands it to every rank (e.g. torch.distributed) */
int tidq_comm_unique_id(uint8_t* id_out /* TIDQ_COMM_ID_BYTES */);
int tidq_comm_create(tidq_ctx* ctx, const uint8_t* id, int32_t nranks, int32_t rank, tidq_comm** out);
int tidq_comm_destroy(tidq_comm* comm);
/* payload bytes this rank sent to OTHER ranks through tidq_table_alltoallv
 * and the device time of those exchanges since the last reset (NVLink
 * roofline accounting: bytes / time vs ~900 GB/s per direction per GPU) */
int tidq_comm_stats(tidq_comm* comm, int32_t reset, uint64_t* bytes_out, double* exchange_ms);
/* rows grouped (stably) by destination rank
 *   h = 0; for each key column v: h = (h ^ v) * 0x9E3779B97F4A7C15 mod 2^64
 *   dest = (h >> 32) % nranks;   counts[r] = rows for rank r */
int tidq_table_partition(tidq_table* t, int32_t n_key_cols, const int32_t* key_cols, int32_t nranks,
                         tidq_table** out, uint64_t* counts);
/* variable all-to-all of a partitioned table (send_counts[r] rows to rank r);
 * received rows are in source-rank order; recv_counts may be NULL */
int tidq_table_alltoallv(tidq_comm* comm, tidq_table* t, const uint64_t* send_counts, tidq_table** out,
                         uint64_t* recv_counts);
/* elementwise sum of n uint64 values over all ranks (pair counts vs row_cap) */
int tidq_comm_allreduce_u64(tidq_comm* comm, const uint64_t* in, uint64_t* out, int32_t n);
/* every rank's rows in rank order (small build sides, result collection) */
int tidq_table_allgather(tidq_comm* comm, tidq_table* t, tidq_table** out);

/* ---- FILTER (query_ops.py:232-252) ------------------------------------ */
/* accepted-ID bitset: bit id set iff regex(str(lexical(id))) matched on host */
int tidq_bitmap_upload(tidq_ctx* ctx, const uint32_t* words, uint64_t n_bits, tidq_bitmap** out);
/* an all-zero device bitmap (e.g. a scan stream's key_bitmap target) */
int tidq_bitmap_create(tidq_ctx* ctx, uint64_t n_bits, tidq_bitmap** out);
int tidq_bitmap_free(tidq_bitmap* b);

/* ---- N-Triples -> TripleID conversion (host cores) ---------------------------
 * The reference's cmd_convert (cli.py:64-114): nt.parse_stream (nt.py:196-224)
 * + Dictionary.encode in first-occurrence order (dictionary.py:71-80) +
 * write_tid (store.py:97-104) + write_id_files (dictionary.py:98-107), parsed
 * by `threads` host threads (0 = all cores).  Writes the reference's
 * temporary files <out_prefix>.tid.tmp and <out_prefix>.tmp.{sid,pid,oid}
 * (the caller renames them, as cli.py:88-91 does); their bytes equal the
 * reference's.  strict != 0: the first malformed line in stream order ->
 * TIDQ_E_PARSE, tidq_last_error() = "line N, byte B: message" (nt.ParseError),
 * nothing written.  Lenient: malformed lines are skipped and counted; with
 * errors_tsv non-null, *errors_tsv receives a malloc'd "line\tbyte\tmessage\n"
 * list (free with tidq_convert_free).  I/O failures -> TIDQ_E_IO with
 * report->io_errno / io_path set. */
typedef struct {
  uint64_t triples;           /* statements converted = .tid rows              */
  uint64_t terms;             /* dictionary size (largest ID)                  */
  uint64_t distinct[3];       /* Dictionary.role_counts(): s, p, o             */
  uint64_t skipped_lines;     /* blank and comment lines (ParseReport.skipped) */
  uint64_t parse_errors;      /* malformed lines skipped (lenient)             */
  uint64_t file_bytes[4];     /* .tid .sid .pid .oid sizes                     */
  uint64_t first_error_line;  /* strict: the failing line and byte offset      */
  uint64_t first_error_offset;
  int32_t io_errno;
  char io_path[4096];
} tidq_convert_report;

int tidq_convert_nt(const char* input, const char* out_prefix, int strict, int threads,
                    tidq_convert_report* report, char** errors_tsv);
int tidq_convert_free(char* p);

#ifdef __cplusplus
}
#endif
#endif /* TIDQ_H */
