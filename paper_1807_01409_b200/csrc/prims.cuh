// Device primitives shared by the table operators: device-wide exclusive
// scan, stable LSD radix sort of (key, row) pairs, order-preserving
// compaction, gathers.  All hand-written (no CUB/Thrust on the path).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "internal.cuh"

namespace tidq {
namespace prims {

// Exclusive scan of n values (uint32 in, uint64 out); returns the total.
uint64_t exclusive_scan(Ctx* c, const uint32_t* in, uint64_t* out, uint64_t n);
uint64_t exclusive_scan(Ctx* c, const uint64_t* in, uint64_t* out, uint64_t n);
// stream-ordered, no host synchronisation
void exclusive_scan_async(Ctx* c, const uint32_t* in, uint64_t* out, uint64_t n);

// Stable LSD radix sort of (keys, vals) by the low `bits` bits of the key.
// keys/vals are sorted in place (double-buffered internally).
void radix_sort_pairs(Ctx* c, uint32_t* keys, uint32_t* vals, uint64_t n, int bits);
void radix_sort_pairs(Ctx* c, uint64_t* keys, uint32_t* vals, uint64_t n, int bits);
// the number of low key bits radix_sort_pairs(n, bits) actually orders by
// (whole digits: >= bits); keys sorted on `bits` bits are grouped by these
int radix_sorted_bits(uint64_t n, int bits);  // for 64-bit keys

// max of a uint32 column (0 for n = 0); synchronises
uint32_t max_u32(Ctx* c, const uint32_t* x, uint64_t n);
// maxima of k <= 8 columns with one host synchronisation
void max_u32_multi(Ctx* c, int k, const uint32_t* const* x, const uint64_t* n, uint32_t* out);

// out[i] = i
void iota(Ctx* c, uint32_t* out, uint64_t n);
// out[i] = src[idx[i]]
void gather_u32(Ctx* c, const uint32_t* src, const uint32_t* idx, uint32_t* out, uint64_t n);

// Order-preserving row selection by a keep bitmap (bit r of word r/32):
// select_count returns the kept total and fills per-1024-row offsets;
// select_write copies the kept rows of n_cols uint32 columns.
uint64_t select_count(Ctx* c, const uint32_t* words, uint64_t n_rows, DevBuf& offs);
// the same without a host round trip: the total is left at offs[(n_rows + 1023) / 1024]
void select_count_async(Ctx* c, const uint32_t* words, uint64_t n_rows, DevBuf& offs);
void select_write(Ctx* c, const uint32_t* words, uint64_t n_rows, const DevBuf& offs, int n_cols,
                  const uint32_t* const* in, uint32_t* const* out);

inline int bits_for(uint64_t max_value) {
  int b = 0;
  while (b < 64 && (max_value >> b)) ++b;
  return b;
}

inline unsigned grid_for(Ctx* c, uint64_t n, int threads, int per_sm = 8) {
  const uint64_t want = (n + threads - 1) / threads;
  const uint64_t cap = uint64_t(c->sm_count) * per_sm;
  return unsigned(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace prims
}  // namespace tidq
