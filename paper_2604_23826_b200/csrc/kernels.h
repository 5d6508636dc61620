// kernels.h — host-callable launchers of the device kernels (all enqueue on `stream`).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace sstat_b200 {

// K1: tiles [job.tile_begin, job.tile_end), p <= 64; persistent grid of
// min(tiles, sms x resident CTAs per SM).
cudaError_t launch_smallp(const TileJob& job, int sms, cudaStream_t stream);
// CTAs per SM of the runtime-height K1 kernel for width p (alignment-independent): the wave size
// of the small-plan tile rule (smallp_tile_rows).
constexpr uint32_t kMaxSmallP = 64;
uint32_t smallp_rt_ctas_per_sm(uint32_t p);

// K1w: 64 < p <= 128 (splitp_handles), K1's register-direct pass with the triangle split over
// warps; tiles of widep_tile_rows(p) rows like K2.
bool splitp_handles(uint32_t p);
cudaError_t launch_splitp(const TileJob& job, int sms, cudaStream_t stream);

// K2: tiles for p > 64 (smem-staged DMMA SYRK), tiles of widep_tile_rows(p) rows.
// *kernels (optional) receives the number of kernels launched (2 when the idle-slot split runs).
cudaError_t launch_widep(const TileJob& job, int sms, cudaStream_t stream, uint32_t* kernels = nullptr);
uint32_t widep_tile_rows(uint32_t p);
constexpr uint32_t kMaxWideP = 2048;  // launch_widep rejects wider rows

// shift[r][j] = first row of local range r (0 when the range is empty).
cudaError_t launch_gather_shift(const double* base, uint64_t base_row, const uint64_t* range_start,
                                const uint64_t* range_count, uint32_t n_ranges, uint32_t p, double* shift,
                                cudaStream_t stream);

// K3a: fold each local range's tile partials in ascending tile order, map the shifted
// moments back to raw sums / X^T X, write [kHdr + r*E] of `rank_buf`, and flag
// non-finite ranges (global index first_range + r) in the header.
// The shift row: shift[r*p], or (shift == nullptr, base != nullptr) the range's first row
// read in place from the resident shard base (absolute row base_row at base[0]).
// chunks: the launch's cluster size = max over its ranges of fold_chunks(tiles of the range).
cudaError_t launch_range_fold(const double* tile_partials, const uint64_t* tile_prefix, const uint64_t* range_count,
                              const double* shift, const double* base, uint64_t base_row, const uint64_t* range_start,
                              uint32_t n_ranges, uint32_t p, uint64_t first_range, double* rank_buf, uint32_t* flags,
                              uint32_t chunks, cudaStream_t stream);

// First non-finite value (row-major) over the flagged local ranges (flags[r] != 0);
// min absolute linear index row*p + col lands in header[1].  No-op when none flagged.
cudaError_t launch_find_nonfinite(const double* base, uint64_t base_row, const uint64_t* range_start,
                                  const uint64_t* range_count, uint32_t n_ranges, uint32_t p, const uint32_t* flags,
                                  double* rank_buf, int grid, cudaStream_t stream);

// K3b: fold over all n_ranges global ranges.  reference_order: ascending from +0.0
// (reduce.hpp:142-145, fold_entry; precision 1 rounds every add through binary32 like
// merge_suffstats, suffstats.cpp:92-98); otherwise the 32-lane fast fold (fold_fast).
// Range r lives in rank q = owner(r) at buf + q*rank_stride + kHdr + (r - first(q))*E.
cudaError_t launch_final_fold(const double* buf, uint64_t rank_stride, uint64_t n_ranges, int world, uint32_t p,
                              uint32_t precision, bool reference_order, double* out, cudaStream_t stream);

// Reference-order accumulation: one sequential mul-then-add chain per (range, entry)
// exactly as accumulate_into<Acc> (suffstats.cpp:56-67); precision 1 = binary32.
// Writes raw range partials out[r*E] and flags non-finite ranges (flags[r], hdr[0]).
// resume_first: range 0 of this launch is a later piece of a range streamed in pieces — its
// chains continue from out[0..E) instead of +0.0 (same operations, same order).
cudaError_t launch_refexact(const double* base, uint64_t base_row, const uint64_t* range_start,
                            const uint64_t* range_count, uint32_t n_ranges, uint32_t p, uint32_t precision,
                            uint64_t first_range, double* hdr, double* out, uint32_t* flags, bool rows_aligned16,
                            bool resume_first, cudaStream_t stream);

// K5: synthetic rows [first_row, first_row + n_rows) (bit-identical to the oracle).
cudaError_t launch_generate(double* dst, uint32_t kind, uint64_t seed, double mu, uint32_t n_int, uint64_t first_row,
                            uint64_t n_rows, uint32_t p, cudaStream_t stream);

// ---- column_sum (reduce.cpp:32-88): 32-byte partials {f64/f32 sum, exact lo, exact hi,
// first non-integral row}; tiles -> ranges -> one ascending final fold.  sequential +
// resume_first: range 0 continues the partial already in range_parts[0] (pieces) ----
cudaError_t launch_colsum(const double* base, uint64_t base_row, uint32_t p, uint32_t column,
                          const uint64_t* range_start, const uint64_t* range_count, const uint64_t* tile_prefix,
                          uint32_t n_ranges, uint64_t tile_begin, uint64_t tile_end, bool sequential,
                          uint32_t precision, void* tile_parts, void* range_parts, int sms, bool resume_first,
                          cudaStream_t stream);
cudaError_t launch_colsum_range_fold(const void* tile_parts, const uint64_t* tile_prefix, uint32_t n_ranges,
                                     void* range_parts, cudaStream_t stream);
cudaError_t launch_colsum_final(const void* buf, uint64_t rank_stride_parts, uint64_t n_ranges, int world,
                                uint32_t precision, void* out, cudaStream_t stream);

// ---- co-moments (suffstats.cpp:107-159) from K1's shifted tile partials ----
cudaError_t launch_comoment_range(const double* tile_partials, const uint64_t* tile_prefix, const uint64_t* range_count,
                                  const double* shift, uint32_t n_ranges, uint32_t p, double* out, uint64_t first_range,
                                  double* rank_hdr, uint32_t* flags, cudaStream_t stream);
cudaError_t launch_comoment_merge(const double* buf, uint64_t rank_stride, uint64_t n_ranges, int world,
                                  const uint64_t* counts, uint32_t p, double* out, cudaStream_t stream);

}  // namespace sstat_b200
