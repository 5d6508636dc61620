// fold.cuh — the per-range fold (K3a) device code.  Blocks of 256 threads.
#pragma once

#include "common.cuh"

namespace sstat_b200 {

// Tile partials come from the previous kernel; read them through L2 (ld.global.cg).
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// Tile folds of one range run kTileLanes interleaved lanes per entry: lane q sums tiles
// t0+q, t0+q+kTileLanes, ... (kFoldInFlight loads in flight, masked tails instead of a serial
// remainder loop), then the lanes are added 0..kTileLanes-1.  A fixed function of the range's
// tile partials; blocks are kTileLanes x 32 threads.  32 lanes x 16 loads in flight keep a
// range of ~2000 small-plan tiles (C1: 1e6 rows in 512-row tiles) to four L2 round trips.
constexpr int kTileLanes = 32;
constexpr int kFoldInFlight = 16;
__device__ __forceinline__ double fold_tiles_lane(const double* __restrict__ tp, uint64_t E, uint64_t e, uint64_t t0,
                                                  uint64_t t1, int q) {
    double s = 0.0;
    const uint64_t T = t1 - t0;
    if ((uint64_t)q >= T) return s;
    const uint32_t cnt = (uint32_t)((T - q + kTileLanes - 1) / kTileLanes);  // this lane's tiles
    const uint64_t stride = (uint64_t)kTileLanes * E;
    const double* ptr = tp + (t0 + q) * E + e;
    for (uint32_t i = 0; i < cnt; i += kFoldInFlight, ptr += kFoldInFlight * stride) {
        const uint32_t m = cnt - i;
        double v[kFoldInFlight];
#pragma unroll
        for (int u = 0; u < kFoldInFlight; ++u) v[u] = (uint32_t)u < m ? ld_cg(ptr + u * stride) : 0.0;
#pragma unroll
        for (int u = 0; u < kFoldInFlight; ++u)
            if ((uint32_t)u < m) s += v[u];
    }
    return s;
}

// Inverse of packed_index: (j, k) with j <= k for packed position i.
__device__ __forceinline__ void unpack_index(uint32_t p, uint32_t i, uint32_t& j, uint32_t& k) {
    const double b = 2.0 * p + 1.0;
    int64_t row = (int64_t)floor((b - sqrt(b * b - 8.0 * i)) * 0.5);
    if (row < 0) row = 0;
    auto start = [p](int64_t jj) { return jj * (int64_t)p - jj * (jj - 1) / 2; };
    while (row > 0 && start(row) > (int64_t)i) --row;
    while (row + 1 < (int64_t)p && start(row + 1) <= (int64_t)i) ++row;
    j = (uint32_t)row;
    k = (uint32_t)(row + ((int64_t)i - start(row)));
}

// K3a for one local range r, by one block of kTileLanes x 32 threads.  The range's tile
// partials are summed in a fixed order (fold_tiles_lane, then lanes 0..kTileLanes-1),
// and the shifted moments map back to raw moments with c = shift row, n = range rows:
//   s_j  = s'_j + n c_j
//   S_jk = S'_jk + c_j s'_k + c_k s'_j + n c_j c_k
// (exact for integer data below 2^53, like the reference's own sums).  A range whose sums
// are non-finite is flagged (any non-finite input makes them so; reduce.hpp:111-134 picks
// the lowest failing range).  sm: (2p + 32 kTileLanes) doubles.  c: the shift row (or nullptr = 0).
// Cross entries [p + x0, p + x1) are this block's slice; every slice block folds the p
// sums (needed for the un-shift) but only slice 0 writes them and flags.
__device__ inline void fold_range_block(const double* __restrict__ tp, uint64_t t0, uint64_t t1, double n,
                                        const double* c, uint32_t p, uint64_t global_range, double* out,
                                        double* rank_hdr, uint32_t* flag, double* sm, uint64_t x0, uint64_t x1) {
    const uint64_t E = partial_len(p);
    double* ssum = sm;
    double* sc = sm + p;
    double* lanes = sm + 2 * p;
    const int le = threadIdx.x & 31, q = threadIdx.x >> 5;
    const bool lead = x0 == 0;
    for (int phase = 0; phase < 2; ++phase) {
        const uint64_t lo = phase == 0 ? 0 : p + x0, hi = phase == 0 ? p : (p + x1 < E ? p + x1 : E);
        for (uint64_t e0 = lo; e0 < hi; e0 += 32) {
            const uint64_t e = e0 + le;
            lanes[q * 32 + le] = e < hi ? fold_tiles_lane(tp, E, e, t0, t1, q) : 0.0;
            __syncthreads();
            if (q == 0 && e < hi) {
                double S = lanes[le];
#pragma unroll
                for (int w = 1; w < kTileLanes; ++w) S += lanes[w * 32 + le];
                if (phase == 0) {
                    const double cj = c ? c[e] : 0.0;
                    ssum[e] = S;
                    sc[e] = cj;
                    if (lead) out[e] = S + n * cj;
                    if (lead && (!isfinite(S) || !isfinite(cj))) {
                        *flag = 1;
                        atomicMin(reinterpret_cast<unsigned long long*>(rank_hdr), (unsigned long long)global_range);
                    }
                } else {
                    if (c) {
                        uint32_t j, k;
                        unpack_index(p, (uint32_t)(e - p), j, k);
                        S = ((S + sc[j] * ssum[k]) + sc[k] * ssum[j]) + (n * sc[j]) * sc[k];
                    }
                    out[e] = S;
                }
            }
            __syncthreads();
        }
    }
}

}  // namespace sstat_b200
