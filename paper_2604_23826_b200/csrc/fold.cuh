// fold.cuh — the per-range fold (K3a) device code.  Blocks of 256 threads.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace sstat_b200 {

namespace cg = cooperative_groups;

// Tile partials come from the previous kernel; read them through L2 (ld.global.cg).
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// Tile folds of one range run kTileLanes interleaved lanes per entry: lane q sums tiles
// t0+q, t0+q+kTileLanes, ... (kFoldInFlight loads in flight, masked tails instead of a serial
// remainder loop), then the lanes are added 0..kTileLanes-1.  A fixed function of the range's
// tile partials; blocks are kTileLanes x 32 threads (512: four per SM, so C2's 480 fold blocks
// run in one wave — 1024-thread blocks measured 2x slower there).
constexpr int kTileLanes = 16;
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

// K3a splits a range's T tile partials into fold_chunks(T) contiguous chunks, one per CTA of a
// thread-block cluster (a range of a small plan has ~2000 tiles: one CTA alone would stream
// them at one SM's L2 bandwidth).  A function of T alone, so every rank folds a range the same
// way.
constexpr uint64_t kChunkTiles = 256;
constexpr uint32_t kMaxChunks = 8;  // portable cluster size
__host__ __device__ inline uint32_t fold_chunks(uint64_t T) {
    const uint64_t c = (T + kChunkTiles - 1) / kChunkTiles;
    return c < 1 ? 1u : c > kMaxChunks ? kMaxChunks : (uint32_t)c;
}

// K3a for one local range, by the CTA of chunk k of a cluster of kTileLanes x 32-thread CTAs.
// Order: within chunk k the tiles are summed by fold_tiles_lane (lane q: tiles q, q + 32, ...
// of the chunk), lanes added 0..kTileLanes-1; CTA 0 then adds the chunk partials 0..C-1 through
// distributed shared memory — a fixed function of the range's tile partials.  The shifted
// moments map back to raw moments with c = shift row, n = range rows:
//   s_j  = s'_j + n c_j
//   S_jk = S'_jk + c_j s'_k + c_k s'_j + n c_j c_k
// (exact for integer data below 2^53, like the reference's own sums).  A range whose sums
// are non-finite is flagged (any non-finite input makes them so; reduce.hpp:111-134 picks
// the lowest failing range).  c: the shift row (or nullptr = 0).  Cross entries
// [p + x0, p + x1) are this block's slice; every slice folds the p sums (needed for the
// un-shift) but only slice 0 writes them and flags.
// sm: fold_smem_doubles(p, x1 - x0) doubles.
__host__ __device__ inline uint64_t fold_smem_doubles(uint32_t p, uint64_t slice) {
    return 2ull * p + 32ull * kTileLanes + p + slice;
}
template <bool CLUSTER>
__device__ inline void fold_range_block(const double* __restrict__ tp, uint64_t t0, uint64_t t1, double n,
                                        const double* c, uint32_t p, uint64_t global_range, double* out,
                                        double* rank_hdr, uint32_t* flag, double* sm, uint64_t x0, uint64_t x1,
                                        uint32_t k) {
    const uint64_t E = partial_len(p);
    double* ssum = sm;
    double* sc = sm + p;
    double* lanes = sm + 2 * p;
    double* cp = lanes + 32 * kTileLanes;  // this chunk's partials: [p sums | the slice's cross]
    const int le = threadIdx.x & 31, q = threadIdx.x >> 5;
    const bool lead = x0 == 0;
    const uint64_t xe = p + x1 < E ? p + x1 : E;  // end of the slice's cross entries
    const uint64_t n_mine = p + (xe - (p + x0));
    const uint64_t T = t1 - t0;
    const uint32_t C = fold_chunks(T);
    const uint64_t ch = (T + C - 1) / C;
    // 1. the chunk partial of every entry of the block
    if (k < C) {
        const uint64_t c0 = t0 + (k * ch < T ? k * ch : T), c1 = t0 + ((k + 1) * ch < T ? (k + 1) * ch : T);
        for (int phase = 0; phase < 2; ++phase) {
            const uint64_t lo = phase == 0 ? 0 : p + x0, hi = phase == 0 ? p : xe;
            for (uint64_t e0 = lo; e0 < hi; e0 += 32) {
                const uint64_t e = e0 + le;
                lanes[q * 32 + le] = e < hi ? fold_tiles_lane(tp, E, e, c0, c1, q) : 0.0;
                __syncthreads();
                if (q == 0 && e < hi) {
                    double S = lanes[le];
#pragma unroll
                    for (int w = 1; w < kTileLanes; ++w) S += lanes[w * 32 + le];
                    cp[phase == 0 ? e : p + (e - p - x0)] = S;
                }
                __syncthreads();
            }
        }
    }
    if constexpr (CLUSTER) {
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
    if (k == 0) {
        // 2. CTA 0: the chunk partials in order 0..C-1 (remote ones through DSMEM)
        if constexpr (CLUSTER) {
            cg::cluster_group cluster = cg::this_cluster();
            for (uint64_t i = threadIdx.x; i < n_mine; i += blockDim.x) {
                double v[kMaxChunks];
#pragma unroll
                for (uint32_t kk = 1; kk < kMaxChunks; ++kk)  // all remote loads in flight, then the adds in order
                    v[kk] = kk < C ? *cluster.map_shared_rank(cp + i, kk) : 0.0;
                double S = cp[i];
#pragma unroll
                for (uint32_t kk = 1; kk < kMaxChunks; ++kk)
                    if (kk < C) S += v[kk];
                cp[i] = S;
            }
            __syncthreads();
        }
        // 3. the range's raw moments
        for (uint64_t i = threadIdx.x; i < p; i += blockDim.x) {
            const double S = cp[i];
            const double cj = c ? c[i] : 0.0;
            ssum[i] = S;
            sc[i] = cj;
            if (lead) out[i] = (S + n * cj) + 0.0;  // + 0.0: a partial is never -0.0, like the reference's
            if (lead && (!isfinite(S) || !isfinite(cj))) {
                *flag = 1;
                atomicMin(reinterpret_cast<unsigned long long*>(rank_hdr), (unsigned long long)global_range);
            }
        }
        __syncthreads();
        for (uint64_t i = p + threadIdx.x; i < n_mine; i += blockDim.x) {
            const uint64_t e = p + x0 + (i - p);
            double S = cp[i];
            if (c) {
                uint32_t j, kk;
                unpack_index(p, (uint32_t)(e - p), j, kk);
                S = ((S + sc[j] * ssum[kk]) + sc[kk] * ssum[j]) + (n * sc[j]) * sc[kk];
            }
            out[e] = S + 0.0;
        }
    }
    if constexpr (CLUSTER) {  // CTA 0's remote reads are done before any CTA of the cluster exits
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
}

}  // namespace sstat_b200
