// common.cuh — shared device-side definitions of the B200 sufficient-statistics engine.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sstat_b200 {

// Rows per accumulation tile.  A tile is the deterministic unit of work: its
// partial depends only on the rows of the tile, so results are bit-identical for
// any grid size, GPU count or staging layout.  K1's tiles are kTileRows = 4096 rows
// (8 warps x 128 k-steps); large plans (at least kBigTileMin tiles of kBigTileRows, p > 8)
// take kBigTileRows = 16384 (a quarter of the per-tile epilogues and partials: C2's K1
// +3 %, profiles/r02_k1_tile_height_ab.log); plans too small to fill the GPU with kTileRows
// take the shortest height whose tiles fit one wave of K1's CTA slots (smallp_tile_rows,
// engine.cu) — a function of the plan alone, the same on every rank.
constexpr uint32_t kTileRows = 4096;
constexpr uint32_t kBigTileRows = 16384;
constexpr uint32_t kMinTileRows = 256;
constexpr uint64_t kFillTiles = 2ull * 148 * 4;   // twice K1's resident CTA slots on a B200
constexpr uint64_t kWaveTiles = 148ull * 4;       // K1's resident CTA slots on a B200 (4 per SM)
constexpr uint64_t kWaveSMs = 148;                // the SMs a tile wave is counted over (B200)
constexpr uint64_t kBigTileMin = 8ull * 148 * 4;  // eight waves of big tiles
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;

// Number of doubles in one canonical partial: sums[p] then the packed upper triangle.
__host__ __device__ inline uint64_t partial_len(uint32_t p) { return p + (uint64_t)p * (p + 1) / 2; }

// SymPacked index (linalg.hpp:58-61), j <= k.
__host__ __device__ inline uint32_t packed_index(uint32_t p, uint32_t j, uint32_t k) {
    return j * p - j * (j - 1) / 2 + (k - j);
}

// Everything a tile kernel needs for one launch.  `base` points at the row with
// absolute index `base_row` (device shard or a staging slot).
struct TileJob {
    const double* base;
    uint64_t base_row;
    const uint64_t* range_start;   // [n_ranges] absolute first row of each local range
    const uint64_t* range_count;   // [n_ranges]
    const uint64_t* tile_prefix;   // [n_ranges + 1] local range r owns tiles [prefix[r], prefix[r+1])
    const double* shift;           // [n_ranges][p] first row of each range, or nullptr (no shift)
    uint32_t n_ranges;
    uint32_t p;
    uint64_t tile_begin, tile_end; // tiles of this launch
    double* tile_partials;         // [n_tiles][partial_len(p)] canonical, shifted space
    unsigned long long* claim;     // 8-byte device scratch for K2's dynamic work split (or nullptr)
    // K2's idle-slot launch: the caller context's own side stream and fork / join events
    // (nullptr: no side launch, the clustered launch takes every tile)
    cudaStream_t side;
    cudaEvent_t fork, join;
    const void** launched;         // (optional) receives the accumulate kernel the launcher chose
    uint32_t tile_rows;            // K1: rows per tile of this plan (smallp_tile_rows)
    uint32_t shift_in_place;       // K1 runtime-height instances, shift == nullptr: the shift row is
                                   // the range's first row read from base (a resident shard)
    int* occupancy;                // K1 query (non-null): receives the CTAs per SM of the kernel the
                                   // launcher would choose; nothing is launched
};

// Range owning tile t (tile_prefix ascending; binary search, O(log R) L2 reads per tile).
__device__ __forceinline__ uint32_t range_of_tile(const uint64_t* prefix, uint32_t n_ranges, uint64_t t) {
    uint32_t lo = 0, hi = n_ranges;  // invariant: prefix[lo] <= t < prefix[hi]
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(prefix + mid) <= t) lo = mid;
        else hi = mid;
    }
    return lo;
}

// FP64 warp MMA D = A(8x4, row) * B(4x8, col) + C on the DMMA tensor pipe.
// Fragments (PTX ISA, mma.m8n8k4 .f64): lane l, g = l>>2, k = l&3 holds
//   A[g][k], B[k][g], C[g][2k], C[g][2k+1].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// Streaming 64/128-bit loads: read once, evict first.
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream2(const double* p) { return __ldcs(reinterpret_cast<const double2*>(p)); }

// Per-rank header in front of the range partials: [0] lowest failing global range
// (UINT64_MAX = none), [1] first non-finite linear index row*p + col (UINT64_MAX = none),
// [2] the rank's status (0 = ok; a failed rank's sstat_status, so its peers fail with it
// instead of waiting in the exchange), [3] spare (0).
constexpr uint32_t kHdr = 4;

// Where range r's partial sits in the gathered rank buffers: rank q = owner(r) with
// first(q) = floor(q R / W), at buf + q*rank_stride + kHdr + (r - first(q))*E.
__host__ __device__ inline const double* range_partial(const double* buf, uint64_t rank_stride, uint64_t n_ranges,
                                                       int world, uint64_t E, uint64_t r) {
    if (world == 1) return buf + kHdr + r * E;
    int q = (int)((r * (uint64_t)world) / n_ranges);
    if (q >= world) q = world - 1;
    while (q > 0 && (uint64_t)q * n_ranges / world > r) --q;
    while (q + 1 < world && (uint64_t)(q + 1) * n_ranges / world <= r) ++q;
    return buf + (uint64_t)q * rank_stride + kHdr + (r - (uint64_t)q * n_ranges / world) * E;
}

// Fast-mode range fold of one entry: 32 interleaved lanes (lane q sums ranges q, q+32, ...
// ascending from +0.0), then the lanes in order 0..31.  A fixed function of the global range
// sequence — identical on every rank and for any GPU count — with 32x shorter dependent chains
// than the reference order (C3's 954 ranges: 30 loads per lane).  fold_lane is one lane (device:
// one thread per lane).
constexpr int kFoldLanes = 32;
__host__ __device__ inline double fold_lane(const double* buf, uint64_t rank_stride, uint64_t n_ranges, int world,
                                            uint64_t E, uint64_t e, int q) {
    double s = 0.0;
    for (uint64_t r = q; r < n_ranges; r += kFoldLanes) s += range_partial(buf, rank_stride, n_ranges, world, E, r)[e];
    return s;
}
__host__ __device__ inline double fold_fast(const double* buf, uint64_t rank_stride, uint64_t n_ranges, int world,
                                            uint64_t E, uint64_t e) {
    double t = 0.0;
    for (int q = 0; q < kFoldLanes; ++q) t += fold_lane(buf, rank_stride, n_ranges, world, E, e, q);
    return t;
}

// The ascending range fold of one entry (reference include/sstat/reduce.hpp:142-145 with
// merge_suffstats, src/suffstats.cpp:86-105): acc starts at +0.0 and adds range 0, 1, ...
// Range r sits in rank q = owner(r), first(q) = floor(q R / W), at
//   buf + q*rank_stride + kHdr + (r - first(q))*E + e.
// Binary32 mode rounds every add through float like merge_suffstats.  The reference-order
// fold of SSTAT_FLAG_REFEXACT / Binary32Diagnostic; shared by the device fold (K3b) and the
// host fold used to check the rank layout.
__host__ __device__ inline double fold_entry(const double* buf, uint64_t rank_stride, uint64_t n_ranges, int world,
                                             uint32_t p, uint32_t precision, uint64_t e) {
    const uint64_t E = partial_len(p);
    double acc = 0.0;
    for (int q = 0; q < world; ++q) {
        const uint64_t f = (uint64_t)q * n_ranges / world, l = (uint64_t)(q + 1) * n_ranges / world;
        const double* part = buf + (uint64_t)q * rank_stride + kHdr + e;
        const uint64_t cnt = l - f;
        if (precision == 1) {
            for (uint64_t r = 0; r < cnt; ++r) acc = (double)((float)acc + (float)part[r * E]);
        } else {
            uint64_t r = 0;
            for (; r + 8 <= cnt; r += 8) {  // 8 loads in flight, adds stay in range order
                double v[8];
                for (int u = 0; u < 8; ++u) v[u] = part[(r + u) * E];
                for (int u = 0; u < 8; ++u) acc += v[u];
            }
            for (; r < cnt; ++r) acc += part[r * E];
        }
    }
    return acc;
}

}  // namespace sstat_b200
