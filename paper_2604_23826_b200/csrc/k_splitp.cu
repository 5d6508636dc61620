// k_splitp.cu — K1w: 64 < p <= 128, K1's register-direct DMMA pass with the triangle split
// over W warps.
//
// Replaces accumulate_into<double> (reference src/suffstats.cpp:50-70) at these widths.  K2's
// rectangles pad the 9-16-block triangle and stream it through a cluster-wide shared-memory
// ring; here the CTA's 8 warps form 8/W row groups of W warps: the W warps of a group read the
// same 4-row k-steps straight from global memory (the group's other warps hit L1/L2), each
// keeps the accumulators of every W-th block of the NB(NB+1)/2-block triangle (block b with
// b % W == part, chosen at compile time so no DMMA is predicated) and part 0 adds the column
// sums.  At the end of a tile the groups' partials meet in shared memory and are added in
// group order into the canonical tile partial.  Tiles are widep_tile_rows(p) rows (as K2),
// so the choice between the two kernels never changes the tile partition.
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace sstat_b200 {
namespace {

constexpr int kU = 2;  // k-steps of loads in flight per warp (default; U below)

// X1: p = 8 NB + 1 — the last column rides outside the DMMA blocks, as in K1's
// k_smallp_x1: part 0 accumulates d_e d_j (j < 8 NB), d_e^2 and the sum of d_e with DFMA.
template <int NB, bool X1 = false>
struct SplitP {
    static constexpr int NBLK = NB * (NB + 1) / 2;
    static constexpr int XV = X1 ? NB * 8 + 2 : 0;     // extra column: x_e x_j, x_e^2, sum
    static constexpr int FRAG = NBLK * 64 + NB * 8 + XV;  // per-group epilogue values
};

template <int NB, int W, int PART>
struct Mine {  // blocks b = PART, PART + W, ... of the canonical (J <= K) enumeration
    static constexpr int N = (SplitP<NB>::NBLK - PART + W - 1) / W;
};

template <int NB>
__device__ __forceinline__ void load_k(const double* __restrict__ rowp, int g, uint32_t p, double (&x)[NB]) {
#pragma unroll
    for (int J = 0; J < NB; ++J) {
        const int c = 8 * J + g;
        x[J] = c < (int)p ? __ldg(rowp + c) : 0.0;
    }
}

// The extra column's state (X1, part 0 only): shift, products with each J, square, sum.
template <int NB>
struct Extra {
    double ce, ae[NB], aee, se;
};

template <int NB, int W, int PART, bool X1>
__device__ __forceinline__ void split_step(const double (&x)[NB], double xe, const double (&c)[NB],
                                           double (&acc)[Mine<NB, W, PART>::N][2], double (&s)[NB], Extra<NB>& ex) {
    double d[NB];
#pragma unroll
    for (int J = 0; J < NB; ++J) {
        d[J] = x[J] - c[J];
        if (PART == 0) s[J] += d[J];
    }
    if (X1 && PART == 0) {
        const double de = xe - ex.ce;
        ex.se += de;
        ex.aee = fma(de, de, ex.aee);
#pragma unroll
        for (int J = 0; J < NB; ++J) ex.ae[J] = fma(d[J], de, ex.ae[J]);
    }
    int b = 0;
#pragma unroll
    for (int J = 0; J < NB; ++J)
#pragma unroll
        for (int K = J; K < NB; ++K, ++b)
            if (b % W == PART) dmma_8x8x4(acc[b / W][0], acc[b / W][1], d[J], d[K]);
}

// Canonical destination of epilogue value e (block values, then the sums) or -1
// (padding / lower mirror of a diagonal block); columns col(J, g) = 8 J + g.
template <int NB, bool X1>
__device__ int split_slot(int e, uint32_t p) {
    constexpr int NBLK = SplitP<NB>::NBLK;
    if (X1 && e >= NBLK * 64 + NB * 8) {  // the extra column 8 NB
        const int x = e - NBLK * 64 - NB * 8, ecol = 8 * NB;
        if (x < NB * 8) return (int)(p + packed_index(p, x, ecol));  // column x = 8 J + g
        if (x == NB * 8) return (int)(p + packed_index(p, ecol, ecol));
        return ecol;  // its sum
    }
    if (e < NBLK * 64) {
        int b = e >> 6;
        const int l = (e & 63) >> 1, m = l >> 2, n = 2 * (l & 3) + (e & 1);
        int J = 0;
        while (b >= NB - J) {
            b -= NB - J;
            ++J;
        }
        const int K = J + b;
        const int a = 8 * J + m, bb = 8 * K + n;
        if (a >= (int)p || bb >= (int)p) return -1;
        if (J == K && a > bb) return -1;
        return (int)(p + packed_index(p, a < bb ? a : bb, a < bb ? bb : a));
    }
    const int e2 = e - NBLK * 64;
    const int a = 8 * (e2 >> 3) + (e2 & 7);
    return a < (int)p ? a : -1;
}

template <int NB, int W, int PART, bool X1, int kU>
__device__ __forceinline__ void split_body(const TileJob& job, uint32_t tile_rows, double* red) {
    using C = SplitP<NB, X1>;
    constexpr bool XP = X1 && PART == 0;  // this warp carries the extra column
    constexpr int G = kWarps / W;  // row groups
    constexpr int NM = Mine<NB, W, PART>::N;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int group = warp / W;
    const int g = lane >> 2, kk = lane & 3;
    const uint32_t p = job.p;
    const uint64_t E = partial_len(p);

    for (uint64_t t = job.tile_begin + blockIdx.x; t < job.tile_end; t += gridDim.x) {
        const uint32_t r = range_of_tile(job.tile_prefix, job.n_ranges, t);
        const uint64_t rs = __ldg(job.range_start + r), rc = __ldg(job.range_count + r);
        const uint64_t row0 = rs + (t - __ldg(job.tile_prefix + r)) * tile_rows;
        const uint64_t left = rs + rc - row0;
        const uint32_t rows = left < tile_rows ? (uint32_t)left : tile_rows;
        const double* __restrict__ tile = job.base + (row0 - job.base_row) * p;
        const double* crow = job.shift != nullptr ? job.shift + (uint64_t)r * p : nullptr;
        double c[NB];
#pragma unroll
        for (int J = 0; J < NB; ++J) c[J] = (crow != nullptr && 8 * J + g < (int)p) ? crow[8 * J + g] : 0.0;
        double acc[NM][2], s[NB];
#pragma unroll
        for (int b = 0; b < NM; ++b) acc[b][0] = acc[b][1] = 0.0;
#pragma unroll
        for (int J = 0; J < NB; ++J) s[J] = 0.0;
        Extra<NB> ex;
        ex.ce = (XP && crow != nullptr) ? crow[8 * NB] : 0.0;
        ex.aee = ex.se = 0.0;
#pragma unroll
        for (int J = 0; J < NB; ++J) ex.ae[J] = 0.0;

        const uint32_t nks = rows >> 2;
        const uint64_t kstride = (uint64_t)G * 4 * p;
        uint32_t ks = group;
        const double* rowp = tile + (uint64_t)(group * 4 + kk) * p;
        for (; ks + G * (kU - 1) < nks; ks += G * kU, rowp += kU * kstride) {
            double x[kU][NB], xe[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                load_k<NB>(rowp + u * kstride, g, p, x[u]);
                xe[u] = XP ? __ldg(rowp + u * kstride + 8 * NB) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) split_step<NB, W, PART, X1>(x[u], xe[u], c, acc, s, ex);
        }
        for (; ks < nks; ks += G, rowp += kstride) {
            double x[NB];
            load_k<NB>(rowp, g, p, x);
            split_step<NB, W, PART, X1>(x, XP ? __ldg(rowp + 8 * NB) : 0.0, c, acc, s, ex);
        }
        // ragged tail (rows % 4): the group whose turn k-step nks is; missing rows add 0
        if ((rows & 3) && group == (int)(nks % G)) {
            const uint32_t row = nks * 4 + kk;
            double x[NB], xe = ex.ce;
            if (row < rows) {
                load_k<NB>(tile + (uint64_t)row * p, g, p, x);
                if (XP) xe = __ldg(tile + (uint64_t)row * p + 8 * NB);
            } else {
#pragma unroll
                for (int J = 0; J < NB; ++J) x[J] = c[J];
            }
            split_step<NB, W, PART, X1>(x, xe, c, acc, s, ex);
        }

        // ---- epilogue: each group's partial into red[group], then the groups in order ----
        double* mine = red + group * C::FRAG;
        {
            int b = 0;
#pragma unroll
            for (int J = 0; J < NB; ++J)
#pragma unroll
                for (int K = J; K < NB; ++K, ++b)
                    if (b % W == PART) {
                        mine[b * 64 + lane * 2] = acc[b / W][0];
                        mine[b * 64 + lane * 2 + 1] = acc[b / W][1];
                    }
        }
        if (PART == 0) {
#pragma unroll
            for (int J = 0; J < NB; ++J) {
                s[J] += __shfl_xor_sync(0xffffffffu, s[J], 1);
                s[J] += __shfl_xor_sync(0xffffffffu, s[J], 2);
            }
            if (kk == 0) {
#pragma unroll
                for (int J = 0; J < NB; ++J) mine[C::NBLK * 64 + J * 8 + g] = s[J];
            }
        }
        if (XP) {  // the extra column, reduced over the 4 rows of a k-step like the sums
#pragma unroll
            for (int J = 0; J < NB; ++J) {
                ex.ae[J] += __shfl_xor_sync(0xffffffffu, ex.ae[J], 1);
                ex.ae[J] += __shfl_xor_sync(0xffffffffu, ex.ae[J], 2);
            }
            ex.aee += __shfl_xor_sync(0xffffffffu, ex.aee, 1);
            ex.aee += __shfl_xor_sync(0xffffffffu, ex.aee, 2);
            ex.se += __shfl_xor_sync(0xffffffffu, ex.se, 1);
            ex.se += __shfl_xor_sync(0xffffffffu, ex.se, 2);
            double* xm = mine + C::NBLK * 64 + NB * 8;
            if (kk == 0) {
#pragma unroll
                for (int J = 0; J < NB; ++J) xm[J * 8 + g] = ex.ae[J];
            }
            if (lane == 0) {
                xm[NB * 8] = ex.aee;
                xm[NB * 8 + 1] = ex.se;
            }
        }
        __syncthreads();
        double* out = job.tile_partials + t * E;
        for (int e = threadIdx.x; e < C::FRAG; e += kThreads) {
            const int slot = split_slot<NB, X1>(e, p);
            if (slot < 0) continue;
            double v = red[e];
#pragma unroll
            for (int q = 1; q < G; ++q) v += red[q * C::FRAG + e];
            out[slot] = v;
        }
        __syncthreads();
    }
}

template <int NB, int W, bool X1, int U>
__global__ void __launch_bounds__(kThreads, 1) k_splitp(TileJob job, uint32_t tile_rows) {
    extern __shared__ double red[];  // [8 / W][FRAG]
    const int part = (threadIdx.x >> 5) % W;
    if (part == 0) split_body<NB, W, 0, X1, U>(job, tile_rows, red);
    else if (part == 1) split_body<NB, W, 1, X1, U>(job, tile_rows, red);
    else if constexpr (W == 4) {
        if (part == 2) split_body<NB, W, 2, X1, U>(job, tile_rows, red);
        else split_body<NB, W, 3, X1, U>(job, tile_rows, red);
    }
}

template <int NB, int W, bool X1 = false, int U = kU>
cudaError_t launch_nb(const TileJob& job, int sms, cudaStream_t stream) {
    constexpr size_t smem = sizeof(double) * (kWarps / W) * SplitP<NB, X1>::FRAG;
    static std::atomic<int> cached[64];
    int dev = 0;
    cudaGetDevice(&dev);
    int per_sm = dev < 64 ? cached[dev].load() : 0;
    if (per_sm == 0) {
        cudaError_t e = cudaFuncSetAttribute(k_splitp<NB, W, X1, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_splitp<NB, W, X1, U>, kThreads, smem);
        if (e != cudaSuccess) return e;
        if (per_sm < 1) per_sm = 1;
        if (getenv("SSTAT_DEBUG")) fprintf(stderr, "k_splitp<%d,%d,%d>: smem=%zu per_sm=%d\n", NB, W, (int)X1, smem, per_sm);
        if (dev < 64) cached[dev].store(per_sm);
    }
    const uint64_t tiles = job.tile_end - job.tile_begin;
    const uint64_t grid = tiles < (uint64_t)sms * per_sm ? tiles : (uint64_t)sms * per_sm;
    if (grid == 0) return cudaSuccess;
    k_splitp<NB, W, X1, U><<<(unsigned)grid, kThreads, smem, stream>>>(job, widep_tile_rows(job.p));
    if (job.launched) *job.launched = (const void*)k_splitp<NB, W, X1, U>;
    return cudaGetLastError();
}

// k-steps of loads in flight per warp, per instance (SSTAT_K1W_U overrides: 2, 3 or 4).
// K1w runs one CTA (8 warps) per SM, so its loads are latency-bound where the registers allow
// more in flight.  Measured (profiles/r01_k1w_u.log, TF/s at U = 2 -> chosen): p = 65 15.3 ->
// 19.2 (U = 4), p = 72 21.7 -> 25.6, p = 73 21.9 -> 24.2, p = 80 21.4 -> 24.2, p = 104 21.7 ->
// 25.0, p = 105 21.9 -> 22.4, p = 112 21.0 -> 21.3 (U = 3); the others lose with U > 2.
// NB = 12 (p = 90-96) with W = 4 at U = 4: p = 92 / 96 17.7 / 16.5 against K2's 15.1 / 16.0
// (U = 2: 14.0 / 13.6; W = 2 spills at every U: 10-14) — profiles/r01_k1w_nb12.log.
template <int NB, bool X1>
constexpr int default_u() {
    if ((NB == 8 && X1) || NB == 12) return 4;
    if (NB == 9 || (NB == 10 && !X1) || NB == 13 || (NB == 14 && !X1)) return 3;
    return 2;
}

template <int NB, int W, bool X1>
cudaError_t launch_u(const TileJob& job, int sms, cudaStream_t stream) {
    int u = default_u<NB, X1>();
    if (const char* env = getenv("SSTAT_K1W_U")) u = atoi(env);
    if (u == 3) return launch_nb<NB, W, X1, 3>(job, sms, stream);
    if (u == 4) return launch_nb<NB, W, X1, 4>(job, sms, stream);
    return launch_nb<NB, W, X1, 2>(job, sms, stream);
}

}  // namespace

// Measured (profiles/r01_p_sweep.log): W = 2 for NB = 9..11 (21-22 TF/s vs K2's 8.5-17.5),
// W = 4 for NB = 12..16 (20-22 TF/s vs 14-21; NB = 12 only with 4 k-steps of loads in flight,
// default_u above), so K1w takes every 64 < p <= 128 (SSTAT_SPLITP=0: K2 there).
bool splitp_handles(uint32_t p) {
    if (const char* env = getenv("SSTAT_SPLITP")) {
        if (atoi(env) == 0) return false;
    }
    return p > 64 && p <= 128;
}

cudaError_t launch_splitp(const TileJob& job, int sms, cudaStream_t stream) {
    // p = 8 NB + 1: NB block rows plus the last column by DFMA (k_smallp_x1's scheme) instead
    // of NB + 1 block rows whose last one holds a single column (measured,
    // profiles/r01_k1w_x1.log: p = 65 / 73 / 81 / 105 / 113 +7 / +9 / +11 / +7 / +1 %, p = 89
    // +23 % over K2); p = 97 keeps the 13-block-row split (the 12-row extra-column instance sits
    // at 254 registers: 13.9 vs 14.7 TF/s at its best U, profiles/r01_k1w_nb12.log) and p = 121
    // NB = 16 (the NB = 15 x1 instance spills: -19 %).
    if (job.p % 8 == 1 && !getenv("SSTAT_K1W_NO_X1")) {
        switch (job.p / 8) {
            case 8: return launch_u<8, 2, true>(job, sms, stream);
            case 9: return launch_u<9, 2, true>(job, sms, stream);
            case 10: return launch_u<10, 2, true>(job, sms, stream);
            case 11: return launch_u<11, 2, true>(job, sms, stream);
            case 13: return launch_u<13, 4, true>(job, sms, stream);
            case 14: return launch_u<14, 4, true>(job, sms, stream);
            default: break;
        }
    }
    switch ((job.p + 7) / 8) {
        case 9: return launch_u<9, 2, false>(job, sms, stream);
        case 10: return launch_u<10, 2, false>(job, sms, stream);
        case 11: return launch_u<11, 2, false>(job, sms, stream);
        case 12: return launch_u<12, 4, false>(job, sms, stream);
        case 13: return launch_u<13, 4, false>(job, sms, stream);
        case 14: return launch_u<14, 4, false>(job, sms, stream);
        case 15: return launch_u<15, 4, false>(job, sms, stream);
        case 16: return launch_u<16, 4, false>(job, sms, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sstat_b200
