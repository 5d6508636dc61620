#pragma once
// k_smallp.cuh — K1: streaming sufficient statistics for p <= 64 on the FP64 DMMA pipe.
// The kernels and their launchers for one tile height TRC are instantiated by one translation
// unit each (k_smallp.cu: runtime height and the dispatch, k_smallp_4k.cu, k_smallp_16k.cu), so
// the three families compile in parallel.
//
// Replaces accumulate_into<double> (reference src/suffstats.cpp:50-70) for one
// accumulation tile (4096 rows; fewer for small plans, job.tile_rows).  Each warp walks k-steps of 4 rows.  Lane
// l = 4g + k loads the values of row k at the NB columns col(J, g), J < NB, straight
// from HBM with coalesced streaming loads (a warp load covers 4 whole rows), subtracts
// the range shift c, and feeds the same register as the A fragment (A[g][k]) of
// column block J and the B fragment (B[k][g]) of column block K of
//     mma.sync.m8n8k4.f64:  C_JK[m][n] += sum_k X[k][col(J,m)] * X[k][col(K,n)].
// The NB(NB+1)/2 upper blocks C_JK (J <= K) cover every column pair exactly once (the
// diagonal blocks twice, symmetrically), so no value is loaded twice and no shared
// memory is touched in the main loop.  Column sums accumulate with DADD on the same
// registers.  The epilogue reduces the 8 warps through shared memory in fixed order
// and writes the tile partial in canonical (sums, SymPacked) order.
//
// Column permutation col(J, g):  VEC (p == 8*NB, NB even): g*NB + J  — each lane reads
// NB contiguous doubles with 128-bit loads;  otherwise J*8 + g — 8 lanes read 8
// consecutive doubles of a row per instruction (64-byte segments).
#include <atomic>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace sstat_b200 {
namespace {

// X1: p = 8 NB + 1 — the last column rides outside the DMMA blocks (see step()).
template <int NB, bool VEC, bool X1 = false>
struct SmallP {
    static constexpr int NBLK = NB * (NB + 1) / 2;
#ifndef SSTAT_U2V
#define SSTAT_U2V 16
#endif
    static constexpr int U = NB <= 2 ? (VEC || NB == 1 ? SSTAT_U2V : 8) : (NB <= 4 ? 8 : 4);  // k-steps in flight per warp
    static constexpr int XV = X1 ? NB * 8 + 2 : 0;                 // extra column: x_e x_j, x_e^2, sum
    static constexpr int FRAG = NBLK * 64 + NB * 8 + XV;           // per-warp epilogue values
    __device__ __forceinline__ static int col(int J, int g) { return VEC ? g * NB + J : J * 8 + g; }
};

template <int NB, bool VEC>
__device__ __forceinline__ void load_row(const double* __restrict__ rowp, int g, uint32_t p, double (&x)[NB]) {
    using C = SmallP<NB, VEC>;
    if constexpr (VEC) {
        const double* q = rowp + g * NB;
#pragma unroll
        for (int i = 0; i < NB / 2; ++i) {
            const double2 v = ld_stream2(q + 2 * i);
            x[2 * i] = v.x;
            x[2 * i + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int J = 0; J < NB; ++J) {
            const int c = C::col(J, g);
            x[J] = (c < (int)p) ? ld_stream(rowp + c) : 0.0;
        }
    }
}

template <int NB>
__device__ __forceinline__ void step(const double (&x)[NB], const double (&c)[NB], double (&acc)[NB * (NB + 1) / 2][2],
                                     double (&s)[NB]) {
    double d[NB];
#pragma unroll
    for (int J = 0; J < NB; ++J) {
        d[J] = x[J] - c[J];
        s[J] += d[J];
    }
    int b = 0;
#pragma unroll
    for (int J = 0; J < NB; ++J)
#pragma unroll
        for (int K = J; K < NB; ++K, ++b) dmma_8x8x4(acc[b][0], acc[b][1], d[J], d[K]);
}

// p = 8 NB + 1: a whole DMMA block for one column would spend NB + 1 DMMAs (16 pipe cycles
// each) on NB * 8 + 1 products per row; instead every lane (g, k) also loads the last column
// e of its row k (8 lanes, one address) and accumulates d_e * d_{col(J, g)} for each J and
// d_e^2 with DFMA (2 pipe cycles each), d_e into its sum.  Fixed order per lane, reduced over
// k and the warps in fixed order in the epilogue: a fixed function of the tile.
template <int NB>
__device__ __forceinline__ void step_x1(const double (&x)[NB], double xe, const double (&c)[NB], double ce,
                                        double (&acc)[NB * (NB + 1) / 2][2], double (&s)[NB], double (&ae)[NB],
                                        double& aee, double& se) {
    double d[NB];
#pragma unroll
    for (int J = 0; J < NB; ++J) {
        d[J] = x[J] - c[J];
        s[J] += d[J];
    }
    const double de = xe - ce;
    se += de;
    aee = fma(de, de, aee);
#pragma unroll
    for (int J = 0; J < NB; ++J) ae[J] = fma(d[J], de, ae[J]);
    int b = 0;
#pragma unroll
    for (int J = 0; J < NB; ++J)
#pragma unroll
        for (int K = J; K < NB; ++K, ++b) dmma_8x8x4(acc[b][0], acc[b][1], d[J], d[K]);
}

// Canonical destination of epilogue value e, or -1 when it is padding or the lower
// mirror of a diagonal block.
template <int NB, bool VEC, bool X1 = false>
__device__ int canonical_slot(int e, uint32_t p) {
    using C = SmallP<NB, VEC, X1>;
    if (X1 && e >= C::NBLK * 64 + NB * 8) {  // the extra column 8 NB
        const int x = e - C::NBLK * 64 - NB * 8;
        const int ecol = 8 * NB;
        if (x < NB * 8) return (int)(p + packed_index(p, x, ecol));  // column x = 8 J + g
        if (x == NB * 8) return (int)(p + packed_index(p, ecol, ecol));
        return ecol;  // its sum
    }
    if (e < C::NBLK * 64) {
        int b = e >> 6;
        const int l = (e & 63) >> 1, m = l >> 2, n = 2 * (l & 3) + (e & 1);
        int J = 0;
        while (b >= NB - J) {
            b -= NB - J;
            ++J;
        }
        const int K = J + b;
        const int a = C::col(J, m), bb = C::col(K, n);
        if (a >= (int)p || bb >= (int)p) return -1;
        if (J == K && a > bb) return -1;
        const int j = a < bb ? a : bb, k = a < bb ? bb : a;
        return (int)(p + packed_index(p, j, k));
    }
    const int e2 = e - C::NBLK * 64;
    const int a = C::col(e2 >> 3, e2 & 7);
    return a < (int)p ? a : -1;
}

// TRC: the tile height as a compile-time constant — kTileRows (the loop is fully unrolled and
// software-pipelined, measured faster) or kBigTileRows (large plans) — or 0: job.tile_rows
// at run time (small plans).
template <int NB, bool VEC, bool X1 = false, uint32_t TRC = kTileRows>
__device__ __forceinline__ void smallp_body(const TileJob& job) {
    using C = SmallP<NB, VEC, X1>;
    constexpr int U = C::U;
    extern __shared__ double red[];  // [kWarps][FRAG]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, kk = lane & 3;
    const uint32_t p = VEC ? 8u * NB : job.p;  // compile-time for the vector layout
    const uint64_t E = partial_len(p);

    for (uint64_t t = job.tile_begin + blockIdx.x; t < job.tile_end; t += gridDim.x) {
        const uint32_t r = range_of_tile(job.tile_prefix, job.n_ranges, t);
        const uint64_t rs = __ldg(job.range_start + r), rc = __ldg(job.range_count + r);
        const uint32_t TR = TRC ? TRC : job.tile_rows;
        const uint64_t row0 = rs + (t - __ldg(job.tile_prefix + r)) * TR;
        const uint64_t left = rs + rc - row0;
        const uint32_t rows = left < TR ? (uint32_t)left : TR;
        const double* __restrict__ tile = job.base + (row0 - job.base_row) * p;

        // shift row c of this range (the gathered table; reading it in place from the shard
        // costs this kernel 16 registers and 1.6% of its bandwidth — measured)
        const double* crow = job.shift != nullptr ? job.shift + (uint64_t)r * p
                             : (!TRC && job.shift_in_place && rc) ? job.base + (rs - job.base_row) * p
                                                               : nullptr;
        double c[NB];
#pragma unroll
        for (int J = 0; J < NB; ++J) {
            const int cj = C::col(J, g);
            c[J] = (crow != nullptr && cj < (int)p) ? crow[cj] : 0.0;
        }
        double acc[C::NBLK][2];
        double s[NB];
#pragma unroll
        for (int b = 0; b < C::NBLK; ++b) acc[b][0] = acc[b][1] = 0.0;
#pragma unroll
        for (int J = 0; J < NB; ++J) s[J] = 0.0;
        // X1: the extra column 8 NB (its shift, d_e x d_j per J, d_e^2, sum)
        const double ce = (X1 && crow != nullptr) ? crow[8 * NB] : 0.0;
        double ae[NB], aee = 0.0, se = 0.0;
#pragma unroll
        for (int J = 0; J < NB; ++J) ae[J] = 0.0;

        const uint32_t nks = rows >> 2;
        const uint32_t kstride = kWarps * 4 * p;  // doubles between a warp's consecutive k-steps
        uint32_t ks = warp;
        const double* rowp = tile + (warp * 4 + kk) * p;
        for (; ks + kWarps * (U - 1) < nks; ks += kWarps * U, rowp += U * kstride) {
            double x[U][NB], xe[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                load_row<NB, VEC>(rowp + u * kstride, g, p, x[u]);
                if (X1) xe[u] = ld_stream(rowp + u * kstride + 8 * NB);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (X1) step_x1<NB>(x[u], xe[u], c, ce, acc, s, ae, aee, se);
                else step<NB>(x[u], c, acc, s);
            }
        }
        if constexpr (TRC == 0 && NB <= 2) {
            // runtime-height tiles (small plans, mostly one per CTA), p <= 17: the warp's last
            // (< U) k-steps in predicated batches of 4 — a round trip per 4 k-steps instead of one
            // each; k-steps past the tile read the shift row and add 0, like the ragged tail below
            // (wider blocks keep the serial loop)
            constexpr int UR = 4;
            for (; ks < nks; ks += kWarps * UR, rowp += UR * kstride) {
                double x[UR][NB], xe[UR];
#pragma unroll
                for (int u = 0; u < UR; ++u) {
                    if (ks + kWarps * u < nks) {
                        load_row<NB, VEC>(rowp + u * kstride, g, p, x[u]);
                        if (X1) xe[u] = ld_stream(rowp + u * kstride + 8 * NB);
                    } else {
#pragma unroll
                        for (int J = 0; J < NB; ++J) x[u][J] = c[J];
                        xe[u] = ce;
                    }
                }
#pragma unroll
                for (int u = 0; u < UR; ++u) {
                    if (X1) step_x1<NB>(x[u], xe[u], c, ce, acc, s, ae, aee, se);
                    else step<NB>(x[u], c, acc, s);
                }
            }
        } else {
            for (; ks < nks; ks += kWarps, rowp += kstride) {
                double x[NB];
                load_row<NB, VEC>(rowp, g, p, x);
                if (X1) step_x1<NB>(x, ld_stream(rowp + 8 * NB), c, ce, acc, s, ae, aee, se);
                else step<NB>(x, c, acc, s);
            }
        }
        // Ragged tail (rows % 4): the warp whose turn k-step nks is; missing rows add 0.
        if ((rows & 3) && warp == (int)(nks % kWarps)) {
            const uint32_t row = nks * 4 + kk;
            double x[NB], xe = ce;
            if (row < rows) {
                load_row<NB, VEC>(tile + (uint64_t)row * p, g, p, x);
                if (X1) xe = ld_stream(tile + (uint64_t)row * p + 8 * NB);
            } else {
#pragma unroll
                for (int J = 0; J < NB; ++J) x[J] = c[J];
            }
            if (X1) step_x1<NB>(x, xe, c, ce, acc, s, ae, aee, se);
            else step<NB>(x, c, acc, s);
        }

        // ---- epilogue: fixed-order reduction to the canonical tile partial ----
#pragma unroll
        for (int J = 0; J < NB; ++J) {
            s[J] += __shfl_xor_sync(0xffffffffu, s[J], 1);
            s[J] += __shfl_xor_sync(0xffffffffu, s[J], 2);
        }
        double* mine = red + warp * C::FRAG;
#pragma unroll
        for (int b = 0; b < C::NBLK; ++b) {
            mine[b * 64 + lane * 2] = acc[b][0];
            mine[b * 64 + lane * 2 + 1] = acc[b][1];
        }
        if (kk == 0) {
#pragma unroll
            for (int J = 0; J < NB; ++J) mine[C::NBLK * 64 + J * 8 + g] = s[J];
        }
        if (X1) {  // the extra column, reduced over the 4 rows of a k-step like the sums
#pragma unroll
            for (int J = 0; J < NB; ++J) {
                ae[J] += __shfl_xor_sync(0xffffffffu, ae[J], 1);
                ae[J] += __shfl_xor_sync(0xffffffffu, ae[J], 2);
            }
            aee += __shfl_xor_sync(0xffffffffu, aee, 1);
            aee += __shfl_xor_sync(0xffffffffu, aee, 2);
            se += __shfl_xor_sync(0xffffffffu, se, 1);
            se += __shfl_xor_sync(0xffffffffu, se, 2);
            double* xm = mine + C::NBLK * 64 + NB * 8;
            if (kk == 0) {
#pragma unroll
                for (int J = 0; J < NB; ++J) xm[J * 8 + g] = ae[J];
            }
            if (lane == 0) {
                xm[NB * 8] = aee;
                xm[NB * 8 + 1] = se;
            }
        }
        __syncthreads();
        double* out = job.tile_partials + t * E;
        for (int e = threadIdx.x; e < C::FRAG; e += kThreads) {
            double v = red[e];
#pragma unroll
            for (int w = 1; w < kWarps; ++w) v += red[w * C::FRAG + e];
            const int slot = canonical_slot<NB, VEC, X1>(e, p);
            if (slot >= 0) out[slot] = v;
        }
        __syncthreads();
    }
}

// The same body under different register budgets.  Unbounded: NB <= 2 compiles to 64
// registers (4 CTAs, 32 warps per SM) and a floor there only changes the allocation for the
// worse.  The wider widths are load-latency-bound at the occupancy their unbounded register
// counts allow, so they take a floor of MINB CTAs per SM (measured per NB, SSTAT_K1_MINB
// overrides): 3 for NB = 3..4 (<= 85 registers, 24 warps; p = 24: 4.2 -> 5.8 TB/s, p = 32:
// 4.2 -> 5.0), 2 for NB = 5 (<= 128; p = 40: +35 %).  NB = 6 spills under a floor of 2 and
// loses 14 %; NB >= 6 stay unbounded.
template <int NB, bool VEC, uint32_t TRC>
__global__ void __launch_bounds__(kThreads) k_smallp(TileJob job) {
    smallp_body<NB, VEC, false, TRC>(job);
}
template <int NB, bool VEC, int MINB, uint32_t TRC>
__global__ void __launch_bounds__(kThreads, MINB) k_smallp_floor(TileJob job) {
    smallp_body<NB, VEC, false, TRC>(job);
}

template <int NB, uint32_t TRC>
__global__ void __launch_bounds__(kThreads) k_smallp_x1(TileJob job) {
    smallp_body<NB, false, true, TRC>(job);
}

template <int NB, uint32_t TRC>
cudaError_t launch_nb_x1(const TileJob& job, int sms, cudaStream_t stream) {
    constexpr size_t smem = sizeof(double) * kWarps * SmallP<NB, false, true>::FRAG;
    static std::atomic<int> cached[64];  // per instantiation (NB, TRC)
    int dev = 0;
    cudaGetDevice(&dev);
    int per_sm = dev < 64 ? cached[dev].load() : 0;
    if (per_sm == 0) {
        cudaError_t e = cudaFuncSetAttribute(k_smallp_x1<NB, TRC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_smallp_x1<NB, TRC>, kThreads, smem);
        if (e != cudaSuccess) return e;
        if (per_sm < 1) per_sm = 1;
        if (dev < 64) cached[dev].store(per_sm);
    }
    if (job.occupancy) {
        *job.occupancy = per_sm;
        return cudaSuccess;
    }
    const uint64_t tiles = job.tile_end - job.tile_begin;
    const uint64_t grid = tiles < (uint64_t)sms * per_sm ? tiles : (uint64_t)sms * per_sm;
    if (grid == 0) return cudaSuccess;
    k_smallp_x1<NB, TRC><<<(unsigned)grid, kThreads, smem, stream>>>(job);
    if (job.launched) *job.launched = (const void*)k_smallp_x1<NB, TRC>;
    return cudaGetLastError();
}

template <int NB, bool VEC, uint32_t TRC>
cudaError_t launch_nb(const TileJob& job, int sms, cudaStream_t stream) {
    constexpr size_t smem = sizeof(double) * kWarps * SmallP<NB, VEC>::FRAG;
    int minb = NB == 3 || NB == 4 ? 3 : (NB == 5 ? 2 : 0);
    if (const char* env = getenv("SSTAT_K1_MINB")) minb = atoi(env);
    void (*kern)(TileJob) = k_smallp<NB, VEC, TRC>;
    if constexpr (NB >= 3 && NB <= 4) {
        if (minb == 3) kern = k_smallp_floor<NB, VEC, 3, TRC>;
        else if (minb == 2) kern = k_smallp_floor<NB, VEC, 2, TRC>;
        else minb = 0;
    } else if constexpr (NB == 5) {
        if (minb == 2) kern = k_smallp_floor<NB, VEC, 2, TRC>;
        else minb = 0;
    } else {
        minb = 0;
    }
    const int variant = minb;  // 0, 2 or 3
    // function attribute + occupancy, once per device and variant (kept off the per-call path)
    static std::atomic<int> cached[4][64];
    int dev = 0;
    cudaGetDevice(&dev);
    int per_sm = dev < 64 ? cached[variant][dev].load() : 0;
    if (per_sm == 0) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
        if (e != cudaSuccess) return e;
        if (per_sm < 1) per_sm = 1;
        if (dev < 64) cached[variant][dev].store(per_sm);
    }
    if (job.occupancy) {
        *job.occupancy = per_sm;
        return cudaSuccess;
    }
    const uint64_t tiles = job.tile_end - job.tile_begin;
    const uint64_t grid = tiles < (uint64_t)sms * per_sm ? tiles : (uint64_t)sms * per_sm;
    if (grid == 0) return cudaSuccess;
    kern<<<(unsigned)grid, kThreads, smem, stream>>>(job);
    if (job.launched) *job.launched = (const void*)kern;
    return cudaGetLastError();
}

template <uint32_t TRC>
cudaError_t launch_smallp_rt(const TileJob& job, int sms, cudaStream_t stream) {
    const uint32_t p = job.p;
    const int nb = (int)((p + 7) / 8);
    // 128-bit loads need p a multiple of 16 and a 16-byte aligned base.
    const bool vec = (p == 8u * nb) && (nb % 2 == 0) && (reinterpret_cast<uintptr_t>(job.base) % 16 == 0);
    // p = 8 NB + 1: the last column by DFMA instead of a nearly empty block row of DMMAs
    // (measured, profiles/r01_k1_x1.log: p = 9 / 17 / 25 / 41 / 49 / 57 +43 / +4 / +20 / +42 /
    // +4 / +8 %)
    if (p % 8 == 1 && p > 1 && !getenv("SSTAT_K1_NO_X1")) {
        switch (p / 8) {
            case 1: return launch_nb_x1<1, TRC>(job, sms, stream);
            case 2: return launch_nb_x1<2, TRC>(job, sms, stream);
            case 3: return launch_nb_x1<3, TRC>(job, sms, stream);
            // NB = 4 (p = 33): 136 registers, one CTA per SM — measured 18 % below the
            // occupancy-floored 5-block-row kernel, which it keeps
            case 5: return launch_nb_x1<5, TRC>(job, sms, stream);
            case 6: return launch_nb_x1<6, TRC>(job, sms, stream);
            case 7: return launch_nb_x1<7, TRC>(job, sms, stream);
            default: break;
        }
    }
    switch (nb) {
        case 1: return launch_nb<1, false, TRC>(job, sms, stream);
        case 2: return vec ? launch_nb<2, true, TRC>(job, sms, stream) : launch_nb<2, false, TRC>(job, sms, stream);
        case 3: return launch_nb<3, false, TRC>(job, sms, stream);
        case 4: return vec ? launch_nb<4, true, TRC>(job, sms, stream) : launch_nb<4, false, TRC>(job, sms, stream);
        case 5: return launch_nb<5, false, TRC>(job, sms, stream);
        case 6: return vec ? launch_nb<6, true, TRC>(job, sms, stream) : launch_nb<6, false, TRC>(job, sms, stream);
        case 7: return launch_nb<7, false, TRC>(job, sms, stream);
        case 8: return vec ? launch_nb<8, true, TRC>(job, sms, stream) : launch_nb<8, false, TRC>(job, sms, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

}  // namespace sstat_b200
