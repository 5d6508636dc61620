// k_widep.cu — K2: wide-p (p > 64) sufficient statistics, a SYRK on the FP64 DMMA pipe.
//
// Replaces accumulate_into<double> (reference src/suffstats.cpp:50-70) where X^T X is
// compute-bound (p(p+2) flops per 8p bytes).  Column blocks of 8 form an nb x nb grid of
// 8x8 output blocks; its upper triangle is cut into 4x4-block rectangles (I <= J).  A
// consumer warp owns one rectangle and runs the same straight-line program for every
// rectangle — 16 DMMA per k-step over 8 operand fragments, no per-block predicates (blocks
// past p multiply zero fragments; a diagonal rectangle's 6 mirrored blocks are computed and
// dropped), so the warp-synchronous DMMAs are never guarded.  C consumer warps (8 or 4,
// chosen per p so the rectangles fill them) form a group = one CTA; ceil(items / C) groups
// cover the triangle, and the groups of a tile run on neighbouring CTAs with equal work.
//
// Warp-specialised pipeline, no CTA-wide barrier in the loop:
//   * producer warp: one elected lane streams each stage of stage_rows rows into a ring of
//     kStages shared-memory slots with TMA bulk copies (cp.async.bulk, one per row, rows
//     padded to pitch = 4 mod 16 doubles so the 4-row fragment reads are conflict-free),
//     completing on the slot's `full` mbarrier (expect_tx); odd p uses 8-byte cp.async from
//     all 32 lanes with cp.async.mbarrier.arrive;
//   * consumer warps: wait `full`, read fragments (next k-step's loads in flight while the
//     current DMMAs issue), subtract the range shift held in registers, DMMA, then arrive on
//     the slot's `empty` mbarrier; one consumer warp per SMSP already saturates its DMMA
//     unit (measured, profiles/r01_fp64_probe.log), two hide each other's load gaps.
// Column sums of rectangle J ride on the warp that owns rectangle (0, J).  Each (tile, group) writes disjoint
// entries of the tile's canonical partial, so the result is a fixed function of the tile.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace sstat_b200 {
namespace {

// Consumer warps per CTA (one rectangle each) are 8 or 4: with the producer that is at
// most 3 warps per SMSP, so the 152-register budget fits the 16K-register SMSP file.
constexpr int kStages = 4;                    // smem ring depth
constexpr int kMaxStageRows = 16;
constexpr int kStageElems = 4096;             // doubles per stage: stage_rows = min(16, 4096/p) & ~3
constexpr int kMaxItems = 4096;
__constant__ uint32_t c_items[kMaxItems];     // [group][consumer]: idle<<28 | I<<14 | J

constexpr uint32_t kIdle = 1u << 28;

struct WideGeom {
    uint32_t p, nb, nr, pitch, n_groups, stage_rows, consumers;
};

__device__ __forceinline__ uint32_t smem_u32(const void* ptr) { return (uint32_t)__cvta_generic_to_shared(ptr); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// Canonical writes of one 8x8 block (column blocks A <= B) from lane (g, kk).
__device__ __forceinline__ void write_block(double* out, uint32_t p, uint32_t A, uint32_t B, int g, int kk,
                                            const double (&c)[2]) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const uint32_t a = A * 8 + g, b = B * 8 + 2 * kk + i;
        if (a >= p || b >= p) continue;
        if (A == B && a > b) continue;
        out[p + packed_index(p, a < b ? a : b, a < b ? b : a)] = c[i];
    }
}

struct UnitInfo {
    uint64_t t;
    uint32_t grp, r, rows;
    const double* tile;
};

__device__ __forceinline__ UnitInfo unit_info(const TileJob& job, const WideGeom& geo, uint32_t tile_rows,
                                              uint64_t u) {
    UnitInfo ui;
    ui.t = job.tile_begin + u / geo.n_groups;
    ui.grp = (uint32_t)(u % geo.n_groups);
    ui.r = range_of_tile(job.tile_prefix, job.n_ranges, ui.t);
    const uint64_t rs = __ldg(job.range_start + ui.r), rc = __ldg(job.range_count + ui.r);
    const uint64_t row0 = rs + (ui.t - __ldg(job.tile_prefix + ui.r)) * tile_rows;
    const uint64_t left = rs + rc - row0;
    ui.rows = left < tile_rows ? (uint32_t)left : tile_rows;
    ui.tile = job.base + (row0 - job.base_row) * geo.p;
    return ui;
}

__global__ void __maxnreg__(152) k_widep(TileJob job, WideGeom geo, uint32_t tile_rows) {
    extern __shared__ __align__(128) double sm[];  // kStages x (stage_rows x pitch) | full[kStages] | empty[kStages]
    const uint32_t p = geo.p, pitch = geo.pitch, nb = geo.nb, srows = geo.stage_rows;
    const uint32_t slot_elems = srows * pitch;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + kStages * slot_elems);
    uint64_t* empty = full + kStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t consumers = geo.consumers;
    const uint64_t units = (job.tile_end - job.tile_begin) * geo.n_groups;
    const bool bulk = (p % 2 == 0) && (reinterpret_cast<uintptr_t>(job.base) % 16 == 0);

    // the column pad [p, pitch) of every slot is never written by the copies: zero it once
    for (uint32_t i = threadIdx.x; i < kStages * srows * (pitch - p); i += blockDim.x) {
        const uint32_t row = i / (pitch - p), col = p + i % (pitch - p);
        sm[row * pitch + col] = 0.0;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], bulk ? 1u : 32u);
            mbar_init(&empty[s], consumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (warp == (int)consumers) {
        // ---------------- producer ----------------
        uint32_t n = 0;  // global stage counter (slot = n % kStages, phase = (n / kStages) & 1)
        for (uint64_t u = blockIdx.x; u < units; u += gridDim.x) {
            const UnitInfo ui = unit_info(job, geo, tile_rows, u);
            const uint32_t n_stages = (ui.rows + srows - 1) / srows;
            const double* crow = job.shift != nullptr ? job.shift + (uint64_t)ui.r * p : nullptr;
            for (uint32_t sidx = 0; sidx < n_stages; ++sidx, ++n) {
                const uint32_t slot = n % kStages, ph = (n / kStages) & 1;
                mbar_wait(&empty[slot], ph ^ 1);
                const uint32_t r0 = sidx * srows;
                const uint32_t vrows = ui.rows - r0 < srows ? ui.rows - r0 : srows;
                double* dst = sm + slot * slot_elems;
                const double* src = ui.tile + (uint64_t)r0 * p;
                // rows past the tile end hold the shift row, so x - c = 0 there (plain stores,
                // ordered before the release of this lane's arrive below)
                for (uint32_t rr = vrows; rr < srows; ++rr)
                    for (uint32_t j = lane; j < p; j += 32) dst[rr * pitch + j] = crow ? crow[j] : 0.0;
                __syncwarp();
                if (bulk) {
                    if (lane == 0) {
                        mbar_arrive_expect_tx(&full[slot], vrows * p * 8);
                        for (uint32_t rr = 0; rr < vrows; ++rr)
                            bulk_g2s(dst + rr * pitch, src + (uint64_t)rr * p, p * 8, &full[slot]);
                    }
                } else {
                    for (uint32_t rr = 0; rr < vrows; ++rr)
                        for (uint32_t j = lane; j < p; j += 32) cp_async8(dst + rr * pitch + j, src + (uint64_t)rr * p + j);
                    cp_async_arrive_noinc(&full[slot]);
                }
            }
        }
        return;
    }

    // ---------------- consumers ----------------
    const int g = lane >> 2, kk = lane & 3;
    const uint64_t E = partial_len(p);
    uint32_t n = 0;
    for (uint64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const UnitInfo ui = unit_info(job, geo, tile_rows, u);
        const uint32_t item = c_items[ui.grp * consumers + warp];
        const bool idle = item & kIdle;
        const uint32_t I = (item >> 14) & 0x3fff, J = item & 0x3fff;
        // fragment a reads column colI + 8a (a < 4, rectangle I) or colJ + 8(a-4) (rectangle J);
        // columns past p read the zero pad with c = 0, rows past the tile end read c
        const int colI = (int)(32 * I) + g, colJ = (int)(32 * J) + g;
        double cw[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const int col = a < 4 ? colI + 8 * a : colJ + 8 * (a - 4);
            cw[a] = (!idle && col < (int)p && job.shift != nullptr) ? job.shift[(uint64_t)ui.r * p + col] : 0.0;
        }
        const bool sums_here = !idle && I == 0;  // rectangle (0, J) sums the columns of rectangle J
        double acc[16][2], sums[4];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) sums[i] = 0.0;

        const uint32_t n_stages = (ui.rows + srows - 1) / srows;
        for (uint32_t sidx = 0; sidx < n_stages; ++sidx, ++n) {
            const uint32_t slot = n % kStages, ph = (n / kStages) & 1;
            mbar_wait(&full[slot], ph);
            if (idle) {  // padding warp of the last group: keep the ring protocol, skip the math
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[slot]);
                continue;
            }
            const double* st = sm + slot * slot_elems + kk * pitch;
            double f[8], raw[8];
#pragma unroll
            for (int a = 0; a < 8; ++a) raw[a] = st[a < 4 ? colI + 8 * a : colJ + 8 * (a - 4)];
#pragma unroll
            for (int q = 0; q < kMaxStageRows / 4; ++q) {
                if (4u * q >= srows) break;
#pragma unroll
                for (int a = 0; a < 8; ++a) f[a] = raw[a] - cw[a];
                if (4u * (q + 1) < srows) {  // next k-step's loads in flight under this one's DMMAs
                    const double* nx = st + 4 * (q + 1) * pitch;
#pragma unroll
                    for (int a = 0; a < 8; ++a) raw[a] = nx[a < 4 ? colI + 8 * a : colJ + 8 * (a - 4)];
                }
#pragma unroll
                for (int a = 0; a < 4; ++a) sums[a] += f[4 + a];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a * 4 + b][0], acc[a * 4 + b][1], f[a], f[4 + b]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
        }

        // ---- epilogue: disjoint canonical entries of the tile partial ----
        double* out = job.tile_partials + ui.t * E;
        if (!idle) {
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const uint32_t A = 4 * I + a, B = 4 * J + b;
                    if (A <= B && B < nb) write_block(out, p, A, B, g, kk, acc[a * 4 + b]);
                }
        }
        if (sums_here) {
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                sums[a] += __shfl_xor_sync(0xffffffffu, sums[a], 1);
                sums[a] += __shfl_xor_sync(0xffffffffu, sums[a], 2);
            }
            if (kk == 0) {
#pragma unroll
                for (int a = 0; a < 4; ++a)
                    if (colJ + 8 * a < (int)p) out[colJ + 8 * a] = sums[a];
            }
        }
    }
}

// Rectangles (I <= J) of the nr x nr rectangle grid, dealt to groups of C consumer warps;
// C = 8 unless C = 4 leaves markedly fewer idle warps.
std::vector<uint32_t> make_items(uint32_t nr, uint32_t& n_groups, uint32_t& consumers) {
    std::vector<uint32_t> items;
    for (uint32_t I = 0; I < nr; ++I)
        for (uint32_t J = I; J < nr; ++J) items.push_back((I << 14) | J);
    // 8 consumers per CTA unless 4 saves more than an eighth of the slots: fewer, fuller
    // groups re-read each tile fewer times
    uint32_t best = 8, best_slots = (uint32_t)((items.size() + 7) / 8) * 8;
    const uint32_t slots4 = (uint32_t)((items.size() + 3) / 4) * 4;
    if (8 * (best_slots - slots4) > best_slots) {
        best = 4;
        best_slots = slots4;
    }
    consumers = best;
    n_groups = best_slots / best;
    while (items.size() < best_slots) items.push_back(kIdle);
    return items;
}

}  // namespace

uint32_t widep_tile_rows(uint32_t) { return 32768; }

cudaError_t launch_widep(const TileJob& job, int sms, cudaStream_t stream) {
    const uint32_t p = job.p;
    if (p > 2048 || p < 2) return cudaErrorInvalidValue;
    WideGeom geo;
    geo.p = p;
    geo.nb = (p + 7) / 8;
    geo.nr = (geo.nb + 3) / 4;
    // pitch = 4 (mod 16) doubles puts the 4 rows of a k-step in distinct 32-byte bank groups,
    // so each half-warp fragment read is one conflict-free wavefront; rows stay 16-B aligned
    geo.pitch = ((p + 15) / 16) * 16 + 4;
    geo.stage_rows = std::min<uint32_t>(kMaxStageRows, (kStageElems / p) & ~3u);
    if (geo.stage_rows < 4) geo.stage_rows = 4;
    std::vector<uint32_t> items = make_items(geo.nr, geo.n_groups, geo.consumers);
    if (items.size() > (size_t)kMaxItems) return cudaErrorInvalidValue;
    cudaError_t e = cudaMemcpyToSymbolAsync(c_items, items.data(), items.size() * 4, 0, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return e;
    const size_t smem = sizeof(double) * kStages * geo.stage_rows * geo.pitch + 2 * kStages * sizeof(uint64_t);
    e = cudaFuncSetAttribute(k_widep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    const int threads = (int)(geo.consumers + 1) * 32;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_widep, threads, smem);
    if (e != cudaSuccess) return e;
    const uint64_t units = (job.tile_end - job.tile_begin) * geo.n_groups;
    const uint64_t cap = (uint64_t)sms * (per_sm > 0 ? per_sm : 1);
    const uint64_t grid = units < cap ? units : cap;
    if (grid == 0) return cudaSuccess;
    k_widep<<<(unsigned)grid, threads, smem, stream>>>(job, geo, widep_tile_rows(p));
    return cudaGetLastError();
}

}  // namespace sstat_b200
