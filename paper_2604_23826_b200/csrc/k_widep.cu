// k_widep.cu — K2: wide-p (p > 64) sufficient statistics, a SYRK on the FP64 DMMA pipe.
//
// Replaces accumulate_into<double> (reference src/suffstats.cpp:50-70) where X^T X is
// compute-bound (p(p+2) flops per 8p bytes).  Column blocks of 8 form an nb x nb grid
// of 8x8 output blocks; its upper triangle is cut into 4x4-block rectangles, and each
// warp owns either one off-diagonal rectangle (16 DMMA per k-step over 8 operand
// fragments) or one diagonal rectangle (10 DMMA over 4 fragments).  Eight warps form a
// CTA ("group"); ceil(items / 8) groups cover the triangle, so one tile of rows is
// visited by every group (the re-reads hit L2).  Rows are staged through shared memory
// by cp.async (LDGSTS, double-buffered) with a 64-byte row pad so the 4-row fragment
// reads are 2-wavefront conflict-free.  Column sums come from the warps that own
// diagonal rectangles.  Each (tile, group) writes disjoint entries of the tile's canonical
// partial, so the result is a fixed function of the tile.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace sstat_b200 {
namespace {

constexpr int kMaxStageRows = 16;
constexpr int kStageElems = 4096;  // doubles per stage (stage_rows = min(16, 4096 / p) & ~3)
constexpr int kMaxItems = 2048;
__constant__ uint32_t c_items[kMaxItems];  // [group][warp]: kind<<28 | I<<14 | J

enum : uint32_t { kFull = 0, kDiag = 1, kIdle = 3 };

struct WideGeom {
    uint32_t p, nb, nr, pitch, n_groups, stage_rows;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

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

__global__ void __launch_bounds__(kThreads, 2) k_widep(TileJob job, WideGeom geo, uint32_t tile_rows) {
    extern __shared__ __align__(16) double sm[];  // stage0 | stage1, each stage_rows x pitch
    const uint32_t p = geo.p, pitch = geo.pitch, nb = geo.nb, srows = geo.stage_rows;
    double* stage[2] = {sm, sm + srows * pitch};
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, kk = lane & 3;
    const uint64_t E = partial_len(p);
    const uint64_t units = (job.tile_end - job.tile_begin) * geo.n_groups;
    const bool vec2 = (p % 2 == 0) && (reinterpret_cast<uintptr_t>(job.base) % 16 == 0);

    // zero the column pad once (columns p .. pitch-1 are never written by the copies)
    for (uint32_t i = threadIdx.x; i < 2 * srows * (pitch - p); i += kThreads) {
        const uint32_t row = i / (pitch - p), col = p + i % (pitch - p);
        sm[row * pitch + col] = 0.0;
    }

    for (uint64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const uint64_t t = job.tile_begin + u / geo.n_groups;
        const uint32_t grp = (uint32_t)(u % geo.n_groups);
        const uint32_t item = c_items[grp * kWarps + warp];
        const uint32_t kind = item >> 28, I = (item >> 14) & 0x3fff, J = item & 0x3fff;

        const uint32_t r = range_of_tile(job.tile_prefix, job.n_ranges, t);
        const uint64_t rs = __ldg(job.range_start + r), rc = __ldg(job.range_count + r);
        const uint64_t row0 = rs + (t - __ldg(job.tile_prefix + r)) * tile_rows;
        const uint64_t left = rs + rc - row0;
        const uint32_t rows = left < tile_rows ? (uint32_t)left : tile_rows;
        const double* __restrict__ tile = job.base + (row0 - job.base_row) * p;

        // this lane's operand columns: blocks 4I+a (a < 4) and, for full rectangles, 4J+b
        const int colI = (int)(32 * I) + g, colJ = (int)(32 * J) + g;  // column of fragment a: col0 + 8a
#define COLW(a) ((a) < 4 ? colI + 8 * (a) : colJ + 8 * ((a) - 4))
        double cw[8];
#pragma unroll
        for (int a = 0; a < 8; ++a)
            cw[a] = (job.shift != nullptr && COLW(a) < (int)p) ? job.shift[(uint64_t)r * p + COLW(a)] : 0.0;
        double acc[16][2];
        double s[4];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) s[i] = 0.0;

        const uint32_t n_stages = (rows + srows - 1) / srows;
        auto issue = [&](uint32_t sidx) {
            const uint32_t srow0 = sidx * srows;
            const uint32_t vrows = rows - srow0 < srows ? rows - srow0 : srows;
            const double* src = tile + (uint64_t)srow0 * p;
            double* dst = stage[sidx & 1];
            if (vec2) {
                const uint32_t n2 = vrows * p / 2;
                for (uint32_t i = threadIdx.x; i < n2; i += kThreads) {
                    const uint32_t e = 2 * i, rr = e / p, cc = e % p;
                    cp_async16(dst + rr * pitch + cc, src + e);
                }
            } else {
                const uint32_t n1 = vrows * p;
                for (uint32_t e = threadIdx.x; e < n1; e += kThreads) cp_async8(dst + (e / p) * pitch + e % p, src + e);
            }
            cp_commit();
        };
        __syncthreads();  // previous unit's readers are done with both stages
        issue(0);
        for (uint32_t sidx = 0; sidx < n_stages; ++sidx) {
            if (sidx + 1 < n_stages) {
                issue(sidx + 1);
                cp_wait<1>();
            } else {
                cp_wait<0>();
            }
            __syncthreads();
            const double* st = stage[sidx & 1];
            const uint32_t srow0 = sidx * srows;
            if (kind != kIdle) {
#pragma unroll 1
                for (uint32_t k4 = 0; k4 < srows; k4 += 4) {
                    const bool vrow = srow0 + k4 + kk < rows;  // rows past the tile end add 0
                    const double* rowp = st + (k4 + kk) * pitch;
                    double f[8];
#pragma unroll
                    for (int a = 0; a < 8; ++a) {
                        if (a >= 4 && kind != kFull) break;
                        f[a] = (vrow && COLW(a) < (int)p) ? rowp[COLW(a)] - cw[a] : 0.0;
                    }
                    if (kind == kFull) {
#pragma unroll
                        for (int a = 0; a < 4; ++a)
#pragma unroll
                            for (int b = 0; b < 4; ++b)
                                if (4 * J + b < nb) dmma_8x8x4(acc[a * 4 + b][0], acc[a * 4 + b][1], f[a], f[4 + b]);
                    } else {
                        int i = 0;
#pragma unroll
                        for (int a = 0; a < 4; ++a) {
                            s[a] += f[a];
#pragma unroll
                            for (int b = a; b < 4; ++b, ++i)
                                if (4 * I + b < nb) dmma_8x8x4(acc[i][0], acc[i][1], f[a], f[b]);
                        }
                    }
                }
            }
            __syncthreads();  // stage sidx & 1 is refilled by the next iteration's issue
        }

        // ---- epilogue: disjoint canonical entries of the tile partial ----
        double* out = job.tile_partials + t * E;
        if (kind == kFull) {
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if (4 * J + b < nb && 4 * I + a < nb) write_block(out, p, 4 * I + a, 4 * J + b, g, kk, acc[a * 4 + b]);
        } else if (kind == kDiag) {
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                s[a] += __shfl_xor_sync(0xffffffffu, s[a], 1);
                s[a] += __shfl_xor_sync(0xffffffffu, s[a], 2);
            }
            int i = 0;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = a; b < 4; ++b, ++i)
                    if (4 * I + b < nb) write_block(out, p, 4 * I + a, 4 * I + b, g, kk, acc[i]);
            if (kk == 0)
#pragma unroll
                for (int a = 0; a < 4; ++a)
                    if (COLW(a) < (int)p) out[COLW(a)] = s[a];
#undef COLW
        }
    }
}

// Work items for p: off-diagonal rectangles (16 DMMA per k-step) and diagonal ones (10).
std::vector<uint32_t> make_items(uint32_t nr, uint32_t& n_groups) {
    std::vector<uint32_t> items;
    for (uint32_t I = 0; I < nr; ++I)
        for (uint32_t J = I + 1; J < nr; ++J) items.push_back((kFull << 28) | (I << 14) | J);
    for (uint32_t D = 0; D < nr; ++D) items.push_back((kDiag << 28) | (D << 14) | D);
    n_groups = (uint32_t)((items.size() + kWarps - 1) / kWarps);
    while (items.size() < n_groups * kWarps) items.push_back(kIdle << 28);
    return items;
}

}  // namespace

uint32_t widep_tile_rows(uint32_t) { return 32768; }

cudaError_t launch_widep(const TileJob& job, int sms, cudaStream_t stream) {
    const uint32_t p = job.p;
    if (p > 1024 || p < 2) return cudaErrorInvalidValue;
    WideGeom geo;
    geo.p = p;
    geo.nb = (p + 7) / 8;
    geo.nr = (geo.nb + 3) / 4;
    geo.pitch = ((geo.nr * 32 + 15) / 16) * 16 + 8;  // >= 32*nr columns, pitch = 8 (mod 16) doubles
    geo.stage_rows = std::min<uint32_t>(kMaxStageRows, (kStageElems / p) & ~3u);
    if (geo.stage_rows < 4) geo.stage_rows = 4;
    std::vector<uint32_t> items = make_items(geo.nr, geo.n_groups);
    if (items.size() > (size_t)kMaxItems) return cudaErrorInvalidValue;
    cudaError_t e = cudaMemcpyToSymbolAsync(c_items, items.data(), items.size() * 4, 0, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return e;
    const size_t smem = sizeof(double) * geo.pitch * 2 * geo.stage_rows;
    e = cudaFuncSetAttribute(k_widep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_widep, kThreads, smem);
    if (e != cudaSuccess) return e;
    const uint64_t units = (job.tile_end - job.tile_begin) * geo.n_groups;
    const uint64_t cap = (uint64_t)sms * (per_sm > 0 ? per_sm : 1);
    const uint64_t grid = units < cap ? units : cap;
    if (grid == 0) return cudaSuccess;
    k_widep<<<(unsigned)grid, kThreads, smem, stream>>>(job, geo, widep_tile_rows(p));
    return cudaGetLastError();
}

}  // namespace sstat_b200
