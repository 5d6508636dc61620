// k_extras.cu — the two passes next to the sufficient-statistics path:
//   * column_sum (reference src/reduce.cpp:32-88): a column's FP64 (or binary32) sum plus an
//     exact 128-bit integer sum while every value is integral and |v| < 2^63 — the
//     identifier validation against n(n+1)/2 (tools/sstat_main.cpp:239-245);
//   * centered co-moments (reference src/suffstats.cpp:107-159): per range, mean and
//     M2 = sum (x - mean)(x - mean)^T from the shifted moments K1 already accumulates
//     (c = the range's first row: mean = c + s'/n, M2 = S' - s' s'^T / n), merged over ranges
//     in ascending order with the pairwise update of merge_comoments.
#include <cstdint>

#include "common.cuh"
#include "fold.cuh"
#include "kernels.h"

namespace sstat_b200 {
namespace {

using u128 = unsigned __int128;
constexpr double kInt63 = 9223372036854775808.0;  // 2^63 (reduce.cpp:28)

// Range / tile partial of column_sum: [float sum, exact lo, exact hi, first non-integral row].
struct ColPart {
    double f;
    unsigned long long lo, hi, bad_row;
};

__device__ __forceinline__ void exact_add(u128& acc, double v, uint64_t row, unsigned long long& bad) {
    // reduce.cpp:56-61: integral and |v| < 2^63 joins the exact sum, else the first such row is noted
    if (v == trunc(v) && fabs(v) < kInt63) acc += (u128)(__int128)(long long)v;
    else if (row < bad) bad = row;
}

// Fast mode: one CTA per tile of kTileRows rows; thread i takes rows i, i+256, ... in order,
// then a fixed pairwise tree over the 256 threads.
__global__ void __launch_bounds__(256) k_colsum_tiles(const double* __restrict__ base, uint64_t base_row, uint32_t p,
                                                      uint32_t column, const uint64_t* __restrict__ range_start,
                                                      const uint64_t* __restrict__ range_count,
                                                      const uint64_t* __restrict__ tile_prefix, uint32_t n_ranges,
                                                      uint64_t tile_begin, uint64_t tile_end, ColPart* out) {
    __shared__ double sf[256];
    __shared__ u128 se[256];
    __shared__ unsigned long long sb[256];
    for (uint64_t t = tile_begin + blockIdx.x; t < tile_end; t += gridDim.x) {
        const uint32_t r = range_of_tile(tile_prefix, n_ranges, t);
        const uint64_t rs = range_start[r], rc = range_count[r];
        const uint64_t row0 = rs + (t - tile_prefix[r]) * kTileRows;
        const uint64_t rows = rs + rc - row0 < kTileRows ? rs + rc - row0 : kTileRows;
        const double* col = base + (row0 - base_row) * p + column;
        double f = 0.0;
        u128 ex = 0;
        unsigned long long bad = ~0ull;
        for (uint64_t i = threadIdx.x; i < rows; i += 256) {
            const double v = __ldcs(col + i * p);
            f += v;
            exact_add(ex, v, row0 + i, bad);
        }
        sf[threadIdx.x] = f;
        se[threadIdx.x] = ex;
        sb[threadIdx.x] = bad;
        __syncthreads();
        for (int w = 128; w > 0; w >>= 1) {
            if ((int)threadIdx.x < w) {
                sf[threadIdx.x] = sf[threadIdx.x] + sf[threadIdx.x + w];
                se[threadIdx.x] += se[threadIdx.x + w];
                sb[threadIdx.x] = sb[threadIdx.x] < sb[threadIdx.x + w] ? sb[threadIdx.x] : sb[threadIdx.x + w];
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            ColPart cp;
            cp.f = sf[0];
            cp.lo = (unsigned long long)se[0];
            cp.hi = (unsigned long long)(se[0] >> 64);
            cp.bad_row = sb[0];
            out[t] = cp;
        }
        __syncthreads();
    }
}

// Per-range fold of the tile partials (ascending tiles), into the rank buffer.
__global__ void k_colsum_range_fold(const ColPart* __restrict__ tiles, const uint64_t* __restrict__ tile_prefix,
                                    uint32_t n_ranges, ColPart* ranges) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_ranges) return;
    double f = 0.0;
    u128 ex = 0;
    unsigned long long bad = ~0ull;
    for (uint64_t t = tile_prefix[r]; t < tile_prefix[r + 1]; ++t) {
        const ColPart cp = tiles[t];
        f += cp.f;
        ex += ((u128)cp.hi << 64) | cp.lo;
        bad = cp.bad_row < bad ? cp.bad_row : bad;
    }
    ColPart o;
    o.f = f;
    o.lo = (unsigned long long)ex;
    o.hi = (unsigned long long)(ex >> 64);
    o.bad_row = bad;
    ranges[r] = o;
}

// Reference order (SSTAT_FLAG_REFEXACT, and always for binary32): one thread per range,
// rows in order, exactly reduce.cpp:43-62 (binary32: f32 += (float)v, stored widened).
__global__ void k_colsum_seq(const double* __restrict__ base, uint64_t base_row, uint32_t p, uint32_t column,
                             const uint64_t* __restrict__ range_start, const uint64_t* __restrict__ range_count,
                             uint32_t n_ranges, uint32_t precision, ColPart* ranges, uint32_t resume_first) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_ranges) return;
    const double* col = base + (range_start[r] - base_row) * p + column;
    double f = 0.0;
    float f32 = 0.0f;
    u128 ex = 0;
    unsigned long long bad = ~0ull;
    if (resume_first && r == 0) {  // a range streamed in pieces: continue its sequential sums
        const ColPart prev = ranges[0];
        f = prev.f;
        f32 = (float)prev.f;
        ex = ((u128)prev.hi << 64) | prev.lo;
        bad = prev.bad_row;
    }
    bool ok = bad == ~0ull;
    for (uint64_t i = 0; i < range_count[r]; ++i) {
        const double v = col[i * p];
        if (precision == 1) f32 = __fadd_rn(f32, __double2float_rn(v));
        else f = __dadd_rn(f, v);
        if (ok) {
            if (v == trunc(v) && fabs(v) < kInt63) {
                ex += (u128)(__int128)(long long)v;
            } else {
                ok = false;
                bad = range_start[r] + i;
            }
        }
    }
    ColPart o;
    o.f = precision == 1 ? (double)f32 : f;
    o.lo = (unsigned long long)ex;
    o.hi = (unsigned long long)(ex >> 64);
    o.bad_row = bad;
    ranges[r] = o;
}

// Final ascending fold over all ranges (merge in reduce.cpp:63-74): float sums add in range
// order from +0.0 (binary32 through float), exact sums add, the note comes from the first
// failing range in fold order.  Range r of rank q lives at buf + q*stride + 1 + (r - first(q))
// (ColPart slots after a one-ColPart rank header {0, status, 0, 0}).  out[0] = the result,
// out[1 + q] = rank q's header.  Thread 0 folds.
__global__ void k_colsum_final(const ColPart* __restrict__ buf, uint64_t rank_stride, uint64_t n_ranges, int world,
                               uint32_t precision, ColPart* out) {
    if (blockIdx.x != 0) return;
    for (int q = threadIdx.x; q < world; q += blockDim.x) out[1 + q] = buf[(uint64_t)q * rank_stride];  // rank headers
    if (threadIdx.x != 0) return;
    double f = 0.0;
    float f32 = 0.0f;
    u128 ex = 0;
    unsigned long long bad = ~0ull;
    for (int q = 0; q < world; ++q) {
        const uint64_t first = (uint64_t)q * n_ranges / world, last = (uint64_t)(q + 1) * n_ranges / world;
        const ColPart* part = buf + (uint64_t)q * rank_stride + 1;
        for (uint64_t r = 0; r < last - first; ++r) {
            const ColPart cp = part[r];
            if (precision == 1) f32 = __fadd_rn(f32, __double2float_rn(cp.f));
            else f = __dadd_rn(f, cp.f);
            ex += ((u128)cp.hi << 64) | cp.lo;
            if (bad == ~0ull && cp.bad_row != ~0ull) bad = cp.bad_row;
        }
    }
    ColPart o;
    o.f = precision == 1 ? (double)f32 : f;
    o.lo = (unsigned long long)ex;
    o.hi = (unsigned long long)(ex >> 64);
    o.bad_row = bad;
    *out = o;
}

// ---------------- co-moments ----------------
// Per local range: mean_j = c_j + s'_j / n, M2_jk = S'_jk - s'_j s'_k / n from the folded
// shifted moments (tile partials, the same order as K3a).  Blocks over (range, M2 slice);
// writes [mean(p) | M2(packed)] and n is implicit (range counts).
__global__ void __launch_bounds__(kTileLanes * 32) k_comoment_range(const double* __restrict__ tp,
                                                        const uint64_t* __restrict__ tile_prefix,
                                                        const uint64_t* __restrict__ range_count,
                                                        const double* __restrict__ shift, uint32_t p, double* out,
                                                        uint64_t first_range, double* rank_hdr, uint32_t* flags,
                                                        uint64_t slice) {
    extern __shared__ double sm[];  // [p] shifted sums, [kTileLanes][32] lanes
    double* ssum = sm;
    double* lanes = sm + p;
    const uint32_t r = blockIdx.x;
    const uint64_t E = partial_len(p);
    const uint64_t t0 = tile_prefix[r], t1 = tile_prefix[r + 1];
    const uint64_t nr = range_count[r];
    const double n = (double)nr;
    const int le = threadIdx.x & 31, q = threadIdx.x >> 5;
    double* o = out + (uint64_t)r * E;
    // blockIdx.y = the slice of M2 entries [p + y slice, p + (y + 1) slice); every slice block
    // folds the p sums (M2 needs them), slice 0 writes the means and the flags
    const uint64_t x0 = (uint64_t)blockIdx.y * slice, x1 = x0 + slice;
    const bool lead = blockIdx.y == 0;
    for (int phase = 0; phase < 2; ++phase) {
        const uint64_t lo = phase == 0 ? 0 : p + x0, hi = phase == 0 ? p : (p + x1 < E ? p + x1 : E);
        for (uint64_t e0 = lo; e0 < hi; e0 += 32) {
            const uint64_t e = e0 + le;
            lanes[q * 32 + le] = e < hi ? fold_tiles_lane(tp, E, e, t0, t1, q) : 0.0;  // K3a's order
            __syncthreads();
            if (q == 0 && e < hi) {
                double S = lanes[le];
                for (int w = 1; w < kTileLanes; ++w) S += lanes[w * 32 + le];
                if (phase == 0) {
                    ssum[e] = S;
                    const double c = shift ? shift[(uint64_t)r * p + e] : 0.0;
                    if (lead) o[e] = nr ? c + S / n : 0.0;
                    if (lead && (!isfinite(S) || !isfinite(c))) {  // check_chunk (suffstats.cpp:33-45), located later
                        flags[r] = 1;
                        atomicMin(reinterpret_cast<unsigned long long*>(rank_hdr), (unsigned long long)(first_range + r));
                    }
                } else {
                    uint32_t j, k;
                    unpack_index(p, (uint32_t)(e - p), j, k);
                    o[e] = nr ? S - ssum[j] * ssum[k] / n : 0.0;
                }
            }
            __syncthreads();
        }
    }
}

// merge_comoments (suffstats.cpp:134-159) over all ranges in ascending order: blocks over the
// M2 entries, ranges sequential.  Every block runs the same mean chain (the p means and the
// deltas, bit-identical across blocks), so each entry sees exactly the single-block sequence
// of operations.  Range r: [mean p | M2 packed] at range_partial(buf, ...), counts[r] rows.
// out: [mean p | M2 packed | rank headers] (block 0 writes the means and headers).
__global__ void __launch_bounds__(256) k_comoment_merge(const double* __restrict__ buf, uint64_t rank_stride,
                                                        uint64_t n_ranges, int world,
                                                        const uint64_t* __restrict__ counts, uint32_t p, double* out) {
    extern __shared__ double sm[];  // [p] mean, [p] delta
    double* mean = sm;
    double* delta = sm + p;
    const uint64_t E = partial_len(p), NP = E - p;
    double* m2 = out + p;
    if (blockIdx.x == 0)  // append the rank headers
        for (uint32_t h = threadIdx.x; h < (uint32_t)world * kHdr; h += blockDim.x)
            out[E + h] = buf[(h / kHdr) * rank_stride + h % kHdr];
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;  // this thread's M2 entry
    const bool has = i < NP;
    uint32_t j = 0, k = 0;
    if (has) unpack_index(p, (uint32_t)i, j, k);
    double acc = 0.0;
    uint64_t na = 0;
    for (uint32_t c = threadIdx.x; c < p; c += blockDim.x) mean[c] = 0.0;
    __syncthreads();
    for (uint64_t r = 0; r < n_ranges; ++r) {
        const uint64_t nb = counts[r];
        if (nb == 0) continue;  // b.n == 0: a unchanged
        const double* pb = range_partial(buf, rank_stride, n_ranges, world, E, r);
        if (na == 0) {  // a.n == 0: a = b
            for (uint32_t c = threadIdx.x; c < p; c += blockDim.x) mean[c] = pb[c];
            if (has) acc = pb[p + i];
            na = nb;
            __syncthreads();
            continue;
        }
        const double dna = (double)na, dnb = (double)nb, dn = dna + dnb;
        for (uint32_t c = threadIdx.x; c < p; c += blockDim.x) delta[c] = __dsub_rn(pb[c], mean[c]);
        __syncthreads();
        const double scale = __ddiv_rn(__dmul_rn(dna, dnb), dn);
        if (has) acc = __dadd_rn(__dadd_rn(acc, pb[p + i]), __dmul_rn(__dmul_rn(delta[j], delta[k]), scale));
        const double frac = __ddiv_rn(dnb, dn);
        __syncthreads();  // every thread has read delta / mean before the means move
        for (uint32_t c = threadIdx.x; c < p; c += blockDim.x) mean[c] = __dadd_rn(mean[c], __dmul_rn(delta[c], frac));
        na += nb;
        __syncthreads();
    }
    if (has) m2[i] = acc;
    if (blockIdx.x == 0)
        for (uint32_t c = threadIdx.x; c < p; c += blockDim.x) out[c] = mean[c];
}

}  // namespace

cudaError_t launch_colsum(const double* base, uint64_t base_row, uint32_t p, uint32_t column,
                          const uint64_t* range_start, const uint64_t* range_count, const uint64_t* tile_prefix,
                          uint32_t n_ranges, uint64_t tile_begin, uint64_t tile_end, bool sequential,
                          uint32_t precision, void* tile_parts, void* range_parts, int sms, bool resume_first,
                          cudaStream_t stream) {
    if (n_ranges == 0) return cudaSuccess;
    if (sequential) {
        k_colsum_seq<<<(n_ranges + 127) / 128, 128, 0, stream>>>(base, base_row, p, column, range_start, range_count,
                                                                  n_ranges, precision, (ColPart*)range_parts,
                                                                  resume_first ? 1u : 0u);
        return cudaGetLastError();
    }
    const uint64_t tiles = tile_end - tile_begin;
    if (tiles > 0) {
        const uint64_t grid = tiles < (uint64_t)sms * 8 ? tiles : (uint64_t)sms * 8;
        k_colsum_tiles<<<(unsigned)grid, 256, 0, stream>>>(base, base_row, p, column, range_start, range_count,
                                                          tile_prefix, n_ranges, tile_begin, tile_end,
                                                          (ColPart*)tile_parts);
    }
    return cudaGetLastError();
}

cudaError_t launch_colsum_range_fold(const void* tile_parts, const uint64_t* tile_prefix, uint32_t n_ranges,
                                     void* range_parts, cudaStream_t stream) {
    if (n_ranges == 0) return cudaSuccess;
    k_colsum_range_fold<<<(n_ranges + 127) / 128, 128, 0, stream>>>((const ColPart*)tile_parts, tile_prefix, n_ranges,
                                                                     (ColPart*)range_parts);
    return cudaGetLastError();
}

cudaError_t launch_colsum_final(const void* buf, uint64_t rank_stride_parts, uint64_t n_ranges, int world,
                                uint32_t precision, void* out, cudaStream_t stream) {
    k_colsum_final<<<1, 32, 0, stream>>>((const ColPart*)buf, rank_stride_parts, n_ranges, world, precision,
                                         (ColPart*)out);
    return cudaGetLastError();
}

cudaError_t launch_comoment_range(const double* tile_partials, const uint64_t* tile_prefix, const uint64_t* range_count,
                                  const double* shift, uint32_t n_ranges, uint32_t p, double* out, uint64_t first_range,
                                  double* rank_hdr, uint32_t* flags, cudaStream_t stream) {
    if (n_ranges == 0) return cudaSuccess;
    const size_t smem = (p + kTileLanes * 32) * sizeof(double);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_comoment_range, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const uint64_t cross = (uint64_t)p * (p + 1) / 2;
    const uint64_t slice = 32ull * ((p + 31) / 32);  // as K3a: the redundant sums fold <= the slice
    const dim3 grid(n_ranges, (unsigned)((cross + slice - 1) / slice));
    k_comoment_range<<<grid, kTileLanes * 32, smem, stream>>>(tile_partials, tile_prefix, range_count, shift, p, out,
                                                              first_range, rank_hdr, flags, slice);
    return cudaGetLastError();
}

cudaError_t launch_comoment_merge(const double* buf, uint64_t rank_stride, uint64_t n_ranges, int world,
                                  const uint64_t* counts, uint32_t p, double* out, cudaStream_t stream) {
    const size_t smem = 2 * p * sizeof(double);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_comoment_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const uint64_t np = (uint64_t)p * (p + 1) / 2;
    k_comoment_merge<<<(unsigned)((np + 255) / 256), 256, smem, stream>>>(buf, rank_stride, n_ranges, world, counts, p,
                                                                          out);
    return cudaGetLastError();
}

}  // namespace sstat_b200
