// k_misc.cu — folds (K3a/K3b), non-finite localisation, reference-order accumulation
// and the measurement generator (K5).
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace sstat_b200 {
namespace {

using ull = unsigned long long;

__device__ __forceinline__ bool finite64(double v) { return isfinite(v); }

// Inverse of packed_index: (j, k) with j <= k for packed position i.
__device__ __forceinline__ void unpack_index(uint32_t p, uint32_t i, uint32_t& j, uint32_t& k) {
    // row j: start(j) = j*p - j(j-1)/2 <= i < start(j+1); estimate then correct
    const double b = 2.0 * p + 1.0;
    int64_t row = (int64_t)floor((b - sqrt(b * b - 8.0 * i)) * 0.5);
    if (row < 0) row = 0;
    auto start = [p](int64_t jj) { return jj * (int64_t)p - jj * (jj - 1) / 2; };
    while (row > 0 && start(row) > (int64_t)i) --row;
    while (row + 1 < (int64_t)p && start(row + 1) <= (int64_t)i) ++row;
    j = (uint32_t)row;
    k = (uint32_t)(row + ((int64_t)i - start(row)));
}

__global__ void k_gather_shift(const double* __restrict__ base, uint64_t base_row, const uint64_t* __restrict__ range_start,
                               const uint64_t* __restrict__ range_count, uint32_t n_ranges, uint32_t p, double* shift) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= (uint64_t)n_ranges * p) return;
    const uint32_t r = (uint32_t)(i / p), j = (uint32_t)(i % p);
    shift[i] = range_count[r] ? base[(range_start[r] - base_row) * p + j] : 0.0;
}

// Lane q of kFoldLanes sums tiles t0+q, t0+q+kFoldLanes, ... of entry e (8 loads in flight).
constexpr int kFoldLanes = 8;

__device__ __forceinline__ double fold_tiles_lane(const double* __restrict__ tp, uint64_t E, uint64_t e, uint64_t t0,
                                                  uint64_t t1, int q) {
    double s = 0.0;
    uint64_t t = t0 + q;
    for (; t + 7 * kFoldLanes < t1; t += 8 * kFoldLanes) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = tp[(t + u * kFoldLanes) * E + e];
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; t < t1; t += kFoldLanes) s += tp[t * E + e];
    return s;
}

// One block (8 warps) per local range.  Tile partials of the range are summed in a fixed
// order (8 interleaved lanes, then lane 0..7), and the shifted moments are mapped back to
// raw moments with c = shift row, n = range rows:
//   s_j  = s'_j + n c_j
//   S_jk = S'_jk + c_j s'_k + c_k s'_j + n c_j c_k
// (exact for integer data below 2^53, like the reference's own sums).
__global__ void __launch_bounds__(256) k_range_fold(const double* __restrict__ tp,
                                                    const uint64_t* __restrict__ tile_prefix,
                                                    const uint64_t* __restrict__ range_count,
                                                    const double* __restrict__ shift, uint32_t p,
                                                    uint64_t first_range, double* rank_buf, uint32_t* flags) {
    extern __shared__ double sm[];  // [p] shifted sums, [p] shift, [kFoldLanes][32] lane partials
    double* ssum = sm;
    double* sc = sm + p;
    double* lanes = sm + 2 * p;
    const uint32_t r = blockIdx.x;
    const uint64_t E = partial_len(p);
    const uint64_t t0 = tile_prefix[r], t1 = tile_prefix[r + 1];
    const double n = (double)range_count[r];
    double* out = rank_buf + kHdr + (uint64_t)r * E;
    const int le = threadIdx.x & 31, q = threadIdx.x >> 5;
    for (int phase = 0; phase < 2; ++phase) {
        const uint64_t lo = phase == 0 ? 0 : p, hi = phase == 0 ? p : E;
        for (uint64_t e0 = lo; e0 < hi; e0 += 32) {
            const uint64_t e = e0 + le;
            lanes[q * 32 + le] = e < hi ? fold_tiles_lane(tp, E, e, t0, t1, q) : 0.0;
            __syncthreads();
            if (q == 0 && e < hi) {
                double S = lanes[le];
#pragma unroll
                for (int w = 1; w < kFoldLanes; ++w) S += lanes[w * 32 + le];
                if (phase == 0) {
                    const double cj = shift ? shift[(uint64_t)r * p + e] : 0.0;
                    ssum[e] = S;
                    sc[e] = cj;
                    out[e] = S + n * cj;
                    if (!finite64(S) || !finite64(cj)) {
                        flags[r] = 1;
                        atomicMin(reinterpret_cast<ull*>(rank_buf), (ull)(first_range + r));
                    }
                } else {
                    if (shift) {
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

// Scans the flagged local ranges for their first non-finite value.  Ranges ascend, so
// the minimum absolute linear index row*p + col lies in the lowest failing range.
__global__ void k_find_nonfinite(const double* __restrict__ base, uint64_t base_row,
                                 const uint64_t* __restrict__ range_start, const uint64_t* __restrict__ range_count,
                                 uint32_t n_ranges, uint32_t p, const uint32_t* __restrict__ flags, double* rank_buf) {
    if (*reinterpret_cast<const ull*>(rank_buf) == ~0ull) return;
    for (uint32_t r = 0; r < n_ranges; ++r) {
        if (!flags[r]) continue;
        const double* rows = base + (range_start[r] - base_row) * p;
        const uint64_t total = range_count[r] * p;
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
             i += (uint64_t)gridDim.x * blockDim.x)
            if (!finite64(rows[i])) atomicMin(reinterpret_cast<ull*>(rank_buf) + 1, (ull)(range_start[r] * p + i));
    }
}

__global__ void k_final_fold(const double* __restrict__ buf, uint64_t rank_stride, uint64_t n_ranges, int world,
                             uint32_t p, uint32_t precision, double* out) {
    const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (e >= partial_len(p)) return;
    out[e] = fold_entry(buf, rank_stride, n_ranges, world, p, precision, e);
}

template <typename Acc>
__device__ __forceinline__ Acc cvt(double v);
template <>
__device__ __forceinline__ double cvt<double>(double v) { return v; }
template <>
__device__ __forceinline__ float cvt<float>(double v) { return __double2float_rn(v); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }

// accumulate_into<Acc> (suffstats.cpp:56-67), one chain per (range, entry):
//   sums:  s  = s + Acc(x_j)                    for each row, ascending
//   cross: S  = S + Acc(x_j) * Acc(x_k)         separate multiply and add
template <typename Acc>
__global__ void k_refexact(const double* __restrict__ base, uint64_t base_row, const uint64_t* __restrict__ range_start,
                           const uint64_t* __restrict__ range_count, uint32_t p, uint64_t first_range, double* hdr,
                           double* out, uint32_t* flags) {
    const uint64_t E = partial_len(p);
    const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint32_t r = blockIdx.y;
    if (e >= E) return;
    const bool is_sum = e < p;
    uint32_t j = (uint32_t)e, k = (uint32_t)e;
    if (!is_sum) unpack_index(p, (uint32_t)(e - p), j, k);
    const double* rows = base + (range_start[r] - base_row) * p;
    const uint64_t n = range_count[r];
    Acc acc = Acc(0);
    uint64_t i = 0;
    constexpr int U = 8;
    for (; i + U <= n; i += U) {
        double xj[U], xk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            xj[u] = rows[(i + u) * p + j];
            xk[u] = rows[(i + u) * p + k];
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            acc = is_sum ? add_rn(acc, cvt<Acc>(xj[u])) : add_rn(acc, mul_rn(cvt<Acc>(xj[u]), cvt<Acc>(xk[u])));
    }
    for (; i < n; ++i) {
        const double a = rows[i * p + j], b = rows[i * p + k];
        acc = is_sum ? add_rn(acc, cvt<Acc>(a)) : add_rn(acc, mul_rn(cvt<Acc>(a), cvt<Acc>(b)));
    }
    const double v = (double)acc;
    out[(uint64_t)r * E + e] = v;
    if (is_sum && !finite64(v)) {
        flags[r] = 1;
        atomicMin(reinterpret_cast<ull*>(hdr), (ull)(first_range + r));
    }
}

// ---- K5 generator: RowRng (rng.hpp:14-38) + Irwin-Hall Gaussians, IEEE ops in fixed order ----
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__global__ void k_generate(double* dst, uint32_t kind, uint64_t seed, double mu, uint32_t n_int, uint64_t first_row,
                           uint64_t n_rows, uint32_t p) {
    const uint64_t golden = 0x9e3779b97f4a7c15ULL;
    const uint64_t mseed = mix64(seed);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_rows;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t index = first_row + i + 1;
        const uint64_t rb = mix64(mseed ^ mix64(index + golden));
        uint64_t pos = 0;
        double* row = dst + i * p;
        uint32_t j = 0;
        if (kind == 0) {
            for (; j < n_int && j < p; ++j) row[j] = (double)(int64_t)(1 + (int64_t)(mix64(rb + (++pos) * golden) % 100));
        } else if (kind == 1) {
            row[0] = (double)index;
            j = 1;
        }
        double zprev = 0.0;
        for (; j < p; ++j) {
            double s = 0.0;
#pragma unroll
            for (int u = 0; u < 12; ++u)
                s = __dadd_rn(s, __dmul_rn((double)(mix64(rb + (++pos) * golden) >> 11), 0x1.0p-53));
            const double z = __dsub_rn(s, 6.0);
            row[j] = __dadd_rn(__dadd_rn(mu, z), __dmul_rn(0.5, zprev));
            zprev = z;
        }
    }
}

}  // namespace

cudaError_t launch_gather_shift(const double* base, uint64_t base_row, const uint64_t* range_start,
                                const uint64_t* range_count, uint32_t n_ranges, uint32_t p, double* shift,
                                cudaStream_t stream) {
    const uint64_t n = (uint64_t)n_ranges * p;
    if (n == 0) return cudaSuccess;
    k_gather_shift<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(base, base_row, range_start, range_count, n_ranges, p,
                                                                    shift);
    return cudaGetLastError();
}

cudaError_t launch_range_fold(const double* tile_partials, const uint64_t* tile_prefix, const uint64_t* range_count,
                              const double* shift, uint32_t n_ranges, uint32_t p, uint64_t first_range,
                              double* rank_buf, uint32_t* flags, cudaStream_t stream) {
    if (n_ranges == 0) return cudaSuccess;
    const size_t smem = (2 * p + kFoldLanes * 32) * sizeof(double);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_range_fold, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k_range_fold<<<n_ranges, 256, smem, stream>>>(tile_partials, tile_prefix, range_count, shift, p,
                                                                     first_range, rank_buf, flags);
    return cudaGetLastError();
}

cudaError_t launch_find_nonfinite(const double* base, uint64_t base_row, const uint64_t* range_start,
                                  const uint64_t* range_count, uint32_t n_ranges, uint32_t p, const uint32_t* flags,
                                  double* rank_buf, int grid, cudaStream_t stream) {
    if (n_ranges == 0) return cudaSuccess;
    k_find_nonfinite<<<grid, 256, 0, stream>>>(base, base_row, range_start, range_count, n_ranges, p, flags, rank_buf);
    return cudaGetLastError();
}

cudaError_t launch_final_fold(const double* buf, uint64_t rank_stride, uint64_t n_ranges, int world, uint32_t p,
                              uint32_t precision, double* out, cudaStream_t stream) {
    const uint64_t E = partial_len(p);
    k_final_fold<<<(unsigned)((E + 127) / 128), 128, 0, stream>>>(buf, rank_stride, n_ranges, world, p, precision, out);
    return cudaGetLastError();
}

cudaError_t launch_refexact(const double* base, uint64_t base_row, const uint64_t* range_start,
                            const uint64_t* range_count, uint32_t n_ranges, uint32_t p, uint32_t precision,
                            uint64_t first_range, double* hdr, double* out, uint32_t* flags, cudaStream_t stream) {
    if (n_ranges == 0) return cudaSuccess;
    const uint64_t E = partial_len(p);
    dim3 grid((unsigned)((E + 127) / 128), n_ranges);
    if (precision == 1)
        k_refexact<float><<<grid, 128, 0, stream>>>(base, base_row, range_start, range_count, p, first_range, hdr, out,
                                                    flags);
    else
        k_refexact<double><<<grid, 128, 0, stream>>>(base, base_row, range_start, range_count, p, first_range, hdr, out,
                                                     flags);
    return cudaGetLastError();
}

cudaError_t launch_generate(double* dst, uint32_t kind, uint64_t seed, double mu, uint32_t n_int, uint64_t first_row,
                            uint64_t n_rows, uint32_t p, cudaStream_t stream) {
    if (n_rows == 0) return cudaSuccess;
    uint64_t blocks = (n_rows + 255) / 256;
    if (blocks > 148ull * 64) blocks = 148ull * 64;
    k_generate<<<(unsigned)blocks, 256, 0, stream>>>(dst, kind, seed, mu, n_int, first_row, n_rows, p);
    return cudaGetLastError();
}

}  // namespace sstat_b200
