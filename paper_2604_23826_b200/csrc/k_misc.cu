// k_misc.cu — folds (K3a/K3b), non-finite localisation, reference-order accumulation
// and the measurement generator (K5).
#include <algorithm>
#include <cfloat>

#include "common.cuh"
#include "fold.cuh"
#include "kernels.h"

namespace sstat_b200 {
namespace {

using ull = unsigned long long;

__device__ __forceinline__ bool finite64(double v) { return isfinite(v); }

__global__ void k_gather_shift(const double* __restrict__ base, uint64_t base_row, const uint64_t* __restrict__ range_start,
                               const uint64_t* __restrict__ range_count, uint32_t n_ranges, uint32_t p, double* shift) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= (uint64_t)n_ranges * p) return;
    const uint32_t r = (uint32_t)(i / p), j = (uint32_t)(i % p);
    shift[i] = range_count[r] ? base[(range_start[r] - base_row) * p + j] : 0.0;
}

// K3a: blocks of kTileLanes x 32 threads over (local range x chunk, cross-entry slice)
// (fold_range_block); CLUSTER: the K chunk CTAs of a range form one thread-block cluster.
// The shift row comes from the table, or (shift == nullptr, base != nullptr) in place as the
// range's first row of the resident shard.
template <bool CLUSTER>
__global__ void __launch_bounds__(kTileLanes * 32) k_range_fold(const double* __restrict__ tp,
                                                    const uint64_t* __restrict__ tile_prefix,
                                                    const uint64_t* __restrict__ range_count,
                                                    const double* __restrict__ shift, const double* base,
                                                    uint64_t base_row, const uint64_t* __restrict__ range_start,
                                                    uint32_t p, uint64_t first_range, double* rank_buf,
                                                    uint32_t* flags, uint64_t slice, uint32_t K) {
    extern __shared__ double sm[];
    const uint32_t r = blockIdx.x / K, k = blockIdx.x % K;
    const double* c = shift ? shift + (uint64_t)r * p
                            : (base && range_count[r] ? base + (range_start[r] - base_row) * p : nullptr);
    const uint64_t x0 = (uint64_t)blockIdx.y * slice, x1 = x0 + slice;  // this block's cross entries
    fold_range_block<CLUSTER>(tp, tile_prefix[r], tile_prefix[r + 1], (double)range_count[r], c, p, first_range + r,
                              rank_buf + kHdr + (uint64_t)r * partial_len(p), rank_buf, flags + r, sm, x0, x1, k);
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

// K3b, reference order (SSTAT_FLAG_REFEXACT / Binary32Diagnostic): one thread per entry.
__global__ void k_final_fold_seq(const double* __restrict__ buf, uint64_t rank_stride, uint64_t n_ranges, int world,
                                 uint32_t p, uint32_t precision, double* out) {
    const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t E = partial_len(p);
    if (blockIdx.x == 0)  // append the rank headers
        for (uint32_t h = threadIdx.x; h < (uint32_t)world * kHdr; h += blockDim.x)
            out[E + h] = buf[(h / kHdr) * rank_stride + h % kHdr];
    if (e >= E) return;
    out[e] = fold_entry(buf, rank_stride, n_ranges, world, p, precision, e);
}

// K3b, fast mode (fold_fast): blocks of kFoldLanes x 32 threads over 32-entry slices.
constexpr int kFoldBlock = kFoldLanes * 32;
__global__ void __launch_bounds__(kFoldBlock) k_final_fold_fast(const double* __restrict__ buf, uint64_t rank_stride,
                                                                uint64_t n_ranges, int world, uint32_t p, double* out) {
    __shared__ double sm[kFoldBlock];
    const uint64_t E = partial_len(p);
    const int le = threadIdx.x & 31, q = threadIdx.x >> 5;
    if (blockIdx.x == 0)  // append the rank headers
        for (uint32_t h = threadIdx.x; h < (uint32_t)world * kHdr; h += blockDim.x)
            out[E + h] = buf[(h / kHdr) * rank_stride + h % kHdr];
    const uint64_t e = blockIdx.x * 32ull + le;
    double s = 0.0;
    if (e < E) {  // fold_lane's order, eight loads in flight ahead of the adds
        constexpr int U = 8;
        uint64_t r = q;
        for (; r + (U - 1) * kFoldLanes < n_ranges; r += U * kFoldLanes) {
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = __ldcg(range_partial(buf, rank_stride, n_ranges, world, E, r + u * kFoldLanes) + e);
#pragma unroll
            for (int u = 0; u < U; ++u) s += v[u];
        }
        for (; r < n_ranges; r += kFoldLanes) s += __ldcg(range_partial(buf, rank_stride, n_ranges, world, E, r) + e);
    }
    sm[q * 32 + le] = s;
    __syncthreads();
    if (q == 0 && e < E) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kFoldLanes; ++w) t += sm[w * 32 + le];
        out[e] = t;
    }
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

// The value accumulate_into adds to an entry for one row: Acc(x_j) for a sum, the separate
// product Acc(x_j) * Acc(x_k) for a cross entry.  Selected before the add, so an entry's
// dependent chain is the add alone (a select after two adds put an FSEL on every step of it).
template <typename Acc>
__device__ __forceinline__ Acc ref_term(bool is_sum, double a, double b) {
    const Acc ca = cvt<Acc>(a);
    const Acc prod = mul_rn(ca, cvt<Acc>(b));
    return is_sum ? ca : prod;
}

// Rows [0, cnt) of a staged chunk x (row-major, p columns) into one entry's chain, 16 rows per
// step (C2: 16 rows 18.8 ms, 8 rows 19.1, 32 rows 24.1).  Same operations in the same order as
// accumulate_into.
template <typename Acc>
__device__ __forceinline__ void ref_rows(Acc& acc, const double* x, uint32_t cnt, uint32_t p, uint32_t j, uint32_t k,
                                         bool is_sum) {
    constexpr int U = 16;
    uint32_t i = 0;
    for (; i + U <= cnt; i += U) {
        double xj[U], xk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            xj[u] = x[(i + u) * p + j];
            xk[u] = x[(i + u) * p + k];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc = add_rn(acc, ref_term<Acc>(is_sum, xj[u], xk[u]));
    }
    for (; i < cnt; ++i) acc = add_rn(acc, ref_term<Acc>(is_sum, x[i * p + j], x[i * p + k]));
}

// accumulate_into<Acc> (suffstats.cpp:56-67), one chain per (range, entry):
//   sums:  s  = s + Acc(x_j)                    for each row, ascending
//   cross: S  = S + Acc(x_j) * Acc(x_k)         separate multiply and add
template <typename Acc>
__global__ void k_refexact(const double* __restrict__ base, uint64_t base_row, const uint64_t* __restrict__ range_start,
                           const uint64_t* __restrict__ range_count, uint32_t p, uint64_t first_range, double* hdr,
                           double* out, uint32_t* flags, uint32_t resume_first) {
    const uint64_t E = partial_len(p);
    const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint32_t r = blockIdx.y;
    if (e >= E) return;
    const bool is_sum = e < p;
    uint32_t j = (uint32_t)e, k = (uint32_t)e;
    if (!is_sum) unpack_index(p, (uint32_t)(e - p), j, k);
    const double* rows = base + (range_start[r] - base_row) * p;
    const uint64_t n = range_count[r];
    Acc acc = resume_first && r == 0 ? (Acc)out[e] : Acc(0);  // the range's chain continues
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
        for (int u = 0; u < U; ++u) acc = add_rn(acc, ref_term<Acc>(is_sum, xj[u], xk[u]));
    }
    for (; i < n; ++i) acc = add_rn(acc, ref_term<Acc>(is_sum, rows[i * p + j], rows[i * p + k]));
    const double v = (double)acc;
    out[(uint64_t)r * E + e] = v;
    if (is_sum && !finite64(v)) {
        flags[r] = 1;
        atomicMin(reinterpret_cast<ull*>(hdr), (ull)(first_range + r));
    }
}

// The same chains for p <= 64 with the rows staged: a block's 128 entries share every row of
// the range, so the block copies chunks of kRefChunk rows into shared memory with cp.async
// (double-buffered) and each chain then runs from shared memory — one dependent multiply-add
// per row instead of one global-memory round trip per 8 rows.  Same operations, same order.
// Chunks of ch = min(256, 6144 / p) rows: two buffers stay within 96 KB.
__device__ __forceinline__ void cp_async8_ca(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
template <typename Acc>
__global__ void __launch_bounds__(128) k_refexact_staged(const double* __restrict__ base, uint64_t base_row,
                                                         const uint64_t* __restrict__ range_start,
                                                         const uint64_t* __restrict__ range_count, uint32_t p,
                                                         uint64_t first_range, double* hdr, double* out,
                                                         uint32_t* flags, uint32_t ch, uint32_t resume_first) {
    extern __shared__ double stage[];  // [2][ch * p]
    const uint64_t E = partial_len(p);
    const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint32_t r = blockIdx.y;
    const bool active = e < E;
    const bool is_sum = e < p;
    uint32_t j = active ? (uint32_t)e : 0, k = j;
    if (active && !is_sum) unpack_index(p, (uint32_t)(e - p), j, k);
    const double* rows = base + (range_start[r] - base_row) * p;
    const uint64_t n = range_count[r];
    const uint32_t chunk_elems = ch * p;
    const uint64_t n_chunks = (n + ch - 1) / ch;
    auto issue = [&](uint64_t c) {
        const uint64_t row0 = c * ch;
        const uint32_t cnt = (uint32_t)((n - row0 < (uint64_t)ch ? n - row0 : ch) * p);
        double* dst = stage + (c & 1) * chunk_elems;
        const double* src = rows + row0 * p;
        for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) cp_async8_ca(dst + i, src + i);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    Acc acc = active && resume_first && r == 0 ? (Acc)out[e] : Acc(0);
    if (n_chunks > 0) issue(0);
    for (uint64_t c = 0; c < n_chunks; ++c) {
        if (c + 1 < n_chunks) {
            issue(c + 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        const double* x = stage + (c & 1) * chunk_elems;
        const uint32_t cnt = (uint32_t)(n - c * ch < (uint64_t)ch ? n - c * ch : ch);
        if (active) ref_rows<Acc>(acc, x, cnt, p, j, k, is_sum);
        __syncthreads();  // the buffer is refilled by the next iteration's issue()
    }
    if (!active) return;
    const double v = (double)acc;
    out[(uint64_t)r * E + e] = v;
    if (is_sum && !finite64(v)) {
        flags[r] = 1;
        atomicMin(reinterpret_cast<ull*>(hdr), (ull)(first_range + r));
    }
}

// The same chains with the chunks streamed by TMA: one thread issues each chunk (contiguous rows,
// 16-byte aligned) as a single bulk copy into a kRefStages-deep shared-memory ring completing on
// the slot's mbarrier, so up to kRefStages chunks are in flight per block instead of one; the
// chains then run exactly as in k_refexact_staged (same operations, same order).
constexpr uint32_t kRefStages = 4;
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <typename Acc>
__global__ void __launch_bounds__(128) k_refexact_tma(const double* __restrict__ base, uint64_t base_row,
                                                      const uint64_t* __restrict__ range_start,
                                                      const uint64_t* __restrict__ range_count, uint32_t p,
                                                      uint64_t first_range, double* hdr, double* out, uint32_t* flags,
                                                      uint32_t ch, uint32_t resume_first) {
    extern __shared__ __align__(128) double stage[];  // [kRefStages][ch * p] | full[kRefStages]
    const uint32_t chunk_elems = ch * p;
    uint64_t* full = reinterpret_cast<uint64_t*>(stage + kRefStages * chunk_elems);
    const uint64_t E = partial_len(p);
    const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint32_t r = blockIdx.y;
    const bool active = e < E;
    const bool is_sum = e < p;
    uint32_t j = active ? (uint32_t)e : 0, k = j;
    if (active && !is_sum) unpack_index(p, (uint32_t)(e - p), j, k);
    const double* rows = base + (range_start[r] - base_row) * p;
    const uint64_t n = range_count[r];
    const uint64_t n_chunks = (n + ch - 1) / ch;
    auto issue = [&](uint64_t c) {  // thread 0
        const uint64_t row0 = c * ch;
        const uint32_t elems = (uint32_t)((n - row0 < (uint64_t)ch ? n - row0 : ch) * p);
        const uint32_t bulk = (elems & ~1u) * 8;  // a whole number of 16-byte units
        double* dst = stage + (c % kRefStages) * chunk_elems;
        const double* src = rows + row0 * p;
        uint64_t* bar = &full[c % kRefStages];
        if (elems & 1) dst[elems - 1] = src[elems - 1];  // odd tail double: a plain store, before the arrive
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bulk)
                     : "memory");
        if (bulk)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                    smem_addr(dst)),
                "l"(src), "r"(bulk), "r"(smem_addr(bar))
                : "memory");
    };
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < kRefStages; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_addr(&full[i])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        for (uint64_t c = 0; c < n_chunks && c < kRefStages; ++c) issue(c);
    }
    __syncthreads();
    Acc acc = active && resume_first && r == 0 ? (Acc)out[e] : Acc(0);
    for (uint64_t c = 0; c < n_chunks; ++c) {
        const uint32_t parity = (uint32_t)((c / kRefStages) & 1);
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "WAIT_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
            "@!P1 bra WAIT_%=;\n"
            "}\n" ::"r"(smem_addr(&full[c % kRefStages])),
            "r"(parity)
            : "memory");
        const double* x = stage + (c % kRefStages) * chunk_elems;
        const uint32_t cnt = (uint32_t)(n - c * ch < (uint64_t)ch ? n - c * ch : ch);
        if (active) ref_rows<Acc>(acc, x, cnt, p, j, k, is_sum);
        __syncthreads();  // every chain is done with the slot: refill it
        if (threadIdx.x == 0 && c + kRefStages < n_chunks) issue(c + kRefStages);
    }
    if (!active) return;
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
                              const double* shift, const double* base, uint64_t base_row, const uint64_t* range_start,
                              uint32_t n_ranges, uint32_t p, uint64_t first_range, double* rank_buf, uint32_t* flags,
                              uint32_t chunks, cudaStream_t stream) {
    if (n_ranges == 0) return cudaSuccess;
    // blocks = ranges x chunks x slices of the cross entries; a slice is as wide as the sums so
    // the redundant sums fold costs at most as much as the slice itself
    const uint64_t cross = (uint64_t)p * (p + 1) / 2;
    const uint64_t slice = 32ull * ((p + 31) / 32);
    const size_t smem = fold_smem_doubles(p, slice) * sizeof(double);
    const uint32_t K = chunks < 1 ? 1 : chunks;
    const dim3 grid(n_ranges * K, (unsigned)((cross + slice - 1) / slice));
    auto kern = K > 1 ? k_range_fold<true> : k_range_fold<false>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = K;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kTileLanes * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = K > 1 ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tile_partials, tile_prefix, range_count, shift, base, base_row,
                                       range_start, p, first_range, rank_buf, flags, slice, K);
    if (e != cudaSuccess) return e;
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
                              uint32_t precision, bool reference_order, double* out, cudaStream_t stream) {
    const uint64_t E = partial_len(p);
    if (reference_order)
        k_final_fold_seq<<<(unsigned)((E + 127) / 128), 128, 0, stream>>>(buf, rank_stride, n_ranges, world, p, precision,
                                                                           out);
    else
        k_final_fold_fast<<<(unsigned)((E + 31) / 32), kFoldBlock, 0, stream>>>(buf, rank_stride, n_ranges, world, p, out);
    return cudaGetLastError();
}

cudaError_t launch_refexact(const double* base, uint64_t base_row, const uint64_t* range_start,
                            const uint64_t* range_count, uint32_t n_ranges, uint32_t p, uint32_t precision,
                            uint64_t first_range, double* hdr, double* out, uint32_t* flags, bool rows_aligned16,
                            bool resume_first, cudaStream_t stream) {
    if (n_ranges == 0) return cudaSuccess;
    const uint32_t rf = resume_first ? 1u : 0u;
    const uint64_t E = partial_len(p);
    dim3 grid((unsigned)((E + 127) / 128), n_ranges);
    // TMA ring when every range starts 16-byte aligned (the caller checks; chunks hold an even
    // number of rows); SSTAT_REFEXACT_STAGED=1 keeps the cp.async kernel for comparison
    if (rows_aligned16 && p <= 64 && !getenv("SSTAT_REFEXACT_STAGED")) {
        uint32_t ch = (16384 / (8 * p)) & ~1u;  // 16 KB stages (three blocks per SM), an even number of rows
        const size_t smem = (size_t)kRefStages * ch * p * sizeof(double) + kRefStages * sizeof(uint64_t);
        cudaError_t e;
        if (precision == 1) {
            e = cudaFuncSetAttribute(k_refexact_tma<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            k_refexact_tma<float><<<grid, 128, smem, stream>>>(base, base_row, range_start, range_count, p,
                                                               first_range, hdr, out, flags, ch, rf);
        } else {
            e = cudaFuncSetAttribute(k_refexact_tma<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            k_refexact_tma<double><<<grid, 128, smem, stream>>>(base, base_row, range_start, range_count, p,
                                                                first_range, hdr, out, flags, ch, rf);
        }
        return cudaGetLastError();
    }
    if (p <= 64) {  // rows staged through shared memory
        const uint32_t ch = std::min<uint32_t>(256, 6144 / p);
        const size_t smem = 2ull * ch * p * sizeof(double);
        cudaError_t e;
        if (precision == 1) {
            e = cudaFuncSetAttribute(k_refexact_staged<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            if (e != cudaSuccess) return e;
            k_refexact_staged<float><<<grid, 128, smem, stream>>>(base, base_row, range_start, range_count, p,
                                                                  first_range, hdr, out, flags, ch, rf);
        } else {
            e = cudaFuncSetAttribute(k_refexact_staged<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            if (e != cudaSuccess) return e;
            k_refexact_staged<double><<<grid, 128, smem, stream>>>(base, base_row, range_start, range_count, p,
                                                                   first_range, hdr, out, flags, ch, rf);
        }
        return cudaGetLastError();
    }
    if (precision == 1)
        k_refexact<float><<<grid, 128, 0, stream>>>(base, base_row, range_start, range_count, p, first_range, hdr, out,
                                                    flags, rf);
    else
        k_refexact<double><<<grid, 128, 0, stream>>>(base, base_row, range_start, range_count, p, first_range, hdr, out,
                                                     flags, rf);
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
