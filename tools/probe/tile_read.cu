// Read-only probe of K1's access pattern at C2 (1e8 x 16 FP64, 12.8 GB): does the order in which
// the CTAs sweep HBM (one contiguous tile per CTA vs the whole grid sweeping one window) set the
// gap between K1 (7.03 TB/s) and a grid-stride read (7.31 TB/s, r01_fp64_probe.log)?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tile_read tile_read.cu && ./tile_read
// Kernels (256 threads, 4 CTAs per SM, 16-byte streaming loads, U loads in flight per thread):
//   grid    grid-stride over the whole array
//   tile    K1's order: CTA b reads tiles b, b + G, ... of TR rows; warp w reads 4-row k-steps
//           w, w + 8, ... of the tile (lane: row kk = l & 3, 16 bytes at column 2 (l >> 2))
//   coop8   8 consecutive CTAs share a tile, CTA c reading its k-steps c, c + 8, ... (the
//           concurrently read tiles drop from 592 to 74)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int P = 16;

__device__ __forceinline__ double2 ldcs2(const double* p) { return __ldcs(reinterpret_cast<const double2*>(p)); }

template <int U>
__global__ void __launch_bounds__(256) k_grid(const double* __restrict__ x, uint64_t n2, double* out) {
    double s = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n2; i += U * stride) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ldcs2(x + 2 * (i + u * stride));
#pragma unroll
        for (int u = 0; u < U; ++u) s += v[u].x + v[u].y;
    }
    for (; i < n2; i += stride) {
        const double2 v = ldcs2(x + 2 * i);
        s += v.x + v.y;
    }
    if (s == 1234.5) out[0] = s;
}

// SPLIT CTAs per tile; each CTA's warps take k-steps sub + SPLIT * (w + 8 i)
template <int U, int SPLIT>
__global__ void __launch_bounds__(256) k_tile(const double* __restrict__ x, uint64_t n_rows, uint32_t TR, double* out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, kk = lane & 3;
    const uint64_t n_tiles = (n_rows + TR - 1) / TR;
    const uint32_t sub = blockIdx.x % SPLIT;
    const uint64_t groups = gridDim.x / SPLIT;
    double s = 0;
    for (uint64_t t = blockIdx.x / SPLIT; t < n_tiles; t += groups) {
        const uint64_t row0 = t * TR;
        const uint32_t rows = (uint32_t)(n_rows - row0 < TR ? n_rows - row0 : TR);
        const uint32_t nks = rows >> 2;
        const uint32_t step = 8 * SPLIT;  // k-steps between a warp's consecutive k-steps
        uint32_t ks = sub + SPLIT * warp;
        const double* base = x + (row0 + kk) * P + 2 * g;
        for (; ks + step * (U - 1) < nks; ks += step * U) {
            double2 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = ldcs2(base + (uint64_t)(ks + u * step) * 4 * P);
#pragma unroll
            for (int u = 0; u < U; ++u) s += v[u].x + v[u].y;
        }
        for (; ks < nks; ks += step) {
            const double2 v = ldcs2(base + (uint64_t)ks * 4 * P);
            s += v.x + v.y;
        }
    }
    if (s == 1234.5) out[0] = s;
}

template <typename F>
float timeit(F&& launch, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    const uint64_t n = 100000000ull;
    const double bytes = n * P * 8.0;
    double *x, *out;
    cudaMalloc(&x, n * P * 8);
    cudaMalloc(&out, 64);
    cudaMemset(x, 0, n * P * 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int G = sms * 4;
    const int reps = 20;
    for (int round = 0; round < 2; ++round) {
        float ms = timeit([&] { k_grid<4><<<G, 256>>>(x, n * P / 2, out); }, reps);
        printf("grid   U4                : %.3f ms %.0f GB/s\n", ms, bytes / ms / 1e6);
        ms = timeit([&] { k_grid<8><<<G, 256>>>(x, n * P / 2, out); }, reps);
        printf("grid   U8                : %.3f ms %.0f GB/s\n", ms, bytes / ms / 1e6);
        for (uint32_t TR : {4096u, 1024u, 512u}) {
            ms = timeit([&] { k_tile<16, 1><<<G, 256>>>(x, n, TR, out); }, reps);
            printf("tile   U16 TR=%4u        : %.3f ms %.0f GB/s\n", TR, ms, bytes / ms / 1e6);
        }
        for (uint32_t TR : {4096u, 8192u, 16384u}) {
            ms = timeit([&] { k_tile<16, 8><<<G, 256>>>(x, n, TR, out); }, reps);
            printf("coop8  U16 TR=%5u       : %.3f ms %.0f GB/s\n", TR, ms, bytes / ms / 1e6);
            ms = timeit([&] { k_tile<8, 8><<<G, 256>>>(x, n, TR, out); }, reps);
            printf("coop8  U8  TR=%5u       : %.3f ms %.0f GB/s\n", TR, ms, bytes / ms / 1e6);
            ms = timeit([&] { k_tile<16, 2><<<G, 256>>>(x, n, TR, out); }, reps);
            printf("coop2  U16 TR=%5u       : %.3f ms %.0f GB/s\n", TR, ms, bytes / ms / 1e6);
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
