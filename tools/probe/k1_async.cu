// K1 (p = 16) prototype: register-direct loads (the shipped K1's scheme) vs a per-warp cp.async
// ring (each lane stages its own 16-byte fragment of the next batches in shared memory, so loads
// stay in flight through the DMMAs and the per-tile epilogue without holding registers).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o k1_async k1_async.cu && ./k1_async
// Both: 16384-row tiles, CTA b takes tiles b, b + G, ...; warp w the k-steps w, w + 8, ... of a
// tile; lane (g, k) = (l >> 2, l & 3) holds X[row k][2g, 2g + 1]; shift, sums, 3 DMMA per k-step;
// per-tile epilogue through shared memory (two barriers, one partial written per tile).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int P = 16;
constexpr uint32_t TR = 16384;
constexpr int KS_W = TR / 4 / 8;  // k-steps per warp per tile

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

struct Acc {
    double c[6] = {0, 0, 0, 0, 0, 0}, s0 = 0, s1 = 0;
    __device__ __forceinline__ void step(double2 v, double2 sh) {
        const double x = v.x - sh.x, y = v.y - sh.y;
        s0 += x;
        s1 += y;
        dmma(c[0], c[1], x, x);
        dmma(c[2], c[3], x, y);
        dmma(c[4], c[5], y, y);
    }
};

__device__ __forceinline__ void epilogue(Acc& a, double* red, double* out, uint64_t t) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* mine = red + warp * 264;
#pragma unroll
    for (int i = 0; i < 6; ++i) mine[i * 32 + lane] = a.c[i];
    mine[192 + lane] = a.s0;
    mine[224 + lane] = a.s1;
    __syncthreads();
    for (int e = threadIdx.x; e < 256; e += 256) {
        double v = red[e];
#pragma unroll
        for (int w = 1; w < 8; ++w) v += red[w * 264 + e];
        if (e < 152) out[t * 152 + e] = v;
    }
    __syncthreads();
    a = Acc{};
}

template <int U>
__global__ void __launch_bounds__(256) k_reg(const double* __restrict__ X, uint64_t n_tiles, double* out) {
    __shared__ double red[8 * 264];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, kk = lane & 3;
    const double2 sh = make_double2(0.5, 0.25);
    Acc a;
    for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const double* base = X + (t * TR + kk) * P + 2 * g;
        for (int ks = warp; ks < KS_W * 8; ks += 8 * U) {
            double2 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = __ldcs(reinterpret_cast<const double2*>(base + (uint64_t)(ks + 8 * u) * 4 * P));
#pragma unroll
            for (int u = 0; u < U; ++u) a.step(v[u], sh);
        }
        epilogue(a, red, out, t);
    }
}

// S slots of B k-steps per warp; the issue side runs S - 1 batches ahead across tiles.
template <int S, int B>
__global__ void __launch_bounds__(256) k_async(const double* __restrict__ X, uint64_t n_tiles, double* out) {
    extern __shared__ __align__(16) double sm[];
    double* red = sm;                                   // 8 x 264 doubles
    double2* ring = reinterpret_cast<double2*>(sm + 8 * 264);  // [8 warps][S][B][32 lanes]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, kk = lane & 3;
    double2* mine = ring + (uint64_t)warp * S * B * 32;
    const double2 sh = make_double2(0.5, 0.25);
    constexpr int NBT = KS_W / B;  // batches per tile per warp
    const uint64_t my_tiles = blockIdx.x < n_tiles ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const uint64_t nb = my_tiles * NBT;
    auto issue = [&](uint64_t q) {
        if (q < nb) {
            const uint64_t t = blockIdx.x + (q / NBT) * gridDim.x;
            const int b0 = (int)(q % NBT) * B;
            const double* base = X + (t * TR + kk) * P + 2 * g;
            double2* dst = mine + (q % S) * B * 32 + lane;
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const double* src = base + (uint64_t)(warp + 8 * (b0 + u)) * 4 * P;
                const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst + u * 32);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
#pragma unroll
    for (int q = 0; q < S - 1; ++q) issue(q);
    Acc a;
    for (uint64_t q = 0; q < nb; ++q) {
        issue(q + S - 1);
        asm volatile("cp.async.wait_group %0;\n" ::"n"(S - 1) : "memory");
        const double2* src = mine + (q % S) * B * 32 + lane;
#pragma unroll
        for (int u = 0; u < B; ++u) a.step(src[u * 32], sh);
        if ((q + 1) % NBT == 0) epilogue(a, red, out, blockIdx.x + (q / NBT) * gridDim.x);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
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

template <int S, int B>
void run_async(const double* X, uint64_t n_tiles, double* out, int sms, double bytes) {
    const size_t smem = (8 * 264 + 8 * S * B * 32 * 2) * sizeof(double);
    cudaFuncSetAttribute(k_async<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_async<S, B>, 256, smem);
    const int G = sms * per_sm;
    float ms = timeit([&] { k_async<S, B><<<G, 256, smem>>>(X, n_tiles, out); }, 20);
    printf("async S=%d B=%2d (%3zu KB smem, %d CTA/SM): %.3f ms %.0f GB/s\n", S, B, smem >> 10, per_sm, ms,
           bytes / ms / 1e6);
}

int main() {
    const uint64_t n_tiles = 6104, n = n_tiles * TR;
    const double bytes = n * P * 8.0;
    double *x, *out;
    cudaMalloc(&x, n * P * 8);
    cudaMalloc(&out, n_tiles * 152 * 8);
    cudaMemset(x, 0, n * P * 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int round = 0; round < 2; ++round) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_reg<16>, 256, 0);
        float ms = timeit([&] { k_reg<16><<<sms * per_sm, 256>>>(x, n_tiles, out); }, 20);
        printf("reg   U=16 (%d CTA/SM)               : %.3f ms %.0f GB/s\n", per_sm, ms, bytes / ms / 1e6);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_reg<8>, 256, 0);
        ms = timeit([&] { k_reg<8><<<sms * per_sm, 256>>>(x, n_tiles, out); }, 20);
        printf("reg   U=8  (%d CTA/SM)               : %.3f ms %.0f GB/s\n", per_sm, ms, bytes / ms / 1e6);
        run_async<2, 8>(x, n_tiles, out, sms, bytes);
        run_async<3, 4>(x, n_tiles, out, sms, bytes);
        run_async<4, 4>(x, n_tiles, out, sms, bytes);
        run_async<3, 8>(x, n_tiles, out, sms, bytes);
        run_async<4, 8>(x, n_tiles, out, sms, bytes);
        run_async<6, 4>(x, n_tiles, out, sms, bytes);
        run_async<8, 4>(x, n_tiles, out, sms, bytes);
    }
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
