// Dependent FP64 add / multiply-add chain latency on one warp (clock64 around N chained ops),
// the bound of the reference-order kernels (one dependent add per row per entry).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dadd_latency dadd_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_add(double* out, double x, int n, long long* cyc) {
    double s = threadIdx.x;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; ++i) s = __dadd_rn(s, x);
    long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
// s = s + (a * b) with the product off the chain (the reference's -ffp-contract=off order)
__global__ void chain_muladd(double* out, const double* v, int n, long long* cyc) {
    double s = threadIdx.x, a = v[0], b = v[1];
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; ++i) {
        const double prod = __dmul_rn(a, b + i);
        s = __dadd_rn(s, prod);
    }
    long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double *out, *v;
    long long* cyc;
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&v, 16);
    cudaMallocManaged(&cyc, 8);
    double h[2] = {1.0000001, 0.5};
    cudaMemcpy(v, h, 16, cudaMemcpyHostToDevice);
    const int n = 1 << 16;
    for (int w : {1, 4, 32}) {
        chain_add<<<1, 32 * w>>>(out, 1e-9, n, cyc);
        cudaDeviceSynchronize();
        printf("dependent DADD chain, %2d warps on one SM: %.2f cycles/add\n", w, (double)*cyc / n);
        chain_muladd<<<1, 32 * w>>>(out, v, n, cyc);
        cudaDeviceSynchronize();
        printf("dependent DMUL+DADD chain, %2d warps:       %.2f cycles/step\n", w, (double)*cyc / n);
    }
    return 0;
}
