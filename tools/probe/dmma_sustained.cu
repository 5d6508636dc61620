// Sustained FP64 DMMA throughput: the K2 consumer loop without its ring (dmma_outer_lds of
// fp64_probe.cu: 12 warps per SM, a 4x4 fragment outer product per k-step from shared memory with
// the shift subtraction) launched back to back for ~4 s; reports the first and the sustained rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_sustained dmma_sustained.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void outer_lds(double* out, int iters) {
  __shared__ double st[4 * 264];
  for (int i = threadIdx.x; i < 4 * 264; i += blockDim.x) st[i] = i * 1e-3;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, kk = lane & 3;
  double acc[16][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0.0;
  double c[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) c[a] = a * 0.5;
  const double* rowp = st + kk * 260 + g;
  for (int i = 0; i < iters; ++i) {
    double f[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) f[a] = rowp[8 * a + (i & 1) * 64] - c[a];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma(acc[a * 4 + b][0], acc[a * 4 + b][1], f[a], f[4 + b]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sms * 384 * sizeof(double));
  const int iters = 200000;  // ~0.1 s per launch
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  outer_lds<<<sms, 384>>>(out, 16);
  cudaDeviceSynchronize();
  const double flop = 2.0 * sms * 12 * (double)iters * 16 * 256;
  auto t_start = std::chrono::steady_clock::now();
  int k = 0;
  double first = 0, last = 0, total_ms = 0, total_flop = 0;
  while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count() < 4.0) {
    cudaEventRecord(e0);
    outer_lds<<<sms, 384>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = flop / (ms * 1e-3) / 1e12;
    if (k == 0) first = tf;
    last = tf;
    total_ms += ms;
    total_flop += flop;
    ++k;
  }
  std::printf("DMMA outer+lds 12 warps/SM: first launch %.2f TF/s, last %.2f TF/s, mean over %d launches (%.1f s) %.2f TF/s\n",
              first, last, k, total_ms * 1e-3, total_flop / (total_ms * 1e-3) / 1e12);
  return 0;
}
