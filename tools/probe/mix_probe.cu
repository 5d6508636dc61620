// mix_probe.cu — are the FP64 DMMA (tensor) and DFMA pipes separate on B200, and what does
// DMMA sustain over a long (power-limited) run?  Build + run: tools/probe/run_mix_probe.sh
#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); std::exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// mode 0: all warps DMMA; 1: all warps DFMA; 2: even warps DMMA, odd warps DFMA;
// 3: every warp interleaves 16 DMMA with 64 DFMA (x 8 lanes of ILP)
__global__ void mix(double* out, int iters, int mode) {
  const int warp = threadIdx.x >> 5;
  double c[16][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i][0] = c[i][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  const bool do_mma = mode == 0 || mode == 3 || (mode == 2 && (warp & 1) == 0);
  const bool do_fma = mode == 1 || mode == 3 || (mode == 2 && (warp & 1) == 1);
  for (int it = 0; it < iters; ++it) {
    if (do_mma) {
#pragma unroll
      for (int j = 0; j < 16; ++j) dmma(c[j][0], c[j][1], a, b);
    }
    if (do_fma) {
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 1.0000001, 1e-9);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main(int argc, char** argv) {
  const double target_ms = argc > 1 ? atof(argv[1]) : 50.0;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, 1 << 26));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"DMMA only", "DFMA only", "DMMA warps + DFMA warps", "DMMA+DFMA interleaved"};
  for (int mode = 0; mode < 4; ++mode) {
    const int wpb = 8, blocks = sms, threads = 32 * wpb;
    int iters = 256;
    float ms = 0;
    for (;;) {  // scale iters to the target duration
      mix<<<blocks, threads>>>(out, iters, mode);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      mix<<<blocks, threads>>>(out, iters, mode);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms >= target_ms * 0.8 || iters > (1 << 26)) break;
      iters = (int)(iters * (target_ms / (ms > 0.01 ? ms : 0.01)) * 1.1);
    }
    double mma_warps = (mode == 0 || mode == 3) ? wpb : (mode == 2 ? wpb / 2 : 0);
    double fma_warps = (mode == 1 || mode == 3) ? wpb : (mode == 2 ? wpb / 2 : 0);
    const double mma_flop = (double)blocks * mma_warps * iters * 16 * 512;
    const double fma_flop = (double)blocks * fma_warps * 32 * iters * 64 * 2;
    std::printf("%-26s %8.1f ms: DMMA %6.2f TF/s + DFMA %6.2f TF/s = %6.2f TF/s\n", names[mode], ms,
                mma_flop / ms / 1e9, fma_flop / ms / 1e9, (mma_flop + fma_flop) / ms / 1e9);
  }
  return 0;
}
