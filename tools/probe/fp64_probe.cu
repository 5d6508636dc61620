// Microbenchmarks that decide the small-p kernel design on B200 (sm_100a):
//   1. DFMA issue throughput (FP64 vector pipe)
//   2. DMMA m8n8k4 f64 throughput (FP64 tensor pipe, legacy warp MMA)
//   3. streaming HBM read bandwidth with 128-bit loads
//   4. a prototype sufficient-statistics pass for p=16 on DMMA fragments
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); std::exit(1);} } while (0)

__global__ void dfma_peak(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void dmma_peak(double* out, int iters) {
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) dmma(c[j][0], c[j][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 4x4 outer product of 8 distinct operand registers (the K2 inner loop without loads)
__global__ void dmma_outer(double* out, int iters) {
  double acc[16][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0.0;
  double f[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) f[a] = threadIdx.x * 1e-3 + a;
  for (int i = 0; i < iters; ++i) {
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

// same, with the operands re-read from shared memory and shifted every k-step (K2's loop)
__global__ void dmma_outer_lds(double* out, int iters) {
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

__global__ void stream_read(const double2* __restrict__ x, size_t n2, double* out) {
  double s0 = 0, s1 = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 v0 = __ldcs(x + i), v1 = __ldcs(x + i + stride), v2 = __ldcs(x + i + 2 * stride), v3 = __ldcs(x + i + 3 * stride);
    s0 += v0.x + v1.x + v2.x + v3.x; s1 += v0.y + v1.y + v2.y + v3.y;
  }
  for (; i < n2; i += stride) { double2 v = __ldcs(x + i); s0 += v.x; s1 += v.y; }
  if (s0 + s1 == 1234.5) out[0] = s0;  // keep the loads alive
}

// Prototype: p=16, each warp walks k-steps of 4 rows; lane (g=l>>2, k=l&3) loads 2 doubles
// X[r+k][2g .. 2g+1] (16 B); column permutation col(J,g) = 2g + J. 3 DMMA per k-step.
template <int U>
__global__ void __launch_bounds__(256) ss16_dmma(const double* __restrict__ X, uint64_t n_rows, double* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  const uint64_t nks = n_rows / 4;
  double c00a = 0, c00b = 0, c01a = 0, c01b = 0, c11a = 0, c11b = 0, s0 = 0, s1 = 0;
  const double2* base = reinterpret_cast<const double2*>(X) + (lane & 3) * 8 + (lane >> 2);
  uint64_t ks = warp;
  for (; ks + (U - 1) * nwarps < nks; ks += U * nwarps) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(base + (ks + u * nwarps) * 32);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      s0 += v[u].x; s1 += v[u].y;
      dmma(c00a, c00b, v[u].x, v[u].x);
      dmma(c01a, c01b, v[u].x, v[u].y);
      dmma(c11a, c11b, v[u].y, v[u].y);
    }
  }
  for (; ks < nks; ks += nwarps) {
    double2 v = __ldcs(base + ks * 32);
    s0 += v.x; s1 += v.y;
    dmma(c00a, c00b, v.x, v.x);
    dmma(c01a, c01b, v.x, v.y);
    dmma(c11a, c11b, v.y, v.y);
  }
  double t = c00a + c00b + c01a + c01b + c11a + c11b + s0 + s1;
  if (t == 1234.5) out[0] = t;
}

// Same pass on the FP64 vector pipe: a row per lane, the 152 entries split over two
// warps (warp-uniform half) reading the row through L1.  Used only to compare pipes.
template <int HALF>
__device__ __forceinline__ void dfma_half(const double* x, double* acc) {
  int o = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j)
#pragma unroll
    for (int k = j; k < 16; ++k) {
      const int e = j * 16 - j * (j - 1) / 2 + (k - j);
      if ((e < 68) == (HALF == 0)) { acc[o] = fma(x[j], x[k], acc[o]); ++o; }
    }
}
__global__ void __launch_bounds__(256) ss16_dfma(const double* __restrict__ X, uint64_t n_rows, double* out) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nthr = gridDim.x * (uint64_t)blockDim.x;
  const int half = (tid >> 5) & 1;
  const uint64_t row0 = (tid >> 6) * 32 + (tid & 31);
  double acc[68];
#pragma unroll
  for (int i = 0; i < 68; ++i) acc[i] = 0;
  for (uint64_t r = row0; r < n_rows; r += nthr >> 1) {
    const double2* rp = reinterpret_cast<const double2*>(X + r * 16);
    double x[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) { double2 v = __ldg(rp + i); x[2 * i] = v.x; x[2 * i + 1] = v.y; }
    if (half == 0) dfma_half<0>(x, acc); else dfma_half<1>(x, acc);
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 68; ++i) t += acc[i];
  if (t == 1234.5) out[0] = t;
}

__global__ void fill(double* x, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x) x[i] = (double)((i * 2654435761u) % 1000) * 1e-3;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  std::printf("device %s SMs %d clock(kHz) %d\n", prop.name, prop.multiProcessorCount, clk);
  const int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 1 << 26));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;

  {  // DFMA
    int iters = 4096, blocks = sms * 8, threads = 256;
    dfma_peak<<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_peak<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fma = (double)blocks * threads * iters * 64;
    std::printf("DFMA: %.2f TFLOP/s (%.1f FMA/clk/SM at base clk)\n", 2 * fma / ms / 1e9, fma / (ms * 1e-3) / sms / (clk * 1e3));
  }
  auto run_dmma = [&](auto kern, int nacc, int warps_per_block) {
    int iters = 2048, blocks = sms * 4, threads = 32 * warps_per_block;
    kern<<<blocks, threads>>>(out, 16);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fma = (double)blocks * (threads / 32) * iters * nacc * 256;
    std::printf("DMMA nacc=%d wpb=%d: %.2f TFLOP/s (%.1f FMA/clk/SM at base clk)\n", nacc, warps_per_block, 2 * fma / ms / 1e9,
                fma / (ms * 1e-3) / sms / (clk * 1e3));
  };
  // occupancy sweep: warps per SM = blocks_per_sm * wpb (grid = sms * blocks_per_sm)
  auto run_occ = [&](auto kern, int nacc, int wpb, int bpsm) {
    int iters = 2048, blocks = sms * bpsm, threads = 32 * wpb;
    kern<<<blocks, threads>>>(out, 16);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fma = (double)blocks * wpb * iters * nacc * 256;
    std::printf("DMMA occupancy: %2d warps/SM, %2d chains/warp: %.2f TFLOP/s\n", wpb * bpsm, nacc, 2 * fma / ms / 1e9);
  };
  for (int w : {1, 2, 4, 8}) run_occ(dmma_peak<16>, 16, w, 1);
  for (int w : {4, 8, 12, 16}) run_occ(dmma_outer, 16, w, 1);
  for (int w : {4, 8, 12, 16}) run_occ(dmma_outer_lds, 16, w, 1);
  run_occ(dmma_peak<16>, 16, 4, 2);
  run_occ(dmma_peak<16>, 16, 4, 4);
  run_dmma(dmma_peak<1>, 1, 4);
  run_dmma(dmma_peak<4>, 4, 4);
  run_dmma(dmma_peak<8>, 8, 8);
  run_dmma(dmma_peak<8>, 8, 16);
  run_dmma(dmma_peak<16>, 16, 8);

  size_t n_rows = 100000000ull;  // 1e8 x 16 doubles = 12.8 GB
  double* X; CK(cudaMalloc(&X, n_rows * 16 * 8));
  fill<<<sms * 8, 256>>>(X, n_rows * 16);
  CK(cudaDeviceSynchronize());
  double bytes = n_rows * 16 * 8.0;
  for (int bpsm : {4, 8, 16}) {
    int blocks = sms * bpsm;
    stream_read<<<blocks, 256>>>((const double2*)X, n_rows * 8, out);
    CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaEventRecord(e0);
      stream_read<<<blocks, 256>>>((const double2*)X, n_rows * 8, out);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    std::printf("stream_read blocks/SM=%d: %.1f GB/s\n", bpsm, bytes / best / 1e6);
  }
  auto run_ss = [&](auto kern, const char* name, int bpsm) {
    int blocks = sms * bpsm;
    kern<<<blocks, 256>>>(X, n_rows, out);
    CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaEventRecord(e0);
      kern<<<blocks, 256>>>(X, n_rows, out);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    std::printf("%s blocks/SM=%d: %.3f ms  %.1f GB/s  %.3e rows/s\n", name, bpsm, best, bytes / best / 1e6, n_rows / (best * 1e-3));
  };
  run_ss(ss16_dmma<4>, "ss16_dmma U4", 8);
  run_ss(ss16_dmma<8>, "ss16_dmma U8", 8);
  run_ss(ss16_dmma<8>, "ss16_dmma U8", 4);
  run_ss(ss16_dmma<16>, "ss16_dmma U16", 4);
  run_ss(ss16_dfma, "ss16_dfma", 1);
  run_ss(ss16_dfma, "ss16_dfma", 2);
  CK(cudaGetLastError());
  return 0;
}
