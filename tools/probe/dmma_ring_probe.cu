// Where K2's consumer loop loses DMMA rate: the sustained probe (12 warps, fixed fragments, 95 %
// of the DMMA peak) morphed step by step toward K2's consumer (no producer, no barriers):
//   v0  outer_lds of dmma_sustained.cu (fragments from two fixed addresses)
//   v1  K2's ring addressing: 8-row stages in a 12-slot ring of padded rows (pitch 260), each warp
//       its own 4 x 4 rectangle (colI, colJ), next k-step's fragments loaded under the DMMAs
//       (consume_stage_rect's schedule), shift from registers
//   v2  v1 without the software pipelining (load, shift, DMMA in order)
//   v3  v1 in a 512-thread CTA whose last 4 warps idle at a barrier (K2's producer warpgroup)
//   v5-v8 isolate: same rectangle for every warp, one ring slot, 128-bit loads
//   v9  v1 + the next stage's first fragments loaded under this stage's last DMMAs
//   v10 16-row stages (6 slots), v11 + cross-stage prefetch, v12 two slots
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_ring_probe dmma_ring_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(384, 1) v0(double* out, int iters) {
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

constexpr int PITCH = 260, RING = 12;

template <bool V128 = false>
__device__ __forceinline__ void load8(double (&r)[8], const double* st, int colI, int colJ) {
    if (V128) {
        const double2 a0 = *reinterpret_cast<const double2*>(st + colI), a1 = *reinterpret_cast<const double2*>(st + colI + 2);
        const double2 b0 = *reinterpret_cast<const double2*>(st + colJ), b1 = *reinterpret_cast<const double2*>(st + colJ + 2);
        r[0] = a0.x; r[1] = a0.y; r[2] = a1.x; r[3] = a1.y; r[4] = b0.x; r[5] = b0.y; r[6] = b1.x; r[7] = b1.y;
        return;
    }
#pragma unroll
    for (int f = 0; f < 8; ++f) r[f] = st[f < 4 ? colI + 8 * f : colJ + 8 * (f - 4)];
}
__device__ __forceinline__ void prep(double (&r)[8], const double (&c)[8]) {
#pragma unroll
    for (int f = 0; f < 8; ++f) r[f] -= c[f];
}
__device__ __forceinline__ void mma16(double (&acc)[16][2], const double (&r)[8]) {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma(acc[a * 4 + b][0], acc[a * 4 + b][1], r[a], r[4 + b]);
}

template <int SROWS, bool PIPE, int NT, bool SAMECOL = false, int NRING = RING, bool V128 = false, bool XST = false>
__global__ void __launch_bounds__(NT, 1) vring(double* out, int stages) {
    extern __shared__ double sm[];
    const int slot_elems = SROWS * PITCH;
    for (int i = threadIdx.x; i < NRING * slot_elems + 64; i += blockDim.x) sm[i] = (i % 977) * 1e-3;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, kk = lane & 3;
    if (warp >= 12) {  // K2's producer warpgroup: idle here
        __syncthreads();
        return;
    }
    const int I = SAMECOL ? 1 : warp % 8, J = SAMECOL ? 4 : (warp + 3) % 8;
    // V128: columns permuted within each 32-column group so lane g's 4 fragments are contiguous
    const int colI = V128 ? 32 * I + 4 * g : 32 * I + g, colJ = V128 ? 32 * J + 4 * g : 32 * J + g;
    double c[8];
#pragma unroll
    for (int f = 0; f < 8; ++f) c[f] = f * 0.25;
    double acc[16][2];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0.0;
    int slot = 0;
    constexpr int Q = SROWS / 4;
    if (XST) {  // the next stage's first fragments are loaded under this stage's last DMMAs
        double ra[8], rb[8];
        load8<V128>(ra, sm + kk * PITCH, colI, colJ);
        for (int s = 0; s < stages; ++s) {
            const double* st = sm + slot * slot_elems + kk * PITCH;
            const int nslot = slot + 1 == NRING ? 0 : slot + 1;
            const double* nst = sm + nslot * slot_elems + kk * PITCH;
#pragma unroll
            for (int q = 0; q < Q; q += 2) {
                load8<V128>(rb, st + 4 * (q + 1) * PITCH, colI, colJ);
                prep(ra, c);
                mma16(acc, ra);
                if (q + 2 < Q) load8<V128>(ra, st + 4 * (q + 2) * PITCH, colI, colJ);
                else load8<V128>(ra, nst, colI, colJ);
                prep(rb, c);
                mma16(acc, rb);
            }
            slot = nslot;
        }
    }
    for (int s = 0; s < (XST ? 0 : stages); ++s) {
        const double* st = sm + slot * slot_elems + kk * PITCH;
        if (PIPE) {
            double ra[8], rb[8];
            load8<V128>(ra, st, colI, colJ);
#pragma unroll
            for (int q = 0; q < Q; q += 2) {
                if (q + 1 < Q) load8<V128>(rb, st + 4 * (q + 1) * PITCH, colI, colJ);
                prep(ra, c);
                mma16(acc, ra);
                if (q + 2 < Q) load8<V128>(ra, st + 4 * (q + 2) * PITCH, colI, colJ);
                if (q + 1 < Q) {
                    prep(rb, c);
                    mma16(acc, rb);
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                double r[8];
                load8<V128>(r, st + 4 * q * PITCH, colI, colJ);
                prep(r, c);
                mma16(acc, r);
            }
        }
        if (++slot == NRING) slot = 0;
    }
    if (NT > 384) __syncthreads();
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i][0] + acc[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float timeit(F&& f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 3;
}

template <int SROWS, bool PIPE, int NT, bool SAMECOL = false, int NRING = RING, bool V128 = false, bool XST = false>
void run_ring(const char* name, double* out, int sms) {
    const int ksteps = 200000, stages = ksteps / (SROWS / 4);
    const size_t smem = ((NRING > 0 ? NRING : 1) * SROWS * PITCH + 64) * sizeof(double);
    auto kern = vring<SROWS, PIPE, NT, SAMECOL, NRING, V128, XST>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const float ms = timeit([&] { kern<<<sms, NT, smem>>>(out, stages); });
    const double flop = 2.0 * sms * 12 * (double)ksteps * 16 * 256;
    printf("%-44s %.2f TF/s (%s)\n", name, flop / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, sms * 512 * sizeof(double));
    for (int round = 0; round < 2; ++round) {
        const int iters = 200000;
        const float ms = timeit([&] { v0<<<sms, 384>>>(out, iters); });
        printf("%-44s %.2f TF/s\n", "v0 fixed fragments", 2.0 * sms * 12 * (double)iters * 16 * 256 / (ms * 1e-3) / 1e12);
        run_ring<8, true, 384>("v1 ring, 8-row stages, pipelined", out, sms);
        run_ring<8, false, 384>("v2 ring, 8-row stages, in order", out, sms);
        run_ring<8, true, 512>("v3 v1 + 4 idle warps (512 threads)", out, sms);
        run_ring<8, true, 384, true>("v5 v1, every warp the same rectangle", out, sms);
        run_ring<8, true, 384, false, 1>("v6 v1, one ring slot", out, sms);
        run_ring<8, true, 384, false, RING, true>("v7 v1 with 128-bit fragment loads", out, sms);
        run_ring<8, true, 384, true, 1>("v8 same rectangle + one slot", out, sms);
        run_ring<8, true, 384, false, RING, false, true>("v9 v1 + cross-stage fragment prefetch", out, sms);
        run_ring<16, true, 384, false, 6>("v10 16-row stages, 6 slots", out, sms);
        run_ring<16, true, 384, false, 6, false, true>("v11 v10 + cross-stage prefetch", out, sms);
        run_ring<8, true, 384, false, 2>("v12 v1, two ring slots", out, sms);
    }
    return 0;
}
