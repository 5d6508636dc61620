// K1 entry point: the runtime-height kernels (small plans) and the dispatch by tile height.
#include "k_smallp.cuh"

#include <algorithm>
#include <atomic>

namespace sstat_b200 {

cudaError_t launch_smallp_4k(const TileJob& job, int sms, cudaStream_t stream);   // k_smallp_4k.cu
cudaError_t launch_smallp_16k(const TileJob& job, int sms, cudaStream_t stream);  // k_smallp_16k.cu

// Full-height tiles (kTileRows, or kBigTileRows for large plans) take the kernels with the
// compile-time tile height; small plans' shorter tiles the runtime-height instances.
cudaError_t launch_smallp(const TileJob& job, int sms, cudaStream_t stream) {
    if (job.tile_rows == kTileRows) return launch_smallp_4k(job, sms, stream);
    if (job.tile_rows == kBigTileRows) return launch_smallp_16k(job, sms, stream);
    return launch_smallp_rt<0>(job, sms, stream);
}

// CTAs per SM of the runtime-height K1 kernel a width p runs (the smaller of the vector-load and
// scalar-load variants where both exist, so it does not depend on the rows' alignment): the wave
// size of the small-plan tile rule.  Cached per (device, p).
uint32_t smallp_rt_ctas_per_sm(uint32_t p) {
    static std::atomic<int> cache[8][kMaxSmallP + 1];
    int dev = 0;
    cudaGetDevice(&dev);
    if (p == 0 || p > kMaxSmallP) return 4;
    std::atomic<int>& slot = cache[dev & 7][p];
    int v = slot.load();
    if (v == 0) {
        int aligned = 0, unaligned = 0;
        TileJob j{};
        j.p = p;
        j.occupancy = &aligned;
        j.base = nullptr;  // 16-byte aligned: the vector variant where p allows it
        if (launch_smallp_rt<0>(j, 1, nullptr) != cudaSuccess) aligned = 4;
        j.occupancy = &unaligned;
        j.base = reinterpret_cast<const double*>(8);  // 8 bytes off: the scalar variant
        if (launch_smallp_rt<0>(j, 1, nullptr) != cudaSuccess) unaligned = 4;
        cudaGetLastError();
        v = std::max(1, std::min(aligned, unaligned));
        slot.store(v);
    }
    return (uint32_t)v;
}

}  // namespace sstat_b200
