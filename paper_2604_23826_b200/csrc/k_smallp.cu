// K1 entry point: the runtime-height kernels (small plans) and the dispatch by tile height.
#include "k_smallp.cuh"

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

}  // namespace sstat_b200
