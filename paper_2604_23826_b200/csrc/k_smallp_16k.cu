// K1 kernels with the compile-time tile height kBigTileRows (16384 rows, large plans).
#include "k_smallp.cuh"

namespace sstat_b200 {
cudaError_t launch_smallp_16k(const TileJob& job, int sms, cudaStream_t stream) {
    return launch_smallp_rt<kBigTileRows>(job, sms, stream);
}
}  // namespace sstat_b200
