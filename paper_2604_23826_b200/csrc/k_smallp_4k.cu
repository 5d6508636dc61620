// K1 kernels with the compile-time tile height kTileRows (4096 rows).
#include "k_smallp.cuh"

namespace sstat_b200 {
cudaError_t launch_smallp_4k(const TileJob& job, int sms, cudaStream_t stream) {
    return launch_smallp_rt<kTileRows>(job, sms, stream);
}
}  // namespace sstat_b200
