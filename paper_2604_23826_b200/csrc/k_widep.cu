// k_widep.cu — K2: wide-p (p > 64) sufficient statistics on the FP64 DMMA pipe.
#include "common.cuh"
#include "kernels.h"

namespace sstat_b200 {

cudaError_t launch_widep(const TileJob&, int, cudaStream_t) { return cudaErrorNotSupported; }

}  // namespace sstat_b200
