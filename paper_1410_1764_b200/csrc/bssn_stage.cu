// bssn_stage.cu -- BSSN fused stage kernels.  Not yet implemented.
#include <cuda_runtime.h>
#include "kernels.hpp"

namespace chemora {
cudaError_t bssn_stage(const StageLaunch&, int, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t bssn_rhs(const StageLaunch&, double*, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace chemora
