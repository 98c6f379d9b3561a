// Register-resident fast kernel (placeholder until the optimized path lands).
#include <cuda_runtime.h>

#include "vd_internal.h"

namespace vd {

bool fast_path_supported(const DecodeLaunch&) { return false; }

cudaError_t launch_fast_i8(const DecodeLaunch&, cudaStream_t) { return cudaErrorNotSupported; }

}  // namespace vd
