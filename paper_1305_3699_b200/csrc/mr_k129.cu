// Channel-count instantiation K = 129 of the RNS Montgomery kernels (see mr_kernels.cuh).
#define MR_K 129
#include "mr_kernels.cuh"

namespace mr {
KernelSet kernels_k129() { return KernelSet{MR_K, upload_base, launch_modexp, launch_combine, launch_mr, launch_modexp_tc, TC_TILES, T, MR_TC_TILES, launch_modexp_tcw}; }
}  // namespace mr
