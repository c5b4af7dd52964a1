// kernels_tc_apply.cu — tcgen05 A.V (placeholder until the tensor-core kernel lands).
#include "kernels.cuh"
namespace ac {
bool apply_tc_supported(int32_t, int32_t, int32_t, int32_t) { return false; }
cudaError_t launch_apply_tc(const ApplyArgs &, int, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace ac
