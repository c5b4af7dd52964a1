// kernels_tc_attend.cu — tcgen05 causal attention (placeholder until the tensor-core kernel lands).
#include "kernels.cuh"
namespace ac {
bool attend_tc_supported(int32_t, int32_t, int32_t) { return false; }
cudaError_t launch_attend_tc(const AttendArgs &, int, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace ac
