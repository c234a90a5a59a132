// Row softmax instantiations for SmKernel::kQuakeUnfused (ablation; see softmax_kernels.cuh).
#include "softmax_kernels.cuh"

namespace qk {

cudaError_t launch_softmax_quake_unfused(const SmPlan& plan, const float* in, float* out, size_t rows,
                                  size_t cols, const SmParams& p, uint32_t* flags,
                                  cudaStream_t stream) {
  return launch_k<SmKernel::kQuakeUnfused>(plan, in, out, rows, cols, p, flags, stream);
}

}  // namespace qk
