// Row softmax instantiations for SmKernel::kQuake2 (see softmax_kernels.cuh).
#include "softmax_kernels.cuh"

namespace qk {

cudaError_t launch_softmax_quake2(const SmPlan& plan, const float* in, float* out, size_t rows,
                                  size_t cols, const SmParams& p, uint32_t* flags,
                                  cudaStream_t stream) {
  return launch_k<SmKernel::kQuake2>(plan, in, out, rows, cols, p, flags, stream);
}

// Clusters of the persistent pipelines resident at once for one launch shape
// (the planner's occupancy probe; variant 4 = kPipe, 6 = kPipeL2, 7 = kPipeS).
int pipe_resident_probe(int variant, int cluster, int threads, size_t smem) {
  if (variant == 7) {
    return resident_clusters(softmax_pipe_s<SmKernel::kQuake2, 40>, cluster, threads, smem);
  }
  if (variant == 6) {
    return resident_clusters(softmax_pipe_l2<SmKernel::kQuake2, 16>, cluster, threads, smem);
  }
  return resident_clusters(softmax_pipe<SmKernel::kQuake2, true, 16>, cluster, threads, smem);
}

}  // namespace qk
