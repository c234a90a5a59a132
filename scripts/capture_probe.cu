// Probe (not product): which CUDA runtime calls keep a stream capture valid.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o build/capture_probe scripts/capture_probe.cu
// Result: profiles/r01_capture_probe.log (only cudaStreamGetDevice invalidates).
#include <cstdio>
#include <functional>
#include <cuda_runtime.h>
__global__ void k(float* p) { asm volatile("griddepcontrol.wait;"); if (p) p[threadIdx.x] = 1.f; }
__global__ void __cluster_dims__(1,1,1) kc(float* p) { if (p) p[threadIdx.x] = 2.f; }
int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  float* d; cudaMalloc(&d, 4096);
  auto probe = [&](const char* what, std::function<cudaError_t()> fn) {
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    cudaError_t e = fn();
    cudaStreamCaptureStatus cs; cudaStreamIsCapturing(s, &cs);
    cudaGraph_t g; cudaError_t e2 = cudaStreamEndCapture(s, &g);
    printf("%-36s -> %-50s still capturing ok: %d, end: %s\n", what, cudaGetErrorString(e), cs == cudaStreamCaptureStatusActive, cudaGetErrorString(e2));
    cudaGetLastError();
  };
  int dev, v;
  probe("cudaGetDevice", [&] { return cudaGetDevice(&dev); });
  probe("cudaStreamIsCapturing", [&] { cudaStreamCaptureStatus c; return cudaStreamIsCapturing(s, &c); });
  probe("cudaStreamGetDevice", [&] { return cudaStreamGetDevice(s, &dev); });
  probe("cudaPointerGetAttributes", [&] { cudaPointerAttributes a; return cudaPointerGetAttributes(&a, d); });
  probe("cudaPointerGetAttributes(host)", [&] { cudaPointerAttributes a; return cudaPointerGetAttributes(&a, &v); });
  probe("cudaDeviceGetAttribute", [&] { return cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, 0); });
  probe("cudaPeekAtLastError", [&] { return cudaPeekAtLastError(); });
  probe("cudaFuncSetAttribute", [&] { return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000); });
  probe("cudaOccupancyMaxActiveBlocksPerSM", [&] { return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, 256, 0); });
  probe("cudaOccupancyMaxActiveClusters", [&] {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(8); cfg.blockDim = dim3(128);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 4; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1; return cudaOccupancyMaxActiveClusters(&v, k, &cfg); });
  probe("launch PDL x2", [&] {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(1); cfg.blockDim = dim3(32); cfg.stream = s;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, d); if (e) return e; return cudaLaunchKernelEx(&cfg, k, d); });
  probe("launch cluster+PDL", [&] {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(4); cfg.blockDim = dim3(32); cfg.stream = s;
    cudaLaunchAttribute at[2]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension; at[1].val.clusterDim.x = 2; at[1].val.clusterDim.y = 1; at[1].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, d); if (e) return e; return cudaLaunchKernelEx(&cfg, k, d); });
  return 0;
}
