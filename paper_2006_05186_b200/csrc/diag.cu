// Diagnostics (not part of the method): FP64 DFMA throughput microbenchmark,
// used by bench.py to state the measured FP64 ceiling beside the derived one
// (MEASURED_PEAKS.json has no FP64 entry).
#include "common.cuh"

namespace bem {
namespace {

__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1234.5678) out[threadIdx.x] = s;  // keep the loop alive
}

}  // namespace
}  // namespace bem

using namespace bem;

extern "C" bem_status bem_debug_fp64_peak(int32_t device, void* cuda_stream, double* flops_per_s) {
  BEM_REQ(flops_per_s, "bem_debug_fp64_peak: NULL output");
  DeviceGuard dg(device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  DBuf<double> out;
  BEM_CK(out.alloc(256));
  const int blocks = nsm * 8, iters = 20000;
  cudaEvent_t e0, e1;
  BEM_CK(cudaEventCreate(&e0));
  BEM_CK(cudaEventCreate(&e1));
  dfma_loop<<<blocks, 256, 0, st>>>(out.p, 100, 0.999999, 1e-7);  // warm-up
  BEM_CK(cudaEventRecord(e0, st));
  dfma_loop<<<blocks, 256, 0, st>>>(out.p, iters, 0.999999, 1e-7);
  BEM_CK(cudaEventRecord(e1, st));
  BEM_CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  BEM_CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *flops_per_s = 2.0 * 16.0 * (double)iters * blocks * 256.0 / (ms * 1e-3);
  return BEM_OK;
}
