// Diagnostics (not part of the method): FP64 DFMA throughput microbenchmark,
// used by bench.py to state the measured FP64 ceiling beside the derived one
// (MEASURED_PEAKS.json has no FP64 entry).
#include "common.cuh"
#include "fastmath.cuh"

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

// FP64 tensor-core (DMMA) throughput: mma.sync m8n8k4 f64, 8 independent
// accumulators per warp.  mode 2 mixes DMMA warps and DFMA warps in one CTA
// to test whether the two share the FP64 datapath.
__global__ void __launch_bounds__(256) dmma_loop(double* out, int iters, int mixed) {
  const int warp = threadIdx.x >> 5;
  if (mixed && (warp & 1)) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters * 2; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = fma(x[i], 0.999999, 1e-7);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 1234.5678) out[threadIdx.x] = s;
    return;
  }
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.5;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5678) out[threadIdx.x] = s;
}

}  // namespace
}  // namespace bem

using namespace bem;

// mode 0: DFMA, 1: DMMA (m8n8k4), 2: half DMMA warps + half DFMA warps.
extern "C" bem_status bem_debug_fp64_peak_ex(int32_t device, void* cuda_stream, int32_t mode, double* flops_per_s) {
  BEM_REQ(flops_per_s, "bem_debug_fp64_peak_ex: NULL output");
  if (mode == 0) return bem_debug_fp64_peak(device, cuda_stream, flops_per_s);
  DeviceGuard dg(device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  DBuf<double> out;
  BEM_CK(out.alloc(256));
  const int blocks = nsm * 4, iters = 20000;
  cudaEvent_t e0, e1;
  BEM_CK(cudaEventCreate(&e0));
  BEM_CK(cudaEventCreate(&e1));
  const int mixed = mode == 2 ? 1 : 0;
  dmma_loop<<<blocks, 256, 0, st>>>(out.p, 100, mixed);
  BEM_CK(cudaEventRecord(e0, st));
  dmma_loop<<<blocks, 256, 0, st>>>(out.p, iters, mixed);
  BEM_CK(cudaEventRecord(e1, st));
  BEM_CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  BEM_CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  // per warp-iteration: 8 DMMA x 512 flop; mixed: half the warps do 2*iters*16*32*2 DFMA flops instead
  const double warps = blocks * 8.0;
  double flops;
  if (!mixed) flops = warps * iters * 8.0 * 512.0;
  else flops = warps / 2 * iters * 8.0 * 512.0 + warps / 2 * (2.0 * iters) * 16.0 * 32.0 * 2.0;
  *flops_per_s = flops / (ms * 1e-3);
  return BEM_OK;
}

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

// ---- hot-path math check: the table-driven exp / sincos of fastmath.cuh (K1, K3
// slice regeneration) evaluated on the device for host inputs.
namespace bem {
namespace {
__global__ void debug_fastmath_kernel(const double* x, int64_t n, double* e, double* sn, double* cs, int v256) {
  __shared__ double et[256];
  __shared__ double2 st[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    et[i] = v256 ? fast::kExp2Tab256[i] : (i < 64 ? fast::kExp2Tab[i] : 0.0);
    st[i] = v256 ? fast::kSinCosTab256[i] : (i < 64 ? fast::kSinCosTab[i] : make_double2(0.0, 0.0));
  }
  __syncthreads();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (v256) {
    e[i] = x[i] <= 0.0 ? fast::exp_neg_tab256(x[i], et) : 0.0;
    fast::sincos_tab256(x[i], st, &sn[i], &cs[i]);
  } else {
    e[i] = x[i] <= 0.0 ? fast::exp_neg_tab(x[i], et) : 0.0;
    fast::sincos_tab(x[i], st, &sn[i], &cs[i]);
  }
}
}  // namespace
}  // namespace bem

extern "C" bem_status bem_debug_fastmath(const double* x, int64_t n, double* e, double* sn, double* cs,
                                         int32_t device, int32_t variant) {
  using namespace bem;
  BEM_REQ(x && e && sn && cs && n >= 0, "bem_debug_fastmath: bad arguments");
  if (n == 0) return BEM_OK;
  DeviceGuard dg(device);
  DBuf<double> dx, de, ds, dc;
  BEM_CK(dx.alloc(n)); BEM_CK(de.alloc(n)); BEM_CK(ds.alloc(n)); BEM_CK(dc.alloc(n));
  BEM_CK(cudaMemcpy(dx.p, x, sizeof(double) * n, cudaMemcpyHostToDevice));
  debug_fastmath_kernel<<<(unsigned)((n + 255) / 256), 256>>>(dx.p, n, de.p, ds.p, dc.p, variant == 256);
  BEM_CK(cudaGetLastError());
  BEM_CK(cudaMemcpy(e, de.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  BEM_CK(cudaMemcpy(sn, ds.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  BEM_CK(cudaMemcpy(cs, dc.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return BEM_OK;
}
