// Diagnostics (not part of the method): one CTA computing D = A B^T with
// tcgen05.mma kind::i8 -- the layout conventions K3's FP64-by-INT8 coupling
// ("far10", far.cu) relies on: A [128][K] int8 either in TMEM (TS: row m -> lane m,
// 4 consecutive K bytes per 32-bit column) or in shared memory, B [N][K] int8 in the
// K-major no-swizzle canonical layout, D [128][N] int32 read back from TMEM.
#include "common.cuh"
#include "tc.cuh"

namespace bem {
namespace {

// canonical K-major no-swizzle byte offset of (row, k) in a [rows][K] int8 tile:
// 8-row x 16-byte core matrices, K-adjacent cores 128 B apart, 8-row groups K*8 B apart
__device__ __forceinline__ uint32_t canon_off(int row, int k, int K) {
  return (uint32_t)((row >> 3) * (K * 8) + (k >> 4) * 128 + (row & 7) * 16 + (k & 15));
}

__global__ void __launch_bounds__(128) i8_gemm_test_kernel(const int8_t* __restrict__ A, const int8_t* __restrict__ B,
                                                          int32_t* __restrict__ D, int K, int N, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t mbar;
  const int t = threadIdx.x, w = t >> 5;
  uint8_t* sB = sm;
  uint8_t* sA = sm + (size_t)N * K;
  for (int i = t; i < N * K / 16; i += 128) {
    const int n = i / (K / 16), kc = i % (K / 16);
    *(uint4*)(sB + canon_off(n, kc * 16, K)) = *(const uint4*)(B + (size_t)n * K + kc * 16);
  }
  if (mode == 1)
    for (int i = t; i < 128 * K / 16; i += 128) {
      const int m = i / (K / 16), kc = i % (K / 16);
      *(uint4*)(sA + canon_off(m, kc * 16, K)) = *(const uint4*)(A + (size_t)m * K + kc * 16);
    }
  if (w == 0) tc::tmem_alloc(&taddr_s, 256);
  if (t == 0) tc::mbar_init(&mbar, 1);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = taddr_s, tD = tbase, tA = tbase + 128;
  const uint32_t lane_base = (uint32_t)(w * 32) << 16;
  if (mode == 0) {
    for (int c = 0; c < K / 4; c += 8) {
      uint32_t v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = *(const uint32_t*)(A + (size_t)t * K + (c + j) * 4);
      tc::tmem_st8(tA + lane_base + c, v);
    }
    tc::wait_st();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (t == 0) {
    const uint32_t id = tc::idesc_i8(128, N);
    for (int kk = 0; kk < K / 32; ++kk) {
      const uint64_t bd = tc::smem_desc(tc::smem_u32(sB) + kk * 256, 128, K * 8);
      if (mode == 0) {
        tc::mma_i8_ts(tD, tA + kk * 8, bd, id, kk > 0);
      } else {
        const uint64_t ad = tc::smem_desc(tc::smem_u32(sA) + kk * 256, 128, K * 8);
        tc::mma_i8_ss(tD, ad, bd, id, kk > 0);
      }
    }
    tc::mma_commit(&mbar);
  }
  __syncwarp();
  tc::mbar_wait(&mbar, 0);
  tc::fence_after();
  for (int c = 0; c < N; c += 16) {
    uint32_t v[16];
    tc::tmem_ld16(tD + lane_base + c, v);
    tc::wait_ld();
#pragma unroll
    for (int j = 0; j < 16; ++j) D[(size_t)t * N + c + j] = (int32_t)v[j];
  }
  tc::fence_before();
  __syncthreads();
  if (w == 0) tc::tmem_dealloc(tbase, 256);
}

}  // namespace
}  // namespace bem

using namespace bem;

extern "C" bem_status bem_debug_i8_gemm(const int8_t* A, const int8_t* B, int32_t* D, int32_t K, int32_t N,
                                        int32_t mode, int32_t device) {
  BEM_REQ(A && B && D, "bem_debug_i8_gemm: NULL argument");
  BEM_REQ(K >= 32 && K <= 512 && K % 32 == 0, "bem_debug_i8_gemm: K must be a multiple of 32 in [32, 512]");
  BEM_REQ(N >= 16 && N <= 128 && N % 16 == 0, "bem_debug_i8_gemm: N must be a multiple of 16 in [16, 128]");
  BEM_REQ(mode == 0 || mode == 1, "bem_debug_i8_gemm: mode 0 (A in TMEM) or 1 (A in smem)");
  DeviceGuard dg(device);
  DBuf<int8_t> dA, dB;
  DBuf<int32_t> dD;
  BEM_CK(dA.alloc((size_t)128 * K)); BEM_CK(dB.alloc((size_t)N * K)); BEM_CK(dD.alloc((size_t)128 * N));
  BEM_CK(cudaMemcpy(dA.p, A, (size_t)128 * K, cudaMemcpyHostToDevice));
  BEM_CK(cudaMemcpy(dB.p, B, (size_t)N * K, cudaMemcpyHostToDevice));
  const size_t smem = (size_t)(N + 128) * K;
  BEM_CK(cudaFuncSetAttribute(i8_gemm_test_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  i8_gemm_test_kernel<<<1, 128, smem>>>(dA.p, dB.p, dD.p, K, N, mode);
  BEM_CK(cudaGetLastError());
  BEM_CK(cudaDeviceSynchronize());
  BEM_CK(cudaMemcpy(D, dD.p, sizeof(int32_t) * 128 * N, cudaMemcpyDeviceToHost));
  return BEM_OK;
}

// ---- tcgen05 kind::i8 issue-rate microbenchmark (diagnostics): one CTA per SM, one thread
// issues `iters` groups of 21 MMAs (M = 128, N, K = 32; the far10 level pattern: six
// accumulators of N columns) with A in TMEM (mode 0) or shared memory (mode 1), a
// commit per group and a wait two groups back.  Returns int8 MACs per second.
namespace bem {
namespace {
__global__ void __launch_bounds__(128, 1) i8_rate_kernel(int iters, int N, int mode, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t mbar[2];
  const int t = threadIdx.x, w = t >> 5;
  for (int i = t; i < 6 * 256 * 32 + 128 * 32 * 6; i += 128) sm[i] = (uint8_t)(i * 7);
  if (w == 0) tc::tmem_alloc(&taddr_s, 512);
  if (t == 0) { tc::mbar_init(&mbar[0], 1); tc::mbar_init(&mbar[1], 1); }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tD = taddr_s, tA = taddr_s + 384;
  const int nacc = N <= 64 ? 6 : N <= 128 ? 3 : 1;  // level accumulators that fit below column 384
  if (mode >= 2 && w == 0) {  // whole warp 0 runs the issue loop, one elected lane issues
    const uint32_t id = tc::idesc_i8(128, N);
    const uint32_t sb = tc::smem_u32(sm);
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int buf = it & 1;
      if (it >= 2) tc::mbar_wait(&mbar[buf], ((it >> 1) - 1) & 1);
#pragma unroll
      for (int ia = 0; ia < 6; ++ia)
#pragma unroll
        for (int ib = 0; ib < 6 - ia; ++ib) {
          const uint64_t bd = tc::smem_desc(sb + ib * (N * 32), 128, 256);
          tc::mma_i8_ts_warp(tD + ((ia + ib) % nacc) * N, tA + ia * 8, bd, id, 1u);
        }
      tc::mma_commit_warp(&mbar[buf]);
    }
    const int last = iters - 1;
    tc::mbar_wait(&mbar[last & 1], (last >> 1) & 1);
    if (t == 0) cyc[blockIdx.x] = clock64() - c0;
  }
  if (mode < 2 && t == 0) {
    const uint32_t id = tc::idesc_i8(128, N);
    const uint32_t sb = tc::smem_u32(sm), sa = tc::smem_u32(sm + 6 * 256 * 32);
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int buf = it & 1;
      if (it >= 2) tc::mbar_wait(&mbar[buf], ((it >> 1) - 1) & 1);
      for (int ia = 0; ia < 6; ++ia)
        for (int ib = 0; ib < 6 - ia; ++ib) {
          const uint64_t bd = tc::smem_desc(sb + ib * (N * 32), 128, 256);
          const uint32_t d = tD + ((ia + ib) % nacc) * N;
          if (mode == 0) tc::mma_i8_ts(d, tA + ia * 8, bd, id, 1u);
          else tc::mma_i8_ss(d, tc::smem_desc(sa + ia * 4096, 128, 256), bd, id, 1u);
        }
      tc::mma_commit(&mbar[buf]);
    }
    const int last = iters - 1;
    tc::mbar_wait(&mbar[last & 1], (last >> 1) & 1);
    cyc[blockIdx.x] = clock64() - c0;
  }
  tc::fence_before();
  __syncthreads();
  if (w == 0) tc::tmem_dealloc(taddr_s, 512);
}
}  // namespace
}  // namespace bem

extern "C" bem_status bem_debug_i8_rate(int32_t N, int32_t mode, int32_t iters, int32_t device, double* macs_per_s,
                                        double* cycles_per_mma) {
  using namespace bem;
  BEM_REQ(macs_per_s && cycles_per_mma, "bem_debug_i8_rate: NULL output");
  BEM_REQ(N == 32 || N == 64 || N == 128 || N == 256, "bem_debug_i8_rate: N in {32, 64, 128, 256}");
  DeviceGuard dg(device);
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  DBuf<long long> cyc;
  BEM_CK(cyc.alloc(nsm));
  const size_t smem = 6 * 256 * 32 + 128 * 32 * 6;
  BEM_CK(cudaFuncSetAttribute(i8_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  i8_rate_kernel<<<nsm, 128, smem>>>(10, N, mode, cyc.p);
  cudaEvent_t e0, e1;
  BEM_CK(cudaEventCreate(&e0));
  BEM_CK(cudaEventCreate(&e1));
  BEM_CK(cudaEventRecord(e0));
  i8_rate_kernel<<<nsm, 128, smem>>>(iters, N, mode, cyc.p);
  BEM_CK(cudaEventRecord(e1));
  BEM_CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  BEM_CK(cudaEventElapsedTime(&ms, e0, e1));
  std::vector<long long> h(nsm);
  BEM_CK(cudaMemcpy(h.data(), cyc.p, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double mmas = 21.0 * iters;
  *macs_per_s = (double)nsm * mmas * 128.0 * N * 32.0 / (ms * 1e-3);
  *cycles_per_mma = (double)h[0] / mmas;
  return BEM_OK;
}

// ---- CTA-pair (cta_group::2) layout test: D = A B^T with M = 256 over a cluster of two
// CTAs.  CTA r holds A rows [128 r, 128 r + 128) in its TMEM and B rows [r N/2, (r + 1) N/2)
// in its shared memory; each CTA reads its 128 D rows x N columns back from its TMEM.
namespace bem {
namespace {
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    i8_pair_test_kernel(const int8_t* __restrict__ A, const int8_t* __restrict__ B, int32_t* __restrict__ D, int K,
                        int N) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t ready, done;
  const int t = threadIdx.x, w = t >> 5;
  const uint32_t rank = tc::cluster_rank();
  const int nh = N / 2;
  for (int i = t; i < nh * K / 16; i += 128) {
    const int n = i / (K / 16), kc = i % (K / 16);
    *(uint4*)(sm + canon_off(n, kc * 16, K)) = *(const uint4*)(B + (size_t)(rank * nh + n) * K + kc * 16);
  }
  if (w == 0) tc::tmem_alloc2(&taddr_s, 256);
  if (t == 0) {
    tc::mbar_init(&ready, 2);
    tc::mbar_init(&done, 1);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::fence_before();
  tc::cluster_sync();
  tc::fence_after();
  const uint32_t tD = taddr_s, tA = taddr_s + 128;
  const uint32_t lane_base = (uint32_t)(w * 32) << 16;
  for (int c = 0; c < K / 4; c += 8) {
    uint32_t v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = *(const uint32_t*)(A + (size_t)(rank * 128 + t) * K + (c + j) * 4);
    tc::tmem_st8(tA + lane_base + c, v);
  }
  tc::wait_st();
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  if (t == 0) tc::mbar_arrive_remote(tc::smem_u32(&ready), 0);
  if (rank == 0 && w == 0) {
    tc::mbar_wait_a(tc::smem_u32(&ready), 0);
    tc::fence_after();
    const uint32_t id = tc::idesc_i8(256, N);
    for (int kk = 0; kk < K / 32; ++kk)
      tc::mma2_i8_ts_warp(tD, tA + kk * 8, tc::smem_desc(tc::smem_u32(sm) + kk * 256, 128, K * 8), id, kk > 0);
    tc::mma2_commit_mc_warp(tc::smem_u32(&done), 3);
  }
  tc::mbar_wait_a(tc::smem_u32(&done), 0);
  tc::fence_after();
  for (int c = 0; c < N; c += 16) {
    uint32_t v[16];
    tc::tmem_ld16(tD + lane_base + c, v);
    tc::wait_ld();
#pragma unroll
    for (int j = 0; j < 16; ++j) D[(size_t)(rank * 128 + t) * N + c + j] = (int32_t)v[j];
  }
  tc::fence_before();
  tc::cluster_sync();
  if (w == 0) tc::tmem_dealloc2(taddr_s, 256);
}
}  // namespace
}  // namespace bem

extern "C" bem_status bem_debug_i8_gemm_pair(const int8_t* A, const int8_t* B, int32_t* D, int32_t K, int32_t N,
                                             int32_t device) {
  using namespace bem;
  BEM_REQ(A && B && D, "bem_debug_i8_gemm_pair: NULL argument");
  BEM_REQ(K >= 32 && K <= 512 && K % 32 == 0, "bem_debug_i8_gemm_pair: K must be a multiple of 32 in [32, 512]");
  BEM_REQ(N >= 32 && N <= 128 && N % 32 == 0, "bem_debug_i8_gemm_pair: N must be a multiple of 32 in [32, 128]");
  DeviceGuard dg(device);
  DBuf<int8_t> dA, dB;
  DBuf<int32_t> dD;
  BEM_CK(dA.alloc((size_t)256 * K)); BEM_CK(dB.alloc((size_t)N * K)); BEM_CK(dD.alloc((size_t)256 * N));
  BEM_CK(cudaMemcpy(dA.p, A, (size_t)256 * K, cudaMemcpyHostToDevice));
  BEM_CK(cudaMemcpy(dB.p, B, (size_t)N * K, cudaMemcpyHostToDevice));
  const size_t smem = (size_t)(N / 2) * K;
  BEM_CK(cudaFuncSetAttribute(i8_pair_test_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  i8_pair_test_kernel<<<2, 128, smem>>>(dA.p, dB.p, dD.p, K, N);
  BEM_CK(cudaGetLastError());
  BEM_CK(cudaDeviceSynchronize());
  BEM_CK(cudaMemcpy(D, dD.p, sizeof(int32_t) * 256 * N, cudaMemcpyDeviceToHost));
  return BEM_OK;
}
