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
