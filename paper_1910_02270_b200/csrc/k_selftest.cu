// On-device self-test of the three tcgen05 MMA shapes the wide pass uses
// (exported as ltfb_selftest_tcgen05 for tests/test_gpu_kernels.py):
//   1. SS  M128 N64 K32: A K-major SW128 [128 x 32], B K-major SW128
//      [N 64 x K 32]                               (enc layer-0 tile, W^T)
//   2. TS  M128 N32 K64: A in TMEM [128 x 64], B K-major SW128 as two
//      [N 32 x K 32] K-blocks                      (dec forward tile, W^T)
//   3. SS  M128 N64 K32: A K-major SW128 [128 x 32], B K-major SW128
//      [N 64 x K 32]                               (dec h-gradient tile, W)
// (tf32 MN-major operands need the 32B-atom swizzle, so every operand of
// the wide pass is staged K-major instead.)
#include "tc_ptx.cuh"

namespace ltfb_dev {

__global__ void __launch_bounds__(128) k_selftest_tc(const float* a1, const float* b1, const float* ah,
                                                      const float* b2, const float* a3, float* d1, float* d2,
                                                      float* d3) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u);
  unsigned char* A1 = sm;            // 16 KB
  unsigned char* B1 = sm + 16384;    // 8 KB (two 4 KB atoms)
  unsigned char* B2 = sm + 24576;    // 8 KB
  unsigned char* A3 = sm + 32768;    // 16 KB
  unsigned char* B2T = sm + 49152;   // 8 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 32; i += 128) {
    const int r = i / 32, c = i % 32;
    *reinterpret_cast<float*>(A1 + tc::sw128_off(r, c)) = a1[i];
    *reinterpret_cast<float*>(A3 + tc::sw128_off(r, c)) = a3[i];
  }
  for (int i = tid; i < 32 * 64; i += 128) {  // b1: [K=32][N=64] row-major -> K-major [64 x 32]
    const int k = i / 64, n = i % 64;
    *reinterpret_cast<float*>(B1 + tc::sw128_off(n, k)) = b1[i];
  }
  for (int i = tid; i < 64 * 32; i += 128) {  // b2: [64][32] row-major
    const int r = i / 32, c = i % 32;
    // test 3 operand: K-major [N=64 rows][K=32]
    *reinterpret_cast<float*>(B2 + tc::sw128_off(r, c)) = b2[i];
    // test 2 operand: b2 as [K=64][N=32] -> K-major [N=32][K=64] in two 32-wide K blocks
    *reinterpret_cast<float*>(B2T + (r / 32) * 4096 + tc::sw128_off(c, r % 32)) = b2[i];
  }
  if (warp == 0) tc::tmem_alloc<256>(&tbase);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t T = tbase;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  {  // A of test 2 into TMEM columns [160, 224)
    float v[32];
    for (int h = 0; h < 2; ++h) {
      for (int j = 0; j < 32; ++j) v[j] = ah[tid * 64 + h * 32 + j];
      tc::tmem_st32(T + lane_base + 160 + 32 * h, v);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (tid == 0) {
    const uint32_t i1 = tc::idesc_tf32(128, 64, 0, 0);
    const uint32_t i2 = tc::idesc_tf32(128, 32, 0, 0);
    const uint32_t i3 = tc::idesc_tf32(128, 64, 0, 0);
    for (int k = 0; k < 4; ++k) {
      const uint64_t ad = tc::sdesc_sw128(tc::smem_u32(A1) + 32 * k, 16, 1024);
      const uint64_t bd = tc::sdesc_sw128(tc::smem_u32(B1) + 32 * k, 16, 1024);
      tc::mma_tf32_ss(T + 0, ad, bd, i1, k > 0);
    }
    for (int k = 0; k < 8; ++k) {
      const uint64_t bd = tc::sdesc_sw128(tc::smem_u32(B2T) + (k / 4) * 4096 + 32 * (k % 4), 16, 1024);
      tc::mma_tf32_ts(T + 64, T + 160 + 8 * k, bd, i2, k > 0);
    }
    for (int k = 0; k < 4; ++k) {
      const uint64_t ad = tc::sdesc_sw128(tc::smem_u32(A3) + 32 * k, 16, 1024);
      const uint64_t bd = tc::sdesc_sw128(tc::smem_u32(B2) + 32 * k, 16, 1024);
      tc::mma_tf32_ss(T + 96, ad, bd, i3, k > 0);
    }
    tc::tc_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  float v[32];
  for (int h = 0; h < 2; ++h) {
    tc::tmem_ld32(T + lane_base + 32 * h, v);
    for (int j = 0; j < 32; ++j) d1[tid * 64 + 32 * h + j] = v[j];
    tc::tmem_ld32(T + lane_base + 96 + 32 * h, v);
    for (int j = 0; j < 32; ++j) d3[tid * 64 + 32 * h + j] = v[j];
  }
  tc::tmem_ld32(T + lane_base + 64, v);
  for (int j = 0; j < 32; ++j) d2[tid * 32 + j] = v[j];
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<256>(T);
}

/// Host wrapper: all pointers are device pointers.
cudaError_t selftest_tc(const float* a1, const float* b1, const float* ah, const float* b2, const float* a3,
                        float* d1, float* d2, float* d3) {
  const int smem = 57344 + 1024;
  cudaFuncSetAttribute(k_selftest_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_selftest_tc<<<1, 128, smem>>>(a1, b1, ah, b2, a3, d1, d2, d3);
  return cudaDeviceSynchronize();
}

}  // namespace ltfb_dev
