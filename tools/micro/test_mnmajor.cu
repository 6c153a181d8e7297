// Dev check: tcgen05.mma kind::tf32 with an MN-major B operand (SWIZZLE_128B)
// read from a TMA-style [64 K rows x 32 N] block pair. D = A B, A [128 x 64]
// from TMEM, B [64 x 64] (K = j rows, N = c). Prints the max error of a few
// (LBO, SBO) descriptor variants against the exact product (small integers).
#include <cstdio>
#include <cmath>
#include "../../paper_1910_02270_b200/csrc/tc_ptx.cuh"
using namespace ltfb_dev;

__device__ float aval(int r, int k) { return (float)(((r * 7 + k * 3) % 9) - 4); }
__device__ float bval(int k, int c) { return (float)(((k * 5 + c * 11) % 7) - 3); }

__global__ void k(float* out, int variant) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw + ((1024u - (tc::smem_u32(smraw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  // B: block kb = c / 32, element (c, j) at j * 128 + (((c % 32) / 4) ^ (j & 7)) * 16 + (c % 4) * 4
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) {
    const int j = i / 64, c = i % 64, kb = c / 32, cc = c % 32;
    float* p = reinterpret_cast<float*>(sm + kb * 8192 + j * 128 + (((cc / 4) ^ (j & 7)) * 16) + (cc % 4) * 4);
    *p = bval(j, c);
  }
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&tbase);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t T = tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, r = warp * 32 + lane;
  const uint32_t la = (uint32_t)(warp * 32) << 16;
  {
    float v[32];
    for (int h = 0; h < 2; ++h) {
      for (int e = 0; e < 32; ++e) v[e] = aval(r, 32 * h + e);
      tc::tmem_st32(T + la + 32 * h, v);
    }
  }
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t b = tc::smem_u32(sm);
    const uint32_t id = tc::idesc_tf32(128, 64, 0, 1);
    uint32_t lbo = 8192, sbo = 1024, step = 1024;
    if (variant == 1) { lbo = 1024; sbo = 8192; }
    if (variant == 2) { lbo = 8192; sbo = 128; step = 1024; }
    for (int kk = 0; kk < 8; ++kk)
      tc::mma_tf32_ts(T + 256, T + 8 * kk, tc::sdesc_sw128(b + step * kk, lbo, sbo), id, kk > 0 ? 1u : 0u);
    tc::tc_commit(&bar);
    tc::mbar_wait(&bar, 0);
  }
  __syncthreads();
  tc::tc_fence_after();
  {
    float v[32];
    for (int h = 0; h < 2; ++h) {
      tc::tmem_ld32(T + la + 256 + 32 * h, v);
      for (int e = 0; e < 32; ++e) {
        double ref = 0;
        for (int kq = 0; kq < 64; ++kq) ref += (double)aval(r, kq) * bval(kq, 32 * h + e);
        out[r * 64 + 32 * h + e] = (float)fabs(v[e] - ref);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(T);
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 64 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int v = 0; v < 3; ++v) {
    k<<<1, 128, 40000>>>(d, v);
    cudaError_t e = cudaDeviceSynchronize();
    float h[128 * 64];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    float mx = 0;
    for (float x : h) mx = fmaxf(mx, x);
    printf("variant %d: %s max abs err %g\n", v, cudaGetErrorString(e), mx);
  }
  return 0;
}
