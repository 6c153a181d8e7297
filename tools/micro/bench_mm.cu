// Microbenchmark (dev tool, not product): cycles per call of the post
// kernel's layer routine `mm` (3xTF32 mma.sync) with warm code, one CTA.
#include "../../paper_1910_02270_b200/csrc/k_post_tpl.cu"
#include <cstdio>

namespace ltfb_dev { namespace ps {
__global__ void k_bench(int reps, long long* out) {
  float* s = S();
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) s[i] = 0.001f * (i % 97);
  __syncthreads();
  MmArgs p{};
  p.M = 16; p.N = 32; p.K = 32;
  p.a = 0; p.asm_ = 32; p.ask = 1;
  p.b = 4096; p.bsk = 32; p.bsn = 1;
  p.ones = -1; p.epi = kEpiFwd; p.ldo = 32; p.out = 10000;
  p.bias = 8192; p.z = 9000; p.act = kLeaky; p.slope = 0.2f;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) { mm(p, 0); __syncthreads(); }
  long long t1 = clock64();
  // pg shape: M = 33 (ones row), N = 32, K = 32
  MmArgs q = p; q.M = 33; q.K = 32; q.asm_ = 1; q.ask = 32; q.ones = 32; q.epi = kEpiPg; q.out = 11000; q.out2 = 12500;
  long long t2 = clock64();
  for (int r = 0; r < reps; ++r) { mm(q, 0); __syncthreads(); }
  long long t3 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / reps; out[1] = (t3 - t2) / reps; }
}
}}

int main() {
  long long* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(ltfb_dev::ps::k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  for (int it = 0; it < 3; ++it) {
    ltfb_dev::ps::k_bench<<<1, 256, 100000>>>(50, d);
    long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("mm fwd 16x32x32: %lld cycles/call; mm pg 33x32x32: %lld (%s)\n", h[0], h[1], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
