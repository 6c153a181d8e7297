// Microbenchmark (dev tool, not product): warm cost of the post kernel's
// warp-local layer routine, transpose and weight-gradient phase, one CTA.
#include "../../paper_1910_02270_b200/csrc/k_post_tpl.cu"
#include <cstdio>

namespace ltfb_dev { namespace ps {
__global__ void k_bench(int reps, long long* out) {
  __shared__ NetS n;
  float* s = S();
  for (int i = threadIdx.x; i < 40000; i += blockDim.x) s[i] = 0.001f * (i % 97);
  if (threadIdx.x == 0) {
    n.L = 1; n.count = 32 * 32 + 32; n.w[0] = 32; n.w[1] = 32; n.act[0] = kLeaky; n.slope[0] = 0.2f;
    n.blob = 0; n.woff[0] = 0; n.boff[0] = 1024; n.T[0] = 2000; n.z[0] = 4000; n.a[0] = 5000; n.dz[0] = 6000;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) { wfwd(8000, n, 0, 2, n.a[0]); __syncthreads(); }
  long long t1 = clock64();
  for (int r = 0; r < reps; ++r) { wgin(n.dz[0], n, 0, 2, 9000, -1, -1, false); __syncthreads(); }
  long long t2 = clock64();
  for (int r = 0; r < reps; ++r) { transpose_net(n); __syncthreads(); }
  long long t3 = clock64();
  for (int r = 0; r < reps; ++r) { pg_net(n, 8000, 16, 10000); __syncthreads(); }
  long long t4 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / reps; out[1] = (t2 - t1) / reps; out[2] = (t3 - t2) / reps; out[3] = (t4 - t3) / reps; }
}
}}

int main() {
  long long* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(ltfb_dev::ps::k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 180000);
  for (int it = 0; it < 3; ++it) {
    ltfb_dev::ps::k_bench<<<1, 256, 180000>>>(50, d);
    long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("wfwd 2 rows 32x32: %lld  wgin: %lld  transpose 32x32: %lld  pg 16 rows 33x32: %lld  (%s)\n", h[0], h[1], h[2], h[3], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
