// Microbenchmark (dev tool): variants of the warp-local layer forward to
// find where the cycles go. One CTA of 256 threads, data in smem.
#include <cstdio>
extern __shared__ float sm[];

template <int IN, int OUT, int NRW>
__device__ __forceinline__ void v_const(int x, int W, int b, int z) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = lane; j < OUT; j += 32) {
    float acc[NRW];
#pragma unroll
    for (int i = 0; i < NRW; ++i) acc[i] = 0.f;
#pragma unroll
    for (int k = 0; k < IN; ++k) {
      const float wv = sm[W + k * OUT + j];
#pragma unroll
      for (int i = 0; i < NRW; ++i) acc[i] = fmaf(sm[x + (warp + 8 * i) * IN + k], wv, acc[i]);
    }
#pragma unroll
    for (int i = 0; i < NRW; ++i) {
      const float v = acc[i] + sm[b + j];
      sm[z + (warp + 8 * i) * OUT + j] = v > 0.f ? v : 0.2f * v;
    }
  }
  __syncwarp();
}

template <int NRW>
__device__ __noinline__ void v_rt(int x, int W, int b, int z, int IN, int OUT) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = lane; j < OUT; j += 32) {
    float acc[NRW];
#pragma unroll
    for (int i = 0; i < NRW; ++i) acc[i] = 0.f;
#pragma unroll 8
    for (int k = 0; k < IN; ++k) {
      const float wv = sm[W + k * OUT + j];
#pragma unroll
      for (int i = 0; i < NRW; ++i) acc[i] = fmaf(sm[x + (warp + 8 * i) * IN + k], wv, acc[i]);
    }
#pragma unroll
    for (int i = 0; i < NRW; ++i) {
      const float v = acc[i] + sm[b + j];
      sm[z + (warp + 8 * i) * OUT + j] = v > 0.f ? v : 0.2f * v;
    }
  }
  __syncwarp();
}

// rows interleaved: x for row i of this warp at x + (warp*NRW + i)*IN? same as above but
// k-split into 2 independent partial chains (more ILP), summed at end (changes order: test only)
__global__ void k_bench(int reps, long long* out, int IN, int OUT) {
  for (int i = threadIdx.x; i < 40000; i += blockDim.x) sm[i] = 0.001f * (i % 97);
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) { v_const<32, 32, 2>(8000, 0, 1024, 12000); __syncthreads(); }
  long long t1 = clock64();
  for (int r = 0; r < reps; ++r) { v_rt<2>(8000, 0, 1024, 12000, IN, OUT); __syncthreads(); }
  long long t2 = clock64();
  for (int r = 0; r < reps; ++r) { __syncthreads(); }
  long long t3 = clock64();
  for (int r = 0; r < reps; ++r) { v_const<32, 32, 4>(8000, 0, 1024, 12000); __syncthreads(); }
  long long t4 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / reps; out[1] = (t2 - t1) / reps; out[2] = (t3 - t2) / reps; out[3] = (t4 - t3) / reps; }
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 180000);
  for (int it = 0; it < 3; ++it) {
    k_bench<<<1, 256, 180000>>>(50, d, 32, 32);
    long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("const 2rows: %lld  rt 2rows: %lld  sync only: %lld  const 4 rows: %lld (%s)\n", h[0], h[1], h[2], h[3], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
