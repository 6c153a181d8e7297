// Microbenchmark (dev tool): cost of executing cold code on B200.
// f<ID>() are distinct noinline functions of ~N dependent-free FFMA/IADD
// instructions; calling 16 distinct ones once (cold) vs one of them 16 times.
#include <cstdio>
template <int ID>
__device__ __noinline__ float f(float x, float y) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = x + i * 0.5f + ID;
#pragma unroll
  for (int r = 0; r < 24; ++r)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], y, 0.25f * (r + ID));
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  return s;
}
template <int N>
__device__ __forceinline__ float call_all(float x, float y) {
  if constexpr (N == 0) return x;
  else return f<N>(call_all<N - 1>(x, y), y);
}
__global__ void k(long long* out, float y) {
  float x = threadIdx.x;
  long long t0 = clock64();
  x = call_all<16>(x, y);  // 16 distinct functions, first touch
  long long t1 = clock64();
  for (int i = 0; i < 16; ++i) x = f<1>(x, y);  // warm (f<1> touched above)
  long long t2 = clock64();
  x = call_all<16>(x, y);  // same 16 again (maybe warm if fits)
  long long t3 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; }
  if (x == 12345.f) out[3] = 1;
}
__global__ void k_evict(float* p) {  // a different big kernel in between (not needed: each launch new)
  p[threadIdx.x] += 1;
}
int main() {
  long long* d; cudaMalloc(&d, 64);
  for (int it = 0; it < 3; ++it) {
    k<<<1, 256>>>(d, 0.999f);
    long long h[3]; cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("16 distinct cold: %lld   same fn x16: %lld   16 distinct again: %lld  (%s)\n", h[0], h[1], h[2], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
