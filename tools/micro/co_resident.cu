// Can a second kernel (grid of G CTAs, dynamic smem SB) start while a
// persistent kernel A (16 CTAs, optional cluster size, dynamic smem SA) is
// resident?  A spins until B's CTA 0 sets a flag (or 1 s passes) and reports
// how long it waited.  nvcc -gencode arch=compute_100a,code=sm_100a -o co co_resident.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void kA(volatile int* flag, unsigned long long* waited) {
  extern __shared__ char sm[];
  if (threadIdx.x == 0) {
    sm[0] = 1;
    const unsigned long long t0 = gt();
    while (*flag == 0 && gt() - t0 < 1000000000ull) __nanosleep(100);
    if (blockIdx.x == 0) *waited = gt() - t0;
  }
  __syncthreads();
}
__global__ void kB(volatile int* flag) {
  extern __shared__ char sm[];
  if (threadIdx.x == 0) sm[0] = 1;
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) { *flag = 1; __threadfence_system(); }
}

int run(int clusterA, int SA, int G, int SB, int threadsB) {
  int* flag; unsigned long long* w;
  cudaMalloc(&flag, 4); cudaMemset(flag, 0, 4);
  cudaMalloc(&w, 8); cudaMemset(w, 0, 8);
  cudaStream_t a, b; cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  cudaFuncSetAttribute(kA, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(kA, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(kB, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaLaunchConfig_t c{}; c.gridDim = dim3(16); c.blockDim = dim3(256); c.dynamicSmemBytes = SA; c.stream = a;
  cudaLaunchAttribute at; at.id = cudaLaunchAttributeClusterDimension; at.val.clusterDim.x = clusterA; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
  c.attrs = &at; c.numAttrs = clusterA > 1 ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&c, kA, (volatile int*)flag, w);
  if (e != cudaSuccess) { printf("launch A: %s\n", cudaGetErrorString(e)); return 1; }
  // let A become resident
  cudaEvent_t ev; cudaEventCreate(&ev);
  for (volatile int i = 0; i < 2000000; ++i) {}
  kB<<<G, threadsB, SB, b>>>((volatile int*)flag);
  e = cudaGetLastError();
  if (e != cudaSuccess) { printf("launch B: %s\n", cudaGetErrorString(e)); return 1; }
  cudaDeviceSynchronize();
  unsigned long long hw; cudaMemcpy(&hw, w, 8, cudaMemcpyDeviceToHost);
  printf("A cluster %2d smemA %6d | B grid %3d smemB %6d thr %d : A waited %.1f us %s\n", clusterA, SA, G, SB, threadsB,
         hw * 1e-3, hw > 900000000ull ? "(NOT concurrent)" : "");
  cudaFree(flag); cudaFree(w);
  return 0;
}

int main() {
  int n; cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", n);
  run(16, 100 * 1024, 132, 200 * 1024, 320);
  run(16, 100 * 1024, 132, 1024, 320);
  run(16, 100 * 1024, 1, 200 * 1024, 320);
  run(8, 100 * 1024, 132, 200 * 1024, 320);
  run(1, 100 * 1024, 132, 200 * 1024, 320);
  run(16, 1024, 132, 200 * 1024, 320);
  run(16, 100 * 1024, 120, 200 * 1024, 320);
  run(16, 100 * 1024, 128, 200 * 1024, 320);
  return 0;
}
