// Microbenchmark (dev tool): tcgen05.mma kind::tf32 throughput for the wide
// pass's small shapes (M = 128, K = 8 per instruction), A from TMEM (.ts) or
// smem (.ss), one CTA. Cycles per instruction, issue -> commit completion.
#include <cstdio>
#include "../../paper_1910_02270_b200/csrc/tc_ptx.cuh"
using namespace ltfb_dev;

__global__ void k(long long* out, int iters) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw + ((1024u - (tc::smem_u32(smraw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f * (i % 13);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&tbase);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  tc::fence_proxy_async();
  const uint32_t T = tbase;
  const uint32_t b = tc::smem_u32(sm), a = tc::smem_u32(sm + 32768);
  uint32_t phase = 0;
  if (threadIdx.x == 0) {
    const int Ns[5] = {32, 64, 128, 256, 64};
    for (int v = 0; v < 7; ++v) {
      const int N = v < 4 ? Ns[v] : 64;
      const uint32_t id = tc::idesc_tf32(128, N, 0, 0);
      const uint64_t bd = tc::sdesc_sw128(b, 16, 1024);
      const uint64_t ad = tc::sdesc_sw128(a, 16, 1024);
      long long t0 = clock64();
      for (int i = 0; i < iters; ++i) {
        if (v < 4) tc::mma_tf32_ts(T + 256, T + 0, bd, id, i > 0);             // same D, A in TMEM
        else if (v == 4) tc::mma_tf32_ts(T + 256 + 64 * (i & 1), T + 0, bd, id, i > 1);  // 2 D regions
        else if (v == 5) tc::mma_tf32_ss(T + 256, ad, bd, id, i > 0);          // A in smem
        else tc::mma_tf32_ts(T + 256 + 64 * (i & 3), T + 0, bd, id, i > 3);  // 4 D regions
      }
      tc::tc_commit(&bar);
      tc::mbar_wait(&bar, phase);
      phase ^= 1;
      long long t1 = clock64();
      out[v] = (t1 - t0);
    }
  }
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(T);
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  const char* names[7] = {"ts N=32 same D", "ts N=64 same D", "ts N=128 same D", "ts N=256 same D",
                          "ts N=64 2 D alternating", "ss N=64 same D", "ts N=64 4 D rotating"};
  for (int it = 0; it < 2; ++it) {
    k<<<1, 128, 70000>>>(d, 512);
    long long h[7]; cudaMemcpy(h, d, 56, cudaMemcpyDeviceToHost);
    for (int v = 0; v < 7; ++v) printf("%-26s %.1f cycles/instr\n", names[v], h[v] / 512.0);
    printf("(%s)\n", cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
