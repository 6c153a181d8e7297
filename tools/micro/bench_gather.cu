// Microbenchmark (dev tool): issue cost and throughput of TMA tile::gather4
// for the wide pass's y tiles (128 random rows x 32 f32 columns of a 1.5 GB
// table), 148 CTAs, 11 tiles each, <= 3 tiles in flight per CTA.
//   mode 0: lane l of one warp issues rows 4l..4l+3 (the product's scheme)
//   mode 1: one thread issues all 32 gather4
//   mode 2: 4 warps, lanes 0-7 each
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_1910_02270_b200/csrc/tc_ptx.cuh"
using namespace ltfb_dev;

__global__ void k(const __grid_constant__ CUtensorMap m, const int* rows, long long* out, int mode, int ncols) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw + ((1024u - (tc::smem_u32(smraw) & 1023u)) & 1023u);
  __shared__ uint64_t full[3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 3; ++s) tc::mbar_init(&full[s], 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  long long t0 = clock64(), issue = 0;
  const int* rr = rows + (blockIdx.x % 64) * 128;
  for (int t = 0; t < 11; ++t) {
    const int s = t % 3;
    if (t >= 3) tc::mbar_wait(&full[s], ((t - 3) / 3) & 1);  // slot reuse: tile t-3 landed
    __syncthreads();
    const int c0 = ((blockIdx.x + t * 148) * 32) % ncols;
    long long i0 = clock64();
    if (mode == 0) {
      if (warp == 0) {
        if (lane == 0) tc::mbar_expect_tx(&full[s], 16384);
        __syncwarp();
        tc::tma_gather4(sm + s * 16384 + 512 * lane, &m, &full[s], c0, rr[4 * lane], rr[4 * lane + 1], rr[4 * lane + 2],
                        rr[4 * lane + 3]);
      }
    } else if (mode == 1) {
      if (threadIdx.x == 0) {
        tc::mbar_expect_tx(&full[s], 16384);
        for (int i = 0; i < 32; ++i)
          tc::tma_gather4(sm + s * 16384 + 512 * i, &m, &full[s], c0, rr[4 * i], rr[4 * i + 1], rr[4 * i + 2], rr[4 * i + 3]);
      }
    } else {
      if (threadIdx.x == 0) tc::mbar_expect_tx(&full[s], 16384);
      __syncthreads();
      if (warp < 4 && lane < 8) {
        const int i = warp * 8 + lane;
        tc::tma_gather4(sm + s * 16384 + 512 * i, &m, &full[s], c0, rr[4 * i], rr[4 * i + 1], rr[4 * i + 2], rr[4 * i + 3]);
      }
    }
    __syncthreads();
    issue += clock64() - i0;
  }
  for (int t = 8; t < 11; ++t) tc::mbar_wait(&full[t % 3], (t / 3) & 1);
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = issue / 11; }
}

int main() {
  const long long N = 8000, C = 49168;
  float* d; cudaMalloc(&d, N * C * 4); cudaMemset(d, 0, N * C * 4);
  std::vector<int> rows(64 * 128); unsigned s = 1;
  for (auto& r : rows) { s = s * 1664525u + 1013904223u; r = (s >> 8) % N; }
  int* rd; cudaMalloc(&rd, rows.size() * 4); cudaMemcpy(rd, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice);
  long long* o; cudaMalloc(&o, 16);
  CUtensorMap m;
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  const cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)N};
  const cuuint64_t strides[1] = {(cuuint64_t)C * 4};
  const cuuint32_t box[2] = {32, 1}, es[2] = {1, 1};
  ((Fn)fp)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 60000);
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 3; ++mode) {
      k<<<148, 256, 60000>>>(m, rd, o, mode, (int)C);
      long long h[2]; cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
      printf("mode %d: 11 tiles %lld cycles (%.0f per tile), issue %lld cycles per tile (%s)\n", mode, h[0], h[0] / 11.0, h[1],
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
