// Microbenchmark (dev tool): issue cost and throughput of TMA tile::gather4
// for the wide pass's y tiles (128 random rows x 32 f32 columns of a 1.5 GB
// table), 148 CTAs, 11 tiles each, <= 3 tiles in flight per CTA.
//   mode 0: lane l of one warp issues rows 4l..4l+3 (the product's scheme)
//   mode 1: one thread issues all 32 gather4
//   mode 2: 4 warps, lanes 0-7 each
//   mode 3: no TMA: 4 warps of cp.async 16 B (LDGSTS) into the SW128 layout
//   mode 4: 2 warps of cp.async (64 threads, 16 ops each per tile)
//   mode 5: one 16 KB cp.async.bulk of a contiguous (pre-laid-out) tile
//   mode 6: eight 2 KB cp.async.bulk by 8 lanes
//   mode 7: two tiled TMA loads (box 32 x 64, SW128) of a [64 x C] weight matrix (16 KB)
//   mode 8: the wide pass's tile: mode-2 y gather (16 KB) + three tiled weight loads (24 KB)
//   mode 9: mode-2 y gather (16 KB) + one 24 KB cp.async.bulk of pre-laid-out weights
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
#include "../../paper_1910_02270_b200/csrc/tc_ptx.cuh"
using namespace ltfb_dev;

__global__ void k(const __grid_constant__ CUtensorMap m, const __grid_constant__ CUtensorMap mw, const int* rows,
                  long long* out, int mode, int ncols, const float* gsrc, int NS, int NT, long long nrows_tab,
                  int SB) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw + ((1024u - (tc::smem_u32(smraw) & 1023u)) & 1023u);
  __shared__ uint64_t full[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) tc::mbar_init(&full[s], mode == 3 ? 128 : (mode == 4 ? 64 : 1));
    tc::fence_barrier_init();
  }
  __syncthreads();
  long long t0 = clock64(), issue = 0;
  const int* rr = rows + (blockIdx.x % 64) * 128;
  for (int t = 0; t < NT; ++t) {
    const int s = t % NS;
    if (t >= NS) tc::mbar_wait(&full[s], ((t - NS) / NS) & 1);  // slot reuse: tile t-NS landed
    __syncthreads();
    const int c0 = ((blockIdx.x + t * 148) * 32) % ncols;
    long long i0 = clock64();
    if (mode == 0) {
      (void)SB;
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
    } else if (mode >= 7) {
      const int c0 = ((blockIdx.x + t * 148) * 32) % (ncols - 32);
      unsigned char* slot = sm + s * SB;
      if (threadIdx.x == 0) tc::mbar_expect_tx(&full[s], mode == 7 ? 16384 : 40960);
      __syncthreads();
      if (mode >= 8 && warp < 4 && lane < 8) {
        const int i = warp * 8 + lane;
        tc::tma_gather4(slot + 512 * i, &m, &full[s], c0, rr[4 * i], rr[4 * i + 1], rr[4 * i + 2], rr[4 * i + 3]);
      }
      if (threadIdx.x == 160) {
        unsigned char* w = slot + (mode == 7 ? 0 : 16384);
        if (mode == 9) {
          const long long off = ((long long)(blockIdx.x + t * 148) * 6144) % ((long long)ncols * nrows_tab - 6144);
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 24576, [%2];" ::"r"(
                           tc::smem_u32(w)), "l"(gsrc + off), "r"(tc::smem_u32(&full[s]))
                       : "memory");
        } else {
          for (int u = 0; u < (mode == 7 ? 2 : 3); ++u) tc::tma_load_2d(w + 8192 * u, &mw, &full[s], (c0 + 32 * u) % (ncols - 32), 0);
        }
      }
    } else if (mode >= 5) {
      const long long off = ((long long)(blockIdx.x + t * 148) * 4096) % ((long long)ncols * nrows_tab - 4096);
      if (mode == 5 && threadIdx.x == 0) {
        tc::mbar_expect_tx(&full[s], 16384);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];" ::"r"(
                         tc::smem_u32(sm + s * 16384)), "l"(gsrc + off), "r"(tc::smem_u32(&full[s]))
                     : "memory");
      }
      if (mode == 6 && warp == 0) {
        if (lane == 0) tc::mbar_expect_tx(&full[s], 16384);
        __syncwarp();
        if (lane < 8)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 2048, [%2];" ::"r"(
                           tc::smem_u32(sm + s * 16384 + lane * 2048)), "l"(gsrc + off + lane * 512), "r"(tc::smem_u32(&full[s]))
                       : "memory");
      }
    } else if (mode >= 3) {
      const int nt = mode == 3 ? 128 : 64;
      if ((int)threadIdx.x < nt) {
        for (int i = threadIdx.x; i < 1024; i += nt) {
          const int r = i >> 3, ch = i & 7;
          const unsigned dst = tc::smem_u32(sm + s * 16384 + r * 128 + ((ch ^ (r & 7)) << 4));
          const float* src = gsrc + (long long)rr[r] * ncols + c0 + ch * 4;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&full[s])) : "memory");
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
  for (int t = NT - NS; t < NT; ++t) tc::mbar_wait(&full[t % NS], (t / NS) & 1);
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = issue / NT; }
}

int main(int argc, char** argv) {
  const int G = argc > 2 ? atoi(argv[2]) : 148;
  const long long N = argc > 1 ? atoll(argv[1]) : 8000, C = 49168;
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
  CUtensorMap mw;
  {
    const cuuint64_t dw[2] = {(cuuint64_t)C, 64};
    const cuuint64_t sw[1] = {(cuuint64_t)C * 4};
    const cuuint32_t bw[2] = {32, 64};
    ((Fn)fp)(&mw, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dw, sw, bw, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int NT = 44;
  for (int mode = 0; mode < 10; ++mode)
    for (int NS : {2, 3, 4, 6, 8}) {
      if (mode < 2 && NS != 3) continue;
      const int SB = mode >= 8 ? 40960 : 16384;
      if (NS * SB + 1024 > 200 * 1024) continue;
      const double bytes = mode >= 8 ? 40960.0 : 16384.0;
      k<<<G, 256, NS * SB + 1024>>>(m, mw, rd, o, mode, (int)C, d, NS, NT, N, SB);
      long long h[2]; cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
      printf("mode %d NS %d: %d tiles %lld cycles (%.0f per tile, %.1f B/clk), issue %lld per tile (%s)\n", mode, NS, NT,
             h[0], h[0] / (double)NT, bytes * NT / h[0], h[1], cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
