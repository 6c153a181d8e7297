// Dev check (not product): TMA tile::gather4 with SWIZZLE_128B into a
// 128-row tile, one gather4 per 4 rows at smem offset 512*i. Prints whether
// the resulting layout equals the 128-B swizzle of a full [128 x 32] box.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap m, const int* rows, float* out) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smraw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" :: "r"(b), "r"(16384));
    for (int i = 0; i < 32; ++i) {
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm + 512 * i);
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                   :: "r"(dst), "l"(&m), "r"(32), "r"(rows[4*i]), "r"(rows[4*i+1]), "r"(rows[4*i+2]), "r"(rows[4*i+3]), "r"(b) : "memory");
    }
  }
  asm volatile("{\n\t.reg .pred P;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n\t}" :: "r"(b));
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) out[i] = reinterpret_cast<float*>(sm)[i];
}

int main() {
  const int N = 1000, C = 96;
  std::vector<float> h(N * C);
  for (int r = 0; r < N; ++r) for (int c = 0; c < C; ++c) h[r * C + c] = r * 1000.0f + c;
  float *d, *o; int* rd;
  cudaMalloc(&d, h.size() * 4); cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&o, 4096 * 4);
  std::vector<int> rows(128); for (int i = 0; i < 128; ++i) rows[i] = (i * 37 + 11) % N;
  cudaMalloc(&rd, 512); cudaMemcpy(rd, rows.data(), 512, cudaMemcpyHostToDevice);
  CUtensorMap m;
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  const cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)N};
  const cuuint64_t strides[1] = {(cuuint64_t)C * 4};
  const cuuint32_t box[2] = {32, 1}, es[2] = {1, 1};
  CUresult r = ((Fn)fp)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 20480);
  k<<<1, 128, 20480>>>(m, rd, o);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> got(4096); cudaMemcpy(got.data(), o, 4096 * 4, cudaMemcpyDeviceToHost);
  int bad_sw = 0, bad_box = 0;
  for (int rr = 0; rr < 128; ++rr) for (int c = 0; c < 32; ++c) {
    const float want = rows[rr] * 1000.0f + 32 + c;
    // address-based 128B swizzle: chunk (c/4) ^ (row % 8)
    const int off_sw = rr * 32 + (((c / 4) ^ (rr % 8)) * 4) + c % 4;
    // box-relative swizzle for 4-row boxes: chunk ^ (row % 4)
    const int off_box = rr * 32 + (((c / 4) ^ (rr % 4)) * 4) + c % 4;
    if (got[off_sw] != want) ++bad_sw;
    if (got[off_box] != want) ++bad_box;
  }
  printf("mismatches: address-based swizzle %d, box-relative %d (of 4096)\n", bad_sw, bad_box);
  return 0;
}
