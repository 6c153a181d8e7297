// Microbenchmark (dev tool, not product): latency of one 16x32x32 dense
// layer (the post kernel's typical micro-phase) under different mappings,
// warm code, one CTA of 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
extern __shared__ float4 sm4[];
#define S (reinterpret_cast<float*>(sm4))
constexpr int X = 0, W = 4096, Z = 9000, LD = 36;

__device__ __forceinline__ void v_scalar() {  // 2 outputs / thread, k-ascending chains
  for (int i = threadIdx.x; i < 512; i += 256) {
    const int r = i >> 5, j = i & 31; float acc = 0.f;
#pragma unroll 8
    for (int k = 0; k < 32; ++k) acc = fmaf(S[X + r * LD + k], S[W + k * 32 + j], acc);
    S[Z + r * LD + j] = acc;
  }
}
__device__ __forceinline__ void v_scalar2() {  // both outputs interleaved
  const int i = threadIdx.x, r0 = i >> 5, j = i & 31, r1 = r0 + 8;
  float a0 = 0.f, a1 = 0.f;
#pragma unroll 8
  for (int k = 0; k < 32; ++k) { const float w = S[W + k * 32 + j]; a0 = fmaf(S[X + r0 * LD + k], w, a0); a1 = fmaf(S[X + r1 * LD + k], w, a1); }
  S[Z + r0 * LD + j] = a0; S[Z + r1 * LD + j] = a1;
}
__device__ __forceinline__ void v_ksplit4() {  // 4 lanes per output pair, 8-long chains, shuffle reduce
  const int t = threadIdx.x, q = t & 3, o = t >> 2;  // 64 groups x 8 outputs... 256/4 = 64 groups
  // group o handles outputs (r = o>>2 .. ) : 512 outputs / 64 groups = 8 outputs per group
  float acc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u] = 0.f;
  const int r = o >> 2, j0 = (o & 3) * 8;  // 16 rows x 4 column blocks of 8
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const int k = q * 8 + kk;
    const float x = S[X + r * LD + k];
    const float4 w0 = *reinterpret_cast<const float4*>(&S[W + k * 32 + j0]);
    const float4 w1 = *reinterpret_cast<const float4*>(&S[W + k * 32 + j0 + 4]);
    acc[0] = fmaf(x, w0.x, acc[0]); acc[1] = fmaf(x, w0.y, acc[1]); acc[2] = fmaf(x, w0.z, acc[2]); acc[3] = fmaf(x, w0.w, acc[3]);
    acc[4] = fmaf(x, w1.x, acc[4]); acc[5] = fmaf(x, w1.y, acc[5]); acc[6] = fmaf(x, w1.z, acc[6]); acc[7] = fmaf(x, w1.w, acc[7]);
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) { acc[u] += __shfl_xor_sync(~0u, acc[u], 1); acc[u] += __shfl_xor_sync(~0u, acc[u], 2); }
  if (q == 0) {
#pragma unroll
    for (int u = 0; u < 8; ++u) S[Z + r * LD + j0 + u] = acc[u];
  }
}
__device__ __forceinline__ void v_rowthread() {  // 2 rows x 8 cols per thread (32 threads)... 16 rows x 4 colblocks = 64 thr x (1 row x 8 cols)
  const int t = threadIdx.x;
  if (t < 64) {
    const int r = t >> 2, j0 = (t & 3) * 8;
    float acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.f;
#pragma unroll 4
    for (int k = 0; k < 32; ++k) {
      const float x = S[X + r * LD + k];
      const float4 w0 = *reinterpret_cast<const float4*>(&S[W + k * 32 + j0]);
      const float4 w1 = *reinterpret_cast<const float4*>(&S[W + k * 32 + j0 + 4]);
      acc[0] = fmaf(x, w0.x, acc[0]); acc[1] = fmaf(x, w0.y, acc[1]); acc[2] = fmaf(x, w0.z, acc[2]); acc[3] = fmaf(x, w0.w, acc[3]);
      acc[4] = fmaf(x, w1.x, acc[4]); acc[5] = fmaf(x, w1.y, acc[5]); acc[6] = fmaf(x, w1.z, acc[6]); acc[7] = fmaf(x, w1.w, acc[7]);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) S[Z + r * LD + j0 + u] = acc[u];
  }
}

__device__ __forceinline__ void v_r4c1() {  // 4 rows x 1 col per thread, LDS.128 broadcast x (128 threads)
  const int t = threadIdx.x;
  if (t < 128) {
    const int j = t & 31, rq = t >> 5;  // rows rq*4 .. rq*4+3
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    const float* x0 = &S[X + (rq * 4 + 0) * LD];
    const float* x1 = &S[X + (rq * 4 + 1) * LD];
    const float* x2 = &S[X + (rq * 4 + 2) * LD];
    const float* x3 = &S[X + (rq * 4 + 3) * LD];
#pragma unroll 2
    for (int k = 0; k < 32; k += 4) {
      const float4 u0 = *reinterpret_cast<const float4*>(x0 + k), u1 = *reinterpret_cast<const float4*>(x1 + k);
      const float4 u2 = *reinterpret_cast<const float4*>(x2 + k), u3 = *reinterpret_cast<const float4*>(x3 + k);
      const float w0 = S[W + (k + 0) * 32 + j], w1 = S[W + (k + 1) * 32 + j], w2 = S[W + (k + 2) * 32 + j], w3 = S[W + (k + 3) * 32 + j];
      a0 = fmaf(u0.x, w0, a0); a0 = fmaf(u0.y, w1, a0); a0 = fmaf(u0.z, w2, a0); a0 = fmaf(u0.w, w3, a0);
      a1 = fmaf(u1.x, w0, a1); a1 = fmaf(u1.y, w1, a1); a1 = fmaf(u1.z, w2, a1); a1 = fmaf(u1.w, w3, a1);
      a2 = fmaf(u2.x, w0, a2); a2 = fmaf(u2.y, w1, a2); a2 = fmaf(u2.z, w2, a2); a2 = fmaf(u2.w, w3, a2);
      a3 = fmaf(u3.x, w0, a3); a3 = fmaf(u3.y, w1, a3); a3 = fmaf(u3.z, w2, a3); a3 = fmaf(u3.w, w3, a3);
    }
    S[Z + (rq * 4 + 0) * LD + j] = a0; S[Z + (rq * 4 + 1) * LD + j] = a1;
    S[Z + (rq * 4 + 2) * LD + j] = a2; S[Z + (rq * 4 + 3) * LD + j] = a3;
  }
}
__device__ __forceinline__ void v_r2c1_all() {  // 2 rows x 1 col, LDS.128 x broadcast, 256 threads
  const int t = threadIdx.x, j = t & 31, rp = t >> 5;  // rows rp, rp+8
  float a0 = 0.f, a1 = 0.f;
  const float* x0 = &S[X + rp * LD];
  const float* x1 = &S[X + (rp + 8) * LD];
#pragma unroll 2
  for (int k = 0; k < 32; k += 4) {
    const float4 u0 = *reinterpret_cast<const float4*>(x0 + k), u1 = *reinterpret_cast<const float4*>(x1 + k);
    const float w0 = S[W + (k + 0) * 32 + j], w1 = S[W + (k + 1) * 32 + j], w2 = S[W + (k + 2) * 32 + j], w3 = S[W + (k + 3) * 32 + j];
    a0 = fmaf(u0.x, w0, a0); a0 = fmaf(u0.y, w1, a0); a0 = fmaf(u0.z, w2, a0); a0 = fmaf(u0.w, w3, a0);
    a1 = fmaf(u1.x, w0, a1); a1 = fmaf(u1.y, w1, a1); a1 = fmaf(u1.z, w2, a1); a1 = fmaf(u1.w, w3, a1);
  }
  S[Z + rp * LD + j] = a0; S[Z + (rp + 8) * LD + j] = a1;
}

__device__ __forceinline__ void split_tf32(float x, unsigned& hi, unsigned& lo) {
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
  const float r = x - __uint_as_float(hi);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(r));
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
template <int SPLIT>
__device__ __forceinline__ void v_hmma() {  // 16x32 output = 4 n-tiles on warps 0-3, K=32 (4 k-steps), 3xTF32
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  if (warp < 4) {
    const int n0 = warp * 8;
    float d[4] = {0, 0, 0, 0}, e[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k0 = 0; k0 < 32; k0 += 8) {
      const float a0 = S[X + gid * LD + k0 + tig], a1 = S[X + (gid + 8) * LD + k0 + tig];
      const float a2 = S[X + gid * LD + k0 + tig + 4], a3 = S[X + (gid + 8) * LD + k0 + tig + 4];
      const float b0 = S[W + (k0 + tig) * 32 + n0 + gid], b1 = S[W + (k0 + tig + 4) * 32 + n0 + gid];
      unsigned ah[4], al[4], bh[2], bl[2];
      split_tf32(a0, ah[0], al[0]); split_tf32(a1, ah[1], al[1]); split_tf32(a2, ah[2], al[2]); split_tf32(a3, ah[3], al[3]);
      split_tf32(b0, bh[0], bl[0]); split_tf32(b1, bh[1], bl[1]);
      if (SPLIT && (k0 & 8)) { mma_tf32(e, al, bh); mma_tf32(e, ah, bl); mma_tf32(e, ah, bh); }
      else { mma_tf32(d, al, bh); mma_tf32(d, ah, bl); mma_tf32(d, ah, bh); }
    }
    const int m = gid, n = n0 + 2 * tig;
    S[Z + m * LD + n] = d[0] + e[0]; S[Z + m * LD + n + 1] = d[1] + e[1];
    S[Z + (m + 8) * LD + n] = d[2] + e[2]; S[Z + (m + 8) * LD + n + 1] = d[3] + e[3];
  }
}

__device__ __forceinline__ void tile_rr(const float* a0, const float* a1, const float* b0, const float* b1, int K,
                                        float& c00, float& c01, float& c10, float& c11) {
#pragma unroll 2
  for (int k = 0; k < K; k += 4) {
    const float4 x = *reinterpret_cast<const float4*>(a0 + k);
    const float4 y = *reinterpret_cast<const float4*>(a1 + k);
    const float4 u = *reinterpret_cast<const float4*>(b0 + k);
    const float4 v = *reinterpret_cast<const float4*>(b1 + k);
    c00 = fmaf(x.x, u.x, c00); c00 = fmaf(x.y, u.y, c00); c00 = fmaf(x.z, u.z, c00); c00 = fmaf(x.w, u.w, c00);
    c01 = fmaf(x.x, v.x, c01); c01 = fmaf(x.y, v.y, c01); c01 = fmaf(x.z, v.z, c01); c01 = fmaf(x.w, v.w, c01);
    c10 = fmaf(y.x, u.x, c10); c10 = fmaf(y.y, u.y, c10); c10 = fmaf(y.z, u.z, c10); c10 = fmaf(y.w, u.w, c10);
    c11 = fmaf(y.x, v.x, c11); c11 = fmaf(y.y, v.y, c11); c11 = fmaf(y.z, v.z, c11); c11 = fmaf(y.w, v.w, c11);
  }
}
// generic runtime-shaped 2x2 tile layer (the v3 post kernel's fwd_layer), WT layout [out][ldt]
__device__ __noinline__ void g_tile(int x, int ldx, int WT, int ldt, int IN, int OUT, int R, int z) {
  const int ncp = (OUT + 1) >> 1, tiles = ((R + 1) >> 1) * ncp;
  for (int t = threadIdx.x; t < tiles; t += 256) {
    const int rp = t / ncp, cp = t - rp * ncp;
    const int r0 = 2 * rp, r1 = min(r0 + 1, R - 1), j0 = 2 * cp, j1 = min(j0 + 1, OUT - 1);
    float c00 = 0.0f, c01 = 0.0f, c10 = 0.0f, c11 = 0.0f;
    tile_rr(&S[x + r0 * ldx], &S[x + r1 * ldx], &S[WT + j0 * ldt], &S[WT + j1 * ldt], IN, c00, c01, c10, c11);
    S[z + r0 * 36 + j0] = c00; S[z + r0 * 36 + j1] = c01; S[z + r1 * 36 + j0] = c10; S[z + r1 * 36 + j1] = c11;
  }
}
// generic runtime scalar: 2 rows per thread sharing the weight load
__device__ __noinline__ void g_scalar2(int x, int ldx, int Wb, int IN, int OUT, int R, int z) {
  const int n = ((R + 1) >> 1) * OUT;
  for (int i = threadIdx.x; i < n; i += 256) {
    const int rp = i / OUT, j = i - rp * OUT, r0 = 2 * rp, r1 = min(r0 + 1, R - 1);
    const float* x0 = &S[x + r0 * ldx]; const float* x1 = &S[x + r1 * ldx]; const float* w = &S[Wb + j];
    float a0 = 0.f, a1 = 0.f;
#pragma unroll 4
    for (int k = 0; k < IN; ++k) { const float wv = w[k * OUT]; a0 = fmaf(x0[k], wv, a0); a1 = fmaf(x1[k], wv, a1); }
    S[z + r0 * 36 + j] = a0; S[z + r1 * 36 + j] = a1;
  }
}
__device__ int g_dims[4];
__device__ __noinline__ void v_call_noinline() { v_scalar2(); }

template <int V>
__global__ void k_bench(int reps, long long* out) {
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) S[i] = 0.001f * (i % 97);
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (V == 0) v_scalar();
    if (V == 1) v_scalar2();
    if (V == 2) v_ksplit4();
    if (V == 3) v_rowthread();
    if (V == 4) v_call_noinline();
    if (V == 5) v_r4c1();
    if (V == 6) v_r2c1_all();
    if (V == 7) v_hmma<0>();
    if (V == 8) v_hmma<1>();
    if (V == 11) g_tile(X, LD, W, 36, g_dims[0], g_dims[1], g_dims[2], Z);
    if (V == 12) g_scalar2(X, LD, W, g_dims[0], g_dims[1], g_dims[2], Z);
    if (V == 10) { if (threadIdx.x < 32) S[Z + threadIdx.x] = S[X + threadIdx.x] + 1.0f; }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[V] = (t1 - t0) / reps;
}

int main() {
  long long* d; cudaMalloc(&d, 128);
  const char* names[] = {"scalar (2 outputs looped)", "scalar2 (2 outputs interleaved)", "ksplit4 + shfl", "row-thread 1x8 float4 (64 thr)", "scalar2 via noinline call", "r4c1 LDS.128 x (128 thr)", "r2c1 LDS.128 x (256 thr)", "hmma 3xtf32 4 warps", "hmma 3xtf32 2 acc chains", "sync only", "tiny store + sync", "generic 2x2 tile (v3)", "generic scalar2"};
  cudaFuncSetAttribute(k_bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k_bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k_bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k_bench<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k_bench<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k_bench<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k_bench<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k_bench<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k_bench<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k_bench<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k_bench<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k_bench<11>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k_bench<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  { int dims[4] = {32, 32, 16, 0}; cudaMemcpyToSymbol(g_dims, dims, 16); }
  for (int it = 0; it < 2; ++it) {
    k_bench<0><<<1, 256, 100000>>>(100, d); k_bench<1><<<1, 256, 100000>>>(100, d); k_bench<2><<<1, 256, 100000>>>(100, d);
    k_bench<3><<<1, 256, 100000>>>(100, d); k_bench<4><<<1, 256, 100000>>>(100, d); k_bench<5><<<1, 256, 100000>>>(100, d); k_bench<6><<<1, 256, 100000>>>(100, d); k_bench<7><<<1, 256, 100000>>>(100, d); k_bench<8><<<1, 256, 100000>>>(100, d); k_bench<9><<<1, 256, 100000>>>(100, d); k_bench<10><<<1, 256, 100000>>>(100, d); k_bench<11><<<1, 256, 100000>>>(100, d); k_bench<12><<<1, 256, 100000>>>(100, d);
    long long h[13]; cudaMemcpy(h, d, 104, cudaMemcpyDeviceToHost);
    for (int v = 0; v < 13; ++v) printf("%-34s %lld cycles/layer\n", names[v], h[v]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
