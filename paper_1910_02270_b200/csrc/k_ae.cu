// Autoencoder pre-training step on the device (surrogate/train_ops.hpp:52-81,
// driven by tournament/runner.hpp:249-279): loss = MAE(dec(enc(y)), y), the
// gradients of every enc / dec parameter, then Adam(enc) and Adam(dec).
//
// Unlike the surrogate step, the AE step needs the weight gradients of the two
// wide layers, so it is three passes over the batch's y rows (gathered from
// the AE source slab through the batch index, never copied):
//
//   K1 enc   Pz[s] = y[:, cols_s] We0[cols_s, :]          split-K partials
//   K2       z0 = sum_s Pz[s] + b0, a0 = act(z0)          fixed split order
//   K3       enc tail, dec head forward (one CTA, block-cooperative)
//   K4 dec   per column tile: o = h Wd + bd, d = o - y, |d| (f64),
//            G = float(1/n) sign(d)          (loss.hpp:24-41)
//            dWd[:, tile] = h^T G, dbd = colsum G  (complete per tile: K = rows)
//            Pg[s] += G Wd[:, tile]^T       split-K partials of dL/dh
//   K5       gh = sum_s Pg[s]; dec head / enc tail backward; gz0 = ga0 act'(z0);
//            db0 = colsum gz0; loss = sum_s |d|_s / n
//   K6 enc   dWe0[tile, :] = y[:, tile]^T gz0  (complete per tile)
//   K7       Adam over the enc blob, then the dec blob (adam.hpp:87-122),
//            in double with explicit round-to-nearest operations.
//
// Every sum has a fixed order (no float atomics); non-finite gradients raise
// per-network flags (integer atomics) that the host turns into the
// reference's NumericError semantics (enc applied before dec is checked).
// The column passes are SIMT fp32 (the AE runs once, before the experiment);
// they are HBM-bound at ~3x the surrogate step's bytes.
#include <cmath>

#include "kernels.hpp"
#include "small_mlp.cuh"

namespace ltfb_dev {
namespace ae {

constexpr int kT = 256;   // threads of the column passes
constexpr int kTN = 32;   // columns per tile
constexpr int kMaxRows = 128;
constexpr int kMaxW = 64;  // E1, D

__device__ __forceinline__ float* smem() {
  extern __shared__ float4 smem4[];
  return reinterpret_cast<float*>(smem4);
}

/// y[r][c0 .. c0 + 32) of the batch into yt [rows x 32] (zero past out).
__device__ __forceinline__ void load_y_tile(const AeArgs& a, float* yt, int c0) {
  const int n = a.n, out = a.m.out;
  for (int i = threadIdx.x; i < n * kTN; i += kT) {
    const int r = i >> 5, c = i & 31;
    yt[i] = c0 + c < out ? a.ysrc[(long long)a.idx[r] * a.m.out_pad + c0 + c] : 0.0f;
  }
}

// K1: split-K partials of y We0. Register tiles: thread (ty, tx) owns rows
// 4 ty .. 4 ty + 3 and features 8 tx .. 8 tx + 7 (32 accumulators); per
// column c one float4 of y^T and two float4 of We feed 32 FMAs (k order =
// column order, as the reference's matmul).
__global__ void __launch_bounds__(kT) k_ae_enc(const __grid_constant__ AeArgs a) {
  float* sm = smem();
  float* yT = sm;                   // [32 cols x 128 rows]
  float* we = yT + kTN * kMaxRows;  // [32 cols x 64]
  const int n = a.n, E1 = a.m.E1, out = a.m.out;
  const float* We = a.enc + a.m.enc_wide_w;
  const int ty = threadIdx.x >> 3, tx = threadIdx.x & 7;  // rows 4 ty.., features 8 tx..
  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
  const int ntiles = (out + kTN - 1) / kTN;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int c0 = t * kTN;
    __syncthreads();
    for (int i = threadIdx.x; i < kMaxRows * kTN; i += kT) {
      const int r = i >> 5, c = i & 31;
      yT[c * kMaxRows + r] =
          (r < n && c0 + c < out) ? a.ysrc[(long long)a.idx[r] * a.m.out_pad + c0 + c] : 0.0f;
    }
    for (int i = threadIdx.x; i < kTN * kMaxW; i += kT) {
      const int c = i >> 6, e = i & 63;
      we[i] = (c0 + c < out && e < E1) ? We[(long long)(c0 + c) * E1 + e] : 0.0f;
    }
    __syncthreads();
#pragma unroll 4
    for (int c = 0; c < kTN; ++c) {
      const float4 y4 = *reinterpret_cast<const float4*>(yT + c * kMaxRows + 4 * ty);
      const float4 w0 = *reinterpret_cast<const float4*>(we + c * kMaxW + 8 * tx);
      const float4 w1 = *reinterpret_cast<const float4*>(we + c * kMaxW + 8 * tx + 4);
      const float yv[4] = {y4.x, y4.y, y4.z, y4.w};
      const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(yv[i], wv[j], acc[i][j]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = 4 * ty + i;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = 8 * tx + j;
      if (e < E1) a.Pz[((long long)blockIdx.x * n + r) * E1 + e] = acc[i][j];
    }
  }
}

// K2: z0 = sum_s Pz[s] + b0, a0 = act(z0); grid n, block E1
__global__ void k_ae_zreduce(const __grid_constant__ AeArgs a) {
  const int r = blockIdx.x, e = threadIdx.x, E1 = a.m.E1, n = a.n;
  float acc = 0.0f;
  for (int s = 0; s < a.S; ++s) acc += a.Pz[((long long)s * n + r) * E1 + e];
  const float z = acc + a.enc[a.m.enc_wide_b + e];
  a.z0[r * E1 + e] = z;
  a.a0[r * E1 + e] = act_apply(a.m.enc_act0, a.m.enc_slope0, z);
}

// K3: enc tail + dec head forward over the batch (one CTA)
__global__ void __launch_bounds__(512) k_ae_small_fwd(const __grid_constant__ AeArgs a) {
  const ModelArgs& m = a.m;
  mlp_forward(m.enc_tail, a.enc, a.a0, m.E1, a.n, a.etz, a.eta, BlockSync{});
  mlp_forward(m.dec_head, a.dec, a.latent, m.lat, a.n, a.dhz, a.dha, BlockSync{});
}

// K4: dec wide layer forward, loss, dWd / dbd, split-K partials of dL/dh.
// All three products are register-tiled from float4 shared-memory operands
// (h, the Wd tile and G are kept in both orientations); every dot product
// keeps the reference's k order (q, then rows, then columns ascending).
__global__ void __launch_bounds__(kT) k_ae_dec(const __grid_constant__ AeArgs a) {
  __shared__ double red[kT];
  float* sm = smem();
  const int n = a.n, D = a.m.D, out = a.m.out;
  float* hs = sm;                          // [128 rows x 64]
  float* hT = hs + kMaxRows * kMaxW;       // [64 x 128 rows]
  float* yt = hT + kMaxW * kMaxRows;       // [128 rows x 32]
  float* wd = yt + kMaxRows * kTN;         // [64 x 32]  Wd tile
  float* wdT = wd + kMaxW * kTN;           // [32 x 64]
  float* G = wdT + kTN * kMaxW;            // [128 rows x 32]
  float* GT = G + kMaxRows * kTN;          // [32 x 128 rows]
  float* bd = GT + kTN * kMaxRows;         // [32]
  const float* Wd = a.dec + a.m.dec_wide_w;
  const float* Bd = a.dec + a.m.dec_wide_b;
  float* dWd = a.gdec + a.m.dec_wide_w;
  float* dbd = a.gdec + a.m.dec_wide_b;
  const float g1 = (float)(1.0 / ((double)n * (double)out));  // loss.hpp:37-39
  for (int i = threadIdx.x; i < kMaxRows * kMaxW; i += kT) {
    const int r = i >> 6, q = i & 63;
    const float v = (r < n && q < D) ? a.h[r * D + q] : 0.0f;
    hs[i] = v;
    hT[q * kMaxRows + r] = v;
  }
  const int ty = threadIdx.x >> 3, tx = threadIdx.x & 7;  // (1) and (3): rows 4 ty ..
  float acc[4][8];  // (3) dL/dh partial: rows 4 ty .. + 3, j = 8 tx .. + 7
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
  double mae = 0.0;
  int bad = 0;
  const int ntiles = (out + kTN - 1) / kTN;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int c0 = t * kTN;
    __syncthreads();
    load_y_tile(a, yt, c0);
    for (int i = threadIdx.x; i < kMaxW * kTN; i += kT) {
      const int jj = i >> 5, c = i & 31;
      const float w = (jj < D && c0 + c < out) ? Wd[(long long)jj * out + c0 + c] : 0.0f;
      wd[i] = w;
      wdT[c * kMaxW + jj] = w;
    }
    if (threadIdx.x < kTN) bd[threadIdx.x] = c0 + (int)threadIdx.x < out ? Bd[c0 + threadIdx.x] : 0.0f;
    __syncthreads();
    {  // (1) forward o = h Wd + b, loss, G: rows 4 ty .., columns 4 tx ..
      float o[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) o[i][j] = 0.0f;
#pragma unroll 4
      for (int q = 0; q < kMaxW; ++q) {
        if (q >= D) break;
        const float4 h4 = *reinterpret_cast<const float4*>(hT + q * kMaxRows + 4 * ty);
        const float4 w4 = *reinterpret_cast<const float4*>(wd + q * kTN + 4 * tx);
        const float hv[4] = {h4.x, h4.y, h4.z, h4.w}, wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) o[i][j] = fmaf(hv[i], wv[j], o[i][j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = 4 * ty + i;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = 4 * tx + j;
          float gv = 0.0f;
          if (r < n && c0 + c < out) {
            const float of = o[i][j] + bd[c];  // mlp.hpp:209-213
            const double d = (double)of - (double)yt[r * kTN + c];
            mae += fabs(d);
            gv = d > 0 ? g1 : (d < 0 ? -g1 : 0.0f);
          }
          G[r * kTN + c] = gv;
          GT[c * kMaxRows + r] = gv;
        }
      }
    }
    __syncthreads();
    {  // (2) dWd[:, tile] = h^T G (rows ascending): j 4 jg .., columns 2 cg ..
      const int jg = threadIdx.x >> 4, cg = threadIdx.x & 15;
      float dw[4][2] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
      float db[2] = {0.f, 0.f};
#pragma unroll 4
      for (int r = 0; r < kMaxRows; ++r) {
        if (r >= n) break;
        const float4 h4 = *reinterpret_cast<const float4*>(hs + r * kMaxW + 4 * jg);
        const float2 g2 = *reinterpret_cast<const float2*>(G + r * kTN + 2 * cg);
        const float hv[4] = {h4.x, h4.y, h4.z, h4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          dw[i][0] = fmaf(hv[i], g2.x, dw[i][0]);
          dw[i][1] = fmaf(hv[i], g2.y, dw[i][1]);
        }
        db[0] += g2.x;
        db[1] += g2.y;
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int c = 2 * cg + k;
        if (c0 + c >= out) continue;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int jj = 4 * jg + i;
          if (jj < D) {
            dWd[(long long)jj * out + c0 + c] = dw[i][k];
            bad |= !isfinite(dw[i][k]);
          }
        }
        if (jg == 0) {
          dbd[c0 + c] = db[k];
          bad |= !isfinite(db[k]);
        }
      }
    }
    // (3) dL/dh partial += G Wd^T over this tile's columns (columns ascending)
#pragma unroll 4
    for (int c = 0; c < kTN; ++c) {
      const float4 g4 = *reinterpret_cast<const float4*>(GT + c * kMaxRows + 4 * ty);
      const float4 w0 = *reinterpret_cast<const float4*>(wdT + c * kMaxW + 8 * tx);
      const float4 w1 = *reinterpret_cast<const float4*>(wdT + c * kMaxW + 8 * tx + 4);
      const float gv[4] = {g4.x, g4.y, g4.z, g4.w};
      const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(gv[i], wv[j], acc[i][j]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = 4 * ty + i;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int jj = 8 * tx + j;
      if (jj < D) a.Pg[((long long)blockIdx.x * n + r) * D + jj] = acc[i][j];
    }
  }
  const double tot = block_sum_det(mae, red);
  if (threadIdx.x == 0) a.mae_part[blockIdx.x] = tot;
  if (bad) atomicOr(&a.flags[1], 1);
}

// K5a: gh = sum_s Pg[s] (fixed split order); grid n, block D
__global__ void k_ae_ghreduce(const __grid_constant__ AeArgs a) {
  const int r = blockIdx.x, j = threadIdx.x, D = a.m.D, n = a.n;
  float acc = 0.0f;
  for (int s = 0; s < a.S; ++s) acc += a.Pg[((long long)s * n + r) * D + j];
  a.gh[r * D + j] = acc;
}

// K5: small-network backward, gz0, db0, loss (one CTA)
__global__ void __launch_bounds__(512) k_ae_small_bwd(const __grid_constant__ AeArgs a) {
  __shared__ int bad_enc, bad_dec;
  const ModelArgs& m = a.m;
  const int n = a.n, D = m.D, E1 = m.E1;
  if (threadIdx.x == 0) {
    bad_enc = 0;
    bad_dec = 0;
  }
  (void)D;
  // dec head (lat -> D): gradient of h -> dec-head params + dL/dlatent
  if (m.dec_head.L > 0)
    mlp_backward(m.dec_head, a.dec, a.latent, m.lat, n, a.dhz, a.dha, a.gh, a.gdec + m.dec_head.base, a.glat,
                 a.tA, a.tB, BlockSync{});
  // enc tail (E1 -> lat): dL/dlatent -> enc-tail params + dL/da0
  if (m.enc_tail.L > 0)
    mlp_backward(m.enc_tail, a.enc, a.a0, E1, n, a.etz, a.eta, a.glat, a.genc + m.enc_tail.base, a.ga0, a.tA,
                 a.tB, BlockSync{});
  __syncthreads();
  for (int i = threadIdx.x; i < n * E1; i += blockDim.x)
    a.gz0[i] = a.ga0[i] * act_deriv(m.enc_act0, m.enc_slope0, a.z0[i], a.a0[i]);
  __syncthreads();
  for (int e = threadIdx.x; e < E1; e += blockDim.x) {
    float s = 0.0f;
    for (int r = 0; r < n; ++r) s += a.gz0[r * E1 + e];
    a.genc[m.enc_wide_b + e] = s;
    if (!isfinite(s)) bad_enc = 1;
  }
  for (long long i = threadIdx.x; i < m.enc_tail.count; i += blockDim.x)
    if (!isfinite(a.genc[m.enc_tail.base + i])) bad_enc = 1;
  for (long long i = threadIdx.x; i < m.dec_head.count; i += blockDim.x)
    if (!isfinite(a.gdec[m.dec_head.base + i])) bad_dec = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (bad_enc) atomicOr(&a.flags[0], 1);
    if (bad_dec) atomicOr(&a.flags[1], 1);
    double t = 0.0;
    for (int s = 0; s < a.S; ++s) t += a.mae_part[s];
    a.loss[0] = t / ((double)n * (double)m.out);
  }
}

// K6: dWe0[tile, :] = y[:, tile]^T gz0 (rows ascending). Thread (cg, eg)
// owns columns 2 cg .. + 1 and features 4 eg .. + 3 of the tile.
__global__ void __launch_bounds__(kT) k_ae_encw(const __grid_constant__ AeArgs a) {
  float* sm = smem();
  const int n = a.n, E1 = a.m.E1, out = a.m.out;
  float* gz = sm;                     // [128 rows x 64]
  float* yt = gz + kMaxRows * kMaxW;  // [128 rows x 32]
  float* dWe = a.genc + a.m.enc_wide_w;
  for (int i = threadIdx.x; i < kMaxRows * kMaxW; i += kT) {
    const int r = i >> 6, e = i & 63;
    gz[i] = (r < n && e < E1) ? a.gz0[r * E1 + e] : 0.0f;
  }
  const int cg = threadIdx.x >> 4, eg = threadIdx.x & 15;
  int bad = 0;
  const int ntiles = (out + kTN - 1) / kTN;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int c0 = t * kTN;
    __syncthreads();
    load_y_tile(a, yt, c0);
    __syncthreads();
    float dw[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll 4
    for (int r = 0; r < kMaxRows; ++r) {
      if (r >= n) break;
      const float2 y2 = *reinterpret_cast<const float2*>(yt + r * kTN + 2 * cg);
      const float4 g4 = *reinterpret_cast<const float4*>(gz + r * kMaxW + 4 * eg);
      const float gv[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        dw[0][e] = fmaf(y2.x, gv[e], dw[0][e]);
        dw[1][e] = fmaf(y2.y, gv[e], dw[1][e]);
      }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int c = 2 * cg + k;
      if (c0 + c >= out) continue;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ee = 4 * eg + e;
        if (ee < E1) {
          dWe[(long long)(c0 + c) * E1 + ee] = dw[k][e];
          bad |= !isfinite(dw[k][e]);
        }
      }
    }
  }
  if (bad) atomicOr(&a.flags[0], 1);
}

// K7: nn/adam.hpp:48-61 over one blob, in double with explicit
// round-to-nearest operations (bit-identical to the reference's loop)
__global__ void __launch_bounds__(256) k_ae_adam(float* __restrict__ p, float* __restrict__ m1,
                                                 float* __restrict__ m2, const float* __restrict__ g,
                                                 long long count, double lr, double b1, double b2, double eps,
                                                 double c1, double c2) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < count;
       e += (long long)gridDim.x * blockDim.x) {
    float m = m1[e], v = m2[e];
    p[e] = adam_elem(p[e], m, v, g[e], lr, b1, b2, eps, c1, c2);
    m1[e] = m;
    m2[e] = v;
  }
}

}  // namespace ae

bool ae_supported(const ModelArgs& m, int rows) {
  return rows >= 1 && rows <= ae::kMaxRows && m.E1 <= ae::kMaxW && m.D <= ae::kMaxW;
}

void launch_ae_passes(const AeArgs& a, cudaStream_t s) {
  static PerDevice attr;
  const int sm_enc = (ae::kMaxRows * ae::kTN + ae::kTN * ae::kMaxW) * 4;
  const int sm_dec = (2 * ae::kMaxRows * ae::kMaxW + ae::kMaxRows * ae::kTN + 2 * ae::kMaxW * ae::kTN +
                      2 * ae::kMaxRows * ae::kTN + ae::kTN) *
                     4;
  const int sm_encw = (ae::kMaxRows * ae::kMaxW + ae::kMaxRows * ae::kTN) * 4;
  attr.once([&] {
    cudaFuncSetAttribute(ae::k_ae_enc, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_enc);
    cudaFuncSetAttribute(ae::k_ae_dec, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_dec);
    cudaFuncSetAttribute(ae::k_ae_encw, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_encw);
  });
  ae::k_ae_enc<<<a.S, ae::kT, sm_enc, s>>>(a);
  ae::k_ae_zreduce<<<a.n, a.m.E1, 0, s>>>(a);
  ae::k_ae_small_fwd<<<1, 512, 0, s>>>(a);
  ae::k_ae_dec<<<a.S, ae::kT, sm_dec, s>>>(a);
  ae::k_ae_ghreduce<<<a.n, a.m.D, 0, s>>>(a);
  ae::k_ae_small_bwd<<<1, 512, 0, s>>>(a);
  ae::k_ae_encw<<<a.S, ae::kT, sm_encw, s>>>(a);
}

void launch_ae_adam(float* p, float* m1, float* m2, const float* g, long long count, double lr, double b1, double b2,
                    double eps, double c1, double c2, int sms, cudaStream_t s) {
  const long long blocks = std::min<long long>((count + 255) / 256, 8LL * sms);
  ae::k_ae_adam<<<(unsigned)std::max<long long>(1, blocks), 256, 0, s>>>(p, m1, m2, g, count, lr, b1, b2, eps, c1,
                                                                          c2);
}

}  // namespace ltfb_dev
