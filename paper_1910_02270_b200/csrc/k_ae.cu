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
#include <cstdio>
#include <cstdlib>

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
  a.gh[r * D + j] = acc * a.gscale;
}

// K2 / K5a for the tcgen05 passes (E1 == D == 64): the split-K sums spread
// over n x 16 float4 outputs with 16 partial groups each (fixed group order).
template <int kMode>  // 0: z0 / a0 from Pz, 1: gh from Pg
__global__ void __launch_bounds__(256) k_ae_reduce_st(const __grid_constant__ AeArgs a) {
  __shared__ float4 part[16][16];
  const int o = threadIdx.x & 15, g = threadIdx.x >> 4;
  const int nq = a.n * 16, q = blockIdx.x * 16 + o;
  const float4* P = reinterpret_cast<const float4*>(kMode == 0 ? a.Pz : a.Pg);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (q < nq) {
    float4 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int s = g + 16 * u;
      v[u] = s < a.S ? __ldcg(P + (long long)s * nq + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      acc.x += v[u].x;
      acc.y += v[u].y;
      acc.z += v[u].z;
      acc.w += v[u].w;
    }
  }
  part[g][o] = acc;
  __syncthreads();
  if (g == 0 && q < nq) {
    float4 t = part[0][o];
    for (int k = 1; k < 16; ++k) {
      t.x += part[k][o].x;
      t.y += part[k][o].y;
      t.z += part[k][o].z;
      t.w += part[k][o].w;
    }
    const float tv[4] = {t.x, t.y, t.z, t.w};
    if (kMode == 0) {
      const float* b0 = a.enc + a.m.enc_wide_b;
      for (int c = 0; c < 4; ++c) {
        const int e = 4 * (q & 15) + c, r = q >> 4;
        const float zz = tv[c] + b0[e];
        a.z0[r * 64 + e] = zz;
        a.a0[r * 64 + e] = act_apply(a.m.enc_act0, a.m.enc_slope0, zz);
      }
    } else {
      reinterpret_cast<float4*>(a.gh)[q] =
          make_float4(tv[0] * a.gscale, tv[1] * a.gscale, tv[2] * a.gscale, tv[3] * a.gscale);
    }
  }
}

// Row-parallel small nets for the tcgen05 path (every width <= 64): four
// batch rows per 256-thread CTA, each layer's W staged in shared memory once
// per CTA. The forward and the backward's dz / dL/dinput chain are
// row-local; the parameter gradients (sums over rows) follow in
// k_ae_grads_rows. Every dot product keeps mlp_forward / mlp_backward's k
// order, so the bits equal the one-CTA kernels'.
constexpr int kRq = 4;  // rows per CTA

__global__ void __launch_bounds__(256) k_ae_fwd_rows(const __grid_constant__ AeArgs a) {
  __shared__ float W[64 * 64], Bv[64], xs[2][kRq][64];
  const int q = threadIdx.x >> 6, j = threadIdx.x & 63;
  const int r = blockIdx.x * kRq + q;
  const bool live = r < a.n;
  const ModelArgs& m = a.m;
  int cur = 0;
  xs[0][q][j] = live ? a.a0[r * 64 + j] : 0.0f;
  auto run = [&](const NetDesc& nd, const float* blob, float* const* z, float* const* act) {
    for (int l = 0; l < nd.L; ++l) {
      const int in = nd.w[l], out = nd.w[l + 1];
      __syncthreads();
      const float* Wg = blob + nd.off_w[l];
#pragma unroll 4
      for (int i = threadIdx.x; i < in * out; i += 256) W[i] = __ldg(Wg + i);
      if (threadIdx.x < out) Bv[threadIdx.x] = __ldg(blob + nd.off_b[l] + threadIdx.x);
      __syncthreads();
      if (live && j < out) {
        const float* x = xs[cur][q];
        float acc = 0.0f;
#pragma unroll 8
        for (int k = 0; k < in; ++k) acc = fmaf(x[k], W[k * out + j], acc);
        const float zz = acc + Bv[j];
        const float av = act_apply(nd.act[l], nd.slope[l], zz);
        z[l][r * out + j] = zz;
        act[l][r * out + j] = av;
        xs[cur ^ 1][q][j] = av;
      }
      cur ^= 1;
    }
  };
  run(m.enc_tail, a.enc, a.etz, a.eta);
  run(m.dec_head, a.dec, a.dhz, a.dha);
}

__global__ void __launch_bounds__(256) k_ae_bwd_rows(const __grid_constant__ AeArgs a) {
  __shared__ float Wt[64 * 64], g[2][kRq][64], dz[kRq][64];
  const int q = threadIdx.x >> 6, j = threadIdx.x & 63;
  const int r = blockIdx.x * kRq + q;
  const bool live = r < a.n;
  const ModelArgs& m = a.m;
  int cur = 0;
  g[0][q][j] = live ? a.gh[r * 64 + j] : 0.0f;
  auto run = [&](const NetDesc& nd, const float* blob, float* const* z, float* const* act, float* const* dzo) {
    for (int l = nd.L - 1; l >= 0; --l) {
      const int in = nd.w[l], out = nd.w[l + 1];
      __syncthreads();
      const float* Wg = blob + nd.off_w[l];
#pragma unroll 4
      for (int i = threadIdx.x; i < in * out; i += 256) {
        const int k = i / out, jj = i - k * out;
        Wt[jj * in + k] = __ldg(Wg + i);
      }
      if (live && j < out) {
        const float d = g[cur][q][j] * act_deriv(nd.act[l], nd.slope[l], z[l][r * out + j], act[l][r * out + j]);
        dz[q][j] = d;
        dzo[l][r * out + j] = d;
      }
      __syncthreads();
      if (live && j < in) {
        float acc = 0.0f;
#pragma unroll 8
        for (int jj = 0; jj < out; ++jj) acc = fmaf(dz[q][jj], Wt[jj * in + j], acc);
        g[cur ^ 1][q][j] = acc;
      }
      cur ^= 1;
    }
  };
  run(m.dec_head, a.dec, a.dhz, a.dha, a.dzh);  // -> dL/dlatent
  run(m.enc_tail, a.enc, a.etz, a.eta, a.dze);  // -> dL/da0
  __syncthreads();
  if (live) {
    const int i = r * 64 + j;
    a.gz0[i] = g[cur][q][j] * act_deriv(m.enc_act0, m.enc_slope0, a.z0[i], a.a0[i]);
  }
}

/// The over-rows sums of the small nets' parameter gradients, one thread
/// per gradient element (rows ascending, as mlp.hpp:268-279 / col_sums):
/// segment s covers dW (kind 0: sum_r below[r][k] dz[r][j], fmaf) or a
/// bias (kind 1: sum_r dz[r][j]); the last block also writes the loss.
struct GradSeg {
  const float* below;
  const float* dz;
  float* dst;
  int in, out, kind, net;
  int start;  // first thread of the segment
};
struct GradSegs {
  GradSeg s[4 * kMaxLayers + 1];
  int n, total;
};

__global__ void __launch_bounds__(256) k_ae_grads_rows(const __grid_constant__ AeArgs a,
                                                       const __grid_constant__ GradSegs gs) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int rows = a.n;
  if (tid < gs.total) {
    int si = 0;
    while (si + 1 < gs.n && tid >= gs.s[si + 1].start) ++si;
    const GradSeg& sg = gs.s[si];
    const int o = tid - sg.start;
    float acc = 0.0f;
    // 32 rows of operands in flight per round trip, summed in row order
    const int k = sg.kind == 0 ? o / sg.out : 0, j = sg.kind == 0 ? o - k * sg.out : o;
    for (int r0 = 0; r0 < rows; r0 += 32) {
      float bv[32], dv[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const int r = r0 + u;
        dv[u] = r < rows ? __ldcg(sg.dz + r * sg.out + j) : 0.0f;
        bv[u] = (sg.kind == 0 && r < rows) ? __ldcg(sg.below + r * sg.in + k) : 0.0f;
      }
      if (sg.kind == 0) {
#pragma unroll
        for (int u = 0; u < 32; ++u)
          if (r0 + u < rows) acc = fmaf(bv[u], dv[u], acc);
      } else {
#pragma unroll
        for (int u = 0; u < 32; ++u)
          if (r0 + u < rows) acc += dv[u];
      }
    }
    sg.dst[o] = acc;
    if (!isfinite(acc)) atomicOr(&a.flags[sg.net], 1);
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x < 32) {  // the loss: mae partials, fixed xor tree
    const int lane = threadIdx.x;
    double v = 0.0;
    for (int s = lane; s < a.S; s += 32) v += a.mae_part[s];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) a.loss[0] = v / ((double)rows * (double)a.m.out);
  }
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

// K7 with the step's outcome decided on the device (train_ops.hpp:71-81,
// adam.hpp:87-122): a non-finite loss or enc gradient applies nothing, a
// non-finite dec gradient applies enc only; t + 1's bias corrections come
// from the host-computed table (1 - std::pow(beta, t)).
/// Adam(enc) and Adam(dec) in one launch, 4 elements per thread and pass
/// (the blobs are 256-B aligned); the last block to finish commits t.
struct AdamPair {
  float* p[2];
  float* m1[2];
  float* m2[2];
  const float* g[2];
  long long count[2];
  double lr[2];
  double b1, b2, eps;
  const double* adam_c;
  Counters* ctr;
  int* flags;  // [0] enc, [1] dec non-finite, [2] blocks done
  const double* loss;
};

__global__ void __launch_bounds__(256) k_ae_adam_pair(const __grid_constant__ AdamPair a) {
  const bool skip0 = !isfinite(*a.loss) || a.flags[0], skip1 = skip0 || a.flags[1];
  const unsigned long long t0 = a.ctr->t[0] + 1, t1 = a.ctr->t[1] + 1;
  const double c[2][2] = {{a.adam_c[2 * t0], a.adam_c[2 * t0 + 1]}, {a.adam_c[2 * t1], a.adam_c[2 * t1 + 1]}};
  const long long q0 = skip0 ? 0 : a.count[0] / 4, q1 = skip1 ? 0 : a.count[1] / 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < q0 + q1; i += stride) {
    const int net = i < q0 ? 0 : 1;
    const long long j = net ? i - q0 : i;
    float4* p4 = reinterpret_cast<float4*>(a.p[net]) + j;
    float4* m4 = reinterpret_cast<float4*>(a.m1[net]) + j;
    float4* v4 = reinterpret_cast<float4*>(a.m2[net]) + j;
    const float4 g = __ldcs(reinterpret_cast<const float4*>(a.g[net]) + j);
    float4 p = *p4, m = *m4, v = *v4;
    const double lr = a.lr[net], c1 = c[net][0], c2 = c[net][1];
    p.x = adam_elem(p.x, m.x, v.x, g.x, lr, a.b1, a.b2, a.eps, c1, c2);
    p.y = adam_elem(p.y, m.y, v.y, g.y, lr, a.b1, a.b2, a.eps, c1, c2);
    p.z = adam_elem(p.z, m.z, v.z, g.z, lr, a.b1, a.b2, a.eps, c1, c2);
    p.w = adam_elem(p.w, m.w, v.w, g.w, lr, a.b1, a.b2, a.eps, c1, c2);
    *p4 = p;
    *m4 = m;
    *v4 = v;
  }
  if (blockIdx.x == 0 && threadIdx.x < 8) {  // the < 4-element tails
    const int net = threadIdx.x >> 2, k = threadIdx.x & 3;
    const long long e = (a.count[net] / 4) * 4 + k;
    if (!(net ? skip1 : skip0) && e < a.count[net]) {
      float m = a.m1[net][e], v = a.m2[net][e];
      a.p[net][e] = adam_elem(a.p[net][e], m, v, a.g[net][e], a.lr[net], a.b1, a.b2, a.eps, c[net][0], c[net][1]);
      a.m1[net][e] = m;
      a.m2[net][e] = v;
    }
  }
  // every block has read t: the last one to finish advances it
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&a.flags[2], 1) == (int)gridDim.x - 1) {
      if (!skip0) a.ctr->t[0] = t0;
      if (!skip1) a.ctr->t[1] = t1;
    }
  }
}

}  // namespace ae

// LTFB_AE_TIMING=1: CUDA events between the tcgen05 AE step's kernels, one
// stderr line per step (µs): enc, reduce z, small fwd, dec, reduce gh,
// small bwd, encw, adam enc, adam dec + t.
namespace {
struct AeTimer {
  bool on = std::getenv("LTFB_AE_TIMING") != nullptr;
  cudaEvent_t ev[12] = {};
  int k = 0;
  void mark(cudaStream_t s) {
    if (!on || k >= 12) return;
    if (!ev[k]) cudaEventCreate(&ev[k]);
    cudaEventRecord(ev[k++], s);
  }
  void report() {
    if (!on || k < 2) return;
    cudaEventSynchronize(ev[k - 1]);
    std::fprintf(stderr, "ae_timing_us");
    for (int i = 1; i < k; ++i) {
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      std::fprintf(stderr, " %.2f", ms * 1e3f);
    }
    std::fprintf(stderr, "\n");
    k = 0;
  }
};
AeTimer& ae_timer() {
  static thread_local AeTimer t;
  return t;
}
}  // namespace

void launch_ae_adam_dev(float* const* p, float* const* m1, float* const* m2, float* const* g, const long long* count,
                        const double* lr, double b1, double b2, double eps, const double* adam_c, Counters* ctr,
                        int* flags, const double* loss, int sms, cudaStream_t s) {
  ae::AdamPair a;
  for (int net = 0; net < 2; ++net) {
    a.p[net] = p[net];
    a.m1[net] = m1[net];
    a.m2[net] = m2[net];
    a.g[net] = g[net];
    a.count[net] = count[net];
    a.lr[net] = lr[net];
  }
  a.b1 = b1;
  a.b2 = b2;
  a.eps = eps;
  a.adam_c = adam_c;
  a.ctr = ctr;
  a.flags = flags;
  a.loss = loss;
  const long long q = (count[0] + count[1]) / 4;
  const long long blocks = std::min<long long>((q + 255) / 256, 8LL * sms);
  AeTimer& tm = ae_timer();
  ae::k_ae_adam_pair<<<(unsigned)std::max<long long>(1, blocks), 256, 0, s>>>(a);
  tm.mark(s);
  tm.report();
}

bool ae_supported(const ModelArgs& m, int rows) {
  return rows >= 1 && rows <= ae::kMaxRows && m.E1 <= ae::kMaxW && m.D <= ae::kMaxW;
}

void launch_ae_passes(const AeArgs& a0, const void* ymap, cudaStream_t s) {
  AeArgs a = a0;
  a.prof = std::getenv("LTFB_AE_PROF") ? 1 : 0;
  if (ymap) {
    prepare_ae_tc();
    a.gscale = (float)(1.0 / ((double)a.n * (double)a.m.out));
    const int red_blocks = (a.n * 16 + 15) / 16;
    AeTimer& tm = ae_timer();
    tm.mark(s);
    launch_ae_enc_tc(ymap, a, s);
    tm.mark(s);
    ae::k_ae_reduce_st<0><<<red_blocks, 256, 0, s>>>(a);
    tm.mark(s);
    const int row_blocks = (a.n + ae::kRq - 1) / ae::kRq;
    ae::k_ae_fwd_rows<<<row_blocks, 256, 0, s>>>(a);
    tm.mark(s);
    launch_ae_dec_tc(ymap, a, s);
    tm.mark(s);
    ae::k_ae_reduce_st<1><<<red_blocks, 256, 0, s>>>(a);
    tm.mark(s);
    ae::k_ae_bwd_rows<<<row_blocks, 256, 0, s>>>(a);
    tm.mark(s);
    {
      ae::GradSegs gs{};
      int total = 0;
      auto add = [&](const float* below, const float* dz, float* dst, int in, int out, int kind, int net) {
        ae::GradSeg& g = gs.s[gs.n++];
        g.below = below;
        g.dz = dz;
        g.dst = dst;
        g.in = in;
        g.out = out;
        g.kind = kind;
        g.net = net;
        g.start = total;
        total += kind == 0 ? in * out : out;
      };
      const ModelArgs& m = a.m;
      for (int l = 0; l < m.dec_head.L; ++l) {
        const NetDesc& nd = m.dec_head;
        add(l == 0 ? a.latent : a.dha[l - 1], a.dzh[l], a.gdec + nd.off_w[l], nd.w[l], nd.w[l + 1], 0, 1);
        add(nullptr, a.dzh[l], a.gdec + nd.off_b[l], nd.w[l], nd.w[l + 1], 1, 1);
      }
      for (int l = 0; l < m.enc_tail.L; ++l) {
        const NetDesc& nd = m.enc_tail;
        add(l == 0 ? a.a0 : a.eta[l - 1], a.dze[l], a.genc + nd.off_w[l], nd.w[l], nd.w[l + 1], 0, 0);
        add(nullptr, a.dze[l], a.genc + nd.off_b[l], nd.w[l], nd.w[l + 1], 1, 0);
      }
      add(nullptr, a.gz0, a.genc + m.enc_wide_b, m.E1, m.E1, 1, 0);  // db0 = col_sums(gz0)
      gs.total = total;
      ae::k_ae_grads_rows<<<(total + 255) / 256, 256, 0, s>>>(a, gs);
    }
    tm.mark(s);
    launch_ae_encw_tc(ymap, a, s);
    tm.mark(s);
    return;
  }
  a.gscale = 1.0f;  // the SIMT dec pass's partials carry G = (1/n) sign
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
