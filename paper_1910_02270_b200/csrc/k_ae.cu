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

// K1: split-K partials of y We0 (thread: e = tid % 64, rows tid / 64 + 4 i)
__global__ void __launch_bounds__(kT) k_ae_enc(const __grid_constant__ AeArgs a) {
  float* sm = smem();
  float* yt = sm;                   // [rows x 32]
  float* we = yt + kMaxRows * kTN;  // [32 x E1]
  const int n = a.n, E1 = a.m.E1, out = a.m.out;
  const float* We = a.enc + a.m.enc_wide_w;
  const int e = threadIdx.x & 63, rg = threadIdx.x >> 6;
  float acc[kMaxRows / 4];
#pragma unroll
  for (int i = 0; i < kMaxRows / 4; ++i) acc[i] = 0.0f;
  const int ntiles = (out + kTN - 1) / kTN;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int c0 = t * kTN;
    __syncthreads();
    load_y_tile(a, yt, c0);
    for (int i = threadIdx.x; i < kTN * E1; i += kT) {
      const int c = i / E1;
      we[i] = c0 + c < out ? We[(long long)(c0 + c) * E1 + (i - c * E1)] : 0.0f;
    }
    __syncthreads();
    if (e < E1)
      for (int c = 0; c < kTN; ++c) {
        const float w = we[c * E1 + e];
#pragma unroll
        for (int i = 0; i < kMaxRows / 4; ++i)
          if (rg + 4 * i < n) acc[i] = fmaf(yt[(rg + 4 * i) * kTN + c], w, acc[i]);
      }
  }
  if (e < E1)
#pragma unroll
    for (int i = 0; i < kMaxRows / 4; ++i)
      if (rg + 4 * i < n) a.Pz[((long long)blockIdx.x * n + rg + 4 * i) * E1 + e] = acc[i];
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

// K4: dec wide layer forward, loss, dWd / dbd, split-K partials of dL/dh
__global__ void __launch_bounds__(kT) k_ae_dec(const __grid_constant__ AeArgs a) {
  __shared__ double red[kT];
  float* sm = smem();
  const int n = a.n, D = a.m.D, out = a.m.out;
  float* hs = sm;                       // [rows x D]
  float* yt = hs + kMaxRows * kMaxW;    // [rows x 32]
  float* wd = yt + kMaxRows * kTN;      // [D x 32]
  float* G = wd + kMaxW * kTN;          // [rows x 33]
  float* bd = G + kMaxRows * (kTN + 1); // [32]
  const float* Wd = a.dec + a.m.dec_wide_w;
  const float* Bd = a.dec + a.m.dec_wide_b;
  float* dWd = a.gdec + a.m.dec_wide_w;
  float* dbd = a.gdec + a.m.dec_wide_b;
  const float g1 = (float)(1.0 / ((double)n * (double)out));  // loss.hpp:37-39
  for (int i = threadIdx.x; i < n * D; i += kT) hs[i] = a.h[i];
  const int j = threadIdx.x & 63, rg = threadIdx.x >> 6;  // gh partial owner
  float acc[kMaxRows / 4];
#pragma unroll
  for (int i = 0; i < kMaxRows / 4; ++i) acc[i] = 0.0f;
  double mae = 0.0;
  int bad = 0;
  const int ntiles = (out + kTN - 1) / kTN;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int c0 = t * kTN;
    __syncthreads();
    load_y_tile(a, yt, c0);
    for (int i = threadIdx.x; i < D * kTN; i += kT) {
      const int jj = i >> 5, c = i & 31;
      wd[i] = c0 + c < out ? Wd[(long long)jj * out + c0 + c] : 0.0f;
    }
    if (threadIdx.x < kTN) bd[threadIdx.x] = c0 + (int)threadIdx.x < out ? Bd[c0 + threadIdx.x] : 0.0f;
    __syncthreads();
    {  // forward + loss + G: c = tid % 32, rows tid / 32 + 8 i
      const int c = threadIdx.x & 31, rr = threadIdx.x >> 5;
      for (int r = rr; r < n; r += 8) {
        float gv = 0.0f;
        if (c0 + c < out) {
          float o = 0.0f;
          for (int q = 0; q < D; ++q) o = fmaf(hs[r * D + q], wd[q * kTN + c], o);
          o += bd[c];  // mlp.hpp:209-213
          const double d = (double)o - (double)yt[r * kTN + c];
          mae += fabs(d);
          gv = d > 0 ? g1 : (d < 0 ? -g1 : 0.0f);
        }
        G[r * (kTN + 1) + c] = gv;
      }
    }
    __syncthreads();
    {  // dWd[:, tile] = h^T G (rows ascending), dbd = colsum G
      const int c = threadIdx.x & 31, jg = threadIdx.x >> 5;
      if (c0 + c < out) {
        for (int jj = jg; jj < D; jj += 8) {
          float s = 0.0f;
          for (int r = 0; r < n; ++r) s = fmaf(hs[r * D + jj], G[r * (kTN + 1) + c], s);
          dWd[(long long)jj * out + c0 + c] = s;
          bad |= !isfinite(s);
        }
        if (jg == 0) {
          float s = 0.0f;
          for (int r = 0; r < n; ++r) s += G[r * (kTN + 1) + c];
          dbd[c0 + c] = s;
          bad |= !isfinite(s);
        }
      }
    }
    if (j < D)  // dL/dh partial: G Wd^T over this tile's columns
      for (int c = 0; c < kTN; ++c) {
        const float w = wd[j * kTN + c];
#pragma unroll
        for (int i = 0; i < kMaxRows / 4; ++i)
          if (rg + 4 * i < n) acc[i] = fmaf(G[(rg + 4 * i) * (kTN + 1) + c], w, acc[i]);
      }
  }
  if (j < D)
#pragma unroll
    for (int i = 0; i < kMaxRows / 4; ++i)
      if (rg + 4 * i < n) a.Pg[((long long)blockIdx.x * n + rg + 4 * i) * D + j] = acc[i];
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

// K6: dWe0[tile, :] = y[:, tile]^T gz0 (rows ascending)
__global__ void __launch_bounds__(kT) k_ae_encw(const __grid_constant__ AeArgs a) {
  float* sm = smem();
  const int n = a.n, E1 = a.m.E1, out = a.m.out;
  float* gz = sm;                     // [rows x E1]
  float* yt = gz + kMaxRows * kMaxW;  // [rows x 32]
  float* dWe = a.genc + a.m.enc_wide_w;
  for (int i = threadIdx.x; i < n * E1; i += kT) gz[i] = a.gz0[i];
  const int e = threadIdx.x & 63, cg = threadIdx.x >> 6;
  int bad = 0;
  const int ntiles = (out + kTN - 1) / kTN;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int c0 = t * kTN;
    __syncthreads();
    load_y_tile(a, yt, c0);
    __syncthreads();
    if (e < E1)
      for (int c = cg; c < kTN; c += 4) {
        if (c0 + c >= out) break;
        float s = 0.0f;
        for (int r = 0; r < n; ++r) s = fmaf(yt[r * kTN + c], gz[r * E1 + e], s);
        dWe[(long long)(c0 + c) * E1 + e] = s;
        bad |= !isfinite(s);
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
    const double gd = (double)g[e];
    const double mi = __dadd_rn(__dmul_rn(b1, (double)m1[e]), __dmul_rn(1.0 - b1, gd));
    const double vi = __dadd_rn(__dmul_rn(b2, (double)m2[e]), __dmul_rn(__dmul_rn(1.0 - b2, gd), gd));
    m1[e] = (float)mi;
    m2[e] = (float)vi;
    p[e] = (float)__dsub_rn((double)p[e], __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mi, c1)),
                                                     __dadd_rn(__dsqrt_rn(__ddiv_rn(vi, c2)), eps)));
  }
}

}  // namespace ae

bool ae_supported(const ModelArgs& m, int rows) {
  return rows >= 1 && rows <= ae::kMaxRows && m.E1 <= ae::kMaxW && m.D <= ae::kMaxW;
}

void launch_ae_passes(const AeArgs& a, cudaStream_t s) {
  static bool attr = false;
  const int sm_enc = (ae::kMaxRows * ae::kTN + ae::kTN * ae::kMaxW) * 4;
  const int sm_dec = (ae::kMaxRows * ae::kMaxW + ae::kMaxRows * ae::kTN + ae::kMaxW * ae::kTN +
                      ae::kMaxRows * (ae::kTN + 1) + ae::kTN) *
                     4;
  const int sm_encw = (ae::kMaxRows * ae::kMaxW + ae::kMaxRows * ae::kTN) * 4;
  if (!attr) {
    cudaFuncSetAttribute(ae::k_ae_enc, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_enc);
    cudaFuncSetAttribute(ae::k_ae_dec, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_dec);
    cudaFuncSetAttribute(ae::k_ae_encw, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_encw);
    attr = true;
  }
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
