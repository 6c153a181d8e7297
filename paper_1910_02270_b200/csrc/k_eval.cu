// Candidate evaluation and the tournament decision on the device
// (surrogate/train_ops.hpp:191-205; tournament/ltfb.hpp:82-88, 135-147;
// train/trainer.hpp:106-127).
//
// Both candidates of a round (local and incoming generator) share the frozen
// decoder and the trainer's tournament slice, so one pass over the slice's y
// serves both: per tile, y and the decoder's wide weights are loaded once and
// each candidate's prediction is compared against them.
//
//   k_eval_small     fwd -> latent -> inv (inverse-MAE row sums) and
//                    dec head -> h, per candidate and row slice
//   k_eval_wide      forward-MAE partials per CTA and candidate
//   k_eval_finalize  fixed-order double reductions, combined metric,
//                    incoming_wins, and (decide mode) adoption: copy the
//                    incoming fwd/inv blobs and zero their Adam moments,
//                    keeping t (trainer.hpp:117-127)
#include <algorithm>
#include <cstdlib>

#include "kernels.hpp"
#include "small_mlp.cuh"

namespace ltfb_dev {

constexpr int kEvalRows = 8;

__global__ void __launch_bounds__(128) k_eval_small(EvalArgs a) {
  __shared__ float bufA[kEvalRows * kMaxSmallWidth];
  __shared__ float bufB[kEvalRows * kMaxSmallWidth];
  __shared__ float lat[kEvalRows * kMaxSmallWidth];
  const ModelArgs& m = a.m;
  const int c = blockIdx.y;
  const int r0 = blockIdx.x * kEvalRows;
  const int nr = min(kEvalRows, a.rows - r0);
  if (nr <= 0) return;
  const BlockSync sync{};
  float* pp[kMaxLayers];
  for (int l = 0; l < kMaxLayers; ++l) pp[l] = (l & 1) ? bufB : bufA;
  // latent = fwd(x)
  mlp_forward(m.fwd, a.cf[c], a.x + (long long)r0 * m.in, m.in, nr, (float* const*)nullptr, pp, sync);
  const float* latent = pp[m.fwd.L - 1];
  for (int i = threadIdx.x; i < nr * m.lat; i += blockDim.x) lat[i] = latent[i];
  sync();
  // recovered = inv(latent); per-row sum of |recovered - x| in double
  mlp_forward(m.inv, a.ci[c], lat, m.lat, nr, (float* const*)nullptr, pp, sync);
  const float* recov = pp[m.inv.L - 1];
  for (int r = threadIdx.x; r < nr; r += blockDim.x) {
    double acc = 0.0;
    const float* xr = a.x + (long long)(r0 + r) * m.in;
    for (int k = 0; k < m.in; ++k) acc += fabs((double)recov[r * m.in + k] - (double)xr[k]);
    a.inv_row[(long long)c * a.rows + r0 + r] = acc;
  }
  sync();
  // h = dec head(latent)
  float* hdst = a.h + ((long long)c * a.rows + r0) * m.D;
  if (m.dec_head.L > 0) {
    mlp_forward(m.dec_head, a.dec, lat, m.lat, nr, (float* const*)nullptr, pp, sync);
    const float* hh = pp[m.dec_head.L - 1];
    for (int i = threadIdx.x; i < nr * m.D; i += blockDim.x) hdst[i] = hh[i];
  } else {
    for (int i = threadIdx.x; i < nr * m.D; i += blockDim.x) hdst[i] = lat[i];
  }
}

// k_eval_small for C5-size slices: 64 rows per CTA (8 warps x 8 rows, each
// warp keeps its rows through every layer: no block barrier between layers),
// the three small nets' parameters staged into shared memory once per CTA,
// lanes = output neurons, each lane 8 k-ordered fmaf chains (one per row) fed
// by one weight load and 8 broadcast row loads (float4 over k where the
// widths allow) -- the 8-row CTAs above re-read the weights through L1 for
// every FMA (0.57 ms for a 225 k-row slice). Same outputs bit for bit: every
// output is the same k-ordered fmaf chain + bias + activation
// (nn/mlp.hpp:201-217), every inverse row sum the same k-ordered double sum.
constexpr int kER2 = 64;

__device__ __forceinline__ void warp_layer(const float* W, const float* b, int in, int out, int kind, float slope,
                                           const float* x, int ldx, float* dst, int ldd) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = lane; j < out; j += 32) {
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
    const float* xr = x + warp * ldx;
    if (((in | ldx) & 3) == 0) {
      for (int k = 0; k < in; k += 4) {
        const float w0 = W[k * out + j], w1 = W[(k + 1) * out + j], w2 = W[(k + 2) * out + j],
                    w3 = W[(k + 3) * out + j];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 xv = *reinterpret_cast<const float4*>(xr + 8 * i * ldx + k);
          acc[i] = fmaf(xv.x, w0, acc[i]);
          acc[i] = fmaf(xv.y, w1, acc[i]);
          acc[i] = fmaf(xv.z, w2, acc[i]);
          acc[i] = fmaf(xv.w, w3, acc[i]);
        }
      }
    } else {
      for (int k = 0; k < in; ++k) {
        const float wv = W[k * out + j];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fmaf(xr[8 * i * ldx + k], wv, acc[i]);
      }
    }
    const float bj = b[j];
#pragma unroll
    for (int i = 0; i < 8; ++i) dst[(warp + 8 * i) * ldd + j] = act_apply(kind, slope, acc[i] + bj);
  }
  __syncwarp();
}

/// Layers of n for the warp's 8 rows; the last layer writes `last` (ld ldl).
__device__ __forceinline__ void warp_mlp(const NetDesc& n, const float* w, const float* x, int ldx, float* bufA,
                                         float* bufB, int ldbuf, float* last, int ldl) {
  const float* cur = x;
  int ldc = ldx;
  for (int l = 0; l < n.L; ++l) {
    const bool top = l + 1 == n.L;
    float* dst = top ? last : ((l & 1) ? bufB : bufA);
    const int ldd = top ? ldl : ldbuf;
    warp_layer(w + (n.off_w[l] - n.base), w + (n.off_b[l] - n.base), n.w[l], n.w[l + 1], n.act[l], n.slope[l],
               cur, ldc, dst, ldd);
    cur = dst;
    ldc = ldd;
  }
}

__global__ void __launch_bounds__(256) k_eval_small_wide(EvalArgs a, int ldbuf) {
  extern __shared__ float4 sm4[];
  float* sm = reinterpret_cast<float*>(sm4);
  const ModelArgs& m = a.m;
  const int c = blockIdx.y;
  const int r0 = blockIdx.x * kER2;
  const int nr = min(kER2, a.rows - r0);
  if (nr <= 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const NetDesc& F = m.fwd;
  const NetDesc& I = m.inv;
  const NetDesc& H = m.dec_head;
  const int ldl = (m.lat + 3) & ~3, ldx = (m.in + 3) & ~3, ldo = (ldbuf + 3) & ~3;
  float* wf = sm;
  float* wi = wf + ((F.count + 3) & ~3);
  float* wh = wi + ((I.count + 3) & ~3);
  float* bufA = wh + (H.L > 0 ? ((H.count + 3) & ~3) : 0);
  float* bufB = bufA + kER2 * ldo;
  float* lat = bufB + kER2 * ldo;
  float* xs = lat + kER2 * ldl;
  float* rec = xs + kER2 * ldx;  // the inverse output [64 x in] (ld ldx)
  // every load of a chunk in flight before the stores (one L2 round trip per chunk)
  auto stage = [&](float* dst, const float* src, int n) {
    constexpr int kU = 8;
    for (int bb = 0; bb < n; bb += kU * (int)blockDim.x) {
      float v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = bb + u * (int)blockDim.x + (int)threadIdx.x;
        v[u] = i < n ? __ldg(src + i) : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = bb + u * (int)blockDim.x + (int)threadIdx.x;
        if (i < n) dst[i] = v[u];
      }
    }
  };
  stage(wf, a.cf[c] + F.base, (int)F.count);
  stage(wi, a.ci[c] + I.base, (int)I.count);
  if (H.L > 0) stage(wh, a.dec + H.base, (int)H.count);
  for (int i = threadIdx.x; i < kER2 * m.in; i += blockDim.x) {  // x rows (zero past the slice)
    const int r = i / m.in, k = i - r * m.in;
    xs[r * ldx + k] = r < nr ? __ldg(a.x + (long long)(r0 + r) * m.in + k) : 0.0f;
  }
  __syncthreads();
  // latent = fwd(x), recovered = inv(latent), h = dec head(latent): warp-local rows
  warp_mlp(F, wf, xs, ldx, bufA, bufB, ldo, lat, ldl);
  warp_mlp(I, wi, lat, ldl, bufA, bufB, ldo, rec, ldx);
  if (lane < 8) {  // per-row sum of |recovered - x| in double, k order
    const int r = warp + 8 * lane;
    if (r < nr) {
      double acc = 0.0;
      for (int k = 0; k < m.in; ++k) acc += fabs((double)rec[r * ldx + k] - (double)xs[r * ldx + k]);
      a.inv_row[(long long)c * a.rows + r0 + r] = acc;
    }
  }
  float* hdst = a.h + ((long long)c * a.rows + r0) * m.D;
  const float* hh = lat;
  int ldh = ldl;
  if (H.L > 0) {
    float* hb = ((H.L - 1) & 1) ? bufB : bufA;  // the buffer the layer rule gives the top layer (never its input)
    warp_mlp(H, wh, lat, ldl, bufA, bufB, ldo, hb, ldo);
    hh = hb;
    ldh = ldo;
  }
  for (int i = 0; i < 8; ++i) {
    const int r = warp + 8 * i;
    if (r < nr)
      for (int j = lane; j < m.D; j += 32) hdst[(long long)r * m.D + j] = hh[r * ldh + j];
  }
}

// Forward-MAE partials, register-tiled: a CTA owns column tiles of 64
// decoder outputs (Wd tile + bias loaded once) and sweeps every 64-row block
// of the slice for both candidates; each thread computes a 4 x 4 block of
// predictions (k-ordered fmaf chains over D) from float4 shared-memory
// loads (h stored k-major, Wd row-major) and accumulates |o - y| in double.
constexpr int kEvT = 64;  // rows / columns per tile
__global__ void __launch_bounds__(256) k_eval_wide(EvalArgs a) {
  extern __shared__ float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  __shared__ double red[256];
  const ModelArgs& m = a.m;
  const int D = m.D, out = m.out, op = m.out_pad;
  float* wd = sm;                // [D][64]      Wd[:, c0 .. c0 + 64)
  float* hT = wd + D * kEvT;     // [D][64]      h of 64 rows, k-major
  float* yt = hT + D * kEvT;     // [64][64 + 4] y block
  float* bd = yt + kEvT * (kEvT + 4);
  const float* Wd = a.dec + m.dec_wide_w;
  const float* Bd = a.dec + m.dec_wide_b;
  const int ncol = (out + kEvT - 1) / kEvT;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;  // 16 x 16 threads, 4 x 4 outputs each
  double acc_c[2] = {0.0, 0.0};
  for (int t = blockIdx.x; t < ncol; t += gridDim.x) {
    const int c0 = t * kEvT;
    __syncthreads();
    for (int i = tid; i < D * kEvT; i += 256) {
      const int j = i >> 6, c = i & 63;
      wd[i] = c0 + c < out ? Wd[(long long)j * out + c0 + c] : 0.0f;
    }
    if (tid < kEvT) bd[tid] = c0 + tid < out ? Bd[c0 + tid] : 0.0f;
    for (int rb = 0; rb < a.rows; rb += kEvT) {
      const int nr = min(kEvT, a.rows - rb);
      __syncthreads();
      for (int i = tid; i < kEvT * kEvT; i += 256) {
        const int r = i >> 6, c = i & 63;
        yt[r * (kEvT + 4) + c] = (r < nr && c0 + c < out) ? a.y[(long long)(rb + r) * op + c0 + c] : 0.0f;
      }
      for (int cand = 0; cand < a.nc; ++cand) {
        __syncthreads();
        for (int i = tid; i < kEvT * D; i += 256) {
          const int r = i / D, k = i - r * D;
          hT[k * kEvT + r] = r < nr ? a.h[((long long)cand * a.rows + rb + r) * D + k] : 0.0f;
        }
        __syncthreads();
        float o[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) o[i][j] = 0.0f;
#pragma unroll 4
        for (int k = 0; k < D; ++k) {
          const float4 hv = *reinterpret_cast<const float4*>(hT + k * kEvT + 4 * ty);
          const float4 wv = *reinterpret_cast<const float4*>(wd + k * kEvT + 4 * tx);
          const float hr[4] = {hv.x, hv.y, hv.z, hv.w}, wc[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) o[i][j] = fmaf(hr[i], wc[j], o[i][j]);
        }
        double sacc = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = 4 * ty + i;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int c = 4 * tx + j;
            if (r < nr && c0 + c < out) {
              const float pred = o[i][j] + bd[c];  // mlp.hpp:209-213
              sacc += fabs((double)pred - (double)yt[r * (kEvT + 4) + c]);
            }
          }
        }
        acc_c[cand] += sacc;
      }
    }
  }
  for (int cand = 0; cand < a.nc; ++cand) {
    const double tot = block_sum_det(acc_c[cand], red);
    if (tid == 0) a.part[(long long)blockIdx.x * a.nc + cand] = tot;
  }
}

__global__ void __launch_bounds__(256) k_eval_finalize(EvalArgs a) {
  __shared__ int s_adopt;
  __shared__ double red[256];
  const ModelArgs& m = a.m;
  double fsum[2] = {0, 0}, isum[2] = {0, 0};
  for (int c = 0; c < a.nc; ++c) {  // fixed-order strided sums + tree: deterministic
    double f = 0.0, inv = 0.0;
    for (int s = threadIdx.x; s < a.S; s += blockDim.x) f += a.part[(long long)s * a.nc + c];
    // the same strided order, 16 loads in flight per thread (a C5-size slice
    // has ~900 rows per thread: one dependent L2 round trip each was 0.4 ms)
    const double* ir = a.inv_row + (long long)c * a.rows;
    constexpr int kU = 16;
    int r = threadIdx.x;
    for (; r + (kU - 1) * (int)blockDim.x < a.rows; r += kU * (int)blockDim.x) {
      double v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = __ldcg(ir + r + u * (int)blockDim.x);
#pragma unroll
      for (int u = 0; u < kU; ++u) inv += v[u];
    }
    for (; r < a.rows; r += blockDim.x) inv += ir[r];
    fsum[c] = block_sum_det(f, red);
    isum[c] = block_sum_det(inv, red);
  }
  if (threadIdx.x == 0) {
    double comb[2] = {0, 0};
    for (int c = 0; c < a.nc; ++c) {
      const double f = fsum[c] / ((double)a.rows * (double)m.out);
      const double inv = isum[c] / ((double)a.rows * (double)m.in);
      comb[c] = a.w_f * f + a.w_i * inv;
      a.out[c * 3 + 0] = f;
      a.out[c * 3 + 1] = inv;
      a.out[c * 3 + 2] = comb[c];
    }
    int adopt = 0;
    if (a.decide && a.nc == 2) {
      // tournament/ltfb.hpp:82-88
      const bool inc_ok = isfinite(comb[1]), loc_ok = isfinite(comb[0]);
      adopt = !inc_ok ? 0 : (!loc_ok ? 1 : (comb[1] < comb[0] ? 1 : 0));
    }
    s_adopt = adopt;
    if (a.ctr) a.ctr->last_adopt = adopt;
  }
  __syncthreads();
  if (!s_adopt) return;
  for (long long i = threadIdx.x; i < a.n_fwd; i += blockDim.x) {
    a.dst_fwd[i] = a.cf[1][i];
    a.m_fwd[i] = 0.0f;
    a.v_fwd[i] = 0.0f;
  }
  for (long long i = threadIdx.x; i < a.n_inv; i += blockDim.x) {
    a.dst_inv[i] = a.ci[1][i];
    a.m_inv[i] = 0.0f;
    a.v_inv[i] = 0.0f;
  }
}

}  // namespace ltfb_dev

namespace ltfb_dev {

std::size_t eval_wide_smem(const ModelArgs& m) {
  return sizeof(float) * (std::size_t)(2 * m.D * kEvT + kEvT * (kEvT + 4) + kEvT);
}

void launch_eval(const EvalArgs& a, cudaStream_t s, const EvalTcHost* tc, bool precise) {
  static PerDevice attr;
  attr.once([] { cudaFuncSetAttribute(k_eval_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); });
  const ModelArgs& m = a.m;
  const int ldbuf = std::max({m.fwd.max_w(), m.inv.max_w(), m.dec_head.L > 0 ? m.dec_head.max_w() : 0, m.lat, m.in});
  auto up4 = [](long long v) { return (v + 3) & ~3LL; };
  const std::size_t sm2 = sizeof(float) * (std::size_t)(up4(m.fwd.count) + up4(m.inv.count) +
                                                        (m.dec_head.L > 0 ? up4(m.dec_head.count) : 0) +
                                                        2 * kER2 * up4(ldbuf) + kER2 * up4(m.lat) +
                                                        2 * kER2 * up4(m.in));
  if (a.rows >= 64 * kER2 && sm2 <= 200 * 1024 && !std::getenv("LTFB_EVAL_SMALL8")) {  // large slices (C5)
    static PerDevice attr;
    attr.once([] { cudaFuncSetAttribute(k_eval_small_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); });
    k_eval_small_wide<<<dim3((a.rows + kER2 - 1) / kER2, a.nc), 256, sm2, s>>>(a, ldbuf);
  } else {
    k_eval_small<<<dim3((a.rows + kEvalRows - 1) / kEvalRows, a.nc), 128, 0, s>>>(a);
  }
  if (tc)
    launch_eval_tc(a, *tc, precise, s);
  else
    k_eval_wide<<<a.S, 256, eval_wide_smem(a.m), s>>>(a);
  k_eval_finalize<<<1, 256, 0, s>>>(a);
}

}  // namespace ltfb_dev
