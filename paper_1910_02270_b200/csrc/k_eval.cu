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

template <int RB, int TN>
__global__ void __launch_bounds__(256) k_eval_wide(EvalArgs a) {
  extern __shared__ float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  __shared__ double red[256];
  const ModelArgs& m = a.m;
  const int D = m.D, out = m.out, op = m.out_pad;
  float* yt = sm;              // RB x TN
  float* wd = yt + RB * TN;    // D x TN
  float* hb = wd + D * TN;     // RB x D
  float* bd = hb + RB * D;     // TN
  const float* Wd = a.dec + m.dec_wide_w;
  const float* Bd = a.dec + m.dec_wide_b;
  const int ncol = (out + TN - 1) / TN;
  const int nrb = (a.rows + RB - 1) / RB;
  const int tid = threadIdx.x, nth = blockDim.x;
  double acc_c[2] = {0.0, 0.0};
  for (int t = blockIdx.x; t < ncol * nrb; t += gridDim.x) {
    const int rb = (t / ncol) * RB, c0 = (t % ncol) * TN;
    const int nr = min(RB, a.rows - rb);
    __syncthreads();
    for (int i = tid; i < RB * TN; i += nth) {
      const int r = i / TN, c = i - r * TN;
      yt[i] = (r < nr && c0 + c < out) ? a.y[(long long)(rb + r) * op + c0 + c] : 0.0f;
    }
    for (int i = tid; i < D * TN; i += nth) {
      const int j = i / TN, c = i - j * TN;
      wd[i] = (c0 + c < out) ? Wd[(long long)j * out + c0 + c] : 0.0f;
    }
    for (int c = tid; c < TN; c += nth) bd[c] = (c0 + c < out) ? Bd[c0 + c] : 0.0f;
    for (int cand = 0; cand < a.nc; ++cand) {
      __syncthreads();
      for (int i = tid; i < RB * D; i += nth) {
        const int r = i / D;
        hb[i] = r < nr ? a.h[((long long)cand * a.rows + rb + r) * D + (i - r * D)] : 0.0f;
      }
      __syncthreads();
      double s = 0.0;
      for (int i = tid; i < RB * TN; i += nth) {
        const int r = i / TN, c = i - r * TN;
        if (r < nr && c0 + c < out) {
          float acc = 0.0f;
          for (int j = 0; j < D; ++j) acc = fmaf(hb[r * D + j], wd[j * TN + c], acc);
          const float o = acc + bd[c];
          s += fabs((double)o - (double)yt[i]);
        }
      }
      acc_c[cand] += s;
    }
  }
  for (int cand = 0; cand < a.nc; ++cand) {
    const double tot = block_sum_det(acc_c[cand], red);
    if (tid == 0) a.part[(long long)blockIdx.x * a.nc + cand] = tot;
  }
}

template __global__ void k_eval_wide<32, 32>(EvalArgs);

__global__ void __launch_bounds__(256) k_eval_finalize(EvalArgs a) {
  __shared__ int s_adopt;
  const ModelArgs& m = a.m;
  if (threadIdx.x == 0) {
    double comb[2] = {0, 0};
    for (int c = 0; c < a.nc; ++c) {
      double f = 0.0, inv = 0.0;
      for (int s = 0; s < a.S; ++s) f += a.part[(long long)s * a.nc + c];
      for (int r = 0; r < a.rows; ++r) inv += a.inv_row[(long long)c * a.rows + r];
      f /= (double)a.rows * (double)m.out;
      inv /= (double)a.rows * (double)m.in;
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
  constexpr int RB = 32, TN = 32;
  return sizeof(float) * (std::size_t)(RB * TN + m.D * TN + RB * m.D + TN);
}

void launch_eval(const EvalArgs& a, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_eval_wide<32, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  k_eval_small<<<dim3((a.rows + kEvalRows - 1) / kEvalRows, a.nc), 128, 0, s>>>(a);
  k_eval_wide<32, 32><<<a.S, 256, eval_wide_smem(a.m), s>>>(a);
  k_eval_finalize<<<1, 256, 0, s>>>(a);
}

}  // namespace ltfb_dev
