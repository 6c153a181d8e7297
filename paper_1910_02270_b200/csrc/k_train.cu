// One LTFB training step on the GPU (train/trainer.hpp:190-290):
//
//   k_gather   data store -> minibatch (epoch_plan.hpp:106-137, store.hpp:140-181)
//   k_pre      fwd(x) with tape, dec head with tape -> h        (small nets)
//   k_wide_*   ONE pass over the y minibatch that serves both sub-steps:
//                enc layer 0 split-K partials  (D-step real latents,
//                  train_ops.hpp:160 -> mlp.hpp:228-231)
//                dec last layer + MAE + sign + h-gradient partials
//                  (G-step, train_ops.hpp:100-104 -> loss.hpp:25-41,
//                   mlp.hpp:268-279; dW/db of the frozen decoder are
//                   never formed)
//   k_post     split-K reductions, enc tail, the discriminator step
//              (BCE, backprop, finite check, Adam) and the generator step
//              (adversarial + cycle paths, fwd backprop, finite checks,
//              Adam on fwd then inv), StepRecord, skip/abort counters.
//
// The wide-pass kernels are in k_wide.cu; this file holds the generic
// (any width) variant used for non-default architectures.
#include <cfloat>

#include "kernels.hpp"
#include "scratch_layout.cuh"
#include "small_mlp.cuh"

namespace ltfb_dev {

__device__ __forceinline__ int batch_rows(const StepArgs& a) {
  const int begin = (int)a.ctr->step_in_epoch * a.B;
  const int left = a.n_part - begin;
  return left < a.B ? left : a.B;
}

// ----------------------------------------------------------------- gather --
// grid (x chunks, B rows). Each row is one contiguous HBM slab row; float4
// copies keep every warp access 512 B-contiguous.
__global__ void __launch_bounds__(256) k_gather(StepArgs a) {
  if (a.ctr->aborted) return;
  const int rows = batch_rows(a);
  const int r = blockIdx.y;
  if (r >= rows) return;
  const unsigned slot = a.perm[a.ctr->epoch & 1][(long long)a.ctr->step_in_epoch * a.B + r];
  const int n4 = a.m.out_pad >> 2;
  const float4* src = reinterpret_cast<const float4*>(a.sy + (long long)slot * a.m.out_pad);
  float4* dst = reinterpret_cast<float4*>(a.yb + (long long)r * a.m.out_pad);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x)
    dst[i] = __ldcs(src + i);
  if (blockIdx.x == 0 && (int)threadIdx.x < a.m.in)
    a.xb[r * a.m.in + threadIdx.x] = a.sx[(long long)slot * a.m.in + threadIdx.x];
}

// -------------------------------------------------------------------- pre --
// fwd forward (tape) and dec-head forward (tape) for a row slice per CTA.
__global__ void __launch_bounds__(128) k_pre(StepArgs a) {
  if (a.ctr->aborted) return;
  const int rows = batch_rows(a);
  const int per = (rows + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per;
  const int nr = min(per, rows - r0);
  if (nr <= 0) return;
  const ModelArgs& m = a.m;
  const ScratchLayout L = make_scratch_layout(m, a.B);
  float* sc = a.scratch;
  float* fz[kMaxLayers];
  float* fa[kMaxLayers];
  for (int l = 0; l < m.fwd.L; ++l) {
    fz[l] = sc + L.fz[l] + (long long)r0 * m.fwd.w[l + 1];
    fa[l] = sc + L.fa[l] + (long long)r0 * m.fwd.w[l + 1];
  }
  mlp_forward(m.fwd, a.p[kFwd], a.xb + r0 * m.in, m.in, nr, fz, fa, BlockSync{});
  if (m.dec_head.L > 0) {
    float* hz[kMaxLayers];
    float* ha[kMaxLayers];
    for (int l = 0; l < m.dec_head.L; ++l) {
      hz[l] = sc + L.hz[l] + (long long)r0 * m.dec_head.w[l + 1];
      ha[l] = sc + L.ha[l] + (long long)r0 * m.dec_head.w[l + 1];
    }
    mlp_forward(m.dec_head, a.p[kDec], fa[m.fwd.L - 1], m.lat, nr, hz, ha, BlockSync{});
  }
}

// ------------------------------------------------------ wide pass, generic --
// Any E1/D (<= 256), any batch. CTA s owns column tiles s, s+S, ... and
// writes one [rows x E1] / [rows x D] partial; K is split over CTAs and
// reduced in fixed order by k_post (deterministic, no float atomics).
template <int RB, int TN>
__global__ void __launch_bounds__(256) k_wide_generic(StepArgs a) {
  if (a.ctr->aborted) return;
  extern __shared__ float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  __shared__ double red[256];
  const ModelArgs& m = a.m;
  const int rows = batch_rows(a);
  const int E1 = m.E1, D = m.D, out = m.out, op = m.out_pad;
  float* accE = sm;                 // RB x E1
  float* accD = accE + RB * E1;     // RB x D
  float* hb = accD + RB * D;        // RB x D
  float* yt = hb + RB * D;          // RB x TN
  float* we = yt + RB * TN;         // TN x E1
  float* wd = we + TN * E1;         // D x TN
  float* st = wd + D * TN;          // RB x TN
  float* bd = st + RB * TN;         // TN
  const float* We = a.p[kEnc] + m.enc_wide_w;
  const float* Wd = a.p[kDec] + m.dec_wide_w;
  const float* Bd = a.p[kDec] + m.dec_wide_b;
  const int ntiles = (out + TN - 1) / TN;
  const int tid = threadIdx.x, nth = blockDim.x;
  double mae = 0.0;
  for (int rb = 0; rb < rows; rb += RB) {
    const int nr = min(RB, rows - rb);
    __syncthreads();
    for (int i = tid; i < RB * E1; i += nth) accE[i] = 0.0f;
    for (int i = tid; i < RB * D; i += nth) {
      accD[i] = 0.0f;
      const int r = i / D;
      hb[i] = r < nr ? a.h[(long long)(rb + r) * D + (i - r * D)] : 0.0f;
    }
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int c0 = t * TN;
      __syncthreads();
      for (int i = tid; i < RB * TN; i += nth) {
        const int r = i / TN, c = i - r * TN;
        yt[i] = (r < nr && c0 + c < out) ? a.yb[(long long)(rb + r) * op + c0 + c] : 0.0f;
      }
      for (int i = tid; i < TN * E1; i += nth) {
        const int c = i / E1;
        we[i] = (c0 + c < out) ? We[(long long)(c0 + c) * E1 + (i - c * E1)] : 0.0f;
      }
      for (int i = tid; i < D * TN; i += nth) {
        const int j = i / TN, c = i - j * TN;
        wd[i] = (c0 + c < out) ? Wd[(long long)j * out + c0 + c] : 0.0f;
      }
      for (int c = tid; c < TN; c += nth) bd[c] = (c0 + c < out) ? Bd[c0 + c] : 0.0f;
      __syncthreads();
      for (int i = tid; i < RB * E1; i += nth) {
        const int r = i / E1, j = i - r * E1;
        float acc = accE[i];
        for (int c = 0; c < TN; ++c) acc = fmaf(yt[r * TN + c], we[c * E1 + j], acc);
        accE[i] = acc;
      }
      for (int i = tid; i < RB * TN; i += nth) {
        const int r = i / TN, c = i - r * TN;
        float s = 0.0f;
        if (r < nr && c0 + c < out) {
          float acc = 0.0f;
          for (int j = 0; j < D; ++j) acc = fmaf(hb[r * D + j], wd[j * TN + c], acc);
          const float o = acc + bd[c];
          const double d = (double)o - (double)yt[i];
          mae += fabs(d);
          s = d > 0 ? 1.0f : (d < 0 ? -1.0f : 0.0f);
        }
        st[i] = s;
      }
      __syncthreads();
      for (int i = tid; i < RB * D; i += nth) {
        const int r = i / D, j = i - r * D;
        float acc = accD[i];
        for (int c = 0; c < TN; ++c) acc = fmaf(st[r * TN + c], wd[j * TN + c], acc);
        accD[i] = acc;
      }
    }
    __syncthreads();
    float* pe = a.P_enc + ((long long)blockIdx.x * a.B + rb) * E1;
    float* pd = a.P_dec + ((long long)blockIdx.x * a.B + rb) * D;
    for (int i = tid; i < nr * E1; i += nth) pe[i] = accE[i];
    for (int i = tid; i < nr * D; i += nth) pd[i] = accD[i];
  }
  const double tot = block_sum_det(mae, red);
  if (tid == 0) a.mae_part[blockIdx.x] = tot;
}

template __global__ void k_wide_generic<32, 32>(StepArgs);

// ------------------------------------------------------------------- Adam --
// nn/adam.hpp:48-61 in double with explicit round-to-nearest operations so
// nothing is contracted into an FMA: with identical inputs the update is
// bit-identical to the reference's scalar loop.
__device__ __forceinline__ void adam_elem(float& p, float g, float& m1, float& m2, double lr,
                                          double b1, double b2, double eps, double c1, double c2) {
  const double gd = (double)g;
  const double mi = __dadd_rn(__dmul_rn(b1, (double)m1), __dmul_rn(1.0 - b1, gd));
  const double vi = __dadd_rn(__dmul_rn(b2, (double)m2), __dmul_rn(__dmul_rn(1.0 - b2, gd), gd));
  m1 = (float)mi;
  m2 = (float)vi;
  const double upd = __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mi, c1)), __dadd_rn(__dsqrt_rn(__ddiv_rn(vi, c2)), eps));
  p = (float)__dsub_rn((double)p, upd);
}

template <class Sync>
__device__ void adam_net(const StepArgs& a, int net, long long n, Sync sync) {
  const unsigned long long t = a.ctr->t[net] + 1;
  const double c1 = a.adam_c[2 * t], c2 = a.adam_c[2 * t + 1];
  float* p = a.p[net];
  const float* g = a.g[net];
  float* m1 = a.mom1[net];
  float* m2 = a.mom2[net];
  for (long long i = sync.rank(); i < n; i += sync.size())
    adam_elem(p[i], g[i], m1[i], m2[i], a.lr[net], a.b1, a.b2, a.eps, c1, c2);
}

__device__ bool all_finite_blk(const float* v, long long n) {
  int ok = 1;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) ok &= isfinite(v[i]) ? 1 : 0;
  return __syncthreads_and(ok) != 0;
}

// ------------------------------------------------------------------- post --
__global__ void __launch_bounds__(512) k_post(StepArgs a) {
  __shared__ double red[512];
  Counters* ctr = a.ctr;
  if (ctr->aborted) return;
  const ModelArgs& m = a.m;
  const int rows = batch_rows(a);
  const ScratchLayout L = make_scratch_layout(m, a.B);
  float* sc = a.scratch;
  const BlockSync sync{};
  const int tid = threadIdx.x, nth = blockDim.x;
  float* fz[kMaxLayers]; float* fa[kMaxLayers];
  float* hz[kMaxLayers]; float* ha[kMaxLayers];
  float* ez[kMaxLayers]; float* ea[kMaxLayers];
  float* cz[kMaxLayers]; float* ca[kMaxLayers];
  float* iz[kMaxLayers]; float* ia[kMaxLayers];
  for (int l = 0; l < kMaxLayers; ++l) {
    fz[l] = sc + L.fz[l]; fa[l] = sc + L.fa[l];
    hz[l] = sc + L.hz[l]; ha[l] = sc + L.ha[l];
    ez[l] = sc + L.ez[l]; ea[l] = sc + L.ea[l];
    cz[l] = sc + L.cz[l]; ca[l] = sc + L.ca[l];
    iz[l] = sc + L.iz[l]; ia[l] = sc + L.ia[l];
  }
  float* tA = sc + L.tA;
  float* tB = sc + L.tB;
  const float* latent = fa[m.fwd.L - 1];
  const int lat = m.lat, E1 = m.E1, D = m.D;

  // ---- enc wide layer: split-K reduction + bias + activation, enc tail ----
  float* e1z = sc + L.e1z;
  float* e1a = sc + L.e1a;
  const float* be = a.p[kEnc] + m.enc_wide_b;
  for (int i = tid; i < rows * E1; i += nth) {
    const int r = i / E1, j = i - r * E1;
    float acc = 0.0f;
    for (int s = 0; s < a.S; ++s) acc += a.P_enc[((long long)s * a.B + r) * E1 + j];
    const float z = acc + be[j];
    e1z[i] = z;
    e1a[i] = act_apply(m.enc_act0, m.enc_slope0, z);
  }
  sync();
  const float* real = e1a;
  if (m.enc_tail.L > 0) {
    mlp_forward(m.enc_tail, a.p[kEnc], e1a, E1, rows, (float* const*)nullptr, ea, sync);
    real = ea[m.enc_tail.L - 1];
  }
  float* stacked = sc + L.stacked;
  for (int i = tid; i < rows * lat; i += nth) {
    stacked[i] = real[i];
    stacked[rows * lat + i] = latent[i];
  }
  // ---- dec path gradient: grad wrt h, then dec head backward ----
  const long long n_fwd = (long long)rows * m.out;
  const float gscale = (float)(1.0 / (double)n_fwd);
  float* gh = sc + L.gh;
  for (int i = tid; i < rows * D; i += nth) {
    const int r = i / D, j = i - r * D;
    float acc = 0.0f;
    for (int s = 0; s < a.S; ++s) acc += a.P_dec[((long long)s * a.B + r) * D + j];
    gh[i] = gscale * acc;
  }
  sync();
  float* gl_dec = sc + L.gl_dec;
  if (m.dec_head.L > 0) {
    mlp_backward(m.dec_head, a.p[kDec], latent, lat, rows, hz, ha, gh, (float*)nullptr, gl_dec, tA,
                 tB, sync);
  } else {
    for (int i = tid; i < rows * lat; i += nth) gl_dec[i] = gh[i];
  }
  double fwd_sum = 0.0;
  if (tid == 0)
    for (int s = 0; s < a.S; ++s) fwd_sum += a.mae_part[s];
  const double fwd_mae = fwd_sum / (double)n_fwd;  // valid on thread 0
  sync();

  // ---- discriminator step (train_ops.hpp:155-186, trainer.hpp:208-229) ----
  const int n2 = 2 * rows;
  mlp_forward(m.disc, a.p[kDisc], stacked, lat, n2, cz, ca, sync);
  float* probs = sc + L.probs;
  float* bgrad = sc + L.bgrad;
  const float* logit = ca[m.disc.L - 1];
  double part = 0.0;
  for (int i = tid; i < n2; i += nth) {
    const float p = stable_sigmoid(logit[i]);
    probs[i] = p;
    const double y = i < rows ? 1.0 : 0.0;
    double pc = (double)p;
    pc = pc < 1e-7 ? 1e-7 : (pc > 1.0 - 1e-7 ? 1.0 - 1e-7 : pc);
    part += y != 0.0 ? -log(pc) : -log(1.0 - pc);
    bgrad[i] = (float)((pc - y) / (double)n2);
  }
  const double d_raw = block_sum_det(part, red) / (double)n2;
  const double d_loss = ((double)rows * d_raw) / (double)rows;  // allreduce.hpp:62-75
  mlp_backward(m.disc, a.p[kDisc], stacked, lat, n2, cz, ca, bgrad, a.g[kDisc], (float*)nullptr, tA,
               tB, sync);
  const long long n_disc = m.disc.count;
  const bool d_ok = isfinite(d_loss) && all_finite_blk(a.g[kDisc], n_disc);
  if (d_ok) {
    adam_net(a, kDisc, n_disc, sync);
  }
  sync();

  // ---- generator step (train_ops.hpp:88-151, trainer.hpp:231-272) ----
  bool g_ok = false;
  double g_total = 0, g_adv = 0, g_cyc = 0;
  if (d_ok) {
    // adversarial path against the just-updated discriminator
    mlp_forward(m.disc, a.p[kDisc], latent, lat, rows, cz, ca, sync);
    const float* lg = ca[m.disc.L - 1];
    double ap = 0.0;
    for (int i = tid; i < rows; i += nth) {
      double pc = (double)stable_sigmoid(lg[i]);
      pc = pc < 1e-7 ? 1e-7 : (pc > 1.0 - 1e-7 ? 1.0 - 1e-7 : pc);
      ap += -log(pc);
      bgrad[i] = (float)((pc - 1.0) / (double)rows) * m.lambda_adv;
    }
    const double adv = block_sum_det(ap, red) / (double)rows;
    float* gl_disc = sc + L.gl_disc;
    mlp_backward(m.disc, a.p[kDisc], latent, lat, rows, cz, ca, bgrad, (float*)nullptr, gl_disc, tA,
                 tB, sync);
    // cycle path
    mlp_forward(m.inv, a.p[kInv], latent, lat, rows, iz, ia, sync);
    const float* rec = ia[m.inv.L - 1];
    float* ig = sc + L.igrad;
    const long long n_cyc = (long long)rows * m.in;
    double cp = 0.0;
    const float pos = (float)(1.0 / (double)n_cyc), neg = (float)(-1.0 / (double)n_cyc);
    for (int i = tid; i < n_cyc; i += nth) {
      const double d = (double)rec[i] - (double)a.xb[i];
      cp += fabs(d);
      ig[i] = (d > 0 ? pos : (d < 0 ? neg : 0.0f)) * m.lambda_cyc;
    }
    const double cyc = block_sum_det(cp, red) / (double)n_cyc;
    float* gl_inv = sc + L.gl_inv;
    mlp_backward(m.inv, a.p[kInv], latent, lat, rows, iz, ia, ig, a.g[kInv], gl_inv, tA, tB, sync);
    float* gl = sc + L.gl;
    for (int i = tid; i < rows * lat; i += nth) gl[i] = (gl_dec[i] + gl_disc[i]) + gl_inv[i];
    sync();
    mlp_backward(m.fwd, a.p[kFwd], a.xb, m.in, rows, fz, fa, gl, a.g[kFwd], (float*)nullptr, tA,
                 tB, sync);
    // thread 0 holds fwd_mae; broadcast through red[0]
    if (tid == 0) red[0] = fwd_mae;
    sync();
    const double fm = red[0];
    sync();
    const double total_raw = fm + (double)m.lambda_adv * adv + (double)m.lambda_cyc * cyc;
    g_total = ((double)rows * total_raw) / (double)rows;
    g_adv = ((double)rows * adv) / (double)rows;
    g_cyc = ((double)rows * cyc) / (double)rows;
    if (isfinite(g_total)) {
      const bool fwd_ok = all_finite_blk(a.g[kFwd], m.fwd.count);
      if (fwd_ok) {
        adam_net(a, kFwd, m.fwd.count, sync);
        const bool inv_ok = all_finite_blk(a.g[kInv], m.inv.count);
        if (inv_ok) {
          adam_net(a, kInv, m.inv.count, sync);
          g_ok = true;
        }
        sync();
        if (tid == 0) {
          ctr->t[kFwd] += 1;
          if (inv_ok) ctr->t[kInv] += 1;
        }
      }
    }
    if (tid == 0) {
      red[1] = fm;
    }
  }
  sync();
  if (tid == 0) {
    if (d_ok) ctr->t[kDisc] += 1;
    const bool skipped = !(d_ok && g_ok);
    StepRec r{};
    r.d_loss = d_ok ? d_loss : 0.0;
    if (g_ok) {
      r.g_total = g_total;
      r.g_fwd = ((double)rows * red[1]) / (double)rows;
      r.g_adv = g_adv;
      r.g_cyc = g_cyc;
    }
    ctr->global_step += 1;
    ctr->step_in_epoch += 1;
    r.step = ctr->global_step;
    r.epoch = ctr->epoch;
    r.flags = (skipped ? 1u : 0u) | (d_ok ? 2u : 0u) | (g_ok ? 4u : 0u);
    if (skipped) {
      ctr->skipped += 1;
      if ((long long)ctr->skipped > (long long)a.abort_threshold) {
        ctr->aborted = 1;
        r.flags |= 8u;
      }
    }
    a.rec[(ctr->global_step - 1) % (unsigned long long)a.rec_cap] = r;
  }
}

// -------------------------------------------------------- epoch control --
__global__ void k_begin_epoch(Counters* ctr, unsigned epoch) {
  ctr->epoch = epoch;
  ctr->step_in_epoch = 0;
}

}  // namespace ltfb_dev

// ------------------------------------------------------------ launchers --
namespace ltfb_dev {

void launch_gather(const StepArgs& a, cudaStream_t s) {
  const int n4 = a.m.out_pad / 4;
  const int gx = (n4 + 256 * 4 - 1) / (256 * 4);
  k_gather<<<dim3(gx, a.B), 256, 0, s>>>(a);
}

void launch_pre(const StepArgs& a, cudaStream_t s) { k_pre<<<a.small_ctas, 128, 0, s>>>(a); }

static std::size_t wide_generic_smem(const ModelArgs& m) {
  constexpr int RB = 32, TN = 32;
  return sizeof(float) * (std::size_t)(RB * m.E1 + 2 * RB * m.D + RB * TN + TN * m.E1 + m.D * TN +
                                       RB * TN + TN);
}

void launch_wide_generic(const StepArgs& a, cudaStream_t s) {
  const std::size_t smem = wide_generic_smem(a.m);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_wide_generic<32, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  k_wide_generic<32, 32><<<a.S, 256, smem, s>>>(a);
}

void launch_post(const StepArgs& a, cudaStream_t s) { k_post<<<1, 512, 0, s>>>(a); }

void launch_begin_epoch(Counters* ctr, unsigned epoch, cudaStream_t s) {
  k_begin_epoch<<<1, 1, 0, s>>>(ctr, epoch);
}

}  // namespace ltfb_dev
