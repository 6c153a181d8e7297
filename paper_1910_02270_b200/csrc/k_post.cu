// Split-K reduction of the wide pass and the small-network half of a
// training step (train/trainer.hpp:208-290 over surrogate/train_ops.hpp):
//
//   k_reduce        fixed-order sums of the wide pass's per-CTA partials
//                   (enc layer-0 pre-activations, dec h-gradients, |d| sums)
//   k_post_cluster  one thread-block cluster of kPostCluster CTAs; each CTA
//                   owns a slice of minibatch rows. Row-parallel work (enc
//                   tail, BCE, MAE-cycle, every backprop) stays CTA-local;
//                   parameter gradients are per-CTA partials reduced in rank
//                   order by the CTA that owns each parameter slice, which
//                   then applies Adam to that slice. Cluster barriers
//                   (release/acquire) order the phases:
//     D-step: disc fwd/bwd on [real; fake] rows -> reduce -> finite check
//             (loss + all grads, adam.hpp:95-102) -> Adam(disc)
//     G-step: adversarial path through the UPDATED disc, cycle path through
//             inv, grad_latent = dec + disc + inv (train_ops.hpp:104-127),
//             fwd backprop -> reduce -> finite checks -> Adam(fwd), Adam(inv)
//     record: StepRecord, skip / abort counters (trainer.hpp:274-289)
#include <cooperative_groups.h>

#include "kernels.hpp"
#include "scratch_layout.cuh"
#include "small_mlp.cuh"

namespace cg = cooperative_groups;

namespace ltfb_dev {

__device__ __forceinline__ int post_rows(const StepArgs& a) {
  const int begin = (int)a.ctr->step_in_epoch * a.B;
  const int left = a.n_part - begin;
  return left < a.B ? left : a.B;
}

// ---------------------------------------------------------------- reduce --
// CTA = 32 consecutive outputs x 8 groups of partials: thread (o, g) sums
// partials g, g+8, ... (each warp load is 128 B contiguous), the 8 group
// sums are then combined in group order -> deterministic, all SMs busy.
constexpr int kRedOut = 32, kRedGroups = 8;
__global__ void __launch_bounds__(kRedOut * kRedGroups) k_reduce(StepArgs a) {
  if (a.ctr->aborted) return;
  __shared__ float part[kRedGroups][kRedOut];
  const int rows = post_rows(a);
  const ModelArgs& m = a.m;
  const ScratchLayout& L = a.L;
  float* red_enc = a.scratch + L.red_enc;
  float* red_dec = a.scratch + L.red_dec;
  const long long ne = (long long)rows * m.E1, nd = (long long)rows * m.D;
  const int o = threadIdx.x % kRedOut, g = threadIdx.x / kRedOut;
  for (long long base = (long long)blockIdx.x * kRedOut; base < ne + nd; base += (long long)gridDim.x * kRedOut) {
    const long long idx = base + o;
    float acc = 0.0f;
    if (idx < ne) {
      const float* p = a.P_enc + idx;
      for (int s = g; s < a.S; s += kRedGroups) acc += p[(long long)s * a.B * m.E1];
    } else if (idx < ne + nd) {
      const float* p = a.P_dec + (idx - ne);
      for (int s = g; s < a.S; s += kRedGroups) acc += p[(long long)s * a.B * m.D];
    }
    part[g][o] = acc;
    __syncthreads();
    if (g == 0 && idx < ne + nd) {
      float t = 0.0f;
      for (int k = 0; k < kRedGroups; ++k) t += part[k][o];
      if (idx < ne) red_enc[idx] = t;
      else red_dec[idx - ne] = t;
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double t = 0.0;
    for (int s = 0; s < a.S; ++s) t += a.mae_part[s];
    *a.mae_total = t;
  }
}

// ------------------------------------------------------------------- Adam --
// nn/adam.hpp:48-61: the shared element update (device_common.cuh)
__device__ __forceinline__ void adam_elem_ref(float& p, float g, float& m1, float& m2, double lr, double b1,
                                              double b2, double eps, double c1, double c2) {
  p = adam_elem(p, m1, m2, g, lr, b1, b2, eps, c1, c2);
}

__device__ void adam_slice(const StepArgs& a, int net, long long lo, long long hi) {
  const unsigned long long t = a.ctr->t[net] + 1;
  const double c1 = a.adam_c[2 * t], c2 = a.adam_c[2 * t + 1];
  float* p = a.p[net];
  const float* g = a.g[net];
  float* m1 = a.mom1[net];
  float* m2 = a.mom2[net];
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x)
    adam_elem_ref(p[i], g[i], m1[i], m2[i], a.lr[net], a.b1, a.b2, a.eps, c1, c2);
}

/// Sums the C per-CTA partials of [lo, hi) in rank order into `dst`;
/// returns 1 if every summed element is finite (block-uniform).
__device__ int reduce_slice(const float* pg, long long stride, int C, long long lo, long long hi,
                            float* dst) {
  int ok = 1;
  for (long long e = lo + threadIdx.x; e < hi; e += blockDim.x) {
    float acc = 0.0f;
    for (int r = 0; r < C; ++r) acc += pg[r * stride + e];
    dst[e] = acc;
    ok &= isfinite(acc) ? 1 : 0;
  }
  return __syncthreads_and(ok);
}

struct Tape {
  float* z[kMaxLayers];
  float* a[kMaxLayers];
};

__device__ Tape tape_at(float* sc, const long long* zo, const long long* ao, const NetDesc& n,
                        long long row0) {
  Tape t;
  for (int l = 0; l < kMaxLayers; ++l) {
    const long long w = l < n.L ? n.w[l + 1] : 0;
    t.z[l] = sc + zo[l] + row0 * w;
    t.a[l] = sc + ao[l] + row0 * w;
  }
  return t;
}

// ------------------------------------------------------------------ post --
__global__ void __cluster_dims__(kPostCluster, 1, 1) __launch_bounds__(kPostThreads)
    k_post_cluster(StepArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double red[kPostThreads];
  __shared__ double s_loss[4];  // d, adv, cyc partials of this CTA
  __shared__ int s_ok[4];       // disc, fwd, inv slice finiteness
  Counters* ctr = a.ctr;
  if (ctr->aborted) return;  // uniform across the cluster
  const ModelArgs& m = a.m;
  const int C = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int rows = post_rows(a);
  const int per = (rows + C - 1) / C;
  const int r0 = min(rank * per, rows);
  const int nr = min(per, rows - r0);
  const ScratchLayout& L = a.L;
  float* sc = a.scratch;
  const BlockSync bs{};
  const int tid = threadIdx.x, nth = blockDim.x;
  const int lat = m.lat, E1 = m.E1, D = m.D;
  float* tA = sc + L.tA + rank * L.tstride;
  float* tB = sc + L.tB + rank * L.tstride;

  const Tape ft = tape_at(sc, L.fz, L.fa, m.fwd, r0);       // from k_pre
  const Tape ht = tape_at(sc, L.hz, L.ha, m.dec_head, r0);  // from k_pre
  const float* latent = ft.a[m.fwd.L - 1];                  // my rows
  const float* xr = a.xb + (long long)r0 * m.in;

  // ---- enc wide layer epilogue + enc tail (real latents) ----
  float* e1z = sc + L.e1z + (long long)r0 * E1;
  float* e1a = sc + L.e1a + (long long)r0 * E1;
  const float* be = a.p[kEnc] + m.enc_wide_b;
  const float* red_enc = sc + L.red_enc + (long long)r0 * E1;
  for (int i = tid; i < nr * E1; i += nth) {
    const float z = red_enc[i] + be[i % E1];
    e1z[i] = z;
    e1a[i] = act_apply(m.enc_act0, m.enc_slope0, z);
  }
  bs();
  const float* real = e1a;
  if (m.enc_tail.L > 0) {
    const Tape et = tape_at(sc, L.ez, L.ea, m.enc_tail, r0);
    mlp_forward(m.enc_tail, a.p[kEnc], e1a, E1, nr, (float* const*)nullptr, et.a, bs);
    real = et.a[m.enc_tail.L - 1];
  }
  float* stacked = sc + L.stacked + 2LL * r0 * lat;  // [real rows; fake rows] of this CTA
  for (int i = tid; i < nr * lat; i += nth) {
    stacked[i] = real[i];
    stacked[nr * lat + i] = latent[i];
  }
  // ---- dec path: dL/dh = (1/n) * sum_c sign(d) W, dec head backward ----
  const long long n_fwd = (long long)rows * m.out;
  const float gscale = (float)(1.0 / (double)n_fwd);
  float* gh = sc + L.gh + (long long)r0 * D;
  const float* red_dec = sc + L.red_dec + (long long)r0 * D;
  for (int i = tid; i < nr * D; i += nth) gh[i] = gscale * red_dec[i];
  bs();
  float* gl_dec = sc + L.gl_dec + (long long)r0 * lat;
  if (m.dec_head.L > 0) {
    mlp_backward(m.dec_head, a.p[kDec], latent, lat, nr, ht.z, ht.a, gh, (float*)nullptr, gl_dec, tA, tB, bs);
  } else {
    for (int i = tid; i < nr * lat; i += nth) gl_dec[i] = gh[i];
    bs();
  }

  // ---- discriminator step ----
  const int n2 = 2 * rows;
  const Tape ct = tape_at(sc, L.cz, L.ca, m.disc, 2LL * r0);
  mlp_forward(m.disc, a.p[kDisc], stacked, lat, 2 * nr, ct.z, ct.a, bs);
  float* bgrad = sc + L.bgrad + 2LL * r0;
  const float* logit = ct.a[m.disc.L - 1];
  double part = 0.0;
  for (int i = tid; i < 2 * nr; i += nth) {
    const float p = stable_sigmoid(logit[i]);
    const double y = i < nr ? 1.0 : 0.0;
    double pc = (double)p;
    pc = pc < 1e-7 ? 1e-7 : (pc > 1.0 - 1e-7 ? 1.0 - 1e-7 : pc);
    part += y != 0.0 ? -log(pc) : -log(1.0 - pc);
    bgrad[i] = (float)((pc - y) / (double)n2);
  }
  part = block_sum_det(part, red);
  const long long sd = round_up_ll(m.disc.count, 32);
  float* pg_disc = sc + L.pg_disc;
  mlp_backward(m.disc, a.p[kDisc], stacked, lat, 2 * nr, ct.z, ct.a, bgrad, pg_disc + rank * sd,
               (float*)nullptr, tA, tB, bs);
  if (tid == 0) s_loss[0] = part;
  cl.sync();  // S1: disc partials + loss partials visible
  double d_sum = 0.0;
  for (int r = 0; r < C; ++r) d_sum += *cl.map_shared_rank(&s_loss[0], r);
  const double d_loss = ((double)rows * (d_sum / (double)n2)) / (double)rows;  // allreduce.hpp:62-75
  const long long dlo = m.disc.count * rank / C, dhi = m.disc.count * (rank + 1) / C;
  const int dok = reduce_slice(pg_disc, sd, C, dlo, dhi, a.g[kDisc]);
  if (tid == 0) s_ok[0] = dok;
  cl.sync();  // S2: slice finiteness visible
  int all_dok = 1;
  for (int r = 0; r < C; ++r) all_dok &= *cl.map_shared_rank(&s_ok[0], r);
  const bool d_ok = isfinite(d_loss) && all_dok;
  if (d_ok) adam_slice(a, kDisc, dlo, dhi);
  cl.sync();  // S3: updated disc visible to every CTA

  // ---- generator step ----
  bool g_ok = false;
  double g_total = 0, g_fwd = 0, g_adv = 0, g_cyc = 0;
  if (d_ok) {
    // adversarial path against the just-updated discriminator
    mlp_forward(m.disc, a.p[kDisc], latent, lat, nr, ct.z, ct.a, bs);
    const float* lg = ct.a[m.disc.L - 1];
    double ap = 0.0;
    for (int i = tid; i < nr; i += nth) {
      double pc = (double)stable_sigmoid(lg[i]);
      pc = pc < 1e-7 ? 1e-7 : (pc > 1.0 - 1e-7 ? 1.0 - 1e-7 : pc);
      ap += -log(pc);
      bgrad[i] = (float)((pc - 1.0) / (double)rows) * m.lambda_adv;
    }
    ap = block_sum_det(ap, red);
    float* gl_disc = sc + L.gl_disc + (long long)r0 * lat;
    mlp_backward(m.disc, a.p[kDisc], latent, lat, nr, ct.z, ct.a, bgrad, (float*)nullptr, gl_disc, tA, tB, bs);
    // cycle path
    const Tape it = tape_at(sc, L.iz, L.ia, m.inv, r0);
    mlp_forward(m.inv, a.p[kInv], latent, lat, nr, it.z, it.a, bs);
    const float* rec = it.a[m.inv.L - 1];
    float* ig = sc + L.igrad + (long long)r0 * m.in;
    const long long n_cyc = (long long)rows * m.in;
    const float pos = (float)(1.0 / (double)n_cyc), neg = (float)(-1.0 / (double)n_cyc);
    double cp = 0.0;
    for (int i = tid; i < nr * m.in; i += nth) {
      const double d = (double)rec[i] - (double)xr[i];
      cp += fabs(d);
      ig[i] = (d > 0 ? pos : (d < 0 ? neg : 0.0f)) * m.lambda_cyc;
    }
    cp = block_sum_det(cp, red);
    const long long si = round_up_ll(m.inv.count, 32), sf = round_up_ll(m.fwd.count, 32);
    float* pg_inv = sc + L.pg_inv;
    float* pg_fwd = sc + L.pg_fwd;
    float* gl_inv = sc + L.gl_inv + (long long)r0 * lat;
    mlp_backward(m.inv, a.p[kInv], latent, lat, nr, it.z, it.a, ig, pg_inv + rank * si, gl_inv, tA, tB, bs);
    float* gl = sc + L.gl + (long long)r0 * lat;
    for (int i = tid; i < nr * lat; i += nth) gl[i] = (gl_dec[i] + gl_disc[i]) + gl_inv[i];
    bs();
    mlp_backward(m.fwd, a.p[kFwd], xr, m.in, nr, ft.z, ft.a, gl, pg_fwd + rank * sf, (float*)nullptr, tA, tB, bs);
    if (tid == 0) {
      s_loss[1] = ap;
      s_loss[2] = cp;
    }
    cl.sync();  // S4: fwd/inv partials + loss partials visible
    double adv_sum = 0.0, cyc_sum = 0.0;
    for (int r = 0; r < C; ++r) {
      adv_sum += *cl.map_shared_rank(&s_loss[1], r);
      cyc_sum += *cl.map_shared_rank(&s_loss[2], r);
    }
    const double adv = adv_sum / (double)rows;
    const double cyc = cyc_sum / (double)n_cyc;
    const double fm = *a.mae_total / (double)n_fwd;
    const double total_raw = fm + (double)m.lambda_adv * adv + (double)m.lambda_cyc * cyc;
    g_total = ((double)rows * total_raw) / (double)rows;
    g_fwd = ((double)rows * fm) / (double)rows;
    g_adv = ((double)rows * adv) / (double)rows;
    g_cyc = ((double)rows * cyc) / (double)rows;
    const long long flo = m.fwd.count * rank / C, fhi = m.fwd.count * (rank + 1) / C;
    const long long ilo = m.inv.count * rank / C, ihi = m.inv.count * (rank + 1) / C;
    const int fok = reduce_slice(pg_fwd, sf, C, flo, fhi, a.g[kFwd]);
    const int iok = reduce_slice(pg_inv, si, C, ilo, ihi, a.g[kInv]);
    if (tid == 0) {
      s_ok[1] = fok;
      s_ok[2] = iok;
    }
    cl.sync();  // S5
    int all_f = 1, all_i = 1;
    for (int r = 0; r < C; ++r) {
      all_f &= *cl.map_shared_rank(&s_ok[1], r);
      all_i &= *cl.map_shared_rank(&s_ok[2], r);
    }
    // trainer.hpp:256-264: g_total finite, then adam_step(fwd) (throws before
    // touching state on a non-finite fwd grad), then adam_step(inv)
    if (isfinite(g_total) && all_f) {
      adam_slice(a, kFwd, flo, fhi);
      if (all_i) {
        adam_slice(a, kInv, ilo, ihi);
        g_ok = true;
      }
      if (rank == 0 && tid == 0) {
        // counters are advanced after the final barrier (readers above)
        s_ok[3] = 1 | (all_i ? 2 : 0);
      }
    } else if (rank == 0 && tid == 0) {
      s_ok[3] = 0;
    }
  }
  cl.sync();  // S6: every CTA is done reading counters and parameters
  if (rank == 0 && tid == 0) {
    if (d_ok) {
      ctr->t[kDisc] += 1;
      if (s_ok[3] & 1) ctr->t[kFwd] += 1;
      if (s_ok[3] & 2) ctr->t[kInv] += 1;
    }
    const bool skipped = !(d_ok && g_ok);
    StepRec r{};
    r.d_loss = d_ok ? d_loss : 0.0;
    if (g_ok) {
      r.g_total = g_total;
      r.g_fwd = g_fwd;
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

void launch_reduce(const StepArgs& a, cudaStream_t s) {
  const long long n = (long long)a.B * (a.m.E1 + a.m.D);
  const int grid = (int)std::min<long long>((n + kRedOut - 1) / kRedOut, 148 * 8);
  k_reduce<<<grid, kRedOut * kRedGroups, 0, s>>>(a);
}

void launch_post(const StepArgs& a, cudaStream_t s) {
  k_post_cluster<<<kPostCluster, kPostThreads, 0, s>>>(a);
}

}  // namespace ltfb_dev
