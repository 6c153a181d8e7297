// Fast path of the small-network half of a training step: the same
// algorithm as k_post_cluster (see k_post.cu for the reference mapping),
// restructured for latency. Used when every small width is <= 64, nets have
// <= 4 layers and the minibatch is <= 128 rows (16 rows per CTA):
//
//   * everything a CTA touches lives in shared memory: its rows' tapes, the
//     current network's weights W [in x out] AND a transposed copy W^T
//     (so both the forward dot products (lane = output neuron) and the
//     input-gradient dot products (lane = input neuron) read consecutive
//     banks), and its partial parameter gradients;
//   * warp-per-row forward / input-gradient, warp-per-input-neuron weight
//     gradients: each lane runs one short dependent FMA chain, many warps
//     interleave;
//   * per-CTA partial gradients are summed in cluster-rank order over
//     DSMEM by the CTA owning each parameter slice, which applies Adam to it
//     (deterministic, no atomics).
#include <cooperative_groups.h>

#include "kernels.hpp"
#include "small_mlp.cuh"

namespace cg = cooperative_groups;

namespace ltfb_dev {

namespace pf {
constexpr int kC = 8;          // CTAs per cluster
constexpr int kThreads = 256;  // 8 warps
constexpr int kRows = 16;      // rows per CTA
constexpr int kMaxW = 64;
constexpr int kMaxL = 4;
}  // namespace pf

/// Smem image of a small network: per layer W [in x out], W^T [out x in], b.
struct SNet {
  float* W[pf::kMaxL];
  float* WT[pf::kMaxL];
  float* b[pf::kMaxL];
};

__device__ __forceinline__ float* bump(float*& p, int n) {
  float* r = p;
  p += (n + 3) & ~3;
  return r;
}

__device__ void carve_net(const NetDesc& n, float*& p, SNet& s) {
  for (int l = 0; l < n.L; ++l) {
    s.W[l] = bump(p, n.w[l] * n.w[l + 1]);
    s.WT[l] = bump(p, n.w[l] * n.w[l + 1]);
    s.b[l] = bump(p, n.w[l + 1]);
  }
}

__device__ void stage_net(const NetDesc& n, const float* __restrict__ blob, const SNet& s) {
  for (int l = 0; l < n.L; ++l) {
    const int in = n.w[l], out = n.w[l + 1];
    const float* W = blob + n.off_w[l];
    for (int i = threadIdx.x; i < in * out; i += blockDim.x) {
      const float v = W[i];
      s.W[l][i] = v;
      const int k = i / out, j = i - k * out;
      s.WT[l][j * in + k] = v;
    }
    for (int j = threadIdx.x; j < out; j += blockDim.x) s.b[l][j] = blob[n.off_b[l] + j];
  }
}

struct STape {
  float* z[pf::kMaxL];
  float* a[pf::kMaxL];
};

__device__ void carve_tape(const NetDesc& n, int rows, float*& p, STape& t) {
  for (int l = 0; l < n.L; ++l) {
    t.z[l] = bump(p, rows * n.w[l + 1]);
    t.a[l] = bump(p, rows * n.w[l + 1]);
  }
}

// warp-per-row forward of one layer
__device__ __forceinline__ void wfwd(const float* x, int in, const float* W, const float* b, int out, int nr,
                                     int kind, float slope, float* z, float* a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = warp; r < nr; r += nw) {
    const float* xr = x + r * in;
    for (int j = lane; j < out; j += 32) {
      float acc = 0.0f;
#pragma unroll 4
      for (int k = 0; k < in; ++k) acc = fmaf(xr[k], W[k * out + j], acc);
      const float zz = acc + b[j];
      if (z) z[r * out + j] = zz;
      a[r * out + j] = act_apply(kind, slope, zz);
    }
  }
}

__device__ void sfwd(const NetDesc& n, const SNet& s, const float* x, int nr, const STape& t) {
  const float* cur = x;
  for (int l = 0; l < n.L; ++l) {
    wfwd(cur, n.w[l], s.W[l], s.b[l], n.w[l + 1], nr, n.act[l], n.slope[l], t.z[l], t.a[l]);
    __syncthreads();
    cur = t.a[l];
  }
}

/// Reverse pass (nn/mlp.hpp:325-361) over the smem tape. pgrad (optional,
/// blob layout relative to n.base) receives this CTA's partial sums; gin
/// (optional) the input gradient. tA/tB: [nr x 64] scratch.
__device__ void sbwd(const NetDesc& n, const SNet& s, const float* x, int nr, const STape& t,
                     const float* gout, float* pgrad, float* gin, float* tA, float* tB) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const float* g = gout;
  for (int l = n.L - 1; l >= 0; --l) {
    const int in = n.w[l], out = n.w[l + 1];
    for (int i = threadIdx.x; i < nr * out; i += blockDim.x)
      tA[i] = g[i] * act_deriv(n.act[l], n.slope[l], t.z[l][i], t.a[l][i]);
    __syncthreads();
    const float* below = l == 0 ? x : t.a[l - 1];
    if (pgrad) {
      float* dW = pgrad + (n.off_w[l] - n.base);
      float* db = pgrad + (n.off_b[l] - n.base);
      for (int k = warp; k < in; k += nw)
        for (int j = lane; j < out; j += 32) {
          float acc = 0.0f;
          for (int r = 0; r < nr; ++r) acc = fmaf(below[r * in + k], tA[r * out + j], acc);
          dW[k * out + j] = acc;
        }
      if (warp == nw - 1)
        for (int j = lane; j < out; j += 32) {
          float acc = 0.0f;
          for (int r = 0; r < nr; ++r) acc += tA[r * out + j];
          db[j] = acc;
        }
    }
    float* gn = l == 0 ? gin : tB;
    if (gn) {
      for (int r = warp; r < nr; r += nw) {
        const float* dzr = tA + r * out;
        for (int k = lane; k < in; k += 32) {
          float acc = 0.0f;
#pragma unroll 4
          for (int j = 0; j < out; ++j) acc = fmaf(dzr[j], s.WT[l][j * in + k], acc);
          gn[r * in + k] = acc;
        }
      }
    }
    __syncthreads();
    // next layer reads tB as its incoming gradient; swap roles via copy-free
    // ping-pong: dz of the next layer goes to tA again, so tB must survive
    // until then -- it does, tA is rewritten only after this barrier.
    g = tB;
  }
}

__device__ __forceinline__ double cta_sum(double v, double* red) { return block_sum_det(v, red); }

__device__ void adam_apply(const StepArgs& a, int net, long long lo, long long hi) {
  const unsigned long long t = a.ctr->t[net] + 1;
  const double c1 = a.adam_c[2 * t], c2 = a.adam_c[2 * t + 1];
  const double lr = a.lr[net], b1 = a.b1, b2 = a.b2, eps = a.eps;
  float* p = a.p[net];
  const float* g = a.g[net];
  float* m1 = a.mom1[net];
  float* m2 = a.mom2[net];
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    float m = m1[i], v = m2[i];
    p[i] = adam_elem(p[i], m, v, g[i], lr, b1, b2, eps, c1, c2);
    m1[i] = m;
    m2[i] = v;
  }
}

/// Rank-ordered DSMEM reduction of [lo, hi) of every CTA's smem partial
/// `pg` into global `dst`; returns block-uniform "all finite".
__device__ int dsmem_reduce(cg::cluster_group& cl, float* pg, int C, long long lo, long long hi, float* dst) {
  int ok = 1;
  for (long long e = lo + threadIdx.x; e < hi; e += blockDim.x) {
    float acc = 0.0f;
    for (int r = 0; r < C; ++r) acc += cl.map_shared_rank(pg, r)[e];
    dst[e] = acc;
    ok &= isfinite(acc) ? 1 : 0;
  }
  return __syncthreads_and(ok);
}

__global__ void __cluster_dims__(pf::kC, 1, 1) __launch_bounds__(pf::kThreads, 1) k_post_fast(StepArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ float4 smem4[];
  __shared__ double red[pf::kThreads];
  __shared__ double s_loss[4];
  __shared__ int s_ok[4];
  Counters* ctr = a.ctr;
  if (ctr->aborted) return;
  const ModelArgs& m = a.m;
  const ScratchLayout& L = a.L;
  const int C = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int rows = min(a.B, a.n_part - (int)ctr->step_in_epoch * a.B);
  const int per = (rows + C - 1) / C;
  const int r0 = min(rank * per, rows);
  const int nr = min(per, rows - r0);
  const int tid = threadIdx.x, nth = blockDim.x;
  const int lat = m.lat, E1 = m.E1, D = m.D, in = m.in;

  // ---- carve shared memory (identical in every CTA: DSMEM peers address
  // each other's partial-gradient buffers by offset) ----
  float* p = reinterpret_cast<float*>(smem4);
  SNet s_et, s_dh, s_disc, s_fwd, s_inv;
  carve_net(m.enc_tail, p, s_et);
  carve_net(m.dec_head, p, s_dh);
  carve_net(m.disc, p, s_disc);
  carve_net(m.inv, p, s_inv);
  carve_net(m.fwd, p, s_fwd);
  STape t_f, t_h, t_e, t_c, t_i;
  carve_tape(m.fwd, pf::kRows, p, t_f);
  carve_tape(m.dec_head, pf::kRows, p, t_h);
  carve_tape(m.enc_tail, pf::kRows, p, t_e);
  carve_tape(m.disc, 2 * pf::kRows, p, t_c);
  carve_tape(m.inv, pf::kRows, p, t_i);
  float* xs = bump(p, pf::kRows * in);
  float* e1z = bump(p, pf::kRows * E1);
  float* e1a = bump(p, pf::kRows * E1);
  float* stacked = bump(p, 2 * pf::kRows * lat);
  float* gh = bump(p, pf::kRows * D);
  float* gl_dec = bump(p, pf::kRows * lat);
  float* gl_disc = bump(p, pf::kRows * lat);
  float* gl_inv = bump(p, pf::kRows * lat);
  float* gl = bump(p, pf::kRows * lat);
  float* bgrad = bump(p, 2 * pf::kRows);
  float* ig = bump(p, pf::kRows * in);
  float* tA = bump(p, 2 * pf::kRows * pf::kMaxW);
  float* tB = bump(p, 2 * pf::kRows * pf::kMaxW);
  float* pg_disc = bump(p, (int)m.disc.count);
  float* pg_fwd = bump(p, (int)m.fwd.count);
  float* pg_inv = bump(p, (int)m.inv.count);

  // ---- stage inputs and weights ----
  const float* sc = a.scratch;
  for (int i = tid; i < nr * in; i += nth) xs[i] = a.xb[r0 * in + i];
  for (int l = 0; l < m.fwd.L; ++l) {
    const int w = m.fwd.w[l + 1];
    for (int i = tid; i < nr * w; i += nth) {
      t_f.z[l][i] = sc[L.fz[l] + (long long)r0 * w + i];
      t_f.a[l][i] = sc[L.fa[l] + (long long)r0 * w + i];
    }
  }
  for (int l = 0; l < m.dec_head.L; ++l) {
    const int w = m.dec_head.w[l + 1];
    for (int i = tid; i < nr * w; i += nth) {
      t_h.z[l][i] = sc[L.hz[l] + (long long)r0 * w + i];
      t_h.a[l][i] = sc[L.ha[l] + (long long)r0 * w + i];
    }
  }
  const float* be = a.p[kEnc] + m.enc_wide_b;
  const float* red_enc = sc + L.red_enc + (long long)r0 * E1;
  for (int i = tid; i < nr * E1; i += nth) {
    const float z = red_enc[i] + be[i % E1];
    e1z[i] = z;
    e1a[i] = act_apply(m.enc_act0, m.enc_slope0, z);
  }
  const long long n_fwd = (long long)rows * m.out;
  const float gscale = (float)(1.0 / (double)n_fwd);
  const float* red_dec = sc + L.red_dec + (long long)r0 * D;
  for (int i = tid; i < nr * D; i += nth) gh[i] = gscale * red_dec[i];
  stage_net(m.enc_tail, a.p[kEnc], s_et);
  stage_net(m.dec_head, a.p[kDec], s_dh);
  stage_net(m.disc, a.p[kDisc], s_disc);
  stage_net(m.inv, a.p[kInv], s_inv);
  stage_net(m.fwd, a.p[kFwd], s_fwd);
  __syncthreads();
  const float* latent = t_f.a[m.fwd.L - 1];

  // ---- real latents (enc tail) and the stacked disc batch ----
  const float* real = e1a;
  if (m.enc_tail.L > 0) {
    sfwd(m.enc_tail, s_et, e1a, nr, t_e);
    real = t_e.a[m.enc_tail.L - 1];
  }
  for (int i = tid; i < nr * lat; i += nth) {
    stacked[i] = real[i];
    stacked[nr * lat + i] = latent[i];
  }
  // ---- dec path input gradient ----
  if (m.dec_head.L > 0) {
    sbwd(m.dec_head, s_dh, latent, nr, t_h, gh, nullptr, gl_dec, tA, tB);
  } else {
    for (int i = tid; i < nr * lat; i += nth) gl_dec[i] = gh[i];
    __syncthreads();
  }

  // ---- discriminator step ----
  const int n2 = 2 * rows;
  sfwd(m.disc, s_disc, stacked, 2 * nr, t_c);
  const float* logit = t_c.a[m.disc.L - 1];
  double part = 0.0;
  for (int i = tid; i < 2 * nr; i += nth) {
    const double y = i < nr ? 1.0 : 0.0;
    double pc = (double)stable_sigmoid(logit[i]);
    pc = pc < 1e-7 ? 1e-7 : (pc > 1.0 - 1e-7 ? 1.0 - 1e-7 : pc);
    part += y != 0.0 ? -log(pc) : -log(1.0 - pc);
    bgrad[i] = (float)((pc - y) / (double)n2);
  }
  part = cta_sum(part, red);
  sbwd(m.disc, s_disc, stacked, 2 * nr, t_c, bgrad, pg_disc, nullptr, tA, tB);
  if (tid == 0) s_loss[0] = part;
  cl.sync();  // S1
  double d_sum = 0.0;
  for (int r = 0; r < C; ++r) d_sum += *cl.map_shared_rank(&s_loss[0], r);
  const double d_loss = ((double)rows * (d_sum / (double)n2)) / (double)rows;
  const long long dlo = m.disc.count * rank / C, dhi = m.disc.count * (rank + 1) / C;
  const int dok = dsmem_reduce(cl, pg_disc, C, dlo, dhi, a.g[kDisc]);
  if (tid == 0) s_ok[0] = dok;
  cl.sync();  // S2
  int all_dok = 1;
  for (int r = 0; r < C; ++r) all_dok &= *cl.map_shared_rank(&s_ok[0], r);
  const bool d_ok = isfinite(d_loss) && all_dok;
  if (d_ok) adam_apply(a, kDisc, dlo, dhi);
  cl.sync();  // S3: updated disc in global memory

  bool g_ok = false;
  double g_total = 0, g_fwd = 0, g_adv = 0, g_cyc = 0;
  int fwd_applied = 0, inv_applied = 0;
  if (d_ok) {
    stage_net(m.disc, a.p[kDisc], s_disc);
    __syncthreads();
    // adversarial path through the updated discriminator
    sfwd(m.disc, s_disc, latent, nr, t_c);
    const float* lg = t_c.a[m.disc.L - 1];
    double ap = 0.0;
    for (int i = tid; i < nr; i += nth) {
      double pc = (double)stable_sigmoid(lg[i]);
      pc = pc < 1e-7 ? 1e-7 : (pc > 1.0 - 1e-7 ? 1.0 - 1e-7 : pc);
      ap += -log(pc);
      bgrad[i] = (float)((pc - 1.0) / (double)rows) * m.lambda_adv;
    }
    ap = cta_sum(ap, red);
    sbwd(m.disc, s_disc, latent, nr, t_c, bgrad, nullptr, gl_disc, tA, tB);
    // cycle path
    sfwd(m.inv, s_inv, latent, nr, t_i);
    const float* rec = t_i.a[m.inv.L - 1];
    const long long n_cyc = (long long)rows * in;
    const float pos = (float)(1.0 / (double)n_cyc), neg = (float)(-1.0 / (double)n_cyc);
    double cp = 0.0;
    for (int i = tid; i < nr * in; i += nth) {
      const double d = (double)rec[i] - (double)xs[i];
      cp += fabs(d);
      ig[i] = (d > 0 ? pos : (d < 0 ? neg : 0.0f)) * m.lambda_cyc;
    }
    cp = cta_sum(cp, red);
    sbwd(m.inv, s_inv, latent, nr, t_i, ig, pg_inv, gl_inv, tA, tB);
    for (int i = tid; i < nr * lat; i += nth) gl[i] = (gl_dec[i] + gl_disc[i]) + gl_inv[i];
    __syncthreads();
    sbwd(m.fwd, s_fwd, xs, nr, t_f, gl, pg_fwd, nullptr, tA, tB);
    if (tid == 0) {
      s_loss[1] = ap;
      s_loss[2] = cp;
    }
    cl.sync();  // S4
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
    const int fok = dsmem_reduce(cl, pg_fwd, C, flo, fhi, a.g[kFwd]);
    const int iok = dsmem_reduce(cl, pg_inv, C, ilo, ihi, a.g[kInv]);
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
    // trainer.hpp:256-264 ordering: g_total, then fwd (throws before any
    // change), then inv (fwd already applied)
    if (isfinite(g_total) && all_f) {
      adam_apply(a, kFwd, flo, fhi);
      fwd_applied = 1;
      if (all_i) {
        adam_apply(a, kInv, ilo, ihi);
        inv_applied = 1;
        g_ok = true;
      }
    }
  }
  cl.sync();  // S6: all reads of counters / DSMEM done
  if (rank == 0 && tid == 0) {
    if (d_ok) ctr->t[kDisc] += 1;
    if (fwd_applied) ctr->t[kFwd] += 1;
    if (inv_applied) ctr->t[kInv] += 1;
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

// ----------------------------------------------------------------- host --
static int net_smem_floats(const NetDesc& n) {
  int f = 0;
  for (int l = 0; l < n.L; ++l) f += 2 * ((n.w[l] * n.w[l + 1] + 3) & ~3) + ((n.w[l + 1] + 3) & ~3);
  return f;
}
static int tape_smem_floats(const NetDesc& n, int rows) {
  int f = 0;
  for (int l = 0; l < n.L; ++l) f += 2 * ((rows * n.w[l + 1] + 3) & ~3);
  return f;
}

std::size_t post_fast_smem(const ModelArgs& m) {
  const int nr = pf::kRows;
  auto r4 = [](int v) { return (v + 3) & ~3; };
  int f = net_smem_floats(m.enc_tail) + net_smem_floats(m.dec_head) + net_smem_floats(m.disc) +
          net_smem_floats(m.inv) + net_smem_floats(m.fwd);
  f += tape_smem_floats(m.fwd, nr) + tape_smem_floats(m.dec_head, nr) + tape_smem_floats(m.enc_tail, nr) +
       tape_smem_floats(m.disc, 2 * nr) + tape_smem_floats(m.inv, nr);
  f += r4(nr * m.in) + 2 * r4(nr * m.E1) + r4(2 * nr * m.lat) + r4(nr * m.D) + 4 * r4(nr * m.lat) + r4(2 * nr) +
       r4(nr * m.in) + 2 * r4(2 * nr * pf::kMaxW);
  f += r4((int)m.disc.count) + r4((int)m.fwd.count) + r4((int)m.inv.count);
  return (std::size_t)f * sizeof(float);
}

bool post_fast_supported(const StepArgs& a) {
  const ModelArgs& m = a.m;
  if (a.B > pf::kC * pf::kRows) return false;
  const NetDesc* nets[5] = {&m.fwd, &m.inv, &m.disc, &m.enc_tail, &m.dec_head};
  for (const NetDesc* n : nets) {
    if (n->L > pf::kMaxL) return false;
    for (int i = 0; i <= n->L; ++i)
      if (n->L > 0 && n->w[i] > pf::kMaxW) return false;
  }
  if (m.E1 > pf::kMaxW || m.D > pf::kMaxW || m.lat > pf::kMaxW || m.in > pf::kMaxW) return false;
  return post_fast_smem(m) <= 200 * 1024;
}

void launch_post_fast(const StepArgs& a, cudaStream_t s) {
  static PerDevice attr;
  const std::size_t smem = post_fast_smem(a.m);
  attr.once([] { cudaFuncSetAttribute(k_post_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); });
  k_post_fast<<<pf::kC, pf::kThreads, smem, s>>>(a);
}

}  // namespace ltfb_dev
