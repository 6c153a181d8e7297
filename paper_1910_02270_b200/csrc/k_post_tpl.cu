// Latency-optimised small-network half of a training step
// (train/trainer.hpp:208-290 over surrogate/train_ops.hpp:88-186), for every
// architecture whose small widths are <= 64 with <= 4 layers per network:
//
//   D-step  real = enc_tail(act(red_enc + b)), fake = fwd(x);
//           disc fwd/bwd on [real; fake] (BCE, loss.hpp:59-88);
//           cluster-ordered gradient reduction; finite check
//           (adam.hpp:95-102); Adam(disc) (adam.hpp:87-122)
//   G-step  dec path  grad_h = (1/n) S Wd^T (from the wide pass) through the
//                     dec head (train_ops.hpp:100-104)
//           adversarial path through the UPDATED disc (train_ops.hpp:106-117)
//           cycle path through inv (train_ops.hpp:119-127)
//           grad_latent = (dec + disc) + inv; fwd backprop; Adam(fwd), then
//           Adam(inv) (trainer.hpp:256-264)
//
// The step is a chain of ~35 dependent micro-phases of 10-50 kFMA each, so
// it is bound by latency and by instruction delivery, not by FLOPs or bytes.
// Profiles of earlier variants (fully unrolled templates: 220 KB of SASS,
// 51 % of stall samples "no_instructions"; straight-line code calling
// helpers: ~3.5 k cycles per layer against ~1.3 k for the same routine with
// warm code) showed that the instruction footprint decides the time. So the
// kernel is an INTERPRETER: the host compiles the step into a program of
// micro-ops (forward layer, backward layer, loss heads, cluster exchange,
// Adam) passed as a kernel parameter, and the device runs one compact loop
// whose handlers stay resident in the instruction cache:
//   * one forward-layer handler and one backward-layer handler (weight- and
//     input-gradient items side by side, dz = g*act'(z) of the layer below
//     applied in the epilogue) serve every layer of every network; operands
//     live in shared memory (blob images, transposed weights, tapes);
//   * one asynchronous staging pass (cp.async) brings every parameter, the
//     owner-slice Adam moments and this CTA's rows in with one global round
//     trip.
//
// One cluster of 8 CTAs; CTA c owns minibatch rows [c*16, c*16+16) and the
// parameter slice [c*n/8, (c+1)*n/8) of every trained network. Partial
// parameter gradients stay in each CTA's shared memory; the owner sums the 8
// partials in rank order over DSMEM (deterministic, no atomics), applies Adam
// to its slice, and the updated discriminator is pulled back over DSMEM.
// Work that does not depend on the D-step (dec-head backward, the whole cycle
// path) runs between the split cluster-barrier arrive and wait.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "kernels.hpp"

namespace cg = cooperative_groups;

namespace ltfb_dev {
namespace ps {

constexpr int kC = 8;          // CTAs per cluster
constexpr int kThreads = 256;  // 8 warps
constexpr int kR = 16;         // minibatch rows per CTA (B <= 128)
constexpr int kMaxL = 4;
constexpr int kMaxW = 64;
constexpr int kMaxOps = 64;

enum OpKind : int {
  kOpFwd = 1,   // z = x W + b, a = act(z)
  kOpBwd,       // weight/bias partial gradients + input gradient of one layer
  kOpDz,        // out = g * act'(z, a)
  kOpBce,       // D-step BCE on [real; fake] logits
  kOpCyc,       // cycle MAE on inv(latent) vs x
  kOpAdv,       // adversarial BCE(ones) on disc(latent)
  kOpArrive,    // cluster barrier arrive (release)
  kOpWait,      // cluster barrier wait (acquire)
  kOpDUpdate,   // disc: owner reduction, finite check, Adam, DSMEM pull
  kOpGUpdate,   // fwd / inv: owner reduction, finite checks, Adam
};

/// One micro-op. Fields by kind (offsets are floats into dynamic smem):
///  (row buffers are [rows x pad8(width)] with zero pad columns)
///  Fwd: p0 x, p1 W [IN x OUT], p2 b, p3 z, p4 a, p5 act, p6 slope bits
///  Bwd: p0 dz [R x OUT], p1 below [R x IN], p2 W [IN x OUT], p3 pgW (or -1),
///       p4 pgb, p5 gin (or -1), p6 epiA (or -1), p7 epiB, p8 z', p9 a',
///       p10 act' (0: none), p11 slope' bits  (' = layer below)
///  Dz:  p0 g, p1 z, p2 a, p3 act, p4 slope bits, p5 out; n = R*OUT
///  Bce/Adv: p0 logits, p1 grad;  Cyc: p0 rec, p1 xs, p2 grad
struct Op {
  int kind, skip_unless_d, R, IN, OUT;
  int p[12];
};

struct Prog {
  int n;
  int xs, e1, be, gh, stacked, gl_dec, gl_inv, gl, one;
  int blob[3];              // staged blobs: disc, fwd, inv
  int count[3];
  int pg[3];                // partial gradients (blob layout)
  int mo[3], vo[3], gr[3];  // owner-slice moments / reduced gradients
  int et_blob, et_count, dh_blob, dh_count;
  int disc_T[kMaxL], disc_W[kMaxL], disc_in[kMaxL], disc_out[kMaxL], disc_L;
  int total;
  Op op[kMaxOps];
};

extern __shared__ float4 smem4[];
__device__ __forceinline__ float* S() { return reinterpret_cast<float*>(smem4); }

__device__ __forceinline__ float act_f(int kind, float s, float z) {
  return kind == kLeaky ? (z > 0.0f ? z : s * z) : (kind == kIdentity ? z : act_apply(kind, s, z));
}
__device__ __forceinline__ float act_d(int kind, float s, float z, float a) {
  return kind == kLeaky ? (z > 0.0f ? 1.0f : s) : (kind == kIdentity ? 1.0f : act_deriv(kind, s, z, a));
}

__device__ __forceinline__ void cp4(int dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(S() + dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_sync() {
  cluster_arrive();
  cluster_wait();
}

__device__ __forceinline__ int pad8(int v) { return (v + 7) & ~7; }

__device__ __forceinline__ void split_tf32(float x, unsigned& hi, unsigned& lo) {
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
  const float r = x - __uint_as_float(hi);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(r));
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

/// Epilogue selector of mm().
enum { kEpiFwd = 0, kEpiGin = 1, kEpiPg = 2 };

/// D(m,n) = sum_k A(m,k) B(k,n) on the tensor cores: warp-level mma.sync
/// m16n8k8 TF32 with the 3xTF32 split (a_hi b_hi + a_hi b_lo + a_lo b_hi,
/// f32 accumulation), which keeps fp32 accuracy. One 16x8 tile per warp at a
/// time, tiles dealt round-robin from warp w0.
///   A(m,k) = s[a + m*asm_ + k*ask] (row `ones` reads as 1: bias gradient)
///   B(k,n) = s[b + k*bsk + n*bsn]
/// K runs to a multiple of 8: every activation / gradient buffer is
/// zero-padded to 8 columns and the whole shared image starts zeroed, so pad
/// products vanish; reads past a weight matrix land in the finite bias /
/// next layer. Epilogues (valid rows m < M):
///   kEpiFwd: v = acc + bias[n]; z = v, a = act(v), row stride ldo, pad cols 0
///   kEpiGin: v = acc [(epiA + v) + epiB] [* act'(z', a')], stride ldo, pad 0
///   kEpiPg : blob layout, m < ones: out[m*N + n]; m == ones: out2[n]
struct MmArgs {
  int M, N, K, a, asm_, ask, b, bsk, bsn, ones, epi, out, out2, ldo;
  int bias, z, act;  // fwd
  float slope;
  int epiA, epiB, dz, da, dact;  // gin
  float dslope;
};

__device__ __noinline__ void mm(const MmArgs p, int w0) {
  float* s = S();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int M = p.M, N = p.N, Kp = pad8(p.K);
  const int nt = (N + 7) >> 3, tiles = ((M + 15) >> 4) * nt;
  for (int t = (warp - w0 + kThreads / 32) % (kThreads / 32); t < tiles; t += kThreads / 32) {
    const int m0 = (t / nt) * 16, n0 = (t % nt) * 8;
    const int ra = m0 + gid, rb = ra + 8;
    const bool oa = ra == p.ones, ob = rb == p.ones;
    const float* Aa = s + p.a + ra * p.asm_ + tig * p.ask;
    const float* Ab = s + p.a + rb * p.asm_ + tig * p.ask;
    const float* Bc = s + p.b + (n0 + gid) * p.bsn + tig * p.bsk;
    const int a4 = 4 * p.ask, a8 = 8 * p.ask, b4 = 4 * p.bsk, b8 = 8 * p.bsk;
    float d[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 2
    for (int k0 = 0; k0 < Kp; k0 += 8) {
      const float av0 = oa ? 1.0f : Aa[0], av1 = ob ? 1.0f : Ab[0];
      const float av2 = oa ? 1.0f : Aa[a4], av3 = ob ? 1.0f : Ab[a4];
      const float bv0 = Bc[0], bv1 = Bc[b4];
      Aa += a8;
      Ab += a8;
      Bc += b8;
      unsigned ah[4], al[4], bh[2], bl[2];
      split_tf32(av0, ah[0], al[0]);
      split_tf32(av1, ah[1], al[1]);
      split_tf32(av2, ah[2], al[2]);
      split_tf32(av3, ah[3], al[3]);
      split_tf32(bv0, bh[0], bl[0]);
      split_tf32(bv1, bh[1], bl[1]);
      mma_tf32(d, al, bh);
      mma_tf32(d, ah, bl);
      mma_tf32(d, ah, bh);
    }
    // accumulator i: row m0 + gid (+8 for i >= 2), col n0 + 2 tig + (i & 1)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + gid + ((i >> 1) << 3), n = n0 + 2 * tig + (i & 1);
      if (m >= M) continue;
      const bool vn = n < N;
      if (p.epi == kEpiPg) {
        if (vn) s[m == p.ones ? p.out2 + n : p.out + m * N + n] = d[i];
        continue;
      }
      const int o = m * p.ldo + n;
      if (p.epi == kEpiFwd) {
        const float v = vn ? d[i] + s[p.bias + n] : 0.0f;
        s[p.z + o] = v;
        s[p.out + o] = vn ? act_f(p.act, p.slope, v) : 0.0f;
      } else {
        float v = d[i];
        if (p.epiA >= 0) v = (s[p.epiA + o] + v) + s[p.epiB + o];
        if (p.dact) v = v * act_d(p.dact, p.dslope, s[p.dz + o], s[p.da + o]);
        s[p.out + o] = vn ? v : 0.0f;
      }
    }
  }
}

/// Forward layer (nn/mlp.hpp:201-217: matmul, add_row_vector, activation).
__device__ __forceinline__ void op_fwd(const Op& o) {
  MmArgs p{};
  p.M = o.R;
  p.N = o.OUT;
  p.K = o.IN;
  p.a = o.p[0];
  p.asm_ = pad8(o.IN);
  p.ask = 1;
  p.b = o.p[1];
  p.bsk = o.OUT;
  p.bsn = 1;
  p.ones = -1;
  p.epi = kEpiFwd;
  p.out = o.p[4];
  p.ldo = pad8(o.OUT);
  p.bias = o.p[2];
  p.z = o.p[3];
  p.act = o.p[5];
  p.slope = __int_as_float(o.p[6]);
  mm(p, 0);
}

/// Reverse of one layer from its dz (nn/mlp.hpp:270-279), two products in
/// one phase: pgW / pgb = below^T [dz] with a row of ones for the bias
/// (fmaf(1, d, acc) == acc + d), and gin = dz W^T with the optional
/// epilogues ((epiA + v) + epiB for grad_latent = dec + disc + inv,
/// train_ops.hpp:104-127; times act'(z', a') when gin is the dz of the layer
/// below).
__device__ __forceinline__ void op_bwd(const Op& o) {
  int w0 = 0;
  if (o.p[3] >= 0) {
    MmArgs p{};
    p.M = o.IN + 1;
    p.N = o.OUT;
    p.K = o.R;
    p.a = o.p[1];
    p.asm_ = 1;
    p.ask = pad8(o.IN);
    p.b = o.p[0];
    p.bsk = pad8(o.OUT);
    p.bsn = 1;
    p.ones = o.IN;
    p.epi = kEpiPg;
    p.out = o.p[3];
    p.out2 = o.p[4];
    mm(p, 0);
    w0 = (((o.IN + 16) >> 4) * ((o.OUT + 7) >> 3)) & 7;
  }
  if (o.p[5] >= 0) {
    MmArgs p{};
    p.M = o.R;
    p.N = o.IN;
    p.K = o.OUT;
    p.a = o.p[0];
    p.asm_ = pad8(o.OUT);
    p.ask = 1;
    p.b = o.p[2];
    p.bsk = 1;
    p.bsn = o.OUT;  // B(k=j, n=i) = W[i][j]
    p.ones = -1;
    p.epi = kEpiGin;
    p.out = o.p[5];
    p.ldo = pad8(o.IN);
    p.epiA = o.p[6];
    p.epiB = o.p[7];
    p.dz = o.p[8];
    p.da = o.p[9];
    p.dact = o.p[10] > 0 ? o.p[10] : 0;
    p.dslope = __int_as_float(o.p[11]);
    mm(p, w0);
  }
}

/// Owner reduction of [lo, hi) over the kC partials at smem offset pg, in
/// rank order, into gr; returns this CTA's "all finite" (block-uniform).
__device__ __noinline__ int reduce_owned(int pg, int lo, int hi, int gr) {
  cg::cluster_group cl = cg::this_cluster();
  float* s = S();
  int ok = 1;
  for (int e = lo + (int)threadIdx.x; e < hi; e += kThreads) {
    float v[kC];
#pragma unroll
    for (int r = 0; r < kC; ++r) v[r] = cl.map_shared_rank(s + pg, r)[e];
    float acc = 0.0f;
#pragma unroll
    for (int r = 0; r < kC; ++r) acc += v[r];
    s[gr + e - lo] = acc;
    ok &= isfinite(acc) ? 1 : 0;
  }
  return __syncthreads_and(ok);
}

/// nn/adam.hpp:48-61 in double with explicit round-to-nearest operations
/// (no FMA contraction): bit-identical to the reference's scalar loop.
__device__ __noinline__ void adam_owned(const StepArgs& a, int net, int lo, int hi, double c1, double c2,
                                        int p_smem, int gr, int mo, int vo) {
  float* s = S();
  const double lr = a.lr[net], b1 = a.b1, b2 = a.b2, eps = a.eps;
  float* p = a.p[net];
  float* m1 = a.mom1[net];
  float* m2 = a.mom2[net];
  for (int e = lo + (int)threadIdx.x; e < hi; e += kThreads) {
    const double gd = (double)s[gr + e - lo];
    const double mi = __dadd_rn(__dmul_rn(b1, (double)s[mo + e - lo]), __dmul_rn(1.0 - b1, gd));
    const double vi = __dadd_rn(__dmul_rn(b2, (double)s[vo + e - lo]), __dmul_rn(__dmul_rn(1.0 - b2, gd), gd));
    m1[e] = (float)mi;
    m2[e] = (float)vi;
    const float pn = (float)__dsub_rn((double)s[p_smem + e],
                                      __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mi, c1)),
                                                __dadd_rn(__dsqrt_rn(__ddiv_rn(vi, c2)), eps)));
    p[e] = pn;
    s[p_smem + e] = pn;
  }
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

/// BCE on clamped sigmoid probabilities (loss.hpp:59-88) for one warp's
/// worth of rows (logits / grad rows padded to 8 floats): returns the
/// warp-summed loss; writes float((p - y) / n) * lambda.
__device__ __noinline__ double bce_rows(int logits, int grad, int n, int n_real, int nr, double n_div,
                                        float lambda) {
  float* s = S();
  const int i = threadIdx.x;  // < 32
  double lv = 0.0;
  if (i < n) {
    const int r = i < n_real ? i : i - n_real;
    const bool valid = r < nr;
    const double y = i < n_real ? 1.0 : 0.0;
    double pc = (double)stable_sigmoid(s[logits + 8 * i]);
    pc = pc < 1e-7 ? 1e-7 : (pc > 1.0 - 1e-7 ? 1.0 - 1e-7 : pc);
    lv = valid ? (y != 0.0 ? -log(pc) : -log(1.0 - pc)) : 0.0;
    s[grad + 8 * i] = valid ? (float)((pc - y) / n_div) * lambda : 0.0f;
  }
  return warp_sum_d(lv);
}

__global__ void __cluster_dims__(kC, 1, 1) __launch_bounds__(kThreads, 1)
    k_post_small(const __grid_constant__ StepArgs a, const __grid_constant__ Prog P) {
  __shared__ double s_loss[4];  // d, adv, cyc partial sums of this CTA
  __shared__ int s_ok[4];       // finite flags of this CTA's owned slices
  __shared__ long long s_ph[kMaxOps + 2];
  cg::cluster_group cl = cg::this_cluster();
  float* s = S();
  Counters* ctr = a.ctr;
  if (ctr->aborted) return;
  const ModelArgs& m = a.m;
  const int tid = threadIdx.x;
  const bool prof = a.phase_prof != 0;
  if (prof && tid == 0) s_ph[0] = clock64();
  const int rank = (int)cl.block_rank();
  const int rows = min(a.B, a.n_part - (int)ctr->step_in_epoch * a.B);
  const int per = (rows + kC - 1) / kC;
  const int r0 = min(rank * per, rows);
  const int nr = max(0, min(per, rows - r0));
  const int in = m.in, E1 = m.E1, D = m.D;
  const int nets3[3] = {kDisc, kFwd, kInv};
  int lo[3], hi[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    lo[q] = P.count[q] * rank / kC;
    hi[q] = P.count[q] * (rank + 1) / kC;
  }

  // ---- zeroed image, then one asynchronous staging pass ----
  {
    float4* z4 = reinterpret_cast<float4*>(s);
    for (int i = tid; i < P.total / 4; i += kThreads) z4[i] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const float* src = a.p[nets3[q]];
    for (int i = tid; i < P.count[q]; i += kThreads) cp4(P.blob[q] + i, src + i);
    for (int e = lo[q] + tid; e < hi[q]; e += kThreads) {
      cp4(P.mo[q] + e - lo[q], a.mom1[nets3[q]] + e);
      cp4(P.vo[q] + e - lo[q], a.mom2[nets3[q]] + e);
    }
  }
  for (int i = tid; i < P.et_count; i += kThreads) cp4(P.et_blob + i, a.p[kEnc] + m.enc_tail.base + i);
  for (int i = tid; i < P.dh_count; i += kThreads) cp4(P.dh_blob + i, a.p[kDec] + m.dec_head.base + i);
  for (int i = tid; i < E1; i += kThreads) cp4(P.be + i, a.p[kEnc] + m.enc_wide_b + i);
  {
    const float* red_enc = a.scratch + a.L.red_enc + (long long)r0 * E1;
    const float* red_dec = a.scratch + a.L.red_dec + (long long)r0 * D;
    const float* xb = a.xb + (long long)r0 * in;
    const int ldi = pad8(in), lde = pad8(E1), ldd = pad8(D);
    for (int i = tid; i < nr * in; i += kThreads) cp4(P.xs + (i / in) * ldi + i % in, xb + i);
    for (int i = tid; i < nr * E1; i += kThreads) cp4(P.e1 + (i / E1) * lde + i % E1, red_enc + i);
    for (int i = tid; i < nr * D; i += kThreads) cp4(P.gh + (i / D) * ldd + i % D, red_dec + i);
  }
  cp_wait_all();
  __syncthreads();
  {
    // enc layer-0 activation of this CTA's rows (pad rows: act(0 + b))
    const int lde = pad8(E1);
    for (int i = tid; i < kR * E1; i += kThreads) {
      const int oo = (i / E1) * lde + i % E1;
      s[P.e1 + oo] = act_apply(m.enc_act0, m.enc_slope0, s[P.e1 + oo] + s[P.be + i % E1]);
    }
    // dL/dh = (1/n) S Wd^T (loss.hpp:37-39; the 1/n scale folded after the sum)
    const float gscale = (float)(1.0 / ((double)rows * (double)m.out));
    for (int i = tid; i < kR * pad8(D); i += kThreads) s[P.gh + i] *= gscale;
  }
  __syncthreads();

  // ---- the program ----
  bool d_ok = true, g_ok = false;
  double d_loss = 0.0, g_total = 0, g_fwd = 0, g_adv = 0, g_cyc = 0;
  int fwd_applied = 0, inv_applied = 0;
  const unsigned long long t_disc = ctr->t[kDisc] + 1, t_fwd = ctr->t[kFwd] + 1, t_inv = ctr->t[kInv] + 1;
  for (int pc = 0; pc < P.n; ++pc) {
    const Op& o = P.op[pc];
    if (o.skip_unless_d && !d_ok) continue;
    switch (o.kind) {
      case kOpFwd: op_fwd(o); break;
      case kOpBwd: op_bwd(o); break;
      case kOpDz:  // OUT = padded width
        for (int i = tid; i < o.R * o.OUT; i += kThreads)
          s[o.p[5] + i] = s[o.p[0] + i] * act_d(o.p[3], __int_as_float(o.p[4]), s[o.p[1] + i], s[o.p[2] + i]);
        break;
      case kOpBce:
        if (tid < 32) {
          const double t = bce_rows(o.p[0], o.p[1], 2 * kR, kR, nr, 2.0 * (double)rows, 1.0f);
          if (tid == 0) s_loss[0] = t;
        }
        break;
      case kOpAdv:
        if (tid < 32) {
          const double t = bce_rows(o.p[0], o.p[1], kR, kR, nr, (double)rows, m.lambda_adv);
          if (tid == 0) s_loss[1] = t;
        }
        break;
      case kOpCyc:
        if (tid < 32) {
          // mae_loss (loss.hpp:24-41) value part and float(1/n)*sign, times lambda_cyc
          const float pos = (float)(1.0 / ((double)rows * (double)in)), neg = -pos;
          double part = 0.0;
          const int ldi = pad8(in);
          for (int i = tid; i < kR * in; i += 32) {
            const int r = i / in, oo = r * ldi + (i - r * in);
            const bool valid = r < nr;
            const double d = (double)s[o.p[0] + oo] - (double)s[o.p[1] + oo];
            if (valid) part += fabs(d);
            s[o.p[2] + oo] = valid ? (d > 0 ? pos : (d < 0 ? neg : 0.0f)) * m.lambda_cyc : 0.0f;
          }
          part = warp_sum_d(part);
          if (tid == 0) s_loss[2] = part;
        }
        break;
      case kOpArrive: cluster_arrive(); break;
      case kOpWait: cluster_wait(); break;
      case kOpDUpdate: {
        const int dok = reduce_owned(P.pg[0], lo[0], hi[0], P.gr[0]);
        if (tid == 0) s_ok[0] = dok;
        double d_sum = 0.0;
        for (int r = 0; r < kC; ++r) d_sum += cl.map_shared_rank(s_loss, r)[0];
        const double n2 = 2.0 * (double)rows;
        d_loss = ((double)rows * (d_sum / n2)) / (double)rows;
        cluster_sync();  // flags
        int all_ok = 1;
        for (int r = 0; r < kC; ++r) all_ok &= cl.map_shared_rank(s_ok, r)[0];
        d_ok = isfinite(d_loss) && all_ok;
        if (d_ok)
          adam_owned(a, kDisc, lo[0], hi[0], a.adam_c[2 * t_disc], a.adam_c[2 * t_disc + 1], P.blob[0], P.gr[0],
                     P.mo[0], P.vo[0]);
        cluster_sync();  // updated slices visible
        if (d_ok) {
          // pull the peers' slices of the updated disc blob over DSMEM
          const int count = P.count[0];
          for (int e = tid; e < count; e += kThreads) {
            int r = (int)(((long long)e * kC) / count);
            while (r + 1 < kC && (long long)count * (r + 1) / kC <= e) ++r;
            while (r > 0 && (long long)count * r / kC > e) --r;
            if (r != rank) s[P.blob[0] + e] = cl.map_shared_rank(s + P.blob[0], r)[e];
          }
        }
        break;
      }
      case kOpGUpdate: {
        cluster_sync();  // fwd / inv partials + adv / cyc sums
        const int fok = reduce_owned(P.pg[1], lo[1], hi[1], P.gr[1]);
        const int iok = reduce_owned(P.pg[2], lo[2], hi[2], P.gr[2]);
        if (tid == 0) {
          s_ok[1] = fok;
          s_ok[2] = iok;
        }
        double adv_sum = 0.0, cyc_sum = 0.0;
        for (int r = 0; r < kC; ++r) {
          adv_sum += cl.map_shared_rank(s_loss, r)[1];
          cyc_sum += cl.map_shared_rank(s_loss, r)[2];
        }
        cluster_sync();  // flags
        int all_f = 1, all_i = 1;
        for (int r = 0; r < kC; ++r) {
          all_f &= cl.map_shared_rank(s_ok, r)[1];
          all_i &= cl.map_shared_rank(s_ok, r)[2];
        }
        const long long n_fwd = (long long)rows * m.out;
        const long long n_cyc = (long long)rows * in;
        const double adv = adv_sum / (double)rows;
        const double cyc = cyc_sum / (double)n_cyc;
        const double fm = *a.mae_total / (double)n_fwd;
        const double total_raw = fm + (double)m.lambda_adv * adv + (double)m.lambda_cyc * cyc;
        g_total = ((double)rows * total_raw) / (double)rows;
        g_fwd = ((double)rows * fm) / (double)rows;
        g_adv = ((double)rows * adv) / (double)rows;
        g_cyc = ((double)rows * cyc) / (double)rows;
        // trainer.hpp:256-264: g_total, then fwd (throws before any change),
        // then inv (fwd already applied)
        if (isfinite(g_total) && all_f) {
          adam_owned(a, kFwd, lo[1], hi[1], a.adam_c[2 * t_fwd], a.adam_c[2 * t_fwd + 1], P.blob[1], P.gr[1],
                     P.mo[1], P.vo[1]);
          fwd_applied = 1;
          if (all_i) {
            adam_owned(a, kInv, lo[2], hi[2], a.adam_c[2 * t_inv], a.adam_c[2 * t_inv + 1], P.blob[2], P.gr[2],
                       P.mo[2], P.vo[2]);
            inv_applied = 1;
            g_ok = true;
          }
        }
        break;
      }
      default: break;
    }
    __syncthreads();
    if (prof && tid == 0) s_ph[pc + 1] = clock64();
  }
  cluster_sync();  // no CTA leaves while peers read its shared memory
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
    if (prof) {
      printf("post ops (kind:cycles):");
      for (int i = 0; i < P.n; ++i) printf(" %d:%lld", P.op[i].kind, s_ph[i + 1] - s_ph[i]);
      printf("\n");
    }
  }
}

// ------------------------------------------------------- host: program --
inline int up4(int v) { return (v + 3) & ~3; }
inline int hpad8(int v) { return (v + 7) & ~7; }

/// Shared-memory image of one network: blob and tape.
struct NetH {
  int L = 0, count = 0, blob = 0;
  int w[kMaxL + 1] = {};
  int act[kMaxL] = {};
  float slope[kMaxL] = {};
  int woff[kMaxL] = {}, boff[kMaxL] = {}, z[kMaxL] = {}, a[kMaxL] = {};
};

class Builder {
 public:
  Prog p{};
  int at = 0;
  int take(int n) {
    const int o = at;
    at += up4(n);
    return o;
  }
  NetH net(const NetDesc& d, int rows) {
    NetH n;
    n.L = d.L;
    n.count = (int)d.count;
    for (int i = 0; i <= d.L; ++i) n.w[i] = d.w[i];
    n.blob = take(n.count);
    for (int l = 0; l < d.L; ++l) {
      n.act[l] = d.act[l];
      n.slope[l] = d.slope[l];
      n.woff[l] = (int)(d.off_w[l] - d.base);
      n.boff[l] = (int)(d.off_b[l] - d.base);
      n.z[l] = take(rows * hpad8(d.w[l + 1]));
      n.a[l] = d.act[l] == kIdentity ? n.z[l] : take(rows * hpad8(d.w[l + 1]));
    }
    return n;
  }
  Op& push(int kind, bool skip, int R, int IN, int OUT) {
    if (p.n >= kMaxOps) throw std::runtime_error("post program too long");
    Op& o = p.op[p.n++];
    o = Op{};
    o.kind = kind;
    o.skip_unless_d = skip ? 1 : 0;
    o.R = R;
    o.IN = IN;
    o.OUT = OUT;
    for (int& v : o.p) v = -1;
    return o;
  }
  /// forward of every layer; the last layer's output goes to `out` (or its tape)
  void fwd(const NetH& n, int x, int R, int out, bool skip) {
    for (int l = 0; l < n.L; ++l) {
      Op& o = push(kOpFwd, skip, R, n.w[l], n.w[l + 1]);
      o.p[0] = l == 0 ? x : n.a[l - 1];
      o.p[1] = n.blob + n.woff[l];
      o.p[2] = n.blob + n.boff[l];
      o.p[3] = n.z[l];
      o.p[4] = (l + 1 == n.L && out >= 0) ? out : n.a[l];
      o.p[5] = n.act[l];
      o.p[6] = __builtin_bit_cast(int, n.slope[l]);
    }
  }
  /// backward from dz of the top layer ([R x OUT]); x = the net's input
  void bwd(const NetH& n, int dz, int x, int R, int pg, int gin0, int epiA, int epiB, int gA, int gB, bool skip) {
    int cur = dz;
    for (int l = n.L - 1; l >= 0; --l) {
      Op& o = push(kOpBwd, skip, R, n.w[l], n.w[l + 1]);
      o.p[0] = cur;
      o.p[1] = l == 0 ? x : n.a[l - 1];
      o.p[2] = n.blob + n.woff[l];
      if (pg >= 0) {
        o.p[3] = pg + n.woff[l];
        o.p[4] = pg + n.boff[l];
      }
      const int nxt = l > 0 ? (cur == gA ? gB : gA) : gin0;
      o.p[5] = nxt;
      if (l == 0) {
        o.p[6] = epiA;
        o.p[7] = epiB;
      }
      o.p[10] = 0;
      if (l > 0) {
        o.p[8] = n.z[l - 1];
        o.p[9] = n.a[l - 1];
        o.p[10] = n.act[l - 1];
        o.p[11] = __builtin_bit_cast(int, n.slope[l - 1]);
      }
      cur = nxt;
    }
  }
};

inline int max_width(const NetDesc& d) {
  int m = 0;
  for (int i = 0; i <= d.L; ++i) m = d.w[i] > m ? d.w[i] : m;
  return m;
}

inline Prog build_program(const ModelArgs& m) {
  Builder b;
  const NetH F = b.net(m.fwd, kR);
  const NetH I = b.net(m.inv, kR);
  const NetH C = b.net(m.disc, 2 * kR);
  const NetH ET = b.net(m.enc_tail, kR);
  const NetH DH = b.net(m.dec_head, kR);
  Prog& p = b.p;
  const NetH* tr[3] = {&C, &F, &I};
  for (int i = 0; i < 3; ++i) {
    p.blob[i] = tr[i]->blob;
    p.count[i] = tr[i]->count;
    p.pg[i] = b.take(tr[i]->count);
    const int sl = tr[i]->count / kC + 2;
    p.mo[i] = b.take(sl);
    p.vo[i] = b.take(sl);
    p.gr[i] = b.take(sl);
  }
  p.et_blob = ET.blob;
  p.et_count = ET.count;
  p.dh_blob = DH.blob;
  p.dh_count = DH.count;
  p.be = b.take(m.E1);
  p.one = b.take(1);
  // row buffers: [rows x pad8(width)], pad columns zero
  p.xs = b.take(kR * hpad8(m.in));
  p.e1 = b.take(kR * hpad8(m.E1));
  p.gh = b.take(kR * hpad8(m.D));
  p.stacked = b.take(2 * kR * hpad8(m.lat));
  p.gl_dec = b.take(kR * hpad8(m.lat));
  p.gl_inv = b.take(kR * hpad8(m.lat));
  p.gl = b.take(kR * hpad8(m.lat));
  const int gc = b.take(2 * kR * 8);
  const int gi = b.take(kR * hpad8(m.in));
  int gw = 2 * kR * hpad8(max_width(m.disc));
  for (const NetDesc* d : {&m.fwd, &m.inv, &m.dec_head}) gw = std::max(gw, kR * hpad8(max_width(*d)));
  gw = std::max(gw, kR * hpad8(m.D));
  const int gA = b.take(gw), gB = b.take(gw);
  const int latent = p.stacked + kR * hpad8(m.lat);
  // real latents (enc tail; with no tail the enc activation IS the latent),
  // fake latents fwd(x), dec-head tape
  if (ET.L > 0) b.fwd(ET, p.e1, kR, p.stacked, false);
  else p.e1 = p.stacked;
  b.fwd(F, p.xs, kR, latent, false);
  if (DH.L > 0) b.fwd(DH, latent, kR, -1, false);
  else p.gh = p.gl_dec;
  // D-step: disc on [real; fake]
  b.fwd(C, p.stacked, 2 * kR, -1, false);
  {
    Op& o = b.push(kOpBce, false, 2 * kR, 0, 0);
    o.p[0] = C.a[C.L - 1];
    o.p[1] = gc;
  }
  b.bwd(C, gc, p.stacked, 2 * kR, p.pg[0], -1, -1, -1, gA, gB, false);
  b.push(kOpArrive, false, 0, 0, 0);
  // independent of the D-step: dec path and the whole cycle path
  if (DH.L > 0) {
    const int L = DH.L - 1;
    Op& o = b.push(kOpDz, false, kR, 0, hpad8(DH.w[L + 1]));
    o.p[0] = p.gh;
    o.p[1] = DH.z[L];
    o.p[2] = DH.a[L];
    o.p[3] = DH.act[L];
    o.p[4] = __builtin_bit_cast(int, DH.slope[L]);
    o.p[5] = gA;
    b.bwd(DH, gA, latent, kR, -1, p.gl_dec, -1, -1, gA, gB, false);
  }
  b.fwd(I, latent, kR, -1, false);
  {
    Op& o = b.push(kOpCyc, false, kR, 0, 0);
    o.p[0] = I.a[I.L - 1];
    o.p[1] = p.xs;
    o.p[2] = gi;
  }
  b.bwd(I, gi, latent, kR, p.pg[2], p.gl_inv, -1, -1, gA, gB, false);
  b.push(kOpWait, false, 0, 0, 0);
  b.push(kOpDUpdate, false, 0, 0, 0);
  // G-step (only if the D-step applied)
  b.fwd(C, latent, kR, -1, true);
  {
    Op& o = b.push(kOpAdv, true, kR, 0, 0);
    o.p[0] = C.a[C.L - 1];
    o.p[1] = gc;
  }
  b.bwd(C, gc, latent, kR, -1, p.gl, p.gl_dec, p.gl_inv, gA, gB, true);
  b.bwd(F, p.gl, p.xs, kR, p.pg[1], -1, -1, -1, gA, gB, true);
  b.push(kOpGUpdate, true, 0, 0, 0);
  p.total = b.at;
  return p;
}

}  // namespace ps

namespace {
constexpr std::size_t kSmemCap = 220 * 1024;  // dynamic shared memory (static ~1 KB on top)
}

int post_tpl_kind(const StepArgs& a) {
  const ModelArgs& m = a.m;
  if (a.B > ps::kC * ps::kR) return 0;
  const NetDesc* nets[5] = {&m.fwd, &m.inv, &m.disc, &m.enc_tail, &m.dec_head};
  for (const NetDesc* n : nets) {
    if (n->L > ps::kMaxL) return 0;
    for (int i = 0; i <= n->L; ++i)
      if (n->L > 0 && n->w[i] > ps::kMaxW) return 0;
  }
  if (m.fwd.L < 1 || m.inv.L < 1 || m.disc.L < 1) return 0;
  if (m.E1 > ps::kMaxW || m.D > ps::kMaxW || m.lat > ps::kMaxW || m.in > ps::kMaxW) return 0;
  try {
    const ps::Prog p = ps::build_program(m);
    if ((std::size_t)p.total * sizeof(float) > kSmemCap) return 0;
  } catch (const std::exception&) {
    return 0;
  }
  return 1;
}

void launch_post_tpl(int kind, const StepArgs& a, cudaStream_t s) {
  (void)kind;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ps::k_post_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCap);
    attr = true;
  }
  static thread_local ps::Prog cache;
  static thread_local const void* cache_key = nullptr;
  static thread_local ModelArgs cache_m{};
  if (cache_key == nullptr || std::memcmp(&cache_m, &a.m, sizeof(ModelArgs)) != 0) {
    cache = ps::build_program(a.m);
    cache_m = a.m;
    cache_key = &cache;
  }
  ps::k_post_small<<<ps::kC, ps::kThreads, (std::size_t)cache.total * sizeof(float), s>>>(a, cache);
}

}  // namespace ltfb_dev
