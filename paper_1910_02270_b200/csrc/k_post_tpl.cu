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
// The step is a chain of ~30 dependent small layer products (16-32 rows,
// <= 64 wide), so it is bound by the latency of that chain, not by FLOPs or
// bytes. Earlier variants synchronised the whole CTA after every layer
// (~35 block barriers, 2-4 k cycles per layer). Here the chain is
// ROW-PARALLEL and WARP-LOCAL: warp w owns minibatch rows w, w+8, ... of its
// CTA and carries them through every forward layer and every input-gradient
// layer with only __syncwarp between layers (activations, dz and the input
// gradients of a row never leave its warp). The only block-wide phases are
// the weight-gradient products, which need all rows: one phase per network
// computes every layer's dW / db at once from the stored tapes and dz.
// Everything lives in shared memory (blob images, transposed weight copies
// for the input gradients, tapes), staged with one cp.async round trip.
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
#include "stream_sync.cuh"
#include "tc_ptx.cuh"

namespace cg = cooperative_groups;

namespace ltfb_dev {
namespace ps {

constexpr int kC = 8;          // CTAs per cluster
constexpr int kThreads = 256;  // 8 warps
constexpr int kWarps = kThreads / 32;
constexpr int kR = 16;         // minibatch rows per CTA (B <= 128)
constexpr int kMaxL = 4;
constexpr int kMaxW = 64;

/// A small network's shared-memory image. Offsets are float indices into the
/// dynamic shared array; tapes are [rows x w[l+1]] row-major.
struct NetS {
  int L, count;
  int w[kMaxL + 1];
  int act[kMaxL];
  float slope[kMaxL];
  int blob;                      // staged blob (W0,b0,W1,b1,...), W [in x out]
  int woff[kMaxL], boff[kMaxL];  // within the blob
  int T[kMaxL];                  // W^T [out x (in + 1)] (input gradients), contiguous from Tall
  int Tall, Tcount;              // the net's W^T region (same layout as StepArgs::pT)
  int z[kMaxL], a[kMaxL];        // forward tape
  int dz[kMaxL];                 // dL/dz per layer (weight gradients)
};

struct Layout {
  NetS net[5];  // kF, kI, kCd, kET, kDH
  int xs, e1, be, gh, stacked, gl_dec, gl_inv, gl, gd, gc, gi;
  int xn;  // x rows of the next step (next_h), prefetched in the prologue
  int pg[3];                // partial gradients disc, fwd, inv (blob layout)
  int mo[3], vo[3], gr[3];  // owner-slice moments / reduced gradients (then new parameters)
  int mt[3], vt[3];         // new moments of the owner slice (committed into mo / vo if applied)
  int total;
};
enum { kF = 0, kI = 1, kCd = 2, kET = 3, kDH = 4 };

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

// ------------------------------------------------ warp-local layer work --
// The calling warp owns rows w + 8 i (i < nrw) of the tape it works on.

// Each routine has one body with compile-time (IN, OUT, NRW) for the shapes
// of the default surrogate architecture (every loop fully unrolled, operand
// addresses immediate) and a runtime-shaped instance (all three 0) for any
// other width <= 64: same arithmetic, same k order, only the schedule differs.
// Measured: in the full kernel every routine runs once per step from a cold
// instruction cache, so the specialised copies (2x faster warm) lose to one
// compact runtime routine reused by every layer. Opt in with
// -DLTFB_POST_SPECIALIZE (for a resident / persistent variant). The runtime
// instances are inlined into the per-network loops (wnet_fwd / wnet_bwd): no
// call per layer (-2 us per step, A/B on one box).
#ifdef LTFB_POST_SPECIALIZE
#define LTFB_FWD_SHAPES(X) \
  X(64, 20, 2) X(5, 32, 2) X(32, 32, 2) X(32, 20, 2) X(20, 64, 2) X(20, 32, 2) X(32, 5, 2) X(32, 1, 2) \
  X(20, 32, 4) X(32, 32, 4) X(32, 1, 4)
#define LTFB_GIN_SHAPES(X) \
  X(32, 1, 4) X(32, 32, 4) X(20, 64, 2) X(32, 5, 2) X(32, 32, 2) X(20, 32, 2) X(32, 1, 2) X(32, 20, 2)
#else
#define LTFB_FWD_SHAPES(X)
#define LTFB_GIN_SHAPES(X)
#endif
constexpr int shape_key(int in, int out, int nrw) { return (in << 16) | (out << 4) | nrw; }

/// z = x W + b, a = act(z) for the warp's rows (nn/mlp.hpp:201-217:
/// matmul, add_row_vector, activation; each output one k-ordered fmaf
/// chain). Lanes are output neurons; x is read as a warp broadcast.
template <int IN_T, int OUT_T, int NRW_T>
__device__ __forceinline__ void wfwd_k(int x, int W, int b, int IN_rt, int OUT_rt, int z, int act,
                                    float slope, int out_a) {
  float* s = S();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr bool kCT = IN_T > 0;
  const int IN = kCT ? IN_T : IN_rt, OUT = kCT ? OUT_T : OUT_rt;
  constexpr int kRows = NRW_T;
#pragma unroll
  for (int j = lane; j < OUT; j += 32) {
    float acc[kRows];
#pragma unroll
    for (int i = 0; i < kRows; ++i) acc[i] = 0.0f;
    const float* w = s + W + j;
    const float* xr = s + x + warp * IN;
    if constexpr (kCT) {
#pragma unroll
      for (int k = 0; k < IN_T; ++k) {
        const float wv = w[k * OUT_T];
#pragma unroll
        for (int i = 0; i < kRows; ++i) acc[i] = fmaf(xr[8 * i * IN_T + k], wv, acc[i]);
      }
    } else if (((IN | x) & 3) == 0) {  // rows 16-B aligned: x read 4 k at a time (same k order)
#pragma unroll 4
      for (int k = 0; k < IN; k += 4) {
        const float w0 = w[k * OUT], w1 = w[(k + 1) * OUT], w2 = w[(k + 2) * OUT], w3 = w[(k + 3) * OUT];
#pragma unroll
        for (int i = 0; i < kRows; ++i) {
          const float4 xv = *reinterpret_cast<const float4*>(xr + 8 * i * IN + k);
          acc[i] = fmaf(xv.x, w0, acc[i]);
          acc[i] = fmaf(xv.y, w1, acc[i]);
          acc[i] = fmaf(xv.z, w2, acc[i]);
          acc[i] = fmaf(xv.w, w3, acc[i]);
        }
      }
    } else {
#pragma unroll 4
      for (int k = 0; k < IN; ++k) {
        const float wv = w[k * OUT];
#pragma unroll
        for (int i = 0; i < kRows; ++i) acc[i] = fmaf(xr[8 * i * IN + k], wv, acc[i]);
      }
    }
    const float bj = s[b + j];
#pragma unroll
    for (int i = 0; i < kRows; ++i) {
      const int o = (warp + 8 * i) * OUT + j;
      const float v = acc[i] + bj;
      s[z + o] = v;
      s[out_a + o] = act_f(act, slope, v);
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void wfwd(int x, const NetS& n, int l, int nrw, int out_a) {
  const int IN = n.w[l], OUT = n.w[l + 1], W = n.blob + n.woff[l], b = n.blob + n.boff[l];
  const int z = n.z[l], act = n.act[l];
  const float sl = n.slope[l];
  switch (shape_key(IN, OUT, nrw)) {
#define X(i, o, r)                                                   \
  case shape_key(i, o, r):                                           \
    wfwd_k<i, o, r>(x, W, b, IN, OUT, z, act, sl, out_a); \
    return;
    LTFB_FWD_SHAPES(X)
#undef X
    default:
      if (nrw == 4)
        wfwd_k<0, 0, 4>(x, W, b, IN, OUT, z, act, sl, out_a);
      else
        wfwd_k<0, 0, 2>(x, W, b, IN, OUT, z, act, sl, out_a);
  }
}

/// Input gradient of layer l for the warp's rows: v = sum_j dz[r][j] W[k][j]
/// (nn/mlp.hpp:278), then (epiA + v) + epiB if epiA >= 0 (grad_latent = dec
/// + disc + inv, train_ops.hpp:104-127), then * act'(z', a') of layer l-1 if
/// dact (the result is then that layer's dz). Lanes are input neurons.
template <int IN_T, int OUT_T, int NRW_T>
__device__ __forceinline__ void wgin_k(int dz, int WT, int IN_rt, int OUT_rt, int out, int epiA, int epiB,
                                    int zp, int ap, int actp, float slope, bool dact) {
  float* s = S();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr bool kCT = IN_T > 0;
  const int IN = kCT ? IN_T : IN_rt, OUT = kCT ? OUT_T : OUT_rt;
  constexpr int kRows = NRW_T;
  const int ldt = IN + 1;  // odd row pitch: conflict-free transposed writes and reads
#pragma unroll
  for (int k = lane; k < IN; k += 32) {
    float acc[kRows];
#pragma unroll
    for (int i = 0; i < kRows; ++i) acc[i] = 0.0f;
    const float* w = s + WT + k;
    const float* dr = s + dz + warp * OUT;
    if constexpr (kCT) {
#pragma unroll
      for (int j = 0; j < OUT_T; ++j) {
        const float wv = w[j * (IN_T + 1)];
#pragma unroll
        for (int i = 0; i < kRows; ++i) acc[i] = fmaf(dr[8 * i * OUT_T + j], wv, acc[i]);
      }
    } else if (((OUT | dz) & 3) == 0) {  // dz rows 16-B aligned: 4 j at a time (same j order)
#pragma unroll 4
      for (int j = 0; j < OUT; j += 4) {
        const float w0 = w[j * ldt], w1 = w[(j + 1) * ldt], w2 = w[(j + 2) * ldt], w3 = w[(j + 3) * ldt];
#pragma unroll
        for (int i = 0; i < kRows; ++i) {
          const float4 dv = *reinterpret_cast<const float4*>(dr + 8 * i * OUT + j);
          acc[i] = fmaf(dv.x, w0, acc[i]);
          acc[i] = fmaf(dv.y, w1, acc[i]);
          acc[i] = fmaf(dv.z, w2, acc[i]);
          acc[i] = fmaf(dv.w, w3, acc[i]);
        }
      }
    } else {
#pragma unroll 4
      for (int j = 0; j < OUT; ++j) {
        const float wv = w[j * ldt];
#pragma unroll
        for (int i = 0; i < kRows; ++i) acc[i] = fmaf(dr[8 * i * OUT + j], wv, acc[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < kRows; ++i) {
      const int o = (warp + 8 * i) * IN + k;
      float v = acc[i];
      if (epiA >= 0) v = (s[epiA + o] + v) + s[epiB + o];
      if (dact) v = v * act_d(actp, slope, s[zp + o], s[ap + o]);
      s[out + o] = v;
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void wgin(int dz, const NetS& n, int l, int nrw, int out, int epiA, int epiB, bool dact) {
  const int IN = n.w[l], OUT = n.w[l + 1], WT = n.T[l];
  const int zp = dact ? n.z[l - 1] : 0, ap = dact ? n.a[l - 1] : 0, actp = dact ? n.act[l - 1] : kIdentity;
  const float sl = dact ? n.slope[l - 1] : 0.0f;
  switch (shape_key(IN, OUT, nrw)) {
#define X(i, o, r)                                                                    \
  case shape_key(i, o, r):                                                            \
    wgin_k<i, o, r>(dz, WT, IN, OUT, out, epiA, epiB, zp, ap, actp, sl, dact); \
    return;
    LTFB_GIN_SHAPES(X)
#undef X
    default:
      if (nrw == 4)
        wgin_k<0, 0, 4>(dz, WT, IN, OUT, out, epiA, epiB, zp, ap, actp, sl, dact);
      else
        wgin_k<0, 0, 2>(dz, WT, IN, OUT, out, epiA, epiB, zp, ap, actp, sl, dact);
  }
}

/// Forward through every layer of n for the warp's rows; the last layer's
/// activation goes to `out` (or its tape if out < 0).
__device__ __noinline__ void wnet_fwd(const NetS& n, int x, int nrw, int out) {
  for (int l = 0; l < n.L; ++l)
    wfwd(l == 0 ? x : n.a[l - 1], n, l, nrw, (l + 1 == n.L && out >= 0) ? out : n.a[l]);
}

/// Input-gradient chain of n for the warp's rows from dz of the top layer
/// (which must already be in n.dz[L-1]); fills n.dz[l] for every layer and,
/// if gin0 >= 0, the net's input gradient (with the optional epilogue).
__device__ __noinline__ void wnet_bwd(const NetS& n, int nrw, int gin0, int epiA, int epiB) {
  for (int l = n.L - 1; l >= 1; --l) wgin(n.dz[l], n, l, nrw, n.dz[l - 1], -1, -1, true);
  if (gin0 >= 0) wgin(n.dz[0], n, 0, nrw, gin0, epiA, epiB, false);
}

// ------------------------------------------------------ block-wide work --
/// Weight / bias partial gradients of every layer of n over the CTA's R rows
/// (nn/mlp.hpp:274-277): pgW[k][j] = sum_r below[r][k] dz[r][j], pgb[j] =
/// sum_r dz[r][j], one pass over the item space of all layers. Row k == IN
/// of a layer is its bias (below == 1, fmaf(1, d, acc) == acc + d).
/// Layers with a 4-aligned input width: thread (k-group, j) owns the four
/// weight gradients dW[4 kg .. 4 kg + 3][j]; per row one float4 of the layer
/// input (a warp broadcast) and one dz feed 4 FMAs, rows ascending as in the
/// reference (nn/mlp.hpp:274-277). Bias gradients by the k-group past IN.
__device__ __forceinline__ void pg_layer4(const NetS& n, int l, int below, int R, int pg) {
  float* s = S();
  const int IN = n.w[l], OUT = n.w[l + 1];
  const int nkg = IN / 4 + 1;  // + the bias group
  const int items = nkg * OUT;
  const float* d0 = s + n.dz[l];
  const int pgW = pg + n.woff[l], pgb = pg + n.boff[l];
  for (int t = threadIdx.x; t < items; t += kThreads) {
    const int kg = t / OUT, j = t - kg * OUT;
    const float* d = d0 + j;
    if (kg < IN / 4) {
      const float4* b4 = reinterpret_cast<const float4*>(s + below) + kg;
      const int bstride = IN / 4;
      float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
#pragma unroll 4
      for (int r = 0; r < R; ++r) {
        const float dv = d[r * OUT];
        const float4 bv = b4[r * bstride];
        a0 = fmaf(bv.x, dv, a0);
        a1 = fmaf(bv.y, dv, a1);
        a2 = fmaf(bv.z, dv, a2);
        a3 = fmaf(bv.w, dv, a3);
      }
      float* dw = s + pgW + 4 * kg * OUT + j;
      dw[0] = a0;
      dw[OUT] = a1;
      dw[2 * OUT] = a2;
      dw[3 * OUT] = a3;
    } else {
      float a0 = 0.0f;
#pragma unroll 4
      for (int r = 0; r < R; ++r) a0 += d[r * OUT];
      s[pgb + j] = a0;
    }
  }
}

__device__ __noinline__ void pg_net(const NetS& n, int x, int R, int pg) {
  float* s = S();
  // per layer: the float4 path where the input width is a multiple of 4,
  // else the pairwise path (same per-element row order either way: outputs
  // are disjoint, so no barrier between layers)
  const int L = n.L;
  for (int l = 0; l < L; ++l) {
    const int IN = n.w[l], OUT = n.w[l + 1];
    const int below = l == 0 ? x : n.a[l - 1];
    if (IN % 4 == 0) {
      pg_layer4(n, l, below, R, pg);
      continue;
    }
    const int items = ((IN + 2) >> 1) * OUT;
    const float* dz = s + n.dz[l];
    const int pgW = pg + n.woff[l], pgb = pg + n.boff[l];
    for (int t = threadIdx.x; t < items; t += kThreads) {
      const int kp = t / OUT, j = t - kp * OUT;
      const int k0 = 2 * kp, k1 = k0 + 1;
      const float* d = dz + j;
      float a0 = 0.0f, a1 = 0.0f;
      if (k1 < IN) {
        const float* b0 = s + below + k0;
#pragma unroll 4
        for (int r = 0; r < R; ++r) {
          const float dv = d[r * OUT];
          a0 = fmaf(b0[r * IN], dv, a0);
          a1 = fmaf(b0[r * IN + 1], dv, a1);
        }
      } else if (k0 < IN) {  // k1 == IN: bias
        const float* b0 = s + below + k0;
#pragma unroll 4
        for (int r = 0; r < R; ++r) {
          const float dv = d[r * OUT];
          a0 = fmaf(b0[r * IN], dv, a0);
          a1 += dv;
        }
      } else {  // k0 == IN: bias only
#pragma unroll 4
        for (int r = 0; r < R; ++r) a0 += d[r * OUT];
      }
      s[k0 < IN ? pgW + k0 * OUT + j : pgb + j] = a0;
      if (k1 <= IN && k0 < IN) s[k1 < IN ? pgW + k1 * OUT + j : pgb + j] = a1;
    }
  }
}

/// W^T copies of every layer of n from its blob image.
__device__ __noinline__ void transpose_net(const NetS& n) {
  float* s = S();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int l = 0; l < n.L; ++l) {
    const int in = n.w[l], out = n.w[l + 1], W = n.blob + n.woff[l], T = n.T[l];
    for (int k = warp; k < in; k += kWarps)
      for (int j = lane; j < out; j += 32) s[T + j * (in + 1) + k] = s[W + k * out + j];
  }
}

/// Owner reduction of [lo, hi) over the kC partials at smem offset pg, in
/// rank order, into gr; returns this CTA's "all finite" (block-uniform).
__device__ __noinline__ int reduce_owned(int pg, int lo, int hi, int gr, int base = 0) {
  cg::cluster_group cl = cg::this_cluster();
  float* s = S();
  int ok = 1;
  for (int e = lo + (int)threadIdx.x; e < hi; e += kThreads) {
    float v[kC];
#pragma unroll
    for (int r = 0; r < kC; ++r) v[r] = cl.map_shared_rank(s + pg, base + r)[e];
    float acc = 0.0f;
#pragma unroll
    for (int r = 0; r < kC; ++r) acc += v[r];
    s[gr + e - lo] = acc;
    ok &= isfinite(acc) ? 1 : 0;
  }
  return __syncthreads_and(ok);
}

/// nn/adam.hpp:48-61 in double with explicit round-to-nearest operations
/// (no FMA contraction): bit-identical to the reference's scalar loop. The
/// owner writes the new parameter to HBM (p and, for weights, the W^T copy
/// pT the next step stages) and, if push, into the blob image and W^T image
/// of every CTA of the cluster (DSMEM stores; visible after the next cluster
/// barrier), so no CTA has to pull or re-transpose the updated network.
/// First half of the owner's Adam step, issued before the cluster learns
/// whether every gradient is finite (so the f64 chain overlaps the barrier):
/// m, v and the new parameter of each owned element are computed in place
/// of the slice's moment and gradient images. Nothing global changes here.
__device__ __noinline__ void adam_compute(const StepArgs& a, int net, const NetS& n, int lo, int hi, double c1,
                                          double c2, int gr, int mo, int vo, int mt, int vt) {
  float* s = S();
  const double lr = a.lr[net], b1 = a.b1, b2 = a.b2, eps = a.eps;
  for (int e = lo + (int)threadIdx.x; e < hi; e += kThreads) {
    float m = s[mo + e - lo], v = s[vo + e - lo];
    s[gr + e - lo] = adam_elem(s[n.blob + e], m, v, s[gr + e - lo], lr, b1, b2, eps, c1, c2);
    s[mt + e - lo] = m;
    s[vt + e - lo] = v;
  }
}

/// Second half (the step is applied): the owner writes m, v, p and, for
/// weights, the W^T copy pT to HBM (the images the next step stages) and, if
/// push, the new value into the blob image and W^T image of every CTA of its
/// half (DSMEM stores; visible after the next cluster barrier), so no CTA
/// has to pull or re-transpose the updated network.
__device__ __noinline__ void adam_commit(const StepArgs& a, int net, const NetS& n, int lo, int hi, int gr, int mo,
                                         int vo, int mt, int vt, int push /* 1 blob, 2 blob + W^T */,
                                         int rbase = 0, int rcount = kC, bool globals = true) {
  cg::cluster_group cl = cg::this_cluster();
  float* s = S();
  float* p = a.p[net];
  float* pT = a.pT[net];
  float* m1 = a.mom1[net];
  float* m2 = a.mom2[net];
  for (int e = lo + (int)threadIdx.x; e < hi; e += kThreads) {
    const float pn = s[gr + e - lo];
    const float mn = s[mt + e - lo], vn = s[vt + e - lo];
    s[mo + e - lo] = mn;  // the owner slice's moments stay resident (streamed step)
    s[vo + e - lo] = vn;
    if (globals) {
      m1[e] = mn;
      m2[e] = vn;
      p[e] = pn;
    } else if (!push) {
      continue;  // nothing else to write
    }
    int t = -1;  // W^T position of a weight element (biases have none)
    for (int l = 0; l < n.L; ++l) {
      const int in = n.w[l], out = n.w[l + 1], q = e - n.woff[l];
      if (q >= 0 && q < in * out) {
        const int k = q / out, j = q - k * out;
        t = n.T[l] + j * (in + 1) + k;
      }
    }
    if (globals && t >= 0) pT[t - n.Tall] = pn;
    if (push) {
      for (int r = rbase; r < rbase + rcount; ++r) {
        float* peer = cl.map_shared_rank(s, r);
        peer[n.blob + e] = pn;
        if (push == 2 && t >= 0) peer[t] = pn;
      }
    }
  }
}

/// The streamed step defers the global p / m / v / W^T writes of the D/G
/// half's commits (disc, fwd) to the end of the run: the owner slice of `net`
/// from this CTA's resident images (blob, moment images), written once.
__device__ __noinline__ void commit_globals(const StepArgs& a, int net, const NetS& n, int lo, int hi, int mo,
                                            int vo) {
  const float* s = S();
  float* p = a.p[net];
  float* pT = a.pT[net];
  for (int e = lo + (int)threadIdx.x; e < hi; e += kThreads) {
    const float pn = s[n.blob + e];
    a.mom1[net][e] = s[mo + e - lo];
    a.mom2[net][e] = s[vo + e - lo];
    p[e] = pn;
    for (int l = 0; l < n.L; ++l) {
      const int in = n.w[l], out = n.w[l + 1], q = e - n.woff[l];
      if (q >= 0 && q < in * out) {
        const int k = q / out, j = q - k * out;
        pT[n.T[l] - n.Tall + j * (in + 1) + k] = pn;
      }
    }
  }
}

__device__ __forceinline__ double clamp_prob(float logit) {
  double pc = (double)stable_sigmoid(logit);
  return pc < 1e-7 ? 1e-7 : (pc > 1.0 - 1e-7 ? 1.0 - 1e-7 : pc);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

/// Fixed-order sum of the per-warp values (block-uniform after the barrier).
__device__ __forceinline__ double sum_warps(const double* w) {
  double t = 0.0;
  for (int i = 0; i < kWarps; ++i) t += w[i];
  return t;
}

// ------------------------------------------------------- shared layout --
inline int up4(int v) { return (v + 3) & ~3; }

inline int max_width(const NetDesc& d) {
  int m = 0;
  for (int i = 0; i <= d.L; ++i) m = d.w[i] > m ? d.w[i] : m;
  return m;
}

inline Layout make_layout(const ModelArgs& m) {
  Layout y{};
  int at = 0;
  auto take = [&](int n) {
    const int o = at;
    at += up4(n);
    return o;
  };
  const NetDesc* d5[5] = {&m.fwd, &m.inv, &m.disc, &m.enc_tail, &m.dec_head};
  const int rows5[5] = {kR, kR, 2 * kR, kR, kR};
  const bool bwd5[5] = {true, true, true, false, true};
  for (int q = 0; q < 5; ++q) {
    const NetDesc& d = *d5[q];
    NetS& n = y.net[q];
    n.L = d.L;
    n.count = (int)d.count;
    for (int i = 0; i <= kMaxL; ++i) n.w[i] = i <= d.L ? d.w[i] : 0;
    n.blob = take(n.count);
    n.Tcount = 0;
    if (bwd5[q])
      for (int l = 0; l < d.L; ++l) n.Tcount += (d.w[l] + 1) * d.w[l + 1];
    n.Tall = take(n.Tcount);
    int tat = n.Tall;
    for (int l = 0; l < kMaxL; ++l) {
      n.act[l] = l < d.L ? d.act[l] : kIdentity;
      n.slope[l] = l < d.L ? d.slope[l] : 0.0f;
      n.woff[l] = l < d.L ? (int)(d.off_w[l] - d.base) : 0;
      n.boff[l] = l < d.L ? (int)(d.off_b[l] - d.base) : 0;
      n.T[l] = n.z[l] = n.a[l] = n.dz[l] = 0;
      if (l >= d.L) continue;
      const int sz = rows5[q] * d.w[l + 1];
      if (bwd5[q]) {  // W^T, row pitch in + 1
        n.T[l] = tat;
        tat += (d.w[l] + 1) * d.w[l + 1];
      }
      n.z[l] = take(sz);
      n.a[l] = n.act[l] == kIdentity ? n.z[l] : take(sz);
      if (bwd5[q]) n.dz[l] = take(sz);
    }
  }
  const NetDesc* tr[3] = {&m.disc, &m.fwd, &m.inv};
  for (int i = 0; i < 3; ++i) {
    y.pg[i] = take((int)tr[i]->count);
    const int sl = (int)tr[i]->count / kC + 8;
    y.mo[i] = take(sl);
    y.vo[i] = take(sl);
    y.gr[i] = take(sl);
    y.mt[i] = take(sl);
    y.vt[i] = take(sl);
  }
  y.be = take(m.E1);
  y.xs = take(kR * m.in);
  y.xn = take(kR * m.in);
  y.e1 = take(kR * m.E1);
  y.gh = take(kR * m.D);
  y.stacked = take(2 * kR * m.lat);
  y.gl_dec = take(kR * m.lat);
  y.gl_inv = take(kR * m.lat);
  y.gl = take(kR * m.lat);
  y.gd = take(kR * m.lat);
  y.gc = take(2 * kR);
  y.gi = take(kR * m.in);
  y.total = at;
  return y;
}


// Cold, once-per-launch parts of the step live in out-of-line functions so
// that the straight-line kernel body stays short and the hot layer routines
// (wfwd / wgin / pg_net) remain resident in the instruction cache.

// debug: fine-grained stamps inside the update phases (LTFB_PHASE_PROF)
__shared__ long long g_st[16];
__shared__ int g_nst;
// 1 in the streamed step's persistent cluster (k_post_loop): parameters and
// the owners' Adam moments stay resident in shared memory across steps
__shared__ int g_persist;
// LTFB_STREAM_PROF: this step's stamp row (cluster rank 0 only), else null
__shared__ unsigned long long* g_pb;
#define GSTAMP(slot) do { if (g_persist && g_pb && threadIdx.x == 0) g_pb[slot] = gtimer(); } while (0)
#define ST()                                                   \
  do {                                                         \
    if (threadIdx.x == 0 && g_nst < 16) g_st[g_nst++] = clock64(); \
  } while (0)

// step constants fetched once in the prologue (their global loads overlap
// the staging copies): Adam bias corrections 1-b1^t, 1-b2^t for the next t of
// disc / fwd / inv, and the wide pass's forward-MAE sum
__shared__ __align__(16) double g_pre[8];  // 16-B aligned: filled by 16-B cp.async

struct Rows {
  int rank, rows, r0, nr;  // rank within the half (row block / owner slice index)
  int lo[3], hi[3];
  int split;               // 1: two halves (16-CTA cluster), the cycle path in the second
};

/// First element of rank r's owner slice of a count-element blob: the even
/// split rounded down to a multiple of 4, so every slice starts 16 B aligned
/// (bulk copies) and the slices tile [0, count).
__host__ __device__ __forceinline__ int owner_lo(int count, int r) {
  return r <= 0 ? 0 : (r >= kC ? count : ((count * r / kC) & ~3));
}

/// Streamed step: the new parameters of net n (adam_compute left them in
/// every owner's gr slice) into this CTA's blob image and, if wT, its W^T
/// image: DSMEM loads from the kC owners at cluster ranks rbase .. rbase+kC-1.
/// Valid from the owners' flag barrier (S5 / S2) until their next
/// adam_compute, which the cluster reaches only after the next S1.
__device__ __noinline__ void pull_net(const NetS& n, int gr, int rbase, bool wT) {
  cg::cluster_group cl = cg::this_cluster();
  float* s = S();
  const int count = n.count;
  int olo[kC + 1];
#pragma unroll
  for (int r = 0; r <= kC; ++r) olo[r] = owner_lo(count, r);
  // kPer elements per thread and round: every remote load of the round is
  // issued before any value is stored (one DSMEM round trip per round)
  constexpr int kPer = 8;
  for (int base = 0; base < count; base += kThreads * kPer) {
    float v[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = base + u * kThreads + (int)threadIdx.x;
      v[u] = 0.0f;
      if (e < count) {
        int r = 0;
#pragma unroll
        for (int q = 1; q < kC; ++q) r += e >= olo[q] ? 1 : 0;
        v[u] = *cl.map_shared_rank(s + gr + (e - olo[r]), rbase + r);
      }
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = base + u * kThreads + (int)threadIdx.x;
      if (e >= count) continue;
      s[n.blob + e] = v[u];
      if (wT)
        for (int l = 0; l < n.L; ++l) {
          const int in = n.w[l], out = n.w[l + 1], q = e - n.woff[l];
          if (q >= 0 && q < in * out) {
            const int k = q / out, jj = q - k * out;
            s[n.T[l] + jj * (in + 1) + k] = v[u];
          }
        }
    }
  }
}

/// Streamed step: this owner's new parameters [lo, hi) (adam_compute left
/// them in its gr slice) into the net's global staging copy, which every CTA
/// refreshes from once the step's decision is known (no extra barrier: the
/// copy is written before the cluster barrier that publishes the decision).
__device__ __forceinline__ void stage_new_params(float* dst, int gr, int lo, int hi) {
  const float* s = S();
  for (int e = lo + (int)threadIdx.x; e < hi; e += kThreads) dst[e] = s[gr + e - lo];
}

/// Streamed step: net n's new parameters from global memory (the owners'
/// adam_commit wrote them before the cluster barrier that precedes this
/// call) into this CTA's blob image (and W^T image if wT).
__device__ __noinline__ void refresh_net(const NetS& n, const float* p, bool wT) {
  float* s = S();
  const int count = n.count;
  constexpr int kPer = 8;
  for (int base = 0; base < count; base += kThreads * kPer) {
    float v[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = base + u * kThreads + (int)threadIdx.x;
      v[u] = e < count ? __ldcg(p + e) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = base + u * kThreads + (int)threadIdx.x;
      if (e >= count) continue;
      s[n.blob + e] = v[u];
      if (wT)
        for (int l = 0; l < n.L; ++l) {
          const int in = n.w[l], out = n.w[l + 1], q = e - n.woff[l];
          if (q >= 0 && q < in * out) {
            const int k = q / out, jj = q - k * out;
            s[n.T[l] + jj * (in + 1) + k] = v[u];
          }
        }
    }
  }
}

/// A host->smem staging job: n floats from src to smem offset dst.
struct Job {
  int dst, n;
  const float* src;
};

/// Splits a job into a 16 B-aligned body moved by one bulk copy (TMA engine)
/// and <= 3 + 3 unaligned edge floats moved by ordinary loads.
__device__ __forceinline__ void job_split(const Job& j, int& head, int& body) {
  const unsigned mis = (unsigned)(reinterpret_cast<uintptr_t>(j.src) & 15u) >> 2;  // floats past alignment
  head = (int)((4u - mis) & 3u);
  if (head > j.n) head = j.n;
  body = ((j.dst + head) & 3) == 0 ? ((j.n - head) & ~3) : 0;
  if (body == 0) head = j.n;  // relatively misaligned: all by loads
}

/// Staging job q of this CTA (0 <= q < kJobs; n == 0 if absent).
constexpr int kJobs = 19;
__device__ __noinline__ Job make_job(int q, const StepArgs& a, const Layout& Y, const Rows& R) {
  const ModelArgs& m = a.m;
  switch (q) {
    case 0: return {Y.net[kF].blob, Y.net[kF].count, a.p[kFwd]};
    case 1: return {Y.net[kI].blob, Y.net[kI].count, a.p[kInv]};
    case 2: return {Y.net[kCd].blob, Y.net[kCd].count, a.p[kDisc]};
    case 3: return {Y.net[kET].blob, Y.net[kET].count, a.p[kEnc] + m.enc_tail.base};
    case 4: return {Y.net[kDH].blob, Y.net[kDH].count, a.p[kDec] + m.dec_head.base};
    case 5: return {Y.net[kF].Tall, Y.net[kF].Tcount, a.pT[kFwd]};
    case 6: return {Y.net[kI].Tall, Y.net[kI].Tcount, a.pT[kInv]};
    case 7: return {Y.net[kCd].Tall, Y.net[kCd].Tcount, a.pT[kDisc]};
    case 8: return {Y.net[kDH].Tall, Y.net[kDH].Tcount, a.pT[kDec]};
    case 9: return {Y.mo[0], R.hi[0] - R.lo[0], a.mom1[kDisc] + R.lo[0]};
    case 10: return {Y.vo[0], R.hi[0] - R.lo[0], a.mom2[kDisc] + R.lo[0]};
    case 11: return {Y.mo[1], R.hi[1] - R.lo[1], a.mom1[kFwd] + R.lo[1]};
    case 12: return {Y.vo[1], R.hi[1] - R.lo[1], a.mom2[kFwd] + R.lo[1]};
    case 13: return {Y.mo[2], R.hi[2] - R.lo[2], a.mom1[kInv] + R.lo[2]};
    case 14: return {Y.vo[2], R.hi[2] - R.lo[2], a.mom2[kInv] + R.lo[2]};
    case 15: return {Y.be, m.E1, a.p[kEnc] + m.enc_wide_b};
    case 16: return {Y.xs, R.nr * m.in, a.xb + (long long)R.r0 * m.in};
    case 17: return {Y.e1, R.nr * m.E1, a.scratch + a.L.red_enc + (long long)R.r0 * m.E1};
    default: return {Y.gh, R.nr * m.D, a.scratch + a.L.red_dec + (long long)R.r0 * m.D};
  }
}

/// One staging pass: the five blob images, the four W^T images, the owner
/// slices of the three Adam moments and this CTA's rows of x / red_enc /
/// red_dec. Job q belongs to one thread (spread over the warps): it adds its
/// bytes to the mbarrier's transaction count, issues one bulk copy (TMA
/// engine) for the 16 B-aligned body and loads the <= 6 unaligned edge
/// floats itself. Then the row transforms.
__device__ __noinline__ void prologue(const StepArgs& a, const Layout& Y, const Rows& R, uint64_t* bar,
                                      int persist = 0) {
  float* s = S();
  const ModelArgs& m = a.m;
  const int tid = threadIdx.x;
  const int in = m.in, E1 = m.E1, D = m.D;
  const int q = (tid & 31) * kWarps + (tid >> 5);  // job of this thread: warps take turns
  // split mode: each half stages only what it reads (the D/G half: no inv
  // blob / W^T / moments, no dec-head W^T, no dL/dh rows -- it takes gl_dec
  // from its partner; the cyc half: no disc, enc tail, fwd W^T, disc / fwd
  // moments or enc rows); ~1/3 fewer bytes through each SM's copy engine
  const int half = R.split ? (int)(cg::this_cluster().block_rank() / kC) : -1;
  constexpr unsigned kSkipDG = (1u << 1) | (1u << 6) | (1u << 8) | (1u << 13) | (1u << 14) | (1u << 18);
  constexpr unsigned kSkipCyc = (1u << 2) | (1u << 3) | (1u << 5) | (1u << 7) | (1u << 9) | (1u << 10) |
                                (1u << 11) | (1u << 12) | (1u << 15) | (1u << 17);
  // streamed step: the reduced wide-pass rows arrive per step (stage_enc_rows / stage_dec_rows)
  const unsigned skip = (half == 0 ? kSkipDG : (half == 1 ? kSkipCyc : 0u)) | (persist ? (1u << 17) | (1u << 18) : 0u);
  if (q < kJobs && !((skip >> q) & 1u)) {
    const Job j = make_job(q, a, Y, R);
    if (j.n > 0 && j.src != nullptr) {
      int h, b;
      job_split(j, h, b);
      if (b > 0) {
        asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(tc::smem_u32(bar)),
                     "r"(4 * b)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                tc::smem_u32(s + j.dst + h)),
            "l"(j.src + h), "r"(4 * b), "r"(tc::smem_u32(bar))
            : "memory");
      }
      for (int e = 0; e < j.n - b; ++e) {  // unaligned edges
        const int o = e < h ? e : e + b;
        s[j.dst + o] = j.src[o];
      }
    }
  }
  // Loads needed only much later go out as cp.async (no stall here): the
  // Adam bias corrections and the MAE total (awaited in d_update), the next
  // step's x rows (awaited in next_h). Only the index loads block.
  if (persist) {
    // per-step constants, next rows and row transforms: the streamed loop
  } else if (tid < 3) {
    const int net = tid == 0 ? kDisc : (tid == 1 ? kFwd : kInv);
    const unsigned long long t = a.ctr->t[net] + 1;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(tc::smem_u32(&g_pre[2 * tid])),
                 "l"(a.adam_c + 2 * t)
                 : "memory");
  } else if (tid == 3) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(tc::smem_u32(&g_pre[6])), "l"(a.mae_total)
                 : "memory");
  }
  if (a.post_next_h && !persist) {  // x rows of the next step of this epoch (used by next_h)
    const int nxt = (int)a.ctr->step_in_epoch + 1;
    if ((long long)nxt * a.B < (long long)a.n_part) {
      const int rows = min(a.B, a.n_part - nxt * a.B);
      const int per = (rows + kC - 1) / kC;
      const int r0 = min(R.rank * per, rows), nr = max(0, min(per, rows - r0));
      const unsigned* perm = a.perm[a.ctr->epoch & 1u] + (long long)nxt * a.B + r0;
      for (int i = tid; i < kR * in; i += kThreads) {
        const int r = i / in, k = i - r * in;
        if (r < nr)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tc::smem_u32(s + Y.xn + i)),
                       "l"(a.sx + (long long)perm[r] * in + k)
                       : "memory");
        else
          s[Y.xn + i] = 0.0f;
      }
    }
  }
  for (int i = tid; i < (kR - R.nr) * in; i += kThreads) s[Y.xs + R.nr * in + i] = 0.0f;  // pad rows
  for (int i = tid; i < (kR - R.nr) * E1; i += kThreads) s[Y.e1 + R.nr * E1 + i] = 0.0f;
  for (int i = tid; i < (kR - R.nr) * D; i += kThreads) s[Y.gh + R.nr * D + i] = 0.0f;
  __syncthreads();
  if (tid == 0) tc::mbar_arrive(bar);
  tc::mbar_wait(bar, 0);
  __syncthreads();
  if (persist) return;
  {
    // enc layer-0 activation of this CTA's rows (pad rows: act(0 + b))
    const int e1 = Y.net[kET].L > 0 ? Y.e1 : Y.stacked;
    for (int i = tid; i < kR * E1; i += kThreads) {
      const int c = i - (i / E1) * E1;
      s[e1 + i] = act_f(m.enc_act0, m.enc_slope0, s[Y.e1 + i] + s[Y.be + c]);
    }
    // dL/dh = (1/n) S Wd^T (loss.hpp:37-39; the 1/n scale folded after the sum)
    const float gscale = (float)(1.0 / ((double)R.rows * (double)m.out));
    const int gh = Y.net[kDH].L > 0 ? Y.gh : Y.gl_dec;
    for (int i = tid; i < kR * D; i += kThreads) s[gh + i] = s[Y.gh + i] * gscale;
  }
  __syncthreads();
}

/// BCE (loss.hpp:59-88) for the calling warp: n_w rows r = warp + 8 lane
/// (lane < n_w); rows r < n_real are real (label 1). Writes the logit
/// gradient float((p - y) / n_div) * lambda to grad[r] and returns the warp's
/// loss sum (float log of the clamped probability, |rel err| ~ 1e-7).
__device__ __noinline__ double bce_warp(int logits, int grad, int n_w, int n_real, int nr, double n_div,
                                        float lambda) {
  float* s = S();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double lv = 0.0;
  if (lane < n_w) {
    const int r = warp + 8 * lane;
    const bool real = r < n_real;
    const bool valid = (real ? r : r - n_real) < nr;
    const double y = real ? 1.0 : 0.0;
    const double pc = clamp_prob(s[logits + r]);
    lv = valid ? -(double)logf((float)(real ? pc : 1.0 - pc)) : 0.0;
    s[grad + r] = valid ? (float)((pc - y) / n_div) * lambda : 0.0f;
  }
  return warp_sum_d(lv);
}

/// Cycle MAE (loss.hpp:24-41) on the warp's rows, times lambda_cyc: the
/// gradient float(1/n) * sign into grad, the warp's |d| sum returned.
__device__ __noinline__ double cyc_warp(int rec, int xs, int grad, int in, int nr, int rows, float lambda_cyc) {
  float* s = S();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float pos = (float)(1.0 / ((double)rows * (double)in)), neg = -pos;
  double part = 0.0;
  for (int i = 0; i < 2; ++i)
    for (int k = lane; k < in; k += 32) {
      const int r = warp + 8 * i, o = r * in + k;
      const bool valid = r < nr;
      const double d = (double)s[rec + o] - (double)s[xs + o];
      if (valid) part += fabs(d);
      s[grad + o] = valid ? (d > 0 ? pos : (d < 0 ? neg : 0.0f)) * lambda_cyc : 0.0f;
    }
  return warp_sum_d(part);
}

/// out = g * act'(z, a) of layer l for the warp's two rows (width w).
__device__ __noinline__ void dz_warp(int g, const NetS& n, int l, int out) {
  float* s = S();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int w = n.w[l + 1];
  for (int i = 0; i < 2; ++i)
    for (int j = lane; j < w; j += 32) {
      const int o = (warp + 8 * i) * w + j;
      s[out + o] = s[g + o] * act_d(n.act[l], n.slope[l], s[n.z[l] + o], s[n.a[l] + o]);
    }
  __syncwarp();
}

/// Field f of a per-CTA shared array from cluster ranks base .. base+kC-1:
/// every remote load issued before any is used (one DSMEM round trip, not
/// kC dependent ones); callers then combine v[0..kC) in rank order.
template <typename T>
__device__ __forceinline__ void from_ranks(T* arr, int f, int base, T (&v)[kC]) {
  cg::cluster_group cl = cg::this_cluster();
#pragma unroll
  for (int r = 0; r < kC; ++r) v[r] = cl.map_shared_rank(arr, base + r)[f];
}

/// Disc update: owner reduction, finite check (adam.hpp:95-102), Adam, and
/// the DSMEM pull of the peers' updated slices + W^T rebuild. Returns d_ok;
/// *d_loss gets the D-step loss (weighted mean of one shard).
__device__ __noinline__ bool d_update(const StepArgs& a, const Layout& Y, const Rows& R, double* s_loss, int* s_ok,
                                      double* d_loss) {
  cg::cluster_group cl = cg::this_cluster();
  float* s = S();
  const int tid = threadIdx.x;
  ST();
  cp_wait_all();  // g_pre (prologue cp.async); reduce_owned's barrier publishes it
  const int dok = reduce_owned(Y.pg[0], R.lo[0], R.hi[0], Y.gr[0]);
  ST();
  if (tid == 0) s_ok[0] = dok;
  const NetS& C = Y.net[kCd];
  adam_compute(a, kDisc, C, R.lo[0], R.hi[0], g_pre[0], g_pre[1], Y.gr[0], Y.mo[0], Y.vo[0], Y.mt[0], Y.vt[0]);
  double d_sum = 0.0;
  {
    double v[kC];
    from_ranks(s_loss, 0, 0, v);
    for (int r = 0; r < kC; ++r) d_sum += v[r];
  }
  cluster_arrive();  // S2: flags (arrive; the loss below overlaps the other CTAs' arrivals)
  const double n2 = 2.0 * (double)R.rows;
  *d_loss = ((double)R.rows * (d_sum / n2)) / (double)R.rows;
  cluster_wait();  // S2
  ST();
  int all_ok = 1;
  {
    int v[kC];
    from_ranks(s_ok, 0, 0, v);
    for (int r = 0; r < kC; ++r) all_ok &= v[r];
  }
  const bool d_ok = isfinite(*d_loss) && all_ok;
  if (d_ok)
    adam_commit(a, kDisc, C, R.lo[0], R.hi[0], Y.gr[0], Y.mo[0], Y.vo[0], Y.mt[0], Y.vt[0], 2, 0, kC, !g_persist);
  ST();
  cluster_sync();  // S3: every owner's updated disc slice (blob + W^T) pushed into every CTA
  return d_ok;
}

/// Generator update (trainer.hpp:231-272): reductions of the fwd / inv
/// partials, loss combination, finite checks and Adam(fwd) then Adam(inv).
__device__ __noinline__ void g_update(const StepArgs& a, const Layout& Y, const Rows& R, double* s_loss, int* s_ok,
                                      double* out /* g_total, g_fwd, g_adv, g_cyc, fwd_applied, inv_applied */) {
  cg::cluster_group cl = cg::this_cluster();
  const ModelArgs& m = a.m;
  const int tid = threadIdx.x;
  ST();
  GSTAMP(29);
  cluster_sync();  // S4: fwd / inv partials + adv / cyc sums
  GSTAMP(30);
  ST();
  // split mode: the inv partials, their reduction and the cycle losses live
  // in the cyc half (ranks kC .. 2kC-1), which also applies Adam(inv)
  const int cb = R.split ? kC : 0;
  const int fok = reduce_owned(Y.pg[1], R.lo[1], R.hi[1], Y.gr[1]);
  const int iok = R.split ? 1 : reduce_owned(Y.pg[2], R.lo[2], R.hi[2], Y.gr[2]);
  adam_compute(a, kFwd, Y.net[kF], R.lo[1], R.hi[1], g_pre[2], g_pre[3], Y.gr[1], Y.mo[1], Y.vo[1], Y.mt[1],
               Y.vt[1]);
  if (g_persist) stage_new_params(a.g[kFwd], Y.gr[1], R.lo[1], R.hi[1]);  // published by S5
  if (!R.split)
    adam_compute(a, kInv, Y.net[kI], R.lo[2], R.hi[2], g_pre[4], g_pre[5], Y.gr[2], Y.mo[2], Y.vo[2], Y.mt[2],
                 Y.vt[2]);
  ST();
  GSTAMP(31);
  if (tid == 0) {
    s_ok[1] = fok;
    if (!R.split) s_ok[2] = iok;
  }
  double adv_sum = 0.0, cyc_sum = 0.0;
  {
    double va[kC], vc[kC];
    from_ranks(s_loss, 1, 0, va);
    from_ranks(s_loss, 2, cb, vc);
    for (int r = 0; r < kC; ++r) {
      adv_sum += va[r];
      cyc_sum += vc[r];
    }
  }
  cluster_arrive();  // S5: flags (arrive; the loss terms below overlap the other CTAs' arrivals)
  const int rows = R.rows;
  const long long n_fwd = (long long)rows * m.out;
  const long long n_cyc = (long long)rows * m.in;
  const double adv = adv_sum / (double)rows;
  const double cyc = cyc_sum / (double)n_cyc;
  const double fm = g_pre[6] / (double)n_fwd;
  const double total_raw = fm + (double)m.lambda_adv * adv + (double)m.lambda_cyc * cyc;
  out[0] = ((double)rows * total_raw) / (double)rows;
  out[1] = ((double)rows * fm) / (double)rows;
  out[2] = ((double)rows * adv) / (double)rows;
  out[3] = ((double)rows * cyc) / (double)rows;
  out[4] = out[5] = 0.0;
  cluster_wait();  // S5
  GSTAMP(27);
  ST();
  // streamed step: the new fwd from the owners' staging copy (written before
  // S5), loaded now so the L2 round trip overlaps the decision below; it
  // replaces this CTA's blob image only if the fwd update is applied
  constexpr int kRf = 8;
  float rv[kRf];
  const NetS& Fn = Y.net[kF];
  const bool prefetch_fwd = g_persist && Fn.count <= kRf * kThreads;
  if (prefetch_fwd)
#pragma unroll
    for (int u = 0; u < kRf; ++u) {
      const int e = u * kThreads + tid;
      rv[u] = e < Fn.count ? __ldcg(a.g[kFwd] + e) : 0.0f;
    }
  int all_f = 1, all_i = 1;
  {
    int vf[kC], vi[kC];
    from_ranks(s_ok, 1, 0, vf);
    from_ranks(s_ok, 2, cb, vi);
    for (int r = 0; r < kC; ++r) {
      all_f &= vf[r];
      all_i &= vi[r];
    }
  }
  // trainer.hpp:256-264: g_total, then fwd (throws before any change),
  // then inv (fwd already applied)
  if (isfinite(out[0]) && all_f) {
    if (g_persist) {
      // streamed step: every CTA takes the new fwd from the staging copy
      // (here if prefetched, else the caller refreshes); the owners commit
      // p / m / v after next_h (off the critical path)
      if (prefetch_fwd)
#pragma unroll
        for (int u = 0; u < kRf; ++u) {
          const int e = u * kThreads + tid;
          if (e < Fn.count) S()[Fn.blob + e] = rv[u];
        }
    } else
      adam_commit(a, kFwd, Y.net[kF], R.lo[1], R.hi[1], Y.gr[1], Y.mo[1], Y.vo[1], Y.mt[1], Y.vt[1],
                  a.post_next_h ? 1 : 0);  // every CTA needs the new fwd blob for next_h
    out[4] = 1.0;
    ST();
    if (all_i) {
      if (!R.split) adam_commit(a, kInv, Y.net[kI], R.lo[2], R.hi[2], Y.gr[2], Y.mo[2], Y.vo[2], Y.mt[2], Y.vt[2], 0);
      out[5] = 1.0;
    }
  }
  ST();
}

/// Counters and the StepRecord (trainer.hpp:274-289); CTA 0, thread 0.
__device__ __noinline__ void finish(const StepArgs& a, bool d_ok, double d_loss, const double* g) {
  Counters* ctr = a.ctr;
  const bool fwd_applied = g[4] != 0.0, inv_applied = g[5] != 0.0;
  const bool g_ok = inv_applied;
  if (d_ok) ctr->t[kDisc] += 1;
  if (fwd_applied) ctr->t[kFwd] += 1;
  if (inv_applied) ctr->t[kInv] += 1;
  const bool skipped = !(d_ok && g_ok);
  StepRec r{};
  r.d_loss = d_ok ? d_loss : 0.0;
  if (g_ok) {
    r.g_total = g[0];
    r.g_fwd = g[1];
    r.g_adv = g[2];
    r.g_cyc = g[3];
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

/// h = dec_head(fwd(x)) and the x rows of the NEXT step of this epoch
/// (what k_gather's row kernel computes, same k-ordered chains), from the
/// updated fwd every CTA holds after S6: the next step then needs no row
/// kernel. Rows of the next minibatch are split over the CTAs like this
/// step's. No-op when this step ends the epoch (the next epoch's plan is not
/// on the device yet; its first step runs the row kernel).
__device__ __noinline__ void next_h(const StepArgs& a, const Layout& Y, int sie, unsigned epoch) {
  float* s = S();
  const ModelArgs& m = a.m;
  const int tid = threadIdx.x;
  const int nxt = sie + 1;
  if ((long long)nxt * a.B >= (long long)a.n_part) return;
  const int rows = min(a.B, a.n_part - nxt * a.B);
  const int rank = (int)cg::this_cluster().block_rank() % kC;
  const int per = (rows + kC - 1) / kC;
  const int r0 = min(rank * per, rows), nr = max(0, min(per, rows - r0));
  (void)epoch;
  const int in = m.in;
  cp_wait_all();  // the xn rows (prologue cp.async)
  __syncthreads();
  for (int i = tid; i < kR * in; i += kThreads) {  // rows prefetched into xn by the prologue
    const float v = s[Y.xn + i];
    if (i < nr * in) a.xb[(long long)r0 * in + i] = v;
    s[Y.xs + i] = v;
  }
  __syncthreads();
  const NetS& F = Y.net[kF];
  const NetS& DH = Y.net[kDH];
  const int latent = Y.stacked + kR * m.lat;
  wnet_fwd(F, Y.xs, 2, latent);
  int fin = latent, w = m.lat;
  if (DH.L > 0) {
    wnet_fwd(DH, latent, 2, -1);
    fin = DH.a[DH.L - 1];
    w = DH.w[DH.L];
  }
  __syncthreads();
  for (int i = tid; i < nr * w; i += kThreads) a.h[(long long)r0 * w + i] = s[fin + i];
}

/// The second half of a 16-CTA cluster (ranks kC .. 2kC-1): the work of the
/// step that does not depend on the D-step -- fwd forward (its own copy),
/// the dec-head backward (dL/dlatent of the forward-MAE term) and the whole
/// cycle path (inv forward, cycle MAE, inv backward, inv weight gradients)
/// -- runs concurrently with the first half's D-step. CTA kC + c owns the
/// same rows as CTA c, which pulls gl_dec / gl_inv over DSMEM after S1. The
/// half mirrors every cluster barrier of the first half (S1 .. S6), reduces
/// the inv partials over its own ranks, and applies Adam(inv) on its owner
/// slices once the step's decision (computed identically from the shared
/// flags and loss sums) says so.
__device__ void stage_dec_rows(const StepArgs& a, const Layout& Y, const Rows& R, const float* red_dec,
                               int S_wide);

/// Streamed step (rs != nullptr): the cycle path runs first, then the wait
/// for the wide pass's dec half of step k (red_dec, the MAE total) and the
/// dec-head backward; *out gets d_ok, fwd_applied, inv_applied (the same
/// decision every CTA of the cluster computes).
__device__ __noinline__ void cyc_half(const StepArgs& a, const Layout& Y, const Rows& R, double* s_loss, int* s_ok,
                                      double* s_wl, const StreamArgs* rs = nullptr, int k = 0,
                                      int* out = nullptr, unsigned* dflag = nullptr) {
  cg::cluster_group cl = cg::this_cluster();
  const ModelArgs& m = a.m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const NetS& F = Y.net[kF];
  const NetS& I = Y.net[kI];
  const NetS& DH = Y.net[kDH];
  const int latent = Y.stacked + kR * m.lat;
  const int nr = R.nr, rows = R.rows;
  wnet_fwd(F, Y.xs, 2, latent);
  if (DH.L > 0) wnet_fwd(DH, latent, 2, -1);  // dec-head tape
  if (DH.L > 0 && !rs) {
    dz_warp(Y.gh, DH, DH.L - 1, DH.dz[DH.L - 1]);
    wnet_bwd(DH, 2, Y.gl_dec, -1, -1);
  }
  wnet_fwd(I, latent, 2, -1);
  {
    const double part = cyc_warp(I.a[I.L - 1], Y.xs, I.dz[I.L - 1], m.in, nr, rows, m.lambda_cyc);
    if (lane == 0) s_wl[warp] = part;
    __syncwarp();
  }
  wnet_bwd(I, 2, Y.gl_inv, -1, -1);
  __syncthreads();
  pg_net(I, latent, kR, Y.pg[2]);
  if (tid == 0) s_loss[2] = sum_warps(s_wl);
  __syncthreads();
  cluster_arrive();  // S1
  cluster_wait();
  cp_wait_all();  // g_pre (prologue cp.async); reduce_owned's barrier publishes it
  const int iok = reduce_owned(Y.pg[2], R.lo[2], R.hi[2], Y.gr[2], kC);
  if (tid == 0) s_ok[2] = iok;
  adam_compute(a, kInv, I, R.lo[2], R.hi[2], g_pre[4], g_pre[5], Y.gr[2], Y.mo[2], Y.vo[2], Y.mt[2], Y.vt[2]);
  if (rs) stage_new_params(a.g[kInv], Y.gr[2], R.lo[2], R.hi[2]);  // published by S2
  cluster_sync();  // S2 (d_update's flags)
  double d_sum = 0.0;
  int all_ok = 1;
  {
    double vd[kC];
    int vo[kC];
    from_ranks(s_loss, 0, 0, vd);
    from_ranks(s_ok, 0, 0, vo);
    for (int r = 0; r < kC; ++r) {
      d_sum += vd[r];
      all_ok &= vo[r];
    }
  }
  const double d_loss = ((double)rows * (d_sum / (2.0 * (double)rows))) / (double)rows;
  const bool d_ok = isfinite(d_loss) && all_ok;
  cluster_sync();  // S3
  if (rs) {
    // streamed step: the discriminator update above ran while the wide pass
    // streamed its dec half; now wait for it (red_dec, the MAE total), run
    // the dec-head backward and hand dL/dlatent (dec, cycle) to the partner
    // CTA at S3b
    __shared__ int s_w;
    if (tid == 0) {
      s_w = wait_counter(&rs->sync->dec_done, (unsigned long long)rs->S_wide * (k + 1), rs->sync, 3) ? 1 : 0;
      if (rs->prof && cg::this_cluster().block_rank() == kC) rs->prof[512 * k + 7] = gtimer();
    }
    __syncthreads();
    stage_dec_rows(a, Y, R, rs->red_dec[k & 1], rs->S_wide);
    if (DH.L > 0) {
      dz_warp(Y.gh, DH, DH.L - 1, DH.dz[DH.L - 1]);
      wnet_bwd(DH, 2, Y.gl_dec, -1, -1);
    }
    __syncthreads();
    // push dL/dlatent (dec, cycle) into the D/G partner (same rows), then
    // raise its flag; it reads them locally (no cluster barrier)
    {
      float* s = S();
      float* peer = cl.map_shared_rank(s, R.rank);
      for (int i = tid; i < kR * m.lat; i += kThreads) {
        peer[Y.gl_dec + i] = s[Y.gl_dec + i];
        peer[Y.gl_inv + i] = s[Y.gl_inv + i];
      }
      __syncthreads();
      if (tid == 0) {
        cl.map_shared_rank(g_pre, R.rank)[6] = g_pre[6];  // the step's forward-MAE total, for g_update
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        const uint32_t fa = tc::smem_u32(dflag);
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(fa), "r"((unsigned)R.rank));
        asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"((unsigned)(k + 1)) : "memory");
      }
    }
  }
  bool f_app = false, i_app = false;
  if (d_ok) {
    cluster_sync();  // S4
    cluster_sync();  // S5
    double adv_sum = 0.0, cyc_sum = 0.0;
    int all_f = 1, all_i = 1;
    {
      double va[kC], vc[kC];
      int vf[kC], vi[kC];
      from_ranks(s_loss, 1, 0, va);
      from_ranks(s_loss, 2, kC, vc);
      from_ranks(s_ok, 1, 0, vf);
      from_ranks(s_ok, 2, kC, vi);
      for (int r = 0; r < kC; ++r) {
        adv_sum += va[r];
        cyc_sum += vc[r];
        all_f &= vf[r];
        all_i &= vi[r];
      }
    }
    const double adv = adv_sum / (double)rows;
    const double cyc = cyc_sum / (double)((long long)rows * m.in);
    const double fm = g_pre[6] / (double)((long long)rows * m.out);
    const double total_raw = fm + (double)m.lambda_adv * adv + (double)m.lambda_cyc * cyc;
    const double total = ((double)rows * total_raw) / (double)rows;
    f_app = isfinite(total) && all_f;
    i_app = f_app && all_i;
    if (isfinite(total) && all_f && all_i)  // trainer.hpp:256-264: inv after fwd
      adam_commit(a, kInv, I, R.lo[2], R.hi[2], Y.gr[2], Y.mo[2], Y.vo[2], Y.mt[2], Y.vt[2],
                  0);  // streamed step: the cyc half pulls the new inv (pull_net)
  }
  if (out) {
    out[0] = d_ok;
    out[1] = f_app;
    out[2] = i_app;
  }
}

__device__ __noinline__ void print_phases(const long long* ph, int n) {
  printf("post phases (cycles):");
  for (int i = 1; i < n; ++i) printf(" %lld", ph[i] - ph[i - 1]);
  printf("\n  update stamps:");
  for (int i = 1; i < g_nst; ++i) printf(" %lld", g_st[i] - g_st[i - 1]);
  printf("\n");
}

__global__ void __launch_bounds__(kThreads, 1)
    k_post_small(const __grid_constant__ StepArgs ap, const __grid_constant__ Layout Lp) {
  __shared__ Layout Y;
  // The argument block lives in shared memory for the whole step: the
  // out-of-line phases read their fields through a reference, and
  // reads of kernel parameters through a generic address are slow.
  __shared__ __align__(16) StepArgs a_s;
  {
    const int* src = reinterpret_cast<const int*>(&ap);
    int* dst = reinterpret_cast<int*>(&a_s);
    for (int i = threadIdx.x; i < (int)(sizeof(StepArgs) / sizeof(int)); i += kThreads) dst[i] = src[i];
    const int* src2 = reinterpret_cast<const int*>(&Lp);
    int* dst2 = reinterpret_cast<int*>(&Y);
    for (int i = threadIdx.x; i < (int)(sizeof(Layout) / sizeof(int)); i += kThreads) dst2[i] = src2[i];
    __syncthreads();
  }
  const StepArgs& a = a_s;
  __shared__ double s_loss[4];       // d, adv, cyc partial sums of this CTA
  __shared__ double s_wl[kWarps];    // per-warp loss partials
  __shared__ int s_ok[4];            // finite flags of this CTA's owned slices
  __shared__ long long s_ph[16];
  __shared__ double s_g[6];
  __shared__ __align__(8) uint64_t s_bar;
  int n_ph = 0;
#define PH()                                                                  \
  do {                                                                        \
    if (a.phase_prof && threadIdx.x == 0 && n_ph < 16) s_ph[n_ph] = clock64(); \
    ++n_ph;                                                                   \
  } while (0)
  PH();
  if (a.ctr->aborted) return;
  const ModelArgs& m = a.m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Rows R;
  const int crank = (int)cg::this_cluster().block_rank();
  R.split = cg::this_cluster().num_blocks() == 2 * kC ? 1 : 0;
  const int half = crank / kC;
  R.rank = crank % kC;
  const int sie = (int)a.ctr->step_in_epoch;
  const unsigned epoch = a.ctr->epoch;
  R.rows = min(a.B, a.n_part - sie * a.B);
  {
    const int per = (R.rows + kC - 1) / kC;
    R.r0 = min(R.rank * per, R.rows);
    R.nr = max(0, min(per, R.rows - R.r0));
  }
  for (int q = 0; q < 3; ++q) {
    const int c = q == 0 ? Y.net[kCd].count : (q == 1 ? Y.net[kF].count : Y.net[kI].count);
    R.lo[q] = owner_lo(c, R.rank);
    R.hi[q] = owner_lo(c, R.rank + 1);
  }
  if (tid == 0) {
    g_nst = 0;
    g_persist = 0;
    tc::mbar_init(&s_bar, 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  prologue(a, Y, R, &s_bar);
  PH();
  if (half == 1) {
    cyc_half(a, Y, R, s_loss, s_ok, s_wl);
    cluster_sync();  // S6
    return;
  }
  const NetS& F = Y.net[kF];
  const NetS& I = Y.net[kI];
  const NetS& C = Y.net[kCd];
  const NetS& ET = Y.net[kET];
  const NetS& DH = Y.net[kDH];
  const int latent = Y.stacked + kR * m.lat;
  const int nr = R.nr, rows = R.rows;

  // ---- D-step forward + input-gradient chain, warp-local (rows w + 8 i) ----
  if (ET.L > 0) wnet_fwd(ET, Y.e1, 2, Y.stacked);  // real latents -> stacked[0, R)
  wnet_fwd(F, Y.xs, 2, latent);                    // fake latents -> stacked[R, 2R)
  if (DH.L > 0 && !R.split) wnet_fwd(DH, latent, 2, -1);  // dec-head tape
  wnet_fwd(C, Y.stacked, 4, -1);                   // disc on [real; fake]: rows w, w+8 | w+16, w+24
  {
    const double lv = bce_warp(C.a[C.L - 1], C.dz[C.L - 1], 4, kR, nr, 2.0 * (double)rows, 1.0f);
    if (lane == 0) s_wl[warp] = lv;
    __syncwarp();
  }
  wnet_bwd(C, 4, -1, -1, -1);  // dz of every disc layer
  __syncthreads();
  PH();
  pg_net(C, Y.stacked, 2 * kR, Y.pg[0]);  // disc weight gradients (all rows)
  if (tid == 0) s_loss[0] = sum_warps(s_wl);
  __syncthreads();
  PH();
  cluster_arrive();  // S1: disc partials + loss published

  // ---- independent of the D-step: dec path, whole cycle path ----
  // (split mode: computed concurrently by the cyc half, see cyc_half)
  if (!R.split && DH.L > 0) {
    dz_warp(Y.gh, DH, DH.L - 1, DH.dz[DH.L - 1]);
    wnet_bwd(DH, 2, Y.gl_dec, -1, -1);
  }
  if (!R.split) {
    wnet_fwd(I, latent, 2, -1);
    {
      const double part = cyc_warp(I.a[I.L - 1], Y.xs, I.dz[I.L - 1], m.in, nr, rows, m.lambda_cyc);
      if (lane == 0) s_wl[warp] = part;
      __syncwarp();
    }
    wnet_bwd(I, 2, Y.gl_inv, -1, -1);
    __syncthreads();
    pg_net(I, latent, kR, Y.pg[2]);
    if (tid == 0) s_loss[2] = sum_warps(s_wl);
  }
  PH();
  cluster_wait();  // S1
  if (R.split) {  // dL/dlatent of the dec and cycle paths from the partner CTA of the cyc half
    cg::cluster_group cl = cg::this_cluster();
    float* s = S();
    const float* pdec = cl.map_shared_rank(s + Y.gl_dec, kC + R.rank);
    const float* pinv = cl.map_shared_rank(s + Y.gl_inv, kC + R.rank);
    for (int i = tid; i < kR * m.lat; i += kThreads) {
      s[Y.gl_dec + i] = pdec[i];
      s[Y.gl_inv + i] = pinv[i];
    }
    __syncthreads();
  }
  PH();

  double d_loss = 0.0;
  const bool d_ok = d_update(a, Y, R, s_loss, s_ok, &d_loss);
  PH();
  if (tid == 0)
    for (int i = 0; i < 6; ++i) s_g[i] = 0.0;
  if (d_ok) {
    // adversarial path through the updated disc, then fwd backprop: warp-local
    wnet_fwd(C, latent, 2, -1);
    {
      const double lv = bce_warp(C.a[C.L - 1], C.dz[C.L - 1], 2, kR, nr, (double)rows, m.lambda_adv);
      if (lane == 0) s_wl[warp] = lv;
      __syncwarp();
    }
    // grad_latent = (dec + disc) + inv, fused into the disc layer-0 input gradient
    wnet_bwd(C, 2, Y.gl, Y.gl_dec, Y.gl_inv);
    dz_warp(Y.gl, F, F.L - 1, F.dz[F.L - 1]);  // fwd's top layer: dz = grad_latent * act'
    wnet_bwd(F, 2, -1, -1, -1);
    __syncthreads();
    PH();
    pg_net(F, Y.xs, kR, Y.pg[1]);
    if (tid == 0) s_loss[1] = sum_warps(s_wl);
    double g[6];
    g_update(a, Y, R, s_loss, s_ok, g);
    if (tid == 0)
      for (int i = 0; i < 6; ++i) s_g[i] = g[i];
    PH();
  }
  cluster_sync();  // S6: updated fwd in every CTA; no CTA leaves while peers read its shared memory
  PH();
  if (a.post_next_h) next_h(a, Y, sie, epoch);
  PH();
  if (R.rank == 0 && tid == 0) {  // first half only (the cyc half returned above)
    finish(a, d_ok, d_loss, s_g);
    if (a.phase_prof) print_phases(s_ph, n_ph < 16 ? n_ph : 16);
  }
#undef PH
}

// ============================================================ streamed step ==
// k_post_loop: the post half of the streamed step. One persistent 16-CTA
// cluster per run of steps inside an epoch, beside the persistent wide pass
// (k_wide_ps) on the other SMs. The blob images, W^T images and the owners'
// Adam moments stay resident in shared memory (the owners push every update
// into the CTAs that read it), so a step stages only its rows of the
// wide-pass sums. Per step k (DeviceTrainer::launch_stream_run):
//   D/G half: wait enc_done(k) -> enc rows -> D-step chain -> S1 -> disc
//             update -> adversarial + fwd backward -> fwd update -> S6 ->
//             next_h (h / x rows of step k+1) -> h_done += 1 -> record
//   cyc half: fwd / inv forward, cycle path, inv gradients -> wait
//             dec_done(k) -> dec rows -> dec-head backward -> S1 -> inv
//             update -> S6 -> next step's x rows
// Skip / abort decisions are the launched kernel's, computed by every CTA
// from the same cluster-shared flags; the counters they need (Adam t, the
// skip count) are tracked locally from the values at launch.

/// This CTA's rows of the reduced enc layer-0 sums (D/G half), enc layer-0
/// bias + activation applied as the launched prologue does (pad rows act(b)).
__device__ __noinline__ void stage_enc_rows(const StepArgs& a, const Layout& Y, const Rows& R, const float* red_enc) {
  float* s = S();
  const ModelArgs& m = a.m;
  const int E1 = m.E1;
  const int e1 = Y.net[kET].L > 0 ? Y.e1 : Y.stacked;
  // every load issued before any is used (one L2 round trip)
  constexpr int kPer = kR * kMaxW / kThreads;
  float v[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int i = (int)threadIdx.x + u * kThreads, r = i / E1;
    v[u] = i < kR * E1 && r < R.nr ? __ldcg(red_enc + (long long)R.r0 * E1 + i) : 0.0f;
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int i = (int)threadIdx.x + u * kThreads;
    if (i < kR * E1) {
      const int c = i - (i / E1) * E1;
      s[e1 + i] = act_f(m.enc_act0, m.enc_slope0, v[u] + s[Y.be + c]);
    }
  }
  __syncthreads();
}

/// This CTA's rows of dL/dh = (1/n) S Wd^T (cyc half), as the launched prologue.
__device__ void stage_dec_rows(const StepArgs& a, const Layout& Y, const Rows& R, const float* red_dec,
                               int S_wide) {
  float* s = S();
  const ModelArgs& m = a.m;
  const int D = m.D;
  const float gscale = (float)(1.0 / ((double)R.rows * (double)m.out));
  const int gh = Y.net[kDH].L > 0 ? Y.gh : Y.gl_dec;
  constexpr int kPer = kR * kMaxW / kThreads;
  float v[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int i = (int)threadIdx.x + u * kThreads;
    v[u] = i < kR * D && i / D < R.nr ? __ldcg(red_dec + (long long)R.r0 * D + i) : 0.0f;
  }
  // the forward-MAE total from the wide CTAs' partials in the same round trip
  // (streamed step; warp 0; the launched wide pass's fixed order: strided
  // partials per lane, then an xor tree)
  double mv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const int lane = (int)threadIdx.x & 31;
  if (S_wide > 0 && threadIdx.x < 32)
#pragma unroll
    for (int u = 0; u < 5; ++u) mv[u] = lane + 32 * u < S_wide ? __ldcg(a.mae_part + lane + 32 * u) : 0.0;
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int i = (int)threadIdx.x + u * kThreads;
    if (i < kR * D) s[gh + i] = v[u] * gscale;
  }
  if (S_wide > 0 && threadIdx.x < 32) {
    double t = (((mv[0] + mv[1]) + mv[2]) + mv[3]) + mv[4];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if (lane == 0) g_pre[6] = t;
  }
  __syncthreads();
}

/// x rows of step `nxt` of the epoch (this CTA's row block) into xn, async.
__device__ __noinline__ void prefetch_next_x(const StepArgs& a, const Layout& Y, const Rows& R, int nxt,
                                             unsigned epoch) {
  float* s = S();
  const int in = a.m.in;
  if ((long long)nxt * a.B >= (long long)a.n_part) return;
  const int rows = min(a.B, a.n_part - nxt * a.B);
  const int per = (rows + kC - 1) / kC;
  const int r0 = min(R.rank * per, rows), nr = max(0, min(per, rows - r0));
  const unsigned* perm = a.perm[epoch & 1u] + (long long)nxt * a.B + r0;
  for (int i = threadIdx.x; i < kR * in; i += kThreads) {
    const int r = i / in, c = i - r * in;
    if (r < nr)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tc::smem_u32(s + Y.xn + i)),
                   "l"(a.sx + (long long)perm[r] * in + c)
                   : "memory");
    else
      s[Y.xn + i] = 0.0f;
  }
}

/// D/G half of the streamed step: the next step's row indices into s_xidx
/// by cp.async (no thread waits on the index loads at the top of the step);
/// prefetch_next_x_from_idx issues the x-row copies once they have landed.
__device__ __forceinline__ void prefetch_next_idx(const StepArgs& a, const Rows& R, int nxt, unsigned epoch,
                                                  unsigned* s_xidx) {
  if ((long long)nxt * a.B >= (long long)a.n_part) return;
  const int rows = min(a.B, a.n_part - nxt * a.B);
  const int per = (rows + kC - 1) / kC;
  const int r0 = min(R.rank * per, rows), nr = max(0, min(per, rows - r0));
  const unsigned* perm = a.perm[epoch & 1u] + (long long)nxt * a.B + r0;
  if ((int)threadIdx.x < nr)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tc::smem_u32(s_xidx + threadIdx.x)),
                 "l"(perm + threadIdx.x)
                 : "memory");
}

/// x rows of step `nxt` into xn from the landed indices (after a cp_wait_all
/// and a CTA barrier), async; same copies as prefetch_next_x.
__device__ __noinline__ void prefetch_next_x_from_idx(const StepArgs& a, const Layout& Y, const Rows& R, int nxt,
                                                      const unsigned* s_xidx) {
  float* s = S();
  const int in = a.m.in;
  if ((long long)nxt * a.B >= (long long)a.n_part) return;
  const int rows = min(a.B, a.n_part - nxt * a.B);
  const int per = (rows + kC - 1) / kC;
  const int r0 = min(R.rank * per, rows), nr = max(0, min(per, rows - r0));
  for (int i = threadIdx.x; i < kR * in; i += kThreads) {
    const int r = i / in, c = i - r * in;
    if (r < nr)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tc::smem_u32(s + Y.xn + i)),
                   "l"(a.sx + (long long)s_xidx[r] * in + c)
                   : "memory");
    else
      s[Y.xn + i] = 0.0f;
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    k_post_loop(const __grid_constant__ StepArgs ap, const __grid_constant__ Layout Lp,
                const __grid_constant__ StreamArgs rp) {
  __shared__ Layout Y;
  __shared__ __align__(16) StepArgs a_s;
  __shared__ __align__(16) StreamArgs r_s;
  {
    const int* src = reinterpret_cast<const int*>(&ap);
    int* dst = reinterpret_cast<int*>(&a_s);
    for (int i = threadIdx.x; i < (int)(sizeof(StepArgs) / sizeof(int)); i += kThreads) dst[i] = src[i];
    const int* src2 = reinterpret_cast<const int*>(&Lp);
    int* dst2 = reinterpret_cast<int*>(&Y);
    for (int i = threadIdx.x; i < (int)(sizeof(Layout) / sizeof(int)); i += kThreads) dst2[i] = src2[i];
    const int* src3 = reinterpret_cast<const int*>(&rp);
    int* dst3 = reinterpret_cast<int*>(&r_s);
    for (int i = threadIdx.x; i < (int)(sizeof(StreamArgs) / sizeof(int)); i += kThreads) dst3[i] = src3[i];
    __syncthreads();
  }
  const StepArgs& a = a_s;
  const StreamArgs& r = r_s;
  __shared__ double s_loss[4];
  __shared__ double s_wl[kWarps];
  __shared__ int s_ok[4];
  __shared__ double s_g[6];
  __shared__ int s_res[3];    // d_ok, fwd applied, inv applied of the step
  __shared__ int s_err[2];    // StepSync::error seen before S6 (step parity; read from rank 0)
  __shared__ int s_w;
  __shared__ unsigned s_dflag;  // D/G half: steps whose gl_dec / gl_inv the cyc partner has pushed
  __shared__ unsigned s_xidx[kR];  // D/G half: the next step's row indices (cp.async)
  __shared__ __align__(8) uint64_t s_bar;
  const ModelArgs& m = a.m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  cg::cluster_group cl = cg::this_cluster();
  StepSync* sy = r.sync;
  Rows R;
  const int crank = (int)cl.block_rank();
  R.split = 1;  // launched only as the 16-CTA split cluster
  const int half = crank / kC;
  R.rank = crank % kC;
  for (int q = 0; q < 3; ++q) {
    const int c = q == 0 ? Y.net[kCd].count : (q == 1 ? Y.net[kF].count : Y.net[kI].count);
    R.lo[q] = owner_lo(c, R.rank);
    R.hi[q] = owner_lo(c, R.rank + 1);
  }
  auto set_rows = [&](int sie) {
    R.rows = min(a.B, a.n_part - sie * a.B);
    const int per = (R.rows + kC - 1) / kC;
    R.r0 = min(R.rank * per, R.rows);
    R.nr = max(0, min(per, R.rows - R.r0));
  };
  // counters this run advances (trainer.hpp:274-289), tracked locally
  unsigned long long t_disc = a.ctr->t[kDisc], t_fwd = a.ctr->t[kFwd], t_inv = a.ctr->t[kInv];
  unsigned long long skipped = a.ctr->skipped;
  if (tid == 0) {
    s_dflag = 0;
    g_nst = 0;
    g_persist = 1;
    tc::mbar_init(&s_bar, 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  if (crank == 0 && tid == 0) {  // resident (host-visible flag: the k_wide_ps path waits for it)
    sy->t_post0 = gtimer();
    *reinterpret_cast<volatile int*>(r.resident_host) = r.run_id;
    __threadfence_system();
  }
  // the wide pass (k_wide2) is a programmatic dependent launch on this
  // stream: it may start as soon as every CTA of this cluster is resident
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (a.ctr->aborted) {  // trainer.hpp:282-288: a run after the abort is all no-ops
    if (crank == 0 && tid == 0) atomicExch(&sy->abort, 1);
    return;
  }
  set_rows(r.sie0);
  prologue(a, Y, R, &s_bar, 1);
  const NetS& F = Y.net[kF];
  const NetS& C = Y.net[kCd];
  const NetS& ET = Y.net[kET];
  const int latent = Y.stacked + kR * m.lat;
  const bool pstamp = r.prof != nullptr && tid == 0 && (crank == 0 || crank == kC);
#define PSTAMP(slot) do { if (pstamp) r.prof[512 * k + (slot)] = gtimer(); } while (0)
  for (int k = 0; k < r.n; ++k) {
    const int sie = r.sie0 + k;
    if (crank == 0) PSTAMP(8);
    if (tid == 0) g_pb = (r.prof && crank == 0) ? r.prof + 512 * k : nullptr;
    set_rows(sie);
    const int nr = R.nr, rows = R.rows;
    if (half == 1) prefetch_next_x(a, Y, R, sie + 1, r.epoch);
    else prefetch_next_idx(a, R, sie + 1, r.epoch, s_xidx);  // rows issued after d_update
    if (tid >= 32 && tid < 35) {  // Adam bias corrections 1 - b^t of this step's t (host std::pow table)
      const int q = tid - 32;     // (not thread 0: it polls the wide pass's counters)
      const unsigned long long t = (q == 0 ? t_disc : (q == 1 ? t_fwd : t_inv)) + 1;
      g_pre[2 * q] = a.adam_c[2 * t];
      g_pre[2 * q + 1] = a.adam_c[2 * t + 1];
    }
    if (half == 1) {
      int res[3];
      cyc_half(a, Y, R, s_loss, s_ok, s_wl, &r, k, res, &s_dflag);
      PSTAMP(15);
      if (tid == 0) {
        s_res[0] = res[0];
        s_res[1] = res[1];
        s_res[2] = res[2];
      }
      // the generator's new parameters from the owners' staging copies
      // (fwd: written before S5, inv: before S2): fwd (blob) and inv (blob
      // + W^T); no further cluster barrier this step
      if (res[1]) refresh_net(F, a.g[kFwd], false);
      if (res[2]) refresh_net(Y.net[kI], a.g[kInv], true);
      cp_wait_all();   // the next step's x rows
      __syncthreads();
      for (int i = tid; i < kR * m.in; i += kThreads) S()[Y.xs + i] = S()[Y.xn + i];
    } else {
      // ---- D-step: wait for the enc half of the wide pass of step k ----
      if (tid == 0)
        s_w = wait_counter(&sy->enc_done, (unsigned long long)r.S_wide * (k + 1), sy, 2) ? 1 : 0;
      PSTAMP(9);
      __syncthreads();
      stage_enc_rows(a, Y, R, r.red_enc[k & 1]);
      GSTAMP(100);
      if (ET.L > 0) wnet_fwd(ET, Y.e1, 2, Y.stacked);  // real latents -> stacked[0, R)
      GSTAMP(101);
      // fake latents -> stacked[R, 2R): from step 1 of the run on, next_h of
      // the previous step computed exactly this tape (same updated fwd, same
      // x rows, same routine; train_ops.hpp:165 and :97 use the same fwd)
      if (k == 0) wnet_fwd(F, Y.xs, 2, latent);
      GSTAMP(102);
      wnet_fwd(C, Y.stacked, 4, -1);                   // disc on [real; fake]
      GSTAMP(103);
      {
        const double lv = bce_warp(C.a[C.L - 1], C.dz[C.L - 1], 4, kR, nr, 2.0 * (double)rows, 1.0f);
        if (lane == 0) s_wl[warp] = lv;
        __syncwarp();
      }
      GSTAMP(104);
      wnet_bwd(C, 4, -1, -1, -1);
      GSTAMP(105);
      __syncthreads();
      pg_net(C, Y.stacked, 2 * kR, Y.pg[0]);
      GSTAMP(106);
      if (tid == 0) {
        s_loss[0] = sum_warps(s_wl);
        s_err[k & 1] = ld_acquire_i(&sy->error);  // read by every CTA at the end of the step (after S1)
      }
      __syncthreads();
      cluster_arrive();  // S1
      cluster_wait();
      GSTAMP(107);
      PSTAMP(10);
      double d_loss = 0.0;
      bool commit_fwd = false;
      const bool d_ok = d_update(a, Y, R, s_loss, s_ok, &d_loss);
      PSTAMP(11);
      prefetch_next_x_from_idx(a, Y, R, sie + 1, s_xidx);  // indices landed (d_update's wait + barriers)
      if (tid == 0)
        for (int i = 0; i < 6; ++i) s_g[i] = 0.0;
      if (d_ok) {
        // adversarial path through the updated disc (train_ops.hpp:106-117):
        // its input gradient waits in gd for the dec / cycle terms
        wnet_fwd(C, latent, 2, -1);
        {
          const double lv = bce_warp(C.a[C.L - 1], C.dz[C.L - 1], 2, kR, nr, (double)rows, m.lambda_adv);
          if (lane == 0) s_wl[warp] = lv;
          __syncwarp();
        }
        wnet_bwd(C, 2, Y.gd, -1, -1);
      }
      if (k > 0) transpose_net(F);  // W^T of the fwd pulled last step (input gradients below)
      GSTAMP(94);
      // the partner's dec-head backward (after the wide pass's dec half):
      // it pushes gl_dec and gl_inv into this CTA's shared memory and then
      // raises s_dflag (release, cluster scope) -- a pairwise hand-off, no
      // cluster barrier
      if (tid == 0) {
        const unsigned want = (unsigned)(k + 1);
        const unsigned long long t0 = gtimer();
        unsigned v;
        for (;;) {
          asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(tc::smem_u32(&s_dflag)) : "memory");
          if (v >= want) break;
          if (gtimer() - t0 > kStreamTimeoutNs) {
            if (atomicCAS(&sy->error, 0, 1) == 0) sy->err_site = 7;
            break;
          }
        }
        // (the partner pushed the step's MAE total into g_pre[6] with them)
      }
      __syncthreads();
      GSTAMP(95);
      if (d_ok) {
        {  // grad_latent = (dec + disc) + inv (train_ops.hpp:104, 116-117, 126-127), the warp's rows
          float* s = S();
          for (int i = 0; i < 2; ++i)
            for (int c = lane; c < m.lat; c += 32) {
              const int o = (warp + 8 * i) * m.lat + c;
              s[Y.gl + o] = (s[Y.gl_dec + o] + s[Y.gd + o]) + s[Y.gl_inv + o];
            }
          __syncwarp();
        }
        GSTAMP(92);
        dz_warp(Y.gl, F, F.L - 1, F.dz[F.L - 1]);
        wnet_bwd(F, 2, -1, -1, -1);
        __syncthreads();
        GSTAMP(93);
        pg_net(F, Y.xs, kR, Y.pg[1]);
        if (tid == 0) s_loss[1] = sum_warps(s_wl);
        double g[6];
        g_update(a, Y, R, s_loss, s_ok, g);
        if (tid == 0)
          for (int i = 0; i < 6; ++i) s_g[i] = g[i];
        PSTAMP(12);
        // the new fwd blob straight from the owners' slices (its W^T image is
        // rebuilt next step while this half waits for the dec half)
        GSTAMP(90);
        // the new fwd from the owners' staging copy (written before S5),
        // unless g_update already took it (prefetched under its decision)
        if (g[4] != 0.0 && F.count > 8 * kThreads) refresh_net(F, a.g[kFwd], false);
        commit_fwd = g[4] != 0.0;
        GSTAMP(91);
        __syncthreads();
        PSTAMP(13);
      }
      if (tid == 0) {
        s_res[0] = d_ok;
        s_res[1] = s_g[4] != 0.0;
        s_res[2] = s_g[5] != 0.0;
      }
      if ((long long)(sie + 1) * a.B < (long long)a.n_part) {
        next_h(a, Y, sie, r.epoch);  // h / x rows of step k+1 (also into this CTA's xs)
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          atomicAdd(&sy->h_done, 1ull);
        }
      }
      PSTAMP(14);
      if (commit_fwd)  // the owners' fwd p / m / v (and W^T) into global memory and their moment images
        adam_commit(a, kFwd, F, R.lo[1], R.hi[1], Y.gr[1], Y.mo[1], Y.vo[1], Y.mt[1], Y.vt[1], 0, 0, kC, false);
      if (R.rank == 0 && tid == 0) finish(a, d_ok, d_loss, s_g);
    }
    // ---- the step's decision, identical in every CTA ----
    __syncthreads();
    const bool d_ok = s_res[0] != 0, f_app = s_res[1] != 0, i_app = s_res[2] != 0;
    if (d_ok) ++t_disc;
    if (f_app) ++t_fwd;
    if (i_app) ++t_inv;
    bool stop = false;
    if (!(d_ok && i_app)) {
      ++skipped;
      stop = (long long)skipped > (long long)a.abort_threshold;  // finish() set ctr->aborted
    }
    if (stop && crank == 0 && tid == 0) {
      __threadfence();
      atomicExch(&sy->abort, 1);
    }
    // a timed-out hand-off anywhere: every CTA reads rank 0's view from before S6
    if (cl.map_shared_rank(s_err, 0)[k & 1]) stop = true;
    if (stop) break;
  }
#undef PSTAMP
  cp_wait_all();
  if (half == 0) {  // the deferred global writes of the run's disc / fwd commits
    __syncthreads();
    commit_globals(a, kDisc, Y.net[kCd], R.lo[0], R.hi[0], Y.mo[0], Y.vo[0]);
    commit_globals(a, kFwd, Y.net[kF], R.lo[1], R.hi[1], Y.mo[1], Y.vo[1]);
  }
  cluster_sync();  // no CTA leaves while peers may still read its shared memory
}

}  // namespace ps

namespace ps {
/// W^T images from the blobs (block q: fwd, inv, disc, dec head).
__global__ void __launch_bounds__(256) k_build_T(const __grid_constant__ StepArgs a) {
  const int q = blockIdx.x;
  const int net = q == 0 ? kFwd : (q == 1 ? kInv : (q == 2 ? kDisc : kDec));
  const NetDesc& d = q == 0 ? a.m.fwd : (q == 1 ? a.m.inv : (q == 2 ? a.m.disc : a.m.dec_head));
  const float* p = a.p[net];
  float* T = a.pT[net];
  if (!T || d.L == 0) return;
  long long at = 0;
  for (int l = 0; l < d.L; ++l) {
    const int in = d.w[l], out = d.w[l + 1], n = (in + 1) * out;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int j = i / (in + 1), k = i - j * (in + 1);
      T[at + i] = k < in ? p[d.off_w[l] + (long long)k * out + j] : 0.0f;
    }
    at += n;
  }
}
}  // namespace ps

long long small_T_floats(const NetDesc& d) {
  long long n = 0;
  for (int l = 0; l < d.L; ++l) n += (long long)(d.w[l] + 1) * d.w[l + 1];
  return n;
}

void launch_build_T(const StepArgs& a, cudaStream_t s) { ps::k_build_T<<<4, 256, 0, s>>>(a); }

namespace {
constexpr std::size_t kSmemCap = 220 * 1024;  // dynamic shared memory (static ~2 KB on top)
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
  const ps::Layout y = ps::make_layout(m);
  if ((std::size_t)y.total * sizeof(float) > kSmemCap) return 0;
  return 1;
}

int post_loop_supported(const StepArgs& a) {
  if (!post_tpl_kind(a) || std::getenv("LTFB_POST_NO_SPLIT")) return 0;
  static PerDevice probe;
  return probe.value([] {
    if (cudaFuncSetAttribute(ps::k_post_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCap) !=
            cudaSuccess ||
        cudaFuncSetAttribute(ps::k_post_loop, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    cudaLaunchConfig_t q{};
    q.gridDim = dim3(2 * ps::kC);
    q.blockDim = dim3(ps::kThreads);
    q.dynamicSmemBytes = kSmemCap;
    cudaLaunchAttribute qa;
    qa.id = cudaLaunchAttributeClusterDimension;
    qa.val.clusterDim.x = 2 * ps::kC;
    qa.val.clusterDim.y = 1;
    qa.val.clusterDim.z = 1;
    q.attrs = &qa;
    q.numAttrs = 1;
    int nclusters = 0;
    const bool ok = cudaOccupancyMaxActiveClusters(&nclusters, ps::k_post_loop, &q) == cudaSuccess && nclusters >= 1;
    cudaGetLastError();
    return ok ? 1 : 0;
  });
}

void launch_post_loop(const StepArgs& a, const StreamArgs& r, cudaStream_t s) {
  static thread_local ps::Layout cache;
  static thread_local ModelArgs cache_m{};
  static thread_local bool have = false;
  if (!have || std::memcmp(&cache_m, &a.m, sizeof(ModelArgs)) != 0) {
    cache = ps::make_layout(a.m);
    cache_m = a.m;
    have = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * ps::kC);
  cfg.blockDim = dim3(ps::kThreads);
  cfg.dynamicSmemBytes = (std::size_t)cache.total * sizeof(float);
  cfg.stream = s;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = 2 * ps::kC;
  at.val.clusterDim.y = 1;
  at.val.clusterDim.z = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, ps::k_post_loop, a, cache, r);
  if (e != cudaSuccess) throw std::runtime_error(std::string("streamed post cluster launch: ") + cudaGetErrorString(e));
}

void launch_post_tpl(int kind, const StepArgs& a, cudaStream_t s) {
  (void)kind;
  static PerDevice attr;
  attr.once([] { cudaFuncSetAttribute(ps::k_post_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCap); });
  static thread_local ps::Layout cache;
  static thread_local ModelArgs cache_m{};
  static thread_local bool have = false;
  if (!have || std::memcmp(&cache_m, &a.m, sizeof(ModelArgs)) != 0) {
    cache = ps::make_layout(a.m);
    cache_m = a.m;
    have = true;
  }
  // one 16-CTA cluster (non-portable size) when the GPU can place it: the
  // cycle path runs in the second half concurrently with the D-step; else
  // one 8-CTA cluster running both in sequence
  static PerDevice split_probe;
  const std::size_t smem = (std::size_t)cache.total * sizeof(float);
  const int split = split_probe.value([] {
    int split = 0;
    if (!std::getenv("LTFB_POST_NO_SPLIT") &&
        cudaFuncSetAttribute(ps::k_post_small, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
      cudaLaunchConfig_t q{};
      q.gridDim = dim3(2 * ps::kC);
      q.blockDim = dim3(ps::kThreads);
      q.dynamicSmemBytes = kSmemCap;
      cudaLaunchAttribute qa;
      qa.id = cudaLaunchAttributeClusterDimension;
      qa.val.clusterDim.x = 2 * ps::kC;
      qa.val.clusterDim.y = 1;
      qa.val.clusterDim.z = 1;
      q.attrs = &qa;
      q.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, ps::k_post_small, &q) == cudaSuccess && nclusters >= 1) split = 1;
    }
    cudaGetLastError();
    return split;
  });
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(split ? 2 * ps::kC : ps::kC);
  cfg.blockDim = dim3(ps::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = cfg.gridDim.x;
  at.val.clusterDim.y = 1;
  at.val.clusterDim.z = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, ps::k_post_small, a, cache);
  if (e != cudaSuccess) throw std::runtime_error(std::string("post kernel launch: ") + cudaGetErrorString(e));
}

}  // namespace ltfb_dev
