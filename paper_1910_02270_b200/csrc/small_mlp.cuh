// Block-cooperative forward / backward of the small dense networks (fwd, inv,
// disc, enc tail, dec head). Widths are <= 256 and row counts <= 2 x batch,
// so every layer is a few thousand MACs: one thread owns one output element
// and sums its dot product in the reference's index order
// (nn/mlp.hpp:280-361 over nn/tensor.hpp:114-175).
//
// `Sync` abstracts the barrier so the same code runs inside one CTA
// (__syncthreads) or across a thread-block cluster.
#pragma once

#include "device_common.cuh"

namespace ltfb_dev {

struct BlockSync {
  __device__ void operator()() const { __syncthreads(); }
  __device__ int rank() const { return threadIdx.x; }
  __device__ int size() const { return blockDim.x; }
};

/// z_l = a_{l-1} W_l + b_l ; a_l = act(z_l) for every layer of `n`.
/// `x` is [rows x w0] with leading dimension ldx; z[l] / a[l] are
/// [rows x w_{l+1}]. z may be null (forward-only use).
template <class Sync>
__device__ void mlp_forward(const NetDesc& n, const float* __restrict__ blob, const float* x,
                            int ldx, int rows, float* const* z, float* const* a, Sync sync) {
  const float* cur = x;
  int ldc = ldx;
  for (int l = 0; l < n.L; ++l) {
    const int in = n.w[l], out = n.w[l + 1];
    const float* W = blob + n.off_w[l];
    const float* b = blob + n.off_b[l];
    const int kind = n.act[l];
    const float slope = n.slope[l];
    for (int idx = sync.rank(); idx < rows * out; idx += sync.size()) {
      const int r = idx / out, j = idx - r * out;
      const float* xr = cur + (long long)r * ldc;
      float acc = 0.0f;
      for (int k = 0; k < in; ++k) acc = fmaf(xr[k], W[k * out + j], acc);
      const float zz = acc + b[j];
      if (z) z[l][idx] = zz;
      a[l][idx] = act_apply(kind, slope, zz);
    }
    sync();
    cur = a[l];
    ldc = out;
  }
}

/// Reverse pass for the tape produced by mlp_forward (nn/mlp.hpp:325-361).
/// gout [rows x w_L]. pgrad (blob layout of this subnet, relative to
/// n.base) and gin [rows x w0] are optional. tA/tB are scratch of
/// rows x max width each. Parameter gradients are sums over `rows`.
template <class Sync>
__device__ void mlp_backward(const NetDesc& n, const float* __restrict__ blob, const float* x,
                             int ldx, int rows, float* const* z, float* const* a,
                             const float* gout, float* pgrad, float* gin, float* tA, float* tB,
                             Sync sync) {
  const float* g = gout;
  for (int l = n.L - 1; l >= 0; --l) {
    const int in = n.w[l], out = n.w[l + 1];
    const float* W = blob + n.off_w[l];
    const int kind = n.act[l];
    const float slope = n.slope[l];
    float* dz = tA;
    for (int idx = sync.rank(); idx < rows * out; idx += sync.size())
      dz[idx] = g[idx] * act_deriv(kind, slope, z[l][idx], a[l][idx]);
    sync();
    const float* below = l == 0 ? x : a[l - 1];
    const int ldb = l == 0 ? ldx : in;
    if (pgrad) {
      float* dW = pgrad + (n.off_w[l] - n.base);
      float* db = pgrad + (n.off_b[l] - n.base);
      for (int idx = sync.rank(); idx < in * out; idx += sync.size()) {
        const int k = idx / out, j = idx - k * out;
        float acc = 0.0f;
        for (int r = 0; r < rows; ++r) acc = fmaf(below[(long long)r * ldb + k], dz[r * out + j], acc);
        dW[idx] = acc;
      }
      for (int j = sync.rank(); j < out; j += sync.size()) {
        float acc = 0.0f;
        for (int r = 0; r < rows; ++r) acc += dz[r * out + j];
        db[j] = acc;
      }
    }
    float* gn = (l == 0) ? gin : tB;
    if (gn) {
      for (int idx = sync.rank(); idx < rows * in; idx += sync.size()) {
        const int r = idx / in, k = idx - r * in;
        const float* dzr = dz + r * out;
        const float* Wk = W + k * out;
        float acc = 0.0f;
        for (int j = 0; j < out; ++j) acc = fmaf(dzr[j], Wk[j], acc);
        gn[idx] = acc;
      }
    }
    sync();
    g = tB;
  }
}

/// Fixed-order block reduction of one double per thread (deterministic).
__device__ inline double block_sum_det(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  const double out = red[0];
  __syncthreads();
  return out;
}

}  // namespace ltfb_dev
