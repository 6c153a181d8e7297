// Device-side building blocks shared by every kernel of the LTFB hot path.
//
// Layout conventions (HBM):
//   * every network is one flat f32 blob in the reference manifest order
//     W0,b0,W1,b1,... with row-major [in x out] weights (nn/mlp.hpp:63-84);
//   * per-row activations are row-major [rows x width];
//   * the data store keeps x [N x input_dim] and y [N x out_pad] slabs, with
//     out_pad = output_dim rounded up to 4 floats (16-byte rows for vector
//     loads and TMA); padding columns are zero.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ltfb_dev {

constexpr int kMaxLayers = 8;     // per small network
constexpr int kMaxSmallWidth = 256;

enum ActKind : int { kIdentity = 0, kRelu = 1, kLeaky = 2, kTanh = 3, kSigmoid = 4 };

/// Descriptor of a stack of small dense layers living inside a blob.
/// `first_layer` lets the enc tail / dec head address a sub-range of the
/// enc/dec blobs whose other layer is the wide one.
struct NetDesc {
  int L = 0;
  int w[kMaxLayers + 1] = {};
  int act[kMaxLayers] = {};
  float slope[kMaxLayers] = {};
  long long off_w[kMaxLayers] = {};
  long long off_b[kMaxLayers] = {};
  long long count = 0;  // parameters in this (sub)net
  long long base = 0;   // offset of the first parameter within the blob
  __host__ __device__ int max_w() const {
    int m = 0;
    for (int i = 0; i <= L; ++i) m = w[i] > m ? w[i] : m;
    return m;
  }
};

// nn/activation.hpp:43-77, float instantiation.
__device__ __forceinline__ float stable_sigmoid(float z) {
  if (z >= 0.0f) return 1.0f / (1.0f + expf(-z));
  const float e = expf(z);
  return e / (1.0f + e);
}
__device__ __forceinline__ float act_apply(int kind, float slope, float z) {
  switch (kind) {
    case kRelu: return z > 0.0f ? z : 0.0f;
    case kLeaky: return z > 0.0f ? z : slope * z;
    case kTanh: return tanhf(z);
    case kSigmoid: return stable_sigmoid(z);
    default: return z;
  }
}
/// act_apply for code that is unrolled many times: the piecewise-linear
/// kinds inline, the transcendental ones behind one out-of-line call, so the
/// instruction footprint stays small.
__device__ __noinline__ float act_apply_slow(int kind, float slope, float z);
__device__ __forceinline__ float act_apply_compact(int kind, float slope, float z) {
  if (kind == kLeaky) return z > 0.0f ? z : slope * z;
  if (kind == kIdentity) return z;
  if (kind == kRelu) return z > 0.0f ? z : 0.0f;
  return act_apply_slow(kind, slope, z);
}
__device__ __noinline__ inline float act_apply_slow(int kind, float slope, float z) { return act_apply(kind, slope, z); }

__device__ __forceinline__ float act_deriv(int kind, float slope, float z, float a) {
  switch (kind) {
    case kRelu: return z > 0.0f ? 1.0f : 0.0f;
    case kLeaky: return z > 0.0f ? 1.0f : slope;
    case kTanh: return 1.0f - a * a;
    case kSigmoid: return a * (1.0f - a);
    default: return 1.0f;
  }
}

__device__ __forceinline__ bool finite_f(float v) { return isfinite(v); }

/// One element of nn/adam.hpp:48-61 (detail::adam_update_range) in double
/// with explicit round-to-nearest operations, so no FMA contraction changes
/// the reference's rounding: m, v are stored as float, the parameter update
/// uses the double mi / vi. Every device Adam (post kernel owners, AE K7)
/// calls this one routine; tests/test_gpu_kernels.py pins it bit-exactly
/// against the reference's adam vectors (tests/golden/nn.npz).
__device__ __forceinline__ float adam_elem(float p, float& m, float& v, float g, double lr, double b1, double b2,
                                           double eps, double c1, double c2) {
  const double gd = (double)g;
  const double mi = __dadd_rn(__dmul_rn(b1, (double)m), __dmul_rn(1.0 - b1, gd));
  const double vi = __dadd_rn(__dmul_rn(b2, (double)v), __dmul_rn(__dmul_rn(1.0 - b2, gd), gd));
  m = (float)mi;
  v = (float)vi;
  return (float)__dsub_rn((double)p, __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mi, c1)), __dadd_rn(__dsqrt_rn(__ddiv_rn(vi, c2)), eps)));
}

/// Per-trainer device counters; every step kernel reads them, the step's
/// last kernel advances them. Kept in device memory so one captured step
/// graph can be replayed.
struct Counters {
  unsigned long long global_step;  // steps executed (skipped ones included)
  unsigned long long t[5];         // Adam step count per network
  unsigned int step_in_epoch;
  unsigned int skipped;
  int aborted;                     // sticky once skipped > threshold
  unsigned int epoch;
  int last_adopt;                  // decision kernel output
  int pad_;
};

/// One StepRecord (train/history.hpp:20-30) as written by the device.
struct StepRec {
  double d_loss, g_total, g_fwd, g_adv, g_cyc;
  unsigned long long step;
  unsigned int epoch;
  unsigned int flags;  // bit0 skipped, bit1 D applied, bit2 G applied, bit3 aborted here
};

enum NetId : int { kEnc = 0, kDec = 1, kFwd = 2, kInv = 3, kDisc = 4 };

}  // namespace ltfb_dev
