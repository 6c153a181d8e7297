// Host-side launch entry points of the device kernels (one per kernel file,
// so no relocatable device code is needed).
#pragma once

#include <cuda_runtime.h>

#include "step_args.cuh"

namespace ltfb_dev {

void launch_gather(const StepArgs& a, cudaStream_t s);
/// One CTA per minibatch row: x from the store through the epoch plan (also
/// written to xb) or from xb, then h = dec_head(fwd(x)).
void launch_row_h(const StepArgs& a, bool x_from_store, cudaStream_t s);
void launch_pre(const StepArgs& a, cudaStream_t s);
void launch_wide_generic(const StepArgs& a, cudaStream_t s);
bool wide_tc_supported(const StepArgs& a);
void launch_wide_tc(const StepArgs& a, cudaStream_t s);

/// Host-side state of the tcgen05 wide pass: K-major fp32 copies of the
/// frozen wide-layer weights, the padded bias, and the TMA descriptors.
struct WideTcParamsHost {
  alignas(64) unsigned char maps[4 * 128];  // CUtensorMap x4 (y, WeT, Wd, WdT)
  alignas(64) unsigned char y_alt[2][128];  // y maps of the host-streamed (e2e) minibatch buffers
  int y_sel = -1;                           // -1: maps[0] (gathered minibatch), else y_alt[y_sel]
  bool precise = true;
  float* bias_pad = nullptr;
  float* wet = nullptr;
  float* wd = nullptr;
  float* wdt = nullptr;
};
/// Builds the TMA descriptors (yb is [yb_rows x out_pad]).
void encode_wide_maps(WideTcParamsHost& p, const StepArgs& a, const float* yb, int yb_rows);
/// (Re)encodes a y map over [yb_rows x out_pad]: which = -1 the store /
/// gathered-minibatch map, 0/1 the host-streamed buffers.
void encode_y_map(WideTcParamsHost& p, int which, const float* yb, const StepArgs& a, int yb_rows);
void launch_prep_wide(const StepArgs& a, const WideTcParamsHost& p, cudaStream_t s);
void launch_wide_tc_params(const WideTcParamsHost& p, const StepArgs& a, cudaStream_t s);
void launch_reduce(const StepArgs& a, cudaStream_t s);
void launch_post(const StepArgs& a, cudaStream_t s);
bool post_fast_supported(const StepArgs& a);
void launch_post_fast(const StepArgs& a, cudaStream_t s);
/// Compile-time-shaped post kernel (k_post_tpl.cu): 0 if no instance
/// matches the model, else the instance id for launch_post_tpl.
/// Floats of a small net's W^T image (sum over layers of (in + 1) * out).
long long small_T_floats(const NetDesc& d);
/// Rebuilds every non-null StepArgs::pT image from the parameter blobs.
void launch_build_T(const StepArgs& a, cudaStream_t s);
int post_tpl_kind(const StepArgs& a);
void launch_post_tpl(int kind, const StepArgs& a, cudaStream_t s);
void launch_begin_epoch(Counters* ctr, unsigned epoch, cudaStream_t s);

std::size_t eval_wide_smem(const ModelArgs& m);
cudaError_t selftest_tc(const float* a1, const float* b1, const float* ah, const float* b2, const float* a3,
                        float* d1, float* d2, float* d3);
void launch_eval(const EvalArgs& a, cudaStream_t s);

}  // namespace ltfb_dev
