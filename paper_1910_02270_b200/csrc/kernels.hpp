// Host-side launch entry points of the device kernels (one per kernel file,
// so no relocatable device code is needed).
#pragma once

#include <cuda_runtime.h>

#include "step_args.cuh"

namespace ltfb_dev {

void launch_gather(const StepArgs& a, cudaStream_t s);
void launch_pre(const StepArgs& a, cudaStream_t s);
void launch_wide_generic(const StepArgs& a, cudaStream_t s);
bool wide_tc_supported(const StepArgs& a);
void launch_wide_tc(const StepArgs& a, cudaStream_t s);
void launch_reduce(const StepArgs& a, cudaStream_t s);
void launch_post(const StepArgs& a, cudaStream_t s);
void launch_begin_epoch(Counters* ctr, unsigned epoch, cudaStream_t s);

std::size_t eval_wide_smem(const ModelArgs& m);
void launch_eval(const EvalArgs& a, cudaStream_t s);

}  // namespace ltfb_dev
