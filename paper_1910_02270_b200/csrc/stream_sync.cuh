// Device-side hand-off primitives of the streamed step (k_wide_ps /
// k_post_loop): acquire loads of the StepSync counters and a bounded wait.
// Every wait gives up after kStreamTimeoutNs and raises StepSync::error, so a
// lost hand-off stops the run (the host raises) instead of hanging the GPU.
#pragma once

#include "step_args.cuh"

namespace ltfb_dev {

constexpr unsigned long long kStreamTimeoutNs = 2000000000ull;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire_i(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

/// Until *ctr >= target (call from one thread); false on abort, error or
/// timeout (site: diagnostic code of the waiting point, kept in err_site).
__device__ __forceinline__ bool wait_counter(const unsigned long long* ctr, unsigned long long target, StepSync* sy,
                                             int site = 1) {
  const unsigned long long t0 = gtimer();
  while (ld_acquire(ctr) < target) {
    if (ld_acquire_i(&sy->abort) || ld_acquire_i(&sy->error)) return false;
    if (gtimer() - t0 > kStreamTimeoutNs) {
      if (atomicCAS(&sy->error, 0, 1) == 0) sy->err_site = site;
      return false;
    }
    __nanosleep(64);
  }
  return true;
}

}  // namespace ltfb_dev
