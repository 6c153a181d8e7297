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
// grid (x chunks [+ 1], B rows). Each row is one contiguous HBM slab row;
// float4 copies keep every warp access 512 B-contiguous. With h_in_gather
// the last CTA column computes h = dec_head(fwd(x)) for its row instead
// (nn/mlp.hpp:201-217, the same k-ordered fmaf chains as k_pre): a few
// dependent L2 round trips, hidden under the copy, so the wide pass finds
// h in HBM/L2 without a separate launch.
__device__ void row_h(const StepArgs& a, int r, unsigned slot) {
  __shared__ float act[2][kMaxSmallWidth];
  __shared__ float wbuf[6144];  // fwd + dec-head blobs (one cp.async round trip)
  const ModelArgs& m = a.m;
  const int t = threadIdx.x;
  const NetDesc* nets[2] = {&m.fwd, &m.dec_head};
  const float* blobs[2] = {a.p[kFwd] + m.fwd.base, a.p[kDec] + m.dec_head.base};
  const int cnt0 = (int)m.fwd.count, cnt1 = (int)m.dec_head.count;
  const bool staged = cnt0 + cnt1 <= 6144;
  if (staged) {
    for (int i = t; i < cnt0 + cnt1; i += blockDim.x) {
      const float* src = i < cnt0 ? blobs[0] + i : blobs[1] + (i - cnt0);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(wbuf + i)),
                   "l"(src)
                   : "memory");
    }
  }
  if (t < m.in) {
    const float x = a.x_from_store ? a.sx[(long long)slot * m.in + t] : a.xb[r * m.in + t];
    act[0][t] = x;
    if (a.x_from_store) a.xb[r * m.in + t] = x;  // the minibatch x for the small nets
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  int cur = 0;
  for (int net = 0; net < 2; ++net) {
    const NetDesc& n = *nets[net];
    const float* blob = staged ? wbuf + (net == 0 ? 0 : cnt0) : blobs[net];
    for (int l = 0; l < n.L; ++l) {
      const int in = n.w[l], out = n.w[l + 1];
      const float* W = blob + (n.off_w[l] - n.base);
      const float* bb = blob + (n.off_b[l] - n.base);
      const bool last = net == 1 && l + 1 == n.L;
      for (int j = t; j < out; j += blockDim.x) {
        float acc = 0.0f;
#pragma unroll 8
        for (int k = 0; k < in; ++k) acc = fmaf(act[cur][k], W[k * out + j], acc);
        const float v = act_apply(n.act[l], n.slope[l], acc + bb[j]);
        if (last) a.h[(long long)r * out + j] = v;
        else act[cur ^ 1][j] = v;
      }
      __syncthreads();
      cur ^= 1;
    }
  }
}

__global__ void __launch_bounds__(256) k_gather(StepArgs a) {
  if (a.ctr->aborted) return;
  const int rows = batch_rows(a);
  const int r = blockIdx.y;
  if (r >= rows) return;
  const long long idx = (long long)a.ctr->step_in_epoch * a.B + r;
  const int nx = gridDim.x - (a.h_in_gather ? 1 : 0);  // copy columns
  if ((int)blockIdx.x >= nx) {
    row_h(a, r, a.x_from_store ? a.perm[a.ctr->epoch & 1][idx] : 0u);
    return;
  }
  const unsigned slot = a.perm[a.ctr->epoch & 1][idx];
  const int n4 = a.m.out_pad >> 2;
  const float4* src = reinterpret_cast<const float4*>(a.sy + (long long)slot * a.m.out_pad);
  float4* dst = reinterpret_cast<float4*>(a.yb + (long long)r * a.m.out_pad);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += nx * blockDim.x) dst[i] = __ldcs(src + i);
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
  const ScratchLayout& L = a.L;
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

// -------------------------------------------------------- epoch control --
__global__ void k_begin_epoch(Counters* ctr, unsigned epoch) {
  ctr->epoch = epoch;
  ctr->step_in_epoch = 0;
}

/// Store rows by slot into a row-major destination slab (the distributed AE
/// batch, runner.hpp:255-277 with the union sharded over the ranks' stores):
/// one CTA per row, float4 copies of the padded row.
__global__ void k_gather_rows(const float* __restrict__ src, const unsigned* __restrict__ slots, int n,
                              float* __restrict__ dst, int out_pad) {
  const int r = blockIdx.x;
  if (r >= n) return;
  const float4* s = reinterpret_cast<const float4*>(src + (long long)slots[r] * out_pad);
  float4* d = reinterpret_cast<float4*>(dst + (long long)r * out_pad);
  for (int i = threadIdx.x; i < out_pad / 4; i += blockDim.x) d[i] = __ldg(s + i);
}

/// Start of a streamed run: the hand-off counters restart, the first step's
/// h counts as ready (the row kernel or the previous run produced it).
__global__ void k_stream_init(StepSync* sy, int run_id, unsigned* grid_bar) {
  // the streamed wide pass's barrier: arrival count and per-CTA flags restart
  for (int i = threadIdx.x; i < 32 + 32 * 160; i += blockDim.x) grid_bar[64 + i] = 0;  // [64, 96 + 32 * 160)
  if (threadIdx.x != 0) return;
  sy->enc_done = 0;
  sy->dec_done = 0;
  sy->h_done = kStreamSignalers;
  sy->abort = 0;
  sy->resident = -run_id;  // error stays sticky: the host reads it after the chunk
  sy->t_post0 = sy->t_wide0 = 0;
  __threadfence();
}

/// Concurrency probe of the streamed step: k_probe_spin waits (<= 50 ms) for
/// k_probe_set, launched on another stream after it. Under tools that
/// serialise kernels (ncu, compute-sanitizer) or when the GPU cannot run the
/// two side by side, the spinner times out and the trainer uses the
/// launched step.
__global__ void k_probe_spin(const volatile int* flag, int* ok) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  int seen = 0;
  for (;;) {
    if (*flag) {
      seen = 1;
      break;
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 50000000ull) break;
    __nanosleep(200);
  }
  *ok = seen;
}
__global__ void k_probe_set(volatile int* flag) {
  *flag = 1;
  __threadfence_system();
}

/// Timer gate (bench timed regions): holds the stream until the host has
/// enqueued the work behind it (*flag != 0), so the device-timed region
/// starts with a full queue; gives up after ~0.5 s so a missed release can
/// never hang the GPU.
__global__ void k_gate(const volatile int* flag) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*flag == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 500000000ull) break;
    __nanosleep(200);
  }
}

}  // namespace ltfb_dev

// ------------------------------------------------------------ launchers --
namespace ltfb_dev {

void launch_gather(const StepArgs& a, cudaStream_t s) {
  const int n4 = a.m.out_pad / 4;
  const int gx = (n4 + 256 * 4 - 1) / (256 * 4);
  k_gather<<<dim3(gx + (a.h_in_gather ? 1 : 0), a.B), 256, 0, s>>>(a);
}

void launch_row_h(const StepArgs& a, bool x_from_store, cudaStream_t s) {
  StepArgs b = a;  // no copy columns: every CTA is a row_h CTA
  b.h_in_gather = 1;
  b.x_from_store = x_from_store ? 1 : 0;
  k_gather<<<dim3(1, a.B), 256, 0, s>>>(b);
}

void launch_pre(const StepArgs& a, cudaStream_t s) { k_pre<<<a.small_ctas, 128, 0, s>>>(a); }

static std::size_t wide_generic_smem(const ModelArgs& m) {
  constexpr int RB = 32, TN = 32;
  return sizeof(float) * (std::size_t)(RB * m.E1 + 2 * RB * m.D + RB * TN + TN * m.E1 + m.D * TN +
                                       RB * TN + TN);
}

void launch_wide_generic(const StepArgs& a, cudaStream_t s) {
  const std::size_t smem = wide_generic_smem(a.m);
  static PerDevice attr;
  attr.once([] { cudaFuncSetAttribute(k_wide_generic<32, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); });
  k_wide_generic<32, 32><<<a.S, 256, smem, s>>>(a);
}


void launch_begin_epoch(Counters* ctr, unsigned epoch, cudaStream_t s) {
  k_begin_epoch<<<1, 1, 0, s>>>(ctr, epoch);
}

void launch_gate(const volatile int* flag, cudaStream_t s) { k_gate<<<1, 1, 0, s>>>(flag); }

void launch_stream_init(StepSync* sy, int run_id, unsigned* grid_bar, cudaStream_t s) {
  k_stream_init<<<1, 256, 0, s>>>(sy, run_id, grid_bar);
}

void launch_gather_rows(const float* src, const unsigned* slots, int n, float* dst, int out_pad, cudaStream_t s) {
  if (n > 0) k_gather_rows<<<n, 256, 0, s>>>(src, slots, n, dst, out_pad);
}

bool probe_concurrency(cudaStream_t a, cudaStream_t b) {
  // load both kernels first: a lazily loaded module waits for the device to idle
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_probe_spin) != cudaSuccess || cudaFuncGetAttributes(&fa, k_probe_set) != cudaSuccess)
    return false;
  int* d = nullptr;
  if (cudaMalloc(&d, 2 * sizeof(int)) != cudaSuccess) return false;
  cudaMemsetAsync(d, 0, 2 * sizeof(int), a);
  cudaStreamSynchronize(a);
  k_probe_spin<<<1, 1, 0, a>>>(d, d + 1);
  k_probe_set<<<1, 1, 0, b>>>(d);
  int ok = 0;
  const bool fine = cudaStreamSynchronize(a) == cudaSuccess && cudaStreamSynchronize(b) == cudaSuccess &&
                    cudaMemcpy(&ok, d + 1, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess;
  cudaFree(d);
  cudaGetLastError();
  return fine && ok == 1;
}

void prepare_stream_kernels() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_stream_init);
  cudaFuncGetAttributes(&fa, k_gate);
  cudaFuncGetAttributes(&fa, k_begin_epoch);
  prepare_wide_ps();
  prepare_wide2();
}

}  // namespace ltfb_dev
