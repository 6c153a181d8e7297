// Host-side launch entry points of the device kernels (one per kernel file,
// so no relocatable device code is needed).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "step_args.cuh"

namespace ltfb_dev {

/// One-time, per-device and thread-safe host setup (kernel function
/// attributes and capability probes live in the device's context: a process
/// that drives several GPUs -- RunConfig.devices round-robins trainers over
/// them -- needs them set once on every device). value() caches one int per
/// device (e.g. a probe result).
class PerDevice {
 public:
  template <class F>
  void once(F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu_);
    if (dev < 0 || dev >= kMax) {
      f();
      return;
    }
    if (!done_[dev]) {
      f();
      done_[dev] = true;
    }
  }
  template <class F>
  int value(F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu_);
    if (dev < 0 || dev >= kMax) return f();
    if (!have_[dev]) {
      val_[dev] = f();
      have_[dev] = true;
    }
    return val_[dev];
  }

 private:
  static constexpr int kMax = 64;
  std::mutex mu_;
  bool done_[kMax] = {};
  bool have_[kMax] = {};
  int val_[kMax] = {};
};

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
  alignas(64) unsigned char wdt64[128];     // WdT with 64-row boxes (k_wide2's 64-column tiles)
  alignas(64) unsigned char y_alt[2][128];  // y maps of the host-streamed (e2e) minibatch buffers
  int y_sel = -1;                           // -1: maps[0] (gathered minibatch), else y_alt[y_sel]
  bool precise = true;
  float* bias_pad = nullptr;
  float* wet = nullptr;
  float* wd = nullptr;
  float* wdt = nullptr;
  // L2 persistence window over the frozen weight copies (one allocation):
  // the weights are re-read every step, y streams through once
  void* l2_base = nullptr;
  std::size_t l2_bytes = 0;
  float l2_hit = 0.0f;  // 0: no window
};
/// Builds the TMA descriptors (yb is [yb_rows x out_pad]).
void encode_wide_maps(WideTcParamsHost& p, const StepArgs& a, const float* yb, int yb_rows);
/// (Re)encodes a y map over [yb_rows x out_pad]: which = -1 the store /
/// gathered-minibatch map, 0/1 the host-streamed buffers.
void encode_y_map(WideTcParamsHost& p, int which, const float* yb, const StepArgs& a, int yb_rows);
void launch_prep_wide(const StepArgs& a, const WideTcParamsHost& p, cudaStream_t s);
void launch_wide_tc_params(const WideTcParamsHost& p, const StepArgs& a, cudaStream_t s);
/// Streamed step (k_wide_ps.cu / k_post_tpl.cu k_post_loop): the persistent
/// two-phase wide pass over S CTAs and the persistent post cluster of a run.
bool wide_ps_supported(const StepArgs& a, int S);
/// Loads every kernel a streamed run launches (lazy module loading must not
/// happen while the persistent post cluster spins).
void prepare_wide_ps();
void prepare_stream_kernels();
/// True if a kernel on stream b runs while one on stream a is resident
/// (false under kernel-serialising tools: the streamed step then stays off).
bool probe_concurrency(cudaStream_t a, cudaStream_t b);
void launch_wide_ps(const WideTcParamsHost& p, const StepArgs& a, const StreamArgs& r, int S, cudaStream_t s);
/// The 64-column-tile wide pass (k_wide2.cu): the streamed step's persistent
/// kernel and the launched step's cooperative one (same arithmetic).
int wide2_tiles(const StepArgs& a);
bool wide2_supported(const StepArgs& a, int S);
void prepare_wide2();
void launch_wide2_stream(const WideTcParamsHost& p, const StepArgs& a, const StreamArgs& r, int S, cudaStream_t s);
void launch_wide2_step(const WideTcParamsHost& p, const StepArgs& a, cudaStream_t s);
/// 1 if the streamed post cluster (16 CTAs, split mode) can run this model here.
int post_loop_supported(const StepArgs& a);
void launch_post_loop(const StepArgs& a, const StreamArgs& r, cudaStream_t s);
/// Resets the run's StepSync (h of the first step counted as ready).
void launch_stream_init(StepSync* sy, int run_id, unsigned* grid_bar, cudaStream_t s);
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
void launch_gate(const volatile int* flag, cudaStream_t s);
/// dst[r] = src[slots[r]] for n rows of out_pad floats (device pointers).
void launch_gather_rows(const float* src, const unsigned* slots, int n, float* dst, int out_pad, cudaStream_t s);

/// Autoencoder pre-training step (k_ae.cu): one batch of n rows of the AE
/// source slab selected by idx; every pointer device memory.
struct AeArgs {
  ModelArgs m;
  int n;  // batch rows (<= 128)
  int S;  // CTAs of the column passes (split count of Pz / Pg)
  const float* ysrc;     // [N x out_pad] AE source rows
  const unsigned* idx;   // [n] rows of ysrc in this batch
  const float* enc;      // parameter blobs
  const float* dec;
  float* genc;           // gradient blobs (same layout)
  float* gdec;
  float* Pz;             // [S x n x E1]
  float* Pg;             // [S x n x D]
  double* mae_part;      // [S]
  float* z0, *a0, *ga0, *gz0;  // [n x E1]
  float* etz[kMaxLayers];      // enc-tail tape
  float* eta[kMaxLayers];
  float* dhz[kMaxLayers];      // dec-head tape
  float* dha[kMaxLayers];
  float* dzh[kMaxLayers];      // dL/dz per layer of the dec head / enc tail [n x w_{l+1}]
  float* dze[kMaxLayers];      // (row-parallel backward, then the over-rows sums)
  const float* latent;   // enc output [n x lat] (eta[L-1], or a0 if the tail is empty)
  const float* h;        // dec-head output [n x D] (dha[L-1], or latent)
  float* gh;             // dL/dh [n x D]
  float* glat;           // dL/dlatent [n x lat] (gh if the head is empty)
  float* tA, *tB;        // [n x max width] backward scratch
  int* flags;            // [2] non-finite gradient: enc, dec
  double* loss;          // [1]
  float gscale;          // dL/dh = gscale * sum_s Pg[s] (the tcgen05 dec pass leaves 1/n out)
  int prof;              // LTFB_AE_PROF: CTA 0 of the tcgen05 dec pass prints per-tile stamps
};
bool ae_supported(const ModelArgs& m, int rows);
/// K1-K6 of an AE step; ymap (a y tensor map over ysrc, encode_ae_y_map)
/// selects the tcgen05 column passes (k_ae_tc.cu), nullptr the SIMT ones.
void launch_ae_passes(const AeArgs& a, const void* ymap, cudaStream_t s);
bool ae_tc_supported(const ModelArgs& m, int rows);
void encode_ae_y_map(void* map, const float* ysrc, int rows, const ModelArgs& m);
void prepare_ae_tc();
void launch_ae_enc_tc(const void* map, const AeArgs& a, cudaStream_t s);
void launch_ae_dec_tc(const void* map, const AeArgs& a, cudaStream_t s);
void launch_ae_encw_tc(const void* map, const AeArgs& a, cudaStream_t s);
void launch_ae_adam(float* p, float* m1, float* m2, const float* g, long long count, double lr, double b1, double b2,
                    double eps, double c1, double c2, int sms, cudaStream_t s);
/// Adam(enc) then Adam(dec) and their t, applied or skipped on the device
/// from the step's loss and non-finite flags (no host round trip).
void launch_ae_adam_dev(float* const* p, float* const* m1, float* const* m2, float* const* g, const long long* count,
                        const double* lr, double b1, double b2, double eps, const double* adam_c, Counters* ctr,
                        int* flags, const double* loss, int sms, cudaStream_t s);

/// Encodes a 2-D f32 tensor map (128-B swizzle) over [rows x cols].
void encode_tile_map(void* map, const float* base, uint64_t cols, uint64_t rows, uint32_t box_cols,
                     uint32_t box_rows);
/// tcgen05 evaluation of the decoder's wide layer (k_eval_tc.cu).
struct EvalTcHost {
  alignas(64) unsigned char maps[2 * 128];  // slice y, WdT
  const float* bias_pad = nullptr;
  bool ready = false;
};
bool eval_tc_supported(const ModelArgs& m);
void encode_eval_maps(EvalTcHost& h, const float* slice_y, int rows, const float* wdt, const ModelArgs& m);
void launch_eval_tc(const EvalArgs& a, const EvalTcHost& h, bool precise, cudaStream_t s);
std::size_t eval_wide_smem(const ModelArgs& m);
cudaError_t selftest_tc(const float* a1, const float* b1, const float* ah, const float* b2, const float* a3,
                        float* d1, float* d2, float* d3);
/// k_eval_small, then the forward-MAE pass (tcgen05 when tc != nullptr,
/// else the SIMT k_eval_wide), then k_eval_finalize.
void launch_eval(const EvalArgs& a, cudaStream_t s, const EvalTcHost* tc = nullptr, bool precise = true);

/// Device synthetic generator (k_synth.cu; synth/generator.hpp:41-206).
struct SynthArgs {
  const std::uint32_t* ids;   // global sample ids per row (nullptr: first + row)
  std::uint64_t first;
  const double* coeffs;       // [S x 31] per-spec tables (SynthGenerator)
  const double* gain;         // [V x C]
  const double* wavelength;   // [C]
  int S, V, C, H, W;
  unsigned g;                 // grid_side(total_n)
  std::uint64_t sampling_seed;
  float* x;                   // [n x 5]
  float* y;                   // [n x y_stride]
  long long y_stride;
};
void launch_synth(const SynthArgs& a, long long n, cudaStream_t s);
}  // namespace ltfb_dev
namespace ltfb::surrogate { struct ModalityDims; }
namespace ltfb_dev {
/// Rows ids[i] (or first + i when ids is null) of a total_n-point sweep into
/// device x [n x 5] / y [n x y_stride]; the per-spec tables come from the
/// host SynthGenerator. Synchronous on `s`.
void synth_generate_device(const ltfb::surrogate::ModalityDims& dims, std::uint64_t spec_seed,
                           double noise_level, const std::uint32_t* ids, std::uint64_t first,
                           std::size_t n, std::uint64_t total_n, std::uint64_t sampling_seed, float* x,
                           float* y, long long y_stride, cudaStream_t s);

}  // namespace ltfb_dev
