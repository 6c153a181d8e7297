// DeviceTrainer: one LTFB trainer resident on one GPU.
//
// Owns every device buffer of the trainer (parameter blobs and Adam state,
// the HBM data store of its partition, the tournament and validation slices,
// the step intermediates) plus one CUDA stream, and drives the step kernels.
// It is the implementation behind both the C ABI (include/ltfb_gpu.h) and the
// C++ drop-in façade (include/ltfb_b200/trainer.hpp), and mirrors the state
// machine of the reference train::Trainer (train/trainer.hpp:41-308):
// epoch plans, D-then-G steps, numeric skip / abort, epoch records,
// tournament evaluation and generator adoption.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "device_common.cuh"
#include "ltfb_b200/types.hpp"
#include "kernels.hpp"
#include "step_args.cuh"

namespace ltfb_b200 {

void cuda_check(cudaError_t e, const char* what);
#define LTFB_CUDA(x) ::ltfb_b200::cuda_check((x), #x)

/// RAII device guard (cudaSetDevice for the current scope).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev);
  ~DeviceGuard();
};

template <typename T>
struct DevBuf {
  T* p = nullptr;
  std::size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void alloc(std::size_t count) {
    release();
    if (count) LTFB_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  std::size_t bytes() const { return n * sizeof(T); }
};

struct TrainerSpec {
  ltfb::surrogate::ModalityDims dims;
  ltfb::surrogate::SurrogateArch arch;
  int trainer_id = 0;
  int device = 0;
  int n_shards = 1;
  std::size_t batch_size = 128;
  std::uint64_t seed = 0;
  int numeric_abort_threshold = 10;
  double w_f = 1.0, w_i = 1.0;
  double lr[5] = {0, 0, 0, 0, 0};  // 0 = arch.adam.lr
  int wide_kernel = 0;             // 0 auto, 1 generic, 2 tcgen05 3xTF32, 3 tcgen05 TF32
  int post_kernel = 0;  // 0 auto, 1 generic cluster, 2 smem fast path, 3 compile-time shapes
};

struct EvalOut {
  ltfb::surrogate::EvalMetric m[2];
  int adopted = 0;
};

/// Nets are indexed like ltfb_dev::NetId: enc, dec, fwd, inv, disc.
class DeviceTrainer {
 public:
  explicit DeviceTrainer(const TrainerSpec& spec);
  ~DeviceTrainer();
  DeviceTrainer(const DeviceTrainer&) = delete;
  DeviceTrainer& operator=(const DeviceTrainer&) = delete;

  const TrainerSpec& spec() const { return spec_; }
  int device() const { return spec_.device; }
  cudaStream_t stream() const { return stream_; }
  std::size_t param_count(int net) const { return counts_[net]; }
  const ltfb::nn::MlpSpec& net_spec(int net) const { return specs_[net]; }

  // ---- parameters & optimizer state (host <-> HBM, blob layout) ----
  void set_params(int net, const float* blob, std::size_t count);
  void get_params(int net, float* blob, std::size_t count);
  void set_adam(int net, const float* m, const float* v, std::uint64_t t);
  void get_adam(int net, float* m, float* v, std::uint64_t* t);

  // ---- data ----
  /// Uploads the partition (slot i = ids[i]) into the HBM store. `owner`
  /// (optional) is the owning shard per slot for shuffle accounting.
  void load_store(const std::uint32_t* ids, std::size_t n, const float* x, const float* y,
                  const std::int32_t* owner = nullptr);
  /// load_store with the partition rendered on the device by the synthetic
  /// generator (rows ids[i] of a total_n-point sweep; k_synth.cu).
  void generate_store(const std::uint32_t* ids, std::size_t n, const std::int32_t* owner,
                      std::uint64_t spec_seed, double noise_level, std::uint64_t sampling_seed,
                      std::uint64_t total_n);
  void set_slice(int which, const float* x, const float* y, std::size_t rows);  // 0 tour, 1 val
  /// set_slice with the slice rendered on the device.
  void generate_slice(int which, const std::uint32_t* ids, std::size_t rows, std::uint64_t spec_seed,
                      double noise_level, std::uint64_t sampling_seed, std::uint64_t total_n);
  std::size_t slice_rows(int which) const { return which == 0 ? tour_rows_ : val_rows_; }

  // ---- training ----
  /// Runs n steps; appends one record per executed step. Returns false if
  /// the numeric abort threshold was exceeded (records end at that step).
  bool train_steps(std::size_t n, std::vector<ltfb::train::StepRecord>& out);
  std::uint64_t step() const { return host_step_; }
  struct EpochInfo {
    std::uint32_t epoch;
    std::uint64_t steps, samples_shuffled;
    double seconds;
    bool partial;
  };
  /// Closed epoch records (epoch >= 1) produced so far; drains the queue.
  std::vector<EpochInfo> take_epochs();
  /// Closes the in-flight epoch as partial (trainer.hpp:129-134).
  void flush_epoch();

  // ---- tournament / evaluation ----
  /// Evaluates candidates (null pointers = this trainer's own fwd/inv) on
  /// slice `which` (0 tournament, 1 validation).
  EvalOut evaluate(int which, const float* cand_fwd_dev, const float* cand_inv_dev, int nc,
                   bool decide, double w_f, double w_i);
  /// Uploads host blobs into the incoming-generator buffer.
  void set_incoming(const float* fwd, const float* inv);
  /// Device pointers of the own [fwd|inv] generator blob and the incoming one.
  float* generator_dev() { return gen_.p; }
  float* incoming_dev() { return incoming_.p; }
  std::size_t generator_floats() const { return counts_[2] + counts_[3]; }
  /// Evaluate local vs incoming on the tournament slice, decide and adopt
  /// on the device (K3 + K9). Requires the incoming buffer filled.
  EvalOut tournament_decide();
  /// Installs fwd/inv blobs and zeroes their moments, keeping t.
  void adopt(const float* fwd, const float* inv);
  void synchronize();

  // ---- autoencoder pre-training (runner.hpp:249-279) ----
  /// One AE step on rows `rows_idx` (slots of the AE source store).
  double ae_step(const std::uint32_t* rows_idx, std::size_t n);
  void load_ae_source(const float* y, std::size_t n);
  /// Distributed AE (C5: the union of the partitions sharded over the ranks'
  /// stores): a zeroed AE source slab of `rows` rows, filled per step from
  /// the stores (ae_fill_from_store, then an all-gather across ranks).
  void ae_alloc_source(std::size_t rows);
  void ae_fill_from_store(const std::uint32_t* slots, std::size_t n, std::size_t dst_row);
  float* ae_source_dev() { return ae_y_.p; }
  std::size_t ae_source_rows() const { return ae_rows_; }
  int out_pad() const { return margs_.out_pad; }

  // exposed for benchmarks: launches one step without reading back
  void enqueue_steps(std::size_t n);
  /// Device-event timer on this trainer's stream (bench.py timed region).
  /// The region starts behind a gate kernel that the next host enqueue
  /// releases, and ends at the last work enqueued before a host wait, so
  /// host latency at the region's two edges is not device time; gaps the
  /// host loop causes inside the region (record read-back, rounds) are.
  void timer_start();
  double timer_stop_ms();
  /// Host waits on stream_ go through here: the gate is released first, and
  /// a running timer's end mark moves to the work enqueued so far.
  void sync_stream();
  void release_gate();
  void mark_enqueued();
  /// When on, every wide-pass launch is bracketed by CUDA events on the
  /// launching stream; kernel_time() returns (total ms, launches).
  void set_kernel_timing(bool on);
  std::pair<double, std::uint64_t> kernel_time(int which);
  /// e2e path: n steps whose minibatches come from HOST memory (x [n x B x
  /// in], y [n x B x out], rows per step = B); each step's batch is copied
  /// H2D inside the call (double-buffered on a copy stream) and its record
  /// read back D2H.
  bool train_steps_host(std::size_t n, const float* x, const float* y,
                        std::vector<ltfb::train::StepRecord>& out);
  std::size_t wide_ctas() const { return S_; }
  const ltfb_dev::StepArgs& step_args() const { return args_; }
  int wide_kernel_kind() const { return wide_kind_; }
  bool wide2() const { return wide2_; }
  /// Wide part of evaluate() on slice `which`: 2 = k_eval_tc (tcgen05), 1 = SIMT k_eval_wide.
  int eval_kind(int which) const { return eval_tc_[which & 1].ready ? 2 : 1; }
  /// Column passes of ae_step for `rows` batch rows: 2 tcgen05, 1 SIMT.
  int ae_kind(int rows) const;
  /// 1 when store-path steps run as the streamed step (persistent two-phase
  /// wide pass + persistent post cluster per run, launch_stream_run).
  bool stream_mode() const { return stream_on_; }
  /// Stamps the next streamed run and keeps its stage averages (µs): step,
  /// phase 1, h -> phase 2 reduced, phase-2 tiles, phase-2 barrier +
  /// reduction, D-step, post chain after the dec half, steps averaged.
  void stream_profile_next() { stream_prof_next_ = true; }
  const double* stream_profile() const { return stream_prof_; }
  std::uint64_t launch_count() const { return launches_; }

 private:
  void build_model_args();
  void ensure_adam_table(std::uint64_t t_max);
  void start_epoch();
  void launch_step();
  void close_epoch_segment(bool epoch_done, bool partial);
  void launch_step_kernels(bool gather, bool row_h);
  bool next_h_on() const;
  bool h_ready_ = false;  // this step's h / x rows were produced by the previous post kernel
  /// Runs `steps` steps of the current epoch as one cached CUDA graph;
  /// false if graphs are off or capture is unsupported (caller launches).
  bool launch_graph(std::size_t steps);
  /// The cached graph of `steps` steps; row_head: its first step runs the
  /// row kernel (x rows + h) -- needed unless the previous step's post
  /// kernel already produced them (h_ready_).
  cudaGraphExec_t graph_for(std::size_t steps, bool row_head = true);
  static constexpr std::size_t kMaxGraphRun = 32;
  /// Streamed step: `steps` steps of the current epoch as one run of the
  /// persistent post cluster (post_stream_) beside the persistent wide pass
  /// (stream_), which overlap across steps through StepSync hand-offs.
  void launch_stream_run(std::size_t steps);
  void check_stream_error();
  bool stream_on_ = false;
  bool stream_prof_next_ = false;
  double stream_prof_[8] = {};
  int S_stream_ = 0;
  int run_id_ = 0;
  cudaStream_t post_stream_ = nullptr;
  cudaEvent_t st_ev_[2] = {nullptr, nullptr};
  ltfb_dev::StepSync* sync_ = nullptr;
  int* resident_ = nullptr;  // pinned, mapped
  DevBuf<float> red2_;       // red_enc / red_dec of the odd steps of a run
  DevBuf<double> mae2_;
  DevBuf<unsigned long long> prof_;  // LTFB_STREAM_PROF stamps

 public:
  /// Captures (without running) the step graphs of every run length the
  /// step loop uses, so no capture lands inside a timed region.
  void prepare_graphs();

 private:

  TrainerSpec spec_;
  ltfb::nn::MlpSpec specs_[5];
  std::size_t counts_[5] = {};
  ltfb_dev::ModelArgs margs_{};
  ltfb_dev::StepArgs args_{};
  cudaStream_t stream_ = nullptr;
  int sm_count_ = 148;
  std::size_t S_ = 0;
  int wide_kind_ = 1;
  bool post_fast_ = false;
  int post_tpl_ = 0;
  std::uint64_t launches_ = 0;
  bool graphs_on_ = true;
  std::map<std::size_t, cudaGraphExec_t> graphs_;
  std::map<std::size_t, std::uint64_t> graph_launches_;
  ltfb_dev::StepArgs graph_args_{};

  DevBuf<float> params_[5], mom1_[5], mom2_[5], grads_[5];
  DevBuf<float> gen_;       // [fwd | inv] contiguous (exchange payload)
  DevBuf<float> incoming_;  // [fwd | inv] of an incoming generator
  DevBuf<float> sx_, sy_;
  void begin_store(const std::uint32_t* ids, std::size_t n, const std::int32_t* owner);
  void finish_store(std::size_t n);
  void finish_slice(int which, std::size_t rows);
  DevBuf<unsigned> perm_[2];
  DevBuf<float> xb_, yb_, pe_, pd_, scratch_;
  // tcgen05 wide pass: K-major fp32 copies of the frozen wide-layer weights + bias
  DevBuf<float> wide_w_;  // WeT | Wd | WdT | bias (one range for the L2 persistence window)
  ltfb_dev::WideTcParamsHost wtp_{};
  bool wide2_ = false;  // k_wide2 (64-column tiles) is the wide pass of both step modes
  bool wide_dirty_ = false;
  bool small_T_dirty_ = true;  // StepArgs::pT images need a rebuild
  DevBuf<float> pT_[5];
  void prepare_params();
  DevBuf<double> mae_part_, mae_total_, adam_c_;
  DevBuf<ltfb_dev::Counters> ctr_;
  DevBuf<unsigned> grid_bar_;
  DevBuf<ltfb_dev::StepRec> rec_;
  std::uint64_t adam_cap_ = 0;
  std::uint64_t t_host_max_ = 0;  // upper bound of any net's t

  // epoch plan (host)
  std::vector<std::uint32_t> part_ids_;
  std::vector<std::int32_t> owner_;
  std::size_t n_part_ = 0;
  std::uint32_t epoch_ = 0;
  std::size_t step_in_epoch_ = 0, steps_per_epoch_ = 0;
  bool have_plan_ = false;
  std::uint64_t host_step_ = 0;
  std::vector<std::uint32_t> perm_slots_[2];
  unsigned* pinned_perm_[2] = {nullptr, nullptr};
  cudaEvent_t perm_ev_[2] = {nullptr, nullptr};
  // epoch accounting
  std::uint64_t epoch_steps_ = 0, epoch_shuffled_ = 0;
  double epoch_seconds_ = 0;
  std::vector<EpochInfo> closed_;
  // epoch starts enqueued by the current train_steps chunk (host bookkeeping
  // before each), so an abort can roll back what its no-op tail advanced
  struct EpochMark {
    std::uint64_t at_step;
    std::uint32_t epoch;
    std::size_t closed, step_in_epoch;
    std::uint64_t steps, shuffled;
    double seconds;
  };
  std::vector<EpochMark> epoch_marks_;
  bool aborted_ = false;  // the device abort flag was seen: later steps are refused
  std::vector<cudaEvent_t> ev_pool_;  // every event created (destroyed with the trainer)
  std::vector<cudaEvent_t> ev_free_;  // events not in use
  struct Segment {
    cudaEvent_t a, b;
  };
  std::vector<Segment> open_segments_;
  // closed epochs whose device time is not resolved yet: the epoch boundary
  // does not wait for the device (closed_[idx].seconds gets the segments'
  // elapsed times at the next sync, resolve_epoch_times)
  struct PendingEpoch {
    std::size_t idx;
    std::vector<Segment> segs;
  };
  std::vector<PendingEpoch> pending_epochs_;
  void resolve_epoch_times();
  void release_event(cudaEvent_t e) { ev_free_.push_back(e); }
  cudaEvent_t seg_start_ = nullptr;
  bool seg_open_ = false;
  cudaEvent_t next_event();

  // slices
  DevBuf<float> tx_, ty_, vx_, vy_;
  std::size_t tour_rows_ = 0, val_rows_ = 0;
  DevBuf<float> eval_h_;
  DevBuf<double> eval_inv_, eval_part_, eval_out_;
  std::size_t eval_S_ = 0;
  ltfb_dev::EvalTcHost eval_tc_[2];

  // timing
  cudaEvent_t tmr_[2] = {nullptr, nullptr};
  bool timer_on_ = false, timer_marked_ = false;
  int* gate_ = nullptr;  // pinned, mapped
  bool gate_armed_ = false;
  bool ktime_on_ = false;
  static constexpr int kTimed = 5;  // gather, small fwd, wide, post, reduce
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> kev_[kTimed];
  std::size_t kev_used_[kTimed] = {};
  double kms_[kTimed] = {};
  std::uint64_t kcount_[kTimed] = {};
  void kernel_mark(int which, bool begin);
  void resolve_kernel_times();
  // e2e streaming
  cudaStream_t copy_stream_ = nullptr;
  DevBuf<float> hx_[2], hy_[2];
  cudaEvent_t h2d_done_[2] = {nullptr, nullptr}, used_done_[2] = {nullptr, nullptr};

  // AE pre-training (k_ae.cu)
  DevBuf<float> ae_y_;
  DevBuf<unsigned> ae_fill_slots_;
  std::size_t ae_rows_ = 0;
  DevBuf<unsigned> ae_idx_;
  DevBuf<double> ae_loss_;
  DevBuf<float> ae_scr_;
  DevBuf<double> ae_part_;
  DevBuf<int> ae_flags_;
  ltfb_dev::AeArgs ae_args_{};
  bool ae_alloc_ = false;
  alignas(64) unsigned char ae_map_[128] = {};  // gather4 map over ae_y_ (tcgen05 passes)
  struct AePinned {
    std::uint32_t idx[128];
    double loss;
    int flags[2];
  };
  AePinned* ae_pin_ = nullptr;  // pinned staging of the batch index and the step's outcome
  const float* ae_map_base_ = nullptr;
  std::size_t ae_map_rows_ = 0;
  void ae_allocate();
};

}  // namespace ltfb_b200
