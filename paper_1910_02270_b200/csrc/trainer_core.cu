#include <chrono>
#include <thread>
// DeviceTrainer implementation (see trainer_core.hpp).
#include "trainer_core.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "kernels.hpp"
#include "ltfb_b200/host_algos.hpp"
#include "scratch_layout.cuh"

namespace ltfb_b200 {

using ltfb::ContractError;
using ltfb::DimensionError;
using ltfb::Error;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw Error(std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
                ") at " + what);
  }
}

DeviceGuard::DeviceGuard(int dev) {
  cudaGetDevice(&prev);
  if (prev != dev) LTFB_CUDA(cudaSetDevice(dev));
}
DeviceGuard::~DeviceGuard() {
  int cur = -1;
  cudaGetDevice(&cur);
  if (prev >= 0 && cur != prev) cudaSetDevice(prev);
}

namespace {

int act_code(const ltfb::nn::Activation& a) {
  switch (a.kind) {
    case ltfb::nn::Act::kIdentity: return ltfb_dev::kIdentity;
    case ltfb::nn::Act::kRelu: return ltfb_dev::kRelu;
    case ltfb::nn::Act::kLeakyRelu: return ltfb_dev::kLeaky;
    case ltfb::nn::Act::kTanh: return ltfb_dev::kTanh;
    case ltfb::nn::Act::kSigmoid: return ltfb_dev::kSigmoid;
  }
  return ltfb_dev::kIdentity;
}

/// Describes layers [first, last) of `spec` as a small-network descriptor
/// whose offsets index the full blob.
ltfb_dev::NetDesc describe(const ltfb::nn::MlpSpec& spec, std::size_t first, std::size_t last) {
  ltfb_dev::NetDesc d{};
  const auto man = ltfb::nn::manifest_for(spec);
  d.L = static_cast<int>(last - first);
  if (d.L > ltfb_dev::kMaxLayers) throw DimensionError("network has more than 8 small layers");
  for (std::size_t l = first; l < last; ++l) {
    const int i = static_cast<int>(l - first);
    d.w[i] = static_cast<int>(spec.layer_widths[l]);
    d.w[i + 1] = static_cast<int>(spec.layer_widths[l + 1]);
    d.act[i] = act_code(spec.activations[l]);
    d.slope[i] = static_cast<float>(spec.activations[l].slope);
    d.off_w[i] = static_cast<long long>(man.entries[2 * l].offset);
    d.off_b[i] = static_cast<long long>(man.entries[2 * l + 1].offset);
  }
  for (int i = 0; i <= d.L; ++i)
    if (d.L > 0 && d.w[i] > ltfb_dev::kMaxSmallWidth)
      throw DimensionError("small-network width " + std::to_string(d.w[i]) + " exceeds 256");
  if (d.L > 0) {
    d.base = d.off_w[0];
    d.count = static_cast<long long>(man.total) - d.base;
    if (last < spec.n_layers()) d.count = static_cast<long long>(man.entries[2 * last].offset) - d.base;
  }
  return d;
}

}  // namespace

DeviceTrainer::DeviceTrainer(const TrainerSpec& spec) : spec_(spec) {
  if (spec_.n_shards < 1) throw ContractError("Trainer: n_shards must be >= 1");
  if (spec_.batch_size < 1) throw ContractError("Trainer: batch_size must be >= 1");
  spec_.dims.validate();
  DeviceGuard g(spec_.device);
  cudaDeviceProp prop{};
  LTFB_CUDA(cudaGetDeviceProperties(&prop, spec_.device));
  sm_count_ = prop.multiProcessorCount;
  LTFB_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));

  // network specs exactly as make_cyclegan builds them (model.hpp:96-132)
  const auto m = ltfb::surrogate::make_cyclegan<float>(spec_.dims, spec_.arch, 0);
  specs_[0] = m.enc_spec;
  specs_[1] = m.dec_spec;
  specs_[2] = m.fwd_spec;
  specs_[3] = m.inv_spec;
  specs_[4] = m.disc_spec;
  for (int i = 0; i < 5; ++i) counts_[i] = ltfb::nn::manifest_for(specs_[i]).total;
  if (spec_.batch_size > 4096) throw ContractError("Trainer: batch_size above 4096 is not supported on the B200 path");
  build_model_args();

  for (int i = 0; i < 5; ++i) {
    if (i == 2 || i == 3) continue;
    params_[i].alloc(counts_[i]);
  }
  gen_.alloc(counts_[2] + counts_[3]);
  incoming_.alloc(counts_[2] + counts_[3]);
  for (int i = 0; i < 5; ++i) {
    mom1_[i].alloc(counts_[i]);
    mom2_[i].alloc(counts_[i]);
    grads_[i].alloc(counts_[i]);
    LTFB_CUDA(cudaMemsetAsync(mom1_[i].p, 0, mom1_[i].bytes(), stream_));
    LTFB_CUDA(cudaMemsetAsync(mom2_[i].p, 0, mom2_[i].bytes(), stream_));
  }
  const int B = static_cast<int>(spec_.batch_size);
  const auto& ma = margs_;
  // wide-pass kernel: tcgen05 (3xTF32 parity or 1xTF32 fast) where the
  // shape allows it, else the generic SIMT kernel
  {
    ltfb_dev::StepArgs probe{};
    probe.m = ma;
    probe.B = B;
    probe.S = sm_count_;  // one wide-pass CTA per SM
    const bool tc_ok = ltfb_dev::wide_tc_supported(probe);
    if (spec_.wide_kernel == 0) wide_kind_ = tc_ok ? 2 : 1;
    else if (spec_.wide_kernel == 1) wide_kind_ = 1;
    else if (spec_.wide_kernel == 2 || spec_.wide_kernel == 3) {
      if (!tc_ok) throw ContractError("tcgen05 wide kernel requested but unsupported for this shape");
      wide_kind_ = spec_.wide_kernel;
    } else {
      throw ContractError("wide_kernel must be 0 (auto), 1 (generic), 2 (tcgen05 3xTF32) or 3 (tcgen05 TF32)");
    }
  }
  // tcgen05 pass: one CTA per SM, but never more CTAs than 32-column tiles
  // (small dims would otherwise pay for idle CTAs in the grid barrier and the
  // split-K reduction)
  S_ = wide_kind_ >= 2 ? std::min<std::size_t>(static_cast<std::size_t>(sm_count_), (ma.out + 31) / 32)
                       : std::min<std::size_t>((ma.out + 31) / 32, static_cast<std::size_t>(sm_count_) * 2);
  const std::size_t yb_rows = std::max<std::size_t>(B, 128);
  xb_.alloc(static_cast<std::size_t>(B) * ma.in);
  yb_.alloc(yb_rows * ma.out_pad);
  LTFB_CUDA(cudaMemsetAsync(yb_.p, 0, yb_.bytes(), stream_));
  pe_.alloc(S_ * B * ma.E1);
  pd_.alloc(S_ * B * ma.D);
  mae_part_.alloc(S_);
  mae_total_.alloc(1);
  const auto lay = ltfb_dev::make_scratch_layout(ma, B);
  scratch_.alloc(static_cast<std::size_t>(lay.total));
  ctr_.alloc(1);
  LTFB_CUDA(cudaMemsetAsync(ctr_.p, 0, sizeof(ltfb_dev::Counters), stream_));
  // [0..1]: the launched wide pass's barrier; from 64 on: the streamed wide
  // pass's per-CTA release flags (one 128-B line each) and its arrival count
  // (k_wide2's launched mode keeps its own region from 5248 on: epoch base,
  // arrival count, per-CTA flags)
  grid_bar_.alloc(5248 + 64 + 32 * 160);
  LTFB_CUDA(cudaMemsetAsync(grid_bar_.p, 0, grid_bar_.bytes(), stream_));
  rec_.alloc(4096);
  for (int i = 0; i < 2; ++i) {
    LTFB_CUDA(cudaEventCreateWithFlags(&perm_ev_[i], cudaEventDisableTiming));
  }

  auto& a = args_;
  a.m = margs_;
  a.B = B;
  a.S = static_cast<int>(S_);
  a.abort_threshold = spec_.numeric_abort_threshold;
  a.rec_cap = static_cast<int>(rec_.n);
  a.phase_prof = std::getenv("LTFB_PHASE_PROF") ? 1 : 0;
  graphs_on_ = !std::getenv("LTFB_NO_GRAPH") && !a.phase_prof;
  a.small_ctas = std::max(1, (B + 15) / 16);
  const auto& h = spec_.arch.adam;
  for (int i = 0; i < 5; ++i) a.lr[i] = spec_.lr[i] > 0 ? spec_.lr[i] : h.lr;
  a.b1 = h.beta1;
  a.b2 = h.beta2;
  a.eps = h.eps;
  for (int i = 0; i < 5; ++i) {
    a.p[i] = i == 2 ? gen_.p : (i == 3 ? gen_.p + counts_[2] : params_[i].p);
    a.mom1[i] = mom1_[i].p;
    a.mom2[i] = mom2_[i].p;
    a.g[i] = grads_[i].p;
  }
  a.xb = xb_.p;
  a.yb = yb_.p;
  a.P_enc = pe_.p;
  a.P_dec = pd_.p;
  a.mae_part = mae_part_.p;
  a.mae_total = mae_total_.p;
  a.scratch = scratch_.p;
  a.L = lay;
  a.h = scratch_.p + (margs_.dec_head.L > 0 ? lay.ha[margs_.dec_head.L - 1] : lay.fa[margs_.fwd.L - 1]);
  a.ctr = ctr_.p;
  a.grid_bar = grid_bar_.p;
  a.rec = rec_.p;
  ensure_adam_table(1024);

  if (wide_kind_ >= 2) {
    const std::size_t nw = 64 * static_cast<std::size_t>(ma.out_pad);
    // one allocation (WeT | Wd | WdT | bias) so one L2 persistence window covers it
    wide_w_.alloc(3 * nw + static_cast<std::size_t>(ma.out_pad));
    wtp_.precise = wide_kind_ == 2;
    wtp_.wet = wide_w_.p;
    wtp_.wd = wide_w_.p + nw;
    wtp_.wdt = wide_w_.p + 2 * nw;
    wtp_.bias_pad = wide_w_.p + 3 * nw;
    if (!std::getenv("LTFB_NO_L2_PERSIST")) {
      int max_persist = 0, max_window = 0;
      cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, spec_.device);
      cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, spec_.device);
      const std::size_t bytes = std::min<std::size_t>(wide_w_.bytes(), static_cast<std::size_t>(max_window));
      if (max_persist > 0 && bytes > 0) {
        std::size_t cur = 0;
        cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
        const std::size_t want = std::min<std::size_t>(static_cast<std::size_t>(max_persist), std::max(cur, bytes));
        if (want > cur) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
        cudaGetLastError();
        wtp_.l2_base = wide_w_.p;
        wtp_.l2_bytes = bytes;
        wtp_.l2_hit = static_cast<float>(std::min(1.0, static_cast<double>(want) / static_cast<double>(bytes)));
      }
    }
    ltfb_dev::encode_wide_maps(wtp_, a, yb_.p, static_cast<int>(yb_rows));
  }
  // post kernel: compile-time-shaped instance when the model matches one,
  // else the shared-memory fast path, else the generic cluster kernel
  post_tpl_ = spec_.post_kernel == 0 || spec_.post_kernel == 3 ? ltfb_dev::post_tpl_kind(a) : 0;
  if (spec_.post_kernel == 3 && post_tpl_ == 0)
    throw ContractError("post_kernel 3 (compile-time shapes) requested but no instance matches this model");
  if (post_tpl_) {  // W^T images the post kernel stages (and its Adam owners maintain)
    const ltfb_dev::NetDesc* d[5] = {nullptr, &margs_.dec_head, &margs_.fwd, &margs_.inv, &margs_.disc};
    for (int i = 1; i < 5; ++i) {
      pT_[i].alloc(static_cast<std::size_t>(std::max<long long>(1, ltfb_dev::small_T_floats(*d[i]))));
      a.pT[i] = pT_[i].p;
    }
    small_T_dirty_ = true;
  }
  // with the tcgen05 wide pass (which reduces its own partials) and the
  // recomputing post kernel, h comes from the gather kernel and k_pre is skipped
  a.h_in_gather = (wide_kind_ >= 2 && post_tpl_) ? 1 : 0;
  a.x_from_store = 1;
  post_fast_ = post_tpl_ == 0 && (spec_.post_kernel == 0 || spec_.post_kernel == 2) &&
               ltfb_dev::post_fast_supported(a);
  if (spec_.post_kernel == 2 && !post_fast_)
    throw ContractError("post_kernel 2 (shared-memory fast path) requested but unsupported for this model");
  {
    wide_dirty_ = true;
  }
  // streamed step: the post cluster takes 2 x kPostCluster SMs for a whole
  // run, the persistent wide pass the others (and, for one split-K order on
  // every path, so do the launched wide passes)
  {
    const bool tool = std::getenv("CUDA_INJECTION64_PATH") != nullptr;  // ncu / compute-sanitizer serialise kernels
    // the 64-column-tile wide pass (k_wide2) for both step modes, on the SMs
    // the post cluster leaves free; LTFB_WIDE_V1=1 (A/B runs) or a shape
    // k_wide2 does not cover: the 32-column kernels (k_wide_ps streamed,
    // k_wide_tc launched)
    int Ss2 = std::min<int>(sm_count_ - 2 * ltfb_dev::kPostCluster, ltfb_dev::wide2_tiles(a));
    if (const char* ws = std::getenv("LTFB_WIDE_CTAS")) Ss2 = std::max(1, std::min(Ss2, std::atoi(ws)));  // A/B runs
    wide2_ = wide_kind_ >= 2 && !std::getenv("LTFB_WIDE_V1") && ltfb_dev::wide2_supported(a, Ss2);
    const int Ss = wide2_ ? Ss2
                          : std::min<int>(sm_count_ - 2 * ltfb_dev::kPostCluster, static_cast<int>((ma.out + 31) / 32));
    // LTFB_NO_STREAM=1: launched steps; =2: launched steps with the streamed
    // step's wide CTA count (the two paths then sum in the same order)
    const char* ns = std::getenv("LTFB_NO_STREAM");
    const bool able = wide_kind_ >= 2 && post_tpl_ && a.h_in_gather && spec_.n_shards == 1 && !a.phase_prof &&
                      (wide2_ || (static_cast<std::size_t>(Ss) <= (ma.out + 31) / 32 &&
                                  ltfb_dev::wide_ps_supported(a, Ss))) &&
                      ltfb_dev::post_loop_supported(a);
    stream_on_ = able && !ns && !tool;
    if (wide2_ || (able && (stream_on_ || tool || (ns && ns[0] == '2')))) {
      S_ = static_cast<std::size_t>(Ss);
      a.S = Ss;
    }
    if (stream_on_) {
      S_stream_ = Ss;
      LTFB_CUDA(cudaMalloc(reinterpret_cast<void**>(&sync_), sizeof(ltfb_dev::StepSync)));
      LTFB_CUDA(cudaMemsetAsync(sync_, 0, sizeof(ltfb_dev::StepSync), stream_));
      LTFB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&resident_), sizeof(int), cudaHostAllocMapped));
      *reinterpret_cast<volatile int*>(resident_) = 0;
      red2_.alloc(static_cast<std::size_t>(B) * (ma.E1 + ma.D));
      mae2_.alloc(1);
      LTFB_CUDA(cudaStreamCreateWithFlags(&post_stream_, cudaStreamNonBlocking));
      for (auto& e : st_ev_) LTFB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ltfb_dev::prepare_stream_kernels();
      // the two persistent kernels must run side by side: a tool that
      // serialises kernels (ncu kernel replay, compute-sanitizer) or a
      // shared GPU turns the streamed step off here, not in a 2 s hand-off timeout
      if (!ltfb_dev::probe_concurrency(stream_, post_stream_)) stream_on_ = false;
    }
  }
  sync_stream();
}

DeviceTrainer::~DeviceTrainer() {
  DeviceGuard g(spec_.device);
  release_gate();
  if (stream_) cudaStreamSynchronize(stream_);
  if (post_stream_) {
    cudaStreamSynchronize(post_stream_);
    cudaStreamDestroy(post_stream_);
  }
  for (auto e : st_ev_)
    if (e) cudaEventDestroy(e);
  if (sync_) cudaFree(sync_);
  if (resident_) cudaFreeHost(resident_);
  if (ae_pin_) cudaFreeHost(ae_pin_);
  if (gate_) cudaFreeHost(gate_);
  for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second);
  for (int i = 0; i < 2; ++i) {
    if (pinned_perm_[i]) cudaFreeHost(pinned_perm_[i]);
    if (perm_ev_[i]) cudaEventDestroy(perm_ev_[i]);
  }
  for (auto e : ev_pool_) cudaEventDestroy(e);
  for (auto e : tmr_)
    if (e) cudaEventDestroy(e);
  for (auto& v : kev_)
    for (auto& pr : v) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  for (int i = 0; i < 2; ++i) {
    if (h2d_done_[i]) cudaEventDestroy(h2d_done_[i]);
    if (used_done_[i]) cudaEventDestroy(used_done_[i]);
  }
  if (copy_stream_) {
    cudaStreamSynchronize(copy_stream_);
    cudaStreamDestroy(copy_stream_);
  }
  if (stream_) cudaStreamDestroy(stream_);
}

void DeviceTrainer::build_model_args() {
  auto& m = margs_;
  m.in = static_cast<int>(spec_.dims.input_dim);
  m.lat = static_cast<int>(spec_.dims.latent_dim);
  m.out = static_cast<int>(spec_.dims.output_dim());
  m.out_pad = (m.out + 3) / 4 * 4;
  const auto& enc = specs_[0];
  const auto& dec = specs_[1];
  const auto em = ltfb::nn::manifest_for(enc);
  const auto dm = ltfb::nn::manifest_for(dec);
  m.E1 = static_cast<int>(enc.layer_widths[1]);
  m.enc_act0 = act_code(enc.activations[0]);
  m.enc_slope0 = static_cast<float>(enc.activations[0].slope);
  m.enc_wide_w = static_cast<long long>(em.entries[0].offset);
  m.enc_wide_b = static_cast<long long>(em.entries[1].offset);
  m.enc_tail = describe(enc, 1, enc.n_layers());
  const std::size_t dl = dec.n_layers() - 1;
  m.D = static_cast<int>(dec.layer_widths[dl]);
  m.dec_wide_w = static_cast<long long>(dm.entries[2 * dl].offset);
  m.dec_wide_b = static_cast<long long>(dm.entries[2 * dl + 1].offset);
  m.dec_head = describe(dec, 0, dl);
  m.fwd = describe(specs_[2], 0, specs_[2].n_layers());
  m.inv = describe(specs_[3], 0, specs_[3].n_layers());
  m.disc = describe(specs_[4], 0, specs_[4].n_layers());
  if (m.E1 > ltfb_dev::kMaxSmallWidth || m.D > ltfb_dev::kMaxSmallWidth)
    throw DimensionError("wide-layer inner width above 256 is not supported on the B200 path");
  m.lambda_adv = static_cast<float>(spec_.arch.lambda_adv);
  m.lambda_cyc = static_cast<float>(spec_.arch.lambda_cyc);
}

void DeviceTrainer::ensure_adam_table(std::uint64_t t_max) {
  if (t_max + 1 <= adam_cap_) return;
  std::uint64_t cap = std::max<std::uint64_t>(1024, adam_cap_ * 2);
  while (cap < t_max + 1) cap *= 2;
  // nn/adam.hpp:113-116: 1 - std::pow(beta, t) in double on the host
  std::vector<double> tab(2 * cap);
  const auto& h = spec_.arch.adam;
  for (std::uint64_t t = 0; t < cap; ++t) {
    tab[2 * t] = 1.0 - std::pow(h.beta1, static_cast<double>(t));
    tab[2 * t + 1] = 1.0 - std::pow(h.beta2, static_cast<double>(t));
  }
  DevBuf<double> nb;
  nb.alloc(tab.size());
  LTFB_CUDA(cudaMemcpyAsync(nb.p, tab.data(), nb.bytes(), cudaMemcpyHostToDevice, stream_));
  sync_stream();
  std::swap(adam_c_.p, nb.p);
  std::swap(adam_c_.n, nb.n);
  adam_cap_ = cap;
  args_.adam_c = adam_c_.p;
  args_.adam_cap = static_cast<long long>(cap);
}

// ------------------------------------------------------------ parameters --
static float* net_ptr(DeviceTrainer& t, DevBuf<float>* params, DevBuf<float>& gen, int net,
                      std::size_t c2) {
  (void)t;
  if (net == 2) return gen.p;
  if (net == 3) return gen.p + c2;
  return params[net].p;
}

void DeviceTrainer::set_params(int net, const float* blob, std::size_t count) {
  if (net == 0 || net == 1) wide_dirty_ = true;
  small_T_dirty_ = true;
  h_ready_ = false;
  if (net < 0 || net > 4) throw ContractError("set_params: bad network index");
  if (count != counts_[net])
    throw ContractError("blob length " + std::to_string(count) + " does not match manifest total " +
                        std::to_string(counts_[net]));
  DeviceGuard g(spec_.device);
  LTFB_CUDA(cudaMemcpyAsync(net_ptr(*this, params_, gen_, net, counts_[2]), blob, count * 4,
                            cudaMemcpyHostToDevice, stream_));
  sync_stream();
}

void DeviceTrainer::get_params(int net, float* blob, std::size_t count) {
  if (net < 0 || net > 4) throw ContractError("get_params: bad network index");
  if (count != counts_[net]) throw ContractError("get_params: wrong blob length");
  DeviceGuard g(spec_.device);
  LTFB_CUDA(cudaMemcpyAsync(blob, net_ptr(*this, params_, gen_, net, counts_[2]), count * 4,
                            cudaMemcpyDeviceToHost, stream_));
  sync_stream();
}

void DeviceTrainer::set_adam(int net, const float* m, const float* v, std::uint64_t t) {
  if (net < 0 || net > 4) throw ContractError("set_adam: bad network index");
  DeviceGuard g(spec_.device);
  const std::size_t n = counts_[net];
  if (m) LTFB_CUDA(cudaMemcpyAsync(mom1_[net].p, m, n * 4, cudaMemcpyHostToDevice, stream_));
  if (v) LTFB_CUDA(cudaMemcpyAsync(mom2_[net].p, v, n * 4, cudaMemcpyHostToDevice, stream_));
  LTFB_CUDA(cudaMemcpyAsync(&ctr_.p->t[net], &t, 8, cudaMemcpyHostToDevice, stream_));
  sync_stream();
  t_host_max_ = std::max(t_host_max_, t);
}

void DeviceTrainer::get_adam(int net, float* m, float* v, std::uint64_t* t) {
  if (net < 0 || net > 4) throw ContractError("get_adam: bad network index");
  DeviceGuard g(spec_.device);
  const std::size_t n = counts_[net];
  if (m) LTFB_CUDA(cudaMemcpyAsync(m, mom1_[net].p, n * 4, cudaMemcpyDeviceToHost, stream_));
  if (v) LTFB_CUDA(cudaMemcpyAsync(v, mom2_[net].p, n * 4, cudaMemcpyDeviceToHost, stream_));
  std::uint64_t tt = 0;
  LTFB_CUDA(cudaMemcpyAsync(&tt, &ctr_.p->t[net], 8, cudaMemcpyDeviceToHost, stream_));
  sync_stream();
  if (t) *t = tt;
}

// ------------------------------------------------------------------ data --
void DeviceTrainer::begin_store(const std::uint32_t* ids, std::size_t n, const std::int32_t* owner) {
  h_ready_ = false;
  if (n == 0) throw ContractError("plan_epoch: empty partition");
  const auto& m = margs_;
  part_ids_.assign(ids, ids + n);
  owner_.assign(n, 0);
  if (owner) owner_.assign(owner, owner + n);
  n_part_ = n;
  sx_.alloc(n * m.in);
  sy_.alloc(n * m.out_pad);
}

void DeviceTrainer::finish_store(std::size_t n) {
  for (int i = 0; i < 2; ++i) {
    perm_[i].alloc(n);
    if (pinned_perm_[i]) cudaFreeHost(pinned_perm_[i]);
    LTFB_CUDA(cudaMallocHost(&pinned_perm_[i], n * sizeof(unsigned)));
    perm_slots_[i].resize(n);
  }
  auto& a = args_;
  a.sx = sx_.p;
  a.sy = sy_.p;
  a.perm[0] = perm_[0].p;
  a.perm[1] = perm_[1].p;
  a.n_part = static_cast<int>(n);
  if (wide_kind_ >= 2) ltfb_dev::encode_y_map(wtp_, -1, sy_.p, a, static_cast<int>(n));  // gather4 source
  steps_per_epoch_ = (n + spec_.batch_size - 1) / spec_.batch_size;
  sync_stream();
}

void DeviceTrainer::load_store(const std::uint32_t* ids, std::size_t n, const float* x,
                               const float* y, const std::int32_t* owner) {
  DeviceGuard g(spec_.device);
  begin_store(ids, n, owner);
  const auto& m = margs_;
  LTFB_CUDA(cudaMemcpyAsync(sx_.p, x, n * m.in * 4, cudaMemcpyHostToDevice, stream_));
  if (m.out_pad == m.out) {
    LTFB_CUDA(cudaMemcpyAsync(sy_.p, y, n * m.out * 4, cudaMemcpyHostToDevice, stream_));
  } else {
    LTFB_CUDA(cudaMemsetAsync(sy_.p, 0, sy_.bytes(), stream_));
    LTFB_CUDA(cudaMemcpy2DAsync(sy_.p, m.out_pad * 4, y, m.out * 4, m.out * 4, n,
                                cudaMemcpyHostToDevice, stream_));
  }
  finish_store(n);
}

void DeviceTrainer::generate_store(const std::uint32_t* ids, std::size_t n, const std::int32_t* owner,
                                   std::uint64_t spec_seed, double noise_level,
                                   std::uint64_t sampling_seed, std::uint64_t total_n) {
  DeviceGuard g(spec_.device);
  for (std::size_t i = 0; i < n; ++i)
    if (ids[i] >= total_n) throw ContractError("DataStore: partition id outside dataset");
  begin_store(ids, n, owner);
  const auto& m = margs_;
  if (m.out_pad != m.out) LTFB_CUDA(cudaMemsetAsync(sy_.p, 0, sy_.bytes(), stream_));
  ltfb_dev::synth_generate_device(spec_.dims, spec_seed, noise_level, ids, 0, n, total_n, sampling_seed,
                                  sx_.p, sy_.p, m.out_pad, stream_);
  finish_store(n);
}

void DeviceTrainer::set_slice(int which, const float* x, const float* y, std::size_t rows) {
  DeviceGuard g(spec_.device);
  const auto& m = margs_;
  DevBuf<float>& bx = which == 0 ? tx_ : vx_;
  DevBuf<float>& by = which == 0 ? ty_ : vy_;
  bx.alloc(rows * m.in);
  by.alloc(rows * m.out_pad);
  if (rows) {
    LTFB_CUDA(cudaMemcpyAsync(bx.p, x, rows * m.in * 4, cudaMemcpyHostToDevice, stream_));
    LTFB_CUDA(cudaMemsetAsync(by.p, 0, by.bytes(), stream_));
    LTFB_CUDA(cudaMemcpy2DAsync(by.p, m.out_pad * 4, y, m.out * 4, m.out * 4, rows,
                                cudaMemcpyHostToDevice, stream_));
  }
  finish_slice(which, rows);
}

void DeviceTrainer::generate_slice(int which, const std::uint32_t* ids, std::size_t rows,
                                   std::uint64_t spec_seed, double noise_level, std::uint64_t sampling_seed,
                                   std::uint64_t total_n) {
  DeviceGuard g(spec_.device);
  for (std::size_t i = 0; i < rows; ++i)
    if (ids[i] >= total_n) throw ContractError("slice id outside dataset");
  const auto& m = margs_;
  DevBuf<float>& bx = which == 0 ? tx_ : vx_;
  DevBuf<float>& by = which == 0 ? ty_ : vy_;
  bx.alloc(rows * m.in);
  by.alloc(rows * m.out_pad);
  if (rows) {
    LTFB_CUDA(cudaMemsetAsync(by.p, 0, by.bytes(), stream_));
    ltfb_dev::synth_generate_device(spec_.dims, spec_seed, noise_level, ids, 0, rows, total_n, sampling_seed,
                                    bx.p, by.p, m.out_pad, stream_);
  }
  finish_slice(which, rows);
}

void DeviceTrainer::finish_slice(int which, std::size_t rows) {
  const auto& m = margs_;
  DevBuf<float>& by = which == 0 ? ty_ : vy_;
  (which == 0 ? tour_rows_ : val_rows_) = rows;
  // tcgen05 eval maps over this slice (weights: the wide pass's K-major copy)
  eval_tc_[which].ready = false;
  if (rows && wide_kind_ >= 2 && ltfb_dev::eval_tc_supported(margs_) && !std::getenv("LTFB_EVAL_SIMT")) {
    ltfb_dev::encode_eval_maps(eval_tc_[which], by.p, static_cast<int>(rows), wtp_.wdt, m);
    eval_tc_[which].bias_pad = wtp_.bias_pad;
    eval_tc_[which].ready = true;
  }
  const std::size_t mx = std::max(tour_rows_, val_rows_);
  if (eval_h_.n < 2 * mx * m.D) {
    eval_h_.alloc(2 * mx * m.D);
    eval_inv_.alloc(2 * mx);
  }
  eval_S_ = static_cast<std::size_t>(sm_count_) * 2;
  if (eval_part_.n < eval_S_ * 2) eval_part_.alloc(eval_S_ * 2);
  if (!eval_out_.p) eval_out_.alloc(6);
  sync_stream();
}

// -------------------------------------------------------------- training --
cudaEvent_t DeviceTrainer::next_event() {
  if (!ev_free_.empty()) {
    cudaEvent_t e = ev_free_.back();
    ev_free_.pop_back();
    return e;
  }
  cudaEvent_t e;
  LTFB_CUDA(cudaEventCreate(&e));
  ev_pool_.push_back(e);
  return e;
}

void DeviceTrainer::resolve_epoch_times() {
  if (pending_epochs_.empty()) return;
  sync_stream();
  for (auto& pe : pending_epochs_) {
    double sec = 0;
    for (const auto& sg : pe.segs) {
      float ms = 0;
      LTFB_CUDA(cudaEventElapsedTime(&ms, sg.a, sg.b));
      sec += ms * 1e-3;
      release_event(sg.a);
      release_event(sg.b);
    }
    if (pe.idx < closed_.size()) closed_[pe.idx].seconds += sec;
  }
  pending_epochs_.clear();
}

void DeviceTrainer::close_epoch_segment(bool epoch_done, bool partial) {
  if (seg_open_) {
    cudaEvent_t e = next_event();
    LTFB_CUDA(cudaEventRecord(e, stream_));
    open_segments_.push_back({seg_start_, e});
    seg_open_ = false;
  }
  if (epoch_done) {
    // this epoch's segments (all recorded on stream_) are timed at the next
    // sync (resolve_epoch_times), so the boundary does not drain the device
    closed_.push_back({epoch_, epoch_steps_, epoch_shuffled_, epoch_seconds_, partial});
    pending_epochs_.push_back({closed_.size() - 1, std::move(open_segments_)});
    open_segments_.clear();
    epoch_steps_ = epoch_shuffled_ = 0;
    epoch_seconds_ = 0;
  }
}

void DeviceTrainer::start_epoch() {
  h_ready_ = false;
  if (have_plan_) close_epoch_segment(true, false);
  epoch_ += 1;
  const int buf = static_cast<int>(epoch_ & 1);
  // epoch_plan.hpp:69-71: shuffle(partition) == partition[shuffle(iota)],
  // because the Fisher-Yates swaps depend only on the length.
  auto& slots = perm_slots_[buf];
  for (std::size_t i = 0; i < n_part_; ++i) slots[i] = static_cast<std::uint32_t>(i);
  ltfb::Rng(ltfb::mix_seed({spec_.seed, epoch_, 0x5caff1eULL})).shuffle(slots);
  release_gate();
  LTFB_CUDA(cudaEventSynchronize(perm_ev_[buf]));  // previous use of this pinned buffer
  std::memcpy(pinned_perm_[buf], slots.data(), n_part_ * sizeof(unsigned));
  LTFB_CUDA(cudaMemcpyAsync(perm_[buf].p, pinned_perm_[buf], n_part_ * sizeof(unsigned),
                            cudaMemcpyHostToDevice, stream_));
  LTFB_CUDA(cudaEventRecord(perm_ev_[buf], stream_));
  ltfb_dev::launch_begin_epoch(ctr_.p, epoch_, stream_);
  ++launches_;
  step_in_epoch_ = 0;
  have_plan_ = true;
}

void DeviceTrainer::launch_step() {
  launch_step_kernels(true, !h_ready_);
  h_ready_ = next_h_on() && step_in_epoch_ + 1 < steps_per_epoch_;
}

// kernel ids for per-kernel timing: 0 gather, 1 pre, 2 wide, 3 post, 4 reduce
void DeviceTrainer::kernel_mark(int which, bool begin) {
  if (!ktime_on_) return;
  auto& v = kev_[which];
  auto& used = kev_used_[which];
  if (begin) {
    if (used == v.size()) {
      cudaEvent_t a, b;
      LTFB_CUDA(cudaEventCreate(&a));
      LTFB_CUDA(cudaEventCreate(&b));
      v.push_back({a, b});
    }
    LTFB_CUDA(cudaEventRecord(v[used].first, stream_));
  } else {
    LTFB_CUDA(cudaEventRecord(v[used].second, stream_));
    ++used;
  }
}

void DeviceTrainer::resolve_kernel_times() {
  for (int k = 0; k < kTimed; ++k) {
    for (std::size_t i = 0; i < kev_used_[k]; ++i) {
      float ms = 0;
      LTFB_CUDA(cudaEventElapsedTime(&ms, kev_[k][i].first, kev_[k][i].second));
      kms_[k] += ms;
      ++kcount_[k];
    }
    kev_used_[k] = 0;
  }
}

void DeviceTrainer::prepare_params() {
  if (wide_kind_ >= 2 && wide_dirty_) {
    ltfb_dev::launch_prep_wide(args_, wtp_, stream_);
    ++launches_;
    wide_dirty_ = false;
  }
  if (post_tpl_ && small_T_dirty_) {
    ltfb_dev::launch_build_T(args_, stream_);
    ++launches_;
    small_T_dirty_ = false;
  }
}

bool DeviceTrainer::next_h_on() const { return wide_kind_ >= 2 && post_tpl_ && args_.h_in_gather; }

void DeviceTrainer::launch_step_kernels(bool gather, bool row_h) {
  // gather == true: the minibatch comes from the HBM store through the epoch
  // plan; false: it was streamed into xb / the y buffer by the host path.
  // row_h == false: the previous step's post kernel already produced this
  // step's h and x rows (post_next_h), so the row kernel is skipped.
  prepare_params();
  std::uint64_t n = 0;
  if (wide_kind_ >= 2) {
    // tcgen05 wide pass gathers y rows from the store itself (tile::gather4);
    // one small kernel brings the x rows and computes h = dec_head(fwd(x))
    if (!(gather && !row_h && next_h_on())) {
      kernel_mark(0, true);
      ltfb_dev::launch_row_h(args_, gather, stream_);
      kernel_mark(0, false);
      ++n;
    }
  } else if (gather) {
    kernel_mark(0, true);
    ltfb_dev::launch_gather(args_, stream_);
    kernel_mark(0, false);
    ++n;
  }
  if (!args_.h_in_gather) {  // k_pre: h and the small-net tapes for the generic post kernels
    kernel_mark(1, true);
    ltfb_dev::launch_pre(args_, stream_);
    kernel_mark(1, false);
    ++n;
  }
  kernel_mark(2, true);
  if (wide_kind_ >= 2 && wide2_) ltfb_dev::launch_wide2_step(wtp_, args_, stream_);
  else if (wide_kind_ >= 2) ltfb_dev::launch_wide_tc_params(wtp_, args_, stream_);
  else ltfb_dev::launch_wide_generic(args_, stream_);
  kernel_mark(2, false);
  ++n;
  if (wide_kind_ < 2) {  // the tcgen05 wide pass reduces its split-K partials itself
    kernel_mark(4, true);
    ltfb_dev::launch_reduce(args_, stream_);
    kernel_mark(4, false);
    ++n;
  }
  kernel_mark(3, true);
  if (post_tpl_) {
    ltfb_dev::StepArgs b = args_;
    b.post_next_h = gather && next_h_on() ? 1 : 0;
    ltfb_dev::launch_post_tpl(post_tpl_, b, stream_);
  }
  else if (post_fast_) ltfb_dev::launch_post_fast(args_, stream_);
  else ltfb_dev::launch_post(args_, stream_);
  kernel_mark(3, false);
  launches_ += n + 1;
}

void DeviceTrainer::timer_start() {
  DeviceGuard g(spec_.device);
  for (auto& e : tmr_)
    if (!e) LTFB_CUDA(cudaEventCreate(&e));
  if (!gate_) LTFB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&gate_), sizeof(int), cudaHostAllocMapped));
  release_gate();
  *reinterpret_cast<volatile int*>(gate_) = 0;
  int* dflag = nullptr;
  LTFB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dflag), gate_, 0));
  ltfb_dev::launch_gate(dflag, stream_);
  gate_armed_ = true;
  LTFB_CUDA(cudaEventRecord(tmr_[0], stream_));
  timer_on_ = true;
  timer_marked_ = false;
}

void DeviceTrainer::release_gate() {
  if (gate_armed_) {
    *reinterpret_cast<volatile int*>(gate_) = 1;
    gate_armed_ = false;
  }
}

void DeviceTrainer::mark_enqueued() {
  if (timer_on_) {
    LTFB_CUDA(cudaEventRecord(tmr_[1], stream_));
    timer_marked_ = true;
  }
}

void DeviceTrainer::sync_stream() {
  mark_enqueued();
  release_gate();
  LTFB_CUDA(cudaStreamSynchronize(stream_));
}

double DeviceTrainer::timer_stop_ms() {
  DeviceGuard g(spec_.device);
  if (!timer_marked_) LTFB_CUDA(cudaEventRecord(tmr_[1], stream_));
  release_gate();
  timer_on_ = false;
  LTFB_CUDA(cudaEventSynchronize(tmr_[1]));
  float ms = 0;
  LTFB_CUDA(cudaEventElapsedTime(&ms, tmr_[0], tmr_[1]));
  return ms;
}

void DeviceTrainer::set_kernel_timing(bool on) {
  DeviceGuard g(spec_.device);
  sync_stream();
  resolve_kernel_times();
  for (int k = 0; k < kTimed; ++k) {
    kms_[k] = 0;
    kcount_[k] = 0;
  }
  ktime_on_ = on;
}

std::pair<double, std::uint64_t> DeviceTrainer::kernel_time(int which) {
  DeviceGuard g(spec_.device);
  sync_stream();
  resolve_kernel_times();
  return {kms_[which], kcount_[which]};
}

void DeviceTrainer::enqueue_steps(std::size_t n) {
  DeviceGuard g(spec_.device);
  if (n_part_ == 0) throw ContractError("train_steps: data store is empty");
  ensure_adam_table(t_host_max_ + host_step_ + n + 1);
  for (std::size_t i = 0; i < n; ++i) {
    if (!have_plan_ || step_in_epoch_ >= steps_per_epoch_) {
      epoch_marks_.push_back(
          {host_step_, epoch_, closed_.size(), step_in_epoch_, epoch_steps_, epoch_shuffled_, epoch_seconds_});
      start_epoch();
    }
    if (!seg_open_) {
      seg_start_ = next_event();
      LTFB_CUDA(cudaEventRecord(seg_start_, stream_));
      seg_open_ = true;
    }
    // data/store.hpp:314-318: deliveries whose owner differs from the
    // consuming shard are counted as shuffled samples.
    const std::size_t begin = step_in_epoch_ * spec_.batch_size;
    const std::size_t rows = std::min(spec_.batch_size, n_part_ - begin);
    if (spec_.n_shards > 1) {
      const auto ranges = ltfb::data::shard_split(rows, spec_.n_shards);
      const auto& slots = perm_slots_[epoch_ & 1];
      for (int s = 0; s < spec_.n_shards; ++s)
        for (std::size_t r = ranges[s].first; r < ranges[s].second; ++r)
          if (owner_[slots[begin + r]] >= 0 && owner_[slots[begin + r]] != s) ++epoch_shuffled_;
    }
    if (stream_on_ && !ktime_on_) {  // streamed step: the rest of this epoch (or of n) as one run
      const std::size_t srun = std::min<std::size_t>(n - i, steps_per_epoch_ - step_in_epoch_);
      launch_stream_run(srun);
      step_in_epoch_ += srun;
      epoch_steps_ += srun;
      host_step_ += srun;
      i += srun - 1;
      continue;
    }
    // a run of steps inside this epoch goes out as one CUDA graph launch
    // runs are powers of two (<= kMaxGraphRun) so a handful of cached
    // graphs covers every position in every epoch
    std::size_t run = std::min<std::size_t>({n - i, steps_per_epoch_ - step_in_epoch_, kMaxGraphRun});
    while (run & (run - 1)) run &= run - 1;
    if (run >= 2 && spec_.n_shards == 1 && launch_graph(run)) {
      step_in_epoch_ += run;
      epoch_steps_ += run;
      host_step_ += run;
      i += run - 1;
      continue;
    }
    launch_step();
    ++step_in_epoch_;
    ++epoch_steps_;
    ++host_step_;
  }
  LTFB_CUDA(cudaGetLastError());
}

void DeviceTrainer::prepare_graphs() {
  DeviceGuard g(spec_.device);
  if (!graphs_on_ || ktime_on_ || spec_.n_shards != 1) return;
  prepare_params();
  for (std::size_t s = 2; s <= kMaxGraphRun; s *= 2)
    for (const bool head : {true, false})
      if ((head || next_h_on()) && !graph_for(s, head)) return;
}

cudaGraphExec_t DeviceTrainer::graph_for(std::size_t steps, bool row_head) {
  row_head = row_head || !next_h_on();
  const std::size_t key = 2 * steps + (row_head ? 1 : 0);
  if (std::memcmp(&graph_args_, &args_, sizeof args_) != 0) {  // pointers or layout changed
    for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second);
    graphs_.clear();
    graph_args_ = args_;
  }
  auto it = graphs_.find(key);
  if (it == graphs_.end()) {
    const std::uint64_t l0 = launches_;
    cudaGraph_t graph = nullptr;
    if (cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      graphs_on_ = false;
      return nullptr;
    }
    for (std::size_t k = 0; k < steps; ++k) launch_step_kernels(true, k == 0 && row_head);
    const cudaError_t e = cudaStreamEndCapture(stream_, &graph);
    cudaGraphExec_t exec = nullptr;
    if (e != cudaSuccess || cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      graphs_on_ = false;  // capture unsupported here: plain launches from now on
      launches_ = l0;
      return nullptr;
    }
    cudaGraphDestroy(graph);
    graph_launches_[key] = launches_ - l0;
    launches_ = l0;
    it = graphs_.emplace(key, exec).first;
  }
  return it->second;
}

bool DeviceTrainer::launch_graph(std::size_t steps) {
  if (!graphs_on_ || ktime_on_) return false;
  prepare_params();  // weight re-layouts stay outside the graph
  const bool head = !h_ready_ || !next_h_on();
  cudaGraphExec_t exec = graph_for(steps, head);
  if (!exec) return false;
  LTFB_CUDA(cudaGraphLaunch(exec, stream_));
  h_ready_ = next_h_on() && step_in_epoch_ + steps < steps_per_epoch_;
  launches_ += graph_launches_[2 * steps + (head ? 1 : 0)];
  return true;
}

void DeviceTrainer::launch_stream_run(std::size_t steps) {
  prepare_params();  // weight re-layouts / W^T images before the run
  if (!h_ready_) {   // h / x rows of the run's first step
    ltfb_dev::launch_row_h(args_, true, stream_);
    ++launches_;
  }
  ++run_id_;
  ltfb_dev::launch_stream_init(sync_, run_id_, grid_bar_.p, stream_);
  ltfb_dev::StreamArgs r{};
  r.n = static_cast<int>(steps);
  r.sie0 = static_cast<int>(step_in_epoch_);
  r.epoch = epoch_;
  r.run_id = run_id_;
  r.S_wide = S_stream_;
  r.sync = sync_;
  LTFB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&r.resident_host), resident_, 0));
  const int B = args_.B;
  r.red_enc[0] = args_.scratch + args_.L.red_enc;
  r.red_dec[0] = args_.scratch + args_.L.red_dec;
  r.red_enc[1] = red2_.p;
  r.red_dec[1] = red2_.p + static_cast<std::size_t>(B) * margs_.E1;
  r.mae_total[0] = args_.mae_total;
  r.mae_total[1] = mae2_.p;
  // an armed profile waits for a run long enough to average (>= 8 steps)
  const bool prof = std::getenv("LTFB_STREAM_PROF") != nullptr || (stream_prof_next_ && steps >= 8);
  if (prof) stream_prof_next_ = false;
  if (prof) {
    if (prof_.n < 512 * steps + 256) prof_.alloc(512 * steps + 256);
    LTFB_CUDA(cudaMemsetAsync(prof_.p, 0, prof_.bytes(), stream_));
    r.prof = prof_.p;
  }
  // the post cluster first (it starts behind everything queued on stream_),
  // then -- once it is resident, so the cooperative wide pass finds exactly
  // its SMs free -- the wide pass on stream_; stream_ then joins post_stream_
  LTFB_CUDA(cudaEventRecord(st_ev_[0], stream_));
  LTFB_CUDA(cudaStreamWaitEvent(post_stream_, st_ev_[0], 0));
  ltfb_dev::launch_post_loop(args_, r, post_stream_);
  if (wide2_) {
    // programmatic dependent launch right behind the cluster on its stream:
    // the device starts the wide pass once the cluster is resident (no host
    // wait between the launches, so the host can run ahead of the device)
    ltfb_dev::launch_wide2_stream(wtp_, args_, r, S_stream_, post_stream_);
    release_gate();
  } else {
    release_gate();
    const auto t0 = std::chrono::steady_clock::now();
    while (*reinterpret_cast<volatile int*>(resident_) != run_id_) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(20)) {
        stream_on_ = false;
        throw ltfb::Error("CUDA error: streamed step: the post cluster did not become resident");
      }
      std::this_thread::yield();
    }
    ltfb_dev::launch_wide_ps(wtp_, args_, r, S_stream_, stream_);
  }
  LTFB_CUDA(cudaEventRecord(st_ev_[1], post_stream_));
  LTFB_CUDA(cudaStreamWaitEvent(stream_, st_ev_[1], 0));
  launches_ += 3;
  h_ready_ = next_h_on() && step_in_epoch_ + steps < steps_per_epoch_;
  if (std::getenv("LTFB_STREAM_DEBUG") || prof) {
    sync_stream();
    check_stream_error();
  }
  if (prof) {  // per-step stage times (us) relative to the wide pass's phase-1 start of each step
    std::vector<unsigned long long> h(512 * steps);
    LTFB_CUDA(cudaMemcpy(h.data(), prof_.p, h.size() * 8, cudaMemcpyDeviceToHost));
    static const char* names[32] = {"w.p1", "w.p1red", "w.p2", "w.p2prod", "w.p2red", "w.hwait", "-", "c.decwait",
                                    "d.start", "d.encwait", "d.S1", "d.dupd", "d.gupd", "d.S6", "d.nexth", "c.end",
                                    "m.p1last", "m.p2first", "m.p2last", "e.p1part", "e.p2part", "w.gs1", "w.gs2",
                                    "e.p2t0", "e.p2t5", "s.p2t0", "s.p2t5", "-", "-", "-", "-", "-"};
    double acc[32] = {}, per_step = 0;
    int cnt = 0;
    for (std::size_t k = 2; k + 1 < steps; ++k, ++cnt) {
      for (int s = 0; s < 32; ++s)
        if (h[512 * k + s]) acc[s] += ((double)h[512 * k + s] - (double)h[512 * k + 0]) * 1e-3;
      per_step += ((double)h[512 * (k + 1)] - (double)h[512 * k]) * 1e-3;
    }
    if (cnt) {
      for (auto& v : acc) v /= cnt;
      stream_prof_[0] = per_step / cnt;               // step
      stream_prof_[1] = acc[1];                       // phase 1 until reduced
      stream_prof_[2] = acc[4] - acc[5];              // h ready -> phase 2 reduced
      stream_prof_[3] = acc[18] - acc[17];            // phase-2 tiles (CTA 0: first MMA2 .. last MMA3 issue)
      stream_prof_[4] = acc[4] - acc[20];             // phase-2 partials -> reduced (barrier + reduction)
      stream_prof_[5] = acc[11] - acc[9];             // D-step (enc rows .. disc update), overlapped
      stream_prof_[6] = acc[14] - acc[7];             // post chain after the dec half (cyc dec wait .. next h)
      stream_prof_[7] = (double)cnt;
      if (!std::getenv("LTFB_STREAM_PROF")) goto done_print;
      std::fprintf(stderr, "stream prof (%d steps, us from w.p1 of the step; step %.2f us):", cnt, per_step);
      for (auto& v : acc) v *= cnt;
      for (int s = 0; s < 32; ++s)
        if (names[s][0] != '-') std::fprintf(stderr, " %s %.1f", names[s], acc[s] / cnt);
      // phase-2 tiles of CTA 0 in step 3: producer issue, staged, MMA2 issued, epilogue done, MMA3 issued
      if (steps > 4) {
        const std::size_t k = 3;
        std::fprintf(stderr, "\n  pull: start %.2f end %.2f (us from c.decwait)",
                     ((double)h[512 * k + 90] - (double)h[512 * k + 7]) * 1e-3,
                     ((double)h[512 * k + 91] - (double)h[512 * k + 7]) * 1e-3);
        std::fprintf(stderr, "\n  D-step (us from d.encwait): enc rows %.2f enc tail %.2f fwd %.2f disc fwd %.2f bce %.2f disc bwd %.2f pg %.2f S1 %.2f",
                     ((double)h[512 * k + 100] - (double)h[512 * k + 9]) * 1e-3,
                     ((double)h[512 * k + 101] - (double)h[512 * k + 9]) * 1e-3,
                     ((double)h[512 * k + 102] - (double)h[512 * k + 9]) * 1e-3,
                     ((double)h[512 * k + 103] - (double)h[512 * k + 9]) * 1e-3,
                     ((double)h[512 * k + 104] - (double)h[512 * k + 9]) * 1e-3,
                     ((double)h[512 * k + 105] - (double)h[512 * k + 9]) * 1e-3,
                     ((double)h[512 * k + 106] - (double)h[512 * k + 9]) * 1e-3,
                     ((double)h[512 * k + 107] - (double)h[512 * k + 9]) * 1e-3);
        std::fprintf(stderr, "\n  post (us from c.decwait): S3b-arrive %.2f S3b %.2f fwd-bwd-start %.2f pg-start %.2f S4-arr %.2f S4 %.2f adam %.2f S5 %.2f gupd %.2f S6 %.2f nexth %.2f",
                     ((double)h[512 * k + 94] - (double)h[512 * k + 7]) * 1e-3,
                     ((double)h[512 * k + 95] - (double)h[512 * k + 7]) * 1e-3,
                     ((double)h[512 * k + 92] - (double)h[512 * k + 7]) * 1e-3,
                     ((double)h[512 * k + 93] - (double)h[512 * k + 7]) * 1e-3,
                     ((double)h[512 * k + 29] - (double)h[512 * k + 7]) * 1e-3,
                     ((double)h[512 * k + 30] - (double)h[512 * k + 7]) * 1e-3,
                     ((double)h[512 * k + 31] - (double)h[512 * k + 7]) * 1e-3,
                     ((double)h[512 * k + 27] - (double)h[512 * k + 7]) * 1e-3,
                     ((double)h[512 * k + 12] - (double)h[512 * k + 7]) * 1e-3,
                     ((double)h[512 * k + 13] - (double)h[512 * k + 7]) * 1e-3,
                     ((double)h[512 * k + 14] - (double)h[512 * k + 7]) * 1e-3);
        {  // phase-2 partials written, per CTA, relative to CTA 0
          std::vector<double> d;
          for (int c = 0; c < S_stream_; ++c)
            if (h[512 * k + 128 + c]) d.push_back(((double)h[512 * k + 128 + c] - (double)h[512 * k + 128]) * 1e-3);
          std::sort(d.begin(), d.end());
          if (!d.empty())
            std::fprintf(stderr, "\n  phase-2 partials per CTA vs CTA 0 (us): min %.2f p10 %.2f median %.2f p90 %.2f max %.2f",
                         d.front(), d[d.size() / 10], d[d.size() / 2], d[d.size() * 9 / 10], d.back());
          std::vector<double> b;
          for (int c = 0; c < S_stream_; ++c)
            if (h[512 * k + 300 + c]) b.push_back(((double)h[512 * k + 300 + c] - (double)h[512 * k + 128]) * 1e-3);
          std::sort(b.begin(), b.end());
          if (!b.empty())
            std::fprintf(stderr, "\n  phase-2 barrier arrival per CTA vs CTA 0 partials (us): min %.2f median %.2f max %.2f; CTA0 pre-sync %.2f",
                         b.front(), b[b.size() / 2], b.back(),
                         ((double)h[512 * k + 299] - (double)h[512 * k + 128]) * 1e-3);
          {  // barrier latency: last arrival vs release, all in us from CTA 0's partials
            const double p0 = (double)h[512 * k + 128];
            double last = -1e30, rel_min = 1e30, rel_max = -1e30;
            for (int c = 0; c < S_stream_; ++c)
              if (h[512 * k + 300 + c]) last = std::max(last, ((double)h[512 * k + 300 + c] - p0) * 1e-3);
            for (int c = 0; c < std::min(40, S_stream_); ++c)
              if (h[512 * k + 432 + c]) {
                rel_min = std::min(rel_min, ((double)h[512 * k + 432 + c] - p0) * 1e-3);
                rel_max = std::max(rel_max, ((double)h[512 * k + 432 + c] - p0) * 1e-3);
              }
            std::fprintf(stderr, "\n  phase-2 barrier (us vs CTA 0 partials): last arrival %.2f, release (CTAs < 40) %.2f .. %.2f",
                         last, rel_min, rel_max);
          }
        }
        if (std::getenv("LTFB_STREAM_PROF") && std::getenv("LTFB_STREAM_PROF")[0] == '2') {
          std::vector<unsigned long long> sm(S_stream_);
          LTFB_CUDA(cudaMemcpy(sm.data(), prof_.p + 512 * steps, S_stream_ * 8, cudaMemcpyDeviceToHost));
          for (std::size_t kk = 2; kk + 1 < steps && kk < 12; ++kk) {
            std::fprintf(stderr, "\n  per CTA step %zu (cta:sm p2part, us vs median, > 1.5 us):", kk);
            std::vector<double> d;
            for (int c = 0; c < S_stream_; ++c) d.push_back((double)h[512 * kk + 128 + c]);
            std::vector<double> srt = d;
            std::sort(srt.begin(), srt.end());
            const double med = srt[srt.size() / 2];
            for (int c = 0; c < S_stream_; ++c)
              if ((d[c] - med) * 1e-3 > 1.5) std::fprintf(stderr, " %d:%llu %.1f", c, sm[c], (d[c] - med) * 1e-3);
          }
        }
        std::fprintf(stderr, "\n  tiles of step 3 (us from w.p2): prod / staged / mma2 / epi / mma3 / O-ready\n");
        for (int j = 0; j < 8; ++j) {
          std::fprintf(stderr, "   t%2d", j);
          for (int e = 0; e < 6; ++e) {
            const unsigned long long v = h[512 * k + 32 + 6 * j + e];
            std::fprintf(stderr, " %7.2f", v ? ((double)v - (double)h[512 * k + 2]) * 1e-3 : -1.0);
          }
          std::fprintf(stderr, "\n");
        }
      }
    done_print:;
      std::fprintf(stderr, "\n");
    }
  }
}

void DeviceTrainer::check_stream_error() {
  if (!stream_on_) return;
  ltfb_dev::StepSync sy{};
  LTFB_CUDA(cudaMemcpy(&sy, sync_, sizeof sy, cudaMemcpyDeviceToHost));
  if (std::getenv("LTFB_STREAM_DEBUG"))
    std::fprintf(stderr, "stream run %d: enc %llu dec %llu h %llu abort %d error %d site %d wide-post start %.1f us\n",
                 run_id_, sy.enc_done, sy.dec_done, sy.h_done, sy.abort, sy.error, sy.err_site,
                 (double)((long long)sy.t_wide0 - (long long)sy.t_post0) * 1e-3);
  if (sy.error) {
    stream_on_ = false;
    throw ltfb::Error("CUDA error: streamed step: a hand-off between the wide pass and the post cluster timed out "
                      "(code " + std::to_string(sy.error) + ", site " + std::to_string(sy.err_site) + ")");
  }
}

bool DeviceTrainer::train_steps(std::size_t n, std::vector<ltfb::train::StepRecord>& out) {
  DeviceGuard g(spec_.device);
  // trainer.hpp:282-288: the skip threshold was exceeded; the device trainer
  // stays aborted, so every later call fails the same way
  if (aborted_ && n > 0) return false;
  std::size_t done = 0;
  while (done < n) {
    const std::size_t chunk = std::min<std::size_t>(n - done, rec_.n);
    const std::uint64_t first = host_step_;
    epoch_marks_.clear();
    enqueue_steps(chunk);
    close_epoch_segment(false, false);
    sync_stream();
    check_stream_error();
    resolve_epoch_times();
    if (ktime_on_) resolve_kernel_times();
    std::vector<ltfb_dev::StepRec> recs(chunk);
    const std::size_t at = first % rec_.n;
    const std::size_t n1 = std::min(chunk, rec_.n - at);
    LTFB_CUDA(cudaMemcpy(recs.data(), rec_.p + at, n1 * sizeof(ltfb_dev::StepRec), cudaMemcpyDeviceToHost));
    if (n1 < chunk)
      LTFB_CUDA(cudaMemcpy(recs.data() + n1, rec_.p, (chunk - n1) * sizeof(ltfb_dev::StepRec),
                           cudaMemcpyDeviceToHost));
    for (std::size_t i = 0; i < chunk; ++i) {
      const auto& r = recs[i];
      ltfb::train::StepRecord s;
      s.trainer = spec_.trainer_id;
      s.step = r.step;
      s.epoch = r.epoch;
      s.d_loss = r.d_loss;
      s.g_total = r.g_total;
      s.g_fwd = r.g_fwd;
      s.g_adv = r.g_adv;
      s.g_cyc = r.g_cyc;
      s.skipped = (r.flags & 1u) != 0;
      out.push_back(s);
      if (r.flags & 8u) {
        // abort: steps enqueued after this one were no-ops on the device;
        // roll the host bookkeeping (step, position in the epoch, epoch
        // starts and the records they closed) back to this step.
        const std::uint64_t valid_end = first + i + 1;  // host step after the aborting step
        std::uint64_t tail = chunk - 1 - i;             // no-op steps in the old epoch
        for (const auto& mk : epoch_marks_) {
          if (mk.at_step < valid_end) continue;
          epoch_ = mk.epoch;
          closed_.resize(std::min(closed_.size(), mk.closed));
          step_in_epoch_ = mk.step_in_epoch;
          epoch_steps_ = mk.steps;
          epoch_shuffled_ = mk.shuffled;
          epoch_seconds_ = mk.seconds;
          tail = mk.at_step - valid_end;
          break;
        }
        step_in_epoch_ -= std::min<std::size_t>(step_in_epoch_, tail);
        epoch_steps_ -= std::min<std::uint64_t>(epoch_steps_, tail);
        host_step_ = valid_end;
        aborted_ = true;
        return false;
      }
    }
    done += chunk;
  }
  return true;
}

std::vector<DeviceTrainer::EpochInfo> DeviceTrainer::take_epochs() {
  DeviceGuard g(spec_.device);
  resolve_epoch_times();
  std::vector<EpochInfo> out;
  out.swap(closed_);
  return out;
}

void DeviceTrainer::flush_epoch() {
  DeviceGuard g(spec_.device);
  if (have_plan_ && step_in_epoch_ > 0) {
    close_epoch_segment(true, step_in_epoch_ < steps_per_epoch_);
  }
  resolve_epoch_times();
}

void DeviceTrainer::synchronize() {
  DeviceGuard g(spec_.device);
  sync_stream();
}

// ----------------------------------------------------------- evaluation --
EvalOut DeviceTrainer::evaluate(int which, const float* cf, const float* ci, int nc, bool decide,
                                double w_f, double w_i) {
  DeviceGuard g(spec_.device);
  const std::size_t rows = which == 0 ? tour_rows_ : val_rows_;
  if (rows == 0) throw ContractError(which == 0 ? "Trainer: no tournament slice configured"
                                                : "evaluate: empty data slice");
  ltfb_dev::EvalArgs e{};
  e.m = margs_;
  e.rows = static_cast<int>(rows);
  e.nc = nc;
  e.S = static_cast<int>(eval_S_);
  e.x = which == 0 ? tx_.p : vx_.p;
  e.y = which == 0 ? ty_.p : vy_.p;
  e.enc = params_[0].p;
  e.dec = params_[1].p;
  const float* own_f = gen_.p;
  const float* own_i = gen_.p + counts_[2];
  e.cf[0] = cf ? cf : own_f;
  e.ci[0] = ci ? ci : own_i;
  e.cf[1] = incoming_.p;
  e.ci[1] = incoming_.p + counts_[2];
  e.h = eval_h_.p;
  e.inv_row = eval_inv_.p;
  e.part = eval_part_.p;
  e.out = eval_out_.p;
  e.w_f = w_f;
  e.w_i = w_i;
  e.decide = decide ? 1 : 0;
  e.dst_fwd = gen_.p;
  e.dst_inv = gen_.p + counts_[2];
  e.m_fwd = mom1_[2].p;
  e.v_fwd = mom2_[2].p;
  e.m_inv = mom1_[3].p;
  e.v_inv = mom2_[3].p;
  e.n_fwd = static_cast<long long>(counts_[2]);
  e.n_inv = static_cast<long long>(counts_[3]);
  e.ctr = ctr_.p;
  const ltfb_dev::EvalTcHost* etc = eval_tc_[which].ready ? &eval_tc_[which] : nullptr;
  if (etc) {
    prepare_params();  // the K-major weight copy the tensor-core pass reads
    e.S = sm_count_;
  }
  ltfb_dev::launch_eval(e, stream_, etc, wide_kind_ == 2);
  if (decide) small_T_dirty_ = true;  // the device may have adopted the incoming generator
  if (decide) h_ready_ = false;
  launches_ += 3;
  LTFB_CUDA(cudaGetLastError());
  double out[6] = {0, 0, 0, 0, 0, 0};
  LTFB_CUDA(cudaMemcpyAsync(out, eval_out_.p, sizeof(double) * 3 * nc, cudaMemcpyDeviceToHost, stream_));
  int adopt = 0;
  LTFB_CUDA(cudaMemcpyAsync(&adopt, &ctr_.p->last_adopt, sizeof(int), cudaMemcpyDeviceToHost, stream_));
  sync_stream();
  EvalOut r;
  for (int c = 0; c < nc; ++c) r.m[c] = {out[3 * c], out[3 * c + 1], out[3 * c + 2]};
  r.adopted = decide ? adopt : 0;
  return r;
}

void DeviceTrainer::set_incoming(const float* fwd, const float* inv) {
  DeviceGuard g(spec_.device);
  LTFB_CUDA(cudaMemcpyAsync(incoming_.p, fwd, counts_[2] * 4, cudaMemcpyHostToDevice, stream_));
  LTFB_CUDA(cudaMemcpyAsync(incoming_.p + counts_[2], inv, counts_[3] * 4, cudaMemcpyHostToDevice, stream_));
  sync_stream();
}

EvalOut DeviceTrainer::tournament_decide() {
  return evaluate(0, nullptr, nullptr, 2, true, spec_.w_f, spec_.w_i);
}

void DeviceTrainer::adopt(const float* fwd, const float* inv) {
  DeviceGuard g(spec_.device);
  small_T_dirty_ = true;
  h_ready_ = false;
  LTFB_CUDA(cudaMemcpyAsync(gen_.p, fwd, counts_[2] * 4, cudaMemcpyHostToDevice, stream_));
  LTFB_CUDA(cudaMemcpyAsync(gen_.p + counts_[2], inv, counts_[3] * 4, cudaMemcpyHostToDevice, stream_));
  for (int net : {2, 3}) {
    LTFB_CUDA(cudaMemsetAsync(mom1_[net].p, 0, counts_[net] * 4, stream_));
    LTFB_CUDA(cudaMemsetAsync(mom2_[net].p, 0, counts_[net] * 4, stream_));
  }
  sync_stream();
}

bool DeviceTrainer::train_steps_host(std::size_t n, const float* x, const float* y,
                                     std::vector<ltfb::train::StepRecord>& out) {
  h_ready_ = false;
  DeviceGuard g(spec_.device);
  if (n_part_ == 0) throw ContractError("train_steps: data store is empty");
  const auto& m = margs_;
  const std::size_t B = spec_.batch_size;
  if (!copy_stream_) {
    LTFB_CUDA(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      hx_[i].alloc(B * m.in);
      hy_[i].alloc(std::max<std::size_t>(B, 128) * m.out_pad);
      if (wide_kind_ >= 2)
        ltfb_dev::encode_y_map(wtp_, i, hy_[i].p, args_, static_cast<int>(std::max<std::size_t>(B, 128)));
      LTFB_CUDA(cudaMemsetAsync(hy_[i].p, 0, hy_[i].bytes(), copy_stream_));
      LTFB_CUDA(cudaEventCreateWithFlags(&h2d_done_[i], cudaEventDisableTiming));
      LTFB_CUDA(cudaEventCreateWithFlags(&used_done_[i], cudaEventDisableTiming));
      LTFB_CUDA(cudaEventRecord(used_done_[i], stream_));
    }
  }
  ensure_adam_table(t_host_max_ + host_step_ + n + 1);
  // order the copy stream after everything already on the compute stream
  LTFB_CUDA(cudaEventRecord(used_done_[0], stream_));
  LTFB_CUDA(cudaEventRecord(used_done_[1], stream_));
  float* keep_x = args_.xb;
  float* keep_y = args_.yb;
  for (std::size_t i = 0; i < n; ++i) {
    if (!have_plan_ || step_in_epoch_ >= steps_per_epoch_) start_epoch();
    const int b = static_cast<int>(i & 1);
    // H2D of this step's minibatch on the copy stream, after the step that
    // last used this buffer has finished with it
    LTFB_CUDA(cudaStreamWaitEvent(copy_stream_, used_done_[b], 0));
    LTFB_CUDA(cudaMemcpyAsync(hx_[b].p, x + i * B * m.in, B * m.in * 4, cudaMemcpyHostToDevice, copy_stream_));
    LTFB_CUDA(cudaMemcpy2DAsync(hy_[b].p, m.out_pad * 4, y + i * B * m.out, m.out * 4, m.out * 4, B,
                                cudaMemcpyHostToDevice, copy_stream_));
    LTFB_CUDA(cudaEventRecord(h2d_done_[b], copy_stream_));
    LTFB_CUDA(cudaStreamWaitEvent(stream_, h2d_done_[b], 0));
    args_.xb = hx_[b].p;
    args_.yb = hy_[b].p;
    args_.y_identity = 1;
    wtp_.y_sel = b;
    launch_step_kernels(false, true);
    wtp_.y_sel = -1;
    args_.y_identity = 0;
    LTFB_CUDA(cudaEventRecord(used_done_[b], stream_));
    ++step_in_epoch_;
    ++epoch_steps_;
    ++host_step_;
  }
  args_.xb = keep_x;
  args_.yb = keep_y;
  LTFB_CUDA(cudaGetLastError());
  std::vector<ltfb_dev::StepRec> recs(n);
  const std::uint64_t first = host_step_ - n;
  for (std::size_t i = 0; i < n; ++i)  // D2H of every step's record
    LTFB_CUDA(cudaMemcpyAsync(&recs[i], rec_.p + (first + i) % rec_.n, sizeof(ltfb_dev::StepRec),
                              cudaMemcpyDeviceToHost, stream_));
  sync_stream();
  bool ok = true;
  for (const auto& r : recs) {
    ltfb::train::StepRecord s;
    s.trainer = spec_.trainer_id;
    s.step = r.step;
    s.epoch = r.epoch;
    s.d_loss = r.d_loss;
    s.g_total = r.g_total;
    s.g_fwd = r.g_fwd;
    s.g_adv = r.g_adv;
    s.g_cyc = r.g_cyc;
    s.skipped = (r.flags & 1u) != 0;
    out.push_back(s);
    if (r.flags & 8u) {
      ok = false;
      break;
    }
  }
  return ok;
}

// ------------------------------------------------- autoencoder pre-training --
int DeviceTrainer::ae_kind(int rows) const {
  // LTFB_AE_SIMT=1: the SIMT column passes (A/B checks)
  const bool simt = std::getenv("LTFB_AE_SIMT") != nullptr;
  return !simt && ltfb_dev::ae_tc_supported(margs_, rows) ? 2 : 1;
}

void DeviceTrainer::ae_allocate() {
  if (ae_alloc_) return;
  const auto& m = margs_;
  const int R = 128;
  auto& a = ae_args_;
  a = {};
  a.m = m;
  a.S = sm_count_;
  std::size_t need = 0;
  auto take = [&](std::size_t n) {
    const std::size_t o = need;
    need += (n + 31) & ~std::size_t(31);
    return o;
  };
  const std::size_t oPz = take((std::size_t)a.S * R * m.E1), oPg = take((std::size_t)a.S * R * m.D);
  const std::size_t oz0 = take(R * m.E1), oa0 = take(R * m.E1), oga0 = take(R * m.E1), ogz0 = take(R * m.E1);
  std::size_t oet[ltfb_dev::kMaxLayers][2] = {}, odh[ltfb_dev::kMaxLayers][2] = {};
  int maxw = std::max(m.E1, m.D);
  std::size_t odz[ltfb_dev::kMaxLayers][2] = {};
  for (int l = 0; l < m.enc_tail.L; ++l) {
    oet[l][0] = take((std::size_t)R * m.enc_tail.w[l + 1]);
    oet[l][1] = take((std::size_t)R * m.enc_tail.w[l + 1]);
    odz[l][0] = take((std::size_t)R * m.enc_tail.w[l + 1]);
    maxw = std::max(maxw, m.enc_tail.max_w());
  }
  for (int l = 0; l < m.dec_head.L; ++l) odz[l][1] = take((std::size_t)R * m.dec_head.w[l + 1]);
  for (int l = 0; l < m.dec_head.L; ++l) {
    odh[l][0] = take((std::size_t)R * m.dec_head.w[l + 1]);
    odh[l][1] = take((std::size_t)R * m.dec_head.w[l + 1]);
    maxw = std::max(maxw, m.dec_head.max_w());
  }
  const std::size_t ogh = take(R * m.D), oglat = take((std::size_t)R * m.lat);
  const std::size_t otA = take((std::size_t)R * maxw), otB = take((std::size_t)R * maxw);
  ae_scr_.alloc(need);
  ae_part_.alloc(a.S);
  ae_flags_.alloc(4);  // enc / dec non-finite flags, Adam blocks done
  ae_loss_.alloc(1);
  ae_idx_.alloc(R);
  float* b = ae_scr_.p;
  a.Pz = b + oPz;
  a.Pg = b + oPg;
  a.z0 = b + oz0;
  a.a0 = b + oa0;
  a.ga0 = b + oga0;
  a.gz0 = b + ogz0;
  for (int l = 0; l < m.enc_tail.L; ++l) {
    a.etz[l] = b + oet[l][0];
    a.eta[l] = b + oet[l][1];
    a.dze[l] = b + odz[l][0];
  }
  for (int l = 0; l < m.dec_head.L; ++l) a.dzh[l] = b + odz[l][1];
  for (int l = 0; l < m.dec_head.L; ++l) {
    a.dhz[l] = b + odh[l][0];
    a.dha[l] = b + odh[l][1];
  }
  a.latent = m.enc_tail.L > 0 ? a.eta[m.enc_tail.L - 1] : a.a0;
  a.h = m.dec_head.L > 0 ? a.dha[m.dec_head.L - 1] : a.latent;
  a.gh = b + ogh;
  a.glat = m.dec_head.L > 0 ? b + oglat : a.gh;
  // with an empty enc tail, dL/da0 is dL/dlatent itself
  a.tA = b + otA;
  a.tB = b + otB;
  a.mae_part = ae_part_.p;
  a.flags = ae_flags_.p;
  a.loss = ae_loss_.p;
  a.idx = ae_idx_.p;
  a.enc = params_[0].p;
  a.dec = params_[1].p;
  a.genc = grads_[0].p;
  a.gdec = grads_[1].p;
  if (m.enc_tail.L == 0) a.ga0 = a.glat;
  ae_alloc_ = true;
}

void DeviceTrainer::load_ae_source(const float* y, std::size_t n) {
  DeviceGuard g(spec_.device);
  if (n == 0) throw ContractError("load_ae_source: empty source");
  const std::size_t out = static_cast<std::size_t>(margs_.out), op = static_cast<std::size_t>(margs_.out_pad);
  ae_y_.alloc(n * op);
  LTFB_CUDA(cudaMemsetAsync(ae_y_.p, 0, ae_y_.bytes(), stream_));
  LTFB_CUDA(cudaMemcpy2DAsync(ae_y_.p, op * 4, y, out * 4, out * 4, n, cudaMemcpyHostToDevice, stream_));
  sync_stream();
  ae_rows_ = n;
}

void DeviceTrainer::ae_alloc_source(std::size_t rows) {
  DeviceGuard g(spec_.device);
  if (rows == 0) throw ContractError("ae_alloc_source: empty source");
  const std::size_t op = static_cast<std::size_t>(margs_.out_pad);
  ae_y_.alloc(rows * op);
  LTFB_CUDA(cudaMemsetAsync(ae_y_.p, 0, ae_y_.bytes(), stream_));
  ae_rows_ = rows;
  sync_stream();
}

void DeviceTrainer::ae_fill_from_store(const std::uint32_t* slots, std::size_t n, std::size_t dst_row) {
  DeviceGuard g(spec_.device);
  if (dst_row + n > ae_rows_) throw ContractError("ae_fill_from_store: rows outside the AE source");
  for (std::size_t i = 0; i < n; ++i)
    if (slots[i] >= n_part_) throw ContractError("ae_fill_from_store: slot outside the store");
  if (n == 0) return;
  if (ae_fill_slots_.n < n) ae_fill_slots_.alloc(std::max<std::size_t>(n, 128));
  LTFB_CUDA(cudaMemcpyAsync(ae_fill_slots_.p, slots, n * 4, cudaMemcpyHostToDevice, stream_));
  ltfb_dev::launch_gather_rows(sy_.p, ae_fill_slots_.p, static_cast<int>(n),
                               ae_y_.p + dst_row * static_cast<std::size_t>(margs_.out_pad), margs_.out_pad, stream_);
  ++launches_;
}

/// surrogate/train_ops.hpp:71-81 on the device: loss, gradients, then
/// Adam(enc) and Adam(dec) with the reference's NumericError semantics
/// (a non-finite loss or enc gradient changes nothing; a non-finite dec
/// gradient leaves enc applied).
double DeviceTrainer::ae_step(const std::uint32_t* rows_idx, std::size_t n) {
  DeviceGuard g(spec_.device);
  if (ae_rows_ == 0) throw ContractError("ae_step: no autoencoder source loaded");
  if (!ltfb_dev::ae_supported(margs_, static_cast<int>(n)))
    throw ContractError("ae_step: supported for 1..128 rows and wide-layer widths <= 64");
  for (std::size_t i = 0; i < n; ++i)
    if (rows_idx[i] >= ae_rows_) throw ContractError("ae_step: row index outside the source");
  ae_allocate();
  auto a = ae_args_;
  a.n = static_cast<int>(n);
  a.ysrc = ae_y_.p;
  if (!ae_pin_) LTFB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ae_pin_), sizeof(AePinned), cudaHostAllocDefault));
  std::memcpy(ae_pin_->idx, rows_idx, n * 4);
  LTFB_CUDA(cudaMemcpyAsync(ae_idx_.p, ae_pin_->idx, n * 4, cudaMemcpyHostToDevice, stream_));
  LTFB_CUDA(cudaMemsetAsync(ae_flags_.p, 0, 16, stream_));
  const void* map = nullptr;
  if (ae_kind(static_cast<int>(n)) == 2) {
    if (ae_map_base_ != ae_y_.p || ae_map_rows_ != ae_rows_) {
      ltfb_dev::encode_ae_y_map(ae_map_, ae_y_.p, static_cast<int>(ae_rows_), margs_);
      ae_map_base_ = ae_y_.p;
      ae_map_rows_ = ae_rows_;
    }
    map = ae_map_;
  }
  ltfb_dev::launch_ae_passes(a, map, stream_);
  launches_ += 7;
  if (map) {
    // one host round trip per step: Adam(enc), Adam(dec) and t decided on
    // the device; the host maps the flags onto the reference's exceptions
    ensure_adam_table(t_host_max_ + 2);
    const auto& h = spec_.arch.adam;
    float* p[2] = {params_[0].p, params_[1].p};
    float* m1[2] = {mom1_[0].p, mom1_[1].p};
    float* m2[2] = {mom2_[0].p, mom2_[1].p};
    float* g[2] = {grads_[0].p, grads_[1].p};
    const long long cnt[2] = {static_cast<long long>(counts_[0]), static_cast<long long>(counts_[1])};
    const double lr[2] = {spec_.lr[0] > 0 ? spec_.lr[0] : h.lr, spec_.lr[1] > 0 ? spec_.lr[1] : h.lr};
    ltfb_dev::launch_ae_adam_dev(p, m1, m2, g, cnt, lr, h.beta1, h.beta2, h.eps, adam_c_.p, ctr_.p, ae_flags_.p,
                                 ae_loss_.p, sm_count_, stream_);
    launches_ += 1;
    LTFB_CUDA(cudaMemcpyAsync(&ae_pin_->loss, ae_loss_.p, 8, cudaMemcpyDeviceToHost, stream_));
    LTFB_CUDA(cudaMemcpyAsync(ae_pin_->flags, ae_flags_.p, 8, cudaMemcpyDeviceToHost, stream_));
    sync_stream();
    t_host_max_ += 1;
    wide_dirty_ = true;
    small_T_dirty_ = true;
    h_ready_ = false;
    const double loss = ae_pin_->loss;
    if (!std::isfinite(loss)) throw ltfb::NumericError("autoencoder_step: non-finite loss");
    if (ae_pin_->flags[0] || ae_pin_->flags[1]) throw ltfb::NumericError("adam_step: non-finite gradient component");
    return loss;
  }
  double loss = 0.0;
  int flags[2] = {0, 0};
  LTFB_CUDA(cudaMemcpyAsync(&loss, ae_loss_.p, 8, cudaMemcpyDeviceToHost, stream_));
  LTFB_CUDA(cudaMemcpyAsync(flags, ae_flags_.p, 8, cudaMemcpyDeviceToHost, stream_));
  sync_stream();
  if (!std::isfinite(loss)) throw ltfb::NumericError("autoencoder_step: non-finite loss");
  const auto& h = spec_.arch.adam;
  auto apply = [&](int net) {
    std::uint64_t t = 0;
    LTFB_CUDA(cudaMemcpy(&t, &ctr_.p->t[net], 8, cudaMemcpyDeviceToHost));
    t += 1;
    const double c1 = 1.0 - std::pow(h.beta1, static_cast<double>(t));
    const double c2 = 1.0 - std::pow(h.beta2, static_cast<double>(t));
    const double lr = spec_.lr[net] > 0 ? spec_.lr[net] : h.lr;
    ltfb_dev::launch_ae_adam(params_[net].p, mom1_[net].p, mom2_[net].p, grads_[net].p,
                             static_cast<long long>(counts_[net]), lr, h.beta1, h.beta2, h.eps, c1, c2, sm_count_,
                             stream_);
    ++launches_;
    LTFB_CUDA(cudaMemcpyAsync(&ctr_.p->t[net], &t, 8, cudaMemcpyHostToDevice, stream_));
    sync_stream();
  };
  wide_dirty_ = true;  // the frozen-weight copies / W^T images follow enc / dec
  small_T_dirty_ = true;
  h_ready_ = false;
  if (flags[0]) throw ltfb::NumericError("adam_step: non-finite gradient component");
  apply(0);
  if (flags[1]) throw ltfb::NumericError("adam_step: non-finite gradient component");
  apply(1);
  return loss;
}

}  // namespace ltfb_b200
