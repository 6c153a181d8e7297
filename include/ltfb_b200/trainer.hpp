// C++ drop-in façade of the B200 path: the reference's train::Trainer and
// tournament::tournament_round surface (train/trainer.hpp:41-134,
// tournament/ltfb.hpp:96-164) over the C ABI of libltfb_gpu.so
// (include/ltfb_gpu.h). Header-only; link with -lltfb_gpu.
//
// Same names, argument meanings and error behaviour as the reference: every
// failing ABI status is rethrown as the reference's exception type
// (ltfb::DimensionError, ContractError, NumericError, ...), with the
// library's message. The model lives in HBM; model() returns a host mirror
// refreshed on demand (value semantics as in the reference).
#pragma once

#include <algorithm>
#include <chrono>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "../ltfb_gpu.h"
#include "host_algos.hpp"
#include "types.hpp"

namespace ltfb_b200 {

using ltfb::surrogate::CycleGan;
using ltfb::surrogate::EvalMetric;
using ltfb::surrogate::ModalityDims;
using ltfb::surrogate::SurrogateArch;

/// Maps a C-ABI status onto the reference's exception taxonomy
/// (core/error.hpp:11-58).
inline void check(int rc) {
  if (rc == LTFB_OK) return;
  const std::string msg = ltfb_last_error();
  switch (rc) {
    case LTFB_EDIMENSION: throw ltfb::DimensionError(msg);
    case LTFB_ECONTRACT: throw ltfb::ContractError(msg);
    case LTFB_ENUMERIC: throw ltfb::NumericError(msg);
    case LTFB_EIO: throw ltfb::IoError(msg);
    case LTFB_ECAPACITY: throw ltfb::CapacityError(msg);
    case LTFB_ESTORECORRUPT: throw ltfb::StoreCorruptError(msg);
    case LTFB_ECONFIG: throw ltfb::ConfigError(msg);
    default: throw ltfb::Error("ltfb_gpu: " + msg);
  }
}

inline ltfb_dims to_c(const ModalityDims& d) {
  return {d.input_dim, d.latent_dim, d.scalar_dim, d.image_views, d.image_channels, d.image_h, d.image_w};
}

/// The architecture a CycleGan was built with (hidden widths from its specs,
/// hidden activation, lambdas and Adam hyper-parameters).
inline ltfb_arch arch_of(const CycleGan<float>& m) {
  ltfb_arch a{};
  ltfb_arch_defaults(&a);
  auto hidden = [](const ltfb::nn::MlpSpec& s, uint32_t* dst, uint32_t* n) {
    const std::size_t L = s.n_layers();
    if (L - 1 > 8) throw ltfb::ContractError("more than 8 hidden layers");
    *n = static_cast<uint32_t>(L - 1);
    for (std::size_t i = 1; i < L; ++i) dst[i - 1] = static_cast<uint32_t>(s.layer_widths[i]);
  };
  hidden(m.enc_spec, a.enc_hidden, &a.n_enc_hidden);
  hidden(m.dec_spec, a.dec_hidden, &a.n_dec_hidden);
  hidden(m.fwd_spec, a.fwd_hidden, &a.n_fwd_hidden);
  hidden(m.inv_spec, a.inv_hidden, &a.n_inv_hidden);
  hidden(m.disc_spec, a.disc_hidden, &a.n_disc_hidden);
  const auto& act = m.fwd_spec.activations.front();
  a.hidden_act = static_cast<int32_t>(act.kind);  // Act order == LTFB_ACT_* order
  a.hidden_slope = act.slope;
  a.lambda_adv = m.lambda_adv;
  a.lambda_cyc = m.lambda_cyc;
  a.lr = m.fwd_opt.hyper.lr;
  a.beta1 = m.fwd_opt.hyper.beta1;
  a.beta2 = m.fwd_opt.hyper.beta2;
  a.eps = m.fwd_opt.hyper.eps;
  return a;
}

/// train/trainer.hpp:26-39 (+ device placement and kernel choice).
struct TrainerConfig {
  int trainer_id = 0;
  int n_shards = 1;
  std::size_t batch_size = 128;
  std::uint64_t seed = 0;
  int numeric_abort_threshold = 10;
  double w_f = 1.0, w_i = 1.0;
  std::vector<std::uint32_t> train_ids, tournament_ids;
  int device = 0;
  int wide_kernel = 0;
};

/// An in-memory dataset: x [total x input_dim], y [total x output_dim],
/// indexed by global sample id (the assemble_tensors view of a
/// DatasetIndex, data/bundle.hpp:134-224).
struct DatasetView {
  ModalityDims dims;
  std::size_t total = 0;
  const float* x = nullptr;
  const float* y = nullptr;
};

/// data/store.hpp:45-57: file-access accounting of the store.
struct AccessCounters {
  std::uint64_t files_opened = 0;
  std::uint64_t bytes_read = 0;
  std::uint64_t samples_shuffled = 0;
};

/// Host view of the trainer's HBM-resident preload store
/// (data/store.hpp:62-99 accessors): the partition, the loader shard that
/// owns each slot (files dealt round-robin to shards, store.hpp:100-135)
/// and the access counters (the preload phase reads every partition record
/// once; training reads no file).
class StoreView {
 public:
  int n_shards() const { return n_shards_; }
  const std::vector<std::uint32_t>& partition() const { return partition_; }
  const std::vector<std::int32_t>& owners() const { return owner_; }
  const AccessCounters& counters() const { return counters_; }
  const std::vector<std::uint32_t>& file_open_counts() const { return file_open_counts_; }
  std::size_t size() const { return partition_.size(); }

 private:
  friend class Trainer;
  int n_shards_ = 1;
  std::vector<std::uint32_t> partition_;
  std::vector<std::int32_t> owner_;
  std::vector<std::uint32_t> file_open_counts_;
  AccessCounters counters_;
};

class Trainer {
 public:
  /// train::Trainer(TrainerConfig, const DatasetIndex&, CycleGan<float>)
  /// (trainer.hpp:43-79) over an in-memory dataset: the partition is
  /// preloaded into HBM; the view's rows count as bundles of
  /// `samples_per_file` records for the store's accounting.
  Trainer(TrainerConfig cfg, const DatasetView& ds, CycleGan<float> model, std::size_t samples_per_file = 500)
      : cfg_(std::move(cfg)), mirror_(std::move(model)) {
    const std::size_t in = mirror_.dims.input_dim, out = mirror_.dims.output_dim();
    const std::size_t files = (ds.total + samples_per_file - 1) / std::max<std::size_t>(1, samples_per_file);
    init([&](const std::vector<std::uint32_t>& ids, float* x, float* y) {
      for (std::size_t i = 0; i < ids.size(); ++i) {
        if (ids[i] >= ds.total) throw ltfb::ContractError("DataStore: partition id outside dataset");
        std::copy_n(ds.x + static_cast<std::size_t>(ids[i]) * in, in, x + i * in);
        std::copy_n(ds.y + static_cast<std::size_t>(ids[i]) * out, out, y + i * out);
      }
    }, [&](std::uint32_t id) { return static_cast<std::size_t>(id) / std::max<std::size_t>(1, samples_per_file); },
         files, static_cast<std::uint64_t>(mirror_.dims.record_floats()) * 4);
  }

  /// train::Trainer(TrainerConfig, const DatasetIndex&, CycleGan<float>)
  /// over LBDS bundle files on disk (data/bundle.hpp:134-224): only the
  /// partition's and the tournament slice's records are read (the preload
  /// of store.hpp:100-135, one pass per file) and made resident in HBM.
  Trainer(TrainerConfig cfg, const ltfb::data::DatasetIndex& index, CycleGan<float> model)
      : cfg_(std::move(cfg)), mirror_(std::move(model)) {
    if (!(index.dims == mirror_.dims)) throw ltfb::DimensionError("Trainer: dataset dims differ from the model's");
    init([&](const std::vector<std::uint32_t>& ids, float* x, float* y) {
      ltfb::data::read_records(index, std::span<const std::uint32_t>(ids), x, y, index.dims.output_dim());
    }, [&](std::uint32_t id) { return index.locate(id).file_idx; }, index.paths.size(), index.stride_bytes());
  }

  /// trainer.hpp:90-97: one model hash per replica (the device trainer
  /// keeps one replica per shard in lockstep: all equal by construction).
  std::vector<std::uint64_t> replica_hashes() {
    return std::vector<std::uint64_t>(static_cast<std::size_t>(cfg_.n_shards), model().model_hash());
  }

  /// trainer.hpp:88-89: the trainer's data store (host view).
  const StoreView& store() const { return store_; }

  int id() const { return cfg_.trainer_id; }
  const TrainerConfig& config() const { return cfg_; }
  ltfb_trainer* handle() { return h_.get(); }
  /// The device state changed behind the mirror (e.g. a device-side adoption).
  void invalidate() { dirty_ = true; }

  /// trainer.hpp:102-104; NumericError once the skip threshold is exceeded
  /// (the records up to the aborting step are kept).
  void train_steps(std::uint64_t n) {
    if (n == 0) return;
    std::vector<ltfb_step_record> recs(n);
    std::uint64_t got = 0;
    const int rc = ltfb_trainer_train_steps(h_.get(), n, recs.data(), &got);
    dirty_ = true;
    for (std::uint64_t i = 0; i < got; ++i) {
      const auto& r = recs[i];
      history_.steps.push_back({cfg_.trainer_id, r.step, r.epoch, r.d_loss, r.g_total, r.g_fwd, r.g_adv, r.g_cyc,
                                r.skipped != 0});
      if (r.skipped) ++history_.skipped_steps;
    }
    drain_epochs();
    check(rc);
  }

  std::uint64_t step() const {
    std::uint64_t s = 0;
    check(ltfb_trainer_step(h_.get(), &s));
    return s;
  }

  /// Host mirror of the HBM-resident model (value semantics).
  const CycleGan<float>& model() {
    if (dirty_) {
      pull_net(LTFB_NET_FWD, mirror_.fwd, mirror_.fwd_opt, mirror_.fwd_spec);
      pull_net(LTFB_NET_INV, mirror_.inv, mirror_.inv_opt, mirror_.inv_spec);
      pull_net(LTFB_NET_DISC, mirror_.disc, mirror_.disc_opt, mirror_.disc_spec);
      dirty_ = false;
    }
    return mirror_;
  }

  /// trainer.hpp:106-112: the trainer's own generator on its tournament slice.
  EvalMetric eval_tournament() {
    ltfb_eval_metric m{};
    check(ltfb_trainer_evaluate(h_.get(), LTFB_SLICE_TOURNAMENT, nullptr, nullptr, cfg_.w_f, cfg_.w_i, &m));
    return {m.forward_mae, m.inverse_mae, m.combined};
  }
  /// ... and a candidate's generator (same frozen decoder).
  EvalMetric eval_tournament(const CycleGan<float>& cand) {
    const auto f = cand.fwd.flatten(), i = cand.inv.flatten();
    ltfb_eval_metric m{};
    check(ltfb_trainer_evaluate(h_.get(), LTFB_SLICE_TOURNAMENT, f.data(), i.data(), cfg_.w_f, cfg_.w_i, &m));
    return {m.forward_mae, m.inverse_mae, m.combined};
  }

  /// The shared validation slice (runner.hpp:319-337 evaluate_all), resident in HBM.
  void set_validation(const float* x, const float* y, std::size_t rows) {
    check(ltfb_trainer_set_slice(h_.get(), LTFB_SLICE_VALIDATION, x, y, rows));
  }
  /// surrogate::evaluate of the trainer's own generator on the validation slice.
  EvalMetric evaluate_validation(double w_f, double w_i) {
    ltfb_eval_metric m{};
    check(ltfb_trainer_evaluate(h_.get(), LTFB_SLICE_VALIDATION, nullptr, nullptr, w_f, w_i, &m));
    return {m.forward_mae, m.inverse_mae, m.combined};
  }

  /// trainer.hpp:117-127: copy fwd / inv, zero their moments, keep t.
  void adopt_generators(const ltfb::nn::MlpParams<float>& fwd, const ltfb::nn::MlpParams<float>& inv) {
    if (!fwd.same_shape(mirror_.fwd) || !inv.same_shape(mirror_.inv))
      throw ltfb::ContractError("adopt_generators: incompatible parameter shapes");
    const auto f = fwd.flatten(), i = inv.flatten();
    check(ltfb_trainer_adopt(h_.get(), f.data(), i.data()));
    dirty_ = true;
  }

  ltfb::train::HistorySegment& history() { return history_; }

  /// trainer.hpp:129-134.
  void flush_epoch_record() {
    check(ltfb_trainer_flush_epoch(h_.get()));
    drain_epochs();
  }

 private:
  struct Deleter {
    void operator()(ltfb_trainer* t) const { ltfb_trainer_destroy(t); }
  };

  void push_model() {
    const std::pair<int, const ltfb::nn::MlpParams<float>*> nets[5] = {
        {LTFB_NET_ENC, &mirror_.enc}, {LTFB_NET_DEC, &mirror_.dec}, {LTFB_NET_FWD, &mirror_.fwd},
        {LTFB_NET_INV, &mirror_.inv}, {LTFB_NET_DISC, &mirror_.disc}};
    const ltfb::nn::AdamState<float>* opts[5] = {&mirror_.enc_opt, &mirror_.dec_opt, &mirror_.fwd_opt,
                                                 &mirror_.inv_opt, &mirror_.disc_opt};
    for (int k = 0; k < 5; ++k) {
      const auto blob = nets[k].second->flatten();
      check(ltfb_trainer_set_params(h_.get(), nets[k].first, blob.data(), blob.size()));
      check(ltfb_trainer_set_adam(h_.get(), nets[k].first, opts[k]->m.data(), opts[k]->v.data(), opts[k]->t));
    }
  }

  void pull_net(int net, ltfb::nn::MlpParams<float>& p, ltfb::nn::AdamState<float>& o,
                const ltfb::nn::MlpSpec& spec) {
    std::vector<float> blob(p.param_count());
    check(ltfb_trainer_get_params(h_.get(), net, blob.data(), blob.size()));
    p = ltfb::nn::MlpParams<float>::unflatten(spec, std::span<const float>(blob));
    check(ltfb_trainer_get_adam(h_.get(), net, o.m.data(), o.v.data(), &o.t));
  }

  void drain_epochs() {
    std::vector<ltfb_epoch_record> buf(1024);
    std::uint64_t n = 0;
    check(ltfb_trainer_take_epochs(h_.get(), buf.data(), buf.size(), &n));
    // training epochs of the preload store read no file (store.hpp:140-181)
    for (std::uint64_t i = 0; i < n; ++i) {
      history_.epochs.push_back({cfg_.trainer_id, buf[i].epoch, buf[i].steps, 0, 0, buf[i].samples_shuffled,
                                 buf[i].seconds, buf[i].partial != 0});
      store_.counters_.samples_shuffled += buf[i].samples_shuffled;
    }
  }

  /// Creates the device trainer, preloads the partition (rows(ids, x, y)
  /// fills host rows of the given ids) and the tournament slice, and writes
  /// the preload phase's epoch-0 record (trainer.hpp:56-73).
  template <class Rows, class FileOf>
  void init(Rows&& rows, FileOf&& file_of, std::size_t n_files, std::uint64_t stride_bytes) {
    if (!mirror_.autoencoder_frozen) throw ltfb::ContractError("Trainer: model autoencoder must be frozen");
    if (cfg_.train_ids.empty()) throw ltfb::ContractError("plan_epoch: empty partition");
    const auto t0 = std::chrono::steady_clock::now();
    const ltfb_dims d = to_c(mirror_.dims);
    const ltfb_arch a = arch_of(mirror_);
    ltfb_trainer_config c{};
    c.trainer_id = cfg_.trainer_id;
    c.device = cfg_.device;
    c.n_shards = cfg_.n_shards;
    c.numeric_abort_threshold = cfg_.numeric_abort_threshold;
    c.batch_size = cfg_.batch_size;
    c.seed = cfg_.seed;
    c.w_f = cfg_.w_f;
    c.w_i = cfg_.w_i;
    c.wide_kernel = cfg_.wide_kernel;
    ltfb_trainer* h = nullptr;
    check(ltfb_trainer_create(&d, &a, &c, &h));
    h_.reset(h);
    push_model();
    // store.hpp:100-135: files covering the partition dealt round-robin to
    // shards in file order; the loader shard owns every record it loads
    store_.n_shards_ = cfg_.n_shards;
    store_.partition_ = cfg_.train_ids;
    store_.file_open_counts_.assign(n_files, 0);
    std::vector<std::size_t> file(cfg_.train_ids.size());
    std::vector<int> loader(n_files, -1);
    std::vector<char> used(n_files, 0);
    for (std::size_t i = 0; i < file.size(); ++i) {
      file[i] = file_of(cfg_.train_ids[i]);
      if (file[i] >= n_files) throw ltfb::ContractError("DataStore: partition id outside dataset");
      used[file[i]] = 1;
    }
    int next = 0;
    for (std::size_t f = 0; f < n_files; ++f)
      if (used[f]) {
        loader[f] = next;
        next = (next + 1) % std::max(1, cfg_.n_shards);
        ++store_.file_open_counts_[f];
        ++store_.counters_.files_opened;
      }
    store_.owner_.resize(file.size());
    for (std::size_t i = 0; i < file.size(); ++i) store_.owner_[i] = loader[file[i]];
    store_.counters_.bytes_read = static_cast<std::uint64_t>(cfg_.train_ids.size()) * stride_bytes;
    // only the partition's rows and the tournament slice's rows on the host
    const std::size_t in = mirror_.dims.input_dim, out = mirror_.dims.output_dim();
    {
      std::vector<float> x(cfg_.train_ids.size() * in), y(cfg_.train_ids.size() * out);
      rows(cfg_.train_ids, x.data(), y.data());
      check(ltfb_trainer_load_store(h_.get(), cfg_.train_ids.data(), cfg_.train_ids.size(), x.data(), y.data(),
                                    store_.owner_.data()));
    }
    if (!cfg_.tournament_ids.empty()) {
      std::vector<float> x(cfg_.tournament_ids.size() * in), y(cfg_.tournament_ids.size() * out);
      rows(cfg_.tournament_ids, x.data(), y.data());
      check(ltfb_trainer_set_slice(h_.get(), LTFB_SLICE_TOURNAMENT, x.data(), y.data(),
                                   cfg_.tournament_ids.size()));
    }
    ltfb::train::EpochRecord rec;
    rec.trainer = cfg_.trainer_id;
    rec.epoch = 0;
    rec.files_opened = store_.counters_.files_opened;
    rec.bytes_read = store_.counters_.bytes_read;
    rec.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    history_.epochs.push_back(rec);
  }

  TrainerConfig cfg_;
  std::unique_ptr<ltfb_trainer, Deleter> h_;
  CycleGan<float> mirror_;
  bool dirty_ = false;
  ltfb::train::HistorySegment history_;
  StoreView store_;
};

struct RoundResult {
  ltfb::train::RoundRecord round;
  std::vector<ltfb::train::TrainerRoundRecord> trainer_records;
  std::vector<ltfb::train::TransferRecord> transfers;
};

/// tournament/ltfb.hpp:96-164: every pair's payloads are captured
/// (device-to-device) before any trainer decides; each side's decision and
/// adoption run in a device kernel (ltfb_trainer_tournament_decide).
inline RoundResult tournament_round(std::vector<std::unique_ptr<Trainer>>& trainers,
                                    const ltfb::tournament::Matching& matching, int round_index) {
  const std::uint64_t step = trainers.front()->step();
  for (auto& t : trainers)
    if (t->step() != step) throw ltfb::ContractError("tournament_round: trainers are not step-synchronized");
  RoundResult rr;
  rr.round.round = round_index;
  rr.round.step = step;
  for (const auto& p : matching.pairs) rr.round.pairs.push_back({p[0], p[1]});
  rr.round.bye = matching.bye;
  std::vector<std::pair<int, int>> exchanges;  // (to, from)
  for (const auto& p : matching.pairs) {
    if (p[0] == p[1]) throw ltfb::ContractError("tournament_round: trainer paired with itself");
    for (const auto& [to, from] : {std::pair{p[0], p[1]}, std::pair{p[1], p[0]}}) {
      const auto& m = trainers[static_cast<std::size_t>(from)]->model();
      const auto f = m.fwd.flatten(), i = m.inv.flatten();
      rr.transfers.push_back({round_index, from, to, "fwd", f.size() * 4,
                              ltfb::hex64(ltfb::fnv1a64(f.data(), f.size() * 4))});
      rr.transfers.push_back({round_index, from, to, "inv", i.size() * 4,
                              ltfb::hex64(ltfb::fnv1a64(i.data(), i.size() * 4))});
      exchanges.push_back({to, from});
    }
  }
  for (const auto& [to, from] : exchanges)
    check(ltfb_trainer_copy_incoming(trainers[static_cast<std::size_t>(to)]->handle(),
                                     trainers[static_cast<std::size_t>(from)]->handle()));
  for (const auto& [to, from] : exchanges) {
    auto& t = *trainers[static_cast<std::size_t>(to)];
    const std::string disc_hash = ltfb::hex64(t.model().disc_hash());
    ltfb_eval_metric loc{}, inc{};
    int32_t adopted = 0;
    check(ltfb_trainer_tournament_decide(t.handle(), &loc, &inc, &adopted));
    t.invalidate();
    rr.trainer_records.push_back({round_index, step, to, from, loc.combined, inc.combined, adopted != 0, disc_hash});
  }
  std::sort(rr.trainer_records.begin(), rr.trainer_records.end(),
            [](const auto& a, const auto& b) { return a.trainer < b.trainer; });
  return rr;
}

}  // namespace ltfb_b200
