// C++ drop-in of tournament::run_experiment (tournament/runner.hpp:232-437)
// over the façade Trainer / tournament_round (trainer.hpp in this directory):
// the same split, autoencoder pre-training (on the device, ltfb_trainer_ae_step),
// per-trainer re-initialisation, chunk loop with validation evaluations,
// LTFB rounds, best-of-k selection and per-trainer summaries, with the
// reference's RunConfig / RunResult names. Header-only; link -lltfb_gpu.
#pragma once

#include <filesystem>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "trainer.hpp"

namespace ltfb_b200 {

/// tournament/runner.hpp:30-44.
enum class RunMode { kSingle, kLtfb, kKIndependent };

/// tournament/runner.hpp:46-78 (B200: the preload store only; `devices`
/// places trainer t on devices[t % size]).
struct RunConfig {
  std::string data_dir;
  bool generate = true;
  std::uint64_t gen_n = 16000;
  std::uint32_t samples_per_file = 500;
  std::uint64_t sampling_seed = 1;
  std::uint64_t spec_seed = 1;
  double noise_level = 0.0;
  ModalityDims dims;
  SurrogateArch arch;
  RunMode mode = RunMode::kSingle;
  int trainers = 1;
  int shards = 1;
  std::size_t batch_size = 128;
  std::uint64_t interval = 100;
  std::uint64_t step_budget = 1000;
  std::uint64_t ae_steps = 2000;
  int threads = 1;
  std::uint64_t seed = 1;
  double validation_fraction = 0.05;
  double tournament_fraction = 0.05;
  int numeric_abort_threshold = 10;
  double w_f = 1.0;
  double w_i = 1.0;
  std::vector<int> devices{0};
};

/// tournament/runner.hpp:80-85.
struct RunResult {
  ltfb::train::RunHistory history;
  int best_trainer = -1;
  EvalMetric best_metric;
  CycleGan<float> best_model;
};

namespace detail {

inline void validate_run_config(const RunConfig& cfg) {  // runner.hpp:91-110
  std::string problems;
  auto bad = [&](const std::string& msg) { problems += msg + "; "; };
  if (cfg.trainers < 1) bad("trainers must be >= 1");
  if (cfg.shards < 1) bad("shards must be >= 1");
  if (cfg.batch_size < 1) bad("batch_size must be >= 1");
  if (cfg.interval < 1) bad("interval must be >= 1");
  if (cfg.threads < 1) bad("threads must be >= 1");
  if (!(cfg.validation_fraction >= 0 && cfg.validation_fraction < 1)) bad("validation_fraction must be in [0,1)");
  if (!(cfg.tournament_fraction >= 0 && cfg.tournament_fraction < 1)) bad("tournament_fraction must be in [0,1)");
  if (cfg.numeric_abort_threshold < 0) bad("numeric_abort_threshold must be >= 0");
  if (cfg.devices.empty()) bad("devices must not be empty");
  if (!problems.empty()) throw ltfb::ConfigError("invalid run config: " + problems);
  cfg.dims.validate();
}

inline std::vector<float> rows_y(const ltfb::data::DatasetIndex& index, const std::vector<std::uint32_t>& ids,
                                 std::vector<float>* x_out = nullptr) {
  const std::size_t in = index.dims.input_dim, out = index.dims.output_dim();
  std::vector<float> x(ids.size() * in), y(ids.size() * out);
  ltfb::data::read_records(index, std::span<const std::uint32_t>(ids), x.data(), y.data(), out);
  if (x_out) *x_out = std::move(x);
  return y;
}

/// runner.hpp:247-279: AE pre-training on the sorted union of the training
/// partitions (batches drawn with replacement by Rng(mix_seed({seed,
/// 0xae1}))) on the device, then frozen.
inline CycleGan<float> pretrain(const RunConfig& cfg, const ltfb::data::DatasetIndex& index,
                                const std::vector<std::vector<std::uint32_t>>& train,
                                std::vector<ltfb::train::PretrainRecord>& log) {
  auto base = ltfb::surrogate::make_cyclegan<float>(cfg.dims, cfg.arch, ltfb::mix_seed({cfg.seed, 0xae0ULL}));
  if (cfg.ae_steps > 0) {
    std::vector<std::uint32_t> uni;
    for (const auto& p : train) uni.insert(uni.end(), p.begin(), p.end());
    std::sort(uni.begin(), uni.end());
    const std::vector<float> ay = rows_y(index, uni);
    const std::size_t rows = uni.size(), b = std::min<std::size_t>(cfg.batch_size, rows);
    const ltfb_dims d = to_c(cfg.dims);
    const ltfb_arch a = arch_of(base);
    ltfb_trainer_config c{};
    c.device = cfg.devices.front();
    c.n_shards = 1;
    c.numeric_abort_threshold = 10;
    c.batch_size = b;
    c.w_f = c.w_i = 1.0;
    ltfb_trainer* h = nullptr;
    check(ltfb_trainer_create(&d, &a, &c, &h));
    std::unique_ptr<ltfb_trainer, void (*)(ltfb_trainer*)> guard(h, [](ltfb_trainer* t) { ltfb_trainer_destroy(t); });
    const ltfb::nn::MlpParams<float>* nets[5] = {&base.enc, &base.dec, &base.fwd, &base.inv, &base.disc};
    const ltfb::nn::AdamState<float>* opts[5] = {&base.enc_opt, &base.dec_opt, &base.fwd_opt, &base.inv_opt,
                                                 &base.disc_opt};
    for (int k = 0; k < 5; ++k) {
      const auto blob = nets[k]->flatten();
      check(ltfb_trainer_set_params(h, k, blob.data(), blob.size()));
      check(ltfb_trainer_set_adam(h, k, opts[k]->m.data(), opts[k]->v.data(), opts[k]->t));
    }
    check(ltfb_trainer_load_ae_source(h, ay.data(), rows));
    std::vector<std::uint32_t> draws(b * cfg.ae_steps);
    check(ltfb_ae_batch_rows(cfg.seed, rows, b, cfg.ae_steps, draws.data()));
    for (std::uint64_t s = 0; s < cfg.ae_steps; ++s) {
      double loss = 0;
      check(ltfb_trainer_ae_step(h, draws.data() + s * b, b, &loss));
      log.push_back({s + 1, loss});
    }
    const std::pair<int, ltfb::nn::MlpParams<float>*> ae[2] = {{LTFB_NET_ENC, &base.enc}, {LTFB_NET_DEC, &base.dec}};
    ltfb::nn::AdamState<float>* aopt[2] = {&base.enc_opt, &base.dec_opt};
    const ltfb::nn::MlpSpec* specs[2] = {&base.enc_spec, &base.dec_spec};
    for (int k = 0; k < 2; ++k) {
      std::vector<float> blob(ae[k].second->param_count());
      check(ltfb_trainer_get_params(h, ae[k].first, blob.data(), blob.size()));
      *ae[k].second = ltfb::nn::MlpParams<float>::unflatten(*specs[k], std::span<const float>(blob));
      check(ltfb_trainer_get_adam(h, ae[k].first, aopt[k]->m.data(), aopt[k]->v.data(), &aopt[k]->t));
    }
  }
  base.autoencoder_frozen = true;
  return base;
}

}  // namespace detail

/// tournament::run_experiment(const RunConfig&, const DatasetIndex&)
/// (runner.hpp:232-437) with the trainers on the GPUs of cfg.devices.
inline RunResult run_experiment(const RunConfig& cfg, const ltfb::data::DatasetIndex& index) {
  detail::validate_run_config(cfg);
  if (!(index.dims == cfg.dims)) throw ltfb::ConfigError("configured dims do not match the dataset on disk");
  const int k = cfg.mode == RunMode::kSingle ? 1 : cfg.trainers;
  const bool rounds_enabled = cfg.mode == RunMode::kLtfb && k >= 2;
  RunResult result;
  result.history.mode = cfg.mode == RunMode::kSingle ? "single" : (cfg.mode == RunMode::kLtfb ? "ltfb" : "k-independent");
  result.history.n_trainers = k;
  const auto split = ltfb::tournament::detail::split_dataset(index.total, k, cfg.validation_fraction,
                                                             cfg.tournament_fraction, cfg.seed, k >= 2);
  const auto base = detail::pretrain(cfg, index, split.train, result.history.pretrain);

  std::vector<std::unique_ptr<Trainer>> trainers;
  for (int t = 0; t < k; ++t) {
    auto model = base;
    ltfb::surrogate::reinit_gan_nets(model, ltfb::mix_seed({cfg.seed, 0x1417ULL, static_cast<std::uint64_t>(t)}));
    TrainerConfig tc;
    tc.trainer_id = t;
    tc.n_shards = cfg.shards;
    tc.batch_size = cfg.batch_size;
    tc.seed = ltfb::mix_seed({cfg.seed, 0x57a7e1ULL, static_cast<std::uint64_t>(t)});
    tc.numeric_abort_threshold = cfg.numeric_abort_threshold;
    tc.w_f = cfg.w_f;
    tc.w_i = cfg.w_i;
    tc.train_ids = split.train[static_cast<std::size_t>(t)];
    tc.tournament_ids = split.tournament[static_cast<std::size_t>(t)];
    tc.device = cfg.devices[static_cast<std::size_t>(t) % cfg.devices.size()];
    trainers.push_back(std::make_unique<Trainer>(std::move(tc), index, model));
  }
  const bool have_validation = !split.validation.empty();
  if (have_validation) {
    std::vector<float> vx;
    const std::vector<float> vy = detail::rows_y(index, split.validation, &vx);
    for (auto& t : trainers) t->set_validation(vx.data(), vy.data(), split.validation.size());
  }
  auto evaluate_all = [&](std::uint64_t at_step) {
    if (!have_validation) return;
    for (auto& t : trainers) {
      const auto m = t->evaluate_validation(cfg.w_f, cfg.w_i);
      t->history().evals.push_back({t->id(), at_step, "validation", m.forward_mae, m.inverse_mae, m.combined});
    }
  };
  evaluate_all(0);
  std::uint64_t done = 0;
  int round_index = 0;
  while (done < cfg.step_budget) {
    const std::uint64_t chunk = std::min<std::uint64_t>(cfg.interval, cfg.step_budget - done);
    for (auto& t : trainers) t->train_steps(chunk);
    done += chunk;
    evaluate_all(done);
    if (rounds_enabled && chunk == cfg.interval) {  // rounds at full interval boundaries only
      ++round_index;
      const auto matching = ltfb::tournament::pair_trainers(k, round_index, ltfb::mix_seed({cfg.seed, 0x9a18ULL}));
      auto round = tournament_round(trainers, matching, round_index);
      result.history.rounds.push_back(std::move(round.round));
      result.history.trainer_rounds.insert(result.history.trainer_rounds.end(), round.trainer_records.begin(),
                                           round.trainer_records.end());
      result.history.transfers.insert(result.history.transfers.end(), round.transfers.begin(),
                                      round.transfers.end());
    }
  }
  for (auto& t : trainers) t->flush_epoch_record();
  for (auto& t : trainers) {  // runner.hpp:171-197 merge_segments
    auto& seg = t->history();
    result.history.steps.insert(result.history.steps.end(), seg.steps.begin(), seg.steps.end());
    result.history.evals.insert(result.history.evals.end(), seg.evals.begin(), seg.evals.end());
    result.history.epochs.insert(result.history.epochs.end(), seg.epochs.begin(), seg.epochs.end());
  }
  auto by = [](const auto& l, const auto& r) { return std::pair(l.step, l.trainer) < std::pair(r.step, r.trainer); };
  std::stable_sort(result.history.steps.begin(), result.history.steps.end(), by);
  std::stable_sort(result.history.evals.begin(), result.history.evals.end(), by);
  std::stable_sort(result.history.epochs.begin(), result.history.epochs.end(), [](const auto& l, const auto& r) {
    return std::pair(l.epoch, l.trainer) < std::pair(r.epoch, r.trainer);
  });
  if (have_validation) {  // best-of-k on the shared validation metric
    double best = std::numeric_limits<double>::infinity();
    for (auto& t : trainers) {
      const auto m = t->evaluate_validation(cfg.w_f, cfg.w_i);
      if (m.combined < best) {
        best = m.combined;
        result.best_trainer = t->id();
        result.best_metric = m;
      }
    }
  } else {
    result.best_trainer = 0;
  }
  result.best_model = trainers[static_cast<std::size_t>(std::max(result.best_trainer, 0))]->model();
  result.history.best_trainer = result.best_trainer;
  result.history.best_metric = result.best_metric;
  for (auto& t : trainers) {  // runner.hpp:395-431
    ltfb::train::TrainerSummary s;
    s.trainer = t->id();
    s.steps = t->step();
    for (const auto& rec : t->history().steps)
      if (!rec.skipped) {
        s.final_d_loss = rec.d_loss;
        s.final_g_total = rec.g_total;
        s.final_g_fwd = rec.g_fwd;
        s.final_g_adv = rec.g_adv;
        s.final_g_cyc = rec.g_cyc;
      }
    for (const auto& rec : t->history().epochs)
      if (rec.epoch > 0 && !rec.partial) s.epochs_completed += 1;
    for (const auto& rec : t->history().evals)
      if (rec.slice == "validation") {
        s.final_val_forward_mae = rec.forward_mae;
        s.final_val_inverse_mae = rec.inverse_mae;
        s.final_val_combined = rec.combined;
      }
    for (const auto& rec : result.history.trainer_rounds)
      if (rec.trainer == t->id()) {
        s.rounds += 1;
        if (rec.kept_incoming) s.incoming_adopted += 1;
      }
    const auto& counters = t->store().counters();
    s.files_opened = counters.files_opened;
    s.bytes_read = counters.bytes_read;
    s.samples_shuffled = counters.samples_shuffled;
    s.skipped_steps = t->history().skipped_steps;
    s.is_best = t->id() == result.best_trainer;
    result.history.summaries.push_back(s);
  }
  return result;
}

/// runner.hpp:203-230 + run_experiment(cfg): the bundles under cfg.data_dir,
/// generated there first (device-independent host generator through the
/// library) when none exist and cfg.generate is set.
inline ltfb::data::DatasetIndex ensure_dataset(const RunConfig& cfg) {
  namespace fs = std::filesystem;
  bool have = false;
  std::error_code ec;
  if (fs::is_directory(cfg.data_dir, ec))
    for (const auto& e : fs::directory_iterator(cfg.data_dir, ec))
      if (e.path().extension() == ".lbds") have = true;
  if (!have) {
    if (!cfg.generate) throw ltfb::IoError("no dataset found under " + cfg.data_dir + " and generation is disabled");
    const ltfb_dims d = to_c(cfg.dims);
    check(ltfb_write_synth_bundles(cfg.data_dir.c_str(), &d, cfg.spec_seed, cfg.noise_level, cfg.gen_n,
                                   cfg.sampling_seed, cfg.samples_per_file, 1));
  }
  return ltfb::data::DatasetIndex::scan_dir(cfg.data_dir);
}

inline RunResult run_experiment(const RunConfig& cfg) { return run_experiment(cfg, ensure_dataset(cfg)); }

}  // namespace ltfb_b200
