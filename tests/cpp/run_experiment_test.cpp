// The C++ run_experiment (include/ltfb_b200/runner.hpp) on the reference's
// tiny_k2 run configuration (oracle/golden_dump.cpp scenario_tournament:
// tests/test_tournament.cpp tiny_run_config, 2 LTFB trainers): prints one
// JSON line with the run's history so tests/test_gpu_parity.py can compare it
// with the reference's run (tests/golden/tournament.npz, prefix tiny_k2_).
#include <unistd.h>

#include <cstdio>
#include <filesystem>

#include "ltfb_b200/runner.hpp"

int main(int argc, char** argv) {
  ltfb_b200::RunConfig cfg;
  cfg.data_dir = (std::filesystem::temp_directory_path() / ("ltfb_run_" + std::to_string(::getpid()))).string();
  cfg.gen_n = 800;
  cfg.samples_per_file = 100;
  cfg.dims.image_views = 1;
  cfg.dims.image_channels = 1;
  cfg.dims.image_h = cfg.dims.image_w = 4;
  cfg.arch.enc_hidden = cfg.arch.dec_hidden = cfg.arch.fwd_hidden = cfg.arch.inv_hidden = cfg.arch.disc_hidden = {8};
  cfg.batch_size = 32;
  cfg.ae_steps = 15;
  cfg.seed = 42;
  cfg.mode = ltfb_b200::RunMode::kLtfb;
  cfg.trainers = 2;
  cfg.interval = 10;
  cfg.step_budget = 30;
  if (argc > 1) cfg.devices = {0, std::atoi(argv[1])};
  const auto res = ltfb_b200::run_experiment(cfg);
  std::filesystem::remove_all(cfg.data_dir);
  const auto& h = res.history;
  auto list = [](const char* name, const auto& v, auto get, bool last = false) {
    std::printf("\"%s\": [", name);
    for (std::size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? ", " : "", (double)get(v[i]));
    std::printf("]%s", last ? "" : ", ");
  };
  std::printf("{");
  list("pretrain_loss", h.pretrain, [](const auto& r) { return r.loss; });
  list("steps_trainer", h.steps, [](const auto& r) { return r.trainer; });
  list("steps_step", h.steps, [](const auto& r) { return r.step; });
  list("steps_d_loss", h.steps, [](const auto& r) { return r.d_loss; });
  list("steps_g_total", h.steps, [](const auto& r) { return r.g_total; });
  list("tr_kept", h.trainer_rounds, [](const auto& r) { return r.kept_incoming ? 1 : 0; });
  list("tr_local", h.trainer_rounds, [](const auto& r) { return r.local_metric; });
  list("evals_combined", h.evals, [](const auto& r) { return r.combined; });
  list("epochs_epoch", h.epochs, [](const auto& r) { return r.epoch; });
  list("epochs_files_opened", h.epochs, [](const auto& r) { return r.files_opened; });
  list("epochs_bytes_read", h.epochs, [](const auto& r) { return r.bytes_read; });
  list("summary_files_opened", h.summaries, [](const auto& r) { return r.files_opened; });
  list("summary_bytes_read", h.summaries, [](const auto& r) { return r.bytes_read; });
  std::printf("\"best_trainer\": %d}\n", res.best_trainer);
  return 0;
}
