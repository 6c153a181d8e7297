// C++ façade smoke/parity program (tests/test_gpu_parity.py runs it): two
// trainers on tiny dims through ltfb_b200::Trainer / tournament_round, the
// reference's own types; prints one JSON line with every step's g_total and
// every round decision so the test can compare it with the Python mirror.
#include <unistd.h>

#include <cstdio>
#include <filesystem>
#include <vector>

#include "ltfb_b200/trainer.hpp"

int main() {
  using namespace ltfb;
  surrogate::ModalityDims dims;
  dims.image_views = 1;
  dims.image_channels = 1;
  dims.image_h = dims.image_w = 4;
  surrogate::SurrogateArch arch;
  arch.enc_hidden = arch.dec_hidden = arch.fwd_hidden = arch.inv_hidden = arch.disc_hidden = {8};
  const std::size_t n = 400, in = dims.input_dim, out = dims.output_dim();
  std::vector<float> x(n * in), y(n * out);
  const ltfb_dims cd = ltfb_b200::to_c(dims);
  ltfb_b200::check(ltfb_synth_generate(&cd, 1, 0.0, 0, n, n, 1, x.data(), y.data(), 1));
  const ltfb_b200::DatasetView ds{dims, n, x.data(), y.data()};
  auto base = surrogate::make_cyclegan<float>(dims, arch, 7);
  base.autoencoder_frozen = true;
  std::vector<std::unique_ptr<ltfb_b200::Trainer>> ts;
  for (int t = 0; t < 2; ++t) {
    auto m = base;
    surrogate::reinit_gan_nets(m, mix_seed({7, 0x1417, static_cast<std::uint64_t>(t)}));
    ltfb_b200::TrainerConfig c;
    c.trainer_id = t;
    c.batch_size = 32;
    c.seed = 100 + t;
    for (std::uint32_t i = 0; i < 180; ++i) c.train_ids.push_back(static_cast<std::uint32_t>(t * 200 + 20 + i));
    for (std::uint32_t i = 0; i < 20; ++i) c.tournament_ids.push_back(static_cast<std::uint32_t>(t * 200 + i));
    ts.push_back(std::make_unique<ltfb_b200::Trainer>(c, ds, m));
  }
  std::printf("{\"g_total\": [");
  bool first = true;
  std::vector<int> kept;
  for (int round = 1; round <= 2; ++round) {
    for (auto& t : ts) t->train_steps(10);
    const auto res = ltfb_b200::tournament_round(ts, tournament::pair_trainers(2, round, 5), round);
    for (const auto& r : res.trainer_records) kept.push_back(r.kept_incoming ? 1 : 0);
  }
  for (auto& t : ts)
    for (const auto& s : t->history().steps) {
      std::printf("%s%.17g", first ? "" : ", ", s.g_total);
      first = false;
    }
  std::printf("], \"kept\": [");
  for (std::size_t i = 0; i < kept.size(); ++i) std::printf("%s%d", i ? ", " : "", kept[i]);
  std::printf("], \"fwd_hash\": \"%s\"}\n", hex64(ts[0]->model().fwd_hash()).c_str());
  {  // the same trainer 0 built from LBDS bundle files (DatasetIndex) trains identically
    std::vector<data::SampleRecord> recs(n);
    for (std::size_t i = 0; i < n; ++i) {
      recs[i].inputs.assign(x.begin() + i * in, x.begin() + (i + 1) * in);
      recs[i].outputs.assign(y.begin() + i * out, y.begin() + (i + 1) * out);
    }
    const auto dir = std::filesystem::temp_directory_path() / ("ltfb_facade_" + std::to_string(::getpid()));
    data::write_bundles(std::span<const data::SampleRecord>(recs), dims, 100, dir);
    const auto index = data::DatasetIndex::scan_dir(dir);
    auto m = base;
    surrogate::reinit_gan_nets(m, mix_seed({7, 0x1417, 0}));
    ltfb_b200::TrainerConfig c;
    c.batch_size = 32;
    c.seed = 100;
    for (std::uint32_t i = 0; i < 180; ++i) c.train_ids.push_back(20 + i);
    for (std::uint32_t i = 0; i < 20; ++i) c.tournament_ids.push_back(i);
    ltfb_b200::Trainer tb(c, index, m);
    tb.train_steps(10);
    if (tb.history().steps.back().g_total != ts[0]->history().steps[9].g_total) return 3;
    // store() / replica_hashes() (trainer.hpp:88-97): the preload read each
    // partition record once from the 2 files covering ids 20..199
    const auto& st = tb.store();
    if (st.size() != 180 || st.counters().files_opened != 2 ||
        st.counters().bytes_read != 180 * dims.record_floats() * 4)
      return 4;
    if (tb.history().epochs.empty() || tb.history().epochs.front().epoch != 0 ||
        tb.history().epochs.front().files_opened != 2)
      return 5;
    const auto hs = tb.replica_hashes();
    if (hs.size() != 1 || hs[0] != tb.model().model_hash()) return 6;
    std::filesystem::remove_all(dir);
  }
  try {  // the reference's error behaviour through the façade
    ts[0]->adopt_generators(ts[1]->model().inv, ts[1]->model().fwd);
    return 2;
  } catch (const ContractError&) {
  }
  return 0;
}
