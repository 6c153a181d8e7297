// TEST INFRASTRUCTURE (oracle) — the reference's own CPU path, timed.
//
// Built by oracle/Makefile from the UNMODIFIED reference headers
// (/root/reference/proj/include) with the OpenBLAS-backed Eigen shim, and
// run by bench.py --impl reference / the cpu_baseline leg on the GPU box's
// host cores. It drives the reference's public API exactly as
// run_experiment does (tournament/runner.hpp:232-437): per-trainer models
// from a shared frozen autoencoder, train::Trainer over an LBDS bundle
// dataset, train_steps chunks on std::async workers, pair_trainers +
// tournament_round. Autoencoder pre-training is excluded (it is not part of
// the timed hot path on either side).
//
//   ref_bench --dims paper|desk --n N --batch B --trainers K --threads T
//             --steps S --warmup W --interval I --dir DIR
// prints one JSON line.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <future>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "ltfb/ltfb.hpp"

using namespace ltfb;
using Clock = std::chrono::steady_clock;

static double secs(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

int main(int argc, char** argv) {
  std::string dims_name = "paper", dir = "/tmp/ltfb_ref_bench";
  std::uint64_t n = 2000, batch = 128, steps = 3, warmup = 1, interval = 0;
  int trainers = 1, threads = 1;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--dims") dims_name = v;
    else if (k == "--n") n = std::stoull(v);
    else if (k == "--batch") batch = std::stoull(v);
    else if (k == "--trainers") trainers = std::stoi(v);
    else if (k == "--threads") threads = std::stoi(v);
    else if (k == "--steps") steps = std::stoull(v);
    else if (k == "--warmup") warmup = std::stoull(v);
    else if (k == "--interval") interval = std::stoull(v);
    else if (k == "--dir") dir = v;
  }
  surrogate::ModalityDims dims;
  if (dims_name == "paper") dims = surrogate::ModalityDims::paper_scale();
  const surrogate::SurrogateArch arch;

  // dataset: synth generator (spec 1, sampling 1) -> LBDS bundles, 500/file
  const auto t_gen0 = Clock::now();
  synth::GeneratorSpec spec;
  spec.dims = dims;
  spec.spec_seed = 1;
  const synth::SynthGenerator gen(spec);
  std::vector<data::SampleRecord> recs(n);
  {
    const std::uint32_t g = synth::grid_side(n);
    const int nt = std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> pool;
    for (int w = 0; w < nt; ++w)
      pool.emplace_back([&, w] {
        for (std::uint64_t i = w; i < n; i += nt) recs[i] = gen.sample(synth::sweep_point(i, g, 1));
      });
    for (auto& th : pool) th.join();
  }
  std::filesystem::remove_all(dir);
  const auto paths = data::write_bundles(recs, dims, 500, dir);
  recs.clear();
  recs.shrink_to_fit();
  const auto index = data::DatasetIndex::scan(paths);
  const double gen_s = secs(t_gen0, Clock::now());

  const int k = trainers;
  const auto split = tournament::detail::split_dataset(index, k, 0.05, 0.05, 1, k >= 2);
  auto base = surrogate::make_cyclegan<float>(dims, arch, mix_seed({1, 0xae0ULL}));
  base.autoencoder_frozen = true;
  std::vector<std::unique_ptr<train::Trainer>> ts;
  const auto t_load0 = Clock::now();
  for (int t = 0; t < k; ++t) {
    auto model = base;
    surrogate::reinit_gan_nets(model, mix_seed({1, 0x1417ULL, static_cast<std::uint64_t>(t)}));
    train::TrainerConfig tc;
    tc.trainer_id = t;
    tc.n_shards = 1;
    tc.batch_size = batch;
    tc.seed = mix_seed({1, 0x57a7e1ULL, static_cast<std::uint64_t>(t)});
    tc.prefetch_depth = threads > 1 ? 1 : 0;
    tc.train_ids = split.train[t];
    tc.tournament_ids = split.tournament[t];
    ts.push_back(std::make_unique<train::Trainer>(tc, index, std::move(model)));
  }
  const double load_s = secs(t_load0, Clock::now());
  auto run_chunk = [&](std::uint64_t chunk) {
    tournament::detail::parallel_for_indices(k, threads, [&](int t) { ts[t]->train_steps(chunk); });
  };
  run_chunk(warmup);
  const auto t0 = Clock::now();
  run_chunk(steps);
  const double train_s = secs(t0, Clock::now());
  double round_s = 0;
  if (k >= 2 && interval == 0) {
    const auto m = tournament::pair_trainers(k, 1, mix_seed({1, 0x9a18ULL}));
    const auto r0 = Clock::now();
    tournament::tournament_round(ts, m, 1);
    round_s = secs(r0, Clock::now());
  }
  const double samples = static_cast<double>(k) * batch * steps;
  std::printf(
      "{\"ms_per_step\": %.6f, \"samples_per_s\": %.6f, \"round_ms\": %.6f, \"trainers\": %d, "
      "\"threads\": %d, \"batch\": %llu, \"steps\": %llu, \"n\": %llu, \"dims\": \"%s\", "
      "\"gen_s\": %.3f, \"load_s\": %.3f, \"tour_rows\": %zu}\n",
      1e3 * train_s / steps, samples / train_s, 1e3 * round_s, k, threads,
      static_cast<unsigned long long>(batch), static_cast<unsigned long long>(steps),
      static_cast<unsigned long long>(n), dims_name.c_str(), gen_s, load_s, split.tournament[0].size());
  std::filesystem::remove_all(dir);
  return 0;
}
