// TEST INFRASTRUCTURE (oracle) — not product code.
//
// Golden-vector dumper. Compiled (by oracle/Makefile) directly against the
// UNMODIFIED reference headers under /root/reference/proj/include plus the
// strict Eigen shim in oracle/shim, it runs fixed, seeded scenarios through
// the reference's own public API and writes every observable into tagged
// little-endian binary files that oracle/make_golden.py turns into the
// committed fixtures tests/golden/*.npz.
//
// Each scenario names the reference entry points it exercises.
#include <algorithm>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "ltfb/ltfb.hpp"
#include "ltfb/bench/output.hpp"

using namespace ltfb;
namespace fs = std::filesystem;

// --------------------------------------------------------------------------
// Tagged binary writer: per array [u32 name_len][name][u8 dtype][u64 n][data]
// dtype: 0=f32 1=f64 2=u32 3=u64 4=i32 5=i64 6=u8
// --------------------------------------------------------------------------
class Dump {
 public:
  explicit Dump(const fs::path& p) : os_(p, std::ios::binary) {
    if (!os_) throw std::runtime_error("cannot open " + p.string());
  }
  template <typename T>
  void put(const std::string& name, const std::vector<T>& v) {
    const std::uint32_t n = static_cast<std::uint32_t>(name.size());
    os_.write(reinterpret_cast<const char*>(&n), 4);
    os_.write(name.data(), n);
    const std::uint8_t code = dtype<T>();
    os_.write(reinterpret_cast<const char*>(&code), 1);
    const std::uint64_t count = v.size();
    os_.write(reinterpret_cast<const char*>(&count), 8);
    os_.write(reinterpret_cast<const char*>(v.data()),
              static_cast<std::streamsize>(count * sizeof(T)));
  }
  template <typename T>
  void scalar(const std::string& name, T v) { put(name, std::vector<T>{v}); }

 private:
  template <typename T>
  static std::uint8_t dtype() {
    if constexpr (std::is_same_v<T, float>) return 0;
    else if constexpr (std::is_same_v<T, double>) return 1;
    else if constexpr (std::is_same_v<T, std::uint32_t>) return 2;
    else if constexpr (std::is_same_v<T, std::uint64_t>) return 3;
    else if constexpr (std::is_same_v<T, std::int32_t>) return 4;
    else if constexpr (std::is_same_v<T, std::int64_t>) return 5;
    else if constexpr (std::is_same_v<T, std::uint8_t>) return 6;
    else static_assert(sizeof(T) == 0, "unsupported dtype");
  }
  std::ofstream os_;
};

template <typename T>
std::vector<T> flat(const nn::MlpParams<T>& p) { return p.flatten(); }

static std::vector<float> uniform_vec(Rng& rng, std::size_t n, double lo,
                                      double hi) {
  std::vector<float> v(n);
  for (auto& x : v) x = static_cast<float>(rng.uniform(lo, hi));
  return v;
}

static surrogate::ModalityDims tiny_dims() {
  surrogate::ModalityDims d;
  d.image_views = 1;
  d.image_channels = 1;
  d.image_h = 4;
  d.image_w = 4;
  return d;
}

static surrogate::SurrogateArch tiny_arch() {
  surrogate::SurrogateArch a;
  a.enc_hidden = {8};
  a.dec_hidden = {8};
  a.fwd_hidden = {8};
  a.inv_hidden = {8};
  a.disc_hidden = {8};
  return a;
}

static void put_dims(Dump& d, const std::string& pfx,
                     const surrogate::ModalityDims& m) {
  d.put(pfx + "dims", std::vector<std::uint32_t>{m.input_dim, m.latent_dim,
                                           m.scalar_dim, m.image_views,
                                           m.image_channels, m.image_h,
                                           m.image_w});
}

static void put_model(Dump& d, const std::string& pfx,
                      const surrogate::CycleGan<float>& m, bool big = true) {
  if (big) {
    d.put(pfx + "enc", flat(m.enc));
    d.put(pfx + "dec", flat(m.dec));
  }
  d.put(pfx + "fwd", flat(m.fwd));
  d.put(pfx + "inv", flat(m.inv));
  d.put(pfx + "disc", flat(m.disc));
  d.put(pfx + "hashes",
        std::vector<std::uint64_t>{m.enc_hash(), m.dec_hash(), m.fwd_hash(),
                                   m.inv_hash(), m.disc_hash(),
                                   m.model_hash()});
}

// strided sample of a large vector (AE grads / enc-dec blobs at desk and
// paper dims); the stride is stored beside it as NAME_stride.
template <typename T>
void put_strided(Dump& d, const std::string& name, const std::vector<T>& v) {
  const std::size_t stride = v.size() < 1000000 ? 97 : 1009;
  std::vector<T> out;
  for (std::size_t i = 0; i < v.size(); i += stride) out.push_back(v[i]);
  d.put(name, out);
  d.scalar(name + "_stride", static_cast<std::uint64_t>(stride));
}

static void put_steps(Dump& d, const std::string& pfx,
                      const std::vector<train::StepRecord>& steps) {
  std::vector<double> dl, gt, gf, ga, gc;
  std::vector<std::uint64_t> st;
  std::vector<std::int32_t> tr;
  std::vector<std::uint32_t> ep;
  std::vector<std::uint8_t> sk;
  for (const auto& s : steps) {
    dl.push_back(s.d_loss);
    gt.push_back(s.g_total);
    gf.push_back(s.g_fwd);
    ga.push_back(s.g_adv);
    gc.push_back(s.g_cyc);
    st.push_back(s.step);
    tr.push_back(s.trainer);
    ep.push_back(s.epoch);
    sk.push_back(s.skipped ? 1 : 0);
  }
  d.put(pfx + "d_loss", dl);
  d.put(pfx + "g_total", gt);
  d.put(pfx + "g_fwd", gf);
  d.put(pfx + "g_adv", ga);
  d.put(pfx + "g_cyc", gc);
  d.put(pfx + "step", st);
  d.put(pfx + "trainer", tr);
  d.put(pfx + "epoch", ep);
  d.put(pfx + "skipped", sk);
}

static void put_epochs(Dump& d, const std::string& pfx,
                       const std::vector<train::EpochRecord>& eps) {
  std::vector<std::int32_t> tr;
  std::vector<std::uint32_t> ep;
  std::vector<std::uint64_t> steps, files, bytes, shuffled;
  std::vector<std::uint8_t> partial;
  for (const auto& e : eps) {
    tr.push_back(e.trainer);
    ep.push_back(e.epoch);
    steps.push_back(e.steps);
    files.push_back(e.files_opened);
    bytes.push_back(e.bytes_read);
    shuffled.push_back(e.samples_shuffled);
    partial.push_back(e.partial ? 1 : 0);
  }
  d.put(pfx + "trainer", tr);
  d.put(pfx + "epoch", ep);
  d.put(pfx + "steps", steps);
  d.put(pfx + "files_opened", files);
  d.put(pfx + "bytes_read", bytes);
  d.put(pfx + "samples_shuffled", shuffled);
  d.put(pfx + "partial", partial);
}

// ---------------------------------------------------------------------------
// rng: core/rng.hpp:13-97
// ---------------------------------------------------------------------------
static void scenario_rng(const fs::path& out) {
  Dump d(out / "rng.bin");
  d.put("mix_seed", std::vector<std::uint64_t>{
                        mix_seed({1}), mix_seed({1, 2}), mix_seed({42, 0xa11}),
                        mix_seed({7, 3, 0x9a12}), mix_seed({0}),
                        mix_seed({~0ULL, 5}), mix_seed({1, 0x57a7e1, 3}),
                        mix_seed({12345, 0, 0x5caff1e})});
  Rng r(12345);
  std::vector<std::uint64_t> nx;
  for (int i = 0; i < 32; ++i) nx.push_back(r.next());
  d.put("next", nx);
  std::vector<double> un;
  for (int i = 0; i < 16; ++i) un.push_back(r.uniform());
  d.put("uniform", un);
  std::vector<std::uint64_t> bn_n{1, 2, 3, 7, 100, 1000003,
                                  (1ULL << 63) + 5};
  std::vector<std::uint64_t> bl;
  for (auto n : bn_n)
    for (int i = 0; i < 8; ++i) bl.push_back(r.below(n));
  d.put("below_n", bn_n);
  d.put("below", bl);
  std::vector<double> nm;
  for (int i = 0; i < 8; ++i) nm.push_back(r.normal());
  d.put("normal", nm);
  std::vector<std::uint32_t> sh(57);
  for (std::uint32_t i = 0; i < 57; ++i) sh[i] = i;
  Rng r2(99);
  r2.shuffle(sh);
  d.put("shuffle57_seed99", sh);
  d.put("fnv_hello", std::vector<std::uint64_t>{fnv1a64("hello", 5)});
}

// ---------------------------------------------------------------------------
// plan: tournament/ltfb.hpp:24-66, runner.hpp:134-169, epoch_plan.hpp:41-137
// ---------------------------------------------------------------------------
static std::vector<data::SampleId> iota_ids(std::size_t n) {
  std::vector<data::SampleId> v(n);
  for (std::size_t i = 0; i < n; ++i) v[i] = static_cast<data::SampleId>(i);
  return v;
}

static void put_parts(Dump& d, const std::string& pfx,
                      const std::vector<std::vector<data::SampleId>>& parts) {
  std::vector<std::uint32_t> cat, sizes;
  for (const auto& p : parts) {
    sizes.push_back(static_cast<std::uint32_t>(p.size()));
    cat.insert(cat.end(), p.begin(), p.end());
  }
  d.put(pfx + "ids", cat);
  d.put(pfx + "sizes", sizes);
}

static void scenario_plan(const fs::path& out, const fs::path& tmp) {
  Dump d(out / "plan.bin");
  put_parts(d, "part_100_4_5_", tournament::partition_dataset(iota_ids(100), 4, 5));
  put_parts(d, "part_1000_7_11_",
            tournament::partition_dataset(iota_ids(1000), 7, 11));
  // pairings
  std::vector<std::int32_t> pk, pr, pa, pb, byes;
  for (int k : {2, 3, 4, 5, 8})
    for (int round = 1; round <= 25; ++round) {
      const auto m = tournament::pair_trainers(k, round, 0x1234);
      for (const auto& p : m.pairs) {
        pk.push_back(k);
        pr.push_back(round);
        pa.push_back(p[0]);
        pb.push_back(p[1]);
      }
      byes.push_back(m.bye);
    }
  d.put("pair_k", pk);
  d.put("pair_round", pr);
  d.put("pair_a", pa);
  d.put("pair_b", pb);
  d.put("pair_byes", byes);
  // dataset splits
  for (auto [total, k, seed] : {std::tuple<std::size_t, int, std::uint64_t>{800, 2, 42},
                               {16000, 4, 101}, {16000, 8, 1}}) {
    data::DatasetIndex idx;
    idx.total = total;
    const auto split = tournament::detail::split_dataset(idx, k, 0.05, 0.05,
                                                         seed, k >= 2);
    const std::string pfx = "split_" + std::to_string(total) + "_" +
                            std::to_string(k) + "_";
    d.put(pfx + "validation", split.validation);
    put_parts(d, pfx + "train_", split.train);
    put_parts(d, pfx + "tour_", split.tournament);
  }
  // epoch plans over a store partition (no preload: no transfers)
  {
    data::DatasetIndex idx;
    idx.total = 800;
    const auto split =
        tournament::detail::split_dataset(idx, 2, 0.05, 0.05, 42, true);
    data::DataStore store(&idx, split.train[0], data::StoreMode::kNone, 2);
    const std::uint64_t seed = mix_seed({42, 0x57a7e1ULL, 0});
    for (std::uint32_t e = 1; e <= 3; ++e) {
      const auto plan = data::plan_epoch(store, e, seed, 32);
      d.put("plan_perm_e" + std::to_string(e), plan.permutation);
      std::vector<std::uint64_t> sl;
      for (auto [b, en] : plan.slices) {
        sl.push_back(b);
        sl.push_back(en);
      }
      d.put("plan_slices_e" + std::to_string(e), sl);
    }
    d.scalar("plan_seed", seed);
  }
  // transfer lists and shuffle counters from a preloaded 3-shard store
  {
    synth::GeneratorSpec spec;
    spec.dims = tiny_dims();
    spec.spec_seed = 3;
    synth::SynthGenerator gen(spec);
    const auto recs = synth::generate_dataset(gen, 600, 17);
    const fs::path dir = tmp / "plan_ds";
    const auto paths = data::write_bundles(recs, spec.dims, 100, dir);
    const auto idx = data::DatasetIndex::scan(paths);
    std::vector<data::SampleId> part;
    for (data::SampleId i = 30; i < 600; ++i) part.push_back(i);
    data::DataStore store(&idx, part, data::StoreMode::kPreload, 3);
    store.preload();
    store.begin_epoch(1);
    const auto plan = data::plan_epoch(store, 1, 5, 64);
    std::vector<std::uint32_t> tid, step;
    std::vector<std::int32_t> own, con;
    for (std::size_t s = 0; s < plan.transfers.size(); ++s)
      for (const auto& t : plan.transfers[s]) {
        step.push_back(static_cast<std::uint32_t>(s));
        tid.push_back(t.id);
        own.push_back(t.owner);
        con.push_back(t.consumer);
      }
    d.put("xfer_step", step);
    d.put("xfer_id", tid);
    d.put("xfer_owner", own);
    d.put("xfer_consumer", con);
    for (std::size_t s = 0; s < plan.n_steps(); ++s)
      data::shuffle_step(store, plan, s);
    d.scalar("xfer_samples_shuffled", store.counters().samples_shuffled);
    d.scalar("xfer_files_opened", store.counters().files_opened);
    d.scalar("xfer_bytes_read", store.counters().bytes_read);
    std::vector<std::int32_t> owners;
    for (data::SampleId i = 30; i < 600; ++i) owners.push_back(store.owner_of(i));
    d.put("xfer_owner_of", owners);
  }
}

// ---------------------------------------------------------------------------
// synth: synth/generator.hpp:71-206
// ---------------------------------------------------------------------------
static void put_records(Dump& d, const std::string& pfx,
                        const std::vector<data::SampleRecord>& recs) {
  std::vector<float> x, y;
  for (const auto& r : recs) {
    x.insert(x.end(), r.inputs.begin(), r.inputs.end());
    y.insert(y.end(), r.outputs.begin(), r.outputs.end());
  }
  d.put(pfx + "x", x);
  d.put(pfx + "y", y);
}

static void scenario_synth(const fs::path& out) {
  Dump d(out / "synth.bin");
  {
    synth::GeneratorSpec spec;
    spec.dims = tiny_dims();
    spec.spec_seed = 3;
    synth::SynthGenerator gen(spec);
    put_records(d, "tiny_", synth::generate_dataset(gen, 200, 17));
    spec.noise_level = 0.1;
    synth::SynthGenerator noisy(spec);
    put_records(d, "tiny_noisy_", synth::generate_dataset(noisy, 20, 17));
  }
  {
    synth::GeneratorSpec spec;  // desk dims
    spec.spec_seed = 1;
    synth::SynthGenerator gen(spec);
    const std::uint32_t g = synth::grid_side(16000);
    std::vector<data::SampleRecord> recs;
    std::vector<std::uint64_t> which{0, 1, 777, 15999};
    for (auto i : which) recs.push_back(gen.sample(synth::sweep_point(i, g, 1)));
    put_records(d, "desk_", recs);
    d.put("desk_which", which);
    d.scalar("grid_side_16000", g);
  }
  {
    synth::GeneratorSpec spec;
    spec.dims = surrogate::ModalityDims::paper_scale();
    spec.spec_seed = 1;
    synth::SynthGenerator gen(spec);
    const std::uint32_t g = synth::grid_side(16000);
    std::vector<data::SampleRecord> recs;
    recs.push_back(gen.sample(synth::sweep_point(12345, g, 1)));
    put_records(d, "paper_", recs);
  }
}

// ---------------------------------------------------------------------------
// nn: mlp.hpp:149-282, loss.hpp:24-88, adam.hpp:87-122
// ---------------------------------------------------------------------------
static void mlp_case(Dump& d, const std::string& pfx, nn::MlpSpec spec,
                     std::size_t rows, std::uint64_t data_seed) {
  const auto params = nn::init_params<float>(spec);
  Rng rng(data_seed);
  auto x = nn::Tensor<float>::from_data(
      {rows, spec.in_dim()}, uniform_vec(rng, rows * spec.in_dim(), -1, 1));
  auto g = nn::Tensor<float>::from_data(
      {rows, spec.out_dim()}, uniform_vec(rng, rows * spec.out_dim(), -1, 1));
  const auto tape = nn::mlp_forward(spec, params, x);
  const auto back = nn::mlp_backward(spec, params, tape, g);
  std::vector<std::uint32_t> widths(spec.layer_widths.begin(),
                                    spec.layer_widths.end());
  std::vector<std::int32_t> acts;
  std::vector<double> slopes;
  for (const auto& a : spec.activations) {
    acts.push_back(static_cast<std::int32_t>(a.kind));
    slopes.push_back(a.slope);
  }
  d.put(pfx + "widths", widths);
  d.put(pfx + "acts", acts);
  d.put(pfx + "slopes", slopes);
  d.scalar(pfx + "init_seed", spec.init_seed);
  d.put(pfx + "params", params.flatten());
  d.put(pfx + "x", x.data);
  d.put(pfx + "gout", g.data);
  d.put(pfx + "out", tape.output().data);
  d.put(pfx + "apply", nn::mlp_apply(spec, params, x).data);
  d.put(pfx + "pgrad", back.param_grads.flatten());
  d.put(pfx + "gin", back.grad_input.data);
}

static void scenario_nn(const fs::path& out) {
  Dump d(out / "nn.bin");
  using nn::Act;
  nn::MlpSpec a;
  a.layer_widths = {7, 5, 3};
  a.activations = {{Act::kLeakyRelu, 0.2}, {Act::kIdentity}};
  a.init_seed = 77;
  mlp_case(d, "mlpA_", a, 4, 5);
  nn::MlpSpec b;
  b.layer_widths = {6, 8, 8, 8, 8, 2};
  b.activations = {{Act::kRelu}, {Act::kTanh}, {Act::kSigmoid},
                   {Act::kLeakyRelu, 0.2}, {Act::kIdentity}};
  b.init_seed = 78;
  mlp_case(d, "mlpB_", b, 9, 6);
  nn::MlpSpec c;  // the default fwd net shape
  c.layer_widths = {5, 32, 32, 20};
  c.activations = {{Act::kLeakyRelu, 0.2}, {Act::kLeakyRelu, 0.2},
                   {Act::kIdentity}};
  c.init_seed = mix_seed({1, 3});
  mlp_case(d, "mlpC_", c, 128, 7);

  // losses
  Rng rng(31);
  auto p = nn::Tensor<float>::from_data({3, 5}, uniform_vec(rng, 15, -1, 1));
  auto t = nn::Tensor<float>::from_data({3, 5}, uniform_vec(rng, 15, -1, 1));
  t[4] = p[4];  // an exact tie (zero subgradient)
  const auto mae = nn::mae_loss(p, t);
  d.put("mae_p", p.data);
  d.put("mae_t", t.data);
  d.scalar("mae_value", mae.value);
  d.put("mae_grad", mae.grad.data);
  auto logits = nn::Tensor<float>::from_data({8, 1}, uniform_vec(rng, 8, -30, 30));
  logits[0] = 0.0f;
  logits[1] = 40.0f;
  logits[2] = -40.0f;
  const auto probs = nn::sigmoid(logits);
  nn::Tensor<float> labels({8, 1});
  for (int i = 0; i < 8; i += 2) labels[i] = 1.0f;
  const auto bce = nn::bce_loss(probs, labels);
  d.put("bce_logits", logits.data);
  d.put("bce_probs", probs.data);
  d.put("bce_labels", labels.data);
  d.scalar("bce_value", bce.value);
  d.put("bce_grad", bce.grad.data);

  // Adam: 3 steps on a 50-parameter blob
  nn::MlpSpec s;
  s.layer_widths = {6, 7, 1};
  s.activations = {{Act::kLeakyRelu, 0.2}, {Act::kIdentity}};
  s.init_seed = 5;
  auto params = nn::init_params<float>(s);
  auto state = nn::AdamState<float>::for_params(params, nn::AdamHyper{});
  d.put("adam_p0", params.flatten());
  for (int step = 1; step <= 3; ++step) {
    auto grads = nn::MlpParams<float>::zeros_like(s);
    std::vector<float> gv = uniform_vec(rng, params.param_count(), -0.1, 0.1);
    auto gp = nn::MlpParams<float>::unflatten(s, gv);
    nn::adam_step(params, gp, state);
    d.put("adam_g" + std::to_string(step), gv);
    d.put("adam_p" + std::to_string(step), params.flatten());
    d.put("adam_m" + std::to_string(step), state.m);
    d.put("adam_v" + std::to_string(step), state.v);
  }
}

// ---------------------------------------------------------------------------
// surrogate: model.hpp:96-147, train_ops.hpp:52-205
// ---------------------------------------------------------------------------
static void surrogate_case(Dump& d, const std::string& pfx,
                           const surrogate::ModalityDims& dims,
                           const surrogate::SurrogateArch& arch,
                           std::uint64_t seed, const nn::Tensor<float>& x,
                           const nn::Tensor<float>& y, bool big_blobs,
                           bool ae_grads, bool store_y) {
  auto m = surrogate::make_cyclegan<float>(dims, arch, seed);
  put_dims(d, pfx, dims);
  d.scalar(pfx + "seed", seed);
  put_model(d, pfx + "init_", m, big_blobs);
  d.put(pfx + "x", x.data);
  if (store_y) d.put(pfx + "y", y.data);
  nn::MlpParams<float> dg, fg, ig, eg, decg;
  const double dl = surrogate::discriminator_backward(m, x, y, &dg);
  d.scalar(pfx + "d_loss", dl);
  d.put(pfx + "disc_grad", flat(dg));
  const auto gl = surrogate::generator_backward(m, x, y, &fg, &ig);
  d.put(pfx + "gen_losses", std::vector<double>{gl.total, gl.fwd, gl.adv, gl.cyc});
  d.put(pfx + "fwd_grad", flat(fg));
  d.put(pfx + "inv_grad", flat(ig));
  const double al = surrogate::autoencoder_backward(m, y, &eg, &decg);
  d.scalar(pfx + "ae_loss", al);
  if (ae_grads) {
    d.put(pfx + "enc_grad", flat(eg));
    d.put(pfx + "dec_grad", flat(decg));
  } else {
    put_strided(d, pfx + "enc_grad_strided", flat(eg));
    put_strided(d, pfx + "dec_grad_strided", flat(decg));
  }
  const auto e1 = surrogate::evaluate(m, x, y);
  const auto e2 = surrogate::evaluate(m, x, y, 0.7, 0.3);
  d.put(pfx + "eval", std::vector<double>{e1.forward_mae, e1.inverse_mae,
                                          e1.combined, e2.forward_mae,
                                          e2.inverse_mae, e2.combined});
  // one full D-then-G step with the *_step API
  m.autoencoder_frozen = true;
  const double ds = surrogate::discriminator_step(m, x, y);
  const auto gs = surrogate::generator_step(m, x, y);
  d.put(pfx + "step_losses", std::vector<double>{ds, gs.total, gs.fwd, gs.adv, gs.cyc});
  put_model(d, pfx + "after_", m, false);
}

static nn::Tensor<float> rows_x(const std::vector<data::SampleRecord>& r) {
  nn::Tensor<float> t({r.size(), r.front().inputs.size()});
  for (std::size_t i = 0; i < r.size(); ++i)
    std::copy(r[i].inputs.begin(), r[i].inputs.end(),
              t.data.begin() + static_cast<std::ptrdiff_t>(i * t.cols()));
  return t;
}
static nn::Tensor<float> rows_y(const std::vector<data::SampleRecord>& r) {
  nn::Tensor<float> t({r.size(), r.front().outputs.size()});
  for (std::size_t i = 0; i < r.size(); ++i)
    std::copy(r[i].outputs.begin(), r[i].outputs.end(),
              t.data.begin() + static_cast<std::ptrdiff_t>(i * t.cols()));
  return t;
}

static void scenario_surrogate(const fs::path& out) {
  Dump d(out / "surrogate.bin");
  {
    Rng rng(8);
    const auto dims = tiny_dims();
    auto x = nn::Tensor<float>::from_data({16, 5}, uniform_vec(rng, 80, 0, 1));
    auto y = nn::Tensor<float>::from_data({16, 31}, uniform_vec(rng, 16 * 31, -1, 2));
    surrogate_case(d, "tiny_", dims, tiny_arch(), 3, x, y, true, true, true);
  }
  {
    surrogate::ModalityDims dims;  // desk
    synth::GeneratorSpec spec;
    spec.spec_seed = 1;
    synth::SynthGenerator gen(spec);
    const auto recs = synth::generate_dataset(gen, 16, 5);
    surrogate_case(d, "desk_", dims, surrogate::SurrogateArch{}, 11,
                   rows_x(recs), rows_y(recs), false, false, true);
  }
  {
    // paper dims: inputs regenerated by the consumer from
    // generate_dataset(spec_seed 1, n = 8, sampling_seed 5)
    const auto dims = surrogate::ModalityDims::paper_scale();
    synth::GeneratorSpec spec;
    spec.dims = dims;
    spec.spec_seed = 1;
    synth::SynthGenerator gen(spec);
    const auto recs = synth::generate_dataset(gen, 8, 5);
    surrogate_case(d, "paper_", dims, surrogate::SurrogateArch{}, 11,
                   rows_x(recs), rows_y(recs), false, false, false);
  }
}

// ---------------------------------------------------------------------------
// trainer: train/trainer.hpp:41-308 (single trainer, Fixture of
// tests/test_trainer.cpp:36-75 generalised)
// ---------------------------------------------------------------------------
struct DataFixture {
  fs::path dir;
  data::DatasetIndex index;
  DataFixture(const fs::path& d, const surrogate::ModalityDims& dims,
              std::uint64_t n, std::size_t per_file, std::uint64_t spec_seed,
              std::uint64_t sampling_seed)
      : dir(d) {
    synth::GeneratorSpec spec;
    spec.dims = dims;
    spec.spec_seed = spec_seed;
    synth::SynthGenerator gen(spec);
    const auto recs = synth::generate_dataset(gen, n, sampling_seed);
    const auto paths = data::write_bundles(recs, dims, per_file, dir);
    index = data::DatasetIndex::scan(paths);
  }
};

static train::TrainerConfig trainer_cfg(const data::DatasetIndex& index,
                                        int shards, std::size_t batch,
                                        std::uint64_t seed,
                                        std::size_t n_tour) {
  train::TrainerConfig tc;
  tc.trainer_id = 0;
  tc.n_shards = shards;
  tc.batch_size = batch;
  tc.store_mode = data::StoreMode::kPreload;
  tc.seed = seed;
  tc.prefetch_depth = 0;
  for (std::size_t i = 0; i < index.total; ++i) {
    if (i < n_tour) tc.tournament_ids.push_back(static_cast<data::SampleId>(i));
    else tc.train_ids.push_back(static_cast<data::SampleId>(i));
  }
  return tc;
}

static void trainer_case(Dump& d, const std::string& pfx,
                         const DataFixture& fx,
                         const surrogate::ModalityDims& dims,
                         const surrogate::SurrogateArch& arch,
                         std::uint64_t model_seed, int shards,
                         std::size_t batch, std::uint64_t seed,
                         std::size_t n_tour, std::size_t steps) {
  auto model = surrogate::make_cyclegan<float>(dims, arch, model_seed);
  model.autoencoder_frozen = true;
  train::Trainer t(trainer_cfg(fx.index, shards, batch, seed, n_tour),
                   fx.index, model);
  const auto e0 = t.eval_tournament(t.model());
  t.train_steps(steps);
  const auto e1 = t.eval_tournament(t.model());
  t.flush_epoch_record();
  put_steps(d, pfx + "steps_", t.history().steps);
  put_epochs(d, pfx + "epochs_", t.history().epochs);
  put_model(d, pfx + "final_", t.model(), false);
  d.put(pfx + "eval0", std::vector<double>{e0.forward_mae, e0.inverse_mae, e0.combined});
  d.put(pfx + "eval1", std::vector<double>{e1.forward_mae, e1.inverse_mae, e1.combined});
  d.put(pfx + "replica_hashes", t.replica_hashes());
  d.put(pfx + "cfg", std::vector<std::uint64_t>{model_seed, static_cast<std::uint64_t>(shards),
                                                batch, seed, n_tour, steps});
  d.put(pfx + "fwd_m", t.model().fwd_opt.m);
  d.put(pfx + "fwd_v", t.model().fwd_opt.v);
  d.put(pfx + "opt_t", std::vector<std::uint64_t>{t.model().fwd_opt.t,
                                                  t.model().inv_opt.t,
                                                  t.model().disc_opt.t});
}

static void scenario_trainer(const fs::path& out, const fs::path& tmp) {
  Dump d(out / "trainer.bin");
  {
    DataFixture fx(tmp / "tr_tiny", tiny_dims(), 600, 100, 3, 17);
    d.put("tiny_data", std::vector<std::uint64_t>{600, 100, 3, 17});
    put_dims(d, "tiny_", tiny_dims());
    trainer_case(d, "tiny_s1_", fx, tiny_dims(), tiny_arch(), 3, 1, 64, 7, 30, 20);
    trainer_case(d, "tiny_s2_", fx, tiny_dims(), tiny_arch(), 3, 2, 64, 7, 30, 20);
    trainer_case(d, "tiny_s4_", fx, tiny_dims(), tiny_arch(), 3, 4, 64, 7, 30, 20);
    // numeric skip -> abort (tests/test_trainer.cpp:208-222)
    auto model = surrogate::make_cyclegan<float>(tiny_dims(), tiny_arch(), 6);
    model.autoencoder_frozen = true;
    for (auto& w : model.fwd.weights)
      for (auto& v : w.data) v = 1e38f;
    auto cfg = trainer_cfg(fx.index, 1, 32, 10, 30);
    cfg.numeric_abort_threshold = 3;
    train::Trainer t(cfg, fx.index, model);
    bool threw = false;
    try {
      t.train_steps(10);
    } catch (const NumericError&) {
      threw = true;
    }
    d.scalar("abort_threw", static_cast<std::uint8_t>(threw));
    put_steps(d, "abort_steps_", t.history().steps);
    d.scalar("abort_skipped", t.history().skipped_steps);
    d.scalar("abort_step", t.step());
  }
  {
    surrogate::ModalityDims dims;  // desk 16x16
    DataFixture fx(tmp / "tr_desk", dims, 400, 100, 1, 1);
    d.put("desk_data", std::vector<std::uint64_t>{400, 100, 1, 1});
    put_dims(d, "desk_", dims);
    // partition 370, B = 32 -> 12 steps/epoch with a short last slice (18)
    trainer_case(d, "desk_s1_", fx, dims, surrogate::SurrogateArch{}, 3, 1, 32, 7, 30, 14);
    trainer_case(d, "desk_s2_", fx, dims, surrogate::SurrogateArch{}, 3, 2, 32, 7, 30, 14);
  }
  {
    const auto dims = surrogate::ModalityDims::paper_scale();
    DataFixture fx(tmp / "tr_paper", dims, 300, 100, 1, 1);
    d.put("paper_data", std::vector<std::uint64_t>{300, 100, 1, 1});
    put_dims(d, "paper_", dims);
    // partition 270, B = 128 -> 3 steps/epoch (128, 128, 14)
    trainer_case(d, "paper_s1_", fx, dims, surrogate::SurrogateArch{}, 3, 1, 128, 7, 30, 4);
  }
}

// activations: trainer cases with the other hidden activations the
// reference supports (nn/activation.hpp:43-77: relu, tanh, sigmoid), tiny and
// desk dims, so the device's activation / derivative paths are pinned too.
static void scenario_activations(const fs::path& out, const fs::path& tmp) {
  Dump d(out / "activations.bin");
  const std::pair<const char*, nn::Act> acts[3] = {
      {"relu", nn::Act::kRelu}, {"tanh", nn::Act::kTanh}, {"sigmoid", nn::Act::kSigmoid}};
  {
    DataFixture fx(tmp / "act_tiny", tiny_dims(), 600, 100, 3, 17);
    d.put("tiny_data", std::vector<std::uint64_t>{600, 100, 3, 17});
    for (const auto& [name, act] : acts) {
      auto arch = tiny_arch();
      arch.hidden_act = nn::Activation{act, 0.0};
      trainer_case(d, std::string("tiny_") + name + "_", fx, tiny_dims(), arch, 3, 1, 64, 7, 30, 20);
    }
  }
  {
    surrogate::ModalityDims dims;  // desk 16x16
    DataFixture fx(tmp / "act_desk", dims, 400, 100, 1, 1);
    d.put("desk_data", std::vector<std::uint64_t>{400, 100, 1, 1});
    for (const auto& [name, act] : acts) {
      surrogate::SurrogateArch arch;
      arch.hidden_act = nn::Activation{act, 0.0};
      trainer_case(d, std::string("desk_") + name + "_", fx, dims, arch, 3, 1, 32, 7, 30, 14);
    }
  }
}

// horizon: the trainer cases of scenario_trainer over 50 steps (SURVEY §7:
// 1e-4 relative over 50 steps, tests/acceptance_test.cpp:210-244), at desk
// and paper dims, several epochs each (the per-epoch reshuffle included).
static void scenario_horizon(const fs::path& out, const fs::path& tmp) {
  Dump d(out / "horizon.bin");
  {
    surrogate::ModalityDims dims;  // desk 16x16
    DataFixture fx(tmp / "hz_desk", dims, 400, 100, 1, 1);
    d.put("desk_data", std::vector<std::uint64_t>{400, 100, 1, 1});
    put_dims(d, "desk_", dims);
    // partition 370, B = 32 -> 12 steps/epoch: 50 steps = 4 epochs + 2
    trainer_case(d, "desk_s50_", fx, dims, surrogate::SurrogateArch{}, 3, 1, 32, 7, 30, 50);
  }
  {
    const auto dims = surrogate::ModalityDims::paper_scale();
    DataFixture fx(tmp / "hz_paper", dims, 1000, 100, 1, 1);
    d.put("paper_data", std::vector<std::uint64_t>{1000, 100, 1, 1});
    put_dims(d, "paper_", dims);
    // partition 970, B = 128 -> 8 steps/epoch (7 x 128 + 74): 50 steps = 6 epochs + 2
    trainer_case(d, "paper_s50_", fx, dims, surrogate::SurrogateArch{}, 3, 1, 128, 7, 30, 50);
  }
}

// ---------------------------------------------------------------------------
// tournament: runner.hpp:232-437 re-driven step by step so pre-round model
// state can be captured for state-injection decision tests. The loop mirrors
// run_experiment; a self-check compares its history against run_experiment.
// ---------------------------------------------------------------------------
static void tournament_case(Dump& d, const std::string& pfx,
                            const tournament::RunConfig& cfg) {
  const auto index = tournament::ensure_dataset(cfg);
  const auto ref = tournament::run_experiment(cfg, index);

  d.put(pfx + "cfg", std::vector<std::uint64_t>{
                         cfg.gen_n, cfg.samples_per_file, cfg.spec_seed,
                         cfg.sampling_seed, static_cast<std::uint64_t>(cfg.trainers),
                         cfg.batch_size, cfg.interval, cfg.step_budget,
                         cfg.ae_steps, cfg.seed,
                         static_cast<std::uint64_t>(cfg.shards)});
  put_dims(d, pfx, cfg.dims);
  std::vector<double> pre;
  for (const auto& p : ref.history.pretrain) pre.push_back(p.loss);
  d.put(pfx + "pretrain_loss", pre);
  put_steps(d, pfx + "steps_", ref.history.steps);
  {
    std::vector<std::int32_t> tr;
    std::vector<std::uint64_t> st;
    std::vector<double> f, i, c;
    for (const auto& e : ref.history.evals) {
      tr.push_back(e.trainer);
      st.push_back(e.step);
      f.push_back(e.forward_mae);
      i.push_back(e.inverse_mae);
      c.push_back(e.combined);
    }
    d.put(pfx + "evals_trainer", tr);
    d.put(pfx + "evals_step", st);
    d.put(pfx + "evals_fwd", f);
    d.put(pfx + "evals_inv", i);
    d.put(pfx + "evals_combined", c);
  }
  {
    std::vector<std::int32_t> rr, pa, pb, bye;
    std::vector<std::uint64_t> rs;
    for (const auto& r : ref.history.rounds) {
      bye.push_back(r.bye);
      rs.push_back(r.step);
      for (const auto& p : r.pairs) {
        rr.push_back(r.round);
        pa.push_back(p[0]);
        pb.push_back(p[1]);
      }
    }
    d.put(pfx + "round_bye", bye);
    d.put(pfx + "round_step", rs);
    d.put(pfx + "round_pair_round", rr);
    d.put(pfx + "round_pair_a", pa);
    d.put(pfx + "round_pair_b", pb);
  }
  {
    std::vector<std::int32_t> rr, tr, peer;
    std::vector<double> lm, im;
    std::vector<std::uint8_t> kept;
    for (const auto& r : ref.history.trainer_rounds) {
      rr.push_back(r.round);
      tr.push_back(r.trainer);
      peer.push_back(r.peer);
      lm.push_back(r.local_metric);
      im.push_back(r.incoming_metric);
      kept.push_back(r.kept_incoming ? 1 : 0);
    }
    d.put(pfx + "tr_round", rr);
    d.put(pfx + "tr_trainer", tr);
    d.put(pfx + "tr_peer", peer);
    d.put(pfx + "tr_local", lm);
    d.put(pfx + "tr_incoming", im);
    d.put(pfx + "tr_kept", kept);
  }
  {
    std::vector<std::int32_t> rr, from, to;
    std::vector<std::uint64_t> bytes;
    std::vector<std::uint8_t> is_fwd;
    for (const auto& t : ref.history.transfers) {
      rr.push_back(t.round);
      from.push_back(t.from_trainer);
      to.push_back(t.to_trainer);
      bytes.push_back(t.bytes);
      is_fwd.push_back(t.payload == "fwd" ? 1 : 0);
    }
    d.put(pfx + "xf_round", rr);
    d.put(pfx + "xf_from", from);
    d.put(pfx + "xf_to", to);
    d.put(pfx + "xf_bytes", bytes);
    d.put(pfx + "xf_is_fwd", is_fwd);
  }
  put_epochs(d, pfx + "epochs_", ref.history.epochs);
  d.scalar(pfx + "best_trainer", static_cast<std::int32_t>(ref.best_trainer));
  d.put(pfx + "best_metric", std::vector<double>{ref.best_metric.forward_mae,
                                                 ref.best_metric.inverse_mae,
                                                 ref.best_metric.combined});
  put_model(d, pfx + "best_model_", ref.best_model, false);
  put_strided(d, pfx + "best_model_enc_strided", flat(ref.best_model.enc));
  put_strided(d, pfx + "best_model_dec_strided", flat(ref.best_model.dec));
  // split ids (so consumers can rebuild tournament slices)
  const int k = cfg.trainers;
  const auto split = tournament::detail::split_dataset(
      index, k, cfg.validation_fraction, cfg.tournament_fraction, cfg.seed, k >= 2);
  d.put(pfx + "split_validation", split.validation);
  put_parts(d, pfx + "split_train_", split.train);
  put_parts(d, pfx + "split_tour_", split.tournament);

  // ---- re-driven loop for pre-round state capture -----------------------
  auto base = surrogate::make_cyclegan<float>(cfg.dims, cfg.arch,
                                              mix_seed({cfg.seed, 0xae0ULL}));
  {
    std::vector<data::SampleId> union_ids;
    for (const auto& part : split.train)
      union_ids.insert(union_ids.end(), part.begin(), part.end());
    std::sort(union_ids.begin(), union_ids.end());
    auto [ax, ay] = data::assemble_tensors(index, union_ids);
    Rng batch_rng(mix_seed({cfg.seed, 0xae1ULL}));
    const std::size_t rows = ay.rows();
    nn::Tensor<float> batch({std::min(cfg.batch_size, rows), cfg.dims.output_dim()});
    std::vector<std::uint32_t> ae_rows;
    for (std::uint64_t s = 0; s < cfg.ae_steps; ++s) {
      for (std::size_t r = 0; r < batch.rows(); ++r) {
        const std::size_t src = static_cast<std::size_t>(batch_rng.below(rows));
        if (s < 2) ae_rows.push_back(static_cast<std::uint32_t>(src));
        std::copy_n(ay.data.begin() + static_cast<std::ptrdiff_t>(src * ay.cols()),
                    ay.cols(),
                    batch.data.begin() + static_cast<std::ptrdiff_t>(r * batch.cols()));
      }
      surrogate::autoencoder_step(base, batch);
    }
    d.put(pfx + "ae_rows_first2", ae_rows);
  }
  base.autoencoder_frozen = true;
  put_strided(d, pfx + "ae_enc_strided", flat(base.enc));
  put_strided(d, pfx + "ae_dec_strided", flat(base.dec));
  d.put(pfx + "ae_hashes", std::vector<std::uint64_t>{base.enc_hash(), base.dec_hash()});
  if (cfg.dims.output_dim() < 10000) {  // tiny and desk: the full frozen AE (state injection)
    d.put(pfx + "ae_enc", flat(base.enc));
    d.put(pfx + "ae_dec", flat(base.dec));
  }
  std::vector<std::unique_ptr<train::Trainer>> trainers;
  for (int t = 0; t < k; ++t) {
    auto model = base;
    surrogate::reinit_gan_nets(model, mix_seed({cfg.seed, 0x1417ULL, static_cast<std::uint64_t>(t)}));
    train::TrainerConfig tc;
    tc.trainer_id = t;
    tc.n_shards = cfg.shards;
    tc.batch_size = cfg.batch_size;
    tc.store_mode = cfg.store_mode;
    tc.seed = mix_seed({cfg.seed, 0x57a7e1ULL, static_cast<std::uint64_t>(t)});
    tc.numeric_abort_threshold = cfg.numeric_abort_threshold;
    tc.prefetch_depth = 0;
    tc.train_ids = split.train[static_cast<std::size_t>(t)];
    tc.tournament_ids = split.tournament[static_cast<std::size_t>(t)];
    trainers.push_back(std::make_unique<train::Trainer>(tc, index, std::move(model)));
  }
  std::uint64_t done = 0;
  int round_index = 0;
  std::vector<float> pre_fwd, pre_inv;
  std::vector<std::uint32_t> pre_fwd_len, pre_inv_len;
  std::vector<std::int32_t> my_kept;
  while (done < cfg.step_budget) {
    const std::uint64_t chunk = std::min<std::uint64_t>(cfg.interval, cfg.step_budget - done);
    for (auto& t : trainers) t->train_steps(chunk);
    done += chunk;
    if (cfg.mode == tournament::RunMode::kLtfb && k >= 2 && chunk == cfg.interval) {
      ++round_index;
      for (auto& t : trainers) {
        const auto f = flat(t->model().fwd);
        const auto iv = flat(t->model().inv);
        pre_fwd.insert(pre_fwd.end(), f.begin(), f.end());
        pre_inv.insert(pre_inv.end(), iv.begin(), iv.end());
        pre_fwd_len.push_back(static_cast<std::uint32_t>(f.size()));
        pre_inv_len.push_back(static_cast<std::uint32_t>(iv.size()));
      }
      const auto matching = tournament::pair_trainers(k, round_index, mix_seed({cfg.seed, 0x9a18ULL}));
      const auto round = tournament::tournament_round(trainers, matching, round_index);
      for (const auto& r : round.trainer_records) my_kept.push_back(r.kept_incoming ? 1 : 0);
    }
  }
  d.put(pfx + "pre_round_fwd", pre_fwd);
  d.put(pfx + "pre_round_inv", pre_inv);
  d.put(pfx + "pre_round_fwd_len", pre_fwd_len);
  d.put(pfx + "pre_round_inv_len", pre_inv_len);
  // self-check: the re-driven loop matches run_experiment's decisions
  std::vector<std::int32_t> ref_kept;
  for (const auto& r : ref.history.trainer_rounds) ref_kept.push_back(r.kept_incoming ? 1 : 0);
  if (ref_kept != my_kept) throw std::runtime_error("re-driven loop diverged from run_experiment");
}

static void scenario_tournament(const fs::path& out, const fs::path& tmp) {
  Dump d(out / "tournament.bin");
  {
    // tests/test_tournament.cpp:38-53 tiny_run_config
    tournament::RunConfig cfg;
    cfg.data_dir = (tmp / "tour_tiny").string();
    cfg.gen_n = 800;
    cfg.samples_per_file = 100;
    cfg.dims = tiny_dims();
    cfg.arch = tiny_arch();
    cfg.batch_size = 32;
    cfg.ae_steps = 15;
    cfg.seed = 42;
    cfg.mode = tournament::RunMode::kLtfb;
    cfg.trainers = 2;
    cfg.interval = 10;
    cfg.step_budget = 30;
    tournament_case(d, "tiny_k2_", cfg);
    cfg.trainers = 4;
    cfg.step_budget = 40;
    tournament_case(d, "tiny_k4_", cfg);
    cfg.trainers = 3;  // odd k: a bye every round
    cfg.step_budget = 30;
    tournament_case(d, "tiny_k3_", cfg);
  }
  {
    tournament::RunConfig cfg;
    cfg.data_dir = (tmp / "tour_desk").string();
    cfg.gen_n = 2000;
    cfg.samples_per_file = 250;
    cfg.batch_size = 32;
    cfg.ae_steps = 20;
    cfg.seed = 7;
    cfg.mode = tournament::RunMode::kLtfb;
    cfg.trainers = 2;
    cfg.interval = 10;
    cfg.step_budget = 30;
    tournament_case(d, "desk_k2_", cfg);
  }
}

// tournament_paper: BASELINE config C2 -- LTFB with 2 trainers at paper dims,
// B = 128, 16,000 samples (runner.hpp:49-66 defaults) so each trainer's
// tournament slice is floor(0.05 * 7600) = 380 rows (runner.hpp:160-165),
// three rounds. ae_steps = 0: the frozen enc / dec are make_cyclegan's
// init (seed mix_seed({seed, 0xae0})), which a consumer rebuilds bit-exactly
// on the host instead of carrying 25 MB of pre-trained weights.
static void scenario_tournament_paper(const fs::path& out, const fs::path& tmp) {
  Dump d(out / "tournament_paper.bin");
  tournament::RunConfig cfg;
  cfg.data_dir = (tmp / "tour_paper").string();
  cfg.gen_n = 16000;
  cfg.samples_per_file = 500;
  cfg.dims = surrogate::ModalityDims::paper_scale();
  cfg.batch_size = 128;
  cfg.ae_steps = 0;
  cfg.seed = 11;
  cfg.mode = tournament::RunMode::kLtfb;
  cfg.trainers = 2;
  cfg.interval = 20;
  cfg.step_budget = 60;
  tournament_case(d, "paper_k2_", cfg);
}

// ---------------------------------------------------------------------------
// run outputs: bench/output.hpp + bench/config.hpp (the run directory the
// reference CLI writes, ltfb_cli.cpp:126-138) for two tiny runs, copied
// verbatim into tests/golden/run_<name>/ by make_golden.py. data_dir is
// relative (golden_dump runs from TMP_DIR) so config.json / config_hash are
// machine-independent.
// ---------------------------------------------------------------------------
static void outputs_case(const fs::path& out, const std::string& name, tournament::RunConfig cfg) {
  cfg.data_dir = "data_" + name;
  const auto index = tournament::ensure_dataset(cfg);
  auto res = tournament::run_experiment(cfg, index);
  res.history.config_hash = bench::config_hash(cfg);
  bench::write_run_outputs(out / ("run_" + name), cfg, res.history, &res.best_model);
}

static void scenario_outputs(const fs::path& out, const fs::path& tmp) {
  const fs::path abs_out = fs::absolute(out);
  const fs::path cwd = fs::current_path();
  fs::current_path(tmp);
  {
    tournament::RunConfig cfg;  // tiny_k2 of scenario_tournament
    cfg.gen_n = 800;
    cfg.samples_per_file = 100;
    cfg.dims = tiny_dims();
    cfg.arch = tiny_arch();
    cfg.batch_size = 32;
    cfg.ae_steps = 15;
    cfg.seed = 42;
    cfg.mode = tournament::RunMode::kLtfb;
    cfg.trainers = 2;
    cfg.interval = 10;
    cfg.step_budget = 30;
    outputs_case(abs_out, "tiny_k2", cfg);
    cfg.mode = tournament::RunMode::kSingle;  // one trainer, no rounds, 2 epochs + a partial
    cfg.trainers = 1;
    cfg.step_budget = 50;
    cfg.interval = 20;
    cfg.seed = 5;
    outputs_case(abs_out, "tiny_single", cfg);
  }
  fs::current_path(cwd);
  // golden_dump's tagged-file convention: one (empty) marker per scenario
  Dump d(out / "outputs.bin");
  d.put("outputs_runs", std::vector<std::uint32_t>{2});
}

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s OUT_DIR TMP_DIR [scenario...]\n", argv[0]);
    return 2;
  }
  const fs::path out = argv[1], tmp = argv[2];
  fs::create_directories(out);
  fs::create_directories(tmp);
  std::vector<std::string> want(argv + 3, argv + argc);
  auto on = [&](const char* s) {
    return want.empty() || std::find(want.begin(), want.end(), s) != want.end();
  };
  try {
    if (on("rng")) scenario_rng(out);
    if (on("plan")) scenario_plan(out, tmp);
    if (on("synth")) scenario_synth(out);
    if (on("nn")) scenario_nn(out);
    if (on("surrogate")) scenario_surrogate(out);
    if (on("trainer")) scenario_trainer(out, tmp);
    if (on("tournament")) scenario_tournament(out, tmp);
    if (on("horizon")) scenario_horizon(out, tmp);
    if (on("activations")) scenario_activations(out, tmp);
    if (on("tournament_paper")) scenario_tournament_paper(out, tmp);
    if (on("outputs")) scenario_outputs(out, tmp);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "golden_dump failed: %s\n", e.what());
    return 1;
  }
  return 0;
}
