// ltfb_b200 — host-side value types of the drop-in API.
//
// These are the types the reference's trainer/model/tournament API passes
// around (errors, seeds, shapes, parameter blobs, the CycleGan value type and
// the history records). They keep the reference's names and meaning so code
// written against /root/reference/proj/include/ltfb compiles against this
// header set; the arithmetic they feed runs on the GPU (libltfb_gpu.so).
//
// Reference correspondence (file:line under /root/reference/proj/include/ltfb):
//   errors            core/error.hpp:11-58
//   Rng / mix_seed    core/rng.hpp:13-97
//   fnv1a64 / hex64   core/hash.hpp:15-40
//   Tensor            nn/tensor.hpp:20-84        (host container only)
//   Activation        nn/activation.hpp:12-20
//   MlpSpec/params    nn/mlp.hpp:23-165
//   AdamHyper/State   nn/adam.hpp:15-47
//   ModalityDims      surrogate/dims.hpp:15-53
//   SurrogateArch,
//   CycleGan, make_cyclegan, reinit_gan_nets   surrogate/model.hpp:18-148
//   EvalMetric/GenLosses  surrogate/train_ops.hpp:20-31
//   history records   train/history.hpp:20-129
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <initializer_list>
#include <numeric>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace ltfb {

// ---------------------------------------------------------------- errors --
// One class per failure kind; the C ABI maps each to a status code
// (include/ltfb_gpu.h, LTFB_E*) and the façade rethrows the same type.
struct Error : std::runtime_error {
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
#define LTFB_B200_ERROR(Name)                                   \
  struct Name : Error {                                         \
    explicit Name(const std::string& m) : Error(m) {}           \
  }
LTFB_B200_ERROR(DimensionError);
LTFB_B200_ERROR(ContractError);
LTFB_B200_ERROR(NumericError);
LTFB_B200_ERROR(IoError);
LTFB_B200_ERROR(CapacityError);
LTFB_B200_ERROR(StoreCorruptError);
LTFB_B200_ERROR(ConfigError);
#undef LTFB_B200_ERROR

// ------------------------------------------------------------------ seeds --
namespace seedmix {
inline constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
inline std::uint64_t step(std::uint64_t& s) {
  s += kGolden;
  std::uint64_t v = s;
  v = (v ^ (v >> 30)) * 0xbf58476d1ce4e5b9ULL;
  v = (v ^ (v >> 27)) * 0x94d049bb133111ebULL;
  return v ^ (v >> 31);
}
}  // namespace seedmix

inline std::uint64_t splitmix64(std::uint64_t& state) { return seedmix::step(state); }

/// Derives a stream seed from a list of words (core/rng.hpp:23-30).
inline std::uint64_t mix_seed(std::initializer_list<std::uint64_t> words) {
  std::uint64_t acc = 0x243f6a8885a308d3ULL;
  for (const std::uint64_t w : words) {
    acc ^= w + seedmix::kGolden + (acc << 6) + (acc >> 2);
    seedmix::step(acc);
  }
  return seedmix::step(acc);
}

/// xoshiro256** with the reference's uniform/below/normal/shuffle mappings
/// (core/rng.hpp:35-97). Host only: every seeded integer decision (pairings,
/// partitions, epoch permutations, init) is made here, bit-exact.
class Rng {
 public:
  using result_type = std::uint64_t;
  explicit Rng(std::uint64_t seed) {
    for (int i = 0; i < 4; ++i) w_[i] = seedmix::step(seed);
  }
  static constexpr result_type min() { return 0; }
  static constexpr result_type max() { return ~result_type{0}; }
  result_type operator()() { return next(); }

  std::uint64_t next() {
    const std::uint64_t out = rol(w_[1] * 5, 7) * 9;
    const std::uint64_t shifted = w_[1] << 17;
    w_[2] ^= w_[0];
    w_[3] ^= w_[1];
    w_[1] ^= w_[2];
    w_[0] ^= w_[3];
    w_[2] ^= shifted;
    w_[3] = rol(w_[3], 45);
    return out;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  std::uint64_t below(std::uint64_t n) {
    const std::uint64_t reject_under = (0 - n) % n;  // 2^64 mod n
    for (;;) {
      const std::uint64_t v = next();
      if (v >= reject_under) return v % n;
    }
  }
  double normal() {
    double u1;
    do u1 = uniform(); while (u1 <= 0.0);
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) *
           std::cos(6.283185307179586476925286766559 * u2);
  }
  template <typename T>
  void shuffle(std::vector<T>& v) {
    for (std::size_t top = v.size(); top > 1; --top)
      std::swap(v[top - 1], v[static_cast<std::size_t>(below(top))]);
  }

 private:
  static std::uint64_t rol(std::uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
  std::uint64_t w_[4];
};

// ------------------------------------------------------------------- hash --
inline constexpr std::uint64_t kFnvBasis = 0xcbf29ce484222325ULL;
inline std::uint64_t fnv1a64(const void* bytes, std::size_t n,
                             std::uint64_t h = kFnvBasis) {
  const auto* p = static_cast<const unsigned char*>(bytes);
  for (const unsigned char* e = p + n; p != e; ++p) h = (h ^ *p) * 0x100000001b3ULL;
  return h;
}
template <typename T>
std::uint64_t hash_span(std::span<const T> v, std::uint64_t h = kFnvBasis) {
  return fnv1a64(v.data(), v.size_bytes(), h);
}
inline std::string hex64(std::uint64_t v) {
  char buf[17];
  for (int i = 15; i >= 0; --i, v >>= 4) buf[i] = "0123456789abcdef"[v & 0xf];
  buf[16] = 0;
  return buf;
}

namespace nn {

// ----------------------------------------------------------------- tensor --
/// Row-major host container (the reference's nn::Tensor minus the math,
/// which runs on the device).
template <typename T>
struct Tensor {
  std::vector<std::size_t> shape;
  std::vector<T> data;
  Tensor() = default;
  explicit Tensor(std::vector<std::size_t> s)
      : shape(std::move(s)), data(count(shape), T{0}) {}
  Tensor(std::initializer_list<std::size_t> s) : Tensor(std::vector<std::size_t>(s)) {}
  static std::size_t count(const std::vector<std::size_t>& s) {
    std::size_t n = 1;
    for (auto d : s) n *= d;
    return n;
  }
  static Tensor from_data(std::vector<std::size_t> s, std::vector<T> d) {
    if (count(s) != d.size()) throw DimensionError("tensor data length does not match shape");
    Tensor t;
    t.shape = std::move(s);
    t.data = std::move(d);
    return t;
  }
  std::size_t size() const { return data.size(); }
  bool empty() const { return data.empty(); }
  std::size_t rows() const { rank2(); return shape[0]; }
  std::size_t cols() const { rank2(); return shape[1]; }
  T& operator()(std::size_t r, std::size_t c) { return data[r * shape[1] + c]; }
  T operator()(std::size_t r, std::size_t c) const { return data[r * shape[1] + c]; }
  T& operator[](std::size_t i) { return data[i]; }
  T operator[](std::size_t i) const { return data[i]; }
  bool all_finite() const {
    return std::all_of(data.begin(), data.end(),
                       [](T v) { return std::isfinite(static_cast<double>(v)); });
  }
  void fill(T v) { std::fill(data.begin(), data.end(), v); }

 private:
  void rank2() const {
    if (shape.size() != 2)
      throw DimensionError("expected a rank-2 tensor, got rank " + std::to_string(shape.size()));
  }
};

// ------------------------------------------------------------ activations --
enum class Act { kIdentity, kRelu, kLeakyRelu, kTanh, kSigmoid };
struct Activation {
  Act kind = Act::kIdentity;
  double slope = 0.01;
  bool operator==(const Activation&) const = default;
};

// ----------------------------------------------------------------- MLPs --
struct MlpSpec {
  std::vector<std::size_t> layer_widths;
  std::vector<Activation> activations;
  std::uint64_t init_seed = 0;
  std::size_t n_layers() const { return layer_widths.empty() ? 0 : layer_widths.size() - 1; }
  std::size_t in_dim() const { return layer_widths.front(); }
  std::size_t out_dim() const { return layer_widths.back(); }
  void validate() const {
    std::string why;
    if (layer_widths.size() < 2) why += "need at least two layer widths; ";
    if (std::any_of(layer_widths.begin(), layer_widths.end(), [](std::size_t w) { return w < 1; }))
      why += "layer widths must be >= 1; ";
    if (!layer_widths.empty() && activations.size() != layer_widths.size() - 1)
      why += "need exactly one activation per layer (" + std::to_string(layer_widths.size() - 1) +
             " expected, " + std::to_string(activations.size()) + " given); ";
    if (!why.empty()) throw ContractError("invalid MlpSpec: " + why);
  }
  bool operator==(const MlpSpec&) const = default;
};

/// Blob manifest: W0, b0, W1, b1, ... with row-major [in x out] weights
/// (nn/mlp.hpp:63-84). The device keeps every network in exactly this
/// layout, so a blob crosses the ABI (and NCCL) as one contiguous copy.
struct BlobManifest {
  struct Entry {
    std::string name;
    std::size_t offset, rows, cols;
    std::size_t count() const { return rows * cols; }
  };
  std::vector<Entry> entries;
  std::size_t total = 0;
  bool operator==(const BlobManifest&) const = default;
};

inline BlobManifest manifest_for(const MlpSpec& spec) {
  spec.validate();
  BlobManifest m;
  for (std::size_t l = 0; l < spec.n_layers(); ++l) {
    const std::size_t in = spec.layer_widths[l], out = spec.layer_widths[l + 1];
    m.entries.push_back({"w" + std::to_string(l), m.total, in, out});
    m.total += in * out;
    m.entries.push_back({"b" + std::to_string(l), m.total, 1, out});
    m.total += out;
  }
  return m;
}

template <typename T>
struct MlpParams {
  std::vector<Tensor<T>> weights;
  std::vector<Tensor<T>> biases;
  std::size_t param_count() const {
    std::size_t n = 0;
    for (std::size_t l = 0; l < weights.size(); ++l) n += weights[l].size() + biases[l].size();
    return n;
  }
  bool same_shape(const MlpParams& o) const {
    if (weights.size() != o.weights.size()) return false;
    for (std::size_t l = 0; l < weights.size(); ++l)
      if (weights[l].shape != o.weights[l].shape || biases[l].shape != o.biases[l].shape) return false;
    return true;
  }
  std::vector<T> flatten() const {
    std::vector<T> blob;
    blob.reserve(param_count());
    for (std::size_t l = 0; l < weights.size(); ++l) {
      blob.insert(blob.end(), weights[l].data.begin(), weights[l].data.end());
      blob.insert(blob.end(), biases[l].data.begin(), biases[l].data.end());
    }
    return blob;
  }
  /// Writes the blob into `dst` (param_count() elements).
  void flatten_into(T* dst) const {
    for (std::size_t l = 0; l < weights.size(); ++l) {
      dst = std::copy(weights[l].data.begin(), weights[l].data.end(), dst);
      dst = std::copy(biases[l].data.begin(), biases[l].data.end(), dst);
    }
  }
  static MlpParams zeros_like(const MlpSpec& spec) {
    MlpParams p;
    for (std::size_t l = 0; l < spec.n_layers(); ++l) {
      p.weights.emplace_back(Tensor<T>({spec.layer_widths[l], spec.layer_widths[l + 1]}));
      p.biases.emplace_back(Tensor<T>({spec.layer_widths[l + 1]}));
    }
    return p;
  }
  static MlpParams unflatten(const MlpSpec& spec, std::span<const T> blob) {
    const BlobManifest man = manifest_for(spec);
    if (blob.size() != man.total)
      throw ContractError("blob length " + std::to_string(blob.size()) +
                          " does not match manifest total " + std::to_string(man.total));
    MlpParams p = zeros_like(spec);
    const T* src = blob.data();
    for (std::size_t l = 0; l < spec.n_layers(); ++l) {
      std::copy_n(src, p.weights[l].size(), p.weights[l].data.begin());
      src += p.weights[l].size();
      std::copy_n(src, p.biases[l].size(), p.biases[l].data.begin());
      src += p.biases[l].size();
    }
    return p;
  }
};

/// U(-sqrt(1/fan_in), +sqrt(1/fan_in)) weights, zero biases, one Rng stream
/// per network (nn/mlp.hpp:235-244). Runs on the host: the init is an
/// integer/double sequence that must be bit-identical to the reference.
template <typename T>
MlpParams<T> init_params(const MlpSpec& spec) {
  spec.validate();
  Rng rng(spec.init_seed);
  MlpParams<T> p = MlpParams<T>::zeros_like(spec);
  for (std::size_t l = 0; l < spec.n_layers(); ++l) {
    const double bound = std::sqrt(1.0 / static_cast<double>(spec.layer_widths[l]));
    for (T& w : p.weights[l].data) w = static_cast<T>(rng.uniform(-bound, bound));
  }
  return p;
}

struct AdamHyper {
  double lr = 0.001, beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
  bool operator==(const AdamHyper&) const = default;
};

template <typename T>
struct AdamState {
  std::vector<T> m, v;
  std::uint64_t t = 0;
  AdamHyper hyper;
  static AdamState for_params(const MlpParams<T>& p, AdamHyper h) {
    AdamState s;
    s.m.assign(p.param_count(), T{0});
    s.v.assign(p.param_count(), T{0});
    s.hyper = h;
    return s;
  }
  void reset_moments() {
    std::fill(m.begin(), m.end(), T{0});
    std::fill(v.begin(), v.end(), T{0});
  }
};

}  // namespace nn

namespace surrogate {

struct ModalityDims {
  std::uint32_t input_dim = 5, latent_dim = 20, scalar_dim = 15;
  std::uint32_t image_views = 3, image_channels = 4, image_h = 16, image_w = 16;
  std::uint32_t image_elems() const { return image_views * image_channels * image_h * image_w; }
  std::uint32_t output_dim() const { return scalar_dim + image_elems(); }
  std::uint32_t record_floats() const { return input_dim + output_dim(); }
  void validate() const {
    const std::pair<std::uint32_t, const char*> fields[] = {
        {input_dim, "input_dim"},     {latent_dim, "latent_dim"},
        {scalar_dim, "scalar_dim"},   {image_views, "image_views"},
        {image_channels, "image_channels"}, {image_h, "image_h"}, {image_w, "image_w"}};
    for (const auto& [v, name] : fields)
      if (v < 1) throw ContractError(std::string("ModalityDims: ") + name + " must be >= 1");
  }
  static ModalityDims paper_scale() {
    ModalityDims d;
    d.image_h = d.image_w = 64;
    return d;
  }
  bool operator==(const ModalityDims&) const = default;
};

struct SurrogateArch {
  std::vector<std::size_t> enc_hidden{64}, dec_hidden{64};
  std::vector<std::size_t> fwd_hidden{32, 32}, inv_hidden{32, 32}, disc_hidden{32, 32};
  nn::Activation hidden_act{nn::Act::kLeakyRelu, 0.2};
  double lambda_adv = 0.01, lambda_cyc = 1.0;
  nn::AdamHyper adam;
  bool operator==(const SurrogateArch&) const = default;
};

/// Host value type of the surrogate (surrogate/model.hpp:36-73). On the
/// drop-in path the authoritative copy lives in HBM; Trainer::model()
/// returns a host mirror refreshed from the device on demand.
template <typename T>
struct CycleGan {
  ModalityDims dims;
  nn::MlpSpec enc_spec, dec_spec, fwd_spec, inv_spec, disc_spec;
  nn::MlpParams<T> enc, dec, fwd, inv, disc;
  nn::AdamState<T> enc_opt, dec_opt, fwd_opt, inv_opt, disc_opt;
  T lambda_adv{}, lambda_cyc{};
  bool autoencoder_frozen = false;

  static std::uint64_t hash_blob(const nn::MlpParams<T>& p) {
    std::uint64_t h = kFnvBasis;
    for (std::size_t l = 0; l < p.weights.size(); ++l) {
      h = hash_span(std::span<const T>(p.weights[l].data), h);
      h = hash_span(std::span<const T>(p.biases[l].data), h);
    }
    return h;
  }
  std::uint64_t enc_hash() const { return hash_blob(enc); }
  std::uint64_t dec_hash() const { return hash_blob(dec); }
  std::uint64_t fwd_hash() const { return hash_blob(fwd); }
  std::uint64_t inv_hash() const { return hash_blob(inv); }
  std::uint64_t disc_hash() const { return hash_blob(disc); }
  std::uint64_t model_hash() const {
    std::uint64_t h = kFnvBasis;
    for (const auto* p : {&enc, &dec, &fwd, &inv, &disc})
      for (std::size_t l = 0; l < p->weights.size(); ++l) {
        h = hash_span(std::span<const T>(p->weights[l].data), h);
        h = hash_span(std::span<const T>(p->biases[l].data), h);
      }
    return h;
  }
};

namespace detail {
inline nn::MlpSpec spec_of(std::size_t in, std::size_t out, const std::vector<std::size_t>& hidden,
                           nn::Activation act, std::uint64_t seed) {
  nn::MlpSpec s;
  s.layer_widths.push_back(in);
  s.layer_widths.insert(s.layer_widths.end(), hidden.begin(), hidden.end());
  s.layer_widths.push_back(out);
  const std::size_t L = s.layer_widths.size() - 1;
  for (std::size_t l = 0; l < L; ++l)
    s.activations.push_back(l + 1 < L ? act : nn::Activation{nn::Act::kIdentity});
  s.init_seed = seed;
  s.validate();
  return s;
}
}  // namespace detail

/// surrogate/model.hpp:96-132. Per-network streams mix_seed({seed, 1..5}).
template <typename T>
CycleGan<T> make_cyclegan(const ModalityDims& dims, const SurrogateArch& arch, std::uint64_t seed) {
  dims.validate();
  CycleGan<T> m;
  m.dims = dims;
  m.lambda_adv = static_cast<T>(arch.lambda_adv);
  m.lambda_cyc = static_cast<T>(arch.lambda_cyc);
  const std::size_t in = dims.input_dim, lat = dims.latent_dim, out = dims.output_dim();
  m.enc_spec = detail::spec_of(out, lat, arch.enc_hidden, arch.hidden_act, mix_seed({seed, 1}));
  m.dec_spec = detail::spec_of(lat, out, arch.dec_hidden, arch.hidden_act, mix_seed({seed, 2}));
  m.fwd_spec = detail::spec_of(in, lat, arch.fwd_hidden, arch.hidden_act, mix_seed({seed, 3}));
  m.inv_spec = detail::spec_of(lat, in, arch.inv_hidden, arch.hidden_act, mix_seed({seed, 4}));
  m.disc_spec = detail::spec_of(lat, 1, arch.disc_hidden, arch.hidden_act, mix_seed({seed, 5}));
  m.enc = nn::init_params<T>(m.enc_spec);
  m.dec = nn::init_params<T>(m.dec_spec);
  m.fwd = nn::init_params<T>(m.fwd_spec);
  m.inv = nn::init_params<T>(m.inv_spec);
  m.disc = nn::init_params<T>(m.disc_spec);
  m.enc_opt = nn::AdamState<T>::for_params(m.enc, arch.adam);
  m.dec_opt = nn::AdamState<T>::for_params(m.dec, arch.adam);
  m.fwd_opt = nn::AdamState<T>::for_params(m.fwd, arch.adam);
  m.inv_opt = nn::AdamState<T>::for_params(m.inv, arch.adam);
  m.disc_opt = nn::AdamState<T>::for_params(m.disc, arch.adam);
  return m;
}

/// surrogate/model.hpp:137-147.
template <typename T>
void reinit_gan_nets(CycleGan<T>& m, std::uint64_t seed) {
  m.fwd_spec.init_seed = mix_seed({seed, 3});
  m.inv_spec.init_seed = mix_seed({seed, 4});
  m.disc_spec.init_seed = mix_seed({seed, 5});
  m.fwd = nn::init_params<T>(m.fwd_spec);
  m.inv = nn::init_params<T>(m.inv_spec);
  m.disc = nn::init_params<T>(m.disc_spec);
  m.fwd_opt = nn::AdamState<T>::for_params(m.fwd, m.fwd_opt.hyper);
  m.inv_opt = nn::AdamState<T>::for_params(m.inv, m.inv_opt.hyper);
  m.disc_opt = nn::AdamState<T>::for_params(m.disc, m.disc_opt.hyper);
}

struct EvalMetric {
  double forward_mae = 0, inverse_mae = 0, combined = 0;
};
struct GenLosses {
  double total = 0, fwd = 0, adv = 0, cyc = 0;
};

}  // namespace surrogate

namespace train {

struct StepRecord {
  int trainer = 0;
  std::uint64_t step = 0;
  std::uint32_t epoch = 0;
  double d_loss = 0, g_total = 0, g_fwd = 0, g_adv = 0, g_cyc = 0;
  bool skipped = false;
};
struct EvalRecord {
  int trainer = 0;
  std::uint64_t step = 0;
  std::string slice;
  double forward_mae = 0, inverse_mae = 0, combined = 0;
};
struct EpochRecord {
  int trainer = 0;
  std::uint32_t epoch = 0;
  std::uint64_t steps = 0, files_opened = 0, bytes_read = 0, samples_shuffled = 0;
  double seconds = 0;
  bool partial = false;
};
struct PretrainRecord {
  std::uint64_t step = 0;
  double loss = 0;
};
struct RoundRecord {
  int round = 0;
  std::uint64_t step = 0;
  std::vector<std::array<int, 2>> pairs;
  int bye = -1;
};
struct TrainerRoundRecord {
  int round = 0;
  std::uint64_t step = 0;
  int trainer = 0, peer = -1;
  double local_metric = 0, incoming_metric = 0;
  bool kept_incoming = false;
  std::string disc_hash;
};
struct TransferRecord {
  int round = 0, from_trainer = 0, to_trainer = 0;
  std::string payload;
  std::uint64_t bytes = 0;
  std::string blob_hash;
};
struct HistorySegment {
  std::vector<StepRecord> steps;
  std::vector<EvalRecord> evals;
  std::vector<EpochRecord> epochs;
  std::uint64_t skipped_steps = 0;
};
struct TrainerSummary {
  int trainer = 0;
  std::uint64_t steps = 0;
  std::uint32_t epochs_completed = 0;
  double final_d_loss = 0, final_g_total = 0, final_g_fwd = 0, final_g_adv = 0, final_g_cyc = 0;
  double final_val_forward_mae = 0, final_val_inverse_mae = 0, final_val_combined = 0;
  std::uint64_t rounds = 0, incoming_adopted = 0, files_opened = 0, bytes_read = 0,
                samples_shuffled = 0, skipped_steps = 0;
  bool is_best = false;
};
struct RunHistory {
  std::string config_hash, mode;
  int n_trainers = 1;
  std::vector<PretrainRecord> pretrain;
  std::vector<StepRecord> steps;
  std::vector<EvalRecord> evals;
  std::vector<EpochRecord> epochs;
  std::vector<RoundRecord> rounds;
  std::vector<TrainerRoundRecord> trainer_rounds;
  std::vector<TransferRecord> transfers;
  int best_trainer = -1;
  surrogate::EvalMetric best_metric;
  std::vector<TrainerSummary> summaries;
};

}  // namespace train
}  // namespace ltfb
