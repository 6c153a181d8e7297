// ltfb_b200 — the integer/seeded host algorithms of the hot path, plus the
// synthetic JAG-shaped data source and the LBDS bundle format.
//
// Everything here must be bit-identical to the reference (pairings,
// partitions, epoch permutations, sample ids, synthetic samples), so it runs
// on the host, where the reference's exact integer and libm sequences can be
// reproduced. The GPU consumes its outputs (permutations become slot lists in
// HBM; bundles and generated samples become the HBM-resident data store).
//
// Reference correspondence (/root/reference/proj/include/ltfb):
//   partition_dataset / Matching / pair_trainers  tournament/ltfb.hpp:24-66
//   incoming_wins (host mirror of the device rule) tournament/ltfb.hpp:82-88
//   split_dataset                                  tournament/runner.hpp:134-169
//   shard_split / epoch permutation                data/epoch_plan.hpp:41-89
//   SampleRecord                                   data/sample.hpp:12-27
//   LBDS bundles, DatasetIndex, assemble_tensors   data/bundle.hpp:25-224
//   SynthGenerator, grid_side, sweep_point,
//   generate_dataset                               synth/generator.hpp:29-206
#pragma once

#include <bit>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <utility>

#include "ltfb_b200/types.hpp"

namespace ltfb {

namespace data {
using SampleId = std::uint32_t;

struct SampleRecord {
  std::vector<float> inputs, outputs;
  bool matches(const surrogate::ModalityDims& d) const {
    return inputs.size() == d.input_dim && outputs.size() == d.output_dim();
  }
  bool operator==(const SampleRecord&) const = default;
};

/// Contiguous row ranges of a minibatch per shard; the first rows % n
/// shards get one extra row (data/epoch_plan.hpp:41-54).
inline std::vector<std::pair<std::size_t, std::size_t>> shard_split(std::size_t rows, int n_shards) {
  std::vector<std::pair<std::size_t, std::size_t>> out;
  const std::size_t n = static_cast<std::size_t>(n_shards);
  std::size_t at = 0;
  for (std::size_t s = 0; s < n; ++s) {
    const std::size_t len = rows / n + (s < rows % n ? 1 : 0);
    out.emplace_back(at, at + len);
    at += len;
  }
  return out;
}

/// Epoch permutation of a partition (data/epoch_plan.hpp:69-71).
inline std::vector<SampleId> epoch_permutation(const std::vector<SampleId>& partition,
                                               std::uint32_t epoch, std::uint64_t seed) {
  std::vector<SampleId> perm = partition;
  Rng(mix_seed({seed, epoch, 0x5caff1eULL})).shuffle(perm);
  return perm;
}

// ----------------------------------------------------------- LBDS bundles --
inline constexpr char kBundleMagic[4] = {'L', 'B', 'D', 'S'};
inline constexpr std::uint32_t kBundleVersion = 1;
inline constexpr std::size_t kBundleHeaderBytes = 40;

namespace detail {
inline void put32(std::ostream& os, std::uint32_t v) {
  unsigned char b[4] = {static_cast<unsigned char>(v), static_cast<unsigned char>(v >> 8),
                        static_cast<unsigned char>(v >> 16), static_cast<unsigned char>(v >> 24)};
  os.write(reinterpret_cast<const char*>(b), 4);
}
inline std::uint32_t get32(std::istream& is, const std::string& ctx) {
  unsigned char b[4];
  if (!is.read(reinterpret_cast<char*>(b), 4)) throw IoError("truncated read in " + ctx);
  return b[0] | (b[1] << 8) | (b[2] << 16) | (static_cast<std::uint32_t>(b[3]) << 24);
}
}  // namespace detail

struct BundleHeader {
  std::uint32_t version = kBundleVersion, sample_count = 0;
  surrogate::ModalityDims dims;
};

inline BundleHeader read_bundle_header(std::istream& is, const std::string& path) {
  char magic[4];
  if (!is.read(magic, 4) || std::memcmp(magic, kBundleMagic, 4) != 0)
    throw IoError("not a bundle file (bad magic): " + path);
  BundleHeader h;
  h.version = detail::get32(is, path);
  if (h.version != kBundleVersion) throw IoError("unsupported bundle version in " + path);
  h.sample_count = detail::get32(is, path);
  std::uint32_t* f[] = {&h.dims.input_dim, &h.dims.latent_dim, &h.dims.scalar_dim,
                        &h.dims.image_views, &h.dims.image_channels, &h.dims.image_h,
                        &h.dims.image_w};
  for (auto* p : f) *p = detail::get32(is, path);
  h.dims.validate();
  return h;
}

inline void write_bundle(const std::filesystem::path& path, const surrogate::ModalityDims& dims,
                         std::span<const SampleRecord> records) {
  static_assert(std::endian::native == std::endian::little, "LBDS writer assumes a little-endian host");
  const std::filesystem::path tmp = path.string() + ".tmp";
  {
    std::ofstream os(tmp, std::ios::binary);
    if (!os) throw IoError("cannot open " + tmp.string() + " for writing");
    os.write(kBundleMagic, 4);
    for (std::uint32_t v : {kBundleVersion, static_cast<std::uint32_t>(records.size()), dims.input_dim,
                            dims.latent_dim, dims.scalar_dim, dims.image_views, dims.image_channels,
                            dims.image_h, dims.image_w})
      detail::put32(os, v);
    for (const SampleRecord& r : records) {
      if (!r.matches(dims)) throw ContractError("sample record does not match the bundle dims");
      os.write(reinterpret_cast<const char*>(r.inputs.data()), r.inputs.size() * 4);
      os.write(reinterpret_cast<const char*>(r.outputs.data()), r.outputs.size() * 4);
    }
    if (!os) throw IoError("write failure on " + tmp.string());
  }
  std::error_code ec;
  std::filesystem::rename(tmp, path, ec);
  if (ec) throw IoError("cannot move bundle into place at " + path.string() + ": " + ec.message());
}

inline std::vector<std::filesystem::path> write_bundles(std::span<const SampleRecord> records,
                                                        const surrogate::ModalityDims& dims,
                                                        std::size_t per_file,
                                                        const std::filesystem::path& dir) {
  if (per_file < 1) throw ContractError("write_bundles: samples_per_file must be >= 1");
  std::error_code ec;
  std::filesystem::create_directories(dir, ec);
  std::vector<std::filesystem::path> paths;
  for (std::size_t at = 0, f = 0; at < records.size(); at += per_file, ++f) {
    char name[32];
    std::snprintf(name, sizeof name, "bundle_%05zu.lbds", f);
    paths.push_back(dir / name);
    write_bundle(paths.back(), dims, records.subspan(at, std::min(per_file, records.size() - at)));
  }
  return paths;
}

/// Global id -> (file, record) over a sorted set of bundle files
/// (data/bundle.hpp:134-193).
struct DatasetIndex {
  surrogate::ModalityDims dims;
  std::vector<std::filesystem::path> paths;
  std::vector<std::uint32_t> counts;
  std::vector<SampleId> bases;
  std::size_t total = 0;

  std::size_t stride_floats() const { return dims.record_floats(); }
  std::size_t stride_bytes() const { return stride_floats() * 4; }
  struct Location {
    std::size_t file_idx;
    std::uint32_t record_idx;
  };
  Location locate(SampleId id) const {
    if (id >= total)
      throw ContractError("sample id " + std::to_string(id) + " outside dataset of " + std::to_string(total));
    const auto it = std::upper_bound(bases.begin(), bases.end(), id);
    const std::size_t f = static_cast<std::size_t>(it - bases.begin()) - 1;
    return {f, id - bases[f]};
  }
  static DatasetIndex scan(const std::vector<std::filesystem::path>& files) {
    if (files.empty()) throw IoError("dataset scan: no bundle files given");
    DatasetIndex ix;
    for (std::size_t i = 0; i < files.size(); ++i) {
      std::ifstream is(files[i], std::ios::binary);
      if (!is) throw IoError("cannot open bundle " + files[i].string());
      const BundleHeader h = read_bundle_header(is, files[i].string());
      if (i == 0) ix.dims = h.dims;
      else if (!(h.dims == ix.dims)) throw IoError("bundle dims mismatch in " + files[i].string());
      ix.paths.push_back(files[i]);
      ix.counts.push_back(h.sample_count);
      ix.bases.push_back(static_cast<SampleId>(ix.total));
      ix.total += h.sample_count;
    }
    return ix;
  }
  static DatasetIndex scan_dir(const std::filesystem::path& dir) {
    std::vector<std::filesystem::path> files;
    std::error_code ec;
    for (const auto& e : std::filesystem::directory_iterator(dir, ec))
      if (e.path().extension() == ".lbds") files.push_back(e.path());
    if (ec) throw IoError("cannot list dataset directory " + dir.string());
    if (files.empty()) throw IoError("no .lbds bundle files under " + dir.string());
    std::sort(files.begin(), files.end());
    return scan(files);
  }
};

/// Reads records for `ids` (in order) into x [n x input] and y [n x output]
/// row-major host arrays; `y_stride` lets the caller read straight into a
/// padded staging buffer. Returns the number of distinct files opened.
inline std::size_t read_records(const DatasetIndex& index, std::span<const SampleId> ids, float* x,
                                float* y, std::size_t y_stride) {
  const std::size_t in = index.dims.input_dim, out = index.dims.output_dim();
  std::ifstream is;
  std::size_t open = static_cast<std::size_t>(-1), opened = 0;
  std::vector<float> rec(index.stride_floats());
  for (std::size_t r = 0; r < ids.size(); ++r) {
    const auto loc = index.locate(ids[r]);
    if (loc.file_idx != open) {
      is.close();
      is.clear();
      is.open(index.paths[loc.file_idx], std::ios::binary);
      if (!is) throw IoError("cannot open bundle " + index.paths[loc.file_idx].string());
      open = loc.file_idx;
      ++opened;
    }
    is.seekg(static_cast<std::streamoff>(kBundleHeaderBytes + loc.record_idx * index.stride_bytes()));
    if (!is.read(reinterpret_cast<char*>(rec.data()), static_cast<std::streamsize>(index.stride_bytes())))
      throw IoError("truncated read in " + index.paths[loc.file_idx].string());
    std::memcpy(x + r * in, rec.data(), in * 4);
    std::memcpy(y + r * y_stride, rec.data() + in, out * 4);
  }
  return opened;
}

/// data/bundle.hpp:198-224.
inline std::pair<nn::Tensor<float>, nn::Tensor<float>> assemble_tensors(const DatasetIndex& index,
                                                                        std::span<const SampleId> ids) {
  nn::Tensor<float> x({ids.size(), index.dims.input_dim});
  nn::Tensor<float> y({ids.size(), index.dims.output_dim()});
  read_records(index, ids, x.data.data(), y.data.data(), index.dims.output_dim());
  return {std::move(x), std::move(y)};
}
}  // namespace data

// --------------------------------------------------------------- synth --
namespace synth {

struct GeneratorSpec {
  surrogate::ModalityDims dims;
  double noise_level = 0.0;
  std::uint64_t spec_seed = 1;
};

inline constexpr double kTwoPi = 6.283185307179586476925286766559;
inline constexpr double kPi = 3.14159265358979323846;
inline constexpr std::size_t kScalarBasisTerms = 31;

/// 1, p_i, p_i p_j (i <= j), sin 2pi p_i, cos 2pi p_i (generator.hpp:41-49).
inline void scalar_basis(std::span<const double> p, double* phi) {
  double* o = phi;
  *o++ = 1.0;
  for (int i = 0; i < 5; ++i) *o++ = p[i];
  for (int i = 0; i < 5; ++i)
    for (int j = i; j < 5; ++j) *o++ = p[i] * p[j];
  for (int i = 0; i < 5; ++i) *o++ = std::sin(kTwoPi * p[i]);
  for (int i = 0; i < 5; ++i) *o++ = std::cos(kTwoPi * p[i]);
}

/// Analytic JAG stand-in (generator.hpp:51-165). The per-spec tables are
/// public so the device generator (data-store population at scale) can be
/// fed the exact same coefficients.
class SynthGenerator {
 public:
  explicit SynthGenerator(GeneratorSpec spec) : spec_(spec) {
    spec_.dims.validate();
    if (spec_.dims.input_dim != 5) throw ContractError("SynthGenerator: input_dim must be 5");
    Rng rng(mix_seed({spec_.spec_seed, 0xc0effULL}));
    coeffs.resize(spec_.dims.scalar_dim * kScalarBasisTerms);
    for (double& c : coeffs) c = rng.uniform(-1.0, 1.0);
    gain.resize(static_cast<std::size_t>(spec_.dims.image_views) * spec_.dims.image_channels);
    for (double& g : gain) g = rng.uniform(0.9, 1.1);
    wavelength.resize(spec_.dims.image_channels);
    for (std::uint32_t c = 0; c < spec_.dims.image_channels; ++c)
      wavelength[c] = (1.0 / (1.0 + 0.25 * c)) * rng.uniform(0.95, 1.05);
  }
  const GeneratorSpec& spec() const { return spec_; }

  /// Writes inputs[5] and outputs[output_dim] for one parameter point.
  void sample_into(std::span<const double> p, float* inputs, float* outputs) const {
    if (p.size() != 5) throw ContractError("synth_sample: expected 5 parameters");
    for (double v : p)
      if (!(v >= 0.0 && v <= 1.0)) throw ContractError("synth_sample: parameters must lie in [0,1]");
    const auto& d = spec_.dims;
    for (int i = 0; i < 5; ++i) inputs[i] = static_cast<float>(p[i]);
    double phi[kScalarBasisTerms];
    scalar_basis(p, phi);
    for (std::uint32_t s = 0; s < d.scalar_dim; ++s) {
      double acc = 0;
      for (std::size_t t = 0; t < kScalarBasisTerms; ++t) acc += coeffs[s * kScalarBasisTerms + t] * phi[t];
      outputs[s] = static_cast<float>(acc);
    }
    render(p, outputs + d.scalar_dim);
    if (spec_.noise_level > 0.0) add_noise(p, outputs);
  }
  data::SampleRecord sample(std::span<const double> p) const {
    data::SampleRecord r;
    r.inputs.resize(spec_.dims.input_dim);
    r.outputs.resize(spec_.dims.output_dim());
    sample_into(p, r.inputs.data(), r.outputs.data());
    return r;
  }

  std::vector<double> coeffs, gain, wavelength;

 private:
  void render(std::span<const double> p, float* out) const {
    const auto& d = spec_.dims;
    const double drive = p[0], theta0 = kPi * p[1], ecc = 1.2 * (p[2] - 0.5);
    const double cx = 0.25 * (p[3] - 0.5), cy = 0.25 * (p[4] - 0.5);
    const double sigma = 0.10 + 0.25 * drive * drive;
    const double amp = 0.4 + 1.8 * drive * drive * drive + 0.3 * std::sin(kTwoPi * drive);
    for (std::uint32_t v = 0; v < d.image_views; ++v) {
      const double theta = theta0 + v * kPi / d.image_views;
      const double ct = std::cos(theta), st = std::sin(theta);
      for (std::uint32_t c = 0; c < d.image_channels; ++c) {
        const double wl = wavelength[c];
        const double sx = sigma * wl * std::exp(ecc), sy = sigma * wl * std::exp(-ecc);
        const double a = amp * gain[v * d.image_channels + c] *
                         std::exp(-static_cast<double>(c) * (0.3 + 0.6 * drive));
        for (std::uint32_t i = 0; i < d.image_h; ++i) {
          const double yy = (static_cast<double>(i) - 0.5 * (d.image_h - 1)) / d.image_h - cy;
          for (std::uint32_t j = 0; j < d.image_w; ++j) {
            const double xx = (static_cast<double>(j) - 0.5 * (d.image_w - 1)) / d.image_w - cx;
            const double xr = ct * xx + st * yy, yr = -st * xx + ct * yy;
            *out++ = static_cast<float>(a * std::exp(-0.5 * (xr * xr / (sx * sx) + yr * yr / (sy * sy))));
          }
        }
      }
    }
  }
  void add_noise(std::span<const double> p, float* outputs) const {
    std::uint64_t h = spec_.spec_seed;
    for (double v : p) h = mix_seed({h, std::bit_cast<std::uint64_t>(v)});
    Rng rng(h);
    const auto& d = spec_.dims;
    for (std::uint32_t s = 0; s < d.scalar_dim; ++s)
      outputs[s] += static_cast<float>(spec_.noise_level * rng.normal());
    for (std::size_t i = d.scalar_dim; i < d.output_dim(); ++i) {
      const double noisy = outputs[i] + spec_.noise_level * 0.5 * rng.normal();
      outputs[i] = static_cast<float>(noisy > 0.0 ? noisy : 0.0);
    }
  }
  GeneratorSpec spec_;
};

inline std::uint32_t grid_side(std::uint64_t n) {
  std::uint32_t g = 1;
  while (static_cast<std::uint64_t>(g) * g * g * g * g < n) ++g;
  return g;
}

/// generator.hpp:177-192: lexicographic g^5 grid (first coordinate
/// slowest), cell centred, with seeded sub-cell jitter.
inline std::array<double, 5> sweep_point(std::uint64_t i, std::uint32_t g, std::uint64_t seed) {
  std::array<double, 5> p{};
  std::uint64_t rem = i;
  for (int k = 4; k >= 0; --k, rem /= g) p[k] = static_cast<double>(rem % g);
  Rng rng(mix_seed({seed, i, 0x9e37ULL}));
  for (int k = 0; k < 5; ++k) p[k] = (p[k] + 0.5 + rng.uniform(-0.4, 0.4)) / g;
  return p;
}

inline std::vector<data::SampleRecord> generate_dataset(const SynthGenerator& gen, std::uint64_t n,
                                                        std::uint64_t sampling_seed) {
  if (n < 1) throw ContractError("generate_dataset: n must be >= 1");
  const std::uint32_t g = grid_side(n);
  std::vector<data::SampleRecord> out;
  out.reserve(n);
  for (std::uint64_t i = 0; i < n; ++i) out.push_back(gen.sample(sweep_point(i, g, sampling_seed)));
  return out;
}
}  // namespace synth

// ----------------------------------------------------------- tournament --
namespace tournament {

inline std::vector<std::vector<data::SampleId>> partition_dataset(std::vector<data::SampleId> ids, int k,
                                                                  std::uint64_t seed) {
  if (k < 1) throw ContractError("partition_dataset: k must be >= 1");
  if (static_cast<std::size_t>(k) > ids.size()) throw ContractError("partition_dataset: k exceeds the number of ids");
  Rng(mix_seed({seed, 0x9a27ULL})).shuffle(ids);
  std::vector<std::vector<data::SampleId>> parts(static_cast<std::size_t>(k));
  auto at = ids.begin();
  for (std::size_t p = 0; p < parts.size(); ++p) {
    const std::size_t len = ids.size() / parts.size() + (p < ids.size() % parts.size() ? 1 : 0);
    parts[p].assign(at, at + static_cast<std::ptrdiff_t>(len));
    at += static_cast<std::ptrdiff_t>(len);
  }
  return parts;
}

struct Matching {
  std::vector<std::array<int, 2>> pairs;
  int bye = -1;
};

inline Matching pair_trainers(int k, int round, std::uint64_t seed) {
  Matching m;
  if (k < 2) return m;
  std::vector<int> order(static_cast<std::size_t>(k));
  std::iota(order.begin(), order.end(), 0);
  Rng(mix_seed({seed, static_cast<std::uint64_t>(round), 0x9a12ULL})).shuffle(order);
  if (k % 2 == 1) {
    m.bye = order.back();
    order.pop_back();
  }
  for (std::size_t i = 0; i + 1 < order.size(); i += 2) m.pairs.push_back({order[i], order[i + 1]});
  return m;
}

/// Host statement of the tournament rule the device decision kernel applies.
inline bool incoming_wins(double local, double incoming) {
  if (!std::isfinite(incoming)) return false;
  if (!std::isfinite(local)) return true;
  return incoming < local;
}

namespace detail {
struct DataSplit {
  std::vector<data::SampleId> validation;
  std::vector<std::vector<data::SampleId>> train, tournament;
};

inline DataSplit split_dataset(std::size_t total, int k, double validation_fraction, double tournament_fraction,
                               std::uint64_t seed, bool need_tournament) {
  std::vector<data::SampleId> ids(total);
  std::iota(ids.begin(), ids.end(), data::SampleId{0});
  Rng(mix_seed({seed, 0xa11ULL})).shuffle(ids);
  const std::size_t n_val = static_cast<std::size_t>(validation_fraction * static_cast<double>(ids.size()));
  DataSplit s;
  s.validation.assign(ids.begin(), ids.begin() + static_cast<std::ptrdiff_t>(n_val));
  auto parts = partition_dataset(std::vector<data::SampleId>(ids.begin() + static_cast<std::ptrdiff_t>(n_val), ids.end()),
                                 k, mix_seed({seed, 0xbbULL}));
  s.train.resize(parts.size());
  s.tournament.resize(parts.size());
  for (std::size_t t = 0; t < parts.size(); ++t) {
    auto& part = parts[t];
    Rng(mix_seed({seed, 0xccULL, t})).shuffle(part);
    std::size_t n_tour = static_cast<std::size_t>(tournament_fraction * static_cast<double>(part.size()));
    if (need_tournament && n_tour == 0 && part.size() > 1) n_tour = 1;
    s.tournament[t].assign(part.begin(), part.begin() + static_cast<std::ptrdiff_t>(n_tour));
    s.train[t].assign(part.begin() + static_cast<std::ptrdiff_t>(n_tour), part.end());
  }
  return s;
}
}  // namespace detail
}  // namespace tournament
}  // namespace ltfb
