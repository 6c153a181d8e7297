// Synthetic JAG-shaped data on the device: the reference's analytic
// generator (synth/generator.hpp:41-206) evaluated straight into the
// HBM-resident data store, so a large partition never exists on the host.
//
// One CTA per (sample, view x channel image); every thread recomputes the
// sample's sweep point (xoshiro256** seeded by mix_seed(seed, id, 0x9e37),
// integer-exact) and the per-image constants, then renders its pixels. The
// (view, channel) == (0, 0) CTA also writes the 5 inputs and the scalar
// outputs (the 31-term basis dot product).
//
// Numerics: every double expression keeps the reference's evaluation order
// and this file is compiled with -fmad=false (build.py), so the only
// differences from the host generator come from the device libm's exp / sin
// / cos (<= 1-2 double ulp); after the fp32 cast the outputs agree to <= 1
// fp32 ulp (tests/test_gpu_parity.py::test_device_synth_matches_host).
#include <cstdint>

#include "kernels.hpp"

namespace ltfb_dev {

namespace {

constexpr double kTwoPi = 6.283185307179586476925286766559;
constexpr double kPi = 3.14159265358979323846;
constexpr int kBasis = 31;
constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

__device__ __forceinline__ std::uint64_t sm_step(std::uint64_t& s) {  // core/rng.hpp:14-21
  s += kGolden;
  std::uint64_t v = s;
  v = (v ^ (v >> 30)) * 0xbf58476d1ce4e5b9ULL;
  v = (v ^ (v >> 27)) * 0x94d049bb133111ebULL;
  return v ^ (v >> 31);
}

__device__ __forceinline__ void mix_word(std::uint64_t& acc, std::uint64_t w) {  // core/rng.hpp:23-30
  acc ^= w + kGolden + (acc << 6) + (acc >> 2);
  sm_step(acc);
}

__device__ __forceinline__ std::uint64_t rol(std::uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

struct DevRng {  // xoshiro256** (core/rng.hpp:35-60)
  std::uint64_t w[4];
  __device__ explicit DevRng(std::uint64_t seed) {
    for (int i = 0; i < 4; ++i) w[i] = sm_step(seed);
  }
  __device__ std::uint64_t next() {
    const std::uint64_t out = rol(w[1] * 5, 7) * 9;
    const std::uint64_t shifted = w[1] << 17;
    w[2] ^= w[0];
    w[3] ^= w[1];
    w[1] ^= w[2];
    w[0] ^= w[3];
    w[2] ^= shifted;
    w[3] = rol(w[3], 45);
    return out;
  }
  __device__ double uniform(double lo, double hi) {
    const double u = static_cast<double>(next() >> 11) * 0x1.0p-53;
    return lo + (hi - lo) * u;
  }
};

/// sweep_point (generator.hpp:177-192): lexicographic g^5 cell + jitter.
__device__ void sweep_point(std::uint64_t id, unsigned g, std::uint64_t seed, double p[5]) {
  std::uint64_t rem = id;
  for (int k = 4; k >= 0; --k, rem /= g) p[k] = static_cast<double>(rem % g);
  std::uint64_t acc = 0x243f6a8885a308d3ULL;
  mix_word(acc, seed);
  mix_word(acc, id);
  mix_word(acc, 0x9e37ULL);
  DevRng rng(sm_step(acc));
  for (int k = 0; k < 5; ++k) p[k] = (p[k] + 0.5 + rng.uniform(-0.4, 0.4)) / static_cast<double>(g);
}

__global__ void __launch_bounds__(256) k_synth(SynthArgs a) {
  const long long r = blockIdx.x;
  const int vc = blockIdx.y;
  const int v = vc / a.C, c = vc % a.C;
  const std::uint64_t id = a.ids ? a.ids[r] : a.first + static_cast<std::uint64_t>(r);
  double p[5];
  sweep_point(id, a.g, a.sampling_seed, p);
  float* yrow = a.y + r * a.y_stride;

  if (vc == 0 && threadIdx.x < 5) a.x[r * 5 + threadIdx.x] = static_cast<float>(p[threadIdx.x]);
  if (vc == 0 && threadIdx.x < static_cast<unsigned>(a.S)) {
    double phi[kBasis];  // scalar_basis (generator.hpp:41-49)
    int o = 0;
    phi[o++] = 1.0;
    for (int i = 0; i < 5; ++i) phi[o++] = p[i];
    for (int i = 0; i < 5; ++i)
      for (int j = i; j < 5; ++j) phi[o++] = p[i] * p[j];
    for (int i = 0; i < 5; ++i) phi[o++] = sin(kTwoPi * p[i]);
    for (int i = 0; i < 5; ++i) phi[o++] = cos(kTwoPi * p[i]);
    const double* cf = a.coeffs + threadIdx.x * kBasis;
    double acc = 0;
    for (int t = 0; t < kBasis; ++t) acc += cf[t] * phi[t];
    yrow[threadIdx.x] = static_cast<float>(acc);
  }

  // render (generator.hpp:118-150), image (v, c)
  const double drive = p[0], theta0 = kPi * p[1], ecc = 1.2 * (p[2] - 0.5);
  const double cx = 0.25 * (p[3] - 0.5), cy = 0.25 * (p[4] - 0.5);
  const double sigma = 0.10 + 0.25 * drive * drive;
  const double amp = 0.4 + 1.8 * drive * drive * drive + 0.3 * sin(kTwoPi * drive);
  const double theta = theta0 + static_cast<double>(v) * kPi / static_cast<double>(a.V);
  const double ct = cos(theta), st = sin(theta);
  const double wl = a.wavelength[c];
  const double sx = sigma * wl * exp(ecc), sy = sigma * wl * exp(-ecc);
  const double sx2 = sx * sx, sy2 = sy * sy;
  const double amp_c = amp * a.gain[v * a.C + c] * exp(-static_cast<double>(c) * (0.3 + 0.6 * drive));
  const double hh = static_cast<double>(a.H), ww = static_cast<double>(a.W);
  const double hc = 0.5 * static_cast<double>(a.H - 1), wc = 0.5 * static_cast<double>(a.W - 1);
  float* img = yrow + a.S + static_cast<long long>(vc) * a.H * a.W;
  const int npix = a.H * a.W;
  for (int q = threadIdx.x; q < npix; q += blockDim.x) {
    const int i = q / a.W, j = q - i * a.W;
    const double yy = (static_cast<double>(i) - hc) / hh - cy;
    const double xx = (static_cast<double>(j) - wc) / ww - cx;
    const double xr = ct * xx + st * yy, yr = -st * xx + ct * yy;
    img[q] = static_cast<float>(amp_c * exp(-0.5 * (xr * xr / sx2 + yr * yr / sy2)));
  }
}

}  // namespace

void launch_synth(const SynthArgs& a, long long n, cudaStream_t s) {
  if (n <= 0) return;
  const dim3 grid(static_cast<unsigned>(n), static_cast<unsigned>(a.V * a.C));
  k_synth<<<grid, 256, 0, s>>>(a);
}

}  // namespace ltfb_dev

// ------------------------------------------------------------------ host --
#include "ltfb_b200/host_algos.hpp"

namespace ltfb_dev {

void synth_generate_device(const ltfb::surrogate::ModalityDims& dims, std::uint64_t spec_seed,
                           double noise_level, const std::uint32_t* ids, std::uint64_t first,
                           std::size_t n, std::uint64_t total_n, std::uint64_t sampling_seed, float* x,
                           float* y, long long y_stride, cudaStream_t s) {
  if (noise_level != 0.0)
    throw ltfb::ContractError("device generator: noise_level must be 0 (the noise stream is sequential)");
  if (total_n < 1) throw ltfb::ContractError("generate_dataset: n must be >= 1");
  ltfb::synth::GeneratorSpec spec;
  spec.dims = dims;
  spec.spec_seed = spec_seed;
  const ltfb::synth::SynthGenerator gen(spec);  // validates dims, input_dim == 5
  if (dims.scalar_dim > 256) throw ltfb::ContractError("device generator: scalar_dim must be <= 256");
  if (y_stride < static_cast<long long>(dims.output_dim()))
    throw ltfb::ContractError("device generator: y row stride below output_dim");
  if (n == 0) return;
  const std::size_t nc = gen.coeffs.size(), ng = gen.gain.size(), nw = gen.wavelength.size();
  std::vector<double> tables(nc + ng + nw);
  std::copy(gen.coeffs.begin(), gen.coeffs.end(), tables.begin());
  std::copy(gen.gain.begin(), gen.gain.end(), tables.begin() + nc);
  std::copy(gen.wavelength.begin(), gen.wavelength.end(), tables.begin() + nc + ng);
  double* dt = nullptr;
  std::uint32_t* di = nullptr;
  auto ck = [](cudaError_t e) {
    if (e != cudaSuccess) throw ltfb::Error(std::string("CUDA error in the device generator: ") + cudaGetErrorString(e));
  };
  ck(cudaMallocAsync(reinterpret_cast<void**>(&dt), tables.size() * sizeof(double), s));
  ck(cudaMemcpyAsync(dt, tables.data(), tables.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  if (ids) {
    ck(cudaMallocAsync(reinterpret_cast<void**>(&di), n * 4, s));
    ck(cudaMemcpyAsync(di, ids, n * 4, cudaMemcpyHostToDevice, s));
  }
  SynthArgs a{};
  a.ids = di;
  a.first = first;
  a.coeffs = dt;
  a.gain = dt + nc;
  a.wavelength = dt + nc + ng;
  a.S = static_cast<int>(dims.scalar_dim);
  a.V = static_cast<int>(dims.image_views);
  a.C = static_cast<int>(dims.image_channels);
  a.H = static_cast<int>(dims.image_h);
  a.W = static_cast<int>(dims.image_w);
  a.g = ltfb::synth::grid_side(total_n);
  a.sampling_seed = sampling_seed;
  a.x = x;
  a.y = y;
  a.y_stride = y_stride;
  launch_synth(a, static_cast<long long>(n), s);
  ck(cudaGetLastError());
  ck(cudaFreeAsync(dt, s));
  if (di) ck(cudaFreeAsync(di, s));
  // the host tables / ids must outlive the async copies
  ck(cudaStreamSynchronize(s));
}

}  // namespace ltfb_dev
