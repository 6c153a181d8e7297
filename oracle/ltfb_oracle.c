/* TEST INFRASTRUCTURE (oracle) — not product code. See ltfb_oracle.h.
 *
 * Plain-C restatement of the reference's LTFB hot path. Citations are to
 * /root/reference/proj/include/ltfb/<file>:<line>. The arithmetic order of
 * every loop is chosen to equal the reference compiled with the strict Eigen
 * shim (oracle/shim/Eigen/Core), so on the same machine results are
 * bit-identical to tests/golden/*.npz; that is what
 * tests/test_oracle_golden.py pins.
 */
#include "ltfb_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ====================================================================== */
/* core/rng.hpp                                                            */
/* ====================================================================== */

/* rng.hpp:13-18 */
uint64_t lo_splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* rng.hpp:23-30 */
uint64_t lo_mix_seed(const uint64_t* parts, int n) {
  uint64_t s = 0x243f6a8885a308d3ULL;
  for (int i = 0; i < n; ++i) {
    s ^= parts[i] + 0x9e3779b97f4a7c15ULL + (s << 6) + (s >> 2);
    (void)lo_splitmix64(&s);
  }
  return lo_splitmix64(&s);
}

static uint64_t mix2(uint64_t a, uint64_t b) {
  const uint64_t p[2] = {a, b};
  return lo_mix_seed(p, 2);
}
static uint64_t mix3(uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t p[3] = {a, b, c};
  return lo_mix_seed(p, 3);
}

/* rng.hpp:39-41 */
void lo_rng_init(lo_rng* r, uint64_t seed) {
  for (int i = 0; i < 4; ++i) r->s[i] = lo_splitmix64(&seed);
}

static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.hpp:46-56 (xoshiro256**) */
uint64_t lo_rng_next(lo_rng* r) {
  uint64_t* s = r->s;
  const uint64_t result = rotl64(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

/* rng.hpp:61-63 */
double lo_rng_uniform(lo_rng* r) {
  return (double)(lo_rng_next(r) >> 11) * 0x1.0p-53;
}
static double rng_uniform_range(lo_rng* r, double lo, double hi) {
  return lo + (hi - lo) * lo_rng_uniform(r);
}

/* rng.hpp:66-71 */
uint64_t lo_rng_below(lo_rng* r, uint64_t n) {
  const uint64_t threshold = (~n + 1) % n;
  uint64_t x = lo_rng_next(r);
  while (x < threshold) x = lo_rng_next(r);
  return x % n;
}

/* rng.hpp:74-80 */
double lo_rng_normal(lo_rng* r) {
  double u1 = lo_rng_uniform(r);
  while (u1 <= 0.0) u1 = lo_rng_uniform(r);
  const double u2 = lo_rng_uniform(r);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

/* rng.hpp:84-89 */
void lo_shuffle_u32(lo_rng* r, uint32_t* v, size_t n) {
  for (size_t i = n; i > 1; --i) {
    const size_t j = (size_t)lo_rng_below(r, i);
    const uint32_t tmp = v[i - 1];
    v[i - 1] = v[j];
    v[j] = tmp;
  }
}
void lo_shuffle_i32(lo_rng* r, int32_t* v, size_t n) {
  for (size_t i = n; i > 1; --i) {
    const size_t j = (size_t)lo_rng_below(r, i);
    const int32_t tmp = v[i - 1];
    v[i - 1] = v[j];
    v[j] = tmp;
  }
}

/* hash.hpp:15-22 */
uint64_t lo_fnv1a64(const void* data, size_t n, uint64_t h) {
  const unsigned char* p = (const unsigned char*)data;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* ====================================================================== */
/* tournament/ltfb.hpp, runner.hpp, data/epoch_plan.hpp                    */
/* ====================================================================== */

/* tournament/ltfb.hpp:24-43 */
int lo_partition(const uint32_t* ids, size_t n, int k, uint64_t seed,
                 uint32_t* out_ids, uint32_t* out_sizes) {
  if (k < 1 || (size_t)k > n) return -1;
  memcpy(out_ids, ids, n * sizeof(uint32_t));
  lo_rng r;
  lo_rng_init(&r, mix2(seed, 0x9a27ULL));
  lo_shuffle_u32(&r, out_ids, n);
  const size_t base = n / (size_t)k, extra = n % (size_t)k;
  for (size_t p = 0; p < (size_t)k; ++p)
    out_sizes[p] = (uint32_t)(base + (p < extra ? 1 : 0));
  return 0;
}

/* tournament/ltfb.hpp:52-66 */
int lo_pair_trainers(int k, int round, uint64_t seed, int32_t* pairs,
                     int32_t* bye) {
  *bye = -1;
  if (k < 2) return 0;
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);
  for (int i = 0; i < k; ++i) order[i] = i;
  lo_rng r;
  lo_rng_init(&r, mix3(seed, (uint64_t)round, 0x9a12ULL));
  lo_shuffle_i32(&r, order, (size_t)k);
  int n = k;
  if (k % 2 == 1) {
    *bye = order[k - 1];
    n = k - 1;
  }
  int np = 0;
  for (int i = 0; i + 1 < n; i += 2) {
    pairs[2 * np] = order[i];
    pairs[2 * np + 1] = order[i + 1];
    ++np;
  }
  free(order);
  return np;
}

/* runner.hpp:134-169 */
int lo_split_dataset(size_t total, int k, double validation_fraction,
                     double tournament_fraction, uint64_t seed,
                     int need_tournament, uint32_t* out_val, size_t* n_val,
                     uint32_t* out_train, uint32_t* train_sizes,
                     uint32_t* out_tour, uint32_t* tour_sizes) {
  uint32_t* ids = (uint32_t*)malloc(sizeof(uint32_t) * (total ? total : 1));
  for (size_t i = 0; i < total; ++i) ids[i] = (uint32_t)i;
  lo_rng r;
  lo_rng_init(&r, mix2(seed, 0xa11ULL));
  lo_shuffle_u32(&r, ids, total);
  const size_t nv = (size_t)(validation_fraction * (double)total);
  memcpy(out_val, ids, nv * sizeof(uint32_t));
  *n_val = nv;
  const size_t pool_n = total - nv;
  uint32_t* parts = (uint32_t*)malloc(sizeof(uint32_t) * (pool_n ? pool_n : 1));
  uint32_t* sizes = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)k);
  if (lo_partition(ids + nv, pool_n, k, mix2(seed, 0xbbULL), parts, sizes) != 0) {
    free(ids);
    free(parts);
    free(sizes);
    return -1;
  }
  size_t off = 0, toff = 0, troff = 0;
  for (int t = 0; t < k; ++t) {
    uint32_t* part = parts + off;
    const size_t len = sizes[t];
    lo_rng pr;
    lo_rng_init(&pr, mix3(seed, 0xccULL, (uint64_t)t));
    lo_shuffle_u32(&pr, part, len);
    size_t n_tour = (size_t)(tournament_fraction * (double)len);
    if (need_tournament && n_tour == 0 && len > 1) n_tour = 1;
    memcpy(out_tour + toff, part, n_tour * sizeof(uint32_t));
    memcpy(out_train + troff, part + n_tour, (len - n_tour) * sizeof(uint32_t));
    tour_sizes[t] = (uint32_t)n_tour;
    train_sizes[t] = (uint32_t)(len - n_tour);
    toff += n_tour;
    troff += len - n_tour;
    off += len;
  }
  free(ids);
  free(parts);
  free(sizes);
  return 0;
}

/* tournament/ltfb.hpp:82-88 */
int lo_incoming_wins(double local, double incoming) {
  if (!isfinite(incoming)) return 0;
  if (!isfinite(local)) return 1;
  return incoming < local;
}

/* data/epoch_plan.hpp:69-71 */
void lo_plan_perm(const uint32_t* partition, size_t n, uint32_t epoch,
                  uint64_t seed, uint32_t* perm_out) {
  memcpy(perm_out, partition, n * sizeof(uint32_t));
  lo_rng r;
  lo_rng_init(&r, mix3(seed, (uint64_t)epoch, 0x5caff1eULL));
  lo_shuffle_u32(&r, perm_out, n);
}

/* ====================================================================== */
/* synth/generator.hpp                                                     */
/* ====================================================================== */
#define LO_TWO_PI 6.283185307179586476925286766559
#define LO_PI 3.14159265358979323846
#define LO_BASIS 31

struct lo_synth {
  uint32_t dims[7];
  uint64_t spec_seed;
  double noise;
  double* coeffs; /* scalar_dim x 31 */
  double* gain;   /* views*channels */
  double* wavelength;
};

/* generator.hpp:51-62 */
lo_synth* lo_synth_create(const uint32_t* dims7, uint64_t spec_seed,
                          double noise_level) {
  if (dims7[0] != 5) return NULL;
  lo_synth* g = (lo_synth*)calloc(1, sizeof(lo_synth));
  memcpy(g->dims, dims7, sizeof(g->dims));
  g->spec_seed = spec_seed;
  g->noise = noise_level;
  lo_rng r;
  lo_rng_init(&r, mix2(spec_seed, 0xc0effULL));
  const size_t nc = (size_t)dims7[2] * LO_BASIS;
  g->coeffs = (double*)malloc(sizeof(double) * nc);
  for (size_t i = 0; i < nc; ++i) g->coeffs[i] = rng_uniform_range(&r, -1.0, 1.0);
  const size_t vc = (size_t)dims7[3] * dims7[4];
  g->gain = (double*)malloc(sizeof(double) * vc);
  for (size_t i = 0; i < vc; ++i) g->gain[i] = rng_uniform_range(&r, 0.9, 1.1);
  g->wavelength = (double*)malloc(sizeof(double) * dims7[4]);
  for (uint32_t c = 0; c < dims7[4]; ++c)
    g->wavelength[c] = (1.0 / (1.0 + 0.25 * c)) * rng_uniform_range(&r, 0.95, 1.05);
  return g;
}

void lo_synth_destroy(lo_synth* g) {
  if (!g) return;
  free(g->coeffs);
  free(g->gain);
  free(g->wavelength);
  free(g);
}

/* generator.hpp:41-49 */
static void scalar_basis(const double* p, double* phi) {
  size_t k = 0;
  phi[k++] = 1.0;
  for (int i = 0; i < 5; ++i) phi[k++] = p[i];
  for (int i = 0; i < 5; ++i)
    for (int j = i; j < 5; ++j) phi[k++] = p[i] * p[j];
  for (int i = 0; i < 5; ++i) phi[k++] = sin(LO_TWO_PI * p[i]);
  for (int i = 0; i < 5; ++i) phi[k++] = cos(LO_TWO_PI * p[i]);
}

/* generator.hpp:102-143 */
static void render_images(const lo_synth* g, const double* p, float* out) {
  const uint32_t V = g->dims[3], C = g->dims[4], H = g->dims[5], W = g->dims[6];
  const double drive = p[0];
  const double theta_base = LO_PI * p[1];
  const double ecc = 1.2 * (p[2] - 0.5);
  const double cx = 0.25 * (p[3] - 0.5);
  const double cy = 0.25 * (p[4] - 0.5);
  const double sigma = 0.10 + 0.25 * drive * drive;
  const double amp = 0.4 + 1.8 * drive * drive * drive + 0.3 * sin(LO_TWO_PI * drive);
  size_t k = 0;
  for (uint32_t v = 0; v < V; ++v) {
    const double theta = theta_base + v * LO_PI / V;
    const double ct = cos(theta), st = sin(theta);
    for (uint32_t c = 0; c < C; ++c) {
      const double wl = g->wavelength[c];
      const double sx = sigma * wl * exp(ecc);
      const double sy = sigma * wl * exp(-ecc);
      const double a = amp * g->gain[v * C + c] * exp(-(double)c * (0.3 + 0.6 * drive));
      for (uint32_t i = 0; i < H; ++i) {
        const double y = ((double)i - 0.5 * (H - 1)) / H - cy;
        for (uint32_t j = 0; j < W; ++j) {
          const double x = ((double)j - 0.5 * (W - 1)) / W - cx;
          const double xr = ct * x + st * y;
          const double yr = -st * x + ct * y;
          const double val = a * exp(-0.5 * (xr * xr / (sx * sx) + yr * yr / (sy * sy)));
          out[k++] = (float)val;
        }
      }
    }
  }
}

/* generator.hpp:72-98 + apply_noise :145-159 */
int lo_synth_sample(const lo_synth* g, const double* p5, float* inputs,
                    float* outputs) {
  for (int i = 0; i < 5; ++i)
    if (!(p5[i] >= 0.0 && p5[i] <= 1.0)) return -1;
  for (int i = 0; i < 5; ++i) inputs[i] = (float)p5[i];
  double phi[LO_BASIS];
  scalar_basis(p5, phi);
  const uint32_t S = g->dims[2];
  for (uint32_t s = 0; s < S; ++s) {
    double acc = 0;
    for (int t = 0; t < LO_BASIS; ++t) acc += g->coeffs[s * LO_BASIS + t] * phi[t];
    outputs[s] = (float)acc;
  }
  render_images(g, p5, outputs + S);
  if (g->noise > 0.0) {
    uint64_t h = g->spec_seed;
    for (int i = 0; i < 5; ++i) {
      uint64_t bits;
      memcpy(&bits, &p5[i], 8);
      h = mix2(h, bits);
    }
    lo_rng r;
    lo_rng_init(&r, h);
    const size_t out_dim = S + (size_t)g->dims[3] * g->dims[4] * g->dims[5] * g->dims[6];
    for (uint32_t s = 0; s < S; ++s) outputs[s] += (float)(g->noise * lo_rng_normal(&r));
    for (size_t i = S; i < out_dim; ++i) {
      const double noisy = outputs[i] + g->noise * 0.5 * lo_rng_normal(&r);
      outputs[i] = (float)(noisy > 0.0 ? noisy : 0.0);
    }
  }
  return 0;
}

/* generator.hpp:168-173 */
uint32_t lo_grid_side(uint64_t n) {
  uint32_t g = 1;
  while ((uint64_t)g * g * g * g * g < n) ++g;
  return g;
}

/* generator.hpp:177-192 */
void lo_sweep_point(uint64_t i, uint32_t g, uint64_t sampling_seed, double* p) {
  uint64_t rem = i;
  for (int k = 4; k >= 0; --k) {
    p[k] = (double)(rem % g);
    rem /= g;
  }
  lo_rng r;
  lo_rng_init(&r, mix3(sampling_seed, i, 0x9e37ULL));
  for (int k = 0; k < 5; ++k) {
    const double jitter = rng_uniform_range(&r, -0.4, 0.4);
    p[k] = (p[k] + 0.5 + jitter) / g;
  }
}

/* generator.hpp:197-206, samples [first, first+n) of a total_n sweep */
int lo_synth_generate(const lo_synth* g, uint64_t first, uint64_t n,
                      uint64_t total_n, uint64_t sampling_seed, float* x,
                      float* y) {
  const uint32_t gs = lo_grid_side(total_n);
  const size_t out_dim =
      g->dims[2] + (size_t)g->dims[3] * g->dims[4] * g->dims[5] * g->dims[6];
  for (uint64_t i = 0; i < n; ++i) {
    double p[5];
    lo_sweep_point(first + i, gs, sampling_seed, p);
    if (lo_synth_sample(g, p, x + i * 5, y + i * out_dim) != 0) return -1;
  }
  return 0;
}

/* ====================================================================== */
/* nn/ (tensor.hpp, activation.hpp, mlp.hpp, loss.hpp, adam.hpp)           */
/* ====================================================================== */

/* activation.hpp:43-50 (float instantiation: std::exp(float) == expf) */
float lo_stable_sigmoid(float z) {
  if (z >= 0.0f) return 1.0f / (1.0f + expf(-z));
  const float e = expf(z);
  return e / (1.0f + e);
}

/* activation.hpp:52-62 */
static float act_apply(int kind, double slope, float z) {
  switch (kind) {
    case LO_IDENTITY: return z;
    case LO_RELU: return z > 0.0f ? z : 0.0f;
    case LO_LEAKY: return z > 0.0f ? z : (float)slope * z;
    case LO_TANH: return tanhf(z);
    case LO_SIGMOID: return lo_stable_sigmoid(z);
  }
  return z;
}

/* activation.hpp:66-77 */
static float act_deriv(int kind, double slope, float z, float a) {
  switch (kind) {
    case LO_IDENTITY: return 1.0f;
    case LO_RELU: return z > 0.0f ? 1.0f : 0.0f;
    case LO_LEAKY: return z > 0.0f ? 1.0f : (float)slope;
    case LO_TANH: return 1.0f - a * a;
    case LO_SIGMOID: return a * (1.0f - a);
  }
  return 1.0f;
}

/* tensor.hpp:114-123 via the strict shim: c(i,j) = sum_k a(i,k) b(k,j) */
static void mm(const float* a, const float* b, float* c, size_t m, size_t kd,
               size_t n) {
  for (size_t i = 0; i < m * n; ++i) c[i] = 0.0f;
  for (size_t i = 0; i < m; ++i)
    for (size_t k = 0; k < kd; ++k) {
      const float aik = a[i * kd + k];
      const float* brow = b + k * n;
      float* crow = c + i * n;
      for (size_t j = 0; j < n; ++j) crow[j] = crow[j] + aik * brow[j];
    }
}
/* tensor.hpp:125-134: c = a^T b, a is [kd x m], b is [kd x n] */
static void mm_tn(const float* a, const float* b, float* c, size_t kd, size_t m,
                  size_t n) {
  for (size_t i = 0; i < m * n; ++i) c[i] = 0.0f;
  for (size_t i = 0; i < m; ++i)
    for (size_t k = 0; k < kd; ++k) {
      const float aik = a[k * m + i];
      const float* brow = b + k * n;
      float* crow = c + i * n;
      for (size_t j = 0; j < n; ++j) crow[j] = crow[j] + aik * brow[j];
    }
}
/* tensor.hpp:136-145: c = a b^T, a is [m x kd], b is [n x kd] */
static void mm_nt(const float* a, const float* b, float* c, size_t m, size_t kd,
                  size_t n) {
  for (size_t i = 0; i < m * n; ++i) c[i] = 0.0f;
  for (size_t i = 0; i < m; ++i)
    for (size_t k = 0; k < kd; ++k) {
      const float aik = a[i * kd + k];
      float* crow = c + i * n;
      for (size_t j = 0; j < n; ++j) crow[j] = crow[j] + aik * b[j * kd + k];
    }
}

size_t lo_mlp_param_count(const uint32_t* w, int L) {
  size_t n = 0;
  for (int l = 0; l < L; ++l) n += (size_t)w[l] * w[l + 1] + w[l + 1];
  return n;
}

/* mlp.hpp:149-163 (manifest) + :235-244 (init_params) */
void lo_mlp_init(const uint32_t* w, int L, uint64_t seed, float* blob) {
  lo_rng r;
  lo_rng_init(&r, seed);
  size_t off = 0;
  for (int l = 0; l < L; ++l) {
    const double a = sqrt(1.0 / (double)w[l]);
    const size_t nw = (size_t)w[l] * w[l + 1];
    for (size_t i = 0; i < nw; ++i) blob[off + i] = (float)rng_uniform_range(&r, -a, a);
    off += nw;
    for (size_t i = 0; i < w[l + 1]; ++i) blob[off + i] = 0.0f;
    off += w[l + 1];
  }
}

typedef struct {
  int L;
  float** z; /* pre-activations per layer */
  float** a; /* activations per layer */
} tape_t;

/* mlp.hpp:280-298 */
static tape_t mlp_forward_tape(const uint32_t* w, const int32_t* acts,
                               const double* slopes, int L, const float* blob,
                               const float* x, size_t rows) {
  tape_t t;
  t.L = L;
  t.z = (float**)malloc(sizeof(float*) * (size_t)L);
  t.a = (float**)malloc(sizeof(float*) * (size_t)L);
  const float* cur = x;
  size_t off = 0;
  for (int l = 0; l < L; ++l) {
    const size_t in = w[l], out = w[l + 1];
    const float* W = blob + off;
    const float* b = blob + off + in * out;
    off += in * out + out;
    float* z = (float*)malloc(sizeof(float) * rows * out);
    float* a = (float*)malloc(sizeof(float) * rows * out);
    mm(cur, W, z, rows, in, out);
    for (size_t r = 0; r < rows; ++r) /* tensor.hpp:148-156 add_row_vector */
      for (size_t c = 0; c < out; ++c) z[r * out + c] = z[r * out + c] + b[c];
    for (size_t i = 0; i < rows * out; ++i) a[i] = act_apply(acts[l], slopes[l], z[i]);
    t.z[l] = z;
    t.a[l] = a;
    cur = a;
  }
  return t;
}

static void tape_free(tape_t* t) {
  for (int l = 0; l < t->L; ++l) {
    free(t->z[l]);
    free(t->a[l]);
  }
  free(t->z);
  free(t->a);
}

void lo_mlp_forward(const uint32_t* w, const int32_t* acts, const double* slopes,
                    int L, const float* blob, const float* x, size_t rows,
                    float* out) {
  tape_t t = mlp_forward_tape(w, acts, slopes, L, blob, x, rows);
  memcpy(out, t.a[L - 1], sizeof(float) * rows * w[L]);
  tape_free(&t);
}

/* mlp.hpp:325-361 */
static void mlp_backward_tape(const uint32_t* w, const int32_t* acts,
                              const double* slopes, int L, const float* blob,
                              const float* x, const tape_t* t, size_t rows,
                              const float* grad_out, float* param_grad,
                              float* grad_in) {
  size_t* offs = (size_t*)malloc(sizeof(size_t) * (size_t)(L + 1));
  offs[0] = 0;
  for (int l = 0; l < L; ++l) offs[l + 1] = offs[l] + (size_t)w[l] * w[l + 1] + w[l + 1];
  float* g = (float*)malloc(sizeof(float) * rows * w[L]);
  memcpy(g, grad_out, sizeof(float) * rows * w[L]);
  for (int l = L - 1; l >= 0; --l) {
    const size_t in = w[l], out = w[l + 1];
    float* dz = (float*)malloc(sizeof(float) * rows * out);
    for (size_t i = 0; i < rows * out; ++i)
      dz[i] = g[i] * act_deriv(acts[l], slopes[l], t->z[l][i], t->a[l][i]);
    const float* below = l == 0 ? x : t->a[l - 1];
    float* dW = param_grad ? param_grad + offs[l] : NULL;
    if (dW) {
      mm_tn(below, dz, dW, rows, in, out);
      float* db = dW + in * out; /* tensor.hpp:159-165 col_sums */
      for (size_t c = 0; c < out; ++c) db[c] = 0.0f;
      for (size_t r = 0; r < rows; ++r)
        for (size_t c = 0; c < out; ++c) db[c] += dz[r * out + c];
    }
    float* gn = (float*)malloc(sizeof(float) * rows * in);
    mm_nt(dz, blob + offs[l], gn, rows, out, in);
    free(g);
    free(dz);
    g = gn;
  }
  if (grad_in) memcpy(grad_in, g, sizeof(float) * rows * w[0]);
  free(g);
  free(offs);
}

void lo_mlp_backward(const uint32_t* w, const int32_t* acts, const double* slopes,
                     int L, const float* blob, const float* x, size_t rows,
                     const float* grad_out, float* param_grad, float* grad_in) {
  tape_t t = mlp_forward_tape(w, acts, slopes, L, blob, x, rows);
  mlp_backward_tape(w, acts, slopes, L, blob, x, &t, rows, grad_out, param_grad,
                    grad_in);
  tape_free(&t);
}

/* loss.hpp:24-41 */
double lo_mae(const float* pred, const float* target, size_t n, float* grad) {
  const double dn = (double)n;
  double acc = 0;
  for (size_t i = 0; i < n; ++i) {
    const double d = (double)pred[i] - (double)target[i];
    acc += fabs(d);
    if (grad) grad[i] = d > 0 ? (float)(1.0 / dn) : (d < 0 ? (float)(-1.0 / dn) : 0.0f);
  }
  return acc / dn;
}

/* loss.hpp:59-80 (labels are exactly 0 or 1 here) */
double lo_bce(const float* probs, const float* labels, size_t n, float* grad) {
  const double dn = (double)n;
  double acc = 0;
  for (size_t i = 0; i < n; ++i) {
    const double y = (double)labels[i];
    double p = (double)probs[i];
    if (p < 1e-7) p = 1e-7;
    if (p > 1.0 - 1e-7) p = 1.0 - 1e-7;
    acc += y != 0.0 ? -log(p) : -log(1.0 - p);
    if (grad) grad[i] = (float)((p - y) / dn);
  }
  return acc / dn;
}

/* adam.hpp:48-61 + :87-122 */
int lo_adam_step(float* params, const float* grads, float* m, float* v, size_t n,
                 uint64_t* t, double lr, double b1, double b2, double eps) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite((double)grads[i])) return -1;
  *t += 1;
  const double c1 = 1.0 - pow(b1, (double)*t);
  const double c2 = 1.0 - pow(b2, (double)*t);
  for (size_t i = 0; i < n; ++i) {
    const double g = (double)grads[i];
    const double mi = b1 * (double)m[i] + (1.0 - b1) * g;
    const double vi = b2 * (double)v[i] + (1.0 - b2) * g * g;
    m[i] = (float)mi;
    v[i] = (float)vi;
    const double update = lr * (mi / c1) / (sqrt(vi / c2) + eps);
    params[i] = (float)((double)params[i] - update);
  }
  return 0;
}

/* ====================================================================== */
/* surrogate/model.hpp, train_ops.hpp                                      */
/* ====================================================================== */
#define LO_MAXL 16
typedef struct {
  int L;
  uint32_t w[LO_MAXL + 1];
  int32_t act[LO_MAXL];
  double slope[LO_MAXL];
  uint64_t seed;
  size_t count;
  float* blob;
  float* m;
  float* v;
  uint64_t t;
} lo_net;

struct lo_gan {
  uint32_t in_dim, latent, out_dim;
  lo_net net[5];
  float lambda_adv, lambda_cyc;
  double lr, b1, b2, eps;
};

/* model.hpp:76-90 make_spec */
static void make_net(lo_net* n, uint32_t in, uint32_t out, const uint32_t* h,
                     int nh, double slope) {
  memset(n, 0, sizeof(*n));
  n->L = nh + 1;
  n->w[0] = in;
  for (int i = 0; i < nh; ++i) n->w[i + 1] = h[i];
  n->w[nh + 1] = out;
  for (int l = 0; l < n->L; ++l) {
    const int hidden = l + 1 < n->L;
    n->act[l] = hidden ? LO_LEAKY : LO_IDENTITY;
    n->slope[l] = hidden ? slope : 0.01;
  }
  n->count = lo_mlp_param_count(n->w, n->L);
  n->blob = (float*)calloc(n->count, sizeof(float));
  n->m = (float*)calloc(n->count, sizeof(float));
  n->v = (float*)calloc(n->count, sizeof(float));
}

lo_gan* lo_gan_create(uint32_t in, uint32_t latent, uint32_t out,
                      const uint32_t* eh, int ne, const uint32_t* dh, int nd,
                      const uint32_t* fh, int nf, const uint32_t* ih, int ni,
                      const uint32_t* ch, int nc, double slope, double la,
                      double lc, double lr, double b1, double b2, double eps) {
  lo_gan* g = (lo_gan*)calloc(1, sizeof(lo_gan));
  g->in_dim = in;
  g->latent = latent;
  g->out_dim = out;
  make_net(&g->net[LO_ENC], out, latent, eh, ne, slope);
  make_net(&g->net[LO_DEC], latent, out, dh, nd, slope);
  make_net(&g->net[LO_FWD], in, latent, fh, nf, slope);
  make_net(&g->net[LO_INV], latent, in, ih, ni, slope);
  make_net(&g->net[LO_DISC], latent, 1, ch, nc, slope);
  g->lambda_adv = (float)la;
  g->lambda_cyc = (float)lc;
  g->lr = lr;
  g->b1 = b1;
  g->b2 = b2;
  g->eps = eps;
  return g;
}

lo_gan* lo_gan_clone(const lo_gan* src) {
  lo_gan* g = (lo_gan*)malloc(sizeof(lo_gan));
  *g = *src;
  for (int i = 0; i < 5; ++i) {
    const size_t b = sizeof(float) * src->net[i].count;
    g->net[i].blob = (float*)malloc(b);
    g->net[i].m = (float*)malloc(b);
    g->net[i].v = (float*)malloc(b);
    memcpy(g->net[i].blob, src->net[i].blob, b);
    memcpy(g->net[i].m, src->net[i].m, b);
    memcpy(g->net[i].v, src->net[i].v, b);
  }
  return g;
}

void lo_gan_destroy(lo_gan* g) {
  if (!g) return;
  for (int i = 0; i < 5; ++i) {
    free(g->net[i].blob);
    free(g->net[i].m);
    free(g->net[i].v);
  }
  free(g);
}

static void net_init(lo_net* n, uint64_t seed) {
  n->seed = seed;
  lo_mlp_init(n->w, n->L, seed, n->blob);
  memset(n->m, 0, sizeof(float) * n->count);
  memset(n->v, 0, sizeof(float) * n->count);
  n->t = 0;
}

/* model.hpp:96-132 */
void lo_gan_init(lo_gan* g, uint64_t seed) {
  for (int i = 0; i < 5; ++i) net_init(&g->net[i], mix2(seed, (uint64_t)(i + 1)));
}

/* model.hpp:137-147 */
void lo_gan_reinit_gan_nets(lo_gan* g, uint64_t seed) {
  net_init(&g->net[LO_FWD], mix2(seed, 3));
  net_init(&g->net[LO_INV], mix2(seed, 4));
  net_init(&g->net[LO_DISC], mix2(seed, 5));
}

float* lo_gan_blob(lo_gan* g, int net, size_t* count) {
  if (count) *count = g->net[net].count;
  return g->net[net].blob;
}
float* lo_gan_moment(lo_gan* g, int net, int which) {
  return which == 0 ? g->net[net].m : g->net[net].v;
}
uint64_t* lo_gan_t(lo_gan* g, int net) { return &g->net[net].t; }

int lo_gan_adam(lo_gan* g, int net, const float* grads) {
  lo_net* n = &g->net[net];
  return lo_adam_step(n->blob, grads, n->m, n->v, n->count, &n->t, g->lr, g->b1,
                      g->b2, g->eps);
}

static tape_t net_fwd(const lo_net* n, const float* x, size_t rows) {
  return mlp_forward_tape(n->w, n->act, n->slope, n->L, n->blob, x, rows);
}
static float* net_out(const tape_t* t) { return t->a[t->L - 1]; }

/* train_ops.hpp:155-172 discriminator_backward */
double lo_disc_backward(const lo_gan* g, const float* x, const float* y,
                        size_t rows, float* disc_grad) {
  const size_t lat = g->latent;
  tape_t te = net_fwd(&g->net[LO_ENC], y, rows);
  tape_t tf = net_fwd(&g->net[LO_FWD], x, rows);
  float* stacked = (float*)malloc(sizeof(float) * 2 * rows * lat);
  memcpy(stacked, net_out(&te), sizeof(float) * rows * lat);
  memcpy(stacked + rows * lat, net_out(&tf), sizeof(float) * rows * lat);
  tape_t td = net_fwd(&g->net[LO_DISC], stacked, 2 * rows);
  float* probs = (float*)malloc(sizeof(float) * 2 * rows);
  float* labels = (float*)calloc(2 * rows, sizeof(float));
  float* grad = (float*)malloc(sizeof(float) * 2 * rows);
  for (size_t i = 0; i < 2 * rows; ++i) probs[i] = lo_stable_sigmoid(net_out(&td)[i]);
  for (size_t i = 0; i < rows; ++i) labels[i] = 1.0f;
  const double loss = lo_bce(probs, labels, 2 * rows, grad);
  const lo_net* d = &g->net[LO_DISC];
  mlp_backward_tape(d->w, d->act, d->slope, d->L, d->blob, stacked, &td, 2 * rows,
                    grad, disc_grad, NULL);
  tape_free(&te);
  tape_free(&tf);
  tape_free(&td);
  free(stacked);
  free(probs);
  free(labels);
  free(grad);
  return loss;
}

/* train_ops.hpp:88-136 generator_backward */
void lo_gen_backward(const lo_gan* g, const float* x, const float* y,
                     size_t rows, float* fwd_grad, float* inv_grad,
                     double* losses) {
  const size_t lat = g->latent, in = g->in_dim, out = g->out_dim;
  tape_t tf = net_fwd(&g->net[LO_FWD], x, rows);
  const float* latent = net_out(&tf);
  /* forward-prediction path */
  tape_t tdec = net_fwd(&g->net[LO_DEC], latent, rows);
  float* mgrad = (float*)malloc(sizeof(float) * rows * out);
  losses[1] = lo_mae(net_out(&tdec), y, rows * out, mgrad);
  float* grad_latent = (float*)malloc(sizeof(float) * rows * lat);
  const lo_net* dn = &g->net[LO_DEC];
  mlp_backward_tape(dn->w, dn->act, dn->slope, dn->L, dn->blob, latent, &tdec, rows,
                    mgrad, NULL, grad_latent);
  /* adversarial path */
  tape_t tdisc = net_fwd(&g->net[LO_DISC], latent, rows);
  float* probs = (float*)malloc(sizeof(float) * rows);
  float* ones = (float*)malloc(sizeof(float) * rows);
  float* agrad = (float*)malloc(sizeof(float) * rows);
  for (size_t i = 0; i < rows; ++i) {
    probs[i] = lo_stable_sigmoid(net_out(&tdisc)[i]);
    ones[i] = 1.0f;
  }
  losses[2] = lo_bce(probs, ones, rows, agrad);
  for (size_t i = 0; i < rows; ++i) agrad[i] *= g->lambda_adv;
  float* dgi = (float*)malloc(sizeof(float) * rows * lat);
  const lo_net* cn = &g->net[LO_DISC];
  mlp_backward_tape(cn->w, cn->act, cn->slope, cn->L, cn->blob, latent, &tdisc, rows,
                    agrad, NULL, dgi);
  for (size_t i = 0; i < rows * lat; ++i) grad_latent[i] += dgi[i];
  /* cycle path */
  tape_t tinv = net_fwd(&g->net[LO_INV], latent, rows);
  float* cgrad = (float*)malloc(sizeof(float) * rows * in);
  losses[3] = lo_mae(net_out(&tinv), x, rows * in, cgrad);
  for (size_t i = 0; i < rows * in; ++i) cgrad[i] *= g->lambda_cyc;
  float* igi = (float*)malloc(sizeof(float) * rows * lat);
  const lo_net* in_n = &g->net[LO_INV];
  mlp_backward_tape(in_n->w, in_n->act, in_n->slope, in_n->L, in_n->blob, latent, &tinv,
                    rows, cgrad, inv_grad, igi);
  for (size_t i = 0; i < rows * lat; ++i) grad_latent[i] += igi[i];
  const lo_net* fn = &g->net[LO_FWD];
  mlp_backward_tape(fn->w, fn->act, fn->slope, fn->L, fn->blob, x, &tf, rows,
                    grad_latent, fwd_grad, NULL);
  losses[0] = losses[1] + (double)g->lambda_adv * losses[2] +
              (double)g->lambda_cyc * losses[3];
  tape_free(&tf);
  tape_free(&tdec);
  tape_free(&tdisc);
  tape_free(&tinv);
  free(mgrad);
  free(grad_latent);
  free(probs);
  free(ones);
  free(agrad);
  free(dgi);
  free(cgrad);
  free(igi);
}

/* train_ops.hpp:52-66 autoencoder_backward */
double lo_ae_backward(const lo_gan* g, const float* y, size_t rows,
                      float* enc_grad, float* dec_grad) {
  const size_t lat = g->latent, out = g->out_dim;
  tape_t te = net_fwd(&g->net[LO_ENC], y, rows);
  tape_t td = net_fwd(&g->net[LO_DEC], net_out(&te), rows);
  float* mgrad = (float*)malloc(sizeof(float) * rows * out);
  const double loss = lo_mae(net_out(&td), y, rows * out, mgrad);
  float* gl = (float*)malloc(sizeof(float) * rows * lat);
  const lo_net* dn = &g->net[LO_DEC];
  mlp_backward_tape(dn->w, dn->act, dn->slope, dn->L, dn->blob, net_out(&te), &td, rows,
                    mgrad, dec_grad, gl);
  const lo_net* en = &g->net[LO_ENC];
  mlp_backward_tape(en->w, en->act, en->slope, en->L, en->blob, y, &te, rows, gl,
                    enc_grad, NULL);
  tape_free(&te);
  tape_free(&td);
  free(mgrad);
  free(gl);
  return loss;
}

/* train_ops.hpp:191-205 evaluate */
void lo_evaluate(const lo_gan* g, const float* x, const float* y, size_t rows,
                 double w_f, double w_i, double* out3) {
  tape_t tf = net_fwd(&g->net[LO_FWD], x, rows);
  tape_t td = net_fwd(&g->net[LO_DEC], net_out(&tf), rows);
  tape_t ti = net_fwd(&g->net[LO_INV], net_out(&tf), rows);
  out3[0] = lo_mae(net_out(&td), y, rows * g->out_dim, NULL);
  out3[1] = lo_mae(net_out(&ti), x, rows * g->in_dim, NULL);
  out3[2] = w_f * out3[0] + w_i * out3[1];
  tape_free(&tf);
  tape_free(&td);
  tape_free(&ti);
}

/* ====================================================================== */
/* train/trainer.hpp:139-290, single shard, preload, no prefetch            */
/* ====================================================================== */
struct lo_trainer {
  lo_gan* gan;
  const float* ds_x;
  const float* ds_y;
  uint32_t* partition;
  size_t n_part, batch;
  uint64_t seed;
  int abort_threshold;
  uint32_t* perm;
  uint32_t epoch;
  size_t step_in_epoch, n_steps_epoch;
  uint64_t global_step, skipped;
  int have_plan;
};

lo_trainer* lo_trainer_create(const lo_gan* model, const float* ds_x,
                              const float* ds_y, const uint32_t* partition,
                              size_t n_part, size_t batch, uint64_t seed,
                              int abort_threshold) {
  lo_trainer* t = (lo_trainer*)calloc(1, sizeof(lo_trainer));
  t->gan = lo_gan_clone(model);
  t->ds_x = ds_x;
  t->ds_y = ds_y;
  t->partition = (uint32_t*)malloc(sizeof(uint32_t) * n_part);
  memcpy(t->partition, partition, sizeof(uint32_t) * n_part);
  t->perm = (uint32_t*)malloc(sizeof(uint32_t) * n_part);
  t->n_part = n_part;
  t->batch = batch;
  t->seed = seed;
  t->abort_threshold = abort_threshold;
  return t;
}

void lo_trainer_destroy(lo_trainer* t) {
  if (!t) return;
  lo_gan_destroy(t->gan);
  free(t->partition);
  free(t->perm);
  free(t);
}

lo_gan* lo_trainer_gan(lo_trainer* t) { return t->gan; }
uint64_t lo_trainer_step(const lo_trainer* t) { return t->global_step; }

/* train/allreduce.hpp:62-75 weighted_mean over a single shard: the
 * reference still forms (rows * v) / rows in double, which is not always
 * exactly v, so the records carry that rounding. */
static double wmean1(double v, size_t rows) {
  double num = 0, den = 0;
  num += (double)rows * v;
  den += (double)rows;
  return num / den;
}

static int all_finite(const float* v, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite((double)v[i])) return 0;
  return 1;
}

size_t lo_trainer_steps(lo_trainer* t, size_t n, double* rec5, uint8_t* skipped,
                        uint32_t* epoch_out) {
  lo_gan* g = t->gan;
  const size_t in = g->in_dim, out = g->out_dim;
  float* x = (float*)malloc(sizeof(float) * t->batch * in);
  float* y = (float*)malloc(sizeof(float) * t->batch * out);
  for (size_t s = 0; s < n; ++s) {
    if (!t->have_plan || t->step_in_epoch >= t->n_steps_epoch) {
      t->epoch += 1; /* trainer.hpp:139-148 start_epoch */
      lo_plan_perm(t->partition, t->n_part, t->epoch, t->seed, t->perm);
      t->n_steps_epoch = (t->n_part + t->batch - 1) / t->batch;
      t->step_in_epoch = 0;
      t->have_plan = 1;
    }
    const size_t begin = t->step_in_epoch * t->batch;
    const size_t rows = (begin + t->batch <= t->n_part) ? t->batch : t->n_part - begin;
    for (size_t r = 0; r < rows; ++r) { /* epoch_plan.hpp:106-137 */
      const uint32_t id = t->perm[begin + r];
      memcpy(x + r * in, t->ds_x + (size_t)id * in, sizeof(float) * in);
      memcpy(y + r * out, t->ds_y + (size_t)id * out, sizeof(float) * out);
    }
    double rec[5] = {0, 0, 0, 0, 0};
    int skip = 0;
    /* D-step, trainer.hpp:208-229 */
    {
      float* dg = (float*)malloc(sizeof(float) * g->net[LO_DISC].count);
      const double dl = wmean1(lo_disc_backward(g, x, y, rows, dg), rows);
      if (!isfinite(dl) || lo_gan_adam(g, LO_DISC, dg) != 0) skip = 1;
      else rec[0] = dl;
      free(dg);
    }
    /* G-step, trainer.hpp:231-272 */
    if (!skip) {
      float* fg = (float*)malloc(sizeof(float) * g->net[LO_FWD].count);
      float* ig = (float*)malloc(sizeof(float) * g->net[LO_INV].count);
      double losses[4];
      lo_gen_backward(g, x, y, rows, fg, ig, losses);
      for (int i = 0; i < 4; ++i) losses[i] = wmean1(losses[i], rows);
      if (!isfinite(losses[0])) {
        skip = 1;
      } else if (!all_finite(fg, g->net[LO_FWD].count)) {
        skip = 1;
      } else {
        lo_gan_adam(g, LO_FWD, fg);
        if (lo_gan_adam(g, LO_INV, ig) != 0) skip = 1;
        else {
          rec[1] = losses[0];
          rec[2] = losses[1];
          rec[3] = losses[2];
          rec[4] = losses[3];
        }
      }
      free(fg);
      free(ig);
    }
    t->global_step += 1;
    t->step_in_epoch += 1;
    memcpy(rec5 + 5 * s, rec, sizeof(rec));
    skipped[s] = (uint8_t)skip;
    epoch_out[s] = t->epoch;
    if (skip) {
      t->skipped += 1;
      if (t->skipped > (uint64_t)t->abort_threshold) {
        free(x);
        free(y);
        return s + 1;
      }
    }
  }
  free(x);
  free(y);
  return n;
}
