/* TEST INFRASTRUCTURE (oracle) — not product code.
 *
 * Plain-C restatement of the reference's hot path (ltfb, header-only C++ at
 * /root/reference/proj/include/ltfb). It is the CHECKER used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg; the product
 * library never links or calls it. Every function names the reference
 * file:line it restates. GEMM order = the strict Eigen shim
 * (oracle/shim/Eigen/Core): k-ascending fp32 sums, no FMA contraction.
 * Pinned against tests/golden/*.npz (generated from the unmodified reference
 * by oracle/make_golden.py) in tests/test_oracle_golden.py.
 */
#ifndef LTFB_ORACLE_H
#define LTFB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- core/rng.hpp:13-97 ---------------------------------------------- */
typedef struct { uint64_t s[4]; } lo_rng;
uint64_t lo_splitmix64(uint64_t* state);
uint64_t lo_mix_seed(const uint64_t* parts, int n);
void lo_rng_init(lo_rng* r, uint64_t seed);
uint64_t lo_rng_next(lo_rng* r);
double lo_rng_uniform(lo_rng* r);
uint64_t lo_rng_below(lo_rng* r, uint64_t n);
double lo_rng_normal(lo_rng* r);
void lo_shuffle_u32(lo_rng* r, uint32_t* v, size_t n);
void lo_shuffle_i32(lo_rng* r, int32_t* v, size_t n);
/* core/hash.hpp:15-22 */
uint64_t lo_fnv1a64(const void* data, size_t n, uint64_t h);

/* ---- tournament/ltfb.hpp:24-88, runner.hpp:134-169 -------------------- */
int lo_partition(const uint32_t* ids, size_t n, int k, uint64_t seed,
                 uint32_t* out_ids, uint32_t* out_sizes);
int lo_pair_trainers(int k, int round, uint64_t seed, int32_t* pairs,
                     int32_t* bye); /* returns number of pairs */
/* writes validation ids (out_val, n_val), concatenated train parts and
 * tournament parts in trainer order; sizes per trainer. */
int lo_split_dataset(size_t total, int k, double validation_fraction,
                     double tournament_fraction, uint64_t seed,
                     int need_tournament, uint32_t* out_val, size_t* n_val,
                     uint32_t* out_train, uint32_t* train_sizes,
                     uint32_t* out_tour, uint32_t* tour_sizes);
int lo_incoming_wins(double local, double incoming);
/* data/epoch_plan.hpp:59-71 (permutation only) */
void lo_plan_perm(const uint32_t* partition, size_t n, uint32_t epoch,
                  uint64_t seed, uint32_t* perm_out);

/* ---- synth/generator.hpp:29-206 ------------------------------------- */
typedef struct lo_synth lo_synth;
/* dims7 = {input, latent, scalar, views, channels, h, w} */
lo_synth* lo_synth_create(const uint32_t* dims7, uint64_t spec_seed,
                          double noise_level);
void lo_synth_destroy(lo_synth* g);
int lo_synth_sample(const lo_synth* g, const double* p5, float* inputs,
                    float* outputs);
uint32_t lo_grid_side(uint64_t n);
void lo_sweep_point(uint64_t i, uint32_t g, uint64_t sampling_seed,
                    double* p5);
int lo_synth_generate(const lo_synth* g, uint64_t first, uint64_t n,
                      uint64_t total_n, uint64_t sampling_seed, float* x,
                      float* y);

/* ---- nn/*.hpp --------------------------------------------------------- */
enum { LO_IDENTITY = 0, LO_RELU = 1, LO_LEAKY = 2, LO_TANH = 3, LO_SIGMOID = 4 };
size_t lo_mlp_param_count(const uint32_t* widths, int n_layers);
void lo_mlp_init(const uint32_t* widths, int n_layers, uint64_t seed,
                 float* blob);
void lo_mlp_forward(const uint32_t* widths, const int32_t* acts,
                    const double* slopes, int n_layers, const float* blob,
                    const float* x, size_t rows, float* out);
void lo_mlp_backward(const uint32_t* widths, const int32_t* acts,
                     const double* slopes, int n_layers, const float* blob,
                     const float* x, size_t rows, const float* grad_out,
                     float* param_grad, float* grad_in);
double lo_mae(const float* pred, const float* target, size_t n, float* grad);
double lo_bce(const float* probs, const float* labels, size_t n, float* grad);
float lo_stable_sigmoid(float z);
/* adam.hpp:87-122; returns -1 (nothing applied) on a non-finite gradient */
int lo_adam_step(float* params, const float* grads, float* m, float* v,
                 size_t n, uint64_t* t, double lr, double beta1, double beta2,
                 double eps);

/* ---- surrogate/model.hpp + train_ops.hpp ------------------------------ */
typedef struct lo_gan lo_gan;
enum { LO_ENC = 0, LO_DEC = 1, LO_FWD = 2, LO_INV = 3, LO_DISC = 4 };
/* hidden_* arrays are the SurrogateArch widths (model.hpp:19-23). */
lo_gan* lo_gan_create(uint32_t input_dim, uint32_t latent_dim,
                      uint32_t output_dim, const uint32_t* enc_h, int n_enc,
                      const uint32_t* dec_h, int n_dec, const uint32_t* fwd_h,
                      int n_fwd, const uint32_t* inv_h, int n_inv,
                      const uint32_t* disc_h, int n_disc, double slope,
                      double lambda_adv, double lambda_cyc, double lr,
                      double beta1, double beta2, double eps);
lo_gan* lo_gan_clone(const lo_gan* g);
void lo_gan_destroy(lo_gan* g);
void lo_gan_init(lo_gan* g, uint64_t seed);           /* make_cyclegan */
void lo_gan_reinit_gan_nets(lo_gan* g, uint64_t seed); /* reinit_gan_nets */
float* lo_gan_blob(lo_gan* g, int net, size_t* count);
float* lo_gan_moment(lo_gan* g, int net, int which /*0 m,1 v*/);
uint64_t* lo_gan_t(lo_gan* g, int net);
int lo_gan_adam(lo_gan* g, int net, const float* grads);
double lo_disc_backward(const lo_gan* g, const float* x, const float* y,
                        size_t rows, float* disc_grad);
void lo_gen_backward(const lo_gan* g, const float* x, const float* y,
                     size_t rows, float* fwd_grad, float* inv_grad,
                     double* losses4 /* total, fwd, adv, cyc */);
double lo_ae_backward(const lo_gan* g, const float* y, size_t rows,
                      float* enc_grad, float* dec_grad);
void lo_evaluate(const lo_gan* g, const float* x, const float* y, size_t rows,
                 double w_f, double w_i, double* out3);

/* ---- train/trainer.hpp:190-290 (single shard, preload) ---------------- */
typedef struct lo_trainer lo_trainer;
/* ds_x/ds_y are indexed by global sample id (row stride input/output dim).
 * The trainer copies the model. */
lo_trainer* lo_trainer_create(const lo_gan* model, const float* ds_x,
                              const float* ds_y, const uint32_t* partition,
                              size_t n_part, size_t batch, uint64_t seed,
                              int abort_threshold);
void lo_trainer_destroy(lo_trainer* t);
/* Runs n steps; per step writes 5 doubles (d, g_total, g_fwd, g_adv, g_cyc),
 * skipped flag and epoch. Returns the number of steps recorded; a value < n
 * means the abort threshold was exceeded at the last recorded step. */
size_t lo_trainer_steps(lo_trainer* t, size_t n, double* rec5,
                        uint8_t* skipped, uint32_t* epoch);
lo_gan* lo_trainer_gan(lo_trainer* t);
uint64_t lo_trainer_step(const lo_trainer* t);

#ifdef __cplusplus
}
#endif
#endif
