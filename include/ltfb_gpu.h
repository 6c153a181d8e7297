/* ltfb_gpu.h — C ABI of the B200-native LTFB hot path (libltfb_gpu.so).
 *
 * The reference (/root/reference/proj, header-only C++20) has no plugin or
 * FFI layer: its "interface" is the C++ API of train::Trainer,
 * tournament::tournament_round and the surrogate::* step functions. This
 * header is the flat C boundary under that API: plain pointers and sizes,
 * opaque handles, int status codes; no C++ or torch types. The C++ drop-in
 * façade (include/ltfb_b200/*.hpp) and the Python package both sit on it.
 *
 * Each entry point names the reference interface it replaces
 * (file:line under /root/reference/proj/include/ltfb).
 *
 * Errors: every function returns LTFB_OK or one LTFB_E* code mapping 1:1
 * onto the reference exception taxonomy (core/error.hpp:11-58);
 * ltfb_last_error() returns the message (thread-local). LTFB_ENUMERIC keeps
 * the reference meaning: the offending update was not applied.
 *
 * Networks are indexed LTFB_NET_ENC..LTFB_NET_DISC; a network crosses the
 * ABI as one float32 blob in the reference manifest order
 * (nn/mlp.hpp:63-84: W0, b0, W1, b1, ... with row-major [in x out] W).
 */
#ifndef LTFB_GPU_H
#define LTFB_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LTFB_ABI_VERSION 1

enum {
  LTFB_OK = 0,
  LTFB_EDIMENSION = 1,    /* DimensionError */
  LTFB_ECONTRACT = 2,     /* ContractError */
  LTFB_ENUMERIC = 3,      /* NumericError */
  LTFB_EIO = 4,           /* IoError */
  LTFB_ECAPACITY = 5,     /* CapacityError */
  LTFB_ESTORECORRUPT = 6, /* StoreCorruptError */
  LTFB_ECONFIG = 7,       /* ConfigError */
  LTFB_ECUDA = 8,         /* device / driver failure (no reference analogue) */
  LTFB_EINTERNAL = 9
};

enum { LTFB_NET_ENC = 0, LTFB_NET_DEC = 1, LTFB_NET_FWD = 2, LTFB_NET_INV = 3, LTFB_NET_DISC = 4 };
enum { LTFB_ACT_IDENTITY = 0, LTFB_ACT_RELU = 1, LTFB_ACT_LEAKY_RELU = 2, LTFB_ACT_TANH = 3,
       LTFB_ACT_SIGMOID = 4 };
enum { LTFB_SLICE_TOURNAMENT = 0, LTFB_SLICE_VALIDATION = 1 };

/* surrogate/dims.hpp:15-53 */
typedef struct {
  uint32_t input_dim, latent_dim, scalar_dim, image_views, image_channels, image_h, image_w;
} ltfb_dims;

/* surrogate/model.hpp:18-30 (hidden widths per network, <= 8 each) */
typedef struct {
  uint32_t enc_hidden[8], dec_hidden[8], fwd_hidden[8], inv_hidden[8], disc_hidden[8];
  uint32_t n_enc_hidden, n_dec_hidden, n_fwd_hidden, n_inv_hidden, n_disc_hidden;
  int32_t hidden_act; /* LTFB_ACT_* */
  double hidden_slope;
  double lambda_adv, lambda_cyc;
  double lr, beta1, beta2, eps; /* nn/adam.hpp:15-22 */
} ltfb_arch;

/* train/trainer.hpp:26-39 (+ device placement) */
typedef struct {
  int32_t trainer_id;
  int32_t device;        /* CUDA ordinal */
  int32_t n_shards;
  int32_t numeric_abort_threshold;
  uint64_t batch_size;
  uint64_t seed;         /* epoch-plan seed */
  double w_f, w_i;
  double lr_fwd, lr_inv, lr_disc; /* 0 = arch.lr (runner.hpp:286-293 lr_jitter) */
  int32_t wide_kernel;   /* 0 auto, 1 generic SIMT, 2 tcgen05 3xTF32 (fp32 parity),
                            3 tcgen05 1xTF32 (perf mode); 2/3 error if unsupported */
  int32_t post_kernel;   /* 0 auto, 1 generic cluster kernel, 2 shared-memory fast path,
                            3 compile-time-shaped kernel (2/3 error if unsupported) */
} ltfb_trainer_config;

/* train/history.hpp:20-30 */
typedef struct {
  uint64_t step;
  uint32_t epoch;
  uint32_t skipped;
  double d_loss, g_total, g_fwd, g_adv, g_cyc;
} ltfb_step_record;

/* train/history.hpp:38-46 */
typedef struct {
  uint32_t epoch;
  uint32_t partial;
  uint64_t steps, samples_shuffled;
  double seconds;
} ltfb_epoch_record;

/* surrogate/train_ops.hpp:20-24 */
typedef struct {
  double forward_mae, inverse_mae, combined;
} ltfb_eval_metric;

typedef struct ltfb_trainer ltfb_trainer;
typedef struct ltfb_comm ltfb_comm;
typedef struct ltfb_dataset ltfb_dataset; /* DatasetIndex over LBDS bundle files */

const char* ltfb_last_error(void);
int ltfb_abi_version(void);
int ltfb_device_count(int* count);

/* Fills *arch with SurrogateArch{} defaults (model.hpp:18-30). */
void ltfb_arch_defaults(ltfb_arch* arch);

/* ---- trainer lifecycle: replaces train::Trainer(TrainerConfig,
 *      DatasetIndex, CycleGan<float>) (trainer.hpp:43-79) ---------------- */
int ltfb_trainer_create(const ltfb_dims* dims, const ltfb_arch* arch,
                        const ltfb_trainer_config* cfg, ltfb_trainer** out);
int ltfb_trainer_destroy(ltfb_trainer* t);
int ltfb_trainer_param_count(const ltfb_trainer* t, int net, uint64_t* count);

/* CycleGan blobs (model.hpp:36-73) <-> HBM. */
int ltfb_trainer_set_params(ltfb_trainer* t, int net, const float* blob, uint64_t count);
int ltfb_trainer_get_params(ltfb_trainer* t, int net, float* blob, uint64_t count);
/* AdamState (adam.hpp:25-47); m/v may be NULL (left unchanged / not read). */
int ltfb_trainer_set_adam(ltfb_trainer* t, int net, const float* m, const float* v, uint64_t step);
int ltfb_trainer_get_adam(ltfb_trainer* t, int net, float* m, float* v, uint64_t* step);

/* DataStore::preload (store.hpp:100-135) into HBM: slot i holds sample
 * ids[i]; x is [n x input_dim], y is [n x output_dim], row-major f32.
 * owner (optional, may be NULL) is the owning shard per slot. */
int ltfb_trainer_load_store(ltfb_trainer* t, const uint32_t* ids, uint64_t n, const float* x,
                            const float* y, const int32_t* owner);
/* ltfb_trainer_load_store with the partition rendered on the device by the
 * synthetic generator (generator.hpp:41-206; sample ids[i] of a total_n-point
 * sweep, noise_level must be 0) instead of uploaded: a large partition never
 * exists on the host. Outputs within 1 fp32 ulp of ltfb_synth_generate_ids. */
int ltfb_trainer_generate_store(ltfb_trainer* t, const uint32_t* ids, uint64_t n, const int32_t* owner,
                                uint64_t spec_seed, double noise_level, uint64_t sampling_seed,
                                uint64_t total_n);
/* ltfb_trainer_set_slice with the slice rendered on the device. */
int ltfb_trainer_generate_slice(ltfb_trainer* t, int which, const uint32_t* ids, uint64_t rows,
                                uint64_t spec_seed, double noise_level, uint64_t sampling_seed,
                                uint64_t total_n);
/* assemble_tensors of the tournament / validation slice (trainer.hpp:74-78,
 * runner.hpp:318) made resident in HBM. */
int ltfb_trainer_set_slice(ltfb_trainer* t, int which, const float* x, const float* y, uint64_t rows);

/* Trainer::train_steps (trainer.hpp:102-104, 190-290). Writes one record
 * per executed step to out (capacity n) and the count to *n_out. Returns
 * LTFB_ENUMERIC when the skip threshold was exceeded (trainer.hpp:283-289);
 * the records up to and including the aborting step are still written. */
int ltfb_trainer_train_steps(ltfb_trainer* t, uint64_t n, ltfb_step_record* out, uint64_t* n_out);
int ltfb_trainer_step(const ltfb_trainer* t, uint64_t* step);
/* Closed epoch records (epochs >= 1) since the last call; *n_out <= cap. */
int ltfb_trainer_take_epochs(ltfb_trainer* t, ltfb_epoch_record* out, uint64_t cap, uint64_t* n_out);
/* Trainer::flush_epoch_record (trainer.hpp:129-134). */
int ltfb_trainer_flush_epoch(ltfb_trainer* t);

/* surrogate::evaluate (train_ops.hpp:191-205) on a resident slice. NULL
 * candidate blobs mean the trainer's own fwd/inv (eval_tournament(model()),
 * trainer.hpp:106-112). */
int ltfb_trainer_evaluate(ltfb_trainer* t, int which, const float* cand_fwd, const float* cand_inv,
                          double w_f, double w_i, ltfb_eval_metric* out);

/* ---- tournament (tournament/ltfb.hpp:96-164) --------------------------- */
/* Size in floats of the generator payload fwd||inv (15,204 B default). */
int ltfb_trainer_generator_floats(const ltfb_trainer* t, uint64_t* n);
/* Own fwd||inv blob to host (TransferRecord hashes, ltfb.hpp:118-131). */
int ltfb_trainer_get_generator(ltfb_trainer* t, float* dst, uint64_t n);
/* Incoming candidate from host memory. */
int ltfb_trainer_set_incoming(ltfb_trainer* t, const float* fwd, const float* inv);
/* Incoming candidate = another in-process trainer's current generator
 * (device-to-device / peer copy; the payload capture of ltfb.hpp:118-131). */
int ltfb_trainer_copy_incoming(ltfb_trainer* dst, ltfb_trainer* src);
/* Evaluate local vs incoming on the tournament slice in one pass, decide
 * with incoming_wins (ltfb.hpp:82-88) IN A DEVICE KERNEL and, if the
 * incoming generator wins, adopt it on the device: copy fwd/inv, zero their
 * Adam moments, keep t (trainer.hpp:117-127). */
int ltfb_trainer_tournament_decide(ltfb_trainer* t, ltfb_eval_metric* local,
                                   ltfb_eval_metric* incoming, int32_t* adopted);
/* Trainer::adopt_generators from host blobs. */
int ltfb_trainer_adopt(ltfb_trainer* t, const float* fwd, const float* inv);

/* ---- autoencoder pre-training (train_ops.hpp:52-81, runner.hpp:249-279) -- */
/* The AE batch source (the sorted union of the training ids, runner.hpp:
 * 251-256): y [n x output_dim], made resident in HBM. */
int ltfb_trainer_load_ae_source(ltfb_trainer* t, const float* y, uint64_t n);
/* surrogate::autoencoder_step (train_ops.hpp:71-81) on source rows
 * idx[0..n): MAE(dec(enc(y)), y), every enc/dec gradient, Adam(enc) then
 * Adam(dec). LTFB_ENUMERIC as the reference: a non-finite loss or enc
 * gradient changes nothing, a non-finite dec gradient leaves enc applied. */
int ltfb_trainer_ae_step(ltfb_trainer* t, const uint32_t* idx, uint64_t n, double* loss);
/* Distributed AE pre-training (runner.hpp:249-279 with the union of the
   training partitions sharded over the ranks' HBM stores, BASELINE config C5):
   a zeroed AE source of `rows` rows; this trainer's store rows (by slot)
   into source rows [dst_row, dst_row + n); ltfb_trainer_ae_allgather then
   assembles every rank's rows (in place, NCCL all-gather on the trainer's
   stream) and ltfb_trainer_ae_step runs on the assembled batch. */
int ltfb_trainer_ae_alloc_source(ltfb_trainer* t, uint64_t rows);
int ltfb_trainer_ae_fill_from_store(ltfb_trainer* t, const uint32_t* slots, uint64_t n, uint64_t dst_row);
/* The runner's AE batch draws (runner.hpp:257-266): steps x batch row
 * indices from Rng(mix_seed({seed, 0xae1})).below(rows), step-major. */
int ltfb_ae_batch_rows(uint64_t seed, uint64_t rows, uint64_t batch, uint64_t steps, uint32_t* out);

/* ---- measurement hooks (bench.py) ------------------------------------- */
/* Host-buffer variant of train_steps (the e2e path): the minibatches of the
 * n steps come from HOST memory, x [n x batch x input_dim] and
 * y [n x batch x output_dim] (pinned for full PCIe rate); every step's batch
 * is copied H2D inside the call (double-buffered on a copy stream that
 * overlaps the previous step's kernels) and its record is read back D2H. */
int ltfb_trainer_train_steps_host(ltfb_trainer* t, uint64_t n, const float* x, const float* y,
                                  ltfb_step_record* out, uint64_t* n_out);
/* Blocks until every kernel / copy queued on the trainer's stream is done. */
int ltfb_trainer_synchronize(ltfb_trainer* t);
/* Captures the CUDA graphs of the step loop (runs of 2..32 steps) without
 * executing them, so that no graph capture lands inside a timed region. */
int ltfb_trainer_prepare_graphs(ltfb_trainer* t);
/* CUDA-event timer on the trainer's stream. */
int ltfb_trainer_timer_start(ltfb_trainer* t);
int ltfb_trainer_timer_stop(ltfb_trainer* t, double* ms);
/* Per-kernel CUDA-event timing inside train_steps (0 gather, 1 small
 * forward, 2 wide pass, 3 post/optimizer). on=1 resets the counters. */
int ltfb_trainer_kernel_timing(ltfb_trainer* t, int on);
int ltfb_trainer_kernel_time(ltfb_trainer* t, int which, double* ms, uint64_t* launches);
/* Which wide-pass kernel is active (1 generic SIMT, 2 tcgen05) and its grid. */
int ltfb_trainer_wide_info(const ltfb_trainer* t, int32_t* kind, int32_t* ctas);
/* Column-tile width of the tcgen05 wide pass: 64 (k_wide2, both step modes)
 * or 32 (k_wide_ps / k_wide_tc); 0 for the generic SIMT pass. */
int ltfb_trainer_wide_tile(const ltfb_trainer* t, int32_t* cols);
/* which kernel evaluates slice `which` (0 tournament, 1 validation): 2 tcgen05 k_eval_tc, 1 SIMT */
int ltfb_trainer_eval_info(const ltfb_trainer* t, int which, int32_t* kind);
/* which column passes ltfb_trainer_ae_step runs for `rows` batch rows:
   2 tcgen05 (k_ae_tc.cu), 1 SIMT (k_ae.cu) */
int ltfb_trainer_ae_info(const ltfb_trainer* t, int32_t rows, int32_t* kind);
/* 1: store-path steps run as the streamed step (a persistent two-phase wide
   pass beside a persistent post cluster per run of steps), 0: launched steps */
int ltfb_trainer_stream_info(const ltfb_trainer* t, int32_t* on);
/* arm != 0: stamp the next streamed run (%globaltimer per stage);
   arm == 0: its stage averages in µs (up to 8): step, phase 1, h -> phase 2
   reduced, phase-2 tiles, phase-2 barrier + reduction, D-step (overlapped),
   post chain after the dec half, number of steps averaged. */
int ltfb_trainer_stream_profile(ltfb_trainer* t, int arm, double* out, int n);
/* Number of kernels this trainer has launched so far (all of them ours). */
int ltfb_trainer_launch_count(const ltfb_trainer* t, uint64_t* launches);

/* Diagnostic: runs the three tcgen05 MMA shapes of the wide pass on the
 * current device (host buffers): a1 [128x32], b1 [32x64], ah [128x64],
 * b2 [64x32], a3 [128x32] -> d1 = a1 b1 [128x64], d2 = ah b2 [128x32],
 * d3 = a3 b2^T [128x64] (kind::tf32 inputs, f32 accumulation). */
int ltfb_selftest_tcgen05(const float* a1, const float* b1, const float* ah, const float* b2, const float* a3,
                          float* d1, float* d2, float* d3);

/* ---- multi-GPU: one trainer per GPU, NCCL point-to-point exchange ------- */
/* nn/adam.hpp:87-122 adam_step_blob: one bias-corrected Adam step over a flat
   blob of n floats (host buffers, updated in place; *t advanced), computed by
   the device Adam kernel every trainer uses (AE K7; the post kernel's owners
   share its element routine). LTFB_ENUMERIC, nothing changed, if a gradient
   component is not finite (adam.hpp:95-102). */
int ltfb_adam_step(float* p, float* m, float* v, const float* g, uint64_t n, uint64_t* t, double lr,
                   double beta1, double beta2, double eps, int device);
int ltfb_nccl_available(void);
int ltfb_nccl_unique_id(uint8_t id[128]);
int ltfb_comm_create(const uint8_t id[128], int nranks, int rank, int device, ltfb_comm** out);
int ltfb_comm_destroy(ltfb_comm* c);
/* Pairwise generator swap with `peer`: ncclSend(own fwd||inv) +
 * ncclRecv(peer's into the incoming buffer) in one group on the trainer's
 * stream (replaces the in-process value copy of ltfb.hpp:118-131). */
int ltfb_trainer_exchange(ltfb_trainer* t, ltfb_comm* c, int peer);
/* Broadcast a network blob from `root` (AE broadcast, runner.hpp:285). */
int ltfb_trainer_broadcast(ltfb_trainer* t, ltfb_comm* c, int net, int root);
/* In-place all-gather of the AE source: rank r contributes rows
   [r * rows_per_rank, (r + 1) * rows_per_rank). */
int ltfb_trainer_ae_allgather(ltfb_trainer* t, ltfb_comm* c, uint64_t rows_per_rank);

/* ---- host algorithms of the path (bit-exact, product implementations) -- */
uint64_t ltfb_mix_seed(const uint64_t* words, int n);                        /* rng.hpp:23-30 */
uint64_t ltfb_fnv1a64(const void* bytes, uint64_t n);                        /* hash.hpp:15-22 */
int ltfb_pair_trainers(int k, int round, uint64_t seed, int32_t* pairs, int32_t* bye,
                       int32_t* n_pairs);                                     /* ltfb.hpp:52-66 */
int ltfb_partition_dataset(const uint32_t* ids, uint64_t n, int k, uint64_t seed,
                           uint32_t* out_ids, uint32_t* sizes);               /* ltfb.hpp:24-43 */
int ltfb_split_dataset(uint64_t total, int k, double validation_fraction,
                       double tournament_fraction, uint64_t seed, int need_tournament,
                       uint32_t* val, uint64_t* n_val, uint32_t* train, uint32_t* train_sizes,
                       uint32_t* tour, uint32_t* tour_sizes);                 /* runner.hpp:134-169 */
int ltfb_epoch_permutation(const uint32_t* partition, uint64_t n, uint32_t epoch, uint64_t seed,
                           uint32_t* out);                                    /* epoch_plan.hpp:59-89 */
int ltfb_incoming_wins(double local, double incoming);                       /* ltfb.hpp:82-88 */
/* generate_dataset rows [first, first+n) of a total_n sweep (generator.hpp:195-206) */
int ltfb_synth_generate(const ltfb_dims* dims, uint64_t spec_seed, double noise_level,
                        uint64_t first, uint64_t n, uint64_t total_n, uint64_t sampling_seed,
                        float* x, float* y, int threads);
/* the samples with global ids `ids` of a total_n sweep, in ids order */
int ltfb_synth_generate_ids(const ltfb_dims* dims, uint64_t spec_seed, double noise_level,
                            const uint32_t* ids, uint64_t n, uint64_t total_n, uint64_t sampling_seed,
                            float* x, float* y, int threads);
/* ltfb_synth_generate_ids on the device: x_dev [n x 5] and y_dev [n x
 * y_stride] are device pointers on `device` (ids may be NULL: rows first..);
 * returns after the rows are written. */
int ltfb_synth_generate_device(const ltfb_dims* dims, uint64_t spec_seed, double noise_level,
                               const uint32_t* ids, uint64_t first, uint64_t n, uint64_t total_n,
                               uint64_t sampling_seed, float* x_dev, float* y_dev, uint64_t y_stride,
                               int device);
/* ---- LBDS bundle datasets (data/bundle.hpp:25-224, runner.hpp:203-230) ----
 * The on-disk dataset the reference trains from: sorted bundle_*.lbds files
 * (40-byte header + records inputs[5] || outputs[out], f32 LE). */
/* DatasetIndex::scan_dir: every *.lbds under dir, sorted by name. */
int ltfb_dataset_open(const char* dir, ltfb_dataset** out);
int ltfb_dataset_destroy(ltfb_dataset* d);
int ltfb_dataset_info(const ltfb_dataset* d, ltfb_dims* dims, uint64_t* total, uint64_t* n_files);
/* bundle file index of each id (DatasetIndex::locate). */
int ltfb_dataset_file_of(const ltfb_dataset* d, const uint32_t* ids, uint64_t n, uint32_t* file_idx);
/* assemble_tensors / read_records: rows ids[i] into x [n x 5] and y
 * [n x output_dim]; *files_opened = distinct files opened (may be NULL). */
int ltfb_dataset_read(const ltfb_dataset* d, const uint32_t* ids, uint64_t n, float* x, float* y,
                      uint64_t* files_opened);
/* ensure_dataset's generation branch: generate_dataset(gen_n) and
 * write_bundles(samples_per_file) into dir (bundle_00000.lbds, ...). */
int ltfb_write_synth_bundles(const char* dir, const ltfb_dims* dims, uint64_t spec_seed, double noise_level,
                             uint64_t gen_n, uint64_t sampling_seed, uint32_t samples_per_file, int threads);
/* make_cyclegan blob init (model.hpp:96-132, mlp.hpp:235-244) */
int ltfb_init_params(const ltfb_dims* dims, const ltfb_arch* arch, uint64_t seed, int net,
                     float* blob, uint64_t count);
int ltfb_net_param_count(const ltfb_dims* dims, const ltfb_arch* arch, int net, uint64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* LTFB_GPU_H */
