// Kernel argument blocks. Passed by value (one constant-bank copy per launch),
// they carry every device pointer a kernel touches so a captured CUDA graph
// of one training step can be replayed without re-binding.
#pragma once

#include "device_common.cuh"

namespace ltfb_dev {

struct ModelArgs {
  int in, lat, out, out_pad;  // input_dim, latent_dim, output_dim, padded row
  int E1;                     // enc wide-layer width (enc layer 0: out -> E1)
  int D;                      // dec wide-layer input width (dec last: D -> out)
  int enc_act0;               // activation of enc layer 0
  float enc_slope0;
  long long enc_wide_w, enc_wide_b;  // offsets inside the enc blob
  long long dec_wide_w, dec_wide_b;  // offsets inside the dec blob
  NetDesc enc_tail;  // enc layers 1.. (E1 -> ... -> lat); L may be 0
  NetDesc dec_head;  // dec layers 0..L-2 (lat -> ... -> D); L may be 0
  NetDesc fwd, inv, disc;
  float lambda_adv, lambda_cyc;
};

/// Offsets (in floats) of the small-network scratch regions; computed once
/// on the host (scratch_layout.cuh) and carried in StepArgs.
struct ScratchLayout {
  long long fz[kMaxLayers], fa[kMaxLayers];  // fwd tape         [B x w]
  long long hz[kMaxLayers], ha[kMaxLayers];  // dec-head tape    [B x w]
  long long ez[kMaxLayers], ea[kMaxLayers];  // enc-tail outputs [B x w]
  long long cz[kMaxLayers], ca[kMaxLayers];  // disc tape        [2B x w]
  long long iz[kMaxLayers], ia[kMaxLayers];  // inv tape         [B x w]
  long long e1z, e1a;                        // enc wide layer   [B x E1]
  long long stacked;                         // [2B x lat]
  long long probs, bgrad;                    // [2B]
  long long gh;                              // [B x D]
  long long gl_dec, gl_disc, gl_inv, gl;     // [B x lat]
  long long igrad;                           // [B x in]
  long long tA, tB;                          // per post CTA: [2 ceil(B/C) x maxw]
  long long tstride;                         // floats per post CTA in tA / tB
  long long red_enc, red_dec;                // reduced wide-pass sums [B x E1], [B x D]
  long long pg_disc, pg_fwd, pg_inv;         // per post CTA partial gradients
  long long total;
};

constexpr int kPostCluster = 8;   // CTAs of the post kernel (one cluster)
constexpr int kPostThreads = 256;

struct StepArgs {
  ModelArgs m;
  int B;            // configured batch size
  int n_part;       // partition size (slots in the store)
  int S;            // split count of the wide pass (partials)
  int abort_threshold;
  int rec_cap;
  int h_in_gather;  // 1: k_gather's last CTA column computes h = dec_head(fwd(x)) per row
  int y_identity;   // wide pass: minibatch row r is row r of the y map (host-streamed buffer)
  int x_from_store; // 1: that h computation reads x through the epoch plan, 0: from xb
  int post_next_h;  // 1: the small-network post kernel also computes h / xb of the next step (store path)
  int phase_prof;   // debug: per-phase clock64 stamps printed by the post kernel (LTFB_PHASE_PROF)
  int small_ctas;   // CTAs of the small-network kernels
  double lr[5], b1, b2, eps;
  long long adam_cap;  // entries of the bias-correction table
  // parameters / optimizer state (blob layout), gradient scratch
  float* p[5];
  float* mom1[5];
  float* mom2[5];
  float* g[5];
  // W^T images of fwd / inv / disc / dec-head ([out x (in + 1)] per layer,
  // layers concatenated) for the small-network post kernel; by NetId, kDec =
  // the dec head. Rebuilt by k_build_T when parameters change from outside a
  // step, kept current by the post kernel's Adam owners.
  float* pT[5];
  // HBM-resident data store and the epoch plan (two buffers, epoch parity)
  const float* sx;
  const float* sy;
  const unsigned* perm[2];
  // minibatch and wide-pass intermediates
  float* xb;
  float* yb;
  float* h;         // [B x D] dec-head output, input of the wide pass
  float* P_enc;     // [S x B x E1]
  float* P_dec;     // [S x B x D]
  double* mae_part; // [S]
  double* mae_total; // [1] reduced forward-MAE sum
  float* scratch;   // small-network tapes
  ScratchLayout L;  // offsets into scratch
  Counters* ctr;
  unsigned* grid_bar;  // [2] arrival count, generation (cooperative wide pass)
  StepRec* rec;
  const double* adam_c;  // [cap x 2]: 1-b1^t, 1-b2^t (host std::pow)
};

/// Hand-offs of the streamed step (DeviceTrainer stream mode) between the
/// persistent wide kernel (k_wide_ps) and the persistent post cluster
/// (k_post_loop). Reset by k_stream_init at the start of every run; the
/// counters only grow inside a run.
struct StepSync {
  unsigned long long enc_done;  // wide CTAs done reducing P_enc (+S per step)
  unsigned long long dec_done;  // wide CTAs done reducing P_dec and the MAE (+S per step)
  unsigned long long h_done;    // post D/G CTAs that wrote the next step's h / x rows (+kStreamSignalers per step)
  int abort;                    // post: numeric abort, the run stops
  int error;                    // a wait timed out (never expected): the run stops, the host raises
  int resident;                 // post: the cluster of run `run_id` is resident
  int err_site;                 // which wait timed out first (diagnostics)
  unsigned long long t_post0, t_wide0;  // %globaltimer at the start of each kernel of the run (diagnostics)
};
/// CTAs of the post cluster that signal h_done (the D/G half, one row block each).
constexpr int kStreamSignalers = 8;

/// One run of the streamed step: n steps inside one epoch.
struct StreamArgs {
  int n;         // steps in the run
  int sie0;      // step_in_epoch of the run's first step
  unsigned epoch;
  int run_id;
  int S_wide;    // CTAs of the persistent wide kernel (split count of the partials)
  StepSync* sync;
  int* resident_host;  // mapped pinned int: the host waits for the post cluster before launching the wide pass
  float* red_enc[2];   // reduced wide-pass sums per step parity [B x E1] / [B x D]
  float* red_dec[2];
  double* mae_total[2];
  unsigned long long* prof;  // LTFB_STREAM_PROF: [n x 16] %globaltimer stamps per step, else null
  int tile_rot;              // k_wide2: CTA c owns the column tiles of index (c + tile_rot) % S
  int tile_donate;           // k_wide2: tiles each of the two slow-placed owners hands to other short owners
};

/// Candidate evaluation (train_ops.hpp:191-205) over a resident slice.
struct EvalArgs {
  ModelArgs m;
  int rows;         // slice rows
  int nc;           // candidates (1 or 2)
  int S;
  const float* x;   // [rows x in]
  const float* y;   // [rows x out_pad]
  const float* enc; // frozen enc/dec blobs
  const float* dec;
  const float* cf[2];  // candidate fwd blobs
  const float* ci[2];  // candidate inv blobs
  float* h;            // [nc x rows x D]
  double* inv_row;     // [nc x rows]
  double* part;        // [S x nc]
  double* out;         // [nc x 3]
  double w_f, w_i;
  // decision + adoption (tournament/ltfb.hpp:135-147, trainer.hpp:117-127)
  int decide;
  float* dst_fwd; float* dst_inv;
  float* m_fwd; float* v_fwd; float* m_inv; float* v_inv;
  long long n_fwd, n_inv;
  Counters* ctr;
};

}  // namespace ltfb_dev
