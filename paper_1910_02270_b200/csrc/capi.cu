#include <cmath>
// C ABI (include/ltfb_gpu.h) over DeviceTrainer and the host algorithms.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>
#include <thread>

#include "ltfb_b200/host_algos.hpp"
#include "kernels.hpp"
#include "ltfb_gpu.h"
#include "trainer_core.hpp"

using ltfb_b200::DeviceGuard;
using ltfb_b200::DeviceTrainer;

struct ltfb_trainer {
  std::unique_ptr<DeviceTrainer> t;
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return LTFB_OK;
  } catch (const ltfb::DimensionError& e) {
    g_err = e.what();
    return LTFB_EDIMENSION;
  } catch (const ltfb::ContractError& e) {
    g_err = e.what();
    return LTFB_ECONTRACT;
  } catch (const ltfb::NumericError& e) {
    g_err = e.what();
    return LTFB_ENUMERIC;
  } catch (const ltfb::IoError& e) {
    g_err = e.what();
    return LTFB_EIO;
  } catch (const ltfb::CapacityError& e) {
    g_err = e.what();
    return LTFB_ECAPACITY;
  } catch (const ltfb::StoreCorruptError& e) {
    g_err = e.what();
    return LTFB_ESTORECORRUPT;
  } catch (const ltfb::ConfigError& e) {
    g_err = e.what();
    return LTFB_ECONFIG;
  } catch (const ltfb::Error& e) {
    g_err = e.what();
    return std::strncmp(e.what(), "CUDA error", 10) == 0 ? LTFB_ECUDA : LTFB_EINTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LTFB_EINTERNAL;
  }
}

ltfb::nn::Activation act_of(int32_t code, double slope) {
  using ltfb::nn::Act;
  switch (code) {
    case LTFB_ACT_IDENTITY: return {Act::kIdentity, slope};
    case LTFB_ACT_RELU: return {Act::kRelu, slope};
    case LTFB_ACT_LEAKY_RELU: return {Act::kLeakyRelu, slope};
    case LTFB_ACT_TANH: return {Act::kTanh, slope};
    case LTFB_ACT_SIGMOID: return {Act::kSigmoid, slope};
  }
  throw ltfb::ConfigError("unknown activation code " + std::to_string(code));
}

ltfb::surrogate::ModalityDims dims_of(const ltfb_dims* d) {
  if (!d) throw ltfb::ContractError("null dims");
  ltfb::surrogate::ModalityDims m;
  m.input_dim = d->input_dim;
  m.latent_dim = d->latent_dim;
  m.scalar_dim = d->scalar_dim;
  m.image_views = d->image_views;
  m.image_channels = d->image_channels;
  m.image_h = d->image_h;
  m.image_w = d->image_w;
  m.validate();
  return m;
}

ltfb::surrogate::SurrogateArch arch_of(const ltfb_arch* a) {
  ltfb::surrogate::SurrogateArch s;
  if (!a) return s;
  auto list = [](const uint32_t* w, uint32_t n) {
    if (n > 8) throw ltfb::ContractError("more than 8 hidden layers");
    return std::vector<std::size_t>(w, w + n);
  };
  s.enc_hidden = list(a->enc_hidden, a->n_enc_hidden);
  s.dec_hidden = list(a->dec_hidden, a->n_dec_hidden);
  s.fwd_hidden = list(a->fwd_hidden, a->n_fwd_hidden);
  s.inv_hidden = list(a->inv_hidden, a->n_inv_hidden);
  s.disc_hidden = list(a->disc_hidden, a->n_disc_hidden);
  s.hidden_act = act_of(a->hidden_act, a->hidden_slope);
  s.lambda_adv = a->lambda_adv;
  s.lambda_cyc = a->lambda_cyc;
  s.adam.lr = a->lr;
  s.adam.beta1 = a->beta1;
  s.adam.beta2 = a->beta2;
  s.adam.eps = a->eps;
  return s;
}

DeviceTrainer& T(ltfb_trainer* t) {
  if (!t || !t->t) throw ltfb::ContractError("null trainer handle");
  return *t->t;
}

// ---------------------------------------------------------------- NCCL ----
// Loaded at run time so the library has no link-time NCCL dependency; in a
// process that already loaded torch, dlopen returns torch's libnccl.so.2.
typedef int nccl_result;
typedef void* nccl_comm;
struct NcclUid {
  char internal[128];
};
struct NcclApi {
  nccl_result (*GetUniqueId)(NcclUid*) = nullptr;
  nccl_result (*CommInitRank)(nccl_comm*, int, NcclUid, int) = nullptr;
  nccl_result (*CommDestroy)(nccl_comm) = nullptr;
  nccl_result (*Send)(const void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  nccl_result (*Recv)(void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  nccl_result (*Bcast)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  nccl_result (*AllGather)(const void*, void*, size_t, int, nccl_comm, cudaStream_t) = nullptr;
  nccl_result (*GroupStart)() = nullptr;
  nccl_result (*GroupEnd)() = nullptr;
  const char* (*ErrStr)(nccl_result) = nullptr;
  bool ok = false;
};
constexpr int kNcclFloat = 7;  // ncclFloat32

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.Bcast = reinterpret_cast<decltype(api.Bcast)>(sym("ncclBroadcast"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.ErrStr = reinterpret_cast<decltype(api.ErrStr)>(sym("ncclGetErrorString"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv &&
             api.Bcast && api.AllGather && api.GroupStart && api.GroupEnd && api.ErrStr;
  });
  return api;
}

void nccl_check(nccl_result r, const char* what) {
  if (r != 0) throw ltfb::Error(std::string("NCCL error at ") + what + ": " + nccl().ErrStr(r));
}

}  // namespace

struct ltfb_comm {
  nccl_comm comm = nullptr;
  int nranks = 0, rank = 0, device = 0;
};

extern "C" {

const char* ltfb_last_error(void) { return g_err.c_str(); }
int ltfb_abi_version(void) { return LTFB_ABI_VERSION; }

int ltfb_device_count(int* count) {
  return guarded([&] { LTFB_CUDA(cudaGetDeviceCount(count)); });
}

void ltfb_arch_defaults(ltfb_arch* a) {
  std::memset(a, 0, sizeof(*a));
  a->enc_hidden[0] = 64;
  a->n_enc_hidden = 1;
  a->dec_hidden[0] = 64;
  a->n_dec_hidden = 1;
  a->fwd_hidden[0] = a->fwd_hidden[1] = 32;
  a->n_fwd_hidden = 2;
  a->inv_hidden[0] = a->inv_hidden[1] = 32;
  a->n_inv_hidden = 2;
  a->disc_hidden[0] = a->disc_hidden[1] = 32;
  a->n_disc_hidden = 2;
  a->hidden_act = LTFB_ACT_LEAKY_RELU;
  a->hidden_slope = 0.2;
  a->lambda_adv = 0.01;
  a->lambda_cyc = 1.0;
  a->lr = 0.001;
  a->beta1 = 0.9;
  a->beta2 = 0.999;
  a->eps = 1e-8;
}

int ltfb_trainer_create(const ltfb_dims* dims, const ltfb_arch* arch, const ltfb_trainer_config* cfg,
                        ltfb_trainer** out) {
  return guarded([&] {
    if (!cfg || !out) throw ltfb::ContractError("null argument");
    ltfb_b200::TrainerSpec s;
    s.dims = dims_of(dims);
    s.arch = arch_of(arch);
    s.trainer_id = cfg->trainer_id;
    s.device = cfg->device;
    s.n_shards = cfg->n_shards;
    s.batch_size = cfg->batch_size;
    s.seed = cfg->seed;
    s.numeric_abort_threshold = cfg->numeric_abort_threshold;
    s.w_f = cfg->w_f;
    s.w_i = cfg->w_i;
    s.lr[2] = cfg->lr_fwd;
    s.lr[3] = cfg->lr_inv;
    s.lr[4] = cfg->lr_disc;
    s.wide_kernel = cfg->wide_kernel;
    s.post_kernel = cfg->post_kernel;
    auto h = std::make_unique<ltfb_trainer>();
    h->t = std::make_unique<DeviceTrainer>(s);
    *out = h.release();
  });
}

int ltfb_trainer_destroy(ltfb_trainer* t) {
  return guarded([&] { delete t; });
}

int ltfb_trainer_param_count(const ltfb_trainer* t, int net, uint64_t* count) {
  return guarded([&] {
    if (net < 0 || net > 4) throw ltfb::ContractError("bad network index");
    *count = T(const_cast<ltfb_trainer*>(t)).param_count(net);
  });
}

int ltfb_trainer_set_params(ltfb_trainer* t, int net, const float* blob, uint64_t count) {
  return guarded([&] { T(t).set_params(net, blob, count); });
}
int ltfb_trainer_get_params(ltfb_trainer* t, int net, float* blob, uint64_t count) {
  return guarded([&] { T(t).get_params(net, blob, count); });
}
int ltfb_trainer_set_adam(ltfb_trainer* t, int net, const float* m, const float* v, uint64_t step) {
  return guarded([&] { T(t).set_adam(net, m, v, step); });
}
int ltfb_trainer_get_adam(ltfb_trainer* t, int net, float* m, float* v, uint64_t* step) {
  return guarded([&] { T(t).get_adam(net, m, v, step); });
}

int ltfb_trainer_load_store(ltfb_trainer* t, const uint32_t* ids, uint64_t n, const float* x,
                            const float* y, const int32_t* owner) {
  return guarded([&] { T(t).load_store(ids, n, x, y, owner); });
}

int ltfb_trainer_set_slice(ltfb_trainer* t, int which, const float* x, const float* y, uint64_t rows) {
  return guarded([&] {
    if (which != 0 && which != 1) throw ltfb::ContractError("bad slice index");
    T(t).set_slice(which, x, y, rows);
  });
}

int ltfb_trainer_generate_store(ltfb_trainer* t, const uint32_t* ids, uint64_t n, const int32_t* owner,
                                uint64_t spec_seed, double noise_level, uint64_t sampling_seed,
                                uint64_t total_n) {
  return guarded([&] { T(t).generate_store(ids, n, owner, spec_seed, noise_level, sampling_seed, total_n); });
}

int ltfb_trainer_generate_slice(ltfb_trainer* t, int which, const uint32_t* ids, uint64_t rows,
                                uint64_t spec_seed, double noise_level, uint64_t sampling_seed,
                                uint64_t total_n) {
  return guarded([&] {
    if (which != 0 && which != 1) throw ltfb::ContractError("bad slice index");
    T(t).generate_slice(which, ids, rows, spec_seed, noise_level, sampling_seed, total_n);
  });
}

int ltfb_trainer_train_steps(ltfb_trainer* t, uint64_t n, ltfb_step_record* out, uint64_t* n_out) {
  bool ok = true;
  std::vector<ltfb::train::StepRecord> recs;
  const int rc = guarded([&] {
    recs.reserve(n);
    ok = T(t).train_steps(n, recs);
  });
  if (n_out) *n_out = recs.size();
  if (out)
    for (std::size_t i = 0; i < recs.size(); ++i) {
      const auto& r = recs[i];
      out[i] = {r.step, r.epoch, r.skipped ? 1u : 0u, r.d_loss, r.g_total, r.g_fwd, r.g_adv, r.g_cyc};
    }
  if (rc != LTFB_OK) return rc;
  if (!ok) {
    g_err = "trainer " + std::to_string(T(t).spec().trainer_id) + " exceeded the numeric skip threshold";
    return LTFB_ENUMERIC;
  }
  return LTFB_OK;
}

int ltfb_trainer_step(const ltfb_trainer* t, uint64_t* step) {
  return guarded([&] { *step = T(const_cast<ltfb_trainer*>(t)).step(); });
}

int ltfb_trainer_take_epochs(ltfb_trainer* t, ltfb_epoch_record* out, uint64_t cap, uint64_t* n_out) {
  return guarded([&] {
    const auto eps = T(t).take_epochs();
    if (eps.size() > cap) throw ltfb::ContractError("take_epochs: capacity too small");
    for (std::size_t i = 0; i < eps.size(); ++i)
      out[i] = {eps[i].epoch, eps[i].partial ? 1u : 0u, eps[i].steps, eps[i].samples_shuffled, eps[i].seconds};
    *n_out = eps.size();
  });
}

int ltfb_trainer_flush_epoch(ltfb_trainer* t) {
  return guarded([&] { T(t).flush_epoch(); });
}

int ltfb_trainer_evaluate(ltfb_trainer* t, int which, const float* cf, const float* ci, double w_f,
                          double w_i, ltfb_eval_metric* out) {
  return guarded([&] {
    auto& tr = T(t);
    const float* df = nullptr;
    const float* di = nullptr;
    if (cf || ci) {
      if (!(cf && ci)) throw ltfb::ContractError("evaluate: pass both candidate blobs or neither");
      tr.set_incoming(cf, ci);
      df = tr.incoming_dev();
      di = tr.incoming_dev() + tr.param_count(2);
    }
    const auto r = tr.evaluate(which, df, di, 1, false, w_f, w_i);
    *out = {r.m[0].forward_mae, r.m[0].inverse_mae, r.m[0].combined};
  });
}

int ltfb_trainer_generator_floats(const ltfb_trainer* t, uint64_t* n) {
  return guarded([&] { *n = T(const_cast<ltfb_trainer*>(t)).generator_floats(); });
}

int ltfb_trainer_get_generator(ltfb_trainer* t, float* dst, uint64_t n) {
  return guarded([&] {
    auto& tr = T(t);
    if (n != tr.generator_floats()) throw ltfb::ContractError("get_generator: wrong length");
    DeviceGuard g(tr.device());
    LTFB_CUDA(cudaMemcpyAsync(dst, tr.generator_dev(), n * 4, cudaMemcpyDeviceToHost, tr.stream()));
    tr.sync_stream();
  });
}

int ltfb_trainer_set_incoming(ltfb_trainer* t, const float* fwd, const float* inv) {
  return guarded([&] { T(t).set_incoming(fwd, inv); });
}

int ltfb_trainer_copy_incoming(ltfb_trainer* dst, ltfb_trainer* src) {
  return guarded([&] {
    auto& d = T(dst);
    auto& s = T(src);
    if (d.generator_floats() != s.generator_floats())
      throw ltfb::ContractError("adopt_generators: incompatible parameter shapes");
    s.synchronize();
    DeviceGuard g(d.device());
    LTFB_CUDA(cudaMemcpyPeerAsync(d.incoming_dev(), d.device(), s.generator_dev(), s.device(),
                                  d.generator_floats() * 4, d.stream()));
    d.sync_stream();
  });
}

int ltfb_trainer_tournament_decide(ltfb_trainer* t, ltfb_eval_metric* local, ltfb_eval_metric* incoming,
                                   int32_t* adopted) {
  return guarded([&] {
    const auto r = T(t).tournament_decide();
    if (local) *local = {r.m[0].forward_mae, r.m[0].inverse_mae, r.m[0].combined};
    if (incoming) *incoming = {r.m[1].forward_mae, r.m[1].inverse_mae, r.m[1].combined};
    if (adopted) *adopted = r.adopted;
  });
}

int ltfb_trainer_adopt(ltfb_trainer* t, const float* fwd, const float* inv) {
  return guarded([&] { T(t).adopt(fwd, inv); });
}

int ltfb_trainer_prepare_graphs(ltfb_trainer* t) {
  return guarded([&] { T(t).prepare_graphs(); });
}

int ltfb_trainer_synchronize(ltfb_trainer* t) {
  return guarded([&] { T(t).synchronize(); });
}

int ltfb_trainer_load_ae_source(ltfb_trainer* t, const float* y, uint64_t n) {
  return guarded([&] {
    if (!y) throw ltfb::ContractError("load_ae_source: null source");
    T(t).load_ae_source(y, n);
  });
}

int ltfb_trainer_ae_alloc_source(ltfb_trainer* t, uint64_t rows) {
  return guarded([&] { T(t).ae_alloc_source(rows); });
}

int ltfb_trainer_ae_fill_from_store(ltfb_trainer* t, const uint32_t* slots, uint64_t n, uint64_t dst_row) {
  return guarded([&] {
    if (!slots && n) throw ltfb::ContractError("ae_fill_from_store: null slots");
    T(t).ae_fill_from_store(slots, n, dst_row);
  });
}

int ltfb_trainer_ae_step(ltfb_trainer* t, const uint32_t* idx, uint64_t n, double* loss) {
  return guarded([&] {
    if (!idx || n == 0) throw ltfb::ContractError("ae_step: empty batch");
    const double l = T(t).ae_step(idx, n);
    if (loss) *loss = l;
  });
}

int ltfb_ae_batch_rows(uint64_t seed, uint64_t rows, uint64_t batch, uint64_t steps, uint32_t* out) {
  return guarded([&] {
    if (rows == 0) throw ltfb::ContractError("ae_batch_rows: empty source");
    ltfb::Rng rng(ltfb::mix_seed({seed, 0xae1ULL}));
    for (uint64_t i = 0; i < batch * steps; ++i) out[i] = static_cast<uint32_t>(rng.below(rows));
  });
}

int ltfb_trainer_train_steps_host(ltfb_trainer* t, uint64_t n, const float* x, const float* y,
                                  ltfb_step_record* out, uint64_t* n_out) {
  bool ok = true;
  std::vector<ltfb::train::StepRecord> recs;
  const int rc = guarded([&] {
    recs.reserve(n);
    ok = T(t).train_steps_host(n, x, y, recs);
  });
  if (n_out) *n_out = recs.size();
  if (out)
    for (std::size_t i = 0; i < recs.size(); ++i) {
      const auto& r = recs[i];
      out[i] = {r.step, r.epoch, r.skipped ? 1u : 0u, r.d_loss, r.g_total, r.g_fwd, r.g_adv, r.g_cyc};
    }
  if (rc != LTFB_OK) return rc;
  if (!ok) {
    g_err = "trainer exceeded the numeric skip threshold";
    return LTFB_ENUMERIC;
  }
  return LTFB_OK;
}

int ltfb_trainer_timer_start(ltfb_trainer* t) {
  return guarded([&] { T(t).timer_start(); });
}
int ltfb_trainer_timer_stop(ltfb_trainer* t, double* ms) {
  return guarded([&] { *ms = T(t).timer_stop_ms(); });
}
int ltfb_trainer_kernel_timing(ltfb_trainer* t, int on) {
  return guarded([&] { T(t).set_kernel_timing(on != 0); });
}
int ltfb_trainer_kernel_time(ltfb_trainer* t, int which, double* ms, uint64_t* launches) {
  return guarded([&] {
    if (which < 0 || which > 4) throw ltfb::ContractError("bad kernel index");
    const auto r = T(t).kernel_time(which);
    *ms = r.first;
    *launches = r.second;
  });
}
int ltfb_trainer_wide_info(const ltfb_trainer* t, int32_t* kind, int32_t* ctas) {
  return guarded([&] {
    auto& tr = T(const_cast<ltfb_trainer*>(t));
    *kind = tr.wide_kernel_kind();
    *ctas = static_cast<int32_t>(tr.wide_ctas());
  });
}

int ltfb_trainer_wide_tile(const ltfb_trainer* t, int32_t* cols) {
  return guarded([&] {
    auto& tr = T(const_cast<ltfb_trainer*>(t));
    *cols = tr.wide_kernel_kind() >= 2 ? (tr.wide2() ? 64 : 32) : 0;
  });
}

int ltfb_trainer_eval_info(const ltfb_trainer* t, int which, int32_t* kind) {
  return guarded([&] {
    if (which < 0 || which > 1) throw ltfb::ContractError("eval_info: which must be 0 or 1");
    *kind = T(const_cast<ltfb_trainer*>(t)).eval_kind(which);
  });
}

int ltfb_trainer_ae_info(const ltfb_trainer* t, int32_t rows, int32_t* kind) {
  return guarded([&] { *kind = T(const_cast<ltfb_trainer*>(t)).ae_kind(rows); });
}

int ltfb_trainer_stream_info(const ltfb_trainer* t, int32_t* on) {
  return guarded([&] { *on = T(const_cast<ltfb_trainer*>(t)).stream_mode() ? 1 : 0; });
}

int ltfb_trainer_stream_profile(ltfb_trainer* t, int arm, double* out, int n) {
  return guarded([&] {
    auto& tr = T(t);
    if (arm) {
      tr.stream_profile_next();
      return;
    }
    if (!out || n < 0) throw ltfb::ContractError("stream_profile: bad output buffer");
    for (int i = 0; i < n && i < 8; ++i) out[i] = tr.stream_profile()[i];
  });
}

int ltfb_trainer_launch_count(const ltfb_trainer* t, uint64_t* launches) {
  return guarded([&] { *launches = T(const_cast<ltfb_trainer*>(t)).launch_count(); });
}

int ltfb_selftest_tcgen05(const float* a1, const float* b1, const float* ah, const float* b2, const float* a3,
                          float* d1, float* d2, float* d3) {
  return guarded([&] {
    const std::size_t n_in[5] = {128 * 32, 32 * 64, 128 * 64, 64 * 32, 128 * 32};
    const float* in[5] = {a1, b1, ah, b2, a3};
    const std::size_t n_out[3] = {128 * 64, 128 * 32, 128 * 64};
    float* outp[3] = {d1, d2, d3};
    float* din[5];
    float* dout[3];
    for (int i = 0; i < 5; ++i) {
      LTFB_CUDA(cudaMalloc(&din[i], n_in[i] * 4));
      LTFB_CUDA(cudaMemcpy(din[i], in[i], n_in[i] * 4, cudaMemcpyHostToDevice));
    }
    for (int i = 0; i < 3; ++i) LTFB_CUDA(cudaMalloc(&dout[i], n_out[i] * 4));
    const cudaError_t e = ltfb_dev::selftest_tc(din[0], din[1], din[2], din[3], din[4], dout[0], dout[1], dout[2]);
    for (int i = 0; i < 3; ++i) {
      if (e == cudaSuccess) LTFB_CUDA(cudaMemcpy(outp[i], dout[i], n_out[i] * 4, cudaMemcpyDeviceToHost));
      cudaFree(dout[i]);
    }
    for (int i = 0; i < 5; ++i) cudaFree(din[i]);
    LTFB_CUDA(e);
  });
}

int ltfb_adam_step(float* p, float* m, float* v, const float* g, uint64_t n, uint64_t* t, double lr, double beta1,
                   double beta2, double eps, int device) {
  return guarded([&] {
    if (!p || !m || !v || !g || !t) throw ltfb::ContractError("adam_step: null buffer");
    // adam.hpp:91-102: every gradient component finite before any state changes
    for (uint64_t i = 0; i < n; ++i)
      if (!std::isfinite(static_cast<double>(g[i]))) throw ltfb::NumericError("adam_step: non-finite gradient component");
    DeviceGuard dg(device);
    const uint64_t tn = *t + 1;
    const double c1 = 1.0 - std::pow(beta1, static_cast<double>(tn));  // adam.hpp:113-116
    const double c2 = 1.0 - std::pow(beta2, static_cast<double>(tn));
    float* d = nullptr;
    LTFB_CUDA(cudaMalloc(&d, std::max<uint64_t>(1, 4 * n) * 4));
    float *dp = d, *dm = d + n, *dv = d + 2 * n, *dg2 = d + 3 * n;
    cudaError_t e = cudaSuccess;
    if (n > 0) {
      const float* src[4] = {p, m, v, g};
      for (int i = 0; i < 4 && e == cudaSuccess; ++i) e = cudaMemcpy(d + i * n, src[i], n * 4, cudaMemcpyHostToDevice);
      if (e == cudaSuccess) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        ltfb_dev::launch_ae_adam(dp, dm, dv, dg2, static_cast<long long>(n), lr, beta1, beta2, eps, c1, c2, sms, 0);
        e = cudaDeviceSynchronize();
      }
      float* dst[3] = {p, m, v};
      for (int i = 0; i < 3 && e == cudaSuccess; ++i) e = cudaMemcpy(dst[i], d + i * n, n * 4, cudaMemcpyDeviceToHost);
    }
    cudaFree(d);
    LTFB_CUDA(e);
    *t = tn;
  });
}

int ltfb_nccl_available(void) { return nccl().ok ? 1 : 0; }

int ltfb_nccl_unique_id(uint8_t id[128]) {
  return guarded([&] {
    if (!nccl().ok) throw ltfb::Error("NCCL library not found");
    NcclUid u;
    nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, 128);
  });
}

int ltfb_comm_create(const uint8_t id[128], int nranks, int rank, int device, ltfb_comm** out) {
  return guarded([&] {
    if (!nccl().ok) throw ltfb::Error("NCCL library not found");
    DeviceGuard g(device);
    NcclUid u;
    std::memcpy(u.internal, id, 128);
    auto c = std::make_unique<ltfb_comm>();
    nccl_check(nccl().CommInitRank(&c->comm, nranks, u, rank), "ncclCommInitRank");
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    *out = c.release();
  });
}

int ltfb_comm_destroy(ltfb_comm* c) {
  return guarded([&] {
    if (c && c->comm) nccl().CommDestroy(c->comm);
    delete c;
  });
}

int ltfb_trainer_exchange(ltfb_trainer* t, ltfb_comm* c, int peer) {
  return guarded([&] {
    auto& tr = T(t);
    if (!c) throw ltfb::ContractError("null communicator");
    if (peer == c->rank) throw ltfb::ContractError("tournament_round: trainer paired with itself");
    DeviceGuard g(tr.device());
    const std::size_t n = tr.generator_floats();
    auto& api = nccl();
    nccl_check(api.GroupStart(), "ncclGroupStart");
    nccl_check(api.Send(tr.generator_dev(), n, kNcclFloat, peer, c->comm, tr.stream()), "ncclSend");
    nccl_check(api.Recv(tr.incoming_dev(), n, kNcclFloat, peer, c->comm, tr.stream()), "ncclRecv");
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
  });
}

int ltfb_trainer_ae_allgather(ltfb_trainer* t, ltfb_comm* c, uint64_t rows_per_rank) {
  return guarded([&] {
    auto& tr = T(t);
    if (!c) throw ltfb::ContractError("null communicator");
    if (rows_per_rank * static_cast<uint64_t>(c->nranks) > tr.ae_source_rows())
      throw ltfb::ContractError("ae_allgather: AE source smaller than rows_per_rank x ranks");
    DeviceGuard g(tr.device());
    const std::size_t count = rows_per_rank * static_cast<std::size_t>(tr.out_pad());
    float* buf = tr.ae_source_dev();
    // in place: rank r's rows sit at [r * rows_per_rank, (r + 1) * rows_per_rank)
    nccl_check(nccl().AllGather(buf + count * static_cast<std::size_t>(c->rank), buf, count, kNcclFloat, c->comm,
                                tr.stream()),
               "ncclAllGather");
  });
}

int ltfb_trainer_broadcast(ltfb_trainer* t, ltfb_comm* c, int net, int root) {
  return guarded([&] {
    auto& tr = T(t);
    if (!c) throw ltfb::ContractError("null communicator");
    if (net != LTFB_NET_ENC && net != LTFB_NET_DEC)
      throw ltfb::ContractError("broadcast: only the shared autoencoder is broadcast");
    DeviceGuard g(tr.device());
    std::vector<float> host(tr.param_count(net));
    // the enc/dec blobs are addressed through get/set to keep one owner of
    // the device layout; the NCCL payload itself is device-resident
    float* dev = nullptr;
    LTFB_CUDA(cudaMalloc(&dev, host.size() * 4));
    if (c->rank == root) {
      tr.get_params(net, host.data(), host.size());
      LTFB_CUDA(cudaMemcpy(dev, host.data(), host.size() * 4, cudaMemcpyHostToDevice));
    }
    nccl_check(nccl().Bcast(dev, dev, host.size(), kNcclFloat, root, c->comm, tr.stream()), "ncclBroadcast");
    tr.sync_stream();
    if (c->rank != root) {
      LTFB_CUDA(cudaMemcpy(host.data(), dev, host.size() * 4, cudaMemcpyDeviceToHost));
      tr.set_params(net, host.data(), host.size());
    }
    cudaFree(dev);
  });
}

// ----------------------------------------------------- host algorithms ---
uint64_t ltfb_mix_seed(const uint64_t* words, int n) {
  std::uint64_t acc = 0x243f6a8885a308d3ULL;
  for (int i = 0; i < n; ++i) {
    acc ^= words[i] + ltfb::seedmix::kGolden + (acc << 6) + (acc >> 2);
    ltfb::seedmix::step(acc);
  }
  return ltfb::seedmix::step(acc);
}

uint64_t ltfb_fnv1a64(const void* bytes, uint64_t n) { return ltfb::fnv1a64(bytes, n); }

int ltfb_pair_trainers(int k, int round, uint64_t seed, int32_t* pairs, int32_t* bye, int32_t* n_pairs) {
  return guarded([&] {
    const auto m = ltfb::tournament::pair_trainers(k, round, seed);
    for (std::size_t i = 0; i < m.pairs.size(); ++i) {
      pairs[2 * i] = m.pairs[i][0];
      pairs[2 * i + 1] = m.pairs[i][1];
    }
    *bye = m.bye;
    *n_pairs = static_cast<int32_t>(m.pairs.size());
  });
}

int ltfb_partition_dataset(const uint32_t* ids, uint64_t n, int k, uint64_t seed, uint32_t* out_ids,
                           uint32_t* sizes) {
  return guarded([&] {
    const auto parts = ltfb::tournament::partition_dataset(std::vector<uint32_t>(ids, ids + n), k, seed);
    std::size_t at = 0;
    for (std::size_t p = 0; p < parts.size(); ++p) {
      sizes[p] = static_cast<uint32_t>(parts[p].size());
      std::memcpy(out_ids + at, parts[p].data(), parts[p].size() * 4);
      at += parts[p].size();
    }
  });
}

int ltfb_split_dataset(uint64_t total, int k, double vf, double tf, uint64_t seed, int need_tournament,
                       uint32_t* val, uint64_t* n_val, uint32_t* train, uint32_t* train_sizes,
                       uint32_t* tour, uint32_t* tour_sizes) {
  return guarded([&] {
    const auto s = ltfb::tournament::detail::split_dataset(total, k, vf, tf, seed, need_tournament != 0);
    std::memcpy(val, s.validation.data(), s.validation.size() * 4);
    *n_val = s.validation.size();
    std::size_t a = 0, b = 0;
    for (int t = 0; t < k; ++t) {
      train_sizes[t] = static_cast<uint32_t>(s.train[t].size());
      tour_sizes[t] = static_cast<uint32_t>(s.tournament[t].size());
      std::memcpy(train + a, s.train[t].data(), s.train[t].size() * 4);
      std::memcpy(tour + b, s.tournament[t].data(), s.tournament[t].size() * 4);
      a += s.train[t].size();
      b += s.tournament[t].size();
    }
  });
}

int ltfb_epoch_permutation(const uint32_t* partition, uint64_t n, uint32_t epoch, uint64_t seed,
                           uint32_t* out) {
  return guarded([&] {
    const auto p = ltfb::data::epoch_permutation(std::vector<uint32_t>(partition, partition + n), epoch, seed);
    std::memcpy(out, p.data(), n * 4);
  });
}

int ltfb_incoming_wins(double local, double incoming) {
  return ltfb::tournament::incoming_wins(local, incoming) ? 1 : 0;
}

static void synth_rows_impl(const ltfb_dims* dims, uint64_t spec_seed, double noise_level,
                            const uint32_t* ids, uint64_t first, uint64_t n, uint64_t total_n,
                            uint64_t sampling_seed, float* x, float* y, int threads) {
  {
    ltfb::synth::GeneratorSpec spec;
    spec.dims = dims_of(dims);
    spec.spec_seed = spec_seed;
    spec.noise_level = noise_level;
    const ltfb::synth::SynthGenerator gen(spec);
    const std::uint32_t g = ltfb::synth::grid_side(total_n);
    const std::size_t in = spec.dims.input_dim, out = spec.dims.output_dim();
    auto work = [&](std::uint64_t a, std::uint64_t b) {
      for (std::uint64_t i = a; i < b; ++i) {
        const std::uint64_t id = ids ? ids[i] : first + i;
        const auto p = ltfb::synth::sweep_point(id, g, sampling_seed);
        gen.sample_into(p, x + i * in, y + i * out);
      }
    };
    const int nt = std::max(1, std::min<int>(threads, static_cast<int>(std::max<std::uint64_t>(1, n / 64))));
    if (nt == 1) {
      work(0, n);
      return;
    }
    std::vector<std::thread> pool;
    for (int w = 0; w < nt; ++w) pool.emplace_back(work, n * w / nt, n * (w + 1) / nt);
    for (auto& th : pool) th.join();
  }
}

static int synth_rows(const ltfb_dims* dims, uint64_t spec_seed, double noise_level,
                      const uint32_t* ids, uint64_t first, uint64_t n, uint64_t total_n,
                      uint64_t sampling_seed, float* x, float* y, int threads) {
  return guarded([&] { synth_rows_impl(dims, spec_seed, noise_level, ids, first, n, total_n, sampling_seed, x, y,
                                       threads); });
}

int ltfb_synth_generate_ids(const ltfb_dims* dims, uint64_t spec_seed, double noise_level,
                            const uint32_t* ids, uint64_t n, uint64_t total_n, uint64_t sampling_seed,
                            float* x, float* y, int threads) {
  return synth_rows(dims, spec_seed, noise_level, ids, 0, n, total_n, sampling_seed, x, y, threads);
}

int ltfb_synth_generate(const ltfb_dims* dims, uint64_t spec_seed, double noise_level, uint64_t first,
                        uint64_t n, uint64_t total_n, uint64_t sampling_seed, float* x, float* y,
                        int threads) {
  return synth_rows(dims, spec_seed, noise_level, nullptr, first, n, total_n, sampling_seed, x, y, threads);
}

int ltfb_synth_generate_device(const ltfb_dims* dims, uint64_t spec_seed, double noise_level,
                               const uint32_t* ids, uint64_t first, uint64_t n, uint64_t total_n,
                               uint64_t sampling_seed, float* x_dev, float* y_dev, uint64_t y_stride,
                               int device) {
  return guarded([&] {
    ltfb_b200::DeviceGuard g(device);
    cudaStream_t s = nullptr;
    LTFB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    try {
      ltfb_dev::synth_generate_device(dims_of(dims), spec_seed, noise_level, ids, first, n, total_n,
                                      sampling_seed, x_dev, y_dev, static_cast<long long>(y_stride), s);
    } catch (...) {
      cudaStreamDestroy(s);
      throw;
    }
    LTFB_CUDA(cudaStreamDestroy(s));
  });
}

struct ltfb_dataset {
  ltfb::data::DatasetIndex index;
};

int ltfb_dataset_open(const char* dir, ltfb_dataset** out) {
  return guarded([&] {
    if (!dir || !out) throw ltfb::ContractError("ltfb_dataset_open: null argument");
    auto* d = new ltfb_dataset{ltfb::data::DatasetIndex::scan_dir(dir)};
    *out = d;
  });
}

int ltfb_dataset_destroy(ltfb_dataset* d) {
  delete d;
  return LTFB_OK;
}

int ltfb_dataset_info(const ltfb_dataset* d, ltfb_dims* dims, uint64_t* total, uint64_t* n_files) {
  return guarded([&] {
    const auto& x = d->index.dims;
    if (dims) *dims = ltfb_dims{x.input_dim, x.latent_dim, x.scalar_dim, x.image_views, x.image_channels,
                                x.image_h, x.image_w};
    if (total) *total = d->index.total;
    if (n_files) *n_files = d->index.paths.size();
  });
}

int ltfb_dataset_file_of(const ltfb_dataset* d, const uint32_t* ids, uint64_t n, uint32_t* file_idx) {
  return guarded([&] {
    for (uint64_t i = 0; i < n; ++i) file_idx[i] = static_cast<uint32_t>(d->index.locate(ids[i]).file_idx);
  });
}

int ltfb_dataset_read(const ltfb_dataset* d, const uint32_t* ids, uint64_t n, float* x, float* y,
                      uint64_t* files_opened) {
  return guarded([&] {
    const std::size_t opened = ltfb::data::read_records(d->index, std::span<const uint32_t>(ids, n), x, y,
                                                        d->index.dims.output_dim());
    if (files_opened) *files_opened = opened;
  });
}

int ltfb_write_synth_bundles(const char* dir, const ltfb_dims* dims, uint64_t spec_seed, double noise_level,
                             uint64_t gen_n, uint64_t sampling_seed, uint32_t samples_per_file, int threads) {
  return guarded([&] {
    if (!dir) throw ltfb::ContractError("ltfb_write_synth_bundles: null directory");
    if (gen_n < 1) throw ltfb::ContractError("generate_dataset: n must be >= 1");
    const auto d = dims_of(dims);
    const std::size_t in = d.input_dim, out = d.output_dim();
    std::vector<float> x(gen_n * in), y(gen_n * out);
    synth_rows_impl(dims, spec_seed, noise_level, nullptr, 0, gen_n, gen_n, sampling_seed, x.data(), y.data(),
                    threads);
    std::vector<ltfb::data::SampleRecord> recs(gen_n);
    for (uint64_t i = 0; i < gen_n; ++i) {
      recs[i].inputs.assign(x.begin() + i * in, x.begin() + (i + 1) * in);
      recs[i].outputs.assign(y.begin() + i * out, y.begin() + (i + 1) * out);
    }
    ltfb::data::write_bundles(recs, d, samples_per_file, dir);
  });
}

int ltfb_net_param_count(const ltfb_dims* dims, const ltfb_arch* arch, int net, uint64_t* count) {
  return guarded([&] {
    const auto m = ltfb::surrogate::make_cyclegan<float>(dims_of(dims), arch_of(arch), 0);
    const ltfb::nn::MlpSpec* s[5] = {&m.enc_spec, &m.dec_spec, &m.fwd_spec, &m.inv_spec, &m.disc_spec};
    if (net < 0 || net > 4) throw ltfb::ContractError("bad network index");
    *count = ltfb::nn::manifest_for(*s[net]).total;
  });
}

int ltfb_init_params(const ltfb_dims* dims, const ltfb_arch* arch, uint64_t seed, int net, float* blob,
                     uint64_t count) {
  return guarded([&] {
    if (net < 0 || net > 4) throw ltfb::ContractError("bad network index");
    auto spec = ltfb::surrogate::make_cyclegan<float>(dims_of(dims), arch_of(arch), 0);
    ltfb::nn::MlpSpec* s[5] = {&spec.enc_spec, &spec.dec_spec, &spec.fwd_spec, &spec.inv_spec, &spec.disc_spec};
    s[net]->init_seed = ltfb::mix_seed({seed, static_cast<std::uint64_t>(net + 1)});
    const auto p = ltfb::nn::init_params<float>(*s[net]);
    if (count != p.param_count()) throw ltfb::ContractError("init_params: wrong blob length");
    p.flatten_into(blob);
  });
}

}  // extern "C"
