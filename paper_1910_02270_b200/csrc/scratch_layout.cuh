// Layout of the per-trainer small-network scratch (tapes and gradients of
// fwd, inv, disc, the enc tail and the dec head). Computed identically on
// host (allocation size) and device (pointer carving).
#pragma once

#include "step_args.cuh"

namespace ltfb_dev {





__host__ __device__ inline long long round_up_ll(long long v, long long a) { return (v + a - 1) / a * a; }

__host__ __device__ inline ScratchLayout make_scratch_layout(const ModelArgs& m, int B) {
  ScratchLayout s{};
  long long at = 0;
  auto take = [&](long long n) {
    const long long o = at;
    at += round_up_ll(n, 32);
    return o;
  };
  auto tape = [&](const NetDesc& n, long long rows, long long* z, long long* a) {
    for (int l = 0; l < kMaxLayers; ++l) z[l] = a[l] = 0;
    for (int l = 0; l < n.L; ++l) {
      z[l] = take(rows * n.w[l + 1]);
      a[l] = take(rows * n.w[l + 1]);
    }
  };
  tape(m.fwd, B, s.fz, s.fa);
  tape(m.dec_head, B, s.hz, s.ha);
  tape(m.enc_tail, B, s.ez, s.ea);
  tape(m.disc, 2LL * B, s.cz, s.ca);
  tape(m.inv, B, s.iz, s.ia);
  s.e1z = take((long long)B * m.E1);
  s.e1a = take((long long)B * m.E1);
  s.stacked = take(2LL * B * m.lat);
  s.probs = take(2LL * B);
  s.bgrad = take(2LL * B);
  s.gh = take((long long)B * m.D);
  s.gl_dec = take((long long)B * m.lat);
  s.gl_disc = take((long long)B * m.lat);
  s.gl_inv = take((long long)B * m.lat);
  s.gl = take((long long)B * m.lat);
  s.igrad = take((long long)B * m.in);
  int mw = m.in > m.lat ? m.in : m.lat;
  const NetDesc* nets[5] = {&m.fwd, &m.inv, &m.disc, &m.enc_tail, &m.dec_head};
  for (const NetDesc* n : nets) mw = n->max_w() > mw ? n->max_w() : mw;
  mw = m.E1 > mw ? m.E1 : mw;
  mw = m.D > mw ? m.D : mw;
  const long long per = (B + kPostCluster - 1) / kPostCluster;
  s.tstride = round_up_ll(2 * per * mw, 32);
  s.tA = take(s.tstride * kPostCluster);
  s.tB = take(s.tstride * kPostCluster);
  s.red_enc = take((long long)B * m.E1);
  s.red_dec = take((long long)B * m.D);
  s.pg_disc = take(kPostCluster * round_up_ll(m.disc.count, 32));
  s.pg_fwd = take(kPostCluster * round_up_ll(m.fwd.count, 32));
  s.pg_inv = take(kPostCluster * round_up_ll(m.inv.count, 32));
  s.total = at;
  return s;
}

}  // namespace ltfb_dev
