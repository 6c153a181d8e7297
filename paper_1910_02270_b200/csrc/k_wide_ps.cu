// The wide pass of the STREAMED step (DeviceTrainer stream mode): one
// persistent cooperative kernel per run of steps inside an epoch, on every
// SM the persistent post cluster (k_post_loop, 16 SMs) leaves free, split
// into two phases per step so that the work that does not need the step's h
// overlaps the post cluster's previous step:
//
//   phase 1 (y and We only)   P_enc += Y We     enc layer-0 split-K partials
//                                               (D-step real latents,
//                                               train_ops.hpp:160); then
//                                               the grid-wide fixed-order
//                                               reduction -> red_enc[k&1]
//                                               and enc_done += 1 per CTA
//   wait for h of the step (StepSync::h_done, written by the post cluster's
//   next_h of the previous step, or the row kernel for the run's first step)
//   phase 2 (y, Wd, Wd^T)     O = h Wd ; d = O + b - Y ; sum |d| ; S = sign d ;
//                             P_dec += S Wd^T   (train_ops.hpp:100-104,
//                                               loss.hpp:25-41, mlp.hpp:278);
//                                               reduction -> red_dec[k&1],
//                                               mae_total[k&1], dec_done
//
// Phase 1 of step k+1 runs while the post cluster finishes step k (its
// generator update and the next h); the post cluster's discriminator step of
// k+1 runs while phase 2 of k+1 streams. The y rows are gathered twice per
// step straight from the HBM store (TMA tile::gather4 through the epoch
// plan); the second read of the 25 MB batch comes from L2.
//
// Arithmetic per tile is k_wide_tc's (3xTF32 fp32-parity mode or 1xTF32 perf
// mode, the same MMA shapes and epilogue), so the streamed step computes what
// the launched step computes; the split-K partition follows the CTA count of
// this kernel, which the trainer also uses for its launched wide passes.
//
// Warp roles (320 threads): w0 TMA producer of the weight tiles, w1 MMA
// issuer + TMEM owner, w2-5 epilogue (TMEM lane quadrants), w6-9 y gather +
// tf32 split. Every ring counter runs on across phases and steps; at a phase
// end the producer and the gathers have already issued the next phase's
// first tiles (bounded by the rings), so the next phase's data arrives under
// the grid barrier, the reduction and the wait for h.
#include <cuda.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "kernels.hpp"
#include "stream_sync.cuh"
#include "tc_ptx.cuh"

namespace ltfb_dev {

namespace wp {
constexpr int kTileN = 32;
constexpr int kW = 64;
constexpr uint32_t kY = 16384;       // [128 x 32] f32
constexpr uint32_t kWt = 8192;       // [64 x 32] f32
constexpr uint32_t kStage = 4 * kWt; // phase 1: WeT hi/lo; phase 2: Wd hi/lo, WdT hi/lo
constexpr int kStages = 4;           // == TMEM y slots
constexpr int kYStages = 3;
constexpr int kMaxQ = 16;            // float4 outputs reduced per CTA (one of P_enc / P_dec)
constexpr int kThreads = 320;
// partial groups of the reduction: k_wide_tc's grouping (10 groups of 32
// threads, group g sums partials g, g + 10, ...), so a streamed step sums
// every output in exactly the launched step's order (bit-identical paths)
constexpr int kG = 10;
constexpr uint32_t kRedOff = kYStages * kY + kStages * kStage;  // reduction scratch
constexpr uint32_t kMaxS = 148;
constexpr uint32_t kSmem = kRedOff + (kMaxS + kG) * kMaxQ * 16 + 1024;
// TMEM columns: one split-K accumulator shared by the phases (P_enc in
// phase 1, P_dec in phase 2: each is read out before the other phase's
// first MMA), the O double buffer, h hi / lo, and a y slot per stage
constexpr uint32_t kPacc = 0, kO0 = 64, kHhi = 128, kHlo = 192, kYbase = 256;
static_assert(kYbase + 64 * kStages <= 512, "TMEM columns");
static_assert(kSmem <= 227 * 1024, "shared memory");
}  // namespace wp

struct WidePsParams {
  CUtensorMap tm_y, tm_wet, tm_wd, tm_wdt;
};

/// Sense-reversing grid barrier of the cooperative launch, with a timeout
/// (a missing CTA raises sync->error instead of hanging the GPU).
/// Grid barrier of the persistent wide pass. Arrival: one release atomic on
/// a counter. Release: the last CTA to arrive bumps every CTA's own flag
/// (one 128-B line per CTA), so the waiting CTAs poll disjoint lines instead
/// of all polling one (measured: ~4 us of release latency with one shared
/// generation word under 131 pollers). `epoch` counts this kernel's barriers
/// (identical in every CTA); flags only grow, so no reset is needed.
__device__ __forceinline__ void grid_sync_t(unsigned* bar, unsigned n, StepSync* sy, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* cnt = bar + 64;
    unsigned* flags = bar + 96;  // flag of CTA c at flags[32 c]
    unsigned old;
    // acq_rel: the last arriver acquires every CTA's writes before it releases the flags
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
    if (old + 1 == n * epoch) {
      // one release fence, then plain (relaxed) flag stores: a release store
      // per flag would fence 132 times
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      for (unsigned c = 0; c < n; ++c)
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(flags + 32 * c), "r"(epoch) : "memory");
    } else {
      const unsigned long long t0 = gtimer();
      unsigned cur;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(flags + 32 * blockIdx.x) : "memory");
        if (cur >= epoch) break;
        if (gtimer() - t0 > kStreamTimeoutNs) {
          if (atomicCAS(&sy->error, 0, 2) == 0) sy->err_site = 6;
          break;
        }
        __nanosleep(32);
      }
    }
  }
  __syncthreads();
}

/// mbarrier wait that traps after kStreamTimeoutNs: a broken hand-off inside
/// the persistent kernel ends it with a launch failure instead of a hang.
__device__ __forceinline__ void mbar_wait_to(uint64_t* bar, uint32_t parity) {
  if (tc::mbar_try_wait(bar, parity)) return;  // the warp sleeps in hardware while it waits
  const unsigned long long t0 = gtimer();
  while (!tc::mbar_try_wait(bar, parity))
    if (gtimer() - t0 > 2 * kStreamTimeoutNs) __trap();
}

template <bool kPrecise>
__global__ void __launch_bounds__(wp::kThreads, 1)
    k_wide_ps(const __grid_constant__ WidePsParams tp, const __grid_constant__ StepArgs a,
              const __grid_constant__ StreamArgs r, const float* __restrict__ bias_pad) {
  using namespace wp;
  if (a.ctr->aborted) return;  // the post cluster leaves at once too
  unsigned bar_epoch = 0;      // grid barriers passed in this launch (k_stream_init zeroes the counter and flags)
  if (blockIdx.x == 0 && threadIdx.x == 0) r.sync->t_wide0 = gtimer();
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kStages], split_done[kStages], sready[kStages], empty[kStages];
  __shared__ uint64_t yfull[kYStages];
  __shared__ uint64_t ofull[2], oempty[2], h_ready, done, rbar;
  __shared__ uint32_t tmem_base;
  __shared__ double red[128];
  __shared__ int s_go;

  StepSync* sy = r.sync;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int out = a.m.out;
  const int ntiles = (out + kTileN - 1) / kTileN;
  const int my_tiles = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int S = (int)gridDim.x;
  // the flat schedule: phase q = 2 k + p (k = step of the run, p = 0 / 1);
  // every phase has my_tiles tiles, running tile index i = q * my_tiles + j
  const int nphase = 2 * r.n;
  auto col0 = [&](int j) { return ((int)blockIdx.x + j * S) * kTileN; };
  auto rows_of = [&](int k) { return min(a.B, a.n_part - (r.sie0 + k) * a.B); };

  auto stage_ptr = [&](int s) { return sm + kYStages * kY + s * kStage; };
  auto Yraw = [&](int sy_) { return sm + sy_ * kY; };
  auto WeH = [&](int s) { return stage_ptr(s); };
  auto WeL = [&](int s) { return stage_ptr(s) + kWt; };
  auto WdH = [&](int s) { return stage_ptr(s); };
  auto WdL = [&](int s) { return stage_ptr(s) + kWt; };
  auto WtH = [&](int s) { return stage_ptr(s) + 2 * kWt; };
  auto WtL = [&](int s) { return stage_ptr(s) + 3 * kWt; };
  auto tYh = [&](int s) { return (uint32_t)(kYbase + 64 * s); };
  auto tYl = [&](int s) { return (uint32_t)(kYbase + 64 * s + 32); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&split_done[s], 128);
      tc::mbar_init(&sready[s], 128);
      tc::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kYStages; ++s) tc::mbar_init(&yfull[s], 1);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&ofull[b], 1);
      tc::mbar_init(&oempty[b], 128);
    }
    tc::mbar_init(&h_ready, 128);
    tc::mbar_init(&done, 1);
    tc::mbar_init(&rbar, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tp.tm_y);
    tc::tma_prefetch(&tp.tm_wet);
    tc::tma_prefetch(&tp.tm_wd);
    tc::tma_prefetch(&tp.tm_wdt);
  }
  if (warp == 1) tc::tmem_alloc<512>(&tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t T = tmem_base;

  // per-tile stamps of phase 2 (CTA 0): slot 32 + 5 j + e
#define TSTAMP(kk, j, e) do { if (r.prof && blockIdx.x == 0 && (j) < 12) r.prof[512 * (kk) + 32 + 5 * (j) + (e)] = gtimer(); } while (0)
  // ---- per-role state that runs on across phases ----
  int prod_next = 0;   // w0: next running tile index whose weights are issued
  int gath_next = 0;   // w6-9: next running tile index whose y rows are gathered
  uint32_t hr_par = 0, done_par = 0, rbar_par = 0;
  int o_run = 0;       // running phase-2 tile count (O double buffer)
  const unsigned* perm = a.perm[r.epoch & 1u];

  // w0: issue the weight tiles of running tiles [prod_next, upto)
  auto produce = [&](int upto) {
    for (; prod_next < upto; ++prod_next) {
      const int i = prod_next;
      const int q = i / max(my_tiles, 1), j = i - q * my_tiles;
      const int s = i % kStages;
      if (lane == 0) {
        if (i >= kStages) mbar_wait_to(&empty[s], ((uint32_t)(i / kStages) & 1u) ^ 1u);
        const int c0 = col0(j);
        if ((q & 1) == 0) {  // phase 1: WeT
          tc::mbar_expect_tx(&full[s], kWt);
          tc::tma_load_2d(WeH(s), &tp.tm_wet, &full[s], c0, 0);
        } else {             // phase 2: Wd (MMA3) and WdT (MMA2, two K-blocks)
          TSTAMP(q >> 1, j, 0);
          tc::mbar_expect_tx(&full[s], 2 * kWt);
          tc::tma_load_2d(WdH(s), &tp.tm_wd, &full[s], c0, 0);
          tc::tma_load_2d(WtH(s), &tp.tm_wdt, &full[s], 0, c0);
          tc::tma_load_2d(WtH(s) + 4096, &tp.tm_wdt, &full[s], 32, c0);
        }
      }
      __syncwarp();
    }
  };
  // w6-9: y rows of running tiles [gath_next, upto) (rows of the tile's step)
  const int tg = (int)threadIdx.x - 192;  // 0..127 in the staging group
  const int gslot = (warp - 6) * 8 + lane;
  auto gather = [&](int upto) {
    for (; gath_next < upto; ++gath_next) {
      const int i = gath_next;
      const int q = i / max(my_tiles, 1), j = i - q * my_tiles;
      const int k = q >> 1, rows = rows_of(k);
      const int sy_ = i % kYStages;
      // expect_tx before any complete_tx; the barrier also orders every
      // staging thread's read of the slot's previous tile before the refill
      if (tg == 0) tc::mbar_expect_tx(&yfull[sy_], kY);
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (lane < 8) {
        const unsigned* pr = perm + (long long)(r.sie0 + k) * a.B;
        int rw[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int rr = 4 * gslot + u;
          rw[u] = (int)pr[rr < rows ? rr : 0];
        }
        tc::tma_gather4(Yraw(sy_) + 512 * gslot, &tp.tm_y, &yfull[sy_], col0(j), rw[0], rw[1], rw[2], rw[3]);
      }
    }
  };

  if (warp == 0) produce(min(kStages, nphase * my_tiles));
  if (warp >= 6) gather(min(kYStages, nphase * my_tiles));

  double mae_e[4] = {0.0, 0.0, 0.0, 0.0};
  int q_done = 0;  // phases executed
  const bool stamp = r.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
#define WSTAMP(slot) do { if (stamp) r.prof[512 * k + (slot)] = gtimer(); } while (0)
  for (int q = 0; q < nphase; ++q) {
    q_done = q + 1;
    const int k = q >> 1;
    const bool ph2 = (q & 1) != 0;
    WSTAMP(ph2 ? 2 : 0);
    const int rows = rows_of(k);
    const int i0 = q * my_tiles, i1 = i0 + my_tiles;
    const int nxt_end = min(i1 + kStages, nphase * my_tiles);
    if (warp == 0) {
      // ------------------------------------------------ TMA producer --
      produce(i1);
      produce(nxt_end);  // the next phase's first tiles (stages free once this phase's MMAs retire)
    } else if (warp == 1) {
      // ---------------------------------------------------- MMA issuer --
      if (lane == 0 && my_tiles > 0) {
        const uint32_t i_enc = tc::idesc_tf32(128, 64, 0, 0);
        const uint32_t i_dec = tc::idesc_tf32(128, 32, 0, 0);
        if (!ph2) {
          for (int i = i0; i < i1; ++i) {
            const int s = i % kStages;
            mbar_wait_to(&split_done[s], (uint32_t)(i / kStages) & 1u);
            tc::tc_fence_after();
            const uint32_t weh = tc::smem_u32(WeH(s)), wel = tc::smem_u32(WeL(s));
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t bh = tc::sdesc_sw128(weh + 32 * kk, 16, 1024);
              tc::mma_tf32_ts(T + kPacc, T + tYh(s) + 8 * kk, bh, i_enc, (i > i0 || kk > 0) ? 1u : 0u);
              if (kPrecise) {
                tc::mma_tf32_ts(T + kPacc, T + tYl(s) + 8 * kk, bh, i_enc, 1u);
                tc::mma_tf32_ts(T + kPacc, T + tYh(s) + 8 * kk, tc::sdesc_sw128(wel + 32 * kk, 16, 1024), i_enc,
                                1u);
              }
            }
            tc::tc_commit(&empty[s]);
          }
          if (r.prof && blockIdx.x == 0) r.prof[512 * k + 16] = gtimer();
        } else {
          mbar_wait_to(&h_ready, hr_par);
          if (r.prof && blockIdx.x == 0) r.prof[512 * k + 17] = gtimer();
          tc::tc_fence_after();
          auto mma3 = [&](int i) {
            const int s = i % kStages;
            tc::tc_fence_after();
            const uint32_t wdh = tc::smem_u32(WdH(s)), wdl = tc::smem_u32(WdL(s));
            for (int kk = 0; kk < 4; ++kk) {
              tc::mma_tf32_ts(T + kPacc, T + tYl(s) + 8 * kk, tc::sdesc_sw128(wdh + 32 * kk, 16, 1024), i_enc,
                              (i > i0 || kk > 0) ? 1u : 0u);
              if (kPrecise)
                tc::mma_tf32_ts(T + kPacc, T + tYl(s) + 8 * kk, tc::sdesc_sw128(wdl + 32 * kk, 16, 1024), i_enc,
                                1u);
            }
            tc::tc_commit(&empty[s]);
          };
          auto mma2 = [&](int i, int ob) {
            const int s = i % kStages;
            tc::tc_fence_after();
            const uint32_t Od = T + kO0 + 32u * (uint32_t)ob;
            const uint32_t wth = tc::smem_u32(WtH(s)), wtl = tc::smem_u32(WtL(s));
            for (int kk = 0; kk < 8; ++kk) {
              const uint32_t boff = (kk / 4) * 4096 + 32 * (kk % 4);
              const uint64_t bh = tc::sdesc_sw128(wth + boff, 16, 1024);
              tc::mma_tf32_ts(Od, T + kHhi + 8 * kk, bh, i_dec, kk > 0 ? 1u : 0u);
              if (kPrecise) {
                tc::mma_tf32_ts(Od, T + kHlo + 8 * kk, bh, i_dec, 1u);
                tc::mma_tf32_ts(Od, T + kHhi + 8 * kk, tc::sdesc_sw128(wtl + boff, 16, 1024), i_dec, 1u);
              }
            }
            tc::tc_commit(&ofull[ob]);
          };
          // dynamic order: MMA3 of a tile as soon as its S is ready (frees
          // the stage), MMA2 of the next tile once staged and an O buffer is free
          int n2 = i0, n3 = i0;
          while (n3 < i1) {
            bool issued = false;
            if (n3 < n2) {
              // sready is arrived once per phase-2 tile: indexed by the phase-2 tile count
              const int o3 = o_run + (n3 - i0);
              if (tc::mbar_test(&sready[o3 % kStages], (uint32_t)(o3 / kStages) & 1u)) {
                TSTAMP(k, n3 - i0, 4);
                mma3(n3++);
                issued = true;
              }
            }
            if (n2 < i1) {
              const int s = n2 % kStages;
              const int oi = o_run + (n2 - i0);
              const bool staged = tc::mbar_test(&split_done[s], (uint32_t)(n2 / kStages) & 1u);
              const bool obuf = oi < 2 || tc::mbar_test(&oempty[oi & 1], ((uint32_t)(oi >> 1) & 1u) ^ 1u);
              if (staged && obuf) {
                mma2(n2, oi & 1);
                TSTAMP(k, n2 - i0, 2);
                ++n2;
                issued = true;
              }
            }
            if (!issued) __nanosleep(20);
          }
          if (r.prof && blockIdx.x == 0) r.prof[512 * k + 18] = gtimer();
        }
        tc::tc_commit(&done);
      }
      __syncwarp();
    } else if (warp >= 2 && warp < 6) {
      // ------------------------------------------------------ epilogue --
      const int quad = warp & 3;
      const int rr = quad * 32 + lane;
      const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
      if (ph2 && my_tiles > 0) {
        // h of this step (the post cluster's next_h, or the row kernel) -> TMEM tf32 hi / lo
        float4 hv[16];
        const float4* hrow = reinterpret_cast<const float4*>(a.h + (long long)rr * kW);
#pragma unroll
        for (int u = 0; u < 16; ++u) hv[u] = rr < rows ? __ldcg(hrow + u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          float v[32], vl[32];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 x4 = hv[half * 8 + u];
            const float xs[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              v[4 * u + e] = kPrecise ? tc::tf32_hi(xs[e]) : xs[e];
              vl[4 * u + e] = xs[e] - v[4 * u + e];
            }
          }
          tc::tmem_st32(T + lane_addr + kHhi + 32 * half, v);
          if (kPrecise) tc::tmem_st32(T + lane_addr + kHlo + 32 * half, vl);
        }
        tc::tc_fence_before();
        tc::mbar_arrive(&h_ready);
        for (int e = 0; e < 4; ++e) mae_e[e] = 0.0;
        const int out_pad = a.m.out_pad;
        auto load_bias = [&](int j, float4* dst) {
          const int c0 = col0(j);
          const float4* bp = reinterpret_cast<const float4*>(bias_pad + c0);
#pragma unroll
          for (int u = 0; u < 8; ++u) dst[u] = c0 + 4 * u < out_pad ? __ldg(bp + u) : make_float4(0.f, 0.f, 0.f, 0.f);
        };
        float4 bnext[8];
        load_bias(0, bnext);
        for (int i = i0; i < i1; ++i) {
          const int j = i - i0;
          const int s = i % kStages;
          const int oi = o_run + j, ob = oi & 1;
          const int c0 = col0(j);
          float4 bcur[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) bcur[u] = bnext[u];
          if (j + 1 < my_tiles) load_bias(j + 1, bnext);
          mbar_wait_to(&ofull[ob], (uint32_t)(oi >> 1) & 1u);
          tc::tc_fence_after();
          float o[32], yv[32];
          tc::tmem_ld32(T + lane_addr + kO0 + 32u * (uint32_t)ob, o);
          tc::tmem_ld32(T + lane_addr + tYh(s), yv);  // raw y (phase 2 stages y unsplit)
          const int nvalid = rr < rows ? min(kTileN, out - c0) : 0;
          float tsum[4] = {0.f, 0.f, 0.f, 0.f};
          float sv[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const float bq[4] = {bcur[c / 4].x, bcur[c / 4].y, bcur[c / 4].z, bcur[c / 4].w};
            const float of = o[c] + bq[c % 4];  // mlp.hpp:209-213
            const bool ok = c < nvalid;
            tsum[c % 4] += ok ? fabsf(of - yv[c]) : 0.0f;  // loss.hpp:25-41
            sv[c] = ok ? (of > yv[c] ? 1.0f : (of < yv[c] ? -1.0f : 0.0f)) : 0.0f;
          }
          tc::tmem_st32(T + lane_addr + tYl(s), sv);
          tc::tc_fence_before();
          tc::mbar_arrive(&oempty[ob]);
          tc::mbar_arrive(&sready[oi % kStages]);
          if (r.prof && blockIdx.x == 0 && rr == 0 && (j == 0 || j == 5)) r.prof[512 * k + (j == 0 ? 23 : 24)] = gtimer();
          if (rr == 0) TSTAMP(k, j, 3);
#pragma unroll
          for (int e = 0; e < 4; ++e) mae_e[e] += (double)tsum[e];
        }
      }
      // partials of this phase out
      float* P = (ph2 ? a.P_dec : a.P_enc) + ((long long)blockIdx.x * a.B + rr) * kW;
      if (my_tiles > 0) {
        mbar_wait_to(&done, done_par);
        tc::tc_fence_after();
      }
      for (int half = 0; half < 2; ++half) {
        float v[32];
        if (my_tiles > 0) tc::tmem_ld32(T + lane_addr + kPacc + 32 * half, v);
        else
          for (int u = 0; u < 32; ++u) v[u] = 0.0f;
        if (rr < rows)
          for (int u = 0; u < 32; u += 4)
            *reinterpret_cast<float4*>(P + 32 * half + u) = make_float4(v[u], v[u + 1], v[u + 2], v[u + 3]);
      }
      tc::tc_fence_before();
      if (r.prof && blockIdx.x == 0 && rr == 0) r.prof[512 * k + (ph2 ? 20 : 19)] = gtimer();
      if (r.prof && ph2 && rr == 0) r.prof[512 * k + 128 + blockIdx.x] = gtimer();
      if (ph2) {
        red[rr] = (mae_e[0] + mae_e[1]) + (mae_e[2] + mae_e[3]);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (rr == 0) {
          double t = 0.0;
          for (int u = 0; u < 128; ++u) t += red[u];
          a.mae_part[blockIdx.x] = t;
        }
      }
    } else {
      // --------------------------------------------- gather + tf32 split --
      const int quad = warp & 3;
      const int rr = quad * 32 + lane;
      const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
      auto split = [&](unsigned char* hi_p, unsigned char* lo_p, int n4) {
        float4* hp = reinterpret_cast<float4*>(hi_p);
        float4* lp = reinterpret_cast<float4*>(lo_p);
#pragma unroll 4
        for (int idx = tg; idx < n4; idx += 128) {
          const float4 v = hp[idx];
          const float4 h = make_float4(tc::tf32_hi(v.x), tc::tf32_hi(v.y), tc::tf32_hi(v.z), tc::tf32_hi(v.w));
          hp[idx] = h;
          lp[idx] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        }
      };
      for (int i = i0; i < i1; ++i) {
        const int s = i % kStages;
        const int sy_ = i % kYStages;
        mbar_wait_to(&yfull[sy_], (uint32_t)(i / kYStages) & 1u);
        mbar_wait_to(&full[s], (uint32_t)(i / kStages) & 1u);
        {
          const unsigned char* yrow = Yraw(sy_) + rr * 128;
          float v[32], vl[32];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint32_t off = (uint32_t)(((u ^ (rr & 7)) & 7) << 4);
            const float4 y4 = *reinterpret_cast<const float4*>(yrow + off);
            const float ys[4] = {y4.x, y4.y, y4.z, y4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              v[4 * u + e] = (kPrecise && !ph2) ? tc::tf32_hi(ys[e]) : ys[e];
              vl[4 * u + e] = ys[e] - v[4 * u + e];
            }
          }
          tc::tmem_st32(T + lane_addr + tYh(s), v);
          if (kPrecise && !ph2) tc::tmem_st32(T + lane_addr + tYl(s), vl);
        }
        // every staging thread has read slot sy_: refill it (tiles of this
        // phase, then the next phase's first ones)
        gather(min(i + 1 + kYStages, nphase * my_tiles));
        if (kPrecise) {
          if (!ph2) {
            split(WeH(s), WeL(s), kWt / 16);
          } else {
            split(WdH(s), WdL(s), kWt / 16);
            split(WtH(s), WtL(s), kWt / 16);
          }
          tc::fence_proxy_async();
        }
        tc::tc_fence_before();
        tc::mbar_arrive(&split_done[s]);
        if (ph2 && r.prof && blockIdx.x == 0 && tg == 0 && (i - i0 == 0 || i - i0 == 5))
          r.prof[512 * k + (i - i0 == 0 ? 25 : 26)] = gtimer();
        if (ph2 && tg == 0) TSTAMP(k, i - i0, 1);
      }
    }
    if (my_tiles > 0) done_par ^= 1u;
    if (ph2) {
      o_run += my_tiles;
      hr_par ^= 1u;
    }

    // ---- phase end: grid-wide fixed-order reduction of this phase's partials ----
    if (ph2) WSTAMP(3);
    if (ph2 && r.prof && blockIdx.x == 0 && threadIdx.x == 64) r.prof[512 * k + 299] = gtimer();
    if (ph2 && r.prof) {
      __syncthreads();
      if (threadIdx.x == 0) r.prof[512 * k + 300 + blockIdx.x] = gtimer();
    }
    grid_sync_t(a.grid_bar, (unsigned)S, sy, ++bar_epoch);
    WSTAMP(ph2 ? 22 : 21);
    {
      const int q_all = rows * (kW / 4);  // float4 outputs of P_enc or P_dec
      const int lo = (int)((long long)q_all * blockIdx.x / S);
      const int hi = (int)((long long)q_all * (blockIdx.x + 1) / S);
      float4* stage = reinterpret_cast<float4*>(sm + kRedOff);                  // [S][kMaxQ]
      float4* part = reinterpret_cast<float4*>(sm + kRedOff) + kMaxS * kMaxQ;  // [kG][kMaxQ]
      const int g = threadIdx.x / 32, o = threadIdx.x % 32;  // o < nq <= kMaxQ active
      const long long pstride4 = (long long)a.B * kW / 4;
      const float4* P4 = reinterpret_cast<const float4*>(ph2 ? a.P_dec : a.P_enc);
      // this CTA's slice [lo, hi) in chunks of kMaxQ outputs (one chunk when
      // S >= 128): every partial's chunk by one bulk copy (TMA engine) per
      // source CTA, then summed in ascending partial order per group
      for (int c0 = lo; c0 < hi; c0 += kMaxQ) {
        const int nq = min(kMaxQ, hi - c0);
        if (threadIdx.x == 0) tc::mbar_expect_tx(&rbar, (uint32_t)(S * nq * 16));
        __syncthreads();
        if ((int)threadIdx.x < S) {
          asm volatile("fence.proxy.async.global;" ::: "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  tc::smem_u32(stage + threadIdx.x * kMaxQ)),
              "l"(P4 + threadIdx.x * pstride4 + c0), "r"(nq * 16), "r"(tc::smem_u32(&rbar))
              : "memory");
        }
        mbar_wait_to(&rbar, rbar_par);
        rbar_par ^= 1u;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        if (o < nq)
          for (int sidx = g; sidx < S; sidx += kG) {
            const float4 v = stage[sidx * kMaxQ + o];
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
          }
        if (o < kMaxQ) part[g * kMaxQ + o] = acc;
        __syncthreads();
        if (g == 0 && o < nq) {
          float4 t = part[o];
          for (int u = 1; u < kG; ++u) {
            const float4 w = part[u * kMaxQ + o];
            t.x += w.x;
            t.y += w.y;
            t.z += w.z;
            t.w += w.w;
          }
          float4* dst = reinterpret_cast<float4*>(ph2 ? r.red_dec[k & 1] : r.red_enc[k & 1]);
          dst[c0 + o] = t;
          __threadfence();
        }
        __syncthreads();  // stage / part are refilled by the next chunk
      }
      if (ph2 && blockIdx.x == 0 && warp == 0) {  // forward-MAE total: strided partials, fixed xor tree
        double v[5];
#pragma unroll
        for (int u = 0; u < 5; ++u) v[u] = lane + 32 * u < S ? __ldcg(a.mae_part + lane + 32 * u) : 0.0;
        double t = (((v[0] + v[1]) + v[2]) + v[3]) + v[4];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        if (lane == 0) {
          *r.mae_total[k & 1] = t;
          __threadfence();
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ph2 ? &sy->dec_done : &sy->enc_done, 1ull);
      }
      WSTAMP(ph2 ? 4 : 1);
    }
    // ---- before phase 2: the epilogue warps wait for this step's h (post
    // cluster / row kernel); the producer and the staging warps run on into
    // phase 2 (the MMA warp waits on h_ready, which the epilogue arrives on) ----
    if (!ph2 && warp >= 2 && warp < 6) {
      if (threadIdx.x == 64) {
        s_go = wait_counter(&sy->h_done, (unsigned long long)kStreamSignalers * (k + 1), sy, 4) ? 1 : 0;
        if (r.prof && blockIdx.x == 0) r.prof[512 * k + 5] = gtimer();
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    // a failed wait (abort / timeout): every CTA sees the flags at the same
    // grid barrier, so all leave together after the next one
    if (ph2) {
      grid_sync_t(a.grid_bar, (unsigned)S, sy, ++bar_epoch);
      if (threadIdx.x == 0) s_go = (ld_acquire_i(&sy->abort) | ld_acquire_i(&sy->error)) ? 0 : 1;
      __syncthreads();
      if (!s_go) break;
    }
  }
  // a run stopped early (abort / timeout) may have next-phase copies in
  // flight: let them land before the CTA's shared memory is released
  {
    const int consumed = q_done * my_tiles;
    if (warp == 0 && lane == 0)
      for (int i = consumed; i < prod_next; ++i) mbar_wait_to(&full[i % kStages], (uint32_t)(i / kStages) & 1u);
    if (warp >= 6 && tg == 0)
      for (int i = consumed; i < gath_next; ++i) mbar_wait_to(&yfull[i % kYStages], (uint32_t)(i / kYStages) & 1u);
  }
#undef WSTAMP
#undef TSTAMP
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(T);
}

// ----------------------------------------------------------------- host --
bool wide_ps_supported(const StepArgs& a, int S) {
  // every CTA owns >= 1 column tile (S <= tiles); the reduction walks its
  // output slice in chunks of kMaxQ
  return a.m.E1 == wp::kW && a.m.D == wp::kW && a.B <= 128 && a.m.out >= wp::kTileN && S >= 1 &&
         S <= (int)wp::kMaxS && S <= (a.m.out + wp::kTileN - 1) / wp::kTileN;
}

static PerDevice g_wide_ps_attr;

/// Loads the streamed step's wide kernels and sets their attributes. Must run
/// before a run starts: with lazy module loading, loading a kernel while the
/// post cluster spins would wait for that cluster to finish (measured: the
/// wide pass started only after the cluster's 2 s hand-off timeout).
void prepare_wide_ps() {
  g_wide_ps_attr.once([] {
    cudaFuncSetAttribute(k_wide_ps<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, wp::kSmem);
    cudaFuncSetAttribute(k_wide_ps<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, wp::kSmem);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_wide_ps<true>);
    cudaFuncGetAttributes(&fa, k_wide_ps<false>);
  });
}

void launch_wide_ps(const WideTcParamsHost& p, const StepArgs& a, const StreamArgs& r, int S, cudaStream_t s) {
  prepare_wide_ps();
  WidePsParams tp;
  std::memcpy(&tp, p.maps, sizeof tp);
  void* args[] = {(void*)&tp, (void*)&a, (void*)&r, (void*)&p.bias_pad};
  const void* fn = p.precise ? (const void*)k_wide_ps<true> : (const void*)k_wide_ps<false>;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(S);
  cfg.blockDim = dim3(wp::kThreads);
  cfg.dynamicSmemBytes = wp::kSmem;
  cfg.stream = s;
  // Not a cooperative launch: a cooperative grid does not start while the
  // post cluster (another kernel) is resident (measured: it waited for the
  // cluster to exit). The grid is exactly the SMs the cluster leaves free at
  // one CTA per SM (shared memory), so every CTA is resident at once in
  // practice; the grid barrier's timeout turns any exception into an error.
  cudaLaunchAttribute at[1];
  int nat = 0;
  if (p.l2_hit > 0.0f) {
    at[0].id = cudaLaunchAttributeAccessPolicyWindow;
    at[0].val.accessPolicyWindow.base_ptr = p.l2_base;
    at[0].val.accessPolicyWindow.num_bytes = p.l2_bytes;
    at[0].val.accessPolicyWindow.hitRatio = p.l2_hit;
    at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    nat = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = nat;
  const cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e != cudaSuccess) throw std::runtime_error(std::string("streamed wide pass launch: ") + cudaGetErrorString(e));
}

static_assert(sizeof(WidePsParams) == 4 * 128, "CUtensorMap packing");

}  // namespace ltfb_dev
