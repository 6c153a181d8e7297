// The wide pass of a training step on the 5th-gen tensor cores, with
// 64-column tiles (round 2b). One kernel body serves both step modes:
//
//   streamed (kStream = true): one persistent kernel per run of steps inside
//     an epoch, beside the persistent post cluster (k_post_loop), two phases
//     per step handed over through StepSync;
//   launched (kStream = false): one cooperative launch per step (CUDA graphs,
//     the host-buffer e2e path, profilers), the two phases back to back.
//
// Both run the same tile -> CTA map, MMA sequence and fixed-order split-K
// reduction, so the two step modes compute the same bits.
//
//   phase 1 (y, We)   P_enc += Y We          enc layer-0 split-K partials
//                                            (D-step real latents,
//                                            train_ops.hpp:160)
//   phase 2 (h, Wd)   O = h Wd ; d = O + b - Y ; sum |d| ; S = sign d ;
//                     P_dec += S Wd^T        (train_ops.hpp:100-104,
//                                            loss.hpp:25-41, mlp.hpp:278)
//
// Why 64 columns (the round-1 / round-2a kernels used 32): a tcgen05 MMA with
// N = 32 costs about what N = 64 costs, and the per-tile stage cycle (TMA ->
// split -> MMA2 -> epilogue -> MMA3) was latency-bound at 1.8 us per 32
// columns. Here a tile of 64 columns moves 64 KB of weights per stage (hi and
// lo tf32 parts of WdT and Wd, or of WeT plus the y block), and:
//   - phase 2 reads its y rows straight from L2 in the epilogue (they were
//     gathered from HBM in phase 1 of the same step), so no y slot is staged;
//   - S overwrites the O buffer it came from in TMEM and is MMA3's A operand
//     there; the O buffer is released by MMA3's commit;
//   - phase 1's A operand is the gathered y block itself (tf32 hi written in
//     place by the split warps); its lo part goes to a TMEM slot per stage.
//
// fp32 parity ("3xTF32", kPrecise): every fp32 operand is split into tf32 hi
// + lo and the products accumulate hi*hi + lo*hi + hi*lo in f32 TMEM per
// K-step; S is exact in tf32, so MMA3 needs S*hi + S*lo. kPrecise = false is
// the 1xTF32 perf mode.
//
// Warp roles (320 threads): w0 TMA producer (weights by lane 0, y row
// gathers by all lanes: rows 4l .. 4l+3), w1 MMA issuer + TMEM owner, w2-5
// epilogue (TMEM lane quadrants), w6-9 tf32 split. Ring counters run on
// across phases and steps, so the next phase's first stages load under the
// grid barrier and the reduction.
#include <cuda.h>

#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "kernels.hpp"
#include "stream_sync.cuh"
#include "tc_ptx.cuh"

namespace ltfb_dev {

namespace w2 {
constexpr int kTileN = 64;
constexpr int kW = 64;
constexpr uint32_t kYBlk = 16384;   // [128 x 32] f32, SW128 (one y K-block)
constexpr uint32_t kWBlk = 8192;    // [64 x 32] f32, SW128 (one weight K-block)
constexpr uint32_t kStage = 65536;  // phase 1: Y (2 blk) | WeT hi | WeT lo; phase 2: WdT hi | WdT lo | Wd hi | Wd lo
constexpr int kStages = 3;
constexpr int kThreads = 320;
constexpr int kG = 9;       // reduction groups: warps 1-9 (the producer warp prefetches meanwhile)
constexpr int kMaxQ = 32;   // float4 outputs per reduction chunk
constexpr int kMaxS = 153;  // <= kG * 17 partials
// phase 2's y tiles land here (one [128 x 32] block per slot, TMA gather4)
// and are copied into the stage's TMEM y slot; the reduction scratch and the
// MAE row sums reuse the slots (idle at phase ends)
constexpr uint32_t kLandOff = kStages * kStage;
constexpr uint32_t kPartOff = kLandOff;
constexpr uint32_t kRedOff = kLandOff + kYBlk;
constexpr uint32_t kSmem = kLandOff + 2 * kYBlk + 1024;
static_assert(kG * kMaxQ * 16 <= kYBlk, "reduction scratch in a landing slot");
// TMEM columns: split-K accumulator (P_enc in phase 1, P_dec in phase 2),
// two O / S buffers, h hi / lo, a y slot per stage (phase 1: y lo; phase 2:
// the raw y tile the epilogue compares against)
constexpr uint32_t kPacc = 0, kO0 = 64, kHhi = 192, kHlo = 256, kYlo = 320;
static_assert(kYlo + 64 * kStages <= 512, "TMEM columns");
static_assert(kSmem <= 227 * 1024, "shared memory");
// launched mode's grid barrier: its own region of StepArgs::grid_bar (the
// streamed barrier uses [64, 96 + 32 * 160)); word 0 the epoch base the next
// launch starts from, then the arrival counter and one 128-B flag per CTA
constexpr int kLaunchBar = 5248;
}  // namespace w2

struct Wide2Params {
  CUtensorMap tm_y, tm_wet, tm_wd, tm_wdt;  // y rows (gather4), WeT / Wd [64 x out_pad], WdT [out_pad x 64] (box 64 rows)
};

/// Grid barrier over `n` CTAs that are all resident: arrival is one release
/// reduction on cnt, and every CTA's leader polls cnt itself (acquire) until
/// it reaches n * epoch (no flag fan-out by the last arriver: measured ~4 us
/// from the last arrival to the release with per-CTA flags after a fence).
/// `epoch` only grows; the comparison is modular. A missing CTA raises
/// sy->error after the timeout (streamed mode) instead of hanging the GPU;
/// launched mode traps.
/// kFull: every thread of the CTA takes part (leader thread 0); else warps
/// 1-9 only (named barrier 3, leader thread 32): the phase-end barrier, which
/// the producer warp skips so its next-phase prefetch never delays it.
template <bool kFull>
__device__ __forceinline__ void grid_sync2(unsigned* cnt, unsigned* flags, unsigned n, StepSync* sy,
                                           unsigned epoch) {
  (void)flags;
  if (kFull) __syncthreads();
  else asm volatile("bar.sync 3, 288;" ::: "memory");
  if (threadIdx.x == (kFull ? 0u : 32u)) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    const unsigned target = n * epoch;
    const unsigned long long t0 = gtimer();
    unsigned cur;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(cnt) : "memory");
      if ((int)(cur - target) >= 0) break;
      if (gtimer() - t0 > kStreamTimeoutNs) {
        if (sy) {
          if (atomicCAS(&sy->error, 0, 2) == 0) sy->err_site = 6;
          break;
        }
        __trap();
      }
    }
  }
  if (kFull) __syncthreads();
  else asm volatile("bar.sync 3, 288;" ::: "memory");
}

/// 8 floats (one 32-B sector) through the non-coherent path, 32-B aligned;
/// zeros when !ok.
__device__ __forceinline__ void ld_nc_v8(const float* p, bool ok, float* v) {
  if (ok) {
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = 0.0f;
  }
}

/// 8 floats through L2 (.cg: data another kernel wrote during this one), 32-B aligned.
__device__ __forceinline__ void ld_cg_v8(const float* p, bool ok, float* v) {
  if (ok) {
    asm volatile("ld.global.cg.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = 0.0f;
  }
}

/// mbarrier wait that traps after 2 x kStreamTimeoutNs: a broken hand-off
/// ends the kernel with a launch failure instead of a hang.
__device__ __forceinline__ void mbar_wait2(uint64_t* bar, uint32_t parity) {
  if (tc::mbar_try_wait(bar, parity)) return;
  const unsigned long long t0 = gtimer();
  while (!tc::mbar_try_wait(bar, parity))
    if (gtimer() - t0 > 2 * kStreamTimeoutNs) __trap();
}

template <bool kPrecise, bool kStream>
__global__ void __launch_bounds__(w2::kThreads, 1)
    k_wide2(const __grid_constant__ Wide2Params tp, const __grid_constant__ StepArgs a,
            const __grid_constant__ StreamArgs r, const float* __restrict__ bias_pad) {
  using namespace w2;
  if (a.ctr->aborted) return;  // (streamed: the post cluster leaves at once too)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kStages], split_done[kStages], empty[kStages];
  __shared__ uint64_t ofull[2], oempty[2], sready[2], h_ready, done, lfull;
  __shared__ uint32_t tmem_base;
  __shared__ int s_go;
  __shared__ unsigned s_base;

  StepSync* sy = kStream ? r.sync : nullptr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int out = a.m.out, out_pad = a.m.out_pad;
  const int ntiles = (out + kTileN - 1) / kTileN;
  const int S = (int)gridDim.x;
  const int lcta = ((int)blockIdx.x + r.tile_rot) % S;  // column-tile owner index (A/B: LTFB_W2_ROT)
  // owner lcta holds tiles lcta, lcta + S, ... (base_tiles of them), except
  // that the first two 'short' owners (lcta L0, L0 + 1: the rotation places
  // them on the SMs that run tiles slowest) hand their last tile_donate tiles
  // to the next 2 * tile_donate short owners, one each (the same map in both
  // step modes: it fixes which tiles a CTA's partial sums)
  const int base_tiles = ntiles > lcta ? (ntiles - 1 - lcta) / S + 1 : 0;
  int my_tiles = base_tiles, extra_tile = -1;
  {
    const int dn = r.tile_donate, n_short = ntiles % S ? S - ntiles % S : 0, L0 = S - n_short;
    if (dn > 0 && n_short >= 2 * (1 + dn) && base_tiles > dn && lcta >= L0) {
      const int o = lcta - L0;
      if (o < 2) {
        my_tiles -= dn;
      } else if (o < 2 + 2 * dn) {
        const int rr = o - 2;
        extra_tile = (L0 + rr / dn) + (base_tiles - 1 - rr % dn) * S;
        my_tiles += 1;
      }
    }
  }
  const int nsteps = kStream ? r.n : 1;
  const int sie0 = kStream ? r.sie0 : (int)a.ctr->step_in_epoch;
  const unsigned epoch = kStream ? r.epoch : a.ctr->epoch;
  const unsigned* perm = a.perm[epoch & 1u];
  const float* ysrc = a.y_identity ? a.yb : a.sy;
  unsigned* bar_cnt = kStream ? a.grid_bar + 64 : a.grid_bar + kLaunchBar + 32;
  unsigned* bar_flags = bar_cnt + 32;
  const int nphase = 2 * nsteps;
  auto col0 = [&](int j) { return (j < base_tiles ? lcta + j * S : extra_tile) * kTileN; };
  auto rows_of = [&](int k) { return min(a.B, a.n_part - (sie0 + k) * a.B); };
  auto nkb_of = [&](int c0) { return c0 + 32 < out ? 2 : 1; };  // y / We / Wd K-blocks inside the matrix
  auto row_index = [&](int k, int rr, int rows) {
    if (a.y_identity) return rr < rows ? rr : 0;
    return (int)perm[(long long)(sie0 + k) * a.B + (rr < rows ? rr : 0)];
  };

  auto stage_ptr = [&](int s) { return sm + s * kStage; };
  auto Yb = [&](int s) { return stage_ptr(s); };                   // y [128 x 64]: 2 K-blocks
  auto WeH = [&](int s) { return stage_ptr(s) + 2 * kYBlk; };      // WeT [64 j x 64 c]: 2 K-blocks
  auto WeL = [&](int s) { return stage_ptr(s) + 2 * kYBlk + 2 * kWBlk; };
  auto WtH = [&](int s) { return stage_ptr(s); };                  // WdT [64 c x 64 j]: 2 K-blocks (j)
  auto WtL = [&](int s) { return stage_ptr(s) + 2 * kWBlk; };
  auto WdH = [&](int s) { return stage_ptr(s) + 4 * kWBlk; };      // Wd [64 j x 64 c]: 2 K-blocks (c)
  auto WdL = [&](int s) { return stage_ptr(s) + 6 * kWBlk; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&split_done[s], 128);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&ofull[b], 1);
      tc::mbar_init(&oempty[b], 1);
      tc::mbar_init(&sready[b], 128);
    }
    tc::mbar_init(&h_ready, 128);
    tc::mbar_init(&done, 1);
    tc::mbar_init(&lfull, 1);
    tc::fence_barrier_init();
    // launched mode: this launch's barrier epochs continue from the last one
    s_base = kStream ? 0u : *reinterpret_cast<volatile unsigned*>(a.grid_bar + kLaunchBar);
    if (kStream && blockIdx.x == 0) r.sync->t_wide0 = gtimer();
    if (kStream && r.prof) {  // SM of every CTA, after the run's step rows (LTFB_STREAM_PROF)
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      r.prof[512ll * r.n + blockIdx.x] = smid;
    }
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
  unsigned bar_epoch = s_base;

  unsigned long long* prof = kStream ? r.prof : nullptr;
#define TSTAMP(kk, j, e) do { if (prof && blockIdx.x == 0 && (j) < 8) prof[512 * (kk) + 32 + 6 * (j) + (e)] = gtimer(); } while (0)
  // ---- per-role state that runs on across phases ----
  int prod_next = 0;  // w0: next running tile index whose operands are issued
  int prod_k = -1;    // w0: step whose gather rows are cached in rw
  int rw[4] = {0, 0, 0, 0};
  uint32_t hr_par = 0, done_par = 0;
  int o_run = 0;      // running phase-2 tile count (O / S double buffer)
  uint32_t l_par = 0; // w6-9: landing-slot phase

  // w0: issue the operands of running tiles [prod_next, upto)
  auto produce = [&](int upto) {
    for (; prod_next < upto; ++prod_next) {
      const int i = prod_next;
      const int q = i / max(my_tiles, 1), j = i - q * my_tiles;
      const int s = i % kStages;
      if (i >= kStages) mbar_wait2(&empty[s], ((uint32_t)(i / kStages) & 1u) ^ 1u);
      const int c0 = col0(j), nkb = nkb_of(c0);
      if ((q & 1) == 0) {  // phase 1: WeT blocks + the y rows of the tile's step
        const int k = q >> 1;
        if (k != prod_k) {
          const int rows = rows_of(k);
#pragma unroll
          for (int u = 0; u < 4; ++u) rw[u] = row_index(k, 4 * lane + u, rows);
          prod_k = k;
        }
        if (lane == 0) {
          tc::mbar_expect_tx(&full[s], (uint32_t)nkb * (kYBlk + kWBlk));
          for (int kb = 0; kb < nkb; ++kb) tc::tma_load_2d(WeH(s) + kb * kWBlk, &tp.tm_wet, &full[s], c0 + 32 * kb, 0);
        }
        __syncwarp();
        for (int kb = 0; kb < nkb; ++kb)
          tc::tma_gather4(Yb(s) + kb * kYBlk + 512 * lane, &tp.tm_y, &full[s], c0 + 32 * kb, rw[0], rw[1], rw[2], rw[3]);
      } else if (lane == 0) {  // phase 2: WdT (MMA2) and Wd (MMA3)
        TSTAMP(q >> 1, j, 0);
        tc::mbar_expect_tx(&full[s], 2 * kWBlk + (uint32_t)nkb * kWBlk);
        for (int kb = 0; kb < 2; ++kb) tc::tma_load_2d(WtH(s) + kb * kWBlk, &tp.tm_wdt, &full[s], 32 * kb, c0);
        for (int kb = 0; kb < nkb; ++kb) tc::tma_load_2d(WdH(s) + kb * kWBlk, &tp.tm_wd, &full[s], c0 + 32 * kb, 0);
      }
      __syncwarp();
    }
  };

  if (warp == 0) produce(min(kStages, nphase * my_tiles));

  double mae_e[4] = {0.0, 0.0, 0.0, 0.0};
  int q_done = 0;
  const bool stamp = prof != nullptr && blockIdx.x == 0 && threadIdx.x == 32;
#define WSTAMP(slot) do { if (stamp) prof[512 * k + (slot)] = gtimer(); } while (0)
  for (int q = 0; q < nphase; ++q) {
    q_done = q + 1;
    const int k = q >> 1;
    const bool ph2 = (q & 1) != 0;
    WSTAMP(ph2 ? 2 : 0);
    const int rows = rows_of(k);
    const int i0 = q * my_tiles, i1 = i0 + my_tiles;
    if (warp == 0) {
      // ------------------------------------------------ TMA producer --
      // phase 2: the gather rows of the next step's phase 1 now (perm loads
      // off the phase end), so the prefetch below is only TMA issues
      if (ph2 && k + 1 < nsteps && prod_k != k + 1) {
        const int rows1 = rows_of(k + 1);
#pragma unroll
        for (int u = 0; u < 4; ++u) rw[u] = row_index(k + 1, 4 * lane + u, rows1);
        prod_k = k + 1;
      }
      produce(i1);
      produce(min(i1 + kStages, nphase * my_tiles));  // the next phase's first tiles, under the barrier
    } else if (warp == 1) {
      // ---------------------------------------------------- MMA issuer --
      if (lane == 0 && my_tiles > 0) {
        const uint32_t id64 = tc::idesc_tf32(128, 64, 0, 0);
        if (!ph2) {
          for (int i = i0; i < i1; ++i) {
            const int s = i % kStages;
            const int nkb = nkb_of(col0(i - i0));
            mbar_wait2(&split_done[s], (uint32_t)(i / kStages) & 1u);
            tc::tc_fence_after();
            const uint32_t yb = tc::smem_u32(Yb(s)), weh = tc::smem_u32(WeH(s)), wel = tc::smem_u32(WeL(s));
            for (int kb = 0; kb < nkb; ++kb)
              for (int kk = 0; kk < 4; ++kk) {
                const uint64_t ah = tc::sdesc_sw128(yb + kb * kYBlk + 32 * kk, 16, 1024);
                const uint64_t bh = tc::sdesc_sw128(weh + kb * kWBlk + 32 * kk, 16, 1024);
                tc::mma_tf32_ss(T + kPacc, ah, bh, id64, (i > i0 || kb > 0 || kk > 0) ? 1u : 0u);
                if (kPrecise) {
                  tc::mma_tf32_ts(T + kPacc, T + kYlo + 64 * s + 32 * kb + 8 * kk, bh, id64, 1u);
                  tc::mma_tf32_ss(T + kPacc, ah, tc::sdesc_sw128(wel + kb * kWBlk + 32 * kk, 16, 1024), id64, 1u);
                }
              }
            tc::tc_commit(&empty[s]);
          }
          if (prof && blockIdx.x == 0) prof[512 * k + 16] = gtimer();
        } else {
          mbar_wait2(&h_ready, hr_par);
          if (prof && blockIdx.x == 0) prof[512 * k + 17] = gtimer();
          tc::tc_fence_after();
          auto mma2 = [&](int i, int ob) {
            const int s = i % kStages;
            tc::tc_fence_after();
            const uint32_t Od = T + kO0 + 64u * (uint32_t)ob;
            const uint32_t wth = tc::smem_u32(WtH(s)), wtl = tc::smem_u32(WtL(s));
            for (int kb = 0; kb < 2; ++kb)
              for (int kk = 0; kk < 4; ++kk) {
                const uint64_t bh = tc::sdesc_sw128(wth + kb * kWBlk + 32 * kk, 16, 1024);
                const uint32_t hoff = 32 * kb + 8 * kk;
                tc::mma_tf32_ts(Od, T + kHhi + hoff, bh, id64, (kb > 0 || kk > 0) ? 1u : 0u);
                if (kPrecise) {
                  tc::mma_tf32_ts(Od, T + kHlo + hoff, bh, id64, 1u);
                  tc::mma_tf32_ts(Od, T + kHhi + hoff, tc::sdesc_sw128(wtl + kb * kWBlk + 32 * kk, 16, 1024), id64,
                                  1u);
                }
              }
            tc::tc_commit(&ofull[ob]);
          };
          auto mma3 = [&](int i, int ob) {
            const int s = i % kStages;
            const int nkb = nkb_of(col0(i - i0));
            tc::tc_fence_after();
            const uint32_t Sa = T + kO0 + 64u * (uint32_t)ob;
            const uint32_t wdh = tc::smem_u32(WdH(s)), wdl = tc::smem_u32(WdL(s));
            for (int kb = 0; kb < nkb; ++kb)
              for (int kk = 0; kk < 4; ++kk) {
                const uint32_t aoff = 32 * kb + 8 * kk;
                tc::mma_tf32_ts(T + kPacc, Sa + aoff, tc::sdesc_sw128(wdh + kb * kWBlk + 32 * kk, 16, 1024), id64,
                                (i > i0 || kb > 0 || kk > 0) ? 1u : 0u);
                if (kPrecise)
                  tc::mma_tf32_ts(T + kPacc, Sa + aoff, tc::sdesc_sw128(wdl + kb * kWBlk + 32 * kk, 16, 1024), id64,
                                  1u);
              }
            tc::tc_commit(&empty[s]);
            tc::tc_commit(&oempty[ob]);
          };
          // dynamic order: MMA3 of a tile as soon as its S is in TMEM (frees
          // the stage and the buffer), MMA2 of the next tile once its stage
          // is split and an O buffer is free
          int n2 = i0, n3 = i0;
          while (n3 < i1) {
            bool issued = false;
            if (n3 < n2) {
              const int o3 = o_run + (n3 - i0);
              if (tc::mbar_test(&sready[o3 & 1], (uint32_t)(o3 >> 1) & 1u)) {
                TSTAMP(k, n3 - i0, 4);
                mma3(n3++, o3 & 1);
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
          if (prof && blockIdx.x == 0) prof[512 * k + 18] = gtimer();
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
        // h of this step -> TMEM (MMA2's A operand): the raw fp32 row is the
        // tf32 hi part (the MMA ignores the low 13 mantissa bits), lo = x -
        // hi. 32-B loads (L2; the post cluster wrote h after the acquire above)
        {
          const float* hrow = a.h + (long long)rr * kW;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            float v[32], vl[32];
#pragma unroll
            for (int u = 0; u < 4; ++u) ld_cg_v8(hrow + 32 * half + 8 * u, rr < rows, v + 8 * u);
#pragma unroll
            for (int e = 0; e < 32; ++e) vl[e] = v[e] - tc::tf32_hi(v[e]);
            tc::tmem_st32(T + lane_addr + kHhi + 32 * half, v);
            if (kPrecise) tc::tmem_st32(T + lane_addr + kHlo + 32 * half, vl);
          }
        }
        tc::tc_fence_before();
        tc::mbar_arrive(&h_ready);
        for (int e = 0; e < 4; ++e) mae_e[e] = 0.0;
        for (int i = i0; i < i1; ++i) {
          const int j = i - i0;
          const int oi = o_run + j, ob = oi & 1;
          const int c0 = col0(j);
          // O of the tile (MMA2 ran after the split warps put the tile's y
          // into the stage's TMEM y slot)
          mbar_wait2(&ofull[ob], (uint32_t)(oi >> 1) & 1u);
          tc::tc_fence_after();
          if (rr == 0) TSTAMP(k, j, 5);
          const uint32_t Ob = T + lane_addr + kO0 + 64u * (uint32_t)ob;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            float o[32], yv[32];
            tc::tmem_ld32(Ob + 32 * half, o);
            tc::tmem_ld32(T + lane_addr + kYlo + 64 * (i % kStages) + 32 * half, yv);
            const int cb = c0 + 32 * half;
            const int nvalid = rr < rows ? max(0, min(32, out - cb)) : 0;
            float tsum[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              float bq[8];
              ld_nc_v8(bias_pad + cb + 8 * u, cb + 8 * u < out_pad, bq);
#pragma unroll
              for (int e8 = 0; e8 < 8; ++e8) {
                const int c = 8 * u + e8;
                const float yq = yv[c];
                const float of = o[c] + bq[e8];  // mlp.hpp:209-213
                const bool ok = c < nvalid;
                tsum[c & 3] += ok ? fabsf(of - yq) : 0.0f;  // loss.hpp:25-41
                o[c] = ok ? (of > yq ? 1.0f : (of < yq ? -1.0f : 0.0f)) : 0.0f;  // S over O in place
              }
            }
            tc::tmem_st32(Ob + 32 * half, o);
#pragma unroll
            for (int e = 0; e < 4; ++e) mae_e[e] += (double)tsum[e];
          }
          tc::tc_fence_before();
          tc::mbar_arrive(&sready[ob]);
          if (prof && blockIdx.x == 0 && rr == 0 && (j == 0 || j == 5)) prof[512 * k + (j == 0 ? 23 : 24)] = gtimer();
          if (rr == 0) TSTAMP(k, j, 3);
        }
      }
      // partials of this phase out
      float* P = (ph2 ? a.P_dec : a.P_enc) + ((long long)blockIdx.x * a.B + rr) * kW;
      if (my_tiles > 0) {
        mbar_wait2(&done, done_par);
        tc::tc_fence_after();
      }
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float v[32];
        if (my_tiles > 0) tc::tmem_ld32(T + lane_addr + kPacc + 32 * half, v);
        else
#pragma unroll
          for (int u = 0; u < 32; ++u) v[u] = 0.0f;
        if (rr < rows)
#pragma unroll
          for (int u = 0; u < 32; u += 4)
            *reinterpret_cast<float4*>(P + 32 * half + u) = make_float4(v[u], v[u + 1], v[u + 2], v[u + 3]);
      }
      tc::tc_fence_before();
      if (prof && blockIdx.x == 0 && rr == 0) prof[512 * k + (ph2 ? 20 : 19)] = gtimer();
      if (prof && ph2 && rr == 0) prof[512 * k + 128 + blockIdx.x] = gtimer();
      if (ph2) {
        // the CTA's MAE partial: a fixed xor tree per warp, then the four
        // warp sums in quadrant order (deterministic)
        double* red = reinterpret_cast<double*>(sm + kRedOff);
        double t = (mae_e[0] + mae_e[1]) + (mae_e[2] + mae_e[3]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        if (lane == 0) red[quad] = t;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (rr == 0) a.mae_part[blockIdx.x] = ((red[0] + red[1]) + red[2]) + red[3];
      }
    } else {
      // ----------------------------------------------------- tf32 split --
      const int quad = warp & 3;
      const int rr = quad * 32 + lane;
      const int tg = (int)threadIdx.x - 192;
      const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
      // tf32 split of an fp32 operand block: the raw block stays the hi part
      // (the MMA reads fp32 containers as tf32 by dropping the low 13
      // mantissa bits -- measured bit-identical to writing the masked value,
      // tools/w2_trunc_check.py), lo = x - hi goes to its own block
      auto split = [&](const unsigned char* hi_p, unsigned char* lo_p, int n4) {
        const float4* hp = reinterpret_cast<const float4*>(hi_p);
        float4* lp = reinterpret_cast<float4*>(lo_p);
#pragma unroll 4
        for (int idx = tg; idx < n4; idx += 128) {
          const float4 v = hp[idx];
          lp[idx] = make_float4(v.x - tc::tf32_hi(v.x), v.y - tc::tf32_hi(v.y), v.z - tc::tf32_hi(v.z),
                                v.w - tc::tf32_hi(v.w));
        }
      };
      // phase 2: the y tile of running tile i is gathered into the landing
      // slots during tile i - 1 and copied into the stage's TMEM y slot
      int grw[4] = {0, 0, 0, 0};
      const int gslot = (warp - 6) * 8 + lane;  // lanes 0-7 of each split warp: rows 4 g .. 4 g + 3
      auto issue_y = [&](int j) {  // all 128 split threads call this
        const int c0 = col0(j), nkb = nkb_of(c0);
        if (tg == 0) tc::mbar_expect_tx(&lfull, (uint32_t)nkb * kYBlk);
        asm volatile("bar.sync 2, 128;" ::: "memory");  // expect_tx first; every thread done reading the slots
        if (lane < 8)
          for (int kb = 0; kb < nkb; ++kb)
            tc::tma_gather4(sm + kLandOff + kb * kYBlk + 512 * gslot, &tp.tm_y, &lfull, c0 + 32 * kb, grw[0], grw[1],
                            grw[2], grw[3]);
      };
      if (ph2 && my_tiles > 0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) grw[u] = row_index(k, 4 * gslot + u, rows);
        issue_y(0);
      }
      for (int i = i0; i < i1; ++i) {
        const int s = i % kStages;
        const int c0 = col0(i - i0), nkb = nkb_of(c0);
        mbar_wait2(&full[s], (uint32_t)(i / kStages) & 1u);
        if (ph2) {
          // the tile's raw y rows -> TMEM y slot s (this thread's row), then
          // the landing slots take the next tile's rows
          mbar_wait2(&lfull, l_par);
          l_par ^= 1u;
          for (int kb = 0; kb < nkb; ++kb) {
            const unsigned char* yrow = sm + kLandOff + kb * kYBlk + rr * 128;
            float v[32];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const uint32_t off = (uint32_t)(((u ^ (rr & 7)) & 7) << 4);
              const float4 y4 = *reinterpret_cast<const float4*>(yrow + off);
              v[4 * u + 0] = y4.x;
              v[4 * u + 1] = y4.y;
              v[4 * u + 2] = y4.z;
              v[4 * u + 3] = y4.w;
            }
            tc::tmem_st32(T + lane_addr + kYlo + 64 * s + 32 * kb, v);
          }
          if (i + 1 < i1) issue_y(i + 1 - i0);
        }
        if (kPrecise) {
          if (!ph2) {
            // y: this thread's row of each K-block, hi in place, lo -> TMEM
            for (int kb = 0; kb < nkb; ++kb) {
              const unsigned char* yrow = Yb(s) + kb * kYBlk + rr * 128;
              float vl[32];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const uint32_t off = (uint32_t)(((u ^ (rr & 7)) & 7) << 4);
                const float4 y4 = *reinterpret_cast<const float4*>(yrow + off);
                vl[4 * u + 0] = y4.x - tc::tf32_hi(y4.x);
                vl[4 * u + 1] = y4.y - tc::tf32_hi(y4.y);
                vl[4 * u + 2] = y4.z - tc::tf32_hi(y4.z);
                vl[4 * u + 3] = y4.w - tc::tf32_hi(y4.w);
              }
              tc::tmem_st32(T + lane_addr + kYlo + 64 * s + 32 * kb, vl);
            }
            split(WeH(s), WeL(s), nkb * (int)kWBlk / 16);
          } else {
            split(WtH(s), WtL(s), 2 * (int)kWBlk / 16);
            split(WdH(s), WdL(s), nkb * (int)kWBlk / 16);
          }
          tc::fence_proxy_async();
        }
        tc::tc_fence_before();
        tc::mbar_arrive(&split_done[s]);
        if (ph2 && prof && blockIdx.x == 0 && tg == 0 && (i - i0 == 0 || i - i0 == 5))
          prof[512 * k + (i - i0 == 0 ? 25 : 26)] = gtimer();
        if (ph2 && tg == 0) TSTAMP(k, i - i0, 1);
      }
    }
    if (my_tiles > 0) done_par ^= 1u;
    if (ph2) {
      o_run += my_tiles;
      hr_par ^= 1u;
    }

    // ---- phase end: grid-wide fixed-order reduction of the partials, by
    // warps 1-9 (the producer is already issuing the next phase's first
    // tiles). Streamed: after each phase (the post cluster needs P_enc
    // before phase 2 ends). Launched: once, after phase 2, for both (the
    // post kernel runs after this kernel) -- the phase-1 partials are in
    // global memory before the epilogue loads h, which phase 2's first MMA
    // waits for, so the shared TMEM accumulator is never overwritten early.
    if (kStream || ph2) {
    ++bar_epoch;
    if (warp != 0) {
    if (ph2) WSTAMP(3);
    if (ph2 && prof && blockIdx.x == 0 && threadIdx.x == 64) prof[512 * k + 299] = gtimer();
    if (ph2 && prof && blockIdx.x < 40 && threadIdx.x == 32) prof[512 * k + 472 + blockIdx.x] = gtimer();
    if (ph2 && prof) {
      asm volatile("bar.sync 3, 288;" ::: "memory");
      if (threadIdx.x == 32) prof[512 * k + 300 + blockIdx.x] = gtimer();
    }
    grid_sync2<false>(bar_cnt, bar_flags, (unsigned)S, sy, bar_epoch);
    WSTAMP(ph2 ? 22 : 21);
    if (ph2 && prof && blockIdx.x < 40 && threadIdx.x == 32) prof[512 * k + 432 + blockIdx.x] = gtimer();
    {
      const int q_all = rows * (kW / 4);  // float4 outputs of P_enc or P_dec
      const int lo = (int)((long long)q_all * blockIdx.x / S);
      const int hi = (int)((long long)q_all * (blockIdx.x + 1) / S);
      float4* part = reinterpret_cast<float4*>(sm + kPartOff);  // [kG][kMaxQ]
      const int g = warp - 1, o = lane;
      const long long pstride4 = (long long)a.B * kW / 4;
      // this CTA's slice [lo, hi) of one reduced matrix, in chunks of kMaxQ
      // outputs: thread (g, o) loads partials g, g + kG, ... of output o
      // (every load issued before the adds: one L2 round trip), sums them
      // in ascending order, then the kG group sums are added in group order
      // -- a fixed order, so the result is deterministic and the same in
      // both step modes
      auto reduce = [&](const float* Pm, float* dst) {
        const float4* P4 = reinterpret_cast<const float4*>(Pm);
        for (int c0 = lo; c0 < hi; c0 += kMaxQ) {
          const int nq = min(kMaxQ, hi - c0);
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          if (o < nq) {
            // absent partials re-read partial g and are not added
            float4 v[kMaxS / kG];
#pragma unroll
            for (int u = 0; u < kMaxS / kG; ++u) {
              const int sidx = g + u * kG < S ? g + u * kG : g;
              const float4* src = P4 + sidx * pstride4 + c0 + o;
              asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                           : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w)
                           : "l"(src));
            }
#pragma unroll
            for (int u = 0; u < kMaxS / kG; ++u)
              if (g + u * kG < S) {
                acc.x += v[u].x;
                acc.y += v[u].y;
                acc.z += v[u].z;
                acc.w += v[u].w;
              }
          }
          part[g * kMaxQ + o] = acc;
          asm volatile("bar.sync 3, 288;" ::: "memory");
          if (g == 0 && o < nq) {
            float4 t = part[o];
            for (int u = 1; u < kG; ++u) {
              const float4 w = part[u * kMaxQ + o];
              t.x += w.x;
              t.y += w.y;
              t.z += w.z;
              t.w += w.w;
            }
            reinterpret_cast<float4*>(dst)[c0 + o] = t;  // published by the fence + release below (streamed)
          }
          asm volatile("bar.sync 3, 288;" ::: "memory");  // part is refilled by the next chunk
        }
      };
      if (kStream) reduce(ph2 ? a.P_dec : a.P_enc, ph2 ? r.red_dec[k & 1] : r.red_enc[k & 1]);
      else {
        reduce(a.P_enc, a.scratch + a.L.red_enc);
        reduce(a.P_dec, a.scratch + a.L.red_dec);
      }
      if (!kStream && ph2 && blockIdx.x == 0 && warp == 1) {  // forward-MAE total: strided partials, fixed xor tree
        // (streamed: the post cluster's cyc half sums the partials itself, off this signal's path)
        double v[5];
#pragma unroll
        for (int u = 0; u < 5; ++u) v[u] = lane + 32 * u < S ? __ldcg(a.mae_part + lane + 32 * u) : 0.0;
        double t = (((v[0] + v[1]) + v[2]) + v[3]) + v[4];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        if (lane == 0) *(kStream ? r.mae_total[k & 1] : a.mae_total) = t;
      }
      if (kStream) {
        asm volatile("bar.sync 3, 288;" ::: "memory");
        if (threadIdx.x == 32) {
          __threadfence();
          atomicAdd(ph2 ? &sy->dec_done : &sy->enc_done, 1ull);
        }
      }
      WSTAMP(ph2 ? 4 : 1);
    }
    }  // warp != 0
    }  // kStream || ph2
    if (kStream) {
      // before phase 2: the epilogue warps wait for this step's h (post
      // cluster / row kernel); the producer and the split warps run on
      if (!ph2 && warp >= 2 && warp < 6) {
        if (threadIdx.x == 64) {
          s_go = wait_counter(&sy->h_done, (unsigned long long)kStreamSignalers * (k + 1), sy, 4) ? 1 : 0;
          if (prof && blockIdx.x == 0) prof[512 * k + 5] = gtimer();
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      // after phase 2: a failed wait (abort / timeout) anywhere -- every CTA
      // sees the flags at the same grid barrier, so all leave together
      if (ph2) {
        grid_sync2<true>(bar_cnt, bar_flags, (unsigned)S, sy, ++bar_epoch);
        if (threadIdx.x == 0) s_go = (ld_acquire_i(&sy->abort) | ld_acquire_i(&sy->error)) ? 0 : 1;
        __syncthreads();
        if (!s_go) break;
      }
    }
  }
  // launched mode: the next launch's barrier epochs start after this one's
  // (every CTA read the base before its first arrival)
  if (!kStream && blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<volatile unsigned*>(a.grid_bar + kLaunchBar) = bar_epoch;
  // a run stopped early (abort / timeout) may have next-phase copies in
  // flight: let them land before the CTA's shared memory is released
  {
    const int consumed = q_done * my_tiles;
    if (warp == 0 && lane == 0)
      for (int i = consumed; i < prod_next; ++i) mbar_wait2(&full[i % kStages], (uint32_t)(i / kStages) & 1u);
  }
#undef WSTAMP
#undef TSTAMP
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(T);
}

// ----------------------------------------------------------------- host --
int wide2_tiles(const StepArgs& a) { return (a.m.out + w2::kTileN - 1) / w2::kTileN; }

bool wide2_supported(const StepArgs& a, int S) {
  // every CTA owns >= 1 column tile; one CTA per SM
  // (32-B row segments: out_pad a multiple of 8 floats)
  return a.m.E1 == w2::kW && a.m.D == w2::kW && a.B <= 128 && a.m.out >= w2::kTileN && a.m.out_pad % 8 == 0 && S >= 1 &&
         S <= w2::kMaxS && S <= wide2_tiles(a);
}

static PerDevice g_wide2_attr;

void prepare_wide2() {
  g_wide2_attr.once([] {
    cudaFuncSetAttribute(k_wide2<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, w2::kSmem);
    cudaFuncSetAttribute(k_wide2<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, w2::kSmem);
    cudaFuncSetAttribute(k_wide2<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, w2::kSmem);
    cudaFuncSetAttribute(k_wide2<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, w2::kSmem);
    // load every instance now (lazy loading while the post cluster spins would wait for it)
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_wide2<true, true>);
    cudaFuncGetAttributes(&fa, k_wide2<false, true>);
    cudaFuncGetAttributes(&fa, k_wide2<true, false>);
    cudaFuncGetAttributes(&fa, k_wide2<false, false>);
  });
}

static void launch_wide2(const WideTcParamsHost& p, const StepArgs& a, const StreamArgs& r0, int S, bool stream,
                         cudaStream_t s) {
  prepare_wide2();
  StreamArgs r = r0;
  // Which CTAs own one column tile fewer (when S does not divide the tile
  // count): the 'short' owner indices are the last n_short; the rotation
  // puts grid CTAs 16, 17, ... on them. Measured: those two CTAs land on the
  // one TPC that shares a GPC with the post cluster (SMs 122/123 on every box
  // measured, whichever tiles they own -- LTFB_W2_ROT A/B) and run each
  // tile ~1.5x slower, so the step's phase-2 barrier waited for them
  // (-2.3 us per step with the rotation). A placement heuristic only: the
  // arithmetic is the same for any rotation given the same rotation in both
  // step modes (it is a property of the trainer's launches, not of the data).
  const int ntiles = wide2_tiles(a);
  const int n_short = ntiles % S ? S - ntiles % S : 0;
  r.tile_rot = n_short > 0 ? ((S - n_short - 16) % S + S) % S : 0;
  if (const char* rot = std::getenv("LTFB_W2_ROT")) r.tile_rot = std::atoi(rot) % std::max(S, 1);
  r.tile_donate = 3;  // (those two CTAs ran 2-6 us behind the median with 5 tiles; A/B: 1, 2, 3 tiles -0.7, -1.3, -1.5 us)
  if (const char* dn = std::getenv("LTFB_W2_DONATE")) r.tile_donate = std::max(0, std::atoi(dn));
  Wide2Params tp;
  std::memcpy(&tp.tm_y, p.y_sel >= 0 ? p.y_alt[p.y_sel] : p.maps, sizeof(CUtensorMap));
  std::memcpy(&tp.tm_wet, p.maps + 128, sizeof(CUtensorMap));
  std::memcpy(&tp.tm_wd, p.maps + 256, sizeof(CUtensorMap));
  std::memcpy(&tp.tm_wdt, p.wdt64, sizeof(CUtensorMap));
  void* args[] = {(void*)&tp, (void*)&a, (void*)&r, (void*)&p.bias_pad};
  const void* fn = stream ? (p.precise ? (const void*)k_wide2<true, true> : (const void*)k_wide2<false, true>)
                          : (p.precise ? (const void*)k_wide2<true, false> : (const void*)k_wide2<false, false>);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(S);
  cfg.blockDim = dim3(w2::kThreads);
  cfg.dynamicSmemBytes = w2::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[3];
  int nat = 0;
  if (stream) {
    // programmatic dependent launch behind the post cluster on the same
    // stream: this grid is scheduled once every post CTA has signalled
    // (griddepcontrol.launch_dependents right after it became resident), so
    // it finds exactly the SMs the cluster leaves free -- no host round trip
    // between the two launches. (This kernel never waits on the post grid's
    // completion: it synchronises with it through StepSync counters.)
    at[nat].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[nat].val.programmaticStreamSerializationAllowed = 1;
    ++nat;
  }
  if (!stream) {
    // launched mode: cooperative, the grid barrier needs every CTA resident.
    // (Streamed mode is not: a cooperative grid does not start while the post
    // cluster -- another kernel -- is resident; its grid is exactly the SMs
    // the cluster leaves free, and the barrier's timeout catches the rest.)
    at[nat].id = cudaLaunchAttributeCooperative;
    at[nat].val.cooperative = 1;
    ++nat;
  }
  if (p.l2_hit > 0.0f) {  // the frozen weights persist in L2 across steps
    at[nat].id = cudaLaunchAttributeAccessPolicyWindow;
    at[nat].val.accessPolicyWindow.base_ptr = p.l2_base;
    at[nat].val.accessPolicyWindow.num_bytes = p.l2_bytes;
    at[nat].val.accessPolicyWindow.hitRatio = p.l2_hit;
    at[nat].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[nat].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    ++nat;
  }
  cfg.attrs = at;
  cfg.numAttrs = nat;
  const cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e != cudaSuccess)
    throw std::runtime_error(std::string(stream ? "streamed" : "launched") + " wide pass launch: " +
                             cudaGetErrorString(e));
}

void launch_wide2_stream(const WideTcParamsHost& p, const StepArgs& a, const StreamArgs& r, int S, cudaStream_t s) {
  launch_wide2(p, a, r, S, true, s);
}

void launch_wide2_step(const WideTcParamsHost& p, const StepArgs& a, cudaStream_t s) {
  StreamArgs r{};
  r.n = 1;
  launch_wide2(p, a, r, a.S, false, s);
}

static_assert(sizeof(Wide2Params) == 4 * 128, "CUtensorMap packing");

}  // namespace ltfb_dev
