// The wide pass of a training step on the 5th-gen tensor cores (sm_100a).
//
// One persistent CTA per SM walks 32-column tiles c0 = 32 t of the output
// dimension (49,167 at paper scale). Per tile, with Y = the minibatch's
// output rows [128 x 32], the frozen weights We (enc layer 0, [out x 64])
// and Wd (dec last layer, [64 x out]) and h = dec-head activations
// [128 x 64] (in TMEM for the whole kernel):
//
//   MMA1  P_enc += Y  We[c0:c0+32, :]         (enc layer-0 split-K partial:
//                                              D-step real latents,
//                                              train_ops.hpp:160)
//   MMA2  O      = h  Wd[:, c0:c0+32]         (dec forward, train_ops.hpp:100)
//   epi   d = O + b - Y ; sum |d| (f64) ; S = sign(d)     (loss.hpp:25-41)
//   MMA3  P_dec += S  Wd[:, c0:c0+32]^T        (dL/dh up to 1/n,
//                                              mlp.hpp:278; dW/db of the
//                                              frozen decoder never formed)
//
// Parity ("3xTF32") mode splits every fp32 operand into hi + lo tf32 parts
// and accumulates hi*hi + lo*hi + hi*lo in f32 TMEM (S is exact in tf32, so
// MMA3 needs only S*hi + S*lo). The operand tiles arrive by TMA as plain
// fp32 (y, and K-major copies WeT / Wd / WdT of the frozen weights, laid
// out once) and are split per tile in shared memory: 40 KB of HBM per tile
// against 32 KB algorithmic (WdT duplicates Wd; a tf32 MN-major operand
// would need the 32-B-atom swizzle, which MMA3's K-major use of Wd excludes).
//
// Warp roles (320 threads): w0 TMA producer, w1 MMA issuer + TMEM owner,
// w2-5 epilogue (TMEM lane quadrants 2,3,0,1), w6-9 tf32 hi/lo split.
// After the tiles the grid synchronises (cooperative launch, one CTA per SM)
// and every CTA sums a slice of the 148 partials in fixed CTA order (the
// deterministic split-K reduction), so no separate reduce kernel runs.
// Pipelines: 2 smem stages of 80 KB (full / split / sready / empty
// mbarriers), 2 TMEM O buffers (ofull / oempty).
#include <cuda.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "kernels.hpp"
#include "tc_ptx.cuh"

namespace ltfb_dev {

namespace wt {
constexpr int kTileN = 32;                 // output columns per tile
constexpr int kRows = 128;                 // MMA M (minibatch rows)
constexpr int kW = 64;                     // E1 == D == 64
constexpr uint32_t kY = 16384;             // [128 x 32] f32
constexpr uint32_t kWt = 8192;             // [64 x 32] f32
constexpr uint32_t kStage = 6 * kWt;  // WeT hi/lo, Wd hi/lo, WdT hi/lo
constexpr int kStages = 3;            // weight stages == TMEM y slots (freed by MMA3)
constexpr int kYStages = 4;           // y landing slots (freed by the split): the row
                                      // gather runs one tile further ahead
constexpr uint32_t kSmem = kYStages * kY + kStages * kStage + 1024;
constexpr int kThreads = 320;
// TMEM columns
constexpr uint32_t kPenc = 0, kPdec = 64, kO0 = 128, kHhi = 192, kHlo = 256;
constexpr uint32_t kYbase = 320;  // + 64 s: y hi [32], y lo / S [32] of stage s
static_assert(kYbase + 64 * kStages <= 512, "TMEM columns");
}  // namespace wt

struct WideTcParams {
  CUtensorMap tm_y, tm_wet, tm_wd, tm_wdt;  // minibatch y, WeT / Wd [64 x out_pad], WdT [out_pad x 64]
};

/// Sense-reversing grid barrier; valid because the kernel is launched
/// cooperatively (every CTA resident). bar[0] arrivals, bar[1] generation.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g0 = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == n - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g0) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

template <bool kPrecise>
__global__ void __launch_bounds__(wt::kThreads, 1)
    k_wide_tc(const __grid_constant__ WideTcParams tp, StepArgs a, const float* __restrict__ bias_pad) {
  using namespace wt;
  if (a.ctr->aborted) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte aligned base for the 128-byte swizzle; offsetting the __shared__
  // array itself (not an integer round trip) keeps every access an LDS/STS
  unsigned char* sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kStages], split_done[kStages], sready[kStages], empty[kStages];
  __shared__ uint64_t yfull[kYStages];
  __shared__ uint64_t ofull[2], oempty[2], h_ready, done, rbar;
  __shared__ uint32_t tmem_base;
  __shared__ double red[128];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rows = min(a.B, a.n_part - (int)a.ctr->step_in_epoch * a.B);
  __shared__ long long s_ph[10];
  __shared__ long long s_ev[16][8];  // debug timeline (LTFB_PHASE_PROF), CTA 0
  const bool prof = a.phase_prof && blockIdx.x == 0;
#define LTFB_EV(i, e) do { if (prof && (i) < 16) s_ev[(i)][(e)] = clock64(); } while (0)
  if (prof && threadIdx.x == 0) s_ph[0] = clock64();
  const int out = a.m.out;
  const int ntiles = (out + kTileN - 1) / kTileN;
  const int my_tiles = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

  auto stage_ptr = [&](int s) { return sm + kYStages * kY + s * kStage; };
  auto Yraw = [&](int sy) { return sm + sy * kY; };                     // y tile [128 x 32] SW128 (gather4)
  auto WeH = [&](int s) { return stage_ptr(s); };                       // WeT [64 j x 32 c] SW128
  auto WeL = [&](int s) { return stage_ptr(s) + kWt; };
  auto WdH = [&](int s) { return stage_ptr(s) + 2 * kWt; };             // Wd  [64 j x 32 c] SW128
  auto WdL = [&](int s) { return stage_ptr(s) + 3 * kWt; };
  auto WtH = [&](int s) { return stage_ptr(s) + 4 * kWt; };             // WdT [32 c x 64 j] as 2 K-blocks
  auto WtL = [&](int s) { return stage_ptr(s) + 5 * kWt; };
  auto tYh = [&](int s) { return (uint32_t)(kYbase + 64 * s); };        // TMEM y hi   [128 x 32]
  auto tYl = [&](int s) { return (uint32_t)(kYbase + 64 * s + 32); };   // TMEM y lo, then S

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&split_done[s], 128);
      tc::mbar_init(&sready[s], 128);
      tc::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kYStages; ++s) {
      tc::mbar_init(&yfull[s], 1);
    }
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

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer --
    // weight tiles only (the y rows are gathered by the staging warps,
    // which refill each y slot as soon as they have read it)
    for (int iw = 0; iw < my_tiles; ++iw) {
      const int s = iw % kStages;
      if (lane == 0) {
        if (iw >= kStages) tc::mbar_wait(&empty[s], ((uint32_t)(iw / kStages) & 1u) ^ 1u);
        const int c0 = ((int)blockIdx.x + iw * (int)gridDim.x) * kTileN;
        LTFB_EV(iw, 0);
        tc::mbar_expect_tx(&full[s], 3 * kWt);
        tc::tma_load_2d(WeH(s), &tp.tm_wet, &full[s], c0, 0);
        tc::tma_load_2d(WdH(s), &tp.tm_wd, &full[s], c0, 0);
        tc::tma_load_2d(WtH(s), &tp.tm_wdt, &full[s], 0, c0);
        tc::tma_load_2d(WtH(s) + 4096, &tp.tm_wdt, &full[s], 32, c0);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer --
    // A operands (y hi / lo, h hi / lo, S) live in TMEM; B operands are the
    // K-major weight tiles in shared memory
    if (lane == 0) {
      const uint32_t i_enc = tc::idesc_tf32(128, 64, 0, 0);
      const uint32_t i_dec = tc::idesc_tf32(128, 32, 0, 0);
      auto mma3 = [&](int j) {  // P_dec += S Wd^T  (S exact in tf32: S*hi + S*lo)
        const int s = j % kStages;
        tc::tc_fence_after();
        const uint32_t wdh = tc::smem_u32(WdH(s)), wdl = tc::smem_u32(WdL(s));
        for (int kk = 0; kk < 4; ++kk) {
          tc::mma_tf32_ts(T + kPdec, T + tYl(s) + 8 * kk, tc::sdesc_sw128(wdh + 32 * kk, 16, 1024), i_enc,
                          (j > 0 || kk > 0) ? 1u : 0u);
          if (kPrecise)
            tc::mma_tf32_ts(T + kPdec, T + tYl(s) + 8 * kk, tc::sdesc_sw128(wdl + 32 * kk, 16, 1024), i_enc, 1u);
        }
        tc::tc_commit(&empty[s]);  // frees the stage for the producer
        LTFB_EV(j, 6);
      };
      auto mma12 = [&](int i) {
        const int s = i % kStages;
        const int b = i & 1;
        tc::tc_fence_after();
        const uint32_t weh = tc::smem_u32(WeH(s)), wel = tc::smem_u32(WeL(s));
        for (int kk = 0; kk < 4; ++kk) {  // MMA1: P_enc += Y We  (K = 8 c per step)
          const uint64_t bh = tc::sdesc_sw128(weh + 32 * kk, 16, 1024);
          tc::mma_tf32_ts(T + kPenc, T + tYh(s) + 8 * kk, bh, i_enc, (i > 0 || kk > 0) ? 1u : 0u);
          if (kPrecise) {
            tc::mma_tf32_ts(T + kPenc, T + tYl(s) + 8 * kk, bh, i_enc, 1u);
            tc::mma_tf32_ts(T + kPenc, T + tYh(s) + 8 * kk, tc::sdesc_sw128(wel + 32 * kk, 16, 1024), i_enc, 1u);
          }
        }
        if (i == 0) {  // h is needed from MMA2 on
          tc::mbar_wait(&h_ready, 0);
          tc::tc_fence_after();
        }
        const uint32_t Od = T + kO0 + 32u * (uint32_t)b;
        const uint32_t wth = tc::smem_u32(WtH(s)), wtl = tc::smem_u32(WtL(s));
        for (int kk = 0; kk < 8; ++kk) {  // MMA2: O = h Wd  (K = 8 j per step, B = WdT K-major)
          const uint32_t boff = (kk / 4) * 4096 + 32 * (kk % 4);
          const uint64_t bh = tc::sdesc_sw128(wth + boff, 16, 1024);
          tc::mma_tf32_ts(Od, T + kHhi + 8 * kk, bh, i_dec, kk > 0 ? 1u : 0u);
          if (kPrecise) {
            tc::mma_tf32_ts(Od, T + kHlo + 8 * kk, bh, i_dec, 1u);
            tc::mma_tf32_ts(Od, T + kHhi + 8 * kk, tc::sdesc_sw128(wtl + boff, 16, 1024), i_dec, 1u);
          }
        }
        tc::tc_commit(&ofull[b]);
        LTFB_EV(i, 3);
      };
      // dynamic order: MMA3 of a tile goes out as soon as its S is ready (so
      // the stage returns to the producer at once), MMA1/2 of the next tile
      // as soon as its operands are staged
      int n12 = 0, n3 = 0;
      while (n3 < my_tiles) {
        bool issued = false;
        if (n3 < n12) {
          const int s = n3 % kStages;
          if (tc::mbar_test(&sready[s], (uint32_t)(n3 / kStages) & 1u)) {
            mma3(n3++);
            issued = true;
          }
        }
        if (n12 < my_tiles) {
          const int s = n12 % kStages;
          const bool staged = tc::mbar_test(&split_done[s], (uint32_t)(n12 / kStages) & 1u);
          const bool obuf = n12 < 2 || tc::mbar_test(&oempty[n12 & 1], ((uint32_t)(n12 >> 1) & 1u) ^ 1u);
          if (staged && obuf) {
            mma12(n12++);
            issued = true;
          }
        }
        if (!issued) __nanosleep(20);
      }
      tc::tc_commit(&done);
    }
  } else if (warp >= 2 && warp < 6) {
    // -------------------------------------------------------- epilogue --
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int r = quad * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    {  // h = dec_head(fwd(x)) (computed by the row kernel / k_pre) -> TMEM as tf32 hi / lo
      float4 hv[16];  // the row's 64 floats, all loads in flight at once
      const float4* hrow = reinterpret_cast<const float4*>(a.h + (long long)r * kW);
#pragma unroll
      for (int q = 0; q < 16; ++q) hv[q] = r < rows ? hrow[q] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float v[32], vl[32];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 x4 = hv[half * 8 + q];
          const float xs[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            v[4 * q + e] = kPrecise ? tc::tf32_hi(xs[e]) : xs[e];
            vl[4 * q + e] = xs[e] - v[4 * q + e];
          }
        }
        tc::tmem_st32(T + lane_addr + kHhi + 32 * half, v);
        if (kPrecise) tc::tmem_st32(T + lane_addr + kHlo + 32 * half, vl);
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&h_ready);
      if (prof && r == 0) s_ph[1] = clock64();
    }
    // |d| sums: fp32 within a tile, four f64 chains across tiles, combined
    // once at the end; the bias of tile i+1 is prefetched while tile i runs
    double mae_e[4] = {0.0, 0.0, 0.0, 0.0};
    const int out_pad = a.m.out_pad;
    auto load_bias = [&](int i, float4* dst) {
      const int c0 = ((int)blockIdx.x + i * (int)gridDim.x) * kTileN;
      const float4* bp = reinterpret_cast<const float4*>(bias_pad + c0);
#pragma unroll
      for (int q = 0; q < 8; ++q) dst[q] = c0 + 4 * q < out_pad ? __ldg(bp + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    float4 bnext[8];
    if (my_tiles > 0) load_bias(0, bnext);
    for (int i = 0; i < my_tiles; ++i) {
      const int s = i % kStages;
      const int b = i & 1;
      const uint32_t phb = (uint32_t)(i >> 1) & 1u;
      const int c0 = ((int)blockIdx.x + i * (int)gridDim.x) * kTileN;
      float4 bcur[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) bcur[q] = bnext[q];
      if (i + 1 < my_tiles) load_bias(i + 1, bnext);
      tc::mbar_wait(&ofull[b], phb);
      if (r == 0) LTFB_EV(i, 4);
      tc::tc_fence_after();
      float o[32], yh[32], yl[32];
      tc::tmem_ld32(T + lane_addr + kO0 + 32u * (uint32_t)b, o);
      tc::tmem_ld32(T + lane_addr + tYh(s), yh);
      if (kPrecise) tc::tmem_ld32(T + lane_addr + tYl(s), yl);
      const int nvalid = r < rows ? min(kTileN, out - c0) : 0;
      // per-tile |d| partials in fp32 (8 terms each), folded into the f64
      // accumulators once per tile: FP64 conversions and adds are the
      // expensive operations of this loop on B200
      float tsum[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      float sv[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const float yv = kPrecise ? yh[c] + yl[c] : yh[c];  // hi + lo == y exactly
        const float bq[4] = {bcur[c / 4].x, bcur[c / 4].y, bcur[c / 4].z, bcur[c / 4].w};
        const float of = o[c] + bq[c % 4];  // dec forward output (mlp.hpp:209-213)
        const bool ok = c < nvalid;
        // loss.hpp:25-41: |p - t| (summed in double per tile below); sign(p - t), 0 at ties
        tsum[c % 4] += ok ? fabsf(of - yv) : 0.0f;
        sv[c] = ok ? (of > yv ? 1.0f : (of < yv ? -1.0f : 0.0f)) : 0.0f;
      }
      tc::tmem_st32(T + lane_addr + tYl(s), sv);  // S replaces y lo (MMA1 has consumed it)
      tc::tc_fence_before();
      tc::mbar_arrive(&oempty[b]);
      tc::mbar_arrive(&sready[s]);
#pragma unroll
      for (int e = 0; e < 4; ++e) mae_e[e] += (double)tsum[e];
      if (r == 0) LTFB_EV(i, 5);
    }
    const double mae = (mae_e[0] + mae_e[1]) + (mae_e[2] + mae_e[3]);
    // ---- partials out ----
    tc::mbar_wait(&done, 0);
    tc::tc_fence_after();
    float* pe = a.P_enc + ((long long)blockIdx.x * a.B + r) * kW;
    float* pd = a.P_dec + ((long long)blockIdx.x * a.B + r) * kW;
    for (int half = 0; half < 2; ++half) {
      float v[32];
      if (my_tiles > 0) {
        tc::tmem_ld32(T + lane_addr + kPenc + 32 * half, v);
      } else {
        for (int j = 0; j < 32; ++j) v[j] = 0.0f;
      }
      if (r < rows)
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(pe + 32 * half + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      if (my_tiles > 0) {
        tc::tmem_ld32(T + lane_addr + kPdec + 32 * half, v);
      }
      if (r < rows)
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(pd + 32 * half + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
    red[r] = mae;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (r == 0) {
      double t = 0.0;
      for (int k = 0; k < 128; ++k) t += red[k];
      a.mae_part[blockIdx.x] = t;
    }
  } else {
    // ------------------------------------------------- operand staging ----
    // thread t owns minibatch row r (its TMEM lane): the gathered y row goes
    // into TMEM as tf32 hi / lo (the A operand of MMA1 and the epilogue's y);
    // in precise mode the weight tiles are split in place in shared memory
    // (hi, plus a lo copy at the same swizzled offset)
    const int t = threadIdx.x - 192;  // 0..127
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    auto split = [&](unsigned char* hi_p, unsigned char* lo_p, int n4) {
      float4* hp = reinterpret_cast<float4*>(hi_p);
      float4* lp = reinterpret_cast<float4*>(lo_p);
#pragma unroll 4
      for (int idx = t; idx < n4; idx += 128) {
        const float4 v = hp[idx];
        const float4 h = make_float4(tc::tf32_hi(v.x), tc::tf32_hi(v.y), tc::tf32_hi(v.z), tc::tf32_hi(v.w));
        hp[idx] = h;
        lp[idx] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
      }
    };
    // y rows come straight from the HBM data store (epoch_plan.hpp:106-137,
    // store.hpp:140-181) with TMA tile::gather4 (4 rows per instruction, 32
    // per tile). One warp issuing all 32 costs ~2 k cycles per tile (the
    // issue serialises); lanes 0-7 of the four staging warps issue 8 each
    // (~0.7 k), so this warp group gathers: gather g covers rows 4g .. 4g+3.
    const int g = (warp - 6) * 8 + lane;  // gather slot of this lane (lanes < 8)
    int rw[4] = {0, 0, 0, 0};
    if (lane < 8) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rr = 4 * g + u;
        if (a.y_identity) {
          rw[u] = rr;  // host-streamed minibatch buffer
        } else {
          const unsigned* perm = a.perm[a.ctr->epoch & 1] + (long long)a.ctr->step_in_epoch * a.B;
          rw[u] = (int)perm[rr < rows ? rr : 0];
        }
      }
    }
    auto gather = [&](int it) {  // all 128 staging threads call this
      const int sy = it % kYStages;
      const int c0 = ((int)blockIdx.x + it * (int)gridDim.x) * kTileN;
      if (t == 0) tc::mbar_expect_tx(&yfull[sy], kY);
      asm volatile("bar.sync 2, 128;" ::: "memory");  // expect_tx before any complete_tx
      if (lane < 8) tc::tma_gather4(Yraw(sy) + 512 * g, &tp.tm_y, &yfull[sy], c0, rw[0], rw[1], rw[2], rw[3]);
    };
    for (int it = 0; it < kYStages && it < my_tiles; ++it) gather(it);
    for (int i = 0; i < my_tiles; ++i) {
      const int s = i % kStages;
      const uint32_t ph = (uint32_t)(i / kStages) & 1u;
      const int sy = i % kYStages;
      tc::mbar_wait(&yfull[sy], (uint32_t)(i / kYStages) & 1u);
      tc::mbar_wait(&full[s], ph);  // weights landed: stage s (and TMEM y slot s) is this tile's
      if (t == 0) LTFB_EV(i, 1);
      {
        const unsigned char* yrow = Yraw(sy) + r * 128;
        float v[32], vl[32];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t off = (uint32_t)(((q ^ (r & 7)) & 7) << 4);
          const float4 y4 = *reinterpret_cast<const float4*>(yrow + off);
          const float ys[4] = {y4.x, y4.y, y4.z, y4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            v[4 * q + e] = kPrecise ? tc::tf32_hi(ys[e]) : ys[e];
            vl[4 * q + e] = ys[e] - v[4 * q + e];
          }
        }
        tc::tmem_st32(T + lane_addr + tYh(s), v);
        if (kPrecise) tc::tmem_st32(T + lane_addr + tYl(s), vl);
      }
      // every staging thread has read its row of slot sy: refill it (the
      // barrier inside gather() orders the reads before the async writes)
      if (i + kYStages < my_tiles) gather(i + kYStages);
      if (kPrecise) {
        split(WeH(s), WeL(s), kWt / 16);
        split(WdH(s), WdL(s), kWt / 16);
        split(WtH(s), WtL(s), kWt / 16);
        tc::fence_proxy_async();
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&split_done[s]);
      if (t == 0) LTFB_EV(i, 2);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(T);
  if (prof && threadIdx.x == 0) s_ph[2] = clock64();

  // ---- grid-wide deterministic split-K reduction of the partials ----
  grid_sync(a.grid_bar, gridDim.x);
  if (prof && threadIdx.x == 0) s_ph[3] = clock64();
  {
    // float4 outputs [rows x 64] of P_enc then of P_dec; CTA c owns a
    // contiguous slice of <= kMaxQ outputs. Thread (g, o) sums partials
    // s = g, g + G, ... of output o (all loads issued before the adds, one
    // L2 round trip), then the G group sums are added in group order: a
    // fixed summation order, so the result is run-to-run deterministic.
    constexpr int kMaxQ = 32;
    const int q_enc = rows * (kW / 4), q_all = 2 * q_enc;
    const int lo = (int)((long long)q_all * blockIdx.x / gridDim.x);
    const int hi = (int)((long long)q_all * (blockIdx.x + 1) / gridDim.x);
    float4* part = reinterpret_cast<float4*>(sm);  // [G][kMaxQ]
    const int G = kThreads / kMaxQ;                // 10 groups
    const int g = threadIdx.x / kMaxQ, o = threadIdx.x % kMaxQ;
    const long long pstride4 = (long long)a.B * kW / 4;
    // this CTA's output slice [lo, hi) in chunks of kMaxQ float4 (one chunk
    // unless the grid is small, e.g. 97 CTAs at desk dims with B = 128):
    // every partial's chunk arrives by one or two bulk copies (TMA engine,
    // one per source CTA) into shared memory
    float4* stage = reinterpret_cast<float4*>(sm + 8192);  // [S][kMaxQ]
    uint32_t rpar = 0;
    for (int c0 = lo; c0 < hi; c0 += kMaxQ) {
      const int c1 = min(hi, c0 + kMaxQ), nq = c1 - c0;
      const int e0 = c0, e1 = min(c1, q_enc), d0 = max(c0, q_enc), d1 = c1;
      const int ne = max(0, e1 - e0), nd = max(0, d1 - d0);
      if (threadIdx.x == 0) tc::mbar_expect_tx(&rbar, (uint32_t)(a.S * nq * 16));
      __syncthreads();
      if ((int)threadIdx.x < a.S) {
        const int sidx = threadIdx.x;
        asm volatile("fence.proxy.async.global;" ::: "memory");
        const uint32_t dst = tc::smem_u32(stage + sidx * kMaxQ);
        const float4* pe4 = reinterpret_cast<const float4*>(a.P_enc) + sidx * pstride4;
        const float4* pd4 = reinterpret_cast<const float4*>(a.P_dec) + sidx * pstride4;
        if (ne > 0)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
              "l"(pe4 + e0), "r"(ne * 16), "r"(tc::smem_u32(&rbar))
              : "memory");
        if (nd > 0)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  dst + 16u * (uint32_t)ne),
              "l"(pd4 + (d0 - q_enc)), "r"(nd * 16), "r"(tc::smem_u32(&rbar))
              : "memory");
      }
      tc::mbar_wait(&rbar, rpar);
      rpar ^= 1u;
      float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      if (o < nq) {
        constexpr int kMaxPer = 16;  // ceil(148 / 10)
#pragma unroll
        for (int u = 0; u < kMaxPer; ++u) {
          const int sidx = g + u * G;
          if (sidx < a.S) {
            const float4 v = stage[sidx * kMaxQ + o];
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
          }
        }
      }
      if (prof && threadIdx.x == 0) s_ph[4] = clock64();
      part[g * kMaxQ + o] = acc;
      __syncthreads();
      if (prof && threadIdx.x == 0) s_ph[5] = clock64();
      if (g == 0 && o < nq) {
        float4 t = part[o];
        for (int k = 1; k < G; ++k) {
          const float4 w = part[k * kMaxQ + o];
          t.x += w.x;
          t.y += w.y;
          t.z += w.z;
          t.w += w.w;
        }
        const int q = c0 + o;
        float4* red_enc = reinterpret_cast<float4*>(a.scratch + a.L.red_enc);
        float4* red_dec = reinterpret_cast<float4*>(a.scratch + a.L.red_dec);
        if (q < q_enc) red_enc[q] = t;
        else red_dec[q - q_enc] = t;
      }
      __syncthreads();  // stage / part are refilled by the next chunk
    }
    if (prof && threadIdx.x == 0) s_ph[6] = clock64();
    if (blockIdx.x == 0 && warp == 0) {  // MAE total: lanes own strided partials, fixed xor tree
      double v[5];
#pragma unroll
      for (int u = 0; u < 5; ++u) v[u] = lane + 32 * u < a.S ? __ldcg(a.mae_part + lane + 32 * u) : 0.0;
      double t = (((v[0] + v[1]) + v[2]) + v[3]) + v[4];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
      if (lane == 0) *a.mae_total = t;
    }
  }
  if (prof && threadIdx.x == 0)
  {
    const long long tend = clock64();
    printf("wide phases (cycles): h %lld, tiles %lld, grid sync %lld, reduce %lld (loads %lld, part sync %lld, "
           "sum+write %lld, mae %lld)\n",
           s_ph[1] - s_ph[0], s_ph[2] - s_ph[0], s_ph[3] - s_ph[2], tend - s_ph[3], s_ph[4] - s_ph[3],
           s_ph[5] - s_ph[4], s_ph[6] - s_ph[5], tend - s_ph[6]);
    for (int i = 0; i < my_tiles && i < 16; ++i)
      printf("  tile %d: issue %lld tma %lld split %lld mma12 %lld epi_in %lld epi_out %lld mma3 %lld\n", i,
             s_ev[i][0] - s_ph[0], s_ev[i][1] - s_ph[0], s_ev[i][2] - s_ph[0], s_ev[i][3] - s_ph[0],
             s_ev[i][4] - s_ph[0], s_ev[i][5] - s_ph[0], s_ev[i][6] - s_ph[0]);
  }
}

// ----------------------------------------------------------------- host --
bool wide_tc_supported(const StepArgs& a) {
  // one CTA per SM (<= 160 partials for the in-kernel reduction's 10 x 16
  // loads); the reduction walks its output slice in chunks, any grid size
  return a.m.E1 == wt::kW && a.m.D == wt::kW && a.B <= wt::kRows && a.m.out >= wt::kTileN && a.S <= 160;
}

void launch_wide_tc(const StepArgs&, cudaStream_t) {
  throw std::runtime_error("launch_wide_tc: use launch_wide_tc_params");
}

void launch_wide_tc_params(const WideTcParamsHost& p, const StepArgs& a, cudaStream_t s) {
  static PerDevice attr;
  attr.once([] {
    cudaFuncSetAttribute(k_wide_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, wt::kSmem);
    cudaFuncSetAttribute(k_wide_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, wt::kSmem);
  });
  WideTcParams tp;
  std::memcpy(&tp, p.maps, sizeof tp);
  if (p.y_sel >= 0) std::memcpy(&tp.tm_y, p.y_alt[p.y_sel], sizeof(CUtensorMap));
  // cooperative: the in-kernel grid barrier needs every CTA resident
  void* args[] = {(void*)&tp, (void*)&a, (void*)&p.bias_pad};
  const void* fn = p.precise ? (const void*)k_wide_tc<true> : (const void*)k_wide_tc<false>;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.S);
  cfg.blockDim = dim3(wt::kThreads);
  cfg.dynamicSmemBytes = wt::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  int nat = 1;
  if (p.l2_hit > 0.0f) {  // frozen weights persist in L2 across steps
    at[1].id = cudaLaunchAttributeAccessPolicyWindow;
    at[1].val.accessPolicyWindow.base_ptr = p.l2_base;
    at[1].val.accessPolicyWindow.num_bytes = p.l2_bytes;
    at[1].val.accessPolicyWindow.hitRatio = p.l2_hit;
    at[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    nat = 2;
  }
  cfg.attrs = at;
  cfg.numAttrs = nat;
  const cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e != cudaSuccess) throw std::runtime_error(std::string("wide pass cooperative launch: ") + cudaGetErrorString(e));
}

// Splits / transposes the frozen wide-layer weights into the K-major tf32
// hi/lo copies the kernel streams (run whenever enc/dec change).
/// Lays the frozen wide-layer weights out for K-major tcgen05 operands, in
/// fp32 (split into tf32 hi / lo per tile in shared memory): WeT [64 x
/// out_pad] (enc layer 0 transposed), Wd [64 x out_pad] (dec last layer,
/// padded to a 16-B row pitch), WdT [out_pad x 64], bias [out_pad]; pad
/// columns zero. Run whenever enc / dec change.
__global__ void k_prep_wide(const float* __restrict__ enc, long long enc_w, const float* __restrict__ dec,
                            long long dec_w, long long dec_b, int out, int out_pad, float* wet, float* wd, float* wdt,
                            float* bias_pad) {
  const long long n = (long long)wt::kW * out_pad;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i / out_pad), c = (int)(i % out_pad);
    const bool ok = c < out;
    wet[i] = ok ? enc[enc_w + (long long)c * wt::kW + j] : 0.0f;  // enc W0 [out x 64]
    const float w = ok ? dec[dec_w + (long long)j * out + c] : 0.0f;  // dec W_last [64 x out]
    wd[i] = w;
    wdt[(long long)c * wt::kW + j] = w;
    if (j == 0) bias_pad[c] = ok ? dec[dec_b + c] : 0.0f;
  }
}

void launch_prep_wide(const StepArgs& a, const WideTcParamsHost& p, cudaStream_t s) {
  k_prep_wide<<<592, 256, 0, s>>>(a.p[kEnc], a.m.enc_wide_w, a.p[kDec], a.m.dec_wide_w, a.m.dec_wide_b, a.m.out,
                                  a.m.out_pad, p.wet, p.wd, p.wdt, p.bias_pad);
}

static_assert(sizeof(WideTcParams) == 4 * 128, "CUtensorMap packing");

namespace {
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}
void encode_2d(CUtensorMap* m, const float* base, uint64_t cols, uint64_t rows, uint32_t box_cols,
               uint32_t box_rows) {
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 4};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                                 es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}
}  // namespace

void encode_tile_map(void* map, const float* base, uint64_t cols, uint64_t rows, uint32_t box_cols,
                     uint32_t box_rows) {
  encode_2d(reinterpret_cast<CUtensorMap*>(map), base, cols, rows, box_cols, box_rows);
}

// y maps are read by tile::gather4: box = one row of 32 columns
void encode_y_map(WideTcParamsHost& p, int which, const float* yb, const StepArgs& a, int yb_rows) {
  CUtensorMap m;
  encode_2d(&m, yb, (uint64_t)a.m.out_pad, (uint64_t)yb_rows, 32, 1);
  std::memcpy(which < 0 ? p.maps : p.y_alt[which], &m, sizeof m);
}

void encode_wide_maps(WideTcParamsHost& p, const StepArgs& a, const float* yb, int yb_rows) {
  WideTcParams tp;
  const uint64_t op = (uint64_t)a.m.out_pad;
  encode_2d(&tp.tm_y, yb, op, (uint64_t)yb_rows, 32, 1);
  encode_2d(&tp.tm_wet, p.wet, op, wt::kW, 32, 64);
  encode_2d(&tp.tm_wd, p.wd, op, wt::kW, 32, 64);
  encode_2d(&tp.tm_wdt, p.wdt, wt::kW, op, 32, 32);
  std::memcpy(p.maps, &tp, sizeof tp);
  CUtensorMap m64;
  encode_2d(&m64, p.wdt, wt::kW, op, 32, 64);  // k_wide2: [64 columns x 32 j] per K-block
  std::memcpy(p.wdt64, &m64, sizeof m64);
}

}  // namespace ltfb_dev
