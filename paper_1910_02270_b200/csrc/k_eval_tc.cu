// Tournament / validation evaluation of the decoder's wide layer on the
// tensor cores (surrogate/train_ops.hpp:191-205 -> nn/loss.hpp:24-53): for
// every candidate c (local, incoming) and every slice row r,
//
//   forward_mae partial = sum_col | (h_c Wd)[r, col] + b[col] - y[r, col] |
//
// with h_c = dec_head(fwd_c(x)) from k_eval_small. One persistent CTA per SM
// owns 64-column tiles of the decoder output; for each 128-row block of the
// slice the rows' h of BOTH candidates sit in TMEM (tf32 hi / lo), and per
// tile one TMA stage brings the y block (two 128-B-swizzled halves) and the
// WdT tile (two K-blocks), which serve both candidates:
//
//   MMA  O_c = h_c WdT_tile^T   (3xTF32: hi*hi + lo*hi + hi*lo, N = 64)
//   epi  |O_c + b - y| in fp32 per tile, then f64 per thread; fixed-order
//        per-CTA sums -> EvalArgs::part, reduced by k_eval_finalize
//
// Warp roles (320 threads): w0 TMA producer, w1 MMA issuer + TMEM owner,
// w2-5 epilogue (also stage h into TMEM per row block), w6-9 tf32 split of
// the weight tile. 3 smem stages of 64 KB, 2 TMEM O buffers per candidate.
#include <cuda.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "kernels.hpp"
#include "small_mlp.cuh"
#include "tc_ptx.cuh"

namespace ltfb_dev {

namespace et {
constexpr int kN = 64;                       // decoder-output columns per tile
constexpr int kW = 64;                       // D (dec-head output width)
constexpr uint32_t kYHalf = 128 * 128;       // [128 rows x 32 cols] f32, SW128
constexpr uint32_t kY = 2 * kYHalf;          // 32 KB
constexpr uint32_t kWk = 64 * 128;           // WdT K-block [64 cols x 32 j] f32, SW128
constexpr uint32_t kWh = 2 * kWk;            // 16 KB (K = 64)
constexpr uint32_t kStage = kY + 2 * kWh;    // y + W hi + W lo
constexpr int kStages = 3;
constexpr uint32_t kSmem = kStages * kStage + 1024;
constexpr int kThreads = 320;
// TMEM: cand c h hi at 128 c, h lo at 128 c + 64; O[b][c] at 256 + 128 b + 64 c
}  // namespace et

struct EvalTcMaps {
  CUtensorMap tm_y;    // slice y [rows x out_pad], box {32, 128}, SW128
  CUtensorMap tm_wdt;  // WdT [out_pad x 64], box {32, 64}, SW128
};

template <bool kPrecise>
__global__ void __launch_bounds__(et::kThreads, 1)
    k_eval_tc(const __grid_constant__ EvalTcMaps tp, const __grid_constant__ EvalArgs a,
              const float* __restrict__ bias_pad) {
  using namespace et;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kStages], split_done[kStages], empty[kStages];
  __shared__ uint64_t ofull[2], oempty[2], h_ready, rb_done;
  __shared__ uint32_t tmem_base;
  __shared__ double red[128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int out = a.m.out, rows = a.rows, nc = a.nc;
  const int ntiles = (out + kN - 1) / kN;
  // CTA grid = column-tile lanes x row groups: with fewer column tiles than
  // SMs (desk dims: 49) the 128-row blocks of a large slice are dealt over
  // row groups too (block rbg = gr + rb * rgn), so a C5-size tournament
  // slice keeps every SM busy; paper dims: one row group, as before
  // A slice with at least one 128-row block per CTA (C5-size slices) is dealt
  // by rows only: each CTA sweeps every column tile of its row blocks, so the
  // rows' h (both candidates, 64 KB per block, not L2-resident at that size)
  // is staged once per block instead of once per column lane (at desk dims
  // 49 lanes re-read it: ~2x the y bytes); the WdT tiles it re-reads instead
  // are L2-resident.
  const int nrb_all = (rows + 127) / 128;
  const int cgn = nrb_all >= (int)gridDim.x ? 1 : min((int)gridDim.x, ntiles);
  const int rgn = max(1, (int)gridDim.x / max(cgn, 1));
  const int cb = (int)blockIdx.x % max(cgn, 1), gr = (int)blockIdx.x / max(cgn, 1);
  const bool active = gr < rgn && gr < nrb_all;
  const int my_tiles = active && ntiles > cb ? (ntiles - 1 - cb) / cgn + 1 : 0;
  const int nrb = active ? (nrb_all - gr + rgn - 1) / rgn : 0;  // this CTA's row blocks
  const int nitems = my_tiles * nrb;  // item q = rb * my_tiles + i
  auto Ys = [&](int s) { return sm + s * kStage; };
  auto Wh = [&](int s) { return sm + s * kStage + kY; };
  auto Wl = [&](int s) { return sm + s * kStage + kY + kWh; };
  auto tile_c0 = [&](int i) { return (cb + i * cgn) * kN; };
  auto rb_row0 = [&](int rb) { return (gr + rb * rgn) * 128; };  // first slice row of local row block rb

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&split_done[s], 128);
      tc::mbar_init(&empty[s], 128);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&ofull[b], 1);
      tc::mbar_init(&oempty[b], 128);
    }
    tc::mbar_init(&h_ready, 128);
    tc::mbar_init(&rb_done, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tp.tm_y);
    tc::tma_prefetch(&tp.tm_wdt);
  }
  if (warp == 1) tc::tmem_alloc<512>(&tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t T = tmem_base;

  if (warp == 0) {
    // ---------------------------------------------------- TMA producer --
    if (lane == 0)
      for (int q = 0; q < nitems; ++q) {
        const int s = q % kStages;
        if (q >= kStages) tc::mbar_wait(&empty[s], ((uint32_t)(q / kStages) & 1u) ^ 1u);
        const int rb = q / my_tiles, c0 = tile_c0(q % my_tiles);
        tc::mbar_expect_tx(&full[s], kY + kWh);
        tc::tma_load_2d(Ys(s), &tp.tm_y, &full[s], c0, rb_row0(rb));
        tc::tma_load_2d(Ys(s) + kYHalf, &tp.tm_y, &full[s], c0 + 32, rb_row0(rb));
        tc::tma_load_2d(Wh(s), &tp.tm_wdt, &full[s], 0, c0);
        tc::tma_load_2d(Wh(s) + kWk, &tp.tm_wdt, &full[s], 32, c0);
      }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer --
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_tf32(128, kN, 0, 0);
      for (int q = 0; q < nitems; ++q) {
        const int s = q % kStages, b = q & 1, i = q % my_tiles, rb = q / my_tiles;
        if (i == 0) tc::mbar_wait(&h_ready, (uint32_t)rb & 1u);
        tc::mbar_wait(&split_done[s], (uint32_t)(q / kStages) & 1u);
        if (q >= 2) tc::mbar_wait(&oempty[b], ((uint32_t)(q >> 1) & 1u) ^ 1u);
        tc::tc_fence_after();
        const uint32_t wh = tc::smem_u32(Wh(s)), wl = tc::smem_u32(Wl(s));
        for (int c = 0; c < nc; ++c) {
          const uint32_t D = T + 256u + 128u * (uint32_t)b + 64u * (uint32_t)c;
          const uint32_t Ah = T + 128u * (uint32_t)c, Al = Ah + 64u;
          for (int kk = 0; kk < 8; ++kk) {  // K = 8 j per step
            const uint32_t boff = (uint32_t)(kk / 4) * kWk + 32u * (uint32_t)(kk % 4);
            const uint64_t bh = tc::sdesc_sw128(wh + boff, 16, 1024);
            tc::mma_tf32_ts(D, Ah + 8 * kk, bh, idesc, kk > 0 ? 1u : 0u);
            if (kPrecise) {
              tc::mma_tf32_ts(D, Al + 8 * kk, bh, idesc, 1u);
              tc::mma_tf32_ts(D, Ah + 8 * kk, tc::sdesc_sw128(wl + boff, 16, 1024), idesc, 1u);
            }
          }
        }
        tc::tc_commit(&ofull[b]);
        if (i + 1 == my_tiles) tc::tc_commit(&rb_done);  // h of this row block no longer read
      }
    }
  } else if (warp < 6) {
    // -------------------------------------------------------- epilogue --
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    double acc[2] = {0.0, 0.0};
    for (int rb = 0; rb < nrb && my_tiles > 0; ++rb) {
      if (rb > 0) {
        tc::mbar_wait(&rb_done, (uint32_t)(rb - 1) & 1u);
        tc::tc_fence_after();
      }
      const int row = rb_row0(rb) + r;
      for (int c = 0; c < nc; ++c) {  // h rows of both candidates -> TMEM (tf32 hi / lo)
        const float4* hp = reinterpret_cast<const float4*>(a.h + ((long long)c * rows + row) * kW);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          float v[32], vl[32];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 x4 = row < rows ? hp[half * 8 + q] : make_float4(0.f, 0.f, 0.f, 0.f);
            const float xs[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              v[4 * q + e] = kPrecise ? tc::tf32_hi(xs[e]) : xs[e];
              vl[4 * q + e] = xs[e] - v[4 * q + e];
            }
          }
          tc::tmem_st32(T + lane_addr + 128u * (uint32_t)c + 32u * (uint32_t)half, v);
          if (kPrecise) tc::tmem_st32(T + lane_addr + 128u * (uint32_t)c + 64u + 32u * (uint32_t)half, vl);
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&h_ready);
      for (int i = 0; i < my_tiles; ++i) {
        const int q = rb * my_tiles + i, s = q % kStages, b = q & 1;
        const int c0 = tile_c0(i);
        float4 bias[16];
        const float4* bp = reinterpret_cast<const float4*>(bias_pad + c0);
#pragma unroll
        for (int k = 0; k < 16; ++k) bias[k] = c0 + 4 * k < a.m.out_pad ? __ldg(bp + k) : make_float4(0.f, 0.f, 0.f, 0.f);
        tc::mbar_wait(&ofull[b], (uint32_t)(q >> 1) & 1u);
        tc::tc_fence_after();
        const int nvalid = row < rows ? min(kN, out - c0) : 0;
        for (int c = 0; c < nc; ++c) {
          float tsum = 0.0f;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            float o[32];
            tc::tmem_ld32(T + lane_addr + 256u + 128u * (uint32_t)b + 64u * (uint32_t)c + 32u * (uint32_t)half, o);
            const unsigned char* yrow = Ys(s) + half * kYHalf + r * 128;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float4 y4 = *reinterpret_cast<const float4*>(yrow + (((k ^ (r & 7)) & 7) << 4));
              const float4 b4 = bias[half * 8 + k];
              const float ys[4] = {y4.x, y4.y, y4.z, y4.w}, bs[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int col = half * 32 + 4 * k + e;
                const float pred = o[4 * k + e] + bs[e];  // mlp.hpp:209-213
                tsum += col < nvalid ? fabsf(pred - ys[e]) : 0.0f;
              }
            }
          }
          acc[c] += (double)tsum;
        }
        tc::tc_fence_before();
        tc::mbar_arrive(&oempty[b]);
        tc::mbar_arrive(&empty[s]);
      }
    }
    for (int c = 0; c < nc; ++c) {  // fixed-order per-CTA sum
      red[r] = acc[c];
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (r == 0) {
        double t = 0.0;
        for (int k = 0; k < 128; ++k) t += red[k];
        a.part[(long long)blockIdx.x * nc + c] = t;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
  } else {
    // ------------------------------------------------ weight tf32 split --
    const int t = threadIdx.x - 192;
    for (int q = 0; q < nitems; ++q) {
      const int s = q % kStages;
      tc::mbar_wait(&full[s], (uint32_t)(q / kStages) & 1u);
      if (kPrecise) {
        float4* hp = reinterpret_cast<float4*>(Wh(s));
        float4* lp = reinterpret_cast<float4*>(Wl(s));
#pragma unroll 4
        for (int idx = t; idx < (int)(kWh / 16); idx += 128) {
          const float4 v = hp[idx];
          const float4 h = make_float4(tc::tf32_hi(v.x), tc::tf32_hi(v.y), tc::tf32_hi(v.z), tc::tf32_hi(v.w));
          hp[idx] = h;
          lp[idx] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        }
        tc::fence_proxy_async();
      }
      tc::mbar_arrive(&split_done[s]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc<512>(T);
}

bool eval_tc_supported(const ModelArgs& m) { return m.D == et::kW; }

void encode_eval_maps(EvalTcHost& h, const float* slice_y, int rows, const float* wdt, const ModelArgs& m) {
  EvalTcMaps mp;
  encode_tile_map(&mp.tm_y, slice_y, (uint64_t)m.out_pad, (uint64_t)rows, 32, 128);
  encode_tile_map(&mp.tm_wdt, wdt, (uint64_t)et::kW, (uint64_t)m.out_pad, 32, 64);
  static_assert(sizeof(EvalTcMaps) == sizeof(h.maps), "map packing");
  std::memcpy(h.maps, &mp, sizeof mp);
}

void launch_eval_tc(const EvalArgs& a, const EvalTcHost& h, bool precise, cudaStream_t s) {
  static PerDevice attr;
  attr.once([] {
    cudaFuncSetAttribute(k_eval_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, et::kSmem);
    cudaFuncSetAttribute(k_eval_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, et::kSmem);
  });
  EvalTcMaps mp;
  std::memcpy(&mp, h.maps, sizeof mp);
  if (precise)
    k_eval_tc<true><<<a.S, et::kThreads, et::kSmem, s>>>(mp, a, h.bias_pad);
  else
    k_eval_tc<false><<<a.S, et::kThreads, et::kSmem, s>>>(mp, a, h.bias_pad);
}

}  // namespace ltfb_dev
