// The three column passes of the autoencoder pre-training step on the
// 5th-gen tensor cores (surrogate/train_ops.hpp:52-81: autoencoder_backward;
// the weight gradients are nn/mlp.hpp:268-279, the bias gradients
// nn/tensor.hpp:159-164 col_sums). k_ae.cu holds the small kernels between
// them (split-K reductions, the enc tail / dec head forward and backward)
// and Adam; its SIMT column passes remain for widths other than 64.
//
// Every pass walks 32-column tiles of the output dimension with one
// persistent CTA per SM, gathers the batch's y rows straight from the AE
// source slab with TMA tile::gather4 (never copied) and computes in 3xTF32
// (fp32 operands split into tf32 hi + lo, products hi*hi + lo*hi + hi*lo
// accumulated in f32 TMEM; sign(d) is exact in tf32, so products with it
// need hi and lo only):
//
//   enc   P_z  += Y[:, tile] We0[tile, :]        A = y (TMEM), B = We0 rows
//                                                 transposed in smem
//   dec   O     = h Wd[:, tile]                   A = h (TMEM)
//         d = O + bd - y, |d| (f64), S = sign(d)  (loss.hpp:25-41)
//         P_g  += S Wd[:, tile]^T                 A = S (TMEM)
//         dWd[:, tile] = g1 (h^T S)               A = [h^T hi ; h^T lo]
//                                                 stacked on 128 TMEM lanes
//         dbd[tile] = col_sums(g1 S)              fp32, rows in order
//   encw  dWe0[tile, :] = y[:, tile]^T gz0        A = [gz0^T hi ; gz0^T lo],
//                                                 [gz0^T hi ; 0]
//
// (g1 = float(1 / (n out)), the MAE gradient scale: P_g is scaled by it in
// the split-K reduction.) The weights are read in the blob's own layout --
// We0 rows of a tile are one contiguous 8 KB block (bulk copy), Wd's rows
// have an unaligned pitch (plain loads) -- and transposed / split in shared
// memory, so Adam updates one copy of every parameter.
//
// Warp roles (320 threads): w0 the dec pass's bias-gradient column sums,
// w1 TMEM owner + MMA issuer, w2-5 epilogue (TMEM lane quadrants 2,3,0,1),
// w6-9 operand staging.
#include <cuda.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "kernels.hpp"
#include "tc_ptx.cuh"

namespace ltfb_dev {
namespace aet {

constexpr int kTileN = 32;       // output columns per tile
constexpr int kW = 64;           // E1 == D == 64
constexpr uint32_t kY = 16384;   // y tile [128 rows x 32] f32
constexpr uint32_t kWt = 8192;   // [64 x 32] f32
constexpr uint32_t kKb = 4096;   // one K-block [32 x 32] f32 of a K = 128 operand
constexpr int kLand = 3;         // y landing slots
constexpr int kThreads = 320;
constexpr int kXs = 33;          // padded row pitch of the lane-exchange buffer

struct Maps {
  CUtensorMap y;  // AE source slab [rows x out_pad], box {32, 1} (gather4)
};

__device__ __forceinline__ unsigned char* align1k(unsigned char* p) {
  return p + ((1024u - (tc::smem_u32(p) & 1023u)) & 1023u);
}

__device__ __forceinline__ int tiles_of_cta(int out) {
  const int ntiles = (out + kTileN - 1) / kTileN;
  return ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
}
__device__ __forceinline__ int tile_c0(int i) { return ((int)blockIdx.x + i * (int)gridDim.x) * kTileN; }

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

/// The y tile's gather slots: lanes 0-7 of the four warps of one 128-thread
/// group issue 8 gathers of 4 rows each (rows past n repeat row idx[0]: they
/// meet zero operands, so they only need to be finite).
struct Gather {
  int rw[4] = {0, 0, 0, 0};
  int g = 0;
  __device__ void init(const AeArgs& a, int group_warp, int lane) {
    g = group_warp * 8 + lane;
    if (lane < 8)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rr = 4 * g + u;
        rw[u] = (int)a.idx[rr < a.n ? rr : 0];
      }
  }
};

/// Row r of a gathered [128 x 32] tile (128-B swizzle) into 32 registers.
__device__ __forceinline__ void read_y_row(const unsigned char* tile, int r, float* v) {
  const unsigned char* row = tile + r * 128;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 y4 = *reinterpret_cast<const float4*>(row + (((q ^ (r & 7)) & 7) << 4));
    v[4 * q] = y4.x;
    v[4 * q + 1] = y4.y;
    v[4 * q + 2] = y4.z;
    v[4 * q + 3] = y4.w;
  }
}

/// Element (row, k) of a K-major operand [rows x 128] stored as four 128-B
/// swizzled K-blocks of [rows x 32] (rows == 32 here).
__device__ __forceinline__ uint32_t kblock_off(uint32_t row, uint32_t k) {
  return (k >> 5) * kKb + tc::sw128_off(row, k & 31u);
}

/// A [n x 64] row-major matrix (n * 256 contiguous bytes) into shared memory
/// by one bulk copy; every calling thread returns once it has landed.
__device__ __forceinline__ void stage_rows(float* dst, const float* src, int n, uint64_t* bar, bool issuer) {
  if (issuer) {
    tc::mbar_expect_tx(bar, (uint32_t)n * kW * 4u);
    bulk_g2s(dst, src, (uint32_t)n * kW * 4u, bar);
  }
  tc::mbar_wait(bar, 0);
}

/// Column j (lanes 0-63: tf32 hi; lanes 64-127: lo, or 0 when lo_zero) of
/// a [n x 64] row-major matrix, written along 128 TMEM columns from `col`:
/// the stacked A operand [M^T hi ; M^T lo] of a K = rows product.
__device__ __forceinline__ void stack_columns_to_tmem(const float* M, int n, int r, uint32_t taddr, bool lo_zero) {
  const int j = r & 63;
  const bool lo = r >= 64;
#pragma unroll 1
  for (int rb = 0; rb < 4; ++rb) {
    float v[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int rr = 32 * rb + u;
      const float x = rr < n ? M[rr * kW + j] : 0.0f;
      const float h = tc::tf32_hi(x);
      v[u] = lo ? (lo_zero ? 0.0f : x - h) : h;
    }
    tc::tmem_st32(taddr + 32 * rb, v);
  }
}

// ------------------------------------------------------------------ enc --
// P_z[cta] = sum over this CTA's tiles of Y[:, tile] We0[tile, :]
__global__ void __launch_bounds__(kThreads, 1) k_ae_enc_tc(const __grid_constant__ Maps mp,
                                                           const __grid_constant__ AeArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = align1k(smem_raw);
  __shared__ uint64_t land[kLand], staged[2], empty[2], done;
  __shared__ uint32_t tmem_base;
  constexpr uint32_t kP = 0, kYs = 64;  // TMEM: P [64]; y hi / lo of slot s at 64 + 64 s (+32)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = a.n, out = a.m.out;
  const int my = tiles_of_cta(out);
  auto Yl = [&](int sl) { return sm + sl * kY; };
  auto Wl = [&](int sl) { return sm + kLand * kY + sl * kWt; };  // We0 rows [32 c x 64 j]
  auto Bh = [&](int s) { return sm + kLand * (kY + kWt) + s * 2 * kWt; };
  auto Bl = [&](int s) { return Bh(s) + kWt; };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kLand; ++s) tc::mbar_init(&land[s], 1);
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&staged[s], 128);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&done, 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&mp.y);
  }
  if (warp == 1) tc::tmem_alloc<256>(&tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t T = tmem_base;

  if (warp == 1) {
    if (lane == 0) {
      const uint32_t idn = tc::idesc_tf32(128, 64, 0, 0);
      for (int i = 0; i < my; ++i) {
        const int s = i & 1;
        tc::mbar_wait(&staged[s], (uint32_t)(i >> 1) & 1u);
        tc::tc_fence_after();
        const uint32_t bh = tc::smem_u32(Bh(s)), bl = tc::smem_u32(Bl(s));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t ah = T + kYs + 64 * s + 8 * kk;
          const uint64_t dh = tc::sdesc_sw128(bh + 32 * kk, 16, 1024);
          tc::mma_tf32_ts(T + kP, ah, dh, idn, (i > 0 || kk > 0) ? 1u : 0u);
          tc::mma_tf32_ts(T + kP, ah + 32, dh, idn, 1u);
          tc::mma_tf32_ts(T + kP, ah, tc::sdesc_sw128(bl + 32 * kk, 16, 1024), idn, 1u);
        }
        tc::tc_commit(&empty[s]);
      }
      tc::tc_commit(&done);
    }
    __syncwarp();
  } else if (warp >= 6) {
    // ---------------------------------------------------------- staging --
    const int t = threadIdx.x - 192;
    const int quad = warp & 3, r = quad * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    Gather G;
    G.init(a, warp - 6, lane);
    const float* We = a.enc + a.m.enc_wide_w;
    auto refill = [&](int it) {
      const int sl = it % kLand, c0 = tile_c0(it);
      const uint32_t wb = (uint32_t)min(kTileN, out - c0) * (uint32_t)(kW * 4);
      if (t == 0) tc::mbar_expect_tx(&land[sl], kY + wb);
      asm volatile("bar.sync 2, 128;" ::: "memory");  // slot reads done; expect_tx before complete_tx
      if (lane < 8) tc::tma_gather4(Yl(sl) + 512 * G.g, &mp.y, &land[sl], c0, G.rw[0], G.rw[1], G.rw[2], G.rw[3]);
      if (t == 0) bulk_g2s(Wl(sl), We + (long long)c0 * kW, wb, &land[sl]);
    };
    for (int it = 0; it < kLand && it < my; ++it) refill(it);
    const int j = t & 63, hc = (t >> 6) * 16;
    for (int i = 0; i < my; ++i) {
      const int sl = i % kLand, s = i & 1;
      const int nv = min(kTileN, out - tile_c0(i));
      tc::mbar_wait(&land[sl], (uint32_t)(i / kLand) & 1u);
      if (i >= 2) tc::mbar_wait(&empty[s], ((uint32_t)(i >> 1) & 1u) ^ 1u);
      tc::tc_fence_after();
      {  // y row r -> TMEM hi / lo (A)
        float v[32], vl[32];
        read_y_row(Yl(sl), r, v);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float h = tc::tf32_hi(v[c]);
          vl[c] = v[c] - h;
          v[c] = h;
        }
        tc::tmem_st32(T + lane_addr + kYs + 64 * s, v);
        tc::tmem_st32(T + lane_addr + kYs + 64 * s + 32, vl);
      }
      {  // We0 rows [c][j] -> B = [64 j x 32 c] K-major hi / lo (rows past out: 0)
        const float* w = reinterpret_cast<const float*>(Wl(sl));
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = hc + 4 * q;
          float x[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) x[e] = c + e < nv ? w[(c + e) * kW + j] : 0.0f;
          const float4 h4 = make_float4(tc::tf32_hi(x[0]), tc::tf32_hi(x[1]), tc::tf32_hi(x[2]), tc::tf32_hi(x[3]));
          *reinterpret_cast<float4*>(Bh(s) + tc::sw128_off(j, c)) = h4;
          *reinterpret_cast<float4*>(Bl(s) + tc::sw128_off(j, c)) =
              make_float4(x[0] - h4.x, x[1] - h4.y, x[2] - h4.z, x[3] - h4.w);
        }
      }
      tc::fence_proxy_async();
      tc::tc_fence_before();
      tc::mbar_arrive(&staged[s]);
      if (i + kLand < my) refill(i + kLand);
    }
  } else if (warp >= 2) {
    // --------------------------------------------------------- partials --
    const int quad = warp & 3, r = quad * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    tc::mbar_wait(&done, 0);
    tc::tc_fence_after();
    float* pz = a.Pz + ((long long)blockIdx.x * n + r) * kW;
    for (int half = 0; half < 2; ++half) {
      float v[32];
      if (my > 0) {
        tc::tmem_ld32(T + lane_addr + kP + 32 * half, v);
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = 0.0f;
      }
      if (r < n)
#pragma unroll
        for (int c = 0; c < 32; c += 4)
          *reinterpret_cast<float4*>(pz + 32 * half + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<256>(T);
}

// ------------------------------------------------------------------ dec --
__global__ void __launch_bounds__(kThreads, 1) k_ae_dec_tc(const __grid_constant__ Maps mp,
                                                           const __grid_constant__ AeArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = align1k(smem_raw);
  __shared__ uint64_t land[kLand], wstaged[2], wempty[2], hready, ofull[2], sready[2], d4full[2], d4empty[2],
      dbdone[2], done, hbar;
  __shared__ uint32_t tmem_base;
  __shared__ double red[128];
  __shared__ long long ev[16][8];
  const bool prof = a.prof && blockIdx.x == 0;
  const long long t_start = clock64();
#define AE_EV(i, e) do { if (prof && (i) < 16) ev[(i)][(e)] = clock64() - t_start; } while (0)
  // TMEM columns
  constexpr uint32_t kHhi = 0, kHlo = 64, kHT = 128, kPg = 256, kO = 320, kD4 = 384, kS = 448;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = a.n, out = a.m.out;
  const int my = tiles_of_cta(out);
  const float g1 = (float)(1.0 / ((double)n * (double)out));  // loss.hpp:37-39
  auto Yl = [&](int sl) { return sm + sl * kY; };
  unsigned char* wbase = sm + kLand * kY;
  auto WkH = [&](int s) { return wbase + s * 4 * kWt; };  // Wd tile [64 j x 32 c] K-major (B of P_g)
  auto WkL = [&](int s) { return WkH(s) + kWt; };
  auto WtH = [&](int s) { return WkH(s) + 2 * kWt; };  // Wd tile^T [32 c x 64 j], 2 K-blocks (B of O)
  auto WtL = [&](int s) { return WkH(s) + 3 * kWt; };
  unsigned char* sbase = wbase + 2 * 4 * kWt;
  auto SB = [&](int b) { return sbase + b * 4 * kKb; };  // S^T [32 c x 128 r], 4 K-blocks (B of dWd)
  float* xch = reinterpret_cast<float*>(sbase + 2 * 4 * kKb);  // [64 x kXs]
  if (threadIdx.x == 0) {
    for (int s = 0; s < kLand; ++s) tc::mbar_init(&land[s], 1);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&wstaged[b], 128);
      tc::mbar_init(&wempty[b], 1);
      tc::mbar_init(&ofull[b], 1);
      tc::mbar_init(&sready[b], 128);
      tc::mbar_init(&d4full[b], 1);
      tc::mbar_init(&d4empty[b], 128);
      tc::mbar_init(&dbdone[b], 1);
    }
    tc::mbar_init(&hready, 128);
    tc::mbar_init(&done, 1);
    tc::mbar_init(&hbar, 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&mp.y);
  }
  if (warp == 1) tc::tmem_alloc<512>(&tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t T = tmem_base;
  int bad = 0;

  if (warp == 0) {
    // ------------------------------------- dbd = col_sums(g1 S), rows in order
    float* dbd = a.gdec + a.m.dec_wide_b;
    for (int i = 0; i < my; ++i) {
      const int b = i & 1;
      const int c0 = tile_c0(i), nv = min(kTileN, out - c0);
      tc::mbar_wait(&sready[b], (uint32_t)(i >> 1) & 1u);
      const unsigned char* sb = SB(b);
      float s = 0.0f;
      for (int r = 0; r < n; ++r) {
        const float v = *reinterpret_cast<const float*>(sb + kblock_off(lane, r));
        s += v > 0.0f ? g1 : (v < 0.0f ? -g1 : 0.0f);
      }
      if (lane < nv) {
        dbd[c0 + lane] = s;
        bad |= !isfinite(s);
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&dbdone[b]);
      if (lane == 0) AE_EV(i, 7);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer --
    if (lane == 0) {
      const uint32_t i64 = tc::idesc_tf32(128, 64, 0, 0), i32 = tc::idesc_tf32(128, 32, 0, 0);
      int n2 = 0, n34 = 0;
      bool have_h = false;
      while (n34 < my) {
        bool issued = false;
        if (n34 < n2) {  // P_g += S Wd^T and dWd = h^T S of tile n34, once its S is staged
          const int b = n34 & 1;
          const uint32_t ph = (uint32_t)(n34 >> 1) & 1u;
          if (tc::mbar_test(&sready[b], ph) && (n34 < 2 || tc::mbar_test(&d4empty[b], ph ^ 1u))) {
            tc::tc_fence_after();
            const uint32_t kh = tc::smem_u32(WkH(b)), kl = tc::smem_u32(WkL(b));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t as = T + kS + 32 * b + 8 * kk;
              tc::mma_tf32_ts(T + kPg, as, tc::sdesc_sw128(kh + 32 * kk, 16, 1024), i64,
                              (n34 > 0 || kk > 0) ? 1u : 0u);
              tc::mma_tf32_ts(T + kPg, as, tc::sdesc_sw128(kl + 32 * kk, 16, 1024), i64, 1u);
            }
            const uint32_t sb = tc::smem_u32(SB(b));
#pragma unroll
            for (int kk = 0; kk < 16; ++kk)
              tc::mma_tf32_ts(T + kD4 + 32 * b, T + kHT + 8 * kk,
                              tc::sdesc_sw128(sb + (kk >> 2) * kKb + 32 * (kk & 3), 16, 1024), i32,
                              kk > 0 ? 1u : 0u);
            tc::tc_commit(&d4full[b]);
            tc::tc_commit(&wempty[b]);
            AE_EV(n34, 4);
            ++n34;
            issued = true;
          }
        }
        if (n2 < my && n2 < n34 + 2) {  // O = h Wd of tile n2 (O buffer freed by tile n2 - 2's S)
          const int s = n2 & 1;
          if (tc::mbar_test(&wstaged[s], (uint32_t)(n2 >> 1) & 1u)) {
            if (!have_h) {
              tc::mbar_wait(&hready, 0);
              have_h = true;
            }
            tc::tc_fence_after();
            const uint32_t od = T + kO + 32 * s;
            const uint32_t th = tc::smem_u32(WtH(s)), tl = tc::smem_u32(WtL(s));
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint32_t boff = (kk >> 2) * kKb + 32 * (kk & 3);
              const uint64_t bh = tc::sdesc_sw128(th + boff, 16, 1024);
              tc::mma_tf32_ts(od, T + kHhi + 8 * kk, bh, i32, kk > 0 ? 1u : 0u);
              tc::mma_tf32_ts(od, T + kHlo + 8 * kk, bh, i32, 1u);
              tc::mma_tf32_ts(od, T + kHhi + 8 * kk, tc::sdesc_sw128(tl + boff, 16, 1024), i32, 1u);
            }
            tc::tc_commit(&ofull[s]);
            AE_EV(n2, 1);
            ++n2;
            issued = true;
          }
        }
        if (!issued) __nanosleep(20);
      }
      tc::tc_commit(&done);
    }
    __syncwarp();
  } else if (warp < 6) {
    // --------------------------------------------------------- epilogue --
    const int t = threadIdx.x - 64;
    const int quad = warp & 3, r = quad * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    {  // h rows -> TMEM hi / lo (A of O); h columns -> stacked [h^T hi ; h^T lo] (A of dWd),
       // from a shared-memory copy of h in the (not yet used) y landing slots 0-1
      float* hs = reinterpret_cast<float*>(Yl(0));
      stage_rows(hs, a.h, n, &hbar, t == 0);
      float v[32], vl[32];
      for (int half = 0; half < 2; ++half) {
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float x = r < n ? hs[r * kW + 32 * half + c] : 0.0f;
          v[c] = tc::tf32_hi(x);
          vl[c] = x - v[c];
        }
        tc::tmem_st32(T + lane_addr + kHhi + 32 * half, v);
        tc::tmem_st32(T + lane_addr + kHlo + 32 * half, vl);
      }
      stack_columns_to_tmem(hs, n, r, T + lane_addr + kHT, false);
      tc::tc_fence_before();
      tc::mbar_arrive(&hready);
    }
    Gather G;
    G.init(a, warp - 2, lane);
    auto refill = [&](int it) {
      const int sl = it % kLand;
      if (t == 0) tc::mbar_expect_tx(&land[sl], kY);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (lane < 8)
        tc::tma_gather4(Yl(sl) + 512 * G.g, &mp.y, &land[sl], tile_c0(it), G.rw[0], G.rw[1], G.rw[2], G.rw[3]);
    };
    for (int it = 0; it < kLand && it < my; ++it) refill(it);
    float* dWd = a.gdec + a.m.dec_wide_w;
    const float* Bd = a.dec + a.m.dec_wide_b;
    // dWd[:, tile j] = g1 (lanes j + lanes 64 + j of D4): the upper quadrants
    // hand their rows over through shared memory
    auto dwd = [&](int jt) {
      const int b = jt & 1;
      const int c0 = tile_c0(jt), nv = min(kTileN, out - c0);
      tc::mbar_wait(&d4full[b], (uint32_t)(jt >> 1) & 1u);
      if (t == 0) AE_EV(jt, 5);
      tc::tc_fence_after();
      float v[32];
      tc::tmem_ld32(T + lane_addr + kD4 + 32 * b, v);
      if (quad >= 2)
#pragma unroll
        for (int c = 0; c < 32; ++c) xch[(r - 64) * kXs + c] = v[c];
      tc::tc_fence_before();
      tc::mbar_arrive(&d4empty[b]);
      asm volatile("bar.sync 3, 128;" ::: "memory");
      if (quad < 2) {
        float* row = dWd + (long long)r * out + c0;
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (c < nv) {
            const float w = (v[c] + xch[r * kXs + c]) * g1;
            row[c] = w;
            bad |= !isfinite(w);
          }
      }
      asm volatile("bar.sync 3, 128;" ::: "memory");
      if (t == 0) AE_EV(jt, 6);
    };
    double mae = 0.0;
    for (int i = 0; i < my; ++i) {
      const int b = i & 1, sl = i % kLand;
      const int c0 = tile_c0(i), nv = min(kTileN, out - c0);
      float bd[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) bd[c] = c < nv ? __ldg(Bd + c0 + c) : 0.0f;
      tc::mbar_wait(&land[sl], (uint32_t)(i / kLand) & 1u);
      tc::mbar_wait(&ofull[b], (uint32_t)(i >> 1) & 1u);
      if (i >= 2) tc::mbar_wait(&dbdone[b], ((uint32_t)(i >> 1) & 1u) ^ 1u);
      if (t == 0) AE_EV(i, 2);
      tc::tc_fence_after();
      float o[32], y[32], sv[32];
      tc::tmem_ld32(T + lane_addr + kO + 32 * b, o);
      read_y_row(Yl(sl), r, y);
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const bool ok = r < n && c < nv;
        const float of = o[c] + bd[c];  // mlp.hpp:209-213
        const double d = (double)of - (double)y[c];
        if (ok) mae += fabs(d);
        sv[c] = ok ? (d > 0 ? 1.0f : (d < 0 ? -1.0f : 0.0f)) : 0.0f;
      }
      tc::tmem_st32(T + lane_addr + kS + 32 * b, sv);
      unsigned char* sb = SB(b);
#pragma unroll
      for (int c = 0; c < 32; ++c) *reinterpret_cast<float*>(sb + kblock_off(c, r)) = sv[c];
      tc::fence_proxy_async();
      tc::tc_fence_before();
      tc::mbar_arrive(&sready[b]);
      if (t == 0) AE_EV(i, 3);
      if (i + kLand < my) refill(i + kLand);
      if (i >= 1) dwd(i - 1);
    }
    if (my > 0) dwd(my - 1);
    tc::mbar_wait(&done, 0);
    tc::tc_fence_after();
    float* pg = a.Pg + ((long long)blockIdx.x * n + r) * kW;
    for (int half = 0; half < 2; ++half) {
      float v[32];
      if (my > 0) {
        tc::tmem_ld32(T + lane_addr + kPg + 32 * half, v);
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = 0.0f;
      }
      if (r < n)
#pragma unroll
        for (int c = 0; c < 32; c += 4)
          *reinterpret_cast<float4*>(pg + 32 * half + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
    }
    red[r] = mae;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (t == 0) {
      double s = 0.0;
      for (int k = 0; k < 128; ++k) s += red[k];
      a.mae_part[blockIdx.x] = s;
    }
  } else {
    // ---------------------------------------------------------- staging --
    // thread (j, 16 columns): the Wd tile's row j, loaded one tile ahead
    const int t = threadIdx.x - 192;
    const int j = t & 63, hc = (t >> 6) * 16;
    const float* Wd = a.dec + a.m.dec_wide_w;
    float wn[16];
    auto load = [&](int it) {
      const int c0 = tile_c0(it), nv = min(kTileN, out - c0);
      const float* row = Wd + (long long)j * out + c0;
#pragma unroll
      for (int u = 0; u < 16; ++u) wn[u] = hc + u < nv ? __ldg(row + hc + u) : 0.0f;
    };
    if (my > 0) load(0);
    for (int i = 0; i < my; ++i) {
      const int s = i & 1;
      float w[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) w[u] = wn[u];
      if (i + 1 < my) load(i + 1);
      if (i >= 2) tc::mbar_wait(&wempty[s], ((uint32_t)(i >> 1) & 1u) ^ 1u);
      float hi[16], lo[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        hi[u] = tc::tf32_hi(w[u]);
        lo[u] = w[u] - hi[u];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t off = tc::sw128_off(j, hc + 4 * q);
        *reinterpret_cast<float4*>(WkH(s) + off) = make_float4(hi[4 * q], hi[4 * q + 1], hi[4 * q + 2], hi[4 * q + 3]);
        *reinterpret_cast<float4*>(WkL(s) + off) = make_float4(lo[4 * q], lo[4 * q + 1], lo[4 * q + 2], lo[4 * q + 3]);
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const uint32_t off = (j >> 5) * kKb + tc::sw128_off(hc + u, j & 31);
        *reinterpret_cast<float*>(WtH(s) + off) = hi[u];
        *reinterpret_cast<float*>(WtL(s) + off) = lo[u];
      }
      tc::fence_proxy_async();
      tc::mbar_arrive(&wstaged[s]);
      if (t == 0) AE_EV(i, 0);
    }
  }
  if (bad) atomicOr(&a.flags[1], 1);
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(T);
  if (prof && threadIdx.x == 0) {
    printf("ae dec pass CTA 0: %d tiles, %lld cycles\n", my, clock64() - t_start);
    for (int i = 0; i < my && i < 16; ++i)
      printf("  tile %d: staged %lld mma2 %lld epi_in %lld sready %lld mma34 %lld dwd_in %lld dwd_out %lld dbd %lld\n", i,
             ev[i][0], ev[i][1], ev[i][2], ev[i][3], ev[i][4], ev[i][5], ev[i][6], ev[i][7]);
  }
#undef AE_EV
}

// ----------------------------------------------------------------- encw --
// dWe0[tile, :] = Y[:, tile]^T gz0: D [128 x 32] = A1 Y^T hi + A2 Y^T lo with
// A1 = [gz0^T hi ; gz0^T lo], A2 = [gz0^T hi ; 0]; dWe0^T = D[0:64] + D[64:128]
__global__ void __launch_bounds__(kThreads, 1) k_ae_encw_tc(const __grid_constant__ Maps mp,
                                                            const __grid_constant__ AeArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = align1k(smem_raw);
  __shared__ uint64_t land[kLand], staged[2], empty[2], aready, dfull[2], dempty[2], gbar;
  __shared__ uint32_t tmem_base;
  constexpr uint32_t kA1 = 0, kA2 = 128, kD = 256;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = a.n, out = a.m.out;
  const int my = tiles_of_cta(out);
  auto Yl = [&](int sl) { return sm + sl * kY; };
  auto YtH = [&](int s) { return sm + kLand * kY + s * 2 * kY; };  // y tile^T [32 c x 128 r], 4 K-blocks
  auto YtL = [&](int s) { return YtH(s) + kY; };
  float* xch = reinterpret_cast<float*>(sm + kLand * kY + 4 * kY);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kLand; ++s) tc::mbar_init(&land[s], 1);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&staged[b], 128);
      tc::mbar_init(&empty[b], 1);
      tc::mbar_init(&dfull[b], 1);
      tc::mbar_init(&dempty[b], 128);
    }
    tc::mbar_init(&aready, 128);
    tc::mbar_init(&gbar, 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&mp.y);
  }
  if (warp == 1) tc::tmem_alloc<512>(&tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t T = tmem_base;
  int bad = 0;

  if (warp == 1) {
    if (lane == 0) {
      const uint32_t i32 = tc::idesc_tf32(128, 32, 0, 0);
      for (int i = 0; i < my; ++i) {
        const int s = i & 1;
        const uint32_t ph = (uint32_t)(i >> 1) & 1u;
        if (i == 0) tc::mbar_wait(&aready, 0);
        tc::mbar_wait(&staged[s], ph);
        if (i >= 2) tc::mbar_wait(&dempty[s], ph ^ 1u);
        tc::tc_fence_after();
        const uint32_t yh = tc::smem_u32(YtH(s)), yl = tc::smem_u32(YtL(s));
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
          const uint32_t boff = (kk >> 2) * kKb + 32 * (kk & 3);
          tc::mma_tf32_ts(T + kD + 32 * s, T + kA1 + 8 * kk, tc::sdesc_sw128(yh + boff, 16, 1024), i32,
                          kk > 0 ? 1u : 0u);
          tc::mma_tf32_ts(T + kD + 32 * s, T + kA2 + 8 * kk, tc::sdesc_sw128(yl + boff, 16, 1024), i32, 1u);
        }
        tc::tc_commit(&dfull[s]);
        tc::tc_commit(&empty[s]);
      }
    }
    __syncwarp();
  } else if (warp >= 2 && warp < 6) {
    // --------------------------------------------------------- epilogue --
    const int quad = warp & 3, r = quad * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    float* gs = xch + 64 * kXs;  // gz0 [n x 64]
    stage_rows(gs, a.gz0, n, &gbar, warp == 2 && lane == 0);
    stack_columns_to_tmem(gs, n, r, T + lane_addr + kA1, false);
    stack_columns_to_tmem(gs, n, r, T + lane_addr + kA2, true);
    tc::tc_fence_before();
    tc::mbar_arrive(&aready);
    float* dWe = a.genc + a.m.enc_wide_w;
    for (int i = 0; i < my; ++i) {
      const int b = i & 1;
      const int c0 = tile_c0(i), nv = min(kTileN, out - c0);
      tc::mbar_wait(&dfull[b], (uint32_t)(i >> 1) & 1u);
      tc::tc_fence_after();
      float v[32];
      tc::tmem_ld32(T + lane_addr + kD + 32 * b, v);
      if (quad >= 2)
#pragma unroll
        for (int c = 0; c < 32; ++c) xch[(r - 64) * kXs + c] = v[c];
      tc::tc_fence_before();
      tc::mbar_arrive(&dempty[b]);
      asm volatile("bar.sync 3, 128;" ::: "memory");
      if (quad < 2) {
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (c < nv) {
            const float w = v[c] + xch[r * kXs + c];
            dWe[(long long)(c0 + c) * kW + r] = w;
            bad |= !isfinite(w);
          }
      }
      asm volatile("bar.sync 3, 128;" ::: "memory");
    }
  } else if (warp >= 6) {
    // ---------------------------------------------------------- staging --
    const int t = threadIdx.x - 192;
    const int quad = warp & 3, r = quad * 32 + lane;
    Gather G;
    G.init(a, warp - 6, lane);
    auto refill = [&](int it) {
      const int sl = it % kLand;
      if (t == 0) tc::mbar_expect_tx(&land[sl], kY);
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (lane < 8)
        tc::tma_gather4(Yl(sl) + 512 * G.g, &mp.y, &land[sl], tile_c0(it), G.rw[0], G.rw[1], G.rw[2], G.rw[3]);
    };
    for (int it = 0; it < kLand && it < my; ++it) refill(it);
    for (int i = 0; i < my; ++i) {
      const int sl = i % kLand, s = i & 1;
      tc::mbar_wait(&land[sl], (uint32_t)(i / kLand) & 1u);
      if (i >= 2) tc::mbar_wait(&empty[s], ((uint32_t)(i >> 1) & 1u) ^ 1u);
      float v[32];
      read_y_row(Yl(sl), r, v);
      unsigned char* yh = YtH(s);
      unsigned char* yl = YtL(s);
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const float h = tc::tf32_hi(v[c]);
        const uint32_t off = kblock_off(c, r);
        *reinterpret_cast<float*>(yh + off) = h;
        *reinterpret_cast<float*>(yl + off) = v[c] - h;
      }
      tc::fence_proxy_async();
      tc::mbar_arrive(&staged[s]);
      if (i + kLand < my) refill(i + kLand);
    }
  }
  if (bad) atomicOr(&a.flags[0], 1);
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(T);
}

constexpr uint32_t kSmemEnc = kLand * (kY + kWt) + 2 * 2 * kWt + 1024;
constexpr uint32_t kSmemDec = kLand * kY + 2 * 4 * kWt + 2 * 4 * kKb + 64 * kXs * 4 + 1024;
constexpr uint32_t kSmemEncw = kLand * kY + 4 * kY + 64 * kXs * 4 + 128 * kW * 4 + 1024;
static_assert(kSmemDec <= 227 * 1024 && kSmemEnc <= 227 * 1024 && kSmemEncw <= 227 * 1024, "shared memory");

}  // namespace aet

bool ae_tc_supported(const ModelArgs& m, int rows) {
  // the staged small kernels between the passes (k_ae.cu) hold <= 64-wide layers
  return rows >= 1 && rows <= 128 && m.E1 == aet::kW && m.D == aet::kW && m.out >= aet::kTileN &&
         m.enc_wide_w % 4 == 0 && m.enc_tail.max_w() <= 64 && m.dec_head.max_w() <= 64;
}

void encode_ae_y_map(void* map, const float* ysrc, int rows, const ModelArgs& m) {
  encode_tile_map(map, ysrc, (uint64_t)m.out_pad, (uint64_t)rows, aet::kTileN, 1);
}

static void launch_one(const void* fn, uint32_t smem, const void* map, const AeArgs& a, cudaStream_t s,
                       const char* what) {
  aet::Maps mp;
  std::memcpy(&mp.y, map, sizeof(CUtensorMap));
  void* args[] = {(void*)&mp, (void*)&a};
  const cudaError_t e = cudaLaunchKernel(fn, dim3(a.S), dim3(aet::kThreads), args, smem, s);
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

void prepare_ae_tc() {
  static PerDevice attr;
  attr.once([] {
    cudaFuncSetAttribute(aet::k_ae_enc_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, aet::kSmemEnc);
    cudaFuncSetAttribute(aet::k_ae_dec_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, aet::kSmemDec);
    cudaFuncSetAttribute(aet::k_ae_encw_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, aet::kSmemEncw);
  });
}

void launch_ae_enc_tc(const void* map, const AeArgs& a, cudaStream_t s) {
  launch_one((const void*)aet::k_ae_enc_tc, aet::kSmemEnc, map, a, s, "AE enc pass (tcgen05)");
}
void launch_ae_dec_tc(const void* map, const AeArgs& a, cudaStream_t s) {
  launch_one((const void*)aet::k_ae_dec_tc, aet::kSmemDec, map, a, s, "AE dec pass (tcgen05)");
}
void launch_ae_encw_tc(const void* map, const AeArgs& a, cudaStream_t s) {
  launch_one((const void*)aet::k_ae_encw_tc, aet::kSmemEncw, map, a, s, "AE encw pass (tcgen05)");
}

}  // namespace ltfb_dev
