// K3b: fused GEMM chain Y = (X . W1) . W2 for E <= 256.
//
// MA kernel (per 64-row block i0, sequential j0 over F tiles):
//   xT  = dot(X[rows, 0:K], W1[0:K, f-tile])          (fp32)
//   xY  = dot(xT, W2[f-tile, 0:E], acc=Y[rows, 0:E])  (Y read-modify-written in Global)
// B200 realisation: one CTA per (128-row block, F split).  The T tile is
// accumulated in TMEM (double buffered), converted to bf16 by the epilogue
// warps into shared memory (the K-major A operand of the second MMA) and Y
// stays in TMEM for the whole F range -- the MA's per-iteration Global
// read-modify-write of Y becomes an on-chip carried accumulator.  With F
// split over S CTAs each writes an fp32 partial; a deterministic reduction
// kernel sums the S partials in ascending order.
#pragma once
#include "sm100.cuh"

namespace nt {

struct ChainParams {
  int N, K, F, E;
  int f_tiles_per_split;  // 128-wide F tiles handled by one CTA
  int splits;
  int row_blocks;
  float* partial;  // [splits, N, E] fp32 (splits > 1) or the fp32 output (splits == 1)
  void* y;         // final output when splits == 1
  long long ldy;
  int out_f32;
};

template <int E>
struct ChainCfg {
  static constexpr int BM = 128, BK = 64, BF = 128;
  static constexpr int X_BYTES = BM * BK * 2;    // 16 KB
  static constexpr int W1_BYTES = BK * BF * 2;   // 16 KB
  static constexpr int STAGE = X_BYTES + W1_BYTES;
  static constexpr int STAGES = 3;
  static constexpr int W2_BYTES = BF * E * 2;    // 32/64 KB
  static constexpr int ST_BYTES = BM * BF * 2;   // 32 KB
  static constexpr int OFF_W2 = STAGES * STAGE;
  static constexpr int OFF_ST = OFF_W2 + W2_BYTES;
  static constexpr int OFF_BAR = OFF_ST + ST_BYTES;
  static constexpr int NBAR = 2 * STAGES + 2 + 2 + 2 + 2 + 1;
  static constexpr int SMEM_BYTES = OFF_BAR + NBAR * 8 + 16 + 1024;
};

constexpr int kChainThreads = 192;

template <int E>
__global__ void __launch_bounds__(kChainThreads, 1)
    chain_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW1,
                 const __grid_constant__ CUtensorMap tmW2, const ChainParams p) {
  using C = ChainCfg<E>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* w2_full = bars + 2 * C::STAGES;   // [1] + pad
  uint64_t* w2_empty = w2_full + 2;           // [1] + pad
  uint64_t* t_full = w2_empty + 2;            // [2]
  uint64_t* t_empty = t_full + 2;             // [2]
  uint64_t* st_full = t_empty + 2;            // [1]
  uint64_t* st_empty = st_full + 1;           // [1]
  uint64_t* y_full = st_empty + 1;            // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR + 2);
  uint8_t* sW2 = smem + C::OFF_W2;
  uint8_t* sT = smem + C::OFF_ST;

  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const int lane = threadIdx.x & 31;
  const int rb = blockIdx.x % p.row_blocks;
  const int split = blockIdx.x / p.row_blocks;
  const int f_tiles_total = (p.F + C::BF - 1) / C::BF;
  const int ft0 = split * p.f_tiles_per_split;
  const int ft1 = min(f_tiles_total, ft0 + p.f_tiles_per_split);
  const int nft = max(0, ft1 - ft0);
  const int k_blocks = (p.K + C::BK - 1) / C::BK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmW1);
    prefetch_tmap(&tmW2);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(w2_full, 1);
    mbar_init(w2_empty, 1);
    for (int a = 0; a < 2; ++a) {
      mbar_init(&t_full[a], 1);
      mbar_init(&t_empty[a], 4);
    }
    mbar_init(st_full, 4);
    mbar_init(st_empty, 1);
    mbar_init(y_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tY = tmem + 256;  // Y accumulator columns [256, 256+E)

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int i = 0; i < nft; ++i) {
        const int ft = ft0 + i;
        for (int kb = 0; kb < k_blocks; ++kb, ++it) {
          const int s = it % C::STAGES;
          mbar_wait(&empty[s], ((it / C::STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], C::STAGE);
          uint8_t* sx = smem + s * C::STAGE;
          uint8_t* sw = sx + C::X_BYTES;
          tma_load_2d(sx, &tmX, &full[s], kb * C::BK, rb * C::BM);
          tma_load_2d(sw, &tmW1, &full[s], ft * C::BF, kb * C::BK);
          tma_load_2d(sw + C::BK * 128, &tmW1, &full[s], ft * C::BF + 64, kb * C::BK);
        }
        // W2 rows of this F tile (single buffer, released by the Y MMA)
        mbar_wait(w2_empty, (i & 1) ^ 1);
        mbar_arrive_expect_tx(w2_full, C::W2_BYTES);
#pragma unroll
        for (int c = 0; c < E / 64; ++c)
          tma_load_2d(sW2 + c * (C::BF * 128), &tmW2, w2_full, c * 64, ft * C::BF);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idT = idesc_bf16(128, C::BF, 0, 1);
      constexpr uint32_t idY = idesc_bf16(128, E, 0, 1);
      const uint32_t sbase = smem_u32(smem);
      const uint32_t sW2a = smem_u32(sW2), sTa = smem_u32(sT);
      auto y_gemm = [&](int i) {
        mbar_wait(st_full, i & 1);
        mbar_wait(w2_full, i & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < C::BF / 16; ++k) {
          const uint64_t ad = sdesc_sw128(sTa + (k >> 2) * (C::BM * 128) + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(sW2a + k * 2048, C::BF * 128, 1024);
          umma_ss(tY, ad, bd, idY, (i > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(st_empty);
        umma_commit(w2_empty);
      };
      int it = 0;
      for (int i = 0; i < nft; ++i) {
        const int a = i & 1;
        mbar_wait(&t_empty[a], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < k_blocks; ++kb, ++it) {
          const int s = it % C::STAGES;
          mbar_wait(&full[s], (it / C::STAGES) & 1);
          tc_fence_after();
          const uint32_t sx = sbase + s * C::STAGE;
          const uint32_t sw = sx + C::X_BYTES;
#pragma unroll
          for (int k = 0; k < C::BK / 16; ++k) {
            const uint64_t ad = sdesc_sw128(sx + k * 32, 16, 1024);
            const uint64_t bd = sdesc_sw128(sw + k * 2048, C::BK * 128, 1024);
            umma_ss(tmem + a * 128, ad, bd, idT, (kb | k) ? 1u : 0u);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&t_full[a]);
        if (i > 0) y_gemm(i - 1);
      }
      if (nft > 0) y_gemm(nft - 1);
      umma_commit(y_full);
    }
  } else {
    const int wq = warp & 3;
    const int r = wq * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    for (int i = 0; i < nft; ++i) {
      const int a = i & 1;
      mbar_wait(&t_full[a], (i >> 1) & 1);
      tc_fence_after();
      // previous Y MMA must be done reading sT
      mbar_wait(st_empty, (i & 1) ^ 1);
#pragma unroll 1
      for (int c = 0; c < C::BF / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + a * 128 + lane_off + c * 32, v);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
        uint8_t* rowp = sT + (c >> 1) * (C::BM * 128) + r * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int chunk = ((c & 1) * 4 + q) ^ (r & 7);
          *reinterpret_cast<uint4*>(rowp + chunk * 16) = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(st_full);
        mbar_arrive(&t_empty[a]);
      }
    }
    mbar_wait(y_full, 0);
    tc_fence_after();
    const int row = rb * 128 + r;
    const bool rv = row < p.N;
    // tcgen05.ld is .sync.aligned: every lane loads, only valid rows store
#pragma unroll 1
    for (int c = 0; c < E / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(tY + lane_off + c * 32, v);
      tmem_wait_ld();
      const int col0 = c * 32;
      if (!rv || col0 >= p.E) continue;
      if (p.splits > 1 || p.out_f32) {
        float* dst = (p.splits > 1) ? p.partial + ((long long)split * p.N + row) * p.E + col0
                                    : static_cast<float*>(p.y) + (long long)row * p.ldy + col0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (col0 + 4 * j < p.E)
            *reinterpret_cast<float4*>(dst + 4 * j) = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                                                  __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
      } else {
        __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.y) + (long long)row * p.ldy + col0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (col0 + 8 * j < p.E)
            *reinterpret_cast<uint4*>(dst + 8 * j) = make_uint4(
                pack_bf16(__uint_as_float(v[8 * j]), __uint_as_float(v[8 * j + 1])),
                pack_bf16(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3])),
                pack_bf16(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5])),
                pack_bf16(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7])));
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Deterministic split-F reduction: Y[n, e] = sum_s partial[s, n, e] (ascending s).
__global__ void chain_reduce_kernel(const float* __restrict__ partial, int splits, int N, int E, void* y,
                                    long long ldy, int out_f32) {
  const long long total = (long long)N * E;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    float acc = partial[idx];
    for (int s = 1; s < splits; ++s) acc += partial[(long long)s * total + idx];
    const long long n = idx / E, e = idx % E;
    if (out_f32)
      static_cast<float*>(y)[n * ldy + e] = acc;
    else
      static_cast<__nv_bfloat16*>(y)[n * ldy + e] = __float2bfloat16_rn(acc);
  }
}

}  // namespace nt
