// K3: tcgen05 GEMM C[M,N] = A[M,K] . B[K,N] (bf16 in, fp32 accumulate in TMEM).
//
// Realises the MA dots of the GEMM-chain kernel (SURVEY.md B.4, Appendix C
// V5/V6): `xT = dot(X[64*i0:+64, 0:K], W1[0:K, 128*j0:+128])` and
// `xY = dot(xT, W2[128*j0:+128, 0:E], acc=Y[...])`, which interpret_ma runs as
// sequential rank-1 updates (tilecc/ma/interp.py:241-251).
//
// Two variants: gemm_kernel (one CTA, M=128 x N=BN tiles) and gemm2_kernel
// (a CTA pair with tcgen05.mma.cta_group::2, M=256 x N=256 tiles, below),
// chosen by nt_gemm from the tile count.
//
// Persistent, warp-specialised:
//   warp 0      TMA producer (A K-major panels, B MN-major panels, SWIZZLE_128B)
//   warp 1      MMA issuer: tcgen05.mma.cta_group::1.kind::f16 M=128 N=BN K=16
//   warps 2-5   epilogue: TMEM -> registers -> global (fp32 or bf16)
// TMEM holds two BN-column accumulators so the epilogue of tile i overlaps
// the main loop of tile i+1.
#pragma once
#include "sm100.cuh"

// experiment switch: 1 = the CTA-pair epilogue reads TMEM but stores nothing
#ifndef NT_GEMM_NO_STORE
#define NT_GEMM_NO_STORE 0
#endif

namespace nt {

// K3's waits suspend instead of re-polling (A/B: GEMM +1.5 %, attention -0.5 % -> K3 only)
#ifndef NT_GEMM_WAIT_HINT
#define NT_GEMM_WAIT_HINT 1
#endif
constexpr bool kGemmWaitHint = NT_GEMM_WAIT_HINT != 0;

struct GemmParams {
  int M, N, K;
  int tiles_m, tiles_n;
  int group_m;  // CTA-pair kernel: tile rows per raster group
  int k_splits;  // single-CTA kernel: K ranges per output tile (fp32 partials to ws)
  int kb_per;    // k-blocks per split
  float* ws;     // [k_splits][M][N] fp32 partials when k_splits > 1
  void* c;
  long long ldc;
};

template <int BN>
struct GemmCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;   // 16 KB
  static constexpr int B_BYTES = BK * BN * 2;   // 32 KB at BN=256
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN == 256) ? 4 : 6;
  static constexpr int SMEM_BAR = STAGES * STAGE;
  static constexpr int NBAR = 2 * STAGES + 4;
  static constexpr int SMEM_BYTES = SMEM_BAR + NBAR * 8 + 16 + 1024;
  static constexpr int TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
};

constexpr int kGemmThreads = 192;

template <int BN, bool OUT_F32>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const GemmParams p) {
  using C = GemmCfg<BN>;
  asm volatile("griddepcontrol.launch_dependents;");  // the split-K reduce may be scheduled
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::SMEM_BAR);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;      // [2]
  uint64_t* tempty = bars + 2 * C::STAGES + 2; // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);

  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const int lane = threadIdx.x & 31;
  const int out_tiles = p.tiles_m * p.tiles_n;
  const int num_tiles = out_tiles * p.k_splits;  // (output tile, K range) work units
  const int k_blocks = (p.K + C::BK - 1) / C::BK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // programmatic dependent launch: nothing is read or written before the preceding
  // kernel on the stream has completed and its memory is visible
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int ot = tile % out_tiles, ks = tile / out_tiles;
        const int mb = ot % p.tiles_m, nb = ot / p.tiles_m;
        const int kb0 = ks * p.kb_per, kb1 = min(k_blocks, kb0 + p.kb_per);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % C::STAGES;
          mbar_wait<kGemmWaitHint>(&empty[s], ((it / C::STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], C::STAGE);
          uint8_t* sa = smem + s * C::STAGE;
          uint8_t* sb = sa + C::A_BYTES;
          tma_load_2d(sa, &tmA, &full[s], kb * C::BK, mb * C::BM);
#pragma unroll
          for (int c = 0; c < BN / 64; ++c)
            tma_load_2d(sb + c * (C::BK * 128), &tmB, &full[s], nb * BN + c * 64, kb * C::BK);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(128, BN, 0, 1);
      const uint32_t sbase = smem_u32(smem);
      int it = 0, tcount = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tcount) {
        const int acc = tcount & 1;
        mbar_wait<kGemmWaitHint>(&tempty[acc], ((tcount >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        const int kb0 = (tile / out_tiles) * p.kb_per, kb1 = min(k_blocks, kb0 + p.kb_per);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % C::STAGES;
          mbar_wait<kGemmWaitHint>(&full[s], (it / C::STAGES) & 1);
          tc_fence_after();
          const uint32_t sa = sbase + s * C::STAGE;
          const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < C::BK / 16; ++k) {
            const uint64_t ad = sdesc_sw128(sa + k * 32, 16, 1024);
            const uint64_t bd = sdesc_sw128(sb + k * 2048, C::BK * 128, 1024);
            umma_ss(d, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    // epilogue warps 2..5 -> TMEM sub-partitions 2,3,0,1
    const int wq = warp & 3;
    const int r = wq * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    int tcount = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tcount) {
      const int acc = tcount & 1;
      const int ot = tile % out_tiles, ks = tile / out_tiles;
      const int mb = ot % p.tiles_m, nb = ot / p.tiles_m;
      mbar_wait<kGemmWaitHint>(&tfull[acc], (tcount >> 1) & 1);
      tc_fence_after();
      const int row = mb * 128 + r;
      const bool rv = row < p.M;
      // split K: fp32 partial rows [ks][row][N] for gemm_splitk_reduce
      float* const part = p.k_splits > 1 ? p.ws + ((long long)ks * p.M + row) * p.N : nullptr;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + acc * BN + lane_off + c * 32, v);
        tmem_wait_ld();
        const int col0 = nb * BN + c * 32;
        if (rv && col0 < p.N) {
          if (OUT_F32 || part) {
            float* cp = part ? part + col0 : static_cast<float*>(p.c) + (long long)row * p.ldc + col0;
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (col0 + 4 * i < p.N)
                *reinterpret_cast<float4*>(cp + 4 * i) =
                    make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
          } else {
            __nv_bfloat16* cp = static_cast<__nv_bfloat16*>(p.c) + (long long)row * p.ldc + col0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (col0 + 8 * i < p.N)
                *reinterpret_cast<uint4*>(cp + 8 * i) = make_uint4(
                    pack_bf16(__uint_as_float(v[8 * i]), __uint_as_float(v[8 * i + 1])),
                    pack_bf16(__uint_as_float(v[8 * i + 2]), __uint_as_float(v[8 * i + 3])),
                    pack_bf16(__uint_as_float(v[8 * i + 4]), __uint_as_float(v[8 * i + 5])),
                    pack_bf16(__uint_as_float(v[8 * i + 6]), __uint_as_float(v[8 * i + 7])));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// C = sum over k_splits of the fp32 partials (N % 4 == 0), cast to bf16 / fp32
__global__ void gemm_splitk_reduce(const float* __restrict__ ws, int splits, int M, int N, void* c, long long ldc,
                                   bool out_f32) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // launched as a dependent of gemm_kernel
  const long long n4 = (long long)M * N / 4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 acc = reinterpret_cast<const float4*>(ws)[i];
    for (int s = 1; s < splits; ++s) {
      const float4 v = reinterpret_cast<const float4*>(ws + (long long)s * M * N)[i];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    const long long e = i * 4;
    const long long row = e / N, col = e % N;
    if (out_f32) {
      *reinterpret_cast<float4*>(static_cast<float*>(c) + row * ldc + col) = acc;
    } else {
      *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(c) + row * ldc + col) =
          make_uint2(pack_bf16(acc.x, acc.y), pack_bf16(acc.z, acc.w));
    }
  }
}

}  // namespace nt

namespace nt {

// ---------------------------------------------------------------------------
// K3 v2: CTA-pair GEMM (tcgen05.mma.cta_group::2, M = 256 x N = 256 per pair).
// Each CTA of a 2-CTA cluster stages its own 128 rows of A and its own half
// (128 columns) of B per k-block; the pair leader issues one M=256 x N=256
// MMA that reads both CTAs' shared memory and accumulates each CTA's 128 rows
// in its own TMEM.  Per SM the shared-memory traffic per FLOP is 2/3 of the
// single-CTA 128x256 kernel (TMA writes 32 KB + MMA reads 32 KB per 512
// tensor clocks = 125 B/clk against 188 B/clk), which is what bounds the
// single-CTA kernel.
//   warp 0      TMA producer (both CTAs; bytes counted on the leader's barrier)
//   warp 1      MMA issuer (leader CTA only)
//   warps 2-5   epilogue (both CTAs): TMEM -> registers -> global
template <bool OUT_F32>
struct Gemm2Cfg {
  static constexpr int BM = 128, BN = 256, BNH = 128, BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;   // 16 KB: this CTA's 128 rows
  static constexpr int B_BYTES = BK * BNH * 2;  // 16 KB: this CTA's 128 columns
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = 6;
  // epilogue staging: one swizzled 32 x 32 C box per epilogue warp (TMA store)
  static constexpr int OBOX = 32 * 32 * (OUT_F32 ? 4 : 2);
  static constexpr int SMEM_O = STAGES * STAGE;
  static constexpr int SMEM_BAR = SMEM_O + 4 * OBOX;
  static constexpr int NBAR = 2 * STAGES + 4;
  static constexpr int SMEM_BYTES = SMEM_BAR + NBAR * 8 + 16 + 1024;
};

// Pair-tile order: groups of p.group_m tile rows walked column by column.  With
// group_m = tiles_m this is plain column order (A panels stay L2-resident when
// A fits); for large A (8192^3: 32 panels = 128 MB) groups of 8 rows keep the
// ~74 tiles in flight on a few A and B panels.
__device__ __forceinline__ void gemm_tile_coords(const GemmParams& p, int tile, int& mb, int& nb) {
  const int per_group = p.group_m * p.tiles_n;
  const int g = tile / per_group, r = tile - g * per_group;
  const int m0 = g * p.group_m;
  const int gm = min(p.tiles_m - m0, p.group_m);
  mb = m0 + r % gm;
  nb = r / gm;
}

template <bool OUT_F32>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmC, const GemmParams p) {
  asm volatile("griddepcontrol.launch_dependents;");  // a PDL-launched successor may stage its prologue
  using C = Gemm2Cfg<OUT_F32>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::SMEM_BAR);
  uint64_t* full = bars;                        // [STAGES] (leader's counts both CTAs' bytes)
  uint64_t* empty = bars + C::STAGES;           // [STAGES] (multicast commit to both CTAs)
  uint64_t* tfull = bars + 2 * C::STAGES;       // [2]
  uint64_t* tempty = bars + 2 * C::STAGES + 2;  // [2] leader: 4 epilogue warps x 2 CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);

  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = (int)cluster_id_x(), npairs = (int)nclusters_x();
  const int num_tiles = p.tiles_m * p.tiles_n;  // tiles of 256 x 256
  const int k_blocks = (p.K + C::BK - 1) / C::BK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    prefetch_tmap(&tmC);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
    fence_barrier_init();
  }
  cluster_sync_all();  // both CTAs' barriers exist before any remote arrive / complete_tx
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: inputs / outputs only after the predecessor
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int tile = pair; tile < num_tiles; tile += npairs) {
        int mb, nb;
        gemm_tile_coords(p, tile, mb, nb);
        for (int kb = 0; kb < k_blocks; ++kb, ++it) {
          const int s = it % C::STAGES;
          mbar_wait<kGemmWaitHint>(&empty[s], ((it / C::STAGES) & 1) ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * C::STAGE);
          uint8_t* sa = smem + s * C::STAGE;
          uint8_t* sb = sa + C::A_BYTES;
          tma_load_2d_pair(sa, &tmA, &full[s], kb * C::BK, mb * 256 + (int)rank * 128);
#pragma unroll
          for (int c = 0; c < C::BNH / 64; ++c)
            tma_load_2d_pair(sb + c * (C::BK * 128), &tmB, &full[s], nb * 256 + (int)rank * 128 + c * 64,
                             kb * C::BK);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = idesc_bf16(256, 256, 0, 1);
      const uint32_t sbase = smem_u32(smem);
      int it = 0, tcount = 0;
      for (int tile = pair; tile < num_tiles; tile += npairs, ++tcount) {
        const int acc = tcount & 1;
        mbar_wait<kGemmWaitHint>(&tempty[acc], ((tcount >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * 256;
        for (int kb = 0; kb < k_blocks; ++kb, ++it) {
          const int s = it % C::STAGES;
          mbar_wait<kGemmWaitHint>(&full[s], (it / C::STAGES) & 1);
          tc_fence_after();
          const uint32_t sa = sbase + s * C::STAGE;
          const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < C::BK / 16; ++k) {
            const uint64_t ad = sdesc_sw128(sa + k * 32, 16, 1024);
            const uint64_t bd = sdesc_sw128(sb + k * 2048, C::BK * 128, 1024);
            umma_ss_pair(d, ad, bd, idesc, (kb | k) ? 1u : 0u);
          }
          umma_commit_pair(&empty[s], 0x3);
        }
        umma_commit_pair(&tfull[acc], 0x3);
      }
    }
  } else {
    // epilogue warps 2..5 -> TMEM sub-partitions 2,3,0,1; this CTA's 128 rows x 256 columns
    const int wq = warp & 3;
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    int tcount = 0;
    for (int tile = pair; tile < num_tiles; tile += npairs, ++tcount) {
      const int acc = tcount & 1;
      int mb, nb;
      gemm_tile_coords(p, tile, mb, nb);
      mbar_wait<kGemmWaitHint>(&tfull[acc], (tcount >> 1) & 1);
      tc_fence_after();
      // TMEM -> registers -> swizzled smem box -> TMA store (edges clipped by TMA)
      uint8_t* stg = smem + C::SMEM_O + (warp - 2) * C::OBOX;
      const int row0 = mb * 256 + (int)rank * 128 + wq * 32;
#pragma unroll 1
      for (int c = 0; c < C::BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + acc * 256 + lane_off + c * 32, v);
        tmem_wait_ld();
        if (lane == 0) bulk_wait_read0();  // previous box has left shared memory
        __syncwarp();
        if (OUT_F32) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<uint4*>(stg + lane * 128 + ((q ^ (lane & 7)) << 4)) =
                make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<uint4*>(stg + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) = make_uint4(
                pack_bf16(__uint_as_float(v[8 * q]), __uint_as_float(v[8 * q + 1])),
                pack_bf16(__uint_as_float(v[8 * q + 2]), __uint_as_float(v[8 * q + 3])),
                pack_bf16(__uint_as_float(v[8 * q + 4]), __uint_as_float(v[8 * q + 5])),
                pack_bf16(__uint_as_float(v[8 * q + 6]), __uint_as_float(v[8 * q + 7])));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && !NT_GEMM_NO_STORE) {
          tma_store_2d(&tmC, stg, nb * C::BN + c * 32, row0);
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(&tempty[acc], 0));  // the leader's barrier
    }
  }
  if (warp >= 2 && lane == 0) bulk_wait0();  // the last C boxes are written
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the leader's MMAs and both epilogues are done with TMEM
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

}  // namespace nt
