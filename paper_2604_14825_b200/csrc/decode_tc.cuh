// K2b: split-KV decode attention on the tensor cores -- HBM-bound.
//
// Same work decomposition and partial format as K2 (decode.cuh): one CTA per
// (split, batch x kv-head group), the group's R = (Hq/Hkv) * Nq query rows run
// the rolling-update recurrence over the split's key range and leave an fp32
// partial (O unnormalised, m, l) for decode_combine_kernel (the repair law,
// tilecc/schedule/repair.py:80-88).  K2 does the dots on the FMA pipe and
// measured issue-bound (ncu: FFMA2 / FADD / SHF / LOP3 carry ~55 % of the stall
// samples; 5.6 TB/s against a 7.4 TB/s TMA read ceiling, tools/ubench/bulk_read.cu).
// Here the dots are tcgen05 MMAs with the R rows padded to M = 128:
//   S(t)  = Q (128 x 128, rows >= R zero) . K(t)^T      SS, 8 x (M128 N128 K16)
//   O    += P(t) (TMEM, bf16) . V(t)                     TS, 8 x (M128 N128 K16)
// 1024 tensor clocks per 128-key K/V tile pair (64 KB) against ~2500 clocks of HBM
// time per SM.  S is double-buffered in TMEM and P has its own columns, so S(t+1)
// is computed while the softmax warp works on S(t): the per-tile chain is the
// softmax alone (~1200 clk: one warp, MUFU-bound), not S + softmax + PV (a first
// version with P aliasing S measured 5.80 TB/s, this chain ~2900 clk per tile).
//   warp 0  softmax (TMEM lanes 0-31; lane = row, lanes < R matter), epilogue
//   warp 1  TMA producer: Q once, then K(t), V(t) through a kDtcStages ring
//   warp 2  MMA issuer (one thread): S(t+1) ahead, PV(t) when P(t) is ready
//   warp 3  idle
// TMEM: S_0 [0,128) S_1 [128,256) P [256,320) O [384,512).
#pragma once
#include "attn_fwd.cuh"
#include "decode.cuh"

namespace nt {

constexpr int kDtcTile = 128;                            // keys per K/V tile
constexpr int kDtcTileBytes = kDtcTile * kDecodeD * 2;   // 32 KB, two 64-dim SW128 panels
constexpr int kDtcHalf = kDtcTile * 128;                 // one panel (16 KB)
constexpr int kDtcStages = 3;                            // K+V tile pairs in flight (192 KB)
constexpr int kDtcThreads = 128;
#ifdef NT_DTC_LOADONLY
constexpr bool kDtcLoadOnly = true;
#else
constexpr bool kDtcLoadOnly = false;
#endif
constexpr int kDtcSmem = kDtcTileBytes /* Q */ + kDtcStages * 2 * kDtcTileBytes + 1024 /* align */ + 256;
// e4m3 K/V (FP8 KV cache): a 128-key tile is one 128-byte panel (16 KB), so twice
// the stages fit -- the same 192 KB in flight
template <bool FP8>
struct DtcCfg {
  static constexpr int TILE = kDtcTile * kDecodeD * (FP8 ? 1 : 2);
  static constexpr int STAGES = FP8 ? 6 : kDtcStages;
  static constexpr int KSTEP = FP8 ? 32 : 16;  // K per tcgen05.mma (kind::f8f6f4 | kind::f16)
  static constexpr int SMEM = TILE + STAGES * 2 * TILE + 1024 + (FP8 ? 512 : 256);  // + barriers
};

// PG: 0 dense K/V ([B, Hkv, M, D] viewed as 5-D pages of M tokens); 1 paged cache with
// page_size a multiple of 128 (one 5-D box {64, 128 tokens, 2 panels} per tile);
// 2 paged with 8/16/32/64-token pages (per page slice and 64-dim panel one 4-D box
// {64, page_size} straight into the canonical [panel][128 keys][128 B] tile -- one
// lane per box, the page ids of the next tile fetched while this one is issued)
// exps of one thread's 64 keys (a half row): P packed as 32 bf16 pairs | 16 e4m3
// quads in key order, the sum of the exps returned
template <bool FP8>
__device__ __forceinline__ float dtc_exp_pass(const uint32_t (&s)[64], float sc, float m, uint32_t (&pk)[32]) {
  const float2 sc2 = make_float2(sc, sc), nm2 = make_float2(-m, -m);
  float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  float2 prev = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const float2 x = ffma2(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), sc2, nm2);
    const float2 e = make_float2(ex2(x.x), ex2(x.y));
    sum2[i & 1] = fadd2(sum2[i & 1], e);
    if constexpr (FP8) {
      if (i & 1) pk[i >> 1] = pack_e4m3x4(prev.x, prev.y, e.x, e.y);
      prev = e;
    } else {
      pk[i] = pack_bf16(e.x, e.y);
    }
  }
  return (sum2[0].x + sum2[0].y) + (sum2[1].x + sum2[1].y);
}

template <int R, int PG = 0, bool FP8 = false>
__global__ void __launch_bounds__(kDtcThreads, 1)
    decode_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const DecodeParams p) {
  constexpr int D = kDecodeD;
  using DC = DtcCfg<FP8>;
  constexpr int kTile = DC::TILE, kStages = DC::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + kTile;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + kStages * 2 * kTile);
  uint64_t* bar_q = bars;
  uint64_t* full = bars + 1;               // [2 * stages]: K(t) / V(t) landed
  uint64_t* empty = full + 2 * kStages;    // [2 * stages]
  uint64_t* bar_s = empty + 2 * kStages;   // [2] S(t) in S_{t%2}
  uint64_t* bar_sf = bar_s + 2;              // [2] S_{t%2} loaded into registers (reusable)
  uint64_t* bar_p = bar_sf + 2;              // P(t) in TMEM
  uint64_t* bar_pv = bar_p + 1;              // PV(t) done (P and O reusable)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_pv + 1);

  const int s = blockIdx.x;
  const int grp = blockIdx.y;  // b * Hkv + hkv
  const int b = grp / p.Hkv, hkv = grp % p.Hkv;
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const int lane = threadIdx.x & 31;
  const int j0 = s * p.keys_per_split;  // multiple of kDtcTile
  const int seq_len = PG ? min(p.M, p.seq_lens[b]) : p.M;
  const int j1 = min(seq_len, j0 + p.keys_per_split);
  const int ntiles = (j1 > j0) ? (j1 - j0 + kDtcTile - 1) / kDtcTile : 0;
#ifdef NT_TRACE
  // debug timeline (tools/trace_decode.py): clock64 per tile for split g_nt_trace_cta of group 0
  unsigned long long* const tr =
      (g_nt_trace && blockIdx.x == g_nt_trace_cta && blockIdx.y == 0) ? g_nt_trace : nullptr;
#define DTC_STAMP(role, t, ev) \
  do { if (tr && (t) < 64) tr[((role) * 64 + (t)) * 8 + (ev)] = clock64(); } while (0)
#else
#define DTC_STAMP(role, t, ev) do {} while (0)
#endif

  // rows >= R of the padded Q tile are zero (S, P, O rows >= R are never read)
  for (int i = threadIdx.x; i < kTile / 16; i += kDtcThreads)
    reinterpret_cast<uint4*>(sQ)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (warp == 1 && lane == 0) {
    prefetch_tmap(&tmQ);
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    mbar_init(bar_q, 1);
    for (int i = 0; i < 2 * kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_s[i], 1);
      mbar_init(&bar_sf[i], 1);
    }
    mbar_init(bar_p, 1);
    mbar_init(bar_pv, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t kColP = 256, kColO = 384;

  if (warp == 1) {
    // ================= TMA producer
    if (ntiles > 0) {
      if (lane == 0) {
        mbar_arrive_expect_tx(bar_q, R * D * (FP8 ? 1 : 2));
        // the group's R rows: box {64 dims (bf16) | 128 dims (e4m3), Nq rows, g heads, 1} per panel
#pragma unroll
        for (int h = 0; h < (FP8 ? 1 : 2); ++h) tma_load_4d(sQ + h * kDtcHalf, &tmQ, bar_q, h * 64, 0, hkv * p.g, b);
      }
      if constexpr (PG == 0) {
        if (lane == 0)
          for (int it = 0; it < 2 * ntiles; ++it) {
            const int slot = it % (2 * kStages);
            mbar_wait(&empty[slot], ((it / (2 * kStages)) & 1) ^ 1, p.err, 1);
#ifdef NT_DTC_COMPUTEONLY
            // experiment (tools/decode_time.py): the consumers alone, on whatever the ring holds
            mbar_arrive(&full[slot]);
            continue;
#endif
            mbar_arrive_expect_tx(&full[slot], kTile);
            DTC_STAMP(3, it >> 1, it & 1);
            if constexpr (FP8)  // one 4-D box {128 e4m3 dims, 128 keys} = one 128-byte panel
              tma_load_4d(sKV + slot * kTile, (it & 1) ? &tmV : &tmK, &full[slot], 0, j0 + (it >> 1) * kDtcTile,
                          hkv, b);
            else  // one 5-D box {64 dims, 128 keys, 2 panels} = [panel][128 keys][128 B]
              tma_load_5d(sKV + slot * kTile, (it & 1) ? &tmV : &tmK, &full[slot], 0, j0 + (it >> 1) * kDtcTile,
                          0, hkv, b);
          }
      } else {
        const int ps = p.page_size;
        const int* bt = p.block_table + (long long)b * p.bt_stride;
        const int last_page = (seq_len - 1) / ps;
        // PG 2: lane = (page slice, panel) -- e4m3: one panel, lane = slice; PG 1: lane 0 only
        const int nsub = (PG == 2) ? kDtcTile / ps : 1;
        const int sub = FP8 ? lane : lane >> 1, panel = FP8 ? 0 : lane & 1;
        const bool active = (PG == 2) ? (lane < (FP8 ? 1 : 2) * nsub) : (lane == 0);
        auto page_of = [&](int t) -> int2 {  // (physical page, token within it) of this lane's slice
          const int tok = j0 + t * kDtcTile + ((PG == 2) ? sub * ps : 0);
          const int pg = tok / ps;
          const int lp = min(pg, last_page);  // past the sequence end: its last page (masked)
          return make_int2(__ldg(bt + lp), tok - pg * ps);
        };
        int2 cur = active ? page_of(0) : make_int2(0, 0);
        for (int t = 0; t < ntiles; ++t) {
          const int2 nxt = (active && t + 1 < ntiles) ? page_of(t + 1) : make_int2(0, 0);
          for (int kv = 0; kv < 2; ++kv) {
            const int it = 2 * t + kv, slot = it % (2 * kStages);
            if (lane == 0) {
              mbar_wait(&empty[slot], ((it / (2 * kStages)) & 1) ^ 1, p.err, 1);
              mbar_arrive_expect_tx(&full[slot], kTile);
            }
            __syncwarp();
            if (active) {
              uint8_t* dst = sKV + slot * kTile;
              const CUtensorMap* m = kv ? &tmV : &tmK;
              if constexpr (PG == 1 && FP8) tma_load_4d(dst, m, &full[slot], 0, cur.y, hkv, cur.x);
              else if constexpr (PG == 1) tma_load_5d(dst, m, &full[slot], 0, cur.y, 0, hkv, cur.x);
              else tma_load_4d(dst + panel * kDtcHalf + sub * ps * 128, m, &full[slot], panel * 64, cur.y, hkv, cur.x);
            }
          }
          cur = nxt;
        }
      }
    }
  } else if (warp == 2) {
    // ================= MMA issuer
#ifdef NT_DTC_LOADONLY
    // experiment (tools/decode_time.py): the producer's stream alone, slots released as they land
    if (lane == 0)
      for (int it = 0; it < 2 * ntiles; ++it) {
        mbar_wait(&full[it % (2 * kStages)], (it / (2 * kStages)) & 1, p.err, 3);
        mbar_arrive(&empty[it % (2 * kStages)]);
      }
    if (false) {
#else
    if (lane == 0 && ntiles > 0) {
#endif
      constexpr uint32_t idS = FP8 ? idesc_e4m3(128, 128, 0, 0) : idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idO = FP8 ? idesc_e4m3(128, D, 0, 1) : idesc_bf16(128, D, 0, 1);
      const uint32_t sQa = smem_u32(sQ), sKVa = smem_u32(sKV);
      mbar_wait(bar_q, 0, p.err, 2);
      auto issue_s = [&](int t) {
        const int gk = 2 * t, slotK = gk % (2 * kStages);
        mbar_wait(&full[slotK], (gk / (2 * kStages)) & 1, p.err, 3);
        if (t >= 2) mbar_wait(&bar_sf[t & 1], ((t >> 1) - 1) & 1, p.err, 6);  // softmax(t-2) read S_{t%2}
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < D / DC::KSTEP; ++k) {
          // 32 bytes of K per instruction, 4 per 128-byte panel row
          const uint32_t off = (k >> 2) * kDtcHalf + (k & 3) * 32;
          const uint64_t ad = sdesc_sw128(sQa + off, 16, 1024), bd = sdesc_sw128(sKVa + slotK * kTile + off, 16, 1024);
          if constexpr (FP8) umma_ss_f8(tmem + (t & 1) * 128, ad, bd, idS, k > 0 ? 1u : 0u);
          else umma_ss(tmem + (t & 1) * 128, ad, bd, idS, k > 0 ? 1u : 0u);
        }
        umma_commit(&bar_s[t & 1]);
        umma_commit(&empty[slotK]);
        DTC_STAMP(0, t, 0);
      };
      issue_s(0);
      for (int t = 0; t < ntiles; ++t) {
        if (t + 1 < ntiles) issue_s(t + 1);
        // PV(t): P from its own TMEM columns, V MN-major from shared memory
        const int gv = 2 * t + 1, slotV = gv % (2 * kStages);
        mbar_wait(bar_p, t & 1, p.err, 4);
        DTC_STAMP(0, t, 1);
        mbar_wait(&full[slotV], (gv / (2 * kStages)) & 1, p.err, 5);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kDtcTile / DC::KSTEP; ++k) {
          // KSTEP keys of V (MN-major, 128-byte rows) x P's 8 TMEM columns (bf16 pairs | e4m3 quads)
          const uint64_t bd = sdesc_sw128(sKVa + slotV * kTile + k * DC::KSTEP * 128, kDtcHalf, 1024);
          if constexpr (FP8) umma_ts_f8(tmem + kColO, tmem + kColP + k * 8, bd, idO, (t > 0 || k > 0) ? 1u : 0u);
          else umma_ts(tmem + kColO, tmem + kColP + k * 8, bd, idO, (t > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(bar_pv);
        umma_commit(&empty[slotV]);
        DTC_STAMP(0, t, 2);
      }
    }
  } else if (warp == 0 && !kDtcLoadOnly) {
    // ================= softmax: two threads per query row (R <= 8 rows live in
    // TMEM lanes 0-15): thread t holds row t % 16, keys (t / 16) * 64 + [0, 64)
    // of each tile, through the .16x32bx2 fragment -- half the exps per thread
    // of a one-row-per-thread loop, which on a 1-group-per-CTA decode is the chain
    const float NINF = f_ninf();
    const float sc = p.scale_log2;
    const uint32_t tO = tmem + kColO, tP = tmem + kColP;  // warp 0: lanes 0-31
    const int half = lane >> 4;
    float m_run = NINF, l_run = 0.f;
    for (int t = 0; t < ntiles; ++t) {
      mbar_wait(&bar_s[t & 1], (t >> 1) & 1, p.err, 8);
      if (lane == 0) DTC_STAMP(1, t, 0);
      tc_fence_after();
      uint32_t sv[64];
      tmem_ld32_x2<64>(tmem + (t & 1) * 128, sv);
      tmem_ld32_x2<64>(tmem + (t & 1) * 128 + 32, sv + 32);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_sf[t & 1]);  // S_{t%2} may take S(t+2)
      if (lane == 0) DTC_STAMP(1, t, 1);
      const int kv0 = j0 + t * kDtcTile + half * 64;
      if (kv0 + 64 > j1) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (kv0 + c >= j1) sv[c] = __float_as_uint(NINF);
      }
      float a0 = __uint_as_float(sv[0]), a1 = __uint_as_float(sv[1]);
#pragma unroll
      for (int c = 2; c + 4 <= 64; c += 4) {
        a0 = fmax3(a0, __uint_as_float(sv[c]), __uint_as_float(sv[c + 1]));
        a1 = fmax3(a1, __uint_as_float(sv[c + 2]), __uint_as_float(sv[c + 3]));
      }
      a0 = fmax3(a0, a1, __uint_as_float(sv[62]));
      float mx = fmaxf(a0, __uint_as_float(sv[63]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));  // the row's other half
      const float m_new = fmaxf(m_run, mx * sc);
      float alpha = 1.0f;
      const bool rescale = __any_sync(0xffffffffu, m_new > m_run + kRescaleLog2);
      if (rescale) {
        alpha = (m_new == NINF) ? 1.0f : ex2(m_run - m_new);
        l_run *= alpha;
        m_run = m_new;
      }
      const float m_use = (m_run == NINF) ? 0.f : m_run;
      uint32_t pk[32];
      l_run += dtc_exp_pass<FP8>(sv, sc, m_use, pk);  // exps into registers (this half's l)
      if (lane == 0) DTC_STAMP(1, t, 2);
      if (t > 0) {
        // PV(t-1) read P(t-1) and wrote O: now P(t) may overwrite it and O be rescaled
        mbar_wait(bar_pv, (t - 1) & 1, p.err, 10);
        if (lane == 0) DTC_STAMP(1, t, 3);
        tc_fence_after();
        // 32x32b: lane t's row; lanes 16-31 are rows past R (nothing reads them)
        if (rescale) attn_rescale_o<D>(tO, alpha);
      }
      if constexpr (FP8) {
        tmem_st16_x2<16>(tP, pk);  // e4m3 quads: columns half * 16 + [0, 16)
      } else {
        tmem_st16_x2<32>(tP, pk);  // bf16 pairs: columns half * 32 + [0, 32)
        tmem_st16_x2<32>(tP + 16, pk + 16);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_p);
      if (lane == 0) DTC_STAMP(1, t, 4);
    }
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 16);  // both halves' sums (same m_run)
    // ---- epilogue: rows < R -> partial (O unnormalised, m, l) in the workspace
    float* w = p.ws + ((long long)grp * p.splits + s) * R * (D + 2);
    if (ntiles > 0) {
      mbar_wait(bar_pv, (ntiles - 1) & 1, p.err, 9);  // the last PV
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + c * 32, o);
        tmem_wait_ld();
        if (lane < R) {  // partial rows are D + 2 floats: 8-byte aligned
#pragma unroll
          for (int q = 0; q < 16; ++q)
            *reinterpret_cast<float2*>(w + lane * (D + 2) + c * 32 + 2 * q) =
                make_float2(__uint_as_float(o[2 * q]) * p.o_scale, __uint_as_float(o[2 * q + 1]) * p.o_scale);
        }
      }
    } else if (lane < R) {
      for (int c = 0; c < D; ++c) w[lane * (D + 2) + c] = 0.f;  // empty split: weight 0, finite O
    }
    if (lane < R) {
      w[lane * (D + 2) + D] = m_run;
      w[lane * (D + 2) + D + 1] = l_run;
    }
  }

  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace nt
