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
// time per SM (e4m3: kind::f8f6f4, K = 32, 4 + 4 MMAs, 16 KB tiles).  S and P are
// double-buffered in TMEM, so S(t+1) is computed while the softmax works on S(t)
// and P(t+1) is stored while PV(t) reads P(t).  An issuing thread blocks on each MMA
// until the tensor pipe takes it, so S and PV have one issuer each; the exps run on
// four warps, one per TMEM lane quarter (DESIGN.md §4 K2b, "What bounds the stream"):
//   warp 1     TMA producer: Q once, then K(t), V(t) through the ring
//   warp 2     S(t) issuer (one thread)          warp 3  PV(t) issuer (one thread)
//   warps 4-7  softmax, warp 4 + q on lane quarter q / keys 32 q + [0, 32) of each
//              tile, an online softmax of its own; the four merged in shared memory
//   warp 0     idle
// TMEM: S_0 [0,128) S_1 [128,256) P_0, P_1 [256,384) O [384,512).
#pragma once
#include "attn_fwd.cuh"
#include "decode.cuh"

namespace nt {

constexpr int kDtcTile = 128;                            // keys per K/V tile
constexpr int kDtcTileBytes = kDtcTile * kDecodeD * 2;   // 32 KB, two 64-dim SW128 panels
constexpr int kDtcHalf = kDtcTile * 128;                 // one panel (16 KB)
constexpr int kDtcStages = 3;                            // K+V tile pairs in flight (192 KB)
// warps 0-3: -, TMA producer, MMA issuer, -; warps 4-7: softmax, one per TMEM lane
// quarter (warp w reaches lanes 32 (w % 4) + [0, 32) only)
constexpr int kDtcThreads = 256;
constexpr int kDtcQuarters = 4;  // key quarters of a tile = softmax warps = partials per split
// Q: the R <= 8 rows fill one 8-row swizzle atom (1 KB) per 64-dim bf16 panel; the
// MMA's A descriptor uses an 8-row-group stride of 0, so that atom is every row
// group of the 128-row tile: rows 32 q + [0, 8) -- TMEM lane quarter q -- hold the
// query rows for every q (rows >= R of the atom are zero)
constexpr int kDtcQBytes = 2048;
// the four quarters' (m, l, O) are merged in shared memory at the end of a split:
// m [4][8], l [4][8], O [4][8][129] fp32 (rows padded against bank conflicts)
constexpr int kDtcMergeBytes = (2 * 4 * 8 + 4 * 8 * 129) * 4;
#ifdef NT_DTC_LOADONLY
constexpr bool kDtcLoadOnly = true;
#else
constexpr bool kDtcLoadOnly = false;
#endif
constexpr int kDtcSmem = kDtcTileBytes /* Q */ + kDtcStages * 2 * kDtcTileBytes + 1024 /* align */ + 256;
// e4m3 K/V (FP8 KV cache): a 128-key tile is one 128-byte panel (16 KB), so twice
// the stages fit -- the same 192 KB in flight
// NT_DTC_E4M3_KPS = 256 moves 256 keys per dense e4m3 ring slot (one 32 KB box: the
// producer alone reads 6.80 TB/s in 16 KB boxes and 7.07 in 32 KB ones; the MMAs and
// the softmax still step in 128-key tiles, SUB per slot).  Measured with the full
// kernel (same box): decode 32K 644 -> 648 us, B=16 8K 89 -> 85 us -- a slot is held
// until both its tiles are consumed, so fewer bytes are in flight; 128 stays default.
#ifndef NT_DTC_E4M3_KPS
#define NT_DTC_E4M3_KPS 128
#endif
template <bool FP8, int PG = 0>
struct DtcCfg {
  static constexpr int KPS = (FP8 && PG == 0) ? NT_DTC_E4M3_KPS : kDtcTile;  // keys per ring slot
  static constexpr int SUB = KPS / kDtcTile;                                 // 128-key tiles per slot
  static constexpr int TILE = KPS * kDecodeD * (FP8 ? 1 : 2);                // bytes per slot
  static constexpr int SUBBYTES = kDtcTile * kDecodeD * (FP8 ? 1 : 2);
  static constexpr int STAGES = (kDtcStages * 2 * kDtcTileBytes) / (2 * TILE);  // 192 KB in flight
  static constexpr int KSTEP = FP8 ? 32 : 16;  // K per tcgen05.mma (kind::f8f6f4 | kind::f16)
  static constexpr int SMEM = kDtcQBytes + STAGES * 2 * TILE + 1024 + 512 + kDtcMergeBytes;  // + align, barriers
};

// PG: 0 dense K/V ([B, Hkv, M, D] viewed as 5-D pages of M tokens); 1 paged cache with
// page_size a multiple of 128 (one 5-D box {64, 128 tokens, 2 panels} per tile);
// 2 paged with 8/16/32/64-token pages (per page slice and 64-dim panel one 4-D box
// {64, page_size} straight into the canonical [panel][128 keys][128 B] tile -- one
// lane per box, the page ids of the next tile fetched while this one is issued)
// exps of one thread's 16 keys (its half of a quarter row): P packed as 8 bf16 pairs
// | 4 e4m3 quads in key order, the sum of the exps returned
template <bool FP8>
__device__ __forceinline__ float dtc_exp_pass(const uint32_t (&s)[16], float sc, float m, uint32_t (&pk)[8]) {
  const float2 sc2 = make_float2(sc, sc), nm2 = make_float2(-m, -m);
  float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  float2 prev = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
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
  using DC = DtcCfg<FP8, PG>;
  constexpr int kTile = DC::TILE, kStages = DC::STAGES, kSub = DC::SUB;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + kDtcQBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + kStages * 2 * kTile);
  uint64_t* bar_q = bars;
  uint64_t* full = bars + 1;               // [2 * stages]: K(t) / V(t) landed
  uint64_t* empty = full + 2 * kStages;    // [2 * stages]
  uint64_t* bar_s = empty + 2 * kStages;   // [2] S(t) in S_{t%2}
  uint64_t* bar_sf = bar_s + 2;              // [2] S_{t%2} loaded into registers (reusable)
  uint64_t* bar_p = bar_sf + 2;              // [2] P(t) in P_{t%2} (4 warps)
  uint64_t* bar_pv = bar_p + 2;              // [2] PV(t) done (P_{t%2} reusable, O current)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_pv + 2);
  float* merge = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 512);

  const int s = blockIdx.x;
  const int grp = blockIdx.y;  // b * Hkv + hkv
  const int b = grp / p.Hkv, hkv = grp % p.Hkv;
  asm volatile("griddepcontrol.launch_dependents;");  // the combine may be scheduled now
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const int lane = threadIdx.x & 31;
  const int j0 = s * p.keys_per_split;  // multiple of kDtcTile
  const int seq_len = PG ? min(p.M, p.seq_lens[b]) : p.M;
  const int j1 = min(seq_len, j0 + p.keys_per_split);
  const int ntiles = (j1 > j0) ? (j1 - j0 + kDtcTile - 1) / kDtcTile : 0;
  const int nslots = (ntiles + kSub - 1) / kSub;  // K (and V) ring slots the split uses
#ifdef NT_TRACE
  // debug timeline (tools/trace_decode.py): clock64 per tile for split g_nt_trace_cta of group 0
  unsigned long long* const tr =
      (g_nt_trace && blockIdx.x == g_nt_trace_cta && blockIdx.y == 0) ? g_nt_trace : nullptr;
#define DTC_STAMP(role, t, ev) \
  do { if (tr && (t) < 64) tr[((role) * 64 + (t)) * 8 + (ev)] = clock64(); } while (0)
#else
#define DTC_STAMP(role, t, ev) do {} while (0)
#endif

  // rows >= R of the Q atom are zero
  for (int i = threadIdx.x; i < kDtcQBytes / 16; i += kDtcThreads)
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
      mbar_init(&bar_sf[i], kDtcQuarters);
      mbar_init(&bar_p[i], kDtcQuarters);
      mbar_init(&bar_pv[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM: S_0 [0,128) S_1 [128,256) P_0, P_1 (64 bf16-pair | 32 e4m3-quad columns each)
  // from 256, O [384,512).  P is double-buffered: P(t+1) is stored while PV(t) reads P(t)
  constexpr uint32_t kColP = 256, kColO = 384, kPCols = FP8 ? 32 : 64;

  if (warp == 1) {
    // ================= TMA producer
    if (ntiles > 0) {
      if (lane == 0) {
        mbar_arrive_expect_tx(bar_q, R * D * (FP8 ? 1 : 2));
        // the group's R rows: box {64 dims (bf16) | 128 dims (e4m3), Nq rows, g heads, 1} per panel
#pragma unroll
        for (int h = 0; h < (FP8 ? 1 : 2); ++h) tma_load_4d(sQ + h * 1024, &tmQ, bar_q, h * 64, 0, hkv * p.g, b);
      }
      if constexpr (PG == 0) {
        if (lane == 0)
          for (int it = 0; it < 2 * nslots; ++it) {
            const int slot = it % (2 * kStages);
            mbar_wait(&empty[slot], ((it / (2 * kStages)) & 1) ^ 1, p.err, 1);
#ifdef NT_DTC_COMPUTEONLY
            // experiment (tools/decode_time.py): the consumers alone, on whatever the ring holds
            mbar_arrive(&full[slot]);
            continue;
#endif
            mbar_arrive_expect_tx(&full[slot], kTile);
            DTC_STAMP(3, it >> 1, it & 1);
            if constexpr (FP8)  // one 4-D box {128 e4m3 dims, KPS keys} = one 128-byte panel
              tma_load_4d(sKV + slot * kTile, (it & 1) ? &tmV : &tmK, &full[slot], 0, j0 + (it >> 1) * DC::KPS,
                          hkv, b);
            else  // one 5-D box {64 dims, 128 keys, 2 panels} = [panel][128 keys][128 B]
              tma_load_5d(sKV + slot * kTile, (it & 1) ? &tmV : &tmK, &full[slot], 0, j0 + (it >> 1) * DC::KPS,
                          0, hkv, b);
          }
      } else {
        const int ps = p.page_size;
        const int* bt = p.block_table + (long long)b * p.bt_stride;
        const int last_page = (seq_len - 1) / ps;
        // PG 2: lane = (page slice, panel) -- e4m3: one panel, lane = slice; PG 1: lane 0 only.
        // When a tile needs <= 16 boxes, K(t) and V(t) go out in one warp step (lanes 0-15
        // K, 16-31 V): half the producer iterations per byte (e4m3 16-token pages: 8 + 8)
        const int nsub = (PG == 2) ? kDtcTile / ps : 1;
        const int per = (PG == 2) ? (FP8 ? 1 : 2) * nsub : 1;  // boxes per K or V tile
        const bool both = per <= 16;
        const int l = both ? (lane & 15) : lane, kvl = both ? (lane >> 4) : 0;
        const int sub = FP8 ? l : l >> 1, panel = FP8 ? 0 : l & 1;
        const bool active = (PG == 2) ? (l < per) : (l == 0);
        auto page_of = [&](int t) -> int2 {  // (physical page, token within it) of this lane's slice
          const int tok = j0 + t * kDtcTile + ((PG == 2) ? sub * ps : 0);
          const int pg = tok / ps;
          const int lp = min(pg, last_page);  // past the sequence end: its last page (masked)
          return make_int2(__ldg(bt + lp), tok - pg * ps);
        };
        int2 cur = active ? page_of(0) : make_int2(0, 0);
        auto issue = [&](int slot, int kv) {
          uint8_t* dst = sKV + slot * kTile;
          const CUtensorMap* m = kv ? &tmV : &tmK;
          if constexpr (PG == 1 && FP8) tma_load_4d(dst, m, &full[slot], 0, cur.y, hkv, cur.x);
          else if constexpr (PG == 1) tma_load_5d(dst, m, &full[slot], 0, cur.y, 0, hkv, cur.x);
          else tma_load_4d(dst + panel * kDtcHalf + sub * ps * 128, m, &full[slot], panel * 64, cur.y, hkv, cur.x);
        };
        for (int t = 0; t < ntiles; ++t) {
          const int2 nxt = (active && t + 1 < ntiles) ? page_of(t + 1) : make_int2(0, 0);
          if (both) {
            const int itK = 2 * t, sK = itK % (2 * kStages), sV = (itK + 1) % (2 * kStages);
            if (lane == 0) {
              mbar_wait(&empty[sK], ((itK / (2 * kStages)) & 1) ^ 1, p.err, 1);
              mbar_wait(&empty[sV], (((itK + 1) / (2 * kStages)) & 1) ^ 1, p.err, 1);
              mbar_arrive_expect_tx(&full[sK], kTile);
              mbar_arrive_expect_tx(&full[sV], kTile);
            }
            __syncwarp();
            if (active) issue(kvl ? sV : sK, kvl);
            cur = nxt;
            continue;
          }
          for (int kv = 0; kv < 2; ++kv) {
            const int it = 2 * t + kv, slot = it % (2 * kStages);
            if (lane == 0) {
              mbar_wait(&empty[slot], ((it / (2 * kStages)) & 1) ^ 1, p.err, 1);
              mbar_arrive_expect_tx(&full[slot], kTile);
            }
            __syncwarp();
            if (active) issue(slot, kv);
          }
          cur = nxt;
        }
      }
    }
  } else if (warp == 2 || warp == 3) {
    // ================= MMA issuers: warp 2 the score MMAs S(t), warp 3 the PV(t) MMAs.
    // An issuing thread blocks for each MMA until the tensor pipe takes it (~64 clk)
    // and spends ~100 clk per mbarrier wait and ~60 per commit even when nothing is
    // pending (tools/trace_decode.py): one thread doing both chains left the tensor
    // pipe idle ~60 % of a tile.  The two chains only meet through the softmax's
    // barriers (S_{t%2} read -> S(t+2); P(t) stored -> PV(t)), so two issuers are safe
#ifdef NT_DTC_LOADONLY
    // experiment (tools/decode_time.py): the producer's stream alone, slots released as they land
    if (lane == 0 && warp == 2)
      for (int it = 0; it < 2 * nslots; ++it) {
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
      // tile t lives in ring slot t / kSub at (t % kSub) x SUBBYTES; a slot is released
      // by the commit after its last tile's MMAs
      auto last_of_slot = [&](int t) { return t % kSub == kSub - 1 || t == ntiles - 1; };
      auto issue_s = [&](int t) {
        const int gk = 2 * (t / kSub), slotK = gk % (2 * kStages);
        const uint32_t so = (t % kSub) * DC::SUBBYTES;
        mbar_wait(&full[slotK], (gk / (2 * kStages)) & 1, p.err, 3);
        DTC_STAMP(0, t, 3);
        if (t >= 2) mbar_wait(&bar_sf[t & 1], ((t >> 1) - 1) & 1, p.err, 6);  // softmax(t-2) read S_{t%2}
        DTC_STAMP(0, t, 4);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < D / DC::KSTEP; ++k) {
          // 32 bytes of K per instruction, 4 per 128-byte panel row
          const uint64_t ad = sdesc_sw128(sQa + (k >> 2) * 1024 + (k & 3) * 32, 16, 0);  // the Q atom, every row group
          const uint64_t bd = sdesc_sw128(sKVa + slotK * kTile + so + (k >> 2) * kDtcHalf + (k & 3) * 32, 16, 1024);
          if constexpr (FP8) umma_ss_f8(tmem + (t & 1) * 128, ad, bd, idS, k > 0 ? 1u : 0u);
          else umma_ss(tmem + (t & 1) * 128, ad, bd, idS, k > 0 ? 1u : 0u);
        }
        DTC_STAMP(0, t, 5);
        umma_commit(&bar_s[t & 1]);
        if (last_of_slot(t)) umma_commit(&empty[slotK]);
        DTC_STAMP(0, t, 0);
      };
      if (warp == 2) {
        mbar_wait(bar_q, 0, p.err, 2);
        for (int t = 0; t < ntiles; ++t) issue_s(t);
      } else for (int t = 0; t < ntiles; ++t) {
        // PV(t): P from its own TMEM columns, V MN-major from shared memory
        const int gv = 2 * (t / kSub) + 1, slotV = gv % (2 * kStages);
        const uint32_t so = (t % kSub) * DC::SUBBYTES;
        mbar_wait(&bar_p[t & 1], (t >> 1) & 1, p.err, 4);
        DTC_STAMP(0, t, 1);
        mbar_wait(&full[slotV], (gv / (2 * kStages)) & 1, p.err, 5);
        DTC_STAMP(0, t, 6);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kDtcTile / DC::KSTEP; ++k) {
          // KSTEP keys of V (MN-major, 128-byte rows) x P's 8 TMEM columns (bf16 pairs | e4m3 quads)
          const uint64_t bd = sdesc_sw128(sKVa + slotV * kTile + so + k * DC::KSTEP * 128, kDtcHalf, 1024);
          const uint32_t ta = tmem + kColP + (t & 1) * kPCols + k * 8;
          if constexpr (FP8) umma_ts_f8(tmem + kColO, ta, bd, idO, (t > 0 || k > 0) ? 1u : 0u);
          else umma_ts(tmem + kColO, ta, bd, idO, (t > 0 || k > 0) ? 1u : 0u);
        }
        DTC_STAMP(0, t, 7);
        umma_commit(&bar_pv[t & 1]);
        if (last_of_slot(t)) umma_commit(&empty[slotV]);
        DTC_STAMP(0, t, 2);
      }
    }
  } else if (warp >= 4 && !kDtcLoadOnly) {
    // ================= softmax: warp 4 + q owns TMEM lane quarter q (its rows 0-7 are
    // the query rows, see kDtcQBytes) and keys 32 q + [0, 32) of every tile; two threads
    // per row through the .16x32bx2 fragment (thread t: row t % 16, keys 32 q +
    // (t / 16) * 16 + [0, 16)).  Each quarter is an independent online softmax -- its
    // own m, l and O rows, P zero outside its key columns -- left as its own partial,
    // so the exps run on all four SMSPs' MUFUs with no exchange between the warps
    const int q = warp & 3;
    const uint32_t lq = (uint32_t)(32 * q) << 16;  // TMEM lane field of this quarter
    const float NINF = f_ninf();
    const float sc = p.scale_log2;
    const uint32_t tO = tmem + lq + kColO, tP = tmem + lq + kColP;
    const int half = lane >> 4;
    float m_run = NINF, l_run = 0.f;
    {
      // P outside this quarter's key columns (and rows 16-31) stays zero all launch
      uint32_t z[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) z[i] = 0u;
#pragma unroll
      for (int c = 0; c < 2 * kPCols / 16; ++c) tmem_st16(tP + c * 16, z);
    }
    for (int t = 0; t < ntiles; ++t) {
      mbar_wait(&bar_s[t & 1], (t >> 1) & 1, p.err, 8);
      if (q == 0 && lane == 0) DTC_STAMP(1, t, 0);
      tc_fence_after();
      uint32_t sv[16];
      tmem_ld16_x2<16>(tmem + lq + (t & 1) * 128 + q * 32, sv);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_sf[t & 1]);  // S_{t%2} may take S(t+2)
      if (q == 0 && lane == 0) DTC_STAMP(1, t, 1);
      const int kv0 = j0 + t * kDtcTile + q * 32 + half * 16;
      if (kv0 + 16 > j1) {
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (kv0 + c >= j1) sv[c] = __float_as_uint(NINF);
      }
      float a0 = fmax3(__uint_as_float(sv[0]), __uint_as_float(sv[1]), __uint_as_float(sv[2]));
      float a1 = fmax3(__uint_as_float(sv[3]), __uint_as_float(sv[4]), __uint_as_float(sv[5]));
#pragma unroll
      for (int c = 6; c + 4 <= 14; c += 4) {
        a0 = fmax3(a0, __uint_as_float(sv[c]), __uint_as_float(sv[c + 1]));
        a1 = fmax3(a1, __uint_as_float(sv[c + 2]), __uint_as_float(sv[c + 3]));
      }
      float mx = fmaxf(fmax3(a0, a1, __uint_as_float(sv[14])), __uint_as_float(sv[15]));
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
      uint32_t pk[8];
      l_run += dtc_exp_pass<FP8>(sv, sc, m_use, pk);  // exps into registers (this half's l)
      if (q == 0 && lane == 0) DTC_STAMP(1, t, 2);
      if (t > 0 && rescale) {
        // O must hold every PV so far before it is rescaled
        mbar_wait(&bar_pv[(t - 1) & 1], ((t - 1) >> 1) & 1, p.err, 10);
        tc_fence_after();
        // 32x32b: lane t's row of this quarter; rows 16-31 are zero
        attn_rescale_o<D>(tO, alpha);
      } else if (t > 1) {
        // PV(t-2) read P_{t%2} (long done): P(t) may overwrite it
        mbar_wait(&bar_pv[t & 1], ((t - 2) >> 1) & 1, p.err, 10);
        tc_fence_after();
      }
      if (q == 0 && lane == 0) DTC_STAMP(1, t, 3);
      const uint32_t tPb = tP + (t & 1) * kPCols;
      if constexpr (FP8) tmem_st4_x2<4>(tPb + q * 8, pk);  // e4m3 quads: columns 8 q + 4 half + [0, 4)
      else tmem_st8_x2<8>(tPb + q * 16, pk);                // bf16 pairs: columns 16 q + 8 half + [0, 8)
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_p[t & 1]);
      if (q == 0 && lane == 0) DTC_STAMP(1, t, 4);
    }
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 16);  // both halves' sums (same m_run)
    // ---- epilogue: merge the four quarters' (m, l, O) (the repair law) in shared
    // memory, rows < R -> the split's partial (O unnormalised, m, l) in the workspace
    float* sm_m = merge;               // [4][8]
    float* sm_l = merge + 32;          // [4][8]
    float* sm_o = merge + 64;          // [4][8][129]
    if (lane < R) sm_m[q * 8 + lane] = m_run;
    named_bar_sync(1, 128);
    float mm = NINF;
#pragma unroll
    for (int qq = 0; qq < kDtcQuarters; ++qq) mm = fmaxf(mm, sm_m[qq * 8 + (lane & 7)]);
    const float wq = (m_run == NINF) ? 0.f : ex2(m_run - mm) * p.o_scale;  // this quarter's weight
    float* so = sm_o + (q * 8 + lane) * 129;
    if (ntiles > 0) {
      mbar_wait(&bar_pv[(ntiles - 1) & 1], ((ntiles - 1) >> 1) & 1, p.err, 9);  // the last PV
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + c * 32, o);
        tmem_wait_ld();
        if (lane < R) {
#pragma unroll
          for (int i = 0; i < 32; ++i) so[c * 32 + i] = __uint_as_float(o[i]) * wq;
        }
      }
    } else if (lane < R) {
      for (int c = 0; c < D; ++c) so[c] = 0.f;  // empty split: weight 0, finite O
    }
    if (lane < R) sm_l[q * 8 + lane] = l_run * (m_run == NINF ? 0.f : ex2(m_run - mm));
    named_bar_sync(1, 128);
    // warp q sums columns 32 q + lane of every row
    float* w = p.ws + ((long long)grp * p.splits + s) * R * (D + 2);
    for (int r = 0; r < R; ++r) {
      float acc = 0.f;
#pragma unroll
      for (int qq = 0; qq < kDtcQuarters; ++qq) acc += sm_o[(qq * 8 + r) * 129 + q * 32 + lane];
      w[r * (D + 2) + q * 32 + lane] = acc;
    }
    if (q == 0 && lane < R) {
      float ll = 0.f;
#pragma unroll
      for (int qq = 0; qq < kDtcQuarters; ++qq) ll += sm_l[qq * 8 + lane];
      w[lane * (D + 2) + D] = mm;
      w[lane * (D + 2) + D + 1] = ll;
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
