// K1: fused attention forward for sm_100a -- realises the auto-scheduler's
// "1 loop, 2 dots, 3 carried accumulators" MA kernel (SURVEY.md B.2,
// tilecc/ma/interp.py:102-280 executes it on the CPU today).
//
// MA semantics per query block (tile t0_i rows), ascending KV tiles j0:
//   S  = Q_s . (K_s * c)^T                       (VDot, fp32 accumulate)
//   m' = max(S [+ Mask], axis=1, init=m)         (VReduce max)
//   a  = exp2(log2e * (m - m'))                  (repair law, tilecc/schedule/repair.py:70-78)
//   P  = exp2(log2e * (S [+ Mask] - m'))
//   l' = sum(P, axis=1, init=l * a)
//   O' = dot(P, V, acc = O * a)
//   O  = O / l   after the loop (telescoped division)
//
// Work item = two 128-row query tiles (256 rows = 256/t0_i consecutive MA
// blocks) of one (batch, head), sharing each 128-row K/V tile (128/t0_j
// consecutive MA j0 iterations; the rolling-update law makes the coarsening
// exact up to rounding).  The kernel is PERSISTENT: a grid of at most one CTA
// per SM walks the item list (heaviest causal items first), each CTA drawing
// its next item from a global counter when it starts one (greedy LPT, like the
// hardware block scheduler), and keeps TMEM, barriers and the K/V ring alive
// across items, so the next item's Q load and first score GEMMs overlap the
// current item's epilogue.  The producer warp draws items and hands them to
// the MMA and softmax warps through a small ring in shared memory.
//
//   warp 0      TMA producer: per item Q0,Q1 (once their previous contents are
//               consumed), then K0,V0,K1,V1,... into a STAGES ring
//   warp 1      MMA issuer (one thread): S_t = Q_t K_j^T (SS), O_t += P_t V_j (TS, P from TMEM)
//   warps 2-3   idle (warpgroup 0 donates registers via setmaxnreg)
//   warps 4-7   softmax + epilogue for tile 0 (one thread per query row = TMEM lane)
//   warps 8-11  softmax + epilogue for tile 1
// TMEM (512 cols): S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [384,384+D);
// P_t (bf16, 64 cols) aliases the first half of S_t.
//
// NQ = 1 ("128-row items"): the same pipeline with ONE query tile per item and
// one softmax warpgroup (256 threads, 256 TMEM columns: S [0,128), O [128,..)),
// sized so that TWO CTAs share an SM.  The two co-resident CTAs are independent
// streams of work items -- each with its own Q, K/V ring and barriers -- so one
// CTA's item boundary (Q landing, first S, epilogue) overlaps the other CTA's
// KV loop, and items are half as long (finer LPT balance).  This is the MA's
// t0_i choice made real on the GPU: 128 vs 256 query rows per work item.
//
// Numerics: bf16 operands, fp32 accumulation, P rounded to bf16 before P.V.
// The scale c is folded into the exp2 constant (c*log2e), which differs from
// the MA's K_s*c only in rounding.  The running max is updated lazily: a warp
// only moves its rows' max (and rescales O, l) when some row's max grew by more
// than RESCALE_LOG2 (values of P stay <= 2^RESCALE_LOG2); the final O/l is the
// same quantity, so this is an exact identity up to rounding.  Rows whose max
// is still -inf use 0 in place of the max (the FA -inf guard the MA lacks,
// SURVEY.md B.14).
#pragma once
#include "sm100.cuh"

namespace nt {

// MASK_BITS: a 0 / -inf Mask packed to one bit per key (nt_mask_to_bits): the
// softmax reads 16 bytes per row per 128-key tile instead of 512 bytes of fp32
enum { MASK_NONE = 0, MASK_CAUSAL = 1, MASK_TENSOR = 2, MASK_BITS = 3 };

struct AttnFwdParams {
  int B, Hq, Hkv, N, M;
  int q_per_kv;
  int n_mblocks;      // ceil(N / rows per item)
  int n_kv_total;     // ceil(M / 128)
  int n_items;        // n_mblocks * B * Hq
  int causal_offset;  // key j visible to query i iff j <= i + causal_offset
  float scale_log2;   // c * log2(e)
  const float* mask;  // MASK_TENSOR: fp32 [N, M]; MASK_BITS: uint32 bit rows (bit j: key j visible)
  long long mask_row_stride;
  void* o;            // output (bf16, or fp32 if OUT_F32), element strides below; D contiguous
  long long o_sb, o_sh, o_sn;
  int* err;  // bit 0: zero denominator (fully masked row); bit 8+k: wait k timed out
  int* work;  // [next, done] dynamic item counter (zero at launch, reset by the last CTA) or null
  float o_scale;  // e4m3 inputs: V's descale (O = o_scale * P.V / l), else 1
  // Split KV (few, long work items -- e.g. one kv-group per GPU at 8 GPUs): an item
  // whose KV range exceeds kv_split tiles becomes ceil(n_kv / kv_split) work units;
  // each writes an fp32 partial (O unnormalised, m, l) that attn_combine_kernel
  // merges with the repair law.  kv_split = 0: one unit per item (n_items units).
  int kv_split;
  int* unit_prefix;  // [n_mblocks + 1] units before each m-block position (written by CTA 0)
  int n_split_mb;    // m-block positions 0 .. n_split_mb-1 (LPT order) hold split items (the merge grid)
  float2* part_ml;   // [unit][256 rows] (m, l)
};
constexpr int kMaxSplitMblocks = 384;  // prefix table size in shared memory

template <int NQ>
constexpr int attn_threads() { return 128 + 128 * NQ; }
constexpr int kAttnThreads = attn_threads<2>();
#ifndef NT_REG_LO64
#define NT_REG_LO64 104  // D=64 register split (88 / 96 / 104 -> softmax 208 / 204 / 200)
#endif
#ifndef NT_REG_LO_NQ1
#define NT_REG_LO_NQ1 64  // NQ = 1 register split (56 / 64 / 72 -> softmax 200 / 192 / 184; 56 spills the issuer)
#endif
constexpr int kItemRing = 4;  // work-item slots handed from the producer to the MMA / softmax warps
constexpr float kRescaleLog2 = 8.0f;
// exp2 on the FMA pipe: 1 in POLY_EVERY pairs of P go through the degree-3
// polynomial (ex2_poly2) instead of MUFU.EX2 (0 = MUFU only), per head dim.
#ifndef NT_POLY_EVERY_D64
#define NT_POLY_EVERY_D64 8  // BERT 58.8 -> 57.5 us with the late PV wait (A/B, r02); D=128: 1/8 slower (446 -> 456 us)
#endif
#ifndef NT_POLY_EVERY_D128
#define NT_POLY_EVERY_D128 0
#endif
// P -> bf16 pack: 0 = cvt.rn.bf16x2.f32 (F2FP), 1 = integer add + byte permute
// (round half up, ALU pipe), 2 = byte permute only (truncation, ALU pipe) with
// the exponent pre-biased by log2(1 + E[rel. truncation error]) so P is
// unbiased on average and l divided by the same factor (kTruncScale).
#ifndef NT_PACK_D64
#define NT_PACK_D64 0
#endif
#ifndef NT_PACK_D128
#define NT_PACK_D128 0
#endif
// control warps (producer / MMA issuer) on the highest warp ids
#ifndef NT_K1_TWO_ISSUERS
#define NT_K1_TWO_ISSUERS 1
#endif
#ifndef NT_ROLES_HIGH
#define NT_ROLES_HIGH 0  // A/B r02: 8K 447 -> 453 us, 2K 49.4 -> 50.1, BERT 57.1 -> 56.5, 1-group 86.8 -> 85.9: off
#endif
// D=64 (SEP_P): wait for PV_t(j-1) after the exp pass instead of before it
// D=128: store P to TMEM after the whole exp pass instead of chunk by chunk
#ifndef NT_P_STORE_LATE
#define NT_P_STORE_LATE 0
#endif
#ifndef NT_SEP_P_LATE
#define NT_SEP_P_LATE 1
#endif
template <int D> constexpr int attn_poly_every() { return D == 64 ? NT_POLY_EVERY_D64 : NT_POLY_EVERY_D128; }
template <int D> constexpr int attn_pack_mode() { return D == 64 ? NT_PACK_D64 : NT_PACK_D128; }
// mean relative truncation error of a bf16 (7 stored mantissa bits) under
// Benford-distributed mantissas: 2^-8 * (1/ln 2) * (1 - 1/2) = 2.818e-3
constexpr float kTruncScale = 1.0028177f;
constexpr float kTruncLog2 = 0.0040601f;  // log2(kTruncScale)

// KV ring depth in 128-key K or V tiles.  The MA kernel's `stages` tunable
// (SetParam stages, tilecc/autosched/scheduler.py:116-124) picks it: stages = 1
// keeps one K/V tile pair (D=128) / two pairs (D=64) in flight, stages >= 2 the
// most shared memory allows (64 KB of K/V per stage).
template <int D, int NQ = 2>
constexpr int attn_kv_slots(int ma_stages) {
  if (NQ == 1) return (D == 128) ? 2 : (ma_stages <= 1 ? 2 : 4);  // half an SM's shared memory
  return (D == 128) ? (ma_stages <= 1 ? 2 : 4) : (ma_stages <= 1 ? 4 : 8);
}

template <int D, int KVS = attn_kv_slots<D>(2), bool OUT_F32 = false, bool FP8 = false, int NQ = 2,
          bool SPLIT = false>
struct AttnCfg {
  static constexpr int BM = 128, BN = 128;
  static constexpr int ROWS = 128 * NQ;          // query rows per work item
  static constexpr int THREADS = attn_threads<NQ>();
  static constexpr int TMEM_COLS = NQ == 2 ? 512 : 256;
  static constexpr int O_COL0 = 128 * NQ;        // TMEM column of O_0 (O_t at O_COL0 + 128 t)
  static constexpr int ESZ = FP8 ? 1 : 2;     // operand bytes (bf16 | e4m3)
  static constexpr int HALF = 128 * 128;      // one 128-row x 128-byte swizzle-128B panel
  static constexpr int PANELS = D * ESZ / 128;
  static constexpr int KSTEP = FP8 ? 32 : 16;  // K per tcgen05.mma (kind::f8f6f4 | kind::f16)
  static constexpr int TQ = BM * D * ESZ;
  static constexpr int TKV = BN * D * ESZ;
  static constexpr int STAGES = KVS;
  // D = 64: O_t needs only 64 TMEM columns, so P_t gets its own 64 columns
  // next to it instead of aliasing S_t.  S_t(j+1) can then be computed as soon
  // as the softmax warps have loaded S_t(j) into registers, i.e. while they
  // compute P_t(j), and the tile's GEMMs leave the softmax critical path.
  static constexpr bool SEP_P = (D == 64);
  // D = 64: Q is double-buffered across work items (the next item's Q lands
  // while the current one runs); D = 128 has no shared memory left for it
  static constexpr int QB = (D == 64 || FP8) ? 2 : 1;
  static constexpr int SMEM_Q = 0;
  static constexpr int SMEM_KV = NQ * QB * TQ;
  // epilogue staging: per softmax warp one 32-row x 32-column O box (TMA store),
  // 64B-swizzled (bf16) / 128B-swizzled (fp32) so the row-per-thread writes are
  // bank-conflict free
  // fp32 O / split-KV partial boxes: 32 columns (128-byte rows, SWIZZLE_128B) or,
  // NQ = 1 (two CTAs per SM, tight shared memory), 16 columns (64-byte rows,
  // SWIZZLE_64B); bf16 boxes are 32 columns of 64-byte rows
  static constexpr int F32_BOX_COLS = NQ == 1 ? 16 : 32;
  static constexpr int OBOX = (OUT_F32 && NQ == 2) ? 32 * 32 * 4 : 32 * 32 * 2;  // split partials are bf16
  static constexpr int SMEM_O = SMEM_KV + STAGES * TKV;
  static constexpr int SMEM_BAR = SMEM_O + 4 * NQ * OBOX;
  static constexpr int NBAR = 4 * QB + 2 * STAGES + 2 + 2 + 2 + 2 + 2 + 2 * kItemRing;
  static constexpr int SMEM_PREFIX = SMEM_BAR + NBAR * 8 + 16 + 4 * kItemRing;
  static constexpr int SMEM_BYTES = SMEM_PREFIX + (SPLIT ? 4 * (kMaxSplitMblocks + 1) : 0) + 1024;  // + alignment slack
  // two CTAs per SM (NQ = 1): 2 x (SMEM_BYTES + 1 KB reserved) <= 228 KB
  static constexpr bool FITS = NQ == 2 ? SMEM_BYTES <= 227 * 1024 : SMEM_BYTES <= (233472 - 2 * 1024) / 2;
};

__device__ __forceinline__ float f_ninf() { return __int_as_float(0xff800000); }

// O_t *= alpha in TMEM (one row per thread).
template <int D>
__device__ __forceinline__ void attn_rescale_o(uint32_t tO, float alpha) {
#pragma unroll
  for (int c = 0; c < D / 16; ++c) {
    uint32_t o[16];
    tmem_ld16(tO + c * 16, o);
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
    tmem_st16(tO + c * 16, o);
  }
}

// P = exp2(S*sc - m) for one 128-key row, packed into pk (bf16 pairs, or e4m3
// quads when FP8: 64 / 32 words) and, when STORE, written to TMEM at tP chunk by
// chunk; returns the row sum of P (fp32, before rounding).
template <bool FP8, bool STORE, int POLY = 0, int PACK = 0, bool EXACT_ZERO = true>
__device__ __forceinline__ float attn_exp_pass(const uint32_t (&s)[128], float sc, float m, uint32_t tP,
                                               uint32_t (&pk)[64]) {
  const float2 sc2 = make_float2(sc, sc);
  const float mb = (PACK == 2 && !FP8) ? -m + kTruncLog2 : -m;
  const float2 nm2 = make_float2(mb, mb);
  float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
    float2 prev = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float s0 = __uint_as_float(s[ch * 32 + 2 * i]), s1 = __uint_as_float(s[ch * 32 + 2 * i + 1]);
      const float2 x = ffma2(make_float2(s0, s1), sc2, nm2);
      float2 e;
      if (POLY > 0 && (i % POLY) == POLY - 1) {
        e = ex2_poly2<EXACT_ZERO>(x);  // FMA-pipe exp2 for 1/POLY of the pairs
      } else {
        e = make_float2(ex2(x.x), ex2(x.y));
      }
      sum2[i & 1] = fadd2(sum2[i & 1], e);
      if (FP8) {
        if (i & 1) pk[ch * 8 + (i >> 1)] = pack_e4m3x4(prev.x, prev.y, e.x, e.y);
        prev = e;
      } else {
        pk[ch * 16 + i] = PACK == 2 ? pack_bf16_trunc(e.x, e.y)
                          : PACK == 1 ? pack_bf16_alu(e.x, e.y) : pack_bf16(e.x, e.y);
      }
    }
    if (STORE) {
      if (!FP8) tmem_st16(tP + ch * 16, pk + ch * 16);
      else if (ch & 1) tmem_st16(tP + (ch >> 1) * 16, pk + (ch >> 1) * 16);  // 64 keys = 16 e4m3-quad columns
    }
  }
  return (sum2[0].x + sum2[0].y) + (sum2[1].x + sum2[1].y);
}

#ifdef NT_TRACE
// Debug timeline (NT_TRACE builds only): clock64 stamps of one CTA's pipeline
// for its first work item.  trace[(role * 64 + iter) * 8 + event]; role 0 MMA,
// 1/2 softmax tile 0/1, 3 producer.
__device__ unsigned long long* g_nt_trace = nullptr;
__device__ int g_nt_trace_cta = 0;
__device__ int g_nt_trace_li = 0;  // which of the CTA's work items the per-step stamps record
__device__ unsigned long long* g_nt_cta_times = nullptr;  // [cta][entry, exit, items] (globaltimer ns)
// The trace controls are read once into registers (nt_tr / nt_tr_li, see
// NT_TRACE_INIT) so a stamp costs a clock read and a store, not a global load.
#define NT_TRACE_INIT                                                                          \
  unsigned long long* const nt_tr = (g_nt_trace && blockIdx.x == g_nt_trace_cta) ? g_nt_trace : nullptr; \
  const int nt_tr_li = g_nt_trace_li
#define NT_TRACE_LI nt_tr_li
#define NT_STAMP(role, iter, ev)                                                               \
  do {                                                                                         \
    if (nt_tr && (iter) < 64) nt_tr[((role) * 64 + (iter)) * 8 + (ev)] = clock64();             \
  } while (0)
#else
#define NT_STAMP(role, iter, ev) do {} while (0)
#define NT_TRACE_LI 0
#define NT_TRACE_INIT do {} while (0)
#endif

// Work item -> coordinates.  Items are ordered heaviest first for causal masks
// (largest query block first: LPT over the strided CTA assignment).
struct AttnItem {
  int b, hq, hkv, q_row0, n_kv;
  int kv_lo;   // first KV tile of this work unit
  int unit;    // work-unit index (partial slot when split)
  bool split;  // the item is split over several units: write an fp32 partial
};

// KV tiles of m-block mb (causal: up to the diagonal of its last row)
template <int MASK, int ROWS = 256>
__device__ __forceinline__ int attn_mb_nkv(const AttnFwdParams& p, int mb) {
  int n_kv = p.n_kv_total;
  if (MASK == MASK_CAUSAL) {
    const int last_q = min(mb * ROWS + ROWS - 1, p.N - 1) + p.causal_offset;
    n_kv = max(min(n_kv, last_q / 128 + 1), 1);
  }
  return n_kv;
}

template <int MASK, int ROWS>
__device__ __forceinline__ AttnItem attn_item(const AttnFwdParams& p, int w) {
  const int BH = p.B * p.Hq;
  const int bh = w % BH;
  const int mbi = w / BH;
  const int mb = (MASK == MASK_CAUSAL) ? (p.n_mblocks - 1 - mbi) : mbi;
  AttnItem it;
  it.hq = bh % p.Hq;
  it.b = bh / p.Hq;
  it.hkv = it.hq / p.q_per_kv;
  it.q_row0 = mb * ROWS;
  it.n_kv = attn_mb_nkv<MASK, ROWS>(p, mb);
  it.kv_lo = 0;
  it.unit = w;
  it.split = false;
  return it;
}

// Work unit w: items in the same LPT order (heaviest m-blocks first); with
// kv_split, m-block position i holds ceil(n_kv / kv_split) x B x Hq units
// (chunk-major), located by a binary search of the prefix table.
template <int MASK, bool SPLIT, int ROWS = 256>
__device__ __forceinline__ AttnItem attn_unit(const AttnFwdParams& p, const int* prefix, int w) {
  if (!SPLIT) return attn_item<MASK, ROWS>(p, w);
  int lo = 0, hi = p.n_mblocks;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (prefix[mid] <= w) lo = mid;
    else hi = mid;
  }
  const int BH = p.B * p.Hq;
  const int r = w - prefix[lo];
  const int c = r / BH, bh = r - c * BH;
  const int mb = (MASK == MASK_CAUSAL) ? (p.n_mblocks - 1 - lo) : lo;
  const int n_full = attn_mb_nkv<MASK, ROWS>(p, mb);
  AttnItem it;
  it.hq = bh % p.Hq;
  it.b = bh / p.Hq;
  it.hkv = it.hq / p.q_per_kv;
  it.q_row0 = mb * ROWS;
  it.kv_lo = c * p.kv_split;
  it.n_kv = min(p.kv_split, n_full - it.kv_lo);
  it.unit = w;
  it.split = n_full > p.kv_split;
  return it;
}

template <int D, int MASK, bool OUT_F32, int KVS, bool FP8 = false, bool SPLIT = false, int NQ = 2>
__global__ void __launch_bounds__(attn_threads<NQ>(), NQ == 2 ? 1 : 2)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                    const __grid_constant__ CUtensorMap tmP, const AttnFwdParams p) {
  using C = AttnCfg<D, KVS, OUT_F32, FP8, NQ, SPLIT>;
  constexpr int ROWS = C::ROWS;
  constexpr int kPoly = FP8 ? 0 : attn_poly_every<D>();
  constexpr int kPack = FP8 ? 0 : attn_pack_mode<D>();
  // register split between warpgroup 0 (producer / MMA issuer) and the softmax
  // warpgroups: NQ = 2: 128 x lo + 256 x hi = 384 x 168; NQ = 1 (two CTAs per
  // SM): 128 x lo + 128 x hi = 256 x 128
  constexpr int kRegSplitLo = NQ == 1 ? NT_REG_LO_NQ1 : (D == 64) ? NT_REG_LO64 : 104;
  static_assert(C::FITS, "K1 shared memory exceeds the per-CTA budget");
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);

  uint8_t* sQ = smem + C::SMEM_Q;
  uint8_t* sKV = smem + C::SMEM_KV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::SMEM_BAR);
  uint64_t* bar_q = bars;                            // [QB][2] Q_t landed
  uint64_t* bar_q_empty = bars + 2 * C::QB;          // [QB][2] last S_t of the item done (Q_t reusable)
  uint64_t* bar_kv_full = bars + 4 * C::QB;          // [STAGES]
  uint64_t* bar_kv_empty = bar_kv_full + C::STAGES;  // [STAGES]
  uint64_t* bar_s_full = bar_kv_empty + C::STAGES;   // [2]
  uint64_t* bar_p_full = bar_s_full + 2;             // [2]
  uint64_t* bar_o_full = bar_p_full + 2;             // [2]
  uint64_t* bar_s_free = bar_o_full + 2;             // [2] SEP_P: S_t loaded into registers (4 warps)
  uint64_t* bar_pv_done = bar_s_free + 2;            // [2] SEP_P: PV_t completed (P_t / O_t reusable)
  uint64_t* bar_item_full = bar_pv_done + 2;         // [kItemRing] item index published
  uint64_t* bar_item_empty = bar_item_full + kItemRing;  // [kItemRing] read by MMA + 8 softmax warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);
  int* item_ring = reinterpret_cast<int*>(tmem_slot + 4);
  int* unit_prefix = reinterpret_cast<int*>(smem + C::SMEM_PREFIX);

  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const int lane = threadIdx.x & 31;
  if (SPLIT) asm volatile("griddepcontrol.launch_dependents;");  // the merge may be scheduled now
  // warp roles: the control warpgroup (TMA producer, MMA issuer, helpers) and the
  // softmax warpgroups.  The SMSP scheduler prefers the highest eligible warp id
  // (B300_MICROARCH.md), so the control warps get the HIGH ids (NT_ROLES_HIGH): the
  // MMA issuer is not starved by the softmax warps sharing its SMSP.
  constexpr int kCtl = NT_ROLES_HIGH ? 4 * NQ : 0;   // producer kCtl, MMA kCtl + 1, helper kCtl + 2
  constexpr int kSm0 = NT_ROLES_HIGH ? 0 : 4;        // first softmax warp
  // MMA-issuing warps: two only where S is computed ahead of the chain (SEP_P, D=64):
  // with P aliasing S (D=128) each tile's PV+S group sits in its chain, and two issuers
  // interleave the groups' MMAs so both finish later (8K 447 -> 550 us; BERT 56.8 -> 55.4)
  constexpr int kIssuers = (NQ == 2 && C::SEP_P && NT_K1_TWO_ISSUERS) ? 2 : 1;
  NT_TRACE_INIT;
  if (threadIdx.x == 0) NT_STAMP(3, 63, 7);  // kernel entry (trace builds)
#ifdef NT_TRACE
  if (threadIdx.x == 0 && g_nt_cta_times) g_nt_cta_times[blockIdx.x * 3] = globaltimer();
#endif

  if (warp == kCtl && lane == 0) {
    prefetch_tmap(&tmQ);
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    prefetch_tmap(&tmO);
    if (SPLIT) prefetch_tmap(&tmP);
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bar_s_full[t], 1);
      mbar_init(&bar_p_full[t], 4);
      mbar_init(&bar_o_full[t], 1);
      mbar_init(&bar_s_free[t], 4);
      mbar_init(&bar_pv_done[t], 1);
    }
    for (int q = 0; q < 2 * C::QB; ++q) {
      mbar_init(&bar_q[q], 1);
      mbar_init(&bar_q_empty[q], 1);
    }
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&bar_kv_full[s], 1);
      mbar_init(&bar_kv_empty[s], kIssuers);
    }
    for (int s = 0; s < kItemRing; ++s) {
      mbar_init(&bar_item_full[s], 1);
      mbar_init(&bar_item_empty[s], kIssuers + 4 * NQ);
    }
    fence_barrier_init();
  }
  if (warp == kCtl + 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  if (SPLIT && warp == kCtl + 2) {
    // split-KV unit prefix over m-block positions (warp scan, 32 positions per step)
    const int BH = p.B * p.Hq;
    int carry = 0;
    for (int base = 0; base < p.n_mblocks; base += 32) {
      const int i = base + lane;
      int cnt = 0;
      if (i < p.n_mblocks) {
        const int mb = (MASK == MASK_CAUSAL) ? (p.n_mblocks - 1 - i) : i;
        cnt = (attn_mb_nkv<MASK, ROWS>(p, mb) + p.kv_split - 1) / p.kv_split * BH;
      }
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, cnt, off);
        if (lane >= off) cnt += v;
      }
      if (i < p.n_mblocks) unit_prefix[i + 1] = carry + cnt;
      carry += __shfl_sync(0xffffffffu, cnt, 31);
    }
    if (lane == 0) unit_prefix[0] = 0;
    __syncwarp();
    if (blockIdx.x == 0)
      for (int i = lane; i <= p.n_mblocks; i += 32) p.unit_prefix[i] = unit_prefix[i];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= kCtl && warp < kCtl + 4) {
    // setmaxnreg only redistributes the launch allocation (384 x 168 = 64512
    // registers): 128 x 104 + 256 x 200 = 64512
    if constexpr (kRegSplitLo == 104) asm volatile("setmaxnreg.dec.sync.aligned.u32 104;");
    else if constexpr (kRegSplitLo == 96) asm volatile("setmaxnreg.dec.sync.aligned.u32 96;");
    else if constexpr (kRegSplitLo == 88) asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
    else if constexpr (kRegSplitLo == 72) asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
    else if constexpr (kRegSplitLo == 64) asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
    else asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (warp == kCtl) {
      // ================= TMA producer
      if (lane == 0) {
        int kv_base = 0;
        for (int li = 0;; ++li) {
          // ---- schedule: first item static, then greedy (LPT order) from the global counter
          const int slot_i = li % kItemRing;
          if (li < 15) NT_STAMP(3, 48 + li, 0);  // trace: producer reaches item li
          if (li >= kItemRing) mbar_wait(&bar_item_empty[slot_i], ((li / kItemRing) - 1) & 1, p.err, 12);
          int w;
          if (li == 0) w = blockIdx.x;
          else if (p.work) w = gridDim.x + atomicAdd(p.work, 1);
          else w = blockIdx.x + li * gridDim.x;
          item_ring[slot_i] = w;
          mbar_arrive(&bar_item_full[slot_i]);
          if (li < 15) NT_STAMP(3, 48 + li, 1);  // trace: item li published
          if (w >= p.n_items) {
#ifdef NT_TRACE
            if (g_nt_cta_times)  // units << 32 | KV steps this CTA ran
              g_nt_cta_times[blockIdx.x * 3 + 2] = ((unsigned long long)li << 32) | (unsigned)(kv_base >> 1);
#endif
            break;
          }
          const AttnItem itm = attn_unit<MASK, SPLIT, ROWS>(p, unit_prefix, w);
          // Q_t of this item may only land once the previous item's last S_t is
          // done; K(0) goes first, into the ring, so it is resident when Q is
          auto load_q = [&]() {
            const int qb = (li % C::QB) * NQ;
            for (int t = 0; t < NQ; ++t) {
              if (li >= C::QB) mbar_wait(&bar_q_empty[qb + t], ((li / C::QB) - 1) & 1, p.err, 11);
              mbar_arrive_expect_tx(&bar_q[qb + t], C::TQ);
#pragma unroll
              for (int h = 0; h < C::PANELS; ++h)
                tma_load_4d(sQ + (qb + t) * C::TQ + h * C::HALF, &tmQ, &bar_q[qb + t], h * 64, itm.q_row0 + t * 128,
                            itm.hq, itm.b);
            }
          };
          for (int it = 0; it < 2 * itm.n_kv; ++it) {
            if (it == 1) load_q();
            const int g = kv_base + it;
            const int slot = g % C::STAGES;
            const uint32_t ph = (g / C::STAGES) & 1;
            if (li == NT_TRACE_LI) NT_STAMP(3, it >> 1, (it & 1) * 2);
            mbar_wait(&bar_kv_empty[slot], ph ^ 1, p.err, 1);
            if (li == NT_TRACE_LI) NT_STAMP(3, it >> 1, (it & 1) * 2 + 1);
            mbar_arrive_expect_tx(&bar_kv_full[slot], C::TKV);
            const CUtensorMap* m = (it & 1) ? &tmV : &tmK;
            const int row = (itm.kv_lo + (it >> 1)) * 128;
#pragma unroll
            for (int h = 0; h < C::PANELS; ++h)
              tma_load_4d(sKV + slot * C::TKV + h * C::HALF, m, &bar_kv_full[slot], h * 64, row, itm.hkv, itm.b);
          }
          if (itm.n_kv == 0) load_q();
          kv_base += 2 * itm.n_kv;
        }
      }
    } else if (warp == kCtl + 1 || (kIssuers == 2 && warp == kCtl + 3)) {
      // ================= MMA issuer(s).  An issuing thread blocks on each MMA until the
      // tensor pipe takes it and spends ~100 clk per mbarrier wait and ~60 per commit
      // (tools/trace_decode.py, tools/ubench/umma_rate.cu); with kIssuers = 2 each
      // query tile has its own issuer (warp kCtl + 1: tile 0, kCtl + 3: tile 1), so one
      // tile's waits and commits overlap the other tile's MMAs.  The tiles only share
      // K/V ring slots (released by both issuers' commits) and the item ring.
      const int t_lo = (kIssuers == 2 && warp == kCtl + 3) ? 1 : 0;
      const int t_hi = kIssuers == 2 ? t_lo + 1 : NQ;
      if (lane == 0) {
        constexpr uint32_t idS = FP8 ? idesc_e4m3(128, 128, 0, 0) : idesc_bf16(128, 128, 0, 0);
        constexpr uint32_t idO = FP8 ? idesc_e4m3(128, D, 0, 1) : idesc_bf16(128, D, 0, 1);
        const uint32_t sQa = smem_u32(sQ), sKVa = smem_u32(sKV);
        int qb = 0;  // Q buffer pair of the current item
        auto issue_s = [&](int t, int slot) {
#pragma unroll
          for (int k = 0; k < D / C::KSTEP; ++k) {
            // 32 bytes of K per instruction, 4 per 128-byte panel row
            const uint32_t off = (k >> 2) * C::HALF + (k & 3) * 32;
            const uint64_t a = sdesc_sw128(sQa + (qb + t) * C::TQ + off, 16, 1024);
            const uint64_t bd = sdesc_sw128(sKVa + slot * C::TKV + off, 16, 1024);
            if (FP8) umma_ss_f8(tmem + t * 128, a, bd, idS, k > 0 ? 1u : 0u);
            else umma_ss(tmem + t * 128, a, bd, idS, k > 0 ? 1u : 0u);
          }
        };
        auto issue_pv = [&](int t, int slot, bool acc) {
#pragma unroll
          for (int k = 0; k < 128 / C::KSTEP; ++k) {
            // KSTEP keys of V (MN-major, 128-byte rows) x P's 8 TMEM columns
            const uint64_t bd = sdesc_sw128(sKVa + slot * C::TKV + k * C::KSTEP * 128, C::HALF, 1024);
            const uint32_t pcol = C::SEP_P ? (C::O_COL0 + t * 128 + 64) : (t * 128);
            if (FP8) umma_ts_f8(tmem + C::O_COL0 + t * 128, tmem + pcol + k * 8, bd, idO, (acc || k > 0) ? 1u : 0u);
            else umma_ts(tmem + C::O_COL0 + t * 128, tmem + pcol + k * 8, bd, idO, (acc || k > 0) ? 1u : 0u);
          }
        };
        // The issue stream runs across work items: the next item's first score
        // GEMMs S_t(0) are issued inside the current item's tail (as soon as S_t's
        // TMEM is free), so the softmax warps find them ready after the epilogue.
        auto fetch = [&](int li) -> int {  // item index of the CTA's li-th item, -1 at the end
          const int slot_i = li % kItemRing;
          mbar_wait(&bar_item_full[slot_i], (li / kItemRing) & 1, p.err, 13);
          const int w = item_ring[slot_i];
          mbar_arrive(&bar_item_empty[slot_i]);
          return w < p.n_items ? w : -1;
        };
        auto wait_q = [&](int li) {
          qb = (li % C::QB) * NQ;
          for (int t = t_lo; t < t_hi; ++t) mbar_wait(&bar_q[qb + t], (li / C::QB) & 1, p.err, 2);
          if (li < 15) NT_STAMP(3, 48 + li, 3);  // trace: MMA has Q of item li
        };
        // S_t(0) of an item from its K(0) at ring index g (both tiles)
        auto first_s = [&](int g, int n_kv) {
          const int slotK = g % C::STAGES;
          mbar_wait(&bar_kv_full[slotK], (g / C::STAGES) & 1, p.err, 3);
          tc_fence_after();
          for (int t = t_lo; t < t_hi; ++t) {
            issue_s(t, slotK);
            umma_commit(&bar_s_full[t]);
            if (n_kv == 1) umma_commit(&bar_q_empty[qb + t]);
          }
          umma_commit(&bar_kv_empty[slotK]);
        };
        int kv_base = 0;
        uint32_t p_phase[2] = {0u, 0u};
        uint32_t sf_phase[2] = {0u, 0u};
        int w = fetch(0);
        int n_kv = w >= 0 ? attn_unit<MASK, SPLIT, ROWS>(p, unit_prefix, w).n_kv : 0;
        if (w >= 0) {
          wait_q(0);
          first_s(0, n_kv);
        }
        for (int li = 0; w >= 0; ++li) {
          // ---- steps j = 1 .. n_kv-1: S_t(j) and PV_t(j-1)
          for (int j = 1; j < n_kv; ++j) {
            const int gK = kv_base + 2 * j;
            const int slotK = gK % C::STAGES;
            const int gV = gK - 1;  // V(j-1)
            const int slotV = gV % C::STAGES;
            if (li == NT_TRACE_LI) NT_STAMP(0, j, 0);
            mbar_wait(&bar_kv_full[slotK], (gK / C::STAGES) & 1, p.err, 3);
            if (li == NT_TRACE_LI) NT_STAMP(0, j, 1);
            tc_fence_after();
            if constexpr (C::SEP_P) {
              // S_t(j) waits only until the softmax warps have read S_t(j-1) out of TMEM
              for (int t = t_lo; t < t_hi; ++t) {
                mbar_wait(&bar_s_free[t], sf_phase[t], p.err, 15);
                sf_phase[t] ^= 1u;
                tc_fence_after();
                if (li == NT_TRACE_LI) NT_STAMP(0, j, 2 + t);
                issue_s(t, slotK);
                umma_commit(&bar_s_full[t]);
                if (j == n_kv - 1) umma_commit(&bar_q_empty[qb + t]);
              }
              umma_commit(&bar_kv_empty[slotK]);
              for (int t = t_lo; t < t_hi; ++t) {
                mbar_wait(&bar_p_full[t], p_phase[t], p.err, 4);
                p_phase[t] ^= 1u;
                if (t == t_lo) mbar_wait(&bar_kv_full[slotV], (gV / C::STAGES) & 1, p.err, 5);
                tc_fence_after();
                if (li == NT_TRACE_LI) NT_STAMP(0, j, 4 + t);
                issue_pv(t, slotV, j - 1 > 0);
                umma_commit(&bar_pv_done[t]);
              }
              umma_commit(&bar_kv_empty[slotV]);
            } else {
              // P_t(j-1) aliases S_t: PV_t(j-1) then S_t(j), tile 0 then tile 1
              for (int t = t_lo; t < t_hi; ++t) {
                mbar_wait(&bar_p_full[t], p_phase[t], p.err, 4);
                p_phase[t] ^= 1u;
                if (li == NT_TRACE_LI) NT_STAMP(0, j, 2 + 2 * t);
                if (t == t_lo) mbar_wait(&bar_kv_full[slotV], (gV / C::STAGES) & 1, p.err, 5);
                tc_fence_after();
                issue_pv(t, slotV, j - 1 > 0);
                if (t == t_hi - 1) umma_commit(&bar_kv_empty[slotV]);
                issue_s(t, slotK);
                umma_commit(&bar_s_full[t]);
                if (j == n_kv - 1) umma_commit(&bar_q_empty[qb + t]);
                if (li == NT_TRACE_LI) NT_STAMP(0, j, 3 + 2 * t);
              }
              umma_commit(&bar_kv_empty[slotK]);
            }
          }
          // ---- tail: PV_t(n_kv-1) -> O complete, interleaved with the next item's S_t(0)
          const int wn = fetch(li + 1);
          const int n_next = wn >= 0 ? attn_unit<MASK, SPLIT, ROWS>(p, unit_prefix, wn).n_kv : 0;
          const int gV = kv_base + 2 * n_kv - 1;
          const int slotV = gV % C::STAGES;
          const int gKn = kv_base + 2 * n_kv;  // ring index of the next item's K(0)
          if constexpr (C::SEP_P) {
            for (int t = t_lo; t < t_hi; ++t) {
              mbar_wait(&bar_s_free[t], sf_phase[t], p.err, 16);
              sf_phase[t] ^= 1u;
            }
            if (wn >= 0) {
              wait_q(li + 1);
              first_s(gKn, n_next);
            }
            for (int t = t_lo; t < t_hi; ++t) {
              mbar_wait(&bar_p_full[t], p_phase[t], p.err, 6);
              p_phase[t] ^= 1u;
              if (t == t_lo) mbar_wait(&bar_kv_full[slotV], (gV / C::STAGES) & 1, p.err, 7);
              tc_fence_after();
              issue_pv(t, slotV, n_kv - 1 > 0);
              umma_commit(&bar_pv_done[t]);
              umma_commit(&bar_o_full[t]);
            }
            umma_commit(&bar_kv_empty[slotV]);
          } else {
            const int slotKn = gKn % C::STAGES;
            for (int t = t_lo; t < t_hi; ++t) {
              mbar_wait(&bar_p_full[t], p_phase[t], p.err, 6);
              p_phase[t] ^= 1u;
              if (t == t_lo) mbar_wait(&bar_kv_full[slotV], (gV / C::STAGES) & 1, p.err, 7);
              tc_fence_after();
              issue_pv(t, slotV, n_kv - 1 > 0);
              umma_commit(&bar_o_full[t]);
              if (wn >= 0) {
                if (t == t_lo) {
                  wait_q(li + 1);
                  mbar_wait(&bar_kv_full[slotKn], (gKn / C::STAGES) & 1, p.err, 3);
                  tc_fence_after();
                }
                issue_s(t, slotKn);
                umma_commit(&bar_s_full[t]);
                if (n_next == 1) umma_commit(&bar_q_empty[qb + t]);
              }
            }
            umma_commit(&bar_kv_empty[slotV]);
            if (wn >= 0) umma_commit(&bar_kv_empty[slotKn]);
          }
          kv_base = gKn;
          w = wn;
          n_kv = n_next;
        }
      }
    }
  } else {
    if constexpr (NQ == 1) {
      if constexpr (kRegSplitLo == 72) asm volatile("setmaxnreg.inc.sync.aligned.u32 184;");
      else if constexpr (kRegSplitLo == 64) asm volatile("setmaxnreg.inc.sync.aligned.u32 192;");
      else asm volatile("setmaxnreg.inc.sync.aligned.u32 200;");
    } else if constexpr (kRegSplitLo == 104) asm volatile("setmaxnreg.inc.sync.aligned.u32 200;");
    else if constexpr (kRegSplitLo == 96) asm volatile("setmaxnreg.inc.sync.aligned.u32 204;");
    else asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
    // ================= softmax (+ lazy O correction + epilogue), one thread per query row
    const int t = (warp - kSm0) / 4;
    const int wq = warp & 3;  // TMEM sub-partition this warp may access
    const int r = wq * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t tS = tmem + t * 128 + lane_off;
    const uint32_t tO = tmem + C::O_COL0 + t * 128 + lane_off;
    const uint32_t tP = C::SEP_P ? (tO + 64) : tS;  // where P_t (bf16 pairs) is stored
    const float NINF = f_ninf();
    const float sc = (MASK == MASK_TENSOR) ? 1.0f : p.scale_log2;
    uint32_t s_phase = 0u;
    int pv_base = 0;  // SEP_P: PV_t completions of earlier items
    // deferred epilogue of the previous item (O_t still in TMEM)
    bool pend = false;
    int pend_li = 0, pend_row0 = 0, pend_hq = 0, pend_b = 0;
    float pend_inv = 0.f;
    bool pend_part = false;  // split-KV unit: O / l_unit goes to the bf16 partial map (row pend_row0)
    auto store_o = [&]() {
      // O / l from TMEM -> swizzled smem box (one row per lane) -> TMA store of
      // 32 rows x 32 columns per warp (rows past N are clipped)
      if (t == 0 && wq == 0 && lane == 0 && pend_li < 16) NT_STAMP(3, 32 + pend_li, 2);  // store_o entry (trace)
      mbar_wait(&bar_o_full[t], pend_li & 1, p.err, 9);
      if (t == 0 && wq == 0 && lane == 0 && pend_li < 15) NT_STAMP(3, 48 + pend_li, 6);  // trace: O complete
      tc_fence_after();
      const float inv = pend_inv;
      uint8_t* stg = smem + C::SMEM_O + (warp - kSm0) * C::OBOX;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + c * 32, o);
        tmem_wait_ld();
        const bool f32box = OUT_F32 && !(SPLIT && pend_part);
        if (C::F32_BOX_COLS == 16 && f32box) {
          // two 16-column fp32 boxes: 64-byte rows, chunk q at q ^ ((row >> 1) & 3) (SWIZZLE_64B)
#pragma unroll
          for (int hbox = 0; hbox < 2; ++hbox) {
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int e = hbox * 16 + 4 * q;
              const uint4 v = make_uint4(__float_as_uint(__uint_as_float(o[e]) * inv),
                                         __float_as_uint(__uint_as_float(o[e + 1]) * inv),
                                         __float_as_uint(__uint_as_float(o[e + 2]) * inv),
                                         __float_as_uint(__uint_as_float(o[e + 3]) * inv));
              *reinterpret_cast<uint4*>(stg + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) = v;
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (SPLIT && pend_part) tma_store_2d(&tmP, stg, c * 32 + hbox * 16, pend_row0);
              else tma_store_4d(&tmO, stg, c * 32 + hbox * 16, pend_row0, pend_hq, pend_b);
              bulk_commit();
            }
          }
          continue;
        }
        if (lane == 0) bulk_wait_read0();  // this warp's previous box has left shared memory
        __syncwarp();
        if (f32box) {
          // 128-byte rows, 16-byte chunk q at q ^ (row & 7) (SWIZZLE_128B)
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint4 v = make_uint4(__float_as_uint(__uint_as_float(o[4 * q]) * inv),
                                       __float_as_uint(__uint_as_float(o[4 * q + 1]) * inv),
                                       __float_as_uint(__uint_as_float(o[4 * q + 2]) * inv),
                                       __float_as_uint(__uint_as_float(o[4 * q + 3]) * inv));
            *reinterpret_cast<uint4*>(stg + lane * 128 + ((q ^ (lane & 7)) << 4)) = v;
          }
        } else {
          // 64-byte rows, 16-byte chunk q at q ^ ((row >> 1) & 3) (SWIZZLE_64B)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 v = make_uint4(pack_bf16(__uint_as_float(o[8 * q]) * inv, __uint_as_float(o[8 * q + 1]) * inv),
                                       pack_bf16(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv),
                                       pack_bf16(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv),
                                       pack_bf16(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv));
            *reinterpret_cast<uint4*>(stg + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) = v;
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (SPLIT && pend_part) tma_store_2d(&tmP, stg, c * 32, pend_row0);
          else tma_store_4d(&tmO, stg, c * 32, pend_row0, pend_hq, pend_b);
          bulk_commit();
        }
      }
      // O_t is read out: the next PV_t (after this warp's next p_full arrival) may overwrite it
      tc_fence_before();
      if (t == 0 && wq == 0 && lane == 0 && pend_li < 16) NT_STAMP(3, 32 + pend_li, 7);  // item end (trace)
    };
    for (int li = 0;; ++li) {
      const int slot_i = li % kItemRing;
      if (t == 0 && wq == 0 && lane == 0 && li < 15) NT_STAMP(3, 48 + li, 4);  // trace: softmax asks for item li
      mbar_wait(&bar_item_full[slot_i], (li / kItemRing) & 1, p.err, 14);
      if (t == 0 && wq == 0 && lane == 0 && li < 15) NT_STAMP(3, 48 + li, 5);
      const int w = item_ring[slot_i];
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_item_empty[slot_i]);
      if (w >= p.n_items) break;
      const AttnItem itm = attn_unit<MASK, SPLIT, ROWS>(p, unit_prefix, w);
      const int qi = itm.q_row0 + t * 128 + r;
      float m_run = NINF, l_run = 0.f;
      if (t == 0 && wq == 0 && lane == 0 && li < 16) NT_STAMP(3, 32 + li, 6);  // item start (trace)

      for (int j = 0; j < itm.n_kv; ++j) {
        if (li == NT_TRACE_LI && lane == 0 && wq == 0) NT_STAMP(1 + t, j, 0);
        mbar_wait(&bar_s_full[t], s_phase, p.err, 8);
        s_phase ^= 1u;
        if (li == NT_TRACE_LI && lane == 0 && wq == 0) NT_STAMP(1 + t, j, 1);
        tc_fence_after();
        uint32_t s[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, s + c * 32);
        tmem_wait_ld();
        if constexpr (C::SEP_P) {  // S_t is in registers: let S_t(j+1) overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_s_free[t]);
        }
        if (li == NT_TRACE_LI && lane == 0 && wq == 0) NT_STAMP(1 + t, j, 2);
        const int kv0 = (itm.kv_lo + j) * 128;
        if (MASK == MASK_TENSOR) {
          const float* mrow = p.mask + (long long)min(qi, p.N - 1) * p.mask_row_stride;
          if (kv0 + 128 <= p.M && (reinterpret_cast<uintptr_t>(mrow) & 15) == 0) {
            // a full tile of a 16-byte aligned row: 32 float4 loads instead of 128 scalar ones
            const float4* m4 = reinterpret_cast<const float4*>(mrow + kv0);
#pragma unroll
            for (int c4 = 0; c4 < 32; ++c4) {
              const float4 mk = __ldg(m4 + c4);
              const float mv[4] = {mk.x, mk.y, mk.z, mk.w};
#pragma unroll
              for (int e = 0; e < 4; ++e)
                s[4 * c4 + e] = __float_as_uint(
                    fmaf(__uint_as_float(s[4 * c4 + e]), p.scale_log2, mv[e] * 1.4426950408889634f));
            }
          } else {
#pragma unroll
            for (int c = 0; c < 128; ++c) {
              const int kv = kv0 + c;
              const float mk = (kv < p.M) ? __ldg(mrow + kv) : NINF;
              s[c] = __float_as_uint(fmaf(__uint_as_float(s[c]), p.scale_log2, mk * 1.4426950408889634f));
            }
          }
        } else if (MASK == MASK_BITS) {
          // 128 visibility bits of this row's KV tile in one 16-byte load (bits past M are 0)
          const uint4 w = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(p.mask) +
                                                             (long long)min(qi, p.N - 1) * p.mask_row_stride +
                                                             (kv0 >> 5)));
          if ((w.x & w.y & w.z & w.w) != 0xffffffffu) {
            const uint32_t wd[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int c = 0; c < 128; ++c)
              if (!((wd[c >> 5] >> (c & 31)) & 1u)) s[c] = __float_as_uint(NINF);
          }
        } else {
          const int lim = (MASK == MASK_CAUSAL) ? min(qi + p.causal_offset, p.M - 1) : (p.M - 1);
          if (kv0 + 127 > lim) {
#pragma unroll
            for (int c = 0; c < 128; ++c)
              if (kv0 + c > lim) s[c] = __float_as_uint(NINF);
          }
        }
        float mx;
        {
          // tree max with 3-input FMNMX3, 4 independent chains over s[0..128)
          float a0 = __uint_as_float(s[0]), a1 = __uint_as_float(s[1]);
          float a2 = __uint_as_float(s[2]), a3 = __uint_as_float(s[3]);
#pragma unroll
          for (int c = 4; c + 8 <= 128; c += 8) {
            a0 = fmax3(a0, __uint_as_float(s[c]), __uint_as_float(s[c + 1]));
            a1 = fmax3(a1, __uint_as_float(s[c + 2]), __uint_as_float(s[c + 3]));
            a2 = fmax3(a2, __uint_as_float(s[c + 4]), __uint_as_float(s[c + 5]));
            a3 = fmax3(a3, __uint_as_float(s[c + 6]), __uint_as_float(s[c + 7]));
          }
          a0 = fmax3(a0, __uint_as_float(s[124]), __uint_as_float(s[125]));
          a1 = fmax3(a1, __uint_as_float(s[126]), __uint_as_float(s[127]));
          mx = fmaxf(fmax3(a0, a1, a2), a3);
        }
        if (li == NT_TRACE_LI && lane == 0 && wq == 0) NT_STAMP(1 + t, j, 3);
        constexpr bool kLate = C::SEP_P && NT_SEP_P_LATE;
        if (C::SEP_P && !kLate && j > 0) {
          // PV_t(j-1) must be complete before O_t is rescaled or P_t overwritten;
          // completions up to j-2 were waited for at j-1, so the parity is exact
          mbar_wait(&bar_pv_done[t], (pv_base + j - 1) & 1, p.err, 10);
          tc_fence_after();
        }
        const float m_new = fmaxf(m_run, mx * sc);
        const bool need = m_new > m_run + kRescaleLog2;
        float alpha = 1.0f;
        const bool rescale = __any_sync(0xffffffffu, need);
        if (rescale) {
          alpha = (m_new == NINF) ? 1.0f : ex2(m_run - m_new);
          if (!kLate && j > 0) attn_rescale_o<D>(tO, alpha);
          l_run *= alpha;
          m_run = m_new;
        }
        const float m_use = (m_run == NINF) ? 0.f : m_run;
        uint32_t pk[64];
        float sum;
        if (kLate) {
          // SEP_P (D=64): P_t(j) overwrites P_t(j-1) and O_t is rescaled only after
          // PV_t(j-1) completed -- wait for that AFTER the exps (into registers), so
          // the PV latency hides behind them instead of stalling the exp phase
          sum = attn_exp_pass<FP8, false, kPoly, kPack, MASK != MASK_NONE>(s, sc, m_use, tP, pk);
          if (j == 0 && pend) {
            store_o();  // the previous item's O (its last PV waited inside)
            pend = false;
          } else if (j > 0) {
            mbar_wait(&bar_pv_done[t], (pv_base + j - 1) & 1, p.err, 10);
            tc_fence_after();
            if (rescale) attn_rescale_o<D>(tO, alpha);
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) tmem_st16(tP + c * 16, pk + c * 16);
        } else if (j == 0 && pend) {
          // first tile of an item while the previous item's O is still in TMEM:
          // exps into registers, then that epilogue (its last PV has had the S load,
          // max and exps to finish), then P -- PV(0) may overwrite O only after it
          sum = attn_exp_pass<FP8, false, kPoly, kPack, MASK != MASK_NONE>(s, sc, m_use, tP, pk);
          store_o();
          pend = false;
          if (!FP8) {
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_st16(tP + c * 16, pk + c * 16);
          } else {
            tmem_st16(tP, pk);
            tmem_st16(tP + 16, pk + 16);
          }
        } else if (!FP8 && NT_P_STORE_LATE) {
          // all exps into registers, then the four P stores back to back
          sum = attn_exp_pass<FP8, false, kPoly, kPack, MASK != MASK_NONE>(s, sc, m_use, tP, pk);
#pragma unroll
          for (int c = 0; c < 4; ++c) tmem_st16(tP + c * 16, pk + c * 16);
        } else {
          sum = attn_exp_pass<FP8, true, kPoly, kPack, MASK != MASK_NONE>(s, sc, m_use, tP, pk);
        }
        if (li == NT_TRACE_LI && lane == 0 && wq == 0) NT_STAMP(1 + t, j, 4);
        l_run += sum;
        tmem_wait_st();
        if (li == NT_TRACE_LI && lane == 0 && wq == 0) NT_STAMP(1 + t, j, 5);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_p_full[t]);
      }

      if (t == 0 && wq == 0 && lane == 0 && li < 16) NT_STAMP(3, 32 + li, 0);  // last tile done (trace)
      pv_base += itm.n_kv;
      if (kPack == 2) l_run *= 1.0f / kTruncScale;  // P was pre-biased by kTruncScale before truncation

      // ---- epilogue.  D=64 (short items): deferred into the next item's first
      // tile, where it overlaps the last PV's latency with that tile's S load, max
      // and exps (BERT 60.3 -> 58.5 us).  D=128: right here -- inside the next
      // tile it would delay P(0) and the chain behind it (8K 450 -> 461 us).
      const bool valid = qi < p.N;
      pend = true;
      pend_li = li;
      pend_part = SPLIT && itm.split;
      if (SPLIT && itm.split) {
        // partial of a split item: (m, l) per row now, O / l as bf16 (store_o) -- half
        // the bytes of an unnormalised fp32 partial (1-group 8K: 128 KB -> 64 KB per
        // unit); a KV range can legitimately miss a causal row (l = 0): the combine checks
        p.part_ml[(long long)itm.unit * ROWS + t * 128 + r] = make_float2(m_run, l_run);
        pend_inv = (l_run > 0.f) ? 1.0f / l_run : 0.f;
        pend_row0 = itm.unit * ROWS + t * 128 + wq * 32;
      } else {
        if (valid && !(l_run > 0.f) && p.err) atomicOr(p.err, 1);
        pend_inv = (l_run > 0.f) ? p.o_scale / l_run : 0.f;
        pend_row0 = itm.q_row0 + t * 128 + wq * 32;
      }
      pend_hq = itm.hq;
      pend_b = itm.b;
      if (t == 0 && wq == 0 && lane == 0 && li < 16) NT_STAMP(3, 32 + li, 1);  // epilogue prepared (trace)
      if (!C::SEP_P) {
        store_o();
        pend = false;
      }
    }
    if (pend) store_o();
    if (lane == 0) bulk_wait0();  // the last O boxes are written before the CTA exits
  }

  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == kCtl + 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
#ifdef NT_TRACE
  if (threadIdx.x == 0 && g_nt_cta_times) g_nt_cta_times[blockIdx.x * 3 + 1] = globaltimer();
#endif
  if (threadIdx.x == 0 && p.work) {
    // every CTA has drawn its terminal item before arriving here: the last one
    // resets the counter for the next launch on this stream
    __threadfence();
    if (atomicAdd(p.work + 1, 1) == (int)gridDim.x - 1) {
      atomicExch(p.work, 0);
      atomicExch(p.work + 1, 0);
    }
  }
}

// Split-KV merge: O[row] = o_scale * sum_c w_c O_c[row] / sum_c w_c l_c with
// w_c = exp2(m_c - max m) (the repair law, tilecc/schedule/repair.py:80-88).
// Block = 32 rows of one (split m-block position, batch x head): 8 warps x 4 rows,
// D/32 columns per lane; the grid covers only the split positions (the heaviest
// m-blocks in LPT order), and each warp issues all its rows' partial loads
// before the FMAs.
constexpr int kCombineRowsPerWarp = 4;
template <int D, int MASK, bool OUT_F32, int ROWS = 256>
__global__ void __launch_bounds__(256) attn_combine_kernel(const __nv_bfloat16* __restrict__ part_o,
                                                           const AttnFwdParams p) {
  // launched as a programmatic dependent of K1: wait for its completion and memory
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int mbi = blockIdx.z, bh = blockIdx.y;
  const int mb = (MASK == MASK_CAUSAL) ? (p.n_mblocks - 1 - mbi) : mbi;
  const int n_full = attn_mb_nkv<MASK, ROWS>(p, mb);
  const int nc = (n_full + p.kv_split - 1) / p.kv_split;
  if (nc <= 1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int BH = p.B * p.Hq;
  const int u0 = p.unit_prefix[mbi] + bh;
  constexpr int CPL = D / 32;  // columns per lane (4 bf16 = 8 bytes at D=128)
  const long long cstride = (long long)BH * ROWS * D;
  const int b = bh / p.Hq, hq = bh % p.Hq;
  auto load = [&](const __nv_bfloat16* src, float (&v)[CPL]) {
    if constexpr (CPL == 4) {
      const uint2 x = __ldg(reinterpret_cast<const uint2*>(src));
      v[0] = __uint_as_float(x.x << 16); v[1] = __uint_as_float(x.x & 0xffff0000u);
      v[2] = __uint_as_float(x.y << 16); v[3] = __uint_as_float(x.y & 0xffff0000u);
    } else {
      const uint32_t x = __ldg(reinterpret_cast<const uint32_t*>(src));
      v[0] = __uint_as_float(x << 16); v[1] = __uint_as_float(x & 0xffff0000u);
    }
  };
#pragma unroll 1
  for (int rr = 0; rr < kCombineRowsPerWarp; ++rr) {
    const int row = blockIdx.x * (8 * kCombineRowsPerWarp) + warp * kCombineRowsPerWarp + rr;  // within the m-block
    const int qr = mb * ROWS + row;
    if (qr >= p.N) break;
    // (m, l) of every chunk in one round trip: lane c holds chunk c (nc <= 32 by construction)
    float mc = f_ninf(), lc = 0.f;
    if (lane < nc) {
      const float2 ml = p.part_ml[(long long)(u0 + lane * BH) * ROWS + row];
      mc = ml.x;
      lc = ml.y;
    }
    const __nv_bfloat16* base = part_o + ((long long)u0 * ROWS + row) * D + lane * CPL;
    float v0[4][CPL];  // the first chunks' rows load while the (m, l) reduction runs
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < nc) load(base + k * cstride, v0[k]);
    float m = mc;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    // chunk weight w_c l_c: the partials are O_c / l_c
    const float wgt = (lane < nc && mc != f_ninf()) ? ex2(mc - m) * lc : 0.f;
    float lsum = wgt;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, off);
    float acc[CPL];
#pragma unroll
    for (int i = 0; i < CPL; ++i) acc[i] = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float w = __shfl_sync(0xffffffffu, wgt, k);
      if (k < nc) {
#pragma unroll
        for (int i = 0; i < CPL; ++i) acc[i] += w * v0[k][i];
      }
    }
    for (int c0 = 4; c0 < nc; c0 += 4) {
      float v[4][CPL];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (c0 + k < nc) load(base + (c0 + k) * cstride, v[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float w = __shfl_sync(0xffffffffu, wgt, (c0 + k) & 31);
        if (c0 + k < nc) {
#pragma unroll
          for (int i = 0; i < CPL; ++i) acc[i] += w * v[k][i];
        }
      }
    }
    if (!(lsum > 0.f)) {
      if (lane == 0 && p.err) atomicOr(p.err, 1);
      lsum = 0.f;
    }
    const float inv = (lsum > 0.f) ? p.o_scale / lsum : 0.f;
    const long long off = (long long)b * p.o_sb + (long long)hq * p.o_sh + (long long)qr * p.o_sn + lane * CPL;
    if (OUT_F32) {
      float* dst = static_cast<float*>(p.o) + off;
#pragma unroll
      for (int i = 0; i < CPL; i += 2) *reinterpret_cast<float2*>(dst + i) = make_float2(acc[i] * inv, acc[i + 1] * inv);
    } else {
      __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.o) + off;
#pragma unroll
      for (int i = 0; i < CPL; i += 2) *reinterpret_cast<uint32_t*>(dst + i) = pack_bf16(acc[i] * inv, acc[i + 1] * inv);
    }
  }
}

}  // namespace nt
