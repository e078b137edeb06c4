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
// CTA = one 128-row query tile (128/t0_i consecutive MA blocks) walking
// 128-row K/V tiles (128/t0_j consecutive MA j0 iterations; the rolling-update
// law makes the coarsening exact up to rounding), ascending like the MA.
//
//   warp 0      TMA producer: Q once, then K0,V0,K1,V1,... into a STAGES ring
//   warp 1      MMA issuer (one thread): S(j+1) = Q K_{j+1}^T (SS) is issued
//               BEFORE O += P(j) V_j (TS, P from TMEM), so the tensor core
//               computes the next scores while the softmax works on P(j)
//   warps 2-3   idle (warpgroup 0 donates registers via setmaxnreg)
//   warps 4-11  softmax: warpgroup h = 0/1 owns key columns [64h, 64h+64) of
//               every row (thread = query row = TMEM lane); the two half-row
//               maxima meet in shared memory once per KV tile
// TMEM (512 cols): S[0] [0,128), S[1] [128,256) double-buffered scores,
// O [256, 256+D); P(j) (bf16, 64 cols) is written back over S[j&1].
//
// Numerics: bf16 operands, fp32 accumulation, P rounded to bf16 before P.V.
// The scale c is folded into the exp2 constant (c*log2e), which differs from
// the MA's K_s*c only in rounding.  The running max is updated lazily: a warp
// only moves its rows' max (and rescales O, l) when some row's max grew by more
// than kRescaleLog2 (values of P stay <= 2^8); the final O/l is the same
// quantity, so this is an exact identity up to rounding.  Rows whose max is
// still -inf use 0 in place of the max (the FA -inf guard the MA lacks,
// SURVEY.md B.14).
#pragma once
#include "sm100.cuh"

namespace nt {

enum { MASK_NONE = 0, MASK_CAUSAL = 1, MASK_TENSOR = 2 };

struct AttnFwdParams {
  int B, Hq, Hkv, N, M;
  int q_per_kv;
  int n_mblocks;      // ceil(N / 128)
  int n_kv_total;     // ceil(M / 128)
  int causal_offset;  // key j visible to query i iff j <= i + causal_offset
  float scale_log2;   // c * log2(e)
  const float* mask;  // MASK_TENSOR: fp32 [N, M]
  long long mask_row_stride;
  float* o_f32;  // fp32 output (OUT_F32), element strides below
  long long o_sb, o_sh, o_sn;
  int* err;  // bit 0: zero denominator (fully masked row); 0x100|k: pipeline timeout
};

constexpr int kAttnThreads = 384;  // 4 control warps + 2 column halves x 4 warps
constexpr int kAttnBM = 128;       // query rows per CTA
constexpr float kRescaleLog2 = 8.0f;
// Fraction of exp2 evaluated by the FMA-pipe polynomial instead of MUFU.EX2
// (1 in NT_POLY_EVERY pairs; 0 = MUFU only).
#ifndef NT_POLY_EVERY
#define NT_POLY_EVERY 0
#endif
constexpr bool kPolyExp = NT_POLY_EVERY > 0;
constexpr int kPolyEvery = NT_POLY_EVERY > 0 ? NT_POLY_EVERY : 1;
// P -> bf16 packing on the ALU (1) or with cvt.rn.bf16x2 (0)
#ifndef NT_PACK_ALU
#define NT_PACK_ALU 0
#endif
constexpr bool kPackAlu = NT_PACK_ALU != 0;

template <int D>
struct AttnCfg {
  static constexpr int BM = 128, BN = 128;
  static constexpr int HALF = 128 * 64 * 2;  // one 128-row x 64-col bf16 swizzle-128B panel
  static constexpr int TQ = BM * D * 2;
  static constexpr int TKV = BN * D * 2;
  static constexpr int STAGES = (D == 128) ? 5 : 8;
  static constexpr int SMEM_Q = 0;
  static constexpr int SMEM_KV = TQ;
  static constexpr int SMEM_BAR = SMEM_KV + STAGES * TKV;
  static constexpr int NBAR = 1 + 2 * STAGES + 2 + 1 + 1 + 1;
  static constexpr int SMEM_RED = SMEM_BAR + NBAR * 8 + 16;  // half-row max / sum exchange (3 KB)
  static constexpr int SMEM_BYTES = SMEM_RED + 768 * 4 + 1024;  // + alignment slack
};

__device__ __forceinline__ float f_ninf() { return __int_as_float(0xff800000); }

#ifdef NT_TRACE
// Debug timeline (NT_TRACE builds only): clock64 stamps of one CTA's pipeline.
// trace[(role * 64 + iter) * 8 + event]; role 0 MMA, 1/2 softmax half 0/1, 3 producer.
__device__ unsigned long long* g_nt_trace = nullptr;
__device__ int g_nt_trace_cta = 0;
#define NT_STAMP(role, iter, ev)                                                               \
  do {                                                                                         \
    if (g_nt_trace && blockIdx.x == g_nt_trace_cta && (iter) < 64)                             \
      g_nt_trace[((role) * 64 + (iter)) * 8 + (ev)] = clock64();                               \
  } while (0)
#else
#define NT_STAMP(role, iter, ev) do {} while (0)
#endif

template <int D, int MASK, bool OUT_F32>
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                    const AttnFwdParams p) {
  using C = AttnCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);

  uint8_t* sQ = smem + C::SMEM_Q;
  uint8_t* sKV = smem + C::SMEM_KV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::SMEM_BAR);
  uint64_t* bar_q = bars;                           // [1]
  uint64_t* bar_kv_full = bars + 1;                 // [STAGES]
  uint64_t* bar_kv_empty = bars + 1 + C::STAGES;    // [STAGES]
  uint64_t* bar_s_full = bars + 1 + 2 * C::STAGES;  // [2] (S buffer parity)
  uint64_t* bar_p_full = bar_s_full + 2;            // [1]
  uint64_t* bar_pv_done = bar_p_full + 1;           // [1]
  uint64_t* bar_o_full = bar_pv_done + 1;           // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);
  float* red = reinterpret_cast<float*>(smem + C::SMEM_RED);

  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const int lane = threadIdx.x & 31;

  // ---- tile coordinates (causal: heaviest query blocks first -> LPT order)
  const int BH = p.B * p.Hq;
  const int bh = blockIdx.x % BH;
  const int mbi = blockIdx.x / BH;
  const int mb = (MASK == MASK_CAUSAL) ? (p.n_mblocks - 1 - mbi) : mbi;
  const int hq = bh % p.Hq;
  const int b = bh / p.Hq;
  const int hkv = hq / p.q_per_kv;
  const int q_row0 = mb * kAttnBM;
  int n_kv = p.n_kv_total;
  if (MASK == MASK_CAUSAL) {
    const int last_q = min(q_row0 + kAttnBM - 1, p.N - 1) + p.causal_offset;
    n_kv = min(n_kv, last_q / 128 + 1);
    n_kv = max(n_kv, 1);
  }

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmQ);
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    if (!OUT_F32) prefetch_tmap(&tmO);
    mbar_init(bar_q, 1);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&bar_kv_full[s], 1);
      mbar_init(&bar_kv_empty[s], 1);
    }
    mbar_init(&bar_s_full[0], 1);
    mbar_init(&bar_s_full[1], 1);
    mbar_init(bar_p_full, 8);
    mbar_init(bar_pv_done, 1);
    mbar_init(bar_o_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // setmaxnreg only redistributes the launch allocation (384 x 168 regs):
    // 128 x 56 + 256 x 224 = 64512
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (warp == 0) {
      // ================= TMA producer
      if (lane == 0) {
        mbar_arrive_expect_tx(bar_q, C::TQ);
#pragma unroll
        for (int h = 0; h < D / 64; ++h) tma_load_4d(sQ + h * C::HALF, &tmQ, bar_q, h * 64, q_row0, hq, b);
        for (int it = 0; it < 2 * n_kv; ++it) {
          const int slot = it % C::STAGES;
          const uint32_t ph = (it / C::STAGES) & 1;
          NT_STAMP(3, it >> 1, (it & 1) * 2);
          mbar_wait(&bar_kv_empty[slot], ph ^ 1, p.err, 1);
          NT_STAMP(3, it >> 1, (it & 1) * 2 + 1);
          mbar_arrive_expect_tx(&bar_kv_full[slot], C::TKV);
          const CUtensorMap* m = (it & 1) ? &tmV : &tmK;
          const int row = (it >> 1) * 128;
#pragma unroll
          for (int h = 0; h < D / 64; ++h)
            tma_load_4d(sKV + slot * C::TKV + h * C::HALF, m, &bar_kv_full[slot], h * 64, row, hkv, b);
        }
      }
    } else if (warp == 1) {
      // ================= MMA issuer: S(0); S(1), PV(0); S(2), PV(1); ...
      if (lane == 0) {
        constexpr uint32_t idS = idesc_bf16(128, 128, 0, 0);
        constexpr uint32_t idO = idesc_bf16(128, D, 0, 1);
        const uint32_t sQa = smem_u32(sQ), sKVa = smem_u32(sKV);
        const uint32_t tO = tmem + 256;
        auto issue_s = [&](int j) {  // S[j&1] = Q K_j^T
          const int it = 2 * j, slot = it % C::STAGES;
          mbar_wait(&bar_kv_full[slot], (it / C::STAGES) & 1, p.err, 3);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = (k >> 2) * C::HALF + (k & 3) * 32;
            const uint64_t a = sdesc_sw128(sQa + off, 16, 1024);
            const uint64_t bd = sdesc_sw128(sKVa + slot * C::TKV + off, 16, 1024);
            umma_ss(tmem + (j & 1) * 128, a, bd, idS, k > 0 ? 1u : 0u);
          }
          umma_commit(&bar_s_full[j & 1]);
          umma_commit(&bar_kv_empty[slot]);
        };
        auto issue_pv = [&](int j) {  // O (+)= P(j) V_j, P(j) in TMEM over S[j&1]
          const int it = 2 * j + 1, slot = it % C::STAGES;
          mbar_wait(&bar_kv_full[slot], (it / C::STAGES) & 1, p.err, 5);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint64_t bd = sdesc_sw128(sKVa + slot * C::TKV + k * 2048, C::HALF, 1024);
            umma_ts(tO, tmem + (j & 1) * 128 + k * 8, bd, idO, (j > 0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&bar_kv_empty[slot]);
          umma_commit(bar_pv_done);
        };
        mbar_wait(bar_q, 0, p.err, 2);
        tc_fence_after();
        NT_STAMP(0, 0, 0);
        issue_s(0);
        for (int j = 0; j < n_kv; ++j) {
          NT_STAMP(0, j, 1);
          if (j + 1 < n_kv) issue_s(j + 1);
          NT_STAMP(0, j, 2);
          mbar_wait(bar_p_full, j & 1, p.err, 4);
          NT_STAMP(0, j, 3);
          tc_fence_after();
          issue_pv(j);
          NT_STAMP(0, j, 4);
        }
        umma_commit(bar_o_full);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    // ================= softmax (+ lazy O correction + epilogue)
    const int h = (warp - 4) >> 2;  // key-column half
    const int wq = warp & 3;        // TMEM sub-partition this warp may access
    const int r = wq * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t tO = tmem + 256 + lane_off;
    const int qi = q_row0 + r;
    const float NINF = f_ninf();
    const float sc = (MASK == MASK_TENSOR) ? 1.0f : p.scale_log2;
    float* xmax = red;         // [2 buffers][2 halves][128 rows]
    float* xsum = red + 512;   // [2 halves][128 rows]
    constexpr int HC = 64;     // key columns per half
    constexpr int DH = D / 2;  // O columns per half
    float m_run = NINF, l_run = 0.f;

    for (int j = 0; j < n_kv; ++j) {
      const uint32_t tS = tmem + (j & 1) * 128 + lane_off;
      if (lane == 0 && wq == 0) NT_STAMP(1 + h, j, 0);
      mbar_wait(&bar_s_full[j & 1], (j >> 1) & 1, p.err, 8);
      if (lane == 0 && wq == 0) NT_STAMP(1 + h, j, 1);
      tc_fence_after();
      uint32_t s[HC];
      tmem_ld32(tS + h * HC, s);
      tmem_ld32(tS + h * HC + 32, s + 32);
      tmem_wait_ld();
      if (lane == 0 && wq == 0) NT_STAMP(1 + h, j, 2);
      const int kv0 = j * 128 + h * HC;
      if (MASK == MASK_TENSOR) {
        const float* mrow = p.mask + (long long)min(qi, p.N - 1) * p.mask_row_stride;
#pragma unroll
        for (int c = 0; c < HC; ++c) {
          const int kv = kv0 + c;
          const float mk = (kv < p.M) ? __ldg(mrow + kv) : NINF;
          s[c] = __float_as_uint(fmaf(__uint_as_float(s[c]), p.scale_log2, mk * 1.4426950408889634f));
        }
      } else {
        const int lim = (MASK == MASK_CAUSAL) ? min(qi + p.causal_offset, p.M - 1) : (p.M - 1);
        if (kv0 + HC - 1 > lim) {
#pragma unroll
          for (int c = 0; c < HC; ++c)
            if (kv0 + c > lim) s[c] = __float_as_uint(NINF);
        }
      }
      float mx;
      {
        // tree max with 3-input FMNMX3, 4 independent chains
        float a0 = __uint_as_float(s[0]), a1 = __uint_as_float(s[1]);
        float a2 = __uint_as_float(s[2]), a3 = __uint_as_float(s[3]);
#pragma unroll
        for (int c = 4; c < HC; c += 8) {
          a0 = fmax3(a0, __uint_as_float(s[c]), __uint_as_float(s[c + 1]));
          a1 = fmax3(a1, __uint_as_float(s[c + 2]), __uint_as_float(s[c + 3]));
          a2 = fmax3(a2, __uint_as_float(s[c + 4]), __uint_as_float(s[c + 5]));
          if (c + 7 < HC) a3 = fmax3(a3, __uint_as_float(s[c + 6]), __uint_as_float(s[c + 7]));
          else a3 = fmaxf(a3, __uint_as_float(s[c + 6]));
        }
        mx = fmaxf(fmax3(a0, a1, a2), a3);
      }
      // exchange the half-row maxima (double-buffered on j: one barrier per KV tile)
      float* xm = xmax + (j & 1) * 256;
      xm[h * 128 + r] = mx;
      named_bar_sync(1, 256);
      mx = fmaxf(mx, xm[(h ^ 1) * 128 + r]);
      if (lane == 0 && wq == 0) NT_STAMP(1 + h, j, 3);
      const float m_new = fmaxf(m_run, mx * sc);
      const bool need = m_new > m_run + kRescaleLog2;
      // both halves hold the same rows (same TMEM lanes) -> identical warp decisions
      if (__any_sync(0xffffffffu, need)) {
        const float alpha = (m_new == NINF) ? 1.0f : ex2(m_run - m_new);
        if (j > 0) {
          // O must hold PV(j-1) before it is rescaled (S(j) no longer implies it);
          // PV(j) cannot complete before P(j) exists, so the parity wait is exact
          mbar_wait(bar_pv_done, (j - 1) & 1, p.err, 10);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < DH / 16; ++c) {
            uint32_t o[16];
            tmem_ld16(tO + h * DH + c * 16, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st16(tO + h * DH + c * 16, o);
          }
        }
        l_run *= alpha;
        m_run = m_new;
      }
      const float m_use = (m_run == NINF) ? 0.f : m_run;
      const float2 sc2 = make_float2(sc, sc);
      const float2 nm2 = make_float2(-m_use, -m_use);
      float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 x = ffma2(make_float2(__uint_as_float(s[ch * 32 + 2 * i]),
                                             __uint_as_float(s[ch * 32 + 2 * i + 1])), sc2, nm2);
          float2 e;
          if (kPolyExp && (i % kPolyEvery) == kPolyEvery - 1) {
            e = ex2_poly2(x);  // FMA-pipe exp2 for 1/kPolyEvery of the pairs
          } else {
            e = make_float2(ex2(x.x), ex2(x.y));
          }
          sum2[i & 1] = fadd2(sum2[i & 1], e);
          pk[i] = kPackAlu ? pack_bf16_alu(e.x, e.y) : pack_bf16(e.x, e.y);
        }
        tmem_st16(tS + h * (HC / 2) + ch * 16, pk);  // P (bf16) over this half's key columns
      }
      const float sum = (sum2[0].x + sum2[0].y) + (sum2[1].x + sum2[1].y);
      if (lane == 0 && wq == 0) NT_STAMP(1 + h, j, 4);
      l_run += sum;
      tmem_wait_st();
      if (lane == 0 && wq == 0) NT_STAMP(1 + h, j, 5);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_p_full);
    }

    // ---- epilogue: O / l  (l = sum of the two half-row partial sums)
    xsum[h * 128 + r] = l_run;
    mbar_wait(bar_o_full, 0, p.err, 9);
    tc_fence_after();
    named_bar_sync(1, 256);
    const float l_tot = l_run + xsum[(h ^ 1) * 128 + r];
    const bool valid = qi < p.N;
    if (valid && h == 0 && !(l_tot > 0.f) && p.err) atomicOr(p.err, 1);
    const float inv = (l_tot > 0.f) ? 1.0f / l_tot : 0.f;
    if (OUT_F32) {
      float* orow = p.o_f32 + (long long)b * p.o_sb + (long long)hq * p.o_sh + (long long)qi * p.o_sn + h * DH;
#pragma unroll
      for (int c = 0; c < DH / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + h * DH + c * 32, o);
        tmem_wait_ld();
        if (valid) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 v = make_float4(__uint_as_float(o[4 * i]) * inv, __uint_as_float(o[4 * i + 1]) * inv,
                                   __uint_as_float(o[4 * i + 2]) * inv, __uint_as_float(o[4 * i + 3]) * inv);
            *reinterpret_cast<float4*>(orow + c * 32 + 4 * i) = v;
          }
        }
      }
    } else {
      uint8_t* stage = sQ;  // Q is dead once O is final
#pragma unroll
      for (int c = 0; c < DH / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + h * DH + c * 32, o);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = pack_bf16(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
        const int col0 = h * DH + c * 32;  // first O column of this 32-column chunk
        uint8_t* rowp = stage + (col0 >> 6) * C::HALF + r * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int chunk = (((col0 & 63) >> 3) + q) ^ (r & 7);
          *reinterpret_cast<uint4*>(rowp + chunk * 16) = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1, 256);
      if (h == 0 && r == 0) {
#pragma unroll
        for (int hh = 0; hh < D / 64; ++hh) tma_store_4d(&tmO, stage + hh * C::HALF, hh * 64, q_row0, hq, b);
        bulk_commit();
        bulk_wait_read0();
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

}  // namespace nt
