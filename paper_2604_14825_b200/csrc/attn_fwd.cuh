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
// CTA = two 128-row query tiles (256 rows = 256/t0_i consecutive MA blocks)
// sharing each 128-row K/V tile (128/t0_j consecutive MA j0 iterations; the
// rolling-update law makes the coarsening exact up to rounding).
//
//   warp 0      TMA producer: Q0,Q1 once, then K0,V0,K1,V1,... into a STAGES ring
//   warp 1      MMA issuer (one thread): S_t = Q_t K_j^T (SS), O_t += P_t V_j (TS, P from TMEM)
//   warps 2-3   idle (warpgroup 0 donates registers via setmaxnreg)
//   warps 4-7   softmax for tile 0 (one thread per query row = TMEM lane)
//   warps 8-11  softmax for tile 1
// TMEM (512 cols): S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [384,384+D);
// P_t (bf16, 64 cols) aliases the first half of S_t.
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

enum { MASK_NONE = 0, MASK_CAUSAL = 1, MASK_TENSOR = 2 };

struct AttnFwdParams {
  int B, Hq, Hkv, N, M;
  int q_per_kv;
  int n_mblocks;    // ceil(N / 256)
  int n_kv_total;   // ceil(M / 128)
  int causal_offset;  // key j visible to query i iff j <= i + causal_offset
  float scale_log2;   // c * log2(e)
  const float* mask;  // MASK_TENSOR: fp32 [N, M]
  long long mask_row_stride;
  float* o_f32;  // fp32 output (OUT_F32), element strides below
  long long o_sb, o_sh, o_sn;
  int* err;  // bit 0: zero denominator (fully masked row); 0x100|k: pipeline timeout
};

constexpr int kAttnThreads = 384;
constexpr float kRescaleLog2 = 8.0f;
// Fraction of exp2 evaluated by the FMA-pipe polynomial instead of MUFU.EX2
// (1 in NT_POLY_EVERY pairs; 0 = MUFU only).  Measured on B200 at Llama 8K
// causal: 0 -> 1177, 8 -> 1163, 4 -> 1157, 2 -> 1107 TFLOP/s (profiles/), so
// the MUFU is not the binding pipe of this kernel yet: off by default.
#ifndef NT_POLY_EVERY
#define NT_POLY_EVERY 0
#endif
constexpr bool kPolyExp = NT_POLY_EVERY > 0;
constexpr int kPolyEvery = NT_POLY_EVERY > 0 ? NT_POLY_EVERY : 1;

template <int D>
struct AttnCfg {
  static constexpr int BM = 128, BN = 128;
  static constexpr int HALF = 128 * 64 * 2;  // one 128-row x 64-col bf16 swizzle-128B panel
  static constexpr int TQ = BM * D * 2;
  static constexpr int TKV = BN * D * 2;
  static constexpr int STAGES = (D == 128) ? 4 : 6;
  static constexpr int SMEM_Q = 0;
  static constexpr int SMEM_KV = 2 * TQ;
  static constexpr int SMEM_BAR = SMEM_KV + STAGES * TKV;
  static constexpr int NBAR = 2 + 2 * STAGES + 2 + 2 + 2;
  static constexpr int SMEM_BYTES = SMEM_BAR + NBAR * 8 + 16 + 1024;  // + alignment slack
};

__device__ __forceinline__ float f_ninf() { return __int_as_float(0xff800000); }

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
  uint64_t* bar_q = bars;                      // [2]
  uint64_t* bar_kv_full = bars + 2;            // [STAGES]
  uint64_t* bar_kv_empty = bars + 2 + C::STAGES;  // [STAGES]
  uint64_t* bar_s_full = bars + 2 + 2 * C::STAGES;  // [2]
  uint64_t* bar_p_full = bar_s_full + 2;            // [2]
  uint64_t* bar_o_full = bar_p_full + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);

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
  const int q_row0 = mb * 256;
  int n_kv = p.n_kv_total;
  if (MASK == MASK_CAUSAL) {
    const int last_q = min(q_row0 + 255, p.N - 1) + p.causal_offset;
    n_kv = min(n_kv, last_q / 128 + 1);
    n_kv = max(n_kv, 1);
  }

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmQ);
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    if (!OUT_F32) prefetch_tmap(&tmO);
    mbar_init(&bar_q[0], 1);
    mbar_init(&bar_q[1], 1);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&bar_kv_full[s], 1);
      mbar_init(&bar_kv_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bar_s_full[t], 1);
      mbar_init(&bar_p_full[t], 4);
      mbar_init(&bar_o_full[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
  if (warp == 0) {
    // ================= TMA producer
    if (lane == 0) {
      for (int t = 0; t < 2; ++t) {
        mbar_arrive_expect_tx(&bar_q[t], C::TQ);
#pragma unroll
        for (int h = 0; h < D / 64; ++h)
          tma_load_4d(sQ + t * C::TQ + h * C::HALF, &tmQ, &bar_q[t], h * 64, q_row0 + t * 128, hq, b);
      }
      for (int it = 0; it < 2 * n_kv; ++it) {
        const int slot = it % C::STAGES;
        const uint32_t ph = (it / C::STAGES) & 1;
        mbar_wait(&bar_kv_empty[slot], ph ^ 1, p.err, 1);
        mbar_arrive_expect_tx(&bar_kv_full[slot], C::TKV);
        const CUtensorMap* m = (it & 1) ? &tmV : &tmK;
        const int row = (it >> 1) * 128;
#pragma unroll
        for (int h = 0; h < D / 64; ++h)
          tma_load_4d(sKV + slot * C::TKV + h * C::HALF, m, &bar_kv_full[slot], h * 64, row, hkv, b);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    if (lane == 0) {
      constexpr uint32_t idS = idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idO = idesc_bf16(128, D, 0, 1);
      const uint32_t sQa = smem_u32(sQ), sKVa = smem_u32(sKV);
      auto issue_s = [&](int t, int slot) {
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * C::HALF + (k & 3) * 32;
          const uint64_t a = sdesc_sw128(sQa + t * C::TQ + off, 16, 1024);
          const uint64_t bd = sdesc_sw128(sKVa + slot * C::TKV + off, 16, 1024);
          umma_ss(tmem + t * 128, a, bd, idS, k > 0 ? 1u : 0u);
        }
      };
      auto issue_pv = [&](int t, int slot, bool acc) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t bd = sdesc_sw128(sKVa + slot * C::TKV + k * 2048, C::HALF, 1024);
          umma_ts(tmem + 256 + t * 128, tmem + t * 128 + k * 8, bd, idO, (acc || k > 0) ? 1u : 0u);
        }
      };
      mbar_wait(&bar_q[0], 0, p.err, 2);
      mbar_wait(&bar_q[1], 0, p.err, 2);
      tc_fence_after();
      for (int j = 0; j < n_kv; ++j) {
        const int itK = 2 * j;
        const int slotK = itK % C::STAGES;
        mbar_wait(&bar_kv_full[slotK], (itK / C::STAGES) & 1, p.err, 3);
        tc_fence_after();
        const int itV = 2 * (j - 1) + 1;
        const int slotV = (itV + C::STAGES) % C::STAGES;
        for (int t = 0; t < 2; ++t) {
          if (j > 0) {
            mbar_wait(&bar_p_full[t], (j - 1) & 1, p.err, 4);
            if (t == 0) mbar_wait(&bar_kv_full[slotV], (itV / C::STAGES) & 1, p.err, 5);
            tc_fence_after();
  #ifndef NT_EXP_NO_PV
          issue_pv(t, slotV, j - 1 > 0);
#endif
            if (t == 1) umma_commit(&bar_kv_empty[slotV]);
          }
#ifndef NT_EXP_NO_S
          issue_s(t, slotK);
#endif
          umma_commit(&bar_s_full[t]);
        }
        umma_commit(&bar_kv_empty[slotK]);
      }
      const int itV = 2 * (n_kv - 1) + 1;
      const int slotV = itV % C::STAGES;
      for (int t = 0; t < 2; ++t) {
        mbar_wait(&bar_p_full[t], (n_kv - 1) & 1, p.err, 6);
        if (t == 0) mbar_wait(&bar_kv_full[slotV], (itV / C::STAGES) & 1, p.err, 7);
        tc_fence_after();
        issue_pv(t, slotV, n_kv - 1 > 0);
        umma_commit(&bar_o_full[t]);
      }
      umma_commit(&bar_kv_empty[slotV]);
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    // ================= softmax (+ lazy O correction + epilogue), one thread per query row
    const int t = (warp - 4) / 4;
    const int wq = warp & 3;  // TMEM sub-partition this warp may access
    const int r = wq * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t tS = tmem + t * 128 + lane_off;
    const uint32_t tO = tmem + 256 + t * 128 + lane_off;
    const int qi = q_row0 + t * 128 + r;
    const float NINF = f_ninf();
    const float sc = (MASK == MASK_TENSOR) ? 1.0f : p.scale_log2;
    float m_run = NINF, l_run = 0.f;

    for (int j = 0; j < n_kv; ++j) {
      mbar_wait(&bar_s_full[t], j & 1, p.err, 8);
      tc_fence_after();
      uint32_t s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, s + c * 32);
      tmem_wait_ld();
      const int kv0 = j * 128;
      if (MASK == MASK_TENSOR) {
        const float* mrow = p.mask + (long long)min(qi, p.N - 1) * p.mask_row_stride;
#pragma unroll
        for (int c = 0; c < 128; ++c) {
          const int kv = kv0 + c;
          const float mk = (kv < p.M) ? __ldg(mrow + kv) : NINF;
          s[c] = __float_as_uint(fmaf(__uint_as_float(s[c]), p.scale_log2, mk * 1.4426950408889634f));
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
        // tree max with 3-input FMNMX3, 4 independent chains
        float a0 = __uint_as_float(s[0]), a1 = __uint_as_float(s[1]);
        float a2 = __uint_as_float(s[2]), a3 = __uint_as_float(s[3]);
#pragma unroll
        for (int c = 4; c < 128; c += 8) {
          a0 = fmax3(a0, __uint_as_float(s[c]), __uint_as_float(s[c + 1]));
          a1 = fmax3(a1, __uint_as_float(s[c + 2]), __uint_as_float(s[c + 3]));
          a2 = fmax3(a2, __uint_as_float(s[c + 4]), __uint_as_float(s[c + 5]));
          if (c + 7 < 128) a3 = fmax3(a3, __uint_as_float(s[c + 6]), __uint_as_float(s[c + 7]));
          else a3 = fmaxf(a3, __uint_as_float(s[c + 6]));
        }
        mx = fmaxf(fmax3(a0, a1, a2), a3);
      }
#ifdef NT_EXP_NO_SOFTMAX
      {
        uint32_t pk[16];
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = s[ch * 32 + 2 * i];
          tmem_st16(tS + ch * 16, pk);
        }
        l_run = 1.f;
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_p_full[t]);
        continue;
      }
#endif
      const float m_new = fmaxf(m_run, mx * sc);
      const bool need = m_new > m_run + kRescaleLog2;
      if (__any_sync(0xffffffffu, need)) {
        const float alpha = (m_new == NINF) ? 1.0f : ex2(m_run - m_new);
        if (j > 0) {
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
        l_run *= alpha;
        m_run = m_new;
      }
      const float m_use = (m_run == NINF) ? 0.f : m_run;
      const float2 sc2 = make_float2(sc, sc);
      const float2 nm2 = make_float2(-m_use, -m_use);
      float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
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
          pk[i] = pack_bf16(e.x, e.y);
        }
        tmem_st16(tS + ch * 16, pk);
      }
      const float sum = (sum2[0].x + sum2[0].y) + (sum2[1].x + sum2[1].y);
      l_run += sum;
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_p_full[t]);
    }

    // ---- epilogue: O / l
    mbar_wait(&bar_o_full[t], 0, p.err, 9);
    tc_fence_after();
    const bool valid = qi < p.N;
    if (valid && !(l_run > 0.f) && p.err) atomicOr(p.err, 1);
    const float inv = (l_run > 0.f) ? 1.0f / l_run : 0.f;
    if (OUT_F32) {
      float* orow = p.o_f32 + (long long)b * p.o_sb + (long long)hq * p.o_sh + (long long)qi * p.o_sn;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + c * 32, o);
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
      uint8_t* stage = sQ + t * C::TQ;  // Q_t is dead once O_t is final
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + c * 32, o);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = pack_bf16(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
        uint8_t* rowp = stage + (c >> 1) * C::HALF + r * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int chunk = ((c & 1) * 4 + q) ^ (r & 7);
          *reinterpret_cast<uint4*>(rowp + chunk * 16) = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1 + t, 128);
      if (r == 0) {
#pragma unroll
        for (int h = 0; h < D / 64; ++h)
          tma_store_4d(&tmO, stage + h * C::HALF, h * 64, q_row0 + t * 128, hq, b);
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
