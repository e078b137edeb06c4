// K2: split-KV decode attention + combine (flash-decoding), HBM-bound.
//
// The reference schedules decode (N = 1 or the 4 GQA-packed q-heads of a kv
// group, M = 32K-128K) as ONE MA block with a sequential KV loop of M/128
// iterations (SURVEY.md B.5, Appendix C V2/V2').  A single block cannot fill
// 148 SMs, so the KV range of every (batch, kv-head) group is split over
// CTAs; each CTA runs the same rolling-update recurrence (m, l, O) over its
// key range and the partial states are merged with the repair law
// O = sum_s O_s 2^(m_s - m) / sum_s l_s 2^(m_s - m)   (tilecc/schedule/repair.py:80-88).
//
// The work is 4 flop/byte (GQA ratio 4), far below the tensor-core ridge, so
// the kernel streams K/V with coalesced 16-byte loads straight into
// registers (software-pipelined one key step ahead) and does the dots on the
// FMA pipe: TPK = max(8, 2R) threads share a key (DPT = 128/TPK dims each), the R rows of
// the group live in registers, partial dots are reduced with shuffles.
#pragma once
#include "sm100.cuh"

namespace nt {

struct DecodeParams {
  const __nv_bfloat16* q;
  long long q_sb, q_sh, q_sn;
  const __nv_bfloat16* k;
  long long k_sb, k_sh, k_sn;
  const __nv_bfloat16* v;
  long long v_sb, v_sh, v_sn;
  void* o;
  long long o_sb, o_sh, o_sn;
  int out_f32;
  int B, Hq, Hkv, Nq, M, g;  // rows per group R = g * Nq
  float scale_log2;
  int splits, keys_per_split;
  float* ws;  // [B*Hkv, splits, R, D + 2]  (O, m, l)
  int* err;
};

constexpr int kDecodeThreads = 128;
constexpr int kDecodeD = 128;

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  f[0] = __uint_as_float(u.x << 16);
  f[1] = __uint_as_float(u.x & 0xffff0000u);
  f[2] = __uint_as_float(u.y << 16);
  f[3] = __uint_as_float(u.y & 0xffff0000u);
  f[4] = __uint_as_float(u.z << 16);
  f[5] = __uint_as_float(u.z & 0xffff0000u);
  f[6] = __uint_as_float(u.w << 16);
  f[7] = __uint_as_float(u.w & 0xffff0000u);
}

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int R>
__global__ void __launch_bounds__(kDecodeThreads, 2) decode_split_kernel(const DecodeParams p) {
  constexpr int D = kDecodeD;
  constexpr int TPK = (2 * R > 8) ? 2 * R : 8;  // threads per key
  constexpr int DPT = D / TPK;                  // dims per thread
  constexpr int KPS = kDecodeThreads / TPK;  // keys per step
  constexpr int NV = DPT / 8;            // 16-byte vectors per thread per row
  static_assert(DPT % 8 == 0, "DPT must be a multiple of 8");
  __shared__ float sm_m[KPS][R];
  __shared__ float sm_l[KPS][R];
  __shared__ float sm_o[KPS][R][D];

  const int s = blockIdx.x;
  const int grp = blockIdx.y;  // b * Hkv + hkv
  const int b = grp / p.Hkv, hkv = grp % p.Hkv;
  const int t = threadIdx.x;
  const int kg = t / TPK, ds = t % TPK;
  const int d0 = ds * DPT;

  float q[R][DPT];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int h = hkv * p.g + r / p.Nq, n = r % p.Nq;
    const __nv_bfloat16* qp = p.q + b * p.q_sb + h * p.q_sh + n * p.q_sn + d0;
#pragma unroll
    for (int i = 0; i < NV; ++i) bf16x8_to_f32(*reinterpret_cast<const uint4*>(qp + 8 * i), &q[r][8 * i]);
#pragma unroll
    for (int i = 0; i < DPT; ++i) q[r][i] *= p.scale_log2;  // fold c*log2e into q
  }
  float o[R][DPT];
  float m[R], l[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    m[r] = __int_as_float(0xff800000);
    l[r] = 0.f;
#pragma unroll
    for (int i = 0; i < DPT; ++i) o[r][i] = 0.f;
  }

  const int j0 = s * p.keys_per_split;
  const int j1 = min(p.M, j0 + p.keys_per_split);
  const __nv_bfloat16* kbase = p.k + b * p.k_sb + hkv * p.k_sh + d0;
  const __nv_bfloat16* vbase = p.v + b * p.v_sb + hkv * p.v_sh + d0;

  // warp-uniform trip count: every lane runs every step (the TPK-lane shuffles
  // below need all lanes of the warp); out-of-range keys contribute nothing.
  const int nsteps = (j1 > j0) ? (j1 - j0 + KPS - 1) / KPS : 0;
  uint4 kc[NV], vc[NV];
  {
    const int j = j0 + kg;
    const bool ok = j < j1;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      kc[i] = ok ? ldg_nc_v4(kbase + (long long)j * p.k_sn + 8 * i) : make_uint4(0, 0, 0, 0);
      vc[i] = ok ? ldg_nc_v4(vbase + (long long)j * p.v_sn + 8 * i) : make_uint4(0, 0, 0, 0);
    }
  }
  for (int st = 0; st < nsteps; ++st) {
    const int j = j0 + st * KPS + kg;
    const bool valid = j < j1;
    // prefetch the next key of this group (one step ahead)
    uint4 kn[NV], vn[NV];
    const int jn = j + KPS;
    const bool okn = jn < j1;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      kn[i] = okn ? ldg_nc_v4(kbase + (long long)jn * p.k_sn + 8 * i) : make_uint4(0, 0, 0, 0);
      vn[i] = okn ? ldg_nc_v4(vbase + (long long)jn * p.v_sn + 8 * i) : make_uint4(0, 0, 0, 0);
    }
    float kf[DPT], vf[DPT];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      bf16x8_to_f32(kc[i], &kf[8 * i]);
      bf16x8_to_f32(vc[i], &vf[8 * i]);
    }
    float sc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float a0 = 0.f, a1 = 0.f;
#pragma unroll
      for (int i = 0; i < DPT; i += 2) {
        a0 = fmaf(q[r][i], kf[i], a0);
        a1 = fmaf(q[r][i + 1], kf[i + 1], a1);
      }
      sc[r] = a0 + a1;
    }
#pragma unroll
    for (int off = 1; off < TPK; off <<= 1)
#pragma unroll
      for (int r = 0; r < R; ++r) sc[r] += __shfl_xor_sync(0xffffffffu, sc[r], off);
    if (valid) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (sc[r] > m[r] + 8.0f) {  // lazy rescale (exact identity; keeps p <= 2^8)
          const float alpha = ex2(m[r] - sc[r]);
          l[r] *= alpha;
#pragma unroll
          for (int i = 0; i < DPT; ++i) o[r][i] *= alpha;
          m[r] = sc[r];
        }
        const float pr = ex2(sc[r] - m[r]);
        l[r] += pr;
#pragma unroll
        for (int i = 0; i < DPT; ++i) o[r][i] = fmaf(pr, vf[i], o[r][i]);
      }
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      kc[i] = kn[i];
      vc[i] = vn[i];
    }
  }

  // ---- merge the KPS key groups of this CTA
  if (ds == 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      sm_m[kg][r] = m[r];
      sm_l[kg][r] = l[r];
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int i = 0; i < DPT; ++i) sm_o[kg][r][d0 + i] = o[r][i];
  __syncthreads();
  float* ws = p.ws + ((long long)grp * p.splits + s) * R * (D + 2);
  for (int idx = t; idx < R * D; idx += kDecodeThreads) {
    const int r = idx / D, d = idx % D;
    float mm = __int_as_float(0xff800000);
#pragma unroll 4
    for (int c = 0; c < KPS; ++c) mm = fmaxf(mm, sm_m[c][r]);
    float ll = 0.f, oo = 0.f;
    if (mm != __int_as_float(0xff800000)) {
#pragma unroll 4
      for (int c = 0; c < KPS; ++c) {
        const float w = ex2(sm_m[c][r] - mm);
        ll = fmaf(sm_l[c][r], w, ll);
        oo = fmaf(sm_o[c][r][d], w, oo);
      }
    }
    ws[r * (D + 2) + d] = oo;
    if (d == 0) {
      ws[r * (D + 2) + D] = mm;
      ws[r * (D + 2) + D + 1] = ll;
    }
  }
}

// combine the split partials of every (group, row); one warp per row
__global__ void decode_combine_kernel(const DecodeParams p, int R) {
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  const int ngroups = p.B * p.Hkv;
  if (row >= ngroups * R) return;
  const int grp = row / R, r = row % R;
  const int b = grp / p.Hkv, hkv = grp % p.Hkv;
  const int h = hkv * p.g + r / p.Nq, n = r % p.Nq;
  constexpr int D = kDecodeD;
  const float* ws = p.ws + (long long)grp * p.splits * R * (D + 2);
  float mm = __int_as_float(0xff800000);
  for (int s = 0; s < p.splits; ++s) mm = fmaxf(mm, ws[(s * R + r) * (D + 2) + D]);
  float ll = 0.f;
  float acc[D / 32];
#pragma unroll
  for (int i = 0; i < D / 32; ++i) acc[i] = 0.f;
  if (mm != __int_as_float(0xff800000)) {
    for (int s = 0; s < p.splits; ++s) {
      const float* w = ws + (s * R + r) * (D + 2);
      const float sc = ex2(w[D] - mm);
      ll = fmaf(w[D + 1], sc, ll);
#pragma unroll
      for (int i = 0; i < D / 32; ++i) acc[i] = fmaf(w[lane + 32 * i], sc, acc[i]);
    }
  }
  if (!(ll > 0.f) && lane == 0 && p.err) atomicOr(p.err, 1);
  const float inv = ll > 0.f ? 1.f / ll : 0.f;
  const long long base = b * p.o_sb + h * p.o_sh + n * p.o_sn;
#pragma unroll
  for (int i = 0; i < D / 32; ++i) {
    const float val = acc[i] * inv;
    if (p.out_f32)
      static_cast<float*>(p.o)[base + lane + 32 * i] = val;
    else
      static_cast<__nv_bfloat16*>(p.o)[base + lane + 32 * i] = __float2bfloat16_rn(val);
  }
}

}  // namespace nt
