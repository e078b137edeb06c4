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
// the kernel is built to stream: a producer warp keeps kDecodeStages K/V tile
// pairs (64 keys each, swizzle-128B) in flight with TMA, and 256 consumer
// threads do the dots on the FMA pipe from shared memory -- 8 (R < 8) or 16
// threads share a key, the R rows of the group live in registers, partial
// dots are reduced with shuffles.
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
  float o_scale;  // K2b e4m3: V's descale, applied to the partial O (1 otherwise)
  int splits, keys_per_split;
  float* ws;  // [B*Hkv, splits, R, D + 2]  (O, m, l)
  int* err;
  // paged KV cache (decode_split_kernel<R, true>): K/V tokens live in pages of
  // `page_size` tokens; block_table[b * bt_stride + i] is the physical page of
  // logical page i of sequence b, seq_lens[b] its key count (<= M)
  const int* block_table;
  int bt_stride, page_size;
  const int* seq_lens;
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

constexpr int kDecodeTile = 64;    // keys per TMA tile
constexpr int kDecodeStages = 6;   // K+V tile pairs in flight per CTA (192 KB)
constexpr int kDecodeConsumers = 256;                    // 8 consumer warps (warpgroups 1-2)
constexpr int kDecodeCTAThreads = 128 + kDecodeConsumers;  // warpgroup 0: TMA producer + 3 idle warps
constexpr int kDecodePanel = kDecodeTile * 128;          // one 64-dim swizzle-128B panel (8 KB)
constexpr int kDecodeTileBytes = 2 * kDecodePanel;       // 64 keys x 128 dims bf16 (16 KB)
constexpr int kDecodeBtChunk = 2048;  // paged: block-table entries staged in shared memory at a time
constexpr int kDecodeSmem = kDecodeStages * 2 * kDecodeTileBytes + 1024 + 2 * kDecodeStages * 8 + 64 + 4 * kDecodeBtChunk;
template <int R>
struct DecodeShape {
  static constexpr int TPK = (R >= 8) ? 16 : 8;  // threads per key
  static constexpr int DPT = kDecodeD / TPK;      // dims per thread (16 or 8)
  static constexpr int NCH = DPT / 8;             // 16-byte chunks per thread per row
  static constexpr int KPS = kDecodeConsumers / TPK;  // keys per consumer step
};

// One CTA = (split, batch x kv-head group).  Warp 0 streams K/V tiles with TMA into a
// kDecodeStages-deep ring; warpgroups 1-2 (256 threads) consume them from shared memory.
// setmaxnreg moves the idle registers of warpgroup 0 to the consumers.
// PG: 0 dense KV, 1 paged (pages of >= 64 tokens), 2 paged with small pages (one
// 5-D TMA box per page slice)
template <int R, int PG = 0>
__global__ void __launch_bounds__(kDecodeCTAThreads, 1)
    decode_split_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                        const DecodeParams p) {
  constexpr int D = kDecodeD;
  using SH = DecodeShape<R>;
  constexpr bool PAGED = PG != 0;
  constexpr int TPK = SH::TPK, DPT = SH::DPT, KPS = SH::KPS, NCH = SH::NCH;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kDecodeStages * 2 * kDecodeTileBytes);
  uint64_t* empty = full + kDecodeStages;
  int* sbt = reinterpret_cast<int*>(empty + kDecodeStages + 8);  // paged: block-table chunk

  const int s = blockIdx.x;
  const int grp = blockIdx.y;  // b * Hkv + hkv
  const int b = grp / p.Hkv, hkv = grp % p.Hkv;
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const int lane = threadIdx.x & 31;
  const int j0 = s * p.keys_per_split;  // multiple of kDecodeTile
  const int seq_len = PAGED ? min(p.M, p.seq_lens[b]) : p.M;
  const int j1 = min(seq_len, j0 + p.keys_per_split);
  const int ntiles = (j1 > j0) ? (j1 - j0 + kDecodeTile - 1) / kDecodeTile : 0;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    for (int i = 0; i < kDecodeStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kDecodeConsumers / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    if (PAGED && warp == 0) {
      // the whole warp stages this split's block-table entries in shared memory
      // (coalesced, 8 independent loads in flight per lane), then issues the
      // page-gather TMAs.  Entries past kDecodeBtChunk are read from global.
      const int rows = min(kDecodeTile, p.page_size);
      const int last_page = (seq_len - 1) / p.page_size;
      const int* bt = p.block_table + (long long)b * p.bt_stride;
      const int first = j0 / p.page_size;
      const int n_pages = (ntiles > 0) ? min(kDecodeBtChunk, min(last_page, (j1 - 1) / p.page_size) - first + 1) : 0;
      for (int i0 = 0; i0 < n_pages; i0 += 32 * 8) {
        int v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u * 32 + lane;
          v[u] = (i < n_pages) ? __ldg(bt + first + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u * 32 + lane;
          if (i < n_pages) sbt[i] = v[u];
        }
      }
      __syncwarp();
      // lane 0 claims the ring slot; small pages (PG 2: 64/rows page slices x K,V
      // boxes per tile) spread the box issues over one lane each -- from one thread
      // they serialised (16-token pages 0.70 -> 0.81 of HBM); with 4 boxes per tile
      // (PG 1) one lane issues all of them (spreading measured 0.853 -> 0.84)
      const int nsub = kDecodeTile / rows;
      const int per_sub = (PG == 2) ? 2 : 4;  // 5-D box (both panels) x K,V | 4-D panel x K,V
      const int jobs = (PG == 2) ? nsub * per_sub : 1;
      const bool pow2 = (p.page_size & (p.page_size - 1)) == 0;
      const int ps_log2 = 31 - __clz(p.page_size);
      for (int t = 0; t < ntiles; ++t) {
        const int slot = t % kDecodeStages;
        if (lane == 0) {
          mbar_wait(&empty[slot], ((t / kDecodeStages) & 1) ^ 1, p.err, 11);
          mbar_arrive_expect_tx(&full[slot], 2 * kDecodeTileBytes);
        }
        __syncwarp();
        if (lane < jobs) {
          uint8_t* sk = smem + slot * 2 * kDecodeTileBytes;
          uint8_t* sv = sk + kDecodeTileBytes;
          if constexpr (PG == 2) {
            const int sub = lane / per_sub;
            const int tok = j0 + t * kDecodeTile + sub * rows;
            // tokens past the sequence end read its last page; the consumers mask them
            const int pg = pow2 ? (tok >> ps_log2) : tok / p.page_size;
            const int in_page = pow2 ? (tok & (p.page_size - 1)) : tok - pg * p.page_size;
            const int lp = min(pg, last_page);
            const int page = (lp - first < n_pages) ? sbt[lp - first] : __ldg(bt + lp);
            const bool is_v = lane & 1;
            // one 5-D box = both 64-dim panels of `rows` tokens: the tile is laid out
            // [sub][panel][rows][128 B] (see the consumer's address below)
            tma_load_5d((is_v ? sv : sk) + sub * 2 * rows * 128, is_v ? &tmV : &tmK, &full[slot], 0, in_page, 0,
                        hkv, page);
          } else {
            const int tok = j0 + t * kDecodeTile;
            const int pg = pow2 ? (tok >> ps_log2) : tok / p.page_size;
            const int in_page = pow2 ? (tok & (p.page_size - 1)) : tok - pg * p.page_size;
            const int lp = min(pg, last_page);
            const int page = (lp - first < n_pages) ? sbt[lp - first] : __ldg(bt + lp);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              tma_load_4d(sk + h * kDecodePanel, &tmK, &full[slot], h * 64, in_page, hkv, page);
              tma_load_4d(sv + h * kDecodePanel, &tmV, &full[slot], h * 64, in_page, hkv, page);
            }
          }
        }
      }
    } else if (!PAGED && warp == 0 && lane == 0) {
      for (int t = 0; t < ntiles; ++t) {
        const int slot = t % kDecodeStages;
        mbar_wait(&empty[slot], ((t / kDecodeStages) & 1) ^ 1, p.err, 11);
        mbar_arrive_expect_tx(&full[slot], 2 * kDecodeTileBytes);
        uint8_t* sk = smem + slot * 2 * kDecodeTileBytes;
        uint8_t* sv = sk + kDecodeTileBytes;
        const int row = j0 + t * kDecodeTile;
        tma_load_5d(sk, &tmK, &full[slot], 0, row, 0, hkv, b);  // both panels of 64 keys
        tma_load_5d(sv, &tmV, &full[slot], 0, row, 0, hkv, b);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
    const int tc = threadIdx.x - 128;
    const int rows_log2 = (PG == 2) ? (31 - __clz(min(kDecodeTile, p.page_size))) : 6;
    const int kg = tc / TPK, ds = tc % TPK;
    const int d0 = ds * DPT;
    const int panel = d0 / 64, chunk = (d0 % 64) / 8;

    // q rows (pre-scaled by c*log2e) and the O accumulators as fp32 pairs (FFMA2)
    float2 q2[R][DPT / 2];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int h = hkv * p.g + r / p.Nq, n = r % p.Nq;
      const __nv_bfloat16* qp = p.q + b * p.q_sb + h * p.q_sh + n * p.q_sn + d0;
      float qf[DPT];
#pragma unroll
      for (int c = 0; c < NCH; ++c) bf16x8_to_f32(*reinterpret_cast<const uint4*>(qp + 8 * c), &qf[8 * c]);
#pragma unroll
      for (int i = 0; i < DPT / 2; ++i) q2[r][i] = make_float2(qf[2 * i] * p.scale_log2, qf[2 * i + 1] * p.scale_log2);
    }
    float2 o2[R][DPT / 2];
    float m[R], l[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      m[r] = __int_as_float(0xff800000);
      l[r] = 0.f;
#pragma unroll
      for (int i = 0; i < DPT / 2; ++i) o2[r][i] = make_float2(0.f, 0.f);
    }

    for (int t = 0; t < ntiles; ++t) {
      const int slot = t % kDecodeStages;
      mbar_wait(&full[slot], (t / kDecodeStages) & 1, p.err, 12);
      const uint8_t* sk = smem + slot * 2 * kDecodeTileBytes;
      const uint8_t* sv = sk + kDecodeTileBytes;
#pragma unroll 2
      for (int u = 0; u < kDecodeTile / KPS; ++u) {
        const int kr = u * KPS + kg;
        const bool valid = j0 + t * kDecodeTile + kr < j1;
        float kf[DPT], vf[DPT];
        // key kr, 16-byte chunk: panel-major tile ([panel][64 keys][128 B]), or for
        // small pages [sub][panel][rows][128 B] with rows = 1 << rows_log2
        const int kbase = (PG == 2)
                              ? (((kr >> rows_log2) * 2 + panel) << (rows_log2 + 7)) + ((kr & ((1 << rows_log2) - 1)) << 7)
                              : panel * kDecodePanel + kr * 128;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const int off = kbase + (((chunk + c) ^ (kr & 7)) << 4);
          bf16x8_to_f32(*reinterpret_cast<const uint4*>(sk + off), &kf[8 * c]);
          bf16x8_to_f32(*reinterpret_cast<const uint4*>(sv + off), &vf[8 * c]);
        }
        float sc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float2 a = make_float2(0.f, 0.f);
#pragma unroll
          for (int i = 0; i < DPT / 2; ++i) a = ffma2(q2[r][i], make_float2(kf[2 * i], kf[2 * i + 1]), a);
          sc[r] = a.x + a.y;
        }
#pragma unroll
        for (int offx = 1; offx < TPK; offx <<= 1)
#pragma unroll
          for (int r = 0; r < R; ++r) sc[r] += __shfl_xor_sync(0xffffffffu, sc[r], offx);
        if (valid) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (sc[r] > m[r] + 8.0f) {  // lazy rescale (exact identity; keeps p <= 2^8)
              const float alpha = ex2(m[r] - sc[r]);
              l[r] *= alpha;
#pragma unroll
              for (int i = 0; i < DPT / 2; ++i)
                o2[r][i] = ffma2(o2[r][i], make_float2(alpha, alpha), make_float2(0.f, 0.f));
              m[r] = sc[r];
            }
            const float pr = ex2(sc[r] - m[r]);
            l[r] += pr;
#pragma unroll
            for (int i = 0; i < DPT / 2; ++i)
              o2[r][i] = ffma2(make_float2(pr, pr), make_float2(vf[2 * i], vf[2 * i + 1]), o2[r][i]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }

    // ---- merge the KPS key groups of this CTA (the ring is dead now: reuse it)
    named_bar_sync(1, kDecodeConsumers);
    float* sm_m = reinterpret_cast<float*>(smem);            // [KPS][R]
    float* sm_l = sm_m + KPS * R;                             // [KPS][R]
    float* sm_o = sm_l + KPS * R;                             // [KPS][R][D]
    if (ds == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        sm_m[kg * R + r] = m[r];
        sm_l[kg * R + r] = l[r];
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int i = 0; i < DPT / 2; ++i) {
        sm_o[(kg * R + r) * D + d0 + 2 * i] = o2[r][i].x;
        sm_o[(kg * R + r) * D + d0 + 2 * i + 1] = o2[r][i].y;
      }
    named_bar_sync(1, kDecodeConsumers);
    float* ws = p.ws + ((long long)grp * p.splits + s) * R * (D + 2);
    for (int idx = tc; idx < R * D; idx += kDecodeConsumers) {
      const int r = idx / D, d = idx % D;
      float mm = __int_as_float(0xff800000);
#pragma unroll
      for (int c = 0; c < KPS; ++c) mm = fmaxf(mm, sm_m[c * R + r]);
      float ll = 0.f, oo = 0.f;
      if (mm != __int_as_float(0xff800000)) {
#pragma unroll
        for (int c = 0; c < KPS; ++c) {
          const float w = ex2(sm_m[c * R + r] - mm);
          ll = fmaf(sm_l[c * R + r], w, ll);
          oo = fmaf(sm_o[(c * R + r) * D + d], w, oo);
        }
      }
      ws[r * (D + 2) + d] = oo;
      if (d == 0) {
        ws[r * (D + 2) + D] = mm;
        ws[r * (D + 2) + D + 1] = ll;
      }
    }
  }
}

// combine the split partials of every (group, row); one warp per row
__global__ void decode_combine_kernel(const DecodeParams p, int R) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // launched as a dependent of the split kernel
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
