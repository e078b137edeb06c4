// C ABI: nt_attn_decode (K2 split-KV decode + combine).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "../../include/nautilus_b200.h"
#include "common_host.h"
#include "decode.cuh"
#include "decode_tc.cuh"

using namespace nt;

namespace {
int sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int choose_splits(int groups, int M, int requested) {
  if (requested > 0) return std::min(requested, std::max(1, (M + 63) / 64));
  // one CTA per SM at a time: pick the split count whose last wave is fullest
  // (wave quantization is the loss of a streaming kernel), among counts that give
  // at least ~2 waves and keep >= 8 key tiles per split
  const int n_sm = sms();
  const int by_length = std::max(1, (M + 511) / 512);
  const int lo = std::max(1, std::min(by_length, (2 * n_sm + groups - 1) / groups));
  const int hi = std::max(lo, std::min(by_length, (16 * n_sm + groups - 1) / groups));
  int best = lo;
  double best_eff = -1.0;
  for (int s = lo; s <= hi; ++s) {
    const double waves = (double)groups * s / n_sm;
    const double eff = waves / std::ceil(waves);
    if (eff > best_eff + 1e-3) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

#ifndef NT_DECODE_PDL
#define NT_DECODE_PDL 1
#endif
// the repair-law combine as a programmatic dependent launch: its CTAs are scheduled
// while the split kernel drains (K2b triggers launch_dependents at entry) and wait in
// griddepcontrol.wait for its completion and memory
int launch_combine(const DecodeParams& p, int R, cudaStream_t st) {
  const int rows = p.B * p.Hkv * R;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((rows + 3) / 4);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = NT_DECODE_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int rc = check_cuda(cudaLaunchKernelEx(&cfg, decode_combine_kernel, p, R), "decode_combine launch");
  g_launches++;
  return rc;
}

template <int R, int PG>
int launch(const CUtensorMap& mk, const CUtensorMap& mv, DecodeParams& p, cudaStream_t st) {
  int rc;
  constexpr auto kern = decode_split_kernel<R, PG>;
  if ((rc = configure_smem<kern>(kDecodeSmem, "cudaFuncSetAttribute(decode)"))) return rc;
  dim3 grid(p.splits, p.B * p.Hkv);
  kern<<<grid, kDecodeCTAThreads, kDecodeSmem, st>>>(mk, mv, p);
  g_launches++;
  if ((rc = check_cuda(cudaGetLastError(), "decode_split launch"))) return rc;
  return launch_combine(p, R, st);
}
template <int PG>
int dispatch(int R, const CUtensorMap& mk, const CUtensorMap& mv, DecodeParams& p, cudaStream_t st) {
  switch (R) {
    case 1: return launch<1, PG>(mk, mv, p, st);
    case 2: return launch<2, PG>(mk, mv, p, st);
    case 4: return launch<4, PG>(mk, mv, p, st);
    default: return launch<8, PG>(mk, mv, p, st);
  }
}
// K2b (tensor-core dots) for dense K/V; NT_DECODE_FMA=1 keeps K2 (A/B experiments)
bool use_tc_decode() {
  static const bool fma = getenv("NT_DECODE_FMA") && atoi(getenv("NT_DECODE_FMA")) != 0;
  return !fma;
}

template <int R, int PG, bool FP8>
int launch_tc(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv, DecodeParams& p, cudaStream_t st) {
  int rc;
  constexpr auto kern = decode_tc_kernel<R, PG, FP8>;
  constexpr int smem = DtcCfg<FP8, PG>::SMEM;
  if ((rc = configure_smem<kern>(smem, "cudaFuncSetAttribute(decode_tc)"))) return rc;
  dim3 grid(p.splits, p.B * p.Hkv);
  kern<<<grid, kDtcThreads, smem, st>>>(mq, mk, mv, p);
  g_launches++;
  if ((rc = check_cuda(cudaGetLastError(), "decode_tc launch"))) return rc;
  return launch_combine(p, R, st);
}

template <int PG, bool FP8 = false>
int dispatch_tc(int R, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv, DecodeParams& p,
                cudaStream_t st) {
  switch (R) {
    case 1: return launch_tc<1, PG, FP8>(mq, mk, mv, p, st);
    case 2: return launch_tc<2, PG, FP8>(mq, mk, mv, p, st);
    case 4: return launch_tc<4, PG, FP8>(mq, mk, mv, p, st);
    default: return launch_tc<8, PG, FP8>(mq, mk, mv, p, st);
  }
}

// the group's rows as one box {64 bf16 | 128 e4m3 dims, Nq, g, 1} (one 128-byte panel)
int make_q_map(CUtensorMap* mq, const nt_tensor4& q, int B, int Hq, int Nq, int g, size_t elem = 2) {
  const int64_t qd[4] = {kDecodeD, Nq, Hq, B};
  const int64_t qs[3] = {q.stride_s, q.stride_h, q.stride_b};
  const int qb[4] = {(int)(128 / elem), Nq, g, 1};
  return make_map_4d_box(mq, q.ptr, qd, qs, qb, elem);
}
}  // namespace

#ifdef NT_TRACE
namespace nt {
// debug builds: this TU's copy of the trace symbols (attn_fwd.cuh) for the K2b timeline
void trace_set_decode(unsigned long long* buf, int cta) {
  cudaMemcpyToSymbol(g_nt_trace, &buf, sizeof(buf));
  cudaMemcpyToSymbol(g_nt_trace_cta, &cta, sizeof(cta));
}
}  // namespace nt
#endif

extern "C" int64_t nt_decode_workspace_bytes(int32_t batch, int32_t heads_kv, int32_t rows_per_group,
                                             int32_t head_dim, int32_t num_splits) {
  return (int64_t)batch * heads_kv * num_splits * rows_per_group * (head_dim + 2) * (int64_t)sizeof(float);
}

extern "C" int nt_attn_decode(const nt_decode_args* a, void* stream) {
  if (!a) return set_error(NT_ERR_INVALID, "null args");
  if (a->head_dim != kDecodeD) return set_error(NT_ERR_UNSUPPORTED, "decode kernel is built for head_dim 128");
  if (a->heads_q % a->heads_kv) return set_error(NT_ERR_INVALID, "heads_q must be a multiple of heads_kv");
  const int g = a->heads_q / a->heads_kv;
  const int R = g * a->seq_q;
  if (R != 1 && R != 2 && R != 4 && R != 8)
    return set_error(NT_ERR_UNSUPPORTED, "decode kernel packs 1, 2, 4 or 8 query rows per kv group");
  if (!a->workspace || a->workspace_bytes < nt_decode_workspace_bytes(a->batch, a->heads_kv, R, a->head_dim,
                                                                      std::max(1, a->num_splits)))
    return set_error(NT_ERR_INVALID, "workspace missing or smaller than nt_decode_workspace_bytes(...)");
  const bool fp8 = a->in_dtype == NT_DTYPE_E4M3;
  if (a->in_dtype != NT_DTYPE_BF16 && !fp8) return set_error(NT_ERR_INVALID, "in_dtype must be bf16 or e4m3");
  if (fp8 && !use_tc_decode()) return set_error(NT_ERR_UNSUPPORTED, "e4m3 decode runs on the tensor-core kernel only");
  const int align = fp8 ? 16 : 8;  // strides in elements: 16 bytes either way
  for (const nt_tensor4* t : {&a->q, &a->k, &a->v})
    if (reinterpret_cast<uintptr_t>(t->ptr) % 16 || t->stride_s % align || t->stride_h % align ||
        t->stride_b % align)
      return set_error(NT_ERR_INVALID, "q/k/v must be 16-byte aligned with 16-byte strides");
  DecodeParams p{};
  p.q = static_cast<const __nv_bfloat16*>(a->q.ptr);
  p.q_sb = a->q.stride_b; p.q_sh = a->q.stride_h; p.q_sn = a->q.stride_s;
  p.k = static_cast<const __nv_bfloat16*>(a->k.ptr);
  p.k_sb = a->k.stride_b; p.k_sh = a->k.stride_h; p.k_sn = a->k.stride_s;
  p.v = static_cast<const __nv_bfloat16*>(a->v.ptr);
  p.v_sb = a->v.stride_b; p.v_sh = a->v.stride_h; p.v_sn = a->v.stride_s;
  p.o = a->o.ptr;
  p.o_sb = a->o.stride_b; p.o_sh = a->o.stride_h; p.o_sn = a->o.stride_s;
  p.out_f32 = a->out_dtype == NT_DTYPE_F32;
  p.B = a->batch; p.Hq = a->heads_q; p.Hkv = a->heads_kv; p.Nq = a->seq_q; p.M = a->seq_kv; p.g = g;
  auto ds = [](float d) { return d == 0.f ? 1.f : d; };
  p.scale_log2 = a->scale * 1.4426950408889634f * (fp8 ? ds(a->q_descale) * ds(a->k_descale) : 1.f);
  p.o_scale = fp8 ? ds(a->v_descale) : 1.f;
  p.splits = std::max(1, a->num_splits);
  // key ranges are whole 64-key TMA tiles
  p.keys_per_split = ((a->seq_kv + p.splits - 1) / p.splits + kDecodeTile - 1) / kDecodeTile * kDecodeTile;
  p.ws = static_cast<float*>(a->workspace);
  p.err = a->err_flag;
  p.seq_lens = nullptr;
  p.block_table = nullptr;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUtensorMap mk, mv;
  int rc;
  if (use_tc_decode()) {
    // K2b: 128-key tiles; the group's R query rows as one 4-D box {64, Nq, g, 1}
    p.keys_per_split = ((a->seq_kv + p.splits - 1) / p.splits + kDtcTile - 1) / kDtcTile * kDtcTile;
    CUtensorMap mq;
    if ((rc = make_q_map(&mq, a->q, a->batch, a->heads_q, a->seq_q, g, fp8 ? 1 : 2))) return rc;
    if (fp8) {  // one 128-byte panel per key: box {128 dims, KPS keys, 1, 1}
      constexpr int kps = DtcCfg<true, 0>::KPS;
      p.keys_per_split = ((a->seq_kv + p.splits - 1) / p.splits + kps - 1) / kps * kps;
      if ((rc = make_map_4d(&mk, a->k.ptr, kDecodeD, a->seq_kv, a->heads_kv, a->batch, a->k.stride_s, a->k.stride_h,
                            a->k.stride_b, kps, 1, 0, CU_TENSOR_MAP_SWIZZLE_128B)))
        return rc;
      if ((rc = make_map_4d(&mv, a->v.ptr, kDecodeD, a->seq_kv, a->heads_kv, a->batch, a->v.stride_s, a->v.stride_h,
                            a->v.stride_b, kps, 1, 0, CU_TENSOR_MAP_SWIZZLE_128B)))
        return rc;
      return dispatch_tc<0, true>(R, mq, mk, mv, p, st);
    }
    if ((rc = make_map_pages_5d(&mk, a->k.ptr, a->seq_kv, a->heads_kv, a->batch, a->k.stride_s, a->k.stride_h,
                                a->k.stride_b, kDtcTile)))
      return rc;
    if ((rc = make_map_pages_5d(&mv, a->v.ptr, a->seq_kv, a->heads_kv, a->batch, a->v.stride_s, a->v.stride_h,
                                a->v.stride_b, kDtcTile)))
      return rc;
    return dispatch_tc<0>(R, mq, mk, mv, p, st);
  }
  // one 5-D box {64 dims, 64 keys, 2 panels} per K or V tile (a batch entry is a "page"
  // of seq_kv tokens): both 64-dim panels in one TMA, laid out [panel][64 keys][128 B]
  if ((rc = make_map_pages_5d(&mk, a->k.ptr, a->seq_kv, a->heads_kv, a->batch, a->k.stride_s, a->k.stride_h,
                              a->k.stride_b, kDecodeTile)))
    return rc;
  if ((rc = make_map_pages_5d(&mv, a->v.ptr, a->seq_kv, a->heads_kv, a->batch, a->v.stride_s, a->v.stride_h,
                              a->v.stride_b, kDecodeTile)))
    return rc;
  return dispatch<0>(R, mk, mv, p, st);
}

extern "C" int nt_attn_decode_paged(const nt_decode_paged_args* a, void* stream) {
  if (!a) return set_error(NT_ERR_INVALID, "null args");
  if (a->head_dim != kDecodeD) return set_error(NT_ERR_UNSUPPORTED, "decode kernel is built for head_dim 128");
  if (a->heads_q % a->heads_kv) return set_error(NT_ERR_INVALID, "heads_q must be a multiple of heads_kv");
  const int g = a->heads_q / a->heads_kv;
  const int R = g * a->seq_q;
  if (R != 1 && R != 2 && R != 4 && R != 8)
    return set_error(NT_ERR_UNSUPPORTED, "decode kernel packs 1, 2, 4 or 8 query rows per kv group");
  const int ps = a->page_size;
  if (ps <= 0 || ps % 8 || (ps < kDecodeTile && kDecodeTile % ps) || (ps > kDecodeTile && ps % kDecodeTile))
    return set_error(NT_ERR_UNSUPPORTED, "page_size must be 8, 16, 32, 64 or a multiple of 64");
  if (!a->workspace || !a->block_table || !a->seq_lens) return set_error(NT_ERR_INVALID, "workspace, block_table and seq_lens required");
  if (a->workspace_bytes < nt_decode_workspace_bytes(a->batch, a->heads_kv, R, a->head_dim, std::max(1, a->num_splits)))
    return set_error(NT_ERR_INVALID, "workspace smaller than nt_decode_workspace_bytes(...)");
  if (a->max_seq_kv <= 0 || a->num_pages <= 0) return set_error(NT_ERR_INVALID, "empty cache");
  const bool fp8 = a->in_dtype == NT_DTYPE_E4M3;
  if (a->in_dtype != NT_DTYPE_BF16 && !fp8) return set_error(NT_ERR_INVALID, "in_dtype must be bf16 or e4m3");
  if (fp8 && (!use_tc_decode() || (kDtcTile % ps && ps % kDtcTile)))
    return set_error(NT_ERR_UNSUPPORTED, "e4m3 paged decode: tensor-core kernel, page_size dividing or a multiple of 128");
  const int align = fp8 ? 16 : 8;  // element strides of 16 bytes
  if (reinterpret_cast<uintptr_t>(a->q.ptr) % 16 || a->q.stride_s % align || a->q.stride_h % align ||
      a->q.stride_b % align)
    return set_error(NT_ERR_INVALID, "q must be 16-byte aligned with 16-byte strides");
  DecodeParams p{};
  p.q = static_cast<const __nv_bfloat16*>(a->q.ptr);
  p.q_sb = a->q.stride_b; p.q_sh = a->q.stride_h; p.q_sn = a->q.stride_s;
  p.o = a->o.ptr;
  p.o_sb = a->o.stride_b; p.o_sh = a->o.stride_h; p.o_sn = a->o.stride_s;
  p.out_f32 = a->out_dtype == NT_DTYPE_F32;
  p.B = a->batch; p.Hq = a->heads_q; p.Hkv = a->heads_kv; p.Nq = a->seq_q; p.M = a->max_seq_kv; p.g = g;
  auto ds = [](float d) { return d == 0.f ? 1.f : d; };
  p.scale_log2 = a->scale * 1.4426950408889634f * (fp8 ? ds(a->q_descale) * ds(a->k_descale) : 1.f);
  p.o_scale = fp8 ? ds(a->v_descale) : 1.f;
  p.splits = std::max(1, a->num_splits);
  p.keys_per_split = ((a->max_seq_kv + p.splits - 1) / p.splits + kDecodeTile - 1) / kDecodeTile * kDecodeTile;
  p.ws = static_cast<float*>(a->workspace);
  p.err = a->err_flag;
  p.block_table = a->block_table;
  p.bt_stride = a->block_table_stride;
  p.page_size = ps;
  p.seq_lens = a->seq_lens;
  CUtensorMap mk, mv;
  int rc;
  if (use_tc_decode() && (kDtcTile % ps == 0 || ps % kDtcTile == 0)) {
    // K2b over the page pool: 128-key tiles gathered page slice by page slice
    p.keys_per_split = ((a->max_seq_kv + p.splits - 1) / p.splits + kDtcTile - 1) / kDtcTile * kDtcTile;
    CUtensorMap mq;
    if ((rc = make_q_map(&mq, a->q, a->batch, a->heads_q, a->seq_q, g, fp8 ? 1 : 2))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (fp8) {  // one 128-byte panel per token: box {128 dims, min(page, 128) tokens}
      const int rows = std::min(ps, kDtcTile);
      if ((rc = make_map_4d(&mk, a->k_pages, kDecodeD, ps, a->heads_kv, a->num_pages, a->token_stride,
                            a->head_stride, a->page_stride, rows, 1, 0, CU_TENSOR_MAP_SWIZZLE_128B)))
        return rc;
      if ((rc = make_map_4d(&mv, a->v_pages, kDecodeD, ps, a->heads_kv, a->num_pages, a->token_stride,
                            a->head_stride, a->page_stride, rows, 1, 0, CU_TENSOR_MAP_SWIZZLE_128B)))
        return rc;
      return ps % kDtcTile == 0 ? dispatch_tc<1, true>(R, mq, mk, mv, p, st) : dispatch_tc<2, true>(R, mq, mk, mv, p, st);
    }
    if (ps % kDtcTile == 0) {
      if ((rc = make_map_pages_5d(&mk, a->k_pages, ps, a->heads_kv, a->num_pages, a->token_stride, a->head_stride,
                                  a->page_stride, kDtcTile)))
        return rc;
      if ((rc = make_map_pages_5d(&mv, a->v_pages, ps, a->heads_kv, a->num_pages, a->token_stride, a->head_stride,
                                  a->page_stride, kDtcTile)))
        return rc;
      return dispatch_tc<1>(R, mq, mk, mv, p, st);
    }
    if ((rc = make_map_4d(&mk, a->k_pages, kDecodeD, ps, a->heads_kv, a->num_pages, a->token_stride, a->head_stride,
                          a->page_stride, ps, 2)))
      return rc;
    if ((rc = make_map_4d(&mv, a->v_pages, kDecodeD, ps, a->heads_kv, a->num_pages, a->token_stride, a->head_stride,
                          a->page_stride, ps, 2)))
      return rc;
    return dispatch_tc<2>(R, mq, mk, mv, p, st);
  }
  const int rows = std::min(ps, kDecodeTile);
  if (rows < kDecodeTile) {  // small pages: one 5-D box per page slice (both 64-dim panels)
    if ((rc = make_map_pages_5d(&mk, a->k_pages, ps, a->heads_kv, a->num_pages, a->token_stride, a->head_stride,
                                a->page_stride, rows)))
      return rc;
    if ((rc = make_map_pages_5d(&mv, a->v_pages, ps, a->heads_kv, a->num_pages, a->token_stride, a->head_stride,
                                a->page_stride, rows)))
      return rc;
  } else {
    if ((rc = make_map_4d(&mk, a->k_pages, kDecodeD, ps, a->heads_kv, a->num_pages, a->token_stride,
                          a->head_stride, a->page_stride, rows, 2)))
      return rc;
    if ((rc = make_map_4d(&mv, a->v_pages, kDecodeD, ps, a->heads_kv, a->num_pages, a->token_stride,
                          a->head_stride, a->page_stride, rows, 2)))
      return rc;
  }
  return rows < kDecodeTile ? dispatch<2>(R, mk, mv, p, static_cast<cudaStream_t>(stream))
                            : dispatch<1>(R, mk, mv, p, static_cast<cudaStream_t>(stream));
}

extern "C" int nt_decode_num_splits(int32_t batch, int32_t heads_kv, int32_t seq_kv, int32_t requested) {
  return choose_splits(batch * heads_kv, seq_kv, requested);
}
