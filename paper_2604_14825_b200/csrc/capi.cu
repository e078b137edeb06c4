// C ABI entry points (include/nautilus_b200.h): argument validation, TMA
// descriptor encoding, launch configuration.  Kernels live in *.cuh.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <queue>
#include <vector>
#include <string>

#include "../../include/nautilus_b200.h"
#include "attn_launch.cuh"
#include "common_host.h"

namespace nt {

thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};
// nt_attn_prepare: run the whole launch path (validation, tensor maps, split plan,
// kernel selection, per-device smem attribute -- which also loads the lazily
// loaded kernel image) but stop before the launch
thread_local bool g_prepare_only = false;
thread_local int g_prepared_ctas_per_sm = 0;
thread_local AttnLaunchFn g_prepared_fn = nullptr;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return set_error(NT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return NT_OK;
}

int num_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// rank-4 map over [B, H, S, D] (dims innermost-first), box {box_inner (default one
// 128-byte row), box_rows, 1, 1}, 128B swizzle unless given
int make_map_4d(CUtensorMap* m, const void* ptr, int64_t D, int64_t S, int64_t H, int64_t B, int64_t sS,
                int64_t sH, int64_t sB, int box_rows, size_t elem, int box_inner, CUtensorMapSwizzle swz) {
  EncodeFn enc = get_encode();
  if (!enc) return set_error(NT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (reinterpret_cast<uintptr_t>(ptr) % 16) return set_error(NT_ERR_INVALID, "tensor base not 16B aligned");
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)S, (cuuint64_t)H, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)(sS * elem), (cuuint64_t)(sH * elem), (cuuint64_t)(sB * elem)};
  for (int i = 0; i < 3; ++i) {
    if (strides[i] % 16) return set_error(NT_ERR_INVALID, "tensor strides must be multiples of 16 bytes");
    if (strides[i] == 0) strides[i] = 16;  // broadcast dims of extent 1
  }
  cuuint32_t box[4] = {(cuuint32_t)(box_inner ? box_inner : 128 / elem), (cuuint32_t)box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUtensorMapDataType dt = elem == 1   ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : elem == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUresult r = enc(m, dt, 4,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(NT_ERR_INVALID, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return NT_OK;
}

// rank-4 map with an explicit box (dims innermost first, strides in elements for dims 1-3)
int make_map_4d_box(CUtensorMap* m, const void* ptr, const int64_t dims[4], const int64_t strides[3],
                    const int box[4], size_t elem) {
  EncodeFn enc = get_encode();
  if (!enc) return set_error(NT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (reinterpret_cast<uintptr_t>(ptr) % 16) return set_error(NT_ERR_INVALID, "tensor base not 16B aligned");
  cuuint64_t d[4], st[3];
  cuuint32_t bx[4], estr[4] = {1, 1, 1, 1};
  for (int i = 0; i < 4; ++i) {
    d[i] = (cuuint64_t)dims[i];
    bx[i] = (cuuint32_t)box[i];
  }
  for (int i = 0; i < 3; ++i) {
    st[i] = (cuuint64_t)(strides[i] * elem);
    if (st[i] % 16) return set_error(NT_ERR_INVALID, "tensor strides must be multiples of 16 bytes");
    if (st[i] == 0) st[i] = 16;
  }
  const CUtensorMapDataType dt = elem == 1   ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : elem == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUresult r = enc(m, dt, 4, const_cast<void*>(ptr), d, st, bx, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(NT_ERR_INVALID, "cuTensorMapEncodeTiled(4d box) failed (" + std::to_string((int)r) + ")");
  return NT_OK;
}

int make_map_2d(CUtensorMap* m, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_inner,
                int box_outer, size_t elem, CUtensorMapSwizzle swz) {
  EncodeFn enc = get_encode();
  if (!enc) return set_error(NT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (reinterpret_cast<uintptr_t>(ptr) % 16) return set_error(NT_ERR_INVALID, "matrix base not 16B aligned");
  if ((ld * elem) % 16) return set_error(NT_ERR_INVALID, "leading dimension must be a multiple of 16 bytes");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * elem)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, elem == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(NT_ERR_INVALID, "cuTensorMapEncodeTiled(2d) failed (" + std::to_string((int)r) + ")");
  return NT_OK;
}

// bf16 page pool viewed as 5-D (d_lo 64, token, d_hi 2, head, page): one box
// {64, rows, 2, 1, 1} brings both 64-dim panels of `rows` tokens of one page
int make_map_pages_5d(CUtensorMap* m, const void* ptr, int64_t page_size, int64_t heads, int64_t pages,
                      int64_t token_stride, int64_t head_stride, int64_t page_stride, int rows) {
  EncodeFn enc = get_encode();
  if (!enc) return set_error(NT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (reinterpret_cast<uintptr_t>(ptr) % 16) return set_error(NT_ERR_INVALID, "page pool base not 16B aligned");
  cuuint64_t dims[5] = {64, (cuuint64_t)page_size, 2, (cuuint64_t)heads, (cuuint64_t)pages};
  cuuint64_t strides[4] = {(cuuint64_t)(token_stride * 2), 128, (cuuint64_t)(head_stride * 2),
                           (cuuint64_t)(page_stride * 2)};
  for (int i = 0; i < 4; ++i)
    if (strides[i] % 16) return set_error(NT_ERR_INVALID, "page pool strides must be multiples of 16 bytes");
  cuuint32_t box[5] = {64, (cuuint32_t)rows, 2, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(NT_ERR_INVALID, "cuTensorMapEncodeTiled(pages 5d) failed (" + std::to_string((int)r) + ")");
  return NT_OK;
}

// ----------------------------------------------------------------- attention
// Split-KV plan (host restatement of attn_unit's prefix): kv_split = 0 unless the
// heaviest item exceeds 2x the per-SM average of KV-tile steps (few, long items:
// one kv-group per GPU at 8 GPUs); then items are cut into ~1.1 x avg-tile units.
// Measured (tools/split_probe.py, Llama 8K causal): Hq=4 131 -> 101 us; Hq=8
// (1.1x) 135 -> 153-185 us -- each unit reloads Q, stores an fp32 partial and
// refills the pipeline, so splitting only pays when the heaviest item dominates.
struct AttnSplit {
  int kv_split = 0, n_units = 0;
  int n_split_mb = 0;  // m-block positions (LPT order: heaviest first) whose items are split
  int64_t bytes = 0, off_ml = 0, off_o = 0;
};
// Query rows per work item: 256 (two 128-row tiles, one CTA per SM) or 128 (one
// tile, two CTAs per SM -- the NQ = 1 instantiations; bf16 Q/K/V only).
// args->item_rows 0 = library choice.
// Library choice: 128-row items when 256-row items would leave more than half
// of the SMs idle (e.g. config 1, one 256-row item: 2 CTAs instead of 1,
// 15.9 -> 13.9 us), and at head_dim 64 with short KV ranges (<= 1024 keys: items of
// <= 8 tiles, whose boundaries two co-resident CTAs hide better -- BERT-base 54.0 ->
// 52.5 us, same box, 3 x 2 runs); otherwise 256 (two tiles share each K/V tile).
static int attn_item_rows(const nt_attn_args* a) {
  if (a->in_dtype == NT_DTYPE_E4M3) return 256;
  if (a->item_rows == 128 || a->item_rows == 256) return a->item_rows;
  if (a->head_dim == 64 && a->seq_kv <= 1024) return 128;
  const long long items256 = (long long)((a->seq_q + 255) / 256) * a->batch * a->heads_q;
  return items256 * 2 < num_sms() ? 128 : 256;
}

static AttnSplit attn_split_plan(const nt_attn_args* a) {
  AttnSplit sp;
  const int rows = attn_item_rows(a);
  const int nmb = (a->seq_q + rows - 1) / rows, nkv_total = (a->seq_kv + 127) / 128;
  const long long BH = (long long)a->batch * a->heads_q;
  sp.n_units = (int)(nmb * BH);
  if (nmb > kMaxSplitMblocks || a->mask_kind == NT_MASK_TENSOR || a->mask_kind == NT_MASK_BITS) return sp;
  auto nkv = [&](int mb) {
    if (a->mask_kind != NT_MASK_CAUSAL) return nkv_total;
    const int last_q = std::min(mb * rows + rows - 1, a->seq_q - 1) + a->causal_offset;
    return std::max(std::min(nkv_total, last_q / 128 + 1), 1);
  };
  long long total = 0;
  int mx = 0;
  for (int mb = 0; mb < nmb; ++mb) {
    total += nkv(mb) * BH;
    mx = std::max(mx, nkv(mb));
  }
  // per resident CTA: one per SM with 256-row items, two with 128-row items
  const double avg = (double)total / (num_sms() * (rows == 128 ? 2 : 1));
  // experiment overrides: NT_ATTN_SPLIT_THRESH (x avg), NT_ATTN_SPLIT_DIV (avg / div tiles per unit)
  static const double thresh = getenv("NT_ATTN_SPLIT_THRESH") ? atof(getenv("NT_ATTN_SPLIT_THRESH")) : 2.0;
  // div 0.9 (units of ~1.1x the per-CTA average) measured best for one kv-group of
  // Llama 8K causal (r02 sweep, main kernel + merge): div 3 102.8 us, 1.5 106.8,
  // 1.2 108.0, 1.0 93.4, 0.9 88.3, 0.75 100.6, 0.6 116.1 -- fewer, longer units
  // write fewer fp32 partials and the merge reads fewer (10 vs 18 us)
  static const double div = getenv("NT_ATTN_SPLIT_DIV") ? atof(getenv("NT_ATTN_SPLIT_DIV")) : 0.9;
  if (mx <= thresh * avg) return sp;
  // >= 4 tiles per unit; <= 32 units per item (the combine holds one chunk per lane)
  const int s_min = std::max(4, (mx + 31) / 32);
  int S = std::max((int)std::ceil(avg / div), s_min);
  if (!getenv("NT_ATTN_SPLIT_DIV")) {
    // pick the chunk size whose greedy schedule (the device work counter hands the
    // units out in LPT order to whichever CTA frees first) has the shortest makespan,
    // each unit charged one extra step for its Q load, partial store and refill:
    // one kv-group of Llama 8K, 148 CTAs -- S = 32 (the 0.9 rule) 33 steps, S = 30 32
    const int ctas = num_sms() * (rows == 128 ? 2 : 1);
    auto makespan = [&](int s) {
      std::priority_queue<double, std::vector<double>, std::greater<double>> free_at;
      for (int c = 0; c < ctas; ++c) free_at.push(0.0);
      double end = 0.0;
      for (int i = 0; i < nmb; ++i) {
        const int n = nkv(a->mask_kind == NT_MASK_CAUSAL ? nmb - 1 - i : i);
        const int nc = n > s ? (n + s - 1) / s : 1;
        for (int c = 0; c < nc; ++c)
          for (long long bh = 0; bh < BH; ++bh) {
            const double t = free_at.top() + std::min(s, n - c * s) + 1.0;
            free_at.pop();
            free_at.push(t);
            end = std::max(end, t);
          }
      }
      return end;
    };
    double best = 1e30;
    for (int s = std::max(s_min, (int)(0.8 * avg)); s <= std::max(s_min, (int)std::ceil(1.3 * avg)); ++s) {
      const double m = makespan(s);
      if (m < best - 1e-9) {
        best = m;
        S = s;
      }
    }
  }
  if (S >= mx) return sp;
  long long units = 0;
  for (int mb = 0; mb < nmb; ++mb) {
    units += (nkv(mb) + S - 1) / S * BH;
    sp.n_split_mb += nkv(mb) > S;
  }
  sp.kv_split = S;
  sp.n_units = (int)units;
  const int64_t prefix_bytes = ((int64_t)(nmb + 1) * 4 + 255) / 256 * 256;
  sp.off_ml = prefix_bytes;
  sp.off_o = sp.off_ml + ((int64_t)units * rows * 8 + 255) / 256 * 256;
  sp.bytes = sp.off_o + (int64_t)units * rows * a->head_dim * 2;  // bf16 partials
  return sp;
}

}  // namespace nt

using namespace nt;

extern "C" int64_t nt_attn_workspace_bytes(const nt_attn_args* a) {
  if (!a || a->seq_q <= 0 || a->seq_kv <= 0 || a->batch <= 0 || a->heads_q <= 0) return 0;
  return attn_split_plan(a).bytes;
}

extern "C" int nt_attn_fwd(const nt_attn_args* a, void* stream);

extern "C" int nt_attn_prepare(const nt_attn_args* a) {
  g_prepare_only = true;
  g_prepared_ctas_per_sm = 0;
  const int rc = nt_attn_fwd(a, nullptr);
  g_prepare_only = false;
  return rc;
}

extern "C" int nt_attn_resident_ctas(const nt_attn_args* a) {
  const int rc = nt_attn_prepare(a);
  return rc ? -rc : g_prepared_ctas_per_sm;
}

// Validation, tensor maps, split plan and kernel parameters of one launch.
static int attn_build(const nt_attn_args* a, AttnMaps& m, AttnFwdParams& p, int& nq_out) {
  if (!a) return set_error(NT_ERR_INVALID, "null args");
  if (a->head_dim != 64 && a->head_dim != 128)
    return set_error(NT_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  if (a->batch <= 0 || a->heads_q <= 0 || a->heads_kv <= 0 || a->seq_q <= 0 || a->seq_kv <= 0)
    return set_error(NT_ERR_INVALID, "non-positive extent");
  if (a->heads_q % a->heads_kv) return set_error(NT_ERR_INVALID, "heads_q must be a multiple of heads_kv");
  if (!(a->scale > 0.f)) return set_error(NT_ERR_UNSUPPORTED, "scale must be positive");
  if (a->mask_kind < NT_MASK_NONE || a->mask_kind > NT_MASK_BITS) return set_error(NT_ERR_INVALID, "unknown mask_kind");
  if (a->mask_kind == NT_MASK_TENSOR && !a->mask) return set_error(NT_ERR_INVALID, "tensor mask missing");
  if (a->mask_kind == NT_MASK_BITS) {
    if (!a->mask || reinterpret_cast<uintptr_t>(a->mask) % 16 || a->mask_stride_row % 4 ||
        a->mask_stride_row < (int64_t)((a->seq_kv + 127) / 128) * 4)
      return set_error(NT_ERR_INVALID, "bit mask: 16-byte aligned rows of >= ceil(seq_kv / 128) * 4 words");
  }
  const bool e4m3 = a->in_dtype == NT_DTYPE_E4M3;
  if (a->in_dtype != NT_DTYPE_BF16 && !e4m3) return set_error(NT_ERR_UNSUPPORTED, "q/k/v must be bf16 or e4m3");
  if (a->item_rows != 0 && a->item_rows != 128 && a->item_rows != 256)
    return set_error(NT_ERR_INVALID, "item_rows must be 0, 128 or 256");
  if (e4m3 && a->item_rows == 128) return set_error(NT_ERR_UNSUPPORTED, "e4m3 attention: 256-row items only");
  const int rows = attn_item_rows(a);
  const int nq = rows / 128;
  if (e4m3 && (a->head_dim != 128 || a->mask_kind == NT_MASK_TENSOR || a->mask_kind == NT_MASK_BITS))
    return set_error(NT_ERR_UNSUPPORTED, "e4m3 attention: head_dim 128, no or causal mask");
  const int D = a->head_dim;
  const size_t in_elem = e4m3 ? 1 : 2;
  m = AttnMaps{};
  CUtensorMap &mq = m.q, &mk = m.k, &mv = m.v, &mo = m.o;
  int rc;
  if ((rc = make_map_4d(&mq, a->q.ptr, D, a->seq_q, a->heads_q, a->batch, a->q.stride_s, a->q.stride_h,
                        a->q.stride_b, 128, in_elem)))
    return rc;
  if ((rc = make_map_4d(&mk, a->k.ptr, D, a->seq_kv, a->heads_kv, a->batch, a->k.stride_s, a->k.stride_h,
                        a->k.stride_b, 128, in_elem)))
    return rc;
  if ((rc = make_map_4d(&mv, a->v.ptr, D, a->seq_kv, a->heads_kv, a->batch, a->v.stride_s, a->v.stride_h,
                        a->v.stride_b, 128, in_elem)))
    return rc;
  // the epilogue writes O by TMA: 32-row x 32-column boxes, swizzled to match
  // the row-per-lane staging writes
  const bool f32 = a->out_dtype == NT_DTYPE_F32;
  if (reinterpret_cast<uintptr_t>(a->o.ptr) % 16 || (a->o.stride_s * (f32 ? 4 : 2)) % 16 ||
      (a->o.stride_h * (f32 ? 4 : 2)) % 16 || (a->o.stride_b * (f32 ? 4 : 2)) % 16)
    return set_error(NT_ERR_INVALID, "output must be 16B aligned with 16B-multiple strides");
  // fp32 boxes: 32 columns (SWIZZLE_128B), or 16 (SWIZZLE_64B) for 128-row items (AttnCfg::F32_BOX_COLS)
  const int f32_cols = nq == 1 ? 16 : 32;
  if ((rc = make_map_4d(&mo, a->o.ptr, D, a->seq_q, a->heads_q, a->batch, a->o.stride_s, a->o.stride_h,
                        a->o.stride_b, 32, f32 ? 4 : 2, f32 ? f32_cols : 32,
                        (f32 && f32_cols == 32) ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B)))
    return rc;
  p = AttnFwdParams{};
  p.B = a->batch;
  p.Hq = a->heads_q;
  p.Hkv = a->heads_kv;
  p.N = a->seq_q;
  p.M = a->seq_kv;
  p.q_per_kv = a->heads_q / a->heads_kv;
  p.n_mblocks = (a->seq_q + rows - 1) / rows;
  p.n_kv_total = (a->seq_kv + 127) / 128;
  p.n_items = p.n_mblocks * a->batch * a->heads_q;
  p.causal_offset = a->causal_offset;
  // e4m3: S = (Q.K^T) q_descale k_descale, O = v_descale P.V / l (a descale of 0 reads as 1)
  const float qd = (e4m3 && a->q_descale != 0.f) ? a->q_descale : 1.f;
  const float kd = (e4m3 && a->k_descale != 0.f) ? a->k_descale : 1.f;
  p.scale_log2 = a->scale * qd * kd * 1.4426950408889634f;
  p.o_scale = (e4m3 && a->v_descale != 0.f) ? a->v_descale : 1.f;
  p.mask = a->mask;
  p.mask_row_stride = a->mask_stride_row;
  p.o = a->o.ptr;
  p.o_sb = a->o.stride_b;
  p.o_sh = a->o.stride_h;
  p.o_sn = a->o.stride_s;
  p.err = a->err_flag;
  p.work = a->work_counter;
  // split KV when the caller provided the workspace nt_attn_workspace_bytes asks for
  const AttnSplit sp = attn_split_plan(a);
  if (sp.kv_split > 0 && a->workspace && a->workspace_bytes >= sp.bytes) {
    char* ws = static_cast<char*>(a->workspace);
    p.kv_split = sp.kv_split;
    p.n_items = sp.n_units;
    p.n_split_mb = sp.n_split_mb;
    p.unit_prefix = reinterpret_cast<int*>(ws);
    p.part_ml = reinterpret_cast<float2*>(ws + sp.off_ml);
    m.part_o = reinterpret_cast<const __nv_bfloat16*>(ws + sp.off_o);
    if ((rc = make_map_2d(&m.p, m.part_o, D, (int64_t)sp.n_units * rows, D, 32, 32, 2, CU_TENSOR_MAP_SWIZZLE_64B)))
      return rc;
  } else {
    m.p = m.o;  // unused (no split)
  }
  nq_out = nq;
  return NT_OK;
}

static int attn_dispatch(const nt_attn_args* a, const AttnMaps& m, const AttnFwdParams& p, int nq, cudaStream_t st) {
  if (a->in_dtype == NT_DTYPE_E4M3) return dispatch_attn_e4m3(a, m, p, st);
  return a->head_dim == 64 ? dispatch_attn_d64(a, m, p, nq, st) : dispatch_attn_d128(a, m, p, nq, st);
}

extern "C" int nt_attn_fwd(const nt_attn_args* a, void* stream) {
  AttnMaps m;
  AttnFwdParams p;
  int nq = 2;
  if (const int rc = attn_build(a, m, p, nq)) return rc;
  return attn_dispatch(a, m, p, nq, static_cast<cudaStream_t>(stream));
}

// ----------------------------------------------------------------- attention plans
struct nt_attn_plan {
  AttnMaps maps;
  AttnFwdParams params;
  AttnLaunchFn fn;
  int device;
};

extern "C" int nt_attn_plan_create(const nt_attn_args* a, nt_attn_plan** out) {
  if (!out) return set_error(NT_ERR_INVALID, "null plan pointer");
  *out = nullptr;
  auto* pl = new nt_attn_plan{};
  int nq = 2;
  int rc = attn_build(a, pl->maps, pl->params, nq);
  if (!rc) {
    g_prepare_only = true;
    g_prepared_fn = nullptr;
    rc = attn_dispatch(a, pl->maps, pl->params, nq, nullptr);
    g_prepare_only = false;
    pl->fn = g_prepared_fn;
    if (!rc && !pl->fn) rc = set_error(NT_ERR_UNSUPPORTED, "no launcher selected");
  }
  if (rc) {
    delete pl;
    return rc;
  }
  cudaGetDevice(&pl->device);
  *out = pl;
  return NT_OK;
}

extern "C" int nt_attn_plan_launch(const nt_attn_plan* pl, void* stream) {
  if (!pl) return set_error(NT_ERR_INVALID, "null plan");
  int dev = -1;
  if (cudaGetDevice(&dev) == cudaSuccess && dev != pl->device)
    return set_error(NT_ERR_INVALID, "attention plan created on device " + std::to_string(pl->device) +
                                         ", launched with device " + std::to_string(dev) + " current");
  return pl->fn(pl->maps, pl->params, static_cast<cudaStream_t>(stream));
}

extern "C" void nt_attn_plan_destroy(nt_attn_plan* pl) { delete pl; }

// ----------------------------------------------------------------- casts
__global__ void cast_f32_bf16_kernel(const float4* __restrict__ src, uint2* __restrict__ dst, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = src[i];
    dst[i] = make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
  }
}
__global__ void cast_f32_bf16_tail(const float* src, __nv_bfloat16* dst, int64_t lo, int64_t n) {
  int64_t i = lo + threadIdx.x;
  if (i < n) dst[i] = __float2bfloat16_rn(src[i]);
}
__global__ void cast_bf16_f32_kernel(const __nv_bfloat16* __restrict__ src, float* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __bfloat162float(src[i]);
}

extern "C" int nt_cast_f32_to_bf16(const float* src, void* dst, int64_t n, void* stream) {
  if (n <= 0) return NT_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool aligned = (reinterpret_cast<uintptr_t>(src) % 16 == 0) && (reinterpret_cast<uintptr_t>(dst) % 8 == 0);
  int64_t n4 = aligned ? n / 4 : 0;
  if (n4) {
    int blocks = (int)std::min<int64_t>((n4 + 255) / 256, 148 * 16);
    cast_f32_bf16_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(src), static_cast<uint2*>(dst), n4);
    g_launches++;
  }
  int64_t lo = n4 * 4;
  while (lo < n) {
    cast_f32_bf16_tail<<<1, 256, 0, st>>>(src, static_cast<__nv_bfloat16*>(dst), lo, n);
    g_launches++;
    lo += 256;
  }
  return check_cuda(cudaGetLastError(), "cast_f32_bf16");
}

extern "C" int nt_cast_bf16_to_f32(const void* src, float* dst, int64_t n, void* stream) {
  if (n <= 0) return NT_OK;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  cast_bf16_f32_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(src), dst, n);
  g_launches++;
  return check_cuda(cudaGetLastError(), "cast_bf16_f32");
}

#ifdef NT_TRACE
// debug builds only: route the K1 pipeline timeline stamps of one CTA into `buf`
namespace nt {
void trace_set_decode(unsigned long long* buf, int cta);
}
extern "C" int nt_debug_set_trace(unsigned long long* buf, int cta, int item) {
  for (auto f : {trace_set_d64, trace_set_d128, trace_set_e4m3}) f(buf, cta, item, nullptr, 0);
  nt::trace_set_decode(buf, cta);
  return check_cuda(cudaGetLastError(), "nt_debug_set_trace");
}
extern "C" int nt_debug_set_cta_times(unsigned long long* buf) {
  for (auto f : {trace_set_d64, trace_set_d128, trace_set_e4m3}) f(nullptr, 0, 0, buf, 1);
  return check_cuda(cudaGetLastError(), "nt_debug_set_cta_times");
}
#endif

// 0 / -inf fp32 Mask -> visibility bits (bit j % 32 of word j / 32 of a row: key j
// visible); words past seq_kv are zero.  Any other value sets *flag bit 0 (the
// mask is not a pure 0 / -inf pattern: use NT_MASK_TENSOR).
__global__ void mask_to_bits_kernel(const float* __restrict__ mask, int64_t n, int64_t m, int64_t stride,
                                    uint32_t* __restrict__ bits, int64_t words, int* flag) {
  const int64_t row = blockIdx.y;
  const float* src = mask + row * stride;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t b = 0;
    bool bad = false;
    const int64_t j0 = w * 32;
    if (j0 < m) {
#pragma unroll 8
      for (int i = 0; i < 32; ++i) {
        const int64_t j = j0 + i;
        if (j < m) {
          const float x = __ldg(src + j);
          if (x == 0.f) b |= 1u << i;
          else if (!(isinf(x) && x < 0.f)) bad = true;
        }
      }
    }
    bits[row * words + w] = b;
    if (bad && flag) atomicOr(flag, 1);
  }
}

extern "C" int nt_mask_to_bits(const float* mask, int64_t seq_q, int64_t seq_kv, int64_t row_stride, uint32_t* bits,
                               int64_t words_per_row, int32_t* flag, void* stream) {
  if (seq_q <= 0 || seq_kv <= 0) return NT_OK;
  if (!mask || !bits || words_per_row < (seq_kv + 127) / 128 * 4 || row_stride < seq_kv || seq_q > 65535)
    return set_error(NT_ERR_INVALID, "nt_mask_to_bits: bad arguments");
  const int64_t words = words_per_row;
  const int tpb = 128;
  const int bx = (int)std::min<int64_t>((words + tpb - 1) / tpb, 64);
  mask_to_bits_kernel<<<dim3(bx, (unsigned)seq_q), tpb, 0, static_cast<cudaStream_t>(stream)>>>(
      mask, seq_q, seq_kv, row_stride, bits, words, flag);
  g_launches++;
  return check_cuda(cudaGetLastError(), "mask_to_bits");
}

extern "C" int nt_memcpy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
                                 int64_t height, void* stream) {
  if (width <= 0 || height <= 0) return NT_OK;
  return check_cuda(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width, (size_t)height,
                                      cudaMemcpyDefault, static_cast<cudaStream_t>(stream)),
                    "cudaMemcpy2DAsync");
}

extern "C" int nt_abi_version(void) { return NT_ABI_VERSION; }
extern "C" const char* nt_last_error(void) { return g_last_error.c_str(); }
extern "C" int64_t nt_launch_count(void) { return g_launches.load(); }
