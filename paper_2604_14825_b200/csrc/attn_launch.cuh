// K1 launch plumbing shared by the per-head-dim translation units (attn_d64.cu,
// attn_d128.cu, attn_e4m3.cu -- split so nvcc builds the instantiations in
// parallel) and capi.cu (validation, tensor maps, split plan).
#pragma once
#include <algorithm>

#include "../../include/nautilus_b200.h"
#include "attn_fwd.cuh"
#include "common_host.h"

#ifndef NT_COMBINE_PDL
#define NT_COMBINE_PDL 1
#endif

namespace nt {

struct AttnMaps {
  CUtensorMap q, k, v, o;
  CUtensorMap p;   // split KV: bf16 partial O / l [units * rows, D]
  const __nv_bfloat16* part_o;  // its base
};

// nt_attn_prepare: everything but the launch (set per call in capi.cu); the
// prepared kernel's resident CTAs per SM are left in g_prepared_ctas_per_sm
extern thread_local bool g_prepare_only;
extern thread_local int g_prepared_ctas_per_sm;
// ... and the fully resolved launcher (instantiation + split/merge), so a plan
// (nt_attn_plan_create) launches with one indirect call and no re-encoding
using AttnLaunchFn = int (*)(const AttnMaps&, const AttnFwdParams&, cudaStream_t);
extern thread_local AttnLaunchFn g_prepared_fn;

// Resident CTAs per SM of a kernel at `threads` / `smem`, once per instantiation.
// Computed from the register, shared-memory and TMEM budgets: the occupancy API
// reports 1 for any kernel that executes tcgen05.alloc, but two CTAs of 256 TMEM
// columns each do co-reside (tools/ubench/occ_probe3.cu: 296 CTAs, 148 same-SM
// overlapping pairs).
template <auto Kern>
int resident_ctas(int threads, int smem, int tmem_cols) {
  static std::atomic<int> occ{0};
  int v = occ.load(std::memory_order_relaxed);
  if (v == 0) {
    int dev = 0, regs_sm = 65536, smem_sm = 233472, reserved = 1024;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, Kern);
    const int warp_regs = ((fa.numRegs * 32 + 255) / 256) * 256;  // allocation unit: 256 per warp
    const int by_regs = regs_sm / std::max(1, warp_regs * ((threads + 31) / 32));
    const int by_smem = smem_sm / std::max(1, smem + (int)fa.sharedSizeBytes + reserved);
    const int by_tmem = 512 / tmem_cols;
    v = std::max(1, std::min(std::min(by_regs, by_smem), std::min(by_tmem, 2048 / threads)));
    occ.store(v, std::memory_order_relaxed);
  }
  return v;
}

template <int D, int MASK, bool F32, int KVS, bool FP8, bool SPLIT, int NQ>
int launch_attn_kernel(const AttnMaps& m, const AttnFwdParams& p, cudaStream_t st) {
  using Cfg = AttnCfg<D, KVS, F32, FP8, NQ, SPLIT>;
  constexpr auto kern = attn_fwd_kernel<D, MASK, F32, KVS, FP8, SPLIT, NQ>;
  const int smem = Cfg::SMEM_BYTES;
  if (const int rc0 = configure_smem<kern>(smem, "cudaFuncSetAttribute(attn_fwd)")) return rc0;
  if constexpr (NQ == 1) {
    // two CTAs per SM need the whole 228 KB carveout
    static std::atomic<uint64_t> carve{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(carve.load() & (1ull << (dev & 63)))) {
      if (const int rc1 = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100),
                                     "cudaFuncSetAttribute(carveout)"))
        return rc1;
      carve.fetch_or(1ull << (dev & 63));
    }
  }
  const int per_sm = resident_ctas<kern>(Cfg::THREADS, smem, Cfg::TMEM_COLS);
  if (g_prepare_only) {
    g_prepared_ctas_per_sm = per_sm;
    cudaFuncAttributes fa;
    if constexpr (SPLIT)
      return check_cuda(cudaFuncGetAttributes(&fa, attn_combine_kernel<D, MASK, F32, Cfg::ROWS>),
                        "cudaFuncGetAttributes(attn_combine)");
    return NT_OK;
  }
  // persistent: as many CTAs as are resident (1 per SM, or 2 with NQ = 1), each
  // drawing work items from the shared counter
  const int grid = std::min(p.n_items, per_sm * num_sms());
  kern<<<grid, Cfg::THREADS, smem, st>>>(m.q, m.k, m.v, m.o, m.p, p);
  g_launches++;
  return check_cuda(cudaGetLastError(), "attn_fwd launch");
}

template <int D, int MASK, bool F32, int KVS, bool FP8, int NQ>
int launch_attn(const AttnMaps& m, const AttnFwdParams& p, cudaStream_t st) {
  if (g_prepare_only) g_prepared_fn = &launch_attn<D, MASK, F32, KVS, FP8, NQ>;
  // the split-KV path is its own instantiation: its extra state costs the
  // unsplit kernel registers (BERT 58 -> 63 us when shared)
  if constexpr (MASK != MASK_TENSOR && MASK != MASK_BITS) {
    if (p.kv_split > 0) {
      int rc = launch_attn_kernel<D, MASK, F32, KVS, FP8, true, NQ>(m, p, st);
      if (rc || g_prepare_only) return rc;
      // split-KV items: merge the bf16 partials.  Programmatic dependent launch: the
      // merge grid is launched while K1 runs (its CTAs take the SMs K1's finished
      // CTAs free) and waits in griddepcontrol.wait for K1's completion and memory
      constexpr int ROWS = 128 * NQ;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(ROWS / (8 * kCombineRowsPerWarp), p.B * p.Hq, p.n_split_mb);
      cfg.blockDim = dim3(256);
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = NT_COMBINE_PDL;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      const int rc2 = check_cuda(cudaLaunchKernelEx(&cfg, attn_combine_kernel<D, MASK, F32, ROWS>, m.part_o, p),
                                 "attn_combine launch");
      g_launches++;
      return rc2;
    }
  }
  return launch_attn_kernel<D, MASK, F32, KVS, FP8, false, NQ>(m, p, st);
}

// the MA `stages` tunable -> K/V ring depth (attn_kv_slots)
template <int D, int MASK, bool F32, bool FP8, int NQ>
int launch_attn_stages(int ma_stages, const AttnMaps& m, const AttnFwdParams& p, cudaStream_t st) {
  constexpr int DS = FP8 ? 64 : D;  // e4m3 K/V tiles are D=64-sized
  constexpr int kShallow = attn_kv_slots<DS, NQ>(1), kDeep = attn_kv_slots<DS, NQ>(2);
  if constexpr (kShallow == kDeep) return launch_attn<D, MASK, F32, kDeep, FP8, NQ>(m, p, st);
  else
    return attn_kv_slots<DS, NQ>(ma_stages) == kShallow ? launch_attn<D, MASK, F32, kShallow, FP8, NQ>(m, p, st)
                                                        : launch_attn<D, MASK, F32, kDeep, FP8, NQ>(m, p, st);
}

template <int D, bool FP8, int NQ>
int dispatch_attn_nq(const nt_attn_args* a, const AttnMaps& m, const AttnFwdParams& p, cudaStream_t st) {
  const bool f32 = a->out_dtype == NT_DTYPE_F32;
  const int sg = a->kv_stages > 0 ? a->kv_stages : 2;  // the MA default (VirtualDevice.stage_default)
  switch (a->mask_kind) {
    case NT_MASK_NONE:
      return f32 ? launch_attn_stages<D, MASK_NONE, true, FP8, NQ>(sg, m, p, st)
                 : launch_attn_stages<D, MASK_NONE, false, FP8, NQ>(sg, m, p, st);
    case NT_MASK_CAUSAL:
      return f32 ? launch_attn_stages<D, MASK_CAUSAL, true, FP8, NQ>(sg, m, p, st)
                 : launch_attn_stages<D, MASK_CAUSAL, false, FP8, NQ>(sg, m, p, st);
    case NT_MASK_TENSOR:
      if constexpr (!FP8)
        return f32 ? launch_attn_stages<D, MASK_TENSOR, true, FP8, NQ>(sg, m, p, st)
                   : launch_attn_stages<D, MASK_TENSOR, false, FP8, NQ>(sg, m, p, st);
      break;
    case NT_MASK_BITS:
      if constexpr (!FP8)
        return f32 ? launch_attn_stages<D, MASK_BITS, true, FP8, NQ>(sg, m, p, st)
                   : launch_attn_stages<D, MASK_BITS, false, FP8, NQ>(sg, m, p, st);
      break;
  }
  return set_error(NT_ERR_INVALID, "unknown mask_kind");
}

#ifdef NT_TRACE
// The trace symbols (attn_fwd.cuh) exist once per translation unit: every TU that
// instantiates K1 defines a setter, capi.cu's nt_debug_set_trace calls them all.
#define NT_DEFINE_TRACE_SETTER(NAME)                                                       \
  void NAME(unsigned long long* buf, int cta, int item, unsigned long long* cta_times, int what) { \
    if (what == 0) {                                                                       \
      cudaMemcpyToSymbol(g_nt_trace, &buf, sizeof(buf));                                   \
      cudaMemcpyToSymbol(g_nt_trace_cta, &cta, sizeof(cta));                               \
      cudaMemcpyToSymbol(g_nt_trace_li, &item, sizeof(item));                              \
    } else {                                                                               \
      cudaMemcpyToSymbol(g_nt_cta_times, &cta_times, sizeof(cta_times));                   \
    }                                                                                      \
  }
void trace_set_d64(unsigned long long*, int, int, unsigned long long*, int);
void trace_set_d128(unsigned long long*, int, int, unsigned long long*, int);
void trace_set_e4m3(unsigned long long*, int, int, unsigned long long*, int);
#else
#define NT_DEFINE_TRACE_SETTER(NAME)
#endif

// defined in attn_d64.cu / attn_d128.cu / attn_e4m3.cu
int dispatch_attn_d64(const nt_attn_args* a, const AttnMaps& m, const AttnFwdParams& p, int nq, cudaStream_t st);
int dispatch_attn_d128(const nt_attn_args* a, const AttnMaps& m, const AttnFwdParams& p, int nq, cudaStream_t st);
int dispatch_attn_e4m3(const nt_attn_args* a, const AttnMaps& m, const AttnFwdParams& p, cudaStream_t st);

}  // namespace nt
