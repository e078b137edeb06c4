// C ABI: nt_gemm (K3) and nt_gemm_chain (K3b).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "../../include/nautilus_b200.h"
#include "chain.cuh"
#include "common_host.h"
#include "gemm.cuh"

#ifndef NT_GEMM_PDL
#define NT_GEMM_PDL 1
#endif

#ifndef NT_GEMM_GROUP
#define NT_GEMM_GROUP 0  // experiment: raster group rows (0 = default 8)
#endif

using namespace nt;

namespace {
// cudaLaunchKernelEx with programmatic stream serialization (the kernel calls
// griddepcontrol.wait before it reads anything an earlier kernel wrote)
template <typename Kern, typename... Args>
int launch_pdl(Kern kern, dim3 grid, dim3 block, int smem, cudaStream_t st, const char* what, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = NT_GEMM_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int rc = check_cuda(cudaLaunchKernelEx(&cfg, kern, args...), what);
  g_launches++;
  return rc;
}
int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, bool F32>
int launch_gemm(const nt_gemm_args* a, cudaStream_t st) {
  CUtensorMap ma, mb;
  int rc;
  if ((rc = make_map_2d(&ma, a->a, a->k, a->m, a->lda, 64, 128, 2, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
  if ((rc = make_map_2d(&mb, a->b, a->n, a->k, a->ldb, 64, 64, 2, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
  GemmParams p{};
  p.M = a->m;
  p.N = a->n;
  p.K = a->k;
  p.tiles_m = (a->m + 127) / 128;
  p.tiles_n = (a->n + BN - 1) / BN;
  const int k_blocks = (a->k + 63) / 64;
  // clamp to what the caller's workspace holds (fp32 M x N partial per split)
  const int64_t per_split = (int64_t)a->m * a->n * (int64_t)sizeof(float);
  const int fits = a->workspace ? (int)std::min<int64_t>(a->workspace_bytes / per_split, 1 << 20) : 0;
  p.k_splits = (a->k_splits > 1 && fits > 1) ? std::min(std::min(a->k_splits, fits), k_blocks) : 1;
  p.kb_per = (k_blocks + p.k_splits - 1) / p.k_splits;
  p.k_splits = (k_blocks + p.kb_per - 1) / p.kb_per;  // no empty K range
  p.ws = static_cast<float*>(a->workspace);
  p.c = a->c;
  p.ldc = a->ldc;
  constexpr auto kern = gemm_kernel<BN, F32>;
  const int smem = GemmCfg<BN>::SMEM_BYTES;
  if ((rc = configure_smem<kern>(smem, "cudaFuncSetAttribute(gemm)"))) return rc;
  const int tiles = p.tiles_m * p.tiles_n * p.k_splits;
  const int grid = std::min(tiles, sm_count());
  // programmatic dependent launches: this GEMM's prologue (barriers, TMEM) overlaps the
  // previous kernel's tail -- e.g. the chain's T = X.W1 -- and griddepcontrol.wait
  // inside holds every read of its inputs until that kernel's memory is visible
  if ((rc = launch_pdl(kern, dim3(grid), dim3(kGemmThreads), smem, st, "gemm launch", ma, mb, p))) return rc;
  if (p.k_splits > 1) {
    const long long n4 = (long long)a->m * a->n / 4;
    const int blocks = (int)std::min<long long>((n4 + 255) / 256, 4LL * sm_count());
    rc = launch_pdl(gemm_splitk_reduce, dim3(blocks), dim3(256), 0, st, "gemm split-K reduce", (const float*)p.ws,
                    p.k_splits, a->m, a->n, a->c, (long long)a->ldc, F32);
  }
  return rc;
}

template <bool F32>
int launch_gemm2(const nt_gemm_args* a, cudaStream_t st) {
  CUtensorMap ma, mb;
  int rc;
  if ((rc = make_map_2d(&ma, a->a, a->k, a->m, a->lda, 64, 128, 2, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
  if ((rc = make_map_2d(&mb, a->b, a->n, a->k, a->ldb, 64, 64, 2, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
  GemmParams p{};
  p.M = a->m;
  p.N = a->n;
  p.K = a->k;
  p.tiles_m = (a->m + 255) / 256;
  p.tiles_n = (a->n + 255) / 256;
  // raster groups only when A's panels would not stay in L2 (~126 MB) next to B's
  const double a_bytes = 2.0 * a->m * a->k;
  p.group_m = (a_bytes > 48e6 && p.tiles_m > 8) ? (NT_GEMM_GROUP > 0 ? NT_GEMM_GROUP : 8) : p.tiles_m;
  p.c = a->c;
  p.ldc = a->ldc;
  CUtensorMap mc;
  if ((rc = make_map_2d(&mc, a->c, a->n, a->m, a->ldc, 32, 32, F32 ? 4 : 2,
                        F32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B)))
    return rc;
  constexpr auto kern = gemm2_kernel<F32>;
  const int smem = Gemm2Cfg<F32>::SMEM_BYTES;
  if ((rc = configure_smem<kern>(smem, "cudaFuncSetAttribute(gemm2)"))) return rc;
  const int tiles = p.tiles_m * p.tiles_n;
  const int grid = 2 * std::min(tiles, sm_count() / 2);  // one CTA pair per tile, persistent
  return launch_pdl(kern, dim3(grid), dim3(kGemmThreads), smem, st, "gemm2 launch", ma, mb, mc, p);
}

// F split so that row_blocks x splits ~ fills the SMs
void chain_split(int n, int f, int* splits_out, int* per_split_out) {
  const int row_blocks = (n + 127) / 128;
  const int f_tiles = (f + 127) / 128;
  int splits = std::max(1, std::min(f_tiles, sm_count() / std::max(1, row_blocks)));
  const int per = (f_tiles + splits - 1) / splits;
  *splits_out = (f_tiles + per - 1) / per;
  *per_split_out = per;
}

template <int E>
int launch_chain(const nt_chain_args* a, cudaStream_t st) {
  CUtensorMap mx, mw1, mw2;
  int rc;
  if ((rc = make_map_2d(&mx, a->x, a->k, a->n, a->ldx, 64, 128, 2, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
  if ((rc = make_map_2d(&mw1, a->w1, a->f, a->k, a->ldw1, 64, 64, 2, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
  if ((rc = make_map_2d(&mw2, a->w2, a->e, a->f, a->ldw2, 64, 128, 2, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
  ChainParams p{};
  p.N = a->n;
  p.K = a->k;
  p.F = a->f;
  p.E = a->e;
  p.row_blocks = (a->n + 127) / 128;
  int splits = 1;
  chain_split(a->n, a->f, &splits, &p.f_tiles_per_split);
  p.splits = splits;
  p.y = a->y;
  p.ldy = a->ldy;
  p.out_f32 = a->out_dtype == NT_DTYPE_F32;
  float* partial = static_cast<float*>(a->workspace);
  if (splits > 1 && (!partial || a->workspace_bytes < (int64_t)splits * a->n * a->e * (int64_t)sizeof(float)))
    return set_error(NT_ERR_INVALID, "chain workspace too small (nt_gemm_chain_workspace_bytes)");
  p.partial = partial;
  constexpr auto kern = chain_kernel<E>;
  const int smem = ChainCfg<E>::SMEM_BYTES;
  if ((rc = configure_smem<kern>(smem, "cudaFuncSetAttribute(chain)"))) return rc;
  kern<<<p.row_blocks * splits, kChainThreads, smem, st>>>(mx, mw1, mw2, p);
  g_launches++;
  if ((rc = check_cuda(cudaGetLastError(), "chain launch"))) return rc;
  if (splits > 1) {
    const long long total = (long long)a->n * a->e;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 4 * sm_count());
    chain_reduce_kernel<<<blocks, 256, 0, st>>>(partial, splits, a->n, a->e, a->y, a->ldy, p.out_f32);
    g_launches++;
    if ((rc = check_cuda(cudaGetLastError(), "chain reduce launch"))) return rc;
  }
  return NT_OK;
}
}  // namespace

extern "C" int nt_gemm(const nt_gemm_args* a, void* stream) {
  if (!a) return set_error(NT_ERR_INVALID, "null args");
  if (a->m <= 0 || a->n <= 0 || a->k <= 0) return set_error(NT_ERR_INVALID, "non-positive extent");
  if (a->k % 8 || a->n % 8) return set_error(NT_ERR_UNSUPPORTED, "K and N must be multiples of 8");
  if (a->ldc % 8) return set_error(NT_ERR_INVALID, "ldc must be a multiple of 8");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool f32 = a->out_dtype == NT_DTYPE_F32;
  if (a->n <= 128) return f32 ? launch_gemm<128, true>(a, st) : launch_gemm<128, false>(a, st);
  // CTA pairs when there are enough 256x256 tiles to give every pair one (B200 A/B,
  // tools/gemm_ab.py: 4096^3 1-SM 103.8 us -> pairs 96.3 us, 8192^3 784 -> 752 us;
  // 4096x1024x4096 (64 pair tiles) stays faster on single CTAs)
  static const bool one_sm = getenv("NT_GEMM_1SM") != nullptr;  // A/B switch
  const long long pair_tiles = (long long)((a->m + 255) / 256) * ((a->n + 255) / 256);
  if (!one_sm && pair_tiles >= sm_count() / 2)
    return f32 ? launch_gemm2<true>(a, st) : launch_gemm2<false>(a, st);
  return f32 ? launch_gemm<256, true>(a, st) : launch_gemm<256, false>(a, st);
}

// Split K over CTAs when the output tiles (128 x 128) cannot give every SM work:
// 4096 x 128 x 4096 has 32 tiles -> 4 K ranges of 1024 (the GEMM-chain's T.W2).
extern "C" int32_t nt_gemm_k_splits(int32_t m, int32_t n, int32_t k) {
  if (m <= 0 || n <= 0 || k <= 0 || n > 128 || n % 4) return 1;
  const int tiles = ((m + 127) / 128) * ((n + 127) / 128);
  const int k_blocks = (k + 63) / 64;
  if (tiles >= sm_count() / 2) return 1;
  return std::max(1, std::min(sm_count() / tiles, k_blocks / 8));  // >= 8 k-blocks per range
}

extern "C" int64_t nt_gemm_workspace_bytes(int32_t m, int32_t n, int32_t k) {
  const int s = nt_gemm_k_splits(m, n, k);
  return s > 1 ? (int64_t)s * m * n * (int64_t)sizeof(float) : 0;
}

extern "C" int64_t nt_gemm_chain_workspace_bytes(int32_t n, int32_t f, int32_t e) {
  int splits = 1, per = 1;
  chain_split(n, f, &splits, &per);
  return splits > 1 ? (int64_t)splits * n * e * (int64_t)sizeof(float) : 0;
}

extern "C" int nt_gemm_chain(const nt_chain_args* a, void* stream) {
  if (!a) return set_error(NT_ERR_INVALID, "null args");
  if (a->n <= 0 || a->k <= 0 || a->f <= 0 || a->e <= 0) return set_error(NT_ERR_INVALID, "non-positive extent");
  if (a->k % 8 || a->f % 8 || a->e % 8) return set_error(NT_ERR_UNSUPPORTED, "K, F, E must be multiples of 8");
  if (a->e > 256) return set_error(NT_ERR_UNSUPPORTED, "fused chain keeps Y in TMEM: E must be <= 256");
  if (a->ldy % 8) return set_error(NT_ERR_INVALID, "ldy must be a multiple of 8");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (a->e <= 64) return launch_chain<64>(a, st);
  if (a->e <= 128) return launch_chain<128>(a, st);
  return launch_chain<256>(a, st);
}

// K2 decode entry points live in decode.cu
