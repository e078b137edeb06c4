// Host-side helpers shared by the C ABI translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <string>

namespace nt {
extern thread_local std::string g_last_error;
extern std::atomic<int64_t> g_launches;
int set_error(int code, const std::string& msg);
int check_cuda(cudaError_t e, const char* what);
int num_sms();  // SMs of the current device (persistent grids)
int make_map_4d(CUtensorMap* m, const void* ptr, int64_t D, int64_t S, int64_t H, int64_t B, int64_t sS,
                int64_t sH, int64_t sB, int box_rows, size_t elem, int box_inner = 0,
                CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B);
int make_map_4d_box(CUtensorMap* m, const void* ptr, const int64_t dims[4], const int64_t strides[3],
                    const int box[4], size_t elem);
int make_map_pages_5d(CUtensorMap* m, const void* ptr, int64_t page_size, int64_t heads, int64_t pages,
                      int64_t token_stride, int64_t head_stride, int64_t page_stride, int rows);
int make_map_2d(CUtensorMap* m, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_inner,
                int box_outer, size_t elem, CUtensorMapSwizzle swz);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute lives in the device's context, so a process that launches on
// several GPUs must set it on each.  Keyed by the kernel's address (one static
// per instantiation), a bit per device ordinal.
template <auto Kern>
int configure_smem(int smem, const char* what) {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return 0;
  const int rc = check_cuda(cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), what);
  if (rc == 0) done.fetch_or(bit, std::memory_order_acq_rel);
  return rc;
}
}  // namespace nt
