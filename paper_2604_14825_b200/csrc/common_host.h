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
int make_map_pages_5d(CUtensorMap* m, const void* ptr, int64_t page_size, int64_t heads, int64_t pages,
                      int64_t token_stride, int64_t head_stride, int64_t page_stride, int rows);
int make_map_2d(CUtensorMap* m, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_inner,
                int box_outer, size_t elem, CUtensorMapSwizzle swz);
}  // namespace nt
