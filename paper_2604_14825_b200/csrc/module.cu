// C ABI for runtime-compiled kernels (include/nautilus_b200.h, "generic MA
// programs"): the SIMT lowering (paper_2604_14825_b200/simt.py) emits CUDA C
// for an MA module, nvcc compiles it to an sm_100a cubin, and these entry
// points load the image, resolve kernels and launch them on a stream.
//
// Reference seam: the CPU executor interpret_ma (tilecc/ma/interp.py:102-148)
// walks the same MA program; SURVEY.md 8(b) sketches this load / launch /
// unload / last-error surface.  The driver API is resolved at run time through
// cudaGetDriverEntryPoint, so libcuda is not a link dependency.
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>
#include <string>

#include "../../include/nautilus_b200.h"
#include "common_host.h"

namespace nt {
namespace {

struct DriverApi {
  CUresult (*module_load_data)(CUmodule*, const void*) = nullptr;
  CUresult (*module_unload)(CUmodule) = nullptr;
  CUresult (*module_get_function)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*func_set_attribute)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*launch_kernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                            CUstream, void**, void**) = nullptr;
  CUresult (*get_error_string)(CUresult, const char**) = nullptr;
  bool ok = false;
};

template <typename F>
bool resolve(const char* name, F* out) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return false;
  *out = reinterpret_cast<F>(p);
  return true;
}

const DriverApi& api() {
  static DriverApi d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.ok = resolve("cuModuleLoadData", &d.module_load_data) && resolve("cuModuleUnload", &d.module_unload) &&
           resolve("cuModuleGetFunction", &d.module_get_function) &&
           resolve("cuFuncSetAttribute", &d.func_set_attribute) && resolve("cuLaunchKernel", &d.launch_kernel) &&
           resolve("cuGetErrorString", &d.get_error_string);
  });
  return d;
}

int drv_error(CUresult r, const char* what) {
  const char* s = nullptr;
  if (api().get_error_string) api().get_error_string(r, &s);
  return set_error(NT_ERR_CUDA, std::string(what) + ": " + (s ? s : "CUDA driver error ") + " (" +
                                    std::to_string(static_cast<int>(r)) + ")");
}

}  // namespace
}  // namespace nt

using namespace nt;

struct nt_module {
  CUmodule mod;
};

extern "C" int nt_module_load(const void* image, size_t nbytes, nt_module** out) {
  if (!image || nbytes == 0 || !out) return set_error(NT_ERR_INVALID, "nt_module_load: null image");
  const DriverApi& d = api();
  if (!d.ok) return set_error(NT_ERR_CUDA, "CUDA driver entry points unavailable");
  int rc = check_cuda(cudaFree(nullptr), "context init");  // make the primary context current
  if (rc) return rc;
  CUmodule m;
  CUresult r = d.module_load_data(&m, image);
  if (r != CUDA_SUCCESS) return drv_error(r, "cuModuleLoadData");
  *out = new nt_module{m};
  return NT_OK;
}

extern "C" int nt_module_function(nt_module* m, const char* entry, void** fn) {
  if (!m || !entry || !fn) return set_error(NT_ERR_INVALID, "nt_module_function: null argument");
  CUfunction f;
  CUresult r = api().module_get_function(&f, m->mod, entry);
  if (r != CUDA_SUCCESS) return drv_error(r, (std::string("cuModuleGetFunction ") + entry).c_str());
  *fn = reinterpret_cast<void*>(f);
  return NT_OK;
}

extern "C" int nt_launch(void* fn, uint32_t grid_x, uint32_t block_x, uint32_t smem_bytes, void** params,
                         void* stream) {
  if (!fn || grid_x == 0 || block_x == 0) return set_error(NT_ERR_INVALID, "nt_launch: bad launch shape");
  const DriverApi& d = api();
  CUfunction f = reinterpret_cast<CUfunction>(fn);
  if (smem_bytes > 48 * 1024) {
    CUresult r = d.func_set_attribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem_bytes);
    if (r != CUDA_SUCCESS) return drv_error(r, "cuFuncSetAttribute(max dynamic smem)");
  }
  CUresult r = d.launch_kernel(f, grid_x, 1, 1, block_x, 1, 1, smem_bytes, static_cast<CUstream>(stream), params,
                               nullptr);
  if (r != CUDA_SUCCESS) return drv_error(r, "cuLaunchKernel");
  g_launches++;
  return NT_OK;
}

extern "C" int nt_module_unload(nt_module* m) {
  if (!m) return NT_OK;
  CUresult r = api().module_unload(m->mod);
  delete m;
  if (r != CUDA_SUCCESS) return drv_error(r, "cuModuleUnload");
  return NT_OK;
}
