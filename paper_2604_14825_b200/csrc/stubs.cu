// Entry points whose kernels are not built yet: fail loudly (no CPU fallback).
#include "../../include/nautilus_b200.h"
#include "common_host.h"
using namespace nt;
extern "C" int64_t nt_decode_workspace_bytes(int32_t, int32_t, int32_t, int32_t, int32_t) { return 0; }
extern "C" int nt_attn_decode(const nt_decode_args*, void*) { return set_error(NT_ERR_UNSUPPORTED, "nt_attn_decode: not built"); }
extern "C" int nt_gemm(const nt_gemm_args*, void*) { return set_error(NT_ERR_UNSUPPORTED, "nt_gemm: not built"); }
extern "C" int nt_gemm_chain(const nt_chain_args*, void*) { return set_error(NT_ERR_UNSUPPORTED, "nt_gemm_chain: not built"); }
