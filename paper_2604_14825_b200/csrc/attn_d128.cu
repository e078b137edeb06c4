// K1 instantiations, head_dim 128 (Llama-3-8B, configs 1/4)
#include "attn_launch.cuh"

namespace nt {
NT_DEFINE_TRACE_SETTER(trace_set_d128)
int dispatch_attn_d128(const nt_attn_args* a, const AttnMaps& m, const AttnFwdParams& p, int nq, cudaStream_t st) {
  return nq == 1 ? dispatch_attn_nq<128, false, 1>(a, m, p, st) : dispatch_attn_nq<128, false, 2>(a, m, p, st);
}
}  // namespace nt
