// K1 instantiations, e4m3 Q/K/V (head_dim 128, no / causal mask; kind::f8f6f4)
#include "attn_launch.cuh"

namespace nt {
NT_DEFINE_TRACE_SETTER(trace_set_e4m3)
int dispatch_attn_e4m3(const nt_attn_args* a, const AttnMaps& m, const AttnFwdParams& p, cudaStream_t st) {
  return dispatch_attn_nq<128, true, 2>(a, m, p, st);
}
}  // namespace nt
