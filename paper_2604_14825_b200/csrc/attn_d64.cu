// K1 instantiations, head_dim 64 (BERT-base, config 3)
#include "attn_launch.cuh"

namespace nt {
NT_DEFINE_TRACE_SETTER(trace_set_d64)
int dispatch_attn_d64(const nt_attn_args* a, const AttnMaps& m, const AttnFwdParams& p, int nq, cudaStream_t st) {
  return nq == 1 ? dispatch_attn_nq<64, false, 1>(a, m, p, st) : dispatch_attn_nq<64, false, 2>(a, m, p, st);
}
}  // namespace nt
