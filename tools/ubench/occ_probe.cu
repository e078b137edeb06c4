// Occupancy probe for the K1 NQ=1 instantiation (two CTAs per SM expected).
#include <cstdio>
#include "../../paper_2604_14825_b200/csrc/attn_fwd.cuh"
using namespace nt;
int main() {
  constexpr auto k = attn_fwd_kernel<128, MASK_CAUSAL, false, 2, false, false, 1>;
  using C = AttnCfg<128, 2, false, false, 1, false>;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k);
  printf("regs %d maxThreads %d static smem %zu local %zu\n", fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes,
         fa.localSizeBytes);
  int smax = 0, regs = 0, rpb = 0, spb = 0;
  cudaDeviceGetAttribute(&smax, cudaDevAttrMaxSharedMemoryPerMultiprocessor, 0);
  cudaDeviceGetAttribute(&regs, cudaDevAttrMaxRegistersPerMultiprocessor, 0);
  cudaDeviceGetAttribute(&rpb, cudaDevAttrReservedSharedMemoryPerBlock, 0);
  cudaDeviceGetAttribute(&spb, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  printf("smem/SM %d regs/SM %d reserved/block %d optin/block %d\n", smax, regs, rpb, spb);
  printf("set max dyn smem: %s\n", cudaGetErrorString(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES)));
  printf("carveout: %s\n", cudaGetErrorString(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100)));
  for (int s : {0, 50000, 100000, C::SMEM_BYTES, 113000}) {
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, 256, s);
    printf("smem %d -> %d blocks/SM (%s)\n", s, n, cudaGetErrorString(e));
  }
  for (int t : {128, 192, 256}) {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, t, 0);
    printf("threads %d smem 0 -> %d\n", t, n);
  }
  return 0;
}
