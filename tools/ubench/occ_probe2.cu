// Which feature limits residency to one CTA per SM: setmaxnreg, tcgen05.alloc, or neither?
#include <cstdio>
#include <cstdint>
__global__ void __launch_bounds__(256, 2) plain(int* x) { if (x) x[threadIdx.x] = 1; }
__global__ void __launch_bounds__(256, 2) with_maxnreg(int* x) {
  if (threadIdx.x < 128) asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
  else asm volatile("setmaxnreg.inc.sync.aligned.u32 192;");
  if (x) x[threadIdx.x] = 1;
}
__global__ void __launch_bounds__(256, 2) with_tmem(int* x) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(slot));
  if (x) x[threadIdx.x] = 1;
}
template <typename K> void q(const char* n, K k) {
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, 256, 0);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k);
  printf("%-14s regs %3d -> %d blocks/SM\n", n, fa.numRegs, b);
}
int main() {
  q("plain", plain);
  q("setmaxnreg", with_maxnreg);
  q("tcgen05.alloc", with_tmem);
  return 0;
}
