// Do two TMEM-allocating CTAs actually co-reside on one SM?  Each CTA records its SM
// and [entry, exit) globaltimer while spinning 200 us; overlap on one SM = co-residency.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
template <bool TMEM>
__global__ void __launch_bounds__(256, 2) k(unsigned long long* rec) {
  __shared__ uint32_t slot;
  uint64_t t0 = gt();
  if (TMEM && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  while (gt() - t0 < 200000) {}
  __syncthreads();
  if (TMEM && threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(slot));
  if (threadIdx.x == 0) {
    uint32_t sm; asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
    rec[blockIdx.x * 3] = sm; rec[blockIdx.x * 3 + 1] = t0; rec[blockIdx.x * 3 + 2] = gt();
  }
}
template <bool TMEM> void run(const char* name) {
  int n = 296;
  unsigned long long* d; cudaMalloc(&d, n * 3 * 8);
  k<TMEM><<<n, 256>>>(d);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(n * 3);
  cudaMemcpy(h.data(), d, n * 3 * 8, cudaMemcpyDeviceToHost);
  int overlaps = 0;
  unsigned long long lo = ~0ull, hi = 0;
  for (int i = 0; i < n; ++i) { lo = std::min(lo, h[i*3+1]); hi = std::max(hi, h[i*3+2]); }
  for (int i = 0; i < n; ++i) for (int j = i + 1; j < n; ++j)
    if (h[i*3] == h[j*3] && h[i*3+1] < h[j*3+2] && h[j*3+1] < h[i*3+2]) overlaps++;
  printf("%s: %d CTAs, overlapping same-SM pairs %d, span %.1f us (%s)\n", name, n, overlaps, (hi - lo) / 1e3,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
int main() { run<false>("no tmem"); run<true>("tmem 256 cols"); return 0; }
