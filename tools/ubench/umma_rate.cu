// tcgen05.mma (kind::f16, bf16 -> fp32, cta_group::1, M = 128) issue throughput vs N,
// SS (A and B from shared memory) and TS (A from TMEM).  One CTA per SM, one issuing
// thread, 4096 MMAs back to back, timed with clock64 around commit + wait.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_14825_b200/csrc/sm100.cuh"
using namespace nt;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) kern(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = idesc_bf16(128, N, 0, 0);
    const uint32_t s0 = smem_u32(smem);
    const uint64_t a = sdesc_sw128(s0, 16, 1024);
    const uint64_t b = sdesc_sw128(s0 + 65536, 16, 1024);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (TS) umma_ts(tmem, tmem + 256, b, id, 1u);
      else umma_ss(tmem, a, b, id, 1u);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, bool TS>
void run() {
  unsigned long long* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto k = kern<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int iters = 4096;
  k<<<sms, 128, 160 * 1024>>>(d, iters);
  k<<<sms, 128, 160 * 1024>>>(d, iters);
  cudaDeviceSynchronize();
  unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  double per = (double)c / iters;
  printf("%s M=128 N=%3d K=16: %6.1f clk/MMA  -> %6.0f FLOP/clk/SM (dense peak 8192)  err=%s\n", TS ? "TS" : "SS", N, per,
         2.0 * 128 * N * 16 / per, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<64, false>(); run<128, false>(); run<256, false>();
  run<64, true>(); run<128, true>(); run<256, true>();
}
