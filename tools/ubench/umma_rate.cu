// tcgen05.mma (kind::f16 bf16 K=16 | kind::f8f6f4 e4m3 K=32 -> fp32, cta_group::1, M = 128)
// issue throughput vs N, SS (A and B from shared memory) and TS (A from TMEM).  One CTA
// per SM, one issuing thread, 4096 MMAs back to back, timed with clock64 around commit +
// wait; and the latency of a group of G MMAs + commit + wait (the decode kernel's S / PV).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_14825_b200/csrc/sm100.cuh"
using namespace nt;

template <int N, bool TS, bool FP8 = false, int G = 0>
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
    constexpr uint32_t id = FP8 ? idesc_e4m3(128, N, 0, 0) : idesc_bf16(128, N, 0, 0);
    const uint32_t s0 = smem_u32(smem);
    const uint64_t a = sdesc_sw128(s0, 16, 1024);
    const uint64_t b = sdesc_sw128(s0 + 65536, 16, 1024);
    auto mma = [&]() {
      if constexpr (FP8) {
        if (TS) umma_ts_f8(tmem, tmem + 256, b, id, 1u);
        else umma_ss_f8(tmem, a, b, id, 1u);
      } else {
        if (TS) umma_ts(tmem, tmem + 256, b, id, 1u);
        else umma_ss(tmem, a, b, id, 1u);
      }
    };
    const unsigned long long t0 = clock64();
    if constexpr (G == 0) {
      for (int i = 0; i < iters; ++i) mma();
      umma_commit(&bar);
      mbar_wait(&bar, 0);
    } else {
      for (int i = 0; i < iters / G; ++i) {
        for (int j = 0; j < G; ++j) mma();
        umma_commit(&bar);
        mbar_wait(&bar, i & 1);
      }
    }
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, bool TS, bool FP8 = false, int G = 0>
void run() {
  unsigned long long* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto k = kern<N, TS, FP8, G>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int iters = 4096;
  k<<<sms, 128, 160 * 1024>>>(d, iters);
  k<<<sms, 128, 160 * 1024>>>(d, iters);
  cudaDeviceSynchronize();
  unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  double per = (double)c / iters;
  const int K = FP8 ? 32 : 16;
  if (G == 0)
    printf("%s %s M=128 N=%3d K=%d: %6.1f clk/MMA  -> %6.0f FLOP/clk/SM  err=%s\n", FP8 ? "e4m3" : "bf16",
           TS ? "TS" : "SS", N, K, per, 2.0 * 128 * N * K / per, cudaGetErrorString(cudaGetLastError()));
  else
    printf("%s %s M=128 N=%3d K=%d: group of %d + commit + wait: %6.1f clk  err=%s\n", FP8 ? "e4m3" : "bf16",
           TS ? "TS" : "SS", N, K, G, per * G, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<64, false>(); run<128, false>(); run<256, false>();
  run<64, true>(); run<128, true>(); run<256, true>();
  run<128, false, true>(); run<128, true, true>(); run<256, false, true>();
  run<128, false, true, 4>(); run<128, true, true, 4>(); run<128, false, false, 8>(); run<128, true, false, 8>();
}
