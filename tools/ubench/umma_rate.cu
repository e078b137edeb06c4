// tcgen05.mma (kind::f16 bf16 K=16 | kind::f8f6f4 e4m3 K=32 -> fp32, cta_group::1, M = 128)
// issue throughput vs N, SS (A and B from shared memory) and TS (A from TMEM).  One CTA
// per SM, one issuing thread, 4096 MMAs back to back, timed with clock64 around commit +
// wait; and the latency of a group of G MMAs + commit + wait (the decode kernel's S / PV).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_14825_b200/csrc/sm100.cuh"
using namespace nt;

// G > 0: groups of G MMAs; C commits after each group (C = 0: one wait per group)
// BMN: B operand MN-major (the decode PV's V); A0: A descriptor with 8-row-group stride 0
template <int N, bool TS, bool FP8 = false, int G = 0, int C = 0, bool BMN = false, bool A0 = false>
__global__ void __launch_bounds__(128, 1) kern(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bars[4];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = FP8 ? idesc_e4m3(128, N, 0, BMN ? 1 : 0) : idesc_bf16(128, N, 0, BMN ? 1 : 0);
    const uint32_t s0 = smem_u32(smem);
    const uint64_t a = sdesc_sw128(s0, 16, A0 ? 0 : 1024);
    const uint64_t b = BMN ? sdesc_sw128(s0 + 65536, 16384, 1024) : sdesc_sw128(s0 + 65536, 16, 1024);
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
    } else if constexpr (C == 0) {
      for (int i = 0; i < iters / G; ++i) {
        for (int j = 0; j < G; ++j) mma();
        umma_commit(&bar);
        mbar_wait(&bar, i & 1);
      }
    } else {
      // commits that nobody waits on (the decode kernel's bar_s / empty / bar_pv arrivals)
      for (int i = 0; i < iters / G; ++i) {
        for (int j = 0; j < G; ++j) mma();
        for (int c = 0; c < C; ++c) umma_commit(&bars[c]);
      }
      umma_commit(&bar);
      mbar_wait(&bar, 0);
    }
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, bool TS, bool FP8 = false, int G = 0, int C = 0, bool BMN = false, bool A0 = false>
void run() {
  unsigned long long* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto k = kern<N, TS, FP8, G, C, BMN, A0>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int iters = 4096;
  k<<<sms, 128, 160 * 1024>>>(d, iters);
  k<<<sms, 128, 160 * 1024>>>(d, iters);
  cudaDeviceSynchronize();
  unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  double per = (double)c / iters;
  const int K = FP8 ? 32 : 16;
  if (G == 0)
    printf("%s %s%s%s M=128 N=%3d K=%d: %6.1f clk/MMA  -> %6.0f FLOP/clk/SM  err=%s\n", FP8 ? "e4m3" : "bf16",
           TS ? "TS" : "SS", BMN ? " B-MN-major" : "", A0 ? " A-SBO0" : "", N, K, per, 2.0 * 128 * N * K / per,
           cudaGetErrorString(cudaGetLastError()));
  else if (C == 0)
    printf("%s %s M=128 N=%3d K=%d: group of %d + commit + wait: %6.1f clk  err=%s\n", FP8 ? "e4m3" : "bf16",
           TS ? "TS" : "SS", N, K, G, per * G, cudaGetErrorString(cudaGetLastError()));
  else
    printf("%s %s M=128 N=%3d K=%d: group of %d + %d commits (no wait): %6.1f clk per group  err=%s\n",
           FP8 ? "e4m3" : "bf16", TS ? "TS" : "SS", N, K, G, C, per * G, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<64, false>(); run<128, false>(); run<256, false>();
  run<64, true>(); run<128, true>(); run<256, true>();
  run<128, false, true>(); run<128, true, true>(); run<256, false, true>();
  run<128, false, true, 4>(); run<128, true, true, 4>(); run<128, false, false, 8>(); run<128, true, false, 8>();
  run<128, false, true, 4, 1>(); run<128, false, true, 4, 2>(); run<128, true, true, 4, 2>();
  run<128, false, false, 8, 1>(); run<128, false, false, 8, 2>();
  run<128, true, true, 0, 0, true>(); run<128, false, true, 0, 0, true>(); run<128, true, false, 0, 0, true>();
  run<128, false, true, 0, 0, false, true>(); run<128, false, false, 0, 0, false, true>();
}
