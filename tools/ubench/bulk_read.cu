// HBM read ceiling for the decode stream: each CTA pulls its slice of a large buffer
// through a ring of STAGES x CHUNK shared-memory slots with cp.async.bulk (TMA, non
// tensor), consumers only release slots.  Reports GB/s for 1 and 2 CTAs per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_14825_b200/csrc/sm100.cuh"
using namespace nt;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(256) stream(const uint8_t* buf, size_t per_cta, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * CHUNK);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 7); }
    fence_barrier_init();
  }
  __syncthreads();
  const uint8_t* base = buf + blockIdx.x * per_cta;
  const int n = (int)(per_cta / CHUNK);
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0)
      for (int i = 0; i < n; ++i) {
        const int s = i % STAGES;
        if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], CHUNK);
        bulk_g2s(sm + s * CHUNK, base + (size_t)i * CHUNK, CHUNK, &full[s]);
      }
  } else {
    unsigned long long acc = 0;
    for (int i = 0; i < n; ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], (i / STAGES) & 1);
      acc += reinterpret_cast<const uint32_t*>(sm + s * CHUNK)[threadIdx.x];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 12345) *sink = acc;
  }
  if (warp == 0) {  // the 8th arrival per slot comes from warp 0's other lanes? no: 7 consumer warps + warp 0 below
  }
}

template <int STAGES, int CHUNK>
void run(const uint8_t* d, size_t bytes, int ctas_per_sm, int sms) {
  const int grid = sms * ctas_per_sm;
  const size_t per = (bytes / grid) / CHUNK * CHUNK;
  const int smem = STAGES * CHUNK + 2 * STAGES * 8 + 64;
  auto k = stream<STAGES, CHUNK>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  k<<<grid, 256, smem>>>(d, per, sink);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k<<<grid, 256, smem>>>(d, per, sink);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("stages %d chunk %6d B ctas/SM %d: %7.1f GB/s (%s)\n", STAGES, CHUNK, ctas_per_sm,
         5.0 * per * grid / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t bytes = (size_t)8 << 30;
  uint8_t* d; cudaMalloc(&d, bytes); cudaMemset(d, 1, bytes);
  run<6, 32768>(d, bytes, 1, sms);
  run<12, 16384>(d, bytes, 1, sms);
  run<3, 32768>(d, bytes, 2, sms);
  run<6, 16384>(d, bytes, 2, sms);
  run<4, 49152>(d, bytes, 1, sms);
  return 0;
}
