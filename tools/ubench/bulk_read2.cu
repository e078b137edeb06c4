// Read ceiling of the decode access pattern: each CTA streams TWO regions (its K and
// V slices) alternately in CHUNK-byte bulk copies through a STAGES-deep ring, vs one
// contiguous region (tools/ubench/bulk_read.cu).  Consumers only release slots.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_14825_b200/csrc/sm100.cuh"
using namespace nt;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int STAGES, int CHUNK, int STREAMS>
__global__ void __launch_bounds__(128) stream(const uint8_t* buf, size_t half_bytes, size_t per_cta,
                                              unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * CHUNK);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  // STREAMS == 2: chunk i comes from region (i & 1) -- K at [0, half), V at [half, 2 half)
  const uint8_t* base0 = buf + blockIdx.x * per_cta;
  const uint8_t* base1 = buf + half_bytes + blockIdx.x * per_cta;
  const int n = (int)(per_cta / CHUNK) * STREAMS;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < n; ++i) {
      const int s = i % STAGES;
      if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], CHUNK);
      const uint8_t* src = STREAMS == 2 ? ((i & 1) ? base1 : base0) + (size_t)(i >> 1) * CHUNK
                                        : base0 + (size_t)i * CHUNK;
      bulk_g2s(sm + s * CHUNK, src, CHUNK, &full[s]);
    }
  } else if (warp == 1) {
    unsigned long long acc = 0;
    for (int i = 0; i < n; ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], (i / STAGES) & 1);
      acc += reinterpret_cast<const uint32_t*>(sm + s * CHUNK)[lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 12345) *sink = acc;
  }
}

template <int STAGES, int CHUNK, int STREAMS>
void run(const uint8_t* d, size_t bytes, int sms, int grid_mult) {
  const int grid = sms * grid_mult;
  const size_t half = bytes / 2;
  const size_t per = (half / grid) / CHUNK * CHUNK;  // per CTA per stream (STREAMS 1: over the first half only... use 2x)
  const size_t per_eff = STREAMS == 2 ? per : 2 * per;
  const int smem = STAGES * CHUNK + 2 * STAGES * 8 + 64;
  auto k = stream<STAGES, CHUNK, STREAMS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  k<<<grid, 128, smem>>>(d, half, per_eff, sink);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k<<<grid, 128, smem>>>(d, half, per_eff, sink);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double moved = 5.0 * (STREAMS == 2 ? 2.0 * per : 2.0 * per) * grid;
  printf("streams %d stages %2d chunk %6d B grid %dx%d: %7.1f GB/s (%s)\n", STREAMS, STAGES, CHUNK, sms, grid_mult,
         moved / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t bytes = (size_t)8 << 30;
  uint8_t* d; cudaMalloc(&d, bytes); cudaMemset(d, 1, bytes);
  run<12, 16384, 1>(d, bytes, sms, 1);
  run<12, 16384, 2>(d, bytes, sms, 1);
  run<6, 32768, 1>(d, bytes, sms, 1);
  run<6, 32768, 2>(d, bytes, sms, 1);
  run<12, 16384, 2>(d, bytes, sms, 7);  // many short CTAs (the split grid)
  run<6, 32768, 2>(d, bytes, sms, 7);
  return 0;
}
