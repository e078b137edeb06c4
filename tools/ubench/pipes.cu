// Microbenchmark: per-SM throughput of MUFU.EX2, F2FP (cvt bf16x2), FFMA2, IADD3+PRMT on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

template <int OP>
__global__ void kern(float* out, int iters, float seed) {
  float a[8];
  uint32_t u[8];
  for (int i = 0; i < 8; ++i) { a[i] = seed * (threadIdx.x + i) * 1e-3f; u[i] = threadIdx.x + i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i])); }
      if (OP == 1) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i+1)&7])); u[i] ^= r; }
      if (OP == 2) { asm volatile("{.reg .b64 x; mov.b64 x, {%0,%1}; fma.rn.f32x2 x, x, x, x; mov.b64 {%0,%1}, x;}" : "+f"(a[i]), "+f"(a[(i+4)&7])); }
      if (OP == 3) { asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i])); }
      if (OP == 4) { uint32_t r; asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(u[i]), "r"(u[(i+1)&7])); u[i] = r + 0x8000u; }
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + (float)u[i];
  if (s == 123.456f) out[threadIdx.x] = s;
}

template <int OP>
void run(const char* name, int threads) {
  float* out; cudaMalloc(&out, 4096 * 4);
  int iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  kern<OP><<<sms, threads>>>(out, iters, 1.0f);
  cudaEventRecord(e0);
  kern<OP><<<sms, threads>>>(out, iters, 1.0f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)sms * threads * iters * 8;
  double per_sm_per_clk = ops / sms / (ms * 1e-3 * clk * 1e3);
  printf("%-28s threads/CTA %4d: %.1f ops/clk/SM (ms %.3f, clk %d MHz)\n", name, threads, per_sm_per_clk, ms, clk / 1000);
}

int main() {
  for (int t : {128, 512, 1024}) {
    run<0>("MUFU.EX2 (ex2.approx.ftz)", t);
    run<1>("F2FP cvt.rn.bf16x2.f32", t);
    run<2>("FFMA2 (pairs counted x1)", t);
    run<3>("FFMA", t);
    run<4>("PRMT + IADD", t);
  }
  return 0;
}
