// MUFU.EX2 throughput: f32 vs f16x2 (exp-elements per clk per SM), and the f16x2 softmax mix.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include "../../paper_2604_14825_b200/csrc/sm100.cuh"
using namespace nt;

__device__ __forceinline__ uint32_t ex2_h2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float2 unpack_h2(uint32_t h) {
  __half2 v = *reinterpret_cast<__half2*>(&h);
  return __half22float2(v);
}

template <int VAR>
__global__ void kern(float* out, int iters, float seed) {
  float s[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) s[i] = seed * (threadIdx.x + i) * 1e-3f - 3.0f;
  float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  uint32_t acc = 0;
  const float2 sc2 = make_float2(1.0001f, 1.0001f), nm2 = make_float2(-0.5f, -0.5f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      float2 x = ffma2(make_float2(s[2 * i], s[2 * i + 1]), sc2, nm2);
      float2 e;
      if (VAR == 0) {
        e = make_float2(ex2(x.x), ex2(x.y));
      } else {
        e = unpack_h2(ex2_h2(pack_h2(x.x, x.y)));
      }
      sum2[i & 1] = fadd2(sum2[i & 1], e);
      acc ^= pack_bf16(e.x, e.y);
      s[2 * i] = e.x * 0.5f;
      s[2 * i + 1] = e.y * 0.5f;
    }
  }
  float r = sum2[0].x + sum2[0].y + sum2[1].x + sum2[1].y + (float)acc;
  for (int i = 0; i < 64; ++i) r += s[i];
  if (r == 123.456f) out[threadIdx.x] = r;
}

template <int VAR>
void run(const char* name, int w) {
  float* out; cudaMalloc(&out, 4096 * 4);
  int iters = 512, threads = 128 * w;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  kern<VAR><<<sms, threads>>>(out, iters, 1.0f);
  cudaEventRecord(e0);
  kern<VAR><<<sms, threads>>>(out, iters, 1.0f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%-28s warps/SMSP %d: %5.2f exp/clk/SM\n", name, w, (double)threads * iters * 64 / (ms * 1e-3 * clk * 1e3));
}
int main() {
  for (int w : {1, 2, 4}) { run<0>("f32 MUFU mix", w); run<1>("f16x2 MUFU mix", w); }
}
