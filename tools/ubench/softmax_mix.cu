// Throughput of the K1 softmax exp-phase instruction mix (FFMA2 -> 2x MUFU.EX2 -> FADD2 + F2FP)
// per SM, for 1 / 2 / 4 warps per SMSP.  Variant bits: 1 = F2FP pack, 2 = FADD2 row sum,
// 4 = FFMA2 scale/shift, 8 = poly exp2 for 1 in 4 pairs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_14825_b200/csrc/sm100.cuh"
using namespace nt;

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
      float2 x = make_float2(s[2 * i], s[2 * i + 1]);
      if (VAR & 4) x = ffma2(x, sc2, nm2);
      float2 e;
      if ((VAR & 8) && (i % 4) == 3) e = ex2_poly2(x);
      else e = make_float2(ex2(x.x), ex2(x.y));
      if (VAR & 2) sum2[i & 1] = fadd2(sum2[i & 1], e);
      if (VAR & 1) acc ^= pack_bf16(e.x, e.y);
      else acc ^= __float_as_uint(e.x) ^ __float_as_uint(e.y);
      s[2 * i] = e.x * 0.5f;   // keep the chain live (FMUL on FMA pipe)
      s[2 * i + 1] = e.y * 0.5f;
    }
  }
  float r = sum2[0].x + sum2[0].y + sum2[1].x + sum2[1].y + (float)acc;
  for (int i = 0; i < 64; ++i) r += s[i];
  if (r == 123.456f) out[threadIdx.x] = r;
}

template <int VAR>
void run(const char* name, int warps_per_smsp) {
  float* out; cudaMalloc(&out, 4096 * 4);
  int iters = 512, threads = 128 * warps_per_smsp;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  kern<VAR><<<sms, threads>>>(out, iters, 1.0f);
  cudaEventRecord(e0);
  kern<VAR><<<sms, threads>>>(out, iters, 1.0f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double elems = (double)threads * iters * 64;  // per SM
  printf("%-34s warps/SMSP %d: %5.2f exp-elements/clk/SM\n", name, warps_per_smsp, elems / (ms * 1e-3 * clk * 1e3));
}

int main() {
  for (int w : {1, 2, 4}) {
    run<0>("MUFU + FMUL only", w);
    run<4>("+FFMA2", w);
    run<6>("+FFMA2 +FADD2", w);
    run<7>("+FFMA2 +FADD2 +F2FP (K1 mix)", w);
    run<15>("K1 mix, poly 1/4", w);
  }
}
