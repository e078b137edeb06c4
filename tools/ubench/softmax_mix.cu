// Throughput of the K1 softmax exp-phase instruction mix per SM, for 1 / 2 / 4 warps
// per SMSP, timed in SM clocks (clock64 inside the kernel, so clock throttling does
// not bias it).  Variant bits: 1 = F2FP pack (cvt.rn.bf16x2.f32), 2 = FADD2 row sum,
// 4 = FFMA2 scale/shift, 8 = poly exp2 for 1 in 4 pairs, 16 = integer pack
// (2 IADD + PRMT, round half up), 32 = PRMT-only pack (truncation).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_14825_b200/csrc/sm100.cuh"
using namespace nt;

__device__ __forceinline__ uint32_t pack_trunc(float lo, float hi) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(__float_as_uint(lo)), "r"(__float_as_uint(hi)));
  return r;
}

template <int VAR>
__global__ void kern(float* out, long long* cyc, int iters, float seed) {
  float s[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) s[i] = seed * (threadIdx.x + i) * 1e-3f - 3.0f;
  float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  uint32_t acc = 0;
  const float2 sc2 = make_float2(1.0001f, 1.0001f), nm2 = make_float2(-0.5f, -0.5f);
  __syncthreads();
  const long long t0 = clock64();
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
      else if (VAR & 16) acc ^= pack_bf16_alu(e.x, e.y);
      else if (VAR & 32) acc ^= pack_trunc(e.x, e.y);
      else acc ^= __float_as_uint(e.x) ^ __float_as_uint(e.y);
      s[2 * i] = e.x * 0.5f;   // keep the chain live (FMUL on FMA pipe)
      s[2 * i + 1] = e.y * 0.5f;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float r = sum2[0].x + sum2[0].y + sum2[1].x + sum2[1].y + (float)acc;
  for (int i = 0; i < 64; ++i) r += s[i];
  if (r == 123.456f) out[threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int VAR>
void run(const char* name, int warps_per_smsp) {
  float* out; cudaMalloc(&out, 4096 * 4);
  long long* cyc; cudaMalloc(&cyc, 1024 * 8);
  int iters = 512, threads = 128 * warps_per_smsp;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  kern<VAR><<<sms, threads>>>(out, cyc, iters, 1.0f);
  kern<VAR><<<sms, threads>>>(out, cyc, iters, 1.0f);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  double elems = (double)threads * iters * 64;  // per SM
  printf("%-36s warps/SMSP %d: %5.2f exp/clk/SM\n", name, warps_per_smsp, elems / mx);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int w : {1, 2, 4}) {
    run<0>("MUFU + FMUL only", w);
    run<4>("+FFMA2", w);
    run<6>("+FFMA2 +FADD2", w);
    run<7>("+FFMA2 +FADD2 +F2FP (K1 mix)", w);
    run<22>("+FFMA2 +FADD2 +int pack (IADD+PRMT)", w);
    run<38>("+FFMA2 +FADD2 +PRMT truncation", w);
    run<15>("K1 mix, poly 1/4", w);
    run<46>("PRMT truncation, poly 1/4", w);
  }
}
