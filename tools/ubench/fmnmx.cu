// Which pipe does the 3-input max (FMNMX3) use on B200?  Throughput alone and mixed with MUFU.EX2.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2604_14825_b200/csrc/sm100.cuh"
using namespace nt;

template <int OP>
__global__ void kern(float* out, int iters, float seed) {
  float a[8], b[8];
  for (int i = 0; i < 8; ++i) { a[i] = seed * (threadIdx.x + i); b[i] = seed - i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = fmax3(a[i], b[i], b[(i + 1) & 7]);          // FMNMX3 only
      if (OP == 1) a[i] = fmaxf(fmaxf(a[i], b[i]), b[(i + 1) & 7]);    // 2x FMNMX
      if (OP == 2) { a[i] = fmax3(a[i], b[i], b[(i + 1) & 7]); b[i] = ex2(b[i]); }  // FMNMX3 + MUFU
      if (OP == 3) { a[i] = fmaxf(fmaxf(a[i], b[i]), b[(i + 1) & 7]); b[i] = ex2(b[i]); }  // 2 FMNMX + MUFU
      if (OP == 4) { b[i] = ex2(b[i]); }  // MUFU only
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + b[i];
  if (s == 123.456f) out[threadIdx.x] = s;
}

template <int OP>
void run(const char* name) {
  float* out; cudaMalloc(&out, 4096 * 4);
  int iters = 4096, threads = 512;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  kern<OP><<<sms, threads>>>(out, iters, 1.0f);
  cudaEventRecord(e0);
  kern<OP><<<sms, threads>>>(out, iters, 1.0f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%-34s %6.2f iterations-elements/clk/SM\n", name, (double)threads * iters * 8 / (ms * 1e-3 * clk * 1e3));
}
int main() {
  run<0>("FMNMX3 (1 instr / elem)");
  run<1>("2x FMNMX (2 instr / elem)");
  run<2>("FMNMX3 + MUFU.EX2");
  run<3>("2x FMNMX + MUFU.EX2");
  run<4>("MUFU.EX2 only");
}
