// Does cvt.rn.bf16x2.f32 (F2FP) share the XU pipe with MUFU.EX2 on B200?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void kern(float* out, int iters, float seed) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i) * 1e-3f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0 || OP == 2) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1 || OP == 2) {
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(r) : "f"(a[i]));
        a[i] = __uint_as_float(r & 0x3fffffffu);
      }
      if (OP == 3) {  // 2 ex2 + 1 f2fp (softmax mix)
        float b = a[(i + 1) & 7];
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(b));
        a[i] = __uint_as_float(r & 0x3fffffffu);
      }
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 123.456f) out[threadIdx.x] = s;
}

template <int OP>
void run(const char* name, int threads, double ops_per_iter_elem) {
  float* out;
  cudaMalloc(&out, 4096 * 4);
  int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  kern<OP><<<sms, threads>>>(out, iters, 1.0f);
  cudaEventRecord(e0);
  kern<OP><<<sms, threads>>>(out, iters, 1.0f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double insts = (double)threads * iters * 8 * ops_per_iter_elem;  // per SM, thread-instructions
  printf("%-34s thr %4d: %.1f thread-instr/clk/SM\n", name, threads, insts / (ms * 1e-3 * clk * 1e3));
}

int main() {
  for (int t : {256, 1024}) {
    run<0>("MUFU.EX2 only", t, 1);
    run<1>("F2FP only (+LOP)", t, 1);
    run<2>("EX2 + F2FP (counted 2/elem)", t, 2);
    run<3>("2 EX2 + 1 F2FP (counted 3)", t, 3);
  }
}
