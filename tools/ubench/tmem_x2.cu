// Probe of the tcgen05.ld/st .16x32bx2 fragment: which (TMEM lane, column) each
// thread of the warp sees, for the 2-threads-per-row softmax of the decode kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tmem_x2 tools/ubench/tmem_x2.cu
#include <cstdio>
#include <cstdint>

__global__ void probe(uint32_t* out) {
  __shared__ uint32_t slot;
  const int lane = threadIdx.x;
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
      (uint32_t)__cvta_generic_to_shared(&slot)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  // 32x32b: thread = lane, value = lane << 16 | column
  for (int c = 0; c < 64; ++c) {
    const uint32_t v = (lane << 16) | c;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(t + c), "r"(v));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x4.b32 {%0,%1,%2,%3}, [%4], 32;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int i = 0; i < 4; ++i) out[lane * 4 + i] = r[i];
  // store through 16x32bx2 at column 64 (+8 for the second half), read back with 32x32b
  const uint32_t w0 = 0xA0000000u | (lane << 8) | 0, w1 = 0xA0000000u | (lane << 8) | 1;
  asm volatile("tcgen05.st.sync.aligned.16x32bx2.x2.b32 [%0], 8, {%1,%2};" ::"r"(t + 64), "r"(w0), "r"(w1));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  for (int c = 0; c < 12; ++c) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(t + 64 + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    out[128 + lane * 12 + c] = v;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncwarp();
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(t));
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 4096 * 4);
  cudaMemset(d, 0xff, 4096 * 4);
  probe<<<1, 32>>>(d);
  uint32_t h[4096];
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  printf("ld 16x32bx2.x4 imm 32: thread -> (lane, col) x4\n");
  for (int l = 0; l < 32; ++l) {
    printf("t%02d:", l);
    for (int i = 0; i < 4; ++i) printf(" (%u,%u)", h[l * 4 + i] >> 16, h[l * 4 + i] & 0xffff);
    printf("\n");
  }
  printf("st 16x32bx2.x2 imm 8 at col 64: lane -> cols 64..75 (writer thread, reg) or -\n");
  for (int l = 0; l < 32; ++l) {
    printf("L%02d:", l);
    for (int c = 0; c < 12; ++c) {
      uint32_t v = h[128 + l * 12 + c];
      if ((v >> 28) == 0xA) printf(" t%u.r%u", (v >> 8) & 0xff, v & 0xff);
      else printf(" -");
    }
    printf("\n");
  }
  return 0;
}
