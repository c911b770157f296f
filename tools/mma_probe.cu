// Micro-probe: throughput of the legacy warp-level TF32 MMA (mma.sync m16n8k8)
// on this B200, to decide whether an M2L on warp MMAs could beat the FP32 SIMT path.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_mma(float* out, int iters) {
  unsigned a0 = __float_as_uint(1.0f + threadIdx.x * 1e-3f), a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3;
  unsigned b0 = __float_as_uint(0.5f), b1 = b0 ^ 1;
  float c[8][4];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mma_bf16(float* out, int iters) {
  unsigned a0 = 0x3f803f80u + threadIdx.x, a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3, b0 = 0x3f003f00u, b1 = b0 ^ 1;
  float c[8][4];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0);
      if (w == 0) k_mma<<<148 * 8, 256>>>(out, iters); else k_mma_bf16<<<148 * 8, 256>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = (w == 0 ? 2.0 * 16 * 8 * 8 : 2.0 * 16 * 8 * 16) * 8 * iters * (148.0 * 8 * 256 / 32);
      if (rep) printf("%s mma.sync: %.3f ms  %.1f TFLOP/s\n", w ? "BF16" : "TF32", ms, fl / ms / 1e9);
    }
  }
  return 0;
}
