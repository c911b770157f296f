// Micro-probe: sustained FP32 FMA throughput of FFMA vs FFMA2 (fma.rn.f32x2)
// on this B200, to set the issue-slot model of the P2P/M2L kernels.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ffma(float* out, int iters, float a, float b) {
  float x[16];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0; for (int i = 0; i < 16; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ unsigned long long f2(unsigned long long x, unsigned long long y, unsigned long long z) {
  unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(y), "l"(z)); return d;
}
__global__ void k_ffma2(float* out, int iters, float a, float b) {
  unsigned long long x[8];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  unsigned long long A = *(unsigned long long*)&av, B = *(unsigned long long*)&bv;
  for (int i = 0; i < 8; ++i) { float2 v = make_float2(threadIdx.x * 1e-3f + i, i + 0.5f); x[i] = *(unsigned long long*)&v; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = f2(x[i], A, B);
  }
  float s = 0; for (int i = 0; i < 8; ++i) { float2 v = *(float2*)&x[i]; s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int which = 0; which < 2; ++which) {
      cudaEventRecord(e0);
      if (which == 0) k_ffma<<<148 * 8, 256>>>(out, iters, 0.999f, 0.001f);
      else k_ffma2<<<148 * 8, 256>>>(out, iters, 0.999f, 0.001f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 16 * iters * 148.0 * 8 * 256;
      if (rep) printf("%s: %.3f ms  %.1f TFLOP/s\n", which ? "FFMA2" : "FFMA ", ms, fl / ms / 1e9);
    }
  }
  return 0;
}
