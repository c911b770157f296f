// umma_probe.cu -- development probe for the tensor-core M2L (not part of the
// product): one CTA runs D[128 x 112] = A[128 x K] . B[112 x K]^T with
// tcgen05.mma kind::tf32 from K-major, non-swizzled core-matrix smem layouts,
// the FP32 accumulator in TMEM, read back with tcgen05.ld.32x32b.  Checks the
// descriptors against a double-precision host product, 1xTF32 and 3xTF32
// (hi/lo split), then times back-to-back MMAs (clock64) for the issue rate.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/umma_probe tools/umma_probe.cu && /tmp/umma_probe
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 112, K = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, SWIZZLE_NONE: element (r, k) of an R-row tile at
//   (k/4) * (R/8 * 128) + (r/8) * 128 + (r%8) * 16 + (k%4) * 4   bytes
// => core matrices of 8 rows x 16 B; LBO = R/8*128 (next 16-B K chunk), SBO = 128 (next 8 rows)
__host__ __device__ inline int off_kmajor(int r, int k, int R) { return (k / 4) * (R / 8 * 128) + (r / 8) * 128 + (r % 8) * 16 + (k % 4) * 4; }

__device__ inline uint64_t desc_kmajor(uint32_t saddr, int R) {
  const uint64_t lbo = (uint64_t)(R / 8 * 128) >> 4, sbo = 128 >> 4;
  return (uint64_t)((saddr >> 4) & 0x3fff) | (lbo << 16) | (sbo << 32) | (1ull << 46);   // version 1, no swizzle
}

__device__ inline float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

__global__ void probe(const float* A, const float* B, float* D1, float* D3, float* Dacc, int racc, long long* cyc,
                      int reps, int raw_hi) {
  extern __shared__ __align__(1024) uint8_t sm[];
  float* Ah = (float*)sm;                       // M x K
  float* Al = (float*)(sm + M * K * 4);
  float* Bh = (float*)(sm + 2 * M * K * 4);     // N x K
  float* Bl = (float*)(sm + 2 * M * K * 4 + N * K * 4);
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float v = A[i], h = tf32_hi(v);
    *(float*)((uint8_t*)Ah + off_kmajor(r, k, M)) = raw_hi ? v : h;   // raw: the tensor core reads x as TF32 itself
    *(float*)((uint8_t*)Al + off_kmajor(r, k, M)) = v - h;
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float v = B[i], h = tf32_hi(v);
    *(float*)((uint8_t*)Bh + off_kmajor(r, k, N)) = h;
    *(float*)((uint8_t*)Bl + off_kmajor(r, k, N)) = v - h;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  // instruction descriptor: F32 accumulate, TF32 A/B, K-major both, N>>3, M>>4
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  uint32_t phase = 0;
  auto mma = [&](uint32_t dcol, const float* a, const float* b, int ks, bool acc) {
    const uint64_t da = desc_kmajor(smem_u32(a) + ks * 2 * (M / 8 * 128), M);
    const uint64_t db = desc_kmajor(smem_u32(b) + ks * 2 * (N / 8 * 128), N);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm + dcol),
                 "l"(da), "l"(db), "r"(idesc), "r"((uint32_t)acc));
  };
  auto commit_wait = [&]() {
    if (tid == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
    asm volatile("{\n\t.reg .pred P1;\n\tWAIT:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@!P1 bra WAIT;\n\t}" ::"r"(smem_u32(&mbar)), "r"(phase));
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
  };
  if (tid == 0) {
    for (int ks = 0; ks < K / 8; ++ks) mma(0, Ah, Bh, ks, ks > 0);          // 1xTF32 into columns [0, N)
    for (int ks = 0; ks < K / 8; ++ks) {                                    // 3xTF32 into columns [128, 128+N)
      mma(128, Ah, Bh, ks, ks > 0);
      mma(128, Al, Bh, ks, true);
      mma(128, Ah, Bl, ks, true);
    }
  }
  __syncwarp();
  commit_wait();
  // accumulation drift: the 3xTF32 product added racc times into columns [256, 256 + N)
  if (tid == 0)
    for (int r = 0; r < racc; ++r)
      for (int ks = 0; ks < K / 8; ++ks) {
        mma(256, Ah, Bh, ks, r > 0 || ks > 0);
        mma(256, Al, Bh, ks, true);
        mma(256, Ah, Bl, ks, true);
      }
  __syncwarp();
  commit_wait();
  if (warp < 4) {
    const int row = warp * 32 + (tid % 32);
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t v[16];
      const uint32_t addr = tm + ((uint32_t)(warp * 32) << 16) + 256 + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 16; ++j) Dacc[row * N + c0 + j] = __uint_as_float(v[j]);
    }
  }
  if (warp < 4) {
    const int row = warp * 32 + (tid % 32);
    for (int part = 0; part < 2; ++part) {
      for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        const uint32_t addr = tm + ((uint32_t)(warp * 32) << 16) + part * 128 + c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        float* D = part ? D3 : D1;
        for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
      }
    }
  }
  // timing: reps x (K/8) MMAs back to back, one commit
  __syncthreads();
  long long t0 = clock64();
  if (tid == 0)
    for (int r = 0; r < reps; ++r)
      for (int ks = 0; ks < K / 8; ++ks) mma(256 - 256 + 0, Ah, Bh, ks, true);
  __syncwarp();
  commit_wait();
  long long t1 = clock64();
  if (tid == 0) *cyc = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(512));
}

int main(int argc, char** argv) {
  std::vector<float> A(M * K), B(N * K);
  srand(1106);
  for (auto& v : A) v = (float)((rand() / (double)RAND_MAX - 0.5) * pow(10.0, (rand() % 7) - 3));
  for (auto& v : B) v = (float)((rand() / (double)RAND_MAX - 0.5) * pow(10.0, (rand() % 5) - 2));
  float *dA, *dB, *d1, *d3, *dacc;
  long long* dc;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&d1, M * N * 4); cudaMalloc(&d3, M * N * 4); cudaMalloc(&dc, 8);
  cudaMalloc(&dacc, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 2 * M * K * 4 + 2 * N * K * 4;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 2000;
  const int racc = argc > 1 ? atoi(argv[1]) : 1000;
  const int raw_hi = argc > 2 ? atoi(argv[2]) : 0;
  probe<<<1, 128, smem>>>(dA, dB, d1, d3, dacc, racc, dc, reps, raw_hi);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> D1(M * N), D3(M * N);
  long long cyc;
  cudaMemcpy(D1.data(), d1, M * N * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(D3.data(), d3, M * N * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  double e1 = 0, e3 = 0, nr = 0, ea = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0, sa = 0;
      for (int k = 0; k < K; ++k) { s += (double)A[i * K + k] * B[j * K + k]; sa += fabs((double)A[i * K + k] * B[j * K + k]); }
      e1 += (D1[i * N + j] - s) * (D1[i * N + j] - s);
      e3 += (D3[i * N + j] - s) * (D3[i * N + j] - s);
      nr += s * s;
      ea = fmax(ea, fabs(D3[i * N + j] - s) / sa);
    }
  std::vector<float> Dc(M * N);
  cudaMemcpy(Dc.data(), dacc, M * N * 4, cudaMemcpyDeviceToHost);
  {
    double e = 0, nr = 0, bias = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * B[j * K + k];
        s *= racc;
        e += (Dc[i * N + j] - s) * (Dc[i * N + j] - s);
        nr += s * s;
        bias += (fabs(Dc[i * N + j]) - fabs(s)) / (fabs(s) + 1e-30);
      }
    printf("accumulating %d x (3xTF32, K=%d) = %d MMAs into one accumulator: rel-L2 %.3e, mean rel |.| bias %.3e\n",
           racc, K, racc * K / 8 * 3, sqrt(e / nr), bias / (M * N));
  }
  printf("rel-L2 error 1xTF32 %.3e  3xTF32 %.3e  (max |err|/sum|ab| 3x %.3e)\n", sqrt(e1 / nr), sqrt(e3 / nr), ea);
  const double macs = (double)reps * (K / 8) * M * N * 8;
  printf("timing: %d MMAs (128x%dx8 tf32) in %lld cycles = %.1f cycles/MMA = %.0f MAC/clk/SM\n", reps * (K / 8), N, cyc,
         (double)cyc / (reps * (K / 8)), macs / cyc);
  return 0;
}
