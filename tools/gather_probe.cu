// gather_probe.cu -- development probe (not part of the product): TMA
// tile::gather4 of 4 arbitrary 32-byte rows per op into a SWIZZLE_32B K-major
// UMMA operand, consumed by tcgen05.mma kind::tf32; checks D = A.B^T on the host.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/gp tools/gather_probe.cu -lcuda && /tmp/gp
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

constexpr int M = 128, N = 112, K = 8, NROWS = 4096, W = 24;   // table [NROWS][24 floats], one 8-float column block per op

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tmap, const int* rows, int col, const float* B, float* D) {
  __shared__ __align__(1024) float As[M * K];         // SW32 K-major: row r at 32 r bytes (16-B chunks swizzled)
  __shared__ __align__(1024) float Bs[N * K];         // no swizzle, core matrices
  __shared__ uint64_t mbar, mdone;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int j = i / K, k = i % K;
    Bs[((k / 4) * (N / 8 * 128) + (j / 8) * 128 + (j % 8) * 16 + (k % 4) * 4) / 4] = B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&mbar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&mdone)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(su(&mbar)),
                 "r"(M * K * 4));
    for (int g = 0; g < M / 4; ++g)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su(As + g * 4 * K)),
          "l"(&tmap), "r"(su(&mbar)), "r"(col), "r"(rows[4 * g]), "r"(rows[4 * g + 1]), "r"(rows[4 * g + 2]),
          "r"(rows[4 * g + 3])
          : "memory");
  }
  asm volatile("{\n\t.reg .pred P1;\n\tW1:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W1;\n\t}" ::"r"(
      su(&mbar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (tid == 0) {
    // A: SWIZZLE_32B (layout type 6), K-major: SBO = 256 B between 8-row groups, LBO unused (1)
    const uint64_t da = (uint64_t)((su(As) >> 4) & 0x3fff) | (1ull << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46) |
                        (6ull << 61);
    const uint64_t db = (uint64_t)((su(Bs) >> 4) & 0x3fff) | ((uint64_t)((N / 8 * 128) >> 4) << 16) |
                        ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da), "l"(db), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&mdone)));
  }
  __syncwarp();
  asm volatile("{\n\t.reg .pred P1;\n\tW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W2;\n\t}" ::"r"(
      su(&mdone)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    const int row = warp * 32 + (tid % 32);
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t v[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(tm + ((uint32_t)(warp * 32) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  std::vector<float> G((size_t)NROWS * W), Bh((size_t)N * K);
  srand(5273);
  for (auto& v : G) v = (float)((rand() / (double)RAND_MAX - 0.5) * 4);
  for (auto& v : Bh) v = (float)((rand() / (double)RAND_MAX - 0.5) * 4);
  std::vector<int> rows(M);
  for (int i = 0; i < M; ++i) rows[i] = rand() % NROWS;
  const int col = 8;                                           // the second 8-float block of each row
  float *dG, *dB, *dD;
  int* dR;
  cudaMalloc(&dG, G.size() * 4); cudaMalloc(&dB, Bh.size() * 4); cudaMalloc(&dD, M * N * 4); cudaMalloc(&dR, M * 4);
  cudaMemcpy(dG, G.data(), G.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bh.data(), Bh.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dR, rows.data(), M * 4, cudaMemcpyHostToDevice);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
  CUtensorMap tmap;
  cuuint64_t gdim[2] = {(cuuint64_t)W, (cuuint64_t)NROWS};
  cuuint64_t gstr[1] = {(cuuint64_t)W * 4};
  cuuint32_t box[2] = {8, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dG, gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  // host copy of the row indices for the kernel's immediate use
  int* hrows;
  cudaMallocManaged(&hrows, M * 4);
  for (int i = 0; i < M; ++i) hrows[i] = rows[i];
  probe<<<1, 128>>>(tmap, hrows, col, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> D(M * N);
  cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  double en = 0, nr = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)G[(size_t)rows[i] * W + col + k] * Bh[j * K + k];
      en += (D[i * N + j] - s) * (D[i * N + j] - s);
      nr += s * s;
    }
  printf("gather4 + SW32 UMMA: rel-L2 error %.3e (1xTF32 level ~1e-3 expected)\n", sqrt(en / nr));
  return 0;
}
