// umma_rate.cu -- development probe (not part of the product): issue rate of
// tcgen05.mma kind::tf32 (K = 8 per instruction) from K-major, non-swizzled
// shared-memory operands, as a function of M and N, with 1 or 2 CTAs per SM.
// One thread per CTA issues `reps` MMAs back to back (cycling over 4 operand
// buffers), one commit, clock64 around it.  Prints cycles per MMA and the
// implied MAC/clk per SM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/umma_rate tools/umma_rate.cu && /tmp/umma_rate
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ inline uint64_t desc_kmajor(uint32_t saddr, int R) {
  const uint64_t lbo = (uint64_t)(R / 8 * 128) >> 4, sbo = 128 >> 4;
  return (uint64_t)((saddr >> 4) & 0x3fff) | (lbo << 16) | (sbo << 32) | (1ull << 46);
}

__global__ void rate(int M, int N, int reps, int issuers, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 4 * (M + N) * 8; i += blockDim.x) ((float*)sm)[i] = 1.0f + (i & 7) * 0.125f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "n"(256));
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
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  long long t0 = clock64();
  if ((tid & 31) == 0 && warp < issuers) {
    for (int r = 0; r < reps; ++r) {
      const int b = r & 3;
      const uint32_t a = smem_u32(sm) + b * M * 32, bb = smem_u32(sm) + 4 * M * 32 + b * N * 32;
      const uint64_t da = desc_kmajor(a, M), db = desc_kmajor(bb, N);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm + (uint32_t)(warp * (256 / issuers))),
                   "l"(da), "l"(db), "r"(idesc), "r"(1u));
    }
  }
  __syncthreads();
  if (tid == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  __syncwarp();
  asm volatile("{\n\t.reg .pred P1;\n\tWAIT:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@!P1 bra WAIT;\n\t}" ::"r"(smem_u32(&mbar)), "r"(0));
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(256));
}

int main() {
  long long* dc;
  cudaMalloc(&dc, 4096 * 8);
  const int reps = 4096;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Cfg { int per_sm, issuers, M, N; };
  const Cfg cfgs[] = {{1, 1, 128, 16}, {1, 2, 128, 16}, {1, 4, 128, 16}, {2, 1, 128, 16}, {2, 2, 128, 16}, {4, 1, 128, 16},
                      {1, 1, 128, 32}, {1, 2, 128, 32}, {1, 4, 128, 32}, {4, 1, 128, 32},
                      {1, 1, 128, 64}, {1, 2, 128, 64}, {1, 4, 128, 64}, {1, 2, 64, 64}, {1, 4, 64, 64}, {1, 2, 128, 112}, {1, 2, 64, 256}};
  for (const Cfg& c : cfgs) {
    const int M = c.M, N = c.N, per_sm = c.per_sm;
    const int smem = per_sm == 1 ? 200 * 1024 : per_sm == 2 ? 100 * 1024 : 50 * 1024;
    const int grid = 148 * per_sm;
    rate<<<grid, 128, smem>>>(M, N, reps, c.issuers, dc);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("error M=%d N=%d\n", M, N); return 1; }
    std::vector<long long> cv(grid);
    cudaMemcpy(cv.data(), dc, grid * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (long long v : cv) avg += v;
    avg /= grid;
    const double mm_per_sm = (double)per_sm * c.issuers * reps;
    printf("CTAs/SM %d issuers/CTA %d  M %3d  N %3d: %6.1f cycles per MMA per SM -> %7.1f MAC/clk/SM\n", per_sm,
           c.issuers, M, N, avg / mm_per_sm, mm_per_sm * M * N * 8 / avg);
  }
  return 0;
}
