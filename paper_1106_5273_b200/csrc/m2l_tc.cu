// m2l_tc.cu -- a9 (M2L) on the 5th-generation tensor cores for
// the levels where every target cell sees the same set of source offsets.
//
// In a uniform periodic octree every cell of a level has the same M2L
// interaction list up to translation: the same D offsets (source level and
// centre offset Delta), in some traversal order.  For a fixed offset d the
// M2L translation is a fixed real-linear map T_d from the source multipole
// (p(p+1)/2 complex = 110 reals at p = 10, component-wise) to the target local
// expansion, so for a level the whole M2L is one dense contraction
//
//   L[(t, c), j] += sum_d sum_i  M[(src(t, d), c), i]  T_d[j, i]
//
// with K = D x 112 (110 padded): the shape tcgen05.mma wants.  Rows are
// (target cell, vorticity component), 512 per CTA as four 128-row
// accumulators (4 x 112 of the 512 TMEM columns); the operator T_d is built
// once per level in double precision from I_{n+k}^{m+l}(D) with the
// (-1)^k sign and the (s_s/s_t)^n scale of P:228 folded in.
//
// Precision (3xTF32): every operand is split x = hi + lo, hi = x with the 13
// low mantissa bits cleared (exactly a TF32 value), lo = x - hi; the product
// is accumulated as hi.hi + lo.hi + hi.lo in FP32 in TMEM (relative error
// ~2^-21, FP32-level; 1xTF32 would be ~1e-3, tools/umma_probe.cu).
//
// Pipeline (one CTA per SM, 17 warps): warps 0-15 own one row each -- they
// gather the row's 8 multipole reals of the current K-block from global
// memory (prefetched two stages ahead), split them and store hi/lo into the
// stage's A tiles (K-major core-matrix layout, no swizzle); thread 0 also
// starts the bulk copy (cp.async.bulk + mbarrier tx count) of the stage's
// pre-split operator slice.  Warp 16 allocates TMEM and one thread issues the
// 12 MMAs of a stage (4 accumulators x 3 products), committing to the stage's
// "empty" mbarrier.  Every kChunk offsets the producers drain the
// accumulators (TMEM lane quarter = warp % 4) into Lc and the MMAs restart.
//
// Which cells take this path is decided per list build: a reference cell's
// offsets define the level's canonical set; a verification kernel checks,
// for every cell of the level, that its list has exactly those offsets and
// that the source the tensor kernel will compute (Morton index of the
// offset cell in the level-ordered cell array) is the list's source.  Cells
// that fail (adaptive trees, partial levels, other ranks' cells) stay on the
// register kernel (m2l.cu), which skips the cells taken here.
#include <algorithm>
#include <cstring>

#include "ctx.cuh"

namespace fmmb {

namespace {

constexpr int kRows = 512;                  // rows (target, component) per CTA
constexpr int kN = 112;                     // local-expansion reals (110 at p = 10, padded)
constexpr int kKB = 8;                      // K per stage (one kind::tf32 MMA)
constexpr int kNKB = 14;                    // K-blocks per offset (112 / 8)
constexpr int kStages = 4;
constexpr int kATile = 128 * kKB * 4;       // one 128-row A tile (hi or lo), bytes
constexpr int kAStage = 4 * 2 * kATile;     // 4 accumulators x (hi, lo)
constexpr int kBHalf = kN * kKB * 4;        // operator slice (hi or lo), bytes
constexpr int kStage = kAStage + 2 * kBHalf;
constexpr int kThreads = kRows + 32;
constexpr int kChunk = 16;                  // offsets accumulated in TMEM between drains
constexpr int kMaxTcLevels = 32;   // (level, parity class) groups
constexpr int kTcP = 10;                    // the tensor path is instantiated for p = 10

// ---------------------------------------------------------------- PTX ----
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(saddr(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra LAB_WAIT;\n\t}" ::"r"(saddr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   saddr(dst)),
               "l"(src), "r"(bytes), "r"(saddr(bar))
               : "memory");
}
// K-major, no-swizzle operand: core matrices of 8 rows x 16 B; LBO = next
// 16-byte K chunk, SBO = next 8 rows (128 B).
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(b))
               : "memory");
}
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// ------------------------------------------------------------ geometry ----
struct TcGeo {
  const int *qx, *qy, *qz, *level;
  long long per[3];                 // periods in half-finest-cell units
  int lvl_begin[kMaxLevel + 2];
};

__device__ __forceinline__ uint32_t spread3_32(uint32_t v) {   // 10-bit spread (levels <= 10)
  v &= 0x3ff;
  v = (v | (v << 16)) & 0x030000ff;
  v = (v | (v << 8)) & 0x0300f00f;
  v = (v | (v << 4)) & 0x030c30c3;
  v = (v | (v << 2)) & 0x09249249;
  return v;
}

// offset code: (dl + 1) << 21 | (vx + 64) << 14 | (vy + 64) << 7 | (vz + 64),
// dl = level_s - level_t in {-1, 0, 1}, v = Delta / 2^(21 - max(lt, ls)) with
// Delta = c_t - c_s - image shift in half-finest-cell units.
__device__ __forceinline__ int code_dl(int code) { return (code >> 21) - 1; }
__device__ __forceinline__ int code_v(int code, int a) { return ((code >> (14 - 7 * a)) & 127) - 64; }

// the cell the tensor kernel reads for target t (centre ct) and offset code:
// c_s = c_t - Delta wrapped into the period, its level-ls Morton index
__device__ __forceinline__ int tc_source(const TcGeo& g, int lt, const long long (&ct)[3], int code) {
  const int dl = code_dl(code), ls = lt + dl, lf = max(lt, ls);
  uint32_t q[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    long long cs = ct[a] - (long long)code_v(code, a) * (1ll << (kMaxLevel - lf));
    const long long P = g.per[a];
    cs %= P;
    if (cs < 0) cs += P;
    q[a] = (uint32_t)(((cs >> (kMaxLevel - ls)) - 1) >> 1);
  }
  return g.lvl_begin[ls] + (int)(spread3_32(q[0]) | (spread3_32(q[1]) << 1) | (spread3_32(q[2]) << 2));
}

// code of one M2L list entry (or -1 if outside the encodable range)
__device__ __forceinline__ int entry_code(const TcGeo& g, int lt, const long long (&ct)[3], uint64_t ent) {
  const int src = (int)((ent >> 5) & 0x7ffffff), img = (int)(ent & 31);
  const int ls = g.level[src], dl = ls - lt;
  if (dl < -1 || dl > 1) return -1;
  const int lf = max(lt, ls);
  const int qs[3] = {g.qx[src], g.qy[src], g.qz[src]};
  const int im[3] = {img % 3 - 1, (img / 3) % 3 - 1, img / 9 - 1};
  int code = (dl + 1) << 21;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const long long cs = (long long)(2 * qs[a] + 1) << (kMaxLevel - ls);
    const long long d = ct[a] - cs - (long long)im[a] * g.per[a];
    const long long u = 1ll << (kMaxLevel - lf);
    if (d % u != 0) return -1;
    const long long v = d / u;
    if (v < -63 || v > 63) return -1;
    code |= (int)(v + 64) << (14 - 7 * a);
  }
  return code;
}

__device__ __forceinline__ void centre(const TcGeo& g, int cell, int lt, long long (&ct)[3]) {
  ct[0] = (long long)(2 * g.qx[cell] + 1) << (kMaxLevel - lt);
  ct[1] = (long long)(2 * g.qy[cell] + 1) << (kMaxLevel - lt);
  ct[2] = (long long)(2 * g.qz[cell] + 1) << (kMaxLevel - lt);
}

// codes of one cell's entries (the level's reference cell)
__global__ void k_tc_ref_codes(const uint64_t* __restrict__ lst, const int* __restrict__ seg_b,
                               const int* __restrict__ seg_e, int cell, int lt, TcGeo g, int* __restrict__ out) {
  long long ct[3];
  centre(g, cell, lt, ct);
  const int b = seg_b[cell], e = seg_e[cell];
  for (int i = b + threadIdx.x; i < e; i += blockDim.x) out[i - b] = entry_code(g, lt, ct, lst[i]);
}

// parity class of a cell: its octant within the parent (the interaction
// list of a cell depends on it, so each class has its own offset set)
__device__ __forceinline__ int parity_class(const TcGeo& g, int c) {
  return (g.qx[c] & 1) | ((g.qy[c] & 1) << 1) | ((g.qz[c] & 1) << 2);
}

// per class: first cell of [lb, le) with a non-empty list
__global__ void k_tc_first(const int* __restrict__ seg_b, const int* __restrict__ seg_e, int lb, int le, TcGeo g,
                           int* __restrict__ out) {
  for (int c = lb + blockIdx.x * blockDim.x + threadIdx.x; c < le; c += gridDim.x * blockDim.x)
    if (seg_e[c] > seg_b[c]) atomicMin(out + parity_class(g, c), c);
}

// per cell: its list is exactly the canonical offsets and every source is
// the one tc_source computes.  Warp per cell; ok cells are appended to tgt.
__global__ void k_tc_verify(const uint64_t* __restrict__ lst, const int* __restrict__ seg_b,
                            const int* __restrict__ seg_e, int lb, int le, int lt, int D, TcGeo g,
                            const short* __restrict__ tbl, int R, int cls, unsigned char* __restrict__ skip,
                            int* __restrict__ tgt, int* __restrict__ ntgt) {
  const int lane = threadIdx.x & 31;
  const int V = 2 * R + 1;
  for (int c = lb + (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); c < le;
       c += (int)((gridDim.x * blockDim.x) >> 5)) {
    if (parity_class(g, c) != cls) continue;
    const int b = seg_b[c], e = seg_e[c];
    bool ok = (e - b) == D;
    long long ct[3];
    centre(g, c, lt, ct);
    for (int i = b + lane; ok && i < e; i += 32) {
      const uint64_t ent = lst[i];
      const int code = entry_code(g, lt, ct, ent);
      bool good = code >= 0;
      if (good) {
        const int dl = code_dl(code), vx = code_v(code, 0), vy = code_v(code, 1), vz = code_v(code, 2);
        good = vx >= -R && vx <= R && vy >= -R && vy <= R && vz >= -R && vz <= R;
        if (good) good = tbl[(((dl + 1) * V + vx + R) * V + vy + R) * V + vz + R] >= 0;
        if (good) good = tc_source(g, lt, ct, code) == (int)((ent >> 5) & 0x7ffffff);
      }
      ok = ok && good;
    }
    ok = __all_sync(0xffffffffu, ok);
    if (lane == 0 && ok) {
      skip[c] = 1;
      tgt[atomicAdd(ntgt, 1)] = c;
    }
  }
}

// operator of one level: T_d[j][i] split into TF32 hi/lo, stored per (d, K-block)
// in the stage layout  [hi | lo] x [K chunk (2)][row group (14)][8 rows][4 floats].
__global__ void k_tc_operator(const int* __restrict__ codes, int lt, unsigned char* __restrict__ op) {
  constexpr int P = kTcP, NC = P * (P + 1) / 2;
  const int d = blockIdx.x;
  const int code = codes[d];
  const int dl = code_dl(code);
  __shared__ double2 I[NC];
  __shared__ double Dv[3];
  if (threadIdx.x < 3) Dv[threadIdx.x] = (double)code_v(code, threadIdx.x) / (double)(1 << (1 + max(0, dl)));
  __syncthreads();
  // irregular harmonics I_n^m(D), n <= p-1 (same recursion as the FP32 kernels, in double)
  if (threadIdx.x < P) {
    const int m = threadIdx.x;
    const double x = Dv[0], y = Dv[1], z = Dv[2];
    const double r2 = x * x + y * y + z * z, ir2 = 1.0 / r2;
    double dr = 1.0 / sqrt(r2), di = 0.0;
    for (int i = 1; i <= m; ++i) {
      const double s = -(double)(2 * i - 1) * ir2;
      const double nr = s * (x * dr - y * di), ni = s * (x * di + y * dr);
      dr = nr;
      di = ni;
    }
    I[ci(m, m)] = make_double2(dr, di);
    if (m + 1 < P) {
      double ar = (2 * m + 1) * z * ir2 * dr, ai = (2 * m + 1) * z * ir2 * di;
      I[ci(m + 1, m)] = make_double2(ar, ai);
      double br = dr, bi = di;
      for (int n = m + 2; n < P; ++n) {
        const double c1 = (double)(2 * n - 1) * z, c2 = (double)(n - 1 - m) * (double)(n - 1 + m);
        const double vr = (c1 * ar - c2 * br) * ir2, vi = (c1 * ai - c2 * bi) * ir2;
        I[ci(n, m)] = make_double2(vr, vi);
        br = ar; bi = ai;
        ar = vr; ai = vi;
      }
    }
  }
  __syncthreads();
  auto Iget = [&](int j, int mm) -> double2 {
    if (mm > j || -mm > j) return make_double2(0.0, 0.0);
    if (mm >= 0) return I[ci(j, mm)];
    const double2 v = I[ci(j, -mm)];
    const double s = (mm & 1) ? -1.0 : 1.0;           // I_j^{-m} = (-1)^m conj(I_j^m)
    return make_double2(s * v.x, -s * v.y);
  };
  const double ratio = ldexp(1.0, -dl);                 // s_s / s_t
  unsigned char* base = op + (size_t)d * kNKB * 2 * kBHalf;
  for (int idx = threadIdx.x; idx < kN * kN; idx += blockDim.x) {
    const int j = idx / kN, i = idx - kN * (idx / kN);
    double v = 0.0;
    if (j < 2 * NC && i < 2 * NC) {
      const int oj = j >> 1, oi = i >> 1;
      int k = 0;
      while ((k + 1) * (k + 2) / 2 <= oj) ++k;
      const int l = oj - k * (k + 1) / 2;
      int n = 0;
      while ((n + 1) * (n + 2) / 2 <= oi) ++n;
      const int m = oi - n * (n + 1) / 2;
      if (n + k <= P - 1) {
        const double2 X = Iget(n + k, m + l);
        const double2 Y = m > 0 ? Iget(n + k, l - m) : make_double2(0.0, 0.0);
        const double cs = (m & 1) ? -1.0 : 1.0;
        const bool re = (j & 1) == 0, a = (i & 1) == 0;
        // L += M X + [m > 0] (-1)^m conj(M) Y,  M = a + i b
        if (re) v = a ? X.x + cs * Y.x : -X.y + cs * Y.y;
        else v = a ? X.y + cs * Y.y : X.x - cs * Y.x;
        v *= ((k & 1) ? -1.0 : 1.0) * pow(ratio, n);
      }
    }
    const float vf = (float)v, hi = tf32_hi(vf), lo = (float)(v - (double)hi);
    const int kb = i / kKB, kk = i % kKB;
    const size_t off = (size_t)kb * 2 * kBHalf + (kk / 4) * (kN / 8 * 128) + (j / 8) * 128 + (j % 8) * 16 + (kk % 4) * 4;
    *(float*)(base + off) = hi;
    *(float*)(base + off + kBHalf) = lo;
  }
}

// ------------------------------------------------------- tensor kernel ----
struct TcLevelArg {
  const int* tgt;
  const int* codes;
  const unsigned char* op;
  int ntgt, lt, D, cta_begin;
};
struct TcArgs {
  TcLevelArg lv[kMaxTcLevels];
  int nlv;
};

__global__ void __launch_bounds__(kThreads, 1) k_m2l_tc(TcArgs args, TcGeo g, const float2* __restrict__ M,
                                                        float2* __restrict__ Lc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full[kStages], empty[kStages], chunk_full, drained;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  // this CTA's level (levels are laid out back to back, longest first)
  int li = 0;
  while (li + 1 < args.nlv && (int)blockIdx.x >= args.lv[li + 1].cta_begin) ++li;
  const TcLevelArg A = args.lv[li];
  const int nit = A.D * kNKB;

  if (warp == kRows / 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], kRows);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&chunk_full, 1);
    mbar_init(&drained, kRows);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;

  if (warp < kRows / 32) {
    // ------------------------------------------------ producers (one row each)
    const int row = (int)blockIdx.x - A.cta_begin;
    const int R = row * kRows + tid;
    const bool valid = R < 3 * A.ntgt;
    const int t = valid ? R / 3 : 0, comp = valid ? R - 3 * (R / 3) : 0;
    const int cell = A.tgt[t];
    long long ct[3];
    centre(g, cell, A.lt, ct);
    const int tau = tid >> 7, rr = tid & 127;
    const int arow = (rr >> 3) * 128 + (rr & 7) * 16;   // byte offset of this row's 16-byte chunk 0
    int pf_d = -1;
    const float2* pf_src = M;
    auto load = [&](int it, float2 (&v)[4]) {
      const int d = it / kNKB, kb = it - kNKB * (it / kNKB);
      if (d != pf_d) {
        pf_d = d;
        const int src = tc_source(g, A.lt, ct, __ldg(A.codes + d));
        pf_src = M + ((size_t)src * 3 + comp) * 55;
      }
      const float2* p = pf_src + kb * 4;
      v[0] = __ldg(p);
      v[1] = __ldg(p + 1);
      v[2] = __ldg(p + 2);
      v[3] = kb == kNKB - 1 ? make_float2(0.f, 0.f) : __ldg(p + 3);   // reals 110, 111 are padding
    };
    // drain: add the accumulator of the finished chunk into Lc.  The tensor
    // cores accumulate FP32 with truncation, so the error grows with the
    // number of MMAs per accumulator (tools/umma_probe.cu: ~1e-8 per MMA);
    // draining every kChunk offsets keeps it at the FP32 register kernel's level.
    const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(tau * 128);
    float2* out = Lc + ((size_t)cell * 3 + comp) * 55;
    auto drain = [&](int chunk) {
      mbar_wait(&chunk_full, chunk & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
      for (int c0 = 0; c0 < kN; c0 += 16) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (valid) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int o = c0 / 2 + q;
            if (o < 55) {
              float2 w = out[o];
              w.x += __uint_as_float(v[2 * q]);
              w.y += __uint_as_float(v[2 * q + 1]);
              out[o] = w;
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(&drained);
    };
    float2 va[4], vb[4], vc[4];
    if (nit > 0) load(0, va);
    if (nit > 1) load(1, vb);
    for (int it = 0; it < nit; ++it) {
      if (it > 0 && it % (kChunk * kNKB) == 0) drain(it / (kChunk * kNKB) - 1);
      if (it + 2 < nit) load(it + 2, vc);
      const int s = it % kStages;
      if (it >= kStages) mbar_wait(&empty[s], ((it / kStages) - 1) & 1);
      unsigned char* st = smem + (size_t)s * kStage;
      // hi / lo split, chunk c holds reals 4c..4c+3 of the K-block
      const float x[8] = {va[0].x, va[0].y, va[1].x, va[1].y, va[2].x, va[2].y, va[3].x, va[3].y};
      float h[8], l[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        h[q] = tf32_hi(x[q]);
        l[q] = x[q] - h[q];
      }
      unsigned char* ah = st + (tau * 2 + 0) * kATile + arow;
      unsigned char* al = st + (tau * 2 + 1) * kATile + arow;
      *(float4*)ah = make_float4(h[0], h[1], h[2], h[3]);
      *(float4*)(ah + 2048) = make_float4(h[4], h[5], h[6], h[7]);
      *(float4*)al = make_float4(l[0], l[1], l[2], l[3]);
      *(float4*)(al + 2048) = make_float4(l[4], l[5], l[6], l[7]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (tid == 0) {
        const int d = it / kNKB, kb = it - kNKB * (it / kNKB);
        mbar_arrive_tx(&full[s], 2 * kBHalf);
        bulk_g2s(st + kAStage, A.op + ((size_t)d * kNKB + kb) * 2 * kBHalf, 2 * kBHalf, &full[s]);
      } else {
        mbar_arrive(&full[s]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) { va[q] = vb[q]; vb[q] = vc[q]; }
    }
    // ------------------------------------------------ epilogue: the last chunk
    if (nit > 0) drain((nit - 1) / (kChunk * kNKB));
  } else if (tid == kRows) {
    // ------------------------------------------------ MMA issuer
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    for (int it = 0; it < nit; ++it) {
      const int s = it % kStages;
      const int cit = it % (kChunk * kNKB);            // position in the chunk: 0 restarts the accumulators
      if (it > 0 && cit == 0) mbar_wait(&drained, (it / (kChunk * kNKB) - 1) & 1);
      mbar_wait(&full[s], (it / kStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t st = saddr(smem + (size_t)s * kStage);
      const uint64_t bh = umma_desc(st + kAStage, kN / 8 * 128), bl = umma_desc(st + kAStage + kBHalf, kN / 8 * 128);
#pragma unroll
      for (int tau = 0; tau < 4; ++tau) {
        const uint64_t ah = umma_desc(st + (tau * 2 + 0) * kATile, 16 * 128);
        const uint64_t al = umma_desc(st + (tau * 2 + 1) * kATile, 16 * 128);
        const uint32_t dt = tmem + tau * 128;
        umma_tf32(dt, ah, bh, idesc, cit > 0 ? 1u : 0u);
        umma_tf32(dt, al, bh, idesc, 1u);
        umma_tf32(dt, ah, bl, idesc, 1u);
      }
      umma_commit(&empty[s]);
      if ((it + 1) % (kChunk * kNKB) == 0 || it + 1 == nit) umma_commit(&chunk_full);
    }
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == kRows / 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

TcGeo make_geo(Ctx& c) {
  TcGeo g{};
  g.qx = c.cells.qx.p; g.qy = c.cells.qy.p; g.qz = c.cells.qz.p; g.level = c.cells.level.p;
  for (int a = 0; a < 3; ++a) g.per[a] = c.per_units[a];
  const int nl = (int)c.level_begin.size();
  for (int l = 0; l < kMaxLevel + 2; ++l) g.lvl_begin[l] = (int)c.level_begin[std::min(l, nl - 1)];
  return g;
}

}  // namespace

// Decide the tensor-core levels/cells for the current lists (once per list
// build) and build their operators.  Host-synchronous (small copies).
void m2l_tc_prepare(Ctx& c) {
  c.tc_valid = true;
  c.tc_levels.clear();
  c.tc_entries = 0;
  c.tc_skip.reserve(std::max<int64_t>(c.ncells, 1));
  FMM_CUDA(cudaMemsetAsync(c.tc_skip.p, 0, std::max<int64_t>(c.ncells, 1), c.stream));
  if (c.cfg.m2l_path != 0 || c.P != kTcP || c.nm2l == 0) return;
  const int nlev = (int)c.level_begin.size() - 1;
  if (nlev > 11) return;                                    // 10-bit Morton spread in tc_source
  const TcGeo g = make_geo(c);
  cudaStream_t st = c.stream;
  struct Cand { int lt, cls, D, R; std::vector<int> codes; std::vector<short> tbl; };
  std::vector<Cand> cands;
  c.tc_tmp.reserve(8);
  for (int l = 2; l < nlev; ++l) {
    const int lb = (int)c.level_begin[l], le = (int)c.level_begin[l + 1];
    if (le - lb < 1024) continue;       // small levels: the register kernel is as fast
    // reference cells: per parity class, the first of the level with a non-empty list
    std::vector<int> ref(8, 0x7fffffff);
    FMM_CUDA(cudaMemcpyAsync(c.tc_tmp.p, ref.data(), 8 * sizeof(int), cudaMemcpyHostToDevice, st));
    FMM_LAUNCH(c, k_tc_first, 148, 256, 0, c.m2l_b.p, c.m2l_e.p, lb, le, g, c.tc_tmp.p);
    FMM_CUDA(cudaMemcpyAsync(ref.data(), c.tc_tmp.p, 8 * sizeof(int), cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaStreamSynchronize(st));
    for (int cls = 0; cls < 8; ++cls) {
      if (ref[cls] == 0x7fffffff) continue;
      int be[2];
      FMM_CUDA(cudaMemcpyAsync(&be[0], c.m2l_b.p + ref[cls], sizeof(int), cudaMemcpyDeviceToHost, st));
      FMM_CUDA(cudaMemcpyAsync(&be[1], c.m2l_e.p + ref[cls], sizeof(int), cudaMemcpyDeviceToHost, st));
      FMM_CUDA(cudaStreamSynchronize(st));
      const int D = be[1] - be[0];
      if (D <= 0 || D > 8192) continue;
      c.tc_codes_tmp.reserve(D);
      FMM_LAUNCH(c, k_tc_ref_codes, 1, 256, 0, c.m2l.p, c.m2l_b.p, c.m2l_e.p, ref[cls], l, g, c.tc_codes_tmp.p);
      Cand cd;
      cd.lt = l;
      cd.cls = cls;
      cd.D = D;
      cd.codes.resize(D);
      FMM_CUDA(cudaMemcpyAsync(cd.codes.data(), c.tc_codes_tmp.p, sizeof(int) * D, cudaMemcpyDeviceToHost, st));
      FMM_CUDA(cudaStreamSynchronize(st));
      std::sort(cd.codes.begin(), cd.codes.end());
      if (cd.codes[0] < 0 || std::adjacent_find(cd.codes.begin(), cd.codes.end()) != cd.codes.end()) continue;
      int R = 0;
      for (int code : cd.codes)
        for (int a = 0; a < 3; ++a) R = std::max(R, std::abs(((code >> (14 - 7 * a)) & 127) - 64));
      const int V = 2 * R + 1;
      cd.R = R;
      cd.tbl.assign((size_t)3 * V * V * V, (short)-1);
      for (int d = 0; d < D; ++d) {
        const int code = cd.codes[d];
        const int dl = (code >> 21) - 1, vx = ((code >> 14) & 127) - 64, vy = ((code >> 7) & 127) - 64,
                  vz = (code & 127) - 64;
        cd.tbl[(((size_t)(dl + 1) * V + vx + R) * V + vy + R) * V + vz + R] = (short)d;
      }
      cands.push_back(std::move(cd));
    }
  }
  if (cands.empty()) return;
  // verify every cell of the candidate levels; collect the targets
  int64_t tgt_total = 0, code_total = 0, op_total = 0;
  for (auto& cd : cands) {
    tgt_total += c.level_begin[cd.lt + 1] - c.level_begin[cd.lt];
    code_total += cd.D;
  }
  c.tc_tgt.reserve(tgt_total);
  c.tc_codes.reserve(code_total);
  c.tc_cnt.reserve(cands.size());
  FMM_CUDA(cudaMemsetAsync(c.tc_cnt.p, 0, sizeof(int) * cands.size(), st));
  int64_t toff = 0, coff = 0;
  std::vector<int64_t> tgt_off, code_off;
  for (size_t i = 0; i < cands.size(); ++i) {
    auto& cd = cands[i];
    const int lb = (int)c.level_begin[cd.lt], le = (int)c.level_begin[cd.lt + 1];
    c.tc_tbl.reserve(cd.tbl.size());
    FMM_CUDA(cudaMemcpyAsync(c.tc_tbl.p, cd.tbl.data(), sizeof(short) * cd.tbl.size(), cudaMemcpyHostToDevice, st));
    FMM_CUDA(cudaMemcpyAsync(c.tc_codes.p + coff, cd.codes.data(), sizeof(int) * cd.D, cudaMemcpyHostToDevice, st));
    const unsigned blocks = (unsigned)std::min<int64_t>((le - lb + 7) / 8, 148 * 16);
    FMM_LAUNCH(c, k_tc_verify, blocks, 256, 0, c.m2l.p, c.m2l_b.p, c.m2l_e.p, lb, le, cd.lt, cd.D, g, c.tc_tbl.p, cd.R,
               cd.cls, c.tc_skip.p, c.tc_tgt.p + toff, c.tc_cnt.p + i);
    FMM_CUDA(cudaStreamSynchronize(st));    // the table buffer is reused by the next level
    tgt_off.push_back(toff);
    code_off.push_back(coff);
    toff += le - lb;
    coff += cd.D;
  }
  std::vector<int> cnt(cands.size());
  FMM_CUDA(cudaMemcpyAsync(cnt.data(), c.tc_cnt.p, sizeof(int) * cands.size(), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  // operators of the levels that have targets
  std::vector<int64_t> op_off(cands.size(), -1);
  for (size_t i = 0; i < cands.size(); ++i)
    if (cnt[i] > 0) {
      op_off[i] = op_total;
      op_total += (int64_t)cands[i].D * kNKB * 2 * kBHalf;
    }
  if (op_total == 0) return;
  c.tc_op.reserve(op_total);
  for (size_t i = 0; i < cands.size(); ++i) {
    if (cnt[i] <= 0) continue;
    FMM_LAUNCH(c, k_tc_operator, (unsigned)cands[i].D, 256, 0, c.tc_codes.p + code_off[i], cands[i].lt,
               c.tc_op.p + op_off[i]);
    TcLevel tl;
    tl.lt = cands[i].lt;
    tl.D = cands[i].D;
    tl.ntgt = cnt[i];
    tl.tgt_off = tgt_off[i];
    tl.code_off = code_off[i];
    tl.op_off = op_off[i];
    c.tc_levels.push_back(tl);
    c.tc_entries += (int64_t)cnt[i] * cands[i].D;
  }
  // longest CTAs first
  std::sort(c.tc_levels.begin(), c.tc_levels.end(), [](const TcLevel& a, const TcLevel& b) { return a.D > b.D; });
}

void m2l_tc_run(Ctx& c) {
  if (c.tc_levels.empty()) return;
  const int smem = kStages * kStage;
  FMM_CUDA(cudaFuncSetAttribute(k_m2l_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const TcGeo g = make_geo(c);
  // (level, class) groups, up to kMaxTcLevels per launch
  for (size_t g0 = 0; g0 < c.tc_levels.size(); g0 += kMaxTcLevels) {
    TcArgs args{};
    int ctas = 0;
    args.nlv = (int)std::min<size_t>(kMaxTcLevels, c.tc_levels.size() - g0);
    for (int i = 0; i < args.nlv; ++i) {
      const TcLevel& tl = c.tc_levels[g0 + i];
      args.lv[i] = {c.tc_tgt.p + tl.tgt_off, c.tc_codes.p + tl.code_off, c.tc_op.p + tl.op_off, tl.ntgt, tl.lt, tl.D,
                    ctas};
      ctas += (int)((3 * (int64_t)tl.ntgt + kRows - 1) / kRows);
    }
    FMM_LAUNCH(c, k_m2l_tc, (unsigned)ctas, kThreads, smem, args, g, c.M.p, c.Lc.p);
  }
}

}  // namespace fmmb
