// m2l_tc.cu -- a9 (M2L) on the 5th-generation tensor cores for
// the levels where every target cell sees the same set of source offsets.
//
// In a uniform periodic octree every cell of a level has the same M2L
// interaction list up to translation and up to the mirror symmetry of its
// octant in the parent: a cell of parity class c = (qx&1, qy&1, qz&1) sees
// the offsets Q_c(S), S the set of the even (class 0) cells and Q_c the
// reflection of the axes whose bit is set.  For a fixed offset d the M2L
// translation is a fixed real-linear map T_d from the source multipole
// (p(p+1)/2 complex = 110 reals at p = 10, component-wise) to the target local
// expansion, and a reflection only changes signs:
//
//   T(Q D) = S_L(Q) T(D) S_M(Q),   S diagonal +-1:
//     x: (n,m) -> (-1)^m conj,  y: conj,  z: (-1)^(n+m)      (I_n^m(QD) likewise)
//
// so a whole level is ONE dense contraction with one operator,
//
//   L[(t, c), j] += S_L(t)_j sum_d sum_i T_d[j, i] S_M(t)_i M[(src(t, d), c), i],
//
// K = D x 112 (110 padded): the shape tcgen05.mma wants.  T_d is built once per
// level in double precision from I_{n+k}^{m+l}(D) with the (-1)^k sign and the
// (s_s/s_t)^n scale of P:228 folded in.  The triangular truncation n + k <= p-1
// makes the rows of T_d that a K-block of inputs (degrees >= n_min) reaches a
// prefix of length (p - n_min)(p - n_min + 1): each K-block's MMA uses only that
// many output columns (N = 112, 80, 64, 48, 32, 32, 32, 16 x 7 at p = 10, a third
// of the dense work) and the operator stores only those rows.
//
// Precision (3xTF32): every operand is split x = hi + lo, hi = x with the 13
// low mantissa bits cleared (exactly a TF32 value), lo = x - hi; the product
// is accumulated as hi.hi + lo.hi + hi.lo in FP32 in TMEM.  The tensor cores
// accumulate with truncation (tools/umma_probe.cu: the error grows ~1e-8 per
// MMA), so the accumulators are drained into Lc every kChunk offsets; the
// result then matches the FP32 register kernel's accuracy against the
// oracle (tests/test_gpu_m2l_tc.py).
//
// Pipeline (two CTAs per SM, 9 warps each): rows are (target, component),
// 256 per CTA as two 128-row accumulators in TMEM.  A stage is TC_KPS = 2
// K-blocks of one offset.  Warps 0-7 gather, for every row, the 2 x 8
// multipole reals of the stage from a packed copy of M (one thread per row,
// one 256-bit load per K-block), apply the row's S_M signs, split hi/lo and
// store the stage's A tiles (K-major core-matrix layout, no swizzle); thread 0
// also bulk-copies the stage's pre-split operator slices (cp.async.bulk,
// mbarrier tx count).  One thread of warp 8 issues the 12 MMAs of a stage and
// commits to the stage's "empty" mbarrier.  Targets are processed in Morton order so concurrently running
// CTAs share their sources in L2.
//
// Which cells take this path is decided per list build, on the unsorted list
// (two passes over it): the first cell of each level with entries fixes the
// level's canonical offsets; every entry is then checked -- its offset,
// reflected into class 0, is in that set, the source the tensor kernel
// computes (Morton index of the offset cell in the level-ordered cell array)
// is the entry's source, and its bit in the target's offset mask was not yet
// set -- and a cell is taken iff none of its entries failed and its mask holds
// all D offsets.  Only the remaining entries are grouped by target (for the
// register kernel), so the big M2L list is never sorted.  Cells that fail (adaptive
// trees, partial levels) stay on the register kernel (m2l.cu), which skips
// the cells taken here.
#include <algorithm>
#include <cstring>

#include <cub/cub.cuh>

#include "ctx.cuh"

namespace fmmb {

namespace {

#ifndef TC_OGROUP
#define TC_OGROUP 0   // offsets per CTA (0: all of the level's); > 0 splits a row block's offsets over CTAs
#endif
#ifndef TC_CHUNK
#define TC_CHUNK 32
#endif
#ifndef TC_PF
#define TC_PF (TC_KPS == 1 ? 6 : 3)
#endif
#ifndef TC_DIAG
#define TC_DIAG 0   // development only (tools/build_variant.py): 1 = every row reads its own cell, 2 = no gathers,
                    // 3 = one MMA per K-block instead of three (timing only: wrong results)
#endif
constexpr int kTcP = 10;                    // the tensor path is instantiated for p = 10
constexpr int kNC = kTcP * (kTcP + 1) / 2;  // 55 complex coefficients
#ifndef TC_ROWS
#define TC_ROWS 256
#endif
#ifndef TC_KPS
#define TC_KPS 2                 // K-blocks per pipeline stage (1 or 2): each stage hand-off (256
                                 // producer arrivals, proxy fences, the MMA issuer's wait, the
                                 // commit) bounds the kernel, so two K-blocks per stage halve the
                                 // hand-offs: C3 M2L phase 68.9 -> 54.4 ms (2 stages of 46 KB)
#endif
#ifndef TC_AT
#define TC_AT 0                  // 1: A operand in TMEM -- producers write the hi/lo tiles with tcgen05.st
                                 // and the MMAs read A from TMEM ([a-tmem] form), so shared memory carries
                                 // only the operator slices.  Correct (test_gpu_m2l_tc.py passes) but slower
                                 // on a B200 at C3 (r02 A/B, profiles/r02_m2l_tmem_a.txt): 256 rows, one CTA
                                 // per SM 66.4 ms, 128 rows, two CTAs per SM 58.7 ms, vs 52.0 ms with A in
                                 // shared memory -- the LSU pipe drops 78% -> 31% but the tensor pipe stays
                                 // at 16-19% busy with the producers waiting on the MMAs' completion
#endif
#ifndef TC_STAGES
#define TC_STAGES (TC_AT ? 4 : (TC_KPS == 1 ? 4 : 2))
#endif
constexpr int kRows = TC_ROWS;              // rows (target, component) per CTA: 128 x kAcc
constexpr int kAcc = kRows / 128;           // TMEM accumulators per CTA
// TC_AT: the accumulators at columns 128 tau, the stages' A tiles (K-block, tau,
// hi | lo) x 8 columns from column 128 kAcc; 256 rows: one CTA per SM owns all 512
// columns, 128 rows: two CTAs per SM with 256 columns each (two MMA issuers per SM)
constexpr int kCtasPerSm = TC_AT ? (kAcc == 2 ? 1 : 2) : 512 / kRows;
constexpr int kTmemCols = TC_AT ? 256 * kAcc : kAcc * 128;
constexpr int kACol0 = 128 * kAcc;
constexpr int kN = 112;                     // local-expansion reals (110, padded)
constexpr int kKB = 8;                      // K per stage (one kind::tf32 MMA)
constexpr int kNKB = 14;                    // K-blocks per offset (112 / 8)
constexpr int kStages = TC_STAGES;
constexpr int kPF = TC_PF;                      // gather prefetch distance (stages)
constexpr int kATile = 128 * kKB * 4;       // one 128-row A tile (hi or lo), bytes
constexpr int kALbo = 16 * 128;             // A tile: stride between its two 16-byte K chunks
constexpr int kKPS = TC_KPS;
constexpr int kSPO = kNKB / kKPS;            // stages per offset
constexpr int kAStage = TC_AT ? 0 : kKPS * kAcc * 2 * kATile;  // K-blocks x accumulators x (hi, lo)
constexpr int kAColsStage = kKPS * kAcc * 16;      // TC_AT: TMEM columns of one stage's A tiles
constexpr int kBMax = kKPS * 2 * kN * kKB * 4;   // operator slices (hi + lo) at N <= 112
constexpr int kStage = kAStage + kBMax;
constexpr int kThreads = kRows + 32;
static_assert(!TC_AT || ((kAcc == 1 || kAcc == 2) && kACol0 + kStages * kAColsStage <= kTmemCols), "TC_AT: TMEM columns");
// offsets accumulated in TMEM between drains: each drain stalls the CTA's MMAs
// (one accumulator set per CTA), so fewer drains are faster (C3: 16 -> 73.0 ms,
// 24 -> 70.5, 32 -> 68.7, 48 -> 67.5) while the truncation drift grows with the
// MMAs per chunk (far-field u vs the oracle, TG 32^3: 1.6e-6, 2.1e-6, 2.5e-6,
// 3.4e-6; register kernel 4.8e-7, bar 1e-5)
constexpr int kChunk = TC_CHUNK;
constexpr int kMaxTcLevels = 16;
constexpr int kMaxMapLevel = 8;             // forest source maps: 8^l entries per level, l <= 8

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
// 16-byte K chunk, SBO = next 8 rows (128 B); descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
// A from tensor memory (lane = row, 8 consecutive 32-bit columns = K), B from shared memory
__device__ __forceinline__ void umma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(b))
               : "memory");
}
__host__ __device__ __forceinline__ float tf32_hi(float x) {
#ifdef __CUDA_ARCH__
  return __uint_as_float(__float_as_uint(x) & 0xffffe000u);
#else
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u &= 0xffffe000u;
  float y;
  std::memcpy(&y, &u, 4);
  return y;
#endif
}

// ------------------------------------------------------------ geometry ----
struct TcGeo {
  const int *qx, *qy, *qz, *level;
  const int4* cq;                   // (qx, qy, qz, level) per cell, packed per list build (verification)
  long long per[3];                 // periods in half-finest-cell units
  int lvl_begin[kMaxLevel + 2];
  const int* map;                   // LET forest (nranks > 1): level-grid Morton index -> cell id (-1 none,
  int map_off[kMaxLevel + 2];       // -2 several trees), per level at map_off; null on one GPU
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
__host__ __device__ __forceinline__ int code_dl(int code) { return (code >> 21) - 1; }
__host__ __device__ __forceinline__ int code_v(int code, int a) { return ((code >> (14 - 7 * a)) & 127) - 64; }
// Q_c: negate the offset components of the axes whose class bit is set
__host__ __device__ __forceinline__ int reflect(int code, int cls) {
  int out = code & (3 << 21);
  for (int a = 0; a < 3; ++a) {
    const int v = code_v(code, a);
    out |= ((((cls >> a) & 1) ? -v : v) + 64) << (14 - 7 * a);
  }
  return out;
}

// the cell the tensor kernel reads for a target (centre ct) and offset code:
// c_s = c_t - Delta wrapped into the period, its level-ls Morton index
// (centres and periods are < 2^23 half-finest-cell units: int arithmetic)
template <typename I>
__device__ __forceinline__ int tc_source(const TcGeo& g, int lt, const I (&ct)[3], int code) {
  const int dl = code_dl(code), ls = lt + dl, lf = max(lt, ls);
  uint32_t q[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int P = (int)g.per[a];
    int cs = (int)ct[a] - code_v(code, a) * (1 << (kMaxLevel - lf));
    cs &= P - 1;                                   // periods are powers of two (checked on the host)
    q[a] = (uint32_t)(((cs >> (kMaxLevel - ls)) - 1) >> 1);
  }
  const int m = (int)(spread3_32(q[0]) | (spread3_32(q[1]) << 1) | (spread3_32(q[2]) << 2));
  if (!g.map) return g.lvl_begin[ls] + m;
  const int off = g.map_off[ls];
  return off < 0 ? -1 : __ldg(g.map + off + m);
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
    const int sh = kMaxLevel - lf;                  // Delta is a multiple of 2^sh for a valid entry
    if (d & ((1ll << sh) - 1)) return -1;
    const long long v = d >> sh;
    if (v < -63 || v > 63) return -1;
    code |= (int)(v + 64) << (14 - 7 * a);
  }
  return code;
}

// the same from the packed cell table: one 16-byte load per cell
__device__ __forceinline__ int entry_code4(const TcGeo& g, int lt, const long long (&ct)[3], uint64_t ent) {
  const int src = (int)((ent >> 5) & 0x7ffffff), img = (int)(ent & 31);
  const int4 sq = __ldg(g.cq + src);
  const int ls = sq.w, dl = ls - lt;
  if (dl < -1 || dl > 1) return -1;
  const int lf = max(lt, ls);
  const int qs[3] = {sq.x, sq.y, sq.z};
  const int im[3] = {img % 3 - 1, (img / 3) % 3 - 1, img / 9 - 1};
  int code = (dl + 1) << 21;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const long long cs = (long long)(2 * qs[a] + 1) << (kMaxLevel - ls);
    const long long d = ct[a] - cs - (long long)im[a] * g.per[a];
    const int sh = kMaxLevel - lf;
    if (d & ((1ll << sh) - 1)) return -1;
    const long long v = d >> sh;
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

// parity class of a cell: its octant within the parent
__device__ __forceinline__ int parity_class(const TcGeo& g, int c) {
  return (g.qx[c] & 1) | ((g.qy[c] & 1) << 1) | ((g.qz[c] & 1) << 2);
}

// (degree, order) of complex coefficient o = n(n+1)/2 + m
__host__ __device__ __forceinline__ void deg_ord(int o, int& n, int& m) {
  n = 0;
  while ((n + 1) * (n + 2) / 2 <= o) ++n;
  m = o - n * (n + 1) / 2;
}
// sign of real r = 2 o + part of a coefficient under the class-c reflection
// (the same pattern for multipoles and locals, see the header)
inline bool refl_negates(int r, int cls) {
  if (r >= 2 * kNC) return false;
  int n, m;
  deg_ord(r >> 1, n, m);
  const int im = r & 1;
  int neg = 0;
  if (cls & 1) neg ^= (m & 1) ^ im;
  if (cls & 2) neg ^= im;
  if (cls & 4) neg ^= (n + m) & 1;
  return neg != 0;
}

// output columns the K-block kb reaches (rows of T_d that are not zero)
inline int kb_cols(int kb) {
  int n, m;
  deg_ord(4 * kb, n, m);                     // lowest degree in the K-block
  const int kmax = kTcP - 1 - n;
  const int rows = (kmax + 1) * (kmax + 2);
  return std::min(kN, std::max(16, (rows + 15) / 16 * 16));
}

struct TcTables {
  int ncols[kNKB];           // N of each K-block's MMA
  int opk[kNKB + 1];         // byte offset of each K-block's slice within one offset's operator
  unsigned char sm[8][kNKB]; // S_M: bit q set = input real 8 kb + q negated, per class
  uint32_t sl[8][4];         // S_L: bit j set = output real j negated, per class
};

TcTables make_tables() {
  TcTables T{};
  int off = 0;
  for (int kb = 0; kb < kNKB; ++kb) {
    T.ncols[kb] = kb_cols(kb);
    T.opk[kb] = off;
    off += 2 * T.ncols[kb] * kKB * 4;
  }
  T.opk[kNKB] = off;
  for (int c = 0; c < 8; ++c) {
    for (int kb = 0; kb < kNKB; ++kb)
      for (int q = 0; q < kKB; ++q)
        if (refl_negates(kb * kKB + q, c)) T.sm[c][kb] |= (unsigned char)(1u << q);
    for (int j = 0; j < kN; ++j)
      if (refl_negates(j, c)) T.sl[c][j >> 5] |= 1u << (j & 31);
  }
  return T;
}

// ---- per-build verification on the unsorted M2L list (emission order) ----
// Every level's parameters at once, so each kernel is one pass over the list.
struct TcVer {
  int nlv;
  int lt[kMaxTcLevels], lb[kMaxTcLevels], le[kMaxTcLevels], D[kMaxTcLevels], R[kMaxTcLevels], W[kMaxTcLevels];
  int ref[kMaxTcLevels];
  int64_t tbl_off[kMaxTcLevels], mask_off[kMaxTcLevels];
};
__device__ __forceinline__ int ver_level(const TcVer& v, int t) {
  for (int k = 0; k < v.nlv; ++k)
    if (t >= v.lb[k] && t < v.le[k]) return k;
  return -1;
}

// offset histogram per candidate level: every entry's offset code, reflected
// into class 0, counted in a dense (dl, v) table of half-width kHR; the
// level's canonical set is then the codes a majority of its cells use
constexpr int kHR = 24;                 // |v| <= 24 finest-level units: covers the theta = 1/2 lists
constexpr int kHV = 2 * kHR + 1;
constexpr int kHBins = 3 * kHV * kHV * kHV;
constexpr int kHSample = 16;             // the histogram samples 1/16 of the entries (163M atomics on ~550 bins otherwise)
__global__ void k_tc_code_hist(const uint64_t* __restrict__ lst, int64_t n, TcVer v, TcGeo g,
                               unsigned* __restrict__ hist) {
  // a sample of the list: runs of 16 consecutive entries (one 128-byte line), each run taken
  // with probability 1/16 by a multiplicative hash of its index (no aliasing with the
  // traversal's regular emission pattern)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if ((((uint32_t)(i >> 4) * 2654435761u) >> 28) != 0) continue;
    const uint64_t ent = lst[i];
    const int t = (int)(ent >> 32);
    const int k = ver_level(v, t);
    if (k < 0) continue;
    const int lt = v.lt[k];
    const int4 tq = __ldg(g.cq + t);
    long long ct[3];
    ct[0] = (long long)(2 * tq.x + 1) << (kMaxLevel - lt);
    ct[1] = (long long)(2 * tq.y + 1) << (kMaxLevel - lt);
    ct[2] = (long long)(2 * tq.z + 1) << (kMaxLevel - lt);
    const int code = entry_code4(g, lt, ct, ent);
    if (code < 0) continue;
    const int c0 = reflect(code, (tq.x & 1) | ((tq.y & 1) << 1) | ((tq.z & 1) << 2));
    const int vx = code_v(c0, 0), vy = code_v(c0, 1), vz = code_v(c0, 2);
    if (vx < -kHR || vx > kHR || vy < -kHR || vy > kHR || vz < -kHR || vz > kHR) continue;
    atomicAdd(&hist[(int64_t)k * kHBins + (((code_dl(c0) + 1) * kHV + vx + kHR) * kHV + vy + kHR) * kHV + vz + kHR], 1u);
  }
}

__global__ void k_tc_count_has(const unsigned char* __restrict__ has, TcVer v, int* __restrict__ cnt) {
  for (int k = 0; k < v.nlv; ++k) {
    int m = 0;
    for (int c = v.lb[k] + (int)(blockIdx.x * blockDim.x + threadIdx.x); c < v.le[k]; c += (int)(gridDim.x * blockDim.x))
      m += has[c] ? 1 : 0;
    for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(&cnt[k], m);
  }
}

// per entry whose target is in a candidate level: its offset, reflected into
// class 0, is in the canonical table and its source is the one tc_source
// computes -> the entry is "good" (bit i of the per-entry words: the tensor
// path may take it) and its offset's bit is set in the target's mask; a bit
// already set is a duplicate (the target then stays off the tensor path).
// Other entries of a target (offsets outside the level's canonical set, or a
// source elsewhere than the canonical cell: adaptive trees) stay on the
// register kernel, whichever path takes the target's canonical ones.
__global__ void k_tc_verify_entries(const uint64_t* __restrict__ lst, int64_t n, TcVer v, TcGeo g,
                                    const short* __restrict__ tbl, unsigned* __restrict__ mask,
                                    unsigned char* __restrict__ bad, unsigned* __restrict__ goodw,
                                    unsigned char* __restrict__ extra) {
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; i0 < n;
       i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + (threadIdx.x & 31);
    bool good = false;
    if (i < n) {
      const uint64_t ent = lst[i];
      const int t = (int)(ent >> 32);
      const int k = ver_level(v, t);
      if (k >= 0) {
        const int lt = v.lt[k], R = v.R[k], V = 2 * R + 1;
        const int4 tq = __ldg(g.cq + t);
        long long ct[3];
        ct[0] = (long long)(2 * tq.x + 1) << (kMaxLevel - lt);
        ct[1] = (long long)(2 * tq.y + 1) << (kMaxLevel - lt);
        ct[2] = (long long)(2 * tq.z + 1) << (kMaxLevel - lt);
        const int code = entry_code4(g, lt, ct, ent);
        good = code >= 0;
        int d = -1;
        if (good) {
          const int c0 = reflect(code, (tq.x & 1) | ((tq.y & 1) << 1) | ((tq.z & 1) << 2));
          const int dl = code_dl(c0), vx = code_v(c0, 0), vy = code_v(c0, 1), vz = code_v(c0, 2);
          good = vx >= -R && vx <= R && vy >= -R && vy <= R && vz >= -R && vz <= R;
          if (good) d = tbl[v.tbl_off[k] + (((dl + 1) * V + vx + R) * V + vy + R) * V + vz + R];
          good = good && d >= 0;
        }
        if (good) good = tc_source(g, lt, ct, code) == (int)((ent >> 5) & 0x7ffffff);
        if (good) {
          const int64_t row = (int64_t)(t - v.lb[k]);
          const unsigned bit = 1u << (d & 31);
          const unsigned old = atomicOr(&mask[v.mask_off[k] + row * v.W[k] + (d >> 5)], bit);
          if (old & bit) bad[v.lb[k] + row] = 1;
        } else {
          extra[t] = 1;                        // an entry the register kernel keeps
        }
      }
    }
    const unsigned w = __ballot_sync(0xffffffffu, good);
    if ((threadIdx.x & 31) == 0 && i0 < n) goodw[i0 >> 5] = w;
  }
}

// per cell of the candidate levels: no duplicate and at least kMinFrac of the
// D canonical offsets present -> taken by the tensor path (appended per level;
// its missing offsets are masked to zero rows in the kernel, and its
// remaining entries stay on the register kernel)
#ifndef TC_MIN_FRAC
#define TC_MIN_FRAC 0.4f
#endif
constexpr float kMinFrac = TC_MIN_FRAC;
__global__ void k_tc_accept(TcVer v, const unsigned* __restrict__ mask, const unsigned char* __restrict__ bad,
                            unsigned char* __restrict__ skip, int* __restrict__ tgt, const int64_t* __restrict__ tgt_off,
                            int* __restrict__ ntgt, unsigned long long* __restrict__ nent,
                            const unsigned char* __restrict__ extra, int* __restrict__ mixed) {
  for (int k = 0; k < v.nlv; ++k) {
    for (int c = v.lb[k] + (int)(blockIdx.x * blockDim.x + threadIdx.x); c < v.le[k]; c += (int)(gridDim.x * blockDim.x)) {
      if (bad[c]) continue;
      int pc = 0;
      const unsigned* m = mask + v.mask_off[k] + (int64_t)(c - v.lb[k]) * v.W[k];
      for (int w = 0; w < v.W[k]; ++w) pc += __popc(m[w]);
      if (pc > 0 && (float)pc >= kMinFrac * (float)v.D[k]) {
        skip[c] = pc == v.D[k] ? 1 : 2;          // 1: every canonical offset (no mask lookups), 2: masked
        tgt[tgt_off[k] + atomicAdd(&ntgt[k], 1)] = c;
        atomicAdd(nent, (unsigned long long)pc);
        if (pc != v.D[k] || extra[c]) *mixed = 1;   // the register kernel keeps entries of a taken cell
      }
    }
  }
}

// operator of one level (class 0 offsets): T_d[j][i] split into TF32 hi/lo,
// per (d, K-block) the rows j < ncols[kb] in the stage layout
//   [hi | lo] x [K chunk (2)][row group (ncols / 8)][8 rows][4 floats].
__global__ void k_tc_operator(const int* __restrict__ codes, TcTables T, unsigned char* __restrict__ op) {
  constexpr int P = kTcP;
  const int d = blockIdx.x;
  const int code = codes[d];
  const int dl = code_dl(code);
  __shared__ double2 I[kNC];
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
  unsigned char* base = op + (size_t)d * T.opk[kNKB];
  for (int kb = 0; kb < kNKB; ++kb) {
    const int nc = T.ncols[kb];
    for (int idx = threadIdx.x; idx < nc * kKB; idx += blockDim.x) {
      const int j = idx / kKB, kk = idx - kKB * (idx / kKB), i = kb * kKB + kk;
      double v = 0.0;
      if (j < 2 * kNC && i < 2 * kNC) {
        int k, l, n, m;
        deg_ord(j >> 1, k, l);
        deg_ord(i >> 1, n, m);
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
      const size_t off = (size_t)T.opk[kb] + (kk / 4) * (nc / 8 * 128) + (j / 8) * 128 + (j % 8) * 16 + (kk % 4) * 4;
      *(float*)(base + off) = hi;
      *(float*)(base + off + nc * kKB * 4) = lo;
    }
  }
}

// packed multipoles: [cell][K-block (14)][component (3)][8 floats] -- the 32-byte
// K-block slices of a cell's three components are adjacent, so the three rows
// (t, c = 0..2) of a target gather one 96-byte run per stage (fewer L1 lines per
// warp request than a [cell][component][112] layout: -9% kernel time at C3);
// reals 110, 111 = 0
constexpr int kMpLine = 6;                         // float4 per (cell, K-block): 3 components x 2
__global__ void k_tc_pack(const float2* __restrict__ M, int64_t ncells, float4* __restrict__ Mp) {
  const int64_t n4 = ncells * kNKB * kMpLine;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const int w = (int)(i % kMpLine);
    const int64_t r2 = i / kMpLine;
    const int kb = (int)(r2 % kNKB);
    const int64_t cell = r2 / kNKB;
    const int comp = w >> 1, ch = w & 1;
    const int q = kb * 2 + ch;                       // float4 index within the 112-real row
    const float2* src = M + (cell * 3 + comp) * kNC + 2 * q;
    const float2 a = src[0];
    const float2 b = 2 * q + 1 < kNC ? src[1] : make_float2(0.f, 0.f);
    Mp[i] = make_float4(a.x, a.y, b.x, b.y);
  }
}

// ------------------------------------------------------- tensor kernel ----
struct TcLevelArg {
  const int* tgt;
  const int* codes;
  const unsigned char* op;
  const unsigned* mask;          // per target cell (cell - lb) x W words: canonical offsets present
  const unsigned char* skip;     // per cell: 1 = every canonical offset, 2 = subset (mask)
  int ntgt, lt, D, cta_begin, lb, W;
  int nblk, gsize;               // CTAs per offset group (row blocks), offsets per group
};
struct TcArgs {
  TcLevelArg lv[kMaxTcLevels];
  int nlv;
};

__global__ void __launch_bounds__(kThreads, kCtasPerSm) k_m2l_tc(TcArgs args, TcTables T, TcGeo g,
                                                        const float4* __restrict__ Mp, float2* __restrict__ Lc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full[kStages], empty[kStages], chunk_full, drained[2];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  int li = 0;
  while (li + 1 < args.nlv && (int)blockIdx.x >= args.lv[li + 1].cta_begin) ++li;
  const TcLevelArg A = args.lv[li];
  // offset groups: CTA (group, row block); all row blocks of a group run before the
  // next group's, so concurrently running CTAs read the sources of nearby offsets
  const int local = (int)blockIdx.x - A.cta_begin;
  const int grp = local / A.nblk, blk = local - grp * A.nblk;
  const int dbase = grp * A.gsize;
  const int nit = min(A.gsize, A.D - dbase) * kSPO;   // pipeline stages
  constexpr int CN = kChunk * kSPO;
  const int nchunk = (nit + CN - 1) / CN;

  if (warp == kRows / 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tbase)), "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], kRows);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&chunk_full, 1);
    mbar_init(&drained[0], kRows);
    mbar_init(&drained[1], kRows);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  const int row0 = blk * kRows;

  if (warp < kRows / 32) {
    // ---------------------------------------------------------- producers
    // gather: thread tid owns row tid (tile tid / 128) and reads its 32-byte
    // K-block slice with one 256-bit load; a warp request covers 32 rows, i.e.
    // ~11 targets x one 96-byte run each
    int ct[3];
    int comp, cls;
    const float* src = (const float*)Mp;
    const unsigned* mrow;
    bool on = false;                       // the row's target has the current offset
    bool allon = true;                     // ... every canonical offset (no mask lookups)
    {
      const int R = row0 + tid;
      const int t = R < 3 * A.ntgt ? R / 3 : 0;
      comp = R < 3 * A.ntgt ? R - 3 * (R / 3) : 0;
      const int cell = A.tgt[t];
      mrow = A.mask + (size_t)(cell - A.lb) * A.W;
      allon = A.skip[cell] == 1;
      cls = parity_class(g, cell);
      ct[0] = (2 * g.qx[cell] + 1) << (kMaxLevel - A.lt);
      ct[1] = (2 * g.qy[cell] + 1) << (kMaxLevel - A.lt);
      ct[2] = (2 * g.qz[cell] + 1) << (kMaxLevel - A.lt);
    }
    int pf_d = -1;
    auto load = [&](int it, float (&v)[8 * kKPS]) {
      const int d = dbase + it / kSPO, kb = (it - kSPO * (it / kSPO)) * kKPS;
      if (d != pf_d) {
        pf_d = d;
        on = allon || ((__ldg(mrow + (d >> 5)) >> (d & 31)) & 1u);
        if (on) {
          const int code = __ldg(A.codes + d);
#if TC_DIAG == 1
          const int s = A.tgt[(row0 + tid) < 3 * A.ntgt ? (row0 + tid) / 3 : 0] + 0 * code;   // diagnostic: no gather spread
#else
          const int s = tc_source(g, A.lt, ct, reflect(code, cls));
#endif
          src = (const float*)Mp + ((size_t)s * kNKB * kMpLine + comp * 2) * 4;
        }
      }
      if (!on) {                                   // offset absent from the target's list: zero row
#pragma unroll
        for (int q = 0; q < 8 * kKPS; ++q) v[q] = 0.f;
        return;
      }
#if TC_DIAG == 2
      for (int q = 0; q < 8 * kKPS; ++q) v[q] = __int_as_float(kb + q);   // diagnostic: no loads
      return;
#endif
#pragma unroll
      for (int b = 0; b < kKPS; ++b)
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(v[8 * b + 0]), "=f"(v[8 * b + 1]), "=f"(v[8 * b + 2]), "=f"(v[8 * b + 3]),
                       "=f"(v[8 * b + 4]), "=f"(v[8 * b + 5]), "=f"(v[8 * b + 6]), "=f"(v[8 * b + 7])
                     : "l"(src + (kb + b) * kMpLine * 4));
    };
    // drains: thread tid owns row tid (TMEM lane quarter = warp % 4); the
    // chunk's sums are added into Lc with vector reductions (REDG.ADD.F32x2:
    // no round trip; one thread per Lc row, so the order is fixed)
    const int Rd = row0 + tid;
    const bool dvalid = Rd < 3 * A.ntgt;
    const int dcell = A.tgt[dvalid ? Rd / 3 : 0], dcomp = dvalid ? Rd - 3 * (Rd / 3) : 0;
    const int dcls = parity_class(g, dcell);
    float2* out = Lc + ((size_t)dcell * 3 + dcomp) * kNC;
    const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((tid >> 7) * 128);
    int next_drain = 0;
    auto drain = [&]() {
      const int chunk = next_drain++;
      mbar_wait(&chunk_full, chunk & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int c0 = 0; c0 < kN; c0 += 16) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (dvalid) {
          const uint32_t sg = (T.sl[dcls][c0 >> 5] >> (c0 & 31)) & 0xffffu;   // S_L of the row's class
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int o = c0 / 2 + q;
            if (o < kNC)
              atomicAdd(out + o, make_float2(__uint_as_float(v[2 * q] ^ (((sg >> (2 * q)) & 1u) << 31)),
                                             __uint_as_float(v[2 * q + 1] ^ (((sg >> (2 * q + 1)) & 1u) << 31))));
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(&drained[chunk & 1]);
    };
    const int rr = tid & 127, tau = tid >> 7;
    const int arow = (rr >> 3) * 128 + (rr & 7) * 16;
    float buf[kPF][8 * kKPS];
#pragma unroll
    for (int u = 0; u < kPF; ++u)
      if (u < nit) load(u, buf[u]);
    for (int it0 = 0; it0 < nit; it0 += kPF) {
#pragma unroll
      for (int u = 0; u < kPF; ++u) {
        const int it = it0 + u;
        if (it < nit) {
          if (it >= CN && it % CN == 0) drain();         // chunk it/CN - 1 is complete
          const int s = it % kStages;
          const int kb0 = (it - kSPO * (it / kSPO)) * kKPS;
          if (it >= kStages) mbar_wait(&empty[s], ((it / kStages) - 1) & 1);
          unsigned char* st = smem + (size_t)s * kStage;
#if TC_AT
          asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
          for (int b = 0; b < kKPS; ++b) {
            const uint32_t sg = (uint32_t)T.sm[cls][kb0 + b];         // S_M of the row's class
            uint32_t hl[16];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const uint32_t x = __float_as_uint(buf[u][8 * b + q]) ^ (((sg >> q) & 1u) << 31);
              const uint32_t h = x & 0xffffe000u;
              hl[q] = h;
              hl[8 + q] = __float_as_uint(__uint_as_float(x) - __uint_as_float(h));
            }
            const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16) +
                                (uint32_t)(kACol0 + s * kAColsStage + (b * kAcc + tau) * 16);
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                ::"r"(ta), "r"(hl[0]), "r"(hl[1]), "r"(hl[2]), "r"(hl[3]), "r"(hl[4]), "r"(hl[5]), "r"(hl[6]),
                  "r"(hl[7]), "r"(hl[8]), "r"(hl[9]), "r"(hl[10]), "r"(hl[11]), "r"(hl[12]), "r"(hl[13]),
                  "r"(hl[14]), "r"(hl[15])
                : "memory");
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;");
#else
#pragma unroll
          for (int b = 0; b < kKPS; ++b) {
            const uint32_t sg = (uint32_t)T.sm[cls][kb0 + b];         // S_M of the row's class
            float hi[8], lo[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float x = __uint_as_float(__float_as_uint(buf[u][8 * b + q]) ^ (((sg >> q) & 1u) << 31));
              hi[q] = tf32_hi(x);
              lo[q] = x - hi[q];
            }
            unsigned char* ah = st + ((b * kAcc + tau) * 2 + 0) * kATile + arow;
            unsigned char* al = st + ((b * kAcc + tau) * 2 + 1) * kATile + arow;
            *(float4*)ah = make_float4(hi[0], hi[1], hi[2], hi[3]);
            *(float4*)(ah + kALbo) = make_float4(hi[4], hi[5], hi[6], hi[7]);
            *(float4*)al = make_float4(lo[0], lo[1], lo[2], lo[3]);
            *(float4*)(al + kALbo) = make_float4(lo[4], lo[5], lo[6], lo[7]);
          }
#ifndef TC_FENCE
#define TC_FENCE 1    // 0: timing experiment only (no generic -> async proxy fence: formally racy)
#endif
          if (TC_FENCE) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
          if (tid == 0) {
            const int d = dbase + it / kSPO, kb = kb0;
            const uint32_t bytes = (uint32_t)(T.opk[kb + kKPS] - T.opk[kb]);
            mbar_arrive_tx(&full[s], bytes);
            bulk_g2s(st + kAStage, A.op + (size_t)d * T.opk[kNKB] + T.opk[kb], bytes, &full[s]);
          } else {
            mbar_arrive(&full[s]);
          }
          if (it + kPF < nit) load(it + kPF, buf[u]);
        }
      }
    }
    while (next_drain < nchunk) drain();
  } else if (tid == kRows) {
    // ---------------------------------------------------------- MMA issuer
    const uint32_t idesc0 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(128 >> 4) << 24);
    for (int it = 0; it < nit; ++it) {
      const int s = it % kStages;
      const int kb0 = (it - kSPO * (it / kSPO)) * kKPS;
      const int chunk = it / CN, cit = it - CN * chunk;   // cit = 0 restarts the chunk's accumulators
      if (cit == 0 && chunk >= 1) mbar_wait(&drained[(chunk - 1) & 1], ((chunk - 1) >> 1) & 1);
      mbar_wait(&full[s], (it / kStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t st = saddr(smem + (size_t)s * kStage);
#pragma unroll
      for (int b = 0; b < kKPS; ++b) {
        const int kb = kb0 + b;
        const int nc = T.ncols[kb];
        const uint32_t boff = (uint32_t)(T.opk[kb] - T.opk[kb0]);
        const uint32_t idesc = idesc0 | ((uint32_t)(nc >> 3) << 17);
        const uint64_t bh = umma_desc(st + kAStage + boff, nc / 8 * 128);
        const uint64_t bl = umma_desc(st + kAStage + boff + nc * kKB * 4, nc / 8 * 128);
#pragma unroll
        for (int tau = 0; tau < kAcc; ++tau) {
          const uint32_t dt = tmem + (uint32_t)(tau * 128);
#if TC_AT
          const uint32_t ah = tmem + (uint32_t)(kACol0 + s * kAColsStage + (b * kAcc + tau) * 16), al = ah + 8;
          umma_tf32_ts(dt, ah, bh, idesc, (cit > 0 || b > 0) ? 1u : 0u);
          umma_tf32_ts(dt, al, bh, idesc, 1u);
          umma_tf32_ts(dt, ah, bl, idesc, 1u);
#else
          const uint64_t ah = umma_desc(st + ((b * kAcc + tau) * 2 + 0) * kATile, 16 * 128);
          const uint64_t al = umma_desc(st + ((b * kAcc + tau) * 2 + 1) * kATile, 16 * 128);
          umma_tf32(dt, ah, bh, idesc, (cit > 0 || b > 0) ? 1u : 0u);
#if TC_DIAG != 3
          umma_tf32(dt, al, bh, idesc, 1u);
          umma_tf32(dt, ah, bl, idesc, 1u);
#endif
#endif
        }
      }
      umma_commit(&empty[s]);
      if (cit == CN - 1 || it + 1 == nit) umma_commit(&chunk_full);
    }
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == kRows / 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
}

// forest source map: every cell of level l (any tree) at its level-grid Morton index;
// a second cell at the same place (ORB cuts through a cell) marks it -2
__global__ void k_tc_map(const int* __restrict__ qx, const int* __restrict__ qy, const int* __restrict__ qz,
                         const int* __restrict__ level, int64_t n, int l, int off, int* __restrict__ map) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (level[i] != l) continue;
    const int m = (int)(spread3_32((uint32_t)qx[i]) | (spread3_32((uint32_t)qy[i]) << 1) | (spread3_32((uint32_t)qz[i]) << 2));
    const int old = atomicCAS(map + off + m, -1, (int)i);
    if (old != -1) atomicExch(map + off + m, -2);
  }
}

__global__ void k_fill_i32(int* p, int64_t n, int v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void k_tc_cq(const int* __restrict__ qx, const int* __restrict__ qy, const int* __restrict__ qz,
                        const int* __restrict__ level, int64_t n, int4* __restrict__ cq) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    cq[i] = make_int4(qx[i], qy[i], qz[i], level[i]);
}

TcGeo make_geo(Ctx& c) {
  TcGeo g{};
  g.qx = c.cells.qx.p; g.qy = c.cells.qy.p; g.qz = c.cells.qz.p; g.level = c.cells.level.p;
  g.cq = c.tc_cq.p;
  for (int a = 0; a < 3; ++a) g.per[a] = c.per_units[a];
  const int nl = (int)c.level_begin.size();
  for (int l = 0; l < kMaxLevel + 2; ++l) g.lvl_begin[l] = (int)c.level_begin[std::min(l, nl - 1)];
  g.map = c.tc_use_map ? c.tc_map.p : nullptr;
  for (int l = 0; l < kMaxLevel + 2; ++l) g.map_off[l] = l < (int)c.tc_map_off.size() ? (int)c.tc_map_off[l] : -1;
  return g;
}

template <typename F>
void tc_cub(Ctx& c, F f) {
  size_t bytes = 0;
  FMM_CUDA(f((void*)nullptr, bytes));
  c.cub_tmp.reserve(bytes);
  FMM_CUDA(f((void*)c.cub_tmp.p, bytes));
  ++c.cub_calls;
}

}  // namespace

// Decide the tensor-core levels/cells for the current lists (once per list
// build) and build their operators.  Host-synchronous (small copies).
void m2l_tc_prepare(Ctx& c) {
  c.tc_valid = true;
  c.tc_mixed = false;
  c.tc_levels.clear();
  c.tc_entries = 0;
  c.tc_skip.reserve(std::max<int64_t>(c.ncells, 1));
  FMM_CUDA(cudaMemsetAsync(c.tc_skip.p, 0, std::max<int64_t>(c.ncells, 1), c.stream));
  if (c.cfg.m2l_path != 0 || c.P != kTcP || c.nm2l == 0) return;
  for (int a = 0; a < 3; ++a)
    if (c.per_units[a] & (c.per_units[a] - 1)) return;       // tc_source wraps with a mask
  const int nlev = (int)c.level_begin.size() - 1;
  if (nlev > 11) return;                                    // 10-bit Morton spread in tc_source
  c.tc_cq.reserve(std::max<int64_t>(c.ncells, 1));
  FMM_LAUNCH(c, k_tc_cq, (unsigned)std::min<int64_t>((c.ncells + 255) / 256, 148 * 8), 256, 0, c.cells.qx.p,
             c.cells.qy.p, c.cells.qz.p, c.cells.level.p, (int64_t)c.ncells, c.tc_cq.p);
  // candidate target levels: >= 1024 cells (smaller levels: the register kernel is as fast)
  // one GPU: a level is "full" when it holds every cell of its grid inside the
  // periodic domain, and tc_source is then the Morton index within the level;
  // otherwise (adaptive trees: partial levels) and on several GPUs (forests)
  // sources are found through per-level maps
  const int64_t tprod = (int64_t)c.cfg.tiles[0] * c.cfg.tiles[1] * c.cfg.tiles[2];
  auto full_level = [&](int l) {
    if (l < 0 || l >= nlev) return false;
    const int64_t want = (1ll << (3 * l)) * tprod / ((int64_t)c.tmax * c.tmax * c.tmax);
    return c.level_begin[l + 1] - c.level_begin[l] == want;
  };
  auto big = [&](int l) { return l >= 2 && l < nlev && c.level_begin[l + 1] - c.level_begin[l] >= 1024; };
  bool any_partial = false;
  for (int l = 2; l < nlev; ++l)
    if (big(l))
      for (int ls = l - 1; ls <= l + 1; ++ls)
        if (ls < nlev && !full_level(ls) && !(ls == l + 1 && ls == nlev)) any_partial = true;
  c.tc_use_map = c.cfg.nranks > 1 || any_partial;
  auto candidate = [&](int l) { return big(l) && (!c.tc_use_map || l + 1 <= kMaxMapLevel); };
  if (c.tc_use_map) {
    // LET forest: sources are found through a per-level map of all trees' cells,
    // built for the source levels (lt - 1, lt, lt + 1) of every candidate level;
    // a level without a map makes tc_source return -1 (entry fails -> register kernel)
    c.tc_map_off.assign(kMaxLevel + 2, -1);
    int64_t tot = 0;
    for (int l = 1; l <= kMaxMapLevel; ++l)
      if (candidate(l - 1) || candidate(l) || candidate(l + 1)) {
        c.tc_map_off[l] = tot;
        tot += 1ll << (3 * l);
      }
    if (tot == 0) return;
    c.tc_map.reserve(std::max<int64_t>(tot, 1));
    FMM_LAUNCH(c, k_fill_i32, (unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 16), 256, 0, c.tc_map.p, tot, -1);
    for (int l = 1; l <= kMaxMapLevel; ++l)
      if (c.tc_map_off[l] >= 0)
        FMM_LAUNCH(c, k_tc_map, (unsigned)std::min<int64_t>((c.ncells + 255) / 256, 148 * 8), 256, 0, c.cells.qx.p,
                   c.cells.qy.p, c.cells.qz.p, c.cells.level.p, (int64_t)c.ncells, l, (int)c.tc_map_off[l], c.tc_map.p);
  }
  const TcGeo g = make_geo(c);
  const TcTables T = make_tables();
  cudaStream_t st = c.stream;
  struct Cand { int lt, D, R; std::vector<int> codes; std::vector<short> tbl; };
  std::vector<Cand> cands;
  const unsigned gl = (unsigned)std::min<int64_t>((c.nm2l + 255) / 256, 148 * 16);
  TcVer v{};
  for (int l = 2; l < nlev && v.nlv < kMaxTcLevels; ++l) {
    if (!candidate(l)) continue;
    v.lt[v.nlv] = l;
    v.lb[v.nlv] = (int)c.level_begin[l];
    v.le[v.nlv] = (int)c.level_begin[l + 1];
    ++v.nlv;
  }
  if (v.nlv == 0) return;
  // one pass: the histogram of every level's offsets (class 0) and its cells with entries
  c.tc_hist.reserve((int64_t)kHBins * v.nlv);
  c.tc_cnt.reserve(kMaxTcLevels);
  FMM_CUDA(cudaMemsetAsync(c.tc_hist.p, 0, sizeof(unsigned) * kHBins * v.nlv, st));
  FMM_CUDA(cudaMemsetAsync(c.tc_cnt.p, 0, sizeof(int) * kMaxTcLevels, st));
  FMM_LAUNCH(c, k_tc_code_hist, gl, 256, 0, c.m2l.p, c.nm2l, v, g, c.tc_hist.p);
  FMM_LAUNCH(c, k_tc_count_has, 148 * 4, 256, 0, c.tc_has.p, v, c.tc_cnt.p);
  std::vector<unsigned> hist((size_t)kHBins * v.nlv);
  std::vector<int> nhas(kMaxTcLevels);
  FMM_CUDA(cudaMemcpyAsync(hist.data(), c.tc_hist.p, sizeof(unsigned) * hist.size(), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaMemcpyAsync(nhas.data(), c.tc_cnt.p, sizeof(int) * kMaxTcLevels, cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  for (int k = 0; k < v.nlv; ++k) {
    const int l = v.lt[k];
    if (nhas[k] <= 0) continue;
    // canonical (class 0) offsets: those a majority of the level's cells with entries use
    // (all of them, each exactly once per cell, on a uniform level)
    Cand cd;
    cd.lt = l;
    for (int dl = -1; dl <= 1; ++dl)
      for (int x = -kHR; x <= kHR; ++x)
        for (int y = -kHR; y <= kHR; ++y)
          for (int z = -kHR; z <= kHR; ++z) {
            const unsigned h = hist[(size_t)k * kHBins + (((dl + 1) * kHV + x + kHR) * kHV + y + kHR) * kHV + z + kHR];
            if (2ll * kHSample * h > (long long)nhas[k]) cd.codes.push_back(((dl + 1) << 21) | ((x + 64) << 14) | ((y + 64) << 7) | (z + 64));
          }
    cd.D = (int)cd.codes.size();
    if (cd.D == 0) continue;
    std::sort(cd.codes.begin(), cd.codes.end());
    int R = 0;
    for (int code : cd.codes)
      for (int a = 0; a < 3; ++a) R = std::max(R, std::abs(code_v(code, a)));
    const int V = 2 * R + 1;
    cd.R = R;
    cd.tbl.assign((size_t)3 * V * V * V, (short)-1);
    for (int d = 0; d < cd.D; ++d) {
      const int code = cd.codes[d];
      cd.tbl[(((size_t)(code_dl(code) + 1) * V + code_v(code, 0) + R) * V + code_v(code, 1) + R) * V +
             code_v(code, 2) + R] = (short)d;
    }
    cands.push_back(std::move(cd));
  }
  if (cands.empty()) return;
  // one pass: verify every entry of the candidate levels' targets, then accept
  // the cells whose list is exactly the canonical set
  int64_t tgt_total = 0, code_total = 0, op_total = 0, tbl_total = 0, mask_total = 0;
  TcVer w{};
  w.nlv = (int)cands.size();
  std::vector<int64_t> tgt_off, code_off;
  for (size_t i = 0; i < cands.size(); ++i) {
    auto& cd = cands[i];
    const int lb = (int)c.level_begin[cd.lt], le = (int)c.level_begin[cd.lt + 1];
    w.lt[i] = cd.lt; w.lb[i] = lb; w.le[i] = le; w.D[i] = cd.D; w.R[i] = cd.R; w.W[i] = (cd.D + 31) / 32;
    w.tbl_off[i] = tbl_total;
    w.mask_off[i] = mask_total;
    tgt_off.push_back(tgt_total);
    code_off.push_back(code_total);
    tbl_total += (int64_t)cd.tbl.size();
    mask_total += (int64_t)(le - lb) * w.W[i];
    tgt_total += le - lb;
    code_total += cd.D;
  }
  c.tc_tgt.reserve(tgt_total);
  c.tc_tgt2.reserve(tgt_total);
  c.tc_codes.reserve(code_total);
  c.tc_tbl.reserve(tbl_total);
  c.tc_mask.reserve(mask_total);
  c.tc_bad.reserve(std::max<int64_t>(c.ncells, 1));
  FMM_CUDA(cudaMemsetAsync(c.tc_mask.p, 0, sizeof(unsigned) * mask_total, st));
  FMM_CUDA(cudaMemsetAsync(c.tc_bad.p, 0, std::max<int64_t>(c.ncells, 1), st));
  FMM_CUDA(cudaMemsetAsync(c.tc_cnt.p, 0, sizeof(int) * kMaxTcLevels, st));
  for (size_t i = 0; i < cands.size(); ++i) {
    FMM_CUDA(cudaMemcpyAsync(c.tc_tbl.p + w.tbl_off[i], cands[i].tbl.data(), sizeof(short) * cands[i].tbl.size(),
                             cudaMemcpyHostToDevice, st));
    FMM_CUDA(cudaMemcpyAsync(c.tc_codes.p + code_off[i], cands[i].codes.data(), sizeof(int) * cands[i].D,
                             cudaMemcpyHostToDevice, st));
  }
  c.tc_off.reserve(kMaxTcLevels);
  FMM_CUDA(cudaMemcpyAsync(c.tc_off.p, tgt_off.data(), sizeof(int64_t) * tgt_off.size(), cudaMemcpyHostToDevice, st));
  c.tc_good.reserve((c.nm2l + 31) / 32 + 1);
  FMM_CUDA(cudaMemsetAsync(c.tc_good.p, 0, sizeof(unsigned) * ((c.nm2l + 31) / 32 + 1), st));
  c.dcount.reserve(1);
  FMM_CUDA(cudaMemsetAsync(c.dcount.p, 0, sizeof(unsigned long long), st));
  c.tc_tmp.reserve(kMaxLevel + 2);
  c.tc_extra.reserve(std::max<int64_t>(c.ncells, 1));
  FMM_CUDA(cudaMemsetAsync(c.tc_extra.p, 0, std::max<int64_t>(c.ncells, 1), st));
  FMM_CUDA(cudaMemsetAsync(c.tc_tmp.p, 0, sizeof(int), st));
  FMM_LAUNCH(c, k_tc_verify_entries, gl, 256, 0, c.m2l.p, c.nm2l, w, g, c.tc_tbl.p, c.tc_mask.p, c.tc_bad.p,
             c.tc_good.p, c.tc_extra.p);
  FMM_LAUNCH(c, k_tc_accept, 148 * 4, 256, 0, w, c.tc_mask.p, c.tc_bad.p, c.tc_skip.p, c.tc_tgt.p, c.tc_off.p,
             c.tc_cnt.p, c.dcount.p, c.tc_extra.p, c.tc_tmp.p);
  FMM_CUDA(cudaStreamSynchronize(st));    // host vectors above are read by the copies
  std::vector<int> cnt(cands.size());
  unsigned long long nent = 0;
  int mixed = 0;
  FMM_CUDA(cudaMemcpyAsync(cnt.data(), c.tc_cnt.p, sizeof(int) * cands.size(), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaMemcpyAsync(&nent, c.dcount.p, sizeof(nent), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaMemcpyAsync(&mixed, c.tc_tmp.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  c.tc_mixed = mixed != 0;                 // else a taken cell's entries are all on the tensor path
  // Morton order of the targets (= cell index order within a level)
  for (size_t i = 0; i < cands.size(); ++i) {
    const int n = cnt[i];
    if (n <= 0) continue;
    const int* in = c.tc_tgt.p + tgt_off[i];
    int* outp = c.tc_tgt2.p + tgt_off[i];
    tc_cub(c, [&](void* tmp, size_t& bytes) {
      return cub::DeviceRadixSort::SortKeys(tmp, bytes, in, outp, n, 0, 32, st);
    });
  }
  std::vector<int64_t> op_off(cands.size(), -1);
  for (size_t i = 0; i < cands.size(); ++i)
    if (cnt[i] > 0) {
      op_off[i] = op_total;
      op_total += (int64_t)cands[i].D * T.opk[kNKB];
    }
  if (op_total == 0) return;
  // the operators depend only on (level, canonical offsets): rebuilt only when those change
  std::vector<int> sig;
  for (size_t i = 0; i < cands.size(); ++i)
    if (cnt[i] > 0) {
      sig.push_back(cands[i].lt);
      sig.push_back(cands[i].D);
      sig.insert(sig.end(), cands[i].codes.begin(), cands[i].codes.end());
    }
  const bool rebuild = sig != c.tc_op_sig || c.tc_op.p == nullptr;
  if (rebuild) {
    c.tc_op.reserve(op_total);
    c.tc_op_sig = sig;
  }
  for (size_t i = 0; i < cands.size(); ++i) {
    if (cnt[i] <= 0) continue;
    if (rebuild)
      FMM_LAUNCH(c, k_tc_operator, (unsigned)cands[i].D, 256, 0, c.tc_codes.p + code_off[i], T, c.tc_op.p + op_off[i]);
    TcLevel tl;
    tl.lt = cands[i].lt;
    tl.D = cands[i].D;
    tl.ntgt = cnt[i];
    tl.tgt_off = tgt_off[i];
    tl.code_off = code_off[i];
    tl.op_off = op_off[i];
    tl.mask_off = w.mask_off[i];
    tl.lb = w.lb[i];
    tl.W = w.W[i];
    c.tc_levels.push_back(tl);
  }
  c.tc_entries = (int64_t)nent;           // the entries the tensor path evaluates (masked rows excluded)
  // longest CTAs first
  std::sort(c.tc_levels.begin(), c.tc_levels.end(), [](const TcLevel& a, const TcLevel& b) { return a.D > b.D; });
}

void m2l_tc_run(Ctx& c) {
  if (c.tc_levels.empty()) return;
  // TC_AT: enough shared memory that no more CTAs than kCtasPerSm (TMEM allocations) share an SM
  const int smem = TC_AT ? std::max(kStages * kStage, (kCtasPerSm == 1 ? 120 : 80) * 1024) : kStages * kStage;
  FMM_CUDA(cudaFuncSetAttribute(k_m2l_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const TcGeo g = make_geo(c);
  const TcTables T = make_tables();
  // packed, 16-byte aligned copy of the multipoles for the row gathers
  c.tc_mp.reserve((size_t)c.ncells * kNKB * kMpLine * 4);
  {
    const int64_t n4 = (int64_t)c.ncells * kNKB * kMpLine;
    FMM_LAUNCH(c, k_tc_pack, (unsigned)std::min<int64_t>((n4 + 255) / 256, 148 * 32), 256, 0, c.M.p,
               (int64_t)c.ncells, (float4*)c.tc_mp.p);
  }
  for (size_t g0 = 0; g0 < c.tc_levels.size(); g0 += kMaxTcLevels) {
    TcArgs args{};
    int ctas = 0;
    args.nlv = (int)std::min<size_t>(kMaxTcLevels, c.tc_levels.size() - g0);
    for (int i = 0; i < args.nlv; ++i) {
      const TcLevel& tl = c.tc_levels[g0 + i];
      const int nblk = (int)((3 * (int64_t)tl.ntgt + kRows - 1) / kRows);
      const int gsize = TC_OGROUP > 0 ? TC_OGROUP : tl.D;
      args.lv[i] = {c.tc_tgt2.p + tl.tgt_off, c.tc_codes.p + tl.code_off, c.tc_op.p + tl.op_off,
                    c.tc_mask.p + tl.mask_off, c.tc_skip.p, tl.ntgt, tl.lt, tl.D, ctas, tl.lb, tl.W, nblk, gsize};
      ctas += nblk * ((tl.D + gsize - 1) / gsize);
    }
    FMM_LAUNCH(c, k_m2l_tc, (unsigned)ctas, kThreads, smem, args, T, g, (const float4*)c.tc_mp.p, c.Lc.p);
  }
}

}  // namespace fmmb
