// p2p.cu -- a12: the near field (P2P, fig:kernels P:103) of Eq. 1 and Eq. 3.
//
// For each list entry (A <- B, img) and i in A, j in B, r = x_i - x_j - img L:
//   u_i += f(r) alpha_j x r,                         f = g(rho)/(4 pi r^3)
//   s_i += f (alpha_j x alpha_i) + (f'/r)(r.alpha_i)(alpha_j x r),
//   f'/r = ((4/sqrt pi) rho^3 e^{-rho^2} - 3 g)/(4 pi r^5), rho = r/(sqrt2 sigma_j)
// (readings Z1, Z3, Z4, Z7).  sum_j f (alpha_j x alpha_i) is
// accumulated as (sum_j f alpha_j) x alpha_i.
//
// Mapping (sm_100a, bound by the FP32 FMA pipe: 75.8% busy at C3, r01 v19): one warp per target leaf, two target
// particles per lane held in registers, so every shared-memory source load
// feeds two pair evaluations.  Each source leaf of the target's segment is
// staged in shared memory as float4 tiles in *target-leaf-centred*
// coordinates -- the image shift and the centring are done once per source in
// double and rounded to FP32 ("Fix B") -- and the FP32
// partial over each tile (<= 64 sources) is added to a per-target FP64
// accumulator ("Fix A").  MUFU ops are the approximate .ftz forms.
//
// Cutoff g (Eq. 2).  Table 1 counts two expf and no erf, i.e. the
// paper's kernel approximated erf (reading Z6).  Here g is evaluated without
// erf: g = 1 - e^{-rho^2} (erfcx(rho) + (2/sqrt pi) rho) with erfcx fitted by a
// degree-6 polynomial in t = 1/(1 + rho/2), and a 9-term Taylor series of
// g/rho^3 in rho^2 for rho < 0.8 (evaluated only when some lane of the warp
// has such a close pair); |g - g_exact| <= 2e-7 (FP32 evaluation, checked by
// the parity tests through fmm_eval_cutoff).  The pair arithmetic of the two
// targets of a lane is packed into FP32x2 (FFMA2) with the source operands
// broadcast, halving the issue slots per pair.  Sources whose every pair
// with the targets has rho >= 4.6 (distance from the source to the tight box
// of the targets >= 4.6 sqrt2 sigma_j, tested once per source while staging) are
// compacted to the front of the tile and take the exact singular branch;
// the rest follow, those farther than rho = 0.8 from the box first, so only the
// last group (sources that may form a close pair) carries the warp vote for the
// close-pair series.  The singular branch:
// there 1 - g < 4e-9 and rho g' = (4/sqrt pi) rho^3 e^{-rho^2} < 1.5e-7 (both
// within reading Z6's 2e-7), so g = 1 and f'/r = -3/(4 pi r^5) in FP32.
// fmm_eval_pair_kernel exports both branches' g and rho g' for the Z6 test.
#include <cub/cub.cuh>

#include "ctx.cuh"

namespace fmmb {

namespace {

constexpr int TP = 64;           // targets per block pass and sources per tile
constexpr int NT = 32;           // threads per block (one warp, 2 targets each)
constexpr float kFarRho2 = 4.6f * 4.6f;
constexpr float kCloseRho2 = 0.64f;   // pairs below take the Taylor series (rho < 0.8)
constexpr int kAdjChunk = 32;    // sources per FP32 partial for source leaves touching the target leaf
#ifndef P2P_MINB
#define P2P_MINB 16      // blocks (warps) per SM the launch bounds target
#endif
#ifndef P2P_UF
#define P2P_UF 6         // unroll of the singular-branch loop
#endif
#ifndef P2P_UN
#define P2P_UN 3         // unroll of the regularised-branch loop (r02 sweep after the three-group
#endif                   // staging, C3 k_p2p ms: 4/4 204.15, 4/3 202.62, 6/3 201.65, 8/3 201.74,
                         // 5/3 203.67, 4/5 203.14; profiles/r02_ab2_p2p_occupancy.txt)
#ifndef P2P_ADJ_MODE
#define P2P_ADJ_MODE 1
#endif   // rho^2 at and beyond which the singular branch is exact to Z6

__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// g(rho) of Eq. 2 from rho, x = rho^2, e = exp(-rho^2): the two pieces.
//   series: g = rho^3 sum_k a_k x^k               (accurate as rho -> 0; used for x < 0.64)
//   erfcx : g = 1 - e (h(t) + (2/sqrt pi) rho),  h ~ erfcx, t = 1/(1 + rho/2)
// s(x) = g / rho^3 = (4/sqrt pi) sum_n (-x)^n / (n! (2n+3))
__device__ __forceinline__ float2 series_s(float2 x) {
  float2 s = make_float2(2.945851975e-06f, 2.945851975e-06f);
  const float a[8] = {-2.633938311e-05f, 2.089590998e-04f, -1.446640003e-03f, 8.548326790e-03f,
                      -4.179182276e-02f, 1.611970216e-01f, -4.513516724e-01f, 7.522527575e-01f};
#pragma unroll
  for (int k = 0; k < 8; ++k) s = __ffma2_rn(s, x, make_float2(a[k], a[k]));
  return s;
}
// T(x) = ((4/sqrt pi) e^{-x} - 3 s(x)) / x = (4/sqrt pi) sum_m (-1)^{m+1} 2(m+1) x^m / ((m+1)! (2m+5))
__device__ __forceinline__ float2 series_t(float2 x) {
  float2 s = make_float2(5.407844333e-07f, 5.407844333e-07f);
  const float a[9] = {-5.330589414e-06f, 4.713363271e-05f, -3.687513618e-04f, 2.507509260e-03f, -1.446639958e-02f,
                      6.838661619e-02f, -2.507509260e-01f, 6.447880955e-01f, -9.027033337e-01f};
#pragma unroll
  for (int k = 0; k < 9; ++k) s = __ffma2_rn(s, x, make_float2(a[k], a[k]));
  return s;
}
__device__ __forceinline__ float2 series_g(float2 rho, float2 x) {
  return __fmul2_rn(series_s(x), __fmul2_rn(rho, x));
}
__device__ __forceinline__ float2 erfcx_g(float2 rho, float2 e) {
  const float2 d = __ffma2_rn(make_float2(0.5f, 0.5f), rho, make_float2(1.f, 1.f));
  const float2 t = make_float2(rcp_approx(d.x), rcp_approx(d.y));
  float2 h = make_float2(6.501056254e-02f, 6.501056254e-02f);
  const float c[6] = {-4.661040902e-01f, 9.906343818e-01f, -3.476467133e-01f, 5.238698721e-01f,
                      2.293880880e-01f, 4.825282376e-03f};
#pragma unroll
  for (int k = 0; k < 6; ++k) h = __ffma2_rn(h, t, make_float2(c[k], c[k]));
  const float2 y = __ffma2_rn(make_float2(1.1283791670955126f, 1.1283791670955126f), rho, h);
  return __ffma2_rn(make_float2(-e.x, -e.y), y, make_float2(1.f, 1.f));
}
// scalar form (same arithmetic) for fmm_eval_cutoff
__device__ __forceinline__ float cutoff_g(float rho, float x, float e) {
  const float2 gs = series_g(make_float2(rho, rho), make_float2(x, x));
  const float2 gl = erfcx_g(make_float2(rho, rho), make_float2(e, e));
  return x < 0.64f ? gs.x : gl.x;
}

struct PCells {
  const int *level, *qx, *qy, *qz, *begin, *count;
};

// Per-tile FP32 accumulators of the lane's two targets, packed (target 0, 1).
// With w_j = alpha_j x (y_j - C) (y_j the source, C its leaf centre) the
// pair sums factor through the source leaf (one product per pair instead of
// the cross product alpha_j x r_ij):
//   sum_j f alpha_j x r_ij   = (sum_j f alpha_j) x (x_i - C) - sum_j f w_j
//   sum_j q alpha_j x r_ij   = (sum_j q alpha_j) x (x_i - C) - sum_j q w_j,   q = fp (r.alpha_i)
// |x_i - C| and |y_j - C| are bounded by the leaf distances, so the
// difference loses at most a few bits (the parity tests bound it).
struct Acc2 {
  float2 fa0, fa1, fa2, fw0, fw1, fw2, qa0, qa1, qa2, qw0, qw1, qw2;
};
__device__ __forceinline__ void zero(Acc2& A) {
  A.fa0 = A.fa1 = A.fa2 = A.fw0 = A.fw1 = A.fw2 = make_float2(0.f, 0.f);
  A.qa0 = A.qa1 = A.qa2 = A.qw0 = A.qw1 = A.qw2 = make_float2(0.f, 0.f);
}
__device__ __forceinline__ float2 bc(float v) { return make_float2(v, v); }

// one source on the lane's two targets, all arithmetic packed FP32x2
// (FFMA2/FMUL2/FADD2).  Shared-memory operands per source:
//   q = (x', y', z', -log2(e)/(2 sigma^2))      a = (alpha/(4 pi), 1/(sqrt2 sigma))
//   w = alpha/(4 pi) x (y - C)
//   c = (1/(2 sqrt2 sigma), (2/sqrt pi)/(sqrt2 sigma), -(4/(3 sqrt pi))/(sqrt2 sigma)^3, 1/(2 sigma^2))  [NEAR only]
// The stretching accumulators carry fp/(-3) (fp = f'/r); flush multiplies by -3.
// MODE 0: the exact singular kernel; MODE 1 / 2: the regularised one, 2 with the
// close-pair series (sources staged as possibly closer than rho = 0.8 to a target):
//   far : f = 1/r^3,  fp/(-3) = 1/r^5
//   near: f = g/r^3,  fp/(-3) = g/r^5 - (4/(3 sqrt pi)) (1/(sqrt2 sigma))^3 e^{-rho^2}/r^2
//         (= ((4/sqrt pi) rho^3 e^{-rho^2} - 3 g)/r^5 / (-3)),
//   g from erfcx with rho = r/(sqrt2 sigma) entering only through FFMA2s on r.
template <int MODE>
__device__ __forceinline__ void pair2(Acc2& A, float2 x0, float2 x1, float2 x2, float2 b0, float2 b1, float2 b2,
                                      const float4 q, const float4 a, const float4 w, const float4 c) {
  constexpr bool NEAR = MODE > 0;
  const float2 rx = __fadd2_rn(x0, bc(-q.x)), ry = __fadd2_rn(x1, bc(-q.y)), rz = __fadd2_rn(x2, bc(-q.z));
  const float2 r2 = __ffma2_rn(rz, rz, __ffma2_rn(ry, ry, __fmul2_rn(rx, rx)));
  float2 inv;
  // r = 0 (the self pair) gives inf/NaN here, but such a pair always takes the
  // close-pair series below (its rho^2 = 0 votes the warp in), which replaces f
  // and f'/r by selection; rho >= 4.6 in the singular branch: r > 0
  inv = make_float2(rsqrt_approx(r2.x), rsqrt_approx(r2.y));
  const float2 inv2 = __fmul2_rn(inv, inv);
  const float2 inv3 = __fmul2_rn(inv2, inv);
  float2 f, fp3;
  if (NEAR) {
    const float2 ea = __fmul2_rn(r2, bc(q.w));                 // -rho^2 log2(e)
    const float2 e = make_float2(ex2_approx(ea.x), ex2_approx(ea.y));
    const float2 r = __fmul2_rn(r2, inv);
    // g = 1 - e (h(t) + (2/sqrt pi) rho), h ~ erfcx, t = 1/(1 + rho/2)
    const float2 d = __ffma2_rn(r, bc(c.x), bc(1.f));
    const float2 tt = make_float2(rcp_approx(d.x), rcp_approx(d.y));
    float2 h = bc(6.501056254e-02f);
    const float hc[6] = {-4.661040902e-01f, 9.906343818e-01f, -3.476467133e-01f, 5.238698721e-01f,
                         2.293880880e-01f, 4.825282376e-03f};
#pragma unroll
    for (int k = 0; k < 6; ++k) h = __ffma2_rn(h, tt, bc(hc[k]));
    const float2 y = __ffma2_rn(r, bc(c.y), h);
    const float2 g = __ffma2_rn(make_float2(-e.x, -e.y), y, bc(1.f));
    f = __fmul2_rn(g, inv3);
    fp3 = __fmul2_rn(__ffma2_rn(bc(c.z), e, f), inv2);
    // close pairs (rho < 0.8, evaluated only when some lane of the warp has
    // one): f = g/r^3 and f'/r from the Taylor series in x = rho^2 without
    // dividing by r, so they stay exact as r -> 0 (r = 0 still contributes 0, Z7):
    //   f = k^{3/2} s(x),  f'/r = k^{5/2} T(x),  k = 1/(2 sigma^2)
    constexpr float ea_close = -0.64f * 1.4426950408889634f;
    if (MODE == 2 && __any_sync(0xffffffffu, fmaxf(ea.x, ea.y) > ea_close)) {
      const float kk = c.w, k32 = kk * a.w, k52 = kk * k32;
      const float2 x = __fmul2_rn(r2, bc(kk));
      const float2 sx = series_s(x), tx = series_t(x);
      const bool c0 = ea.x > ea_close, c1 = ea.y > ea_close;
      f = make_float2(c0 ? (r2.x > 0.f ? k32 * sx.x : 0.f) : f.x, c1 ? (r2.y > 0.f ? k32 * sx.y : 0.f) : f.y);
      fp3 = make_float2(c0 ? (r2.x > 0.f ? (-1.f / 3.f) * k52 * tx.x : 0.f) : fp3.x,
                        c1 ? (r2.y > 0.f ? (-1.f / 3.f) * k52 * tx.y : 0.f) : fp3.y);
    }
  } else {
    f = inv3;
    fp3 = __fmul2_rn(inv3, inv2);
  }
  A.fa0 = __ffma2_rn(f, bc(a.x), A.fa0); A.fa1 = __ffma2_rn(f, bc(a.y), A.fa1); A.fa2 = __ffma2_rn(f, bc(a.z), A.fa2);
  A.fw0 = __ffma2_rn(f, bc(w.x), A.fw0); A.fw1 = __ffma2_rn(f, bc(w.y), A.fw1); A.fw2 = __ffma2_rn(f, bc(w.z), A.fw2);
  const float2 qq = __fmul2_rn(fp3, __ffma2_rn(rz, b2, __ffma2_rn(ry, b1, __fmul2_rn(rx, b0))));
  A.qa0 = __ffma2_rn(qq, bc(a.x), A.qa0); A.qa1 = __ffma2_rn(qq, bc(a.y), A.qa1); A.qa2 = __ffma2_rn(qq, bc(a.z), A.qa2);
  A.qw0 = __ffma2_rn(qq, bc(w.x), A.qw0); A.qw1 = __ffma2_rn(qq, bc(w.y), A.qw1); A.qw2 = __ffma2_rn(qq, bc(w.z), A.qw2);
}

// per-target FP64 accumulators live in shared memory ([quantity][lane], 18
// per lane: the two targets' u, s, sum f alpha), freeing registers for
// occupancy; each tile's FP32 sums are combined (in FP64) once per tile:
//   u += fa x (x_i - C) - fw,   s += -3 (qa x (x_i - C) - qw),   F += fa
constexpr int kDQ = 18;
__device__ __forceinline__ void flush(double (*sD)[NT], int lane, const Acc2& A, float2 X0, float2 X1, float2 X2,
                                      float C0, float C1, float C2) {
  // tile sums in FP32 (packed over the two targets), then into the FP64 accumulators
  const float2 x = __fadd2_rn(X0, bc(-C0)), y = __fadd2_rn(X1, bc(-C1)), z = __fadd2_rn(X2, bc(-C2));
  const float2 u0 = __fadd2_rn(__ffma2_rn(A.fa1, z, __fmul2_rn(A.fa2, __fmul2_rn(y, bc(-1.f)))), __fmul2_rn(A.fw0, bc(-1.f)));
  const float2 u1 = __fadd2_rn(__ffma2_rn(A.fa2, x, __fmul2_rn(A.fa0, __fmul2_rn(z, bc(-1.f)))), __fmul2_rn(A.fw1, bc(-1.f)));
  const float2 u2 = __fadd2_rn(__ffma2_rn(A.fa0, y, __fmul2_rn(A.fa1, __fmul2_rn(x, bc(-1.f)))), __fmul2_rn(A.fw2, bc(-1.f)));
  const float2 s0 = __fadd2_rn(__ffma2_rn(A.qa1, z, __fmul2_rn(A.qa2, __fmul2_rn(y, bc(-1.f)))), __fmul2_rn(A.qw0, bc(-1.f)));
  const float2 s1 = __fadd2_rn(__ffma2_rn(A.qa2, x, __fmul2_rn(A.qa0, __fmul2_rn(z, bc(-1.f)))), __fmul2_rn(A.qw1, bc(-1.f)));
  const float2 s2 = __fadd2_rn(__ffma2_rn(A.qa0, y, __fmul2_rn(A.qa1, __fmul2_rn(x, bc(-1.f)))), __fmul2_rn(A.qw2, bc(-1.f)));
  const float2 v[9] = {u0, u1, u2, s0, s1, s2, A.fa0, A.fa1, A.fa2};
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const double w = q >= 3 && q < 6 ? -3.0 : 1.0;     // s carries fp/(-3)
    sD[q][lane] += w * (double)v[q].x;
    sD[9 + q][lane] += w * (double)v[q].y;
  }
}

// leaf-local FP32 source data (a12 staging, once per evaluate): for every
// particle of every leaf, (x - c_leaf) rounded from double and w = 1/(2 sigma^2),
// and sqrt(w) = 1/(sqrt2 sigma) in the free fourth lane of (alpha, .)
__global__ void k_leaf_local(const int* __restrict__ leaf, const unsigned char* __restrict__ cflag, PCells c,
                             int64_t c0, int64_t ncells, double lo0, double lo1, double lo2, double L,
                             const float4* __restrict__ pos, float4* __restrict__ posl, float4* __restrict__ alp) {
  const int lane = threadIdx.x & 31;
  for (int64_t cell = c0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); cell < ncells;
       cell += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    if (!leaf[cell] || (cflag && cflag[cell])) continue;     // LET: frontier cells and body-less leaves hold no particles
    const double s = L / (double)(1 << c.level[cell]);
    const double cx = lo0 + (c.qx[cell] + 0.5) * s, cy = lo1 + (c.qy[cell] + 0.5) * s, cz = lo2 + (c.qz[cell] + 0.5) * s;
    const int b = c.begin[cell], n = c.count[cell];
    for (int i = lane; i < n; i += 32) {
      const float4 p = pos[b + i];
      const float w = 1.0f / (2.0f * p.w * p.w);
      posl[b + i] = make_float4((float)((double)p.x - cx), (float)((double)p.y - cy), (float)((double)p.z - cz), w);
      alp[b + i].w = sqrtf(w);
    }
  }
}

// SPL > 1 (small target leaves, <= 64/SPL particles): the warp's lanes form SPL
// groups holding the same 64/SPL targets (two per lane as always), and group g
// takes sources g, g + SPL, ... of every tile (the tile's far and near parts are
// padded with zero-strength sources to multiples of SPL so every lane runs the
// same loop trips); each lane keeps its FP64 accumulators, and the groups' sums
// are added in a fixed order at the end.  Lanes are otherwise idle on leaves
// with few particles (adaptive trees, SURVEY 8d stress variants).
template <int MINB, int UF, int UN, bool ACC, int SPL>
__global__ void __launch_bounds__(NT, MINB) k_p2p(const int* __restrict__ leaf_ids, const int* __restrict__ seg_b,
                                            const int* __restrict__ seg_e, const uint64_t* __restrict__ lst,
                                            PCells c, double lo0, double lo1, double lo2, double L,
                                            double px, double py, double pz,
                                            const float4* __restrict__ posl, const float4* __restrict__ alp,
                                            float* __restrict__ un, float* __restrict__ sn,
                                            unsigned long long* __restrict__ near_pairs) {
  constexpr int NG = NT / SPL;        // lanes per source group
  constexpr int TPASS = 2 * NG;       // targets per pass
  __shared__ float4 sx[TP + 12];   // (x', y', z', -log2(e)/(2 sigma^2))   (+ SPL padding of 3 parts)
  __shared__ float4 sa[TP + 12];   // (alpha/(4 pi), 1/(sqrt2 sigma))
  __shared__ float4 sw[TP + 12];   // alpha/(4 pi) x (y - C), C = the source leaf centre
  __shared__ float4 sc[TP + 12];   // near-kernel constants of the source (see pair2)
  __shared__ double sD[kDQ][NT];
  __shared__ float2 sB[3][NT];   // the lane's target alpha pairs (reloaded as aligned register pairs)
  const float k4 = (float)(1.0 / (4.0 * kPi));
  const int lane = threadIdx.x;
  const int grpl = lane / NG, pl = lane - NG * (lane / NG);   // source group, target pair
  const int leaf = leaf_ids[blockIdx.x];
  const int lev = c.level[leaf], tb = c.begin[leaf], tcnt = c.count[leaf];
  const double s = L / (double)(1 << lev);
  const double cx = lo0 + (c.qx[leaf] + 0.5) * s, cy = lo1 + (c.qy[leaf] + 0.5) * s,
               cz = lo2 + (c.qz[leaf] + 0.5) * s;
  const int eb = seg_b[leaf], ee = seg_e[leaf];
  if (ACC && eb >= ee) return;                    // second pass (remote sources): nothing to add
  const float hst = (float)(0.5 * s);
  unsigned long long nnear = 0;                   // pairs evaluated with the regularised kernel
  for (int t0 = 0; t0 < tcnt; t0 += TPASS) {
    const int i0 = t0 + pl, i1 = t0 + pl + NG;
    const bool v0 = i0 < tcnt, v1 = i1 < tcnt;
    // absent targets sit far away so they never trigger the close-pair branch
    float x00 = 1e4f, x01 = 1e4f, x02 = 1e4f, x10 = 1e4f, x11 = 1e4f, x12 = 1e4f;
    float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
    if (v0) {
      const float4 p = posl[tb + i0];                // leaf-local = target-frame coordinates
      x00 = p.x; x01 = p.y; x02 = p.z;
      a0 = alp[tb + i0];
    }
    if (v1) {
      const float4 p = posl[tb + i1];
      x10 = p.x; x11 = p.y; x12 = p.z;
      a1 = alp[tb + i1];
    }
    // packed once per target pass (the target alphas live only in these pairs,
    // so the loops need no register moves to re-pair them)
    const float2 X0 = make_float2(x00, x10), X1 = make_float2(x01, x11), X2 = make_float2(x02, x12);
    float2 B0 = make_float2(a0.x, a1.x), B1 = make_float2(a0.y, a1.y), B2 = make_float2(a0.z, a1.z);
    sB[0][lane] = B0;
    sB[1][lane] = B1;
    sB[2][lane] = B2;
    // tight box of this pass's targets (centre bc, half extent bh): the far test
    // below measures a source's distance to it (absent targets excluded)
    float bc[3], bh[3];
    {
      const float xs[3][2] = {{x00, x10}, {x01, x11}, {x02, x12}};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        float lo = fminf(v0 ? xs[a][0] : 1e30f, v1 ? xs[a][1] : 1e30f);
        float hi = fmaxf(v0 ? xs[a][0] : -1e30f, v1 ? xs[a][1] : -1e30f);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
          hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        bc[a] = 0.5f * (lo + hi);
        bh[a] = 0.5f * (hi - lo) * 1.0001f + 1e-7f * hst;   // rounding margin
      }
    }
#pragma unroll
    for (int q = 0; q < kDQ; ++q) sD[q][lane] = 0.0;
    for (int e = eb; e < ee; ++e) {
      const uint64_t ent = lst[e];
      const int src = (int)((ent >> 5) & 0x7ffffff), img = (int)(ent & 31);
      // the source leaf centre in the target frame (image shift included), in
      // double then rounded: sources are y' + C with y' their leaf-local coordinates
      const double ss = L / (double)(1 << c.level[src]);
      const float C0 = (float)(lo0 + (c.qx[src] + 0.5) * ss + (img % 3 - 1) * px - cx);
      const float C1 = (float)(lo1 + (c.qy[src] + 0.5) * ss + ((img / 3) % 3 - 1) * py - cy);
      const float C2 = (float)(lo2 + (c.qz[src] + 0.5) * ss + (img / 9 - 1) * pz - cz);
      const int sb = c.begin[src], scnt = c.count[src];
      // source leaf touching (or equal to) the target leaf: |C_d| <= s_t/2 + s_s/2 on every axis
      const float reach = (float)(0.5 * (s + ss)) * 1.0001f;
      const bool adj = fabsf(C0) <= reach && fabsf(C1) <= reach && fabsf(C2) <= reach;
#if P2P_ADJ_MODE == 1
      const int tstep = adj ? kAdjChunk : TP;     // touching leaf: FP32 partials over 32 sources (below)
#else
      const int tstep = TP;
#endif
      for (int s0 = 0; s0 < scnt; s0 += tstep) {
        __syncwarp();
        // stage the tile, far sources first: a source is "far" when it is
        // >= 4.6 sqrt2 sigma_j from the whole target leaf cube, so every pair
        // it forms has rho >= 4.6 (then 1 - g < 4e-9 and rho g' < 1.5e-7: the
        // exact singular branch, reading Z6)
        float4 qv[2], av[2], wv[2], cv[2];
        bool fj[2], vj[2], cj[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = s0 + lane + h * NT;
          vj[h] = j < scnt && j < s0 + tstep;
          fj[h] = cj[h] = false;
          if (vj[h]) {
            const float4 p = posl[sb + j];               // (y - C, 1/(2 sigma^2))
            const float4 a = alp[sb + j];
            const float w = p.w;
            const float qx = p.x + C0, qy = p.y + C1, qz = p.z + C2;
            const float aw = a.w;                        // sqrt(w) (k_leaf_local)
            qv[h] = make_float4(qx, qy, qz, -1.4426950408889634f * w);
            av[h] = make_float4(a.x * k4, a.y * k4, a.z * k4, aw);
            wv[h] = make_float4(av[h].y * p.z - av[h].z * p.y, av[h].z * p.x - av[h].x * p.z,
                                av[h].x * p.y - av[h].y * p.x, 0.f);
            cv[h] = make_float4(0.5f * aw, 1.1283791670955126f * aw, -0.75225277806367504f * aw * aw * aw, w);
            const float gx = fmaxf(0.f, fabsf(qx - bc[0]) - bh[0]), gy = fmaxf(0.f, fabsf(qy - bc[1]) - bh[1]),
                        gz = fmaxf(0.f, fabsf(qz - bc[2]) - bh[2]);
            const float d2w = (gx * gx + gy * gy + gz * gz) * w;
            fj[h] = d2w >= kFarRho2 * 1.0001f;
            cj[h] = !fj[h] && d2w < kCloseRho2 * 1.0001f;   // may form a pair with rho < 0.8
          }
        }
        const unsigned lt = (1u << lane) - 1u;
        const unsigned f0 = __ballot_sync(0xffffffffu, fj[0]), f1 = __ballot_sync(0xffffffffu, fj[1]);
        const unsigned n0 = __ballot_sync(0xffffffffu, vj[0] && !fj[0] && !cj[0]),
                       n1 = __ballot_sync(0xffffffffu, vj[1] && !fj[1] && !cj[1]);
        const unsigned k0 = __ballot_sync(0xffffffffu, cj[0]), k1 = __ballot_sync(0xffffffffu, cj[1]);
        const int nfar = __popc(f0) + __popc(f1), nnc = __popc(n0) + __popc(n1), ncl = __popc(k0) + __popc(k1);
        const int nj = nfar + nnc + ncl;
        // tile order: far | near | near with possible close pairs; SPL > 1: each part
        // padded to a multiple of SPL
        const int nfarP = (nfar + SPL - 1) / SPL * SPL;
        const int nncE = nfarP + (nnc + SPL - 1) / SPL * SPL;
        const int njP = nncE + (ncl + SPL - 1) / SPL * SPL;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (!vj[h]) continue;
          const int dst = fj[h] ? (h == 0 ? __popc(f0 & lt) : __popc(f0) + __popc(f1 & lt))
                        : cj[h] ? nncE + (h == 0 ? __popc(k0 & lt) : __popc(k0) + __popc(k1 & lt))
                                : nfarP + (h == 0 ? __popc(n0 & lt) : __popc(n0) + __popc(n1 & lt));
          sx[dst] = qv[h];
          sa[dst] = av[h];
          sw[dst] = wv[h];
          sc[dst] = cv[h];
        }
        if (SPL > 1) {
          // zero-strength padding sources far from the targets (finite kernel values)
          const int pf = nfarP - nfar, pn = nncE - nfarP - nnc, pc = njP - nncE - ncl;
          if (lane < pf + pn + pc) {
            const int dst = lane < pf ? nfar + lane : (lane < pf + pn ? nfarP + nnc + (lane - pf) : nncE + ncl + (lane - pf - pn));
            sx[dst] = make_float4(1e4f, 1e4f, 1e4f, -1.4426950408889634f);
            sa[dst] = make_float4(0.f, 0.f, 0.f, 1.f);
            sw[dst] = make_float4(0.f, 0.f, 0.f, 0.f);
            sc[dst] = make_float4(0.5f, 1.1283791670955126f, -0.75225277806367504f, 1.f);
          }
        }
        __syncwarp();
        nnear += (unsigned long long)(nj - nfar) * (unsigned long long)min(TPASS, tcnt - t0);
        {
          // reloaded per tile as 64-bit pairs so they sit in aligned register
          // pairs (otherwise ptxas re-pairs them with 6 MOVs per source: 218 -> 204 ms at C3)
          const unsigned b = (unsigned)__cvta_generic_to_shared(&sB[0][lane]);
          asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(B0.x), "=f"(B0.y) : "r"(b));
          asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(B1.x), "=f"(B1.y) : "r"(b + 8 * NT));
          asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(B2.x), "=f"(B2.y) : "r"(b + 16 * NT));
        }
        // FP32 partials added into the FP64 accumulators by flush: per tile of
        // 64 sources, or 32 for a source leaf that touches the target leaf (its
        // close pairs carry the largest terms, and the factorisation through C
        // amplifies their rounding by |x_i - C|/|r|; FP32 emulation at C4:
        // stretching rel-L2 8.9e-6 -> 4.6e-6).  P2P_ADJ_MODE 1 stages
        // such a leaf in tiles of 32 (emulation: 6.2e-6; 16: 4.6e-6 at +2 ms more); mode 0 chunks the loops; mode 2 does neither.
        Acc2 A;
        zero(A);
#pragma unroll UF
        for (int jj = grpl; jj < nfarP; jj += SPL) pair2<0>(A, X0, X1, X2, B0, B1, B2, sx[jj], sa[jj], sw[jj], sa[jj]);
#pragma unroll UN
        for (int jj = nfarP + grpl; jj < nncE; jj += SPL)
          pair2<1>(A, X0, X1, X2, B0, B1, B2, sx[jj], sa[jj], sw[jj], sc[jj]);
#pragma unroll 2
        for (int jj = nncE + grpl; jj < njP; jj += SPL)
          pair2<2>(A, X0, X1, X2, B0, B1, B2, sx[jj], sa[jj], sw[jj], sc[jj]);
        flush(sD, lane, A, X0, X1, X2, C0, C1, C2);
      }
    }
    // s += (sum_j f alpha_j) x alpha_i; SPL > 1: the groups' sums, in group order
    if (SPL > 1) __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!(h == 0 ? v0 : v1) || grpl != 0) continue;
      const float4 ai = h == 0 ? a0 : a1;
      double Dv[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        double acc = sD[9 * h + q][pl];
#pragma unroll
        for (int k = 1; k < SPL; ++k) acc += sD[9 * h + q][pl + k * NG];
        Dv[q] = acc;
      }
      const double u0 = Dv[0], u1 = Dv[1], u2 = Dv[2], s0 = Dv[3], s1 = Dv[4], s2 = Dv[5];
      const double f0 = Dv[6], f1 = Dv[7], f2 = Dv[8];
      const int64_t o = 3 * (int64_t)(tb + (h == 0 ? i0 : i1));
      const float r[6] = {(float)u0, (float)u1, (float)u2, (float)(s0 + (f1 * ai.z - f2 * ai.y)),
                          (float)(s1 + (f2 * ai.x - f0 * ai.z)), (float)(s2 + (f0 * ai.y - f1 * ai.x))};
      if (ACC) {
        un[o] += r[0]; un[o + 1] += r[1]; un[o + 2] += r[2];
        sn[o] += r[3]; sn[o + 1] += r[4]; sn[o + 2] += r[5];
      } else {
        un[o] = r[0]; un[o + 1] = r[1]; un[o + 2] = r[2];
        sn[o] = r[3]; sn[o + 1] = r[4]; sn[o + 2] = r[5];
      }
    }
    if (SPL > 1) __syncwarp();                    // the next pass clears sD
  }
  if (lane == 0 && nnear) atomicAdd(near_pairs, nnear);
}

__global__ void k_eval_cutoff(const float* __restrict__ rho, int64_t n, float* __restrict__ g) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float r = rho[i];
    const float x = r * r;
    g[i] = cutoff_g(r, x, ex2_approx(x * -1.4426950408889634f));
  }
}

// The pair arithmetic of k_p2p (pair2, both branches) on one source at the
// origin with sqrt2 sigma = 1 and targets at r = rho on the x axis (two rho per
// thread, as the lane pairs of k_p2p), alpha_j = alpha_i = x-hat: fa0 = f and
// qa0 = r fp/(-3).  The regularised factors are reported relative to the
// singular ones of the same code (same rsqrt of the same r^2), which isolates
// the cutoff approximation (reading Z6) from the FP32 evaluation of 1/r^k:
//   g = f_reg / f_sing,   rho g' = 3 g - 3 fp_reg / fp_sing
// (f = g/r^3, f'/r = (rho g' - 3 g)/r^5).  branch 0 = the selection
// k_p2p applies (singular, i.e. g = 1 and rho g' = 0, iff rho^2 >= kFarRho2),
// branch 1 = the regularised branch at every rho.
__global__ void k_eval_pair(const float* __restrict__ rho, int64_t n, int branch, float* __restrict__ g,
                            float* __restrict__ rgp) {
  // no early exit: pair2<2> votes across the whole warp
  const int64_t i0 = 2 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
  const float r0 = i0 < n ? rho[i0] : 1.f, r1 = i0 + 1 < n ? rho[i0 + 1] : 1.f;
  const float w = 1.0f;                                     // 1/(2 sigma^2) with sqrt2 sigma = 1
  const float4 q = make_float4(0.f, 0.f, 0.f, -1.4426950408889634f * w);
  const float aw = sqrtf(w);
  const float4 a = make_float4(1.f, 0.f, 0.f, aw);
  const float4 wv = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 cv = make_float4(0.5f * aw, 1.1283791670955126f * aw, -0.75225277806367504f * aw * aw * aw, w);
  const float2 X0 = make_float2(r0, r1), X1 = make_float2(0.f, 0.f), X2 = make_float2(0.f, 0.f);
  const float2 B0 = make_float2(1.f, 1.f), B1 = make_float2(0.f, 0.f), B2 = make_float2(0.f, 0.f);
  Acc2 An, Af;
  zero(An);
  zero(Af);
  pair2<2>(An, X0, X1, X2, B0, B1, B2, q, a, wv, cv);
  pair2<0>(Af, X0, X1, X2, B0, B1, B2, q, a, wv, a);
  const float rr[2] = {r0, r1};
  const float fn[2] = {An.fa0.x, An.fa0.y}, ff[2] = {Af.fa0.x, Af.fa0.y};
  const float pn[2] = {An.qa0.x, An.qa0.y}, pf[2] = {Af.qa0.x, Af.qa0.y};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t i = i0 + h;
    if (i >= n) continue;
    const bool sing = branch == 0 && rr[h] * rr[h] >= kFarRho2;
    if (rr[h] <= 0.f) { g[i] = 0.f; rgp[i] = 0.f; continue; }       // r = 0 contributes nothing (Z7)
    const double gd = sing ? 1.0 : (double)fn[h] / (double)ff[h];
    double rg;
    if (sing) {
      rg = 0.0;
    } else if (rr[h] * rr[h] < 0.64f) {
      // series branch: f'/r from T(x); 3 g - rho g' = 3 fp_reg/fp_sing (no cancellation here)
      rg = 3.0 * gd - 3.0 * (double)pn[h] / (double)pf[h];
    } else {
      // erfcx branch: fp/(-3) = c.z e/r^2 + f/r^2, so rho g' = (4/sqrt pi) rho^3 e with the
      // kernel's e = ex2.approx(-rho^2 log2 e) (pair2's r^2 and q.w; read directly, since
      // 3 g - 3 fp_reg/fp_sing cancels to FP32 resolution when g -> 1)
      const float r2 = rr[h] * rr[h];
      const float e = ex2_approx(r2 * q.w);
      rg = 2.2567583341910251 * (double)e * (double)rr[h] * (double)rr[h] * (double)rr[h];
    }
    g[i] = (float)gd;
    rgp[i] = (float)rg;
  }
}

// leaf size classes for the P2P variants: 0 = > 32 particles (SPL 1), 1 = 17..32 (SPL 2), 2 = <= 16 (SPL 4)
__device__ __forceinline__ int leaf_class(int n) { return n > 32 ? 0 : (n > 16 ? 1 : 2); }
struct LeafClass {
  const int* count;
  int cl;
  __device__ __forceinline__ bool operator()(const int& id) const { return leaf_class(count[id]) == cl; }
};

}  // namespace

void eval_pair_kernel(Ctx& c, const float* rho, int64_t n, int branch, float* g, float* rgp) {
  FMM_LAUNCH(c, k_eval_pair, nblocks((n + 1) / 2, 256), 256, 0, rho, n, branch, g, rgp);
}

void p2p_pass(Ctx& c, float* u_near, float* s_near, int part) {
  if (c.nleaves == 0) return;
  c.dnear.reserve(1);
  if (part != 2) FMM_CUDA(cudaMemsetAsync(c.dnear.p, 0, sizeof(unsigned long long), c.stream));
  PCells pc{c.cells.level.p, c.cells.qx.p, c.cells.qy.p, c.cells.qz.p, c.cells.begin.p, c.cells.count.p};
  // 16 blocks/SM (128 registers), far loop unrolled 6x, near 3x: the best of
  // the occupancy/unroll sweeps on C3 (r01 v16: <16,4,4> 201.8 ms, <16,4,2> 204.0, <16,4,1> 203.1, <16,8,2> 204.8,
  // <12,4,2> 210.2; r02 with the three-group staging: <16,6,3> 201.65 vs <16,4,4> 204.15, 14 or 15 blocks no gain)
  // Prefetching the next list entry while the current tile is evaluated does not pay (r01 v23 A/B,
  // tools/p2p_ab.sh, bit-identical results): its cell-table reads 200.35 -> 200.80 ms, plus its first
  // source tile 207.53 ms (40 B of spills); the tile-boundary load latency is hidden by the other warps.
  // part 1 / 2 (nranks > 1): the entries with local sources while the LET is in flight, then the
  // received sources' entries added (fig:flow_chart)
  c.posl.reserve(std::max<int64_t>(c.nsrc, 1));
  const bool multi = c.cfg.nranks > 1;
  const int64_t c0 = part == 2 ? c.nloc_cells : 0, c1 = part == 1 ? c.nloc_cells : c.ncells;
  if (c1 > c0)
    FMM_LAUNCH(c, k_leaf_local, (unsigned)std::min<int64_t>((c1 - c0 + 7) / 8, 148 * 32), 256, 0, c.cells.leaf.p,
               multi ? c.cflag.p : nullptr, pc, c0, c1, c.lo[0], c.lo[1], c.lo[2], c.L, c.pos.p, c.posl.p, c.alp.p);
  const int* sb = part == 2 ? c.p2p_m.p : c.p2p_b.p;
  const int* se = part == 1 ? c.p2p_m.p : c.p2p_e.p;
  // leaves by size class (once per set_particles): small leaves take the source-split variants
  if (!c.leaf_cls_valid) {
    // stable (Morton order kept within a class: neighbouring blocks then share their
    // source leaves in L2; an atomic scatter scrambled it: +0.9 ms at C3)
    c.leaf_cls.reserve(std::max<int64_t>(c.nleaves, 1));
    c.dflag.reserve(8);
    int off = 0;
    for (int cl = 0; cl < 3; ++cl) {
      LeafClass pred{c.cells.count.p, cl};
      const int* in = c.leaf_ids.p;
      int* out = c.leaf_cls.p + off;
      int* ns = c.dflag.p;
      const int nn = (int)c.nleaves;
      size_t bytes = 0;
      FMM_CUDA(cub::DeviceSelect::If(nullptr, bytes, in, out, ns, nn, pred, c.stream));
      c.cub_tmp.reserve(bytes);
      FMM_CUDA(cub::DeviceSelect::If((void*)c.cub_tmp.p, bytes, in, out, ns, nn, pred, c.stream));
      ++c.cub_calls;
      int h = 0;
      FMM_CUDA(cudaMemcpyAsync(&h, c.dflag.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
      FMM_CUDA(cudaStreamSynchronize(c.stream));
      c.leaf_cls_n[cl] = h;
      off += h;
    }
    c.leaf_cls_valid = true;
  }
  const int* ids[3] = {c.leaf_cls.p, c.leaf_cls.p + c.leaf_cls_n[0], c.leaf_cls.p + c.leaf_cls_n[0] + c.leaf_cls_n[1]};
#define P2P_ARGS sb, se, c.p2p.p, pc, c.lo[0], c.lo[1], c.lo[2], c.L, c.per[0], c.per[1], c.per[2], c.posl.p, c.alp.p, \
                 u_near, s_near, c.dnear.p
  if (part == 2) {
    if (c.leaf_cls_n[0]) FMM_LAUNCH(c, (k_p2p<P2P_MINB, P2P_UF, P2P_UN, true, 1>), (unsigned)c.leaf_cls_n[0], NT, 0, ids[0], P2P_ARGS);
    if (c.leaf_cls_n[1]) FMM_LAUNCH(c, (k_p2p<P2P_MINB, P2P_UF, P2P_UN, true, 2>), (unsigned)c.leaf_cls_n[1], NT, 0, ids[1], P2P_ARGS);
    if (c.leaf_cls_n[2]) FMM_LAUNCH(c, (k_p2p<P2P_MINB, P2P_UF, P2P_UN, true, 4>), (unsigned)c.leaf_cls_n[2], NT, 0, ids[2], P2P_ARGS);
  } else {
    if (c.leaf_cls_n[0]) FMM_LAUNCH(c, (k_p2p<P2P_MINB, P2P_UF, P2P_UN, false, 1>), (unsigned)c.leaf_cls_n[0], NT, 0, ids[0], P2P_ARGS);
    if (c.leaf_cls_n[1]) FMM_LAUNCH(c, (k_p2p<P2P_MINB, P2P_UF, P2P_UN, false, 2>), (unsigned)c.leaf_cls_n[1], NT, 0, ids[1], P2P_ARGS);
    if (c.leaf_cls_n[2]) FMM_LAUNCH(c, (k_p2p<P2P_MINB, P2P_UF, P2P_UN, false, 4>), (unsigned)c.leaf_cls_n[2], NT, 0, ids[2], P2P_ARGS);
  }
#undef P2P_ARGS
}

void eval_cutoff(Ctx& c, const float* rho, int64_t n, float* g) {
  FMM_LAUNCH(c, k_eval_cutoff, nblocks(n, 256), 256, 0, rho, n, g);
}

}  // namespace fmmb
