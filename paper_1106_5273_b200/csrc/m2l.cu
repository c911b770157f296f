// m2l.cu -- a9: batched M2L (the far-field hot loop) for orders
// p <= 10, register-blocked for sm_100a.
//
//   L~_k^l(t) += (-1)^k sum_{n<p-k} sum_{|m|<=n} M~_n^m(s) (s_s/s_t)^n I_{n+k}^{m+l}(D/s_t)
//
// The paper maps one expansion coefficient to a thread and one target cell to
// a thread block (fig:m2l_gpu); with O(p^4) work concentrated in the
// low-degree coefficients that mapping leaves most threads idle.  Here one
// warp owns one target cell and the 30 active lanes are (source subset s,
// component c): lane (s, c) walks sources s, s+10, s+20, ... of the target's
// M2L segment and keeps *all* p(p+1)/2 local coefficients of component c in
// registers (Lr/Li) together with the source's multipole component (Mr/Mi).
// Per source the 55 irregular harmonics I_j^m(D/s_t), j <= p-1, are built once,
// column-parallel across the warp, into shared memory; the fully unrolled
// accumulation then reads each I_j^m exactly once and issues the 1210
// complex multiply-adds per component as packed FP32x2 FMAs (FFMA2, two per
// complex MAC, the scalar M parts broadcast) with all indices, conjugations
// and signs resolved at compile time.  The ten
// subsets' partial locals are reduced in a fixed order at the end
// (deterministic), so no float atomics are used.
#include <type_traits>

#include "ctx.cuh"

namespace fmmb {

namespace {

constexpr int kSub = 10;   // source subsets (x 3 components = 30 lanes)

struct MCells {
  const int *level, *qx, *qy, *qz;
  long long per[3];           // image shifts (half-finest-cell units)
};


template <int P>
struct Dims {
  static constexpr int NC = P * (P + 1) / 2;
  static constexpr int P2 = P;                    // M2L needs I_j for j = n + k <= p - 1 only
  static constexpr int NC2 = P2 * (P2 + 1) / 2;
  // per source: 2 float4 per (j, m) = {I, (-Im, Re)} and {I^{-m}, (-Im, Re) of I^{-m}}; the
  // stride (float4 units) is 7 mod 8 so the ten subsets spread over the 8 bank groups
  static constexpr int S = 2 * NC2 + ((7 - (2 * NC2) % 8) + 8) % 8;
};

// Is holds, per (j, mp): Is[2 ci] = (Re I, Im I, -Im I, Re I) of I_j^mp and
// Is[2 ci + 1] the same for I_j^{-mp} = (-1)^mp conj(I_j^mp).  For a complex
// M = (ar, ai):  M * I = ar (Re I, Im I) + ai (-Im I, Re I).
template <int P>
__device__ __forceinline__ void m2l_accumulate(const float4* __restrict__ Is, const float (&Mr)[Dims<P>::NC],
                                               const float (&Mi)[Dims<P>::NC], float2 (&L)[Dims<P>::NC]) {
  sfor<P - 1, -1, -1>([&](auto J) {                // I degree j = n + k, high -> low
    constexpr int j = decltype(J)::value;
    sfor<j, -1, -1>([&](auto MPc) {
      constexpr int mp = decltype(MPc)::value;
      const float4 ip = Is[2 * ci(j, mp)];
      const float2 Bp = make_float2(ip.x, ip.y), Bq = make_float2(ip.z, ip.w);
      float2 Cp = Bp, Cq = Bq;
      if constexpr (mp > 0) {
        const float4 in = Is[2 * ci(j, mp) + 1];
        Cp = make_float2(in.x, in.y);
        Cq = make_float2(in.z, in.w);
      }
      // four passes over the (n, l) targets of this I_j^{mp}: each pass issues
      // one FFMA2 per local coefficient, so consecutive FFMA2s are independent
      // (a single pass would chain four dependent FFMA2s on the same L[o])
      sfor<0, 4, 1>([&](auto PSc) {
        constexpr int ps = decltype(PSc)::value;
        sfor<0, j + 1, 1>([&](auto Nc) {
          constexpr int n = decltype(Nc)::value;
          constexpr int k = j - n;
          sfor<0, k + 1, 1>([&](auto Lc_) {
            constexpr int l = decltype(Lc_)::value;
            constexpr int o = ci(k, l);
            if constexpr (ps < 2) {
              constexpr int m1 = mp - l;             // term with I_j^{+mp}
              if constexpr (m1 >= -n && m1 <= n) {
                constexpr int ma = m1 >= 0 ? m1 : -m1;
                constexpr float s = (m1 < 0 && (ma & 1)) ? -1.f : 1.f;   // M_n^m = (-1)^m conj(M_n^{-m})
                constexpr float si = m1 < 0 ? -s : s;
                if constexpr (ps == 0) L[o] = __ffma2_rn(make_float2(s * Mr[ci(n, ma)], s * Mr[ci(n, ma)]), Bp, L[o]);
                else L[o] = __ffma2_rn(make_float2(si * Mi[ci(n, ma)], si * Mi[ci(n, ma)]), Bq, L[o]);
              }
            } else {
              constexpr int m2 = -mp - l;            // term with I_j^{-mp}
              if constexpr (mp > 0 && m2 >= -n) {
                constexpr int ma = -m2;
                constexpr float s = (ma & 1) ? -1.f : 1.f;
                if constexpr (ps == 2) L[o] = __ffma2_rn(make_float2(s * Mr[ci(n, ma)], s * Mr[ci(n, ma)]), Cp, L[o]);
                else L[o] = __ffma2_rn(make_float2(-s * Mi[ci(n, ma)], -s * Mi[ci(n, ma)]), Cq, L[o]);
              }
            }
          });
        });
      });
    });
  });
}

// column m of I_j^m(D), j = m .. P-1, written in the expanded layout above
template <int P>
__device__ void irregular_column_x(float x, float y, float z, int m, float4* __restrict__ Is) {
  const float r2 = x * x + y * y + z * z;
  const float ir2 = 1.0f / r2;
  float dr = rsqrtf(r2), di = 0.f;
  for (int i = 1; i <= m; ++i) {
    const float s = -(float)(2 * i - 1) * ir2;
    const float nr = s * (x * dr - y * di), ni = s * (x * di + y * dr);
    dr = nr;
    di = ni;
  }
  const float ts = (m & 1) ? -1.f : 1.f;
  auto put = [&](int n, float vr, float vi) {
    Is[2 * ci(n, m)] = make_float4(vr, vi, -vi, vr);
    Is[2 * ci(n, m) + 1] = make_float4(ts * vr, -ts * vi, ts * vi, ts * vr);
  };
  put(m, dr, di);
  if (m + 1 >= P) return;
  float ar = (float)(2 * m + 1) * z * ir2 * dr, ai = (float)(2 * m + 1) * z * ir2 * di;
  put(m + 1, ar, ai);
  float br = dr, bi = di;
  for (int n = m + 2; n < P; ++n) {
    const float c1 = (float)(2 * n - 1) * z, c2 = (float)(n - 1 - m) * (float)(n - 1 + m);
    const float vr = (c1 * ar - c2 * br) * ir2, vi = (c1 * ai - c2 * bi) * ir2;
    put(n, vr, vi);
    br = ar; bi = ai;
    ar = vr; ai = vi;
  }
}

template <int P>
__global__ void __launch_bounds__(32) k_m2l_reg(const int* __restrict__ seg_b, const int* __restrict__ seg_e,
                                                const uint64_t* __restrict__ lst, MCells c,
                                                const float2* __restrict__ M, float2* __restrict__ Lc,
                                                const unsigned char* __restrict__ skip) {
  using D = Dims<P>;
  constexpr int NC = D::NC, P2 = D::P2, S = D::S;
  extern __shared__ float4 sm4[];                  // [kSub][S] harmonics, later the reduction buffer
  __shared__ float4 Dsh[kSub];
  const int t = blockIdx.x;
  const int b = seg_b[t], e = seg_e[t];
  if (b == e) return;                              // no entry left for the register kernel
  (void)skip;                                      // (the segments hold only register-path entries)
  const int lane = threadIdx.x;
  const int sub = lane / 3, comp = lane - 3 * (lane / 3);
  const bool act = sub < kSub;
  const int lt = c.level[t];
  const long long ctx = (long long)(2 * c.qx[t] + 1) << (kMaxLevel - lt);
  const long long cty = (long long)(2 * c.qy[t] + 1) << (kMaxLevel - lt);
  const long long ctz = (long long)(2 * c.qz[t] + 1) << (kMaxLevel - lt);
  const float inv_st = ldexpf(1.0f, -(kMaxLevel + 1 - lt));

  float2 L[NC];
#pragma unroll
  for (int o = 0; o < NC; ++o) L[o] = make_float2(0.f, 0.f);

#pragma unroll 1
  for (int q0 = b; q0 < e; q0 += kSub) {
    // D / s_t of the round's sources (exact: integer centres, power-of-2 scale)
    if (lane < kSub) {
      const int q = q0 + lane;
      float4 dv = make_float4(1.f, 1.f, 1.f, 0.f);
      if (q < e) {
        const uint64_t ent = lst[q];
        const int src = (int)((ent >> 5) & 0x7ffffff), img = (int)(ent & 31);
        const int ls = c.level[src];
        const int ix = img % 3 - 1, iy = (img / 3) % 3 - 1, iz = img / 9 - 1;
        const long long dx = ctx - ((long long)(2 * c.qx[src] + 1) << (kMaxLevel - ls)) - (long long)ix * c.per[0];
        const long long dy = cty - ((long long)(2 * c.qy[src] + 1) << (kMaxLevel - ls)) - (long long)iy * c.per[1];
        const long long dz = ctz - ((long long)(2 * c.qz[src] + 1) << (kMaxLevel - ls)) - (long long)iz * c.per[2];
        dv = make_float4((float)dx * inv_st, (float)dy * inv_st, (float)dz * inv_st, 1.f);
      }
      Dsh[lane] = dv;
    }
    __syncwarp();
    // irregular harmonics, one column (source s, order m) per task
#pragma unroll 1
    for (int task = lane; task < kSub * P2; task += 32) {
      const int s = task / P2, m = task - P2 * (task / P2);
      const float4 dv = Dsh[s];
      irregular_column_x<P>(dv.x, dv.y, dv.z, m, sm4 + s * S);
    }
    // this lane's source multipole component, scaled by (s_s/s_t)^n
    float Mr[NC], Mi[NC];
    {
      const int q = q0 + sub;
      const bool valid = act && q < e;
      int src = 0;
      float ratio = 0.f;
      if (valid) {
        src = (int)((lst[q] >> 5) & 0x7ffffff);
        ratio = ldexpf(1.0f, lt - c.level[src]);
      }
      const float2* Ms = M + ((int64_t)src * 3 + comp) * NC;
      float pw = valid ? 1.f : 0.f;
#pragma unroll
      for (int n = 0; n < P; ++n) {
#pragma unroll
        for (int m = 0; m <= n; ++m) {
          const float2 v = valid ? __ldg(Ms + ci(n, m)) : make_float2(0.f, 0.f);
          Mr[ci(n, m)] = v.x * pw;
          Mi[ci(n, m)] = v.y * pw;
        }
        pw *= ratio;
      }
    }
    __syncwarp();
    m2l_accumulate<P>(sm4 + (act ? sub : 0) * S, Mr, Mi, L);
    __syncwarp();
  }

  // deterministic reduction over the source subsets
  float2* red = (float2*)sm4;                      // [kSub][3][NC]
  if (act) {
#pragma unroll
    for (int o = 0; o < NC; ++o) red[(sub * 3 + comp) * NC + o] = L[o];
  }
  __syncwarp();
  for (int i = lane; i < 3 * NC; i += 32) {
    const int cc = i / NC, o = i - NC * (i / NC);
    int k = 0;
    while ((k + 1) * (k + 2) / 2 <= o) ++k;
    float sr = 0.f, si = 0.f;
    for (int s = 0; s < kSub; ++s) {
      const float2 v = red[(s * 3 + cc) * NC + o];
      sr += v.x;
      si += v.y;
    }
    const float sg = (k & 1) ? -1.f : 1.f;
    float2* d = Lc + (int64_t)t * 3 * NC + i;
    const float2 old = *d;
    *d = make_float2(old.x + sg * sr, old.y + sg * si);
  }
}

template <int P>
void launch_reg(Ctx& c) {
  using D = Dims<P>;
  size_t sm = sizeof(float4) * (size_t)kSub * D::S;
  size_t red = sizeof(float2) * (size_t)kSub * 3 * D::NC;
  if (red > sm) sm = red;
  MCells mc{c.cells.level.p, c.cells.qx.p, c.cells.qy.p, c.cells.qz.p, {c.per_units[0], c.per_units[1], c.per_units[2]}};
  FMM_LAUNCH(c, k_m2l_reg<P>, (unsigned)c.ncells, 32, sm, c.m2l_b.p, c.m2l_e.p, c.m2lr.p, mc, c.M.p, c.Lc.p,
             c.tc_skip.p);
}

}  // namespace

// returns false if no register-blocked instantiation exists for this order
bool m2l_pass_reg(Ctx& c) {
  switch (c.P) {
    case 4: launch_reg<4>(c); return true;
    case 6: launch_reg<6>(c); return true;
    case 8: launch_reg<8>(c); return true;
    case 10: launch_reg<10>(c); return true;
    default: return false;
  }
}

}  // namespace fmmb
