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
// complex multiply-adds per component as straight FFMA chains with all
// indices, conjugations and signs resolved at compile time.  The ten
// subsets' partial locals are reduced in a fixed order at the end
// (deterministic), so no float atomics are used.
#include <type_traits>

#include "ctx.cuh"

namespace fmmb {

namespace {

constexpr int kSub = 10;   // source subsets (x 3 components = 30 lanes)

struct MCells {
  const int *level, *qx, *qy, *qz;
};

__host__ __device__ constexpr int ci(int n, int m) { return n * (n + 1) / 2 + m; }

template <int P>
struct Dims {
  static constexpr int NC = P * (P + 1) / 2;
  static constexpr int P2 = P;                    // M2L needs I_j for j = n + k <= p - 1 only
  static constexpr int NC2 = P2 * (P2 + 1) / 2;
  static constexpr int S = (NC2 & 1) ? NC2 : NC2 + 1;   // odd stride (float2) => conflict-free subsets
};

// acc += A * B (complex), every sign a compile-time constant
__device__ __forceinline__ void cmac(float& xr, float& xi, float ar, float ai, float br, float bi) {
  xr = fmaf(ar, br, xr);
  xr = fmaf(-ai, bi, xr);
  xi = fmaf(ar, bi, xi);
  xi = fmaf(ai, br, xi);
}

// compile-time loop: f(integral_constant<int, i>) for i = B, B+S, ... (excluding E)
template <int B, int E, int S, typename F>
__device__ __forceinline__ void sfor(F&& f) {
  if constexpr ((S > 0 && B < E) || (S < 0 && B > E)) {
    f(std::integral_constant<int, B>{});
    sfor<B + S, E, S>(f);
  }
}

template <int P>
__device__ __forceinline__ void m2l_accumulate(const float2* __restrict__ Is, const float (&Mr)[Dims<P>::NC],
                                               const float (&Mi)[Dims<P>::NC], float (&Lr)[Dims<P>::NC],
                                               float (&Li)[Dims<P>::NC]) {
  sfor<P - 1, -1, -1>([&](auto J) {                // I degree j = n + k, high -> low
    constexpr int j = decltype(J)::value;
    sfor<j, -1, -1>([&](auto MPc) {
      constexpr int mp = decltype(MPc)::value;
      const float2 iv = Is[ci(j, mp)];
      const float ir = iv.x, ii = iv.y;
      constexpr float ts = (mp & 1) ? -1.f : 1.f;  // I_j^{-mp} = ts conj(I_j^mp)
      sfor<0, j + 1, 1>([&](auto Nc) {
        constexpr int n = decltype(Nc)::value;
        constexpr int k = j - n;
        sfor<0, k + 1, 1>([&](auto Lc_) {
          constexpr int l = decltype(Lc_)::value;
          constexpr int o = ci(k, l);
          constexpr int m1 = mp - l;               // term with I_j^{+mp}
          if constexpr (m1 >= -n && m1 <= n) {
            if constexpr (m1 >= 0) {
              cmac(Lr[o], Li[o], Mr[ci(n, m1)], Mi[ci(n, m1)], ir, ii);
            } else {
              constexpr float s = ((-m1) & 1) ? -1.f : 1.f;   // M_n^m = s conj(M_n^{-m})
              cmac(Lr[o], Li[o], s * Mr[ci(n, -m1)], -s * Mi[ci(n, -m1)], ir, ii);
            }
          }
          constexpr int m2 = -mp - l;              // term with I_j^{-mp}
          if constexpr (mp > 0 && m2 >= -n) {
            constexpr float s = ((-m2) & 1) ? -1.f : 1.f;
            cmac(Lr[o], Li[o], s * Mr[ci(n, -m2)], -s * Mi[ci(n, -m2)], ts * ir, -ts * ii);
          }
        });
      });
    });
  });
}

template <int P>
__global__ void __launch_bounds__(32) k_m2l_reg(const int* __restrict__ seg_b, const int* __restrict__ seg_e,
                                                const uint64_t* __restrict__ lst, MCells c,
                                                const float2* __restrict__ M, float2* __restrict__ Lc) {
  using D = Dims<P>;
  constexpr int NC = D::NC, P2 = D::P2, S = D::S;
  extern __shared__ float2 sm[];                   // [kSub][S] harmonics, later the reduction buffer
  __shared__ float4 Dsh[kSub];
  const int t = blockIdx.x;
  const int b = seg_b[t], e = seg_e[t];
  if (b == e) return;
  const int lane = threadIdx.x;
  const int sub = lane / 3, comp = lane - 3 * (lane / 3);
  const bool act = sub < kSub;
  const int lt = c.level[t];
  const long long ctx = (long long)(2 * c.qx[t] + 1) << (kMaxLevel - lt);
  const long long cty = (long long)(2 * c.qy[t] + 1) << (kMaxLevel - lt);
  const long long ctz = (long long)(2 * c.qz[t] + 1) << (kMaxLevel - lt);
  const float inv_st = ldexpf(1.0f, -(kMaxLevel + 1 - lt));

  float Lr[NC], Li[NC];
#pragma unroll
  for (int o = 0; o < NC; ++o) { Lr[o] = 0.f; Li[o] = 0.f; }

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
        const long long dx = ctx - ((long long)(2 * c.qx[src] + 1) << (kMaxLevel - ls)) - (long long)ix * (1ll << (kMaxLevel + 1));
        const long long dy = cty - ((long long)(2 * c.qy[src] + 1) << (kMaxLevel - ls)) - (long long)iy * (1ll << (kMaxLevel + 1));
        const long long dz = ctz - ((long long)(2 * c.qz[src] + 1) << (kMaxLevel - ls)) - (long long)iz * (1ll << (kMaxLevel + 1));
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
      irregular_column<float>(dv.x, dv.y, dv.z, m, P2, (cpx<float>*)(sm + s * S));
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
    m2l_accumulate<P>(sm + (act ? sub : 0) * S, Mr, Mi, Lr, Li);
    __syncwarp();
  }

  // deterministic reduction over the source subsets
  float2* red = sm;                                // [kSub][3][NC]
  if (act) {
#pragma unroll
    for (int o = 0; o < NC; ++o) red[(sub * 3 + comp) * NC + o] = make_float2(Lr[o], Li[o]);
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
  size_t sm = sizeof(float2) * (size_t)kSub * D::S;
  size_t red = sizeof(float2) * (size_t)kSub * 3 * D::NC;
  if (red > sm) sm = red;
  MCells mc{c.cells.level.p, c.cells.qx.p, c.cells.qy.p, c.cells.qz.p};
  FMM_LAUNCH(c, k_m2l_reg<P>, (unsigned)c.ncells, 32, sm, c.m2l_b.p, c.m2l_e.p, c.m2l.p, mc, c.M.p, c.Lc.p);
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
