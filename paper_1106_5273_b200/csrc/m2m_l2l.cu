// m2m_l2l.cu -- a6 M2M and a10 L2L for p <= 10, register-blocked.
//
//   M2M:  M~_n^m(parent) += sum_{k <= n} sum_l  M~_{n-k}^{m-l}(child) 2^{-(n-k)} conj(R_k^l(d))
//   L2L:  L~_a^b(child)  += 2^{-(a+1)} sum_{k >= a} sum_l  L~_k^l(parent) conj(R_{k-a}^{l-b}(d))
//
// d = child centre - parent centre in parent-side units, one of the 8 octant
// vectors (+-1/4, +-1/4, +-1/4), so R_k^l(d) comes from the per-context table of
// the octants (expansions.cu) staged once per block in shared memory.  A warp
// owns one parent; lane (q, c) = (child q, vorticity component c), 24 lanes.  The
// lane keeps its input expansion (55 complex at p = 10) and its 55 output
// coefficients in registers; the loops over (n, m, k, l) are unrolled at compile
// time with the R_k^l of the lane's octant read once each from shared memory
// (expanded float4 layout: every complex multiply-add is two FFMA2).  M2M sums
// the eight children's shifted expansions in a fixed order through shared memory
// (deterministic); L2L adds each child's result into its local expansion.
// The generic runtime-p kernels in expansions.cu serve other orders.
#include "ctx.cuh"

namespace fmmb {

namespace {

struct TCells {
  const int *qx, *qy, *qz, *leaf, *child_begin, *nchild;
};

__device__ __forceinline__ int octant_of(const TCells& c, int ch, int p) {
  return (c.qx[ch] - 2 * c.qx[p]) | ((c.qy[ch] - 2 * c.qy[p]) << 1) | ((c.qz[ch] - 2 * c.qz[p]) << 2);
}

// Rs[o][2 ci(k, l)]     = (c, -d, d, c)  for R_k^l = c + i d        (l >= 0)
// Rs[o][2 ci(k, l) + 1] = the same for R_k^{-l} = (-1)^l conj(R_k^l)
// so that for X = a + i b:  X conj(R) = a (c, -d) + b (d, c).
template <int P>
__device__ void stage_octants(const float2* __restrict__ R8, float4* __restrict__ Rs) {
  constexpr int NC = P * (P + 1) / 2;
  for (int i = threadIdx.x; i < 8 * NC; i += blockDim.x) {
    const int o = i / NC, k = i - NC * (i / NC);
    int n = 0;
    while ((n + 1) * (n + 2) / 2 <= k) ++n;
    const int l = k - n * (n + 1) / 2;
    const float2 r = R8[i];
    const float t = (l & 1) ? -1.f : 1.f;
    Rs[(o * NC + k) * 2] = make_float4(r.x, -r.y, r.y, r.x);
    Rs[(o * NC + k) * 2 + 1] = make_float4(t * r.x, t * r.y, -t * r.y, t * r.x);
  }
}

__device__ __forceinline__ void cmac_conj(float2& acc, float a, float b, const float4 r) {
  acc = __ffma2_rn(make_float2(a, a), make_float2(r.x, r.y), acc);
  acc = __ffma2_rn(make_float2(b, b), make_float2(r.z, r.w), acc);
}

template <int P>
__global__ void __launch_bounds__(32) k_m2m_reg(int64_t first, TCells c, const float2* __restrict__ R8,
                                                float2* __restrict__ M) {
  constexpr int NC = P * (P + 1) / 2;
  __shared__ float4 Rs[8 * NC * 2];
  __shared__ float2 red[3][8][NC];
  const int p = (int)(first + blockIdx.x);
  if (c.leaf[p]) return;
  stage_octants<P>(R8, Rs);
  const int lane = threadIdx.x, q = lane / 3, comp = lane - 3 * (lane / 3);
  const int cb = c.child_begin[p], nch = c.nchild[p];
  const bool act = lane < 24 && q < nch;
  const int oct = act ? octant_of(c, cb + q, p) : 0;
  // the child's multipole component, scaled by 2^{-n}
  float Mr[NC], Mi[NC];
  {
    const float2* src = M + ((int64_t)(cb + (act ? q : 0)) * 3 + comp) * NC;
    sfor<0, P, 1>([&](auto Nc) {
      constexpr int n = decltype(Nc)::value;
      constexpr float sc = 1.0f / (float)(1 << n);
      sfor<0, n + 1, 1>([&](auto Mc) {
        constexpr int m = decltype(Mc)::value;
        const float2 v = act ? src[ci(n, m)] : make_float2(0.f, 0.f);
        Mr[ci(n, m)] = sc * v.x;
        Mi[ci(n, m)] = sc * v.y;
      });
    });
  }
  float2 acc[NC];
#pragma unroll
  for (int o = 0; o < NC; ++o) acc[o] = make_float2(0.f, 0.f);
  __syncwarp();
  const float4* R = Rs + oct * NC * 2;
  // (k, l) outer: each R_k^l read once, applied to every output it reaches
  sfor<0, P, 1>([&](auto Kc) {
    constexpr int k = decltype(Kc)::value;
    sfor<-k, k + 1, 1>([&](auto Lc_) {
      constexpr int l = decltype(Lc_)::value;
      const float4 r = R[2 * ci(k, l >= 0 ? l : -l) + (l >= 0 ? 0 : 1)];
      sfor<k, P, 1>([&](auto Nc) {
        constexpr int n = decltype(Nc)::value;
        constexpr int nn = n - k;
        sfor<0, n + 1, 1>([&](auto Mc) {
          constexpr int m = decltype(Mc)::value;
          constexpr int mm = m - l;
          if constexpr (mm >= -nn && mm <= nn) {
            if constexpr (mm >= 0) {
              cmac_conj(acc[ci(n, m)], Mr[ci(nn, mm)], Mi[ci(nn, mm)], r);
            } else {
              constexpr float t = ((-mm) & 1) ? -1.f : 1.f;   // M_n^{-m} = (-1)^m conj(M_n^m)
              cmac_conj(acc[ci(n, m)], t * Mr[ci(nn, -mm)], -t * Mi[ci(nn, -mm)], r);
            }
          }
        });
      });
    });
  });
  if (act)
#pragma unroll
    for (int o = 0; o < NC; ++o) red[comp][q][o] = acc[o];
  __syncwarp();
  for (int i = lane; i < 3 * NC; i += 32) {
    const int cc = i / NC, o = i - NC * (i / NC);
    float2 s = make_float2(0.f, 0.f);
    for (int qq = 0; qq < nch; ++qq) {
      const float2 v = red[cc][qq][o];
      s.x += v.x;
      s.y += v.y;
    }
    M[((int64_t)p * 3 + cc) * NC + o] = s;
  }
}

template <int P>
__global__ void __launch_bounds__(32) k_l2l_reg(int64_t pfirst, int64_t clo, int64_t chi, TCells c,
                                                const float2* __restrict__ R8, float2* __restrict__ Lc) {
  constexpr int NC = P * (P + 1) / 2;
  __shared__ float4 Rs[8 * NC * 2];
  const int p = (int)(pfirst + blockIdx.x);
  if (c.leaf[p]) return;
  const int lane = threadIdx.x, q = lane / 3, comp = lane - 3 * (lane / 3);
  const int cb = c.child_begin[p], nch = c.nchild[p];
  const int ch = cb + q;
  const bool act = lane < 24 && q < nch && ch >= clo && ch < chi;   // this rank's children
  if (!__any_sync(0xffffffffu, act)) return;
  stage_octants<P>(R8, Rs);
  const int oct = act ? octant_of(c, ch, p) : 0;
  // the parent's local component
  float Lr[NC], Li[NC];
  {
    const float2* src = Lc + ((int64_t)p * 3 + comp) * NC;
#pragma unroll
    for (int o = 0; o < NC; ++o) {
      const float2 v = src[o];
      Lr[o] = v.x;
      Li[o] = v.y;
    }
  }
  float2 acc[NC];
#pragma unroll
  for (int o = 0; o < NC; ++o) acc[o] = make_float2(0.f, 0.f);
  __syncwarp();
  const float4* R = Rs + oct * NC * 2;
  // R_{kr}^{lr} outer (kr = k - a, lr = l - b), each read once
  sfor<0, P, 1>([&](auto KRc) {
    constexpr int kr = decltype(KRc)::value;
    sfor<-kr, kr + 1, 1>([&](auto LRc) {
      constexpr int lr = decltype(LRc)::value;
      const float4 r = R[2 * ci(kr, lr >= 0 ? lr : -lr) + (lr >= 0 ? 0 : 1)];
      sfor<0, P - kr, 1>([&](auto Ac) {
        constexpr int a = decltype(Ac)::value;
        constexpr int k = a + kr;
        sfor<0, a + 1, 1>([&](auto Bc) {
          constexpr int b = decltype(Bc)::value;
          constexpr int l = lr + b;
          if constexpr (l >= -k && l <= k) {
            if constexpr (l >= 0) {
              cmac_conj(acc[ci(a, b)], Lr[ci(k, l)], Li[ci(k, l)], r);
            } else {
              constexpr float t = ((-l) & 1) ? -1.f : 1.f;      // L_k^{-l} = (-1)^l conj(L_k^l)
              cmac_conj(acc[ci(a, b)], t * Lr[ci(k, -l)], -t * Li[ci(k, -l)], r);
            }
          }
        });
      });
    });
  });
  if (act) {
    float2* d = Lc + ((int64_t)ch * 3 + comp) * NC;
    sfor<0, P, 1>([&](auto Ac) {
      constexpr int a = decltype(Ac)::value;
      constexpr float sc = 1.0f / (float)(2 << a);               // 2^{-(a+1)}
      sfor<0, a + 1, 1>([&](auto Bc) {
        constexpr int b = decltype(Bc)::value;
        float2 v = d[ci(a, b)];
        v.x += sc * acc[ci(a, b)].x;
        v.y += sc * acc[ci(a, b)].y;
        d[ci(a, b)] = v;
      });
    });
  }
}

TCells tcells(Ctx& c) {
  return {c.cells.qx.p, c.cells.qy.p, c.cells.qz.p, c.cells.leaf.p, c.cells.child_begin.p, c.cells.nchild.p};
}

template <int P>
void m2m_launch(Ctx& c, int64_t first, int64_t cnt, const float2* R8) {
  FMM_LAUNCH(c, k_m2m_reg<P>, (unsigned)cnt, 32, 0, first, tcells(c), R8, c.M.p);
}
template <int P>
void l2l_launch(Ctx& c, int64_t pfirst, int64_t pcnt, int64_t clo, int64_t chi, const float2* R8) {
  FMM_LAUNCH(c, k_l2l_reg<P>, (unsigned)pcnt, 32, 0, pfirst, clo, chi, tcells(c), R8, c.Lc.p);
}

}  // namespace

// M2M of the parents [first, first + cnt) (all their children are local); false: no instantiation for this p
bool m2m_level_reg(Ctx& c, int64_t first, int64_t cnt, const float2* R8) {
  if (cnt <= 0) return true;
  switch (c.P) {
    case 4: m2m_launch<4>(c, first, cnt, R8); return true;
    case 6: m2m_launch<6>(c, first, cnt, R8); return true;
    case 8: m2m_launch<8>(c, first, cnt, R8); return true;
    case 10: m2m_launch<10>(c, first, cnt, R8); return true;
    default: return false;
  }
}

// L2L into the children [clo, chi) of one level, parents [pfirst, pfirst + pcnt)
bool l2l_level_reg(Ctx& c, int64_t pfirst, int64_t pcnt, int64_t clo, int64_t chi, const float2* R8) {
  if (pcnt <= 0) return true;
  switch (c.P) {
    case 4: l2l_launch<4>(c, pfirst, pcnt, clo, chi, R8); return true;
    case 6: l2l_launch<6>(c, pfirst, pcnt, clo, chi, R8); return true;
    case 8: l2l_launch<8>(c, pfirst, pcnt, clo, chi, R8); return true;
    case 10: l2l_launch<10>(c, pfirst, pcnt, clo, chi, R8); return true;
    default: return false;
  }
}

}  // namespace fmmb
