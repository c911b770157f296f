// l2p.cu -- a11: L2P for orders p <= 10, compile-time unrolled (the generic
// runtime-p kernel in expansions.cu serves the other orders).
//
// For a particle at y = (x - c)/s in a leaf of side s, shift the normalised
// local L~ to the particle keeping degrees 1 and 2:
//   L'_a^b = s^{-a-1} sum_{k>=a} sum_l L~_k^l conj(R_{k-a}^{l-b}(y)),
// then grad phi = (-Re L'_1^1, -Im L'_1^1, Re L'_1^0) and the Hessian from
// L'_2^{0,1,2};  u = (1/4pi) eps_abc d_b phi_c, s = (1/4pi) alpha_d eps_abc H^c_db.
// One thread per particle keeps its 55 regular harmonics in registers; the
// leaf's local expansion sits in shared memory in an expanded layout so each
// complex multiply-add is two FFMA2 with the harmonic parts broadcast:
//   L conj(R) = Re R (Re L, Im L) + Im R (Im L, -Re L).
#include "ctx.cuh"

namespace fmmb {

namespace {

struct LCells {
  const int *level, *qx, *qy, *qz, *begin, *count;
};

template <int P>
__device__ __forceinline__ void regular_unrolled(float x, float y, float z, float (&Rr)[P * (P + 1) / 2],
                                                 float (&Ri)[P * (P + 1) / 2]) {
  const float r2 = x * x + y * y + z * z;
  Rr[0] = 1.f;
  Ri[0] = 0.f;
  sfor<1, P, 1>([&](auto Mc) {
    constexpr int m = decltype(Mc)::value;
    constexpr float s = -1.0f / (2 * m);
    const float pr = Rr[ci(m - 1, m - 1)], pi = Ri[ci(m - 1, m - 1)];
    Rr[ci(m, m)] = s * (x * pr - y * pi);
    Ri[ci(m, m)] = s * (x * pi + y * pr);
  });
  sfor<0, P - 1, 1>([&](auto Mc) {
    constexpr int m = decltype(Mc)::value;
    Rr[ci(m + 1, m)] = z * Rr[ci(m, m)];
    Ri[ci(m + 1, m)] = z * Ri[ci(m, m)];
  });
  sfor<0, P, 1>([&](auto Mc) {
    constexpr int m = decltype(Mc)::value;
    sfor<m + 2, P, 1>([&](auto Nc) {
      constexpr int n = decltype(Nc)::value;
      constexpr float inv = 1.0f / ((n - m) * (n + m));
      constexpr float c1 = (2 * n - 1) * inv;
      Rr[ci(n, m)] = c1 * z * Rr[ci(n - 1, m)] - inv * r2 * Rr[ci(n - 2, m)];
      Ri[ci(n, m)] = c1 * z * Ri[ci(n - 1, m)] - inv * r2 * Ri[ci(n - 2, m)];
    });
  });
}

// outputs q = 0..4 : (a,b) = (1,0) (1,1) (2,0) (2,1) (2,2)
template <int P>
__device__ __forceinline__ void shift_to_point(const float4* __restrict__ Ls, const float (&Rr)[P * (P + 1) / 2],
                                               const float (&Ri)[P * (P + 1) / 2], float2 (&out)[5]) {
  sfor<0, 5, 1>([&](auto Qc) { out[decltype(Qc)::value] = make_float2(0.f, 0.f); });
  sfor<P - 1, 0, -1>([&](auto Kc) {               // k = p-1 .. 1, high -> low
    constexpr int k = decltype(Kc)::value;
    sfor<0, k + 1, 1>([&](auto Lc_) {
      constexpr int l = decltype(Lc_)::value;
      const float4 lp = Ls[2 * ci(k, l)];          // L_k^l:  (Re, Im, Im, -Re)
      float4 ln = lp;
      if constexpr (l > 0) ln = Ls[2 * ci(k, l) + 1];   // L_k^{-l}
      sfor<0, 5, 1>([&](auto Qc) {
        constexpr int q = decltype(Qc)::value;
        constexpr int a = q < 2 ? 1 : 2;
        constexpr int b = q < 2 ? q : q - 2;
        constexpr int ka = k - a;
        if constexpr (ka >= 0) {
          // term with L_k^{+l}: R index (ka, l - b)
          constexpr int r1 = l - b;
          if constexpr (r1 >= -ka && r1 <= ka) {
            constexpr int ra = r1 >= 0 ? r1 : -r1;
            constexpr float sr = (r1 < 0 && (ra & 1)) ? -1.f : 1.f;   // R_n^{-m} = (-1)^m conj(R_n^m)
            constexpr float si = r1 < 0 ? -sr : sr;
            const float rr = sr * Rr[ci(ka, ra)], ri = si * Ri[ci(ka, ra)];
            out[q] = __ffma2_rn(make_float2(rr, rr), make_float2(lp.x, lp.y), out[q]);
            out[q] = __ffma2_rn(make_float2(ri, ri), make_float2(lp.z, lp.w), out[q]);
          }
          // term with L_k^{-l}: R index (ka, -l - b)
          if constexpr (l > 0) {
            constexpr int r2 = -l - b;
            if constexpr (r2 >= -ka) {
              constexpr int ra = -r2;
              constexpr float sr = (ra & 1) ? -1.f : 1.f;
              constexpr float si = -sr;
              const float rr = sr * Rr[ci(ka, ra)], ri = si * Ri[ci(ka, ra)];
              out[q] = __ffma2_rn(make_float2(rr, rr), make_float2(ln.x, ln.y), out[q]);
              out[q] = __ffma2_rn(make_float2(ri, ri), make_float2(ln.z, ln.w), out[q]);
            }
          }
        }
      });
    });
  });
}

template <int P>
__global__ void __launch_bounds__(64) k_l2p_reg(const int* __restrict__ leaf_ids, LCells c, double lo0, double lo1,
                                                double lo2, double L, const float4* __restrict__ pos,
                                                const float4* __restrict__ alp, const float2* __restrict__ Lc,
                                                float* __restrict__ uf, float* __restrict__ sf) {
  constexpr int NC = P * (P + 1) / 2;
  __shared__ float4 Ls[3][2 * NC];
  const int leaf = leaf_ids[blockIdx.x];
  const int lev = c.level[leaf], b = c.begin[leaf], cnt = c.count[leaf];
  const double s = L / (double)(1 << lev);
  const double cx = lo0 + (c.qx[leaf] + 0.5) * s, cy = lo1 + (c.qy[leaf] + 0.5) * s, cz = lo2 + (c.qz[leaf] + 0.5) * s;
  for (int i = threadIdx.x; i < 3 * NC; i += blockDim.x) {
    const int comp = i / NC, o = i - comp * NC;
    int n = 0;
    while ((n + 1) * (n + 2) / 2 <= o) ++n;
    const int m = o - n * (n + 1) / 2;
    const float2 v = Lc[(int64_t)leaf * 3 * NC + i];
    const float t = (m & 1) ? -1.f : 1.f;            // L^{-m} = (-1)^m conj(L^m)
    Ls[comp][2 * o] = make_float4(v.x, v.y, v.y, -v.x);
    Ls[comp][2 * o + 1] = make_float4(t * v.x, -t * v.y, -t * v.y, -t * v.x);
  }
  __syncthreads();
  const float is2 = (float)(1.0 / (s * s)), is3 = (float)(1.0 / (s * s * s));
  const float k4 = (float)(1.0 / (4.0 * kPi));
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    // keep the local-expansion loads inside the loop (hoisting them would need
    // 6 p(p+1)/2 float4 registers)
    asm volatile("" ::: "memory");
    const float4 p = pos[b + i];
    float Rr[NC], Ri[NC];
    regular_unrolled<P>((float)(((double)p.x - cx) / s), (float)(((double)p.y - cy) / s),
                        (float)(((double)p.z - cz) / s), Rr, Ri);
    float gr[3][3], H[3][6];
    sfor<0, 3, 1>([&](auto Cc) {
      constexpr int comp = decltype(Cc)::value;
      float2 o[5];
      shift_to_point<P>(Ls[comp], Rr, Ri, o);
      gr[comp][0] = -o[1].x * is2;
      gr[comp][1] = -o[1].y * is2;
      gr[comp][2] = o[0].x * is2;
      H[comp][0] = 0.5f * (-o[2].x + o[4].x) * is3;   // xx
      H[comp][1] = 0.5f * (-o[2].x - o[4].x) * is3;   // yy
      H[comp][2] = o[2].x * is3;                      // zz
      H[comp][3] = 0.5f * o[4].y * is3;               // xy
      H[comp][4] = -o[3].x * is3;                     // xz
      H[comp][5] = -o[3].y * is3;                     // yz
    });
    // H^c_{db}: 0 xx, 1 yy, 2 zz, 3 xy, 4 xz, 5 yz
    const float4 ai = alp[b + i];
    const float u0 = gr[2][1] - gr[1][2], u1 = gr[0][2] - gr[2][0], u2 = gr[1][0] - gr[0][1];
    // s_a = alpha_d eps_abc H^c_db
    const float s0 = ai.x * (H[2][3] - H[1][4]) + ai.y * (H[2][1] - H[1][5]) + ai.z * (H[2][5] - H[1][2]);
    const float s1 = ai.x * (H[0][4] - H[2][0]) + ai.y * (H[0][5] - H[2][3]) + ai.z * (H[0][2] - H[2][4]);
    const float s2 = ai.x * (H[1][0] - H[0][3]) + ai.y * (H[1][3] - H[0][1]) + ai.z * (H[1][4] - H[0][5]);
    const int64_t o3 = 3 * (int64_t)(b + i);
    uf[o3] = k4 * u0; uf[o3 + 1] = k4 * u1; uf[o3 + 2] = k4 * u2;
    sf[o3] = k4 * s0; sf[o3 + 1] = k4 * s1; sf[o3 + 2] = k4 * s2;
  }
}

// a5 P2M for p <= 10: M~_n^m(c) = sum_j alpha_j conj(R_n^m((x_j - c)/s)) per
// component.  Thread per particle (64 per pass) with its 55 regular harmonics
// in registers; one component at a time the products go through shared memory
// ([particle][coefficient], stride 57 float2: conflict-free) and 55 threads sum
// a coefficient column each, particles in order.
template <int P>
__global__ void __launch_bounds__(64) k_p2m_reg(const int* __restrict__ leaf_ids, LCells c, double lo0, double lo1,
                                                double lo2, double L, const float4* __restrict__ pos,
                                                const float4* __restrict__ alp, float2* __restrict__ M) {
  constexpr int NC = P * (P + 1) / 2, LD = NC + (NC % 2 == 0 ? 1 : 2);
  static_assert(LD % 2 == 1, "odd row stride in 8-byte words");
  __shared__ float2 S[64][LD];
  const int tid = threadIdx.x;
  const int leaf = leaf_ids[blockIdx.x];
  const int lev = c.level[leaf], b = c.begin[leaf], cnt = c.count[leaf];
  const double s = L / (double)(1 << lev);
  const double cx = lo0 + (c.qx[leaf] + 0.5) * s, cy = lo1 + (c.qy[leaf] + 0.5) * s, cz = lo2 + (c.qz[leaf] + 0.5) * s;
  float2 acc[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  for (int j0 = 0; j0 < cnt; j0 += 64) {
    const int i = j0 + tid;
    const bool v = i < cnt;
    float Rr[NC], Ri[NC];
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    if (v) {
      const float4 p = pos[b + i];
      a = alp[b + i];
      regular_unrolled<P>((float)(((double)p.x - cx) / s), (float)(((double)p.y - cy) / s),
                          (float)(((double)p.z - cz) / s), Rr, Ri);
    } else {
#pragma unroll
      for (int k = 0; k < NC; ++k) Rr[k] = Ri[k] = 0.f;
    }
    const int nr = min(64, cnt - j0);
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) {
      const float ac = comp == 0 ? a.x : (comp == 1 ? a.y : a.z);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < NC; ++k) S[tid][k] = make_float2(ac * Rr[k], -ac * Ri[k]);
      __syncthreads();
      if (tid < NC) {
        float2 w = acc[comp];
        for (int r = 0; r < nr; ++r) {
          const float2 q = S[r][tid];
          w.x += q.x;
          w.y += q.y;
        }
        acc[comp] = w;
      }
    }
  }
  if (tid < NC)
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) M[((int64_t)leaf * 3 + comp) * NC + tid] = acc[comp];
}

template <int P>
void launch_p2m(Ctx& c) {
  LCells lc{c.cells.level.p, c.cells.qx.p, c.cells.qy.p, c.cells.qz.p, c.cells.begin.p, c.cells.count.p};
  FMM_LAUNCH(c, k_p2m_reg<P>, (unsigned)c.nleaves, 64, 0, c.leaf_ids.p, lc, c.lo[0], c.lo[1], c.lo[2], c.L, c.pos.p,
             c.alp.p, c.M.p);
}

template <int P>
void launch(Ctx& c, float* u_far, float* s_far) {
  LCells lc{c.cells.level.p, c.cells.qx.p, c.cells.qy.p, c.cells.qz.p, c.cells.begin.p, c.cells.count.p};
  FMM_LAUNCH(c, k_l2p_reg<P>, (unsigned)c.nleaves, 64, 0, c.leaf_ids.p, lc, c.lo[0], c.lo[1], c.lo[2], c.L, c.pos.p,
             c.alp.p, c.Lc.p, u_far, s_far);
}

}  // namespace

bool l2p_pass_reg(Ctx& c, float* u_far, float* s_far) {
  if (c.nleaves == 0) return true;
  switch (c.P) {
    case 4: launch<4>(c, u_far, s_far); return true;
    case 6: launch<6>(c, u_far, s_far); return true;
    case 8: launch<8>(c, u_far, s_far); return true;
    case 10: launch<10>(c, u_far, s_far); return true;
    default: return false;
  }
}

bool p2m_pass_reg(Ctx& c) {
  if (c.nleaves == 0) return true;
  switch (c.P) {
    case 4: launch_p2m<4>(c); return true;
    case 6: launch_p2m<6>(c); return true;
    case 8: launch_p2m<8>(c); return true;
    case 10: launch_p2m<10>(c); return true;
    default: return false;
  }
}

}  // namespace fmmb
