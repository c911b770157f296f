// p2p.cu -- a12: the near field (P2P, fig:kernels P:103) of Eq. 1 and Eq. 3.
//
// For each list entry (A <- B, img) and i in A, j in B, r = x_i - x_j - img L:
//   u_i += f(r) alpha_j x r,                         f = g(rho)/(4 pi r^3)
//   s_i += f (alpha_j x alpha_i) + (f'/r)(r.alpha_i)(alpha_j x r),
//   f'/r = ((4/sqrt pi) rho^3 e^{-rho^2} - 3 g)/(4 pi r^5), rho = r/(sqrt2 sigma_j)
// (readings Z1, Z3, Z4, Z7).  sum_j f (alpha_j x alpha_i) is
// accumulated as (sum_j f alpha_j) x alpha_i.
//
// Mapping: one thread block per target leaf, one target particle per thread
// held in registers; each source leaf of the target's segment is staged in
// shared memory as float4 tiles in *target-leaf-centred* coordinates -- the
// image shift and the centring are done once per source in double and rounded
// to FP32 ("Fix B") -- and the FP32 partial over each tile
// (<= 64 sources) is added to a per-target FP64 accumulator ("Fix A").
#include "ctx.cuh"

namespace fmmb {

namespace {

constexpr int TP = 64;

struct PCells {
  const int *level, *qx, *qy, *qz, *begin, *count;
};

__global__ void __launch_bounds__(TP) k_p2p(const int* __restrict__ leaf_ids, const int* __restrict__ seg_b,
                                            const int* __restrict__ seg_e, const uint64_t* __restrict__ lst,
                                            PCells c, double lo0, double lo1, double lo2, double L,
                                            const float4* __restrict__ pos, const float4* __restrict__ alp,
                                            float* __restrict__ un, float* __restrict__ sn) {
  __shared__ float4 sx[TP];   // (x', y', z', 1/(2 sigma^2))
  __shared__ float4 sa[TP];   // (alpha/(4 pi), 1/(sqrt2 sigma))
  const float k4 = (float)(1.0 / (4.0 * kPi));
  int leaf = leaf_ids[blockIdx.x];
  int lev = c.level[leaf], tb = c.begin[leaf], tcnt = c.count[leaf];
  double s = L / (double)(1 << lev);
  double cx = lo0 + (c.qx[leaf] + 0.5) * s, cy = lo1 + (c.qy[leaf] + 0.5) * s, cz = lo2 + (c.qz[leaf] + 0.5) * s;
  int eb = seg_b[leaf], ee = seg_e[leaf];
  for (int t0 = 0; t0 < tcnt; t0 += TP) {
    int i = t0 + threadIdx.x;
    bool valid = i < tcnt;
    float xi0 = 0.f, xi1 = 0.f, xi2 = 0.f;
    float4 ai = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) {
      float4 p = pos[tb + i];
      xi0 = (float)((double)p.x - cx);
      xi1 = (float)((double)p.y - cy);
      xi2 = (float)((double)p.z - cz);
      ai = alp[tb + i];
    }
    double du0 = 0, du1 = 0, du2 = 0, ds0 = 0, ds1 = 0, ds2 = 0, dA0 = 0, dA1 = 0, dA2 = 0;
    for (int e = eb; e < ee; ++e) {
      uint64_t ent = lst[e];
      int src = (int)((ent >> 5) & 0x7ffffff), img = (int)(ent & 31);
      double shx = (img % 3 - 1) * L - cx, shy = ((img / 3) % 3 - 1) * L - cy, shz = (img / 9 - 1) * L - cz;
      int sb = c.begin[src], scnt = c.count[src];
      for (int s0 = 0; s0 < scnt; s0 += TP) {
        __syncthreads();
        int j = s0 + threadIdx.x;
        if (j < scnt) {
          float4 p = pos[sb + j];
          float4 a = alp[sb + j];
          float kk = 1.0f / (2.0f * p.w * p.w);
          sx[threadIdx.x] = make_float4((float)((double)p.x + shx), (float)((double)p.y + shy),
                                        (float)((double)p.z + shz), kk);
          sa[threadIdx.x] = make_float4(a.x * k4, a.y * k4, a.z * k4, sqrtf(kk));
        }
        __syncthreads();
        int nj = min(TP, scnt - s0);
        if (valid) {
          float pu0 = 0.f, pu1 = 0.f, pu2 = 0.f, ps0 = 0.f, ps1 = 0.f, ps2 = 0.f, pA0 = 0.f, pA1 = 0.f, pA2 = 0.f;
          for (int jj = 0; jj < nj; ++jj) {
            float4 q = sx[jj];
            float4 a = sa[jj];
            float rx = xi0 - q.x, ry = xi1 - q.y, rz = xi2 - q.z;
            float r2 = rx * rx + ry * ry + rz * rz;
            float inv = r2 > 0.f ? rsqrtf(r2) : 0.f;
            float rho2 = r2 * q.w;
            float rho = r2 * inv * a.w;
            float ex = __expf(-rho2);
            float g = erff(rho) - 1.1283791670955126f * rho * ex;
            float inv2 = inv * inv;
            float inv3 = inv2 * inv;
            float f = g * inv3;
            float fp = (2.2567583341910252f * rho * rho2 * ex - 3.0f * g) * inv3 * inv2;
            float c0 = a.y * rz - a.z * ry, c1 = a.z * rx - a.x * rz, c2 = a.x * ry - a.y * rx;
            pu0 += f * c0; pu1 += f * c1; pu2 += f * c2;
            pA0 += f * a.x; pA1 += f * a.y; pA2 += f * a.z;
            float qq = fp * (rx * ai.x + ry * ai.y + rz * ai.z);
            ps0 += qq * c0; ps1 += qq * c1; ps2 += qq * c2;
          }
          du0 += pu0; du1 += pu1; du2 += pu2;
          ds0 += ps0; ds1 += ps1; ds2 += ps2;
          dA0 += pA0; dA1 += pA1; dA2 += pA2;
        }
      }
    }
    if (valid) {
      // (sum_j f alpha_j) x alpha_i
      ds0 += dA1 * ai.z - dA2 * ai.y;
      ds1 += dA2 * ai.x - dA0 * ai.z;
      ds2 += dA0 * ai.y - dA1 * ai.x;
      int64_t o = 3 * (int64_t)(tb + i);
      un[o] = (float)du0; un[o + 1] = (float)du1; un[o + 2] = (float)du2;
      sn[o] = (float)ds0; sn[o + 1] = (float)ds1; sn[o + 2] = (float)ds2;
    }
  }
}

}  // namespace

void p2p_pass(Ctx& c, float* u_near, float* s_near) {
  if (c.nleaves == 0) return;
  PCells pc{c.cells.level.p, c.cells.qx.p, c.cells.qy.p, c.cells.qz.p, c.cells.begin.p, c.cells.count.p};
  FMM_LAUNCH(c, k_p2p, (unsigned)c.nleaves, TP, 0, c.leaf_ids.p, c.p2p_b.p, c.p2p_e.p, c.p2p.p, pc, c.lo[0], c.lo[1],
                                                  c.lo[2], c.L, c.pos.p, c.alp.p, u_near, s_near);
  FMM_LAUNCH_CHECK();
}

}  // namespace fmmb
