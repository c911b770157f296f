// rbf.cu -- NEXT-4: radial-basis-function reinitialisation of the
// particle field, "a radial basis function interpolation for reinitialized
// Gaussian distributions", onto particles that are "reinitialized to
// the same position every time", so the tree is reused.
//
// The Gaussian core of Eq. 2 is the vorticity of one particle:
//   zeta_s(r) = (2 pi s^2)^{-3/2} exp(-r^2 / (2 s^2)),   g(rho) = int_0^r 4 pi t^2 zeta_s(t) dt
// so the old field's vorticity at the new sites y_i is
//   b_i = sum_n sum_j alpha_j zeta_{sigma_j}(y_i - x_j - n L)                     (1)
// and the new strengths beta (core sigma0 on every site) solve the collocation
// system (the Gaussian basis is the RBF; SURVEY 8f reading):
//   sum_n sum_k beta_k zeta_{sigma0}(y_i - y_k - n L) = b_i                       (2)
// A is symmetric positive definite, so (2) is solved by conjugate gradients on
// the three components at once.  Both sums run over the P2P lists of the tree
// (near field): every pair the lists leave out lies in an M2L-accepted cell pair,
// >= (1/theta - 1)(r_A + r_B) apart, where zeta is below e^{-24} of its peak
// for sigma <= h and 4h leaves (reading R1 in DESIGN.md).  Single GPU.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ctx.cuh"

namespace fmmb {

namespace {

constexpr int TP = 64;   // targets per pass and sources per tile
constexpr int NT = 32;   // one warp per target leaf, two targets per lane

struct GCellsR {
  const int *level, *qx, *qy, *qz, *begin, *count;
};

// out[3 i + c] (sorted order, double) = sum over the list entries of target
// leaf A of sum_{j in B} q_{j,c} zeta_{sigma_j}(x_i - x_j - img L).  Sources are
// staged in the target-leaf frame (shift in double, then FP32); FP32 tile
// partials are added in double.  r = 0 is a regular point of zeta (the self
// term is included).
__global__ void __launch_bounds__(NT) k_gauss(const int* __restrict__ leaf_ids, const int* __restrict__ seg_b,
                                              const int* __restrict__ seg_e, const uint64_t* __restrict__ lst,
                                              GCellsR c, double lo0, double lo1, double lo2, double L, double px,
                                              double py, double pz, const float4* __restrict__ pos,
                                              const float4* __restrict__ q, double* __restrict__ out) {
  __shared__ float4 sx[TP];   // (x', y', z', -log2(e) / (2 sigma^2))
  __shared__ float4 sq[TP];   // q (2 pi sigma^2)^{-3/2}
  const int lane = threadIdx.x;
  const int leaf = leaf_ids[blockIdx.x];
  const int lev = c.level[leaf], tb = c.begin[leaf], tcnt = c.count[leaf];
  const double s = L / (double)(1 << lev);
  const double cx = lo0 + (c.qx[leaf] + 0.5) * s, cy = lo1 + (c.qy[leaf] + 0.5) * s, cz = lo2 + (c.qz[leaf] + 0.5) * s;
  const int eb = seg_b[leaf], ee = seg_e[leaf];
  for (int t0 = 0; t0 < tcnt; t0 += TP) {
    float xt[2][3];
    double acc[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = t0 + lane + h * NT;
      const float4 p = i < tcnt ? pos[tb + i] : make_float4(0.f, 0.f, 0.f, 1.f);
      xt[h][0] = (float)((double)p.x - cx);
      xt[h][1] = (float)((double)p.y - cy);
      xt[h][2] = (float)((double)p.z - cz);
    }
    // tight box of this pass's targets: sources farther than 6 sigma_j from it
    // add below e^{-18} of a peak term (under the FP32 resolution of the sums)
    // and are not staged
    float bcen[3], bhw[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const bool v0 = t0 + lane < tcnt, v1 = t0 + lane + NT < tcnt;
      float lo = fminf(v0 ? xt[0][d] : 1e30f, v1 ? xt[1][d] : 1e30f);
      float hi = fmaxf(v0 ? xt[0][d] : -1e30f, v1 ? xt[1][d] : -1e30f);
      for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      }
      bcen[d] = 0.5f * (lo + hi);
      bhw[d] = 0.5f * (hi - lo) * 1.0001f;
    }
    for (int e = eb; e < ee; ++e) {
      const uint64_t ent = lst[e];
      const int src = (int)((ent >> 5) & 0x7ffffff), img = (int)(ent & 31);
      // source j of image img sits at x_j + img L; in the target frame x_j + img L - c
      const double sh0 = (img % 3 - 1) * px - cx, sh1 = ((img / 3) % 3 - 1) * py - cy, sh2 = (img / 9 - 1) * pz - cz;
      const int sb = c.begin[src], scnt = c.count[src];
      for (int s0 = 0; s0 < scnt; s0 += TP) {
        __syncwarp();
        float4 vx[2], vq[2];
        bool keep[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = s0 + lane + h * NT;
          keep[h] = false;
          if (j < scnt) {
            const float4 p = pos[sb + j];
            const float4 a = q[sb + j];
            const float w = 1.0f / (2.0f * p.w * p.w);
            const float k = (float)(1.0 / (2.0 * kPi * sqrt(2.0 * kPi))) / (p.w * p.w * p.w);   // (2 pi)^{-3/2} / s^3
            vx[h] = make_float4((float)((double)p.x + sh0), (float)((double)p.y + sh1), (float)((double)p.z + sh2),
                                -1.4426950408889634f * w);
            vq[h] = make_float4(a.x * k, a.y * k, a.z * k, 0.f);
            const float gx = fmaxf(0.f, fabsf(vx[h].x - bcen[0]) - bhw[0]), gy = fmaxf(0.f, fabsf(vx[h].y - bcen[1]) - bhw[1]),
                        gz = fmaxf(0.f, fabsf(vx[h].z - bcen[2]) - bhw[2]);
            keep[h] = (gx * gx + gy * gy + gz * gz) * w < 18.0f;
          }
        }
        const unsigned lt = (1u << lane) - 1u;
        const unsigned k0 = __ballot_sync(0xffffffffu, keep[0]), k1 = __ballot_sync(0xffffffffu, keep[1]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (!keep[h]) continue;
          const int dst = h == 0 ? __popc(k0 & lt) : __popc(k0) + __popc(k1 & lt);
          sx[dst] = vx[h];
          sq[dst] = vq[h];
        }
        __syncwarp();
        const int nj = __popc(k0) + __popc(k1);
        float part[2][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
        for (int jj = 0; jj < nj; ++jj) {
          const float4 v = sx[jj], a = sq[jj];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float dx = xt[h][0] - v.x, dy = xt[h][1] - v.y, dz = xt[h][2] - v.z;
            const float e2 = exp2f((dx * dx + dy * dy + dz * dz) * v.w);
            part[h][0] += e2 * a.x;
            part[h][1] += e2 * a.y;
            part[h][2] += e2 * a.z;
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
          for (int d = 0; d < 3; ++d) acc[h][d] += (double)part[h][d];
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = t0 + lane + h * NT;
      if (i < tcnt)
        for (int d = 0; d < 3; ++d) out[3 * (int64_t)(tb + i) + d] = acc[h][d];
    }
  }
}

__global__ void k_to_f4(const double* __restrict__ v, int64_t n, float4* __restrict__ q) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    q[i] = make_float4((float)v[3 * i], (float)v[3 * i + 1], (float)v[3 * i + 2], 0.f);
}

// union sorted slot i with caller index idx[i] >= n0 (a site): sites[idx[i] - n0] = v[i]
__global__ void k_take_sites(const double* __restrict__ v, const uint32_t* __restrict__ idx, int64_t N, int64_t n0,
                             double* __restrict__ sites) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = (int64_t)idx[i] - n0;
    if (j >= 0)
      for (int d = 0; d < 3; ++d) sites[3 * j + d] = v[3 * i + d];
  }
}

// caller order -> sorted order (dir 0) or sorted -> caller as float (dir 1)
__global__ void k_permute(const double* __restrict__ v, const uint32_t* __restrict__ idx, int64_t n,
                          double* __restrict__ sorted_out, float* __restrict__ caller_out, int dir) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx[i];
    for (int d = 0; d < 3; ++d) {
      if (dir == 0) sorted_out[3 * i + d] = v[3 * j + d];
      else caller_out[3 * j + d] = (float)v[3 * i + d];
    }
  }
}

__global__ void k_dot(const double* __restrict__ a, const double* __restrict__ b, int64_t n, double* __restrict__ out) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += a[i] * b[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    out[blockIdx.x] = t;                           // per-block partial: summed in order on the host
  }
}

// x += a p, r -= a Ap
__global__ void k_cg1(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                      const double* __restrict__ ap, int64_t n, double a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += a * p[i];
    r[i] -= a * ap[i];
  }
}

// p = r + b p
__global__ void k_cg2(double* __restrict__ p, const double* __restrict__ r, int64_t n, double b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = r[i] + b * p[i];
}

__global__ void k_set_alpha(const double* __restrict__ v, int64_t n, float4* __restrict__ alp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    alp[i] = make_float4((float)v[3 * i], (float)v[3 * i + 1], (float)v[3 * i + 2], 0.f);
}

unsigned gridn(int64_t n) {
  unsigned b = nblocks(n, 256);
  return b > 148 * 8 ? 148 * 8 : b;
}

}  // namespace

// out (sorted order, [ntot][3] double) = Gaussian sums (1)/(2) of the strengths
// q (sorted, float4) over the context's P2P lists
void gauss_pass(Ctx& c, const float4* q, double* out) {
  FMM_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * 3 * std::max<int64_t>(c.ntot, 1), c.stream));
  if (c.nleaves == 0) return;
  GCellsR gc{c.cells.level.p, c.cells.qx.p, c.cells.qy.p, c.cells.qz.p, c.cells.begin.p, c.cells.count.p};
  FMM_LAUNCH(c, k_gauss, (unsigned)c.nleaves, NT, 0, c.leaf_ids.p, c.p2p_b.p, c.p2p_e.p, c.p2p.p, gc, c.lo[0],
             c.lo[1], c.lo[2], c.L, c.per[0], c.per[1], c.per[2], c.pos.p, q, out);
  FMM_LAUNCH_CHECK();
}

// NEXT-4: b at the sites from the old particles (tree of the union), then the
// sites' tree and CG on (2).  The context ends holding the sites with the new
// strengths (ready for evaluate).  Returns the iterations and the relative
// residual ||b - A beta|| / ||b|| of the last iterate.
void rbf_reinit_impl(Ctx& c, int64_t n, const float* x, const float* alpha, const float* sigma, int64_t m,
                     const float* y, float sigma0, double tol, int maxit, float* beta_out, int* iters, double* resid) {
  cudaStream_t st = c.stream;
  const int64_t N = n + m;
  c.st_x.reserve(3 * N); c.st_a.reserve(3 * N); c.st_s.reserve(N);
  if (n > 0) {
    FMM_CUDA(cudaMemcpyAsync(c.st_x.p, x, sizeof(float) * 3 * n, cudaMemcpyDefault, st));
    FMM_CUDA(cudaMemcpyAsync(c.st_a.p, alpha, sizeof(float) * 3 * n, cudaMemcpyDefault, st));
    FMM_CUDA(cudaMemcpyAsync(c.st_s.p, sigma, sizeof(float) * n, cudaMemcpyDefault, st));
  }
  FMM_CUDA(cudaMemcpyAsync(c.st_x.p + 3 * n, y, sizeof(float) * 3 * m, cudaMemcpyDefault, st));
  FMM_CUDA(cudaMemsetAsync(c.st_a.p + 3 * n, 0, sizeof(float) * 3 * m, st));
  fill_f32(c, c.st_s.p + n, m, sigma0);
  // (1): the old field at the sites (sites carry zero strength in the union)
  c.rbf_b.reserve(3 * std::max<int64_t>(m, 1));
  c.rbf_v.reserve(3 * std::max<int64_t>(N, 1));
  set_particles_impl(c, N, c.st_x.p, c.st_a.p, c.st_s.p);
  build_lists(c);
  gauss_pass(c, c.alp.p, c.rbf_v.p);
  FMM_LAUNCH(c, k_take_sites, gridn(N), 256, 0, c.rbf_v.p, c.idx.p, N, n, c.rbf_b.p);
  // (2): the sites alone
  c.st_xh.reserve(3 * m);
  FMM_CUDA(cudaMemcpyAsync(c.st_xh.p, c.st_x.p + 3 * n, sizeof(float) * 3 * m, cudaMemcpyDeviceToDevice, st));
  set_particles_impl(c, m, c.st_xh.p, c.st_a.p + 3 * n, c.st_s.p + n);
  build_lists(c);
  const int64_t L3 = 3 * m;
  c.rbf_x.reserve(L3); c.rbf_r.reserve(L3); c.rbf_p.reserve(L3); c.rbf_ap.reserve(L3);
  c.rbf_q.reserve(std::max<int64_t>(m, 1));
  c.rbf_dot.reserve(148 * 8);
  std::vector<double> part(148 * 8);
  FMM_LAUNCH(c, k_permute, gridn(m), 256, 0, c.rbf_b.p, c.idx.p, m, c.rbf_r.p, nullptr, 0);   // r = b (x0 = 0)
  FMM_CUDA(cudaMemsetAsync(c.rbf_x.p, 0, sizeof(double) * L3, st));
  FMM_CUDA(cudaMemcpyAsync(c.rbf_p.p, c.rbf_r.p, sizeof(double) * L3, cudaMemcpyDeviceToDevice, st));
  auto dot = [&](const double* a, const double* b) {   // deterministic: fixed grid, ordered host sum
    const unsigned g = gridn(L3);
    FMM_LAUNCH(c, k_dot, g, 256, 0, a, b, L3, c.rbf_dot.p);
    FMM_CUDA(cudaMemcpyAsync(part.data(), c.rbf_dot.p, sizeof(double) * g, cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaStreamSynchronize(st));
    double v = 0.0;
    for (unsigned k = 0; k < g; ++k) v += part[k];
    return v;
  };
  const double bb = dot(c.rbf_r.p, c.rbf_r.p);
  double rr = bb;
  int it = 0;
  static const bool dbg = getenv("FMM_RBF_DEBUG") != nullptr;   // development: residual history on stderr
  if (bb > 0.0) {
    while (it < maxit && rr > tol * tol * bb) {
      FMM_LAUNCH(c, k_to_f4, gridn(m), 256, 0, c.rbf_p.p, m, c.rbf_q.p);
      gauss_pass(c, c.rbf_q.p, c.rbf_ap.p);
      const double pap = dot(c.rbf_p.p, c.rbf_ap.p);
      if (dbg) fprintf(stderr, "rbf it %d  |r|/|b| %.3e  pAp/pp %.3e\n", it, sqrt(rr / bb), pap / dot(c.rbf_p.p, c.rbf_p.p));
      if (!(pap > 0.0)) break;                        // A is SPD: only rounding can get here
      const double a = rr / pap;
      FMM_LAUNCH(c, k_cg1, gridn(L3), 256, 0, c.rbf_x.p, c.rbf_r.p, c.rbf_p.p, c.rbf_ap.p, L3, a);
      const double rn = dot(c.rbf_r.p, c.rbf_r.p);
      FMM_LAUNCH(c, k_cg2, gridn(L3), 256, 0, c.rbf_p.p, c.rbf_r.p, L3, rn / rr);
      rr = rn;
      ++it;
    }
  }
  *iters = it;
  *resid = bb > 0.0 ? sqrt(rr / bb) : 0.0;
  // the context now holds the reinitialised particles (same tree, new strengths)
  FMM_LAUNCH(c, k_set_alpha, gridn(m), 256, 0, c.rbf_x.p, m, c.alp.p);
  c.st_u.reserve(3 * m);
  FMM_LAUNCH(c, k_permute, gridn(m), 256, 0, c.rbf_x.p, c.idx.p, m, nullptr, c.st_u.p, 1);
  FMM_CUDA(cudaMemcpyAsync(beta_out, c.st_u.p, sizeof(float) * 3 * m, cudaMemcpyDefault, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  c.evaluated = false;
}

}  // namespace fmmb
