// expansions.cu -- the far-field operators of fig:kernels:
// P2M (a5), M2M (a6), M2L (a9), periodic far layers (a8), L2L
// (a10) and L2P (a11), on scaled solid harmonics (Cheng et al.).
// Coefficients are stored normalised by the cell side s (reading Z18):
// M~_n = M_n / s^n and L~_n = L_n s^(n+1), so every translation is evaluated
// on O(1) vectors (D / s_target, d / s_parent) and the dynamic range of the
// FP32 coefficients stays small; sums run from high to low degree.
// Layout: float2 [cell][component][n(n+1)/2 + m], 0 <= m <= n < p.
#include "ctx.cuh"

namespace fmmb {

namespace {

__device__ __forceinline__ void nm_of(int k, int& n, int& m) {
  n = (int)((sqrtf(8.0f * k + 1.0f) - 1.0f) * 0.5f);
  while (n * (n + 1) / 2 > k) --n;
  while ((n + 1) * (n + 2) / 2 <= k) ++n;
  m = k - n * (n + 1) / 2;
}

__device__ __forceinline__ cpx<float> ld(const float2* p) { float2 v = *p; return {v.x, v.y}; }

struct GCells {
  const int *level, *qx, *qy, *qz, *begin, *count, *parent, *child_begin, *nchild, *leaf;
};
GCells gcells(Ctx& c) {
  return {c.cells.level.p, c.cells.qx.p, c.cells.qy.p, c.cells.qz.p, c.cells.begin.p, c.cells.count.p,
          c.cells.parent.p, c.cells.child_begin.p, c.cells.nchild.p, c.cells.leaf.p};
}

struct Geo { double lo[3]; double L; double per[3]; long long per_units[3]; int tmax; };

// ---------------------------------------------------------------- P2M (a5)
// one block per leaf; 32 particles per chunk build their R_n^m((x - c)/s)
// in shared memory, then thread o = (component, coefficient) accumulates
// alpha_{j,comp} conj(R) over the chunk in particle order.
__global__ void k_p2m(int P, const int* __restrict__ leaf_ids, GCells c, Geo g, const float4* __restrict__ pos,
                      const float4* __restrict__ alp, float2* __restrict__ M) {
  extern __shared__ float2 sm[];
  const int nc = P * (P + 1) / 2;
  cpx<float>* R = (cpx<float>*)sm;             // [32][nc]
  float4* A = (float4*)(sm + 32 * nc);          // [32]
  int leaf = leaf_ids[blockIdx.x];
  int lev = c.level[leaf], b = c.begin[leaf], cnt = c.count[leaf];
  double s = g.L / (double)(1 << lev);
  double cx = g.lo[0] + (c.qx[leaf] + 0.5) * s, cy = g.lo[1] + (c.qy[leaf] + 0.5) * s,
         cz = g.lo[2] + (c.qz[leaf] + 0.5) * s;
  int o = threadIdx.x;
  int comp = o / nc, k = o % nc;
  cpx<float> acc = {0.f, 0.f};
  for (int j0 = 0; j0 < cnt; j0 += 32) {
    int nj = min(32, cnt - j0);
    if (threadIdx.x < nj) {
      float4 p = pos[b + j0 + threadIdx.x];
      float y0 = (float)(((double)p.x - cx) / s), y1 = (float)(((double)p.y - cy) / s),
            y2 = (float)(((double)p.z - cz) / s);
      regular_harmonics<float>(y0, y1, y2, P, R + threadIdx.x * nc);
      A[threadIdx.x] = alp[b + j0 + threadIdx.x];
    }
    __syncthreads();
    if (o < 3 * nc) {
      for (int jj = 0; jj < nj; ++jj) {
        float4 a4 = A[jj];
        float a = comp == 0 ? a4.x : (comp == 1 ? a4.y : a4.z);
        cpx<float> r = R[jj * nc + k];
        acc.re += a * r.re;
        acc.im -= a * r.im;
      }
    }
    __syncthreads();
  }
  if (o < 3 * nc) M[((int64_t)leaf * 3 + comp) * nc + k] = make_float2(acc.re, acc.im);
}

// ---------------------------------------------------------------- M2M (a6)
// M~_n^m(parent) = sum_{k,l} conj(R_k^l(d/s_p)) M~_{n-k}^{m-l}(child) 2^{-(n-k)}
// Rd of the 8 child octants: R_n^m(d) for d = (+-1/4, +-1/4, +-1/4) in parent
// side units (octant o = (qx&1) | (qy&1) << 1 | (qz&1) << 2 of the child);
// built once per context, shared by M2M and L2L.
__global__ void k_octant_harmonics(int P, float2* __restrict__ R8) {
  const int o = threadIdx.x;
  if (o >= 8) return;
  const float dx = 0.5f * ((float)(o & 1) - 0.5f), dy = 0.5f * ((float)((o >> 1) & 1) - 0.5f),
              dz = 0.5f * ((float)((o >> 2) & 1) - 0.5f);
  regular_harmonics<float>(dx, dy, dz, P, (cpx<float>*)(R8 + o * (P * (P + 1) / 2)));
}

__device__ __forceinline__ int child_octant(const GCells& c, int ch, int p) {
  return (c.qx[ch] - 2 * c.qx[p]) | ((c.qy[ch] - 2 * c.qy[p]) << 1) | ((c.qz[ch] - 2 * c.qz[p]) << 2);
}

__global__ void k_m2m(int P, int64_t first, GCells c, const float2* __restrict__ R8, float2* __restrict__ M) {
  extern __shared__ float2 sm[];
  const int nc = P * (P + 1) / 2;
  cpx<float>* Rd = (cpx<float>*)sm;             // [8][nc]
  cpx<float>* Ms = (cpx<float>*)(sm + 8 * nc);  // [8][3][nc]: the children's multipoles
  int p = (int)(first + blockIdx.x);
  if (c.leaf[p]) return;
  int cb = c.child_begin[p], nch = c.nchild[p];
  for (int i = threadIdx.x; i < nch * nc; i += blockDim.x) {
    const int q = i / nc, k = i - nc * (i / nc);
    const float2 r = R8[child_octant(c, cb + q, p) * nc + k];
    Rd[i] = {r.x, r.y};
  }
  // the children are consecutive cells: one contiguous block of multipoles
  for (int i = threadIdx.x; i < nch * 3 * nc; i += blockDim.x) {
    const float2 v = M[(int64_t)cb * 3 * nc + i];
    Ms[i] = {v.x, v.y};
  }
  __syncthreads();
  int o = threadIdx.x;
  if (o >= 3 * nc) return;
  int comp = o / nc, k = o % nc, n, m;
  nm_of(k, n, m);
  cpx<float> acc = {0.f, 0.f};
  for (int q = 0; q < nch; ++q) {
    const cpx<float>* R = Rd + q * nc;
    const cpx<float>* Mc = Ms + (q * 3 + comp) * nc;
    for (int kk = n; kk >= 0; --kk) {
      int nn = n - kk;
      float sc = ldexpf(1.0f, -nn);
      for (int l = -kk; l <= kk; ++l) {
        int mm = m - l;
        if (mm < -nn || mm > nn) continue;
        cpx<float> t = cmulc(cget(Mc, nn, mm), cget(R, kk, l));
        acc.re += sc * t.re;
        acc.im += sc * t.im;
      }
    }
  }
  M[((int64_t)p * 3 + comp) * nc + k] = make_float2(acc.re, acc.im);
}

// ---------------------------------------------------------------- M2L (a9)
// One block per target cell (the paper's mapping: a target cell per
// thread block, source cells staged in shared memory one after another); a
// thread per local coefficient (k, l) for all three components.
// L~_k^l(t) += (-1)^k sum_{n<p-k} sum_m M~_n^m(s) (s_s/s_t)^n I_{n+k}^{m+l}(D/s_t)
// with D = c_t - c_s - img L evaluated exactly from integer cell coordinates.
__global__ void k_m2l(int P, int64_t ncells, const int* __restrict__ seg_b, const int* __restrict__ seg_e,
                      const uint64_t* __restrict__ lst, GCells c, Geo g, const float2* __restrict__ M,
                      float2* __restrict__ Lc) {
  extern __shared__ float2 sm[];
  const int nc = P * (P + 1) / 2;
  const int P2 = P;   // I_j for j = n + k <= p - 1
  const int nc2 = P2 * (P2 + 1) / 2;
  cpx<float>* Is = (cpx<float>*)sm;            // [nc2]
  cpx<float>* Ms = (cpx<float>*)(sm + nc2);    // [3][nc]
  int t = blockIdx.x;
  int b = seg_b[t], e = seg_e[t];
  if (b == e) return;
  int lt = c.level[t];
  long long ctx = (long long)(2 * c.qx[t] + 1) << (kMaxLevel - lt);
  long long cty = (long long)(2 * c.qy[t] + 1) << (kMaxLevel - lt);
  long long ctz = (long long)(2 * c.qz[t] + 1) << (kMaxLevel - lt);
  float inv_st = ldexpf(1.0f, -(kMaxLevel + 1 - lt));
  int k = 0, l = 0;
  if ((int)threadIdx.x < nc) nm_of(threadIdx.x, k, l);
  cpx<float> acc[3] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
  for (int q = b; q < e; ++q) {
    uint64_t ent = lst[q];
    int src = (int)((ent >> 5) & 0x7ffffff), img = (int)(ent & 31);
    int ls = c.level[src];
    int ix = img % 3 - 1, iy = (img / 3) % 3 - 1, iz = img / 9 - 1;
    long long dx = ctx - ((long long)(2 * c.qx[src] + 1) << (kMaxLevel - ls)) - (long long)ix * g.per_units[0];
    long long dy = cty - ((long long)(2 * c.qy[src] + 1) << (kMaxLevel - ls)) - (long long)iy * g.per_units[1];
    long long dz = ctz - ((long long)(2 * c.qz[src] + 1) << (kMaxLevel - ls)) - (long long)iz * g.per_units[2];
    float Dx = (float)dx * inv_st, Dy = (float)dy * inv_st, Dz = (float)dz * inv_st;
    for (int i = threadIdx.x; i < 3 * nc; i += blockDim.x) {
      int kk = i % nc, n, m;
      nm_of(kk, n, m);
      float sc = ldexpf(1.0f, (lt - ls) * n);
      float2 v = M[(int64_t)src * 3 * nc + i];
      Ms[i] = {v.x * sc, v.y * sc};
    }
    for (int m = threadIdx.x; m < P2; m += blockDim.x) irregular_column<float>(Dx, Dy, Dz, m, P2, Is);
    __syncthreads();
    if ((int)threadIdx.x < nc) {
      for (int n = P - 1 - k; n >= 0; --n)
        for (int m = -n; m <= n; ++m) {
          cpx<float> I = cget(Is, n + k, m + l);
          for (int comp = 0; comp < 3; ++comp) {
            cpx<float> Mv = cget(Ms + comp * nc, n, m);
            acc[comp].re += Mv.re * I.re - Mv.im * I.im;
            acc[comp].im += Mv.re * I.im + Mv.im * I.re;
          }
        }
    }
    __syncthreads();
  }
  if ((int)threadIdx.x < nc) {
    float sg = (k & 1) ? -1.f : 1.f;
    for (int comp = 0; comp < 3; ++comp) {
      float2* d = Lc + ((int64_t)t * 3 + comp) * nc + threadIdx.x;
      float2 v = *d;
      *d = make_float2(v.x + sg * acc[comp].re, v.y + sg * acc[comp].im);
    }
  }
}

// --------------------------------------------- periodic far layers (a8)
// Double precision (the work is O(1) in N: 702 (k-1) M2L per far target).
// far_M[j] holds M^{(j+1)} about the domain centre c0, normalised by L 3^j
// (L = root cube side).  M^{(1)} is the root multipole shifted from the root
// cube centre to c0 (the same point unless the domain is tiled, Z27).
__global__ void k_far_super(int P, int k, Geo g, const float2* __restrict__ Mroot, double* __restrict__ farM) {
  extern __shared__ double smd[];
  const int nc = P * (P + 1) / 2;
  cpx<double>* R = (cpx<double>*)smd;                // [nc]
  cpx<double>* F = (cpx<double>*)farM;
  cpx<double>* T = F + (k - 1) * 3 * nc;             // scratch: root multipole (double)
  int o = threadIdx.x;
  for (int i = o; i < 3 * nc; i += blockDim.x) T[i] = {(double)Mroot[i].x, (double)Mroot[i].y};
  for (int j = 0; j + 1 < k; ++j) {
    // j = 0: root (cube centre) -> c0 at the same scale; j >= 1: 27 shifted copies of M^{(j)}
    const cpx<double>* Mj = j == 0 ? T : F + (j - 1) * 3 * nc;
    cpx<double>* Mn = F + j * 3 * nc;
    int comp = o / nc, kk0 = o % nc, n = 0, m = 0;
    if (o < 3 * nc) nm_of(kk0, n, m);
    cpx<double> acc = {0, 0};
    const int ncopy = j == 0 ? 1 : 27;
    for (int C3 = 0; C3 < ncopy; ++C3) {
      __syncthreads();
      if (o == 0) {
        double dx, dy, dz, sc;
        if (j == 0) {   // d = root centre - c0, in units of L
          dx = 0.5 - 0.5 * g.per[0] / g.L; dy = 0.5 - 0.5 * g.per[1] / g.L; dz = 0.5 - 0.5 * g.per[2] / g.L;
          sc = 1.0;
        } else {        // d = C (.) per 3^{j-1}, in units of L 3^j
          dx = (C3 % 3 - 1) * g.per[0] / g.L / 3.0;
          dy = ((C3 / 3) % 3 - 1) * g.per[1] / g.L / 3.0;
          dz = (C3 / 9 - 1) * g.per[2] / g.L / 3.0;
          sc = 1.0 / 3.0;
        }
        (void)sc;
        regular_harmonics<double>(dx, dy, dz, P, R);
      }
      __syncthreads();
      if (o < 3 * nc) {
        for (int kk = n; kk >= 0; --kk) {
          int nn = n - kk;
          double sc = j == 0 ? 1.0 : pow(3.0, -nn);
          for (int l = -kk; l <= kk; ++l) {
            int mm = m - l;
            if (mm < -nn || mm > nn) continue;
            cpx<double> t2 = cmulc(cget(Mj + comp * nc, nn, mm), cget(R, kk, l));
            acc.re += sc * t2.re;
            acc.im += sc * t2.im;
          }
        }
      }
    }
    __syncthreads();
    if (o < 3 * nc) Mn[comp * nc + kk0] = acc;
    __syncthreads();
  }
}

// block (x = target, y = chunk): chunk = (layer j - 1) * 26 + (neighbour I != 0);
// the 27 children C of that neighbour are summed here, the chunks are summed
// in a fixed order by k_far_reduce (deterministic).
// In a tiled domain (Z27) the first far layer uses the tiles' own multipoles
// (level-1 cells, radius (sqrt3/2) box_len) instead of the elongated domain's,
// which keeps the convergence ratio of the cubic case.
__global__ void k_far_m2l(int P, int k, const int* __restrict__ targets, int ntg, GCells c, Geo g,
                          const double* __restrict__ farM, int ntile, const float2* __restrict__ Mtop,
                          double2* __restrict__ part) {
  extern __shared__ double smd[];
  const int nc = P * (P + 1) / 2;
  const int P2 = P;   // I_j for j = n + k <= p - 1
  const int nc2 = P2 * (P2 + 1) / 2;
  cpx<double>* Is = (cpx<double>*)smd;          // [nc2]
  cpx<double>* Ms = Is + nc2;                   // [3][nc]
  const cpx<double>* F = (const cpx<double>*)farM;
  const int t = targets[blockIdx.x];
  const int chunk = blockIdx.y;
  const int j = 1 + chunk / 26;
  int I3 = chunk % 26;
  if (I3 >= kImgCentre) ++I3;
  const int lt = c.level[t];
  const double st = g.L / (double)(1 << lt);
  const double rx = (c.qx[t] + 0.5) * st - 0.5 * g.per[0], ry = (c.qy[t] + 0.5) * st - 0.5 * g.per[1],
               rz = (c.qz[t] + 0.5) * st - 0.5 * g.per[2];   // c_t - c_0 (domain centre)
  int kq = 0, lq = 0;
  if ((int)threadIdx.x < nc) nm_of(threadIdx.x, kq, lq);
  cpx<double> acc[3] = {{0, 0}, {0, 0}, {0, 0}};
  double scale = g.L;
  for (int jj = 1; jj < j; ++jj) scale *= 3.0;
  const double f3 = scale / g.L;   // 3^{j-1}
  const bool tiled = ntile > 0 && j == 1;
  const int nsrc = tiled ? ntile : 1;
  for (int ts = 0; ts < nsrc; ++ts) {
    double tox = 0, toy = 0, toz = 0;            // source centre offset from c0
    __syncthreads();
    if (tiled) {
      const int o = ts;                          // tile ts = the level-1 cell of octant ts (x fastest, Z27)
      const double s1 = 0.5 * g.L;
      tox = ((o & 1) + 0.5) * s1 - 0.5 * g.per[0];
      toy = (((o >> 1) & 1) + 0.5) * s1 - 0.5 * g.per[1];
      toz = (((o >> 2) & 1) + 0.5) * s1 - 0.5 * g.per[2];
      const double ratio = s1 / st;
      for (int i = threadIdx.x; i < 3 * nc; i += blockDim.x) {
        int kk = i % nc, n, m;
        nm_of(kk, n, m);
        const double sc = pow(ratio, n);
        const float2 v = Mtop[(int64_t)(1 + o) * 3 * nc + i];
        Ms[i] = {(double)v.x * sc, (double)v.y * sc};
      }
    } else {
      const double ratio = scale / st;
      for (int i = threadIdx.x; i < 3 * nc; i += blockDim.x) {
        int kk = i % nc, n, m;
        nm_of(kk, n, m);
        const double sc = pow(ratio, n);
        const cpx<double> v = F[(j - 1) * 3 * nc + i];
        Ms[i] = {v.re * sc, v.im * sc};
      }
    }
    for (int C3 = 0; C3 < 27; ++C3) {
      double ox = 3 * (I3 % 3 - 1) + (C3 % 3 - 1), oy = 3 * ((I3 / 3) % 3 - 1) + ((C3 / 3) % 3 - 1),
             oz = 3 * (I3 / 9 - 1) + (C3 / 9 - 1);
      double Dx = (rx - ox * g.per[0] * f3 - tox) / st, Dy = (ry - oy * g.per[1] * f3 - toy) / st,
             Dz = (rz - oz * g.per[2] * f3 - toz) / st;
      __syncthreads();
      for (int m = threadIdx.x; m < P2; m += blockDim.x) irregular_column<double>(Dx, Dy, Dz, m, P2, Is);
      __syncthreads();
      if ((int)threadIdx.x < nc) {
        for (int n = P - 1 - kq; n >= 0; --n)
          for (int m = -n; m <= n; ++m) {
            cpx<double> I = cget(Is, n + kq, m + lq);
            for (int comp = 0; comp < 3; ++comp) {
              cpx<double> Mv = cget(Ms + comp * nc, n, m);
              acc[comp].re += Mv.re * I.re - Mv.im * I.im;
              acc[comp].im += Mv.re * I.im + Mv.im * I.re;
            }
          }
      }
    }
  }
  if ((int)threadIdx.x < nc) {
    const double sg = (kq & 1) ? -1.0 : 1.0;
    for (int comp = 0; comp < 3; ++comp)
      part[((int64_t)chunk * ntg + blockIdx.x) * 3 * nc + comp * nc + threadIdx.x] =
          make_double2(sg * acc[comp].re, sg * acc[comp].im);
  }
}

__global__ void k_far_reduce(int nc, int nchunk, const int* __restrict__ targets, int ntg,
                             const double2* __restrict__ part, float2* __restrict__ Lc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntg * 3 * nc) return;
  const int ti = i / (3 * nc), o = i - ti * 3 * nc;
  double sr = 0, si = 0;
  for (int ch = 0; ch < nchunk; ++ch) {
    const double2 v = part[((int64_t)ch * ntg + ti) * 3 * nc + o];
    sr += v.x;
    si += v.y;
  }
  float2* d = Lc + (int64_t)targets[ti] * 3 * nc + o;
  const float2 old = *d;
  *d = make_float2((float)((double)old.x + sr), (float)((double)old.y + si));
}

// ---------------------------------------------------------------- L2L (a10)
// L~_a^b(child) += 2^{-(a+1)} sum_{k>=a,l} L~_k^l(parent) conj(R_{k-a}^{l-b}(d/s_p))
__global__ void k_l2l(int P, int64_t first, GCells c, const float2* __restrict__ R8, float2* __restrict__ Lc) {
  extern __shared__ float2 sm[];
  const int nc = P * (P + 1) / 2;
  cpx<float>* Rd = (cpx<float>*)sm;          // [nc]
  cpx<float>* Lp = (cpx<float>*)(sm + nc);   // [3][nc]
  int ch = (int)(first + blockIdx.x);
  int p = c.parent[ch];
  const int oct = child_octant(c, ch, p);
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    const float2 r = R8[oct * nc + i];
    Rd[i] = {r.x, r.y};
  }
  for (int i = threadIdx.x; i < 3 * nc; i += blockDim.x) Lp[i] = ld(Lc + (int64_t)p * 3 * nc + i);
  __syncthreads();
  int o = threadIdx.x;
  if (o >= 3 * nc) return;
  int comp = o / nc, kk0 = o % nc, a, bb;
  nm_of(kk0, a, bb);
  cpx<float> acc = {0.f, 0.f};
  for (int k = P - 1; k >= a; --k)
    for (int l = -k; l <= k; ++l) {
      int ka = k - a, lb = l - bb;
      if (lb < -ka || lb > ka) continue;
      cpx<float> t = cmulc(cget(Lp + comp * nc, k, l), cget(Rd, ka, lb));
      acc.re += t.re;
      acc.im += t.im;
    }
  float sc = ldexpf(1.0f, -(a + 1));
  float2* d = Lc + ((int64_t)ch * 3 + comp) * nc + kk0;
  float2 v = *d;
  *d = make_float2(v.x + sc * acc.re, v.y + sc * acc.im);
}

// ---------------------------------------------------------------- L2P (a11)
// Shift L~ to the particle keeping degrees 1..2 (8c-2 item 16):
// L'_a^b = s^{-a-1} sum_{k>=a,l} L~_k^l conj(R_{k-a}^{l-b}(y)), y = (x - c)/s;
// grad phi = (-Re L'_1^1, -Im L'_1^1, Re L'_1^0); Hessian from L'_2^{0,1,2};
// u = (1/4pi) eps_abc d_b phi_c, s = (1/4pi) alpha_d eps_abc H^c_db.
__global__ void k_l2p(int P, const int* __restrict__ leaf_ids, GCells c, Geo g, const float4* __restrict__ pos,
                      const float4* __restrict__ alp, const float2* __restrict__ Lc, float* __restrict__ uf,
                      float* __restrict__ sf) {
  extern __shared__ float2 sm[];
  const int nc = P * (P + 1) / 2;
  cpx<float>* Ls = (cpx<float>*)sm;               // [3][nc]
  cpx<float>* Rall = (cpx<float>*)(sm + 3 * nc);  // [32][nc]
  int leaf = leaf_ids[blockIdx.x];
  int lev = c.level[leaf], b = c.begin[leaf], cnt = c.count[leaf];
  double s = g.L / (double)(1 << lev);
  double cx = g.lo[0] + (c.qx[leaf] + 0.5) * s, cy = g.lo[1] + (c.qy[leaf] + 0.5) * s,
         cz = g.lo[2] + (c.qz[leaf] + 0.5) * s;
  for (int i = threadIdx.x; i < 3 * nc; i += blockDim.x) Ls[i] = ld(Lc + (int64_t)leaf * 3 * nc + i);
  __syncthreads();
  float is2 = (float)(1.0 / (s * s)), is3 = (float)(1.0 / (s * s * s));
  const float k4 = (float)(1.0 / (4.0 * kPi));
  cpx<float>* R = Rall + threadIdx.x * nc;
  for (int i0 = 0; i0 < cnt; i0 += blockDim.x) {
    int i = i0 + threadIdx.x;
    if (i >= cnt) break;
    float4 p = pos[b + i];
    float y0 = (float)(((double)p.x - cx) / s), y1 = (float)(((double)p.y - cy) / s), y2 = (float)(((double)p.z - cz) / s);
    regular_harmonics<float>(y0, y1, y2, P, R);
    float gr[3][3], H[3][6];
    for (int comp = 0; comp < 3; ++comp) {
      const cpx<float>* Lq = Ls + comp * nc;
      cpx<float> Lp[5];   // (1,0) (1,1) (2,0) (2,1) (2,2)
      const int A_[5] = {1, 1, 2, 2, 2}, B_[5] = {0, 1, 0, 1, 2};
      for (int q = 0; q < 5; ++q) {
        int a = A_[q], bb = B_[q];
        cpx<float> acc = {0.f, 0.f};
        for (int k = P - 1; k >= a; --k)
          for (int l = -k; l <= k; ++l) {
            int ka = k - a, lb = l - bb;
            if (lb < -ka || lb > ka) continue;
            cpx<float> t = cmulc(cget(Lq, k, l), cget(R, ka, lb));
            acc.re += t.re;
            acc.im += t.im;
          }
        Lp[q] = acc;
      }
      gr[comp][0] = -Lp[1].re * is2;
      gr[comp][1] = -Lp[1].im * is2;
      gr[comp][2] = Lp[0].re * is2;
      H[comp][0] = 0.5f * (-Lp[2].re + Lp[4].re) * is3;   // xx
      H[comp][1] = 0.5f * (-Lp[2].re - Lp[4].re) * is3;   // yy
      H[comp][2] = Lp[2].re * is3;                         // zz
      H[comp][3] = 0.5f * Lp[4].im * is3;                  // xy
      H[comp][4] = -Lp[3].re * is3;                        // xz
      H[comp][5] = -Lp[3].im * is3;                        // yz
    }
    // H(c)[d][b] accessor
    auto Hc = [&](int comp, int d, int bb) -> float {
      if (d == bb) return H[comp][d];
      int lo_ = min(d, bb), hi_ = max(d, bb);
      return lo_ == 0 ? (hi_ == 1 ? H[comp][3] : H[comp][4]) : H[comp][5];
    };
    float4 ai = alp[b + i];
    float av[3] = {ai.x, ai.y, ai.z};
    float u0 = gr[2][1] - gr[1][2], u1 = gr[0][2] - gr[2][0], u2 = gr[1][0] - gr[0][1];
    float s0 = 0.f, s1 = 0.f, s2 = 0.f;
    for (int d = 0; d < 3; ++d) {
      s0 += av[d] * (Hc(2, d, 1) - Hc(1, d, 2));
      s1 += av[d] * (Hc(0, d, 2) - Hc(2, d, 0));
      s2 += av[d] * (Hc(1, d, 0) - Hc(0, d, 1));
    }
    int64_t o = 3 * (int64_t)(b + i);
    uf[o] = k4 * u0; uf[o + 1] = k4 * u1; uf[o + 2] = k4 * u2;
    sf[o] = k4 * s0; sf[o + 1] = k4 * s1; sf[o + 2] = k4 * s2;
  }
}

inline int round32(int v) { return (v + 31) / 32 * 32; }

}  // namespace

static Geo geo(const Ctx& c) {
  return {{c.lo[0], c.lo[1], c.lo[2]}, c.L, {c.per[0], c.per[1], c.per[2]},
          {c.per_units[0], c.per_units[1], c.per_units[2]}, c.tmax};
}

// the 8 child-octant harmonic tables (depend on p only)
const float2* octant_r(Ctx& c) {
  if (c.r8_order != c.P) {
    c.r8.reserve((size_t)8 * c.nc);
    FMM_LAUNCH(c, k_octant_harmonics, 1, 32, 0, c.P, c.r8.p);
    c.r8_order = c.P;
  }
  return c.r8.p;
}

// gather (dir 0: M rows of the listed cells -> packed buffer) or scatter (dir 1)
__global__ void k_cells_copy(const int* __restrict__ ids, int64_t nid, int64_t rows, const float2* __restrict__ src,
                             float2* __restrict__ dst, int dir) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nid * rows; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / rows, r = i - k * rows, cell = ids[k];
    if (dir == 0) dst[i] = src[cell * rows + r];
    else dst[cell * rows + r] = src[i];
  }
}

void upward_pass(Ctx& c) {
  cudaStream_t st = c.stream;
  int P = c.P, nc = c.nc;
  GCells gc = gcells(c);
  if (c.nleaves > 0 && !p2m_pass_reg(c)) {
    size_t sm = sizeof(float2) * (32 * nc) + sizeof(float4) * 32;
    FMM_LAUNCH(c, k_p2m, (unsigned)c.nleaves, round32(3 * nc), sm, P, c.leaf_ids.p, gc, geo(c), c.pos.p, c.alp.p, c.M.p);
    FMM_LAUNCH_CHECK();
  }
  // M2M over this rank's (local-tree) cells
  int nlev = (int)c.level_begin.size() - 1;
  for (int l = nlev - 2; l >= 0; --l) {
    int64_t first = c.loc_lo[l], cnt = c.loc_hi[l] - c.loc_lo[l];
    if (cnt <= 0) continue;
    if (!m2m_level_reg(c, first, cnt, octant_r(c)))
      FMM_LAUNCH(c, k_m2m, (unsigned)cnt, round32(3 * nc), sizeof(float2) * 32 * nc, P, first, gc, octant_r(c), c.M.p);
  }
  // (nranks > 1: the root and level-1 multipoles of all ranks are summed by
  // let_exchange into top_M for the periodic far field)
}

void m2l_pass(Ctx& c) {
  if (c.nm2l == 0) {
    for (auto& e : c.ev_m2l) FMM_CUDA(cudaEventRecord(e, c.stream));
    return;
  }
  // tensor-core M2L on the uniform levels (m2l_tc.cu), decided once per list build
  if (!c.tc_valid) {
    m2l_tc_prepare(c);      // decides which targets the tensor path takes (verified entry by entry)
    m2l_reg_segments(c);    // the remaining entries, grouped by target for the register kernels
  }
  FMM_CUDA(cudaEventRecord(c.ev_m2l[0], c.stream));
  m2l_tc_run(c);
  FMM_CUDA(cudaEventRecord(c.ev_m2l[1], c.stream));
  if (!m2l_pass_reg(c)) {   // register-blocked kernel (m2l.cu) for p in {4, 6, 8, 10}, else the generic one
    int P = c.P, nc = c.nc, P2 = P, nc2 = P2 * (P2 + 1) / 2;
    size_t sm = sizeof(float2) * (nc2 + 3 * nc);
    FMM_LAUNCH(c, k_m2l, (unsigned)c.ncells, round32(nc), sm, P, c.ncells, c.m2l_b.p, c.m2l_e.p, c.m2lr.p, gcells(c),
               geo(c), c.M.p, c.Lc.p);
    FMM_LAUNCH_CHECK();
  }
  FMM_CUDA(cudaEventRecord(c.ev_m2l[2], c.stream));
}

// phase 1: the super-cell multipoles and the far layers' M2L into per-chunk
// partials (independent of the M2L list: may run beside it); phase 2: the
// fixed-order reduction of the partials into the locals; 3: both
void periodic_far_pass(Ctx& c, int phase) {
  int k = c.cfg.images;
  if (phase & 1) c.far_ntg = 0;
  if (k < 2 || c.ncells == 0) { if (phase & 1) c.far_m2l = 0; return; }
  if (!(phase & 1)) {
    if (c.far_ntg > 0)
      FMM_LAUNCH(c, k_far_reduce, nblocks((int64_t)c.far_ntg * 3 * c.nc, 128), 128, 0, c.nc, c.far_nchunk, c.far_tg.p,
                 c.far_ntg, c.far_part.p, c.Lc.p);
    return;
  }
  c.far_m2l = 0;
  int P = c.P, nc = c.nc, P2 = P, nc2 = P2 * (P2 + 1) / 2;
  // far targets: cells of side box_len / 4 (level 2 + log2 tmax) and leaves above
  // (this rank's cells only)
  const int lt = 2 + (c.tmax == 2 ? 1 : 0);
  std::vector<int> tg;
  for (size_t i = 0; i < c.host_leaf_top.size(); ++i) {
    if (!c.host_leaf_top[i]) continue;
    int l = 0;
    while (l + 1 < (int)c.level_begin.size() && (int64_t)i >= c.level_begin[l + 1]) ++l;
    if ((int64_t)i >= c.loc_lo[l] && (int64_t)i < c.loc_hi[l]) tg.push_back((int)i);
  }
  if ((int)c.level_begin.size() > lt + 1)
    for (int64_t i = c.loc_lo[lt]; i < c.loc_hi[lt]; ++i) tg.push_back((int)i);
  if (tg.empty()) return;
  // sources: the root multipole (slot 0) and the tiles' (level-1 cells, slots 1 + octant) --
  // summed over the ranks by let_exchange, from the local tree here on one GPU
  if (c.cfg.nranks == 1) top_multipoles(c, c.stream);
  c.far_M.reserve((size_t)k * 3 * nc * 2);
  FMM_LAUNCH(c, k_far_super, 1, round32(3 * nc), sizeof(double) * 2 * nc, P, k, geo(c), c.top_M.p, c.far_M.p);
  FMM_LAUNCH_CHECK();
  c.far_tg.reserve(tg.size() + 1);
  // (pageable source: the call returns once tg has been staged, so tg may go)
  FMM_CUDA(cudaMemcpyAsync(c.far_tg.p, tg.data(), sizeof(int) * tg.size(), cudaMemcpyHostToDevice, c.stream));
  size_t sm = sizeof(double) * 2 * (nc2 + 3 * nc);
  const int ntg = (int)tg.size(), nchunk = 26 * (k - 1);
  c.far_part.reserve((size_t)nchunk * ntg * 3 * nc);
  const int ntile = c.tmax > 1 ? c.cfg.tiles[0] * c.cfg.tiles[1] * c.cfg.tiles[2] : 0;
  FMM_LAUNCH(c, k_far_m2l, dim3(ntg, nchunk), round32(nc), sm, P, k, c.far_tg.p, ntg, gcells(c), geo(c), c.far_M.p,
             ntile, c.top_M.p, c.far_part.p);
  c.far_ntg = ntg;
  c.far_nchunk = nchunk;
  if (phase & 2)
    FMM_LAUNCH(c, k_far_reduce, nblocks((int64_t)ntg * 3 * nc, 128), 128, 0, nc, nchunk, c.far_tg.p, ntg, c.far_part.p,
               c.Lc.p);
  FMM_LAUNCH_CHECK();
  c.far_m2l = (int64_t)tg.size() * 702 * (k - 1 + (ntile > 1 ? ntile - 1 : 0));
}

void downward_pass(Ctx& c, float* u_far, float* s_far) {
  cudaStream_t st = c.stream;
  int P = c.P, nc = c.nc;
  GCells gc = gcells(c);
  int nlev = (int)c.level_begin.size() - 1;
  for (int l = 1; l < nlev; ++l) {
    int64_t first = c.loc_lo[l], cnt = c.loc_hi[l] - first;
    if (cnt <= 0) continue;
    if (!l2l_level_reg(c, c.level_begin[l - 1], c.level_begin[l] - c.level_begin[l - 1], first, first + cnt,
                       octant_r(c)))
      FMM_LAUNCH(c, k_l2l, (unsigned)cnt, round32(3 * nc), sizeof(float2) * 4 * nc, P, first, gc, octant_r(c), c.Lc.p);
    FMM_LAUNCH_CHECK();
  }
  if (c.nleaves > 0 && !l2p_pass_reg(c, u_far, s_far)) {
    size_t sm = sizeof(float2) * (3 * nc + 32 * nc);
    FMM_LAUNCH(c, k_l2p, (unsigned)c.nleaves, 32, sm, P, c.leaf_ids.p, gc, geo(c), c.pos.p, c.alp.p, c.Lc.p, u_far, s_far);
    FMM_LAUNCH_CHECK();
  }
}

void set_expansion_smem_limits() {
  int big = 200 * 1024;
  cudaFuncSetAttribute(k_p2m, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  cudaFuncSetAttribute(k_l2p, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  cudaFuncSetAttribute(k_m2l, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  cudaFuncSetAttribute(k_far_m2l, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
}

}  // namespace fmmb
