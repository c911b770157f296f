// tree.cu -- a1-a4 of the hot path: ingest/validate, periodic
// wrap, 63-bit Morton keys, stable device radix sort (Z17),
// gather into sorted SoA, and the level-by-level octree.
// All of it is HBM-bound streaming work; one thread per particle,
// grid-stride loops, coalesced float4/uint64 traffic.
#include <algorithm>
#include <climits>
#include <cstring>

#include <cub/cub.cuh>

#include "ctx.cuh"

namespace fmmb {

namespace {

// order-preserving float <-> int map for atomicMin/atomicMax
__device__ __forceinline__ int fkey(float f) {
  int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__host__ __forceinline__ float fkey_inv(int i) {
  int j = i >= 0 ? i : i ^ 0x7fffffff;
  float f;
  memcpy(&f, &j, 4);
  return f;
}

// dflag[0] |= 1 non-finite, 2 sigma <= 0; dflag[1..6] = min/max keys of x,y,z
__global__ void k_validate(const float* __restrict__ x, const float* __restrict__ a,
                           const float* __restrict__ s, int64_t n, int* dflag, int want_box) {
  int bad = 0;
  int mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {INT_MIN, INT_MIN, INT_MIN};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int d = 0; d < 3; ++d) {
      float xv = x[3 * i + d], av = a[3 * i + d];
      if (!isfinite(xv) || !isfinite(av)) bad |= 1;
      int k = fkey(xv);
      mn[d] = min(mn[d], k);
      mx[d] = max(mx[d], k);
    }
    float sv = s[i];
    if (!isfinite(sv)) bad |= 1;
    else if (!(sv > 0.0f)) bad |= 2;
  }
  for (int o = 16; o > 0; o >>= 1) {
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    for (int d = 0; d < 3; ++d) {
      mn[d] = min(mn[d], __shfl_xor_sync(0xffffffffu, mn[d], o));
      mx[d] = max(mx[d], __shfl_xor_sync(0xffffffffu, mx[d], o));
    }
  }
  if ((threadIdx.x & 31) == 0) {
    if (bad) atomicOr(dflag, bad);
    if (want_box)
      for (int d = 0; d < 3; ++d) {
        atomicMin(&dflag[1 + d], mn[d]);
        atomicMax(&dflag[4 + d], mx[d]);
      }
  }
}

__device__ __forceinline__ uint64_t spread3(uint64_t v) {
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
__device__ __forceinline__ int compact3(uint64_t v) {
  v &= 0x1249249249249249ull;
  v = (v ^ (v >> 2)) & 0x10c30c30c30c30c3ull;
  v = (v ^ (v >> 4)) & 0x100f00f00f00f00full;
  v = (v ^ (v >> 8)) & 0x1f0000ff0000ffull;
  v = (v ^ (v >> 16)) & 0x1f00000000ffffull;
  v = (v ^ (v >> 32)) & 0x1fffffull;
  return (int)v;
}

struct Box { double lo[3]; double L, scale; double per[3]; int periodic; };

// a1 wrap (periodic) + a2 keys.  Quantisation is IEEE double with explicit
// round-to-nearest intrinsics (no FMA contraction, Z16/Z19):
// q = clamp(floor((x - lo) * (2^21 / L)), 0, 2^21 - 1); bits interleaved with
// x in the lowest bit of every triple.
__global__ void k_keys(const float* __restrict__ x, const float* __restrict__ s, int64_t n, Box b,
                       float4* __restrict__ pos_tmp, uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float xw[3];
    uint64_t key = 0;
    for (int d = 0; d < 3; ++d) {
      double v = (double)x[3 * i + d];
      if (b.periodic && (v < b.lo[d] || v >= b.lo[d] + b.per[d])) {
        double w = __dsub_rn(v, __dmul_rn(b.per[d], floor(__ddiv_rn(__dsub_rn(v, b.lo[d]), b.per[d]))));
        v = (double)(float)w;
      }
      xw[d] = (float)v;
      double t = floor(__dmul_rn(__dsub_rn(v, b.lo[d]), b.scale));
      uint64_t q = t < 0.0 ? 0ull : (t > 2097151.0 ? 2097151ull : (uint64_t)t);
      key |= spread3(q) << d;
    }
    pos_tmp[i] = make_float4(xw[0], xw[1], xw[2], s[i]);
    keys[i] = key;
    idx[i] = (uint32_t)i;
  }
}

__global__ void k_gather(const float4* __restrict__ pos_tmp, const float* __restrict__ a,
                         const uint32_t* __restrict__ idx, int64_t n, float4* __restrict__ pos,
                         float4* __restrict__ alp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t j = idx[i];
    pos[i] = pos_tmp[j];
    alp[i] = make_float4(a[3 * (int64_t)j], a[3 * (int64_t)j + 1], a[3 * (int64_t)j + 2], 0.0f);
  }
}

struct CellPtrs {
  int *level, *qx, *qy, *qz, *begin, *count, *parent, *child_begin, *nchild, *leaf;
};
CellPtrs ptrs(Cells& c) {
  return {c.level.p, c.qx.p, c.qy.p, c.qz.p, c.begin.p, c.count.p, c.parent.p, c.child_begin.p, c.nchild.p, c.leaf.p};
}

__global__ void k_root(CellPtrs c, int64_t n, int ncrit) {
  c.level[0] = 0; c.qx[0] = c.qy[0] = c.qz[0] = 0;
  c.begin[0] = 0; c.count[0] = (int)n; c.parent[0] = -1;
  c.child_begin[0] = -1; c.nchild[0] = 0;
  c.leaf[0] = n <= ncrit ? 1 : 0;
}

__global__ void k_fill_int(int* p, int64_t n, int v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

// level l: a particle is active if its level-(l-1) cell exists and is not a
// leaf; a new cell starts where the level-l key prefix changes.
__global__ void k_level_flags(const uint64_t* __restrict__ keys, const int* __restrict__ pcell,
                              const int* __restrict__ leaf, int64_t n, int l, int* __restrict__ flag) {
  int sh = 3 * (kMaxLevel - l);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int pc = pcell[i];
    int act = pc >= 0 && !leaf[pc];
    int f = 0;
    if (act) {
      if (i == 0) f = 1;
      else {
        int pp = pcell[i - 1];
        f = (pp != pc) || ((keys[i] >> sh) != (keys[i - 1] >> sh));
      }
    }
    flag[i] = f;
  }
}

// scan = inclusive scan of flag; new cell of an active particle = base + scan - 1
__global__ void k_level_fill(const uint64_t* __restrict__ keys, const int* __restrict__ pcell,
                             const int* __restrict__ flag, const int* __restrict__ scan, CellPtrs c,
                             int64_t n, int l, int base, int* __restrict__ pcell_new) {
  int sh = 3 * (kMaxLevel - l);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int pc = pcell[i];
    int act = pc >= 0 && !c.leaf[pc];
    if (!act) { pcell_new[i] = -1; continue; }
    int cell = base + scan[i] - 1;
    pcell_new[i] = cell;
    if (flag[i]) {
      uint64_t pre = keys[i] >> sh;
      c.level[cell] = l;
      c.qx[cell] = compact3(pre);
      c.qy[cell] = compact3(pre >> 1);
      c.qz[cell] = compact3(pre >> 2);
      c.begin[cell] = (int)i;
      c.parent[cell] = pc;
      if ((int)i == c.begin[pc]) c.child_begin[pc] = cell;
      atomicAdd(&c.nchild[pc], 1);
    }
  }
}

__global__ void k_level_end(const int* __restrict__ pcell_new, CellPtrs c, int64_t n, int l, int ncrit) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int cell = pcell_new[i];
    if (cell < 0) continue;
    if (i == n - 1 || pcell_new[i + 1] != cell) {
      int cnt = (int)i + 1 - c.begin[cell];
      c.count[cell] = cnt;
      c.leaf[cell] = (cnt <= ncrit || l == kMaxLevel) ? 1 : 0;
      c.child_begin[cell] = -1;
      c.nchild[cell] = 0;
    }
  }
}

__global__ void k_leaf_flags(const int* __restrict__ leaf, int64_t nc, int* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = leaf[i];
}

__global__ void k_scatter_leaves(const int* __restrict__ leaf, const int* __restrict__ scan, int64_t nc,
                                 int* __restrict__ ids) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x)
    if (leaf[i]) ids[scan[i] - 1] = (int)i;
}

// local leaves (this rank's targets) and the traversal's target filter
__global__ void k_local_flags(const int* __restrict__ leaf, const int* __restrict__ begin,
                              const int* __restrict__ count, int64_t nc, int64_t off, int64_t n,
                              int* __restrict__ lflag, int* __restrict__ tgt_ok) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = begin[i], e = b + count[i];
    lflag[i] = (leaf[i] && b >= off && e <= off + n) ? 1 : 0;
    tgt_ok[i] = (b < off + n && e > off) ? 1 : 0;
  }
}

// per level: first and last cell overlapping [off, off + n) -- the cells whose
// multipoles (partial if they straddle a rank boundary) and locals this rank
// computes; the straddlers' partial multipoles are all-reduced (upward_pass)
__global__ void k_local_range(const int* __restrict__ level, const int* __restrict__ begin,
                              const int* __restrict__ count, int64_t nc, int64_t off, int64_t n,
                              int* __restrict__ lo, int* __restrict__ hi) {
  // cells are level-ordered, so a warp's cells span at most a few levels:
  // reduce within the warp per level before the atomics (one per warp and level
  // instead of one per cell)
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; i0 < nc;
       i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + lane;
    bool in = false;
    int lv = -1;
    if (i < nc) {
      const int64_t b = begin[i], e = b + count[i];
      in = b < off + n && e > off;
      lv = level[i];
    }
    unsigned todo = __ballot_sync(0xffffffffu, in);
    while (todo) {
      const int l = __shfl_sync(0xffffffffu, lv, __ffs(todo) - 1);
      const unsigned same = __ballot_sync(0xffffffffu, in && lv == l);
      if (lane == __ffs(same) - 1) {
        atomicMin(&lo[l], (int)(i0 + __ffs(same) - 1));
        atomicMax(&hi[l], (int)(i0 + 31 - __clz(same)));
      }
      todo &= ~same;
    }
  }
}

// ---- balanced partition (cfg.partition = 1, NEXT-3 / P:113-129) ----
struct Splits { int64_t o[9]; int P; };

__global__ void k_iota_u32(uint32_t* __restrict__ p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (uint32_t)i;
}

// this rank's block [g0, g0 + n) of the gathered keys -> global sorted positions
__global__ void k_ginv(const uint32_t* __restrict__ gsrc, int64_t N, int64_t g0, int64_t n, int* __restrict__ ginv) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < N; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = (int64_t)gsrc[g] - g0;
    if (j >= 0 && j < n) ginv[j] = (int)g;
  }
}

// split k (1 <= k < P): the leaf holding global position k N / P, rounded to
// its nearer boundary, so no leaf is cut (leaves in Morton order: the splits
// are non-decreasing).  out[0] = 0, out[P] = N.
__global__ void k_splits(const int* __restrict__ begin, const int* __restrict__ count,
                         const int* __restrict__ child_begin, const int* __restrict__ nchild,
                         const int* __restrict__ leaf, int64_t N, int P, int64_t* __restrict__ out) {
  const int k = threadIdx.x;
  if (k > P) return;
  if (k == 0 || k == P) { out[k] = k == 0 ? 0 : N; return; }
  const int64_t x = (int64_t)k * N / P;
  int cell = 0;
  while (!leaf[cell]) {
    const int cb = child_begin[cell], nc = nchild[cell];
    int next = cb + nc - 1;
    for (int q = 0; q < nc; ++q)
      if (x < (int64_t)begin[cb + q] + count[cb + q]) { next = cb + q; break; }
    cell = next;
  }
  const int64_t b = begin[cell], e = b + count[cell];
  out[k] = (x - b <= e - x) ? b : e;
}

__device__ __forceinline__ int split_owner(const Splits& s, int64_t g) {
  int q = 0;
  while (q + 1 < s.P && g >= s.o[q + 1]) ++q;
  return q;
}

__global__ void k_owner_count(const int* __restrict__ ginv, int64_t n, Splits s, int* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[split_owner(s, ginv[i])], 1);
}

// records in local sorted order (owners non-decreasing): (x, y, z, sigma), (alpha, global position)
__global__ void k_redist_pack(const int* __restrict__ ginv, const uint32_t* __restrict__ idx,
                              const float4* __restrict__ pos_tmp, const float* __restrict__ a, int64_t n,
                              float4* __restrict__ rec) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx[i];
    rec[2 * i] = pos_tmp[j];
    rec[2 * i + 1] = make_float4(a[3 * j], a[3 * j + 1], a[3 * j + 2], __int_as_float(ginv[i]));
  }
}

__global__ void k_redist_unpack(const float4* __restrict__ rec, int64_t m, float4* __restrict__ pos,
                                float4* __restrict__ alp, int* __restrict__ recv_gp) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    const float4 al = rec[2 * k + 1];
    const int g = __float_as_int(al.w);
    pos[g] = rec[2 * k];
    alp[g] = make_float4(al.x, al.y, al.z, 0.0f);
    recv_gp[k] = g;
  }
}

// cells of level >= 2 with a split strictly inside their particle range
__global__ void k_strad(const int* __restrict__ begin, const int* __restrict__ count, int64_t c0, int64_t nc, Splits s,
                        int* __restrict__ list, int* __restrict__ cnt) {
  for (int64_t i = c0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = begin[i], e = b + count[i];
    bool st = false;
    for (int k = 1; k < s.P; ++k) st |= (b < s.o[k] && s.o[k] < e);
    if (st) list[atomicAdd(cnt, 1)] = (int)i;
  }
}

template <typename F>
void cub_call(Ctx& c, F f) {
  size_t bytes = 0;
  FMM_CUDA(f((void*)nullptr, bytes));
  c.cub_tmp.reserve(bytes);
  FMM_CUDA(f((void*)c.cub_tmp.p, bytes));
  ++c.cub_calls;
}

}  // namespace

static unsigned grid_for(int64_t n) {
  unsigned b = nblocks(n, 256);
  return b > 148 * 16 ? 148 * 16 : b;
}

// Balanced partition, after the global tree is built (every rank holds the
// same global key order and octree): cut the Morton curve into nranks
// equal-count ranges moved to the nearest leaf boundary, send every local
// particle to its owner (grouped ncclSend/ncclRecv) and scatter the received
// ones into the global-position arrays.  Cells that hold a split point (levels
// >= 2) are recorded: their multipoles are sums of per-rank partials.
static void balanced_redistribute(Ctx& c, int64_t n, const float* a, const std::vector<int64_t>& goff) {
  cudaStream_t st = c.stream;
  const int P = c.cfg.nranks, R = c.cfg.rank;
  const int64_t N = c.ntot;
  c.req_off.reserve(P + 1);
  FMM_LAUNCH(c, k_splits, 1, 32, 0, c.cells.begin.p, c.cells.count.p, c.cells.child_begin.p, c.cells.nchild.p,
             c.cells.leaf.p, N, P, c.req_off.p);
  c.rank_off.assign(P + 1, 0);
  FMM_CUDA(cudaMemcpyAsync(c.rank_off.data(), c.req_off.p, sizeof(int64_t) * (P + 1), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  c.off = c.rank_off[R];
  c.nown = c.rank_off[R + 1] - c.rank_off[R];
  Splits sp{};
  sp.P = P;
  for (int q = 0; q <= P; ++q) sp.o[q] = c.rank_off[q];
  // owners of the local particles and the per-peer record counts
  c.ginv.reserve(std::max<int64_t>(n, 1));
  c.dflag.reserve(std::max(8, P));
  FMM_CUDA(cudaMemsetAsync(c.dflag.p, 0, sizeof(int) * P, st));
  if (n > 0) {
    FMM_LAUNCH(c, k_ginv, grid_for(N), 256, 0, c.gsrc.p, N, goff[R], n, c.ginv.p);
    FMM_LAUNCH(c, k_owner_count, grid_for(n), 256, 0, c.ginv.p, n, sp, c.dflag.p);
  }
  std::vector<int> sc(P);
  FMM_CUDA(cudaMemcpyAsync(sc.data(), c.dflag.p, sizeof(int) * P, cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  c.red_scnt.assign(P, 0);
  for (int q = 0; q < P; ++q) c.red_scnt[q] = sc[q];
  c.red_rcnt = alltoall_i64(c, c.red_scnt);
  int64_t nrecv = 0;
  for (int q = 0; q < P; ++q) nrecv += c.red_rcnt[q];
  if (nrecv != c.nown) throw FmmError(FMM_E_INTERNAL, "balanced partition: received particle count mismatch");
  // records (32 B each) in local sorted order = grouped by owner
  c.red_send.reserve(2 * std::max<int64_t>(n, 1));
  c.red_recv.reserve(2 * std::max<int64_t>(c.nown, 1));
  c.recv_gp.reserve(std::max<int64_t>(c.nown, 1));
  if (n > 0) FMM_LAUNCH(c, k_redist_pack, grid_for(n), 256, 0, c.ginv.p, c.idx.p, c.pos_tmp.p, a, n, c.red_send.p);
  std::vector<int64_t> soff(P, 0), sb(P, 0), roff(P, 0), rb(P, 0);
  int64_t so = 0, ro = 0;
  for (int q = 0; q < P; ++q) {
    soff[q] = 32 * so;
    roff[q] = 32 * ro;
    sb[q] = q == R ? 0 : 32 * c.red_scnt[q];
    rb[q] = q == R ? 0 : 32 * c.red_rcnt[q];
    so += c.red_scnt[q];
    ro += c.red_rcnt[q];
  }
  if (c.red_scnt[R] > 0)
    FMM_CUDA(cudaMemcpyAsync((char*)c.red_recv.p + roff[R], (const char*)c.red_send.p + soff[R], 32 * c.red_scnt[R],
                             cudaMemcpyDeviceToDevice, st));
  alltoallv_bytes(c, c.red_send.p, soff, sb, c.red_recv.p, roff, rb);
  c.redist_bytes = 32 * (n - c.red_scnt[R]);
  if (c.nown > 0)
    FMM_LAUNCH(c, k_redist_unpack, grid_for(c.nown), 256, 0, c.red_recv.p, c.nown, c.pos.p, c.alp.p, c.recv_gp.p);
  // straddling cells (levels >= 2; levels 0-1 are all-reduced as a whole)
  const int64_t c0 = c.level_begin.size() > 2 ? c.level_begin[2] : c.ncells;
  c.strad.reserve(64 * P + 1);
  FMM_CUDA(cudaMemsetAsync(c.dflag.p, 0, sizeof(int), st));
  if (c.ncells > c0)
    FMM_LAUNCH(c, k_strad, grid_for(c.ncells - c0), 256, 0, c.cells.begin.p, c.cells.count.p, c0, c.ncells, sp,
               c.strad.p, c.dflag.p);
  int ns = 0;
  FMM_CUDA(cudaMemcpyAsync(&ns, c.dflag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  if (ns > 64 * P) throw FmmError(FMM_E_INTERNAL, "balanced partition: too many straddling cells");
  std::vector<int> ids(ns);
  if (ns) FMM_CUDA(cudaMemcpyAsync(ids.data(), c.strad.p, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  std::sort(ids.begin(), ids.end());                 // same order on every rank (all-reduce layout)
  if (ns) FMM_CUDA(cudaMemcpyAsync(c.strad.p, ids.data(), sizeof(int) * ns, cudaMemcpyHostToDevice, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  c.nstrad = ns;
}

void set_particles_impl(Ctx& c, int64_t n, const float* x, const float* a, const float* s) {
  cudaStream_t st = c.stream;
  c.n = n;
  c.launches = 0;
  c.cub_calls = 0;
  c.have_particles = false;
  c.lists_valid = false;
  c.evaluated = false;
  c.ncells = 0;
  c.nleaves = 0;
  c.level_begin.assign(1, 0);
  FMM_CUDA(cudaEventRecord(c.ev[PH_SET0], st));

  // a1: validation (+ bounding box for free space, Z16)
  c.dflag.reserve(8);
  int init[8] = {0, INT_MAX, INT_MAX, INT_MAX, INT_MIN, INT_MIN, INT_MIN, 0};
  FMM_CUDA(cudaMemcpyAsync(c.dflag.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
  int periodic = c.cfg.images > 0;
  if (n > 0) {
    FMM_LAUNCH(c, k_validate, grid_for(n), 256, 0, x, a, s, n, c.dflag.p, !periodic);
    FMM_LAUNCH_CHECK();
  }
  int h[8];
  FMM_CUDA(cudaMemcpyAsync(h, c.dflag.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  if (h[0] & 1) throw FmmError(FMM_E_NONFINITE, "non-finite x, alpha or sigma");
  if (h[0] & 2) throw FmmError(FMM_E_SIGMA, "sigma <= 0");

  Box b{};
  b.periodic = periodic;
  if (periodic) {
    for (int d = 0; d < 3; ++d) { b.lo[d] = c.cfg.box_lo[d]; b.per[d] = c.per[d]; }
    b.L = c.cfg.box_len * c.tmax;
  } else if (n > 0) {
    double ext = 0;
    for (int d = 0; d < 3; ++d) {
      double mn = (double)fkey_inv(h[1 + d]), mx = (double)fkey_inv(h[4 + d]);
      b.lo[d] = mn;
      if (mx - mn > ext) ext = mx - mn;
    }
    b.L = ext > 0 ? ext * (1.0 + 0x1p-20) : 1.0;
  } else {
    b.L = 1.0;
  }
  b.scale = 2097152.0 / b.L;
  for (int d = 0; d < 3; ++d) c.lo[d] = b.lo[d];
  c.L = b.L;

  if (n == 0 && c.cfg.nranks == 1) {
    c.ntot = 0;
    c.off = 0;
    c.rank_off.assign(2, 0);
    FMM_CUDA(cudaEventRecord(c.ev[PH_KEYS], st));
    FMM_CUDA(cudaEventRecord(c.ev[PH_SORT], st));
    FMM_CUDA(cudaEventRecord(c.ev[PH_TREE], st));
    c.have_particles = true;
    return;
  }

  // a2: keys
  const int P = c.cfg.nranks, R = c.cfg.rank;
  const bool multi = P > 1;
  c.balanced = multi && c.cfg.partition == 1;
  c.redist_bytes = 0;
  std::vector<int64_t> goff(P + 1, 0);        // balanced: the ranks' blocks of the gathered keys
  c.pos_tmp.reserve(n); c.keys_tmp.reserve(n); c.idx_tmp.reserve(n); c.idx.reserve(n);
  FMM_LAUNCH(c, k_keys, grid_for(n), 256, 0, x, s, n, b, c.pos_tmp.p, c.keys_tmp.p, c.idx_tmp.p);
  FMM_CUDA(cudaEventRecord(c.ev[PH_KEYS], st));

  // a3: stable LSD radix sort on the 63 key bits
  uint64_t* ksorted;
  if (multi) { c.keys_loc.reserve(n); ksorted = c.keys_loc.p; }
  else { c.keys.reserve(n); ksorted = c.keys.p; }
  if (n > 0) {
    uint64_t *kin = c.keys_tmp.p, *kout = ksorted;
    uint32_t *vin = c.idx_tmp.p, *vout = c.idx.p;
    int nn = (int)n;
    cub_call(c, [&](void* tmp, size_t& bytes) {
      return cub::DeviceRadixSort::SortPairs(tmp, bytes, kin, kout, vin, vout, nn, 0, 63, st);
    });
  }
  // a14: global key order = the ranks' sorted keys concatenated in rank order
  // (each rank owns a contiguous Morton range: octants [8R/P, 8(R+1)/P))
  c.rank_off.assign(P + 1, 0);
  if (c.balanced) {
    // every rank's sorted keys gathered (rank blocks), then one stable global
    // sort: ties keep (rank, local order), so each rank's particles appear in
    // its local sorted order.  The owners are decided after the tree (below).
    std::vector<int64_t> cnt = allgather_i64(c, n);
    for (int q = 0; q < P; ++q) goff[q + 1] = goff[q] + cnt[q];
    const int64_t NT = goff[P];
    if (NT >= (1ll << 31)) throw FmmError(FMM_E_ARG, "more than 2^31 particles in total");
    c.keys_gat.reserve(std::max<int64_t>(NT, 1));
    if (n > 0) FMM_CUDA(cudaMemcpyAsync(c.keys_gat.p + goff[R], ksorted, 8 * n, cudaMemcpyDeviceToDevice, st));
    std::vector<int64_t> soff(P, 0), sb(P, 0), roff(P, 0), rb(P, 0);
    for (int q = 0; q < P; ++q) {
      if (q == R) continue;
      sb[q] = 8 * n;
      roff[q] = 8 * goff[q];
      rb[q] = 8 * cnt[q];
    }
    alltoallv_bytes(c, ksorted, soff, sb, c.keys_gat.p, roff, rb);
    c.ntot = NT;
    c.keys.reserve(std::max<int64_t>(NT, 1));
    c.gsrc.reserve(std::max<int64_t>(NT, 1));
    c.gsrc_tmp.reserve(std::max<int64_t>(NT, 1));
    if (NT > 0) {
      FMM_LAUNCH(c, k_iota_u32, grid_for(NT), 256, 0, c.gsrc_tmp.p, NT);
      uint64_t *kin = c.keys_gat.p, *kout = c.keys.p;
      uint32_t *vin = c.gsrc_tmp.p, *vout = c.gsrc.p;
      int nn = (int)NT;
      cub_call(c, [&](void* tmp, size_t& bytes) {
        return cub::DeviceRadixSort::SortPairs(tmp, bytes, kin, kout, vin, vout, nn, 0, 63, st);
      });
    }
  } else if (multi) {
    if (n > 0) {
      uint64_t kk[2];
      FMM_CUDA(cudaMemcpyAsync(&kk[0], ksorted, 8, cudaMemcpyDeviceToHost, st));
      FMM_CUDA(cudaMemcpyAsync(&kk[1], ksorted + n - 1, 8, cudaMemcpyDeviceToHost, st));
      FMM_CUDA(cudaStreamSynchronize(st));
      const int o0 = (int)(kk[0] >> 60), o1 = (int)(kk[1] >> 60);
      // refined mode: octants [8r/P, 8(r+1)/P); tiled mode (Z27): octant r = tile r
      const int olo = c.tmax > 1 ? R : 8 * R / P, ohi = c.tmax > 1 ? R + 1 : 8 * (R + 1) / P;
      if (o0 < olo || o1 >= ohi)
        throw FmmError(FMM_E_ARG, "rank holds particles outside its Morton range (top octants it owns)");
    }
    std::vector<int64_t> cnt = allgather_i64(c, n);
    for (int q = 0; q < P; ++q) c.rank_off[q + 1] = c.rank_off[q] + cnt[q];
    c.ntot = c.rank_off[P];
    c.off = c.rank_off[R];
    c.keys.reserve(c.ntot);
    if (n > 0) FMM_CUDA(cudaMemcpyAsync(c.keys.p + c.off, ksorted, 8 * n, cudaMemcpyDeviceToDevice, st));
    std::vector<int64_t> soff(P, 0), sb(P, 0), roff(P, 0), rb(P, 0);
    for (int q = 0; q < P; ++q) {
      if (q == R) continue;
      sb[q] = 8 * n;
      roff[q] = 8 * c.rank_off[q];
      rb[q] = 8 * cnt[q];
    }
    alltoallv_bytes(c, ksorted, soff, sb, c.keys.p, roff, rb);
  } else {
    c.ntot = n;
    c.off = 0;
    c.rank_off[1] = n;
  }
  const int64_t N = c.ntot;
  c.pos.reserve(N); c.alp.reserve(N);
  c.nown = n;
  if (n > 0 && !c.balanced) FMM_LAUNCH(c, k_gather, grid_for(n), 256, 0, c.pos_tmp.p, a, c.idx.p, n, c.pos.p + c.off, c.alp.p + c.off);
  FMM_CUDA(cudaEventRecord(c.ev[PH_SORT], st));
  if (N == 0) {
    FMM_CUDA(cudaEventRecord(c.ev[PH_TREE], st));
    FMM_CUDA(cudaStreamSynchronize(st));
    c.have_particles = true;
    return;
  }

  // a4: cells level by level
  size_t capc = (size_t)(2 * (N / (c.cfg.ncrit + 1)) + 64);
  c.cells.reserve_keep(capc, 0, st);
  c.pcell_a.reserve(N); c.pcell_b.reserve(N); c.flags.reserve(N); c.scan.reserve(N);
  FMM_LAUNCH(c, k_root, 1, 1, 0, ptrs(c.cells), N, c.cfg.ncrit);
  FMM_LAUNCH(c, k_fill_int, grid_for(N), 256, 0, c.pcell_a.p, N, 0);
  FMM_LAUNCH_CHECK();
  int64_t ncells = 1;
  c.level_begin.assign({0, 1});
  int* pc_old = c.pcell_a.p;
  int* pc_new = c.pcell_b.p;
  for (int l = 1; l <= kMaxLevel; ++l) {
    FMM_LAUNCH(c, k_level_flags, grid_for(N), 256, 0, c.keys.p, pc_old, c.cells.leaf.p, N, l, c.flags.p);
    FMM_LAUNCH_CHECK();
    {
      int* fin = c.flags.p;
      int* fout = c.scan.p;
      int nn = (int)N;
      cub_call(c, [&](void* tmp, size_t& bytes) {
        return cub::DeviceScan::InclusiveSum(tmp, bytes, fin, fout, nn, st);
      });
    }
    int total = 0;
    FMM_CUDA(cudaMemcpyAsync(&total, c.scan.p + (N - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaStreamSynchronize(st));
    if (total == 0) break;
    if ((size_t)(ncells + total) > c.cells.level.cap) c.cells.reserve_keep((size_t)(ncells + total) * 2, ncells, st);
    FMM_LAUNCH(c, k_level_fill, grid_for(N), 256, 0, c.keys.p, pc_old, c.flags.p, c.scan.p, ptrs(c.cells), N, l,
                                              (int)ncells, pc_new);
    FMM_LAUNCH(c, k_level_end, grid_for(N), 256, 0, pc_new, ptrs(c.cells), N, l, c.cfg.ncrit);
    FMM_LAUNCH_CHECK();
    ncells += total;
    c.level_begin.push_back(ncells);
    int* t = pc_old; pc_old = pc_new; pc_new = t;
  }
  c.ncells = ncells;
  if (ncells >= (1ll << 27)) throw FmmError(FMM_E_ARG, "more than 2^27 cells; raise ncrit");
  if (c.balanced) balanced_redistribute(c, n, a, goff);

  // local leaf list (this rank's targets), traversal filter, per-level local cell ranges
  c.leaf_ids.reserve(ncells);
  c.tgt_ok.reserve(ncells);
  FMM_LAUNCH(c, k_local_flags, grid_for(ncells), 256, 0, c.cells.leaf.p, c.cells.begin.p, c.cells.count.p, ncells,
             c.off, c.nown, c.flags.p, c.tgt_ok.p);
  {
    int* fin = c.flags.p;
    int* fout = c.scan.p;
    int nn = (int)ncells;
    cub_call(c, [&](void* tmp, size_t& bytes) {
      return cub::DeviceScan::InclusiveSum(tmp, bytes, fin, fout, nn, st);
    });
  }
  FMM_LAUNCH(c, k_scatter_leaves, grid_for(ncells), 256, 0, c.flags.p, c.scan.p, ncells, c.leaf_ids.p);
  const int nlev = (int)c.level_begin.size() - 1;
  {
    std::vector<int> init(2 * (kMaxLevel + 1));
    for (int l = 0; l <= kMaxLevel; ++l) { init[l] = INT_MAX; init[kMaxLevel + 1 + l] = -1; }
    c.need.reserve(2 * (kMaxLevel + 1));
    FMM_CUDA(cudaMemcpyAsync(c.need.p, init.data(), sizeof(int) * init.size(), cudaMemcpyHostToDevice, st));
    FMM_LAUNCH(c, k_local_range, grid_for(ncells), 256, 0, c.cells.level.p, c.cells.begin.p, c.cells.count.p, ncells,
               c.off, c.nown, c.need.p, c.need.p + kMaxLevel + 1);
    FMM_CUDA(cudaMemcpyAsync(init.data(), c.need.p, sizeof(int) * init.size(), cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaStreamSynchronize(st));
    c.loc_lo.assign(nlev, 0);
    c.loc_hi.assign(nlev, 0);
    for (int l = 0; l < nlev; ++l) {
      if (init[kMaxLevel + 1 + l] >= 0) { c.loc_lo[l] = init[l]; c.loc_hi[l] = init[kMaxLevel + 1 + l] + 1; }
      else { c.loc_lo[l] = c.loc_hi[l] = c.level_begin[l]; }
    }
  }
  int nl = 0;
  FMM_CUDA(cudaMemcpyAsync(&nl, c.scan.p + (ncells - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
  const int ltop = 2 + (c.tmax == 2 ? 1 : 0);   // far-field target level (side box_len / 4)
  int64_t ntop = (int)c.level_begin.size() > ltop ? c.level_begin[ltop] : ncells;
  c.host_leaf_top.resize(ntop);
  FMM_CUDA(cudaMemcpyAsync(c.host_leaf_top.data(), c.cells.leaf.p, sizeof(int) * ntop, cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaEventRecord(c.ev[PH_TREE], st));
  FMM_CUDA(cudaStreamSynchronize(st));
  c.nleaves = nl;
  c.have_particles = true;
}

}  // namespace fmmb
