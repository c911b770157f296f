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

// a2-a4 on this rank's n particles (caller order): keys, stable sort, gather
// and the octree, level by level; cells [0, ncells) in canonical (level, key)
// order.  On several GPUs this is the local tree of the LET forest (let.cu).
static void build_local_tree(Ctx& c, int64_t n, const float* x, const float* a, const float* s, const Box& b) {
  cudaStream_t st = c.stream;
  c.pos_tmp.reserve(n); c.keys_tmp.reserve(n); c.idx_tmp.reserve(n); c.idx.reserve(n); c.keys.reserve(n);
  FMM_LAUNCH(c, k_keys, grid_for(n), 256, 0, x, s, n, b, c.pos_tmp.p, c.keys_tmp.p, c.idx_tmp.p);
  FMM_CUDA(cudaEventRecord(c.ev[PH_KEYS], st));
  // a3: stable LSD radix sort on the 63 key bits
  if (n > 0) {
    uint64_t *kin = c.keys_tmp.p, *kout = c.keys.p;
    uint32_t *vin = c.idx_tmp.p, *vout = c.idx.p;
    int nn = (int)n;
    cub_call(c, [&](void* tmp, size_t& bytes) {
      return cub::DeviceRadixSort::SortPairs(tmp, bytes, kin, kout, vin, vout, nn, 0, 63, st);
    });
  }
  c.pos.reserve(n); c.alp.reserve(n);
  if (n > 0) FMM_LAUNCH(c, k_gather, grid_for(n), 256, 0, c.pos_tmp.p, a, c.idx.p, n, c.pos.p, c.alp.p);
  FMM_CUDA(cudaEventRecord(c.ev[PH_SORT], st));
  const int64_t N = n;
  c.ncells = c.nloc_cells = 0;
  c.nleaves = 0;
  c.level_begin.assign(1, 0);
  c.host_leaf_top.clear();
  if (N == 0) return;

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
  c.ncells = c.nloc_cells = ncells;
  if (ncells >= (1ll << 27)) throw FmmError(FMM_E_ARG, "more than 2^27 cells; raise ncrit");

  // leaf list (the targets), per-level cell ranges
  c.leaf_ids.reserve(ncells);
  FMM_LAUNCH(c, k_leaf_flags, grid_for(ncells), 256, 0, c.cells.leaf.p, ncells, c.flags.p);
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
  c.loc_lo.assign(nlev, 0);
  c.loc_hi.assign(nlev, 0);
  for (int l = 0; l < nlev; ++l) { c.loc_lo[l] = c.level_begin[l]; c.loc_hi[l] = c.level_begin[l + 1]; }
  int nl = 0;
  FMM_CUDA(cudaMemcpyAsync(&nl, c.scan.p + (ncells - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
  const int ltop = 2 + (c.tmax == 2 ? 1 : 0);   // far-field target level (side box_len / 4)
  int64_t ntop = (int)c.level_begin.size() > ltop ? c.level_begin[ltop] : ncells;
  c.host_leaf_top.resize(ntop);
  FMM_CUDA(cudaMemcpyAsync(c.host_leaf_top.data(), c.cells.leaf.p, sizeof(int) * ntop, cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  c.nleaves = nl;
}

void set_particles_impl(Ctx& c, int64_t n, const float* x, const float* a, const float* s) {
  cudaStream_t st = c.stream;
  c.n = n;
  c.launches = 0;
  c.cub_calls = 0;
  c.have_particles = false;
  c.lists_valid = false;
  c.evaluated = false;
  c.ncells = c.nloc_cells = 0;
  c.nleaves = 0;
  c.nsrc = 0;
  c.leaf_cls_valid = false;
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

  const int P = c.cfg.nranks;
  const bool multi = P > 1;
  c.balanced = multi && c.cfg.partition >= 1;
  c.redist_bytes = 0;
  c.n_caller = n;
  if (c.balanced) {
    // NEXT-3: ORB multisection of the wrapped positions, then every particle to its owner
    c.pos_tmp.reserve(n); c.keys_tmp.reserve(n); c.idx_tmp.reserve(n);
    if (n > 0) FMM_LAUNCH(c, k_keys, grid_for(n), 256, 0, x, s, n, b, c.pos_tmp.p, c.keys_tmp.p, c.idx_tmp.p);
    orb_redistribute(c, n, x, a, s, c.pos_tmp.p);
    n = c.n_own;
    x = c.px.p;
    a = c.pa.p;
    s = c.ps.p;
    c.n = n;
  }
  c.nown = n;
  build_local_tree(c, n, x, a, s, b);
  if (multi) {
    std::vector<int64_t> all = allgather_i64(c, n);
    c.ntot = 0;
    for (int64_t v : all) c.ntot += v;
    let_setup(c);           // a14: the LET of every peer, merged into the cell table as a forest
  } else {
    c.ntot = n;
    c.nsrc = n;
  }
  c.off = 0;
  FMM_CUDA(cudaEventRecord(c.ev[PH_TREE], st));
  FMM_CUDA(cudaStreamSynchronize(st));
  c.have_particles = true;
}

}  // namespace fmmb
