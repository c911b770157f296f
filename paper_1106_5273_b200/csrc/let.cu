// let.cu -- a14: the local essential tree on B200s.
//
// Every rank builds the octree of its own particles only (the same Morton
// cells of the common root box, so no global index is needed), and
// sends every other rank the part of that tree the other rank's traversal can
// reach -- its LET -- chosen by the sender alone with a conservative LET-MAC
// against the receiver's domain (the bounding box of its particles):
//
//   accept B (send its multipole, do not open it) iff
//       (1 + theta) max(2 r_B, rleaf_q) + r_B < theta d_B,
//       d_B = min over the first-layer images of |c_B + shift - box_q|.
//
// Reading Z25: the paper assumes the target cell has the source's
// size (r_A = r_B) and its centre on the box edge.  The receiver's traversal
// (Alg. 1, split the larger cell) only meets B against targets with r_A <= 2 r_B
// unless the target is a leaf, and a target cell's centre can lie up to r_A
// outside the box of its particles, so its MAC r_A + r_B < theta R_AB holds
// whenever (1 + theta) 2 r_B + r_B < theta d_B -- the test above.  Larger leaf
// targets (adaptive trees: the receiver's leaves near this rank's domain are
// coarser than this rank's cells) are covered by replacing 2 r_B with
// max(2 r_B, rleaf_q), the radius of the largest leaf of q that can meet a
// cell of this rank (k_leaf_reach; one int per pair of ranks).  Leaves are
// sent with their bodies unless accepted (MAC-first) or always (leaf-first,
// where leaf pairs are P2P before any MAC).  The receiver's traversal counts
// every pair it cannot resolve with what it received (Alg. 2's remote branch,
// "M2L with the smallest cell that is available"): zero
// for the uniform trees of C4/C5 (checked by the multi-GPU tests).
//
// set_particles: the walk (level-synchronous count/scan/write rounds over
// (cell, receiver) items, like the traversal), one stable 3-bit radix sort
// into receiver-major order, the 40-byte cell records (geometry, count,
// flags, parent/child links within the record list, body offsets) exchanged
// with grouped ncclSend/ncclRecv, and the received records appended to the
// local cell table as further trees of a forest: local cells keep ids
// [0, nloc), tree t's records take [nloc + base_t, ...), its bodies the
// particle slots [n + bbase_t, ...).
// evaluate: the multipoles of the sent cells and the sent bodies are gathered
// and exchanged on the communication stream while the local near field runs
// (fig:flow_chart); NCCL receives them straight into the M and particle
// arrays (one contiguous block per sender).
#include <algorithm>
#include <climits>
#include <cstring>

#include <cub/cub.cuh>

#include "ctx.cuh"

namespace fmmb {

namespace {

enum { D_FRONTIER = 1, D_OPEN = 2, D_BODIES = 3, D_MONLY = 4 };

struct LetCells {
  const int *level, *qx, *qy, *qz, *leaf, *child_begin, *nchild, *count, *parent;
};

struct LetGeo {
  double lo[3], L, per[3];
  double theta;
  int leaf_first;
  double blo[8][3], bhi[8][3];
  double rleaf[8];        // receiver q: largest radius of its leaves that can meet cells of this rank (k_leaf_reach)
};

// record sent to the receiver: geometry, count, flags and links within the list
struct LetRec {
  int level, qx, qy, qz, count, flags, parent, child, nchild, body_off;
};
enum { F_LEAF = 1, F_FRONTIER = 2, F_BODIES = 4 };

__device__ __forceinline__ double box_dist2(const double c[3], const LetGeo& g, int q) {
  double d2 = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double v = c[a] < g.blo[q][a] ? g.blo[q][a] - c[a] : (c[a] > g.bhi[q][a] ? c[a] - g.bhi[q][a] : 0.0);
    d2 += v * v;
  }
  return d2;
}

// LET-MAC decision for item (cell, receiver q)
__global__ void k_let_count(const uint64_t* __restrict__ front, int64_t nf, LetCells c, LetGeo g,
                            int* __restrict__ nch, unsigned char* __restrict__ dec) {
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= nf) return;
  const uint64_t it = front[f];
  const int cell = (int)(it >> 4), q = (int)(it & 15);
  const int l = c.level[cell];
  const double s = g.L / (double)(1 << l);
  const double ctr[3] = {g.lo[0] + (c.qx[cell] + 0.5) * s, g.lo[1] + (c.qy[cell] + 0.5) * s,
                         g.lo[2] + (c.qz[cell] + 0.5) * s};
  double dmin2 = 1e300;
  for (int img = 0; img < 27; ++img) {
    const double sh[3] = {(img % 3 - 1) * g.per[0], ((img / 3) % 3 - 1) * g.per[1], (img / 9 - 1) * g.per[2]};
    const double cc[3] = {ctr[0] + sh[0], ctr[1] + sh[1], ctr[2] + sh[2]};
    dmin2 = fmin(dmin2, box_dist2(cc, g, q));
  }
  const double r = 0.8660254037844386 * s;
  const double ra = fmax(2.0 * r, g.rleaf[q]);              // the largest target B can meet there
  const double lhs = ((1.0 + g.theta) * ra + r) / g.theta * (1.0 + 1e-9);
  const bool acc = lhs * lhs < dmin2;
  int d, k = 0;
  if (c.leaf[cell]) d = (g.leaf_first || !acc) ? D_BODIES : D_MONLY;
  else if (acc) d = D_FRONTIER;
  else { d = D_OPEN; k = c.nchild[cell]; }
  dec[f] = (unsigned char)d;
  nch[f] = k;
}

// the largest radius of this rank's leaves that can be paired with a smaller
// cell B (r_B < r_A / 2) of rank q's domain: only a leaf target keeps meeting
// ever smaller sources (Alg. 1 never splits a leaf), and it fails the MAC with
// B only if R < (r_A + r_B)/theta, with R >= d(c_A, box_q) - r_B; so leaves
// with d(c_A, box_q) < (1.5/theta + 0.5) r_A count (first-layer images included)
__global__ void k_leaf_reach(const int* __restrict__ leaf_ids, int64_t nl, LetCells c, LetGeo g, int P, int R,
                             unsigned* __restrict__ rmax) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nl; k += (int64_t)gridDim.x * blockDim.x) {
    const int cell = leaf_ids[k];
    const int l = c.level[cell];
    const double s = g.L / (double)(1 << l);
    const double ctr[3] = {g.lo[0] + (c.qx[cell] + 0.5) * s, g.lo[1] + (c.qy[cell] + 0.5) * s,
                           g.lo[2] + (c.qz[cell] + 0.5) * s};
    const double r = 0.8660254037844386 * s, reach = (1.5 / g.theta + 0.5) * r * (1.0 + 1e-9);
    for (int q = 0; q < P; ++q) {
      if (q == R) continue;
      double dmin2 = 1e300;
      for (int img = 0; img < 27; ++img) {
        const double cc[3] = {ctr[0] + (img % 3 - 1) * g.per[0], ctr[1] + ((img / 3) % 3 - 1) * g.per[1],
                              ctr[2] + (img / 9 - 1) * g.per[2]};
        dmin2 = fmin(dmin2, box_dist2(cc, g, q));
      }
      if (dmin2 < reach * reach) atomicMax(&rmax[q], __float_as_uint((float)(r * (1.0 + 1e-6))));
    }
  }
}

// records (receiver << 40 | decision << 32 | cell) and the next level's items
__global__ void k_let_write(const uint64_t* __restrict__ front, int64_t nf, LetCells c,
                            const unsigned char* __restrict__ dec, const int* __restrict__ off,
                            uint64_t* __restrict__ next, uint64_t* __restrict__ rec) {
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= nf) return;
  const uint64_t it = front[f];
  const int cell = (int)(it >> 4), q = (int)(it & 15);
  rec[f] = ((uint64_t)q << 40) | ((uint64_t)dec[f] << 32) | (uint64_t)cell;
  if (dec[f] == D_OPEN) {
    const int cb = c.child_begin[cell], nc = c.nchild[cell];
    for (int k = 0; k < nc; ++k) next[off[f] + k] = ((uint64_t)(cb + k) << 4) | (uint64_t)q;
  }
}

struct QTab { int64_t start[9]; int64_t bbase[9]; int P; };

__global__ void k_let_hist(const uint64_t* __restrict__ rec, int64_t nr, int* __restrict__ cnt) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nr; k += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[(int)(rec[k] >> 40)], 1);
}

// order-preserving float <-> int map for atomicMin/atomicMax
__device__ __forceinline__ int fkey(float f) {
  int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}

__global__ void k_bbox(const float4* __restrict__ pos, int64_t n, int* __restrict__ out) {
  int mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {INT_MIN, INT_MIN, INT_MIN};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 p = pos[i];
    const float v[3] = {p.x, p.y, p.z};
    for (int d = 0; d < 3; ++d) { mn[d] = min(mn[d], fkey(v[d])); mx[d] = max(mx[d], fkey(v[d])); }
  }
  for (int o = 16; o > 0; o >>= 1)
    for (int d = 0; d < 3; ++d) {
      mn[d] = min(mn[d], __shfl_xor_sync(0xffffffffu, mn[d], o));
      mx[d] = max(mx[d], __shfl_xor_sync(0xffffffffu, mx[d], o));
    }
  if ((threadIdx.x & 31) == 0)
    for (int d = 0; d < 3; ++d) { atomicMin(&out[d], mn[d]); atomicMax(&out[3 + d], mx[d]); }
}

__global__ void k_let_recof(const uint64_t* __restrict__ rec, int64_t nr, QTab t, int64_t nloc, int* __restrict__ recof) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nr; k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = rec[k];
    const int q = (int)(r >> 40), cell = (int)(r & 0xffffffffull);
    recof[(int64_t)q * nloc + cell] = (int)(k - t.start[q]);
  }
}

__global__ void k_let_bodycount(const uint64_t* __restrict__ rec, int64_t nr, const int* __restrict__ count,
                                int64_t* __restrict__ bc) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nr; k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = rec[k];
    const int d = (int)((r >> 32) & 255), cell = (int)(r & 0xffffffffull);
    bc[k] = d == D_BODIES ? count[cell] : 0;
  }
}

__global__ void k_let_records(const uint64_t* __restrict__ rec, int64_t nr, LetCells c, QTab t, int64_t nloc,
                              const int* __restrict__ recof, const int64_t* __restrict__ boff,
                              LetRec* __restrict__ out, int* __restrict__ scell) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nr; k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = rec[k];
    const int q = (int)(r >> 40), d = (int)((r >> 32) & 255), cell = (int)(r & 0xffffffffull);
    const int* ro = recof + (int64_t)q * nloc;
    LetRec o;
    o.level = c.level[cell];
    o.qx = c.qx[cell];
    o.qy = c.qy[cell];
    o.qz = c.qz[cell];
    o.count = c.count[cell];
    o.flags = (d == D_BODIES || d == D_MONLY ? F_LEAF : 0) | (d == D_FRONTIER ? F_FRONTIER : 0) |
              (d == D_BODIES ? F_BODIES : 0);
    o.parent = cell == 0 ? -1 : ro[c.parent[cell]];
    o.child = d == D_OPEN ? ro[c.child_begin[cell]] : -1;
    o.nchild = d == D_OPEN ? c.nchild[cell] : 0;
    o.body_off = (int)(boff[k] - t.bbase[q]);
    out[k] = o;
    scell[k] = cell;
  }
}

// the body records (receiver-major): local cell and global offset in the body send buffer
struct IsBodies {
  const uint64_t* rec;
  __device__ __forceinline__ bool operator()(const int64_t& k) const { return ((rec[k] >> 32) & 255) == D_BODIES; }
};

__global__ void k_iota64(int64_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = i;
}

// receiver: the peers' records appended to the cell table as trees of a forest
struct RTab { int64_t start[9]; int64_t cbase[9]; int64_t bbase[9]; int np; };

struct MCells {
  int *level, *qx, *qy, *qz, *begin, *count, *parent, *child_begin, *nchild, *leaf;
};

__global__ void k_let_merge(const LetRec* __restrict__ in, int64_t nr, RTab t, MCells c, unsigned char* __restrict__ cflag) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nr; k += (int64_t)gridDim.x * blockDim.x) {
    int j = 0;
    while (j + 1 < t.np && k >= t.start[j + 1]) ++j;
    const int64_t kk = k - t.start[j];
    const int64_t id = t.cbase[j] + kk;
    const LetRec r = in[k];
    c.level[id] = r.level;
    c.qx[id] = r.qx;
    c.qy[id] = r.qy;
    c.qz[id] = r.qz;
    c.count[id] = r.count;
    c.parent[id] = r.parent >= 0 ? (int)(t.cbase[j] + r.parent) : -1;
    c.child_begin[id] = r.child >= 0 ? (int)(t.cbase[j] + r.child) : -1;
    c.nchild[id] = r.nchild;
    c.leaf[id] = (r.flags & (F_LEAF | F_FRONTIER)) ? 1 : 0;
    c.begin[id] = (r.flags & F_BODIES) ? (int)(t.bbase[j] + r.body_off) : 0;
    // 2: frontier (an internal cell whose children were not sent), 4: leaf without bodies
    cflag[id] = (unsigned char)(((r.flags & F_FRONTIER) ? 2 : 0) | (((r.flags & F_LEAF) && !(r.flags & F_BODIES)) ? 4 : 0));
  }
}

// evaluate: gather the sent multipoles and bodies (receiver-major record order)
__global__ void k_let_gather_m(const int* __restrict__ scell, int64_t nr, int nc3, const float2* __restrict__ M,
                               float2* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nr * nc3; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / nc3, i = e - k * nc3;
    out[e] = M[(int64_t)scell[k] * nc3 + i];
  }
}

__global__ void k_let_gather_b(const int64_t* __restrict__ brec, const int* __restrict__ scell,
                               const int64_t* __restrict__ boff, const int* __restrict__ begin,
                               const int* __restrict__ count, const float4* __restrict__ pos,
                               const float4* __restrict__ alp, float4* __restrict__ op, float4* __restrict__ oa) {
  const int64_t k = brec[blockIdx.x];
  const int cell = scell[k];
  const int b = begin[cell], n = count[cell];
  const int64_t o = boff[k];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    op[o + i] = pos[b + i];
    oa[o + i] = alp[b + i];
  }
}

// top multipoles for the periodic far field: slot 0 = root, 1 + o = level-1 cell of octant o
__global__ void k_top_gather(const int* __restrict__ level, const int* __restrict__ qx, const int* __restrict__ qy,
                             const int* __restrict__ qz, int64_t ncand, int nc3, const float2* __restrict__ M,
                             float2* __restrict__ top) {
  const int cell = blockIdx.x;
  if (cell >= ncand) return;
  const int l = level[cell];
  if (l > 1) return;
  const int slot = l == 0 ? 0 : 1 + (qx[cell] | (qy[cell] << 1) | (qz[cell] << 2));
  for (int i = threadIdx.x; i < nc3; i += blockDim.x) top[(int64_t)slot * nc3 + i] = M[(int64_t)cell * nc3 + i];
}

unsigned grid_for(int64_t n) {
  unsigned b = nblocks(n, 256);
  return b > 148 * 16 ? 148 * 16 : b;
}

template <typename F>
void cub_call(Ctx& c, F f) {
  size_t bytes = 0;
  FMM_CUDA(f((void*)nullptr, bytes));
  c.cub_tmp.reserve(bytes);
  FMM_CUDA(f((void*)c.cub_tmp.p, bytes));
  ++c.cub_calls;
}

float fkey_inv_host(int i) {
  int j = i >= 0 ? i : i ^ 0x7fffffff;
  float f;
  memcpy(&f, &j, 4);
  return f;
}

}  // namespace

// bounding box (min xyz, max xyz) of n float4 positions, synchronous
void bbox_of(Ctx& c, const float4* pos, int64_t n, float out[6]) {
  cudaStream_t st = c.stream;
  int init[6] = {INT_MAX, INT_MAX, INT_MAX, INT_MIN, INT_MIN, INT_MIN};
  c.dflag.reserve(8);
  FMM_CUDA(cudaMemcpyAsync(c.dflag.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
  if (n > 0) FMM_LAUNCH(c, k_bbox, grid_for(n), 256, 0, pos, n, c.dflag.p);
  int h[6];
  FMM_CUDA(cudaMemcpyAsync(h, c.dflag.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  for (int k = 0; k < 6; ++k) out[k] = fkey_inv_host(h[k]);
}

// set_particles (nranks > 1), after the local tree: LET structure for every
// peer, exchanged and merged into the cell table (see the header).
void let_setup(Ctx& c) {
  cudaStream_t st = c.stream;
  const int P = c.cfg.nranks, R = c.cfg.rank;
  const int64_t nloc = c.nloc_cells, n = c.n;
  // the ranks' domains: bounding boxes of their (wrapped) particles
  double mybox[7] = {0, 0, 0, 0, 0, 0, 0};
  if (n > 0) {
    float h[6];
    bbox_of(c, c.pos.p, n, h);
    for (int a = 0; a < 3; ++a) { mybox[a] = h[a]; mybox[3 + a] = h[3 + a]; }
    mybox[6] = 1.0;
  }
  const std::vector<double> boxes = allgather_f64(c, mybox, 7);
  LetGeo g{};
  for (int a = 0; a < 3; ++a) { g.lo[a] = c.lo[a]; g.per[a] = c.per[a]; }
  g.L = c.L;
  g.theta = (double)c.cfg.theta_num / (double)c.cfg.theta_den;
  g.leaf_first = c.cfg.traversal;
  for (int q = 0; q < P; ++q)
    for (int a = 0; a < 3; ++a) { g.blo[q][a] = boxes[7 * q + a]; g.bhi[q][a] = boxes[7 * q + 3 + a]; }
  LetCells lc{c.cells.level.p, c.cells.qx.p, c.cells.qy.p, c.cells.qz.p, c.cells.leaf.p, c.cells.child_begin.p,
              c.cells.nchild.p, c.cells.count.p, c.cells.parent.p};
  // every rank tells every other rank how large its leaves near that rank's domain are
  {
    c.dflag.reserve(std::max(8, P));
    FMM_CUDA(cudaMemsetAsync(c.dflag.p, 0, sizeof(int) * P, st));
    if (c.nleaves > 0)
      FMM_LAUNCH(c, k_leaf_reach, grid_for(c.nleaves), 256, 0, c.leaf_ids.p, c.nleaves, lc, g, P, R,
                 (unsigned*)c.dflag.p);
    std::vector<unsigned> rm(P);
    FMM_CUDA(cudaMemcpyAsync(rm.data(), c.dflag.p, sizeof(unsigned) * P, cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaStreamSynchronize(st));
    std::vector<int64_t> send(P), got;
    for (int q = 0; q < P; ++q) send[q] = (int64_t)rm[q];
    got = alltoall_i64(c, send);
    for (int q = 0; q < P; ++q) {
      float f;
      const unsigned u = (unsigned)got[q];
      memcpy(&f, &u, 4);
      g.rleaf[q] = q == R ? 0.0 : (double)f;
    }
  }
  // 1. the walk
  std::vector<uint64_t> seeds;
  if (n > 0)
    for (int q = 0; q < P; ++q)
      if (q != R && boxes[7 * q + 6] > 0.5) seeds.push_back((uint64_t)q);     // (root 0, receiver q)
  int64_t nf = (int64_t)seeds.size(), nrec = 0;
  c.front_a.reserve(std::max<int64_t>(nf, 1024));
  c.let_rec.reserve(1 << 16);
  if (nf) FMM_CUDA(cudaMemcpyAsync(c.front_a.p, seeds.data(), 8 * nf, cudaMemcpyHostToDevice, st));
  while (nf > 0) {
    c.cnt_p2p.reserve(nf + 1);
    c.off_p2p.reserve(nf + 1);
    c.let_dec.reserve(nf + 1);
    FMM_LAUNCH(c, k_let_count, nblocks(nf, 256), 256, 0, c.front_a.p, nf, lc, g, c.cnt_p2p.p, c.let_dec.p);
    {
      const int* in = c.cnt_p2p.p;
      int* out = c.off_p2p.p;
      const int nn = (int)nf;
      cub_call(c, [&](void* tmp, size_t& bytes) { return cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, nn, st); });
    }
    int tail[2];
    FMM_CUDA(cudaMemcpyAsync(&tail[0], c.off_p2p.p + nf - 1, 4, cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaMemcpyAsync(&tail[1], c.cnt_p2p.p + nf - 1, 4, cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaStreamSynchronize(st));
    const int64_t nn = (int64_t)tail[0] + tail[1];
    c.let_rec.grow_keep(nrec + nf, nrec, st);
    c.front_b.reserve(std::max<int64_t>(nn, 1));
    FMM_LAUNCH(c, k_let_write, nblocks(nf, 256), 256, 0, c.front_a.p, nf, lc, c.let_dec.p, c.off_p2p.p, c.front_b.p,
               c.let_rec.p + nrec);
    nrec += nf;
    std::swap(c.front_a.p, c.front_b.p);
    std::swap(c.front_a.cap, c.front_b.cap);
    nf = nn;
  }
  // 2. receiver-major order (stable: levels ascending, key order within a level)
  c.let_rec2.reserve(std::max<int64_t>(nrec, 1));
  if (nrec > 1) {
    uint64_t* in = c.let_rec.p;
    uint64_t* out = c.let_rec2.p;
    const int nn = (int)nrec;
    cub_call(c, [&](void* tmp, size_t& bytes) { return cub::DeviceRadixSort::SortKeys(tmp, bytes, in, out, nn, 40, 44, st); });
  } else if (nrec == 1) {
    FMM_CUDA(cudaMemcpyAsync(c.let_rec2.p, c.let_rec.p, 8, cudaMemcpyDeviceToDevice, st));
  }
  std::vector<int64_t> nrec_s(P, 0);
  {
    c.dflag.reserve(std::max(8, P));
    FMM_CUDA(cudaMemsetAsync(c.dflag.p, 0, sizeof(int) * P, st));
    if (nrec) FMM_LAUNCH(c, k_let_hist, grid_for(nrec), 256, 0, c.let_rec2.p, nrec, c.dflag.p);
    std::vector<int> h(P);
    FMM_CUDA(cudaMemcpyAsync(h.data(), c.dflag.p, sizeof(int) * P, cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaStreamSynchronize(st));
    for (int q = 0; q < P; ++q) nrec_s[q] = h[q];
  }
  QTab qt{};
  qt.P = P;
  for (int q = 0, acc = 0; q < P; ++q) { qt.start[q] = acc; acc += (int)nrec_s[q]; }
  qt.start[P] = nrec;
  // 3. records: links within each receiver's list, body offsets
  c.let_recof.reserve(std::max<int64_t>((int64_t)P * nloc, 1));
  c.let_boff.reserve(std::max<int64_t>(nrec, 1) + 1);
  c.let_scell.reserve(std::max<int64_t>(nrec, 1));
  c.let_srec.reserve(std::max<int64_t>(nrec, 1) * sizeof(LetRec));
  std::vector<int64_t> nbody_s(P, 0);
  if (nrec) {
    FMM_LAUNCH(c, k_let_recof, grid_for(nrec), 256, 0, c.let_rec2.p, nrec, qt, nloc, c.let_recof.p);
    FMM_CUDA(cudaMemsetAsync(c.let_boff.p, 0, 8 * (nrec + 1), st));
    FMM_LAUNCH(c, k_let_bodycount, grid_for(nrec), 256, 0, c.let_rec2.p, nrec, c.cells.count.p, c.let_boff.p);
    {
      int64_t* p = c.let_boff.p;
      const int nn = (int)(nrec + 1);
      cub_call(c, [&](void* tmp, size_t& bytes) { return cub::DeviceScan::ExclusiveSum(tmp, bytes, p, p, nn, st); });
    }
    std::vector<int64_t> bstart(P + 1, 0);
    for (int q = 0; q <= P; ++q)
      FMM_CUDA(cudaMemcpyAsync(&bstart[q], c.let_boff.p + qt.start[q], 8, cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaStreamSynchronize(st));
    for (int q = 0; q < P; ++q) { qt.bbase[q] = bstart[q]; nbody_s[q] = bstart[q + 1] - bstart[q]; }
    FMM_LAUNCH(c, k_let_records, grid_for(nrec), 256, 0, c.let_rec2.p, nrec, lc, qt, nloc, c.let_recof.p, c.let_boff.p,
               (LetRec*)c.let_srec.p, c.let_scell.p);
    // body records (receiver-major), for the per-evaluate gather
    c.let_brec.reserve(std::max<int64_t>(nrec, 1) * 2);
    FMM_LAUNCH(c, k_iota64, grid_for(nrec), 256, 0, c.let_brec.p + nrec, nrec);
    c.dsel.reserve(1);
    {
      const int64_t* in = c.let_brec.p + nrec;
      int64_t* out = c.let_brec.p;
      int* ns = c.dsel.p;
      const int nn = (int)nrec;
      IsBodies pred{c.let_rec2.p};
      cub_call(c, [&](void* tmp, size_t& bytes) { return cub::DeviceSelect::If(tmp, bytes, in, out, ns, nn, pred, st); });
    }
    int nb = 0;
    FMM_CUDA(cudaMemcpyAsync(&nb, c.dsel.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaStreamSynchronize(st));
    c.let_nbrec = nb;
  } else {
    c.let_nbrec = 0;
  }
  c.let_nrec_s = nrec_s;
  c.let_nbody_s = nbody_s;
  c.let_nsend_rec = nrec;
  // 4. sizes and records to the peers
  c.let_nrec_r = alltoall_i64(c, nrec_s);
  c.let_nbody_r = alltoall_i64(c, nbody_s);
  int64_t nrr = 0, nbr = 0;
  for (int q = 0; q < P; ++q) { nrr += c.let_nrec_r[q]; nbr += c.let_nbody_r[q]; }
  c.let_rrec.reserve(std::max<int64_t>(nrr, 1) * sizeof(LetRec));
  {
    std::vector<int64_t> soff(P), sb(P), roff(P), rb(P);
    int64_t so = 0, ro = 0;
    for (int q = 0; q < P; ++q) {
      soff[q] = (int64_t)sizeof(LetRec) * so;
      roff[q] = (int64_t)sizeof(LetRec) * ro;
      sb[q] = (int64_t)sizeof(LetRec) * nrec_s[q];
      rb[q] = (int64_t)sizeof(LetRec) * c.let_nrec_r[q];
      so += nrec_s[q];
      ro += c.let_nrec_r[q];
    }
    alltoallv_bytes(c, c.let_srec.p, soff, sb, c.let_rrec.p, roff, rb);
  }
  // 5. merge: tree of peer q at cells [nloc + cbase_q, ...), bodies at [n + bbase_q, ...)
  c.let_cbase.assign(P + 1, 0);
  c.let_bbase.assign(P + 1, 0);
  RTab rt{};
  int np = 0;
  int64_t cb = 0, bb = 0, rs = 0;
  c.let_peer.clear();
  for (int q = 0; q < P; ++q) {
    c.let_cbase[q] = nloc + cb;
    c.let_bbase[q] = n + bb;
    if (q == R || c.let_nrec_r[q] == 0) continue;
    rt.start[np] = rs;
    rt.cbase[np] = nloc + cb;
    rt.bbase[np] = n + bb;
    c.let_peer.push_back(q);
    ++np;
    rs += c.let_nrec_r[q];
    cb += c.let_nrec_r[q];
    bb += c.let_nbody_r[q];
  }
  rt.np = np;
  rt.start[np] = rs;
  const int64_t ncells = nloc + nrr;
  if (ncells >= (1ll << 27)) throw FmmError(FMM_E_ARG, "more than 2^27 cells with the LET; raise ncrit");
  c.cells.reserve_keep((size_t)ncells, (size_t)nloc, st);
  c.cflag.reserve(std::max<int64_t>(ncells, 1));
  FMM_CUDA(cudaMemsetAsync(c.cflag.p, 0, std::max<int64_t>(ncells, 1), st));
  MCells mc{c.cells.level.p, c.cells.qx.p, c.cells.qy.p, c.cells.qz.p, c.cells.begin.p, c.cells.count.p,
            c.cells.parent.p, c.cells.child_begin.p, c.cells.nchild.p, c.cells.leaf.p};
  if (nrr) FMM_LAUNCH(c, k_let_merge, grid_for(nrr), 256, 0, (const LetRec*)c.let_rrec.p, nrr, rt, mc, c.cflag.p);
  c.ncells = ncells;
  c.nsrc = n + nbr;
  c.pos.grow_keep((size_t)std::max<int64_t>(c.nsrc, 1), (size_t)n, st);
  c.alp.grow_keep((size_t)std::max<int64_t>(c.nsrc, 1), (size_t)n, st);
  // the peers' roots (traversal seeds) and whether they are leaves
  c.let_roots.clear();
  c.let_root_leaf.clear();
  for (int j = 0; j < np; ++j) {
    const int id = (int)rt.cbase[j];
    int lf = 0;
    FMM_CUDA(cudaMemcpyAsync(&lf, c.cells.leaf.p + id, sizeof(int), cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaStreamSynchronize(st));
    c.let_roots.push_back(id);
    c.let_root_leaf.push_back(lf);
  }
  int64_t scells = 0, sbody = 0;
  for (int q = 0; q < P; ++q) { scells += nrec_s[q]; sbody += nbody_s[q]; }
  const int64_t mb = (int64_t)3 * c.nc * 8;
  c.let_bytes_sent = scells * mb + 32 * sbody;
  c.let_bytes_recv = nrr * mb + 32 * nbr;
  c.let_cells = nrr;
  c.let_leaves = nbr;
}

// evaluate (nranks > 1): the LET payload -- multipoles of the sent cells and the
// sent bodies -- and the top multipoles' all-reduce, enqueued on stream cs
// after the upward pass (the caller orders cs after it).
void let_exchange(Ctx& c, cudaStream_t cs) {
  const int P = c.cfg.nranks, R = c.cfg.rank;
  const int nc3 = 3 * c.nc;
  const int64_t nr = c.let_nsend_rec;
  int64_t nbs = 0;
  for (int q = 0; q < P; ++q) nbs += c.let_nbody_s[q];
  c.let_sM.reserve((size_t)std::max<int64_t>(nr, 1) * nc3);
  c.let_sP.reserve((size_t)std::max<int64_t>(nbs, 1));
  c.let_sA.reserve((size_t)std::max<int64_t>(nbs, 1));
  if (nr) FMM_LAUNCH_ON(c, cs, k_let_gather_m, grid_for(nr * nc3), 256, 0, c.let_scell.p, nr, nc3, c.M.p, c.let_sM.p);
  if (c.let_nbrec)
    FMM_LAUNCH_ON(c, cs, k_let_gather_b, (unsigned)c.let_nbrec, 64, 0, c.let_brec.p, c.let_scell.p, c.let_boff.p,
                  c.cells.begin.p, c.cells.count.p, c.pos.p, c.alp.p, c.let_sP.p, c.let_sA.p);
  std::vector<CommSeg> segs;
  int64_t mo = 0, bo = 0;
  for (int q = 0; q < P; ++q) {
    if (q != R) {
      segs.push_back({true, q, c.let_sM.p + mo * nc3, (int64_t)8 * nc3 * c.let_nrec_s[q]});
      segs.push_back({true, q, c.let_sP.p + bo, 16 * c.let_nbody_s[q]});
      segs.push_back({true, q, c.let_sA.p + bo, 16 * c.let_nbody_s[q]});
      segs.push_back({false, q, c.M.p + c.let_cbase[q] * nc3, (int64_t)8 * nc3 * c.let_nrec_r[q]});
      segs.push_back({false, q, c.pos.p + c.let_bbase[q], 16 * c.let_nbody_r[q]});
      segs.push_back({false, q, c.alp.p + c.let_bbase[q], 16 * c.let_nbody_r[q]});
    }
    mo += c.let_nrec_s[q];
    bo += c.let_nbody_s[q];
  }
  alltoallv_multi(c, segs, cs);
  // root (slot 0) and level-1 cells (slots 1..8) of every rank's tree, summed: the
  // periodic far field's sources (a8) and the tiles' multipoles (Z27)
  top_multipoles(c, cs);
  allreduce_sum_f32(c, (float*)c.top_M.p, 2 * 9 * (int64_t)nc3, cs);
}

// slots 0..8 of c.top_M from the local tree (zeros where this rank has no cell)
void top_multipoles(Ctx& c, cudaStream_t cs) {
  const int nc3 = 3 * c.nc;
  c.top_M.reserve((size_t)9 * nc3);
  FMM_CUDA(cudaMemsetAsync(c.top_M.p, 0, sizeof(float2) * 9 * nc3, cs));
  const int64_t ncand = c.level_begin.size() > 2 ? c.level_begin[2] : c.nloc_cells;
  if (ncand > 0)
    FMM_LAUNCH_ON(c, cs, k_top_gather, (unsigned)ncand, 128, 0, c.cells.level.p, c.cells.qx.p, c.cells.qy.p,
                  c.cells.qz.p, ncand, nc3, c.M.p, c.top_M.p);
}

}  // namespace fmmb
