// traverse.cu -- a7: dual tree traversal (Alg. 1, Alg. 2
// P:171-187) on the device, level-synchronously.  The paper's stack of cell
// pairs becomes a frontier array: every round pops the whole frontier,
// splits the larger cell of each pair (equal radius => split B, never split a
// leaf: reading Z10) and applies Interact to each child pair (MAC-first or
// leaf-first, reading Z11).  Each round is a count pass, three exclusive scans
// and a write pass, so no atomics decide where entries go; the lists are then
// radix-sorted into the canonical (target, source, image) order (Z20) and cut
// into per-target segments for the P2P and M2L kernels.  The MAC is the exact
// integer form of r_A + r_B < theta R (Z9).
#include <cub/cub.cuh>

#include "ctx.cuh"

namespace fmmb {

namespace {

struct TCells {
  const int *level, *qx, *qy, *qz, *child_begin, *nchild, *leaf, *count;
  const unsigned char* cflag;   // LET forest (nranks > 1): 2 = frontier, 4 = leaf without bodies; else null
};

struct TParams {
  unsigned long long lhs_k;   // 3 * theta_den^2
  unsigned long long rhs_k;   // theta_num^2
  int leaf_first;
  long long per[3];           // domain periods in half-finest-cell units (image shifts)
};

__device__ __forceinline__ uint64_t pack(int A, int B, int img) {
  return ((uint64_t)A << 32) | ((uint64_t)B << 5) | (uint64_t)img;
}

// MAC (Z9): 3 den^2 (2^{21-a} + 2^{21-b})^2 < num^2 |Delta|^2 on integers in
// units of half the finest cell; |Delta| includes the first-layer image shift.
__device__ __forceinline__ bool mac_accept(const TCells& c, const TParams& p, int A, int B, int img) {
  int la = c.level[A], lb = c.level[B];
  int ix = img % 3 - 1, iy = (img / 3) % 3 - 1, iz = img / 9 - 1;
  long long dx = ((long long)(2 * c.qx[A] + 1) << (kMaxLevel - la)) - ((long long)(2 * c.qx[B] + 1) << (kMaxLevel - lb)) - (long long)ix * p.per[0];
  long long dy = ((long long)(2 * c.qy[A] + 1) << (kMaxLevel - la)) - ((long long)(2 * c.qy[B] + 1) << (kMaxLevel - lb)) - (long long)iy * p.per[1];
  long long dz = ((long long)(2 * c.qz[A] + 1) << (kMaxLevel - la)) - ((long long)(2 * c.qz[B] + 1) << (kMaxLevel - lb)) - (long long)iz * p.per[2];
  unsigned long long d2 = (unsigned long long)(dx * dx) + (unsigned long long)(dy * dy) + (unsigned long long)(dz * dz);
  unsigned long long ss = (1ull << (kMaxLevel - la)) + (1ull << (kMaxLevel - lb));
  return p.lhs_k * ss * ss < p.rhs_k * d2;
}

// Alg. 2 Interact: 0 = M2L, 1 = P2P, 2 = push, 3 = M2L by the remote branch.
// A remote source received without what the pair needs -- a frontier cell
// (children not sent) that would be split, or a leaf without bodies -- takes
// "the M2L translation with the smallest cell that is available" (Alg. 2,
// P:176-179); such fallbacks are counted (zero when the LET-MAC is
// complete).  Frontier cells carry the leaf flag, so they are never split.
__device__ __forceinline__ int interact(const TCells& c, const TParams& p, int A, int B, int img) {
  const bool leaves = c.leaf[A] && c.leaf[B];
  const int fl = c.cflag ? c.cflag[B] : 0;
  if (p.leaf_first) {
    if (leaves) {
      if (fl & 2) return mac_accept(c, p, A, B, img) ? 0 : 3;   // internal in its own tree
      return (fl & 4) ? 3 : 1;
    }
    return mac_accept(c, p, A, B, img) ? 0 : 2;
  }
  if (mac_accept(c, p, A, B, img)) return 0;
  if (leaves) return fl ? 3 : 1;
  return 2;
}

// Alg. 1 body for frontier pair f: split B if A is a leaf or (B is not a leaf
// and r_B >= r_A, i.e. level_B <= level_A); otherwise split A.
template <bool WRITE>
__global__ void k_expand(const uint64_t* __restrict__ front, int64_t nf, TCells c, TParams p,
                         int* __restrict__ cm, int* __restrict__ cp, int* __restrict__ cq,
                         const int* __restrict__ om, const int* __restrict__ op, const int* __restrict__ oq,
                         uint64_t* __restrict__ m2l, uint64_t* __restrict__ p2p, uint64_t* __restrict__ next,
                         unsigned char* __restrict__ has_m2l, unsigned long long* __restrict__ fallback) {
  int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= nf) return;
  uint64_t e = front[f];
  int A = (int)(e >> 32), B = (int)((e >> 5) & 0x7ffffff), img = (int)(e & 31);
  bool split_b = c.leaf[A] || (!c.leaf[B] && c.level[B] <= c.level[A]);
  int cb = split_b ? c.child_begin[B] : c.child_begin[A];
  int nch = split_b ? c.nchild[B] : c.nchild[A];
  int nm = 0, np = 0, nq = 0;
  int bm = 0, bp = 0, bq = 0;
  if (WRITE) { bm = om[f]; bp = op[f]; bq = oq[f]; }
  for (int k = 0; k < nch; ++k) {
    int a = split_b ? A : cb + k;
    int b = split_b ? cb + k : B;
    int d = interact(c, p, a, b, img);
    if (d == 3) {
      if (WRITE) atomicAdd(fallback, 1ull);
      d = 0;
    }
    if (d == 0) {
      if (WRITE) {
        m2l[bm + nm] = pack(a, b, img);
        if (!split_b) has_m2l[a] = 1;              // has_m2l: for m2l_tc_prepare (A's flag: below)
      }
      ++nm;
    }
    else if (d == 1) { if (WRITE) p2p[bp + np] = pack(a, b, img); ++np; }
    else { if (WRITE) next[bq + nq] = pack(a, b, img); ++nq; }
  }
  if (WRITE && split_b && nm > 0) has_m2l[A] = 1;
  if (!WRITE) { cm[f] = nm; cp[f] = np; cq[f] = nq; }
}

__global__ void k_clear2(int* a, int* b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) { a[i] = 0; b[i] = 0; }
}

__global__ void k_segments(const uint64_t* __restrict__ lst, int64_t n, int* __restrict__ sb, int* __restrict__ se) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int t = (int)(lst[i] >> 32);
    if (i == 0 || (int)(lst[i - 1] >> 32) != t) sb[t] = (int)i;
    if (i == n - 1 || (int)(lst[i + 1] >> 32) != t) se[t] = (int)(i + 1);
  }
}

// p2p_m[t] = the first entry of target t's segment with a remote source
__global__ void k_remote_split(const uint64_t* __restrict__ lst, int64_t n, int nloc, int* __restrict__ pm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t e = lst[i];
    const int t = (int)(e >> 32), s = (int)((e >> 5) & 0x7ffffff);
    if (s < nloc) continue;
    if (i == 0) { pm[t] = 0; continue; }
    const uint64_t f = lst[i - 1];
    if ((int)(f >> 32) != t || (int)((f >> 5) & 0x7ffffff) < nloc) pm[t] = (int)i;
  }
}

__global__ void k_pair_count(const uint64_t* __restrict__ lst, int64_t n, const int* __restrict__ count,
                             unsigned long long* out) {
  unsigned long long acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t e = lst[i];
    acc += (unsigned long long)count[e >> 32] * (unsigned long long)count[(e >> 5) & 0x7ffffff];
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

template <typename F>
void cub_call(Ctx& c, F f) {
  size_t bytes = 0;
  FMM_CUDA(f((void*)nullptr, bytes));
  c.cub_tmp.reserve(bytes);
  FMM_CUDA(f((void*)c.cub_tmp.p, bytes));
  ++c.cub_calls;
}

void exclusive_scan(Ctx& c, const int* in, int* out, int64_t n) {
  cub_call(c, [&](void* tmp, size_t& bytes) {
    return cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, (int)n, c.stream);
  });
}

// begin_bit = 0: the canonical (target, source, image) order; begin_bit = 32:
// grouped by target only, stable, i.e. the traversal's (deterministic)
// emission order within a target
void sort_list(Ctx& c, DBuf<uint64_t>& lst, int64_t n, int begin_bit = 0) {
  if (n <= 1) return;
  c.sort_tmp.reserve(n);
  uint64_t* in = lst.p;
  uint64_t* out = c.sort_tmp.p;
  // the target field (bits 32..58) only holds cell ids < ncells: sort no higher
  int nb = 1;
  while (nb < 27 && (1ll << nb) < c.ncells) ++nb;
  const int end_bit = 32 + nb;
  cub_call(c, [&](void* tmp, size_t& bytes) {
    return cub::DeviceRadixSort::SortKeys(tmp, bytes, in, out, (int)n, begin_bit, end_bit, c.stream);
  });
  std::swap(lst.p, c.sort_tmp.p);
  std::swap(lst.cap, c.sort_tmp.cap);
}

}  // namespace

struct NotTaken {
  const unsigned char* skip;
  __device__ __forceinline__ bool operator()(const uint64_t& e) const { return !skip[(int)(e >> 32)]; }
};

// entry i stays on the register kernel unless its target is on the tensor path
// and the tensor path verified this entry (m2l_tc_prepare's per-entry bits)
struct OnRegisterPath {
  const uint64_t* lst;
  const unsigned char* skip;
  const unsigned* good;
  __device__ __forceinline__ char operator()(const int64_t& i) const {
    if (!skip[(int)(lst[i] >> 32)]) return 1;
    return ((good[i >> 5] >> (i & 31)) & 1u) ? 0 : 1;
  }
};

// the M2L entries the tensor path does not take (target not taken, or entry
// not verified), in emission order (stable select), grouped by target (stable sort), with
// per-target segments m2l_b/m2l_e for the register kernels
void m2l_reg_segments(Ctx& c) {
  cudaStream_t st = c.stream;
  c.nm2lr = 0;
  c.m2l_b.reserve(std::max<int64_t>(c.ncells, 1)); c.m2l_e.reserve(std::max<int64_t>(c.ncells, 1));
  FMM_LAUNCH(c, k_clear2, nblocks(std::max<int64_t>(c.ncells, 1), 256), 256, 0, c.m2l_b.p, c.m2l_e.p, c.ncells);
  if (c.nm2l == 0) return;
  c.m2lr.reserve(c.nm2l);
  c.dsel.reserve(1);
  const uint64_t* in = c.m2l.p;
  uint64_t* out = c.m2lr.p;
  int* nsel = c.dsel.p;
  const int n = (int)c.nm2l;
  if (c.tc_mixed) {
    cub::CountingInputIterator<int64_t> idx(0);
    cub::TransformInputIterator<char, OnRegisterPath, cub::CountingInputIterator<int64_t>> flags(
        idx, OnRegisterPath{c.m2l.p, c.tc_skip.p, c.tc_good.p});
    cub_call(c, [&](void* tmp, size_t& bytes) {
      return cub::DeviceSelect::Flagged(tmp, bytes, in, flags, out, nsel, n, st);
    });
  } else {
    // every entry of a taken cell is on the tensor path (uniform levels): by target alone
    NotTaken pred{c.tc_skip.p};
    cub_call(c, [&](void* tmp, size_t& bytes) {
      return cub::DeviceSelect::If(tmp, bytes, in, out, nsel, n, pred, st);
    });
  }
  int ns = 0;
  FMM_CUDA(cudaMemcpyAsync(&ns, c.dsel.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  c.nm2lr = ns;
  sort_list(c, c.m2lr, c.nm2lr, 32);
  if (c.nm2lr) FMM_LAUNCH(c, k_segments, nblocks(c.nm2lr, 256), 256, 0, c.m2lr.p, c.nm2lr, c.m2l_b.p, c.m2l_e.p);
}

void build_lists(Ctx& c) {
  c.tc_valid = false;
  cudaStream_t st = c.stream;
  c.np2p = c.nm2l = 0;
  c.p2p_pairs = 0;
  c.let_fallback = 0;
  if (c.nloc_cells == 0) { c.lists_valid = true; return; }
  const bool multi = c.cfg.nranks > 1;
  TCells tc{c.cells.level.p, c.cells.qx.p, c.cells.qy.p, c.cells.qz.p, c.cells.child_begin.p,
            c.cells.nchild.p, c.cells.leaf.p, c.cells.count.p, multi ? c.cflag.p : nullptr};
  c.dfallback.reserve(1);
  FMM_CUDA(cudaMemsetAsync(c.dfallback.p, 0, sizeof(unsigned long long), st));
  TParams tp{3ull * (unsigned long long)c.cfg.theta_den * (unsigned long long)c.cfg.theta_den,
             (unsigned long long)c.cfg.theta_num * (unsigned long long)c.cfg.theta_num, c.cfg.traversal,
             {c.per_units[0], c.per_units[1], c.per_units[2]}};

  // seeds (8c-2 item 7): Interact(root, root_t, img) for the 27 first-layer
  // images (k >= 1) or the zero image, for every tree t of the forest (the
  // local tree and the peers' LETs, nranks > 1).  A root pair never passes
  // the MAC (|Delta| <= sqrt(3) L while r_A + r_B = sqrt(3) L and theta < 1),
  // and a received root is never a frontier or a leaf without bodies (the
  // LET-MAC cannot accept a root), so a seed is P2P iff both roots are
  // leaves, else it is pushed.
  std::vector<uint64_t> seeds, pseeds;
  const bool root_leaf = c.host_leaf_top.size() > 0 && c.host_leaf_top[0];
  std::vector<int> roots{0}, rleaf{root_leaf ? 1 : 0};
  for (size_t j = 0; j < c.let_roots.size() && multi; ++j) {
    roots.push_back(c.let_roots[j]);
    rleaf.push_back(c.let_root_leaf[j]);
  }
  for (size_t t = 0; t < roots.size(); ++t) {
    std::vector<int> imgs;
    if (c.cfg.images > 0) for (int img = 0; img < 27; ++img) imgs.push_back(img);
    else imgs.push_back(kImgCentre);
    for (int img : imgs) {
      const uint64_t e = ((uint64_t)roots[t] << 5) | (uint64_t)img;      // target = local root 0
      (root_leaf && rleaf[t] ? pseeds : seeds).push_back(e);
    }
  }
  int64_t nf = (int64_t)seeds.size();
  c.front_a.reserve(std::max<int64_t>(1024, nf));
  c.front_b.reserve(1024);
  c.tc_has.reserve(std::max<int64_t>(c.ncells, 1));
  FMM_CUDA(cudaMemsetAsync(c.tc_has.p, 0, std::max<int64_t>(c.ncells, 1), st));
  c.p2p.reserve(std::max<int64_t>(1 << 16, (int64_t)pseeds.size()));
  c.m2l.reserve(1 << 16);
  if (!pseeds.empty()) {
    FMM_CUDA(cudaMemcpyAsync(c.p2p.p, pseeds.data(), sizeof(uint64_t) * pseeds.size(), cudaMemcpyHostToDevice, st));
    c.np2p = (int64_t)pseeds.size();
  }
  if (nf) FMM_CUDA(cudaMemcpyAsync(c.front_a.p, seeds.data(), sizeof(uint64_t) * nf, cudaMemcpyHostToDevice, st));
  FMM_CUDA(cudaStreamSynchronize(st));          // host vectors above are read by the copies

  while (nf > 0) {
    c.cnt_m2l.reserve(nf + 1); c.cnt_p2p.reserve(nf + 1); c.cnt_push.reserve(nf + 1);
    c.off_m2l.reserve(nf + 1); c.off_p2p.reserve(nf + 1); c.off_push.reserve(nf + 1);
    unsigned g = nblocks(nf, 256);
    FMM_LAUNCH(c, k_expand<false>, g, 256, 0, c.front_a.p, nf, tc, tp, c.cnt_m2l.p, c.cnt_p2p.p, c.cnt_push.p,
                                       nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    FMM_LAUNCH_CHECK();
    exclusive_scan(c, c.cnt_m2l.p, c.off_m2l.p, nf);
    exclusive_scan(c, c.cnt_p2p.p, c.off_p2p.p, nf);
    exclusive_scan(c, c.cnt_push.p, c.off_push.p, nf);
    int tail[6];
    FMM_CUDA(cudaMemcpyAsync(&tail[0], c.off_m2l.p + nf - 1, 4, cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaMemcpyAsync(&tail[1], c.cnt_m2l.p + nf - 1, 4, cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaMemcpyAsync(&tail[2], c.off_p2p.p + nf - 1, 4, cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaMemcpyAsync(&tail[3], c.cnt_p2p.p + nf - 1, 4, cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaMemcpyAsync(&tail[4], c.off_push.p + nf - 1, 4, cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaMemcpyAsync(&tail[5], c.cnt_push.p + nf - 1, 4, cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaStreamSynchronize(st));
    int64_t add_m = (int64_t)tail[0] + tail[1], add_p = (int64_t)tail[2] + tail[3], add_q = (int64_t)tail[4] + tail[5];
    if (c.nm2l + add_m >= (1ll << 31) || c.np2p + add_p >= (1ll << 31))
      throw FmmError(FMM_E_ARG, "interaction list exceeds 2^31 entries");
    c.m2l.grow_keep(c.nm2l + add_m, c.nm2l, st);
    c.p2p.grow_keep(c.np2p + add_p, c.np2p, st);
    c.front_b.reserve(add_q);
    FMM_LAUNCH(c, k_expand<true>, g, 256, 0, c.front_a.p, nf, tc, tp, nullptr, nullptr, nullptr, c.off_m2l.p,
                                      c.off_p2p.p, c.off_push.p, c.m2l.p + c.nm2l, c.p2p.p + c.np2p, c.front_b.p,
                                      c.tc_has.p, c.dfallback.p);
    FMM_LAUNCH_CHECK();
    c.nm2l += add_m;
    c.np2p += add_p;
    std::swap(c.front_a.p, c.front_b.p);
    std::swap(c.front_a.cap, c.front_b.cap);
    nf = add_q;
  }

  // per-target segments of the P2P list (fixes the near-field summation
  // order; deterministic).  The M2L list stays in the
  // traversal's (deterministic) emission order: the tensor path verifies it
  // entry by entry, and only the entries it does not take are grouped by
  // target for the register kernels (m2l_reg_segments, after m2l_tc_prepare);
  // fmm_get_lists returns the canonical order
  // canonical (target, source, image) order: consecutive target leaves then
  // read their source leaves in nearly the same order, which keeps the P2P
  // kernel's source reads in L2 (grouped by target only, the traversal's
  // emission order saves 1.8 ms of sorting but raises the P2P kernel's DRAM
  // traffic from 1.8 to 10.2 GB per launch, r02 prof2), and on several GPUs the
  // local sources (ids < nloc) precede the received ones in every segment
  sort_list(c, c.p2p, c.np2p);
  c.p2p_b.reserve(c.ncells); c.p2p_e.reserve(c.ncells);
  FMM_LAUNCH(c, k_clear2, nblocks(c.ncells, 256), 256, 0, c.p2p_b.p, c.p2p_e.p, c.ncells);
  if (c.np2p) FMM_LAUNCH(c, k_segments, nblocks(c.np2p, 256), 256, 0, c.p2p.p, c.np2p, c.p2p_b.p, c.p2p_e.p);
  if (multi) {
    // a14 overlap: per target, the entries with local sources (ids < nloc, first
    // in canonical order) run while the LET is in flight, the rest after it
    c.p2p_m.reserve(c.ncells);
    FMM_CUDA(cudaMemcpyAsync(c.p2p_m.p, c.p2p_e.p, sizeof(int) * c.ncells, cudaMemcpyDeviceToDevice, st));
    if (c.np2p)
      FMM_LAUNCH(c, k_remote_split, nblocks(c.np2p, 256), 256, 0, c.p2p.p, c.np2p, (int)c.nloc_cells, c.p2p_m.p);
  }
  c.dcount.reserve(1);
  FMM_CUDA(cudaMemsetAsync(c.dcount.p, 0, sizeof(unsigned long long), st));
  if (c.np2p) {
    unsigned g = nblocks(c.np2p, 256);
    if (g > 148 * 8) g = 148 * 8;
    FMM_LAUNCH(c, k_pair_count, g, 256, 0, c.p2p.p, c.np2p, c.cells.count.p, c.dcount.p);
  }
  FMM_LAUNCH_CHECK();
  unsigned long long pairs = 0;
  FMM_CUDA(cudaMemcpyAsync(&pairs, c.dcount.p, sizeof(pairs), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  c.p2p_pairs = (int64_t)pairs;
  unsigned long long fb = 0;
  FMM_CUDA(cudaMemcpyAsync(&fb, c.dfallback.p, sizeof(fb), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  c.let_fallback = (int64_t)fb;
  c.lists_valid = true;
}

}  // namespace fmmb
