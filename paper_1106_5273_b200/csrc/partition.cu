// partition.cu -- NEXT-3: the paper's load-balancing partition,
// orthogonal recursive multisection, on B200s.
//
// "Bisecting the domain involves the calculation of the median of the particle
// distribution for a given direction, and doing this recursively in orthogonal
// directions (x, y, z, x, y, ...)"; multisection searches for "something other
// than the median": "searching for the 3N/7-th element will enable the domain
// to be split between 3 and 4 processes".  Here a group of m ranks
// holding N_g particles is split along axis (depth mod 3) at the
// floor(N_g m1 / m)-th element, m1 = floor(m / 2), until every group is one
// rank; P <= 8 gives at most three levels.
//
// The parallel nth-element is a distributed radix select over 64-bit keys
// (order-preserving bits of the coordinate, then a unique particle id
// (rank, caller index), so ties in a lattice plane are broken and the split
// is exact): eight passes of 8 bits, each a per-rank device histogram of
// every active group's candidates followed by one NCCL all-reduce of the
// histograms -- no sort anywhere, as the paper's nth-element is "much faster
// than any sorting algorithm".  One more counting pass (k_orb_tie) moves a
// cut that would leave a sparse sliver of a lattice plane on one side to the
// plane's edge (reading Z28): such slivers, on the far side of an octant
// boundary, became coarse leaves with near lists of ~10^5 leaves.  The
// subdomains are the (rectangular) ORB boxes the dual traversal and the LET
// handle.
//
// Redistribution: every particle goes to the rank of its final group
// (records grouped by owner with a stable 4-bit radix sort, grouped
// ncclSend/ncclRecv); the receive order is kept, so evaluate sends results
// back along the reverse exchange into every rank's caller order.
#include <algorithm>
#include <climits>

#include <cub/cub.cuh>

#include "ctx.cuh"

namespace fmmb {

namespace {

// order-preserving map float -> uint32
__device__ __forceinline__ uint32_t fbits(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ unsigned long long orb_key(const float4 p, int axis, uint32_t id) {
  const float c = axis == 0 ? p.x : (axis == 1 ? p.y : p.z);
  return ((unsigned long long)fbits(c) << 32) | id;
}

// per-group histograms of one 8-bit digit of the ORB keys of the candidates
__global__ void k_orb_hist(const float4* __restrict__ pos, int64_t n, const unsigned char* __restrict__ grp,
                           uint32_t id0, OrbPass op, unsigned long long* __restrict__ hist) {
  __shared__ unsigned int sh[kMaxGroups * 256];
  for (int i = threadIdx.x; i < op.ngroups * 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int g = grp[i];
    if (!op.active[g]) continue;
    const unsigned long long k = orb_key(pos[i], op.axis[g], id0 + (uint32_t)i);
    const int up = op.shift + 8;
    if (up < 64 && (k >> up) != (op.prefix[g] >> up)) continue;
    atomicAdd(&sh[g * 256 + (int)((k >> op.shift) & 255ull)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < op.ngroups * 256; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], (unsigned long long)sh[i]);
}

// per active group: particles whose axis coordinate lies below / on the
// selected element's coordinate (cnt[2 g] / cnt[2 g + 1])
__global__ void k_orb_tie(const float4* __restrict__ pos, int64_t n, const unsigned char* __restrict__ grp,
                          OrbPass op, unsigned long long* __restrict__ cnt) {
  __shared__ unsigned int sh[2 * kMaxGroups];
  if (threadIdx.x < 2 * kMaxGroups) sh[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int g = grp[i];
    if (!op.active[g]) continue;
    const uint32_t cb = (uint32_t)(orb_key(pos[i], op.axis[g], 0u) >> 32), cs = (uint32_t)(op.prefix[g] >> 32);
    if (cb < cs) atomicAdd(&sh[2 * g], 1u);
    else if (cb == cs) atomicAdd(&sh[2 * g + 1], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 2 * kMaxGroups && sh[threadIdx.x]) atomicAdd(&cnt[threadIdx.x], (unsigned long long)sh[threadIdx.x]);
}

// split: particles of an active group with key < prefix (the selected
// element) go to the low subgroup, the others to the high one
__global__ void k_orb_split(const float4* __restrict__ pos, int64_t n, unsigned char* __restrict__ grp, uint32_t id0,
                            OrbPass op) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int g = grp[i];
    if (!op.active[g]) { grp[i] = (unsigned char)op.lo_id[g]; continue; }
    const unsigned long long k = orb_key(pos[i], op.axis[g], id0 + (uint32_t)i);
    grp[i] = (unsigned char)(k < op.prefix[g] ? op.lo_id[g] : op.hi_id[g]);
  }
}

__global__ void k_fill_u8(unsigned char* p, int64_t n, unsigned char v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

struct OwnerMap { int owner[kMaxGroups]; };

__global__ void k_owner_keys(const unsigned char* __restrict__ grp, int64_t n, OwnerMap om, uint32_t* __restrict__ okey,
                             uint32_t* __restrict__ iota, int* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int o = om.owner[grp[i]];
    okey[i] = (uint32_t)o;
    iota[i] = (uint32_t)i;
    atomicAdd(&cnt[o], 1);
  }
}

// records in send order (grouped by owner): (x, y, z, sigma) wrapped, (alpha, 0)
__global__ void k_red_pack(const uint32_t* __restrict__ sidx, int64_t n, const float4* __restrict__ pos,
                           const float* __restrict__ a, float4* __restrict__ rec) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = sidx[k];
    rec[2 * k] = pos[i];
    rec[2 * k + 1] = make_float4(a[3 * i], a[3 * i + 1], a[3 * i + 2], 0.f);
  }
}

// received records -> this rank's particle arrays x[m][3], alpha[m][3], sigma[m]
__global__ void k_red_unpack(const float4* __restrict__ rec, int64_t m, float* __restrict__ x, float* __restrict__ a,
                             float* __restrict__ s) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    const float4 p = rec[2 * k], q = rec[2 * k + 1];
    x[3 * k] = p.x; x[3 * k + 1] = p.y; x[3 * k + 2] = p.z;
    s[k] = p.w;
    a[3 * k] = q.x; a[3 * k + 1] = q.y; a[3 * k + 2] = q.z;
  }
}

// results of this rank's particles (local caller order = receive order) -> 6-float records
__global__ void k_ret_pack(const float* __restrict__ u, const float* __restrict__ s, int64_t m, float* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x)
    for (int d = 0; d < 3; ++d) {
      out[6 * k + d] = u[3 * k + d];
      out[6 * k + 3 + d] = s[3 * k + d];
    }
}

// records back in send order -> the caller's order (sidx[k] = caller index of send slot k)
__global__ void k_ret_unpack(const float* __restrict__ in, const uint32_t* __restrict__ sidx, int64_t n,
                             float* __restrict__ u, float* __restrict__ s) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = 3 * (int64_t)sidx[k];
    for (int d = 0; d < 3; ++d) {
      u[o + d] = in[6 * k + d];
      s[o + d] = in[6 * k + 3 + d];
    }
  }
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

}  // namespace

// ORB groups of the caller's particles (pos: wrapped (x, y, z, sigma), caller
// order).  With reuse, the stored cuts of the first call assign the particles
// (the paper partitions once); otherwise they are selected anew.
static void orb_groups(Ctx& c, const float4* pos, int64_t n, bool reuse, std::vector<int>& owner_of_group) {
  cudaStream_t st = c.stream;
  const int P = c.cfg.nranks, R = c.cfg.rank;
  const uint32_t id0 = (uint32_t)R << 28;
  if (n >= (1ll << 28)) throw FmmError(FMM_E_ARG, "partition >= 1: at most 2^28 particles per rank");
  c.orb_grp.reserve(std::max<int64_t>(n, 1));
  if (n > 0) FMM_LAUNCH(c, k_fill_u8, grid_for(n), 256, 0, c.orb_grp.p, n, (unsigned char)0);
  // group table: rank ranges [lo, hi) and global counts
  struct G { int lo, hi; long long cnt; };
  std::vector<G> groups;
  if (!reuse) {
    c.orb_passes.clear();
    std::vector<int64_t> all = allgather_i64(c, n);
    long long N = 0;
    for (int64_t v : all) N += v;
    groups.push_back({0, P, N});
    c.orb_hist.reserve(kMaxGroups * 256);
    std::vector<unsigned long long> h(kMaxGroups * 256);
    for (int depth = 0; depth < 8; ++depth) {
      bool any = false;
      for (auto& g : groups) any |= g.hi - g.lo > 1;
      if (!any) break;
      OrbPass op{};
      op.ngroups = (int)groups.size();
      std::vector<long long> kth(groups.size(), 0);
      for (size_t gi = 0; gi < groups.size(); ++gi) {
        const int m = groups[gi].hi - groups[gi].lo;
        op.active[gi] = m > 1;
        op.axis[gi] = depth % 3;               // x, y, z, x, ...
        op.prefix[gi] = 0;
        kth[gi] = m > 1 ? groups[gi].cnt * (m / 2) / m : 0;
      }
      for (int pass = 0; pass < 8; ++pass) {    // radix select, 8 bits per pass from the top
        op.shift = 56 - 8 * pass;
        FMM_CUDA(cudaMemsetAsync(c.orb_hist.p, 0, sizeof(unsigned long long) * op.ngroups * 256, st));
        if (n > 0) FMM_LAUNCH(c, k_orb_hist, grid_for(n), 256, 0, pos, n, c.orb_grp.p, id0, op, c.orb_hist.p);
        allreduce_sum_u64(c, c.orb_hist.p, op.ngroups * 256);
        FMM_CUDA(cudaMemcpyAsync(h.data(), c.orb_hist.p, sizeof(unsigned long long) * op.ngroups * 256,
                                 cudaMemcpyDeviceToHost, st));
        FMM_CUDA(cudaStreamSynchronize(st));
        for (int gi = 0; gi < op.ngroups; ++gi) {
          if (!op.active[gi] || groups[gi].cnt == 0) continue;
          long long below = 0;
          int dg = 0;
          for (; dg < 256; ++dg) {
            const long long cnt = (long long)h[gi * 256 + dg];
            if (below + cnt > kth[gi]) break;
            below += cnt;
          }
          if (dg == 256) throw FmmError(FMM_E_INTERNAL, "ORB radix select: element not found");
          kth[gi] -= below;
          op.prefix[gi] |= (unsigned long long)dg << op.shift;
        }
      }
      // ties (reading Z28): when the selected element's coordinate is shared by
      // a plane of particles and only a sparse part of that plane (< 1/4) would
      // fall on one side, the cut moves to the plane's boundary (cost <= 5% of
      // a rank's share); otherwise the id tie-break keeps the split exact
      FMM_CUDA(cudaMemsetAsync(c.orb_hist.p, 0, sizeof(unsigned long long) * 2 * kMaxGroups, st));
      if (n > 0) FMM_LAUNCH(c, k_orb_tie, grid_for(n), 256, 0, pos, n, c.orb_grp.p, op, c.orb_hist.p);
      allreduce_sum_u64(c, c.orb_hist.p, 2 * kMaxGroups);
      FMM_CUDA(cudaMemcpyAsync(h.data(), c.orb_hist.p, sizeof(unsigned long long) * 2 * kMaxGroups,
                               cudaMemcpyDeviceToHost, st));
      FMM_CUDA(cudaStreamSynchronize(st));
      // relabel: active groups split into (low, high), the others keep one id
      std::vector<G> next;
      for (int gi = 0; gi < op.ngroups; ++gi) {
        const G g = groups[gi];
        if (!op.active[gi]) { op.lo_id[gi] = op.hi_id[gi] = (int)next.size(); next.push_back(g); continue; }
        const int m = g.hi - g.lo, m1 = m / 2;
        long long nlow = g.cnt * m1 / m;
        const long long below = (long long)h[2 * gi], plane = (long long)h[2 * gi + 1];
        const unsigned long long cs = op.prefix[gi] >> 32;
        if (g.cnt > 0 && plane > 1 && cs < 0xffffffffull) {
          const long long dlo = nlow - below, dhi = below + plane - nlow;
          const long long shift = std::min(dlo, dhi);
          if (4 * shift < plane && 20 * shift <= g.cnt / m) {
            if (dlo <= dhi) { op.prefix[gi] = cs << 32; nlow = below; }
            else { op.prefix[gi] = (cs + 1) << 32; nlow = below + plane; }
          }
        }
        op.lo_id[gi] = (int)next.size();
        next.push_back({g.lo, g.lo + m1, nlow});
        op.hi_id[gi] = (int)next.size();
        next.push_back({g.lo + m1, g.hi, g.cnt - nlow});
      }
      if ((int)next.size() > kMaxGroups) throw FmmError(FMM_E_INTERNAL, "ORB: too many groups");
      if (n > 0) FMM_LAUNCH(c, k_orb_split, grid_for(n), 256, 0, pos, n, c.orb_grp.p, id0, op);
      c.orb_passes.push_back(op);
      groups.swap(next);
    }
    c.orb_owner.clear();
    for (auto& g : groups) c.orb_owner.push_back(g.lo);
  } else {
    for (const OrbPass& op : c.orb_passes)
      if (n > 0) FMM_LAUNCH(c, k_orb_split, grid_for(n), 256, 0, pos, n, c.orb_grp.p, id0, op);
  }
  owner_of_group = c.orb_owner;
}

// partition >= 1: ORB groups, then every caller particle to its owner.  On
// return c.px/pa/ps hold this rank's particles (receive order) and c.n_own
// their count; c.red_* describe the exchange for the way back.
void orb_redistribute(Ctx& c, int64_t n, const float* x, const float* a, const float* s, const float4* pos_wrapped) {
  cudaStream_t st = c.stream;
  const int P = c.cfg.nranks, R = c.cfg.rank;
  const bool reuse = !c.orb_passes.empty() && ((c.cfg.partition == 2 && c.orb_fixed) || c.orb_reuse_next);
  c.orb_reuse_next = false;
  std::vector<int> owner_of_group;
  orb_groups(c, pos_wrapped, n, reuse, owner_of_group);
  if (c.cfg.partition == 2) c.orb_fixed = true;
  OwnerMap om{};
  for (int g = 0; g < kMaxGroups; ++g) om.owner[g] = g < (int)owner_of_group.size() ? owner_of_group[g] : 0;
  // owners, grouped stably (send order), counts per peer
  c.red_okey.reserve(2 * std::max<int64_t>(n, 1));
  c.red_sidx.reserve(2 * std::max<int64_t>(n, 1));
  c.dflag.reserve(std::max(8, P));
  FMM_CUDA(cudaMemsetAsync(c.dflag.p, 0, sizeof(int) * P, st));
  uint32_t* okey = c.red_okey.p;
  uint32_t* iota = c.red_sidx.p + std::max<int64_t>(n, 1);
  if (n > 0) {
    FMM_LAUNCH(c, k_owner_keys, grid_for(n), 256, 0, c.orb_grp.p, n, om, okey, iota, c.dflag.p);
    uint32_t* kout = c.red_okey.p + std::max<int64_t>(n, 1);
    uint32_t* vout = c.red_sidx.p;
    const int nn = (int)n;
    cub_call(c, [&](void* tmp, size_t& bytes) {
      return cub::DeviceRadixSort::SortPairs(tmp, bytes, okey, kout, iota, vout, nn, 0, 4, st);
    });
  }
  std::vector<int> sc(P);
  FMM_CUDA(cudaMemcpyAsync(sc.data(), c.dflag.p, sizeof(int) * P, cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  c.red_scnt.assign(P, 0);
  for (int q = 0; q < P; ++q) c.red_scnt[q] = sc[q];
  c.red_rcnt = alltoall_i64(c, c.red_scnt);
  int64_t m = 0;
  for (int q = 0; q < P; ++q) m += c.red_rcnt[q];
  c.red_send.reserve(2 * std::max<int64_t>(n, 1));
  c.red_recv.reserve(2 * std::max<int64_t>(m, 1));
  if (n > 0) FMM_LAUNCH(c, k_red_pack, grid_for(n), 256, 0, c.red_sidx.p, n, pos_wrapped, a, c.red_send.p);
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
  c.px.reserve(3 * std::max<int64_t>(m, 1));
  c.pa.reserve(3 * std::max<int64_t>(m, 1));
  c.ps.reserve(std::max<int64_t>(m, 1));
  if (m > 0) FMM_LAUNCH(c, k_red_unpack, grid_for(m), 256, 0, c.red_recv.p, m, c.px.p, c.pa.p, c.ps.p);
  c.n_caller = n;
  c.n_own = m;
  (void)x;
  (void)s;
}

// results of this rank's own particles (u_loc, s_loc: local caller order) back
// to the ranks that passed them, into their caller order (u, s: device)
void orb_return(Ctx& c, const float* u_loc, const float* s_loc, float* u, float* s) {
  cudaStream_t st = c.stream;
  const int P = c.cfg.nranks, R = c.cfg.rank;
  const int64_t m = c.n_own, n = c.n_caller;
  c.ret_send.reserve(6 * std::max<int64_t>(m, 1));
  c.ret_recv.reserve(6 * std::max<int64_t>(n, 1));
  if (m > 0) FMM_LAUNCH(c, k_ret_pack, grid_for(m), 256, 0, u_loc, s_loc, m, c.ret_send.p);
  std::vector<int64_t> soff(P, 0), sb(P, 0), roff(P, 0), rb(P, 0);
  int64_t so = 0, ro = 0;
  for (int q = 0; q < P; ++q) {              // the reverse of orb_redistribute's exchange
    soff[q] = 24 * so;
    roff[q] = 24 * ro;
    sb[q] = q == R ? 0 : 24 * c.red_rcnt[q];
    rb[q] = q == R ? 0 : 24 * c.red_scnt[q];
    so += c.red_rcnt[q];
    ro += c.red_scnt[q];
  }
  if (c.red_rcnt[R] > 0)
    FMM_CUDA(cudaMemcpyAsync((char*)c.ret_recv.p + roff[R], (const char*)c.ret_send.p + soff[R], 24 * c.red_rcnt[R],
                             cudaMemcpyDeviceToDevice, st));
  alltoallv_bytes(c, c.ret_send.p, soff, sb, c.ret_recv.p, roff, rb);
  if (n > 0) FMM_LAUNCH(c, k_ret_unpack, grid_for(n), 256, 0, c.ret_recv.p, c.red_sidx.p, n, u, s);
}

}  // namespace fmmb
