// let.cu -- a14: the local essential tree exchange on B200s.
//
// Every rank holds the global octree structure (built from the all-gathered
// Morton keys, so global cell ids agree on all ranks) and traverses it for its
// own targets only.  The source cells of its M2L list that another rank owns
// need their multipole; the source leaves of its P2P list that another rank
// owns need their bodies.  That set is exactly the part of the global tree the
// rank must receive -- the LET -- so instead of the paper's conservative
// LET-MAC estimate (which "sends a larger portion ... than is
// exactly required" and needs the M2L fallback of Alg. 2 when it misses), the
// exchange here is exact and the fallback count is zero by construction:
//   1. mark remote sources (kind 1: multipole, kind 2: bodies),
//   2. group the requests by owner (stable radix sort on the owner rank),
//   3. grouped ncclSend/ncclRecv of the request ids (the paper's single
//      non-homogeneous all-to-all),
//   4. owners pack multipoles (3 x p(p+1)/2 complex) and bodies (x, sigma,
//      alpha) straight into the send buffer, one block per request,
//   5. grouped ncclSend/ncclRecv of the replies, unpacked into the global M
//      and particle arrays at the requested cells' slots.
#include <cub/cub.cuh>

#include "ctx.cuh"

namespace fmmb {

namespace {

__global__ void k_mark_remote(const uint64_t* __restrict__ lst, int64_t n, int kind, const int* __restrict__ begin,
                              const int* __restrict__ count, int64_t off, int64_t nloc, int* __restrict__ need) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)((lst[i] >> 5) & 0x7ffffff);
    const int64_t b = begin[s], e = b + count[s];
    if (!(b >= off && e <= off + nloc)) atomicOr(&need[s], kind);
  }
}

__global__ void k_need_flags(const int* __restrict__ need, int64_t nc, int* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = need[i] ? 1 : 0;
}

struct Offs { int64_t o[9]; int P; };

__device__ __forceinline__ int owner_of(const Offs& ro, int64_t b) {
  int q = 0;
  while (q + 1 < ro.P && b >= ro.o[q + 1]) ++q;
  return q;
}

// request word: cell id (27 bits) | kind << 27
__global__ void k_need_scatter(const int* __restrict__ need, const int* __restrict__ scan, int64_t nc,
                               const int* __restrict__ begin, Offs ro, int* __restrict__ ids, int* __restrict__ own) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x) {
    if (need[i]) {
      const int k = scan[i] - 1;
      ids[k] = (int)i | (need[i] << 27);
      own[k] = owner_of(ro, begin[i]);
    }
  }
}

__global__ void k_owner_hist(const int* __restrict__ own, int64_t n, int* __restrict__ hist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&hist[own[i]], 1);
}

__device__ __forceinline__ int64_t req_bytes(int word, const int* __restrict__ count, int64_t mb) {
  const int cell = word & 0x7ffffff, kind = word >> 27;
  return ((kind & 1) ? mb : 0) + ((kind & 2) ? 32ll * count[cell] : 0);
}

__global__ void k_req_sizes(const int* __restrict__ words, int64_t n, const int* __restrict__ count, int64_t mb,
                            int64_t* __restrict__ sz) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    sz[i] = req_bytes(words[i], count, mb);
}

// owner side: one block per received request
__global__ void k_let_pack(const int* __restrict__ words, const int64_t* __restrict__ off, const int* __restrict__ begin,
                           const int* __restrict__ count, const float2* __restrict__ M, int nc3,
                           const float4* __restrict__ pos, const float4* __restrict__ alp, int64_t mb,
                           char* __restrict__ out) {
  const int w = words[blockIdx.x];
  const int cell = w & 0x7ffffff, kind = w >> 27;
  char* dst = out + off[blockIdx.x];
  if (kind & 1) {
    const float2* src = M + (int64_t)cell * nc3;
    float2* d = (float2*)dst;
    for (int i = threadIdx.x; i < nc3; i += blockDim.x) d[i] = src[i];
    dst += mb;
  }
  if (kind & 2) {
    const int b = begin[cell], cnt = count[cell];
    float4* d = (float4*)dst;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      d[i] = pos[b + i];
      d[cnt + i] = alp[b + i];
    }
  }
}

// requester side: one block per own request (same order as sent)
__global__ void k_let_unpack(const int* __restrict__ words, const int64_t* __restrict__ off,
                             const int* __restrict__ begin, const int* __restrict__ count, float2* __restrict__ M,
                             int nc3, float4* __restrict__ pos, float4* __restrict__ alp, int64_t mb,
                             const char* __restrict__ in) {
  const int w = words[blockIdx.x];
  const int cell = w & 0x7ffffff, kind = w >> 27;
  const char* src = in + off[blockIdx.x];
  if (kind & 1) {
    float2* d = M + (int64_t)cell * nc3;
    const float2* s = (const float2*)src;
    for (int i = threadIdx.x; i < nc3; i += blockDim.x) d[i] = s[i];
    src += mb;
  }
  if (kind & 2) {
    const int b = begin[cell], cnt = count[cell];
    const float4* s = (const float4*)src;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      pos[b + i] = s[i];
      alp[b + i] = s[cnt + i];
    }
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

unsigned grid_for(int64_t n) {
  unsigned b = nblocks(n, 256);
  return b > 148 * 16 ? 148 * 16 : b;
}

}  // namespace

void let_exchange(Ctx& c) {
  const int P = c.cfg.nranks;
  c.let_bytes_sent = c.let_bytes_recv = c.let_cells = c.let_leaves = 0;
  if (P <= 1) return;
  cudaStream_t st = c.stream;
  const int64_t nc = c.ncells;
  const int nc3 = 3 * c.nc;
  const int64_t mb = ((int64_t)nc3 * 8 + 15) / 16 * 16;
  Offs ro{};
  ro.P = P;
  for (int q = 0; q <= P; ++q) ro.o[q] = c.rank_off[q];

  // 1. remote sources of this rank's lists
  c.need.reserve(nc);
  FMM_CUDA(cudaMemsetAsync(c.need.p, 0, sizeof(int) * nc, st));
  if (c.nm2l)
    FMM_LAUNCH(c, k_mark_remote, grid_for(c.nm2l), 256, 0, c.m2l.p, c.nm2l, 1, c.cells.begin.p, c.cells.count.p,
               c.off, c.nown, c.need.p);
  if (c.np2p)
    FMM_LAUNCH(c, k_mark_remote, grid_for(c.np2p), 256, 0, c.p2p.p, c.np2p, 2, c.cells.begin.p, c.cells.count.p,
               c.off, c.nown, c.need.p);
  // 2. compact (ascending cell id) and group by owner (stable)
  c.flags.reserve(nc);
  c.scan.reserve(nc);
  FMM_LAUNCH(c, k_need_flags, grid_for(nc), 256, 0, c.need.p, nc, c.flags.p);
  {
    int* fin = c.flags.p;
    int* fout = c.scan.p;
    int nn = (int)nc;
    cub_call(c, [&](void* tmp, size_t& bytes) { return cub::DeviceScan::InclusiveSum(tmp, bytes, fin, fout, nn, st); });
  }
  int nreq = 0;
  FMM_CUDA(cudaMemcpyAsync(&nreq, c.scan.p + nc - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  c.need_ids.reserve(nreq + 1); c.need_ids2.reserve(nreq + 1);
  c.req_owner.reserve(nreq + 1); c.req_owner2.reserve(nreq + 1);
  if (nreq > 0) {
    FMM_LAUNCH(c, k_need_scatter, grid_for(nc), 256, 0, c.need.p, c.scan.p, nc, c.cells.begin.p, ro, c.need_ids.p,
               c.req_owner.p);
    int *kin = c.req_owner.p, *kout = c.req_owner2.p, *vin = c.need_ids.p, *vout = c.need_ids2.p;
    int nn = nreq;
    cub_call(c, [&](void* tmp, size_t& bytes) {
      return cub::DeviceRadixSort::SortPairs(tmp, bytes, kin, kout, vin, vout, nn, 0, 4, st);
    });
  }
  std::vector<int> hist(P, 0);
  c.dflag.reserve(16);
  FMM_CUDA(cudaMemsetAsync(c.dflag.p, 0, sizeof(int) * P, st));
  if (nreq > 0) FMM_LAUNCH(c, k_owner_hist, grid_for(nreq), 256, 0, c.req_owner2.p, nreq, c.dflag.p);
  FMM_CUDA(cudaMemcpyAsync(hist.data(), c.dflag.p, sizeof(int) * P, cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));

  // 3. request counts and ids
  std::vector<int64_t> scnt(P), soff(P, 0);
  for (int q = 0; q < P; ++q) { scnt[q] = hist[q]; if (q) soff[q] = soff[q - 1] + scnt[q - 1]; }
  std::vector<int64_t> rcnt = alltoall_i64(c, scnt), roff(P, 0);
  for (int q = 1; q < P; ++q) roff[q] = roff[q - 1] + rcnt[q - 1];
  const int64_t nin = roff[P - 1] + rcnt[P - 1];
  c.req_in.reserve(nin + 1);
  {
    std::vector<int64_t> sb(P), so(P), rb(P), rof(P);
    for (int q = 0; q < P; ++q) { sb[q] = 4 * scnt[q]; so[q] = 4 * soff[q]; rb[q] = 4 * rcnt[q]; rof[q] = 4 * roff[q]; }
    alltoallv_bytes(c, c.need_ids2.p, so, sb, c.req_in.p, rof, rb);
  }

  // 4. reply layout: owner side (received requests) and requester side (own requests)
  c.req_off.reserve(nin + nreq + 2);
  int64_t* in_sz = c.req_off.p;              // [nin] sizes then exclusive offsets (in place via scan)
  int64_t* my_sz = c.req_off.p + nin + 1;    // [nreq]
  if (nin > 0) FMM_LAUNCH(c, k_req_sizes, grid_for(nin), 256, 0, c.req_in.p, nin, c.cells.count.p, mb, in_sz);
  if (nreq > 0) FMM_LAUNCH(c, k_req_sizes, grid_for(nreq), 256, 0, c.need_ids2.p, (int64_t)nreq, c.cells.count.p, mb, my_sz);
  // per-request byte offsets (exclusive scans, in place) and per-peer totals
  auto excl_scan = [&](int64_t* p, int64_t n) {
    if (n <= 0) return;
    int nn = (int)n;
    cub_call(c, [&](void* tmp, size_t& bytes) { return cub::DeviceScan::ExclusiveSum(tmp, bytes, p, p, nn, st); });
  };
  // totals first (need the sizes): copy sizes to host segment sums via a second scan copy
  std::vector<int64_t> in_sizes(nin), my_sizes(nreq);
  if (nin) FMM_CUDA(cudaMemcpyAsync(in_sizes.data(), in_sz, 8 * nin, cudaMemcpyDeviceToHost, st));
  if (nreq) FMM_CUDA(cudaMemcpyAsync(my_sizes.data(), my_sz, 8 * nreq, cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> sbytes(P, 0), sboff(P, 0), rbytes(P, 0), rboff(P, 0);
  for (int q = 0; q < P; ++q) {
    for (int64_t i = roff[q]; i < roff[q] + rcnt[q]; ++i) sbytes[q] += in_sizes[i];
    for (int64_t i = soff[q]; i < soff[q] + scnt[q]; ++i) rbytes[q] += my_sizes[i];
    if (q) { sboff[q] = sboff[q - 1] + sbytes[q - 1]; rboff[q] = rboff[q - 1] + rbytes[q - 1]; }
  }
  excl_scan(in_sz, nin);
  excl_scan(my_sz, nreq);
  const int64_t stot = sboff[P - 1] + sbytes[P - 1], rtot = rboff[P - 1] + rbytes[P - 1];
  c.let_send.reserve(stot + 16);
  c.let_recv.reserve(rtot + 16);
  if (nin > 0)
    FMM_LAUNCH(c, k_let_pack, (unsigned)nin, 128, 0, c.req_in.p, in_sz, c.cells.begin.p, c.cells.count.p, c.M.p, nc3,
               c.pos.p, c.alp.p, mb, c.let_send.p);
  // 5. replies
  alltoallv_bytes(c, c.let_send.p, sboff, sbytes, c.let_recv.p, rboff, rbytes);
  if (nreq > 0)
    FMM_LAUNCH(c, k_let_unpack, (unsigned)nreq, 128, 0, c.need_ids2.p, my_sz, c.cells.begin.p, c.cells.count.p, c.M.p,
               nc3, c.pos.p, c.alp.p, mb, c.let_recv.p);
  c.let_bytes_sent = stot;
  c.let_bytes_recv = rtot;
  int64_t ncell = 0, nleaf = 0;
  {
    std::vector<int> words(nreq);
    if (nreq) FMM_CUDA(cudaMemcpyAsync(words.data(), c.need_ids2.p, 4 * nreq, cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaStreamSynchronize(st));
    for (int w : words) { if ((w >> 27) & 1) ++ncell; if ((w >> 27) & 2) ++nleaf; }
  }
  c.let_cells = ncell;
  c.let_leaves = nleaf;
}

}  // namespace fmmb
