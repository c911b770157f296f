// comm.cu -- the multi-GPU plumbing of a14: one NCCL communicator
// per context (the 128-byte ncclUniqueId is broadcast by the caller, e.g. with
// torch.distributed), all collectives enqueued on the library stream.
//
// The paper sends the whole LET with one non-homogeneous MPI_Alltoallv
// (P:192).  NCCL 2.28 has no alltoallv, so every variable-size
// exchange here is a grouped ncclSend/ncclRecv (ncclGroupStart/End) over
// NVLink/NVSwitch.
#include <nccl.h>

#include "ctx.cuh"

namespace fmmb {

#define FMM_NCCL(x)                                                                              \
  do {                                                                                           \
    ncclResult_t r_ = (x);                                                                       \
    if (r_ != ncclSuccess)                                                                       \
      throw FmmError(FMM_E_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_) + " at " +      \
                                     __FILE__ + ":" + std::to_string(__LINE__));                 \
  } while (0)

void comm_init(Ctx& c) {
  if (c.cfg.nranks <= 1) return;
  if (!c.cfg.nccl_id) throw FmmError(FMM_E_ARG, "nranks > 1 needs cfg.nccl_id");
  ncclUniqueId id;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(&id, c.cfg.nccl_id, sizeof(id));
  ncclComm_t comm;
  FMM_NCCL(ncclCommInitRank(&comm, c.cfg.nranks, id, c.cfg.rank));
  c.comm = (void*)comm;
}

void comm_unique_id(void* out) {
  ncclUniqueId id;
  FMM_NCCL(ncclGetUniqueId(&id));
  memcpy(out, &id, sizeof(id));
}

void comm_destroy(Ctx& c) {
  if (c.comm) ncclCommDestroy((ncclComm_t)c.comm);
  c.comm = nullptr;
}

// every rank contributes one int64; returns all of them (host), synchronous
std::vector<int64_t> allgather_i64(Ctx& c, int64_t v) {
  const int P = c.cfg.nranks;
  c.comm_i64.reserve(2 * P);
  FMM_CUDA(cudaMemcpyAsync(c.comm_i64.p + c.cfg.rank, &v, sizeof(int64_t), cudaMemcpyHostToDevice, c.stream));
  FMM_NCCL(ncclAllGather(c.comm_i64.p + c.cfg.rank, c.comm_i64.p, 1, ncclInt64, (ncclComm_t)c.comm, c.stream));
  std::vector<int64_t> out(P);
  FMM_CUDA(cudaMemcpyAsync(out.data(), c.comm_i64.p, sizeof(int64_t) * P, cudaMemcpyDeviceToHost, c.stream));
  FMM_CUDA(cudaStreamSynchronize(c.stream));
  return out;
}

// send[q] int64 to every peer q, receive recv[q] from every q (alltoall of one value), synchronous
std::vector<int64_t> alltoall_i64(Ctx& c, const std::vector<int64_t>& send) {
  const int P = c.cfg.nranks;
  c.comm_i64.reserve(2 * P);
  FMM_CUDA(cudaMemcpyAsync(c.comm_i64.p, send.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice, c.stream));
  FMM_NCCL(ncclGroupStart());
  for (int q = 0; q < P; ++q) {
    FMM_NCCL(ncclSend(c.comm_i64.p + q, 1, ncclInt64, q, (ncclComm_t)c.comm, c.stream));
    FMM_NCCL(ncclRecv(c.comm_i64.p + P + q, 1, ncclInt64, q, (ncclComm_t)c.comm, c.stream));
  }
  FMM_NCCL(ncclGroupEnd());
  std::vector<int64_t> out(P);
  FMM_CUDA(cudaMemcpyAsync(out.data(), c.comm_i64.p + P, sizeof(int64_t) * P, cudaMemcpyDeviceToHost, c.stream));
  FMM_CUDA(cudaStreamSynchronize(c.stream));
  return out;
}

// byte-granular alltoallv: send[q] = (offset, bytes) into sbuf, recv[q] into rbuf (stream-ordered)
void alltoallv_bytes(Ctx& c, const void* sbuf, const std::vector<int64_t>& soff, const std::vector<int64_t>& sbytes,
                     void* rbuf, const std::vector<int64_t>& roff, const std::vector<int64_t>& rbytes) {
  const int P = c.cfg.nranks;
  FMM_NCCL(ncclGroupStart());
  for (int q = 0; q < P; ++q) {
    if (sbytes[q] > 0)
      FMM_NCCL(ncclSend((const char*)sbuf + soff[q], (size_t)sbytes[q], ncclChar, q, (ncclComm_t)c.comm, c.stream));
    if (rbytes[q] > 0)
      FMM_NCCL(ncclRecv((char*)rbuf + roff[q], (size_t)rbytes[q], ncclChar, q, (ncclComm_t)c.comm, c.stream));
  }
  FMM_NCCL(ncclGroupEnd());
}

void allreduce_sum_f32(Ctx& c, float* p, int64_t n, cudaStream_t st) {
  FMM_NCCL(ncclAllReduce(p, p, (size_t)n, ncclFloat32, ncclSum, (ncclComm_t)c.comm, st ? st : c.stream));
}

void allreduce_sum_u64(Ctx& c, unsigned long long* p, int64_t n) {
  FMM_NCCL(ncclAllReduce(p, p, (size_t)n, ncclUint64, ncclSum, (ncclComm_t)c.comm, c.stream));
}

// every rank's n doubles (host in, host out [P][n]), synchronous
std::vector<double> allgather_f64(Ctx& c, const double* v, int n) {
  const int P = c.cfg.nranks;
  c.comm_f64.reserve((size_t)P * n);
  FMM_CUDA(cudaMemcpyAsync(c.comm_f64.p + (size_t)c.cfg.rank * n, v, sizeof(double) * n, cudaMemcpyHostToDevice,
                           c.stream));
  FMM_NCCL(ncclAllGather(c.comm_f64.p + (size_t)c.cfg.rank * n, c.comm_f64.p, (size_t)n, ncclFloat64,
                         (ncclComm_t)c.comm, c.stream));
  std::vector<double> out((size_t)P * n);
  FMM_CUDA(cudaMemcpyAsync(out.data(), c.comm_f64.p, sizeof(double) * P * n, cudaMemcpyDeviceToHost, c.stream));
  FMM_CUDA(cudaStreamSynchronize(c.stream));
  return out;
}

// grouped send/recv of several (buffer, bytes) segments per peer in one NCCL group, on stream st
void alltoallv_multi(Ctx& c, const std::vector<CommSeg>& segs, cudaStream_t st) {
  FMM_NCCL(ncclGroupStart());
  for (const CommSeg& g : segs) {
    if (g.bytes <= 0) continue;
    if (g.send) FMM_NCCL(ncclSend(g.ptr, (size_t)g.bytes, ncclChar, g.peer, (ncclComm_t)c.comm, st));
    else FMM_NCCL(ncclRecv((void*)g.ptr, (size_t)g.bytes, ncclChar, g.peer, (ncclComm_t)c.comm, st));
  }
  FMM_NCCL(ncclGroupEnd());
}

}  // namespace fmmb
