// ctx.cuh -- the library-owned context behind the opaque fmm_ctx handle, and
// the internal entry points of each pipeline stage.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "common.cuh"

namespace fmmb {

// Octree cells in canonical (level, key) order, SoA, int32 (a4).
struct Cells {
  DBuf<int> level, qx, qy, qz, begin, count, parent, child_begin, nchild, leaf;
  void reserve_keep(size_t n, size_t keep, cudaStream_t s) {
    DBuf<int>* all[] = {&level, &qx, &qy, &qz, &begin, &count, &parent, &child_begin, &nchild, &leaf};
    for (auto* b : all) b->grow_keep(n, keep, s);
  }
};

// a level whose cells all take the tensor-core M2L (m2l_tc.cu)
struct TcLevel {
  int lt = 0, D = 0, ntgt = 0, lb = 0, W = 0;
  int64_t tgt_off = 0, code_off = 0, op_off = 0, mask_off = 0;
};

enum Phase { PH_SET0, PH_KEYS, PH_SORT, PH_TREE, PH_EVAL0, PH_UP, PH_TRAV, PH_M2L, PH_P2P, PH_DOWN, PH_FIN, PH_N };

// one depth of the ORB recursive multisection (partition.cu)
constexpr int kMaxGroups = 8;
struct OrbPass {
  int ngroups;                          // groups of this depth
  int active[kMaxGroups];               // group is split at this depth
  int axis[kMaxGroups];                 // x, y, z, x, ...
  unsigned long long prefix[kMaxGroups];   // the selected element's key (low part: keys below it)
  int shift;                            // radix-select digit = (key >> shift) & 255
  int lo_id[kMaxGroups], hi_id[kMaxGroups];   // group ids of the next depth
};

// one segment of a grouped NCCL exchange
struct CommSeg {
  bool send;
  int peer;
  const void* ptr;
  int64_t bytes;
};

struct Ctx {
  fmm_config cfg{};
  int P = 10, nc = 55;
  cudaStream_t stream = nullptr, stream2 = nullptr;
  cudaStream_t mstream = nullptr;            // far field beside the near field (high priority)
  int concurrent = 0;                        // 0: M2L then P2P; 1: P2P first, M2L beside; 2: M2L first, P2P beside
  bool own_stream = false;
  std::string err;
  bool poisoned = false;

  // ---- multi-GPU (a14): local tree + LET forest (let.cu), ORB partition (partition.cu) ----
  void* comm = nullptr;                      // ncclComm_t
  cudaStream_t cstream = nullptr;            // LET exchange (overlaps the local near field)
  cudaEvent_t ev_up = nullptr, ev_let0 = nullptr, ev_let1 = nullptr, ev_p2p_loc = nullptr;
  DBuf<int64_t> comm_i64;
  DBuf<double> comm_f64;
  int64_t ntot = 0, off = 0;                 // particles over all ranks; off = 0 (kept for the stats)
  int64_t nloc_cells = 0;                    // cells of the local tree: ids [0, nloc_cells)
  int64_t nsrc = 0;                          // particle slots: local [0, n), received bodies [n, nsrc)
  std::vector<int64_t> loc_lo, loc_hi;       // per level: the local tree's cells
  // LET, send side (receiver-major records, fixed per set_particles)
  DBuf<uint64_t> let_rec, let_rec2;
  DBuf<unsigned char> let_dec;
  DBuf<int> let_recof, let_scell;
  DBuf<int64_t> let_boff, let_brec;
  DBuf<char> let_srec, let_rrec;
  int64_t let_nsend_rec = 0, let_nbrec = 0;
  std::vector<int64_t> let_nrec_s, let_nbody_s, let_nrec_r, let_nbody_r, let_cbase, let_bbase;
  std::vector<int> let_peer, let_roots, let_root_leaf;
  DBuf<float2> let_sM;
  DBuf<float4> let_sP, let_sA;
  DBuf<unsigned char> cflag;                 // [ncells] 2 = frontier (children not sent), 4 = leaf without bodies
  DBuf<unsigned long long> dfallback;
  int64_t let_fallback = 0;
  int64_t let_bytes_sent = 0, let_bytes_recv = 0, let_cells = 0, let_leaves = 0;
  double ms_let = 0.0, ms_let_exposed = 0.0;
  DBuf<float2> top_M;                        // root + level-1 multipoles, summed over ranks (a8, Z27)
  // ORB partition (cfg.partition >= 1)
  bool balanced = false, orb_fixed = false, orb_reuse_next = false;
  std::vector<OrbPass> orb_passes;
  std::vector<int> orb_owner;
  DBuf<unsigned char> orb_grp;
  DBuf<unsigned long long> orb_hist;
  DBuf<uint32_t> red_okey, red_sidx;         // send order: red_sidx[k] = caller index of send slot k
  DBuf<float4> red_send, red_recv;
  std::vector<int64_t> red_scnt, red_rcnt;
  DBuf<float> px, pa, ps;                    // this rank's particles after the redistribution
  int64_t n_caller = 0, n_own = 0, nown = 0, redist_bytes = 0;
  DBuf<float> ret_send, ret_recv, loc_u, loc_s;
  // tensor-core M2L source map for forests (m2l_tc.cu): level grid -> cell id
  DBuf<int> tc_map;
  bool tc_use_map = false;
  bool tc_mixed = false;                     // some taken cell keeps register-path entries (per-entry select)
  DBuf<unsigned char> tc_extra;
  std::vector<int64_t> tc_map_off;

  // ---- particles and tree (set_particles) ----
  int64_t n = 0;
  bool have_particles = false;
  double lo[3] = {0, 0, 0}, L = 1.0;         // key box: the root cube
  double per[3] = {1, 1, 1};                 // periods of the (tiled) periodic domain
  long long per_units[3] = {1ll << 22, 1ll << 22, 1ll << 22};   // periods in half-finest-cell units
  int tmax = 1;                              // largest tiles[d]
  DBuf<float> stage_x, stage_a, stage_s;    // host-input staging
  DBuf<float4> pos_tmp, pos, alp;           // sorted: (x,y,z,sigma), (alpha,0)
  DBuf<float4> posl;                         // leaf-local (x - c_leaf, 1/(2 sigma^2)) for P2P staging
  DBuf<uint64_t> keys_tmp, keys;
  DBuf<uint32_t> idx_tmp, idx;               // idx[i] = caller index of sorted slot i
  DBuf<unsigned char> cub_tmp;
  DBuf<int> pcell_a, pcell_b, flags, scan, dflag;
  DBuf<int> leaf_ids;
  DBuf<int> leaf_cls;                        // leaf ids by size class (P2P variants), counts below
  int64_t leaf_cls_n[3] = {0, 0, 0};
  bool leaf_cls_valid = false;
  Cells cells;
  int64_t ncells = 0, nleaves = 0;
  std::vector<int64_t> level_begin;          // cells of level l: [level_begin[l], level_begin[l+1])
  std::vector<int> host_leaf_top;            // leaf flags of levels 0..1 (far targets)

  // ---- lists (traversal) ----
  bool lists_valid = false;
  DBuf<uint64_t> p2p, m2l, sort_tmp, front_a, front_b;
  DBuf<uint64_t> m2lr;                       // M2L entries the register kernels take, grouped by target
  int64_t nm2lr = 0;
  DBuf<int> dsel;                            // selected-count output of cub::DeviceSelect
  DBuf<unsigned> tc_mask;                    // tensor-path verification: offset bitmask per cell
  DBuf<unsigned> tc_good, tc_hist;           // per M2L entry: taken by the tensor path (bit); offset histogram
  DBuf<unsigned char> tc_bad, tc_has;        // tc_has[t]: cell t has M2L entries (written by the traversal)
  DBuf<int64_t> tc_off;
  DBuf<int4> tc_cq;                          // packed (qx, qy, qz, level) for the verification
  DBuf<int> cnt_m2l, cnt_p2p, cnt_push, off_m2l, off_p2p, off_push;
  int64_t np2p = 0, nm2l = 0, p2p_pairs = 0;
  DBuf<int> p2p_b, p2p_e, p2p_m, m2l_b, m2l_e;   // p2p_m: first remote-source entry (nranks > 1)
  DBuf<unsigned long long> dcount, dnear;
  int64_t p2p_near_pairs = 0;                // pairs of the last P2P on regularised tiles
  // tensor-core M2L (m2l_tc.cu): decided once per list build
  bool tc_valid = false;
  std::vector<TcLevel> tc_levels;
  int64_t tc_entries = 0;                    // M2L list entries handled by the tensor path
  DBuf<unsigned char> tc_skip;               // [ncells] 1 = the register kernel skips the cell
  DBuf<int> tc_tmp, tc_codes_tmp, tc_tgt, tc_tgt2, tc_codes, tc_cnt;
  DBuf<float> tc_mp;                         // packed multipoles [cell][3][112] for the row gathers
  DBuf<short> tc_tbl;
  DBuf<unsigned char> tc_op;                 // pre-split operators, [level][d][K-block][hi|lo]
  std::vector<int> tc_op_sig;                // (level, D, offsets) the operators were built for

  // ---- expansions and results ----
  DBuf<float2> M, Lc;                        // [ncells][3][nc], normalised (Z18)
  DBuf<float2> r8;                           // R_n^m of the 8 child-octant shifts (M2M, L2L)
  int r8_order = 0;
  DBuf<double> far_M;                        // periodic super-cell multipoles
  DBuf<double2> far_part;                    // per-chunk partial far-field locals
  DBuf<int> far_tg;                          // far-field target cells
  int far_ntg = 0, far_nchunk = 0;
  DBuf<float> u_near, s_near, u_far, s_far;  // sorted order, [n][3]
  DBuf<float> stage_u, stage_ds;             // host-output staging
  bool evaluated = false;
  int64_t far_m2l = 0;

  // ---- counters ----
  int64_t launches = 0, cub_calls = 0;       // since the last set_particles

  // ---- time step (NEXT-1) ----
  DBuf<float> st_x, st_a, st_s, st_u, st_da, st_xh, st_ah, st_sh;

  // ---- RBF reinitialisation (NEXT-4) ----
  DBuf<double> rbf_b, rbf_v, rbf_x, rbf_r, rbf_p, rbf_ap, rbf_dot;
  DBuf<float4> rbf_q;

  // ---- timing ----
  cudaEvent_t ev[PH_N + 1] = {};
  cudaEvent_t ev_fork = nullptr, ev_trav = nullptr;   // upward-pass / traversal overlap
  cudaEvent_t ev_m2l[3] = {};                          // M2L sub-phases: start, tensor done, register done
  cudaEvent_t ev_far = nullptr;                        // far layers (phase 1) done on the side stream
  bool overlapped = false;
  fmm_stats stats{};
};

// pipeline stages (each enqueues on ctx.stream; throws FmmError)
void set_particles_impl(Ctx& c, int64_t n, const float* x, const float* a, const float* s);
void build_lists(Ctx& c);
void m2l_reg_segments(Ctx& c);
void upward_pass(Ctx& c);
void m2l_pass(Ctx& c);
bool m2l_pass_reg(Ctx& c);
void m2l_tc_prepare(Ctx& c);
void m2l_tc_run(Ctx& c);
bool l2p_pass_reg(Ctx& c, float* u_far, float* s_far);
bool p2m_pass_reg(Ctx& c);
bool m2m_level_reg(Ctx& c, int64_t first, int64_t cnt, const float2* R8);
bool l2l_level_reg(Ctx& c, int64_t pfirst, int64_t pcnt, int64_t clo, int64_t chi, const float2* R8);
void comm_init(Ctx& c);
void comm_unique_id(void* out);
void comm_destroy(Ctx& c);
std::vector<int64_t> allgather_i64(Ctx& c, int64_t v);
std::vector<int64_t> alltoall_i64(Ctx& c, const std::vector<int64_t>& send);
void alltoallv_bytes(Ctx& c, const void* sbuf, const std::vector<int64_t>& soff, const std::vector<int64_t>& sbytes,
                     void* rbuf, const std::vector<int64_t>& roff, const std::vector<int64_t>& rbytes);
void allreduce_sum_f32(Ctx& c, float* p, int64_t n, cudaStream_t st = nullptr);
void allreduce_sum_u64(Ctx& c, unsigned long long* p, int64_t n);
std::vector<double> allgather_f64(Ctx& c, const double* v, int n);
void alltoallv_multi(Ctx& c, const std::vector<CommSeg>& segs, cudaStream_t st);
void let_setup(Ctx& c);
void let_exchange(Ctx& c, cudaStream_t cs);
void top_multipoles(Ctx& c, cudaStream_t cs);
void bbox_of(Ctx& c, const float4* pos, int64_t n, float out[6]);
void orb_redistribute(Ctx& c, int64_t n, const float* x, const float* a, const float* s, const float4* pos_wrapped);
void orb_return(Ctx& c, const float* u_loc, const float* s_loc, float* u, float* s);
void step_stage_update(Ctx& c, const float* x, const float* a, const float* s, const float* u, const float* da,
                       int64_t n, double h, double two_nu_t, float* xo, float* ao, float* so);
void periodic_far_pass(Ctx& c, int phase = 3);
void fill_f32(Ctx& c, float* p, int64_t n, float v);
void downward_pass(Ctx& c, float* u_far, float* s_far);
void p2p_pass(Ctx& c, float* u_near, float* s_near, int part = 0);   // part: 0 all, 1 local sources, 2 remote (adds)
void eval_cutoff(Ctx& c, const float* rho, int64_t n, float* g);
void eval_pair_kernel(Ctx& c, const float* rho, int64_t n, int branch, float* g, float* rgp);
void gauss_pass(Ctx& c, const float4* q, double* out);
void rbf_reinit_impl(Ctx& c, int64_t n, const float* x, const float* alpha, const float* sigma, int64_t m,
                     const float* y, float sigma0, double tol, int maxit, float* beta_out, int* iters, double* resid);

}  // namespace fmmb

struct fmm_ctx {
  fmmb::Ctx c;
};
