/*
 * fmm.h -- C ABI of the B200-native FMM evaluator for the vortex particle
 * method of Yokota, Barba, Narumi & Yasuoka, "Petascale turbulence simulation
 * using a highly parallel fast multipole method on GPUs" (arXiv 1106.5273).
 * Citations "P:n" are lines of that paper's text; "Zn" are the
 * readings of ambiguous passages listed in DESIGN.md.
 *
 * What the library computes.  For N vortex particles with positions
 * x_j, strengths alpha_j (= gamma_j, Eq. 1) and core widths sigma_j:
 *
 *   u_i         = sum_j alpha_j x grad G g_sigma              (Eq. 1)
 *   dalpha_i/dt = sum_j grad(alpha_j x grad G g_sigma).alpha_i (Eq. 3)
 *
 * with G = 1/(4 pi r), g the Gaussian cutoff of Eq. 2 evaluated with the
 * source's sigma_j (Z4), the physical sign u_i = sum g alpha_j x (x_i - x_j) /
 * (4 pi r^3) (Z1), the classical stretching (alpha_i . grad) u (Z3), and pairs
 * at r = 0 contributing nothing (Z7).  Sources = targets = the set particles.
 * The sums are evaluated by the FMM: Morton-key octree,
 * dual tree traversal (Alg. 1-2) emitting P2P and M2L lists,
 * spherical-harmonic expansions of order p (Z8), and -- when
 * images > 0 -- the periodic cube [lo, lo+L)^3 with 3^k image boxes per
 * dimension (Z14).  The far field uses the singular kernel
 * (Z5).  All kernels run on the GPU in FP32 with FP64 accumulation of P2P tile
 * partials ("single precision ... double-precision accuracy").
 *
 * Conventions for every call:
 *  - Return value: fmm_status, FMM_OK == 0.  No C++ exception crosses the ABI.
 *    fmm_last_error(ctx) returns a message for the last failing call.
 *  - Arrays: contiguous, row-major FP32.  A pointer may be device memory on
 *    cfg.device or host memory (pageable or pinned); the library detects which
 *    with cudaPointerGetAttributes and copies host data itself.
 *  - Stream ordering: all work runs on cfg.stream.  With cfg.stream == NULL the
 *    library creates a *blocking* stream, which is ordered with the legacy
 *    default stream (where torch's default stream enqueues): inputs written
 *    there are complete before the library reads them.  With a caller stream,
 *    the caller orders its producers/consumers with that stream.
 *  - Ownership: the caller owns every array it passes.  set_particles copies
 *    its inputs and returns after validation; evaluate overwrites the caller's
 *    output arrays and returns when they are valid (stream synchronised).
 *  - After FMM_E_CUDA, FMM_E_NCCL or FMM_E_INTERNAL the context is poisoned:
 *    only fmm_destroy is legal (further calls return FMM_E_STATE).
 *  - One host thread per context.  No CPU fallback exists: every step of the
 *    evaluation runs in this library's CUDA kernels.
 */
#ifndef FMM_B200_H
#define FMM_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fmm_ctx fmm_ctx;

typedef enum {
  FMM_OK = 0,
  FMM_E_ARG = 1,        /* bad config, null pointer with n > 0, n < 0          */
  FMM_E_NONFINITE = 2,  /* non-finite x, alpha or sigma                 */
  FMM_E_SIGMA = 3,      /* sigma <= 0                                   */
  FMM_E_STATE = 4,      /* evaluate before set_particles; poisoned context     */
  FMM_E_OOM = 5,        /* device allocation failed                            */
  FMM_E_CUDA = 6,       /* CUDA runtime error (context poisoned)               */
  FMM_E_NCCL = 7,       /* NCCL error (context poisoned)                       */
  FMM_E_INTERNAL = 8,   /* invariant violated (context poisoned)               */
  FMM_E_NOCONV = 9      /* fmm_rbf_reinit: CG reached maxit above tol; the
                           outputs hold the last iterate and its residual       */
} fmm_status;

typedef struct {
  uint32_t struct_size;          /* = sizeof(fmm_config): ABI versioning              */
  int32_t  order;                /* p: degrees n = 0..p-1 (Z8); default 10; 2 <= p <= 16 */
  int32_t  theta_num, theta_den; /* MAC r_A + r_B < theta R (Z9); theta = num/den,
                                    1 <= num < den <= 64; default 1/2                  */
  int32_t  ncrit;                /* leaf iff count <= ncrit or level 21 (Z13); dflt 64 */
  int32_t  images;               /* k: 3^k image boxes per dimension (Z14);
                                    0 = free space; 0 <= k <= 6; default 3             */
  double   box_lo[3], box_len;   /* periodic cell (images > 0): default lo = -pi,
                                    L = 2 pi; ignored in free space (Z16)      */
  int32_t  traversal;            /* 0 = MAC-first (default), 1 = leaf-first (Z11)      */
  int32_t  device;               /* CUDA ordinal                                       */
  void*    stream;               /* cudaStream_t for all work; NULL = library-owned    */
  int32_t  rank, nranks;         /* 1 <= nranks <= 8 (one NVLink node), one rank per GPU;
                                    nranks > 1 needs images >= 1 (see partition)       */
  const void* nccl_id;           /* 128-byte ncclUniqueId when nranks > 1 (all ranks
                                    pass the same id, e.g. broadcast by torch.distributed) */
  int32_t  tiles[3];             /* periodic domain of tiles[d] cubes of side box_len per
                                    axis (reading Z27, weak scaling); tiles[d] in {1, 2},
                                    default (1,1,1).  Tile t is top-level octant t of the
                                    root cube (x fastest); any rank may hold any part  */
  int32_t  m2l_path;             /* 0 (default): tensor-core M2L (tcgen05, 3xTF32) on the
                                    levels whose cells share one offset set, register
                                    kernel elsewhere; 1: register (CUDA-core) kernel only */
  int32_t  partition;            /* multi-GPU domain decomposition (a14, NEXT-3):
                                    0 (default): every rank's targets are the particles it
                                    passes (e.g. its octant blocks or tiles);
                                    1: ORB recursive multisection at every
                                    set_particles -- the particles (any distribution, any
                                    subset per rank) are split at the nth element of x,
                                    y, z, ... (distributed radix select, NCCL all-reduce of
                                    histograms) into nranks equal-count boxes and moved to
                                    their owners; evaluate returns every rank its own
                                    particles' results in its caller order;
                                    2: as 1, with the cuts of the first set_particles kept
                                    ("the partitioning is performed only once").
                                    Every rank then builds the octree of its own particles
                                    and exchanges local essential trees      */
} fmm_config;

/* Per-phase device times of the last set_particles / evaluate (CUDA events on
 * the library stream, ms) and the work counters of the last evaluate. */
typedef struct {
  uint32_t struct_size;          /* = sizeof(fmm_stats)                                */
  int64_t  n, ncells, nleaves, nlevels;
  int64_t  p2p_list, m2l_list;   /* list entries (cell pairs)                          */
  int64_t  p2p_pairs;            /* particle pairs evaluated by P2P                    */
  int64_t  far_m2l;              /* M2L of the periodic far layers (a8)                */
  double   model_flops;          /* 174 * p2p_pairs (Table 1)               */
  int64_t  launches;             /* this library's kernel launches since set_particles */
  int64_t  cub_calls;            /* CUB device-wide calls (radix sort, scan) since then */
  int64_t  p2p_near_pairs;       /* pairs of P2P tiles evaluated with the cutoff g (the
                                    rest took the exact singular branch, rho >= 4.6)   */
  double   ms_keys, ms_sort, ms_tree;                  /* set_particles: a1-a4         */
  double   ms_upward, ms_traverse, ms_m2l, ms_p2p, ms_downward, ms_finalize;
  double   ms_set_total, ms_eval_total;
  /* multi-GPU (a14): global particle count and the last LET exchange */
  int64_t  ntot;
  int64_t  let_bytes_sent, let_bytes_recv;  /* reply payload bytes                       */
  int64_t  let_cells, let_leaves;           /* remote multipoles / leaves received         */
  double   ms_let;                          /* exchange time (CUDA events, incl. requests) */
  int64_t  m2l_tc_list;                     /* M2L entries evaluated on the tensor cores    */
  int64_t  own_begin, own_count;            /* global sorted positions this rank owns        */
  int64_t  redist_bytes;                    /* partition = 1: particle bytes sent by set_particles */
  int64_t  m2l_reg_list;                    /* M2L entries evaluated by the register (CUDA-core) kernel */
  double   ms_m2l_tc, ms_m2l_reg;           /* M2L phase split: tensor-core kernel (+ its pack), register kernel */
  double   ms_let_exposed;                  /* LET wait of the main stream after the local near field */
  int64_t  let_fallback;                    /* pairs resolved by Alg. 2's remote branch (M2L with the
                                               smallest cell received): 0 = complete LET */
  int64_t  nranks;
  int64_t  ncells_local;                    /* cells of this rank's own tree (ids [0, ncells_local));
                                               the rest of ncells are the peers' LETs          */
} fmm_stats;

/* Fill cfg with the defaults listed above. */
void fmm_config_default(fmm_config* cfg);

/* Create a context on cfg->device.  Errors: FMM_E_ARG (invalid field),
 * FMM_E_CUDA, FMM_E_NCCL.  *out is NULL on failure. */
fmm_status fmm_create(const fmm_config* cfg, fmm_ctx** out);

/* a1-a4: copy and validate n particles -- x[n][3], alpha[n][3],
 * sigma[n] -- wrap them into the periodic cell when images > 0, build
 * 63-bit Morton keys (Z16), radix-sort them (stable, Z17) and
 * build the octree.  n = 0 is valid.  Errors: FMM_E_ARG,
 * FMM_E_NONFINITE, FMM_E_SIGMA, FMM_E_OOM, FMM_E_CUDA. */
fmm_status fmm_set_particles(fmm_ctx* ctx, int64_t n, const float* x,
                             const float* alpha, const float* sigma);

/* a5-a13: P2M, M2M, dual tree traversal, periodic far field, M2L, L2L, L2P,
 * P2P; writes u[n][3] (Eq. 1) and dalpha_dt[n][3] (Eq. 3) in the caller's
 * particle order (overwrite, Z28).  Errors: FMM_E_STATE, FMM_E_ARG, FMM_E_CUDA. */
fmm_status fmm_evaluate(fmm_ctx* ctx, float* u, float* dalpha_dt);

/* As fmm_evaluate but writes only the selected parts: bit 0 = near field
 * (P2P), bit 1 = far field (M2L/L2L/L2P incl. periodic layers).  parts = 3 is
 * fmm_evaluate.  Used by the parity tests (near field on identical lists). */
fmm_status fmm_evaluate_parts(fmm_ctx* ctx, int32_t parts, float* u, float* dalpha_dt);

fmm_status fmm_destroy(fmm_ctx* ctx);
const char* fmm_last_error(const fmm_ctx* ctx);
fmm_status fmm_get_stats(const fmm_ctx* ctx, fmm_stats* s);

/* ---- inspection (tests): host output arrays, valid after set_particles ---- */
/* Sizes; lists are built by the first evaluate after set_particles, or here. */
fmm_status fmm_get_sizes(fmm_ctx* ctx, int64_t* ncells, int64_t* np2p, int64_t* nm2l);
/* Key box: lo[3] and side L (periodic cell, or the bounding cube, Z16). */
fmm_status fmm_get_box(const fmm_ctx* ctx, double* lo, double* L);
/* keys[n] sorted ascending and perm[n] = caller index of sorted slot i. */
fmm_status fmm_get_keys(const fmm_ctx* ctx, uint64_t* keys, int64_t* perm);
/* cells[ncells][10] = level, qx, qy, qz, begin, count, parent, child_begin,
 * nchild, is_leaf in canonical (level, key) order; child_begin = -1 for leaves. */
fmm_status fmm_get_cells(const fmm_ctx* ctx, int64_t* cells);
/* p2p[np2p][3], m2l[nm2l][3] = (target cell, source cell, image index) sorted
 * by (target, source, image); image index = (ix+1) + 3(iy+1) + 9(iz+1). */
fmm_status fmm_get_lists(fmm_ctx* ctx, int64_t* p2p, int64_t* m2l);
/* Normalised expansions after evaluate (Z18): M~_n = M_n / s^n,
 * L~_n = L_n s^(n+1), s = cell side; [ncells][3][p(p+1)/2] complex FP32
 * (interleaved re, im) -- either pointer may be NULL. */
fmm_status fmm_get_expansions(const fmm_ctx* ctx, float* M, float* L);

/* NEXT-1: one vortex-method time step around the evaluation:
 * midpoint RK2 -- (u1, s1) = FMM(x, alpha, sigma); x_h = x + dt/2 u1,
 * alpha_h = alpha + dt/2 s1, sigma_h^2 = sigma^2 + nu dt; (u2, s2) =
 * FMM(x_h, alpha_h, sigma_h); x += dt u2, alpha += dt s2, sigma^2 += 2 nu dt
 * (Eq. 4, exact).  x[n][3], alpha[n][3], sigma[n] are read and overwritten
 * (host or device).  Single GPU in this build.  Errors: FMM_E_ARG, plus those
 * of set_particles / evaluate. */
fmm_status fmm_step(fmm_ctx* ctx, int64_t n, float* x, float* alpha, float* sigma, double dt, double nu);

/* NEXT-2 (the paper's second FMM workload, velocity on a uniform
 * lattice for spectra): the velocity of Eq. 1 at nt target points
 * y[nt][3] that carry no vorticity, induced by the n particles (x, alpha,
 * sigma) given here.  Evaluated as one FMM over the union of the particles and
 * the targets (targets enter with alpha = 0, so they change no sum; their
 * positions shape the tree exactly as extra particles would).  Writes
 * u[nt][3] (overwrite); pointers may be device or host memory.  The context
 * then holds the union as its particle set (as after fmm_set_particles).
 * Single-GPU in this build.  Errors: as fmm_set_particles / fmm_evaluate. */
fmm_status fmm_evaluate_targets(fmm_ctx* ctx, int64_t n, const float* x, const float* alpha,
                                const float* sigma, int64_t nt, const float* y, float* u);

/* NEXT-4: radial-basis-function reinitialisation of the particle
 * field onto m new sites ("radial basis function interpolation for
 * reinitialized Gaussian distributions"; the sites are the same every
 * time, so their tree is reused).  With the Gaussian core of Eq. 2,
 * zeta_s(r) = (2 pi s^2)^(-3/2) exp(-r^2 / (2 s^2)), the old field's vorticity at
 * site i is b_i = sum_j alpha_j zeta_{sigma_j}(y_i - x_j) (periodic images as the
 * config's first layer) and the new strengths beta[m][3] (core sigma0 on every
 * site) solve sum_k beta_k zeta_{sigma0}(y_i - y_k) = b_i by conjugate gradients
 * (A is symmetric positive definite) to ||b - A beta|| <= tol ||b||, at most
 * maxit iterations.  Both sums run over the P2P lists of the tree (DESIGN.md
 * reading R1).  Inputs x[n][3], alpha[n][3], sigma[n], y[m][3]; output
 * beta[m][3] in the order of y (overwrite); pointers host or device.  *iters
 * and *resid (may be NULL) receive the iteration count and the final relative
 * residual.  Afterwards the context holds the sites with strengths beta and
 * core sigma0 (evaluate may follow).  Single GPU in this build.  Errors:
 * FMM_E_ARG (bad arguments, nranks > 1, sigma0 <= 0, tol <= 0, maxit < 1),
 * FMM_E_NOCONV (maxit reached above tol; outputs hold the last iterate), and
 * those of set_particles. */
fmm_status fmm_rbf_reinit(fmm_ctx* ctx, int64_t n, const float* x, const float* alpha, const float* sigma,
                          int64_t m, const float* y, float sigma0, double tol, int32_t maxit, float* beta,
                          int32_t* iters, double* resid);

/* Multi-GPU bootstrap: writes a fresh 128-byte ncclUniqueId into id (one rank
 * calls it and broadcasts the bytes to the others, e.g. via torch.distributed;
 * every rank then passes them as fmm_config.nccl_id).  Errors: FMM_E_NCCL. */
fmm_status fmm_comm_unique_id(void* id);

/* The device's P2P pair arithmetic (a12: k_p2p's pair code) as functions of
 * rho = r/(sqrt2 sigma_j): g(rho) of Eq. 2 and rho g'(rho) = (4/sqrt pi) rho^3
 * e^{-rho^2}, recovered from the kernel's f = g/(4 pi r^3) and f'/r =
 * (rho g' - 3 g)/(4 pi r^5) as ratios to the kernel's own
 * singular factors (g = f_reg/f_sing, rho g' = 3 g - 3 fp_reg/fp_sing), so the
 * cutoff approximation of reading Z6 is measured apart from the FP32 1/r^k.
 * branch 0 = the selection k_p2p applies (exact singular kernel, g = 1 and
 * rho g' = 0, iff rho >= 4.6), 1 = the regularised branch at every rho.
 * rho[n] in; g[n], rho_gp[n] out; host or device pointers.  Errors: FMM_E_ARG. */
fmm_status fmm_eval_pair_kernel(fmm_ctx* ctx, int64_t n, const float* rho, int32_t branch, float* g,
                                float* rho_gp);

/* The device's FP32 evaluation of the Eq. 2 cutoff g(rho) used by P2P
 * (reading Z6: any approximation with |g - g_exact| <= 2e-7).  rho[n] in,
 * g[n] out; host or device pointers.  Used by the parity tests. */
fmm_status fmm_eval_cutoff(fmm_ctx* ctx, int64_t n, const float* rho, float* g);

/* Debug modes of the loaded library, read once from the environment at the
 * first allocation: bit 0 = FMM_POISON=1 (every device buffer starts as 0xFF
 * bytes and carries a 4 KB guard zone checked after every API call; a damaged
 * zone fails the call with FMM_E_INTERNAL).  Test infrastructure only
 * (tests/test_gpu_poison.py); no compute, no errors. */
int32_t fmm_debug_mode(void);

#ifdef __cplusplus
}
#endif
#endif
