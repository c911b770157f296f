/*
 * oracle/fmm_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct double-precision CPU oracle for the FMM
 * evaluation of the regularised Biot-Savart velocity (Eq. 1)
 * and vortex-stretching term (Eq. 3).  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  It shares no code, header, table or constant
 * generator with the CUDA product path (paper_1106_5273_b200/csrc).
 *
 * Two parts:
 *   c-1  or_direct(): the plain definition -- an O(N^2 * 27^k) direct sum.
 *   c-2  or_fmm_*():  the FMM step by step in the paper's order: Morton keys
 *        (P:114), octree, dual tree traversal (Alg. 1 P:150-169,
 *        Alg. 2), P2M/M2M/M2L/L2L/L2P/P2P (fig:kernels P:103),
 *        periodic images.
 * Every reading of an ambiguous passage is listed in DESIGN.md ("Readings").
 */
#ifndef FMM_ORACLE_H
#define FMM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Eq. 2: g(rho) = erf(rho) - (2/sqrt(pi)) rho exp(-rho^2). */
double or_cutoff_g(double rho);

/* c-1: direct sum over the image lattice Lambda_k = {-(3^k-1)/2..(3^k-1)/2}^3
 * (k = 0: free space).  Targets xt[nt][3] carrying at[nt][3] (alpha_i, needed
 * by Eq. 3); sources xs[ns][3], as[ns][3], sig[ns].  Outputs u[nt][3] and
 * s[nt][3] are overwritten.  Pairs with r == 0 contribute 0 (reading Z7). */
void or_direct(int64_t nt, const double* xt, const double* at,
               int64_t ns, const double* xs, const double* as, const double* sig,
               double box_len, int images, double* u, double* s);

/* Solid harmonics, complex interleaved (re,im),
 * index n(n+1)/2+m for 0<=m<=n<P. */
void or_regular(double x, double y, double z, int P, double* R);
void or_irregular(double x, double y, double z, int P, double* I);

/* Single operators in physical (un-normalised) units; coefficient arrays
 * hold one component: P(P+1)/2 complex values. */
void or_p2m(int P, int64_t n, const double* x, const double* q, const double c[3], double* M);
void or_m2m(int P, const double* Mc, const double d[3] /* c_child - c_parent */, double* Mp);
void or_m2l(int P, const double* M, const double D[3] /* c_t - c_s */, double* L);
void or_l2l(int P, const double* Lp, const double d[3] /* c_child - c_parent */, double* Lc);
/* potential, gradient (3) and Hessian (xx,yy,zz,xy,xz,yz) of
 * phi(c + y) = sum L conj(R(y)) at y = d. */
void or_l2p_derivs(int P, const double* L, const double d[3], double* phi, double* grad, double* hess);
/* potential of a multipole at D = x - c_s */
double or_m2p(int P, const double* M, const double D[3]);

typedef struct {
  int order;                 /* p: degrees 0..p-1 (reading Z8)                 */
  int theta_num, theta_den;  /* MAC r_A + r_B < theta R (reading Z9)            */
  int ncrit;                 /* leaf iff count <= ncrit or level == 21          */
  int images;                /* k; 0 = free space                               */
  double box_lo[3], box_len; /* periodic cell (ignored for images == 0)         */
  int traversal;             /* 0 = MAC-first, 1 = leaf-first (Alg. 2 printed)  */
} or_cfg;

typedef struct or_fmm or_fmm;

/* Build keys, sort and tree (a1-a4). x, a: [n][3]; sig: [n]. */
or_fmm* or_fmm_new(int64_t n, const double* x, const double* a, const double* sig, const or_cfg* cfg);
void    or_fmm_free(or_fmm* f);
/* Dual tree traversal -> canonical P2P and M2L lists (a7). */
void    or_fmm_traverse(or_fmm* f);
/* Full evaluation (a5, a6, a8-a12): fills near and far parts. */
void    or_fmm_evaluate(or_fmm* f);

int64_t or_fmm_ncells(const or_fmm* f);
int64_t or_fmm_np2p(const or_fmm* f);
int64_t or_fmm_nm2l(const or_fmm* f);
/* box used for keys: lo[3], L */
void    or_fmm_box(const or_fmm* f, double* lo, double* L);
/* sorted keys [n] and permutation perm[i] = original index of sorted slot i */
void    or_fmm_keys(const or_fmm* f, uint64_t* keys, int64_t* perm);
/* wrapped positions actually used, caller order, [n][3] */
void    or_fmm_positions(const or_fmm* f, double* x);
/* cells: int64 [ncells][10] = level, qx, qy, qz, begin, count, parent,
 * child_begin, nchild, is_leaf */
void    or_fmm_cells(const or_fmm* f, int64_t* out);
/* lists: int64 [n][3] = (target cell, source cell, image index 0..26) */
void    or_fmm_p2p_list(const or_fmm* f, int64_t* out);
void    or_fmm_m2l_list(const or_fmm* f, int64_t* out);
/* normalised coefficients (reading Z18): M~_n = M_n / s^n, L~_n = L_n s^(n+1),
 * s = cell side; layout [ncells][3][P(P+1)/2] complex interleaved. */
void    or_fmm_multipoles(const or_fmm* f, double* out);
void    or_fmm_locals(const or_fmm* f, double* out);
/* results in caller order, [n][3] each */
void    or_fmm_results(const or_fmm* f, double* u_near, double* s_near, double* u_far, double* s_far);
/* near field of the selected target leaves only (8c-2 item 18 restricted to
 * their P2P entries; the traversal's target side restricted to their
 * ancestors): for each leaves[k] in order, its particles in sorted order ->
 * pidx (caller index), u[.][3], s[.][3]; *np2p = the leaves' P2P entries.
 * Returns the particle count written, -1 if a listed cell is not a leaf. */
int64_t or_fmm_near_subset(or_fmm* f, int64_t nsel, const int64_t* leaves, int64_t* pidx, double* u, double* s,
                           int64_t* np2p);
/* traversal completeness: per particle (caller order) number of source
 * particles covered by P2P + M2L + periodic far field. */
void    or_fmm_coverage(const or_fmm* f, int64_t* cover);

#ifdef __cplusplus
}
#endif
#endif
