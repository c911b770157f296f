/*
 * oracle/fmm_oracle.c -- TEST INFRASTRUCTURE ONLY (see fmm_oracle.h).
 *
 * A plain double-precision CPU implementation of the FMM-based evaluation of
 * PAPER.md Eqs. 1-3, written in the paper's order and notation.  It exists to
 * check the CUDA product path; nothing here is tuned.  OpenMP parallelises the
 * outer loops over independent targets only (no reordering of any sum).
 *
 * Citations: P:n = /root/reference/PAPER.md line n; Zn = reading n in
 * DESIGN.md (copied from SURVEY.md 8c).  Compile with -ffp-contract=off so the
 * key quantisation (Z16/Z19) is plain IEEE double arithmetic.
 */
#include "fmm_oracle.h"
#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;
#define OR_PI 3.14159265358979323846
#define OR_MAXLEVEL 21            /* 64-bit keys: 21 levels            */
#define OR_IMG_CENTRE 13          /* image index of the zero shift             */

static inline int cidx(int n, int m) { return n * (n + 1) / 2 + m; }

/* value of coefficient (n, m) for any sign of m: C_n^{-m} = (-1)^m conj(C_n^m)
 * (8c-2 item 10; holds for R, I, M and L because the sources are real). */
static inline cplx cget(const cplx* C, int n, int m)
{
  if (m >= 0) return C[cidx(n, m)];
  cplx v = conj(C[cidx(n, -m)]);
  return (m & 1) ? -v : v;
}

/* ------------------------------------------------------------------------ */
/* Eq. 2                                                             */
/* ------------------------------------------------------------------------ */
double or_cutoff_g(double rho)
{
  return erf(rho) - 2.0 / sqrt(OR_PI) * rho * exp(-rho * rho);
}

/* One source j on one target i, r = x_i - x_j - nL.
 * Eq. 1:  u_i += gamma_j x grad(G g),  G = 1/(4 pi r) -- physical sign,
 *                i.e. u_i += f(r) (alpha_j x r), f = g/(4 pi r^3)  (reading Z1).
 * Eq. 3:  ds_i = (alpha_i . grad_x)[f (alpha_j x r)]
 *                     = f (alpha_j x alpha_i) + (f'/r)(r.alpha_i)(alpha_j x r)
 *                (classical scheme, reading Z3), with
 *                f'/r = ((4/sqrt(pi)) rho^3 e^{-rho^2} - 3 g) / (4 pi r^5).
 * sigma is the source's (reading Z4); r == 0 contributes 0 (reading Z7). */
static void pair_kernel(const double r[3], const double aj[3], double sigj,
                        const double ai[3], double u[3], double s[3])
{
  double r2 = r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
  if (r2 == 0.0) return;
  double rr = sqrt(r2);
  double rho = rr / (sqrt(2.0) * sigj);
  double e = exp(-rho * rho);
  double g = erf(rho) - 2.0 / sqrt(OR_PI) * rho * e;
  double f = g / (4.0 * OR_PI * r2 * rr);
  double fp = (4.0 / sqrt(OR_PI) * rho * rho * rho * e - 3.0 * g) / (4.0 * OR_PI * r2 * r2 * rr);
  double c[3] = {aj[1] * r[2] - aj[2] * r[1], aj[2] * r[0] - aj[0] * r[2], aj[0] * r[1] - aj[1] * r[0]};
  double ca[3] = {aj[1] * ai[2] - aj[2] * ai[1], aj[2] * ai[0] - aj[0] * ai[2], aj[0] * ai[1] - aj[1] * ai[0]};
  double rda = r[0] * ai[0] + r[1] * ai[1] + r[2] * ai[2];
  for (int d = 0; d < 3; ++d) {
    u[d] += f * c[d];
    s[d] += f * ca[d] + fp * rda * c[d];
  }
}

static int ipow3(int k) { int v = 1; while (k-- > 0) v *= 3; return v; }

/* ------------------------------------------------------------------------ */
/* c-1: direct sum over the cube-truncated image lattice         */
/* (readings Z14/Z15).                                          */
/* ------------------------------------------------------------------------ */
void or_direct(int64_t nt, const double* xt, const double* at,
               int64_t ns, const double* xs, const double* as, const double* sig,
               double box_len, int images, double* u, double* s)
{
  int side = ipow3(images), h = (side - 1) / 2;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t i = 0; i < nt; ++i) {
    double ui[3] = {0, 0, 0}, si[3] = {0, 0, 0};
    for (int iz = -h; iz <= h; ++iz)
      for (int iy = -h; iy <= h; ++iy)
        for (int ix = -h; ix <= h; ++ix) {
          double sh[3] = {ix * box_len, iy * box_len, iz * box_len};
          for (int64_t j = 0; j < ns; ++j) {
            double r[3];
            for (int d = 0; d < 3; ++d) r[d] = xt[3 * i + d] - xs[3 * j + d] - sh[d];
            pair_kernel(r, &as[3 * j], sig[j], &at[3 * i], ui, si);
          }
        }
    for (int d = 0; d < 3; ++d) { u[3 * i + d] = ui[d]; s[3 * i + d] = si[d]; }
  }
}

/* ------------------------------------------------------------------------ */
/* Solid harmonics (Cheng et al. basis cited at P:109; recurrences 8c-2 8-9). */
/* R_n^m = r^n P_n^m(cos t) e^{i m phi}/(n+m)!,                               */
/* I_n^m = (n-m)! P_n^m(cos t) e^{i m phi}/r^{n+1}  (Condon-Shortley P).       */
/* ------------------------------------------------------------------------ */
static void regular_c(double x, double y, double z, int P, cplx* R)
{
  double r2 = x * x + y * y + z * z;
  cplx xy = x + I * y;
  R[0] = 1.0;
  for (int m = 1; m < P; ++m) R[cidx(m, m)] = -xy / (2.0 * m) * R[cidx(m - 1, m - 1)];
  for (int m = 0; m + 1 < P; ++m) R[cidx(m + 1, m)] = z * R[cidx(m, m)];
  for (int m = 0; m < P; ++m)
    for (int n = m + 2; n < P; ++n)
      R[cidx(n, m)] = ((2.0 * n - 1.0) * z * R[cidx(n - 1, m)] - r2 * R[cidx(n - 2, m)]) /
                      ((double)(n - m) * (double)(n + m));
}

static void irregular_c(double x, double y, double z, int P, cplx* Iv)
{
  double r2 = x * x + y * y + z * z;
  cplx xy = x + I * y;
  Iv[0] = 1.0 / sqrt(r2);
  for (int m = 1; m < P; ++m) Iv[cidx(m, m)] = -(2.0 * m - 1.0) * xy / r2 * Iv[cidx(m - 1, m - 1)];
  for (int m = 0; m + 1 < P; ++m) Iv[cidx(m + 1, m)] = (2.0 * m + 1.0) * z / r2 * Iv[cidx(m, m)];
  for (int m = 0; m < P; ++m)
    for (int n = m + 2; n < P; ++n)
      Iv[cidx(n, m)] = ((2.0 * n - 1.0) * z * Iv[cidx(n - 1, m)] -
                        (double)(n - 1 - m) * (double)(n - 1 + m) * Iv[cidx(n - 2, m)]) / r2;
}

void or_regular(double x, double y, double z, int P, double* R)
{
  regular_c(x, y, z, P, (cplx*)R);
}
void or_irregular(double x, double y, double z, int P, double* Iv)
{
  irregular_c(x, y, z, P, (cplx*)Iv);
}

/* ------------------------------------------------------------------------ */
/* The six operators of fig:kernels for one scalar Laplace     */
/* expansion; the vector kernels use three of them (one per alpha component). */
/* ------------------------------------------------------------------------ */

/* P2M (8c-2 item 12): M_n^m = sum_j q_j conj(R_n^m(x_j - c)). */
static void p2m_c(int P, int64_t n, const double* x, const double* q, int qstride,
                  const double c[3], cplx* M, cplx* Rbuf)
{
  for (int64_t j = 0; j < n; ++j) {
    regular_c(x[3 * j] - c[0], x[3 * j + 1] - c[1], x[3 * j + 2] - c[2], P, Rbuf);
    double qj = q[qstride * j];
    for (int i = 0; i < P * (P + 1) / 2; ++i) M[i] += qj * conj(Rbuf[i]);
  }
}

/* M2M (a6): M_n^m(parent) += sum_{k,l} conj(R_k^l(d)) M_{n-k}^{m-l}(child),
 * d = c_child - c_parent. */
static void m2m_c(int P, const cplx* Mc, const cplx* Rd, cplx* Mp)
{
  for (int n = 0; n < P; ++n)
    for (int m = 0; m <= n; ++m) {
      cplx acc = 0;
      for (int k = 0; k <= n; ++k)
        for (int l = -k; l <= k; ++l) {
          int nn = n - k, mm = m - l;
          if (mm < -nn || mm > nn) continue;
          acc += conj(cget(Rd, k, l)) * cget(Mc, nn, mm);
        }
      Mp[cidx(n, m)] += acc;
    }
}

/* M2L (a9): L_k^l += (-1)^k sum_{n<p-k} sum_m M_n^m I_{n+k}^{m+l}(D),
 * D = c_t - c_s (image shift included).  Terms are summed from high to low
 * degree n. */
static void m2l_c(int P, const cplx* M, const cplx* ID, cplx* L)
{
  for (int k = 0; k < P; ++k)
    for (int l = 0; l <= k; ++l) {
      cplx acc = 0;
      for (int n = P - 1 - k; n >= 0; --n)
        for (int m = -n; m <= n; ++m) acc += cget(M, n, m) * cget(ID, n + k, m + l);
      L[cidx(k, l)] += (k & 1) ? -acc : acc;
    }
}

/* L2L (a10): L_a^b(child) += sum_{k>=a,l} L_k^l(parent) conj(R_{k-a}^{l-b}(d)),
 * d = c_child - c_parent; summed from high to low k. */
static void l2l_c(int P, int Pout, const cplx* Lp, const cplx* Rd, cplx* Lc)
{
  for (int a = 0; a < Pout; ++a)
    for (int b = 0; b <= a; ++b) {
      cplx acc = 0;
      for (int k = P - 1; k >= a; --k)
        for (int l = -k; l <= k; ++l) {
          int kk = k - a, ll = l - b;
          if (ll < -kk || ll > kk) continue;
          acc += cget(Lp, k, l) * conj(cget(Rd, kk, ll));
        }
      Lc[cidx(a, b)] += acc;
    }
}

void or_p2m(int P, int64_t n, const double* x, const double* q, const double c[3], double* M)
{
  cplx* R = malloc(sizeof(cplx) * P * (P + 1) / 2);
  p2m_c(P, n, x, q, 1, c, (cplx*)M, R);
  free(R);
}

void or_m2m(int P, const double* Mc, const double d[3], double* Mp)
{
  cplx* R = malloc(sizeof(cplx) * P * (P + 1) / 2);
  regular_c(d[0], d[1], d[2], P, R);
  m2m_c(P, (const cplx*)Mc, R, (cplx*)Mp);
  free(R);
}

void or_m2l(int P, const double* M, const double D[3], double* L)
{
  int P2 = 2 * P - 1;
  cplx* Iv = malloc(sizeof(cplx) * P2 * (P2 + 1) / 2);
  irregular_c(D[0], D[1], D[2], P2, Iv);
  m2l_c(P, (const cplx*)M, Iv, (cplx*)L);
  free(Iv);
}

void or_l2l(int P, const double* Lp, const double d[3], double* Lc)
{
  cplx* R = malloc(sizeof(cplx) * P * (P + 1) / 2);
  regular_c(d[0], d[1], d[2], P, R);
  l2l_c(P, P, (const cplx*)Lp, R, (cplx*)Lc);
  free(R);
}

/* L2P (a11, 8c-2 item 16): shift L to the point keeping degrees <= 2, then
 * grad phi = (-Re L'_1^1, -Im L'_1^1, Re L'_1^0),
 * H_zz = Re L'_2^0, H_xx = (-Re L'_2^0 + Re L'_2^2)/2,
 * H_yy = (-Re L'_2^0 - Re L'_2^2)/2, H_xy = Im L'_2^2 / 2,
 * H_xz = -Re L'_2^1, H_yz = -Im L'_2^1. */
static void l2p_derivs_c(int P, const cplx* L, const double d[3], cplx* Rbuf,
                         double* phi, double grad[3], double hess[6])
{
  cplx Ls[6] = {0, 0, 0, 0, 0, 0};
  regular_c(d[0], d[1], d[2], P, Rbuf);
  l2l_c(P, P < 3 ? P : 3, L, Rbuf, Ls);
  *phi = creal(Ls[0]);
  grad[0] = -creal(Ls[cidx(1, 1)]);
  grad[1] = -cimag(Ls[cidx(1, 1)]);
  grad[2] = creal(Ls[cidx(1, 0)]);
  double l20 = creal(Ls[cidx(2, 0)]), l22r = creal(Ls[cidx(2, 2)]), l22i = cimag(Ls[cidx(2, 2)]);
  hess[0] = (-l20 + l22r) / 2.0;       /* xx */
  hess[1] = (-l20 - l22r) / 2.0;       /* yy */
  hess[2] = l20;                       /* zz */
  hess[3] = l22i / 2.0;                /* xy */
  hess[4] = -creal(Ls[cidx(2, 1)]);    /* xz */
  hess[5] = -cimag(Ls[cidx(2, 1)]);    /* yz */
}

void or_l2p_derivs(int P, const double* L, const double d[3], double* phi, double* grad, double* hess)
{
  cplx* R = malloc(sizeof(cplx) * P * (P + 1) / 2);
  l2p_derivs_c(P, (const cplx*)L, d, R, phi, grad, hess);
  free(R);
}

double or_m2p(int P, const double* Mv, const double D[3])
{
  const cplx* M = (const cplx*)Mv;
  cplx* Iv = malloc(sizeof(cplx) * P * (P + 1) / 2);
  irregular_c(D[0], D[1], D[2], P, Iv);
  double phi = 0;
  for (int n = P - 1; n >= 0; --n)
    for (int m = -n; m <= n; ++m) phi += creal(cget(M, n, m) * cget(Iv, n, m));
  free(Iv);
  return phi;
}

/* ------------------------------------------------------------------------ */
/* c-2: the FMM, step by step                                                 */
/* ------------------------------------------------------------------------ */
struct or_fmm {
  or_cfg cfg;
  int P, nc;                 /* order, coefficients per component           */
  int64_t n;
  double *x, *a, *sig;       /* caller order; x wrapped (a1)                */
  double lo[3], L;           /* key box                                     */
  uint64_t* keys;            /* sorted                                      */
  int64_t* perm;             /* sorted slot -> caller index                 */
  double *xs, *as, *ss;      /* sorted copies                               */
  int64_t ncells, capcells;
  int64_t *level, *qx, *qy, *qz, *begin, *count, *parent, *child_begin, *nchild, *leaf;
  int64_t level_begin[OR_MAXLEVEL + 2];
  int nlevels;
  int64_t np2p, nm2l, capp2p, capm2l;
  int64_t *p2p, *m2l;        /* (tgt, src, img) triples                     */
  cplx *M, *Lc;              /* [ncells][3][nc], physical units             */
  double *u_near, *s_near, *u_far, *s_far;   /* caller order               */
};

/* a1: periodic wrap into [lo, lo+L) in double, rounded to the FP32 input
 * precision. */
static double wrap_coord(double v, double lo, double L)
{
  if (v >= lo && v < lo + L) return v;
  double w = v - L * floor((v - lo) / L);
  return (double)(float)w;
}

/* a2 (Z16): q = floor((x - lo) 2^21 / L) in IEEE double
 * (no FMA), clamped; interleave with x in the lowest bit of each triple. */
static uint64_t morton_key(const double* x, const double lo[3], double L)
{
  double scale = 2097152.0 / L;
  uint64_t q[3];
  for (int d = 0; d < 3; ++d) {
    double t = (x[d] - lo[d]) * scale;
    double f = floor(t);
    int64_t qi = (int64_t)f;
    if (f < 0) qi = 0;
    if (f > 2097151.0) qi = 2097151;
    q[d] = (uint64_t)qi;
  }
  uint64_t key = 0;
  for (int b = 0; b < OR_MAXLEVEL; ++b)
    for (int d = 0; d < 3; ++d) key |= ((q[d] >> b) & 1ull) << (3 * b + d);
  return key;
}

typedef struct { uint64_t key; int64_t idx; } keyidx;
static int cmp_keyidx(const void* pa, const void* pb)
{
  const keyidx* a = pa; const keyidx* b = pb;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  return a->idx < b->idx ? -1 : (a->idx > b->idx ? 1 : 0);
}

static void grow_cells(or_fmm* f)
{
  if (f->ncells < f->capcells) return;
  int64_t cap = f->capcells ? 2 * f->capcells : 1024;
  int64_t** arrs[] = {&f->level, &f->qx, &f->qy, &f->qz, &f->begin, &f->count,
                      &f->parent, &f->child_begin, &f->nchild, &f->leaf};
  for (unsigned i = 0; i < sizeof(arrs) / sizeof(arrs[0]); ++i)
    *arrs[i] = realloc(*arrs[i], sizeof(int64_t) * cap);
  f->capcells = cap;
}

static int64_t add_cell(or_fmm* f, int64_t lev, int64_t qx, int64_t qy, int64_t qz,
                        int64_t b, int64_t c, int64_t par)
{
  grow_cells(f);
  int64_t i = f->ncells++;
  f->level[i] = lev; f->qx[i] = qx; f->qy[i] = qy; f->qz[i] = qz;
  f->begin[i] = b; f->count[i] = c; f->parent[i] = par;
  f->child_begin[i] = -1; f->nchild[i] = 0; f->leaf[i] = 1;
  return i;
}

or_fmm* or_fmm_new(int64_t n, const double* x, const double* a, const double* sig, const or_cfg* cfg)
{
  or_fmm* f = calloc(1, sizeof(or_fmm));
  f->cfg = *cfg;
  f->P = cfg->order;
  f->nc = f->P * (f->P + 1) / 2;
  f->n = n;
  f->x = malloc(sizeof(double) * 3 * (n ? n : 1));
  f->a = malloc(sizeof(double) * 3 * (n ? n : 1));
  f->sig = malloc(sizeof(double) * (n ? n : 1));
  memcpy(f->a, a, sizeof(double) * 3 * n);
  memcpy(f->sig, sig, sizeof(double) * n);

  /* key box (Z16): the periodic cell, or the bounding cube of the FP32 data */
  if (cfg->images > 0) {
    for (int d = 0; d < 3; ++d) f->lo[d] = cfg->box_lo[d];
    f->L = cfg->box_len;
    for (int64_t i = 0; i < n; ++i)
      for (int d = 0; d < 3; ++d) f->x[3 * i + d] = wrap_coord(x[3 * i + d], f->lo[d], f->L);
  } else {
    memcpy(f->x, x, sizeof(double) * 3 * n);
    double mn[3] = {0, 0, 0}, mx[3] = {0, 0, 0};
    for (int64_t i = 0; i < n; ++i)
      for (int d = 0; d < 3; ++d) {
        double v = f->x[3 * i + d];
        if (i == 0 || v < mn[d]) mn[d] = v;
        if (i == 0 || v > mx[d]) mx[d] = v;
      }
    double ext = 0;
    for (int d = 0; d < 3; ++d) { f->lo[d] = mn[d]; if (mx[d] - mn[d] > ext) ext = mx[d] - mn[d]; }
    f->L = ext > 0 ? ext * (1.0 + 0x1p-20) : 1.0;
  }

  /* a2-a3: keys and a stable sort by key (ties by caller index, Z17) */
  keyidx* ki = malloc(sizeof(keyidx) * (n ? n : 1));
  for (int64_t i = 0; i < n; ++i) { ki[i].key = morton_key(&f->x[3 * i], f->lo, f->L); ki[i].idx = i; }
  qsort(ki, n, sizeof(keyidx), cmp_keyidx);
  f->keys = malloc(sizeof(uint64_t) * (n ? n : 1));
  f->perm = malloc(sizeof(int64_t) * (n ? n : 1));
  f->xs = malloc(sizeof(double) * 3 * (n ? n : 1));
  f->as = malloc(sizeof(double) * 3 * (n ? n : 1));
  f->ss = malloc(sizeof(double) * (n ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    f->keys[i] = ki[i].key; f->perm[i] = ki[i].idx;
    for (int d = 0; d < 3; ++d) { f->xs[3 * i + d] = f->x[3 * ki[i].idx + d]; f->as[3 * i + d] = f->a[3 * ki[i].idx + d]; }
    f->ss[i] = f->sig[ki[i].idx];
  }
  free(ki);

  /* a4: octree of cubic cells over Morton prefixes, built
   * level by level; a cell is a leaf iff count <= ncrit or level == 21;
   * empty octants are not created; canonical order (level, key). */
  for (int l = 0; l <= OR_MAXLEVEL + 1; ++l) f->level_begin[l] = 0;
  f->nlevels = 0;
  if (n > 0) {
    add_cell(f, 0, 0, 0, 0, 0, n, -1);
    int64_t lb = 0;
    for (int l = 0; l <= OR_MAXLEVEL; ++l) {
      int64_t le = f->ncells;
      f->level_begin[l] = lb;
      f->nlevels = l + 1;
      for (int64_t c = lb; c < le; ++c) {
        if (f->count[c] <= cfg->ncrit || l == OR_MAXLEVEL) { f->leaf[c] = 1; continue; }
        f->leaf[c] = 0;
        f->child_begin[c] = f->ncells;
        int64_t i = f->begin[c], end = f->begin[c] + f->count[c];
        int sh = 3 * (OR_MAXLEVEL - 1 - l);
        while (i < end) {
          uint64_t oct = (f->keys[i] >> sh) & 7ull;
          int64_t j = i;
          while (j < end && ((f->keys[j] >> sh) & 7ull) == oct) ++j;
          add_cell(f, l + 1, 2 * f->qx[c] + (int64_t)(oct & 1), 2 * f->qy[c] + (int64_t)((oct >> 1) & 1),
                   2 * f->qz[c] + (int64_t)((oct >> 2) & 1), i, j - i, c);
          i = j;
        }
        f->nchild[c] = f->ncells - f->child_begin[c];
      }
      lb = le;
      if (lb == f->ncells) break;
    }
    f->level_begin[f->nlevels] = f->ncells;
  }
  return f;
}

void or_fmm_free(or_fmm* f)
{
  if (!f) return;
  free(f->x); free(f->a); free(f->sig); free(f->keys); free(f->perm);
  free(f->xs); free(f->as); free(f->ss);
  free(f->level); free(f->qx); free(f->qy); free(f->qz); free(f->begin); free(f->count);
  free(f->parent); free(f->child_begin); free(f->nchild); free(f->leaf);
  free(f->p2p); free(f->m2l); free(f->M); free(f->Lc);
  free(f->u_near); free(f->s_near); free(f->u_far); free(f->s_far);
  free(f);
}

/* geometry (8c-2 item 2): side s_l = L/2^l, centre lo + (q + 1/2) s_l */
static double cell_side(const or_fmm* f, int64_t c) { return f->L / (double)(1ll << f->level[c]); }
static void cell_centre(const or_fmm* f, int64_t c, double ctr[3])
{
  double s = cell_side(f, c);
  ctr[0] = f->lo[0] + ((double)f->qx[c] + 0.5) * s;
  ctr[1] = f->lo[1] + ((double)f->qy[c] + 0.5) * s;
  ctr[2] = f->lo[2] + ((double)f->qz[c] + 0.5) * s;
}

static void img_shift(int img, int v[3]) { v[0] = img % 3 - 1; v[1] = (img / 3) % 3 - 1; v[2] = img / 9 - 1; }

/* MAC (reading Z9, 8c-2 item 3): accept iff r_A + r_B < theta R with
 * r = (sqrt 3 / 2) side and R the distance between geometric centres
 * (image shift included), evaluated exactly on integers in units of half the
 * finest cell: 3 den^2 (2^{21-a} + 2^{21-b})^2 < num^2 |Delta|^2. */
static int mac_accept(const or_fmm* f, int64_t A, int64_t B, int img)
{
  int v[3]; img_shift(img, v);
  int64_t ca[3] = {f->qx[A], f->qy[A], f->qz[A]}, cb[3] = {f->qx[B], f->qy[B], f->qz[B]};
  __int128 d2 = 0;
  for (int d = 0; d < 3; ++d) {
    int64_t xa = (2 * ca[d] + 1) << (OR_MAXLEVEL - f->level[A]);
    int64_t xb = (2 * cb[d] + 1) << (OR_MAXLEVEL - f->level[B]);
    int64_t dd = xa - xb - (int64_t)v[d] * (1ll << (OR_MAXLEVEL + 1));
    d2 += (__int128)dd * dd;
  }
  __int128 ssum = (__int128)(1ll << (OR_MAXLEVEL - f->level[A])) + (__int128)(1ll << (OR_MAXLEVEL - f->level[B]));
  __int128 lhs = (__int128)3 * f->cfg.theta_den * f->cfg.theta_den * ssum * ssum;
  __int128 rhs = (__int128)f->cfg.theta_num * f->cfg.theta_num * d2;
  return lhs < rhs;
}

static void push3(int64_t** arr, int64_t* len, int64_t* cap, int64_t a, int64_t b, int64_t c)
{
  if (*len >= *cap) { *cap = *cap ? 2 * *cap : 4096; *arr = realloc(*arr, sizeof(int64_t) * 3 * *cap); }
  (*arr)[3 * *len] = a; (*arr)[3 * *len + 1] = b; (*arr)[3 * *len + 2] = c; ++*len;
}

typedef struct { int64_t* v; int64_t len, cap; } stack3;

/* Alg. 2 Interact (reading Z11).  MAC-first: MAC -> M2L; both
 * leaves -> P2P; else push.  Leaf-first (as printed): both leaves -> P2P;
 * MAC -> M2L; else push.  (The remote branch, only exists with a
 * LET and is not reachable in a single-domain oracle run.)  The three
 * destinations are passed in (the f's own lists, or a target subset's). */
typedef struct { int64_t *p2p, np2p, capp2p, *m2l, nm2l, capm2l; } lists3;
static void interact_into(or_fmm* f, stack3* st, lists3* out, int64_t A, int64_t B, int img)
{
  int both_leaves = f->leaf[A] && f->leaf[B];
  if (f->cfg.traversal == 0) {
    if (mac_accept(f, A, B, img)) push3(&out->m2l, &out->nm2l, &out->capm2l, A, B, img);
    else if (both_leaves) push3(&out->p2p, &out->np2p, &out->capp2p, A, B, img);
    else push3(&st->v, &st->len, &st->cap, A, B, img);
  } else {
    if (both_leaves) push3(&out->p2p, &out->np2p, &out->capp2p, A, B, img);
    else if (mac_accept(f, A, B, img)) push3(&out->m2l, &out->nm2l, &out->capm2l, A, B, img);
    else push3(&st->v, &st->len, &st->cap, A, B, img);
  }
}

static int cmp_triple(const void* pa, const void* pb)
{
  const int64_t* a = pa; const int64_t* b = pb;
  for (int i = 0; i < 3; ++i) if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  return 0;
}

/* Alg. 1 Evaluate with reading Z10 (equal radius => split B;
 * never split a leaf) and 8c-2 item 7 (seeds: Interact(root, root, img) for
 * the 27 first-layer images when k >= 1). */
/* The traversal loop over (A, B, img) pairs; keep (may be NULL) restricts the
 * target side to the flagged cells: a pair whose target cell is not flagged is
 * dropped, which with keep = "ancestor-or-self of a selected leaf" yields
 * exactly the full traversal's entries whose target lies on those paths (no
 * descendant of an unflagged cell is flagged, so no entry for a selected cell
 * can come from such a pair). */
static void traverse_into(or_fmm* f, const char* keep, lists3* out)
{
  if (f->ncells == 0) return;
  stack3 st = {0, 0, 0};
  if (f->cfg.images > 0) {
    for (int img = 0; img < 27; ++img) interact_into(f, &st, out, 0, 0, img);
  } else {
    interact_into(f, &st, out, 0, 0, OR_IMG_CENTRE);
  }
  while (st.len > 0) {
    --st.len;
    int64_t A = st.v[3 * st.len], B = st.v[3 * st.len + 1];
    int img = (int)st.v[3 * st.len + 2];
    int split_b = f->leaf[A] || (!f->leaf[B] && f->level[B] <= f->level[A]);
    if (split_b) {
      for (int64_t b = f->child_begin[B]; b < f->child_begin[B] + f->nchild[B]; ++b) interact_into(f, &st, out, A, b, img);
    } else {
      for (int64_t a = f->child_begin[A]; a < f->child_begin[A] + f->nchild[A]; ++a)
        if (!keep || keep[a]) interact_into(f, &st, out, a, B, img);
    }
  }
  free(st.v);
  /* canonical order (reading Z20): sort by (target, source, image) */
  qsort(out->p2p, out->np2p, 3 * sizeof(int64_t), cmp_triple);
  qsort(out->m2l, out->nm2l, 3 * sizeof(int64_t), cmp_triple);
}

void or_fmm_traverse(or_fmm* f)
{
  lists3 L = {f->p2p, 0, f->capp2p, f->m2l, 0, f->capm2l};
  traverse_into(f, NULL, &L);
  f->p2p = L.p2p; f->np2p = L.np2p; f->capp2p = L.capp2p;
  f->m2l = L.m2l; f->nm2l = L.nm2l; f->capm2l = L.capm2l;
}

/* Near field (8c-2 item 18: c-1 restricted to P2P list entries) of the
 * selected target leaves only, for sizes where the full traversal or P2P is
 * too slow: the traversal above with the target side restricted to the
 * ancestors-or-self of the selected leaves, then c-1 over each selected
 * leaf's P2P entries in canonical order (the same arithmetic and summation
 * order as or_fmm_evaluate's P2P).  For each selected leaf in the given order,
 * its particles (sorted order) are written to pidx (caller index), u, s.
 * Returns the number of particles written, or -1 if a cell is not a leaf. */
int64_t or_fmm_near_subset(or_fmm* f, int64_t nsel, const int64_t* leaves, int64_t* pidx, double* u, double* s,
                           int64_t* np2p_out)
{
  char* keep = calloc(f->ncells ? f->ncells : 1, 1);
  for (int64_t k = 0; k < nsel; ++k) {
    int64_t c = leaves[k];
    if (c < 0 || c >= f->ncells || !f->leaf[c]) { free(keep); return -1; }
    for (; c >= 0; c = f->parent[c]) keep[c] = 1;
  }
  lists3 L = {NULL, 0, 0, NULL, 0, 0};
  if (nsel > 0) traverse_into(f, keep, &L);
  int64_t* seg = calloc(f->ncells + 1, sizeof(int64_t));
  for (int64_t e = 0; e < L.np2p; ++e) seg[L.p2p[3 * e] + 1]++;
  for (int64_t c = 0; c < f->ncells; ++c) seg[c + 1] += seg[c];
  int64_t* first = malloc(sizeof(int64_t) * (nsel ? nsel : 1));
  int64_t m = 0;
  for (int64_t k = 0; k < nsel; ++k) { first[k] = m; m += f->count[leaves[k]]; }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t k = 0; k < nsel; ++k) {
    int64_t t = leaves[k];
    for (int64_t i = f->begin[t]; i < f->begin[t] + f->count[t]; ++i) {
      double ui[3] = {0, 0, 0}, si[3] = {0, 0, 0};
      for (int64_t e = seg[t]; e < seg[t + 1]; ++e) {
        int64_t sc = L.p2p[3 * e + 1];
        int v[3]; img_shift((int)L.p2p[3 * e + 2], v);
        for (int64_t j = f->begin[sc]; j < f->begin[sc] + f->count[sc]; ++j) {
          double r[3];
          for (int d = 0; d < 3; ++d) r[d] = f->xs[3 * i + d] - f->xs[3 * j + d] - v[d] * f->L;
          pair_kernel(r, &f->as[3 * j], f->ss[j], &f->as[3 * i], ui, si);
        }
      }
      int64_t o = first[k] + (i - f->begin[t]);
      pidx[o] = f->perm[i];
      for (int d = 0; d < 3; ++d) { u[3 * o + d] = ui[d]; s[3 * o + d] = si[d]; }
    }
  }
  if (np2p_out) *np2p_out = L.np2p;
  free(first); free(seg); free(keep); free(L.p2p); free(L.m2l);
  return m;
}

/* segment boundaries of a target-sorted list */
static int64_t* segments(const int64_t* lst, int64_t len, int64_t ncells)
{
  int64_t* seg = calloc(ncells + 1, sizeof(int64_t));
  for (int64_t i = 0; i < len; ++i) seg[lst[3 * i] + 1]++;
  for (int64_t c = 0; c < ncells; ++c) seg[c + 1] += seg[c];
  return seg;
}

/* a8: periodic far field for layers j = 1..k-1 (reading Z14):
 * M^{(1)} = root multipole (side L, centred on the domain); for each layer the
 * 26 neighbour super-cells I != 0 and their 27 children C contribute an M2L
 * from M^{(j)} placed at c0 + (3I + C) 3^{j-1} L into every far target (cells
 * at level 2, or leaves above level 2); then M^{(j+1)} = sum_C M2M(M^{(j)} at
 * c0 + C 3^{j-1} L -> c0). */
static void periodic_far(or_fmm* f)
{
  int k = f->cfg.images;
  if (k < 2 || f->ncells == 0) return;
  int P = f->P, nc = f->nc, P2 = 2 * P - 1;
  double c0[3]; cell_centre(f, 0, c0);
  cplx* Mj = calloc(3 * nc, sizeof(cplx));
  memcpy(Mj, f->M, sizeof(cplx) * 3 * nc);
  cplx* Mnext = calloc(3 * nc, sizeof(cplx));
  cplx* R = malloc(sizeof(cplx) * nc);
  double scale = f->L;
  for (int j = 1; j <= k - 1; ++j) {
#pragma omp parallel
    {
      cplx* Iv = malloc(sizeof(cplx) * P2 * (P2 + 1) / 2);
#pragma omp for schedule(dynamic, 1)
      for (int64_t t = 0; t < f->ncells; ++t) {
        if (!(f->level[t] == 2 || (f->leaf[t] && f->level[t] < 2))) continue;
        double ct[3]; cell_centre(f, t, ct);
        for (int I3 = 0; I3 < 27; ++I3) {
          if (I3 == OR_IMG_CENTRE) continue;
          int vi[3]; img_shift(I3, vi);
          for (int C3 = 0; C3 < 27; ++C3) {
            int vc[3]; img_shift(C3, vc);
            double D[3];
            for (int d = 0; d < 3; ++d) D[d] = ct[d] - (c0[d] + (3.0 * vi[d] + vc[d]) * scale);
            irregular_c(D[0], D[1], D[2], P2, Iv);
            for (int c = 0; c < 3; ++c) m2l_c(P, Mj + c * nc, Iv, f->Lc + (t * 3 + c) * nc);
          }
        }
      }
      free(Iv);
    }
    memset(Mnext, 0, sizeof(cplx) * 3 * nc);
    for (int C3 = 0; C3 < 27; ++C3) {
      int vc[3]; img_shift(C3, vc);
      regular_c(vc[0] * scale, vc[1] * scale, vc[2] * scale, P, R);   /* d = c_child - c_parent */
      for (int c = 0; c < 3; ++c) m2m_c(P, Mj + c * nc, R, Mnext + c * nc);
    }
    memcpy(Mj, Mnext, sizeof(cplx) * 3 * nc);
    scale *= 3.0;
  }
  free(Mj); free(Mnext); free(R);
}

void or_fmm_evaluate(or_fmm* f)
{
  int64_t n = f->n, nc = f->nc;
  int P = f->P, P2 = 2 * P - 1;
  if (f->np2p == 0 && f->nm2l == 0) or_fmm_traverse(f);
  free(f->M); free(f->Lc);
  f->M = calloc((size_t)(f->ncells ? f->ncells : 1) * 3 * nc, sizeof(cplx));
  f->Lc = calloc((size_t)(f->ncells ? f->ncells : 1) * 3 * nc, sizeof(cplx));
  double* un = calloc(3 * (n ? n : 1), sizeof(double));
  double* sn = calloc(3 * (n ? n : 1), sizeof(double));
  double* uf = calloc(3 * (n ? n : 1), sizeof(double));
  double* sf = calloc(3 * (n ? n : 1), sizeof(double));

  /* a5 P2M at leaves, a6 M2M bottom-up ("upward") */
#pragma omp parallel
  {
    cplx* R = malloc(sizeof(cplx) * nc);
#pragma omp for schedule(dynamic, 16)
    for (int64_t c = 0; c < f->ncells; ++c) {
      if (!f->leaf[c]) continue;
      double ctr[3]; cell_centre(f, c, ctr);
      for (int comp = 0; comp < 3; ++comp)
        p2m_c(P, f->count[c], &f->xs[3 * f->begin[c]], &f->as[3 * f->begin[c] + comp], 3, ctr,
              f->M + (c * 3 + comp) * nc, R);
    }
    free(R);
  }
  for (int l = f->nlevels - 2; l >= 0; --l) {
#pragma omp parallel
    {
      cplx* R = malloc(sizeof(cplx) * nc);
#pragma omp for schedule(dynamic, 16)
      for (int64_t c = f->level_begin[l]; c < f->level_begin[l + 1]; ++c) {
        if (f->leaf[c]) continue;
        double cp[3]; cell_centre(f, c, cp);
        for (int64_t ch = f->child_begin[c]; ch < f->child_begin[c] + f->nchild[c]; ++ch) {
          double cc[3]; cell_centre(f, ch, cc);
          regular_c(cc[0] - cp[0], cc[1] - cp[1], cc[2] - cp[2], P, R);
          for (int comp = 0; comp < 3; ++comp) m2m_c(P, f->M + (ch * 3 + comp) * nc, R, f->M + (c * 3 + comp) * nc);
        }
      }
      free(R);
    }
  }

  /* a9 M2L over the list (grouped by target so each target is owned by one
   * thread), then a8 periodic far layers */
  int64_t* seg = segments(f->m2l, f->nm2l, f->ncells);
#pragma omp parallel
  {
    cplx* Iv = malloc(sizeof(cplx) * P2 * (P2 + 1) / 2);
#pragma omp for schedule(dynamic, 8)
    for (int64_t t = 0; t < f->ncells; ++t) {
      double ct[3]; cell_centre(f, t, ct);
      for (int64_t e = seg[t]; e < seg[t + 1]; ++e) {
        int64_t s = f->m2l[3 * e + 1];
        int v[3]; img_shift((int)f->m2l[3 * e + 2], v);
        double cs[3]; cell_centre(f, s, cs);
        double D[3];
        for (int d = 0; d < 3; ++d) D[d] = ct[d] - cs[d] - v[d] * f->L;
        irregular_c(D[0], D[1], D[2], P2, Iv);
        for (int comp = 0; comp < 3; ++comp) m2l_c(P, f->M + (s * 3 + comp) * nc, Iv, f->Lc + (t * 3 + comp) * nc);
      }
    }
    free(Iv);
  }
  free(seg);
  periodic_far(f);

  /* a10 L2L top-down */
  for (int l = 0; l + 1 < f->nlevels; ++l) {
#pragma omp parallel
    {
      cplx* R = malloc(sizeof(cplx) * nc);
#pragma omp for schedule(dynamic, 16)
      for (int64_t c = f->level_begin[l]; c < f->level_begin[l + 1]; ++c) {
        if (f->leaf[c]) continue;
        double cp[3]; cell_centre(f, c, cp);
        for (int64_t ch = f->child_begin[c]; ch < f->child_begin[c] + f->nchild[c]; ++ch) {
          double cc[3]; cell_centre(f, ch, cc);
          regular_c(cc[0] - cp[0], cc[1] - cp[1], cc[2] - cp[2], P, R);
          for (int comp = 0; comp < 3; ++comp) l2l_c(P, P, f->Lc + (c * 3 + comp) * nc, R, f->Lc + (ch * 3 + comp) * nc);
        }
      }
      free(R);
    }
  }

  /* a11 L2P: u_far = (1/4pi) eps_abc d_b phi_c, s_far = (1/4pi) alpha_d eps_abc H^c_db */
#pragma omp parallel
  {
    cplx* R = malloc(sizeof(cplx) * nc);
#pragma omp for schedule(dynamic, 16)
    for (int64_t c = 0; c < f->ncells; ++c) {
      if (!f->leaf[c]) continue;
      double ctr[3]; cell_centre(f, c, ctr);
      for (int64_t i = f->begin[c]; i < f->begin[c] + f->count[c]; ++i) {
        double d[3] = {f->xs[3 * i] - ctr[0], f->xs[3 * i + 1] - ctr[1], f->xs[3 * i + 2] - ctr[2]};
        double g[3][3], H[3][3][3];
        for (int comp = 0; comp < 3; ++comp) {
          double phi, hs[6];
          l2p_derivs_c(P, f->Lc + (c * 3 + comp) * nc, d, R, &phi, g[comp], hs);
          H[comp][0][0] = hs[0]; H[comp][1][1] = hs[1]; H[comp][2][2] = hs[2];
          H[comp][0][1] = H[comp][1][0] = hs[3];
          H[comp][0][2] = H[comp][2][0] = hs[4];
          H[comp][1][2] = H[comp][2][1] = hs[5];
        }
        const double* ai = &f->as[3 * i];
        double k4 = 1.0 / (4.0 * OR_PI);
        /* u_a = eps_abc d_b phi_c */
        double u[3] = {g[2][1] - g[1][2], g[0][2] - g[2][0], g[1][0] - g[0][1]};
        double s[3];
        for (int aa = 0; aa < 3; ++aa) s[aa] = 0;
        for (int dd = 0; dd < 3; ++dd) {
          s[0] += ai[dd] * (H[2][dd][1] - H[1][dd][2]);
          s[1] += ai[dd] * (H[0][dd][2] - H[2][dd][0]);
          s[2] += ai[dd] * (H[1][dd][0] - H[0][dd][1]);
        }
        int64_t o = f->perm[i];
        for (int aa = 0; aa < 3; ++aa) { uf[3 * o + aa] = k4 * u[aa]; sf[3 * o + aa] = k4 * s[aa]; }
      }
    }
    free(R);
  }

  /* a12 P2P over the list, grouped by target leaf */
  int64_t* pseg = segments(f->p2p, f->np2p, f->ncells);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < f->ncells; ++t) {
    if (pseg[t] == pseg[t + 1]) continue;
    for (int64_t i = f->begin[t]; i < f->begin[t] + f->count[t]; ++i) {
      double ui[3] = {0, 0, 0}, si[3] = {0, 0, 0};
      for (int64_t e = pseg[t]; e < pseg[t + 1]; ++e) {
        int64_t s = f->p2p[3 * e + 1];
        int v[3]; img_shift((int)f->p2p[3 * e + 2], v);
        for (int64_t j = f->begin[s]; j < f->begin[s] + f->count[s]; ++j) {
          double r[3];
          for (int d = 0; d < 3; ++d) r[d] = f->xs[3 * i + d] - f->xs[3 * j + d] - v[d] * f->L;
          pair_kernel(r, &f->as[3 * j], f->ss[j], &f->as[3 * i], ui, si);
        }
      }
      int64_t o = f->perm[i];
      for (int d = 0; d < 3; ++d) { un[3 * o + d] = ui[d]; sn[3 * o + d] = si[d]; }
    }
  }
  free(pseg);
  free(f->u_near); free(f->s_near); free(f->u_far); free(f->s_far);
  f->u_near = un; f->s_near = sn; f->u_far = uf; f->s_far = sf;
}

/* ------------------------------------------------------------------------ */
/* getters                                                                    */
/* ------------------------------------------------------------------------ */
int64_t or_fmm_ncells(const or_fmm* f) { return f->ncells; }
int64_t or_fmm_np2p(const or_fmm* f) { return f->np2p; }
int64_t or_fmm_nm2l(const or_fmm* f) { return f->nm2l; }
void or_fmm_box(const or_fmm* f, double* lo, double* L)
{
  for (int d = 0; d < 3; ++d) lo[d] = f->lo[d];
  *L = f->L;
}
void or_fmm_keys(const or_fmm* f, uint64_t* keys, int64_t* perm)
{
  memcpy(keys, f->keys, sizeof(uint64_t) * f->n);
  memcpy(perm, f->perm, sizeof(int64_t) * f->n);
}
void or_fmm_positions(const or_fmm* f, double* x) { memcpy(x, f->x, sizeof(double) * 3 * f->n); }
void or_fmm_cells(const or_fmm* f, int64_t* out)
{
  for (int64_t c = 0; c < f->ncells; ++c) {
    int64_t* o = out + 10 * c;
    o[0] = f->level[c]; o[1] = f->qx[c]; o[2] = f->qy[c]; o[3] = f->qz[c];
    o[4] = f->begin[c]; o[5] = f->count[c]; o[6] = f->parent[c];
    o[7] = f->child_begin[c]; o[8] = f->nchild[c]; o[9] = f->leaf[c];
  }
}
void or_fmm_p2p_list(const or_fmm* f, int64_t* out) { memcpy(out, f->p2p, sizeof(int64_t) * 3 * f->np2p); }
void or_fmm_m2l_list(const or_fmm* f, int64_t* out) { memcpy(out, f->m2l, sizeof(int64_t) * 3 * f->nm2l); }

static void normalised(const or_fmm* f, const cplx* src, int local, double* out)
{
  cplx* o = (cplx*)out;
  for (int64_t c = 0; c < f->ncells; ++c) {
    double s = cell_side(f, c);
    for (int comp = 0; comp < 3; ++comp)
      for (int n = 0; n < f->P; ++n) {
        double fac = local ? pow(s, n + 1) : pow(s, -n);
        for (int m = 0; m <= n; ++m) o[(c * 3 + comp) * f->nc + cidx(n, m)] = src[(c * 3 + comp) * f->nc + cidx(n, m)] * fac;
      }
  }
}
void or_fmm_multipoles(const or_fmm* f, double* out) { normalised(f, f->M, 0, out); }
void or_fmm_locals(const or_fmm* f, double* out) { normalised(f, f->Lc, 1, out); }

void or_fmm_results(const or_fmm* f, double* u_near, double* s_near, double* u_far, double* s_far)
{
  size_t b = sizeof(double) * 3 * f->n;
  if (!f->u_near) return;
  memcpy(u_near, f->u_near, b); memcpy(s_near, f->s_near, b);
  memcpy(u_far, f->u_far, b); memcpy(s_far, f->s_far, b);
}

void or_fmm_coverage(const or_fmm* f, int64_t* cover)
{
  int64_t* cs = calloc(f->n ? f->n : 1, sizeof(int64_t));
  for (int64_t e = 0; e < f->np2p; ++e) {
    int64_t t = f->p2p[3 * e], s = f->p2p[3 * e + 1];
    for (int64_t i = f->begin[t]; i < f->begin[t] + f->count[t]; ++i) cs[i] += f->count[s];
  }
  for (int64_t e = 0; e < f->nm2l; ++e) {
    int64_t t = f->m2l[3 * e], s = f->m2l[3 * e + 1];
    for (int64_t i = f->begin[t]; i < f->begin[t] + f->count[t]; ++i) cs[i] += f->count[s];
  }
  int64_t far = 0;
  if (f->cfg.images >= 2) {
    int64_t p27 = 1;
    for (int j = 0; j < f->cfg.images; ++j) p27 *= 27;
    far = f->n * (p27 - 27);
  }
  for (int64_t i = 0; i < f->n; ++i) cover[f->perm[i]] = cs[i] + far;
  free(cs);
}
