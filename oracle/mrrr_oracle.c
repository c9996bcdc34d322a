/*
 * oracle/mrrr_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, sequential-per-item CPU implementation of the mixed
 * double/quadruple MRRR hot path of arXiv 1401.4950, used to prove
 * parity of the CUDA path.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with
 * paper_1401_4950_b200/ (the product); the two are written independently
 * from DESIGN.md "Algorithm" (S0-S10), which restates the paper.
 *
 *   x-arithmetic = IEEE binary64 (double), no contraction (-ffp-contract=off)
 *   y-arithmetic = IEEE binary128 (__float128, libquadmath)
 *   (double/quadruple realisation; Table tab:precisions P:5552-5571)
 *
 * Built a second time with -DORACLE_SD (liboracle_sd.so): the single/double
 * realisation, y-arithmetic = binary64, epsilon_x = 2^-24,
 * gaptol 1e-5 -- the same steps with the constants of the #ifdef block below.
 *
 * Every function cites the passage it follows as P:<line> and the
 * DESIGN.md reading (A-<n>) where the paper is silent or garbled.
 *
 * Parity pins: see tests/test_oracle_*.py.  Functions with no pin beyond
 * consistency are marked "parity unpinned" below (cluster eigenvector bases,
 * RQI iteration counts / twist index).
 */
#include <float.h>
#include <math.h>
#include <omp.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef __float128 qreal;  /* binary128: the test tools below (residuals, Jacobi), both realisations */

#ifdef ORACLE_SD
/* Single/double realisation: binary32 input and output, ALL computations in      */
/* binary64 ("we carry out all computations in the former"), gaptol fixed to 1e-5.       */
/* Compiled from this same file with -DORACLE_SD into liboracle_sd.so; DESIGN.md "Single/double" lists the    */
/* reading of every constant below.                                                                              */
typedef double yreal;
#define EPS_X 0x1p-24          /* epsilon_x = epsilon_s: the binary32 output precision, Table tab:precisions */
#define EPS_Y 0x1p-53          /* y = binary64 */
#define XI_SCALE 0x1p-24       /* perturbation xi = eps_x: |xi| <= 2^-25 */
#define KELG_RATIO 0x1p29      /* eps_x / eps_y of eq:newkelgbound P:6052-6056 */
#define Y_FULLREL 0x1p-50      /* "full accuracy" of the bisection fallback in binary64 (a few ulps, A-14) */
#define DEFAULT_GAPTOL 1e-5
#define YFABS fabs
#define YFINITE isfinite
#define YFMAX fmax
#define YISINF isinf
#define YISNAN isnan
#define YSQRT sqrt
#define YSIGNBIT signbit
#else
typedef __float128 yreal;      /* double/quadruple realisation */
#define EPS_X 0x1p-53          /* epsilon_x, Table tab:precisions P:5559 */
#define EPS_Y 0x1p-104         /* conservative y unit roundoff for thresholds (A-14) */
#define XI_SCALE 0x1p-53       /* |xi| <= 2^-54 = eps_x / 2 (A-9) */
#define KELG_RATIO 0x1p51      /* eps_x / eps_y of eq:newkelgbound P:6052-6056 (A-35) */
#define Y_FULLREL 0x1p-98Q     /* a few eps_y (A-14) */
#define DEFAULT_GAPTOL 1e-10
#define YFABS fabsq
#define YFINITE finiteq
#define YFMAX fmaxq
#define YISINF isinfq
#define YISNAN isnanq
#define YSQRT sqrtq
#define YSIGNBIT signbitq
#endif
/* the arithmetic of the eigenvalue approximations (x-bisection, intervals, shifts) is binary64 in both     */
/* realisations: Gershgorin inflation, interval inflation nu and the shift offsets scale with its epsilon    */
#define EPS_A 0x1p-53
#define ATOL (2.0 * DBL_MIN)   /* atol = 2 omega */
#define RTOL_Y 0x1p-50         /* "full accuracy" of cluster ends in y (A-12) */
#define GROWTH 64.0            /* element growth threshold (A-11), relaxed by eq:newkelgbound (A-35) */
#define MAX_ATTEMPTS 6         /* shift attempts (A-11) */
#define MAX_RQI 10             /* RQI cap (A-14) */
#define MAXD 8                 /* representation tree depth cap */
#define DEFAULT_SEED 0x4D52525233ULL

enum {
  ST_DMAX = 0, ST_NCLUSTERS, ST_LARGEST, ST_UNCERTIFIED, ST_ATTEMPTS, ST_RQI_ITERS,
  ST_RQI_FALLBACK, ST_BRACKET_FIX, ST_ROOT_BACKOFF, ST_FAILED, ST_NEGX, ST_NEGY,
  ST_GETVEC, ST_ZPIV, ST_ESTOP, ST_SUPPORT, ST_NSTATS = 16
};

typedef struct {
  double gaptol;      /* <= 0 -> DEFAULT_GAPTOL (1e-10; single/double 1e-5) */
  uint64_t seed;      /* perturbation key, 0 -> DEFAULT_SEED */
  int32_t root_side;  /* 0 auto (S3 rule), 1 left, 2 right */
  int32_t threads;    /* 0 -> OpenMP default */
  int32_t roots_only; /* 1: stop after S5 (split, roots, root bisection of the computed set; diagnostics only) */
  int32_t early_stop; /* 1: early classification stop of the root bisection (S5', A-41) */
  int32_t support;    /* 1: numerical-support truncation of every singleton vector (S10', A-42) */
} oracle_opts;

typedef struct {      /* every pointer optional */
  int32_t *nblocks;     /* [1] */
  int32_t *block_start; /* [n+1] */
  double *mu;           /* [n] per block */
  int32_t *side;        /* [n] per block: 0 trivial (size 1), 1 left, 2 right */
  double *root_lo;      /* [n] per global position, NaN if not computed */
  double *root_hi;      /* [n] */
  int32_t *root_gstart; /* [n] 1 starts a root group, 0 member, -1 not computed */
  int32_t *depth;       /* [k] */
  int32_t *grp_first;   /* [MAXD*k] global position of group start at each depth, -1 */
  int32_t *grp_last;    /* [MAXD*k] */
  double *fin_lo;       /* [k] final-node interval (node frame) */
  double *fin_hi;       /* [k] */
  int64_t *stats;       /* [16] */
} oracle_diag;

static int64_t g_stats[ST_NSTATS];
#define STAT_ADD(i, v) do { _Pragma("omp atomic") g_stats[i] += (v); } while (0)
static void stat_max(int i, int64_t v) {
#pragma omp critical(oracle_statmax)
  { if (v > g_stats[i]) g_stats[i] = v; }
}

/* SignBit(d) of Alg. negcountLDL remark (2), P:7159-7161 (A-6); a NaN counts 0. */
static inline int sbx(double x) { return signbit(x) && !isnan(x); }
static inline int sby(yreal x) { return YSIGNBIT(x) && !YISNAN(x); }
static inline int sbq(qreal x) { return signbitq(x) && !isnanq(x); }
static inline double dmax(double a, double b) { return (b > a) ? b : a; }
static inline double dmin(double a, double b) { return (b < a) ? b : a; }

/* ------------------------------------------------------------------------- */
/* Perturbation PRNG: counter-based SplitMix64 (A-9; "any (fixed) sequence of  */
/* pseudo-random numbers").  xi in [-XI_SCALE/2, XI_SCALE/2).     */
/* ------------------------------------------------------------------------- */
double oracle_xi(uint64_t seed, uint64_t idx) {
  uint64_t z = seed + (idx + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z ^= z >> 31;
  double u = (double)(z >> 11) * 0x1p-53;
  return (u - 0.5) * XI_SCALE;
}

/* ------------------------------------------------------------------------- */
/* S1 ||T||_1 and S2 split, eq:tolsplit P:3028-3038 with the mixed */
/* rule |beta_i| <= eps_x sqrt(n) ||T|| of the unreduced input, P:5712-5719 (A-7) */
/* ------------------------------------------------------------------------- */
double oracle_norm1(int64_t n, const double *d, const double *e) {
  double t = 0.0;
  for (int64_t i = 0; i < n; i++) {
    double a = (i > 0) ? fabs(e[i - 1]) : 0.0;
    double b = (i < n - 1) ? fabs(e[i]) : 0.0;
    double c = (a + fabs(d[i])) + b;
    t = dmax(t, c);
  }
  return t;
}

/* writes block starts; returns the number of blocks */
int64_t oracle_split(int64_t n, const double *d, const double *e, int32_t *starts) {
  double tnorm = oracle_norm1(n, d, e);
  double tol = (EPS_X * sqrt((double)n)) * tnorm;
  int64_t nb = 0;
  starts[nb++] = 0;
  for (int64_t i = 0; i < n - 1; i++)
    if (fabs(e[i]) <= tol) starts[nb++] = (int32_t)(i + 1);
  starts[nb] = (int32_t)n;
  return nb;
}

/* Alg. gershgorin, with |beta_1| (A-3); nb >= 2 */
void oracle_gershgorin(int64_t nb, const double *a, const double *b, double *gl_out, double *gu_out,
                       double *t_out) {
  double gl = a[0] - fabs(b[0]), gu = a[0] + fabs(b[0]);
  for (int64_t i = 1; i < nb - 1; i++) {
    gl = dmin(gl, (a[i] - fabs(b[i - 1])) - fabs(b[i]));
    gu = dmax(gu, (a[i] + fabs(b[i - 1])) + fabs(b[i]));
  }
  gl = dmin(gl, a[nb - 1] - fabs(b[nb - 2]));
  gu = dmax(gu, a[nb - 1] + fabs(b[nb - 2]));
  double bnorm = dmax(fabs(gl), fabs(gu));
  double t = ((double)(2 * nb + 10) * bnorm) * EPS_A;
  *gl_out = gl - t;
  *gu_out = gu + t;
  if (t_out) *t_out = t;
}

/* ------------------------------------------------------------------------- */
/* Alg. negcountLDL P:7092-7119 in x-arithmetic, with dll = d l l precomputed */
/* (remark (1) P:7167-7168).                                                  */
/* ------------------------------------------------------------------------- */
int64_t oracle_negcount_x(int64_t nb, const double *d, const double *dll, double sigma) {
  int64_t count = 0;
  double s = -sigma, dp, q;
  for (int64_t i = 0; i < nb - 1; i++) {
    dp = d[i] + s;
    if (isinf(s) && isinf(dp)) q = 1.0;
    else q = s / dp;
    s = q * dll[i] - sigma;
    count += sbx(dp);
  }
  dp = d[nb - 1] + s;
  count += sbx(dp);
  return count;
}

/* the same count in y-arithmetic (binary128) */
static int64_t negcount_q(int64_t nb, const yreal *d, const yreal *dll, yreal sigma) {
  int64_t count = 0;
  yreal s = -sigma, dp, q;
  for (int64_t i = 0; i < nb - 1; i++) {
    dp = d[i] + s;
    if (YISINF(s) && YISINF(dp)) q = 1;
    else q = s / dp;
    s = q * dll[i] - sigma;
    count += sby(dp);
  }
  dp = d[nb - 1] + s;
  count += sby(dp);
  return count;
}

/* test helper: oracle_negcount_x at many shifts (OpenMP over the shifts) */
void oracle_negcount_x_many(int64_t nb, const double *d, const double *dll, int64_t ns, const double *sig,
                            int64_t *counts) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t t = 0; t < ns; t++) counts[t] = oracle_negcount_x(nb, d, dll, sig[t]);
}

/* Alg. negcountT P:7055-7077 in binary128 on T - (mu + sigma) I (pin helper) */
int64_t oracle_negcount_t_q(int64_t n, const double *a, const double *b, double mu, double sigma) {
  qreal sh = (qreal)mu + (qreal)sigma;
  int64_t count = 0;
  qreal dd = (qreal)a[0] - sh;
  count += sbq(dd);
  for (int64_t i = 1; i < n; i++) {
    qreal bb = (qreal)b[i - 1];
    dd = ((qreal)a[i] - sh) - bb * bb / dd;
    count += sbq(dd);
  }
  return count;
}

/* ------------------------------------------------------------------------- */
/* Alg. Bisection P:3077-3111 with the A-4 loop reading and the exact          */
/* midpoint w = wl + (wu - wl)/2 (A-5).                                       */
/* ------------------------------------------------------------------------- */
static inline int bis_continue(double wl, double wu, double rtol) {
  double tol = dmax(rtol * dmax(fabs(wl), fabs(wu)), ATOL);
  return fabs(wu - wl) > tol;
}

void oracle_bisect_x(int64_t nb, const double *d, const double *dll, int64_t j, double rtol,
                     double *plo, double *phi) {
  double wl = *plo, wu = *phi;
  int64_t ev = 0;
  while (bis_continue(wl, wu, rtol)) {
    double werr = (wu - wl) / 2;
    double w = wl + werr;
    ev++;
    if (oracle_negcount_x(nb, d, dll, w) < j) wl = w;
    else wu = w;
  }
  STAT_ADD(ST_NEGX, ev);
  *plo = wl;
  *phi = wu;
}

static void bisect_y_fp64pts(int64_t nb, const yreal *d, const yreal *dll, int64_t j, double rtol,
                             double *plo, double *phi) {
  double wl = *plo, wu = *phi;
  int64_t ev = 0;
  while (bis_continue(wl, wu, rtol)) {
    double w = wl + (wu - wl) / 2;
    ev++;
    if (negcount_q(nb, d, dll, (yreal)w) < j) wl = w;
    else wu = w;
  }
  STAT_ADD(ST_NEGY, ev);
  *plo = wl;
  *phi = wu;
}

/* Dyadic start interval (A-5 / DESIGN.md rule W): the smallest aligned       */
/* power-of-two grid interval covering [lo, hi]; every later midpoint is exact. */
void oracle_dyadic_widen(double lo, double hi, double *slo, double *shi) {
  double w = hi - lo;
  int ex;
  double f = frexp(w, &ex);
  double h = (f == 0.5) ? ldexp(1.0, ex - 1) : ldexp(1.0, ex);
  for (;;) {
    double a = floor(lo / h);
    if ((a + 1) * h >= hi) { *slo = a * h; *shi = (a + 1) * h; return; }
    if ((a + 2) * h >= hi) { *slo = a * h; *shi = (a + 2) * h; return; }
    h = 2 * h;
  }
}

/* Bracket repair ("inflate the input interval until the condition */
/* is met"): Require NegCount(lo) < j <= NegCount(hi).                         */
static void bracket_x(int64_t nb, const double *d, const double *dll, int64_t j, double *plo, double *phi) {
  double lo = *plo, hi = *phi;
  int64_t fix = 0;
  for (int it = 0; it < 64 && oracle_negcount_x(nb, d, dll, lo) >= j; it++) { lo = lo - (hi - lo); fix++; }
  for (int it = 0; it < 64 && oracle_negcount_x(nb, d, dll, hi) < j; it++) { hi = hi + (hi - lo); fix++; }
  STAT_ADD(ST_NEGX, 2 + 2 * fix);
  if (fix) STAT_ADD(ST_BRACKET_FIX, fix);
  *plo = lo;
  *phi = hi;
}

static void bracket_y(int64_t nb, const yreal *d, const yreal *dll, int64_t j, double *plo, double *phi) {
  double lo = *plo, hi = *phi;
  int64_t fix = 0;
  for (int it = 0; it < 64 && negcount_q(nb, d, dll, (yreal)lo) >= j; it++) { lo = lo - (hi - lo); fix++; }
  for (int it = 0; it < 64 && negcount_q(nb, d, dll, (yreal)hi) < j; it++) { hi = hi + (hi - lo); fix++; }
  STAT_ADD(ST_NEGY, 2 + 2 * fix);
  if (fix) STAT_ADD(ST_BRACKET_FIX, fix);
  *plo = lo;
  *phi = hi;
}

/* reldist(j, j+1) >= gaptol, Classification P:3272-3292 */
int oracle_is_boundary(double lo1, double hi1, double lo2, double hi2, double gaptol) {
  double num = lo2 - hi1;
  double den = dmax(dmax(fabs(lo1), fabs(hi1)), dmax(fabs(lo2), fabs(hi2)));
  return (num / den) >= gaptol;
}

/* ------------------------------------------------------------------------- */
/* Alg. dstqds P:3324-3351 and Alg. dqds P:3366-3393 (A-1, A-2 readings) in y */
/* ------------------------------------------------------------------------- */
static void dstqds_q(int64_t nb, const yreal *d, const yreal *dl, const yreal *dll, yreal tau,
                     yreal *dplus, yreal *lplus, yreal *s_out) {
  yreal s = -tau, q;
  for (int64_t i = 0; i < nb - 1; i++) {
    if (s_out) s_out[i] = s;
    dplus[i] = s + d[i];
    if (YISINF(s) && YISINF(dplus[i])) q = 1;
    else q = s / dplus[i];
    lplus[i] = dl[i] / dplus[i];
    s = q * dll[i] - tau;
  }
  if (s_out) s_out[nb - 1] = s;
  dplus[nb - 1] = s + d[nb - 1];
}

static void dqds_q(int64_t nb, const yreal *d, const yreal *dl, const yreal *dll, yreal tau,
                   yreal *omega, yreal *uminus, yreal *p_out) {
  yreal p = d[nb - 1] - tau, q;
  if (p_out) p_out[nb - 1] = p;
  for (int64_t i = nb - 2; i >= 0; i--) {
    omega[i + 1] = p + dll[i];                       /* A-1: omega^-(i+1) */
    if (YISINF(p) && YISINF(omega[i + 1])) q = 1;    /* A-2 guard */
    else q = p / omega[i + 1];
    uminus[i] = dl[i] / omega[i + 1];
    p = q * d[i] - tau;
    if (p_out) p_out[i] = p;
  }
  omega[0] = p;
}

/* ------------------------------------------------------------------------- */
/* representations                                                             */
/* ------------------------------------------------------------------------- */
typedef struct {
  int64_t nb;
  yreal *d, *l, *dl, *dll;   /* M_y: N-representation + cached dl, dll */
  double *dx, *dllx;         /* M_x = fl64(M_y) copy for x-bisection */
  yreal sigma;               /* accumulated shift: lambda[T] = lambda[M] + sigma */
  double spdiam;             /* spdiam[M_root] = gu - gl of the block */
  int depth;
} rep_t;

static rep_t *rep_alloc(int64_t nb) {
  rep_t *r = calloc(1, sizeof(rep_t));
  r->nb = nb;
  r->d = malloc(sizeof(yreal) * nb);
  r->l = malloc(sizeof(yreal) * nb);
  r->dl = malloc(sizeof(yreal) * nb);
  r->dll = malloc(sizeof(yreal) * nb);
  r->dx = malloc(sizeof(double) * nb);
  r->dllx = malloc(sizeof(double) * nb);
  return r;
}
static void rep_free(rep_t *r) {
  if (!r) return;
  free(r->d); free(r->l); free(r->dl); free(r->dll); free(r->dx); free(r->dllx);
  free(r);
}
/* derived data of a representation from (d, l) in y */
static void rep_derive(rep_t *r) {
  int64_t nb = r->nb;
  for (int64_t i = 0; i < nb - 1; i++) {
    r->dl[i] = r->d[i] * r->l[i];
    r->dll[i] = r->dl[i] * r->l[i];
  }
  r->dl[nb - 1] = 0; r->dll[nb - 1] = 0; r->l[nb - 1] = 0;
  for (int64_t i = 0; i < nb; i++) r->dx[i] = (double)r->d[i];
  for (int64_t i = 0; i < nb - 1; i++) {
    double lx = (double)r->l[i];
    r->dllx[i] = (r->dx[i] * lx) * lx;
  }
  r->dllx[nb - 1] = 0;
}

/* ------------------------------------------------------------------------- */
/* S3: root shift and root LDL^T (Alg. mrrr L1 P:2773-2774; definite root      */
/* P:2444-2448; A-8), then the random perturbation into y        */
/* (Alg. mrrr L2 P:2775-2776, mixed xi = eps_x P:5757-5770; A-9).             */
/* Returns 0 on success.                                                       */
/* ------------------------------------------------------------------------- */
/* the factorization loop of S3 from a start shift mu0: mu0, then mu0 -/+ 2^j t, j = 1..10 (A-8) */
static int root_factor_from(int64_t nb, const double *a, const double *b, int left, double mu0, double t,
                            double *mu_out, double *dx, double *lx, int *backoffs) {
  for (int j = 0; j <= 10; j++) {
    double mu = left ? ((j == 0) ? mu0 : mu0 - ldexp(t, j)) : ((j == 0) ? mu0 : mu0 + ldexp(t, j));
    dx[0] = a[0] - mu;
    for (int64_t i = 0; i < nb - 1; i++) {
      lx[i] = b[i] / dx[i];
      dx[i + 1] = (a[i + 1] - mu) - lx[i] * b[i];
    }
    int ok = 1;
    for (int64_t i = 0; i < nb && ok; i++)
      ok = isfinite(dx[i]) && (left ? (dx[i] > 0) : (dx[i] < 0));
    if (ok) { *mu_out = mu; if (backoffs) *backoffs = j; return 0; }
  }
  return -1;
}

int oracle_root_x(int64_t nb, const double *a, const double *b, int left, double *mu_out,
                  double *dx, double *lx, double *gl_out, double *gu_out, int *backoffs) {
  double gl, gu, t;
  oracle_gershgorin(nb, a, b, &gl, &gu, &t);
  *gl_out = gl; *gu_out = gu;
  return root_factor_from(nb, a, b, left, left ? gl : gu, t, mu_out, dx, lx, backoffs);
}

/* pin hook: the same back-off loop started from a caller-chosen shift mu0 with step t (a start inside the */
/* spectrum forces the back-off, which the inflated Gershgorin start never needs, A-32)           */
int oracle_root_x_from(int64_t nb, const double *a, const double *b, int left, double mu0, double t,
                       double *mu_out, double *dx, double *lx, int *backoffs) {
  return root_factor_from(nb, a, b, left, mu0, t, mu_out, dx, lx, backoffs);
}

static rep_t *make_root(int64_t n, int64_t s, int64_t nb, const double *d, const double *e, int left,
                        uint64_t seed, double *mu_out, double *gl_out, double *gu_out) {
  rep_t *r = rep_alloc(nb);
  double *lx = malloc(sizeof(double) * nb);
  int backoffs = 0;
  if (oracle_root_x(nb, d + s, e + s, left, mu_out, r->dx, lx, gl_out, gu_out, &backoffs) != 0) {
    free(lx); rep_free(r); return NULL;
  }
  if (backoffs) STAT_ADD(ST_ROOT_BACKOFF, backoffs);
  for (int64_t i = 0; i < nb; i++) {
    double x = r->dx[i];
    r->d[i] = (yreal)x + (yreal)(x * oracle_xi(seed, (uint64_t)(s + i)));
  }
  for (int64_t i = 0; i < nb - 1; i++) {
    double x = lx[i];
    r->l[i] = (yreal)x + (yreal)(x * oracle_xi(seed, (uint64_t)(n + s + i)));
  }
  r->l[nb - 1] = 0;
  rep_derive(r);   /* dx = fl64(d_y): == d_x exactly for |xi| < 2^-54; single/double: dx = d_y */
  free(lx);
  r->sigma = (yreal)(*mu_out);
  r->spdiam = *gu_out - *gl_out;
  r->depth = 0;
  return r;
}

/* ------------------------------------------------------------------------- */
/* S9: Getvec (Alg. Getvec, remarks P:3456-3482) in y.             */
/* r_io == 0: full twisted factorization and r = argmin |gamma_k| (A-16),      */
/* c = NegCount(LDL^T - lam I) from D+ (P:3477-3480).                          */
/* r_io > 0 (1-based, fixed after iteration 1): only the twisted  */
/* factorization with index r; c = inertia of Delta_r.                         */
/* ------------------------------------------------------------------------- */
typedef struct { yreal *dp, *lp, *sv, *om, *um, *gam, *z; } gv_ws;

static void gv_alloc(gv_ws *w, int64_t nb) {
  w->dp = malloc(sizeof(yreal) * nb); w->lp = malloc(sizeof(yreal) * nb);
  w->sv = malloc(sizeof(yreal) * nb); w->om = malloc(sizeof(yreal) * nb);
  w->um = malloc(sizeof(yreal) * nb); w->gam = malloc(sizeof(yreal) * nb);
  w->z = malloc(sizeof(yreal) * nb);
}
static void gv_free(gv_ws *w) {
  free(w->dp); free(w->lp); free(w->sv); free(w->om); free(w->um); free(w->gam); free(w->z);
}

static void getvec_q(const rep_t *M, yreal lam, int64_t *r_io, gv_ws *w, yreal *gamma_out, yreal *zz_out,
                     int64_t *c_out) {
  const int64_t nb = M->nb;
  const yreal *d = M->d, *dl = M->dl, *dll = M->dll;
  yreal *dp = w->dp, *lp = w->lp, *om = w->om, *um = w->um, *z = w->z;
  int64_t r, c = 0;
  yreal gamma;
  STAT_ADD(ST_GETVEC, 1);
  if (*r_io == 0) {
    dstqds_q(nb, d, dl, dll, lam, dp, lp, w->sv);
    for (int64_t i = 0; i < nb; i++) c += sby(dp[i]);
    /* dqds with gamma_k = s(k) + d(k)/omega(k+1) * p(k+1) folded in */
    yreal p = d[nb - 1] - lam, q;
    w->gam[nb - 1] = w->sv[nb - 1] + d[nb - 1];
    for (int64_t i = nb - 2; i >= 0; i--) {
      om[i + 1] = p + dll[i];
      if (YISINF(p) && YISINF(om[i + 1])) q = 1;
      else q = p / om[i + 1];
      um[i] = dl[i] / om[i + 1];
      w->gam[i] = w->sv[i] + (d[i] / om[i + 1]) * p;
      p = q * d[i] - lam;
    }
    om[0] = p;
    r = -1;
    yreal best = 0;
    for (int64_t k = 0; k < nb; k++) {
      if (YISNAN(w->gam[k])) continue;
      yreal ag = YFABS(w->gam[k]);
      if (r < 0 || ag < best) { r = k; best = ag; }
    }
    if (r < 0) { *r_io = 0; *gamma_out = NAN; *zz_out = NAN; *c_out = c; return; }
    gamma = w->gam[r];
    *r_io = r + 1;
  } else {
    r = *r_io - 1;
    yreal s = -lam, q;
    for (int64_t i = 0; i < r; i++) {
      dp[i] = s + d[i];
      if (YISINF(s) && YISINF(dp[i])) q = 1;
      else q = s / dp[i];
      lp[i] = dl[i] / dp[i];
      s = q * dll[i] - lam;
      c += sby(dp[i]);
    }
    if (r == nb - 1) {
      gamma = s + d[nb - 1];
    } else {
      yreal p = d[nb - 1] - lam;
      gamma = 0;
      for (int64_t i = nb - 2; i >= r; i--) {
        om[i + 1] = p + dll[i];
        if (YISINF(p) && YISINF(om[i + 1])) q = 1;
        else q = p / om[i + 1];
        um[i] = dl[i] / om[i + 1];
        if (i == r) gamma = s + (d[r] / om[r + 1]) * p;
        p = q * d[i] - lam;
        c += sby(om[i + 1]);
      }
    }
    c += sby(gamma);
  }
  /* solve N_r^T z = e_r with zero-pivot substitution;          */
  /* DESIGN.md reading A-25: immediate neighbours first, undefined refs := 0 */
  for (int64_t i = 0; i < nb; i++) z[i] = 0;
  z[r] = 1;
  if (r > 0 && dp[r - 1] != 0) z[r - 1] = -lp[r - 1] * z[r];
  if (r < nb - 1 && om[r + 1] != 0) z[r + 1] = -um[r] * z[r];
  for (int64_t i = r - 1; i >= 0; i--) {
    if (dp[i] != 0) z[i] = -lp[i] * z[i + 1];
    else {
      STAT_ADD(ST_ZPIV, 1);
      yreal num = (i + 1 < nb - 1) ? dl[i + 1] : 0, zz2 = (i + 2 < nb) ? z[i + 2] : 0;
      yreal v = -(num / dl[i]) * zz2;
      z[i] = YFINITE(v) ? v : 0;
    }
  }
  for (int64_t i = r; i < nb - 1; i++) {
    if (om[i + 1] != 0) z[i + 1] = -um[i] * z[i];
    else {
      STAT_ADD(ST_ZPIV, 1);
      yreal num = (i >= 1) ? dl[i - 1] : 0, zm = (i >= 1) ? z[i - 1] : 0;
      yreal v = -(num / dl[i]) * zm;
      z[i + 1] = YFINITE(v) ? v : 0;
    }
  }
  yreal zz = 0;
  for (int64_t i = 0; i < nb; i++) zz += z[i] * z[i];
  *gamma_out = gamma;
  *zz_out = zz;
  *c_out = c;
}

/* y-bisection to full accuracy (fallback of RQI): Alg. Bisection P:3077-3111 on the  */
/* y-representation with y-arithmetic counts, stopping at relative width 2^-98 of |lambda| (a few eps_y,    */
/* A-14) or at atol = 2 omega.  Pinned: tests/test_oracle_branches.py (binary128 Jacobi).     */
static yreal bisect_y_full(const rep_t *M, int64_t j, yreal lo, yreal hi) {
  for (int it = 0; it < 400; it++) {
    yreal m = YFMAX(YFABS(lo), YFABS(hi));
    if (!(hi - lo > YFMAX(Y_FULLREL * m, (yreal)ATOL))) break;
    yreal w = lo + (hi - lo) / 2;
    STAT_ADD(ST_NEGY, 1);
    if (negcount_q(M->nb, M->d, M->dll, w) < j) lo = w;
    else hi = w;
  }
  return lo + (hi - lo) / 2;
}

/* RQI for a singleton, Alg. stask P:4026-4074 with the mixed stopping rule    */
/* ||r|| <= k_rs gap eps_x sqrt(n), k_rs = 1 (A-14, A-15).       */
/* j is the 1-based index in M; [lo, hi] its x-interval; gap > 0.             */
/* S10' numerical support (Getvec remark (2): "for all i < i_first and i > i_last, z(i) can be set */
/* to zero ... easily detected and exploited"; A-42).  The paper gives no rule.  Reading: cutting z   */
/* at the edge between rows i and i+1 (coupling dl(i), the off-diagonal of LDL^T) changes the residual of the  */
/* twisted solution (z(r) = 1) by exactly |dl(i)| (|z(i)| + |z(i+1)|) in two entries, so by the gap theorem     */
/* the cut vector stays within angle ~eps_x of the eigenvector when that term is <= gap eps_x.  Going outward */
/* from r, the support ends at the first edge with |dl(i)| (|z(i)| + |z(i+1)|) <= gap eps_x; the entries past */
/* it are set to zero.  Returns ||z||^2 of the truncated vector.                                                */
static yreal numerical_support(const rep_t *M, yreal *z, int64_t r, double gap) {
  const int64_t nb = M->nb;
  const yreal tau = (yreal)(gap * EPS_X);
  int64_t first = 0, last = nb - 1;  /* 0-based support [first, last]; r is 0-based */
  for (int64_t i = r - 1; i >= 0; i--)
    if (YFABS(M->dl[i]) * (YFABS(z[i]) + YFABS(z[i + 1])) <= tau) { first = i + 1; break; }
  for (int64_t i = r; i < nb - 1; i++)
    if (YFABS(M->dl[i]) * (YFABS(z[i]) + YFABS(z[i + 1])) <= tau) { last = i; break; }
  for (int64_t i = 0; i < first; i++) z[i] = 0;
  for (int64_t i = last + 1; i < nb; i++) z[i] = 0;
  STAT_ADD(ST_SUPPORT, last - first + 1);
  yreal zz = 0;
  for (int64_t i = first; i <= last; i++) zz += z[i] * z[i];
  return zz;
}

static void rqi_singleton(const rep_t *M, int64_t j, double lo, double hi, double gap, int support,
                          double *W_out, double *zcol, gv_ws *w) {
  const int64_t nb = M->nb;
  double mid = lo + (hi - lo) / 2;
  double nu = (100.0 * (double)nb) * EPS_A;
  yreal blo = (yreal)(lo - nu * fabs(lo)), bhi = (yreal)(hi + nu * fabs(hi));
  yreal lam = (yreal)mid, gamma, zz;
  double thr1 = (gap * EPS_X) * sqrt((double)nb);
  int64_t r = 0, c, iters = 0;
  int accepted = 0;
  for (int it = 0; it < MAX_RQI && !accepted; it++) {
    getvec_q(M, lam, &r, w, &gamma, &zz, &c);
    iters++;
    if (r == 0 || !YFINITE(zz) || zz == 0) break;
    yreal nz = YSQRT(zz);
    yreal resid = YFABS(gamma) / nz, rqc = gamma / zz;
    /* stopping tests of Alg. stask: ||r|| <= tol1 (mixed: k_rs gap eps_x sqrt(n)) */
    /* or |RQC| < tol2 |lam| with tol2 = 4 eps_y (A-14)                                                        */
    if ((double)resid <= thr1 || YFABS(rqc) < 4 * EPS_Y * YFABS(lam)) { accepted = 1; break; }
    if (c < j) blo = lam; else bhi = lam;
    yreal nl = lam + rqc;
    int ok = ((c < j) ? (rqc > 0) : (rqc < 0)) && (blo < nl) && (nl < bhi);
    if (ok) lam = nl;
    else break;
  }
  STAT_ADD(ST_RQI_ITERS, iters);
  if (!accepted) {
    STAT_ADD(ST_RQI_FALLBACK, 1);
    lam = bisect_y_full(M, j, blo, bhi);
    getvec_q(M, lam, &r, w, &gamma, &zz, &c);
  }
  if (support && r > 0) zz = numerical_support(M, w->z, r - 1, gap);
  yreal nz = YSQRT(zz);
  *W_out = (double)(lam + M->sigma);
  for (int64_t i = 0; i < nb; i++) zcol[i] = (double)(w->z[i] / nz);
}

/* ------------------------------------------------------------------------- */
/* tree traversal (depth-first)                                   */
/* ------------------------------------------------------------------------- */
typedef struct {
  int64_t n, k, ldz, bstart;  /* global size, #outputs, ldz, block start */
  const int32_t *colmap;      /* [nb+1] 1-based local -> output column or -1 */
  double gaptol, rtol;
  int support;                /* S10' (A-42) */
  double *W, *Z;
  oracle_diag *dg;
} ctx_t;

static void process_group(const ctx_t *cx, const rep_t *M, double *lo, double *hi, int64_t p, int64_t q);

static void emit_depth_info(const ctx_t *cx, int depth, int64_t p, int64_t q) {
  oracle_diag *dg = cx->dg;
  if (!dg || !dg->grp_first || depth >= MAXD) return;
  for (int64_t j = p; j <= q; j++) {
    int32_t col = cx->colmap[j];
    if (col < 0) continue;
    dg->grp_first[(int64_t)depth * cx->k + col] = (int32_t)(cx->bstart + p - 1);
    dg->grp_last[(int64_t)depth * cx->k + col] = (int32_t)(cx->bstart + q - 1);
  }
}

static int group_selected(const ctx_t *cx, int64_t p, int64_t q) {
  for (int64_t j = p; j <= q; j++) if (cx->colmap[j] >= 0) return 1;
  return 0;
}

static void do_singleton(const ctx_t *cx, const rep_t *M, const double *lo, const double *hi, int64_t j) {
  int32_t col = cx->colmap[j];
  if (col < 0) return;
  double mid = lo[j] + (hi[j] - lo[j]) / 2;
  double gl = (j > 1 && !isnan(lo[j - 1])) ? mid - hi[j - 1] : INFINITY;
  double gr = (j < M->nb && !isnan(lo[j + 1])) ? lo[j + 1] - mid : INFINITY;
  double gap = dmin(gl, gr);
  gv_ws w;
  gv_alloc(&w, M->nb);
  double *zc = malloc(sizeof(double) * M->nb);
  double Wv;
  rqi_singleton(M, j, lo[j], hi[j], gap, cx->support, &Wv, zc, &w);
  cx->W[col] = Wv;
  double *Zc = cx->Z + (int64_t)col * cx->ldz;
  for (int64_t i = 0; i < cx->n; i++) Zc[i] = 0.0;
  memcpy(Zc + cx->bstart, zc, sizeof(double) * M->nb);
  if (cx->dg) {
    if (cx->dg->depth) cx->dg->depth[col] = M->depth;
    if (cx->dg->fin_lo) { cx->dg->fin_lo[col] = lo[j]; cx->dg->fin_hi[col] = hi[j]; }
  }
  stat_max(ST_DMAX, M->depth);
  free(zc);
  gv_free(&w);
}

/* S8: a cluster {p..q} of M: Alg. spectrumshift P:3499-3545 (+ remarks,       */
/* A-11, A-12), child intervals P:3576-3590 (A-13), reclassify, recurse.       */
static void do_cluster(const ctx_t *cx, const rep_t *M, const double *lo, const double *hi, int64_t p,
                       int64_t q) {
  const int64_t nb = M->nb;
  STAT_ADD(ST_NCLUSTERS, 1);
  stat_max(ST_LARGEST, q - p + 1);
  double nu = (100.0 * (double)nb) * EPS_A;
  /* (a) refine the extremal eigenvalues of M_y (y-arithmetic), starting from their x-intervals */
  /* (A-12'': the eigenvalue of M_y lies within ~n eps_x |lambda| of M_x's; bracket repair in y widens the     */
  /* start by its own width on a failing side, on the same dyadic grid)                                        */
  double Lp = lo[p], Hp = hi[p];
  double Lq = lo[q], Hq = hi[q];
  oracle_dyadic_widen(Lp, Hp, &Lp, &Hp);
  oracle_dyadic_widen(Lq, Hq, &Lq, &Hq);
  bracket_y(nb, M->d, M->dll, p, &Lp, &Hp);
  bracket_y(nb, M->d, M->dll, q, &Lq, &Hq);
  bisect_y_fp64pts(nb, M->d, M->dll, p, RTOL_Y, &Lp, &Hp);
  bisect_y_fp64pts(nb, M->d, M->dll, q, RTOL_Y, &Lq, &Hq);
  /* (b) tau_l = lam_p_low - 100 eps |.|, tau_r = lam_q_up + 100 eps |.| */
  double offl = (100.0 * EPS_A) * fabs(Lp), offr = (100.0 * EPS_A) * fabs(Hq);
  double taul = Lp - offl, taur = Hq + offr;
  /* (c) attempts */
  yreal *dpl = malloc(sizeof(yreal) * nb), *lpl = malloc(sizeof(yreal) * nb);
  yreal *dpr = malloc(sizeof(yreal) * nb), *lpr = malloc(sizeof(yreal) * nb);
  yreal *bd = malloc(sizeof(yreal) * nb), *bl = malloc(sizeof(yreal) * nb);
  double best_g = INFINITY, best_tau = 0;
  int have_best = 0, certified = 0;
  /* growth bound of the mixed solver, eq:newkelgbound P:6052-6056 (A-35): k_elg <= max(original, eps_x / (eps_y */
  /* sqrt(n))), with the original bound G = 64 of A-11                                                             */
  double gthr = dmax(GROWTH, KELG_RATIO / sqrt((double)nb)) * M->spdiam;
  for (int a = 0; a < MAX_ATTEMPTS; a++) {
    STAT_ADD(ST_ATTEMPTS, 1);
    dstqds_q(nb, M->d, M->dl, M->dll, (yreal)taul, dpl, lpl, NULL);
    dstqds_q(nb, M->d, M->dl, M->dll, (yreal)taur, dpr, lpr, NULL);
    int vl = 1, vr = 1;
    double gl = 0, gr = 0;
    for (int64_t i = 0; i < nb; i++) {
      if (YISNAN(dpl[i]) || (i < nb - 1 && YISNAN(lpl[i]))) vl = 0;
      if (YISNAN(dpr[i]) || (i < nb - 1 && YISNAN(lpr[i]))) vr = 0;
      gl = dmax(gl, fabs((double)dpl[i]));
      gr = dmax(gr, fabs((double)dpr[i]));
    }
    int pick = 0; /* 1 left, 2 right */
    if (vl && vr) pick = (gl <= gr) ? 1 : 2;
    else if (vl) pick = 1;
    else if (vr) pick = 2;
    if (pick) {
      double g = (pick == 1) ? gl : gr;
      if (g < best_g) {
        best_g = g; best_tau = (pick == 1) ? taul : taur; have_best = 1;
        memcpy(bd, (pick == 1) ? dpl : dpr, sizeof(yreal) * nb);
        memcpy(bl, (pick == 1) ? lpl : lpr, sizeof(yreal) * nb);
      }
      if (g <= gthr) { certified = 1; break; }
    }
    taul = taul - ldexp(offl, a);
    taur = taur + ldexp(offr, a);
  }
  free(dpl); free(lpl); free(dpr); free(lpr);
  if (!have_best) {
    STAT_ADD(ST_FAILED, 1);
    free(bd); free(bl);
    for (int64_t j = p; j <= q; j++) do_singleton(cx, M, lo, hi, j);
    return;
  }
  if (!certified) STAT_ADD(ST_UNCERTIFIED, 1);
  /* (d) child representation M_y, M_x */
  rep_t *C = rep_alloc(nb);
  memcpy(C->d, bd, sizeof(yreal) * nb);
  memcpy(C->l, bl, sizeof(yreal) * nb);
  free(bd); free(bl);
  rep_derive(C);
  C->sigma = M->sigma + (yreal)best_tau;
  C->spdiam = M->spdiam;
  C->depth = M->depth + 1;
  /* (e) child intervals */
  double *clo = malloc(sizeof(double) * (nb + 2)), *chi = malloc(sizeof(double) * (nb + 2));
  for (int64_t j = 0; j < nb + 2; j++) clo[j] = chi[j] = NAN;
  double tau = best_tau;
  if (p > 1 && !isnan(lo[p - 1])) { clo[p - 1] = lo[p - 1] - tau; chi[p - 1] = hi[p - 1] - tau; }
  if (q < nb && !isnan(lo[q + 1])) { clo[q + 1] = lo[q + 1] - tau; chi[q + 1] = hi[q + 1] - tau; }
#pragma omp taskloop grainsize(1) shared(clo, chi, C, lo, hi)
  for (int64_t j = p; j <= q; j++) {
    /* the cluster ends start from their y-refined intervals, which bracket the eigenvalues of M_y itself: the  */
    /* inner inflation then covers only the y-arithmetic shift, nu_y = 100 n eps_y (A-13'); the others from    */
    /* their x-intervals with nu                                                                                */
    const int end = (j == p || j == q);
    const double nin = end ? (100.0 * (double)nb) * EPS_Y : nu;
    const double lj = (j == p) ? Lp : (j == q) ? Lq : lo[j], hj = (j == p) ? Hp : (j == q) ? Hq : hi[j];
    double a1 = lj - nin * fabs(lj);
    double b1 = a1 - tau;
    double l2 = b1 - nu * fabs(b1);
    double c1 = hj + nin * fabs(hj);
    double e1 = c1 - tau;
    double h2 = e1 + nu * fabs(e1);
    double L, H;
    oracle_dyadic_widen(l2, h2, &L, &H);
    bracket_x(nb, C->dx, C->dllx, j, &L, &H);
    oracle_bisect_x(nb, C->dx, C->dllx, j, cx->rtol, &L, &H);
    clo[j] = L;
    chi[j] = H;
  }
  /* (f) reclassify and recurse */
  if (C->depth >= MAXD) {
    STAT_ADD(ST_FAILED, 1);
    for (int64_t j = p; j <= q; j++) do_singleton(cx, C, clo, chi, j);
  } else {
    int64_t g0 = p;
    for (int64_t j = p + 1; j <= q + 1; j++) {
      if (j == q + 1 || oracle_is_boundary(clo[j - 1], chi[j - 1], clo[j], chi[j], cx->gaptol)) {
        int64_t g1 = j - 1;
        if (group_selected(cx, g0, g1)) {
#pragma omp task firstprivate(g0, g1) shared(C, clo, chi)
          process_group(cx, C, clo, chi, g0, g1);
        }
        g0 = j;
      }
    }
#pragma omp taskwait
  }
  free(clo); free(chi);
  rep_free(C);
}

static void process_group(const ctx_t *cx, const rep_t *M, double *lo, double *hi, int64_t p, int64_t q) {
  emit_depth_info(cx, M->depth, p, q);
  if (p == q) do_singleton(cx, M, lo, hi, p);
  else do_cluster(cx, M, lo, hi, p, q);
}

/* ------------------------------------------------------------------------- */
/* driver: S0-S10, Alg. mrrr P:2762-2816 / Alg. mrrr2 */
/* ------------------------------------------------------------------------- */
typedef struct {
  int64_t s, nb;
  int left;
  double mu, gl, gu;
  rep_t *root;
  double *lo, *hi;   /* [nb+2], 1-based, NaN = not computed */
  double *s1lo, *s1hi; /* [nb+2] stage-1 intervals of the early stop (S5'), NaN = not computed */
  int64_t ca, cb;    /* computed range */
  int64_t jl, ju;    /* selected range (ju < jl: none) */
  int32_t *colmap;   /* [nb+2] */
} blk_t;

typedef struct { double v; int64_t b, j; } rank_t;
static int rank_cmp(const void *x, const void *y) {
  const rank_t *a = x, *b = y;
  if (a->v < b->v) return -1;
  if (a->v > b->v) return 1;
  if (a->b != b->b) return (a->b < b->b) ? -1 : 1;
  return (a->j < b->j) ? -1 : (a->j > b->j);
}

static void root_bisect_one(blk_t *B, int64_t j, double rtol) {
  double lo = B->left ? 0.0 : -B->hi[0], hi = B->left ? B->hi[0] : 0.0;  /* hi[0] holds 2^E */
  oracle_bisect_x(B->nb, B->root->dx, B->root->dllx, j, rtol, &lo, &hi);
  B->lo[j] = lo;
  B->hi[j] = hi;
}

/* ------------------------------------------------------------------------- */
/* S5' Early classification stop: "only sufficient accuracy to  */
/* classify eigenvalues into well-separated and clustered is needed ...        */
/* Depending on the absolute gap of the eigenvalue, the refinement can be      */
/* stopped earlier on" (sec. 3.2.2 remark (3); A-41).   */
/* Stage 1 bisects index j to rtol_c = max(rtol, 2^-(10 + ceil(log2 n)));      */
/* j (2 <= j <= nb-1) stops there when both neighbour pairs are already        */
/* classification boundaries (reldist >= gaptol) and its width is */
/* at most 2^-7 of its absolute gap; every other index continues from its      */
/* stage-1 interval to rtol -- the same bisection path, hence the same final   */
/* interval as without the stop.  A stopped interval contains the stage-1      */
/* intervals' final refinements of the full run, so reldist only grows: the    */
/* cluster boundaries are those of the full run.                               */
/* ------------------------------------------------------------------------- */
double oracle_es_rtol(int64_t n, double rtol) {
  int e = 0;
  while (e < 62 && ((int64_t)1 << e) < n) e++;   /* ceil(log2 n) */
  return dmax(rtol, ldexp(1.0, -(10 + e)));
}
/* the stop test of index j from the stage-1 intervals of j-1, j, j+1 */
int oracle_es_stop(double llo, double lhi, double clo, double chi, double rlo, double rhi, double gaptol) {
  if (!oracle_is_boundary(llo, lhi, clo, chi, gaptol) || !oracle_is_boundary(clo, chi, rlo, rhi, gaptol)) return 0;
  double gap = dmin(clo - lhi, rlo - chi);
  return (chi - clo) <= ldexp(gap, -7);
}
static void stage1_one(blk_t *B, int64_t j, double rtol_c) {
  if (j < 1 || j > B->nb || !isnan(B->s1lo[j])) return;
  double lo = B->left ? 0.0 : -B->hi[0], hi = B->left ? B->hi[0] : 0.0;
  oracle_bisect_x(B->nb, B->root->dx, B->root->dllx, j, rtol_c, &lo, &hi);
  B->s1lo[j] = lo;
  B->s1hi[j] = hi;
}
/* stage 2 of index j (its stage-1 interval and its neighbours' computed): stop, or continue to rtol */
static void stage2_one(blk_t *B, int64_t j, double rtol, double gaptol) {
  double lo = B->s1lo[j], hi = B->s1hi[j];
  if (j >= 2 && j <= B->nb - 1 &&
      oracle_es_stop(B->s1lo[j - 1], B->s1hi[j - 1], lo, hi, B->s1lo[j + 1], B->s1hi[j + 1], gaptol)) {
    STAT_ADD(ST_ESTOP, 1);
  } else {
    oracle_bisect_x(B->nb, B->root->dx, B->root->dllx, j, rtol, &lo, &hi);
  }
  B->lo[j] = lo;
  B->hi[j] = hi;
}
/* one index with the early stop (guard extension, one at a time) */
static void root_bisect_es(blk_t *B, int64_t j, double rtol_c, double rtol, double gaptol) {
  for (int64_t x = j - 1; x <= j + 1; x++) stage1_one(B, x, rtol_c);
  stage2_one(B, j, rtol, gaptol);
}

static int mrrr_scaled(int64_t n, const double *d, const double *e, int64_t il, int64_t iu, const oracle_opts *op,
                       double *W, double *Z, int64_t ldz, oracle_diag *dg);

/* S0 scaling (P:3026-3027 defers it; A-21): when the largest |entry| a = max(|alpha_i|, |beta_i|)  */
/* lies outside [2^-500, 2^500] the solve runs on 2^s T with 2^s a in [1/2, 1) (so 2^s ||T||_1 < 3) -- a     */
/* power of two, so every step of the scaled solve is the exact image of the unscaled one away from         */
/* over/underflow -- and W is scaled back by 2^-s (Z is scale invariant).  Diagnostics (mu, intervals) stay  */
/* in the scaled frame.                                                                                      */
int oracle_mrrr(int64_t n, const double *d, const double *e, int64_t il, int64_t iu, const oracle_opts *op,
                double *W, double *Z, int64_t ldz, oracle_diag *dg) {
  if (n < 1) return -4;
  if (il < 1 || il > n) return -5;
  if (iu < il || iu > n) return -6;
  if (!d || (n > 1 && !e)) return -2;
  if (ldz < n) return -9;
  for (int64_t i = 0; i < n; i++) if (!isfinite(d[i]) || (i < n - 1 && !isfinite(e[i]))) return 1;
  double amax = 0;
  for (int64_t i = 0; i < n; i++) amax = dmax(amax, fabs(d[i]));
  for (int64_t i = 0; i < n - 1; i++) amax = dmax(amax, fabs(e[i]));
  if (amax == 0 || (amax >= 0x1p-500 && amax <= 0x1p500))
    return mrrr_scaled(n, d, e, il, iu, op, W, Z, ldz, dg);
  int ex;
  frexp(amax, &ex);   /* amax = f 2^ex, f in [1/2, 1) */
  double *ds = malloc(sizeof(double) * n), *es = malloc(sizeof(double) * (n > 1 ? n - 1 : 1));
  for (int64_t i = 0; i < n; i++) ds[i] = ldexp(d[i], -ex);
  for (int64_t i = 0; i < n - 1; i++) es[i] = ldexp(e[i], -ex);
  int rc = mrrr_scaled(n, ds, es, il, iu, op, W, Z, ldz, dg);
  if (rc == 0)
    for (int64_t j = 0; j < iu - il + 1; j++) W[j] = ldexp(W[j], ex);
  free(ds);
  free(es);
  return rc;
}

/* the solve proper (S1-S10) on an input with ||T||_1 in range (or 0) */
static int mrrr_scaled(int64_t n, const double *d, const double *e, int64_t il, int64_t iu, const oracle_opts *op,
                       double *W, double *Z, int64_t ldz, oracle_diag *dg) {
  double gaptol = (op && op->gaptol > 0) ? op->gaptol : DEFAULT_GAPTOL;
  uint64_t seed = (op && op->seed) ? op->seed : DEFAULT_SEED;
  int force = op ? op->root_side : 0;
  if (op && op->threads > 0) omp_set_num_threads(op->threads);
  double rtol = 1e-2 * gaptol;
  int es = op ? op->early_stop : 0;  /* S5' (A-41) */
  double rtol_c = es ? oracle_es_rtol(n, rtol) : rtol;
  int64_t k = iu - il + 1;
  memset(g_stats, 0, sizeof(g_stats));

  /* S1-S2 */
  int32_t *starts = malloc(sizeof(int32_t) * (n + 1));
  int64_t nblk = oracle_split(n, d, e, starts);
  if (dg && dg->nblocks) dg->nblocks[0] = (int32_t)nblk;
  if (dg && dg->block_start) memcpy(dg->block_start, starts, sizeof(int32_t) * (nblk + 1));
  if (dg && dg->root_lo) for (int64_t i = 0; i < n; i++) { dg->root_lo[i] = NAN; dg->root_hi[i] = NAN; }
  if (dg && dg->root_gstart) for (int64_t i = 0; i < n; i++) dg->root_gstart[i] = -1;
  if (dg && dg->grp_first) for (int64_t i = 0; i < MAXD * k; i++) { dg->grp_first[i] = -1; dg->grp_last[i] = -1; }

  blk_t *B = calloc(nblk, sizeof(blk_t));
  int single = (nblk == 1);
  for (int64_t b = 0; b < nblk; b++) {
    B[b].s = starts[b];
    B[b].nb = starts[b + 1] - starts[b];
    int64_t nb = B[b].nb;
    B[b].lo = malloc(sizeof(double) * (nb + 2));
    B[b].hi = malloc(sizeof(double) * (nb + 2));
    B[b].colmap = malloc(sizeof(int32_t) * (nb + 2));
    B[b].s1lo = malloc(sizeof(double) * (nb + 2));
    B[b].s1hi = malloc(sizeof(double) * (nb + 2));
    for (int64_t j = 0; j < nb + 2; j++) {
      B[b].lo[j] = B[b].hi[j] = NAN; B[b].colmap[j] = -1;
      B[b].s1lo[j] = B[b].s1hi[j] = NAN;
    }
    if (single) { B[b].jl = il; B[b].ju = iu; }
    else { B[b].jl = 1; B[b].ju = nb; }
  }

  /* S3: roots */
  int err = 0;
  for (int64_t b = 0; b < nblk && !err; b++) {
    blk_t *X = &B[b];
    if (X->nb == 1) {
      X->mu = 0; X->left = 1;
      X->lo[1] = X->hi[1] = d[X->s];
      X->ca = X->cb = 1;
      if (dg && dg->mu) dg->mu[b] = 0;
      if (dg && dg->side) dg->side[b] = 0;
      continue;
    }
    X->left = (force == 1) ? 1 : (force == 2) ? 0 : ((X->jl - 1) <= (X->nb - X->ju));
    X->root = make_root(n, X->s, X->nb, d, e, X->left, seed, &X->mu, &X->gl, &X->gu);
    if (!X->root) { err = 2; break; }
    if (dg && dg->mu) dg->mu[b] = X->mu;
    if (dg && dg->side) dg->side[b] = X->left ? 1 : 2;
    /* start interval [0, 2^E] (left) / [-2^E, 0] (right), verified (S5) */
    double x = X->left ? (X->gu - X->mu) : (X->mu - X->gl);
    int ex;
    double f = frexp(x, &ex);
    double P = (f == 0.5) ? ldexp(1.0, ex - 1) : ldexp(1.0, ex);
    for (int it = 0; it < 64; it++) {
      int64_t c = oracle_negcount_x(X->nb, X->root->dx, X->root->dllx, X->left ? P : -P);
      STAT_ADD(ST_NEGX, 1);
      if (X->left ? (c == X->nb) : (c == 0)) break;
      P = 2 * P;
    }
    X->hi[0] = P;   /* scratch slot: 2^E */
    /* S4/S5 computed set */
    X->ca = (X->jl > 1) ? X->jl - 1 : X->jl;
    X->cb = (X->ju < X->nb) ? X->ju + 1 : X->ju;
    if (!single) { X->ca = 1; X->cb = X->nb; }
  }
  if (err) goto done;

  /* S5: root bisection of the computed sets (Alg. Bisection per index) */
  for (int64_t b = 0; b < nblk; b++) {
    blk_t *X = &B[b];
    if (X->nb == 1) continue;
    if (es) {
      /* S5': stage 1 of the computed set and its neighbours, then the stop test / stage 2 per index */
      int64_t a1 = X->ca > 1 ? X->ca - 1 : 1, b1 = X->cb < X->nb ? X->cb + 1 : X->nb;
#pragma omp parallel for schedule(dynamic, 4)
      for (int64_t j = a1; j <= b1; j++) stage1_one(X, j, rtol_c);
#pragma omp parallel for schedule(dynamic, 4)
      for (int64_t j = X->ca; j <= X->cb; j++) stage2_one(X, j, rtol, gaptol);
    } else {
#pragma omp parallel for schedule(dynamic, 4)
      for (int64_t j = X->ca; j <= X->cb; j++) root_bisect_one(X, j, rtol);
    }
    /* guard extension while clustered (single-block subsets) */
    while (X->ca > 1 && !oracle_is_boundary(X->lo[X->ca], X->hi[X->ca], X->lo[X->ca + 1], X->hi[X->ca + 1], gaptol)) {
      X->ca--;
      if (es) root_bisect_es(X, X->ca, rtol_c, rtol, gaptol);
      else root_bisect_one(X, X->ca, rtol);
    }
    while (X->cb < X->nb && !oracle_is_boundary(X->lo[X->cb - 1], X->hi[X->cb - 1], X->lo[X->cb], X->hi[X->cb], gaptol)) {
      X->cb++;
      if (es) root_bisect_es(X, X->cb, rtol_c, rtol, gaptol);
      else root_bisect_one(X, X->cb, rtol);
    }
    X->hi[0] = NAN;
  }

  if (op && op->roots_only) {
    for (int64_t b = 0; b < nblk; b++) {
      blk_t *X = &B[b];
      if (dg && dg->root_lo)
        for (int64_t j = X->ca; j <= X->cb; j++) { dg->root_lo[X->s + j - 1] = X->lo[j]; dg->root_hi[X->s + j - 1] = X->hi[j]; }
      if (dg && dg->root_gstart)
        for (int64_t j = X->ca; j <= X->cb; j++)
          dg->root_gstart[X->s + j - 1] = (j == X->ca) ? 1 : oracle_is_boundary(X->lo[j - 1], X->hi[j - 1], X->lo[j], X->hi[j], gaptol);
    }
    goto done;
  }

  /* S4: selection -> output columns */
  if (single) {
    for (int64_t j = il; j <= iu; j++) B[0].colmap[j] = (int32_t)(j - il);
  } else {
    rank_t *R = malloc(sizeof(rank_t) * n);
    int64_t m = 0;
    for (int64_t b = 0; b < nblk; b++)
      for (int64_t j = 1; j <= B[b].nb; j++) {
        double mid = B[b].lo[j] + (B[b].hi[j] - B[b].lo[j]) / 2;
        R[m].v = (B[b].nb == 1) ? mid : mid + B[b].mu;
        R[m].b = b; R[m].j = j; m++;
      }
    qsort(R, (size_t)m, sizeof(rank_t), rank_cmp);
    for (int64_t r = il; r <= iu; r++) B[R[r - 1].b].colmap[R[r - 1].j] = (int32_t)(r - il);
    free(R);
  }

  /* diagnostics: root intervals and root groups */
  for (int64_t b = 0; b < nblk; b++) {
    blk_t *X = &B[b];
    if (dg && dg->root_lo)
      for (int64_t j = X->ca; j <= X->cb; j++) { dg->root_lo[X->s + j - 1] = X->lo[j]; dg->root_hi[X->s + j - 1] = X->hi[j]; }
    if (dg && dg->root_gstart)
      for (int64_t j = X->ca; j <= X->cb; j++)
        dg->root_gstart[X->s + j - 1] = (j == X->ca) ? 1 : oracle_is_boundary(X->lo[j - 1], X->hi[j - 1], X->lo[j], X->hi[j], gaptol);
  }

  /* S6-S10: classify and process groups intersecting the selection */
#pragma omp parallel
#pragma omp single
  for (int64_t b = 0; b < nblk; b++) {
    blk_t *X = &B[b];
    if (X->nb == 1) {
      int32_t col = X->colmap[1];
      if (col >= 0) {
        W[col] = d[X->s];
        double *Zc = Z + (int64_t)col * ldz;
        for (int64_t i = 0; i < n; i++) Zc[i] = 0.0;
        Zc[X->s] = 1.0;
        if (dg && dg->depth) dg->depth[col] = 0;
        if (dg && dg->fin_lo) { dg->fin_lo[col] = d[X->s]; dg->fin_hi[col] = d[X->s]; }
        if (dg && dg->grp_first) { dg->grp_first[col] = (int32_t)X->s; dg->grp_last[col] = (int32_t)X->s; }
      }
      continue;
    }
    ctx_t *cx = malloc(sizeof(ctx_t));
    cx->n = n; cx->k = k; cx->ldz = ldz; cx->bstart = X->s; cx->colmap = X->colmap;
    cx->gaptol = gaptol; cx->rtol = rtol; cx->support = op ? op->support : 0; cx->W = W; cx->Z = Z; cx->dg = dg;
    int64_t g0 = X->ca;
    for (int64_t j = X->ca + 1; j <= X->cb + 1; j++) {
      if (j == X->cb + 1 || oracle_is_boundary(X->lo[j - 1], X->hi[j - 1], X->lo[j], X->hi[j], gaptol)) {
        int64_t g1 = j - 1;
        if (group_selected(cx, g0, g1)) {
#pragma omp task firstprivate(g0, g1, X, cx)
          process_group(cx, X->root, X->lo, X->hi, g0, g1);
        }
        g0 = j;
      }
    }
#pragma omp taskwait
    free(cx);
  }

done:
  if (dg && dg->stats) memcpy(dg->stats, g_stats, sizeof(g_stats));
  for (int64_t b = 0; b < nblk; b++) {
    rep_free(B[b].root);
    free(B[b].lo); free(B[b].hi); free(B[b].colmap); free(B[b].s1lo); free(B[b].s1hi);
  }
  free(B);
  free(starts);
  return err;
}

/* ------------------------------------------------------------------------- */
/* verification helpers (test tools, not part of the method)                    */
/* ------------------------------------------------------------------------- */

/* ||T z_j - W_j z_j||_2 evaluated in binary128 (fp64 products are exact) */
void oracle_residuals(int64_t n, const double *d, const double *e, int64_t k, const double *W, const double *Z,
                      int64_t ldz, double *res) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < k; j++) {
    const double *z = Z + j * ldz;
    qreal acc = 0, lam = (qreal)W[j];
    for (int64_t i = 0; i < n; i++) {
      qreal t = ((qreal)d[i] - lam) * (qreal)z[i];
      if (i > 0) t += (qreal)e[i - 1] * (qreal)z[i - 1];
      if (i < n - 1) t += (qreal)e[i] * (qreal)z[i + 1];
      acc += t * t;
    }
    res[j] = (double)sqrtq(acc);
  }
}

/* exact-ish dot (binary128 accumulation of exact fp64 products) */
static double dotq(int64_t n, const double *x, const double *y) {
  qreal acc = 0;
  for (int64_t i = 0; i < n; i++) acc += (qreal)x[i] * (qreal)y[i];
  return (double)acc;
}

/* max over the given pairs of |z_i . z_j - delta_ij| */
double oracle_ortho_pairs(int64_t n, const double *Z, int64_t ldz, int64_t npairs, const int64_t *pi,
                          const int64_t *pj) {
  double mx = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(max : mx)
  for (int64_t t = 0; t < npairs; t++) {
    double v = dotq(n, Z + pi[t] * ldz, Z + pj[t] * ldz) - (pi[t] == pj[t] ? 1.0 : 0.0);
    v = fabs(v);
    if (v > mx) mx = v;
  }
  return mx;
}

/* full max |Z^T Z - I| over columns [0, k) */
double oracle_ortho_full(int64_t n, int64_t k, const double *Z, int64_t ldz) {
  double mx = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(max : mx)
  for (int64_t i = 0; i < k; i++)
    for (int64_t j = i; j < k; j++) {
      double v = fabs(dotq(n, Z + i * ldz, Z + j * ldz) - (i == j ? 1.0 : 0.0));
      if (v > mx) mx = v;
    }
  return mx;
}

/* cyclic Jacobi on the dense T in binary128 (brute force for n <= 64; a test */
/* tool independent of MRRR).  Eigenvalues ascending into w (as hi/lo pairs).  */
static void jacobi_q(int64_t n, qreal *A, double *w_hi, double *w_lo) {
  for (int sweep = 0; sweep < 100; sweep++) {
    qreal off = 0, dia = 0;
    for (int64_t p = 0; p < n; p++) {
      dia += A[p * n + p] * A[p * n + p];
      for (int64_t q = p + 1; q < n; q++) off += A[p * n + q] * A[p * n + q];
    }
    if (off <= 1e-70Q * dia || off == 0) break;
    for (int64_t p = 0; p < n; p++)
      for (int64_t q = p + 1; q < n; q++) {
        qreal apq = A[p * n + q];
        if (apq == 0) continue;
        qreal theta = (A[q * n + q] - A[p * n + p]) / (2 * apq);
        qreal t = (theta >= 0 ? 1 : -1) / (fabsq(theta) + sqrtq(theta * theta + 1));
        qreal c = 1 / sqrtq(t * t + 1), s = t * c;
        for (int64_t r = 0; r < n; r++) {
          qreal arp = A[r * n + p], arq = A[r * n + q];
          A[r * n + p] = c * arp - s * arq;
          A[r * n + q] = s * arp + c * arq;
        }
        for (int64_t r = 0; r < n; r++) {
          qreal apr = A[p * n + r], aqr = A[q * n + r];
          A[p * n + r] = c * apr - s * aqr;
          A[q * n + r] = s * apr + c * aqr;
        }
      }
  }
  qreal *ev = malloc(sizeof(qreal) * n);
  for (int64_t i = 0; i < n; i++) ev[i] = A[i * n + i];
  for (int64_t i = 1; i < n; i++) {
    qreal v = ev[i];
    int64_t j = i - 1;
    while (j >= 0 && ev[j] > v) { ev[j + 1] = ev[j]; j--; }
    ev[j + 1] = v;
  }
  for (int64_t i = 0; i < n; i++) { w_hi[i] = (double)ev[i]; w_lo[i] = (double)(ev[i] - (qreal)w_hi[i]); }
  free(ev);
}

void oracle_jacobi(int64_t n, const double *d, const double *e, double *w_hi, double *w_lo) {
  qreal *A = calloc((size_t)(n * n), sizeof(qreal));
  for (int64_t i = 0; i < n; i++) A[i * n + i] = d[i];
  for (int64_t i = 0; i < n - 1; i++) { A[i * n + i + 1] = e[i]; A[(i + 1) * n + i] = e[i]; }
  jacobi_q(n, A, w_hi, w_lo);
  free(A);
}

/* the same brute force on L D L^T (unit lower bidiagonal L = (1, l)) multiplied out in binary128 */
void oracle_jacobi_ldl(int64_t n, const double *d, const double *l, double *w_hi, double *w_lo) {
  qreal *A = calloc((size_t)(n * n), sizeof(qreal));
  for (int64_t i = 0; i < n; i++) {
    A[i * n + i] = (qreal)d[i] + ((i > 0) ? ((qreal)d[i - 1] * (qreal)l[i - 1]) * (qreal)l[i - 1] : 0);
    if (i < n - 1) { A[i * n + i + 1] = (qreal)d[i] * (qreal)l[i]; A[(i + 1) * n + i] = A[i * n + i + 1]; }
  }
  jacobi_q(n, A, w_hi, w_lo);
  free(A);
}

/* -------- unit-level wrappers for pins (y values exchanged as hi/lo pairs) -------- */
static void q_out(yreal v, double *hi, double *lo) { *hi = (double)v; *lo = (double)(v - (yreal)(*hi)); }

void oracle_dstqds(int64_t nb, const double *d, const double *l, double tau, double *dp_hi, double *dp_lo,
                   double *lp_hi, double *s_hi) {
  yreal *D = malloc(sizeof(yreal) * nb), *DL = malloc(sizeof(yreal) * nb), *DLL = malloc(sizeof(yreal) * nb);
  yreal *dp = malloc(sizeof(yreal) * nb), *lp = malloc(sizeof(yreal) * nb), *s = malloc(sizeof(yreal) * nb);
  for (int64_t i = 0; i < nb; i++) {
    D[i] = d[i];
    DL[i] = (i < nb - 1) ? (yreal)d[i] * (yreal)l[i] : 0;
    DLL[i] = (i < nb - 1) ? DL[i] * (yreal)l[i] : 0;
  }
  dstqds_q(nb, D, DL, DLL, (yreal)tau, dp, lp, s);
  for (int64_t i = 0; i < nb; i++) {
    double dummy;
    q_out(dp[i], &dp_hi[i], dp_lo ? &dp_lo[i] : &dummy);
    if (i < nb - 1 && lp_hi) lp_hi[i] = (double)lp[i];
    if (s_hi) s_hi[i] = (double)s[i];
  }
  free(D); free(DL); free(DLL); free(dp); free(lp); free(s);
}

void oracle_dqds(int64_t nb, const double *d, const double *l, double tau, double *om_hi, double *um_hi,
                 double *p_hi) {
  yreal *D = malloc(sizeof(yreal) * nb), *DL = malloc(sizeof(yreal) * nb), *DLL = malloc(sizeof(yreal) * nb);
  yreal *om = malloc(sizeof(yreal) * nb), *um = malloc(sizeof(yreal) * nb), *p = malloc(sizeof(yreal) * nb);
  for (int64_t i = 0; i < nb; i++) {
    D[i] = d[i];
    DL[i] = (i < nb - 1) ? (yreal)d[i] * (yreal)l[i] : 0;
    DLL[i] = (i < nb - 1) ? DL[i] * (yreal)l[i] : 0;
  }
  dqds_q(nb, D, DL, DLL, (yreal)tau, om, um, p);
  for (int64_t i = 0; i < nb; i++) {
    om_hi[i] = (double)om[i];
    if (i < nb - 1 && um_hi) um_hi[i] = (double)um[i];
    if (p_hi) p_hi[i] = (double)p[i];
  }
  free(D); free(DL); free(DLL); free(om); free(um); free(p);
}

/* Getvec on LDL^T given in fp64 (d, l), lambda given as hi+lo; r_io as in getvec_q. */
void oracle_getvec(int64_t nb, const double *d, const double *l, double lam_hi, double lam_lo, int64_t *r_io,
                   double *z_out, double *gamma_hi, double *zz_hi, int64_t *c_out) {
  rep_t *M = rep_alloc(nb);
  for (int64_t i = 0; i < nb; i++) { M->d[i] = d[i]; M->l[i] = (i < nb - 1) ? (yreal)l[i] : 0; }
  rep_derive(M);
  gv_ws w;
  gv_alloc(&w, nb);
  yreal g, zz;
  getvec_q(M, (yreal)lam_hi + (yreal)lam_lo, r_io, &w, &g, &zz, c_out);
  for (int64_t i = 0; i < nb; i++) z_out[i] = (double)w.z[i];
  *gamma_hi = (double)g;
  *zz_hi = (double)zz;
  gv_free(&w);
  rep_free(M);
}

/* the y-root built by S3 (for the "fl64(M_y) == M_x" pin) */
int oracle_root_y(int64_t n, const double *d, const double *e, int64_t s, int64_t nb, int left, uint64_t seed,
                  double *mu, double *dy_hi, double *dy_lo, double *ly_hi, double *ly_lo, double *dx, double *dllx) {
  double gl, gu;
  rep_t *r = make_root(n, s, nb, d, e, left, seed ? seed : DEFAULT_SEED, mu, &gl, &gu);
  if (!r) return -1;
  for (int64_t i = 0; i < nb; i++) {
    q_out(r->d[i], &dy_hi[i], &dy_lo[i]);
    q_out(r->l[i], &ly_hi[i], &ly_lo[i]);
    dx[i] = r->dx[i];
    dllx[i] = r->dllx[i];
  }
  rep_free(r);
  return 0;
}

int oracle_maxd(void) { return MAXD; }

/* -------- pins of the branches no full solve of the test matrices reaches (tests/test_oracle_branches.py) */
void oracle_stats_read(int64_t *out) { memcpy(out, g_stats, sizeof(g_stats)); }
void oracle_stats_reset(void) { memset(g_stats, 0, sizeof(g_stats)); }

static rep_t *rep_from_fp64(int64_t nb, const double *d, const double *l) {
  rep_t *M = rep_alloc(nb);
  for (int64_t i = 0; i < nb; i++) { M->d[i] = d[i]; M->l[i] = (i < nb - 1) ? (yreal)l[i] : 0; }
  rep_derive(M);
  M->sigma = 0;
  M->depth = 0;
  double sp = 0;
  for (int64_t i = 0; i < nb; i++) sp = dmax(sp, fabs(d[i]));
  M->spdiam = sp;
  return M;
}

/* bracket repair in x (on M_x = fl64 data) and in y; returns the number of widening steps */
int64_t oracle_bracket_x(int64_t nb, const double *dx, const double *dllx, int64_t j, double *lo, double *hi) {
  int64_t before = g_stats[ST_BRACKET_FIX];
  bracket_x(nb, dx, dllx, j, lo, hi);
  return g_stats[ST_BRACKET_FIX] - before;
}
int64_t oracle_bracket_y(int64_t nb, const double *d, const double *l, int64_t j, double *lo, double *hi) {
  rep_t *M = rep_from_fp64(nb, d, l);
  int64_t before = g_stats[ST_BRACKET_FIX];
  bracket_y(nb, M->d, M->dll, j, lo, hi);
  rep_free(M);
  return g_stats[ST_BRACKET_FIX] - before;
}

/* y-bisection to full accuracy of eigenvalue j (1-based) of L D L^T from [lo, hi] */
void oracle_bisect_y_full(int64_t nb, const double *d, const double *l, int64_t j, double lo, double hi,
                          double *lam_hi, double *lam_lo) {
  rep_t *M = rep_from_fp64(nb, d, l);
  q_out(bisect_y_full(M, j, (yreal)lo, (yreal)hi), lam_hi, lam_lo);
  rep_free(M);
}

/* the singleton RQI of S9 on L D L^T (sigma = 0) from the x-interval [lo, hi] with gap; *fallbacks = 1 when */
/* the RQI ended in the bisection fallback of P:3481-3482                                                    */
void oracle_rqi(int64_t nb, const double *d, const double *l, int64_t j, double lo, double hi, double gap,
                int32_t support, double *W, double *z, int64_t *iters, int64_t *fallbacks) {
  rep_t *M = rep_from_fp64(nb, d, l);
  gv_ws w;
  gv_alloc(&w, nb);
  int64_t i0 = g_stats[ST_RQI_ITERS], f0 = g_stats[ST_RQI_FALLBACK];
  rqi_singleton(M, j, lo, hi, gap, support, W, z, &w);
  *iters = g_stats[ST_RQI_ITERS] - i0;
  *fallbacks = g_stats[ST_RQI_FALLBACK] - f0;
  gv_free(&w);
  rep_free(M);
}
