// kernels_sd.cuh -- the single/double realisation of the mixed-precision MRRR:
// binary32 input and output, every computation in binary64, gaptol fixed to 1e-5.  The x-path
// kernels (split, root chain, NegCount bisection, classification) are shared with the double/double-double
// solver; the y-representation is binary64 (the dd rows carry zero low words) and these kernels hold the
// steps whose arithmetic changes:
//
//   k_f2d / k_w_d2f / k_z_d2f   "data conversion is only necessary when reading the input and writing the
//                               output": binary32 <-> binary64 at the boundary.
//   k_sd_attempt                S8(c) shift attempts: Alg. dstqds P:3324-3351 in binary64, growth max|d+| and
//                               validity, in the operation order of the reference loop (the child data decide
//                               integer outputs, so they must be bit-identical to the oracle's binary64 run).
//   k_sd_build                  S8(d) child representation (d+, l+) and its derived rows dl = d l, dll = dl l
//                               (P:4145-4147), sigma accumulated in binary64.
//
// The singleton RQI runs the segmented passes of kernels_rqi3.cuh with their binary64 step (seg_pass_sd).
#pragma once
#include "kernels_vec.cuh"

__global__ void k_f2d(const float *__restrict__ x, double *y, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = (double)x[i];
}
__global__ void k_w_d2f(const double *__restrict__ x, float *y, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __double2float_rn(x[i]);
}
// Z (binary64, leading dimension n) -> binary32 with leading dimension ldz; blockIdx.y = column
__global__ void k_z_d2f(const double *__restrict__ Zd, float *Z, long long n, long long ldz) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long c = blockIdx.y;
  if (i < n) Z[c * ldz + i] = __double2float_rn(Zd[c * n + i]);
}

// IEEE binary64 quotient (the fast sequence where its range test passes, __ddiv_rn otherwise), with the
// infinity guard of Alg. dstqds: q := 1 when s and d+ are both infinite
__device__ __forceinline__ double sd_quot(double s, double b) {
  const double q = div_fast_nocheck(s, b);
  return div_range_ok(s, b, q) ? q : __ddiv_rn(s, b);
}

// one row of Alg. dstqds in binary64, in the reference order: d+ = s + d, q = s / d+, l+ = dl / d+,
// s' = q dll - tau
__device__ __forceinline__ void sd_dstqds_row(double &s, double d, double dl, double dll, double tau, double &dp,
                                              double &lp) {
  dp = __dadd_rn(s, d);
  const double q = (isinf(s) && isinf(dp)) ? 1.0 : sd_quot(s, dp);
  lp = sd_quot(dl, dp);
  s = __dsub_rn(__dmul_rn(q, dll), tau);
}

// S8(c): attempts a0 .. a0+na-1 of every open cluster, thread per (cluster, attempt, side); growth g = max |d+|
// and validity (no NaN among d+, l+) as the oracle's do_cluster forms them; k_clu_select_multi replays the
// sequential acceptance
__global__ void k_sd_attempt(const Cluster *__restrict__ cl, int ncl, const RepDesc *__restrict__ reps,
                             const YElt *__restrict__ my, const ShiftState *__restrict__ ss, int a0, int na,
                             double *gval, int *valid) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2LL * na * ncl) return;
  const int c = (int)(t / (2 * na)), ia = (int)((t >> 1) % na), side = (int)(t & 1);
  const ShiftState S = ss[c];
  if (S.done) return;
  double tau = side ? S.taur : S.taul;
  for (int b = a0; b < a0 + ia; b++) tau = side ? __dadd_rn(tau, ldexp(S.offr, b)) : __dsub_rn(tau, ldexp(S.offl, b));
  const RepDesc R = reps[cl[c].rep];
  const YElt *y = my + R.off;
  double s = -tau, g = 0.0;
  int v = 1;
  for (int i = 0; i < R.nb - 1; i++) {
    double dp, lp;
    sd_dstqds_row(s, __ldg(&y[i].d_hi), __ldg(&y[i].dl_hi), __ldg(&y[i].dll_hi), tau, dp, lp);
    v &= !(isnan(dp) || isnan(lp));
    g = dmaxd(g, fabs(dp));
  }
  const double dn = __dadd_rn(s, __ldg(&y[R.nb - 1].d_hi));
  v &= !isnan(dn);
  gval[t] = dmaxd(g, fabs(dn));
  valid[t] = v;
}

// S8(d): child representation of cluster c (rep id repbase + c, rows at poolbase + c * nbmax): d = d+,
// l = l+ of dstqds(M, tau_best); rows dl = d l, dll = dl l, M_x = (d, dll) (the oracle's rep_derive with
// y = binary64, where fl64(M_y) = M_y); sigma = fl64(sigma_parent + tau).  No valid shift: nb = -1 (the
// members go back to the parent as singletons, as in the double/dd path).
__global__ void k_sd_build(const Cluster *__restrict__ cl, int ncl, RepDesc *reps, const ShiftState *__restrict__ ss,
                           double2 *mx, YElt *my, int repbase, long long poolbase, int nbmax) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
  const ShiftState S = ss[c];
  const RepDesc P = reps[cl[c].rep];
  RepDesc R = P;
  R.off = poolbase + (long long)c * nbmax;
  R.depth = P.depth + 1;
  R.sig_hi = __dadd_rn(P.sig_hi, S.best_tau);
  R.sig_lo = 0.0;
  if (!S.have_best) R.nb = -1;
  reps[repbase + c] = R;
  if (!S.have_best) return;
  const YElt *y = my + P.off;
  YElt *yc = my + R.off;
  double2 *xc = mx + R.off;
  const double tau = S.best_tau;
  double s = -tau;
  for (int i = 0; i < P.nb - 1; i++) {
    double dp, lp;
    sd_dstqds_row(s, __ldg(&y[i].d_hi), __ldg(&y[i].dl_hi), __ldg(&y[i].dll_hi), tau, dp, lp);
    const double dl = __dmul_rn(dp, lp), dll = __dmul_rn(dl, lp);
    YElt e;
    e.d_hi = dp; e.d_lo = 0.0; e.dl_hi = dl; e.dl_lo = 0.0; e.dll_hi = dll; e.dll_lo = 0.0;
    yc[i] = e;
    xc[i] = make_double2(dp, dll);
  }
  const double dn = __dadd_rn(s, __ldg(&y[P.nb - 1].d_hi));
  YElt e;
  e.d_hi = dn; e.d_lo = 0.0; e.dl_hi = e.dl_lo = e.dll_hi = e.dll_lo = 0.0;
  yc[P.nb - 1] = e;
  xc[P.nb - 1] = make_double2(dn, 0.0);
}
