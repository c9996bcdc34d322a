// kernels_vec.cuh -- cluster path (S8: Alg. spectrumshift, mixed
// precision P:5969-5971, depth-first P:6110-6132) and the singleton RQI /
// eigenvector kernel (S9-S10: Alg. Getvec, Alg. stask
// P:4026-4074, mixed stop P:6074-6108, convert-on-write P:6156-6158).
#pragma once
#include "kernels.cuh"

__device__ __forceinline__ dd ld_d(const YElt *y) { return dd_make(__ldg(&y->d_hi), __ldg(&y->d_lo)); }
__device__ __forceinline__ dd ld_dl(const YElt *y) { return dd_make(__ldg(&y->dl_hi), __ldg(&y->dl_lo)); }
__device__ __forceinline__ dd ld_dll(const YElt *y) { return dd_make(__ldg(&y->dll_hi), __ldg(&y->dll_lo)); }

// RQI form of a representation (derived once per representation, y-arithmetic): with
//   g(i) = d(i+1) + dll(i),  c2(i) = dl(i)^2 = d(i) dll(i),
// the stationary and progressive transforms become one recurrence on the pivots,
//   dstqds:  d+(i+1)  = (g(i)   - lam) - c2(i) / d+(i),      d+(0)     = d(0) - lam
//   dqds  :  omega(i) = (g(i-1) - lam) - c2(i) / omega(i+1), omega(n-1) = g(n-2) - lam, g(-1) = d(0)
// (Alg. dstqds: s(i+1) = s(i) dll(i) / d+(i) - lam = dll(i) - c2(i)/d+(i) - lam; Alg. dqds
// P:3366-3393 with A-1: p(i) = p(i+1) d(i) / omega(i+1) - lam = d(i) - c2(i)/omega(i+1) - lam).  The
// dependent chain per step is one dd division and one dd subtraction; l+(i) = dl(i)/d+(i),
// u-(i) = dl(i)/omega(i+1) and the twist quantity gamma_k = s(k) + t(k) = d+(k) - c2(k)/omega(k+1)
// come off the chain.  Element i holds c2(i), dl(i), gf = g(i), gb = g(i-1).
// (struct QElt is defined in kernels.cuh)

__global__ void k_build_q(const RepDesc *__restrict__ reps, const int *__restrict__ rlist, int r0, int nr,
                          const YElt *__restrict__ my, QElt *mq) {
  const int rid = rlist ? rlist[blockIdx.x] : r0 + (int)blockIdx.x;
  if ((int)blockIdx.x >= nr) return;
  const RepDesc R = reps[rid];
  if (R.nb < 2) return;
  const YElt *y = my + R.off;
  QElt *q = mq + R.off;
  // blockIdx.y splits the rows (a representation's rows are independent here)
  // 16-byte loads and stores (YElt = 3 double2, QElt = 4 double2; both 16-byte aligned)
  const double2 *y2 = reinterpret_cast<const double2 *>(y);
  double2 *q2 = reinterpret_cast<double2 *>(q);
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < R.nb; i += blockDim.x * gridDim.y) {
    const double2 vd = __ldg(y2 + 3LL * i), vdl = __ldg(y2 + 3LL * i + 1), vdll = __ldg(y2 + 3LL * i + 2);
    dd d = dd_make(vd.x, vd.y), dl = dd_make(vdl.x, vdl.y), dll = dd_make(vdll.x, vdll.y);
    dd c2 = dd_mul(dl, dl);
    dd gf = dd_from(0.0), gb = d;
    if (i < R.nb - 1) {
      const double2 vn = __ldg(y2 + 3LL * (i + 1));
      gf = dd_add(dd_make(vn.x, vn.y), dll);
    }
    if (i > 0) {
      const double2 vp = __ldg(y2 + 3LL * (i - 1) + 2);
      gb = dd_add(d, dd_make(vp.x, vp.y));
    }
    q2[4LL * i] = make_double2(c2.hi, c2.lo);
    q2[4LL * i + 1] = make_double2(dl.hi, dl.lo);
    q2[4LL * i + 2] = make_double2(gf.hi, gf.lo);
    q2[4LL * i + 3] = make_double2(gb.hi, gb.lo);
  }
}

// one qd step shared by dstqds (Alg. dstqds) and dqds (Alg. dqds, A-1/A-2):
//   den = x + a; q = (|x| = inf and |den| = inf) ? 1 : x / den; out = b / den; xn = q * c - lam
// dstqds: x = s(i), a = d(i), b = dl(i), c = dll(i)  -> den = d+(i), out = l+(i), xn = s(i+1)
// dqds  : x = p(i+1), a = dll(i), b = dl(i), c = d(i) -> den = omega(i+1), out = u-(i), xn = p(i)
// The two quotients by den share one dd reciprocal (tolerance-level difference to x/den).
__device__ __forceinline__ void qd_step(dd x, dd a, dd b, dd c, dd lam, dd &den, dd &rr, dd &out, dd &xn) {
  den = dd_add(x, a);
  rr = dd_rcp(den);
  dd q = (dd_isinf(x) && dd_isinf(den)) ? dd_from(1.0) : dd_mul(x, rr);
  out = dd_mul(b, rr);
  xn = dd_sub(dd_mul(q, c), lam);
}

// ---------------------------------------------------------------------------
// S8(a): y-refinement nodes for the two cluster ends
// ---------------------------------------------------------------------------
__global__ void k_clu_yref_init(const Cluster *__restrict__ cl, int ncl, const RepDesc *__restrict__ reps,
                                const double *__restrict__ ilo, const double *__restrict__ ihi, BNode *bn) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
  Cluster C = cl[c];
  // start: the end's x-interval itself (A-12''); the y bracket verification repairs it on a failing side
  for (int side = 0; side < 2; side++) {
    int j = side ? C.q : C.p;
    double L = ilo[C.ibase + j], H = ihi[C.ibase + j];
    dyadic_widen(L, H, &L, &H);
    BNode b;
    b.lo = L; b.hi = H; b.clo = 0; b.chi = 0; b.j = j; b.rep = C.rep;
    b.needLo = 1; b.needHi = 1; b.fixes = 0; b.j2 = j;
    b.obase = 2LL * c + side - j;
    bn[2 * c + side] = b;
  }
}

// per-cluster shift state
struct ShiftState {
  double taul, taur, offl, offr, best_g, best_tau;
  int have_best, done, certified, attempts;
};

__global__ void k_clu_shift_init(int ncl, const double *__restrict__ ylo, const double *__restrict__ yhi,
                                 ShiftState *ss) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
  double Lp = ylo[2 * c], Hq = yhi[2 * c + 1];
  ShiftState s;
  s.offl = __dmul_rn(__dmul_rn(100.0, EPS_X), fabs(Lp));
  s.offr = __dmul_rn(__dmul_rn(100.0, EPS_X), fabs(Hq));
  s.taul = __dsub_rn(Lp, s.offl);
  s.taur = __dadd_rn(Hq, s.offr);
  s.best_g = INFINITY; s.best_tau = 0.0;
  s.have_best = 0; s.done = 0; s.certified = 0; s.attempts = 0;
  ss[c] = s;
}

// growth max|fl64(d+)| and validity (no NaN) of dstqds(M_y, tau) (Alg. dstqds): fast pass on the
// pivot-recurrence form (QElt), the careful IEEE pass (qd_step) if a pivot leaves [2^-1000, 2^1000]
__device__ void dstqds_growth(const YElt *__restrict__ y, const QElt *__restrict__ q, int nb, double tau_x, double &g,
                              int &valid) {
  const dd tau = dd_from(tau_x);
  {
    dd den = dd_sub(dd_make(__ldg(&q[0].gb_hi), __ldg(&q[0].gb_lo)), tau);
    double gm = 0.0;
    bool ok = true;
    for (int i = 0; i < nb - 1; i++) {
      const double b = den.hi;
      ok &= (fabs(b) > 0x1p-1000) && (fabs(b) < 0x1p1000);
      gm = dmaxd(gm, fabs(b));
      const double r = rcp_seed(b);
      double ee = __fma_rn(-b, r, 1.0);
      ee = __fma_rn(ee, ee, ee);
      const double r1 = __fma_rn(r, ee, r);
      const double e2 = __fma_rn(-b, r1, 1.0);
      const double r2 = __fma_rn(r1, e2, r1);
      const dd c2 = dd_make(__ldg(&q[i].c2_hi), __ldg(&q[i].c2_lo));
      const double h = __dmul_rn(c2.hi, r1);
      double t = __fma_rn(-h, b, c2.hi);
      t = __dadd_rn(t, c2.lo);
      t = __fma_rn(-h, den.lo, t);
      const dd P = dd_make(h, __dmul_rn(t, r2));
      den = dd_sub_nf(dd_sub_nf(dd_make(__ldg(&q[i].gf_hi), __ldg(&q[i].gf_lo)), tau), P);
    }
    ok &= isfinite(den.hi) && isfinite(den.lo);
    if (ok) {
      g = dmaxd(gm, fabs(den.hi));
      valid = 1;
      return;
    }
  }
  dd s = dd_neg(tau);
  double gm = 0.0;
  int okv = 1;
  for (int i = 0; i < nb - 1; i++) {
    dd den, rr, out, xn;
    qd_step(s, ld_d(y + i), ld_dl(y + i), ld_dll(y + i), tau, den, rr, out, xn);
    okv &= !(isnan(den.hi) || isnan(out.hi));
    gm = dmaxd(gm, fabs(den.hi));
    s = xn;
  }
  dd den = dd_add(s, ld_d(y + nb - 1));
  okv &= !isnan(den.hi);
  g = dmaxd(gm, fabs(den.hi));
  valid = okv;
}

// S8(c) attempts a0 .. a0+na-1 of every open cluster at once (the shift sequence of Alg. spectrumshift is
// fixed in advance: tau_l(a+1) = tau_l(a) - 2^a off_l, tau_r(a+1) = tau_r(a) + 2^a off_r), thread per
// (cluster, attempt, side); k_clu_select_multi then replays the sequential acceptance
__global__ void k_clu_attempt_multi(const Cluster *__restrict__ cl, int ncl, const RepDesc *__restrict__ reps,
                                    const YElt *__restrict__ my, const QElt *__restrict__ mq,
                                    const ShiftState *__restrict__ ss, int a0, int na, double *gval, int *valid) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2LL * na * ncl) return;
  const int c = (int)(t / (2 * na)), ia = (int)((t >> 1) % na), side = (int)(t & 1);
  const ShiftState S = ss[c];
  if (S.done) return;
  double tau = side ? S.taur : S.taul;
  for (int b = a0; b < a0 + ia; b++) tau = side ? __dadd_rn(tau, ldexp(S.offr, b)) : __dsub_rn(tau, ldexp(S.offl, b));
  const RepDesc R = reps[cl[c].rep];
  double g;
  int v;
  dstqds_growth(my + R.off, mq + R.off, R.nb, tau, g, v);
  gval[t] = g;
  valid[t] = v;
}

__global__ void k_clu_select_multi(const Cluster *__restrict__ cl, int ncl, const RepDesc *__restrict__ reps,
                                   ShiftState *ss, const double *__restrict__ gval, const int *__restrict__ valid,
                                   int a0, int na, int *ndone, long long *stats, double kelg) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
  ShiftState s = ss[c];
  if (s.done) { atomicAdd(ndone, 1); return; }
  // mixed-precision growth bound eq:newkelgbound P:6052-6056 (A-35): max(G, eps_x / (eps_y sqrt(n))) spdiam,
  // kelg = eps_x / eps_y (2^51 double/dd, 2^29 single/double)
  const RepDesc Rg = reps[cl[c].rep];
  const double gthr = __dmul_rn(dmaxd(GROWTH, __ddiv_rn(kelg, sqrt((double)Rg.nb))), Rg.spdiam);
  for (int a = a0; a < a0 + na && !s.done; a++) {
    atomicAdd((unsigned long long *)&stats[ST_ATTEMPTS], 1ull);
    const long long o = ((long long)c * na + (a - a0)) * 2;
    int vl = valid[o], vr = valid[o + 1];
    double gl = gval[o], gr = gval[o + 1];
    int pick = 0;
    if (vl && vr) pick = (gl <= gr) ? 1 : 2;
    else if (vl) pick = 1;
    else if (vr) pick = 2;
    s.attempts++;
    if (pick) {
      double g = (pick == 1) ? gl : gr;
      if (g < s.best_g) { s.best_g = g; s.best_tau = (pick == 1) ? s.taul : s.taur; s.have_best = 1; }
      if (g <= gthr) { s.done = 1; s.certified = 1; }
    }
    if (!s.done) {
      s.taul = __dsub_rn(s.taul, ldexp(s.offl, a));
      s.taur = __dadd_rn(s.taur, ldexp(s.offr, a));
      if (a == MAX_ATTEMPTS - 1) {
        s.done = 1;
        if (s.have_best) atomicAdd((unsigned long long *)&stats[ST_UNCERTIFIED], 1ull);
      }
    }
  }
  if (s.done) atomicAdd(ndone, 1);
  ss[c] = s;
}

// S8(d): child representation M_y = (d+, l+) of dstqds(M_y, tau_best) and its x copy.
// Child rep id = repbase + c, data at pool offset poolbase + c * nbmax.
// one row of the fast child build: l+(i) = dl(i)/d+(i) and c2(i)/d+(i) from the reciprocal pair of d+(i),
// the child's y-row (d, dl, dll) and x-row (d, dll); returns d+(i+1) (the y_step recurrence)
// the row's parent data (c2, dl, gf of q[i]) as three 16-byte values: callers that run a chain of rows load them
// a few rows ahead (the chain's dependent steps otherwise wait on each row's load: stall_long_sb 38 % on C3)
struct QRow { double2 c2, dl, gf; };
__device__ __forceinline__ QRow ld_qrow(const QElt *__restrict__ q, int i) {
  const double2 *p = reinterpret_cast<const double2 *>(q + i);
  QRow r;
  r.c2 = __ldg(p);
  r.dl = __ldg(p + 1);
  r.gf = __ldg(p + 2);
  return r;
}
__device__ __forceinline__ dd clu_build_row_v(dd den, const QRow &qr, int i, dd tau, YElt *yc, double2 *xc, bool &ok,
                                              bool staged) {
  const double b = den.hi;
  ok &= (fabs(b) > 0x1p-1000) && (fabs(b) < 0x1p1000);
  const double r = rcp_seed(b);
  double ee = __fma_rn(-b, r, 1.0);
  ee = __fma_rn(ee, ee, ee);
  const double r1 = __fma_rn(r, ee, r);
  const double e2 = __fma_rn(-b, r1, 1.0);
  const double r2 = __fma_rn(r1, e2, r1);
  const dd dlp = dd_make(qr.dl.x, qr.dl.y);
  const dd c2 = dd_make(qr.c2.x, qr.c2.y);
  double h = __dmul_rn(dlp.hi, r1), t = __fma_rn(-h, b, dlp.hi);
  t = __fma_rn(-h, den.lo, __dadd_rn(t, dlp.lo));
  const dd out = fast_two_sum(h, __dmul_rn(t, r2));  // l+(i) = dl(i) / d+(i)
  h = __dmul_rn(c2.hi, r1);
  t = __fma_rn(-h, b, c2.hi);
  t = __fma_rn(-h, den.lo, __dadd_rn(t, c2.lo));
  const dd Pq = dd_make(h, __dmul_rn(t, r2));        // c2(i) / d+(i)
  if (yc) {
    const dd dl = dd_mul(den, out);
    const dd dll = dd_mul(dl, out);
    YElt e;
    e.d_hi = den.hi; e.d_lo = den.lo; e.dl_hi = dl.hi; e.dl_lo = dl.lo; e.dll_hi = dll.hi; e.dll_lo = dll.lo;
    const double dx = den.hi, lx = out.hi;
    const double2 xe = make_double2(dx, __dmul_rn(__dmul_rn(dx, lx), lx));
    if (staged) { *yc = e; *xc = xe; }  // shared-memory staging slot of row i
    else { yc[i] = e; xc[i] = xe; }
  }
  return dd_sub_nf(dd_sub_nf(dd_make(qr.gf.x, qr.gf.y), tau), Pq);
}
__device__ __forceinline__ dd clu_build_row(dd den, const QElt *__restrict__ q, int i, dd tau, YElt *yc, double2 *xc,
                                            bool &ok, bool staged = false) {
  const double b = den.hi;
  ok &= (fabs(b) > 0x1p-1000) && (fabs(b) < 0x1p1000);
  const double r = rcp_seed(b);
  double ee = __fma_rn(-b, r, 1.0);
  ee = __fma_rn(ee, ee, ee);
  const double r1 = __fma_rn(r, ee, r);
  const double e2 = __fma_rn(-b, r1, 1.0);
  const double r2 = __fma_rn(r1, e2, r1);
  const dd dlp = dd_make(__ldg(&q[i].dl_hi), __ldg(&q[i].dl_lo));
  const dd c2 = dd_make(__ldg(&q[i].c2_hi), __ldg(&q[i].c2_lo));
  double h = __dmul_rn(dlp.hi, r1), t = __fma_rn(-h, b, dlp.hi);
  t = __fma_rn(-h, den.lo, __dadd_rn(t, dlp.lo));
  const dd out = fast_two_sum(h, __dmul_rn(t, r2));  // l+(i) = dl(i) / d+(i)
  h = __dmul_rn(c2.hi, r1);
  t = __fma_rn(-h, b, c2.hi);
  t = __fma_rn(-h, den.lo, __dadd_rn(t, c2.lo));
  const dd Pq = dd_make(h, __dmul_rn(t, r2));        // c2(i) / d+(i)
  if (yc) {
    const dd dl = dd_mul(den, out);
    const dd dll = dd_mul(dl, out);
    YElt e;
    e.d_hi = den.hi; e.d_lo = den.lo; e.dl_hi = dl.hi; e.dl_lo = dl.lo; e.dll_hi = dll.hi; e.dll_lo = dll.lo;
    const double dx = den.hi, lx = out.hi;
    const double2 xe = make_double2(dx, __dmul_rn(__dmul_rn(dx, lx), lx));
    if (staged) { *yc = e; *xc = xe; }  // shared-memory staging slot of row i
    else { yc[i] = e; xc[i] = xe; }
  }
  return dd_sub_nf(dd_sub_nf(dd_make(__ldg(&q[i].gf_hi), __ldg(&q[i].gf_lo)), tau), Pq);
}
__device__ void clu_build_one(int c, const Cluster *__restrict__ cl, RepDesc *reps, const ShiftState *__restrict__ ss,
                              double2 *mx, YElt *my, const QElt *__restrict__ mq, int repbase, long long poolbase,
                              int nbmax);
__global__ void k_clu_build(const Cluster *__restrict__ cl, int ncl, RepDesc *reps, const ShiftState *__restrict__ ss,
                            double2 *mx, YElt *my, const QElt *__restrict__ mq, int repbase, long long poolbase,
                            int nbmax) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
  clu_build_one(c, cl, reps, ss, mx, my, mq, repbase, poolbase, nbmax);
}
__device__ void clu_build_one(int c, const Cluster *__restrict__ cl, RepDesc *reps, const ShiftState *__restrict__ ss,
                              double2 *mx, YElt *my, const QElt *__restrict__ mq, int repbase, long long poolbase,
                              int nbmax) {
  ShiftState S = ss[c];
  RepDesc P = reps[cl[c].rep];
  RepDesc R = P;
  R.off = poolbase + (long long)c * nbmax;
  R.depth = P.depth + 1;
  dd sig = dd_add_d(dd_make(P.sig_hi, P.sig_lo), S.best_tau);
  R.sig_hi = sig.hi; R.sig_lo = sig.lo;
  if (!S.have_best) R.nb = -1;  // failed: members go back to the parent as singletons
  reps[repbase + c] = R;
  if (!S.have_best) return;
  const YElt *y = my + P.off;
  YElt *yc = my + R.off;
  double2 *xc = mx + R.off;
  dd tau = dd_from(S.best_tau);
  if (mq) {  // fast pass on the pivot-recurrence form; the careful pass below if a pivot leaves the range
    const QElt *q = mq + P.off;
    dd den = dd_sub(dd_make(__ldg(&q[0].gb_hi), __ldg(&q[0].gb_lo)), tau);
    bool ok = true;
    for (int i = 0; i < P.nb - 1; i++) den = clu_build_row(den, q, i, tau, yc, xc, ok);
    ok &= isfinite(den.hi) && isfinite(den.lo);
    if (ok) {
      YElt e;
      e.d_hi = den.hi; e.d_lo = den.lo; e.dl_hi = e.dl_lo = e.dll_hi = e.dll_lo = 0.0;
      yc[P.nb - 1] = e;
      xc[P.nb - 1] = make_double2(den.hi, 0.0);
      return;
    }
  }
  dd s = dd_neg(tau);
  for (int i = 0; i < P.nb - 1; i++) {
    dd den, rr, out, xn;
    qd_step(s, ld_d(y + i), ld_dl(y + i), ld_dll(y + i), tau, den, rr, out, xn);
    // rep_derive: dl = d l, dll = dl l (y); dx = fl64(d), dllx = (dx lx) lx
    dd dl = dd_mul(den, out);
    dd dll = dd_mul(dl, out);
    YElt e;
    e.d_hi = den.hi; e.d_lo = den.lo; e.dl_hi = dl.hi; e.dl_lo = dl.lo; e.dll_hi = dll.hi; e.dll_lo = dll.lo;
    yc[i] = e;
    double dx = den.hi, lx = out.hi;
    xc[i] = make_double2(dx, __dmul_rn(__dmul_rn(dx, lx), lx));
    s = xn;
  }
  dd den = dd_add(s, ld_d(y + P.nb - 1));
  YElt e;
  e.d_hi = den.hi; e.d_lo = den.lo; e.dl_hi = e.dl_lo = e.dll_hi = e.dll_lo = 0.0;
  yc[P.nb - 1] = e;
  xc[P.nb - 1] = make_double2(den.hi, 0.0);
}

// S8(e): child start intervals (A-13) for members; neighbours shifted by -tau.
// segment of cluster c: cseg[c] .. cseg[c] + (q-p+2): index j -> cseg[c] + (j - p + 1)
__global__ void k_clu_child_starts(const Cluster *__restrict__ cl, int ncl, const RepDesc *__restrict__ reps,
                                   const ShiftState *__restrict__ ss, const long long *__restrict__ cseg,
                                   const long long *__restrict__ bnoff, const double *__restrict__ ilo,
                                   const double *__restrict__ ihi, double *clo, double *chi, BNode *bn, int repbase,
                                   const double *__restrict__ ylo, const double *__restrict__ yhi, double eps_y) {
  // member j's start: (lambda(1 +- nu_in) - tau)(1 +- nu) (A-13); the cluster ends p, q start from
  // their y-refined intervals (they bracket M_y's own eigenvalues), so their inner inflation only covers the
  // y-arithmetic shift: nu_in = 100 n eps_y (A-13'); the other members from their x-intervals with nu_in = nu
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
  Cluster C = cl[c];
  ShiftState S = ss[c];
  if (!S.have_best) return;
  int nb = reps[C.rep].nb;
  double nu = __dmul_rn(__dmul_rn(100.0, (double)nb), EPS_X);
  const double nuy = __dmul_rn(__dmul_rn(100.0, (double)nb), eps_y);
  double tau = S.best_tau;
  long long base = cseg[c] - (C.p - 1);  // child ibase
  const double lpm = (C.p > 1) ? ilo[C.ibase + C.p - 1] : NAN;  // (p = 1 has no left neighbour: no read before ilo)
  if (C.p > 1 && !isnan(lpm)) {
    clo[base + C.p - 1] = __dsub_rn(lpm, tau);
    chi[base + C.p - 1] = __dsub_rn(ihi[C.ibase + C.p - 1], tau);
  } else {
    clo[base + C.p - 1] = NAN; chi[base + C.p - 1] = NAN;
  }
  double lqp = (C.q < nb) ? ilo[C.ibase + C.q + 1] : NAN;
  if (C.q < nb && !isnan(lqp)) {
    clo[base + C.q + 1] = __dsub_rn(lqp, tau);
    chi[base + C.q + 1] = __dsub_rn(ihi[C.ibase + C.q + 1], tau);
  } else {
    clo[base + C.q + 1] = NAN; chi[base + C.q + 1] = NAN;
  }
  long long o = bnoff[c];
  for (int j = C.p; j <= C.q; j++) {
    const bool end = (j == C.p || j == C.q);
    const double nin = end ? nuy : nu;
    double lo = (j == C.p) ? ylo[2 * c] : (j == C.q) ? ylo[2 * c + 1] : ilo[C.ibase + j];
    double hi = (j == C.p) ? yhi[2 * c] : (j == C.q) ? yhi[2 * c + 1] : ihi[C.ibase + j];
    double a1 = __dsub_rn(lo, __dmul_rn(nin, fabs(lo)));
    double b1 = __dsub_rn(a1, tau);
    double l2 = __dsub_rn(b1, __dmul_rn(nu, fabs(b1)));
    double c1 = __dadd_rn(hi, __dmul_rn(nin, fabs(hi)));
    double e1 = __dsub_rn(c1, tau);
    double h2 = __dadd_rn(e1, __dmul_rn(nu, fabs(e1)));
    double L, H;
    dyadic_widen(l2, h2, &L, &H);
    BNode b;
    b.lo = L; b.hi = H; b.clo = 0; b.chi = 0; b.j = j; b.rep = repbase + c;
    b.needLo = 1; b.needHi = 1; b.fixes = 0; b.j2 = j;
    b.obase = base;
    bn[o + (j - C.p)] = b;
  }
}

// S8(f): reclassify the members in the child; singletons -> RQI list, clusters -> next level.
// Failed clusters (no valid shift) send their members to the RQI list on the parent rep.
__global__ void k_clu_classify(const Cluster *__restrict__ cl, int ncl, const RepDesc *__restrict__ reps,
                               const ShiftState *__restrict__ ss, const long long *__restrict__ cseg,
                               const double *__restrict__ ilo, const double *__restrict__ ihi,
                               const double *__restrict__ clo, const double *__restrict__ chi,
                               const int *__restrict__ colmap, double gaptol, int repbase, Singleton *sing, int *nsing,
                               Cluster *nxt, int *nnxt, int *grp_first, int *grp_last, int kout, long long *stats) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
  Cluster C = cl[c];
  ShiftState S = ss[c];
  const RepDesc P = reps[C.rep];
  int bstart = P.bstart, nb = P.nb;
  bool failed = !S.have_best;
  if (failed) atomicAdd((unsigned long long *)&stats[ST_FAILED], 1ull);
  const double *lo = failed ? ilo : clo;
  const double *hi = failed ? ihi : chi;
  long long base = failed ? C.ibase : (cseg[c] - (C.p - 1));
  int rep = failed ? C.rep : repbase + c;
  int depth = failed ? P.depth : P.depth + 1;
  bool all_single = failed || depth >= MAXD;
  if (!failed && depth >= MAXD) atomicAdd((unsigned long long *)&stats[ST_FAILED], 1ull);
  int g0 = C.p;
  for (int j = C.p + 1; j <= C.q + 1; j++) {
    bool brk = (j == C.q + 1) || all_single ||
               is_boundary(lo[base + j - 1], hi[base + j - 1], lo[base + j], hi[base + j], gaptol);
    if (!brk) continue;
    int g1 = j - 1;
    bool sel = false;
    for (int t = g0; t <= g1; t++) sel |= (colmap[bstart + t - 1] >= 0);
    if (sel) {
      if (grp_first && !failed && depth < MAXD) {
        for (int t = g0; t <= g1; t++) {
          int col = colmap[bstart + t - 1];
          if (col >= 0) {
            grp_first[(long long)depth * kout + col] = bstart + g0 - 1;
            grp_last[(long long)depth * kout + col] = bstart + g1 - 1;
          }
        }
      }
      if (g0 == g1 || all_single) {
        for (int t = g0; t <= g1; t++) {
          int col = colmap[bstart + t - 1];
          if (col < 0) continue;
          double mid = bis_mid(lo[base + t], hi[base + t]);
          double ln = lo[base + t - 1], hn = hi[base + t - 1];
          double lr = lo[base + t + 1];
          double gl = (t > 1 && !isnan(ln)) ? __dsub_rn(mid, hn) : INFINITY;
          double gr = (t < nb && !isnan(lr)) ? __dsub_rn(lr, mid) : INFINITY;
          int k = atomicAdd(nsing, 1);
          Singleton s;
          s.lo = lo[base + t]; s.hi = hi[base + t]; s.gap = dmind(gl, gr);
          s.rep = rep; s.j = t; s.col = col; s.pad = 0;
          sing[k] = s;
        }
      } else {
        int k = atomicAdd(nnxt, 1);
        Cluster D;
        D.ibase = base; D.rep = rep; D.p = g0; D.q = g1; D.depth = depth;
        nxt[k] = D;
        atomicAdd((unsigned long long *)&stats[ST_NCLUSTERS], 1ull);
        atomicMax((unsigned long long *)&stats[ST_LARGEST], (unsigned long long)(g1 - g0 + 1));
      }
    }
    g0 = j;
  }
}

// ---------------------------------------------------------------------------
// S9/S10: RQI + Getvec + output.  One thread per singleton.  Workspace A, B
// (dd, interleaved [i * S + t]): A = s (forward) then u- (backward), B = l+.
// Zero pivots are marked by a NaN low word (never produced by dd ops).
// ---------------------------------------------------------------------------
__device__ __forceinline__ dd dd_mark() { return dd_make(0.0, __longlong_as_double(0x7ff8000000000000ll)); }
__device__ __forceinline__ bool is_mark(dd x) { return isnan(x.lo); }

struct GV {
  dd gamma, zz;
  int r, c;
};

// representation element as three 16-byte loads
struct YV {
  dd d, dl, dll;
};
__device__ __forceinline__ YV ldy(const YElt *__restrict__ y, int i) {
  const double2 *q = reinterpret_cast<const double2 *>(y + i);
  double2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  YV v;
  v.d = dd_make(a.x, a.y);
  v.dl = dd_make(b.x, b.y);
  v.dll = dd_make(c.x, c.y);
  return v;
}
// RQI workspace: streamed through L2 with evict-first hints so it does not push the representation
// (read by every lane at every step) out of L2
__device__ __forceinline__ dd ldw(const dd *w, long long off) {
  double2 a = __ldcs(reinterpret_cast<const double2 *>(w + off));
  return dd_make(a.x, a.y);
}
__device__ __forceinline__ void stw(dd *w, long long off, dd v) {
  __stcs(reinterpret_cast<double2 *>(w + off), make_double2(v.hi, v.lo));
}

// z solve of N_r^T z = e_r with zero-pivot substitution (A-25); returns ||z||^2.
// Backward branch (i = r-1 .. 0, uses l+ in B) then forward branch (i = r .. nb-2, uses u- in A),
// as one loop over k with the workspace prefetched two steps ahead.  If Zc != nullptr writes
// fl64(z_i * inv) to Zc[i].
// tau >= 0 (Zc only): numerical support (A-42) -- on each side, the rows past the first edge i with
// |dl(i)| (|z(i)| + |z(i+1)|) <= tau are written as zeros (||z||^2 stays the full one)
__device__ __noinline__ dd zsolve(const YElt *__restrict__ y, int nb, int r, const dd *A, const dd *B, long long S, dd inv,
                     double *Zc, double tau = -1.0) {
  dd zz = dd_from(1.0);
  bool cutL = false, cutR = false;
  if (Zc) Zc[r] = inv.hi;
  const int K = nb - 1;
  if (K <= 0) return zz;
  // z(r+1) by the regular recurrence for the backward branch's substitution at i = r-1
  dd zp1 = dd_from(0.0);
  if (r < nb - 1) {
    dd u = ldw(A, (long long)r * S);
    if (!is_mark(u)) zp1 = dd_neg(u);
  }
#define WOFF(k) ((long long)((k) < r ? (r - 1 - (k)) : (k)) * S)
#define WLD(k) ((k) < r ? ldw(B, WOFF(k)) : ldw(A, WOFF(k)))
  dd w0 = WLD(0), w1 = WLD(min(1, K - 1));
  dd z1 = dd_from(1.0), z2 = zp1;  // z(i+1), z(i+2) for the backward branch
  dd zrm1 = dd_from(0.0);
  for (int k = 0; k < K; k++) {
    int k2 = min(k + 2, K - 1);
    dd w2 = WLD(k2);
    const bool bw = k < r;
    const int i = bw ? (r - 1 - k) : k;
    if (k == r) { z2 = zrm1; z1 = dd_from(1.0); }  // forward branch: z(i), z(i-1)
    dd z;
    if (!is_mark(w0)) {
      z = dd_neg(dd_mul(w0, z1));
    } else {
      int in = bw ? i + 1 : i - 1;
      dd num = (bw ? (in < nb - 1) : (in >= 0)) ? ld_dl(y + in) : dd_from(0.0);
      dd v = dd_neg(dd_mul(dd_div(num, ld_dl(y + i)), z2));
      z = isfinite(v.hi) ? v : dd_from(0.0);
    }
    zz = dd_add(zz, dd_mul(z, z));
    if (Zc) {
      bool &cut = bw ? cutL : cutR;
      if (!cut && tau >= 0.0 &&
          __dmul_rn(fabs(__ldg(&y[i].dl_hi)), __dadd_rn(fabs(z.hi), fabs(z1.hi))) <= tau) cut = true;
      Zc[bw ? i : i + 1] = cut ? 0.0 : dd_mul(z, inv).hi;
    }
    if (bw && i == r - 1) zrm1 = z;
    z2 = z1;
    z1 = z;
    w0 = w1;
    w1 = w2;
  }
#undef WLD
#undef WOFF
  return zz;
}

// y-bisection to relative width 2^-98 (RQI fallback)
// stop at relative width 2^-98 of |lambda| or absolute width 2^-100 spdiam, whichever is larger (A-29)
__device__ __noinline__ dd bisect_y_full(const YElt *__restrict__ y, const QElt *__restrict__ q, int nb, int j, dd lo, dd hi,
                            double spdiam) {
  const dd afloor = dd_from(__dmul_rn(0x1p-100, spdiam));
  for (int it = 0; it < 200; it++) {
    dd m = dd_lt(dd_abs(lo), dd_abs(hi)) ? dd_abs(hi) : dd_abs(lo);
    dd w = dd_sub(hi, lo);
    dd tol = dd_mul_d(m, 0x1p-98);
    if (dd_lt(tol, afloor)) tol = afloor;
    if (!dd_lt(tol, w)) break;
    dd mid = dd_add(lo, dd_mul_d(w, 0.5));
    if ((q ? negcount_y_q(q, y, nb, mid) : negcount_y(y, nb, mid)) < j) lo = mid;
    else hi = mid;
  }
  return dd_add(lo, dd_mul_d(dd_sub(hi, lo), 0.5));
}

// size-1 blocks (S2): eigenpair (alpha_s, e_s)
__global__ void k_trivial(const double *__restrict__ d, const int *__restrict__ starts, int nblk,
                          const int *__restrict__ colmap, double *W, double *Z, long long ldz, int *diag_depth,
                          double *fin_lo, double *fin_hi, int *grp_first, int *grp_last, double *rlo, double *rhi) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  int s = starts[b];
  if (starts[b + 1] - s != 1) return;
  rlo[s] = d[s];
  rhi[s] = d[s];
  int col = colmap[s];
  if (col < 0) return;
  W[col] = d[s];
  Z[(long long)col * ldz + s] = 1.0;
  if (diag_depth) { diag_depth[col] = 0; fin_lo[col] = d[s]; fin_hi[col] = d[s]; }
  if (grp_first) { grp_first[col] = s; grp_last[col] = s; }
}
