// kernels_vec.cuh -- cluster path (S8: Alg. spectrumshift, mixed
// precision P:5969-5971, depth-first P:6110-6132) and the singleton RQI /
// eigenvector kernel (S9-S10: Alg. Getvec, Alg. stask
// P:4026-4074, mixed stop P:6074-6108, convert-on-write P:6156-6158).
#pragma once
#include "kernels.cuh"

__device__ __forceinline__ dd ld_d(const YElt *y) { return dd_make(__ldg(&y->d_hi), __ldg(&y->d_lo)); }
__device__ __forceinline__ dd ld_dl(const YElt *y) { return dd_make(__ldg(&y->dl_hi), __ldg(&y->dl_lo)); }
__device__ __forceinline__ dd ld_dll(const YElt *y) { return dd_make(__ldg(&y->dll_hi), __ldg(&y->dll_lo)); }

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
  int nb = reps[C.rep].nb;
  double nu = __dmul_rn(__dmul_rn(100.0, (double)nb), EPS_X);
  for (int side = 0; side < 2; side++) {
    int j = side ? C.q : C.p;
    double lo = ilo[C.ibase + j], hi = ihi[C.ibase + j];
    double L = __dsub_rn(lo, __dmul_rn(nu, fabs(lo)));
    double H = __dadd_rn(hi, __dmul_rn(nu, fabs(hi)));
    dyadic_widen(L, H, &L, &H);
    BNode b;
    b.lo = L; b.hi = H; b.clo = 0; b.chi = 0; b.j = j; b.rep = C.rep;
    b.needLo = 1; b.needHi = 1; b.fixes = 0; b.pad = 0;
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

// S8(c): growth of dstqds(M_y, tau) for both candidate shifts, thread per (cluster, side)
__global__ void k_clu_attempt(const Cluster *__restrict__ cl, int ncl, const RepDesc *__restrict__ reps,
                              const YElt *__restrict__ my, const ShiftState *__restrict__ ss, double *gval,
                              int *valid) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2 * ncl) return;
  int c = t >> 1, side = t & 1;
  if (ss[c].done) return;
  RepDesc R = reps[cl[c].rep];
  const YElt *y = my + R.off;
  dd tau = dd_from(side ? ss[c].taur : ss[c].taul);
  dd s = dd_neg(tau);
  double g = 0.0;
  int ok = 1;
  for (int i = 0; i < R.nb - 1; i++) {
    dd den, rr, out, xn;
    qd_step(s, ld_d(y + i), ld_dl(y + i), ld_dll(y + i), tau, den, rr, out, xn);
    ok &= !(isnan(den.hi) || isnan(out.hi));
    g = dmaxd(g, fabs(den.hi));
    s = xn;
  }
  dd den = dd_add(s, ld_d(y + R.nb - 1));
  ok &= !isnan(den.hi);
  g = dmaxd(g, fabs(den.hi));
  gval[t] = g;
  valid[t] = ok;
}

__global__ void k_clu_select(const Cluster *__restrict__ cl, int ncl, const RepDesc *__restrict__ reps,
                             ShiftState *ss, const double *__restrict__ gval, const int *__restrict__ valid, int a,
                             int *ndone, long long *stats) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
  ShiftState s = ss[c];
  if (s.done) { atomicAdd(ndone, 1); return; }
  atomicAdd((unsigned long long *)&stats[ST_ATTEMPTS], 1ull);
  double gthr = __dmul_rn(GROWTH, reps[cl[c].rep].spdiam);
  int vl = valid[2 * c], vr = valid[2 * c + 1];
  double gl = gval[2 * c], gr = gval[2 * c + 1];
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
  if (s.done) atomicAdd(ndone, 1);
  ss[c] = s;
}

// S8(d): child representation M_y = (d+, l+) of dstqds(M_y, tau_best) and its x copy.
// Child rep id = repbase + c, data at pool offset poolbase + c * nbmax.
__global__ void k_clu_build(const Cluster *__restrict__ cl, int ncl, RepDesc *reps, const ShiftState *__restrict__ ss,
                            double2 *mx, YElt *my, int repbase, long long poolbase, int nbmax) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
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
                                   const double *__restrict__ ihi, double *clo, double *chi, BNode *bn, int repbase) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
  Cluster C = cl[c];
  ShiftState S = ss[c];
  if (!S.have_best) return;
  int nb = reps[C.rep].nb;
  double nu = __dmul_rn(__dmul_rn(100.0, (double)nb), EPS_X);
  double tau = S.best_tau;
  long long base = cseg[c] - (C.p - 1);  // child ibase
  double lpm = ilo[C.ibase + C.p - 1];
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
    double lo = ilo[C.ibase + j], hi = ihi[C.ibase + j];
    double a1 = __dsub_rn(lo, __dmul_rn(nu, fabs(lo)));
    double b1 = __dsub_rn(a1, tau);
    double l2 = __dsub_rn(b1, __dmul_rn(nu, fabs(b1)));
    double c1 = __dadd_rn(hi, __dmul_rn(nu, fabs(hi)));
    double e1 = __dsub_rn(c1, tau);
    double h2 = __dadd_rn(e1, __dmul_rn(nu, fabs(e1)));
    double L, H;
    dyadic_widen(l2, h2, &L, &H);
    BNode b;
    b.lo = L; b.hi = H; b.clo = 0; b.chi = 0; b.j = j; b.rep = repbase + c;
    b.needLo = 1; b.needHi = 1; b.fixes = 0; b.pad = 0;
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
__device__ __forceinline__ dd ldw(const dd *w, long long off) {
  double2 a = *reinterpret_cast<const double2 *>(w + off);
  return dd_make(a.x, a.y);
}
__device__ __forceinline__ void stw(dd *w, long long off, dd v) {
  *reinterpret_cast<double2 *>(w + off) = make_double2(v.hi, v.lo);
}

// Getvec: r < 0 -> full twisted factorization + twist search (iteration 1);
// r >= 0 (0-based) -> only the r-twisted factorization.
// Representation elements and workspace values are prefetched two steps ahead.
__device__ void getvec_dd(const YElt *__restrict__ y, int nb, dd lam, int r, dd *A, dd *B, long long S, GV &g) {
  int cnt = 0;
  const int last = nb - 1;
  if (r < 0) {
    dd s = dd_neg(lam);
    YV c0 = ldy(y, 0), c1 = ldy(y, min(1, last));
    for (int i = 0; i < last; i++) {
      YV c2 = ldy(y, min(i + 2, last));
      dd den, rr, out, xn;
      qd_step(s, c0.d, c0.dl, c0.dll, lam, den, rr, out, xn);
      stw(A, (long long)i * S, s);
      stw(B, (long long)i * S, (den.hi == 0.0) ? dd_mark() : out);
      cnt += dd_sb(den);
      s = xn;
      c0 = c1;
      c1 = c2;
    }
    dd dlast = c0.d;  // y[nb-1].d
    dd dn = dd_add(s, dlast);
    cnt += dd_sb(dn);
    dd gam = dn;  // gamma_n = s(n) + d(n) = d+(n)
    int rbest = -1;
    dd best = dd_from(INFINITY), gbest = gam;
    if (!isnan(gam.hi)) { rbest = last; best = dd_abs(gam); }
    dd p = dd_sub(dlast, lam);
    if (last >= 1) {
      YV b0 = ldy(y, last - 1), b1 = ldy(y, max(last - 2, 0));
      dd a0 = ldw(A, (long long)(last - 1) * S), a1 = ldw(A, (long long)max(last - 2, 0) * S);
      for (int i = last - 1; i >= 0; i--) {
        int i2 = max(i - 2, 0);
        YV b2 = ldy(y, i2);
        dd a2 = ldw(A, (long long)i2 * S);
        dd den, rr, out, xn;
        qd_step(p, b0.dll, b0.dl, b0.d, lam, den, rr, out, xn);
        dd gi = dd_add(a0, dd_mul(dd_mul(b0.d, rr), p));
        stw(A, (long long)i * S, (den.hi == 0.0) ? dd_mark() : out);
        if (!isnan(gi.hi)) {
          dd ag = dd_abs(gi);
          if (!dd_lt(best, ag)) { best = ag; rbest = i; gbest = gi; }
        }
        p = xn;
        b0 = b1; b1 = b2;
        a0 = a1; a1 = a2;
      }
    }
    g.r = rbest;
    g.gamma = gbest;
  } else {
    dd s = dd_neg(lam), gamma = dd_from(0.0);
    dd dlast = ldy(y, last).d;
    dd p = dd_sub(dlast, lam);
    // unified loop: k < r forward dstqds step i = k; else backward dqds step i = nb-2-(k-r)
    const int K = last;
#define IDX(k) ((k) < r ? (k) : last - 1 - ((k) - r))
    YV c0 = ldy(y, IDX(0)), c1 = ldy(y, IDX(min(1, max(K - 1, 0))));
    for (int k = 0; k < K; k++) {
      YV c2 = ldy(y, IDX(min(k + 2, K - 1)));
      const bool fw = k < r;
      const int i = IDX(k);
      dd den, rr, out, xn;
      qd_step(fw ? s : p, fw ? c0.d : c0.dll, c0.dl, fw ? c0.dll : c0.d, lam, den, rr, out, xn);
      if (fw) {
        stw(B, (long long)i * S, (den.hi == 0.0) ? dd_mark() : out);
        s = xn;
      } else {
        stw(A, (long long)i * S, (den.hi == 0.0) ? dd_mark() : out);
        if (i == r) gamma = dd_add(s, dd_mul(dd_mul(c0.d, rr), p));
        p = xn;
      }
      cnt += dd_sb(den);
      c0 = c1;
      c1 = c2;
    }
#undef IDX
    if (r == last) gamma = dd_add(s, dlast);
    cnt += dd_sb(gamma);
    g.r = r;
    g.gamma = gamma;
  }
  g.c = cnt;
}

// z solve of N_r^T z = e_r with zero-pivot substitution (A-25); returns ||z||^2.
// Backward branch (i = r-1 .. 0, uses l+ in B) then forward branch (i = r .. nb-2, uses u- in A),
// as one loop over k with the workspace prefetched two steps ahead.  If Zc != nullptr writes
// fl64(z_i * inv) to Zc[i].
__device__ dd zsolve(const YElt *__restrict__ y, int nb, int r, const dd *A, const dd *B, long long S, dd inv,
                     double *Zc) {
  dd zz = dd_from(1.0);
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
    if (Zc) Zc[bw ? i : i + 1] = dd_mul(z, inv).hi;
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
__device__ dd bisect_y_full(const YElt *__restrict__ y, int nb, int j, dd lo, dd hi) {
  for (int it = 0; it < 200; it++) {
    dd m = dd_lt(dd_abs(lo), dd_abs(hi)) ? dd_abs(hi) : dd_abs(lo);
    dd w = dd_sub(hi, lo);
    if (!dd_lt(dd_mul_d(m, 0x1p-98), w)) break;
    dd mid = dd_add(lo, dd_mul_d(w, 0.5));
    if (negcount_y(y, nb, mid) < j) lo = mid;
    else hi = mid;
  }
  return dd_add(lo, dd_mul_d(dd_sub(hi, lo), 0.5));
}

__global__ void __launch_bounds__(64) k_rqi(const Singleton *__restrict__ sg, int ns, const RepDesc *__restrict__ reps,
                                            const YElt *__restrict__ my, dd *wsA, dd *wsB, long long S, double *W,
                                            double *Z, long long ldz, int *diag_depth, double *fin_lo, double *fin_hi,
                                            long long *stats) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ns) return;
  const Singleton s = sg[t];
  const RepDesc R = reps[s.rep];
  const int nb = R.nb, j = s.j;
  const YElt *y = my + R.off;
  dd *A = wsA + t, *B = wsB + t;
  double mid = bis_mid(s.lo, s.hi);
  double nu = __dmul_rn(__dmul_rn(100.0, (double)nb), EPS_X);
  dd blo = dd_from(__dsub_rn(s.lo, __dmul_rn(nu, fabs(s.lo))));
  dd bhi = dd_from(__dadd_rn(s.hi, __dmul_rn(nu, fabs(s.hi))));
  dd lam = dd_from(mid);
  double thr1 = __dmul_rn(__dmul_rn(s.gap, EPS_X), sqrt((double)nb));
  int r = -1, iters = 0;
  long long qd = 0, qdg = 0, zs = 0;
  bool accepted = false;
  GV g;
  dd nz = dd_from(1.0);
  for (int it = 0; it < MAX_RQI && !accepted; it++) {
    if (r < 0) { qd += 2 * (nb - 1); qdg += nb - 1; } else qd += nb - 1;
    getvec_dd(y, nb, lam, r, A, B, S, g);
    iters++;
    r = g.r;
    if (r < 0) break;
    zs += nb - 1;
    dd zz = zsolve(y, nb, r, A, B, S, dd_from(0.0), nullptr);
    if (!isfinite(zz.hi) || zz.hi == 0.0) break;
    nz = dd_sqrt(zz);
    dd resid = dd_div(dd_abs(g.gamma), nz);
    dd rqc = dd_div(g.gamma, zz);
    if (resid.hi <= thr1 || dd_lt(dd_abs(rqc), dd_mul_d(dd_abs(lam), 4.0 * EPS_Y))) { accepted = true; break; }
    if (g.c < j) blo = lam; else bhi = lam;
    dd nl = dd_add(lam, rqc);
    bool ok = ((g.c < j) ? (rqc.hi > 0.0) : (rqc.hi < 0.0)) && dd_lt(blo, nl) && dd_lt(nl, bhi);
    if (ok) lam = nl;
    else break;
  }
  atomicAdd((unsigned long long *)&stats[ST_RQI_ITERS], (unsigned long long)iters);
  atomicAdd((unsigned long long *)&stats[ST_QD_STEPS], (unsigned long long)qd);
  atomicAdd((unsigned long long *)&stats[ST_QDG_STEPS], (unsigned long long)qdg);
  atomicAdd((unsigned long long *)&stats[ST_Z_STEPS], (unsigned long long)zs);
  atomicAdd((unsigned long long *)&stats[ST_ZW_STEPS], (unsigned long long)(nb - 1));
  atomicAdd((unsigned long long *)&stats[ST_GETVEC], (unsigned long long)iters);
  if (!accepted) {
    atomicAdd((unsigned long long *)&stats[ST_RQI_FALLBACK], 1ull);
    lam = bisect_y_full(y, nb, j, blo, bhi);
    getvec_dd(y, nb, lam, r, A, B, S, g);
    atomicAdd((unsigned long long *)&stats[ST_GETVEC], 1ull);
    r = g.r;
    if (r < 0) r = 0;
    dd zz = zsolve(y, nb, r, A, B, S, dd_from(0.0), nullptr);
    nz = dd_sqrt(zz);
  }
  dd sig = dd_make(R.sig_hi, R.sig_lo);
  W[s.col] = dd_add(lam, sig).hi;
  double *Zc = Z + (long long)s.col * ldz + R.bstart;
  zsolve(y, nb, r, A, B, S, dd_rcp(nz), Zc);
  if (diag_depth) {
    diag_depth[s.col] = R.depth;
    fin_lo[s.col] = s.lo;
    fin_hi[s.col] = s.hi;
  }
  atomicMax((unsigned long long *)&stats[ST_DMAX], (unsigned long long)R.depth);
}

// ---------------------------------------------------------------------------
// S9/S10, two lanes per singleton (adjacent lanes of a warp): lane F runs the
// dstqds recurrence forward (i = 0, 1, ...), lane B the dqds recurrence
// backward (i = n-2, n-3, ...), concurrently.  ||z||^2 of the twisted solve
// comes from the recurrences S_{k+1} = l+(k)^2 (1 + S_k) (sum of z(i)^2, i < k)
// and T_k = u-(k)^2 (1 + T_{k+1}) (sum of z(i)^2, i > k): ||z||^2 = 1 + S_r + T_r,
// so no z pass is needed inside the RQI (zero pivots fall back to the explicit
// z solve).  Workspace (dd, [i * S + pair]): Ws = s(i), Wt = d(i) p(i+1) /
// omega(i+1), WS = S_i, WT = T_i (iteration 1 only), WL = l+(i), WU = u-(i).
// ---------------------------------------------------------------------------
struct PairWS {
  dd *s, *t, *S, *T, *L, *U;
};

// the two lanes of a pair always take identical control paths; shuffles use the pair mask only
__device__ __forceinline__ unsigned pair_mask() { return 3u << ((threadIdx.x & 31) & ~1u); }
__device__ __forceinline__ int lane_F() { return (threadIdx.x & 31) & ~1; }
__device__ __forceinline__ int lane_B() { return (threadIdx.x & 31) | 1; }
__device__ __forceinline__ dd shfl_dd(dd v, int src_xor) {
  unsigned m = pair_mask();
  return dd_make(__shfl_xor_sync(m, v.hi, src_xor), __shfl_xor_sync(m, v.lo, src_xor));
}
__device__ __forceinline__ dd shfl_dd_from(dd v, int lane) {
  unsigned m = pair_mask();
  return dd_make(__shfl_sync(m, v.hi, lane), __shfl_sync(m, v.lo, lane));
}
__device__ __forceinline__ int shfl_i_from(int v, int lane) { return __shfl_sync(pair_mask(), v, lane); }

// returns (identically in both lanes) gamma_r, ||z||^2 (or NaN if a zero pivot broke the recurrences),
// the twist r and the inertia count c (A-26)
__device__ void getvec_pair(const YElt *__restrict__ y, int nb, dd lam, int r, bool isB, const PairWS &w,
                            long long S, GV &g) {
  const int last = nb - 1;
  const int nsteps = (r < 0) ? last : (isB ? last - r : r);
  dd x = isB ? dd_sub(ldy(y, last).d, lam) : dd_neg(lam);  // F: s(0); B: p(n-1)
  dd acc = dd_from(0.0);                                   // F: S_i; B: T_{i+1}
  dd tr = dd_from(0.0);                                    // B: t(r)
  int cnt = 0;
#define PIX(k) (isB ? (last - 1 - (k)) : (k))
  if (nsteps > 0) {
    YV c0 = ldy(y, PIX(0)), c1 = ldy(y, PIX(min(1, nsteps - 1)));
    for (int k = 0; k < nsteps; k++) {
      YV c2 = ldy(y, PIX(min(k + 2, nsteps - 1)));
      const int i = PIX(k);
      const long long off = (long long)i * S;
      dd den, rr, out, xn;
      qd_step(x, isB ? c0.dll : c0.d, c0.dl, isB ? c0.d : c0.dll, lam, den, rr, out, xn);
      dd o2 = dd_mul(out, out);
      if (!isB) {
        if (r < 0) { stw(w.s, off, x); stw(w.S, off, acc); }
        stw(w.L, off, (den.hi == 0.0) ? dd_mark() : out);
        acc = dd_mul(o2, dd_add_d(acc, 1.0));
      } else {
        if (r < 0 || i == r) {
          dd t = dd_mul(dd_mul(c0.d, rr), x);
          if (r < 0) stw(w.t, off, t);
          else tr = t;
        }
        stw(w.U, off, (den.hi == 0.0) ? dd_mark() : out);
        acc = dd_mul(o2, dd_add_d(acc, 1.0));
        if (r < 0) stw(w.T, off, acc);
      }
      cnt += dd_sb(den);
      x = xn;
      c0 = c1;
      c1 = c2;
    }
  }
#undef PIX
  __syncwarp(pair_mask());
  if (r < 0) {
    // F: x = s(n-1), acc = S_{n-1}, cnt = NegCount(LDL^T - lam I) (full D+) once d+(n-1) is added
    dd glast = isB ? dd_from(0.0) : dd_add(x, ldy(y, last).d);
    if (!isB) cnt += dd_sb(glast);
    // argmin over non-NaN |gamma_k|, ties to the smallest k: F scans [0, h), B scans [h, last)
    const int h = last / 2;
    int k0 = isB ? h : 0, k1 = isB ? last : h;
    int kb = -1;
    dd best = dd_from(INFINITY), gb = dd_from(0.0);
    for (int k = k0; k < k1; k++) {
      dd gk = dd_add(ldw(w.s, (long long)k * S), ldw(w.t, (long long)k * S));
      if (isnan(gk.hi)) continue;
      dd ag = dd_abs(gk);
      if (kb < 0 || dd_lt(ag, best)) { kb = k; best = ag; gb = gk; }
    }
    dd obest = shfl_dd(best, 1), ogb = shfl_dd(gb, 1);
    int okb = __shfl_xor_sync(pair_mask(), kb, 1);
    if (!isB) {  // merge: lower range wins ties
      if (okb >= 0 && (kb < 0 || dd_lt(obest, best))) { kb = okb; best = obest; gb = ogb; }
      if (!isnan(glast.hi) && (kb < 0 || dd_lt(dd_abs(glast), best))) { kb = last; best = dd_abs(glast); gb = glast; }
    }
    kb = shfl_i_from(kb, lane_F());
    gb = shfl_dd_from(gb, lane_F());
    cnt = shfl_i_from(cnt, lane_F());
    g.r = kb;
    g.gamma = gb;
    g.c = cnt;
    dd part = dd_from(0.0);
    if (kb >= 0) {
      if (!isB) part = (kb == last) ? acc : ldw(w.S, (long long)kb * S);
      else part = (kb == last) ? dd_from(0.0) : ldw(w.T, (long long)kb * S);
    }
    dd other = shfl_dd(part, 1);
    g.zz = dd_add_d(dd_add(part, other), 1.0);
  } else {
    // F: x = s(r), acc = S_r; B: tr = t(r), acc = T_r
    dd sr = shfl_dd_from(x, lane_F());
    dd t_r = shfl_dd_from(tr, lane_B());
    int cF = shfl_i_from(cnt, lane_F());
    int cB = shfl_i_from(cnt, lane_B());
    dd gamma = (r == last) ? dd_add(sr, ldy(y, last).d) : dd_add(sr, t_r);
    g.r = r;
    g.gamma = gamma;
    g.c = cF + cB + dd_sb(gamma);
    dd other = shfl_dd(acc, 1);
    g.zz = dd_add_d(dd_add(acc, other), 1.0);
  }
}

// Branch-free version of getvec_pair for the common case: dd ops without special-value handling,
// lane-dependent operand offsets instead of selects, two-ahead prefetch, prefetched argmin scan.
// Returns false (in both lanes) if the qd recurrence of either lane left the finite range (a zero
// pivot / IEEE infinity), in which case the caller reruns getvec_pair.
struct Elt3 {
  double2 a, b, c;
};
__device__ __forceinline__ Elt3 ld3(const YElt *__restrict__ y, int i, int oa, int oc) {
  const double2 *q = reinterpret_cast<const double2 *>(y + i);
  Elt3 e;
  e.a = __ldg(q + oa);
  e.b = __ldg(q + 1);
  e.c = __ldg(q + oc);
  return e;
}
__device__ __forceinline__ dd D(double2 v) { return dd_make(v.x, v.y); }

__device__ bool getvec_pair_fast(const YElt *__restrict__ y, int nb, dd lam, int r, bool isB, const PairWS &w,
                                 long long S, GV &g) {
  const int last = nb - 1;
  const int nsteps = (r < 0) ? last : (isB ? last - r : r);
  const int oa = isB ? 2 : 0, oc = isB ? 0 : 2;  // F: a = d, c = dll; B: a = dll, c = d (double2 slots)
  dd x = isB ? dd_sub_nf(ldy(y, last).d, lam) : dd_neg(lam);
  dd acc = dd_from(0.0), tr = dd_from(0.0);
  int cnt = 0;
  dd *P1 = isB ? w.t : w.s, *P2 = isB ? w.T : w.S, *P3 = isB ? w.U : w.L;
  const bool it1 = r < 0;
#define FIX(k) (isB ? (last - 1 - (k)) : (k))
  if (nsteps > 0) {
    Elt3 e0 = ld3(y, FIX(0), oa, oc), e1 = ld3(y, FIX(min(1, nsteps - 1)), oa, oc);
    for (int k = 0; k < nsteps; k++) {
      Elt3 e2 = ld3(y, FIX(min(k + 2, nsteps - 1)), oa, oc);
      const long long off = (long long)FIX(k) * S;
      const dd a = D(e0.a), b = D(e0.b), c = D(e0.c);
      dd den = dd_add_nf(x, a);
      dd rr = dd_rcp_nf(den);
      dd q = dd_mul_nf(x, rr);
      dd out = dd_mul_nf(b, rr);
      dd xn = dd_sub_nf(dd_mul_nf(q, c), lam);
      dd accn = dd_mul_nf(dd_mul_nf(out, out), dd_add_d_nf(acc, 1.0));
      if (it1) {
        dd t = dd_mul_nf(dd_mul_nf(c, rr), x);  // B: d(i)/omega(i+1) p(i+1)
        stw(P1, off, isB ? t : x);
        stw(P2, off, isB ? accn : acc);
      } else if (isB && k == nsteps - 1) {
        tr = dd_mul_nf(dd_mul_nf(c, rr), x);
      }
      stw(P3, off, out);
      cnt += dd_sb(den);
      x = xn;
      acc = accn;
      e0 = e1;
      e1 = e2;
    }
  }
#undef FIX
  const unsigned pm = pair_mask();
  bool ok = isfinite(x.hi) && isfinite(x.lo);
  ok = __shfl_xor_sync(pm, (int)ok, 1) && ok;
  __syncwarp(pm);
  if (!ok) return false;
  if (it1) {
    dd glast = isB ? dd_from(0.0) : dd_add(x, ldy(y, last).d);
    if (!isB) cnt += dd_sb(glast);
    const int h = last / 2;
    const int k0 = isB ? h : 0, k1 = isB ? last : h;
    int kb = -1;
    dd best = dd_from(INFINITY), gb = dd_from(0.0);
    if (k1 > k0) {
      const int kl = k1 - 1;
      dd s0 = ldw(w.s, (long long)k0 * S), t0 = ldw(w.t, (long long)k0 * S);
      dd s1 = ldw(w.s, (long long)min(k0 + 1, kl) * S), t1 = ldw(w.t, (long long)min(k0 + 1, kl) * S);
      dd s2 = ldw(w.s, (long long)min(k0 + 2, kl) * S), t2 = ldw(w.t, (long long)min(k0 + 2, kl) * S);
      for (int k = k0; k < k1; k++) {
        const int kn = min(k + 3, kl);
        dd s3 = ldw(w.s, (long long)kn * S), t3 = ldw(w.t, (long long)kn * S);
        dd gk = dd_add(s0, t0);
        dd ag = dd_abs(gk);
        bool take = !isnan(gk.hi) && (kb < 0 || dd_lt(ag, best));
        kb = take ? k : kb;
        best = take ? ag : best;
        gb = take ? gk : gb;
        s0 = s1; s1 = s2; s2 = s3;
        t0 = t1; t1 = t2; t2 = t3;
      }
    }
    dd obest = shfl_dd(best, 1), ogb = shfl_dd(gb, 1);
    int okb = __shfl_xor_sync(pm, kb, 1);
    if (!isB) {  // merge: the lower range wins ties, then k = n-1
      if (okb >= 0 && (kb < 0 || dd_lt(obest, best))) { kb = okb; best = obest; gb = ogb; }
      if (!isnan(glast.hi) && (kb < 0 || dd_lt(dd_abs(glast), best))) { kb = last; best = dd_abs(glast); gb = glast; }
    }
    kb = shfl_i_from(kb, lane_F());
    gb = shfl_dd_from(gb, lane_F());
    cnt = shfl_i_from(cnt, lane_F());
    g.r = kb;
    g.gamma = gb;
    g.c = cnt;
    dd part = dd_from(0.0);
    if (kb >= 0) {
      if (!isB) part = (kb == last) ? acc : ldw(w.S, (long long)kb * S);
      else part = (kb == last) ? dd_from(0.0) : ldw(w.T, (long long)kb * S);
    }
    dd other = shfl_dd(part, 1);
    g.zz = dd_add_d(dd_add(part, other), 1.0);
  } else {
    dd sr = shfl_dd_from(x, lane_F());
    dd t_r = shfl_dd_from(tr, lane_B());
    int cF = shfl_i_from(cnt, lane_F());
    int cB = shfl_i_from(cnt, lane_B());
    dd gamma = (r == last) ? dd_add(sr, ldy(y, last).d) : dd_add(sr, t_r);
    g.r = r;
    g.gamma = gamma;
    g.c = cF + cB + dd_sb(gamma);
    dd other = shfl_dd(acc, 1);
    g.zz = dd_add_d(dd_add(acc, other), 1.0);
  }
  return true;
}

// final pass of the pair: z(r) = 1, F writes rows r-1 .. 0, B rows r+1 .. n-1 (A-25 order of the
// zero-pivot substitutions reproduced: z(r+1) pre-value, then z(r-1), then z(r+1))
__device__ void zwrite_pair(const YElt *__restrict__ y, int nb, int r, bool isB, const PairWS &w, long long S,
                            dd inv, double *Zc) {
  const int last = nb - 1;
  dd zp1 = dd_from(0.0), zm1 = dd_from(0.0);
  dd ur = (r < last) ? ldw(w.U, (long long)r * S) : dd_from(0.0);
  if (r < last && !is_mark(ur)) zp1 = dd_neg(ur);  // pre-value
  if (r > 0) {
    dd l = ldw(w.L, (long long)(r - 1) * S);
    if (!is_mark(l)) zm1 = dd_neg(l);
    else {
      dd num = (r < last) ? ld_dl(y + r) : dd_from(0.0);
      dd v = dd_neg(dd_mul(dd_div(num, ld_dl(y + r - 1)), zp1));
      zm1 = isfinite(v.hi) ? v : dd_from(0.0);
    }
  }
  if (r < last && is_mark(ur)) {
    dd num = (r >= 1) ? ld_dl(y + r - 1) : dd_from(0.0);
    dd v = dd_neg(dd_mul(dd_div(num, ld_dl(y + r)), zm1));
    zp1 = isfinite(v.hi) ? v : dd_from(0.0);
  }
  if (!isB) {
    Zc[r] = inv.hi;
    if (r > 0) Zc[r - 1] = dd_mul(zm1, inv).hi;
  } else if (r < last) {
    Zc[r + 1] = dd_mul(zp1, inv).hi;
  }
  // F: i = r-2 .. 0 with z1 = z(i+1), z2 = z(i+2); B: computes z(i+1), i = r+1 .. last-1, z1 = z(i), z2 = z(i-1)
  const int nsteps = isB ? max(last - 1 - r, 0) : max(r - 1, 0);
  dd z1 = isB ? zp1 : zm1, z2 = dd_from(1.0);
  const dd *arr = isB ? w.U : w.L;
#define ZIX(k) (isB ? (r + 1 + (k)) : (r - 2 - (k)))
  if (nsteps > 0) {
    dd w0 = ldw(arr, (long long)ZIX(0) * S), w1 = ldw(arr, (long long)ZIX(min(1, nsteps - 1)) * S);
    for (int k = 0; k < nsteps; k++) {
      dd w2 = ldw(arr, (long long)ZIX(min(k + 2, nsteps - 1)) * S);
      const int i = ZIX(k);
      dd z;
      if (!is_mark(w0)) {
        z = dd_neg(dd_mul(w0, z1));
      } else {
        int in = isB ? i - 1 : i + 1;
        dd num = (isB ? (in >= 0) : (in < last)) ? ld_dl(y + in) : dd_from(0.0);
        dd v = dd_neg(dd_mul(dd_div(num, ld_dl(y + i)), z2));
        z = isfinite(v.hi) ? v : dd_from(0.0);
      }
      Zc[isB ? i + 1 : i] = dd_mul(z, inv).hi;
      z2 = z1;
      z1 = z;
      w0 = w1;
      w1 = w2;
    }
  }
#undef ZIX
}

__global__ void __launch_bounds__(64) k_rqi2(const Singleton *__restrict__ sg, int ns, const RepDesc *__restrict__ reps,
                                             const YElt *__restrict__ my, dd *ws, long long S, long long nbmax,
                                             double *W, double *Z, long long ldz, int *diag_depth, double *fin_lo,
                                             double *fin_hi, long long *stats) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const bool isB = gt & 1;
  const int pid = gt >> 1;  // workspace column (padded grid: S >= #pairs launched)
  const bool active = pid < ns;
  const Singleton s = sg[active ? pid : ns - 1];  // idle pairs shadow the last singleton in their own columns
  const RepDesc R = reps[s.rep];
  const int nb = R.nb, j = s.j;
  const YElt *y = my + R.off;
  const long long plane = nbmax * S;
  PairWS w;
  w.s = ws + pid; w.t = ws + plane + pid; w.S = ws + 2 * plane + pid; w.T = ws + 3 * plane + pid;
  w.L = ws + 4 * plane + pid; w.U = ws + 5 * plane + pid;
  double mid = bis_mid(s.lo, s.hi);
  double nu = __dmul_rn(__dmul_rn(100.0, (double)nb), EPS_X);
  dd blo = dd_from(__dsub_rn(s.lo, __dmul_rn(nu, fabs(s.lo))));
  dd bhi = dd_from(__dadd_rn(s.hi, __dmul_rn(nu, fabs(s.hi))));
  dd lam = dd_from(mid);
  double thr1 = __dmul_rn(__dmul_rn(s.gap, EPS_X), sqrt((double)nb));
  int r = -1, iters = 0;
  long long qd = 0, qdg = 0, zs = 0;
  bool accepted = false;
  GV g;
  dd zz = dd_from(1.0);
  for (int it = 0; it < MAX_RQI && !accepted; it++) {
    if (r < 0) { qd += 2 * (nb - 1); qdg += nb - 1; } else qd += nb - 1;
    if (!getvec_pair_fast(y, nb, lam, r, isB, w, S, g)) getvec_pair(y, nb, lam, r, isB, w, S, g);
    iters++;
    r = g.r;
    if (r < 0) break;
    zz = g.zz;
    if (!isfinite(zz.hi)) {  // zero pivot inside: explicit z solve (lane F), broadcast
      zs += nb - 1;
      if (!isB) zz = zsolve(y, nb, r, w.U, w.L, S, dd_from(0.0), nullptr);
      zz = shfl_dd_from(zz, lane_F());
    }
    if (!isfinite(zz.hi) || zz.hi == 0.0) break;
    dd nz = dd_sqrt(zz);
    dd resid = dd_div(dd_abs(g.gamma), nz);
    dd rqc = dd_div(g.gamma, zz);
    if (resid.hi <= thr1 || dd_lt(dd_abs(rqc), dd_mul_d(dd_abs(lam), 4.0 * EPS_Y))) { accepted = true; break; }
    if (g.c < j) blo = lam; else bhi = lam;
    dd nl = dd_add(lam, rqc);
    bool ok = ((g.c < j) ? (rqc.hi > 0.0) : (rqc.hi < 0.0)) && dd_lt(blo, nl) && dd_lt(nl, bhi);
    if (ok) lam = nl;
    else break;
  }
  if (!accepted) {
    if (active && !isB) atomicAdd((unsigned long long *)&stats[ST_RQI_FALLBACK], 1ull);
    lam = bisect_y_full(y, nb, j, blo, bhi);
    getvec_pair(y, nb, lam, r, isB, w, S, g);
    if (r < 0) qdg += nb - 1;
    qd += (r < 0) ? 2 * (nb - 1) : nb - 1;
    iters++;
    r = g.r < 0 ? 0 : g.r;
    zz = g.zz;
    if (!isfinite(zz.hi)) {
      zs += nb - 1;
      if (!isB) zz = zsolve(y, nb, r, w.U, w.L, S, dd_from(0.0), nullptr);
      zz = shfl_dd_from(zz, lane_F());
    }
  }
  dd inv = dd_rcp(dd_sqrt(zz));
  if (active) {
    double *Zc = Z + (long long)s.col * ldz + R.bstart;
    zwrite_pair(y, nb, r, isB, w, S, inv, Zc);
    if (!isB) {
      dd sig = dd_make(R.sig_hi, R.sig_lo);
      W[s.col] = dd_add(lam, sig).hi;
      if (diag_depth) {
        diag_depth[s.col] = R.depth;
        fin_lo[s.col] = s.lo;
        fin_hi[s.col] = s.hi;
      }
      atomicAdd((unsigned long long *)&stats[ST_RQI_ITERS], (unsigned long long)iters);
      atomicAdd((unsigned long long *)&stats[ST_QD_STEPS], (unsigned long long)qd);
      atomicAdd((unsigned long long *)&stats[ST_QDG_STEPS], (unsigned long long)qdg);
      atomicAdd((unsigned long long *)&stats[ST_Z_STEPS], (unsigned long long)zs);
      atomicAdd((unsigned long long *)&stats[ST_ZW_STEPS], (unsigned long long)(nb - 1));
      atomicAdd((unsigned long long *)&stats[ST_GETVEC], (unsigned long long)iters);
      atomicMax((unsigned long long *)&stats[ST_DMAX], (unsigned long long)R.depth);
    }
  }
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
