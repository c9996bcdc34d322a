// kernels_rqi.cuh -- singleton RQI + eigenvector kernel (S9/S10: Alg. Getvec, Alg. stask
// P:4026-4074, mixed stopping rule P:6074-6108, convert-on-write P:6156-6158), two lanes per singleton.
//
// Lane F (even) runs the dstqds recurrence forward (i = 0, 1, ...), lane B (odd) the dqds recurrence
// backward (i = n-2, n-3, ...), in lock step.  The twist quantities gamma_k = s(k) + d(k) p(k+1) /
// omega(k+1) and the norms ||z_k||^2 = 1 + S_k + T_k of the twisted solves, with
//     S_{k+1} = l+(k)^2 (1 + S_k)   (sum of z(i)^2, i < k),   T_k = u-(k)^2 (1 + T_{k+1})   (i > k),
// are formed on the fly: for the lower half of k lane B combines its own t(k), T_k with the s(k), S_k
// that lane F wrote earlier in the same pass, for the upper half lane F combines with what B wrote
// (they meet in the middle, where one shuffle exchanges the values).  So iteration 1 is one pass of
// n steps per lane and no separate argmin or z pass is needed inside the RQI.  Later iterations (twist
// r fixed) run F on 0..r-1 and B on n-2..r and store l+ / u- for the final z solve.
//
// Workspace: dd planes [i * S + pair]: P0 = s(i) / t(i), P1 = S_i / T_i (iteration 1, each
// index written by exactly one lane), P2 = l+(i) for i < r and u-(i) for i >= r (contiguous per pair).
//
// The hot loops use the branch-free dd operations (dd_*_nf); if a lane's recurrence leaves the finite
// range (a zero pivot: IEEE infinity) the pass is rerun with the careful operations,
// the infinity guard q := 1 and zero-pivot marks for the substitution formulas of Getvec.
#pragma once
#include "kernels_vec.cuh"

#ifndef MRRR_RQI_PD
#define MRRR_RQI_PD 2  // prefetch ring depth of the RQI step loops (2 measured best on C2)
#endif

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

template <bool C> __device__ __forceinline__ dd OADD(dd a, dd b) { if constexpr (C) return dd_add(a, b); else return dd_add_nf(a, b); }
template <bool C> __device__ __forceinline__ dd OSUB(dd a, dd b) { if constexpr (C) return dd_sub(a, b); else return dd_sub_nf(a, b); }
template <bool C> __device__ __forceinline__ dd OMUL(dd a, dd b) { if constexpr (C) return dd_mul(a, b); else return dd_mul_nf(a, b); }
template <bool C> __device__ __forceinline__ dd ORCP(dd a) { if constexpr (C) return dd_rcp(a); else return dd_rcp_nf(a); }
template <bool C> __device__ __forceinline__ dd OADD1(dd a) { if constexpr (C) return dd_add_d(a, 1.0); else return dd_add_d_nf(a, 1.0); }

struct Elt3 {
  double2 a, b, c;
};
// element i of the representation with lane-dependent operand order (F: a = d, c = dll; B: a = dll, c = d)
__device__ __forceinline__ Elt3 ld3(const YElt *__restrict__ y, int i, int oa, int oc) {
  const double2 *q = reinterpret_cast<const double2 *>(y + i);
  Elt3 e;
  e.a = __ldg(q + oa);
  e.b = __ldg(q + 1);
  e.c = __ldg(q + oc);
  return e;
}
__device__ __forceinline__ dd D2(double2 v) { return dd_make(v.x, v.y); }

struct Cand {  // twist candidate of one lane: |gamma|, gamma, k, ||z_k||^2 - 1
  dd best, gam, st;
  int k;
};
__device__ __forceinline__ void cand_take(Cand &c, dd g, dd st, int k, bool tie_wins) {
  if (isnan(g.hi)) return;
  dd a = dd_abs(g);
  bool take = (c.k < 0) || dd_lt(a, c.best) || (tie_wins && !dd_lt(c.best, a));
  if (take) { c.best = a; c.gam = g; c.st = st; c.k = k; }
}

// one qd step (dstqds for F, dqds for B; see qd_step) plus the ||z||^2 recurrence
template <bool C>
__device__ __forceinline__ void qd_math(dd x, dd a, dd b, dd c, dd lam, dd acc, dd &den, dd &rr, dd &out, dd &xn,
                                        dd &accn) {
  den = OADD<C>(x, a);
  rr = ORCP<C>(den);
  dd q = OMUL<C>(x, rr);
  if constexpr (C) q = (dd_isinf(x) && dd_isinf(den)) ? dd_from(1.0) : q;
  out = OMUL<C>(b, rr);
  xn = OSUB<C>(OMUL<C>(q, c), lam);
  accn = OMUL<C>(OMUL<C>(out, out), OADD1<C>(acc));
}

enum { PH_STORE = 0, PH_COMBINE = 1, PH_FIXED = 2 };

// steps k0 .. k1-1 of one lane (F: row i = k, B: row i = n-2-k) with the representation elements and
// (phase B) the other lane's halves read PD steps ahead through compile-time-indexed rings.
template <bool C, int MODE>
__device__ __forceinline__ void run_phase(const YElt *__restrict__ y, int last, int k0, int k1, bool isB, int oa,
                                          int oc, dd lam, int r, dd *P0, dd *P1, dd *P2, long long S, dd &x, dd &acc,
                                          int &cnt, Cand &cd, dd &tr) {
  constexpr int PD = MRRR_RQI_PD;
  if (k0 >= k1) return;
#define GIX(k) (isB ? (last - 1 - (k)) : (k))
  Elt3 er[PD];
  dd pq[PD], ps[PD];
#pragma unroll
  for (int u = 0; u < PD; u++) {
    const int kk = min(k0 + u, k1 - 1);
    er[u] = ld3(y, GIX(kk), oa, oc);
    if (MODE == PH_COMBINE) {
      pq[u] = ldw(P0, (long long)GIX(kk) * S);
      ps[u] = ldw(P1, (long long)GIX(kk) * S);
    }
  }
  for (int kb = k0; kb < k1; kb += PD) {
#pragma unroll
    for (int u = 0; u < PD; u++) {
      const int k = kb + u;
      if (k < k1) {
        const Elt3 e0 = er[u];
        const int kn = min(k + PD, k1 - 1);
        er[u] = ld3(y, GIX(kn), oa, oc);
        dd other, ost;
        if (MODE == PH_COMBINE) {
          other = pq[u];
          ost = ps[u];
          pq[u] = ldw(P0, (long long)GIX(kn) * S);
          ps[u] = ldw(P1, (long long)GIX(kn) * S);
        }
        const int i = GIX(k);
        const dd c = D2(e0.c);
        dd den, rr, out, xn, accn;
        qd_math<C>(x, D2(e0.a), D2(e0.b), c, lam, acc, den, rr, out, xn, accn);
        if (MODE == PH_STORE || MODE == PH_COMBINE) {
          // F: (s(i), S_i) before the update; B: t(i) = d(i) p(i+1) / omega(i+1) and T_i after it
          dd mine = isB ? OMUL<C>(OMUL<C>(c, rr), x) : x;
          dd myst = isB ? accn : acc;
          if (MODE == PH_STORE) {
            stw(P0, (long long)i * S, mine);
            stw(P1, (long long)i * S, myst);
          } else {
            cand_take(cd, OADD<C>(mine, other), OADD<C>(myst, ost), i, isB);
          }
        } else {
          if (isB && k == k1 - 1) tr = OMUL<C>(OMUL<C>(c, rr), x);  // B's last row is r
          if constexpr (C) stw(P2, i, (den.hi == 0.0) ? dd_mark() : out);
          else stw(P2, i, out);
        }
        cnt += dd_sb(den);
        x = xn;
        acc = accn;
      }
    }
  }
#undef GIX
}

// One Getvec of the pair at shift lam.  r < 0: full twisted factorization and twist
// search (iteration 1, no l+/u- stored); r >= 0: the r-twisted factorization, storing l+/u- in P2.
// Returns false (both lanes) if the fast pass left the finite range.  On return (both lanes):
// g.r, g.gamma = gamma_r, g.zz = ||z||^2 (NaN/inf if the closed form broke down), g.c = inertia (A-26).
template <bool C>
__device__ __noinline__ bool getvec_pair_t(const YElt *__restrict__ y, int nb, dd lam, int r, bool isB, dd *P0, dd *P1, dd *P2,
                              long long S, GV &g) {
  const unsigned pm = pair_mask();
  const int last = nb - 1;
  const bool it1 = r < 0;
  const int nsteps = it1 ? last : (isB ? last - r : r);
  const int oa = isB ? 2 : 0, oc = isB ? 0 : 2;
  dd x = isB ? OSUB<C>(ldy(y, last).d, lam) : dd_neg(lam);  // F: s(0); B: p(n-1)
  dd acc = dd_from(0.0), tr = dd_from(0.0);
  int cnt = 0;
  Cand cd;
  cd.k = -1; cd.best = dd_from(INFINITY); cd.gam = dd_from(0.0); cd.st = dd_from(0.0);
  if (it1) {
    // iteration 1: rows i with 2i < n-2 are reached first by the lane that stores its half of gamma_i
    // (phase A); the lanes meet at i = (n-2)/2 if n-1 is odd; after one __syncwarp every remaining row
    // (phase B) combines with the other lane's half written in phase A.
    const int kA = last / 2;
    run_phase<C, PH_STORE>(y, last, 0, kA, isB, oa, oc, lam, r, P0, P1, P2, S, x, acc, cnt, cd, tr);
    if (last & 1) {
      const int i = kA;
      Elt3 e = ld3(y, i, oa, oc);
      dd den, rr, out, xn, accn;
      qd_math<C>(x, D2(e.a), D2(e.b), D2(e.c), lam, acc, den, rr, out, xn, accn);
      dd mine = isB ? OMUL<C>(OMUL<C>(D2(e.c), rr), x) : x;
      dd myst = isB ? accn : acc;
      dd om = shfl_dd(mine, 1), ost = shfl_dd(myst, 1);
      if (!isB) cand_take(cd, OADD<C>(mine, om), OADD<C>(myst, ost), i, false);
      cnt += dd_sb(den);
      x = xn;
      acc = accn;
    }
    __syncwarp(pm);
    run_phase<C, PH_COMBINE>(y, last, kA + (last & 1), last, isB, oa, oc, lam, r, P0, P1, P2, S, x, acc, cnt, cd,
                             tr);
  } else {
    run_phase<C, PH_FIXED>(y, last, 0, nsteps, isB, oa, oc, lam, r, P0, P1, P2, S, x, acc, cnt, cd, tr);
  }
  if constexpr (!C) {
    bool ok = isfinite(x.hi) && isfinite(x.lo);
    ok = __shfl_xor_sync(pm, (int)ok, 1) && ok;
    if (!ok) return false;
  }
  __syncwarp(pm);
  if (it1) {
    // F: x = s(n-1), acc = S_{n-1}; gamma_n = d+(n) closes the full NegCount
    if (!isB) {
      dd glast = OADD<C>(x, ldy(y, last).d);
      cnt += dd_sb(glast);
      cand_take(cd, glast, acc, last, false);
    }
    dd ob = shfl_dd(cd.best, 1), og = shfl_dd(cd.gam, 1), ost = shfl_dd(cd.st, 1);
    int ok_ = __shfl_xor_sync(pm, cd.k, 1);
    if (!isB) {  // B's candidates are the lower indices: they win ties
      if (ok_ >= 0 && (cd.k < 0 || !dd_lt(cd.best, ob))) { cd.best = ob; cd.gam = og; cd.st = ost; cd.k = ok_; }
    }
    g.r = shfl_i_from(cd.k, lane_F());
    g.gamma = shfl_dd_from(cd.gam, lane_F());
    g.zz = dd_add_d(shfl_dd_from(cd.st, lane_F()), 1.0);
    g.c = shfl_i_from(cnt, lane_F());
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

// ---------------------------------------------------------------------------
// Fast Getvec on the RQI form (QElt, kernels_vec.cuh): the pivot recurrence
//   den' = (g - lam) - c2 / den
// with the dd quotient formed from the fp64 reciprocal pair of den.hi (MUFU seed + Newton), so the
// dependent chain per step is: reciprocal of den.hi, one quotient residual, one dd subtraction.
// F lane: den = d+(i), stores (iteration 1) d+(i) and S_i; B lane: den = omega(i+1), stores
// c2(i)/omega(i+1) and T_i; gamma_i = d+(i) - c2(i)/omega(i+1).  Any pivot outside [2^-1000, 2^1000]
// or a non-finite state sends the pair to the careful pass (getvec_pair_t<true>).
// ---------------------------------------------------------------------------
struct QV {
  dd c2, dl, g;
};
struct Q3 {
  double2 c2, dl, g;
};
__device__ __forceinline__ Q3 ldq(const QElt *__restrict__ q, int i, int og) {
  const double2 *p = reinterpret_cast<const double2 *>(q + i);
  Q3 v;
  v.c2 = __ldg(p);
  v.dl = __ldg(p + 1);
  v.g = __ldg(p + og);
  return v;
}
// nu / den from the reciprocal pair (r1 ~ 1/den.hi, r2 refined): unnormalized (hi, lo)
__device__ __forceinline__ dd qdiv(dd nu, dd den, double r1, double r2) {
  const double h = __dmul_rn(nu.hi, r1);
  double t = __fma_rn(-h, den.hi, nu.hi);
  t = __dadd_rn(t, nu.lo);
  t = __fma_rn(-h, den.lo, t);
  return dd_make(h, __dmul_rn(t, r2));
}
// a + b + c in dd with the three high words summed exactly (TwoSum cascade) and the low words and the
// two rounding errors in fp64: absolute error ~u^2 (|a| + |b| + |c|), i.e. a u^2-relative perturbation
// of the representation data and of the shift (the mixed-stability scale of the qd transforms)
__device__ __forceinline__ dd dd_sum3_nf(dd a, dd b, dd c) {
  const dd s1 = two_sum(a.hi, b.hi);
  const dd s2 = two_sum(s1.hi, c.hi);
  const double lo = __dadd_rn(__dadd_rn(__dadd_rn(a.lo, b.lo), c.lo), __dadd_rn(s1.lo, s2.lo));
  return two_sum(s2.hi, lo);
}
// twist candidate kept lazily: gamma = ga - gb and ||z||^2 - 1 = sa + sb are formed in dd only for the
// winner; candidates are ranked by an fp64 evaluation of |ga - gb| (the twist index is parity-unpinned,
// A-16; the winner's gamma_r used by the RQC is the dd value)
struct CandL {
  double best;
  dd ga, gb, sa, sb;
  int k;
};
__device__ __forceinline__ void candl_init(CandL &c) {
  c.best = INFINITY; c.k = -1;
  c.ga = c.gb = c.sa = c.sb = dd_from(0.0);
}
__device__ __forceinline__ void candl_take(CandL &c, dd ga, dd gb, dd sa, dd sb, int k, bool tie_wins) {
  const double g = __dadd_rn(__dsub_rn(ga.hi, gb.hi), __dsub_rn(ga.lo, gb.lo));
  if (isnan(g)) return;
  const double a = fabs(g);
  const bool take = (c.k < 0) || (a < c.best) || (tie_wins && !(c.best < a));
  if (take) { c.best = a; c.ga = ga; c.gb = gb; c.sa = sa; c.sb = sb; c.k = k; }
}

// FULL: l+/u- (out) and the norm recurrence in dd (passes that store the factors for the z solve);
// otherwise (twist-search pass) out and S/T in fp64: they only feed the twist candidates' ||z||^2 for
// the RQC and the acceptance test, whose relative accuracy needs are ~eps_x
template <bool FULL>
__device__ __forceinline__ void q_step(dd den, const Q3 &e, dd lam, dd acc, dd &P, dd &out, dd &dn, dd &accn,
                                       bool &ok) {
  const double b = den.hi;
  const double r = rcp_seed_dd(b);
  double ee = __fma_rn(-b, r, 1.0);
  ee = __fma_rn(ee, ee, ee);
  const double r1 = __fma_rn(r, ee, r);
  const double e2 = __fma_rn(-b, r1, 1.0);
  const double r2 = __fma_rn(r1, e2, r1);
  P = qdiv(D2(e.c2), den, r1, r2);
  dn = dd_sum3_nf(D2(e.g), dd_neg(lam), dd_neg(P));
  if (FULL) {
    const dd o = qdiv(D2(e.dl), den, r1, r2);
    out = fast_two_sum(o.hi, o.lo);
    accn = dd_mul_nf(dd_mul_nf(out, out), dd_add_d_nf(acc, 1.0));
  } else {
    const double o = __dmul_rn(e.dl.x, r2);
    const double o2 = __dmul_rn(o, o);
    out = dd_from(o);
    accn = dd_from(__fma_rn(o2, acc.hi, o2));
  }
  ok &= (fabs(b) > 0x1p-1000) && (fabs(b) < 0x1p1000);
}

// Per-lane prefetch ring in shared memory, filled by cp.async (no register cost): slot k holds the
// representation row of step k (c2, dl, g) and, when combining, the other lane's stored half of
// row k (P0, P1), issued MRRR_RQI_RING steps ahead of use.
#ifndef MRRR_RQI_RING
#define MRRR_RQI_RING 8
#endif
struct RingSlot {
  double2 c2, dl, g, p0, p1;
};
__device__ __forceinline__ void cp16(void *sdst, const void *gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp8(void *sdst, const void *gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int MODE>
__device__ __forceinline__ void run_phase_q(const QElt *__restrict__ q, int last, int k0, int k1, bool isB, int og,
                                            dd lam, dd *P0, dd *P1, dd *P2, long long S, dd &den, dd &acc, int &cnt,
                                            CandL &cd, dd &tr, bool &ok, RingSlot *ring) {
  constexpr int R = MRRR_RQI_RING;
  if (k0 >= k1) return;
#define GIX(k) (isB ? (last - 1 - (k)) : (k))
  auto issue = [&](int k, int slot) {
    const int i = GIX(min(k, k1 - 1));
    const double2 *p = reinterpret_cast<const double2 *>(q + i);
    cp16(&ring[slot].c2, p);
    cp16(&ring[slot].dl, p + 1);
    cp16(&ring[slot].g, p + og);
    if (MODE == PH_COMBINE) {
      cp16(&ring[slot].p0, P0 + (long long)i * S);
      cp16(&ring[slot].p1, P1 + (long long)i * S);
    }
    cp_commit();
  };
#pragma unroll
  for (int u = 0; u < R; u++) issue(k0 + u, u);
  // registers hold the current row; the next row is read from shared memory one step ahead
  cp_wait<R - 1>();
  Q3 en;
  dd on = dd_from(0.0), osn = dd_from(0.0);
  en.c2 = ring[0].c2;
  en.dl = ring[0].dl;
  en.g = ring[0].g;
  if (MODE == PH_COMBINE) {
    on = D2(ring[0].p0);
    osn = D2(ring[0].p1);
  }
#pragma unroll 2
  for (int k = k0; k < k1; k++) {
    const int slot = (k - k0) & (R - 1);
    const Q3 e0 = en;
    const dd other = on, ost = osn;
    cp_wait<R - 2>();  // the group of step k+1 has landed
    const int sn = (slot + 1) & (R - 1);
    en.c2 = ring[sn].c2;
    en.dl = ring[sn].dl;
    en.g = ring[sn].g;
    if (MODE == PH_COMBINE) {
      on = D2(ring[sn].p0);
      osn = D2(ring[sn].p1);
    }
    const int i = GIX(k);
    dd P, out, dn, accn;
    q_step<MODE == PH_FIXED>(den, e0, lam, acc, P, out, dn, accn, ok);
    if (MODE == PH_STORE || MODE == PH_COMBINE) {
      const dd mine = isB ? fast_two_sum(P.hi, P.lo) : den;
      const dd myst = isB ? accn : acc;
      if (MODE == PH_STORE) {
        stw(P0, (long long)i * S, mine);
        stw(P1, (long long)i * S, myst);
      } else {
        // gamma_i = d+(i) - c2(i)/omega(i+1): F holds the first term, B the second
        if (isB) candl_take(cd, other, mine, ost, myst, i, true);
        else candl_take(cd, mine, other, myst, ost, i, false);
      }
    } else {
      if (isB && k == k1 - 1) tr = fast_two_sum(P.hi, P.lo);  // B's last row is r: c2(r)/omega(r+1)
      stw(P2, i, out);
    }
    cnt += dd_sb(den);
    den = dn;
    acc = accn;
    issue(k + R, slot);  // slot k was read into registers last step: refill it R steps ahead
  }
  cp_wait<0>();
#undef GIX
}

// one Getvec of the pair on the RQI form; returns false (both lanes) if the careful pass is needed
__device__ __noinline__ bool getvec_pair_q(const QElt *__restrict__ q, int nb, dd lam, int r, bool isB, dd *P0, dd *P1, dd *P2,
                              long long S, GV &g) {
  extern __shared__ __align__(16) unsigned char rqi_smem[];
  RingSlot *ring = reinterpret_cast<RingSlot *>(rqi_smem) + threadIdx.x * MRRR_RQI_RING;
  const unsigned pm = pair_mask();
  const int last = nb - 1;
  const bool it1 = r < 0;
  const int og = isB ? 3 : 2;
  // F: d+(0) = d(0) - lam = gb(0) - lam;  B: omega(n-1) = g(n-2) - lam = gb(n-1) - lam
  const int i0 = isB ? last : 0;
  dd den = dd_sub_nf(dd_make(__ldg(&q[i0].gb_hi), __ldg(&q[i0].gb_lo)), lam);
  dd acc = dd_from(0.0), tr = dd_from(0.0);
  int cnt = 0;
  bool ok = true;
  CandL cd;
  candl_init(cd);
  if (it1) {
    const int kA = last / 2;
    run_phase_q<PH_STORE>(q, last, 0, kA, isB, og, lam, P0, P1, P2, S, den, acc, cnt, cd, tr, ok, ring);
    if (last & 1) {
      const int i = kA;
      const Q3 e = ldq(q, i, og);
      dd P, out, dn, accn;
      q_step<false>(den, e, lam, acc, P, out, dn, accn, ok);
      const dd mine = isB ? fast_two_sum(P.hi, P.lo) : den;
      const dd myst = isB ? accn : acc;
      const dd om = shfl_dd(mine, 1), ost = shfl_dd(myst, 1);
      if (!isB) candl_take(cd, mine, om, myst, ost, i, false);
      cnt += dd_sb(den);
      den = dn;
      acc = accn;
    }
    __syncwarp(pm);
    run_phase_q<PH_COMBINE>(q, last, kA + (last & 1), last, isB, og, lam, P0, P1, P2, S, den, acc, cnt, cd, tr, ok, ring);
  } else {
    const int nsteps = isB ? last - r : r;
    run_phase_q<PH_FIXED>(q, last, 0, nsteps, isB, og, lam, P0, P1, P2, S, den, acc, cnt, cd, tr, ok, ring);
  }
  ok = ok && isfinite(den.hi) && isfinite(den.lo) && isfinite(acc.hi) && isfinite(acc.lo);
  ok = __shfl_xor_sync(pm, (int)ok, 1) && ok;
  if (!ok) return false;
  __syncwarp(pm);
  if (it1) {
    if (!isB) {  // F: den = d+(n-1) = gamma_n closes the full NegCount
      cnt += dd_sb(den);
      candl_take(cd, den, dd_from(0.0), acc, dd_from(0.0), last, false);
    }
    const double ob = __shfl_xor_sync(pm, cd.best, 1);
    const dd oga = shfl_dd(cd.ga, 1), ogb = shfl_dd(cd.gb, 1), osa = shfl_dd(cd.sa, 1), osb = shfl_dd(cd.sb, 1);
    const int ok_ = __shfl_xor_sync(pm, cd.k, 1);
    if (!isB) {  // B's candidates are the lower indices: they win ties
      if (ok_ >= 0 && (cd.k < 0 || !(cd.best < ob))) { cd.best = ob; cd.ga = oga; cd.gb = ogb; cd.sa = osa; cd.sb = osb; cd.k = ok_; }
    }
    g.r = shfl_i_from(cd.k, lane_F());
    g.gamma = shfl_dd_from(dd_sub(cd.ga, cd.gb), lane_F());
    g.zz = dd_add_d(shfl_dd_from(dd_add(cd.sa, cd.sb), lane_F()), 1.0);
    g.c = shfl_i_from(cnt, lane_F());
  } else {
    const dd dr = shfl_dd_from(den, lane_F());
    const dd t_r = shfl_dd_from(tr, lane_B());
    const int cF = shfl_i_from(cnt, lane_F());
    const int cB = shfl_i_from(cnt, lane_B());
    const dd gamma = (r == last) ? dr : dd_sub(dr, t_r);
    g.r = r;
    g.gamma = gamma;
    g.c = cF + cB + dd_sb(gamma);
    const dd other = shfl_dd(acc, 1);
    g.zz = dd_add_d(dd_add(acc, other), 1.0);
  }
  return true;
}

// returns true if the careful (IEEE special value) pass had to run
// (force_careful: fault injection of the GPU tests, MRRR_FAULT bit 1 -- every Getvec takes the careful pass)
__device__ __forceinline__ bool getvec_pair_any(const YElt *__restrict__ y, const QElt *__restrict__ qy, int nb, dd lam,
                                                int r, bool isB, dd *P0, dd *P1, dd *P2, long long S, GV &g,
                                                bool force_careful = false) {
  if (!force_careful && getvec_pair_q(qy, nb, lam, r, isB, P0, P1, P2, S, g)) return false;
  getvec_pair_t<true>(y, nb, lam, r, isB, P0, P1, P2, S, g);
  return true;
}

// per-singleton hand-off from k_rqi2 to k_zwrite
struct ZMeta {
  double inv_hi, inv_lo;  // 1 / ||z||
  int r, careful;         // twist index; 1 if the last Getvec ran the careful pass (zero-pivot marks in P2)
};

// S10 output: z(r) = 1, z(i) = -l+(i) z(i+1) (i < r), z(i+1) = -u-(i) z(i) (i >= r), written as
// fl64(z / ||z||) into column col of Z.  One warp per singleton: the two products are computed tile by
// tile (32 rows) as warp prefix products of dd factors, times the carry of the previous tile, so the
// P2 reads and the Z column stores are coalesced.  (Rounding order differs from the sequential
// recurrence only at the dd level.)  Careful passes (zero pivots, A-25 substitutions) use lane 0 and
// the sequential zsolve.
__device__ __forceinline__ dd shfl_up_dd(dd v, int off) {
  return dd_make(__shfl_up_sync(0xffffffffu, v.hi, off), __shfl_up_sync(0xffffffffu, v.lo, off));
}
__device__ __forceinline__ dd shfl_idx_dd(dd v, int lane) {
  return dd_make(__shfl_sync(0xffffffffu, v.hi, lane), __shfl_sync(0xffffffffu, v.lo, lane));
}

// Same output as k_zwrite, HBM-streaming form: a warp takes tiles of 32 x ZC rows; the tile's factors are
// staged in shared memory by cp.async (coalesced, one tile ahead), each lane multiplies its own chunk of ZC
// consecutive factors sequentially, one warp scan combines the 32 chunk products, and the z values go back
// through shared memory so the Z column stores are coalesced.  2 dd products per row instead of the 7 of
// the per-row warp scan; 1/||z|| rides in the carry.
constexpr int ZC = 8, ZT = 32 * ZC, ZP = ZT + 32;  // rows per lane chunk, rows per tile, padded tile
__device__ __forceinline__ int zpad(int m) { return m + m / ZC; }  // chunk stride ZC + 1: conflict-free
// status (segmented RQI, kernels_rqi3.cuh): the RqiState ints of singleton w start at status[w * stride]:
// [0] status (1 accepted), [2] light, [3] pad -- rerun marker of a z window too short for the support
__global__ void __launch_bounds__(128) k_zwrite_chunk(const Singleton *__restrict__ sg, int ns,
                                                      const RepDesc *__restrict__ reps, const YElt *__restrict__ my,
                                                      const dd *__restrict__ P2base, long long S,
                                                      const ZMeta *__restrict__ zm, double *Z, long long ldz,
                                                      double eps_sup, int *status = nullptr, int status_stride = 0,
                                                      int zwin = 0, int rerun = 0, int *nrerun = nullptr) {
  // eps_sup > 0: numerical support (S10', Getvec remark (2) P:3459-3463, A-42): going outward from r,
  // the column ends at the first edge i with |dl(i)| (|z(i)| + |z(i+1)|) <= gap eps_x (z(r) = 1), i.e. on the
  // normalised values <= gap eps_x / ||z||; the rows past it are written as zeros without reading their factors.
  // inv_hi == 0 (accepted on an RQC-only pass, k_zrc recomputed the factors of the rows within zwin of r): a
  // measuring sweep over the window finds both ends and ||z||^2 over the support (dd), then the write sweep;
  // a support that reaches the window's edge before the matrix's marks the singleton for a stored pass (rerun).
  __shared__ __align__(16) double2 sbuf[4][2][ZP];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w = blockIdx.x * 4 + wib;
  if (w >= ns) return;
  int *stw_ = status ? status + (long long)w * status_stride : nullptr;
  if (stw_ && stw_[0] != 1) return;
  if (stw_ && rerun && stw_[3] != 1) return;
  const ZMeta m = zm[w];
  const Singleton s = sg[w];
  const RepDesc R = reps[s.rep];
  const int nb = R.nb, r = m.r, last = nb - 1;
  dd inv = dd_make(m.inv_hi, m.inv_lo);
  const dd *P = P2base + (long long)w * S;
  double *Zc = Z + (long long)s.col * ldz + R.bstart;
  const YElt *y = my + R.off;
  const double tau = eps_sup > 0.0 ? __dmul_rn(s.gap, eps_sup) : -1.0;  // gap eps_x on z with z(r) = 1
  if (m.careful) {
    if (lane == 0) zsolve(y, nb, r, P, P, 1, inv, Zc, tau);
    return;
  }
  const bool win = m.inv_hi == 0.0 && tau >= 0.0;
  double2(*buf)[ZP] = sbuf[wib];
  // one side: rows r-1, r-2, ... (side 0) or r+1, r+2, ... (side 1); phase 0 measures (cut and sum of squares of
  // the unnormalised z, no stores), phase 1 writes with the measured cut, phase 2 detects and writes
  auto zside = [&](int side, int phase, int lenA, int cutIn, dd &sum) -> int {
    const int len = side ? last - r : r;
    const int lim = phase == 0 ? lenA : len;  // rows whose factors exist
    const dd carry0 = phase == 0 ? dd_from(1.0) : inv;
    const double tauT = phase == 0 ? tau : __dmul_rn(tau, inv.hi);
    double prevv = carry0.hi;
    int cut = phase == 1 ? cutIn : len;
    const int ntile = (min(lim, phase == 1 ? cut : lim) + ZT - 1) / ZT;
    auto issue = [&](int t) {
      double2 *b = buf[t & 1];
#pragma unroll
      for (int u = 0; u < ZC; u++) {
        const int ml = lane + 32 * u, mm = t * ZT + ml;
        if (mm < lim) cp16(&b[zpad(ml)], P + (side ? r + mm : r - 1 - mm));
      }
      cp_commit();
    };
    if (ntile > 0) issue(0);
    dd carry = carry0;
    int t = 0;
    for (; t < ntile; t++) {
      if (t + 1 < ntile) issue(t + 1);
      else cp_commit();
      cp_wait<1>();
      __syncwarp();
      double2 *b = buf[t & 1];
      const int m0 = t * ZT, mc = m0 + lane * ZC;
      dd p[ZC];
      dd acc = dd_from(1.0);
#pragma unroll
      for (int e = 0; e < ZC; e++) {
        if (mc + e < lim) {
          const double2 f = b[lane * (ZC + 1) + e];
          const dd nf = dd_make(-f.x, -f.y);
          acc = (e == 0) ? nf : dd_mul_nf(acc, nf);
        }
        p[e] = acc;
      }
      __syncwarp();
      dd v = acc;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const dd o = shfl_up_dd(v, off);
        if (lane >= off) v = dd_mul_nf(o, v);
      }
      dd ex = shfl_up_dd(v, 1);
      const dd E = lane ? dd_mul_nf(carry, ex) : carry;
      carry = dd_mul_nf(carry, shfl_idx_dd(v, 31));
      double *sd = reinterpret_cast<double *>(b);
      dd zv[ZC];
#pragma unroll
      for (int e = 0; e < ZC; e++) {
        zv[e] = dd_mul_nf(E, p[e]);
        sd[lane * (ZC + 1) + e] = zv[e].hi;
      }
      __syncwarp();
      if (phase != 1 && tau >= 0.0) {
        // edge between this row and the previous one (towards r): dl(r - 1 - mm) on the left, dl(r + mm) on the right
        int c = len;
#pragma unroll
        for (int e = ZC - 1; e >= 0; e--) {
          const int mm = mc + e;
          if (mm < lim) {
            const double vv = sd[lane * (ZC + 1) + e];
            const double pv = e ? sd[lane * (ZC + 1) + e - 1] : (lane ? sd[lane * (ZC + 1) - 2] : prevv);  // (ZC + 1)-stride chunks
            const double dl = fabs(__ldg(&y[side ? r + mm : r - 1 - mm].dl_hi));
            if (__dmul_rn(dl, __dadd_rn(fabs(vv), fabs(pv))) <= tauT) c = mm;
          }
        }
        cut = __reduce_min_sync(0xffffffffu, c);
        prevv = sd[zpad(ZT - 1)];
      }
      if (phase == 0) {
#pragma unroll
        for (int e = 0; e < ZC; e++)
          if (mc + e < min(cut, lim)) sum = dd_add_nf(sum, dd_mul_nf(zv[e], zv[e]));
      }
      __syncwarp();
      if (phase != 0) {
#pragma unroll
        for (int u = 0; u < ZC; u++) {
          const int ml = lane + 32 * u, mm = m0 + ml;
          if (mm < len) Zc[side ? r + 1 + mm : r - 1 - mm] = mm < cut ? sd[zpad(ml)] : 0.0;
        }
      }
      __syncwarp();
      if (cut < len && cut < m0 + ZT) {
        t++;
        break;
      }
    }
    cp_wait<0>();  // drain the prefetch of the next tile
    __syncwarp();
    if (phase != 0 && t * ZT < len) {
      // rows past the support: one contiguous range [a, b) of the column, stored as 16-byte zeros
      const int a = side ? r + 1 + t * ZT : 0, b = side ? r + 1 + len : r - t * ZT;
      double *z0 = Zc + a;
      const int head = (reinterpret_cast<uintptr_t>(z0) & 15) ? 1 : 0, cnt = b - a;
      if (head && lane == 0) z0[0] = 0.0;
      double2 *z2 = reinterpret_cast<double2 *>(z0 + head);
      const int n2 = (cnt - head) >> 1;
      for (int u = lane; u < n2; u += 32) z2[u] = make_double2(0.0, 0.0);
      if (((cnt - head) & 1) && lane == 0) z0[cnt - 1] = 0.0;
    }
    return cut;
  };
  if (!win) {
    if (lane == 0) Zc[r] = inv.hi;
    dd unused = dd_from(0.0);
    for (int side = 0; side < 2; side++)
      if ((side ? last - r : r) > 0) zside(side, 2, 0, 0, unused);
    return;
  }
  // window rows with recomputed factors: l+ rows [r - zwin, r), u- rows [r, r + zwin] (clipped)
  const int lenL = r, lenR = last - r;
  const int avL = min(r, zwin), avR = min(r + zwin, nb - 2) - r + 1;
  dd sum = dd_from(0.0);
  const int cL = lenL > 0 ? zside(0, 0, min(avL, lenL), 0, sum) : 0;
  const int cR = lenR > 0 ? zside(1, 0, min(avR, lenR), 0, sum) : 0;
  if ((lenL > 0 && cL >= min(avL, lenL) && avL < lenL) || (lenR > 0 && cR >= min(avR, lenR) && avR < lenR)) {
    if (lane == 0 && stw_) {  // the support reaches past the window: a stored pass at the same lambda, then again
      stw_[0] = 0;
      stw_[2] = 0;
      stw_[3] = 1;
      atomicAdd(nrerun, 1);
    }
    return;
  }
  // ||z||^2 over the support: the lanes' partial sums plus z(r)^2 = 1
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sum = dd_add_nf(sum, dd_make(__shfl_xor_sync(0xffffffffu, sum.hi, off),
                                                                      __shfl_xor_sync(0xffffffffu, sum.lo, off)));
  inv = dd_rcp(dd_sqrt(dd_add_d(sum, 1.0)));
  if (lane == 0) Zc[r] = inv.hi;
  if (lenL > 0) zside(0, 1, 0, cL, sum);
  if (lenR > 0) zside(1, 1, 0, cR, sum);
}

__global__ void __launch_bounds__(64) k_rqi2(const Singleton *__restrict__ sg, int ns, const RepDesc *__restrict__ reps,
                                             const YElt *__restrict__ my, const QElt *__restrict__ mq, dd *ws,
                                             long long S, long long nbmax,
                                             double *W, ZMeta *zmeta, int *diag_depth, double *fin_lo,
                                             double *fin_hi, long long *stats, int fault, int sd, double eps_x,
                                             double eps_y) {
  // fault (MRRR_FAULT, GPU tests only): bit 0 skips the RQI iterations (every singleton takes the bisection
  // fallback of P:3481-3482), bit 1 sends every Getvec through the careful IEEE pass
  const bool fc = (fault & 2) != 0;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const bool isB = gt & 1;
  const int pid = gt >> 1;  // workspace column (padded grid: S >= #pairs launched)
  const bool active = pid < ns;
  const Singleton s = sg[active ? pid : ns - 1];  // idle pairs shadow the last singleton in their own columns
  const RepDesc R = reps[s.rep];
  const int nb = R.nb, j = s.j;
  const YElt *y = my + R.off;
  const QElt *qy = mq + R.off;
  const long long plane = nbmax * S;
  // P0, P1 planes [row * S + pair]; P2 (l+/u- of the r-twisted pass) contiguous per pair (k_zwrite reads
  // it row-parallel within a warp)
  dd *P0 = ws + pid, *P1 = ws + plane + pid, *P2 = ws + 2 * plane + (long long)pid * nbmax;
  double mid = bis_mid(s.lo, s.hi);
  double nu = __dmul_rn(__dmul_rn(100.0, (double)nb), EPS_X);
  dd blo = dd_from(__dsub_rn(s.lo, __dmul_rn(nu, fabs(s.lo))));
  dd bhi = dd_from(__dadd_rn(s.hi, __dmul_rn(nu, fabs(s.hi))));
  dd lam = dd_from(mid);
  double thr1 = __dmul_rn(__dmul_rn(s.gap, eps_x), sqrt((double)nb));
  int r = -1, iters = 0;
  long long qd = 0, qdg = 0, zs = 0;
  bool accepted = false, lu_valid = false, careful = false;
  GV g;
  dd zz = dd_from(1.0);
  for (int it = 0; it < ((fault & 1) ? 0 : MAX_RQI) && !accepted; it++) {
    if (r < 0) { qd += 2 * (nb - 1); qdg += nb - 1; } else qd += nb - 1;
    lu_valid = r >= 0;
    careful = getvec_pair_any(y, qy, nb, lam, r, isB, P0, P1, P2, S, g, fc);
    iters++;
    r = g.r;
    if (r < 0) break;
    zz = g.zz;
    if (!isfinite(zz.hi)) {  // closed form broke down (overflow / zero pivot): explicit z solve (A-25)
      if (!lu_valid) { careful = getvec_pair_any(y, qy, nb, lam, r, isB, P0, P1, P2, S, g, fc); lu_valid = true; qd += nb - 1; }
      zs += nb - 1;
      if (!isB) zz = zsolve(y, nb, r, P2, P2, 1, dd_from(0.0), nullptr);
      zz = shfl_dd_from(zz, lane_F());
    }
    if (!isfinite(zz.hi) || zz.hi == 0.0) break;
    dd nz = dd_sqrt(zz);
    dd resid = dd_div(dd_abs(g.gamma), nz);
    dd rqc = dd_div(g.gamma, zz);
    // tol2: |RQC| < 4 eps_y |lam|, not below the representation's y-rounding 2^-100 spdiam (A-30)
    dd tol2 = dd_mul_d(dd_abs(lam), 4.0 * eps_y);
    if (dd_lt(tol2, dd_from(__dmul_rn(0x1p-100, R.spdiam)))) tol2 = dd_from(__dmul_rn(0x1p-100, R.spdiam));
    if (resid.hi <= thr1 || dd_lt(dd_abs(rqc), tol2)) { accepted = true; break; }
    if (g.c < j) blo = lam; else bhi = lam;
    dd nl = sd ? dd_from(__dadd_rn(lam.hi, rqc.hi)) : dd_add(lam, rqc);  // sd: lambda kept in binary64
    const bool sgn = (g.c < j) ? (rqc.hi > 0.0) : (rqc.hi < 0.0);
    bool ok = sgn && dd_lt(blo, nl) && dd_lt(nl, bhi);
#ifdef MRRR_DEBUG_RQI
    if (!ok && active && !isB)
      printf("RQI reject j=%d it=%d r=%d c=%d resid=%.3e thr1=%.3e rqc=%.3e lam=%.17e blo=%.17e bhi=%.17e careful=%d\n", j,
             it, r, g.c, resid.hi, thr1, rqc.hi, lam.hi, blo.hi, bhi.hi, (int)careful);
#endif
    if (ok) lam = nl;
    else {
      if (active && !isB) atomicAdd((unsigned long long *)&stats[sgn ? ST_RQI_REJ_BRACKET : ST_RQI_REJ_SIGN], 1ull);
      break;
    }
  }
  if (!accepted) {
    if (active && !isB) atomicAdd((unsigned long long *)&stats[ST_RQI_FALLBACK], 1ull);
    lam = bisect_y_full(y, qy, nb, j, blo, bhi, R.spdiam);
    lu_valid = r >= 0;
    careful = getvec_pair_any(y, qy, nb, lam, r, isB, P0, P1, P2, S, g, fc);
    if (r < 0) qdg += nb - 1;
    qd += (r < 0) ? 2 * (nb - 1) : nb - 1;
    iters++;
    r = g.r < 0 ? 0 : g.r;
    zz = g.zz;
  }
  if (!lu_valid) {  // accepted on a twist-search pass: one r-twisted pass to store l+ / u- (and its dd ||z||^2)
    careful = getvec_pair_any(y, qy, nb, lam, r, isB, P0, P1, P2, S, g, fc);
    qd += nb - 1;
    zz = g.zz;
  }
  if (!isfinite(zz.hi) || zz.hi == 0.0) {
    zs += nb - 1;
    if (!isB) zz = zsolve(y, nb, r, P2, P2, 1, dd_from(0.0), nullptr);
    zz = shfl_dd_from(zz, lane_F());
  }
  dd inv = dd_rcp(dd_sqrt(zz));
  if (active) {
    if (!isB) {
      ZMeta zmv;
      zmv.inv_hi = inv.hi; zmv.inv_lo = inv.lo; zmv.r = r; zmv.careful = careful ? 1 : 0;
      if (careful) atomicAdd((unsigned long long *)&stats[ST_CAREFUL], 1ull);
      zmeta[pid] = zmv;
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
