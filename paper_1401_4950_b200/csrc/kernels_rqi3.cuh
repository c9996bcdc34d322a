// kernels_rqi3.cuh -- singleton RQI (S9/S10: Alg. Getvec, Alg. stask, mixed stop
// P:6074-6108) with segmented passes.
//
// The qd recurrences of a twisted factorization contract away from the eigenvector's peak (a perturbation
// of d+(i) is multiplied by l+(i)^2 = (z(i)/z(i+1))^2 < 1 where z grows), so each pass is split into K
// segments per lane that run concurrently: segment k starts W rows early from a guess, records its state
// when it reaches its first row, and is accepted only if that state equals, bit for bit, the predecessor's
// exact end state (then every operation of the segment saw the sequential operands).  A singleton with a
// mismatch, or whose fast pass left the finite range, is handed to the two-lane kernel k_rqi2 (which also
// runs the careful IEEE pass and the bisection fallback), so results never depend on a guess.
//
//   k_rqi3_init     RQI state: lambda = interval midpoint, bracket, acceptance threshold.
//   k_twist_lane    iteration 1's twist search in x-arithmetic (A-31) over row-aligned chunks: the
//                   F lane stores d+(i), the B lane forms gamma(i) = d+(i) - c2(i)/omega(i+1) and keeps the
//                   chunk's argmin (k_twist_lane_dd: the same in dd, for child frames).
//   k_twist_pick2   junction check and r = argmin |gamma_k| (ties: smallest k) over the verified chunks.
//   k_fixed_chunk   the r-twisted factorization in y-arithmetic (dd), chunk-major and segmented: l+/u- into
//                   P2, the partial norms S/T as per-chunk affine maps, inertia counts, gamma_r's two halves.
//   k_fixed_step    junction check, gamma_r, ||z||^2, inertia; the stask decision: accept (write W and
//                   the z-write metadata), or apply the RQC and run another k_fixed_chunk, or hand over.
#pragma once
#include "kernels_rqi.cuh"

struct RqiState {
  double lam_hi, lam_lo, blo_hi, blo_lo, bhi_hi, bhi_lo, thr1;
  int r, it, status, wide;  // status: 0 active, 1 accepted, 2 handed to k_rqi2; wide: 8x warm-up
  int light, pad;           // light: RQC-only (no factors stored) passes still due before a stored one
};

// per (singleton, lane, segment) record of a segmented pass
struct SegRec {
  double in_hi, in_lo, out_hi, out_lo;  // state entering the segment's first row, state after its last
  double A, B_hi, B_lo;                 // partial norm: S_end = A * S_start + B (fixed pass)
  double t_hi, t_lo;                    // B lane's c2(r)/omega(r+1) (segment that ends at row r)
  int cnt, ok, empty, pad;              // empty: the lane has fewer steps than segments
};

__global__ void k_rqi3_init(const Singleton *__restrict__ sg, int ns, const RepDesc *__restrict__ reps,
                            RqiState *st, double eps_x, double rtol, int *mode0) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ns) return;
  const Singleton s = sg[i];
  const int nb = reps[s.rep].nb;
  const double nu = __dmul_rn(__dmul_rn(100.0, (double)nb), EPS_X);
  RqiState q;
  q.lam_hi = bis_mid(s.lo, s.hi);
  q.lam_lo = 0.0;
  q.blo_hi = __dsub_rn(s.lo, __dmul_rn(nu, fabs(s.lo)));
  q.blo_lo = 0.0;
  q.bhi_hi = __dadd_rn(s.hi, __dmul_rn(nu, fabs(s.hi)));
  q.bhi_lo = 0.0;
  q.thr1 = __dmul_rn(__dmul_rn(s.gap, eps_x), sqrt((double)nb));  // k_rs gap eps_x sqrt(n)
  q.r = -1;
  q.it = 0;
  q.status = 0;
  q.wide = 0;
  // the first pass only corrects lambda-hat (its factors are not the accepted vector's); an interval left at the
  // early-stop tolerance (A-41: wider than the classification rtol; its midpoint within 2^-8 gap of lambda)
  // takes a second one -- measured: two corrections from there, one from an rtol interval
  q.light = bis_continue(s.lo, s.hi, rtol) ? 2 : 1;
  q.pad = 0;
  if (q.light == 2) atomicOr(mode0, 3);  // the first pass: the x-arithmetic one (mode 3) when any is due
  st[i] = q;
}

// F lane step t = row t; B lane step t = row nb-2-t.  Row data of a lane: c2(i), gf(i) (F) or gb(i) (B).
// balanced split of a singleton's 2K segment threads between its lanes (F: r steps, B: nb-1-r): each lane
// gets segments in proportion to its length, at least one each, so the 2K threads run chains of about
// (nb-1)/(2K) + W steps whatever r is (F segment 0 must exist even for r = 0: it reports d+(0))
__device__ __forceinline__ int seg_kf(int nb, int r, int K2) {
  const int tot = nb - 1, sf = r, sb = nb - 1 - r;
  if (sb <= 0) return K2 - 1;
  if (sf <= 0 || tot <= 0) return 1;
  return min(max((int)(((long long)K2 * sf + tot / 2) / tot), 1), K2 - 1);
}
__device__ __forceinline__ int seg_row(bool isB, int nb, int t) { return isB ? nb - 2 - t : t; }

// ---------------------------------------------------------------------------
// Twist search in two passes over row-aligned chunks (A-31; replaces k_twist_seg + k_twist_pick):
// k_twist_f runs the forward lane over chunk c = rows [cL, (c+1)L) and stores TF[row * S + i] = d+(row);
// k_twist_b runs the backward lane over the same chunk, forms gamma(row) = TF(row) - c2(row)/omega(row+1)
// on the fly and keeps the chunk's argmin |gamma| (only TF is stored: half the traffic of storing both
// lanes); k_twist_pick2 takes the argmin over the chunks where both lanes are verified (every junction
// state bit-identical to its exact predecessor's exit).  Thread (chunk c, singleton i), consecutive
// threads = consecutive singletons on one chunk: shared row loads, coalesced TF stores and loads.
// ---------------------------------------------------------------------------
// one warp (32 singletons) stages its singletons' records in shared memory with coalesced 16-byte loads
// (the per-thread record walks are otherwise a chain of dependent cache misses); returns this thread's copy
__device__ __forceinline__ const void *stage_recs(const void *rec, int bytes, int ns, uint4 *sm) {
  const int i0 = blockIdx.x * 32, lane = threadIdx.x & 31, n16 = bytes / 16;
  for (int q = 0; q < 32 && i0 + q < ns; q++) {
    const uint4 *src = reinterpret_cast<const uint4 *>(reinterpret_cast<const char *>(rec) + (long long)(i0 + q) * bytes);
    for (int u = lane; u < n16; u += 32) sm[q * n16 + u] = src[u];
  }
  __syncwarp();
  return sm + lane * n16;
}
struct TwRec {
  double in, out;       // lane state entering the chunk's first step / after its last step
  double best, scale;   // B: the chunk's min |gamma| and max(|TF|, |TB|) at its argmin
  int ok, empty, row, pad;
  double in_lo, out_lo;  // dd twist search (child frames): low words of the states
};
__device__ __forceinline__ double tw_lam(const RqiState &S) {
  // evaluated a fraction of the inflated bracket away from lambda-hat, so that |gamma_r| stays well above
  // the fp64 rounding of its terms however close lambda-hat is (r is eigenvector j's peak either way)
  return __dadd_rn(S.lam_hi, ldexp(__dsub_rn(S.bhi_hi, S.blo_hi), -8));
}
template <bool ISB>
__global__ void __launch_bounds__(128) k_twist_lane(const Singleton *__restrict__ sg, int ns,
                                                    const RepDesc *__restrict__ reps, const QElt *__restrict__ mq,
                                                    const RqiState *__restrict__ st, int KT, int Wu, double *TF,
                                                    long long S_, TwRec *rec) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (long long)ns * KT) return;
  const int i = (int)(g % ns), c = (int)(g / ns);
  const RqiState S = st[i];
  if (S.status != 0) return;
  TwRec *R = rec + ((long long)i * KT + c) * 2 + (ISB ? 1 : 0);
  const RepDesc Rp = reps[sg[i].rep];
  const int nb = Rp.nb, steps = nb - 1;
  const QElt *q = mq + Rp.off;
  const double lam = tw_lam(S);
  const int L = max((steps + KT - 1) / KT, 1);
  const int lo = min(c * L, steps), hi = min(lo + L, steps);
  double *T = TF + i;
#define TROW(row) T[(long long)(row) * S_]
  if (hi <= lo) {
    R->empty = 1;
    R->ok = 1;
    if (!ISB && c == 0 && steps == 0) TROW(0) = __dsub_rn(__ldg(&q[0].gb_hi), lam);  // nb = 1: gamma = d+(0)
    return;
  }
  // F: steps t = rows lo..hi-1; B: steps t = nb-1-hi .. nb-2-lo (rows hi-1 .. lo)
  const int t0 = ISB ? nb - 1 - hi : lo, t1 = ISB ? nb - 1 - lo : hi;
  const int tw = (t0 == 0) ? 0 : max(t0 - Wu, 0);
  const int rs = ISB ? nb - 1 - tw : tw;
  double den = __dsub_rn(__ldg(&q[rs].gb_hi), lam);  // exact at t = 0, a guess elsewhere
  double din = den, best = INFINITY, scale = 0.0;
  int brow = -1;
  bool ok = true;
  constexpr int PF = 8;
  double rc[PF], rg[PF], rf[PF];  // B also prefetches TF(row): the stored forward lane streams from HBM
  auto ld = [&](int t, int u) {
    const int row = max(seg_row(ISB, nb, min(t, t1 - 1)), 0);
    rc[u] = __ldg(&q[row].c2_hi);
    rg[u] = ISB ? __ldg(&q[row].gb_hi) : __ldg(&q[row].gf_hi);
    if (ISB) rf[u] = (t >= t0) ? __ldcs(T + (long long)row * S_) : 0.0;
  };
  auto step = [&](int t, double c2, double gg, double tf) {
    if (t == t0) din = den;
    const double P = div_fast_nocheck(c2, den);
    if (t >= t0) {
      const int row = seg_row(ISB, nb, t);
      if (ISB) {  // gamma(row) = d+(row) - c2(row)/omega(row+1); rows visited downwards: ties to the smaller row
        const double gm = fabs(__dsub_rn(tf, P));
        if (gm <= best) { best = gm; brow = row; scale = fmax(fabs(tf), fabs(P)); }
      } else {
        TROW(row) = den;
      }
    }
    den = __dsub_rn(__dsub_rn(gg, lam), P);
    ok &= isfinite(den) && den != 0.0;
  };
#pragma unroll
  for (int u = 0; u < PF; u++) ld(tw + u, u);
  int t = tw;
  for (; t + PF <= t1; t += PF) {
#pragma unroll
    for (int u = 0; u < PF; u++) {
      const double c2 = rc[u], gg = rg[u], tf = ISB ? rf[u] : 0.0;
      ld(t + u + PF, u);
      step(t + u, c2, gg, tf);
    }
  }
#pragma unroll
  for (int u = 0; u < PF; u++)
    if (t + u < t1) step(t + u, rc[u], rg[u], ISB ? rf[u] : 0.0);
  if (!ISB && hi == steps) TROW(nb - 1) = den;  // gamma_n = d+(n)
#undef TROW
  R->in = din;
  R->out = den;
  R->in_lo = 0.0;
  R->out_lo = 0.0;
  R->best = best;
  R->scale = scale;
  R->row = brow;
  R->ok = ok ? 1 : 0;
  R->empty = 0;
}
// r = argmin |gamma| over the chunks verified in both lanes (F: the prefix of chunks whose entry states
// chain exactly from row 0; B: the suffix chaining exactly from row nb-2), plus gamma_n = d+(n) when the
// whole F lane is verified; ties to the smaller row.  Unresolved (|gamma_r| within 2^-46 of its terms) or
// no candidate: handed over.
__global__ void k_twist_pick2(const Singleton *__restrict__ sg, int ns, const RepDesc *__restrict__ reps,
                              RqiState *st, int KT, const double *__restrict__ TF, const dd *__restrict__ TFd,
                              long long S_, const TwRec *__restrict__ rec, double res, long long *stats, int stage) {
  extern __shared__ uint4 recsm[];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const TwRec *Rs = stage ? reinterpret_cast<const TwRec *>(stage_recs(rec, 2 * KT * (int)sizeof(TwRec), ns, recsm))
                          : rec + (long long)i * KT * 2;
  unsigned ho = 0, rows = 0;
  if (i < ns && st[i].status == 0) {
    const int nb = reps[sg[i].rep].nb;
    const TwRec *R = Rs;
    int kf = 0, prev = -1;  // F: chunks 0..kf-1 verified
    for (; kf < KT; kf++) {
      const TwRec &a = R[2 * kf];
      if (a.empty) continue;
      if (!a.ok || (prev >= 0 && (__double_as_longlong(a.in) != __double_as_longlong(R[2 * prev].out) ||
                                  __double_as_longlong(a.in_lo) != __double_as_longlong(R[2 * prev].out_lo))))
        break;
      prev = kf;
    }
    int kb = KT - 1;  // B: chunks kb+1..KT-1 verified
    prev = -1;
    for (; kb >= 0; kb--) {
      const TwRec &a = R[2 * kb + 1];
      if (a.empty) continue;
      if (!a.ok || (prev >= 0 && (__double_as_longlong(a.in) != __double_as_longlong(R[2 * prev + 1].out) ||
                                  __double_as_longlong(a.in_lo) != __double_as_longlong(R[2 * prev + 1].out_lo))))
        break;
      prev = kb;
    }
    double best = INFINITY, sc = 0.0;
    int bk = -1;
    for (int c = kb + 1; c < kf; c++) {  // chunks verified in both lanes (ascending rows: ties keep the smaller)
      const TwRec &a = R[2 * c + 1];
      if (a.empty || a.row < 0) continue;
      if (a.best < best) { best = a.best; bk = a.row; sc = a.scale; }
    }
    if (kf == KT) {  // gamma_n = d+(n) (B contributes 0) once the whole F lane is exact
      const double tn = fabs(TFd ? TFd[(long long)(nb - 1) * S_ + i].hi : TF[(long long)(nb - 1) * S_ + i]);
      if (tn < best) { best = tn; bk = nb - 1; sc = tn; }
    }
    if (bk < 0 || !(best > res * sc)) {
      st[i].status = 2;
      ho = 1;
    } else {
      st[i].r = bk;
      rows = (unsigned)(2 * (nb - 1));
    }
  }
  ho = __reduce_add_sync(0xffffffffu, ho);
  rows = __reduce_add_sync(0xffffffffu, rows);
  if ((threadIdx.x & 31) == 0) {
    if (ho) atomicAdd((unsigned long long *)&stats[ST_HO_TWIST], (unsigned long long)ho);
    if (rows) atomicAdd((unsigned long long *)&stats[ST_TWIST_ROWS], (unsigned long long)rows);
  }
}

// the r-twisted factorization in dd: F steps 0..r-1, B steps 0..nb-2-r (rows nb-2 .. r)
// one segment of a fixed-lambda pass: steps t in [tw, t1) of lane isB (F: row t, B: row nb-2-t), warm-up
// [tw, t0) from a guess (the recurrence alone), result in *R (entry state at t0, exit state, partial norm,
// inertia count).  LIGHT: the RQC-only pass (no factors stored, norm in fp64; A-31 note in DESIGN.md).
__device__ __forceinline__ bool rcp_nr2(double b, double &r1, double &r2) {
  const double rc = rcp_seed_dd(b);
  double ee = __fma_rn(-b, rc, 1.0);
  ee = __fma_rn(ee, ee, ee);
  r1 = __fma_rn(rc, ee, rc);
  const double e2 = __fma_rn(-b, r1, 1.0);
  r2 = __fma_rn(r1, e2, r1);
  return (fabs(b) > 0x1p-1000) && (fabs(b) < 0x1p1000);
}
#ifndef MRRR_ZG
#define MRRR_ZG 8
#endif
constexpr int ZG = MRRR_ZG;            // factor rows per bulk store
constexpr int ZSTRIDE = 2 * ZG + 1;  // double2 per thread: two groups + pad (16-byte lanes, conflict-free)

// L2 prefetch of the row PFD steps ahead (child frames: each singleton streams its own representation
// from HBM; the root's rows are L2-resident and shared, so no hint is issued there)
constexpr int PFD = 16;
__device__ __forceinline__ void l2_prefetch(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
template <bool LIGHT, bool PF>
__device__ __forceinline__ void seg_pass_t(const QElt *__restrict__ q, int nb, int isB, int t0, int t1, int tw,
                                           dd lam, dd nlam, dd *P, SegRec *R, double2 *stg, dd *zin = nullptr,
                                           int zrow = -1) {
  constexpr bool pf = PF;
  R->empty = 0;
  const int rs = isB ? nb - 1 - tw : tw, og = isB ? 3 : 2;
  dd den = dd_sub_nf(dd_make(__ldg(&q[rs].gb_hi), __ldg(&q[rs].gb_lo)), lam);
  bool ok = true;
  if (pf)
    for (int u = 0; u < PFD; u++) l2_prefetch(q + min(max(seg_row(isB, nb, tw + u), 0), nb - 1));
  for (int t = tw; t < t0; t++) {
    if (pf) l2_prefetch(q + min(max(seg_row(isB, nb, t + PFD), 0), nb - 1));
    const double2 *pq = reinterpret_cast<const double2 *>(q + seg_row(isB, nb, t));
    const dd c2 = D2(__ldg(pq)), gg = D2(__ldg(pq + og));
    double r1, r2;
    ok &= rcp_nr2(den.hi, r1, r2);
    den = dd_sum3_nf(gg, nlam, dd_neg(qdiv(c2, den, r1, r2)));
  }
  const dd din = den;
  dd Pq = dd_from(0.0), Bs = dd_from(0.0);
  double A = 1.0;
  int cnt = 0, ng = 0, grp = 0;
  // the next row is loaded one step ahead (the loads otherwise sit on the recurrence's critical path)
  const int dq = isB ? -4 : 4;  // double2 per QElt row, in the lane's direction
  const double2 *pq = reinterpret_cast<const double2 *>(q + min(max(seg_row(isB, nb, t0), 0), nb - 1));
  double2 nc2 = __ldg(pq), ndl = __ldg(pq + 1), ngg = __ldg(pq + og);
  if (pf && t0 > tw)
    for (int u = 0; u < PFD; u++) l2_prefetch(q + min(max(seg_row(isB, nb, t0 + u), 0), nb - 1));
  for (int t = t0; t < t1; t++) {
    if (pf) l2_prefetch(q + min(max(seg_row(isB, nb, t + PFD), 0), nb - 1));
    const int row = seg_row(isB, nb, t);
    if (LIGHT && row == zrow) *zin = den;  // the lane's state entering row zrow (z recompute window, k_zrc)
    const dd c2 = D2(nc2), dl = D2(ndl), gg = D2(ngg);
    if (t + 1 < t1) pq += dq;
    nc2 = __ldg(pq);
    ndl = __ldg(pq + 1);
    ngg = __ldg(pq + og);
    double r1, r2;
    ok &= rcp_nr2(den.hi, r1, r2);
    Pq = qdiv(c2, den, r1, r2);
    if (LIGHT) {
      const double o = __dmul_rn(dl.hi, r2), o2 = __dmul_rn(o, o);
      A = __dmul_rn(o2, A);
      Bs.hi = __fma_rn(o2, Bs.hi, o2);
    } else {
      const dd o = qdiv(dl, den, r1, r2);
      const dd out = fast_two_sum(o.hi, o.lo);
      if (stg) {  // stage; B lanes fill their group backwards so it is ascending in memory
        stg[grp * ZG + (isB ? ZG - 1 - ng : ng)] = make_double2(out.hi, out.lo);
        if (++ng == ZG || t + 1 == t1) {
          const int low = isB ? row : row - ng + 1;
          bulk_store(P + low, stg + grp * ZG + (isB ? ZG - ng : 0), (unsigned)(ng * sizeof(double2)));
          grp ^= 1;
          ng = 0;
          bulk_wait_read<1>();  // the other group's previous store has read its rows
        }
      } else {
        stw(P, row, out);
      }
      const dd o2 = dd_mul_nf(out, out);
      A = __dmul_rn(o2.hi, A);
      Bs = dd_mul_nf(o2, dd_add_d_nf(Bs, 1.0));
    }
    cnt += dd_sb(den);
    den = dd_sum3_nf(gg, nlam, dd_neg(Pq));
  }
  if (!LIGHT && stg) bulk_wait_all();
  ok &= isfinite(den.hi) && isfinite(den.lo) && isfinite(Bs.hi);
  R->in_hi = din.hi;
  R->in_lo = din.lo;
  R->out_hi = den.hi;
  R->out_lo = den.lo;
  R->A = A;
  R->B_hi = Bs.hi;
  R->B_lo = Bs.lo;
  const dd tl = fast_two_sum(Pq.hi, Pq.lo);  // B lane: c2(r)/omega(r+1) of the step on row r
  R->t_hi = tl.hi;
  R->t_lo = tl.lo;
  R->cnt = cnt;
  R->ok = ok ? 1 : 0;
}
__device__ __forceinline__ void seg_pass(const QElt *__restrict__ q, int nb, int isB, int t0, int t1, int tw,
                                         bool light, dd lam, dd nlam, dd *P, SegRec *R, double2 *stg = nullptr,
                                         bool pf = false, dd *zin = nullptr, int zrow = -1) {
  if (pf) {
    if (light) seg_pass_t<true, true>(q, nb, isB, t0, t1, tw, lam, nlam, P, R, nullptr, zin, zrow);
    else seg_pass_t<false, true>(q, nb, isB, t0, t1, tw, lam, nlam, P, R, stg);
  } else {
    if (light) seg_pass_t<true, false>(q, nb, isB, t0, t1, tw, lam, nlam, P, R, nullptr, zin, zrow);
    else seg_pass_t<false, false>(q, nb, isB, t0, t1, tw, lam, nlam, P, R, stg);
  }
}

// Z recompute window (numerical support, A-42): a singleton accepted on an RQC-only pass is not
// repeated as a stored pass.  Its factors l+ (rows [zf, r)) and u- (rows [r, zb]) are recomputed from the exact
// lane states the accepted pass recorded entering rows zf and zb, with the stored pass's operations, so the
// z write reads the same bits it would have read after a stored pass -- but only ZWIN rows on each side.
__device__ __forceinline__ int zwin_f(int r, int win) { return max(r - win, 0); }
__device__ __forceinline__ int zwin_b(int nb, int r, int win) { return min(r + win, nb - 2); }
// thread per (singleton, lane): lane F recomputes l+(row) for rows [zf, r), lane B u-(row) for rows zb .. r (down),
// from the states k_fixed_chunk recorded entering rows zf / zb in the accepted RQC-only pass (exact states: every
// junction of that pass verified), with the stored pass's operations (seg_pass_t<false>), into the factor plane
__global__ void __launch_bounds__(128) k_zrc(const Singleton *__restrict__ sg, int ns, const RepDesc *__restrict__ reps,
                                             const QElt *__restrict__ mq, const RqiState *__restrict__ st,
                                             const ZMeta *__restrict__ zm, const dd *__restrict__ zin, dd *P2,
                                             long long nbmax, int zwin) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= 2LL * ns) return;
  const int i = (int)(g % ns), isB = (int)(g / ns);
  if (st[i].status != 1 || zm[i].inv_hi != 0.0 || zm[i].careful) return;
  const RqiState S = st[i];
  const RepDesc Rp = reps[sg[i].rep];
  const int nb = Rp.nb, r = S.r;
  const QElt *q = mq + Rp.off;
  dd *P = P2 + (long long)i * nbmax;
  const dd lam = dd_make(S.lam_hi, S.lam_lo), nlam = dd_neg(lam);
  int t0, t1;  // lane steps: F step t = row t, B step t = row nb-2-t
  if (!isB) {
    t0 = zwin_f(r, zwin);
    t1 = r;
  } else {
    if (r > nb - 2) return;
    t0 = nb - 2 - zwin_b(nb, r, zwin);
    t1 = nb - 1 - r;
  }
  if (t1 <= t0) return;
  const int og = isB ? 3 : 2;
  dd den = zin[2LL * i + isB];
  // rows loaded ZPF steps ahead (a ring of registers): the loads stay off the recurrence's critical path
  constexpr int ZPF = 8;
  double2 rc[ZPF], rd[ZPF], rg[ZPF];
  auto ld = [&](int t, int u) {
    const double2 *pq = reinterpret_cast<const double2 *>(q + seg_row(isB, nb, min(t, t1 - 1)));
    rc[u] = __ldg(pq);
    rd[u] = __ldg(pq + 1);
    rg[u] = __ldg(pq + og);
  };
#pragma unroll
  for (int u = 0; u < ZPF; u++) ld(t0 + u, u);
  for (int tb = t0; tb < t1; tb += ZPF)
#pragma unroll
  for (int u = 0; u < ZPF; u++) {
    const int t = tb + u;
    if (t >= t1) break;
    const int row = seg_row(isB, nb, t);
    const dd c2 = D2(rc[u]), dl = D2(rd[u]), gg = D2(rg[u]);
    ld(t + ZPF, u);
    double r1, r2;
    rcp_nr2(den.hi, r1, r2);
    const dd Pq = qdiv(c2, den, r1, r2);
    const dd o = qdiv(dl, den, r1, r2);
    stw(P, row, fast_two_sum(o.hi, o.lo));
    den = dd_sum3_nf(gg, nlam, dd_neg(Pq));
  }
}
// after a rerun's stored pass: a singleton that did not accept there goes to the two-lane kernel
__global__ void k_zrc_settle(RqiState *st, int ns) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ns || st[i].pad != 1) return;
  if (st[i].status == 0) st[i].status = 2;
}
static_assert(offsetof(RqiState, wide) == offsetof(RqiState, status) + 4 &&
                  offsetof(RqiState, light) == offsetof(RqiState, status) + 8 &&
                  offsetof(RqiState, pad) == offsetof(RqiState, status) + 12,
              "k_zwrite_chunk reads status / light / pad at int offsets 0 / 2 / 3");

// the same segment in binary64 (single/double realisation): den' = (g - lam) - c2 / den with the
// IEEE quotients c2/den and dl/den from one reciprocal pair of den (fast range; a pivot outside it flags the
// segment, as in the dd pass); factors stored with zero low words, partial norms in binary64
__device__ __forceinline__ double sd_q2(double a, double b, double r1, double r2) {
  const double q0 = __dmul_rn(a, r1);
  return __fma_rn(__fma_rn(-b, q0, a), r2, q0);
}
template <bool LIGHT>
__device__ __forceinline__ void seg_pass_sd(const QElt *__restrict__ q, int nb, int isB, int t0, int t1, int tw,
                                            double lam, dd *P, SegRec *R, double2 *stg) {
  R->empty = 0;
  const int rs = isB ? nb - 1 - tw : tw, og = isB ? 6 : 4;  // double offset of g in a QElt row
  double den = __dsub_rn(__ldg(&q[rs].gb_hi), lam);
  bool ok = true;
  for (int t = tw; t < t0; t++) {
    const double *pq = reinterpret_cast<const double *>(q + seg_row(isB, nb, t));
    const double c2 = __ldg(pq), gg = __ldg(pq + og);
    double r1, r2;
    ok &= rcp_nr2(den, r1, r2);
    den = __dsub_rn(__dsub_rn(gg, lam), sd_q2(c2, den, r1, r2));
  }
  const double din = den;
  double Pq = 0.0, A = 1.0, Bs = 0.0;
  int cnt = 0, ng = 0, grp = 0;
  const int dq = isB ? -8 : 8;  // doubles per QElt row, in the lane's direction
  const double *pq = reinterpret_cast<const double *>(q + min(max(seg_row(isB, nb, t0), 0), nb - 1));
  double nc2 = __ldg(pq), ndl = __ldg(pq + 2), ngg = __ldg(pq + og);
  for (int t = t0; t < t1; t++) {
    const int row = seg_row(isB, nb, t);
    const double c2 = nc2, dl = ndl, gg = ngg;
    if (t + 1 < t1) pq += dq;
    nc2 = __ldg(pq);
    ndl = __ldg(pq + 2);
    ngg = __ldg(pq + og);
    double r1, r2;
    ok &= rcp_nr2(den, r1, r2);
    Pq = sd_q2(c2, den, r1, r2);
    const double out = LIGHT ? __dmul_rn(dl, r2) : sd_q2(dl, den, r1, r2);
    if (!LIGHT) {
      if (stg) {
        stg[grp * ZG + (isB ? ZG - 1 - ng : ng)] = make_double2(out, 0.0);
        if (++ng == ZG || t + 1 == t1) {
          const int low = isB ? row : row - ng + 1;
          bulk_store(P + low, stg + grp * ZG + (isB ? ZG - ng : 0), (unsigned)(ng * sizeof(double2)));
          grp ^= 1;
          ng = 0;
          bulk_wait_read<1>();
        }
      } else {
        P[row] = dd_make(out, 0.0);
      }
    }
    const double o2 = __dmul_rn(out, out);
    A = __dmul_rn(o2, A);
    Bs = __fma_rn(o2, Bs, o2);
    cnt += (signbit(den) && !isnan(den)) ? 1 : 0;
    den = __dsub_rn(__dsub_rn(gg, lam), Pq);
  }
  if (!LIGHT && stg) bulk_wait_all();
  ok &= isfinite(den) && isfinite(Bs);
  R->in_hi = din;
  R->in_lo = 0.0;
  R->out_hi = den;
  R->out_lo = 0.0;
  R->A = A;
  R->B_hi = Bs;
  R->B_lo = 0.0;
  R->t_hi = Pq;
  R->t_lo = 0.0;
  R->cnt = cnt;
  R->ok = ok ? 1 : 0;
}

// Chunk-major form of k_fixed_seg: the rows 0..nb-2 are cut into K2 fixed chunks of L rows.  Thread
// (slot c, singleton i), c < K2, runs chunk c's primary part: its F part (rows [lo, min(hi, r))) if the
// chunk starts below r (chunk 0 always: it reports d+(0) even when r = 0), else the whole chunk as B part;
// slot K2 runs the B part (rows [r, hi)) of the chunk holding r when that chunk's primary is its F part.
// Each thread runs ONE part, with its direction as data, so F and B lanes of a warp share the instruction
// stream; consecutive threads are consecutive singletons on the same chunk, so on a shared
// representation a warp loads one or two distinct rows per step (the lane-major layout loads 32).
// Records: rec[(i * K2 + c) * 2 + lane] (lane 0 F, 1 B); parts that do not exist are marked empty.
// dd twist search for child frames (the fp64 search rarely resolves gamma there: a child representation's
// eigenvalues are tiny next to its pivots): k_twist_lane's two passes with the y-arithmetic step of the
// fixed passes (one dd quotient, one dd three-term sum) and d+ stored in dd.
template <bool ISB>
__global__ void __launch_bounds__(128) k_twist_lane_dd(const Singleton *__restrict__ sg, int ns,
                                                       const RepDesc *__restrict__ reps,
                                                       const QElt *__restrict__ mq, const RqiState *__restrict__ st,
                                                       int KT, int Wu, dd *TF, long long S_, TwRec *rec) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (long long)ns * KT) return;
  const int i = (int)(g % ns), c = (int)(g / ns);
  const RqiState S = st[i];
  if (S.status != 0) return;
  TwRec *R = rec + ((long long)i * KT + c) * 2 + (ISB ? 1 : 0);
  const RepDesc Rp = reps[sg[i].rep];
  const int nb = Rp.nb, steps = nb - 1;
  const QElt *q = mq + Rp.off;
  const dd lam = dd_add_d(dd_make(S.lam_hi, S.lam_lo), ldexp(__dsub_rn(S.bhi_hi, S.blo_hi), -8)), nlam = dd_neg(lam);
  const int L = max((steps + KT - 1) / KT, 1);
  const int lo = min(c * L, steps), hi = min(lo + L, steps);
  dd *T = TF + i;
  if (hi <= lo) {
    R->empty = 1;
    R->ok = 1;
    if (!ISB && c == 0 && steps == 0) T[0] = dd_sub_nf(dd_make(__ldg(&q[0].gb_hi), __ldg(&q[0].gb_lo)), lam);
    return;
  }
  const int t0 = ISB ? nb - 1 - hi : lo, t1 = ISB ? nb - 1 - lo : hi;
  const int tw = (t0 == 0) ? 0 : max(t0 - Wu, 0);
  const int rs = ISB ? nb - 1 - tw : tw, og = ISB ? 3 : 2;
  dd den = dd_sub_nf(dd_make(__ldg(&q[rs].gb_hi), __ldg(&q[rs].gb_lo)), lam);
  dd din = den;
  double best = INFINITY, scale = 0.0;
  int brow = -1;
  bool ok = true;
  constexpr int PF = 4;
  double2 rc[PF], rg[PF], rf[PF];
  auto ld = [&](int t, int u) {
    const int row = max(seg_row(ISB, nb, min(t, t1 - 1)), 0);
    const double2 *pq = reinterpret_cast<const double2 *>(q + row);
    rc[u] = __ldg(pq);
    rg[u] = __ldg(pq + og);
    if (ISB) rf[u] = (t >= t0) ? __ldcs(reinterpret_cast<const double2 *>(T + (long long)row * S_)) : make_double2(0, 0);
  };
  auto step = [&](int t, double2 c2v, double2 gv, double2 tfv) {
    if (t == t0) din = den;
    double r1, r2;
    ok &= rcp_nr2(den.hi, r1, r2);
    const dd P = qdiv(D2(c2v), den, r1, r2);
    if (t >= t0) {
      const int row = seg_row(ISB, nb, t);
      if (ISB) {
        const dd gmd = dd_sub(D2(tfv), P);
        const double gm = fabs(gmd.hi);
        if (gm <= best) { best = gm; brow = row; scale = fmax(fabs(tfv.x), fabs(P.hi)); }
      } else {
        T[(long long)row * S_] = den;
      }
    }
    den = dd_sum3_nf(D2(gv), nlam, dd_neg(P));
  };
#pragma unroll
  for (int u = 0; u < PF; u++) ld(tw + u, u);
  int t = tw;
  for (; t + PF <= t1; t += PF) {
#pragma unroll
    for (int u = 0; u < PF; u++) {
      const double2 c2 = rc[u], gg = rg[u], tf = ISB ? rf[u] : make_double2(0, 0);
      ld(t + u + PF, u);
      step(t + u, c2, gg, tf);
    }
  }
#pragma unroll
  for (int u = 0; u < PF; u++)
    if (t + u < t1) step(t + u, rc[u], rg[u], ISB ? rf[u] : make_double2(0, 0));
  if (!ISB && hi == steps) T[(long long)(nb - 1) * S_] = den;  // gamma_n = d+(n)
  ok &= isfinite(den.hi) && isfinite(den.lo);
  R->in = din.hi;
  R->in_lo = din.lo;
  R->out = den.hi;
  R->out_lo = den.lo;
  R->best = best;
  R->scale = scale;
  R->row = brow;
  R->ok = ok ? 1 : 0;
  R->empty = 0;
}

#ifndef MRRR_FC_MINB
#define MRRR_FC_MINB 1
#endif
__global__ void __launch_bounds__(128, MRRR_FC_MINB) k_fixed_chunk(const Singleton *__restrict__ sg, int ns,
                                                     const RepDesc *__restrict__ reps, const QElt *__restrict__ mq,
                                                     const RqiState *__restrict__ st, int K2, int Wu, dd *P2,
                                                     long long nbmax, SegRec *rec, int bulk, int sd,
                                                     const int *__restrict__ modep, dd *zin = nullptr,
                                                     int zwin = 0) {
  // 3: the x-arithmetic RQC-only passes (S.light == 2), 0: the dd RQC-only passes (S.light == 1), 1: the stored
  // ones (S.light == 0), 2: none left (k_rqi_mode)
  const int mode = *modep;
  if (mode == 2) return;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (long long)ns * (K2 + 1)) return;
  const int i = (int)(g % ns), slot = (int)(g / ns);
  const RqiState S = st[i];
  if (S.status != 0 || S.light != (mode == 3 ? 2 : mode == 0 ? 1 : 0)) return;
  const RepDesc Rp = reps[sg[i].rep];
  const int nb = Rp.nb, r = S.r, steps = nb - 1;
  const int L = max((steps + K2 - 1) / K2, 1), W = S.wide ? 8 * Wu : Wu;
  const int cr = (r < steps) ? r / L : -1;  // chunk holding row r (none when r = nb-1: B has no steps)
  auto bounds = [&](int c, int &lo, int &hi) {
    lo = min(c * L, steps);
    hi = min(lo + L, steps);
  };
  auto fprim = [&](int c, int lo) { return c == 0 || lo < r; };
  SegRec *R0 = rec + (long long)i * K2 * 2;
  int isB, t0, t1;
  SegRec *R;
  if (slot < K2) {
    int lo, hi;
    bounds(slot, lo, hi);
    if (fprim(slot, lo)) {
      isB = 0;
      t0 = lo;
      t1 = max(min(hi, r), lo);
      R = R0 + 2 * slot;
      if (slot != cr) {
        R0[2 * slot + 1].empty = 1;
        R0[2 * slot + 1].ok = 1;
      }
    } else {
      R0[2 * slot].empty = 1;
      R0[2 * slot].ok = 1;
      R = R0 + 2 * slot + 1;
      if (hi <= lo) {
        R->empty = 1;
        R->ok = 1;
        return;
      }
      isB = 1;
      t0 = nb - 1 - hi;
      t1 = nb - 1 - lo;
    }
  } else {
    if (cr < 0) return;
    int lo, hi;
    bounds(cr, lo, hi);
    if (!fprim(cr, lo)) return;  // the primary thread runs the whole chunk as B part
    isB = 1;
    t0 = nb - 1 - hi;
    t1 = nb - 1 - r;
    R = R0 + 2 * cr + 1;
  }
  const bool light = S.light != 0;
  const QElt *q = mq + Rp.off;
  const dd lam = dd_make(S.lam_hi, S.lam_lo), nlam = dd_neg(lam);
  __shared__ __align__(16) double2 stage[128 * ZSTRIDE];
  const int tw = t0 == 0 ? 0 : max(t0 - W, 0);
  double2 *stg = bulk ? stage + threadIdx.x * ZSTRIDE : nullptr;
  // sd: the single/double realisation's binary64 passes; S.light == 2: the first of two RQC-only passes from an
  // interval left at the early-stop tolerance (A-41) -- a correction from 2^-8 gap needs only ~2^-24 gap
  // relative accuracy, which x-arithmetic on fl64 of the representation gives (the dd passes that follow
  // decide the eigenpair), at about half the issue cost of the dd pass
  if (sd || mode == 3) {
    if (light) seg_pass_sd<true>(q, nb, isB, t0, t1, tw, S.lam_hi, P2 + (long long)i * nbmax, R, nullptr);
    else seg_pass_sd<false>(q, nb, isB, t0, t1, tw, S.lam_hi, P2 + (long long)i * nbmax, R, stg);
    return;
  }
  // zwin > 0: record the lane's state entering the first row of the z recompute window (k_zrc); rows the
  // window does not reach (zf = 0, zb = nb - 2) start from the lane's exact start instead
  int zrow = -1;
  if (zin && light) zrow = isB ? zwin_b(nb, r, zwin) : zwin_f(r, zwin);
  seg_pass(q, nb, isB, t0, t1, tw, light, lam, nlam, P2 + (long long)i * nbmax, R, stg, Rp.depth > 0,
           zin ? zin + 2LL * i + isB : nullptr, zrow);
}

// thread per singleton: junctions, gamma_r, ||z||^2, inertia, and the stask decision
// per-thread counter increments, summed per warp before one atomic each
struct FsInc {
  unsigned nact, wide, hofixed, horqc, iters, light, qd, zw, dmax, nlight;  // nact / nlight: active, next pass
};                                                                           // stored / RQC-only
__device__ __forceinline__ void fixed_step_body(int i, const Singleton *__restrict__ sg,
                                                const RepDesc *__restrict__ reps, RqiState *st, int K,
                                                const SegRec *__restrict__ F, double *W, ZMeta *zmeta,
                                                int *diag_depth, double *fin_lo, double *fin_hi, FsInc &inc,
                                                int sd, double eps_y, int mode, int zrc) {
  RqiState S = st[i];
  if (S.status != 0 || S.light != (mode == 3 ? 2 : mode == 0 ? 1 : 0)) return;
  const Singleton s = sg[i];
  const RepDesc Rp = reps[s.rep];
  const int nb = Rp.nb, r = S.r, j = s.j;
  bool good = true;
  dd Ssum = dd_from(0.0), Tsum = dd_from(0.0), dr = dd_from(0.0), tr = dd_from(0.0);
  int c = 0;
  for (int ln = 0; ln < 2; ln++) {
    // chunk layout: F records at [2c], B records at [2c + 1] walked from the last chunk down
    const SegRec *X = F;
    const int Kl = 2 * K;
    int prev = -1;
    dd acc = dd_from(0.0);
    for (int kk = 0; kk < Kl; kk++) {
      const int k = 2 * (ln ? Kl - 1 - kk : kk) + ln;
      const SegRec &a = X[k];
      if (a.empty) continue;
      good &= a.ok != 0;
      if (prev >= 0)
        good &= __double_as_longlong(a.in_hi) == __double_as_longlong(X[prev].out_hi) &&
                __double_as_longlong(a.in_lo) == __double_as_longlong(X[prev].out_lo);
      acc = dd_add(dd_mul_d(acc, a.A), dd_make(a.B_hi, a.B_lo));
      c += a.cnt;
      prev = k;
    }
    if (ln == 0) {
      Ssum = acc;
      if (prev >= 0) dr = dd_make(X[prev].out_hi, X[prev].out_lo);  // d+(r): F's exact end state
    } else {
      Tsum = acc;
      if (prev >= 0) tr = dd_make(X[prev].t_hi, X[prev].t_lo);     // c2(r)/omega(r+1): B's last step
    }
  }
  if (!good) {
    if (!S.wide) {  // a warm-up too short for this singleton: repeat the pass with an 8x longer one
      st[i].wide = 1;
      if (S.light) inc.nlight++; else inc.nact++;
      inc.wide++;
      return;
    }
    st[i].status = 2;
    inc.hofixed++;
    return;
  }
  // single/double: gamma_r = d+(r) - c2(r)/omega(r+1) in binary64
  const dd gamma = (r == nb - 1) ? dr : (sd ? dd_from(__dsub_rn(dr.hi, tr.hi)) : dd_sub(dr, tr));
  c += dd_sb(gamma);
  const dd zz = dd_add_d(dd_add(Ssum, Tsum), 1.0);
  dd lam = dd_make(S.lam_hi, S.lam_lo), blo = dd_make(S.blo_hi, S.blo_lo), bhi = dd_make(S.bhi_hi, S.bhi_lo);
  S.it++;
  inc.iters++;
  const bool was_light = S.light != 0;
  if (was_light) inc.light += (unsigned)(nb - 1);
  else inc.qd += (unsigned)(nb - 1);
  bool accepted = false, handover = false;
  if (!isfinite(zz.hi) || zz.hi == 0.0) {
    handover = true;
  } else {
    const dd nz = dd_sqrt(zz);
    const dd resid = dd_div(dd_abs(gamma), nz);
    const dd rqc = dd_div(gamma, zz);
    dd tol2 = dd_mul_d(dd_abs(lam), 4.0 * eps_y);  // A-30
    if (dd_lt(tol2, dd_from(__dmul_rn(0x1p-100, Rp.spdiam)))) tol2 = dd_from(__dmul_rn(0x1p-100, Rp.spdiam));
    if (resid.hi <= S.thr1 || dd_lt(dd_abs(rqc), tol2)) {
      if (was_light && !(zrc && mode == 0)) {  // accepted on an RQC-only pass: repeat it at the same lambda with
        S.light = 0;                           // the factors stored
        inc.nact++;
        st[i] = S;
        return;
      }
      accepted = true;  // zrc: accepted on a dd RQC-only pass; k_zrc recomputes the factors of the z window
    } else {
      if (c < j) blo = lam; else bhi = lam;
      const dd nl = sd ? dd_from(__dadd_rn(lam.hi, rqc.hi)) : dd_add(lam, rqc);  // sd: lambda in binary64
      const bool okc = ((c < j) ? (rqc.hi > 0.0) : (rqc.hi < 0.0)) && dd_lt(blo, nl) && dd_lt(nl, bhi);
      if (okc && S.it < MAX_RQI) lam = nl;
      else handover = true;  // bisection fallback / iteration cap: the two-lane kernel redoes this singleton
      // RQC-only passes still due (k_rqi3_init); zrc: every pass is one until acceptance (the factors of the
      // accepted one come from k_zrc), so no stored pass runs
      S.light = was_light ? max(S.light - 1, zrc ? 1 : 0) : 0;
    }
  }
  if (accepted) {
    const dd inv = dd_rcp(dd_sqrt(zz));
    ZMeta zm;
    zm.inv_hi = inv.hi; zm.inv_lo = inv.lo; zm.r = r; zm.careful = 0;
    if (was_light) { zm.inv_hi = 0.0; zm.inv_lo = 0.0; }  // 1/||z|| over the support: k_zwrite_chunk computes it
    zmeta[i] = zm;
    const dd sig = dd_make(Rp.sig_hi, Rp.sig_lo);
    W[s.col] = dd_add(lam, sig).hi;
    if (diag_depth) {
      diag_depth[s.col] = Rp.depth;
      fin_lo[s.col] = s.lo;
      fin_hi[s.col] = s.hi;
    }
    inc.zw += (unsigned)(nb - 1);
    inc.dmax = max(inc.dmax, (unsigned)Rp.depth);
    S.status = 1;
  } else if (handover) {
    S.status = 2;
    inc.horqc++;
  } else if (S.light) {
    inc.nlight++;
  } else {
    inc.nact++;
  }
  S.lam_hi = lam.hi; S.lam_lo = lam.lo;
  S.blo_hi = blo.hi; S.blo_lo = blo.lo;
  S.bhi_hi = bhi.hi; S.bhi_lo = bhi.lo;
  st[i] = S;
}

__global__ void k_fixed_step(const Singleton *__restrict__ sg, int ns, const RepDesc *__restrict__ reps,
                             RqiState *st, int K, const SegRec *__restrict__ rec, double *W,
                             ZMeta *zmeta, int *diag_depth, double *fin_lo, double *fin_hi, long long *stats,
                             int *nactive, int stage, int sd, double eps_y, const int *__restrict__ modep,
                             int zrc = 0) {
  const int mode = *modep;
  if (mode == 2) return;
  extern __shared__ uint4 recsm[];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int per = 4 * K;  // records per singleton: 2K chunks x 2 lanes
  const SegRec *F = stage ? reinterpret_cast<const SegRec *>(stage_recs(rec, per * (int)sizeof(SegRec), ns, recsm))
                          : rec + (long long)i * per;
  FsInc inc = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (i < ns) fixed_step_body(i, sg, reps, st, K, F, W, zmeta, diag_depth, fin_lo, fin_hi, inc, sd, eps_y, mode, zrc);
  const unsigned fm = 0xffffffffu;
  const unsigned nact = __reduce_add_sync(fm, inc.nact), wide = __reduce_add_sync(fm, inc.wide);
  const unsigned hof = __reduce_add_sync(fm, inc.hofixed), hor = __reduce_add_sync(fm, inc.horqc);
  const unsigned it = __reduce_add_sync(fm, inc.iters), li = __reduce_add_sync(fm, inc.light);
  const unsigned qd = __reduce_add_sync(fm, inc.qd), zw = __reduce_add_sync(fm, inc.zw);
  const unsigned dm = __reduce_max_sync(fm, inc.dmax), nl = __reduce_add_sync(fm, inc.nlight);
  if ((threadIdx.x & 31) == 0) {
    if (nact) atomicAdd(nactive, (int)nact);
    if (nl) atomicAdd(nactive + 1, (int)nl);
    if (wide) atomicAdd((unsigned long long *)&stats[ST_SEG_WIDE], (unsigned long long)wide);
    if (hof) atomicAdd((unsigned long long *)&stats[ST_HO_FIXED], (unsigned long long)hof);
    if (hor) atomicAdd((unsigned long long *)&stats[ST_HO_RQC], (unsigned long long)hor);
    if (it) {
      atomicAdd((unsigned long long *)&stats[ST_RQI_ITERS], (unsigned long long)it);
      atomicAdd((unsigned long long *)&stats[ST_GETVEC], (unsigned long long)it);
    }
    if (li) atomicAdd((unsigned long long *)&stats[ST_QD_LIGHT], (unsigned long long)li);
    if (qd) atomicAdd((unsigned long long *)&stats[ST_QD_STEPS], (unsigned long long)qd);
    if (zw) atomicAdd((unsigned long long *)&stats[ST_ZW_STEPS], (unsigned long long)zw);
    if (dm) atomicMax((unsigned long long *)&stats[ST_DMAX], (unsigned long long)dm);
  }
}

// mode of pass p + 1 from pass p's mode and the counts it left (q[3p] singletons active for a stored pass,
// q[3p + 1] for an RQC-only pass, q[3p + 2] the mode): light passes first, then the stored passes of everyone
// waiting, 2 when nothing is left; the host enqueues several passes between its checks
__global__ void k_rqi_mode(int *q, int p) {
  const int m = q[3 * p + 2], a0 = q[3 * p], a1 = q[3 * p + 1];
  q[3 * (p + 1) + 2] = (m == 2) ? 2 : (m == 3) ? 0 : (m == 0) ? (a1 > 0 ? 0 : 1) : (a1 > 0 ? 0 : (a0 > 0 ? 1 : 2));
}

// singletons handed over (status != 1) for the two-lane kernel k_rqi2
__global__ void k_rqi3_collect(const Singleton *__restrict__ sg, int ns, const RqiState *__restrict__ st,
                               Singleton *hand, int *nhand) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ns) return;
  if (st[i].status != 1) hand[atomicAdd(nhand, 1)] = sg[i];
}
