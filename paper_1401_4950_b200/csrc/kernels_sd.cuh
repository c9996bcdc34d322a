// kernels_sd.cuh -- the single/double realisation of the mixed-precision MRRR:
// binary32 input and output, every computation in binary64, gaptol fixed to 1e-5.  The x-path
// kernels (split, root chain, NegCount bisection, classification) are shared with the double/double-double
// solver; the y-representation is binary64 (the dd rows carry zero low words) and these kernels hold the
// steps whose arithmetic changes:
//
//   k_f2d / k_w_d2f / k_z_d2f   "data conversion is only necessary when reading the input and writing the
//                               output": binary32 <-> binary64 at the boundary.
//   k_sd_seg / _combine         S8(c) shift attempts and S8(d) child representations: Alg. dstqds
//                               in binary64 in the operation order of the reference loop (the child data decide
//                               integer outputs, so they must be bit-identical to the oracle's binary64 run):
//                               growth max|d+| and validity per attempt; the child rows d = d+, dl = d l,
//                               dll = dl l and sigma accumulated in binary64.  Segmented chains
//                               with bit-exact junctions (sequential recomputation where a junction fails).
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

// shift of chain t: attempt mode (na > 0): t = (cluster, attempt a0 + ia, side) as in k_clu_attempt_multi; build
// mode (na == 0): t = cluster, tau = its accepted shift
__device__ __forceinline__ double sd_chain_tau(const ShiftState &S, long long t, int a0, int na) {
  if (na == 0) return S.best_tau;
  const int ia = (int)((t >> 1) % na), side = (int)(t & 1);
  double tau = side ? S.taur : S.taul;
  for (int b = a0; b < a0 + ia; b++) tau = side ? __dadd_rn(tau, ldexp(S.offr, b)) : __dsub_rn(tau, ldexp(S.offl, b));
  return tau;
}
__device__ __forceinline__ int sd_chain_cluster(long long t, int na) { return na ? (int)(t / (2 * na)) : (int)t; }

// rows [b, e) of dstqds(M, tau) from state s: growth / validity over the rows, child rows written when yc != 0;
// the last row (b .. e reaching nb-1) adds d+(nb) = s + d(nb).  The parent rows are loaded PF rows ahead into a
// register ring (the recurrence would otherwise wait for every row's L2 / HBM latency)
__device__ __forceinline__ void sd_rows(const YElt *__restrict__ y, int nb, int b, int e, double tau, double &s,
                                        double &g, int &v, YElt *yc, double2 *xc) {
  constexpr int PF = 8;
  double rd[PF], rl[PF], rll[PF];
  auto ld = [&](int i, int u) {
    const int ii = min(i, nb - 1);
    rd[u] = __ldg(&y[ii].d_hi);
    rl[u] = __ldg(&y[ii].dl_hi);
    rll[u] = __ldg(&y[ii].dll_hi);
  };
  auto row = [&](int i, double d, double dl, double dll) {
    double dp, lp;
    sd_dstqds_row(s, d, dl, dll, tau, dp, lp);
    v &= !(isnan(dp) || isnan(lp));
    g = dmaxd(g, fabs(dp));
    if (yc) {
      const double dlc = __dmul_rn(dp, lp), dllc = __dmul_rn(dlc, lp);
      YElt el;
      el.d_hi = dp; el.d_lo = 0.0; el.dl_hi = dlc; el.dl_lo = 0.0; el.dll_hi = dllc; el.dll_lo = 0.0;
      yc[i] = el;
      xc[i] = make_double2(dp, dllc);
    }
  };
#pragma unroll
  for (int u = 0; u < PF; u++) ld(b + u, u);
  int i = b;
  for (; i + PF <= e; i += PF) {
#pragma unroll
    for (int u = 0; u < PF; u++) {
      const double d = rd[u], dl = rl[u], dll = rll[u];
      ld(i + u + PF, u);
      row(i + u, d, dl, dll);
    }
  }
#pragma unroll
  for (int u = 0; u < PF; u++)
    if (i + u < e) row(i + u, rd[u], rl[u], rll[u]);
  if (e == nb - 1) {
    const double dn = __dadd_rn(s, __ldg(&y[nb - 1].d_hi));
    v &= !isnan(dn);
    g = dmaxd(g, fabs(dn));
    if (yc) {
      YElt el;
      el.d_hi = dn; el.d_lo = 0.0; el.dl_hi = el.dl_lo = el.dll_hi = el.dll_lo = 0.0;
      yc[nb - 1] = el;
      xc[nb - 1] = make_double2(dn, 0.0);
    }
  }
}

// build mode: the child representation descriptor (rep id repbase + c, rows at poolbase + c * nbmax), sigma =
// fl64(sigma_parent + tau); no valid shift: nb = -1 (members go back to the parent as singletons, as in the
// double/dd path)
__device__ __forceinline__ void sd_child_desc(const Cluster *__restrict__ cl, int c, RepDesc *reps,
                                              const ShiftState &S, int repbase, long long poolbase, int nbmax) {
  const RepDesc P = reps[cl[c].rep];
  RepDesc R = P;
  R.off = poolbase + (long long)c * nbmax;
  R.depth = P.depth + 1;
  R.sig_hi = __dadd_rn(P.sig_hi, S.best_tau);
  R.sig_lo = 0.0;
  if (!S.have_best) R.nb = -1;
  reps[repbase + c] = R;
}

// S8(c)/(d) as segmented chains: chain t's rows 0..nb-2 in K segments, segment k started Wu rows early from the
// guess q = 1 (s = dll(w0-1) - tau); it records its entry state at its first row and its exit state, and is
// accepted by k_sd_seg_combine only if the entry equals the predecessor's exit bit for bit (then it applied
// every operation to the sequential operands; otherwise the chain is recomputed sequentially there).
// Thread = (segment k, chain t), chains fastest: a warp runs one segment of 32 chains (shared parent rows).
struct SegSD {
  double s_in, s_out, g;
  int valid, empty;
};
__global__ void __launch_bounds__(128) k_sd_seg(const Cluster *__restrict__ cl, const RepDesc *__restrict__ reps,
                                                const YElt *__restrict__ my, const ShiftState *__restrict__ ss,
                                                long long T, int a0, int na, int K, int Wu, SegSD *seg,
                                                double2 *mx, YElt *myc, long long poolbase, int nbmax) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= T * K) return;
  const long long t = g % T;
  const int k = (int)(g / T);
  SegSD *o = seg + t * K + k;
  const int c = sd_chain_cluster(t, na);
  const ShiftState S = ss[c];
  if ((na && S.done) || (!na && !S.have_best)) { o->empty = 1; return; }
  const RepDesc R = reps[cl[c].rep];
  const int nb = R.nb, steps = nb - 1;
  int bk, ek, w0;
  if (steps >= 2 * K * Wu) {
    const int L = (steps + K - 1) / K;
    bk = min(k * L, steps);
    ek = min(bk + L, steps);
    w0 = (k == 0) ? 0 : max(bk - Wu, 0);
  } else {
    if (k > 0) { o->empty = 1; return; }
    bk = 0; ek = steps; w0 = 0;
  }
  const double tau = sd_chain_tau(S, t, a0, na);
  const YElt *y = my + R.off;
  double s = (w0 == 0) ? -tau : __dsub_rn(__ldg(&y[w0 - 1].dll_hi), tau);
  double gg = 0.0;
  int v = 1;
  sd_rows(y, nb, w0, bk, tau, s, gg, v, nullptr, nullptr);  // warm-up (no growth / validity, bk < nb - 1)
  gg = 0.0;
  v = 1;
  o->s_in = s;
  const long long off = poolbase + (long long)c * nbmax;
  sd_rows(y, nb, bk, ek, tau, s, gg, v, na ? nullptr : myc + off, na ? nullptr : mx + off);
  o->s_out = s;
  o->g = gg;
  o->valid = v;
  o->empty = 0;
}
// junctions of chain t; accepted: growth / validity (attempts) or the descriptor (build); else the chain is
// recomputed sequentially (and its child rows rewritten)
__global__ void k_sd_seg_combine(const Cluster *__restrict__ cl, RepDesc *reps, const YElt *__restrict__ my,
                                 const ShiftState *__restrict__ ss, long long T, int a0, int na, int K,
                                 const SegSD *__restrict__ seg, double *gval, int *valid, double2 *mx, YElt *myc,
                                 int repbase, long long poolbase, int nbmax, int *nfb) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int c = sd_chain_cluster(t, na);
  const ShiftState S = ss[c];
  if (na && S.done) return;
  if (!na) {
    sd_child_desc(cl, c, reps, S, repbase, poolbase, nbmax);
    if (!S.have_best) return;
  }
  const SegSD *R = seg + t * K;
  bool good = true;
  double gg = 0.0;
  int v = 1, prev = -1;
  for (int k = 0; k < K && good; k++) {
    const SegSD &a = R[k];
    if (a.empty) continue;
    good = prev < 0 || __double_as_longlong(a.s_in) == __double_as_longlong(R[prev].s_out);
    gg = dmaxd(gg, a.g);
    v &= a.valid;
    prev = k;
  }
  if (!good) {
    atomicAdd(nfb, 1);
    const RepDesc P = reps[cl[c].rep];
    const double tau = sd_chain_tau(S, t, a0, na);
    const long long off = poolbase + (long long)c * nbmax;
    double s = -tau;
    gg = 0.0;
    v = 1;
    sd_rows(my + P.off, P.nb, 0, P.nb - 1, tau, s, gg, v, na ? nullptr : myc + off, na ? nullptr : mx + off);
  }
  if (na) {
    gval[t] = gg;
    valid[t] = v;
  }
}
