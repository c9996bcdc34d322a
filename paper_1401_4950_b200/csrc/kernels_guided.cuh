// kernels_guided.cuh -- guided rounds of the shared-tree bisection (S5, Alg. Bisection).
//
// The bisection result is fixed by the sequence of decisions NegCount(w) < j at the midpoints w of
// index j's path; any set of evaluated midpoints that contains the path reproduces the sequential
// intervals bit for bit.  A node that holds exactly one eigenvalue (isolated: NegCount(hi) -
// NegCount(lo) = 1) therefore does not need the full k-section subtree: it evaluates the "tube" of
// tree nodes that intersect [est - u, est + u] around an estimate of its eigenvalue, whole levels at a
// time, up to a point budget.  The walker then follows the actual path through the evaluated points;
// where the path leaves the tube (or the budget ends) the node continues next round.  Without an
// estimate (u = inf) the tube is the complete subtree: a k-section.
//
// The estimate is Laguerre's iteration for det(M - sigma I) (all roots real) from the derivatives
// G = f'/f, H = -(f'/f)' that the tube chains accumulate alongside the Sturm recurrence (the
// derivative of s(i) w.r.t. sigma; the chain's reciprocal of d+(i) is reused).  The estimate only
// steers which midpoints are evaluated; it never enters a decision.
#pragma once
#include "kernels.cuh"

// split the node list into k-section nodes (K) and tube nodes (P); P nodes get their point budget in pad
__global__ void k_node_split(const Node *__restrict__ nodes, int nnode, Node *K, int *nK, Node *P, int *nP,
                             int bud_full, int bud_tube) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnode) return;
  Node nd = nodes[i];
  if (node_isolated(nd)) {
    nd.pad = (isinf(nd.u) || isnan(nd.est)) ? bud_full : bud_tube;
    P[atomicAdd(nP, 1)] = nd;
  } else {
    K[atomicAdd(nK, 1)] = nd;
  }
}

__global__ void k_tube_count(const Node *__restrict__ P, int nP, double rtol, int *offs) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nP) return;
  const Node nd = P[i];
  offs[i] = tube_enum(nd, rtol, nd.pad, -1, nullptr);
}

// exclusive scan of offs[0..n) in place, offs[n] = total; *total_out = total (one CTA)
__global__ void __launch_bounds__(1024) k_scan_excl(int *offs, int n, int *total_out) {
  __shared__ int part[1024];
  const int t = threadIdx.x;
  const int chunk = (n + 1023) / 1024;
  const int i0 = t * chunk, i1 = min(i0 + chunk, n);
  int s = 0;
  for (int i = i0; i < i1; i++) s += offs[i];
  part[t] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    int v = (t >= o) ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int run = (t > 0) ? part[t - 1] : 0;
  for (int i = i0; i < i1; i++) {
    int c = offs[i];
    offs[i] = run;
    run += c;
  }
  if (t == 1023) {
    offs[n] = part[1023];
    *total_out = part[1023];
  }
}

// Laguerre step for det(M - sigma I) of degree N from G = f'/f and H = -(f'/f)'
__device__ __forceinline__ double laguerre_est(double sig, double G, double H, double N) {
  if (!isfinite(G) || !isfinite(H)) return NAN;
  double disc = (N - 1.0) * (N * H - G * G);
  disc = sqrt(disc > 0.0 ? disc : 0.0);
  const double den = (G >= 0.0) ? G + disc : G - disc;
  if (den == 0.0) return NAN;
  return sig - N / den;
}

// Walk every tube node along its index's path through the evaluated midpoints; emit the finished
// interval or the node where the path left the tube, with a new estimate from the two deepest points.
__global__ void k_tube_update(const Node *__restrict__ P, int nP, const int *__restrict__ offs,
                              const int *__restrict__ counts, const double *__restrict__ dS,
                              const double *__restrict__ dG, const double *__restrict__ dH,
                              const RepDesc *__restrict__ reps, Node *next, int *nnext, double *out_lo,
                              double *out_hi, double rtol, unsigned long long *alg) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nP) return;
  const Node nd = P[i];
  const int j = nd.b;
  const int base = offs[i];
  const bool full = isinf(nd.u) || isnan(nd.est);
  const double x1 = full ? -INFINITY : __dsub_rn(nd.est, nd.u), x2 = full ? INFINITY : __dadd_rn(nd.est, nd.u);
  double L1 = nd.lo, H1 = nd.hi, L2 = nd.lo, H2 = nd.hi;
  double wl = nd.lo, wu = nd.hi;
  int cum = 0;
  unsigned used = 0;
  double s1 = NAN, G1 = NAN, H1v = NAN, s2 = NAN, G2 = NAN, H2v = NAN;
  for (int l = 0; l < 1100; l++) {
    if (!bis_continue(wl, wu, rtol)) {
      out_lo[nd.obase + j] = wl;
      out_hi[nd.obase + j] = wu;
      if (used) atomicAdd(alg, (unsigned long long)used);
      return;
    }
    if (!bis_continue(L1, H1, rtol) || !bis_continue(L2, H2, rtol)) break;
    const double W = __dsub_rn(H1, L1);
    const double q = __ddiv_rn(__dsub_rn(L2, L1), W);
    if (!(q >= 0.0) || q > (double)nd.pad) break;
    const int cnt = (int)q + 1;
    if (cum + cnt > nd.pad) break;
    if (wl < L1 || wl > L2) break;  // the path left the tube
    const double o = __ddiv_rn(__dsub_rn(wl, L1), W);
    const int idx = cum + (int)o;
    const double w = bis_mid(wl, wu);
    const int c = base + idx;
    if (!(o >= 0.0) || idx >= cum + cnt || __double_as_longlong(dS[c]) != __double_as_longlong(w)) break;
    used++;
    s2 = s1; G2 = G1; H2v = H1v;
    s1 = w; G1 = dG[c]; H1v = dH[c];
    if (counts[c] < j) wl = w;
    else wu = w;
    cum += cnt;
    const double w1 = bis_mid(L1, H1);
    if (x1 >= w1) L1 = w1; else H1 = w1;
    const double w2 = bis_mid(L2, H2);
    if (x2 <= w2) H2 = w2; else L2 = w2;
  }
  if (used) atomicAdd(alg, (unsigned long long)used);
  Node c = nd;
  c.lo = wl;
  c.hi = wu;
  c.est = NAN;
  c.u = INFINITY;
  const double N = (double)reps[nd.rep].nb;
  const double e1 = isnan(s1) ? NAN : laguerre_est(s1, G1, H1v, N);
  if (isfinite(e1) && e1 > wl && e1 < wu) {
    const double e2 = isnan(s2) ? NAN : laguerre_est(s2, G2, H2v, N);
    double u = isfinite(e2) ? 2.0 * fabs(e1 - e2) : 0.25 * fabs(e1 - s1);
    const double fl = 2.0 * N * EPS_X * fabs(e1);
    c.est = e1;
    c.u = fmax(fmax(u, fl), 0x1p-1020);
  }
  next[atomicAdd(nnext, 1)] = c;
}

// ---------------------------------------------------------------------------
// Representation-grouped k-section rounds (child bisection, S8(e)): the nodes of a round are sorted by
// representation so that every CTA evaluates chains of ONE child representation and streams it once
// through shared memory by TMA (instead of every chain reading its own copy from HBM).
// ---------------------------------------------------------------------------
__global__ void k_rep_hist(const Node *__restrict__ nodes, int nnode, int rep0, int *hist) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nnode) atomicAdd(&hist[nodes[i].rep - rep0], 1);
}
__global__ void k_rep_scatter(const Node *__restrict__ nodes, int nnode, int rep0, int *cursor, Node *sorted) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnode) return;
  const Node nd = nodes[i];
  sorted[atomicAdd(&cursor[nd.rep - rep0], 1)] = nd;
}
__global__ void k_rep_ctas(const int *__restrict__ node_off, int nrep, long long P, int *ctas) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nrep) ctas[r] = (int)(((long long)(node_off[r + 1] - node_off[r]) * P + 127) / 128);
}

__global__ void __launch_bounds__(128) k_negcount_grp(const Node *__restrict__ nodes, int m,
                                                      const int *__restrict__ node_off,
                                                      const int *__restrict__ cta_off, int nrep,
                                                      const RepDesc *__restrict__ reps,
                                                      const double2 *__restrict__ mx, int *counts) {
  extern __shared__ __align__(128) unsigned char neg_smem[];
  double2 *buf = reinterpret_cast<double2 *>(neg_smem);
  __shared__ __align__(8) uint64_t bar[2];
  const int b = blockIdx.x;
  int lo = 0, hi = nrep - 1;  // representation r with cta_off[r] <= b < cta_off[r + 1]
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (cta_off[mid] <= b) lo = mid; else hi = mid - 1;
  }
  const int r = lo;
  const long long P = (1LL << m) - 1;
  const long long nc = (long long)(node_off[r + 1] - node_off[r]) * P;
  const long long cr = (long long)(b - cta_off[r]) * 128 + threadIdx.x;
  const bool act = cr < nc;
  const long long crc = act ? cr : nc - 1;
  const long long node = node_off[r] + crc / P;
  const int pt = (int)(crc % P) + 1;
  const Node nd = nodes[node];
  const double sig = node_point(nd, m, pt);
  const RepDesc R = reps[nd.rep];
  const double2 *M = mx + R.off;
  const int nb = R.nb;
  const int ntile = (nb + NEG_TILE - 1) / NEG_TILE;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int t = 0; t < 2 && t < ntile; t++) {
      int len = min(NEG_TILE, nb - t * NEG_TILE);
      tma_load_1d(buf + t * NEG_TILE, M + (long long)t * NEG_TILE, (unsigned)(len * sizeof(double2)), &bar[t]);
    }
  }
  __syncthreads();
  int cnt;
  bool ok;
  double G, H;
  neg_tiles<false>(buf, bar, M, nb, ntile, sig, cnt, ok, G, H);
  if (!ok) cnt = negcount_x_careful(M, nb, sig);
  if (act) counts[node * P + pt - 1] = cnt;
}
