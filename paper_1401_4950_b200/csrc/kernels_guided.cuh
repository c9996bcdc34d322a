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

// ---------------------------------------------------------------------------
// Segmented x-NegCount (latency splitting, bit-exact).  The stationary recurrence of Alg. negcountLDL,
// s(i+1) = s(i) dll(i) / (d(i) + s(i)) - sigma, is strongly contracting on a positive definite root
// (a perturbation of s(i) is multiplied by l+(i)^2): started W rows early from a guess, a segment's
// trajectory becomes BIT-IDENTICAL to the true one within far fewer than W rows.  So a chain is split
// into K segments evaluated concurrently: segment k (k >= 1) runs rows [b_k - W, b_k) from the guess
// s = -sigma without counting, records its state s_in at row b_k, then counts rows [b_k, b_{k+1}) and
// records s_out.  k_seg_combine accepts segment k only if s_in(k) equals, bit for bit, s_out(k-1) of an
// accepted predecessor -- then every operation of the segment was applied to the same operands as in the
// sequential recurrence, and its count is exact.  A chain with a mismatch (or a division that left the
// fast range) is finished from the last exact state with the IEEE operations (seg_chain_count).
// The count is therefore identical to the sequential NegCount in every case; only the latency changes
// (rows per lane: (nb-1)/K + W instead of nb-1).
// ---------------------------------------------------------------------------
struct SegOut {
  double s_in, s_out;
  int cnt, ok;
};

// Staged rows per tile: 2 x 512 rows x 16 B = 16 KB per CTA, so that the register limit (64 per thread: 8 CTAs of
// 128 threads per SM) and not shared memory bounds residency -- a round's grid then fits in one wave of
// 148 x 8 CTAs (with 1024-row tiles, 33 KB per CTA, only 6 fit and a 1024-CTA round ran 1.15 waves)
#ifndef SEG_TILE
#define SEG_TILE 512
#endif
// CH chains per thread (chains c0 + j * 128 of the CTA's 128 * CH): the CTA's chains all run segment k
// over the same staged rows, so a thread interleaves CH independent recurrences on one shared-memory
// row load (instruction-level parallelism where a round has few chains, fewer loads per step)
template <int CH>
__global__ void __launch_bounds__(128) k_negcount_seg(const Node *__restrict__ nodes, int nnode, int m,
                                                      const ExplicitChain *__restrict__ ex, int nex,
                                                      const RepDesc *__restrict__ reps,
                                                      const double2 *__restrict__ mx, int K, int L, int Wu,
                                                      SegOut *seg, const int *__restrict__ dnn, int mmax,
                                                      long long target) {
  extern __shared__ __align__(128) unsigned char neg_smem[];
  double2 *buf = reinterpret_cast<double2 *>(neg_smem);  // [2][SEG_TILE]
  __shared__ __align__(8) uint64_t bar[2];
  if (dnn) {  // device-driven round: node count and depth from the previous round
    nnode = *dnn;
    m = round_m(nnode, mmax, target);
  }
  const long long nn = (long long)nnode * ((1 << m) - 1);
  const long long tot = nn + nex;
  // 1-D grid, segment index fastest: the live CTAs are the first ones dispatched (device-driven rounds
  // launch a grid sized for the largest possible round; its idle tail exits without delaying them)
  const long long cb = (long long)(blockIdx.x / K) * blockDim.x * CH;
  if (cb >= tot) return;  // whole CTA idle (uniform exit)
  const int k = blockIdx.x % K;
  double sig[CH];
  bool act[CH];
  int rep = 0;
#pragma unroll
  for (int j = 0; j < CH; j++) {
    const long long c = cb + threadIdx.x + j * blockDim.x;
    act[j] = c < tot;
    double sj;
    int rj;
    chain_of(nodes, m, nn, ex, act[j] ? c : tot - 1, sj, rj);
    sig[j] = sj;
    rep = rj;
  }
  const RepDesc R = reps[rep];  // one representation for the whole launch (root)
  const int nb = R.nb;
  const double2 *M = mx + R.off;
  const int bk = min(k * L, nb - 1), ek = (k == K - 1) ? nb - 1 : min((k + 1) * L, nb - 1);
  const int w0 = (k == 0) ? 0 : max(bk - Wu, 0);
  const int r1 = (k == K - 1) ? nb : ek;  // staged rows [w0, r1): the last segment also stages row nb-1
  const int nrow = r1 - w0;
  const int ntile = (nrow + SEG_TILE - 1) / SEG_TILE;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int t = 0; t < 2 && t < ntile; t++) {
      int len = min(SEG_TILE, nrow - t * SEG_TILE);
      tma_load_1d(buf + t * SEG_TILE, M + w0 + (long long)t * SEG_TILE, (unsigned)(len * sizeof(double2)), &bar[t]);
    }
  }
  __syncthreads();
  double s[CH], s_in[CH];
  int cnt[CH];
  bool ok = true;
#pragma unroll
  for (int j = 0; j < CH; j++) {
    s[j] = -sig[j];
    s_in[j] = -sig[j];
    cnt[j] = 0;
  }
  for (int t = 0; t < ntile; t++) {
    const int b = t & 1;
    mbar_wait(&bar[b], (unsigned)((t >> 1) & 1));
    const double2 *T = buf + b * SEG_TILE;
    const int row0 = w0 + t * SEG_TILE;
    const int len = min(SEG_TILE, ek - row0);  // recurrence steps in this tile (rows < ek)
    int kk = 0;
    // warm-up rows (before bk): no counting
    const int nw = max(0, min(len, bk - row0));
#pragma unroll 4
    for (; kk < nw; kk++) {
      const double2 mm = T[kk];
#pragma unroll
      for (int j = 0; j < CH; j++) {
        const double dp = __dadd_rn(mm.x, s[j]);
        const double q = div_fast_nocheck(s[j], dp);
        ok &= div_range_ok(s[j], dp, q);
        s[j] = __dsub_rn(__dmul_rn(q, mm.y), sig[j]);
      }
    }
    if (row0 + kk == bk) {
#pragma unroll
      for (int j = 0; j < CH; j++) s_in[j] = s[j];
    }
#pragma unroll 8
    for (; kk < len; kk++) {
      const double2 mm = T[kk];
#pragma unroll
      for (int j = 0; j < CH; j++) {
        const double dp = __dadd_rn(mm.x, s[j]);
        const double q = div_fast_nocheck(s[j], dp);
        ok &= div_range_ok(s[j], dp, q);
        s[j] = __dsub_rn(__dmul_rn(q, mm.y), sig[j]);
        cnt[j] += (int)((unsigned)__double2hiint(dp) >> 31);
      }
    }
    if (k == K - 1 && t == ntile - 1) {
      const double dl = T[nb - 1 - row0].x;
#pragma unroll
      for (int j = 0; j < CH; j++) cnt[j] += sbx(__dadd_rn(dl, s[j]));
    }
    __syncthreads();
    if (threadIdx.x == 0 && t + 2 < ntile) {
      int len2 = min(SEG_TILE, nrow - (t + 2) * SEG_TILE);
      tma_load_1d(buf + b * SEG_TILE, M + w0 + (long long)(t + 2) * SEG_TILE, (unsigned)(len2 * sizeof(double2)),
                  &bar[b]);
    }
  }
#pragma unroll
  for (int j = 0; j < CH; j++) {
    if (bk == w0) s_in[j] = -sig[j];  // no warm-up (k = 0): the exact start
    if (act[j]) {
      SegOut o;
      o.s_in = s_in[j];
      o.s_out = s[j];
      o.cnt = cnt[j];
      o.ok = ok ? 1 : 0;  // one flag for the thread's chains: a failed range test sends both to the careful tail
      seg[(cb + threadIdx.x + j * blockDim.x) * K + k] = o;
    }
  }
}

// accept segments along the verified chain of exact states; queue the rest for the careful tail
// verified count of chain c from its K segment records; a chain whose junctions do not all verify is
// finished here with the careful IEEE operations from its last exact state (rare)
__device__ __forceinline__ int seg_chain_count(const SegOut *__restrict__ seg, int K, long long c,
                                               const Node *__restrict__ nodes, int m, long long nn,
                                               const ExplicitChain *__restrict__ ex,
                                               const RepDesc *__restrict__ reps, const double2 *__restrict__ mx,
                                               int L, int *nfb) {
  const SegOut *S = seg + c * K;
  int total = 0, k = 0;
  double s_exact = S[0].s_in;  // -sigma
  if ((K & 7) == 0) {  // batches of eight records loaded before their part of the junction walk (the loads of a
    bool run = true;   // one-at-a-time walk are a chain of dependent misses: 32 segments cost ~20 us per round)
    for (int k0 = 0; k0 < K && run; k0 += 8) {
      SegOut o[8];
#pragma unroll
      for (int u = 0; u < 8; u++) o[u] = S[k0 + u];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        run = run && o[u].ok && (k0 + u == 0 || __double_as_longlong(o[u].s_in) == __double_as_longlong(s_exact));
        if (run) {
          total += o[u].cnt;
          s_exact = o[u].s_out;
          k = k0 + u + 1;
        }
      }
    }
  } else {
    for (; k < K; k++) {
      const SegOut o = S[k];
      if (!o.ok) break;
      if (k > 0 && __double_as_longlong(o.s_in) != __double_as_longlong(s_exact)) break;
      total += o.cnt;
      s_exact = o.s_out;
    }
  }
  if (k == K) return total;
  double sig;
  int rep;
  chain_of(nodes, m, nn, ex, c, sig, rep);
  const RepDesc R = reps[rep];
  const double2 *M = mx + R.off;
  const int nb = R.nb;
  double s = s_exact;
  int cnt = total;
  // re-run the failed segment k exactly from the last exact state; where the state it reaches equals, bit for
  // bit, the next segment's recorded entry state, that segment saw the sequential operands: take its count and
  // exit state and walk on (near an eigenvalue only the segments past the eigenvector's peak, where the forward
  // recurrence expands, fail -- the rest of the chain need not be re-run)
  while (k < K) {
    const int bk = min(k * L, nb - 1), ek = (k == K - 1) ? nb - 1 : min((k + 1) * L, nb - 1);
    for (int r = bk; r < ek; r++) {
      const double2 mm = M[r];
      const double dp = __dadd_rn(mm.x, s);
      const double q = (isinf(s) && isinf(dp)) ? 1.0 : __ddiv_rn(s, dp);
      s = __dsub_rn(__dmul_rn(q, mm.y), sig);
      cnt += sbx(dp);
    }
    k++;
    while (k < K) {
      const SegOut o = S[k];
      if (!o.ok || __double_as_longlong(o.s_in) != __double_as_longlong(s)) break;
      cnt += o.cnt;  // the last segment's record includes the final row's term
      s = o.s_out;
      k++;
      if (k == K) { atomicAdd(nfb, 1); return cnt; }
    }
  }
  cnt += sbx(__dadd_rn(M[nb - 1].x, s));
  atomicAdd(nfb, 1);
  return cnt;
}
__global__ void k_seg_combine(long long tot, long long nn, int K, const SegOut *__restrict__ seg, int *counts,
                              int *excounts, int *nfb, const int *__restrict__ dnn, int mmax, long long target,
                              long long *negx, const Node *__restrict__ nodes, int nnode, int m,
                              const ExplicitChain *__restrict__ ex, const RepDesc *__restrict__ reps,
                              const double2 *__restrict__ mx, int L) {
  if (dnn) {
    nnode = *dnn;
    m = round_m(nnode, mmax, target);
    nn = (long long)nnode * ((1 << m) - 1);
    tot = nn;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd((unsigned long long *)negx, (unsigned long long)tot);
  }
  long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= tot) return;
  const int cnt = seg_chain_count(seg, K, c, nodes, m, nn, ex, reps, mx, L, nfb);
  if (c < nn) counts[c] = cnt;
  else excounts[c - nn] = cnt;
}
// One segmented round's bookkeeping in one launch: thread per node counts the node's 2^m - 1 chains
// (junction walk) and then runs the shared-tree update for the node's 2^m leaves (rounds without
// explicit chains; host- or device-driven)
__global__ void k_seg_round(int nnode, int m, int K, const SegOut *__restrict__ seg, int *counts,
                            const Node *__restrict__ nodes, const RepDesc *__restrict__ reps,
                            const double2 *__restrict__ mx, int L, Node *next, int *nnext, double *out_lo,
                            double *out_hi, double rtol, unsigned long long *alg, int *nmulti, int *nfb,
                            const int *__restrict__ dnn, int mmax, long long target, long long *negx) {
  if (dnn) {
    nnode = *dnn;
    m = round_m(nnode, mmax, target);
    if (blockIdx.x == 0 && threadIdx.x == 0)
      atomicAdd((unsigned long long *)negx, (unsigned long long)((long long)nnode * ((1 << m) - 1)));
  }
  const long long P = (1LL << m) - 1, nn = (long long)nnode * P;
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= nnode) return;
  for (long long j = 0; j < P; j++) counts[id * P + j] = seg_chain_count(seg, K, id * P + j, nodes, m, nn, nullptr,
                                                                         reps, mx, L, nfb);
  for (int p = 0; p < (1 << m); p++)
    bisect_update_body((id << m) + p, nodes, nnode, m, counts, next, nnext, out_lo, out_hi, rtol, alg, nmulti);
}


// ---------------------------------------------------------------------------
// Segmented y-NegCount (q-form, dd): thread (segment k, chain c) runs rows [bk, ek) of chain c after a
// warm-up of Wu rows from the no-coupling guess; consecutive threads are consecutive chains on the same
// segment (on one representation their row loads coincide).  Chains too short for K segments run whole
// in segment 0.  k_seg_combine_y accepts a chain iff every junction state is bit-identical to its
// predecessor's exit (then the count equals the sequential negcount_y_q's); the rest are recounted whole.
// ---------------------------------------------------------------------------
struct SegOutY {
  double in_hi, in_lo, out_hi, out_lo;
  int cnt, ok, empty, pad;
};
__global__ void __launch_bounds__(128) k_negcount_seg_y(const Node *__restrict__ nodes, int nnode, int m,
                                                        const ExplicitChain *__restrict__ ex, int nex,
                                                        const RepDesc *__restrict__ reps, const QElt *__restrict__ mq,
                                                        int K, int Wu, SegOutY *seg) {
  const long long nn = (long long)nnode * ((1 << m) - 1), tot = nn + nex;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= tot * K) return;
  const int k = (int)(g / tot);
  const long long c = g % tot;
  double sig;
  int rep;
  chain_of(nodes, m, nn, ex, c, sig, rep);
  const RepDesc R = reps[rep];
  const int nb = R.nb, steps = nb - 1;
  SegOutY *o = seg + c * K + k;
  int bk, ek, w0;
  if (steps >= 2 * K * Wu) {
    const int L = (steps + K - 1) / K;
    bk = min(k * L, steps);
    ek = min(bk + L, steps);
    w0 = (k == 0) ? 0 : max(bk - Wu, 0);
  } else {
    if (k > 0) {
      o->empty = 1;
      o->ok = 1;
      return;
    }
    bk = 0;
    ek = steps;
    w0 = 0;
  }
  const dd sigma = dd_from(sig);
  const double2 *p = reinterpret_cast<const double2 *>(mq + R.off);
  const double2 gb0 = __ldg(p + 4 * w0 + 3);
  dd den = dd_sub_nf(dd_make(gb0.x, gb0.y), sigma);  // gb(w0) - sigma: exact at row 0, a guess elsewhere
  dd din = den;
  int cnt = 0;
  bool ok = true;
  double2 c2n = __ldg(p + 4 * w0), gn = __ldg(p + 4 * w0 + 2);
  for (int i = w0; i < ek; i++) {
    const double2 c2v = c2n, gv = gn;
    const int in = min(i + 1, nb - 1);
    c2n = __ldg(p + 4 * in);
    gn = __ldg(p + 4 * in + 2);
    if (i == bk) din = den;
    if (i >= bk) cnt += dd_sb(den);
    den = y_step(den, c2v, gv, sigma, ok);
  }
  if (ek == steps) cnt += dd_sb(den);  // den(nb-1) closes the count
  o->in_hi = din.hi;
  o->in_lo = din.lo;
  o->out_hi = den.hi;
  o->out_lo = den.lo;
  o->cnt = cnt;
  o->ok = (ok && isfinite(den.hi) && isfinite(den.lo)) ? 1 : 0;
  o->empty = 0;
}
__global__ void k_seg_combine_y(long long tot, long long nn, int K, const SegOutY *__restrict__ seg, int *counts,
                                int *excounts, long long *fb, int *nfb) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= tot) return;
  const SegOutY *S = seg + c * K;
  int total = 0, prev = -1;
  bool good = true;
  for (int k = 0; k < K && good; k++) {
    const SegOutY &o = S[k];
    if (o.empty) continue;
    good = o.ok != 0;
    if (good && prev >= 0)
      good = __double_as_longlong(o.in_hi) == __double_as_longlong(S[prev].out_hi) &&
             __double_as_longlong(o.in_lo) == __double_as_longlong(S[prev].out_lo);
    total += o.cnt;
    prev = k;
  }
  if (good) {
    if (c < nn) counts[c] = total;
    else excounts[c - nn] = total;
    return;
  }
  fb[atomicAdd(nfb, 1)] = c;
}
__global__ void k_seg_fallback_y(const long long *__restrict__ fb, const int *__restrict__ nfb,
                                 const Node *__restrict__ nodes, int nnode, int m,
                                 const ExplicitChain *__restrict__ ex, const RepDesc *__restrict__ reps,
                                 const QElt *__restrict__ mq, const YElt *__restrict__ my, int *counts,
                                 int *excounts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *nfb) return;
  const long long c = fb[i], nn = (long long)nnode * ((1 << m) - 1);
  double sig;
  int rep;
  chain_of(nodes, m, nn, ex, c, sig, rep);
  const RepDesc R = reps[rep];
  const int cnt = negcount_y_q(mq + R.off, my + R.off, R.nb, dd_from(sig));
  if (c < nn) counts[c] = cnt;
  else excounts[c - nn] = cnt;
}

// ---------------------------------------------------------------------------
// Segmented x-NegCount for launches whose chains evaluate many representations (child bisection):
// thread (segment k, chain c), per-thread loads with PF rows in flight, the step of negcount_x_fast
// (division fast path, sticky range test).  k_seg_combine_xg accepts a chain iff every junction state
// is bit-identical to its predecessor's exit; the rest are recounted whole by negcount_x_fast (which
// reruns the careful IEEE chain if its own range test fails), so counts equal negcount_x's.
// ---------------------------------------------------------------------------
struct SegOutX {
  double in, out;
  int cnt, ok, empty, pad;
};
// one segment of k_negcount_seg_xg with the IEEE quotient at every step (q_ieee): used for sigma = +-0, where the
// state stays a signed zero that the fast sequence's range test rejects (every segment would fail its junction
// and the whole chain would rerun sequentially)
__device__ __noinline__ void seg_xg_exact(const double2 *__restrict__ M, int nb, int steps, int w0, int bk, int ek,
                                          double sig, SegOutX *o) {
  double s = -sig, s_in = -sig;
  int cnt = 0;
  for (int i = w0; i < ek; i++) {
    if (i == bk) s_in = s;
    const double2 mm = __ldg(M + i);
    const double dp = __dadd_rn(mm.x, s);
    s = __dsub_rn(__dmul_rn(q_ieee(s, dp), mm.y), sig);
    if (i >= bk) cnt += sbx(dp);
  }
  if (ek == steps) cnt += sbx(__dadd_rn(__ldg(M + nb - 1).x, s));
  o->in = s_in;
  o->out = s;
  o->cnt = cnt;
  o->ok = 1;
  o->empty = 0;
}
__global__ void __launch_bounds__(128) k_negcount_seg_xg(const Node *__restrict__ nodes, int nnode, int m,
                                                         const ExplicitChain *__restrict__ ex, int nex,
                                                         const RepDesc *__restrict__ reps,
                                                         const double2 *__restrict__ mx, int K, int Wu,
                                                         SegOutX *seg) {
  constexpr int PF = 8;
  const long long nn = (long long)nnode * ((1 << m) - 1), tot = nn + nex;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= tot * K) return;
  const int k = (int)(g / tot);
  const long long c = g % tot;
  double sig;
  int rep;
  chain_of(nodes, m, nn, ex, c, sig, rep);
  const RepDesc R = reps[rep];
  const int nb = R.nb, steps = nb - 1;
  SegOutX *o = seg + c * K + k;
  int bk, ek, w0;
  if (steps >= 2 * K * Wu) {
    const int L = (steps + K - 1) / K;
    bk = min(k * L, steps);
    ek = min(bk + L, steps);
    w0 = (k == 0) ? 0 : max(bk - Wu, 0);
  } else {
    if (k > 0) {
      o->empty = 1;
      o->ok = 1;
      return;
    }
    bk = 0;
    ek = steps;
    w0 = 0;
  }
  const double2 *M = mx + R.off;
  if (sig == 0.0) {  // (rare: the first midpoint of a child interval symmetric about 0) exact IEEE steps
    seg_xg_exact(M, nb, steps, w0, bk, ek, sig, o);
    return;
  }
  double s = -sig, s_in = -sig;
  int cnt = 0;
  bool ok = true;
  double2 ring[PF];
#pragma unroll
  for (int u = 0; u < PF; u++) ring[u] = __ldg(M + min(w0 + u, nb - 1));
  auto step = [&](int i, double2 mm) {
    if (i == bk) s_in = s;
    const double dp = __dadd_rn(mm.x, s);
    const double q = div_fast_nocheck(s, dp);
    ok &= div_range_ok(s, dp, q);
    s = __dsub_rn(__dmul_rn(q, mm.y), sig);
    if (i >= bk) cnt += (int)((unsigned)__double2hiint(dp) >> 31);
  };
  int i = w0;
  for (; i + PF <= ek; i += PF) {
#pragma unroll
    for (int u = 0; u < PF; u++) {
      const double2 mm = ring[u];
      ring[u] = __ldg(M + min(i + u + PF, nb - 1));
      step(i + u, mm);
    }
  }
#pragma unroll
  for (int u = 0; u < PF; u++)
    if (i + u < ek) step(i + u, ring[u]);
  if (ek == steps) cnt += sbx(__dadd_rn(__ldg(M + nb - 1).x, s));
  o->in = s_in;
  o->out = s;
  o->cnt = cnt;
  o->ok = (ok && !isnan(s)) ? 1 : 0;
  o->empty = 0;
}
struct FbX {
  long long c;
  double s;   // last exact state: entering segment k's first row
  int k, cnt;  // first unverified segment, count of the verified rows before it
};
__global__ void k_seg_combine_xg(long long tot, long long nn, int K, const SegOutX *__restrict__ seg, int *counts,
                                 int *excounts, FbX *fb, int *nfb, long long *stats) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= tot) return;
  const SegOutX *S = seg + c * K;
  int total = 0, prev = -1, k = 0;
  for (; k < K; k++) {
    const SegOutX &o = S[k];
    if (o.empty) continue;
    if (!o.ok) break;
    if (prev >= 0 && __double_as_longlong(o.in) != __double_as_longlong(S[prev].out)) break;
    total += o.cnt;
    prev = k;
  }
  if (k == K) {
    if (c < nn) counts[c] = total;
    else excounts[c - nn] = total;
    return;
  }
  FbX f;
  f.c = c;
  f.s = (prev >= 0) ? S[prev].out : S[0].in;  // S[0].in = -sigma (exact start)
  f.k = (prev >= 0) ? k : 0;
  f.cnt = (prev >= 0) ? total : 0;
  fb[atomicAdd(nfb, 1)] = f;
  atomicAdd((unsigned long long *)&stats[ST_XG_FB], 1ull);
}
// careful (IEEE) evaluation from the first unverified segment's first row with the last exact state, re-joining
// the recorded segments: after running a segment exactly, the next segment's result is taken over as soon as its
// recorded entry state equals the exact one bit for bit (then it saw the sequential operands); only the segments
// whose warm-up did not converge are re-run (one or two per chain instead of the whole tail)
__global__ void k_seg_fallback_xg(const FbX *__restrict__ fb, const int *__restrict__ nfb,
                                  const Node *__restrict__ nodes, int nnode, int m,
                                  const ExplicitChain *__restrict__ ex, const RepDesc *__restrict__ reps,
                                  const double2 *__restrict__ mx, int K, int Wu, int *counts, int *excounts,
                                  const SegOutX *__restrict__ seg, long long *stats) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *nfb) return;
  const FbX f = fb[i];
  const long long nn = (long long)nnode * ((1 << m) - 1);
  double sig;
  int rep;
  chain_of(nodes, m, nn, ex, f.c, sig, rep);
  const RepDesc R = reps[rep];
  const double2 *M = mx + R.off;
  const int nb = R.nb, steps = nb - 1;
  const bool segd = steps >= 2 * K * Wu;
  const int L = segd ? (steps + K - 1) / K : steps;
  const SegOutX *S = seg + f.c * K;
  double s = f.s;
  int cnt = f.cnt;
  // the IEEE operations, with the verified division fast path where its range test passes (bit-identical);
  // the child representation streams from HBM: PF rows in flight
  constexpr int PF = 8;
  auto step = [&](double2 mm) {
    const double dp = __dadd_rn(mm.x, s);
    double q = div_fast_nocheck(s, dp);
    if (!div_range_ok(s, dp, q))
      q = (s == 0.0 && dp != 0.0 && !isnan(dp)) ? __dmul_rn(s, copysign(1.0, dp))  // exact signed zero
          : (isinf(s) && isinf(dp))             ? 1.0
                                                : __ddiv_rn(s, dp);
    s = __dsub_rn(__dmul_rn(q, mm.y), sig);
    cnt += sbx(dp);
  };
  auto run_rows = [&](int r0, int r1) {  // steps on rows [r0, r1)
    double2 ring[PF];
#pragma unroll
    for (int u = 0; u < PF; u++) ring[u] = __ldg(M + min(r0 + u, nb - 1));
    int r = r0;
    for (; r + PF <= r1; r += PF) {
#pragma unroll
      for (int u = 0; u < PF; u++) {
        const double2 mm = ring[u];
        ring[u] = __ldg(M + min(r + u + PF, nb - 1));
        step(mm);
      }
    }
#pragma unroll
    for (int u = 0; u < PF; u++)
      if (r + u < r1) step(ring[u]);
  };
  int k = f.k;
  if (!segd) {
    run_rows(0, steps);
  } else {
    while (k < K) {
      const int bk = min(k * L, steps), ek = min(bk + L, steps);
      run_rows(bk, ek);  // segment k exactly
      atomicAdd((unsigned long long *)&stats[ST_XG_FBSEG], 1ull);
      k++;
      // re-join: take over every following segment whose entry state is the exact one
      while (k < K) {
        const SegOutX o = S[k];
        if (o.empty) { k++; continue; }
        if (!o.ok || __double_as_longlong(o.in) != __double_as_longlong(s)) break;
        cnt += o.cnt;  // (the segment that ends at the last step also counted the final row)
        s = o.out;
        const int ekk = min(min(k * L, steps) + L, steps);
        k++;
        if (ekk == steps) {
          if (f.c < nn) counts[f.c] = cnt;
          else excounts[f.c - nn] = cnt;
          return;
        }
      }
    }
  }
  cnt += sbx(__dadd_rn(__ldg(M + nb - 1).x, s));
  if (f.c < nn) counts[f.c] = cnt;
  else excounts[f.c - nn] = cnt;
}

// ---------------------------------------------------------------------------
// Segmented shift attempts (Alg. spectrumshift step 3): the growth max|d+| of dstqds(M_y, tau) for every
// (cluster, attempt, side) chain, split into K verified segments like the y-count (the fast q-form step
// y_step is shared with dstqds_growth, so a verified chain gives its growth bit for bit); chains that do
// not verify are recomputed whole by dstqds_growth.
// ---------------------------------------------------------------------------
struct SegG {
  double in_hi, in_lo, out_hi, out_lo, gmax;
  int ok, empty;
};
__device__ __forceinline__ double attempt_tau(const ShiftState &S, int a0, int ia, int side) {
  double tau = side ? S.taur : S.taul;
  for (int b = a0; b < a0 + ia; b++) tau = side ? __dadd_rn(tau, ldexp(S.offr, b)) : __dsub_rn(tau, ldexp(S.offl, b));
  return tau;
}
__global__ void __launch_bounds__(128) k_clu_attempt_seg(const Cluster *__restrict__ cl, int ncl,
                                                         const RepDesc *__restrict__ reps,
                                                         const QElt *__restrict__ mq,
                                                         const ShiftState *__restrict__ ss, int a0, int na, int K,
                                                         int Wu, SegG *seg) {
  const long long T = 2LL * na * ncl;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= T * K) return;
  const int k = (int)(g / T);
  const long long t = g % T;
  const int c = (int)(t / (2 * na)), ia = (int)((t >> 1) % na), side = (int)(t & 1);
  const ShiftState S = ss[c];
  SegG *o = seg + t * K + k;
  if (S.done) {
    o->empty = 1;
    o->ok = 1;
    return;
  }
  const dd tau = dd_from(attempt_tau(S, a0, ia, side));
  const RepDesc R = reps[cl[c].rep];
  const int nb = R.nb, steps = nb - 1;
  int bk, ek, w0;
  if (steps >= 2 * K * Wu) {
    const int L = (steps + K - 1) / K;
    bk = min(k * L, steps);
    ek = min(bk + L, steps);
    w0 = (k == 0) ? 0 : max(bk - Wu, 0);
  } else {
    if (k > 0) {
      o->empty = 1;
      o->ok = 1;
      return;
    }
    bk = 0;
    ek = steps;
    w0 = 0;
  }
  const double2 *p = reinterpret_cast<const double2 *>(mq + R.off);
  const double2 gb0 = __ldg(p + 4 * w0 + 3);
  dd den = dd_sub(dd_make(gb0.x, gb0.y), tau);  // dstqds_growth's start (exact at row 0, a guess elsewhere)
  dd din = den;
  double gm = 0.0;
  bool ok = true;
  double2 c2n = __ldg(p + 4 * w0), gn = __ldg(p + 4 * w0 + 2);
  for (int i = w0; i < ek; i++) {
    const double2 c2v = c2n, gv = gn;
    const int in = min(i + 1, nb - 1);
    c2n = __ldg(p + 4 * in);
    gn = __ldg(p + 4 * in + 2);
    if (i == bk) din = den;
    if (i >= bk) gm = dmaxd(gm, fabs(den.hi));
    den = y_step(den, c2v, gv, tau, ok);
  }
  if (ek == steps) {
    ok &= isfinite(den.hi) && isfinite(den.lo);
    gm = dmaxd(gm, fabs(den.hi));
  }
  o->in_hi = din.hi;
  o->in_lo = din.lo;
  o->out_hi = den.hi;
  o->out_lo = den.lo;
  o->gmax = gm;
  o->ok = ok ? 1 : 0;
  o->empty = 0;
}
__global__ void k_clu_attempt_combine(const Cluster *__restrict__ cl, int ncl, const RepDesc *__restrict__ reps,
                                      const YElt *__restrict__ my, const QElt *__restrict__ mq,
                                      const ShiftState *__restrict__ ss, int a0, int na, int K,
                                      const SegG *__restrict__ seg, double *gval, int *valid) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2LL * na * ncl) return;
  const int c = (int)(t / (2 * na)), ia = (int)((t >> 1) % na), side = (int)(t & 1);
  const ShiftState S = ss[c];
  if (S.done) return;
  const SegG *R = seg + t * K;
  double g = 0.0;
  int prev = -1;
  bool good = true;
  for (int k = 0; k < K && good; k++) {
    const SegG &a = R[k];
    if (a.empty) continue;
    good = a.ok != 0 && (prev < 0 || (__double_as_longlong(a.in_hi) == __double_as_longlong(R[prev].out_hi) &&
                                      __double_as_longlong(a.in_lo) == __double_as_longlong(R[prev].out_lo)));
    g = dmaxd(g, a.gmax);
    prev = k;
  }
  if (good) {
    gval[t] = g;
    valid[t] = 1;
    return;
  }
  const RepDesc Rp = reps[cl[c].rep];
  double gg;
  int v;
  dstqds_growth(my + Rp.off, mq + Rp.off, Rp.nb, attempt_tau(S, a0, ia, side), gg, v);
  gval[t] = gg;
  valid[t] = v;
}

// Segmented child build (S8(d)): thread (segment k, cluster c) runs the fast pass of clu_build_one over rows
// [bk, ek) after a warm-up and writes those child rows; k_clu_build_combine verifies the junctions and
// rebuilds the clusters that do not verify whole (clu_build_one), so the child representation is bit for
// bit the sequential one.  Records: SegG (gmax unused).
#ifndef MRRR_BG
#define MRRR_BG 4
#endif
constexpr int BG = MRRR_BG;  // child rows per bulk store in k_clu_build_seg
__global__ void __launch_bounds__(128) k_clu_build_seg(const Cluster *__restrict__ cl, int ncl,
                                                       const RepDesc *__restrict__ reps,
                                                       const ShiftState *__restrict__ ss, double2 *mx, YElt *my,
                                                       const QElt *__restrict__ mq, long long poolbase, int nbmax,
                                                       int K, int Wu, SegG *seg) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  // a warp whose 32 threads all exist decides below, with all its lanes, whether it stores cooperatively
  const bool warp_full = (g | 31) < (long long)ncl * K;
  if (g >= (long long)ncl * K) return;
  const int k = (int)(g / ncl), c = (int)(g % ncl);
  const ShiftState S = ss[c];
  SegG *o = seg + (long long)c * K + k;
  const RepDesc P = reps[cl[c].rep];
  const int nb = P.nb, steps = nb - 1;
  int bk = 0, ek = steps, w0 = 0;
  bool live = S.have_best != 0;
  if (steps >= 2 * K * Wu) {
    const int L = (steps + K - 1) / K;
    bk = min(k * L, steps);
    ek = min(bk + L, steps);
    w0 = (k == 0) ? 0 : max(bk - Wu, 0);
  } else if (k > 0) {
    live = false;
  }
  bool coop = false;
  if (warp_full) {  // every lane reaches these collectives (no lane has returned yet)
    const int bk0 = __shfl_sync(0xffffffffu, bk, 0), ek0 = __shfl_sync(0xffffffffu, ek, 0);
    coop = __all_sync(0xffffffffu, live && bk0 == bk && ek0 == ek);
  }
  if (!live) {
    o->empty = 1;
    o->ok = 1;
    return;
  }
  const long long off = poolbase + (long long)c * nbmax;
  YElt *yc = my + off;
  double2 *xc = mx + off;
  const dd tau = dd_from(S.best_tau);
  const QElt *q = mq + P.off;
  dd den = dd_sub(dd_make(__ldg(&q[w0].gb_hi), __ldg(&q[w0].gb_lo)), tau);
  dd din = den;
  bool ok = true;
  // rows prefetched PFB ahead in a register ring (the parent rows are shared by the warp's lanes, L2-resident)
  constexpr int PFB = 4;
  QRow ring[PFB];
#pragma unroll
  for (int u = 0; u < PFB; u++) ring[u] = ld_qrow(q, min(w0 + u, steps - 1));
  int slot = 0;
  auto next_row = [&](int i) -> QRow {  // row i's data; refills its slot with row i + PFB
    QRow cur = ring[0];
#pragma unroll
    for (int u = 0; u < PFB; u++) if (u == slot) cur = ring[u];
    const QRow nx = ld_qrow(q, min(i + PFB, steps - 1));
#pragma unroll
    for (int u = 0; u < PFB; u++) if (u == slot) ring[u] = nx;
    slot = (slot + 1 == PFB) ? 0 : slot + 1;
    return cur;
  };
  for (int i = w0; i < bk; i++) den = clu_build_row_v(den, next_row(i), i, tau, nullptr, nullptr, ok, false);
  din = den;
  // the rows are staged in shared memory and written by bulk (TMA-engine) copies of BG-row runs: a warp's lanes
  // are different clusters, so plain stores scattered 32 partial lines per instruction (store-bound: C3's child
  // build moved 8.6 GB at 0.66 TB/s)
  extern __shared__ __align__(16) unsigned char bsm[];
  YElt *sy = reinterpret_cast<YElt *>(bsm) + threadIdx.x * 2 * BG;
  double2 *sx = reinterpret_cast<double2 *>(bsm + (size_t)blockDim.x * 2 * BG * sizeof(YElt)) + threadIdx.x * 2 * BG;
  int grp = 0, ng = 0;
  // a full warp on one row range (the usual case: 32 sibling clusters of one frame length on segment k) stores
  // cooperatively: every 2 BG rows, one 16-byte store per lane writes one cluster's 2 BG YElt rows (6 BG chunks)
  // and its 2 BG x-rows (2 BG chunks) -- 32 contiguous runs per 32 store instructions instead of 64 small
  // bulk copies per lane (those ran the 8.6 GB of C3's child rows at 1.7 TB/s)
  const int lane = threadIdx.x & 31;
  constexpr int CG = 2 * BG;  // rows per cooperative store (the two staging groups as one buffer)
  if (coop) {
    const long long offl0 = poolbase + (long long)c * nbmax;
    for (int i = bk; i < ek; i++) {
      den = clu_build_row_v(den, next_row(i), i, tau, sy + ng, sx + ng, ok, true);
      if (++ng == CG || i + 1 == ek) {
        const int low = i - ng + 1;
        __syncwarp();
        const int ny = 3 * ng;  // 16-byte chunks of the YElt rows (48 B each); then ng chunks of x-rows
        for (int l = 0; l < 32; l++) {
          const long long offl = __shfl_sync(0xffffffffu, offl0, l);
          const double2 *src_y = reinterpret_cast<const double2 *>(sy - (lane - l) * 2 * BG);
          const double2 *src_x = sx - (lane - l) * 2 * BG;
          if (lane < ny) reinterpret_cast<double2 *>(my + offl + low)[lane] = src_y[lane];
          else if (lane < ny + ng) (mx + offl + low)[lane - ny] = src_x[lane - ny];
        }
        __syncwarp();
        ng = 0;
      }
    }
  } else {
    for (int i = bk; i < ek; i++) {
      den = clu_build_row_v(den, next_row(i), i, tau, sy + grp * BG + ng, sx + grp * BG + ng, ok, true);
      if (++ng == BG || i + 1 == ek) {
        const int low = i - ng + 1;
        bulk_store(yc + low, sy + grp * BG, (unsigned)(ng * sizeof(YElt)));
        bulk_store(xc + low, sx + grp * BG, (unsigned)(ng * sizeof(double2)));
        grp ^= 1;
        ng = 0;
        bulk_wait_read<2>();  // the other group's two stores have read their rows
      }
    }
    bulk_wait_all();
  }
  if (ek == steps) {
    ok &= isfinite(den.hi) && isfinite(den.lo);
    YElt e;
    e.d_hi = den.hi; e.d_lo = den.lo; e.dl_hi = e.dl_lo = e.dll_hi = e.dll_lo = 0.0;
    yc[nb - 1] = e;
    xc[nb - 1] = make_double2(den.hi, 0.0);
  }
  o->in_hi = din.hi;
  o->in_lo = din.lo;
  o->out_hi = den.hi;
  o->out_lo = den.lo;
  o->ok = ok ? 1 : 0;
  o->empty = 0;
}
__global__ void k_clu_build_combine(const Cluster *__restrict__ cl, int ncl, RepDesc *reps,
                                    const ShiftState *__restrict__ ss, double2 *mx, YElt *my,
                                    const QElt *__restrict__ mq, int repbase, long long poolbase, int nbmax, int K,
                                    const SegG *__restrict__ seg, int *nfb) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
  const ShiftState S = ss[c];
  bool good = S.have_best;
  const SegG *R = seg + (long long)c * K;
  int prev = -1;
  for (int k = 0; k < K && good; k++) {
    const SegG &a = R[k];
    if (a.empty) continue;
    good = a.ok != 0 && (prev < 0 || (__double_as_longlong(a.in_hi) == __double_as_longlong(R[prev].out_hi) &&
                                      __double_as_longlong(a.in_lo) == __double_as_longlong(R[prev].out_lo)));
    prev = k;
  }
  if (good) {  // rows are in place: the representation descriptor (as clu_build_one writes it)
    const RepDesc P = reps[cl[c].rep];
    RepDesc Rc = P;
    Rc.off = poolbase + (long long)c * nbmax;
    Rc.depth = P.depth + 1;
    const dd sig = dd_add_d(dd_make(P.sig_hi, P.sig_lo), S.best_tau);
    Rc.sig_hi = sig.hi;
    Rc.sig_lo = sig.lo;
    reps[repbase + c] = Rc;
    return;
  }
  if (S.have_best) atomicAdd(nfb, 1);
  clu_build_one(c, cl, reps, ss, mx, my, mq, repbase, poolbase, nbmax);  // whole (also the failed-shift case)
}
