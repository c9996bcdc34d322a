// mrrr.cu -- host orchestrator and C ABI of libmrrr.so (include/mrrr.h).
// Sequencing of DESIGN.md S0-S10 on one CUDA stream; every numerical step is
// a kernel from kernels.cuh / kernels_vec.cuh.  Host code only sizes
// workspace, launches, and reads back small counters that size the next
// launch (node / group / cluster counts).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is opened at run time (mrrr_eig_dist)

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mrrr.h"
#include "kernels.cuh"
#include "kernels_vec.cuh"
#include "kernels_rqi.cuh"
#include "kernels_guided.cuh"
#include "kernels_rqi3.cuh"
#include "kernels_sd.cuh"

namespace {

thread_local std::string g_last_cuda_error = "no error";
thread_local std::string g_last_nccl_error = "no error";

struct Buf {
  void *p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) { p = nullptr; return e; }
    cap = want;
    return cudaSuccess;
  }
  // grow to >= bytes keeping the first `keep` bytes (stream-ordered copy)
  cudaError_t grow_keep(size_t bytes, size_t keep, cudaStream_t st) {
    if (bytes <= cap) return cudaSuccess;
    void *q = nullptr;
    cudaError_t e = cudaMalloc(&q, bytes);
    if (e != cudaSuccess) return e;
    if (p && keep) {
      e = cudaMemcpyAsync(q, p, std::min(keep, cap), cudaMemcpyDeviceToDevice, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) { cudaFree(q); return e; }
    }
    if (p) cudaFree(p);
    p = q;
    cap = bytes;
    return cudaSuccess;
  }
  void release() { if (p) cudaFree(p); p = nullptr; cap = 0; }
  template <class T> T *as() const { return reinterpret_cast<T *>(p); }
};

struct Err {
  int code;
};

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t _e = (x);                                                                  \
    if (_e != cudaSuccess) {                                                               \
      g_last_cuda_error = std::string(#x) + ": " + cudaGetErrorString(_e);                 \
      throw Err{_e == cudaErrorMemoryAllocation ? MRRR_ERR_NOMEM : MRRR_ERR_CUDA};         \
    }                                                                                      \
  } while (0)

inline unsigned nblocks_for(long long n, int bs) { return (unsigned)std::max<long long>(1, (n + bs - 1) / bs); }

// counters block on the device: reset/readback in one copy
enum { C_NNEXT = 0, C_NEX, C_NPEND, C_NREADY, C_NSING, C_NCLUS, C_NNXT, C_NDONE, C_NK, C_NP, C_NPC, C_NFB,
       C_NMULTI, C_NACT, C_NLIGHT, C_NCOUNTERS = 16 };

}  // namespace

struct mrrr_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  double gaptol = 1e-10;
  uint64_t seed = 0x4D52525233ULL;
  int root_side = 0;
  uint32_t flags = 0;
  long long ws_limit = 0;
  long long target_chains = 16384;  // k-section budget per round, segmented root chains (C2: 1 level per round)
  long long target_y = 8192;    // k-section budget of the (segmented) y-count rounds (less speculation)
  long long target_chains_small = 8192;  // ... when fewer than 4096 indices are wanted (a rank's shard)
  long long target_unseg = 32768;   // k-section budget per round of whole-length root chains (C1: 3-4 levels)
  long long target_child = 8192;    // ... of child-frame rounds (less speculation on long child chains)
  int mmax = 16;
  bool neg_tma = true;  // x-NegCount with TMA-staged representation tiles (k_negcount_tma)
  bool grouped = true;  // child bisection with CTAs grouped by representation (k_negcount_grp)
  int seg_k = 8, seg_w = 128;  // segmented root NegCount: segments per chain, warm-up rows (k_negcount_seg)
  bool zrc_child = true;       // ... also for child frames (MRRR_ZRC_CHILD=0: stored passes there)
  int zwin = 256;              // z recompute window of singletons accepted on an RQC-only pass (0: stored passes)
  int fuse_mmax = 2;           // host-driven segmented rounds fuse walk + update (k_seg_round) up to this depth
  bool rqi_seg = true;         // segmented RQI passes (kernels_rqi3.cuh); MRRR_RQISEG=0: the two-lane kernel only
  int rqi_segk = 8, rqi_segw = 0;  // rqi_segw 0: by frame length (128 up to 16K rows, else 192)
  long long rqi_threads = 131072;  // adaptive RQI segment count target (threads per segmented pass)
  bool rqi_seg_child = true;   // segmented RQI for child-frame singletons (dd twist search)
  int segchild_min = 8;        // ... when the level has at least this many singletons per child representation
  // deferred tails: a child level whose singletons go to the two-lane kernel only (few singletons per child) runs
  // it on a side stream while the levels above finish (MRRR_DEFER_TAIL=0: in order on the solve stream)
  bool defer_tail = true;
  bool synccheck = false;  // MRRR_SYNCCHECK: synchronise after every launch check (fault localisation)
  long long tail_max_bytes = 1LL << 30;  // largest two-lane workspace a deferred tail may hold (3 dd planes)
  cudaStream_t s_tail = nullptr;
  cudaEvent_t ev_tail_in = nullptr, ev_tail_done = nullptr;
  bool tail_pending = false;
  long long twdd_root_max = 0;  // root blocks up to this size take the dd twist search (MRRR_TWDD_ROOT)
  bool rqi_bulk = true;        // k_fixed_chunk stores the factors by bulk copies of staged 8-row runs
  int segy_k = 16, segy_w = 128;  // segmented y-NegCount, shift growth, child build (MRRR_SEGYK=1: unsegmented)
  int segx_k = 16, segx_w = 128;  // segmented many-representation x-NegCount (child rounds with long chains)
  long long cur_nbmax = 0;       // longest representation of the current child bisection (0: segx off)
  bool stage_attr = false, rec_stage = false;  // record staging in shared memory (MRRR_RECSTAGE=1; slower on C2)
  size_t stage_lim = 0;
  long long seg_ch2 = 0;  // segmented rounds with at most this many chains run two chains per thread (slower on C2)
  long long seg_threads = 262144;  // adaptive segment count: more segments while a round has fewer threads
  int seg_minlen = 512;            // ... and the segments stay this long (long chains: C5b, a rank's C5a shard)
  int dev_frac = 0;            // ... once the indices still sharing nodes are at most 1/dev_frac of the nodes (0: by n)
  bool dev_stable = true;      // device-driven rounds once every node holds one index (exact grids)
  bool round_ev = true;  // per-round timing events of the device-driven rounds (MRRR_ROUNDEV=0: ~2.7 us less per
                         // event on C2, 5.49 -> 5.33 ms, but no per-launch kernel time for the roofline)
  long long es2_target = 4096;  // early stop, stage 2: k-section budget (C2: 2 levels per round; measured
  int es2_minlen = 256;          // 16384 -> 4096 and 512 -> 256-row segments: 2.89 -> 2.53 ms)  (MRRR_ES2_*)
  int dev_rb = 16;            // rounds per device-driven batch (32: empty tail rounds cost a rank's short run)
  bool dev_rounds = false;     // segmented rounds enqueued in batches on device-side counters (MRRR_DEVROUNDS=1;
                               // slower on C2: the oversized early-exit grids cost more than the saved syncs)
  int max_nodes = 0;           // bound on live bisection nodes (indices in the computed set)  // tube point budgets: no estimate (4 full levels) / with estimate
  bool l2_persist = true;
  long long rqi_seg_min = 2048; // root blocks up to this size skip the segmented RQI (MRRR_RQISEGMIN)
  bool bmerge = true;            // start nodes sharing a start interval bisected as one node (MRRR_BMERGE=0: off)
  bool nonlocal = false;         // this solve's root rounds found non-contracting recurrences (see run_bisection)
  bool sd = false;             // this solve runs the single/double realisation (mrrr_seig)
  double gaptol_sd = 1e-5;     // its fixed gaptol
  int segsd_k = 32;            // segments per binary64 dstqds chain (shift attempts, child builds; MRRR_SEGSDK)
  int fault = 0;               // MRRR_FAULT: fault injection for the GPU tests (k_rqi2: bit 0 fallback, bit 1 careful)
  long long l2_max_window = 0;

  // buffers
  Buf starts, scal, binfo, bside, blist, cab, mx, my, mq, lscratch, reps, rlo, rhi, colmap, gstart;
  Buf s1lo, s1hi, esr;  // early classification stop (S5'): stage-1 intervals, decision ranges
  Buf rqmode;           // segmented RQI: per-pass counters and mode (k_rqi_mode)
  Buf nodesK, nodesP, offsP, dS, dG, dH;  // guided bisection rounds
  Buf zinb, zrcb;                         // z recompute window: lane states; rerun counter, mode, scratch
  Buf repoff, repcur, repcta;             // representation-grouped rounds
  Buf segout, rnd;                        // segmented NegCount; per-round device counters
  Buf gpart;                              // k_root_gersh partial bounds
  Buf tail_ws, tail_sing, tail_zmeta;     // deferred tail: two-lane planes, its singleton list, its z metadata
  static constexpr int LVL_MAX = 64;      // per-level cluster lists and singleton copies (kept across solves: a
  Buf lvl_L[LVL_MAX], lvl_NX[LVL_MAX], lvl_SG[LVL_MAX];  // cudaFree would wait for a deferred tail)
  Buf segouty, segfby, segoutx, segoutg;  // segmented y-NegCount / many-representation x-NegCount / growth
  Buf rqst, rqrec, hand;                  // segmented RQI state, segment records, handed-over singletons
  Buf nodesA, nodesB, counts, ex, excounts, exmap, bnA, bnB, sing, clusA, clusB, ss, gval, valid, cseg, bnoff,
      ipool_lo, ipool_hi, yref_lo, yref_hi, wsA, wsB, stats, cnt, ddepth, dgf, dgl, dflo, dfhi, hd, he, hW, hZ, zmeta,
      hd2, sdin, sdW, sdZ, sdhin, sdhW, sdhZ, segsd;
  int *h_cnt = nullptr;  // pinned counters
  int *h_small = nullptr;  // pinned scratch for the small device-to-host reads of a solve (64 ints)
  std::vector<int> h_rounds = std::vector<int>(258);  // node counts of the device-driven rounds

  // results of the last call
  long long last_n = 0, last_k = 0;
  int last_nblk = 0;
  long long stats_h[ST_N] = {0};
  double times[12] = {0};
  std::vector<int> h_starts;
  cudaEvent_t ev[8];
  ncclComm_t comm = nullptr;   // mrrr_eig_dist communicator (created on first use)
  char comm_id[128] = {0};
  int comm_rank = -1, comm_world = 0;
  Buf dWl, dmeta, dmetas, dpad, dparts;  // mrrr_eig_dist staging
  double rqi_ms = 0, neg_ms = 0;
  // kernel timing without host round trips: event pairs recorded on the stream during the solve, read only when
  // mrrr_get_times asks (cudaEventElapsedTime between rounds left the GPU idle: ~4 us per call, 30 per C2 solve)
  std::vector<cudaEvent_t> tev;
  int ntev = 0;
  std::vector<std::pair<int, int>> tneg, trq;
  bool times_dirty = false;
  long long neg_launches = 0, neg_len = 0;
  long long rqi_launches = 0;
  long long host_rounds = 0, host_launches = 0;
};

namespace {

void read_counters(mrrr_t h) {
  CK(cudaMemcpyAsync(h->h_cnt, h->cnt.p, C_NCOUNTERS * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
}
void zero_counters(mrrr_t h) { CK(cudaMemsetAsync(h->cnt.p, 0, C_NCOUNTERS * sizeof(int), h->stream)); }

__global__ void k_fill(double *p, long long n, double v) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}
__global__ void k_fill_i(int *p, long long n, int v) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}
__global__ void k_colmap_range(int *colmap, long long n, long long lo1, long long hi1) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) colmap[i] = (i + 1 >= lo1 && i + 1 <= hi1) ? (int)(i + 1 - lo1) : -1;
}

// root start nodes + end verification chains (S5)
__global__ void k_root_nodes(const int *__restrict__ blist, int nbl, const int *__restrict__ starts,
                             const double *__restrict__ binfo, const int *__restrict__ cab, Node *nodes,
                             ExplicitChain *ex) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nbl) return;
  int blk = blist[t];
  int s = starts[blk], nb = starts[blk + 1] - s;
  const double *bi = binfo + 16 * blk;
  double P = bi[4];
  bool left = bi[6] == 1.0;
  Node nd;
  nd.lo = left ? 0.0 : -P;
  nd.hi = left ? P : 0.0;
  nd.a = 0; nd.b = nb;
  nd.wlo = cab[2 * blk]; nd.whi = cab[2 * blk + 1];
  nd.rep = blk; nd.pad = 0;
  nd.obase = (long long)s - 1;
  nd.est = NAN; nd.u = INFINITY;
  nodes[t] = nd;
  ex[t] = ExplicitChain{left ? P : -P, blk, 0};
}

// guard-extension batches of the single block: one start node per side with indices [w[2k], w[2k+1]]
__global__ void k_guard_nodes(const int *__restrict__ starts, const double *__restrict__ binfo, int w0, int w1,
                              int w2, int w3, Node *nodes) {
  const int t = threadIdx.x;
  const int wlo = t ? w2 : w0, whi = t ? w3 : w1;
  const int nb = starts[1] - starts[0];
  const double P = binfo[4];
  const bool left = binfo[6] == 1.0;
  Node nd;
  nd.lo = left ? 0.0 : -P;
  nd.hi = left ? P : 0.0;
  nd.a = 0; nd.b = nb;
  nd.wlo = wlo; nd.whi = whi;
  nd.rep = 0; nd.pad = 0;
  nd.obase = (long long)starts[0] - 1;
  nd.est = NAN; nd.u = INFINITY;
  nodes[t] = nd;
}

// verification of NegCount at the far root end; doubles P where it fails; flags a restart
__global__ void k_root_verify(const int *__restrict__ blist, int nbl, const int *__restrict__ starts, double *binfo,
                              const int *__restrict__ excounts, int *restart) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nbl) return;
  int blk = blist[t];
  int nb = starts[blk + 1] - starts[blk];
  double *bi = binfo + 16 * blk;
  bool left = bi[6] == 1.0;
  bool ok = left ? (excounts[t] == nb) : (excounts[t] == 0);
  if (!ok) { bi[4] = 2.0 * bi[4]; atomicAdd(restart, 1); }
}

// guard extension test on the root intervals of block 0 (single-block subsets)
__global__ void k_guard_check(const int *__restrict__ cab, const double *__restrict__ rlo,
                              const double *__restrict__ rhi, int nb, double gaptol, int *need) {
  int ca = cab[0], cb = cab[1];
  // positions: index j at j-1 (single block starts at 0)
  need[0] = (ca > 1 && !is_boundary(rlo[ca - 1], rhi[ca - 1], rlo[ca], rhi[ca], gaptol)) ? 1 : 0;
  need[1] = (cb < nb && !is_boundary(rlo[cb - 2], rhi[cb - 2], rlo[cb - 1], rhi[cb - 1], gaptol)) ? 1 : 0;
}

// the guard-extension rule over already computed indices (single block, positions j-1): left, from ca while
// index ca is not separated from ca+1 step outward (not below lo_far); right likewise from cb (not above hi_far)
__global__ void k_guard_scan(int *cab, int lo_far, int hi_far, const double *__restrict__ rlo,
                             const double *__restrict__ rhi, int nb, double gaptol) {
  int ca = cab[0], cb = cab[1];
  while (ca > 1 && ca > lo_far && !is_boundary(rlo[ca - 1], rhi[ca - 1], rlo[ca], rhi[ca], gaptol)) ca--;
  while (cb < nb && cb < hi_far && !is_boundary(rlo[cb - 2], rhi[cb - 2], rlo[cb - 1], rhi[cb - 1], gaptol)) cb++;
  cab[0] = ca;
  cab[1] = cb;
}

// S5' early classification stop (sec. 3.2.2 remark (3) P:3204-3210; A-41; oracle
// stage1_one/stage2_one): index j of a block (2 <= j <= nb-1) keeps its stage-1 interval (rtol_c) when both
// neighbour pairs are classification boundaries and its width is at most 2^-7 of its absolute gap
__device__ __forceinline__ bool es_stop(const double *__restrict__ s1lo, const double *__restrict__ s1hi, long long i,
                                        int j, int nb, double gaptol) {
  if (j < 2 || j > nb - 1) return false;
  const double llo = s1lo[i - 1], lhi = s1hi[i - 1], clo = s1lo[i], chi = s1hi[i], rlo = s1lo[i + 1], rhi = s1hi[i + 1];
  if (!is_boundary(llo, lhi, clo, chi, gaptol) || !is_boundary(clo, chi, rlo, rhi, gaptol)) return false;
  const double gap = dmind(__dsub_rn(clo, lhi), __dsub_rn(rlo, chi));
  return __dsub_rn(chi, clo) <= ldexp(gap, -7);
}
// one thread per index of the ranges rng[r] = {block, ja, jb, offset} (1-based within the block, offsets
// prefix-summed): stopped indices take their stage-1 interval; the continuing ones form one stage-2 node per
// run of consecutive continuing indices sharing a stage-1 interval (a stage-1 node holding several indices)
struct EsRange { int blk, ja, jb, off; };
__global__ void k_es_decide(const EsRange *__restrict__ rng, int nr, int total, const int *__restrict__ starts,
                            const double *__restrict__ s1lo, const double *__restrict__ s1hi, double *rlo,
                            double *rhi, double gaptol, Node *nodes, int *nnode, long long *stats) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  bool stop = false;
  if (t < total) {
    int lo = 0, hi = nr - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (rng[mid].off <= t) lo = mid; else hi = mid - 1;
    }
    const EsRange R = rng[lo];
    const int s = starts[R.blk], nb = starts[R.blk + 1] - s;
    const int j = R.ja + (t - R.off);
    const long long i = (long long)s + j - 1;
    stop = es_stop(s1lo, s1hi, i, j, nb, gaptol);
    if (stop) {
      rlo[i] = s1lo[i];
      rhi[i] = s1hi[i];
    } else {
      auto same = [&](long long x, long long y) {
        return __double_as_longlong(s1lo[x]) == __double_as_longlong(s1lo[y]) &&
               __double_as_longlong(s1hi[x]) == __double_as_longlong(s1hi[y]);
      };
      const bool start = !(j > R.ja && same(i - 1, i) && !es_stop(s1lo, s1hi, i - 1, j - 1, nb, gaptol));
      if (start) {
        int je = j;
        while (je < R.jb && same(i, i + (je + 1 - j)) && !es_stop(s1lo, s1hi, i + (je + 1 - j), je + 1, nb, gaptol)) je++;
        Node nd;
        nd.lo = s1lo[i];
        nd.hi = s1hi[i];
        nd.a = j - 1; nd.b = je;
        nd.wlo = j; nd.whi = je;
        nd.rep = R.blk; nd.pad = 0;
        nd.obase = (long long)s - 1;
        nd.est = NAN; nd.u = INFINITY;
        nodes[atomicAdd(nnode, 1)] = nd;
      }
    }
  }
  const unsigned ns = __reduce_add_sync(0xffffffffu, stop ? 1u : 0u);
  if ((threadIdx.x & 31) == 0 && ns) atomicAdd((unsigned long long *)&stats[ST_ESTOP], (unsigned long long)ns);
}

// multi-block ranking of T-frame midpoints (S4/S6): rank = #{keys before mine}
__global__ void k_rank(const double *__restrict__ d, const int *__restrict__ starts, int nblk,
                       const double *__restrict__ binfo, const double *__restrict__ rlo,
                       const double *__restrict__ rhi, long long n, double *keys) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int lo = 0, hi = nblk - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (starts[mid] <= i) lo = mid; else hi = mid - 1;
  }
  int blk = lo;
  int nbk = starts[blk + 1] - starts[blk];
  keys[i] = (nbk == 1) ? d[i] : __dadd_rn(bis_mid(rlo[i], rhi[i]), binfo[16 * blk]);
}
// multi-block selection (S4/S6): the global rank of position i is its place in the order of (key, position),
// found by a bitonic sort of (key, position) pairs padded to a power of two N2 (O(N2 log^2 N2) work instead of
// the O(n^2) all-pairs count).  Stages with partner distance j >= BT/2 run one global pass per (k, j); all
// smaller distances of a stage run in one shared-memory pass over BT-element tiles.
constexpr int BT = 2048;  // elements per shared-memory tile (1024 threads)
__device__ __forceinline__ bool rank_before(double ka, long long ia, double kb, long long ib) {
  return ka < kb || (ka == kb && ia < ib);
}
__global__ void k_rank_init(const double *__restrict__ keys, long long n, long long N2, double *sk, long long *si) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N2) return;
  sk[i] = (i < n) ? keys[i] : INFINITY;
  si[i] = i;
}
__device__ __forceinline__ void bitonic_cmp(double *sk, long long *si, long long a, long long b, bool up) {
  const double ka = sk[a], kb = sk[b];
  const long long ia = si[a], ib = si[b];
  if (rank_before(kb, ib, ka, ia) == up) {
    sk[a] = kb; sk[b] = ka;
    si[a] = ib; si[b] = ia;
  }
}
__global__ void k_bitonic_global(double *sk, long long *si, long long N2, long long k, long long j) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N2 / 2) return;
  const long long a = (t / j) * 2 * j + (t % j), b = a + j;
  bitonic_cmp(sk, si, a, b, (a & k) == 0);
}
// substages j = jmax .. 1 of stage k (jmax < BT) on one BT-element tile in shared memory
__global__ void __launch_bounds__(BT / 2) k_bitonic_tile(double *sk, long long *si, long long N2, long long k0,
                                                         long long k1, long long jmax) {
  __shared__ double tk[BT];
  __shared__ long long ti[BT];
  const long long base = (long long)blockIdx.x * BT;
  for (int u = threadIdx.x; u < BT; u += blockDim.x) { tk[u] = sk[base + u]; ti[u] = si[base + u]; }
  __syncthreads();
  // stages k = k0, 2 k0, .., k1 (each from its own jmax); the first stage starts at jmax
  for (long long k = k0; k <= k1; k <<= 1) {
    for (long long j = (k == k0) ? jmax : k / 2; j >= 1; j >>= 1) {
      const int t = threadIdx.x;
      const int a = (int)((t / j) * 2 * j + (t % j)), b = a + (int)j;
      const bool up = ((base + a) & k) == 0;
      const double ka = tk[a], kb = tk[b];
      const long long ia = ti[a], ib = ti[b];
      if (rank_before(kb, ib, ka, ia) == up) {
        tk[a] = kb; tk[b] = ka;
        ti[a] = ib; ti[b] = ia;
      }
      __syncthreads();
    }
  }
  for (int u = threadIdx.x; u < BT; u += blockDim.x) { sk[base + u] = tk[u]; si[base + u] = ti[u]; }
}
__global__ void k_rank_scatter(const long long *__restrict__ si, long long n, long long il, long long iu, int *colmap) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const long long rank = p + 1;
  colmap[si[p]] = (rank >= il && rank <= iu) ? (int)(rank - il) : -1;
}

// self-test 1: div_fast/div_ieee vs __ddiv_rn on random bit patterns (wide exponent range) and specials
__global__ void k_selftest_div(long long n, uint64_t seed, unsigned long long *bad) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t z1 = seed + (2 * i + 1) * 0x9E3779B97F4A7C15ull, z2 = seed + (2 * i + 2) * 0x9E3779B97F4A7C15ull;
  z1 = (z1 ^ (z1 >> 30)) * 0xBF58476D1CE4E5B9ull; z1 = (z1 ^ (z1 >> 27)) * 0x94D049BB133111EBull; z1 ^= z1 >> 31;
  z2 = (z2 ^ (z2 >> 30)) * 0xBF58476D1CE4E5B9ull; z2 = (z2 ^ (z2 >> 27)) * 0x94D049BB133111EBull; z2 ^= z2 >> 31;
  double a, b;
  if (i % 4 == 0) {  // raw bit patterns: every exponent, subnormals, inf, nan
    a = __longlong_as_double((long long)z1);
    b = __longlong_as_double((long long)z2);
  } else {           // the NegCount regime: O(1) magnitudes with random signs and scales
    a = ((double)(z1 >> 11) * 0x1p-53 - 0.5) * ldexp(1.0, (int)(z1 & 63) - 32);
    b = ((double)(z2 >> 11) * 0x1p-53 - 0.5) * ldexp(1.0, (int)(z2 & 63) - 32);
    if ((i & 255) == 1) b = 0.0;
    if ((i & 255) == 2) a = 0.0;
    if ((i & 255) == 3) b = -0.0;
    if ((i & 255) == 5) { a = INFINITY; b = -INFINITY; }
  }
  if (i % 4 == 1) {  // near-midpoint quotients: a = RN(b * (m +- half an ulp)) +- a few ulps
    b = __longlong_as_double((long long)((z2 & 0x000FFFFFFFFFFFFFull) | (0x3FFull << 52)));
    double mq = __longlong_as_double((long long)((z1 & 0x000FFFFFFFFFFFFFull) | (0x3FFull << 52)));
    mq = __dadd_rn(mq, ((z1 >> 7) & 1) ? 0x1p-53 : -0x1p-53);
    a = __longlong_as_double(__double_as_longlong(__dmul_rn(b, mq)) + (long long)((z2 >> 5) % 5) - 2);
  }
  double q1 = div_ieee(a, b), q2 = __ddiv_rn(a, b);
  bool same = (__double_as_longlong(q1) == __double_as_longlong(q2)) || (isnan(q1) && isnan(q2));
  double q3 = div_fast_nocheck(a, b);  // the NegCount / root variant: must agree whenever its range test passes
  if (div_range_ok(a, b, q3) && __double_as_longlong(q3) != __double_as_longlong(q2) && !(isnan(q3) && isnan(q2)))
    same = false;
  if (!same) atomicAdd(bad, 1ull);
}

// base segment count of the segmented root rounds for a chain of nb rows: seg_k when a segment spans at least
// 2 warm-ups, else 1 (whole chains).  Short chains are not cut further: C1's 1-2-1 recurrence does not contract
// (no localisation), so its segments never verify (measured: 3 segments at n = 1000 fell back, 6x slower).
int seg_base_k(mrrr_t h, long long nb) {
  return (nb - 1) >= 2LL * h->seg_k * h->seg_w ? h->seg_k : 1;
}

void launch_check(mrrr_t h, int line = __builtin_LINE()) {
  h->host_launches++;
  CK(cudaGetLastError());
  if (h->synccheck) {  // MRRR_SYNCCHECK (debugging): a fault is reported at the launch site that caused it
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) {
      g_last_cuda_error = std::string("kernels launched before mrrr.cu:") + std::to_string(line) + ": " +
                          cudaGetErrorString(e);
      throw Err{MRRR_ERR_CUDA};
    }
  }
}

// record the next pool event on the stream; returns its index (the pool grows on first use)
int tev_rec(mrrr_t h) {
  if (h->ntev >= (int)h->tev.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    h->tev.push_back(e);
  }
  const int i = h->ntev++;
  CK(cudaEventRecord(h->tev[i], h->stream));
  return i;
}

// NegCount chains: node grid points then explicit (rep, sigma) chains; CH chains per thread (x path)
template <bool Y>
void launch_negcount(mrrr_t h, const Node *nodes, int nnode, int m, int nex, const Node *nodesP = nullptr,
                     int nP = 0, const int *offsP = nullptr, int nPc = 0, double rtol = 0.0) {
  long long tot = (long long)nnode * ((1LL << m) - 1) + nPc + nex;
  if (!Y && nPc == 0 && h->segx_k > 1 && tot > 0 && h->cur_nbmax >= 2LL * h->segx_k * h->segx_w) {
    // segmented x-count over many representations (kernels_guided.cuh), junctions verified bit-exact
    const int K = h->segx_k;
    CK(h->segoutx.ensure(sizeof(SegOutX) * tot * K));
    CK(h->segfby.ensure(sizeof(FbX) * tot));
    CK(cudaMemsetAsync(h->cnt.as<int>() + C_NFB, 0, sizeof(int), h->stream));
    k_negcount_seg_xg<<<nblocks_for(tot * K, 128), 128, 0, h->stream>>>(
        nodes, nnode, m, h->ex.as<ExplicitChain>(), nex, h->reps.as<RepDesc>(), h->mx.as<double2>(), K, h->segx_w,
        h->segoutx.as<SegOutX>());
    k_seg_combine_xg<<<nblocks_for(tot, 128), 128, 0, h->stream>>>(tot, tot - nex, K, h->segoutx.as<SegOutX>(),
                                                                   h->counts.as<int>(), h->excounts.as<int>(),
                                                                   h->segfby.as<FbX>(), h->cnt.as<int>() + C_NFB,
                                                                   h->stats.as<long long>());
    k_seg_fallback_xg<<<nblocks_for(tot, 128), 128, 0, h->stream>>>(
        h->segfby.as<FbX>(), h->cnt.as<int>() + C_NFB, nodes, nnode, m, h->ex.as<ExplicitChain>(),
        h->reps.as<RepDesc>(), h->mx.as<double2>(), K, h->segx_w, h->counts.as<int>(), h->excounts.as<int>(),
        h->segoutx.as<SegOutX>(), h->stats.as<long long>());
    launch_check(h);
    return;
  }
  if (!Y && h->neg_tma) {
    k_negcount_tma<<<nblocks_for(tot, 128), 128, 2 * NEG_TILE * sizeof(double2), h->stream>>>(
        nodes, nnode, m, nodesP, nP, offsP, nPc, rtol, h->ex.as<ExplicitChain>(), nex, h->reps.as<RepDesc>(),
        h->mx.as<double2>(), h->counts.as<int>(), h->excounts.as<int>(), h->dS.as<double>(), h->dG.as<double>(),
        h->dH.as<double>());
    launch_check(h);
    return;
  }
  if (Y && h->segy_k > 1 && tot > 0) {
    // segmented y-count (kernels_guided.cuh): K segments per chain, junctions verified bit-exact
    const int K = h->segy_k;
    CK(h->segouty.ensure(sizeof(SegOutY) * tot * K));
    CK(h->segfby.ensure(sizeof(long long) * tot));
    CK(cudaMemsetAsync(h->cnt.as<int>() + C_NFB, 0, sizeof(int), h->stream));
    k_negcount_seg_y<<<nblocks_for(tot * K, 128), 128, 0, h->stream>>>(
        nodes, nnode, m, h->ex.as<ExplicitChain>(), nex, h->reps.as<RepDesc>(), h->mq.as<QElt>(), K, h->segy_w,
        h->segouty.as<SegOutY>());
    k_seg_combine_y<<<nblocks_for(tot, 128), 128, 0, h->stream>>>(tot, tot - nex, K, h->segouty.as<SegOutY>(),
                                                                  h->counts.as<int>(), h->excounts.as<int>(),
                                                                  h->segfby.as<long long>(), h->cnt.as<int>() + C_NFB);
    k_seg_fallback_y<<<nblocks_for(tot, 128), 128, 0, h->stream>>>(
        h->segfby.as<long long>(), h->cnt.as<int>() + C_NFB, nodes, nnode, m, h->ex.as<ExplicitChain>(),
        h->reps.as<RepDesc>(), h->mq.as<QElt>(), h->my.as<YElt>(), h->counts.as<int>(), h->excounts.as<int>());
    launch_check(h);
    return;
  }
  const ExplicitChain *ex = h->ex.as<ExplicitChain>();
  k_negcount<Y, 1><<<nblocks_for(tot, 128), 128, 0, h->stream>>>(
      nodes, nnode, m, ex, nex, h->reps.as<RepDesc>(), h->mx.as<double2>(), h->my.as<YElt>(), h->mq.as<QElt>(),
      h->counts.as<int>(), h->excounts.as<int>());
  launch_check(h);
}

__global__ void k_set_int(int *p, int v) { *p = v; }


// dynamic shared memory for the record-staging kernels (k_twist_pick2, k_fixed_step): the bytes if they fit
// the opt-in per-block limit (attributes raised once per handle), else 0 (the kernels then read global)
size_t stage_bytes(mrrr_t h, size_t bytes) {
  if (!h->stage_attr) {
    int dev = 0, lim = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&lim, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    h->stage_lim = (size_t)std::min(lim, 160 * 1024);
    CK(cudaFuncSetAttribute(k_twist_pick2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->stage_lim));
    CK(cudaFuncSetAttribute(k_fixed_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->stage_lim));
    h->stage_attr = true;
  }
  return (h->rec_stage && bytes <= h->stage_lim) ? bytes : 0;
}

// Segmented rounds driven by device-side node counters: round r reads its node count from nn[r] and the
// update writes nn[r+1], so batches of rounds are enqueued without a host round trip (kernels of empty
// rounds exit at once); the host checks the count once per batch.
void run_rounds_device(mrrr_t h, Node *cur, Node *nxt, int nnode, int nb, int maxnodes, double *out_lo,
                       double *out_hi, double rtol, int mcap = 0) {
  // mcap > 0 (stable phase: every node holds one wanted index, so the node count can only shrink): the
  // k-section depth stays at most mcap, so every round has at most nnode * (2^mcap - 1) chains and the
  // grids are sized exactly (depth is free: the dyadic grid makes any schedule bit-identical)
  const int MAXR = 256, RB = h->dev_rb;
  const int mmax = mcap > 0 ? mcap : h->mmax;
  const long long maxch = mcap > 0 ? (long long)maxnodes * ((1LL << mcap) - 1)
                                   : std::max<long long>(h->target_chains, maxnodes) + 128;
  // segments per chain: the host rounds' rule (more segments while the rounds have few chains)
  int K = seg_base_k(h, nb);
  while (2 * K <= 64 && maxch * 2 * K <= h->seg_threads && (nb - 1) >= 2 * (2 * K) * h->seg_w &&
         (nb - 1) / (2 * K) >= h->seg_minlen)
    K *= 2;
  const int L = (nb - 1 + K - 1) / K;
  CK(h->rnd.ensure(sizeof(int) * 2 * (MAXR + 2)));
  CK(h->counts.ensure(sizeof(int) * maxch));
  CK(h->segout.ensure(sizeof(SegOut) * maxch * K));
  std::vector<std::pair<int, int>> rp;  // timing events of each round
  int *nn = h->rnd.as<int>(), *nfb = nn + MAXR + 2;
  CK(cudaMemsetAsync(h->rnd.p, 0, sizeof(int) * 2 * (MAXR + 2), h->stream));
  k_set_int<<<1, 1, 0, h->stream>>>(nn, nnode);
  launch_check(h);
  unsigned long long *alg = (unsigned long long *)(h->stats.as<long long>() + ST_NEGX_ALG);
  long long *negx = h->stats.as<long long>() + ST_NEGX;
  int r = 0;
  long long known = nnode;  // node count of round r (read back once per batch)
  for (;;) {
    // grids for a batch: the node count can at most double per round (a node splits in two), and a round
    // has at most max(target, nodes) chains; CTAs beyond the live count exit at once
    long long bound = known;
    if (mcap <= 0)
      for (int b = 0; b < RB; b++) bound = std::min<long long>(2 * bound, maxnodes);
    const long long chmax = mcap > 0 ? maxch : std::min<long long>(maxch, std::max<long long>(bound, h->target_chains) + 128);
    const unsigned gseg = (unsigned)((chmax / 128 + 1) * K);
    const unsigned g1 = (unsigned)(chmax / 128 + 1);
    for (int b = 0; b < RB && r < MAXR; b++, r++) {
      Node *in = (r & 1) ? nxt : cur, *out = (r & 1) ? cur : nxt;
      SegOut *sg = h->segout.as<SegOut>();
      const int ea = h->round_ev ? tev_rec(h) : -1;
      k_negcount_seg<1><<<gseg, 128, 2 * SEG_TILE * sizeof(double2), h->stream>>>(
          in, 0, 0, nullptr, 0, h->reps.as<RepDesc>(), h->mx.as<double2>(), K, L, h->seg_w, sg,
          nn + r, mmax, h->target_chains);
      rp.push_back({ea, h->round_ev ? tev_rec(h) : -1});
      // junction walk (careful tail inline) and shared-tree update in one launch
      k_seg_round<<<g1 * 4, 32, 0, h->stream>>>(0, 0, K, sg, h->counts.as<int>(), in,
                                             h->reps.as<RepDesc>(), h->mx.as<double2>(), L, out, nn + r + 1, out_lo,
                                             out_hi, rtol, alg, nullptr, nfb + r, nn + r, mmax, h->target_chains, negx);
      launch_check(h);
      h->host_launches += 3;
    }
    // node counts of every round so far (the last one decides; the others count the rounds that ran)
    CK(cudaMemcpyAsync(h->h_rounds.data(), nn, sizeof(int) * (r + 1), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    const int left = h->h_rounds[r];
    if (left == 0) {
      std::vector<int> fb(r);
      CK(cudaMemcpy(fb.data(), nfb, sizeof(int) * r, cudaMemcpyDeviceToHost));
      for (int i = 0; i < r; i++) h->stats_h[ST_ROOT_FB] += fb[i];
      break;
    }
    known = left;
    if (r >= MAXR) { g_last_cuda_error = "bisection did not converge in 256 rounds"; throw Err{MRRR_ERR_CUDA}; }
  }
  for (int i = 0; i < r; i++) {
    if (h->h_rounds[i] == 0) break;
    if (rp[i].first >= 0) h->tneg.push_back(rp[i]);
    h->neg_launches++;
    h->host_rounds++;
  }
}

template <bool Y>
void run_bisection(mrrr_t h, int nnode, double *out_lo, double *out_hi, double rtol, int nverify,
                   const int *blist_dev, int nbl, bool *restart, int rep0 = -1, int nrep = 0, int single_nb = 0);

// k-section rounds with the nodes grouped by representation (child bisection over many child RRRs)
void run_bisection_grouped(mrrr_t h, int nnode, double *out_lo, double *out_hi, double rtol, int rep0, int nrep) {
  Node *cur = h->nodesA.as<Node>(), *nxt = h->nodesB.as<Node>();
  unsigned long long *alg = (unsigned long long *)(h->stats.as<long long>() + ST_NEGX_ALG);
  CK(h->repoff.ensure(sizeof(int) * (nrep + 1)));
  CK(h->repcur.ensure(sizeof(int) * (nrep + 1)));
  CK(h->repcta.ensure(sizeof(int) * (nrep + 1)));
  while (nnode > 0) {
    CK(h->nodesK.ensure(sizeof(Node) * nnode));
    int m = 1;
    while (m < h->mmax && (long long)nnode * ((1LL << (m + 1)) - 1) <= h->target_child) m++;
    const long long P = (1LL << m) - 1;
    // few chains per representation (e.g. thousands of 2-clusters): a CTA per representation would run
    // latency-bound waves; then the per-thread kernel runs on the rep-sorted nodes (a warp's lanes share
    // one or two representations, so their row loads coalesce)
    // (long child chains: the segmented per-thread path instead, on the same rep-sorted nodes)
    const bool per_cta = (long long)nnode * P >= 64LL * nrep &&
                         !(h->segx_k > 1 && h->cur_nbmax >= 2LL * h->segx_k * h->segx_w);
    zero_counters(h);
    CK(cudaMemsetAsync(h->repoff.p, 0, sizeof(int) * (nrep + 1), h->stream));
    k_rep_hist<<<nblocks_for(nnode, 128), 128, 0, h->stream>>>(cur, nnode, rep0, h->repoff.as<int>());
    launch_check(h);
    k_scan_excl<<<1, 1024, 0, h->stream>>>(h->repoff.as<int>(), nrep, h->cnt.as<int>() + C_NPC);
    launch_check(h);
    CK(cudaMemcpyAsync(h->repcur.p, h->repoff.p, sizeof(int) * (nrep + 1), cudaMemcpyDeviceToDevice, h->stream));
    k_rep_scatter<<<nblocks_for(nnode, 128), 128, 0, h->stream>>>(cur, nnode, rep0, h->repcur.as<int>(),
                                                                 h->nodesK.as<Node>());
    launch_check(h);
    k_rep_ctas<<<nblocks_for(nrep, 128), 128, 0, h->stream>>>(h->repoff.as<int>(), nrep, P, h->repcta.as<int>());
    launch_check(h);
    k_scan_excl<<<1, 1024, 0, h->stream>>>(h->repcta.as<int>(), nrep, h->cnt.as<int>() + C_NK);
    launch_check(h);
    read_counters(h);
    const int ncta = h->h_cnt[C_NK];
    const long long nch = (long long)nnode * P;
    CK(h->counts.ensure(std::max<long long>(nch, 1) * sizeof(int)));
    zero_counters(h);
    const int ea = tev_rec(h);
    if (per_cta) {
      k_negcount_grp<<<ncta, 128, 2 * NEG_TILE * sizeof(double2), h->stream>>>(
          h->nodesK.as<Node>(), m, h->repoff.as<int>(), h->repcta.as<int>(), nrep, h->reps.as<RepDesc>(),
          h->mx.as<double2>(), h->counts.as<int>());
      launch_check(h);
    } else {
      launch_negcount<false>(h, h->nodesK.as<Node>(), nnode, m, 0);
    }
    h->tneg.push_back({ea, tev_rec(h)});
    k_bisect_update<<<nblocks_for((long long)nnode << m, 128), 128, 0, h->stream>>>(
        h->nodesK.as<Node>(), nnode, m, h->counts.as<int>(), nxt, h->cnt.as<int>() + C_NNEXT, out_lo, out_hi, rtol,
        alg);
    launch_check(h);
    read_counters(h);
    h->host_rounds++;
    h->stats_h[ST_NEGX] += nch;
    h->neg_launches++;
    nnode = h->h_cnt[C_NNEXT];
    std::swap(cur, nxt);
  }
}

// shared-tree / k-section bisection rounds until every node is finished (S5, S8)
template <bool Y>
void run_bisection(mrrr_t h, int nnode, double *out_lo, double *out_hi, double rtol, int nverify,
                   const int *blist_dev, int nbl, bool *restart, int rep0, int nrep, int single_nb) {
  if (!Y && rep0 >= 0 && nrep > 1 && h->neg_tma && h->grouped) {
    run_bisection_grouped(h, nnode, out_lo, out_hi, rtol, rep0, nrep);
    return;
  }
  Node *cur = h->nodesA.as<Node>(), *nxt = h->nodesB.as<Node>();
  bool first = true;
  bool seg_on = !Y && single_nb > 0 && h->neg_tma && seg_base_k(h, single_nb) > 1 && !h->nonlocal;
  while (nnode > 0) {
    const long long target = seg_on ? h->target_chains
                            : (Y && h->segy_k > 1) ? h->target_y
                            : (rep0 >= 0) ? h->target_child
                                          : h->target_unseg;
    int m = 1;
    while (m < h->mmax && (long long)nnode * ((1LL << (m + 1)) - 1) <= target) m++;
    long long P = (1LL << m) - 1;
    long long nch = (long long)nnode * P;
    CK(h->counts.ensure(std::max<long long>(nch, 1) * sizeof(int)));
    int nex = first ? nverify : 0;
    bool fused = false;  // the segmented round's update ran inside k_seg_round
    zero_counters(h);
    const int ea = tev_rec(h);
    int eb = -1;
    if (seg_on) {
      // segmented chains (kernels_guided.cuh): K concurrent segments per NegCount, verified bit-exact.
      // Rounds with few chains (one point per node) cut them into more segments, so that about
      // seg_threads threads keep the SMs busy (a round is latency-bound below that)
      const long long tot = nch + nex;
      int K = seg_base_k(h, single_nb);
      while (2 * K <= 64 && tot * 2 * K <= h->seg_threads && (single_nb - 1) >= 2 * (2 * K) * h->seg_w &&
             (single_nb - 1) / (2 * K) >= h->seg_minlen)
        K *= 2;
      const int L = (single_nb - 1 + K - 1) / K;
      CK(h->segout.ensure(sizeof(SegOut) * tot * K));
      const int CH = (tot <= h->seg_ch2) ? 2 : 1;  // few chains: two per thread (ILP)
      const unsigned grid = (unsigned)((tot + 128 * CH - 1) / (128 * CH) * K);
      if (CH == 2)
        k_negcount_seg<2><<<grid, 128, 2 * SEG_TILE * sizeof(double2), h->stream>>>(
            cur, nnode, m, h->ex.as<ExplicitChain>(), nex, h->reps.as<RepDesc>(), h->mx.as<double2>(), K, L,
            h->seg_w, h->segout.as<SegOut>(), nullptr, 0, 0);
      else
        k_negcount_seg<1><<<grid, 128, 2 * SEG_TILE * sizeof(double2), h->stream>>>(
            cur, nnode, m, h->ex.as<ExplicitChain>(), nex, h->reps.as<RepDesc>(), h->mx.as<double2>(), K, L,
            h->seg_w, h->segout.as<SegOut>(), nullptr, 0, 0);
      launch_check(h);
      eb = tev_rec(h);
      if (nex == 0 && m <= h->fuse_mmax) {  // junction walk and shared-tree update in one launch (a thread per
                                              // node walks its 2^m - 1 chains: only while m is small)
        k_seg_round<<<nblocks_for(nnode, 32), 32, 0, h->stream>>>(
            nnode, m, K, h->segout.as<SegOut>(), h->counts.as<int>(), cur, h->reps.as<RepDesc>(), h->mx.as<double2>(),
            L, nxt, h->cnt.as<int>() + C_NNEXT, out_lo, out_hi, rtol,
            (unsigned long long *)(h->stats.as<long long>() + ST_NEGX_ALG), h->cnt.as<int>() + C_NMULTI,
            h->cnt.as<int>() + C_NFB, nullptr, 0, 0, nullptr);
        fused = true;
      } else {
        k_seg_combine<<<nblocks_for(tot, 128), 128, 0, h->stream>>>(
            tot, nch, K, h->segout.as<SegOut>(), h->counts.as<int>(), h->excounts.as<int>(), h->cnt.as<int>() + C_NFB,
            nullptr, 0, 0, nullptr, cur, nnode, m, h->ex.as<ExplicitChain>(), h->reps.as<RepDesc>(),
            h->mx.as<double2>(), L);
      }
      launch_check(h);
    } else {
      launch_negcount<Y>(h, cur, nnode, m, nex);
      eb = tev_rec(h);
    }
    if (nex > 0) {
      k_root_verify<<<nblocks_for(nbl, 128), 128, 0, h->stream>>>(blist_dev, nbl, h->starts.as<int>(),
                                                                  h->binfo.as<double>(), h->excounts.as<int>(),
                                                                  h->cnt.as<int>() + C_NEX);
      launch_check(h);
    }
    if (!fused) {
      k_bisect_update<<<nblocks_for((long long)nnode << m, 128), 128, 0, h->stream>>>(
          cur, nnode, m, h->counts.as<int>(), nxt, h->cnt.as<int>() + C_NNEXT, out_lo, out_hi, rtol,
          (unsigned long long *)(h->stats.as<long long>() + (Y ? ST_NEGY_ALG : ST_NEGX_ALG)),
          h->cnt.as<int>() + C_NMULTI);
      launch_check(h);
    }
    read_counters(h);
    h->host_rounds++;
    h->stats_h[Y ? ST_NEGY : ST_NEGX] += nch + nex;
    if (seg_on) h->stats_h[ST_ROOT_FB] += h->h_cnt[C_NFB];
    if (seg_on && (long long)h->h_cnt[C_NFB] * 4 > nch + nex) {
      // most segment junctions failed: the recurrence does not contract on this matrix (delocalised
      // eigenvectors, e.g. the 1-2-1, Clement, Hermite and prescribed-spectrum families), so every chain fell
      // back to its sequential tail; the remaining rounds run whole chains, and the singleton RQI skips its
      // segmented passes (their twist search would hand every singleton over)
      seg_on = false;
      h->nonlocal = true;
    }
    if (!Y) {
      h->tneg.push_back({ea, eb});
      h->neg_launches++;
    }
    if (nex > 0 && h->h_cnt[C_NEX] > 0) { *restart = true; return; }
    nnode = h->h_cnt[C_NNEXT];
    std::swap(cur, nxt);
    first = false;
    if (!Y && seg_on && h->dev_rounds && nnode > 0) {
      run_rounds_device(h, cur, nxt, nnode, single_nb, std::max(nnode, h->max_nodes), out_lo, out_hi, rtol);
      return;
    }
    // the looser bound oversizes the grids by up to 1/frac: worth it while rounds are short (measured:
    // frac 4 at n <= 16K, 16 for the long chains of n = 65536)
    const int dfrac = h->dev_frac > 0 ? h->dev_frac : (single_nb <= 16384 ? 4 : 16);
    if (!Y && seg_on && h->dev_stable && nnode > 0 && (long long)h->h_cnt[C_NMULTI] * dfrac <= nnode) {
      // near-stable phase: the node count can grow by at most the indices still sharing nodes (few), so
      // the remaining rounds run without host round trips on grids sized for that bound
      const long long maxn = (long long)nnode + h->h_cnt[C_NMULTI];
      int mcap = 1;
      while (mcap < h->mmax && maxn * ((1LL << (mcap + 1)) - 1) <= target) mcap++;
      run_rounds_device(h, cur, nxt, nnode, single_nb, (int)maxn, out_lo, out_hi, rtol, mcap);
      return;
    }
  }
}

// bracket verification / repair rounds for per-index start intervals; ready nodes land in nodesA
template <bool Y>
int run_brackets(mrrr_t h, int nbn) {
  BNode *cur = h->bnA.as<BNode>(), *pend = h->bnB.as<BNode>();
  // consecutive start nodes with identical start intervals: one shared node per run
  if (nbn > 1 && h->bmerge) {
    k_bnode_mark<<<nblocks_for(nbn, 128), 128, 0, h->stream>>>(cur, nbn);
    k_bnode_merge<<<nblocks_for(nbn, 128), 128, 0, h->stream>>>(cur, nbn);
    launch_check(h);
  }
  Node *ready = h->nodesA.as<Node>();
  int nready = 0;
  zero_counters(h);
  while (nbn > 0) {
    CK(cudaMemsetAsync(h->cnt.as<int>() + C_NEX, 0, sizeof(int), h->stream));
    CK(cudaMemsetAsync(h->cnt.as<int>() + C_NPEND, 0, sizeof(int), h->stream));
    k_bracket_chains<<<nblocks_for(nbn, 128), 128, 0, h->stream>>>(cur, nbn, h->ex.as<ExplicitChain>(),
                                                                  h->exmap.as<int>(), h->cnt.as<int>() + C_NEX);
    launch_check(h);
    read_counters(h);
    int nex = h->h_cnt[C_NEX];
    if (nex > 0) {
      launch_negcount<Y>(h, nullptr, 0, 1, nex);
      k_bracket_scatter<<<nblocks_for(nex, 128), 128, 0, h->stream>>>(cur, h->exmap.as<int>(), h->excounts.as<int>(),
                                                                      nex);
      launch_check(h);
      h->stats_h[Y ? ST_NEGY : ST_NEGX] += nex;
    }
    k_bracket_update<<<nblocks_for(nbn, 128), 128, 0, h->stream>>>(cur, nbn, pend, h->cnt.as<int>() + C_NPEND, ready,
                                                                  h->cnt.as<int>() + C_NREADY,
                                                                  h->stats.as<long long>());
    launch_check(h);
    read_counters(h);
    h->host_rounds++;
    nbn = h->h_cnt[C_NPEND];
    nready = h->h_cnt[C_NREADY];
    std::swap(cur, pend);
  }
  return nready;
}

// keep the representation pool (read by every RQI lane at every step) resident in L2 while the
// workspace streams past it: persisting access-policy window on the handle's stream
// numerical-support threshold of the Z write (S10', A-42): eps_x of the realisation, 0 when MRRR_FULL_SUPPORT
double eps_support(mrrr_t h) {
  if (h->flags & MRRR_FULL_SUPPORT) return 0.0;
  return h->sd ? 0x1p-24 : EPS_X;
}

void l2_pin_reps(mrrr_t h, bool on) {
  if (!h->l2_persist) return;
  cudaStreamAttrValue v;
  memset(&v, 0, sizeof(v));
  if (on) {
    Buf &hot = h->mq;  // the representation form the RQI lanes stream
    size_t bytes = std::min<size_t>(hot.cap, (size_t)h->l2_max_window);
    v.accessPolicyWindow.base_ptr = hot.p;
    v.accessPolicyWindow.num_bytes = bytes;
    v.accessPolicyWindow.hitRatio = 1.0f;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  }
  cudaStreamSetAttribute(h->stream, cudaStreamAttributeAccessPolicyWindow, &v);
  cudaGetLastError();
}

void run_rqi(mrrr_t h, int ns, long long nbmax, double *W, double *Z, long long ldz, bool allow_seg,
             bool child = false, const Singleton *list = nullptr) {
  if (ns <= 0) return;
  l2_pin_reps(h, true);
  // workspace per singleton: 3 dd planes (the two-lane kernel's P0, P1, P2; the segmented passes use the first
  // for the twist search and the second for the stored factors)
  long long per = 3LL * (long long)sizeof(dd) * std::max<long long>(nbmax, 1);
  long long budget = std::min<long long>(h->ws_limit / 2, 64LL << 30);
  long long bmax = std::max<long long>(32, budget / per);
  long long batch = std::min<long long>(ns, bmax);
  long long stride = (batch + 31) / 32 * 32;  // pairs launched per batch (grid padding)
  CK(h->wsA.ensure((size_t)3 * stride * nbmax * sizeof(dd)));
  bool diag = (h->flags & MRRR_KEEP_DIAG) != 0;
  for (long long b0 = 0; b0 < ns; b0 += batch) {
    long long nb = std::min<long long>(batch, ns - b0);
    const int rq0 = tev_rec(h);
    CK(h->zmeta.ensure(sizeof(ZMeta) * stride));
    const Singleton *sgb = (list ? list : h->sing.as<Singleton>()) + b0;
    int nold = (int)nb;
    if (h->rqi_seg && allow_seg) {
      // segmented passes (kernels_rqi3.cuh); singletons they hand over go through k_rqi2 below
      // segments per lane: at least rqi_segk; more when the batch has few singletons (a rank's shard),
      // so that about rqi_threads threads run, as long as a chunk stays longer than the warm-up
      int K = h->rqi_segk;
      // warm-up rows: 128 suffice up to n = 16K (no retries measured); longer frames get 192
      int Wu = h->rqi_segw > 0 ? h->rqi_segw : (nbmax <= 16384 ? 128 : 192);
      if (h->sd && (h->nonlocal || nbmax <= h->rqi_seg_min)) {
        // single/double on short or non-contracting frames: every chunk starts at row 0 (a warm-up over the whole
        // frame), so every junction holds by construction and the binary64 passes never hand over for a junction
        K = 1;
        Wu = (int)nbmax;
      }
      while (2 * K <= 32 && (long long)nb * 2 * (2 * K) <= h->rqi_threads && (nbmax - 1) >= 2 * (2 * K) * Wu) K *= 2;
      // z recompute window (k_zrc): root frames of the double/dd solve with the numerical support on
      const bool zrc = h->zwin > 0 && (!child || h->zrc_child) && !h->sd && eps_support(h) > 0.0 && nbmax > 2LL * h->zwin;
      if (zrc) {
        CK(h->zinb.ensure(sizeof(dd) * 2 * stride));
        CK(h->zrcb.ensure(sizeof(int) * 4));
        CK(cudaMemsetAsync(h->zrcb.p, 0, sizeof(int) * 4, h->stream));
        k_set_int<<<1, 1, 0, h->stream>>>(h->zrcb.as<int>() + 1, 1);  // the rerun's pass mode: stored
      }
      CK(h->rqst.ensure(sizeof(RqiState) * stride));
      CK(h->rqrec.ensure(sizeof(SegRec) * stride * 4 * K));  // chunk layout: 2K chunks x 2 lanes
      CK(h->hand.ensure(sizeof(Singleton) * stride));
      double *TF = reinterpret_cast<double *>(h->wsA.as<dd>());  // [row * stride + singleton]
      dd *P2s = h->wsA.as<dd>() + stride * nbmax;                 // after TF
      RqiState *rs = h->rqst.as<RqiState>();
      SegRec *rec = h->rqrec.as<SegRec>();
      const int MAXP = 2 * MAX_RQI + 4;
      CK(h->rqmode.ensure(sizeof(int) * 3 * (MAXP + 1)));
      int *qm = h->rqmode.as<int>();
      CK(cudaMemsetAsync(qm, 0, sizeof(int) * 3 * (MAXP + 1), h->stream));  // pass 0: mode 0 (or 3, k_rqi3_init)
      k_rqi3_init<<<nblocks_for(nb, 128), 128, 0, h->stream>>>(sgb, (int)nb, h->reps.as<RepDesc>(), rs,
                                                                h->sd ? 0x1p-24 : EPS_X, 1e-2 * h->gaptol, qm + 2);
      const int KT = 2 * K;
      TwRec *trec = reinterpret_cast<TwRec *>(rec);
      const size_t tsb = stage_bytes(h, 32 * 2 * KT * sizeof(TwRec));
      if (child || nbmax <= h->twdd_root_max) {
        // child frames: the dd twist search (d+ in dd over the first plane)
        dd *TFd = h->wsA.as<dd>();
        k_twist_lane_dd<false><<<nblocks_for((long long)KT * nb, 128), 128, 0, h->stream>>>(
            sgb, (int)nb, h->reps.as<RepDesc>(), h->mq.as<QElt>(), rs, KT, Wu, TFd, stride, trec);
        k_twist_lane_dd<true><<<nblocks_for((long long)KT * nb, 128), 128, 0, h->stream>>>(
            sgb, (int)nb, h->reps.as<RepDesc>(), h->mq.as<QElt>(), rs, KT, Wu, TFd, stride, trec);
        k_twist_pick2<<<nblocks_for(nb, 32), 32, tsb, h->stream>>>(sgb, (int)nb, h->reps.as<RepDesc>(), rs, KT, nullptr,
                                                                 TFd, stride, trec, 0x1p-90, h->stats.as<long long>(),
                                                                 tsb ? 1 : 0);
      } else {
        // twist search: forward lane stores d+, backward lane forms gamma and the per-chunk argmin
        k_twist_lane<false><<<nblocks_for((long long)KT * nb, 128), 128, 0, h->stream>>>(
            sgb, (int)nb, h->reps.as<RepDesc>(), h->mq.as<QElt>(), rs, KT, Wu, TF, stride, trec);
        k_twist_lane<true><<<nblocks_for((long long)KT * nb, 128), 128, 0, h->stream>>>(
            sgb, (int)nb, h->reps.as<RepDesc>(), h->mq.as<QElt>(), rs, KT, Wu, TF, stride, trec);
        k_twist_pick2<<<nblocks_for(nb, 32), 32, tsb, h->stream>>>(sgb, (int)nb, h->reps.as<RepDesc>(), rs, KT, TF,
                                                                 nullptr, stride, trec, 0x1p-46,
                                                                 h->stats.as<long long>(), tsb ? 1 : 0);
      }
      launch_check(h);
      // passes by mode: the RQC-only (light) passes of every singleton that still has one due run before the
      // stored passes, so a singleton that needs two light passes (a start left at the early-stop tolerance)
      // does not put a stored pass and a second light pass into two separate launches of the others.  The mode
      // of each pass is decided on the device (k_rqi_mode); the host checks after batches of passes.
      const size_t fsb = stage_bytes(h, 32 * 4 * K * sizeof(SegRec));
      int p = 0;
      for (int batch = 3; p < MAXP; batch = 1) {  // first batch: light, stored, and one spare pass (or x-light,
                                                  // light, stored)
        for (int b = 0; b < batch && p < MAXP; b++, p++) {
          k_fixed_chunk<<<nblocks_for((2 * K + 1) * nb, 128), 128, 0, h->stream>>>(
              sgb, (int)nb, h->reps.as<RepDesc>(), h->mq.as<QElt>(), rs, 2 * K, Wu, P2s, nbmax, rec,
              h->rqi_bulk ? 1 : 0, h->sd ? 1 : 0, qm + 3 * p + 2, zrc ? h->zinb.as<dd>() : nullptr, h->zwin);
          k_fixed_step<<<nblocks_for(nb, 32), 32, fsb, h->stream>>>(
              sgb, (int)nb, h->reps.as<RepDesc>(), rs, K, rec, W, h->zmeta.as<ZMeta>(),
              diag ? h->ddepth.as<int>() : nullptr, diag ? h->dflo.as<double>() : nullptr,
              diag ? h->dfhi.as<double>() : nullptr, h->stats.as<long long>(), qm + 3 * p, fsb ? 1 : 0,
              h->sd ? 1 : 0, h->sd ? 0x1p-53 : EPS_Y, qm + 3 * p + 2, zrc ? 1 : 0);
          k_rqi_mode<<<1, 1, 0, h->stream>>>(qm, p);
          launch_check(h);
          h->host_launches += 2;
        }
        CK(cudaMemcpyAsync(h->h_small, qm + 3 * p + 2, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        const int nm = h->h_small[0];
        if (nm == 2) break;
      }
      int *stat = reinterpret_cast<int *>(reinterpret_cast<char *>(rs) + offsetof(RqiState, status));
      int *zc = zrc ? h->zrcb.as<int>() : nullptr;
      if (zrc)
        k_zrc<<<nblocks_for(2 * nb, 128), 128, 0, h->stream>>>(sgb, (int)nb, h->reps.as<RepDesc>(), h->mq.as<QElt>(),
                                                             rs, h->zmeta.as<ZMeta>(), h->zinb.as<dd>(), P2s, nbmax,
                                                             h->zwin);
      k_zwrite_chunk<<<nblocks_for(nb, 4), 128, 0, h->stream>>>(
          sgb, (int)nb, h->reps.as<RepDesc>(), h->my.as<YElt>(), P2s, nbmax, h->zmeta.as<ZMeta>(), Z, ldz,
          eps_support(h), stat, (int)(sizeof(RqiState) / sizeof(int)), zrc ? h->zwin : 0, 0, zc);
      launch_check(h);
      if (zrc) {
        // supports that reach past the recompute window: a stored pass at the accepted lambda, then their z
        CK(cudaMemcpyAsync(h->h_small, zc, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        const int nre = h->h_small[0];
        h->stats_h[ST_ZRC_RERUN] += nre;
        if (nre > 0) {
          k_fixed_chunk<<<nblocks_for((2 * K + 1) * nb, 128), 128, 0, h->stream>>>(
              sgb, (int)nb, h->reps.as<RepDesc>(), h->mq.as<QElt>(), rs, 2 * K, Wu, P2s, nbmax, rec,
              h->rqi_bulk ? 1 : 0, 0, zc + 1);
          k_fixed_step<<<nblocks_for(nb, 32), 32, fsb, h->stream>>>(
              sgb, (int)nb, h->reps.as<RepDesc>(), rs, K, rec, W, h->zmeta.as<ZMeta>(),
              diag ? h->ddepth.as<int>() : nullptr, diag ? h->dflo.as<double>() : nullptr,
              diag ? h->dfhi.as<double>() : nullptr, h->stats.as<long long>(), zc + 2, fsb ? 1 : 0, 0, EPS_Y,
              zc + 1, 0);
          k_zrc_settle<<<nblocks_for(nb, 128), 128, 0, h->stream>>>(rs, (int)nb);
          k_zwrite_chunk<<<nblocks_for(nb, 4), 128, 0, h->stream>>>(
              sgb, (int)nb, h->reps.as<RepDesc>(), h->my.as<YElt>(), P2s, nbmax, h->zmeta.as<ZMeta>(), Z, ldz,
              eps_support(h), stat, (int)(sizeof(RqiState) / sizeof(int)), 0, 1, nullptr);
          launch_check(h);
        }
      }
      CK(cudaMemsetAsync(h->cnt.as<int>() + C_NFB, 0, sizeof(int), h->stream));
      k_rqi3_collect<<<nblocks_for(nb, 128), 128, 0, h->stream>>>(sgb, (int)nb, rs, h->hand.as<Singleton>(),
                                                                  h->cnt.as<int>() + C_NFB);
      launch_check(h);
      CK(cudaMemcpyAsync(h->h_small, h->cnt.as<int>() + C_NFB, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      nold = h->h_small[0];
      sgb = h->hand.as<Singleton>();
      h->stats_h[ST_RQI_HANDOVER] += nold;
    }
    if (nold > 0) {
      k_rqi2<<<nblocks_for(2 * nold, 64), 64, 64 * MRRR_RQI_RING * sizeof(RingSlot), h->stream>>>(
          sgb, nold, h->reps.as<RepDesc>(), h->my.as<YElt>(), h->mq.as<QElt>(), h->wsA.as<dd>(), stride, nbmax, W,
          h->zmeta.as<ZMeta>(), diag ? h->ddepth.as<int>() : nullptr, diag ? h->dflo.as<double>() : nullptr,
          diag ? h->dfhi.as<double>() : nullptr, h->stats.as<long long>(), h->fault, h->sd ? 1 : 0,
          h->sd ? 0x1p-24 : EPS_X, h->sd ? 0x1p-53 : EPS_Y);
      launch_check(h);
      k_zwrite_chunk<<<nblocks_for(nold, 4), 128, 0, h->stream>>>(
          sgb, nold, h->reps.as<RepDesc>(), h->my.as<YElt>(), h->wsA.as<dd>() + 2 * stride * nbmax, nbmax,
          h->zmeta.as<ZMeta>(), Z, ldz, eps_support(h));
    }
    launch_check(h);
    h->trq.push_back({rq0, tev_rec(h)});
    h->rqi_launches++;
  }
  l2_pin_reps(h, false);
}

// the solve stream waits for the deferred tail (before anything that could overwrite what the tail reads: the
// representation slots of the next chunk, the end of the solve)
void join_tail(mrrr_t h) {
  if (h->tail_pending) CK(cudaStreamWaitEvent(h->stream, h->ev_tail_done, 0));
}

// two-lane workspace of a deferred tail of ns singletons on frames of up to nbmax rows
long long tail_bytes(int ns, long long nbmax) {
  const long long stride = ((long long)ns + 31) / 32 * 32;
  return 3LL * stride * std::max<long long>(nbmax, 1) * (long long)sizeof(dd);
}

// a child level's singletons that go to the two-lane kernel only (run_rqi with allow_seg false): the same two
// launches as run_rqi's k_rqi2 branch, on the side stream after the solve stream's current work (the child
// representations), with their own workspace and a copy of the singleton list; the levels above go on meanwhile
void launch_tail(mrrr_t h, int ns, long long nbmax, double *W, double *Z, long long ldz) {
  if (!h->s_tail) {
    CK(cudaStreamCreate(&h->s_tail));
    CK(cudaEventCreateWithFlags(&h->ev_tail_in, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_tail_done, cudaEventDisableTiming));
  }
  if (h->tail_pending) CK(cudaStreamSynchronize(h->s_tail));  // its buffers are reused below
  h->tail_pending = false;
  const long long stride = ((long long)ns + 31) / 32 * 32;
  CK(h->tail_ws.ensure((size_t)tail_bytes(ns, nbmax)));
  CK(h->tail_sing.ensure(sizeof(Singleton) * stride));
  CK(h->tail_zmeta.ensure(sizeof(ZMeta) * stride));
  CK(cudaMemcpyAsync(h->tail_sing.p, h->sing.p, sizeof(Singleton) * ns, cudaMemcpyDeviceToDevice, h->stream));
  CK(cudaEventRecord(h->ev_tail_in, h->stream));
  CK(cudaStreamWaitEvent(h->s_tail, h->ev_tail_in, 0));
  const bool diag = (h->flags & MRRR_KEEP_DIAG) != 0;
  const Singleton *sgb = h->tail_sing.as<Singleton>();
  k_rqi2<<<nblocks_for(2 * ns, 64), 64, 64 * MRRR_RQI_RING * sizeof(RingSlot), h->s_tail>>>(
      sgb, ns, h->reps.as<RepDesc>(), h->my.as<YElt>(), h->mq.as<QElt>(), h->tail_ws.as<dd>(), stride, nbmax, W,
      h->tail_zmeta.as<ZMeta>(), diag ? h->ddepth.as<int>() : nullptr, diag ? h->dflo.as<double>() : nullptr,
      diag ? h->dfhi.as<double>() : nullptr, h->stats.as<long long>(), h->fault, h->sd ? 1 : 0,
      h->sd ? 0x1p-24 : EPS_X, h->sd ? 0x1p-53 : EPS_Y);
  CK(cudaGetLastError());
  k_zwrite_chunk<<<nblocks_for(ns, 4), 128, 0, h->s_tail>>>(
      sgb, ns, h->reps.as<RepDesc>(), h->my.as<YElt>(), h->tail_ws.as<dd>() + 2 * stride * nbmax, nbmax,
      h->tail_zmeta.as<ZMeta>(), Z, ldz, eps_support(h));
  CK(cudaGetLastError());
  CK(cudaEventRecord(h->ev_tail_done, h->s_tail));
  h->tail_pending = true;
  h->host_launches += 2;  // (not in the RQI phase events: it overlaps other phases)
}

struct ClusterLevel {
  int ncl;
};

// depth-first processing of a cluster list (S8), chunked to bound the child pool
void process_clusters(mrrr_t h, Cluster *list_dev, int ncl, int rep_top, long long pool_top, long long ipool_top,
                      long long nbmax, bool from_ipool, double *W, double *Z, long long ldz, long long kout,
                      int level) {
  if (ncl <= 0) return;
  bool diag = (h->flags & MRRR_KEEP_DIAG) != 0;
  // copy the list to host (for chunking / segment offsets)
  std::vector<Cluster> hl(ncl);
  CK(cudaMemcpyAsync(hl.data(), list_dev, sizeof(Cluster) * ncl, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  long long per_child = nbmax * (long long)(sizeof(double2) + sizeof(YElt));
  long long budget = std::max<long long>(per_child, h->ws_limit / 4 - pool_top * (long long)(sizeof(double2) + sizeof(YElt)));
  int chunk = (int)std::max<long long>(1, std::min<long long>(ncl, budget / per_child));
  const bool keep = level < mrrr_ctx::LVL_MAX;  // per-level buffers kept in the handle (no cudaFree mid-solve)
  for (int c0 = 0; c0 < ncl; c0 += chunk) {
    int nc = std::min(chunk, ncl - c0);
    join_tail(h);  // a deferred tail of the previous chunk reads representation slots this chunk overwrites
    // own copy of this chunk's cluster list (device list buffers are reused by recursion)
    Buf Lloc;
    Buf &L = keep ? h->lvl_L[level] : Lloc;
    CK(L.ensure(sizeof(Cluster) * nc));
    CK(cudaMemcpyAsync(L.p, hl.data() + c0, sizeof(Cluster) * nc, cudaMemcpyHostToDevice, h->stream));
    Cluster *cl = L.as<Cluster>();
    // grow the pools (keeping live data): child reps, their data, interval segments
    int repbase = rep_top;
    long long poolbase = pool_top;
    if (h->tail_pending) {  // a reallocated pool must not be freed under a running tail
      const size_t pe = (size_t)(poolbase + (long long)nc * nbmax);
      if (h->reps.cap < sizeof(RepDesc) * (size_t)(repbase + nc) || h->mx.cap < sizeof(double2) * pe ||
          h->my.cap < sizeof(YElt) * pe || h->mq.cap < sizeof(QElt) * pe)
        CK(cudaStreamSynchronize(h->s_tail));
    }
    CK(h->reps.grow_keep(sizeof(RepDesc) * (size_t)(repbase + nc), sizeof(RepDesc) * (size_t)repbase, h->stream));
    CK(h->mx.grow_keep(sizeof(double2) * (size_t)(poolbase + (long long)nc * nbmax),
                       sizeof(double2) * (size_t)poolbase, h->stream));
    CK(h->my.grow_keep(sizeof(YElt) * (size_t)(poolbase + (long long)nc * nbmax), sizeof(YElt) * (size_t)poolbase,
                       h->stream));
    CK(h->mq.grow_keep(sizeof(QElt) * (size_t)(poolbase + (long long)nc * nbmax), sizeof(QElt) * (size_t)poolbase,
                       h->stream));
    long long stot = 0, btot = 0;
    for (int c = 0; c < nc; c++) { stot += hl[c0 + c].q - hl[c0 + c].p + 3; btot += hl[c0 + c].q - hl[c0 + c].p + 1; }
    CK(h->ipool_lo.grow_keep(sizeof(double) * (size_t)(ipool_top + stot), sizeof(double) * (size_t)ipool_top, h->stream));
    CK(h->ipool_hi.grow_keep(sizeof(double) * (size_t)(ipool_top + stot), sizeof(double) * (size_t)ipool_top, h->stream));
    const double *ilo = from_ipool ? h->ipool_lo.as<double>() : h->rlo.as<double>();
    const double *ihi = from_ipool ? h->ipool_hi.as<double>() : h->rhi.as<double>();
    // (a) y-refined ends
    CK(h->bnA.ensure(sizeof(BNode) * std::max<long long>(2LL * nc, 1)));
    CK(h->bnB.ensure(sizeof(BNode) * std::max<long long>(2LL * nc, 1)));
    CK(h->ex.ensure(sizeof(ExplicitChain) * 4LL * nc + 64));
    CK(h->excounts.ensure(sizeof(int) * 4LL * nc + 64));
    CK(h->exmap.ensure(sizeof(int) * 4LL * nc + 64));
    CK(h->nodesA.ensure(sizeof(Node) * std::max<long long>(2LL * nc, 1)));
    CK(h->nodesB.ensure(sizeof(Node) * std::max<long long>(2LL * nc, 1)));
    CK(h->yref_lo.ensure(sizeof(double) * 2LL * nc));
    CK(h->yref_hi.ensure(sizeof(double) * 2LL * nc));
    k_clu_yref_init<<<nblocks_for(nc, 128), 128, 0, h->stream>>>(cl, nc, h->reps.as<RepDesc>(), ilo, ihi,
                                                                 h->bnA.as<BNode>());
    launch_check(h);
    bool dummy = false;
    if (h->sd) {
      // single/double: y = binary64, so the y-count is the x-count on M_x = M_y (the same operations): the
      // x-path brackets and bisection with the y tolerance
      const int nr = run_brackets<false>(h, 2 * nc);
      h->cur_nbmax = nbmax;
      run_bisection<false>(h, nr, h->yref_lo.as<double>(), h->yref_hi.as<double>(), RTOL_Y, 0, nullptr, 0, &dummy);
      h->cur_nbmax = 0;
    } else {
      const int nr = run_brackets<true>(h, 2 * nc);
      run_bisection<true>(h, nr, h->yref_lo.as<double>(), h->yref_hi.as<double>(), RTOL_Y, 0, nullptr, 0, &dummy);
    }
    // (b, c) shifts
    CK(h->ss.ensure(sizeof(ShiftState) * nc));
    CK(h->gval.ensure(sizeof(double) * 2LL * nc));
    CK(h->valid.ensure(sizeof(int) * 2LL * nc));
    k_clu_shift_init<<<nblocks_for(nc, 128), 128, 0, h->stream>>>(nc, h->yref_lo.as<double>(), h->yref_hi.as<double>(),
                                                                  h->ss.as<ShiftState>());
    launch_check(h);
    // attempt 0 for every cluster, then the remaining attempts of the open clusters in one launch
    CK(h->gval.ensure(sizeof(double) * 2LL * (MAX_ATTEMPTS - 1) * nc));
    CK(h->valid.ensure(sizeof(int) * 2LL * (MAX_ATTEMPTS - 1) * nc));
    for (int a0 = 0; a0 < MAX_ATTEMPTS;) {
      const int na = (a0 == 0) ? 1 : MAX_ATTEMPTS - a0;
      CK(cudaMemsetAsync(h->cnt.as<int>() + C_NDONE, 0, sizeof(int), h->stream));
      if (h->sd) {  // binary64 dstqds in the reference order, segmented chains (kernels_sd.cuh)
        const long long T = 2LL * na * nc;
        int K = std::max(1, h->segsd_k);
        while (K > 1 && nbmax - 1 < 2LL * K * h->segy_w) K /= 2;  // segments at least two warm-ups long
        CK(h->segsd.ensure(sizeof(SegSD) * T * K));
        CK(cudaMemsetAsync(h->cnt.as<int>() + C_NFB, 0, sizeof(int), h->stream));
        k_sd_seg<<<nblocks_for(T * K, 128), 128, 0, h->stream>>>(cl, h->reps.as<RepDesc>(), h->my.as<YElt>(),
                                                                 h->ss.as<ShiftState>(), T, a0, na, K, h->segy_w,
                                                                 h->segsd.as<SegSD>(), nullptr, nullptr, 0, 0);
        k_sd_seg_combine<<<nblocks_for(T, 64), 64, 0, h->stream>>>(
            cl, h->reps.as<RepDesc>(), h->my.as<YElt>(), h->ss.as<ShiftState>(), T, a0, na, K, h->segsd.as<SegSD>(),
            h->gval.as<double>(), h->valid.as<int>(), nullptr, nullptr, 0, 0, 0, h->cnt.as<int>() + C_NFB);
      } else if (h->segy_k > 1) {  // growth chains split into verified segments (latency: n/K + W rows per thread)
        const int K = h->segy_k;
        const long long T = 2LL * na * nc;
        CK(h->segoutg.ensure(sizeof(SegG) * T * K));
        k_clu_attempt_seg<<<nblocks_for(T * K, 128), 128, 0, h->stream>>>(
            cl, nc, h->reps.as<RepDesc>(), h->mq.as<QElt>(), h->ss.as<ShiftState>(), a0, na, K, h->segy_w,
            h->segoutg.as<SegG>());
        k_clu_attempt_combine<<<nblocks_for(T, 64), 64, 0, h->stream>>>(
            cl, nc, h->reps.as<RepDesc>(), h->my.as<YElt>(), h->mq.as<QElt>(), h->ss.as<ShiftState>(), a0, na, K,
            h->segoutg.as<SegG>(), h->gval.as<double>(), h->valid.as<int>());
      } else {
        k_clu_attempt_multi<<<nblocks_for(2LL * na * nc, 64), 64, 0, h->stream>>>(
            cl, nc, h->reps.as<RepDesc>(), h->my.as<YElt>(), h->mq.as<QElt>(), h->ss.as<ShiftState>(), a0, na,
            h->gval.as<double>(), h->valid.as<int>());
      }
      launch_check(h);
      k_clu_select_multi<<<nblocks_for(nc, 128), 128, 0, h->stream>>>(
          cl, nc, h->reps.as<RepDesc>(), h->ss.as<ShiftState>(), h->gval.as<double>(), h->valid.as<int>(), a0, na,
          h->cnt.as<int>() + C_NDONE, h->stats.as<long long>(), h->sd ? 0x1p29 : 0x1p51);
      launch_check(h);
      read_counters(h);
      if (h->h_cnt[C_NDONE] >= nc) break;
      a0 += na;
    }
    // (d) children
    if (h->sd) {
      int K = std::max(1, h->segsd_k);
      while (K > 1 && nbmax - 1 < 2LL * K * h->segy_w) K /= 2;
      CK(h->segsd.ensure(sizeof(SegSD) * (long long)nc * K));
      CK(cudaMemsetAsync(h->cnt.as<int>() + C_NFB, 0, sizeof(int), h->stream));
      k_sd_seg<<<nblocks_for((long long)nc * K, 128), 128, 0, h->stream>>>(
          cl, h->reps.as<RepDesc>(), h->my.as<YElt>(), h->ss.as<ShiftState>(), nc, 0, 0, K, h->segy_w,
          h->segsd.as<SegSD>(), h->mx.as<double2>(), h->my.as<YElt>(), poolbase, (int)nbmax);
      k_sd_seg_combine<<<nblocks_for(nc, 64), 64, 0, h->stream>>>(
          cl, h->reps.as<RepDesc>(), h->my.as<YElt>(), h->ss.as<ShiftState>(), nc, 0, 0, K, h->segsd.as<SegSD>(),
          nullptr, nullptr, h->mx.as<double2>(), h->my.as<YElt>(), repbase, poolbase, (int)nbmax,
          h->cnt.as<int>() + C_NFB);
    } else if (h->segy_k > 1) {  // child rows built by verified segments (latency n/K + W rows per thread)
      const int K = h->segy_k;
      CK(h->segoutg.ensure(sizeof(SegG) * (long long)nc * K));
      const size_t bsb = (size_t)128 * 2 * BG * (sizeof(YElt) + sizeof(double2));
      static bool bsb_set = false;
      if (!bsb_set) {
        CK(cudaFuncSetAttribute(k_clu_build_seg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsb));
        bsb_set = true;
      }
      k_clu_build_seg<<<nblocks_for((long long)nc * K, 128), 128, bsb, h->stream>>>(
          cl, nc, h->reps.as<RepDesc>(), h->ss.as<ShiftState>(), h->mx.as<double2>(), h->my.as<YElt>(),
          h->mq.as<QElt>(), poolbase, (int)nbmax, K, h->segy_w, h->segoutg.as<SegG>());
      CK(cudaMemsetAsync(h->cnt.as<int>() + C_NFB, 0, sizeof(int), h->stream));
      k_clu_build_combine<<<nblocks_for(nc, 64), 64, 0, h->stream>>>(
          cl, nc, h->reps.as<RepDesc>(), h->ss.as<ShiftState>(), h->mx.as<double2>(), h->my.as<YElt>(),
          h->mq.as<QElt>(), repbase, poolbase, (int)nbmax, K, h->segoutg.as<SegG>(), h->cnt.as<int>() + C_NFB);
    } else {
      k_clu_build<<<nblocks_for(nc, 64), 64, 0, h->stream>>>(cl, nc, h->reps.as<RepDesc>(), h->ss.as<ShiftState>(),
                                                             h->mx.as<double2>(), h->my.as<YElt>(), h->mq.as<QElt>(),
                                                             repbase, poolbase, (int)nbmax);
    }
    launch_check(h);
    k_build_q<<<dim3(nc, (unsigned)std::min<long long>(64, std::max<long long>(1, (nbmax + 255) / 256 / std::max(1, nc / 148 + 1)))),
                256, 0, h->stream>>>(h->reps.as<RepDesc>(), nullptr, repbase, nc, h->my.as<YElt>(),
                                         h->mq.as<QElt>());
    launch_check(h);
    // (e) child starts: segments and BNode offsets from the host copy
    std::vector<long long> seg(nc), bo(nc);
    {
      long long s1 = 0, b1 = 0;
      for (int c = 0; c < nc; c++) {
        const Cluster &C = hl[c0 + c];
        seg[c] = ipool_top + s1;
        s1 += C.q - C.p + 3;
        bo[c] = b1;
        b1 += C.q - C.p + 1;
      }
    }
    CK(h->cseg.ensure(sizeof(long long) * nc));
    CK(h->bnoff.ensure(sizeof(long long) * nc));
    CK(cudaMemcpyAsync(h->cseg.p, seg.data(), sizeof(long long) * nc, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->bnoff.p, bo.data(), sizeof(long long) * nc, cudaMemcpyHostToDevice, h->stream));
    CK(h->bnA.ensure(sizeof(BNode) * std::max<long long>(btot, 1)));
    CK(h->bnB.ensure(sizeof(BNode) * std::max<long long>(btot, 1)));
    CK(h->ex.ensure(sizeof(ExplicitChain) * 2 * btot + 64));
    CK(h->excounts.ensure(sizeof(int) * 2 * btot + 64));
    CK(h->exmap.ensure(sizeof(int) * 2 * btot + 64));
    CK(h->nodesA.ensure(sizeof(Node) * std::max<long long>(btot, 1)));
    CK(h->nodesB.ensure(sizeof(Node) * std::max<long long>(btot, 1)));
    // BNodes of failed clusters are never written: mark them as finished by pre-filling
    CK(cudaMemsetAsync(h->bnA.p, 0, sizeof(BNode) * btot, h->stream));
    k_clu_child_starts<<<nblocks_for(nc, 64), 64, 0, h->stream>>>(
        cl, nc, h->reps.as<RepDesc>(), h->ss.as<ShiftState>(), h->cseg.as<long long>(), h->bnoff.as<long long>(), ilo,
        ihi, h->ipool_lo.as<double>(), h->ipool_hi.as<double>(), h->bnA.as<BNode>(), repbase,
        h->yref_lo.as<double>(), h->yref_hi.as<double>(), h->sd ? 0x1p-53 : EPS_Y);
    launch_check(h);
    h->cur_nbmax = nbmax;  // chain-length hint for the segmented child counts
    int nrd = run_brackets<false>(h, (int)btot);
    run_bisection<false>(h, nrd, h->ipool_lo.as<double>(), h->ipool_hi.as<double>(), 1e-2 * h->gaptol, 0, nullptr, 0,
                         &dummy, repbase, nc);
    h->cur_nbmax = 0;
    // (f) reclassify
    CK(h->sing.ensure(sizeof(Singleton) * std::max<long long>(btot, 1)));
    Buf NXloc;
    Buf &NX = keep ? h->lvl_NX[level] : NXloc;
    CK(NX.ensure(sizeof(Cluster) * std::max<long long>(btot, 1)));
    zero_counters(h);
    k_clu_classify<<<nblocks_for(nc, 64), 64, 0, h->stream>>>(
        cl, nc, h->reps.as<RepDesc>(), h->ss.as<ShiftState>(), h->cseg.as<long long>(), ilo, ihi,
        h->ipool_lo.as<double>(), h->ipool_hi.as<double>(), h->colmap.as<int>(), h->gaptol, repbase,
        h->sing.as<Singleton>(), h->cnt.as<int>() + C_NSING, NX.as<Cluster>(), h->cnt.as<int>() + C_NNXT,
        diag ? h->dgf.as<int>() : nullptr, diag ? h->dgl.as<int>() : nullptr, (int)kout, h->stats.as<long long>());
    launch_check(h);
    read_counters(h);
    int ns = h->h_cnt[C_NSING], nnx = h->h_cnt[C_NNXT];
    // child frames: the segmented passes with the dd twist search when the child representations are shared
    // by enough singletons for their row loads to coincide (else each lane streams its own representation
    // from HBM and the two-lane kernel is faster: measured C3, 2 singletons per child, vs C4, up to 256)
    // (single/double: always the segmented passes -- their fixed passes run in binary64, k_rqi2 in dd)
    const bool segq = h->sd || (h->rqi_seg_child && ns >= (long long)h->segchild_min * nc);
    if (ns > 0 && !segq && h->defer_tail && keep && tail_bytes(ns, nbmax) <= h->tail_max_bytes) {
      // few singletons per child, two-lane kernel only: a deferred tail on the side stream, overlapping the
      // deeper levels and the RQI of the levels above (C4: the depth-2 pair under the depth-1 passes)
      launch_tail(h, ns, nbmax, W, Z, ldz);
      process_clusters(h, NX.as<Cluster>(), nnx, repbase + nc, poolbase + (long long)nc * nbmax, ipool_top + stot,
                       nbmax, true, W, Z, ldz, kout, level + 1);
    } else if (ns > 0 && nnx > 0 && h->defer_tail && keep) {
      // deeper levels first (a tail found there overlaps this level's passes), then this level's singletons
      // from a copy of their list (the recursion rewrites h->sing); the results do not depend on the order
      Buf &SG = h->lvl_SG[level];
      CK(SG.ensure(sizeof(Singleton) * ns));
      CK(cudaMemcpyAsync(SG.p, h->sing.p, sizeof(Singleton) * ns, cudaMemcpyDeviceToDevice, h->stream));
      process_clusters(h, NX.as<Cluster>(), nnx, repbase + nc, poolbase + (long long)nc * nbmax, ipool_top + stot,
                       nbmax, true, W, Z, ldz, kout, level + 1);
      run_rqi(h, ns, nbmax, W, Z, ldz, segq, true, SG.as<Singleton>());
    } else {
      run_rqi(h, ns, nbmax, W, Z, ldz, segq, true);
      process_clusters(h, NX.as<Cluster>(), nnx, repbase + nc, poolbase + (long long)nc * nbmax, ipool_top + stot,
                       nbmax, true, W, Z, ldz, kout, level + 1);
    }
    CK(cudaStreamSynchronize(h->stream));
    if (!keep) {
      NX.release();
      L.release();
    }
  }
}

// ownership rule of a multi-GPU shard within the selection [il, iu]: an owned unit
// starts at every root group start inside [il, iu] and at il itself (a group that begins before il
// is cut there, as the 1-GPU solve cuts it with its column map); the rank owns every unit that
// STARTS in its shard [sl, su], and the last such unit may extend past su (through min(jmax, iu),
// jmax = the end of the computed range).  The owned ranges of the ranks therefore partition
// [il, iu].  gstart[j-1] = 1 iff index j starts a root group.  Empty ownership: jlo = su + 1, jhi = su.
static void shard_owner(const int32_t *gstart, long long n, long long il, long long iu, long long sl,
                        long long su, long long jmax, long long *jlo_out, long long *jhi_out) {
  long long jlo = -1, jhi;
  const long long jend = std::min(std::min(jmax, iu), n);
  auto unit_start = [&](long long j) { return j == il || gstart[j - 1] == 1; };
  for (long long j = sl; j <= su; j++)
    if (unit_start(j)) { jlo = j; break; }
  if (jlo > 0) {
    long long last = jlo;
    for (long long j = sl; j <= su; j++)
      if (unit_start(j)) last = j;
    jhi = last;
    while (jhi < jend && gstart[jhi] == 0) jhi++;
  } else {
    jlo = su + 1;
    jhi = su;
  }
  *jlo_out = jlo;
  *jhi_out = jhi;
}

int solve(mrrr_t h, const double *d, const double *e, long long n, long long il, long long iu, double *W, double *Z,
          long long ldz, long long shard_lo, long long shard_hi, long long *jlo_out, long long *jhi_out,
          long long ncols_cap) {
  cudaStream_t st = h->stream;
  const bool shard = shard_lo > 0;
  const long long k = iu - il + 1;
  h->last_n = n;
  h->last_k = k;
  h->host_rounds = h->host_launches = 0;
  h->nonlocal = false;
  h->rqi_ms = 0;
  h->rqi_launches = 0;
  h->neg_ms = 0;
  h->neg_launches = 0;
  h->ntev = 0;
  h->tneg.clear();
  h->trq.clear();
  h->times_dirty = false;
  memset(h->stats_h, 0, sizeof(h->stats_h));
  bool diag = (h->flags & MRRR_KEEP_DIAG) != 0;

  CK(h->starts.ensure(sizeof(int) * (n + 2)));
  CK(h->scal.ensure(64));
  CK(h->cnt.ensure(sizeof(int) * C_NCOUNTERS));
  if (h->tail_pending) CK(cudaStreamSynchronize(h->s_tail));  // (a solve that threw may have left one running)
  CK(h->stats.ensure(sizeof(long long) * ST_N));
  CK(cudaMemsetAsync(h->stats.p, 0, sizeof(long long) * ST_N, st));
  CK(cudaEventRecord(h->ev[0], st));

  // S1/S2 (and the S0 scale test: the largest |entry| comes out of the same pass)
  struct ScalRec { int nblk, err; double tnorm, amax; };
  const double eps_split = h->sd ? 0x1p-24 : EPS_X;  // eps_x of the split rule
  k_split<1024><<<1, 1024, 0, st>>>(d, e, n, h->starts.as<int>(), h->scal.as<int>(), (double *)(h->scal.as<char>() + 8),
                                    h->scal.as<int>() + 1, (double *)(h->scal.as<char>() + 16), eps_split);
  launch_check(h);
  ScalRec hs;
  static_assert(sizeof(ScalRec) <= 64 * sizeof(int), "pinned scratch");
  CK(cudaMemcpyAsync(h->h_small, h->scal.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  memcpy(&hs, h->h_small, sizeof(hs));
  if (hs.err) return MRRR_ERR_NONFINITE;
  // S0 scaling (A-21): max |entry| outside [2^-500, 2^500] -> solve 2^-ex T (exact power of two,
  // max |entry| in [1/2, 1)) and scale W back at the end; Z is scale invariant
  int scale_ex = 0;
  if (hs.amax != 0.0 && (hs.amax < 0x1p-500 || hs.amax > 0x1p500)) {
    std::frexp(hs.amax, &scale_ex);
    CK(h->hd2.ensure(sizeof(double) * 2 * n));
    double *ds = h->hd2.as<double>(), *es = ds + n;
    k_scale2<<<nblocks_for(n, 256), 256, 0, st>>>(d, ds, n, -scale_ex);
    if (n > 1) k_scale2<<<nblocks_for(n - 1, 256), 256, 0, st>>>(e, es, n - 1, -scale_ex);
    d = ds;
    e = es;
    k_split<1024><<<1, 1024, 0, st>>>(d, e, n, h->starts.as<int>(), h->scal.as<int>(),
                                      (double *)(h->scal.as<char>() + 8), h->scal.as<int>() + 1,
                                      (double *)(h->scal.as<char>() + 16), eps_split);
    launch_check(h);
    CK(cudaMemcpyAsync(h->h_small, h->scal.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    memcpy(&hs, h->h_small, sizeof(hs));
  }
  struct ScaleBack {  // W of the computed columns back to the input's scale on every successful return path
    mrrr_t h; double *W; long long cnt; int ex;
    void run() { if (ex && cnt > 0) k_scale2<<<nblocks_for(cnt, 256), 256, 0, h->stream>>>(W, W, cnt, ex); }
  } scale_back{h, W, 0, scale_ex};
  const int nblk = hs.nblk;
  h->last_nblk = nblk;
  h->h_starts.assign(nblk + 1, 0);
  if (nblk == 1) { h->h_starts[0] = 0; h->h_starts[1] = (int)n; }
  else CK(cudaMemcpy(h->h_starts.data(), h->starts.p, sizeof(int) * (nblk + 1), cudaMemcpyDeviceToHost));
  const bool single = (nblk == 1);
  if (shard && !single) { g_last_cuda_error = "shards of split matrices are not supported"; return MRRR_ERR_CUDA; }

  // per-block side / computed ranges (S3/S4)
  std::vector<int> bside(nblk, 1), cab(2 * nblk), blist;
  long long nbmax = 1, ncomp = 0;
  for (int b = 0; b < nblk; b++) {
    int nb = h->h_starts[b + 1] - h->h_starts[b];
    nbmax = std::max<long long>(nbmax, nb);
    long long jl = 1, ju = nb;
    if (single) {
      jl = shard ? shard_lo : il;
      ju = shard ? shard_hi : iu;
    }
    bool left = (h->root_side == 1) ? true : (h->root_side == 2) ? false : ((jl - 1) <= (nb - ju));
    if (shard && h->root_side == 0) left = (il - 1) <= (n - iu);  // every rank must build the same root
    bside[b] = left ? 1 : 2;
    long long ca = jl, cb = ju;
    if (single && nb > 1) { ca = (jl > 1) ? jl - 1 : jl; cb = (ju < nb) ? ju + 1 : ju; }
    cab[2 * b] = (int)ca;
    cab[2 * b + 1] = (int)cb;
    if (nb > 1) { blist.push_back(b); ncomp += cb - ca + 1; }
  }
  const int nbl = (int)blist.size();
  CK(h->bside.ensure(sizeof(int) * nblk));
  CK(h->cab.ensure(sizeof(int) * 2 * nblk));
  CK(h->blist.ensure(sizeof(int) * std::max(nbl, 1)));
  CK(h->binfo.ensure(sizeof(double) * 16 * nblk));
  CK(cudaMemcpyAsync(h->bside.p, bside.data(), sizeof(int) * nblk, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(h->cab.p, cab.data(), sizeof(int) * 2 * nblk, cudaMemcpyHostToDevice, st));
  if (nbl) CK(cudaMemcpyAsync(h->blist.p, blist.data(), sizeof(int) * nbl, cudaMemcpyHostToDevice, st));

  // pools: root reps at [0, n); children appended (sized by the workspace budget)
  CK(h->mx.ensure(sizeof(double2) * (n + 1)));
  CK(h->my.ensure(sizeof(YElt) * (n + 1)));
  CK(h->mq.ensure(sizeof(QElt) * (n + 1)));
  CK(h->lscratch.ensure(sizeof(double) * 2 * n));
  CK(h->reps.ensure(sizeof(RepDesc) * (nblk + 1)));
  CK(h->rlo.ensure(sizeof(double) * n));
  CK(h->rhi.ensure(sizeof(double) * n));
  CK(h->colmap.ensure(sizeof(int) * n));
  CK(h->gstart.ensure(sizeof(int) * n));
  if (diag) {
    CK(h->ddepth.ensure(sizeof(int) * k));
    CK(h->dgf.ensure(sizeof(int) * MAXD * k));
    CK(h->dgl.ensure(sizeof(int) * MAXD * k));
    CK(h->dflo.ensure(sizeof(double) * k));
    CK(h->dfhi.ensure(sizeof(double) * k));
    k_fill_i<<<nblocks_for(MAXD * k, 256), 256, 0, st>>>(h->dgf.as<int>(), MAXD * k, -1);
    k_fill_i<<<nblocks_for(MAXD * k, 256), 256, 0, st>>>(h->dgl.as<int>(), MAXD * k, -1);
  }
  k_fill<<<nblocks_for(n, 256), 256, 0, st>>>(h->rlo.as<double>(), n, NAN);
  k_fill<<<nblocks_for(n, 256), 256, 0, st>>>(h->rhi.as<double>(), n, NAN);
  launch_check(h);

  // S3 root
  if (nbl) {
    // long blocks: the Gershgorin reduction and the representation rows over G CTAs per block (k_root
    // keeps the serial chain)
    const int G = n >= 32768 ? (int)std::min<long long>(64, n / 4096) : 0;
    if (G > 1) {
      CK(h->gpart.ensure(sizeof(double) * 2 * (size_t)nbl * G));
      k_root_gersh<256><<<dim3(nbl, G), 256, 0, st>>>(d, e, h->starts.as<int>(), h->blist.as<int>(), G,
                                                      h->gpart.as<double>());
      launch_check(h);
    }
    k_root<256><<<nbl, 256, 0, st>>>(d, e, n, h->starts.as<int>(), h->blist.as<int>(), h->bside.as<int>(), h->seed,
                                     h->binfo.as<double>(), h->mx.as<double2>(), h->my.as<YElt>(),
                                     h->lscratch.as<double>(), h->reps.as<RepDesc>(),
                                     G > 1 ? h->gpart.as<double>() : nullptr, G > 1 ? G : 0, h->sd ? 1 : 0);
    launch_check(h);
    if (G > 1) {
      k_root_derive<256><<<dim3(nbl, G), 256, 0, st>>>(n, h->starts.as<int>(), h->blist.as<int>(), h->seed,
                                                       h->binfo.as<double>(), h->mx.as<double2>(), h->my.as<YElt>(),
                                                       h->lscratch.as<double>(), G, h->sd ? 1 : 0);
      launch_check(h);
    }
    k_build_q<<<dim3(nbl, (unsigned)std::min<long long>(64, std::max<long long>(1, (n + 255) / 256 / std::max(1, nbl / 148 + 1)))),
                256, 0, st>>>(h->reps.as<RepDesc>(), h->blist.as<int>(), 0, nbl, h->my.as<YElt>(),
                                   h->mq.as<QElt>());
    launch_check(h);
  }
  CK(cudaEventRecord(h->ev[1], st));

  // S5 root bisection
  const double rtol = 1e-2 * h->gaptol;
  // k-section budget: few wanted indices (a rank's shard) -> the smaller budget (3 levels per round for
  // ~1K nodes instead of 4: less speculation where the rounds are throughput-bound anyway)
  const long long tc_saved = h->target_chains;
  if (ncomp < 4096 && h->target_chains_small > 0) h->target_chains = std::min(h->target_chains, h->target_chains_small);
  struct RestoreTC {
    mrrr_t h;
    long long v;
    ~RestoreTC() { h->target_chains = v; }
  } restore_tc{h, tc_saved};
  // S5' early classification stop (MRRR_EARLY_STOP, A-41): stage 1 bisects to rtol_c into s1lo/s1hi
  // (the computed set and one neighbour on each side), k_es_decide keeps the stopped intervals and runs the
  // others on from their stage-1 nodes to rtol (the same paths, so the same intervals as without the stop)
  const bool es = (h->flags & MRRR_EARLY_STOP) != 0;
  double rtol_c = rtol;
  if (es) {
    int ex = 0;
    while (ex < 62 && (1LL << ex) < n) ex++;  // ceil(log2 n), as oracle_es_rtol
    rtol_c = std::max(rtol, std::ldexp(1.0, -(10 + ex)));
    CK(h->s1lo.ensure(sizeof(double) * n));
    CK(h->s1hi.ensure(sizeof(double) * n));
    k_fill<<<nblocks_for(n, 256), 256, 0, st>>>(h->s1lo.as<double>(), n, NAN);
    k_fill<<<nblocks_for(n, 256), 256, 0, st>>>(h->s1hi.as<double>(), n, NAN);
    launch_check(h);
  }
  double *b1lo = es ? h->s1lo.as<double>() : h->rlo.as<double>(), *b1hi = es ? h->s1hi.as<double>() : h->rhi.as<double>();
  auto es_stage2 = [&](const std::vector<EsRange> &rg0) {
    std::vector<EsRange> rg;
    int total = 0;
    for (EsRange r : rg0)
      if (r.jb >= r.ja) { r.off = total; total += r.jb - r.ja + 1; rg.push_back(r); }
    if (total == 0) return;
    CK(h->esr.ensure(sizeof(EsRange) * rg.size()));
    CK(cudaMemcpyAsync(h->esr.p, rg.data(), sizeof(EsRange) * rg.size(), cudaMemcpyHostToDevice, st));
    h->max_nodes = std::max(h->max_nodes, total + 2);
    CK(h->nodesA.grow_keep(sizeof(Node) * (size_t)h->max_nodes, 0, st));
    CK(h->nodesB.grow_keep(sizeof(Node) * (size_t)h->max_nodes, 0, st));
    zero_counters(h);
    k_es_decide<<<nblocks_for(total, 128), 128, 0, st>>>(h->esr.as<EsRange>(), (int)rg.size(), total,
                                                         h->starts.as<int>(), h->s1lo.as<double>(),
                                                         h->s1hi.as<double>(), h->rlo.as<double>(),
                                                         h->rhi.as<double>(), h->gaptol, h->nodesA.as<Node>(),
                                                         h->cnt.as<int>() + C_NNEXT, h->stats.as<long long>());
    launch_check(h);
    read_counters(h);
    const int nn2 = h->h_cnt[C_NNEXT];
    if (nn2 > 0) {
      // stage 2 holds few nodes (C2: ~1,100 of 8,192) for ~17 levels: latency-bound rounds, so fewer k-section
      // points per node and shorter segments than the throughput rounds of stage 1
      struct Keep {
        mrrr_t h; long long tc; int ml;
        ~Keep() { h->target_chains = tc; h->seg_minlen = ml; }
      } keep{h, h->target_chains, h->seg_minlen};
      if (h->es2_target > 0) h->target_chains = h->es2_target;
      if (h->es2_minlen > 0) h->seg_minlen = h->es2_minlen;
      bool rs = false;
      run_bisection<false>(h, nn2, h->rlo.as<double>(), h->rhi.as<double>(), rtol, 0, nullptr, 0, &rs, -1, 0,
                           single ? (int)n : 0);
    }
  };
  if (nbl) {
    long long cap = std::max<long long>(ncomp + 2, nbl);
    h->max_nodes = (int)cap;
    CK(h->nodesA.ensure(sizeof(Node) * cap));
    CK(h->nodesB.ensure(sizeof(Node) * cap));
    CK(h->ex.ensure(sizeof(ExplicitChain) * (nbl + 64)));
    CK(h->excounts.ensure(sizeof(int) * (nbl + 64)));
    // a single block's subset (or shard) bisects GUARD_MARGIN indices beyond each guard in the same run, so that
    // a cluster that straddles the edge is usually covered without a guard-extension pass (the indices the
    // extension rule does not reach are reset to "not computed" below)
    const int GUARD_MARGIN = 32;
    std::vector<int> cabm = cab;
    if (single && nbl) {
      if (cab[0] > 1) cabm[0] = std::max(1, cab[0] - GUARD_MARGIN);
      if (cab[1] < (int)n) cabm[1] = std::min((int)n, cab[1] + GUARD_MARGIN);
    }
    std::vector<int> cabs = cabm;  // stage-1 range: with the early stop, one decision neighbour on each side
    if (es && single && nbl) {
      cabs[0] = std::max(1, cabm[0] - 1);
      cabs[1] = std::min((int)n, cabm[1] + 1);
    }
    if (cabs != cab) {
      h->max_nodes = std::max<int>(h->max_nodes, cabs[1] - cabs[0] + 3);
      CK(h->nodesA.grow_keep(sizeof(Node) * (size_t)h->max_nodes, 0, st));
      CK(h->nodesB.grow_keep(sizeof(Node) * (size_t)h->max_nodes, 0, st));
      CK(cudaMemcpyAsync(h->cab.p, cabs.data(), sizeof(int) * 2, cudaMemcpyHostToDevice, st));
    }
    for (int attempt = 0; attempt < 64; attempt++) {
      k_root_nodes<<<nblocks_for(nbl, 128), 128, 0, st>>>(h->blist.as<int>(), nbl, h->starts.as<int>(),
                                                          h->binfo.as<double>(), h->cab.as<int>(), h->nodesA.as<Node>(),
                                                          h->ex.as<ExplicitChain>());
      launch_check(h);
      bool restart = false;
      run_bisection<false>(h, nbl, b1lo, b1hi, es ? rtol_c : rtol, nbl, h->blist.as<int>(), nbl, &restart, -1, 0,
                           single ? (int)n : 0);
      if (!restart) break;
    }
    if (es) {
      std::vector<EsRange> rg;
      if (single) rg.push_back({0, cabm[0], cabm[1], 0});
      else
        for (int b : blist) rg.push_back({b, 1, h->h_starts[b + 1] - h->h_starts[b], 0});
      es_stage2(rg);
    }
    if (cabs != cab) CK(cudaMemcpyAsync(h->cab.p, cab.data(), sizeof(int) * 2, cudaMemcpyHostToDevice, st));
    // root definiteness
    std::vector<double> hb(16 * nblk);
    CK(cudaMemcpy(hb.data(), h->binfo.p, sizeof(double) * 16 * nblk, cudaMemcpyDeviceToHost));
    for (int b : blist) {
      if (hb[16 * b + 8] == 0.0) return MRRR_ERR_ROOT;
      h->stats_h[ST_ROOT_BACKOFF] += (long long)hb[16 * b + 7];
    }
    // guard extension (single block, S5): the oracle bisects one more index at a time while the outermost
    // computed index is not separated from its inner neighbour.  Here the indices beyond each unseparated end are
    // bisected in doubling batches (1, 2, 4, ... indices in one shared-tree run), k_guard_scan walks their
    // boundaries outward from the old end exactly as the one-at-a-time rule does, and the indices the rule never
    // reaches are reset to "not computed" -- the same computed set and intervals, in O(log) passes instead of one
    // pass per index of a cluster that straddles a subset or shard edge (255 passes in C4's clusters)
    if (single && nbl) {
      int nb = (int)n;
      int step[2] = {256, 256};  // extension batches: 256 indices per side, then doubling
      int far[2] = {cabm[0], cabm[1]};  // outermost computed index per side (margin and batches overshoot the rule)
      for (int it = 0; it < 64; it++) {
        // walk outward from the current ends over the computed indices: the one-at-a-time rule's stopping point
        CK(cudaMemcpyAsync(h->cab.p, cab.data(), sizeof(int) * 2, cudaMemcpyHostToDevice, st));
        k_guard_scan<<<1, 1, 0, st>>>(h->cab.as<int>(), far[0], far[1], h->rlo.as<double>(), h->rhi.as<double>(),
                                      nb, h->gaptol);
        launch_check(h);
        CK(cudaMemcpyAsync(cab.data(), h->cab.p, sizeof(int) * 2, cudaMemcpyDeviceToHost, st));
        k_guard_check<<<1, 1, 0, st>>>(h->cab.as<int>(), h->rlo.as<double>(), h->rhi.as<double>(), nb, h->gaptol,
                                       h->cnt.as<int>() + 8);
        launch_check(h);
        read_counters(h);
        const bool need[2] = {h->h_cnt[8] != 0, h->h_cnt[9] != 0};
        if (!need[0] && !need[1]) break;
        // both sides' batches beyond the computed extents, in one shared-tree run
        int w[4] = {0, -1, 0, -1}, nn = 0;
        for (int side = 0; side < 2; side++) {
          if (!need[side]) continue;
          const int a = side ? far[1] + 1 : std::max(1, far[0] - step[0]);
          const int b = side ? std::min(nb, far[1] + step[1]) : far[0] - 1;
          step[side] *= 2;
          if (a > b) continue;
          w[2 * nn] = a;
          w[2 * nn + 1] = b;
          nn++;
          far[side] = side ? b : a;
        }
        if (nn > 0) {
          // node capacity: every index of the batches may separate
          h->max_nodes = std::max(h->max_nodes, (w[1] - w[0] + 1) + (w[3] - w[2] + 1) + 2);
          CK(h->nodesA.grow_keep(sizeof(Node) * (size_t)h->max_nodes, 0, st));
          CK(h->nodesB.grow_keep(sizeof(Node) * (size_t)h->max_nodes, 0, st));
          // early stop: stage 1 of the batches and their decision neighbours, then the decisions and stage 2
          int we[4] = {w[0], w[1], w[2], w[3]};
          if (es)
            for (int q = 0; q < nn; q++) { we[2 * q] = std::max(1, w[2 * q] - 1); we[2 * q + 1] = std::min(nb, w[2 * q + 1] + 1); }
          h->max_nodes = std::max(h->max_nodes, (we[1] - we[0] + 1) + (we[3] - we[2] + 1) + 2);
          CK(h->nodesA.grow_keep(sizeof(Node) * (size_t)h->max_nodes, 0, st));
          CK(h->nodesB.grow_keep(sizeof(Node) * (size_t)h->max_nodes, 0, st));
          k_guard_nodes<<<1, nn, 0, st>>>(h->starts.as<int>(), h->binfo.as<double>(), we[0], we[1], we[2], we[3],
                                          h->nodesA.as<Node>());
          launch_check(h);
          bool rs = false;
          run_bisection<false>(h, nn, b1lo, b1hi, es ? rtol_c : rtol, 0, nullptr, 0, &rs, -1, 0, nb);
          if (es) {
            std::vector<EsRange> rg;
            for (int q = 0; q < nn; q++) rg.push_back({0, w[2 * q], w[2 * q + 1], 0});
            es_stage2(rg);
          }
        }
      }
      CK(cudaMemcpyAsync(h->cab.p, cab.data(), sizeof(int) * 2, cudaMemcpyHostToDevice, st));
      // indices a batch computed beyond the rule's stopping point: not computed (as in the oracle)
      if (far[0] < cab[0]) {
        k_fill<<<nblocks_for(cab[0] - far[0], 256), 256, 0, st>>>(h->rlo.as<double>() + far[0] - 1, cab[0] - far[0], NAN);
        k_fill<<<nblocks_for(cab[0] - far[0], 256), 256, 0, st>>>(h->rhi.as<double>() + far[0] - 1, cab[0] - far[0], NAN);
      }
      if (far[1] > cab[1]) {
        k_fill<<<nblocks_for(far[1] - cab[1], 256), 256, 0, st>>>(h->rlo.as<double>() + cab[1], far[1] - cab[1], NAN);
        k_fill<<<nblocks_for(far[1] - cab[1], 256), 256, 0, st>>>(h->rhi.as<double>() + cab[1], far[1] - cab[1], NAN);
      }
      launch_check(h);
    }
  }
  CK(cudaEventRecord(h->ev[2], st));

  // S4/S6 selection and classification
  if (single) {
    long long lo1 = il, hi1 = iu;
    if (shard) { lo1 = 1; hi1 = n; }
    k_colmap_range<<<nblocks_for(n, 256), 256, 0, st>>>(h->colmap.as<int>(), n, lo1, hi1);
    launch_check(h);
  } else {
    Buf keys;
    CK(keys.ensure(sizeof(double) * n));
    k_rank<<<nblocks_for(n, 256), 256, 0, st>>>(d, h->starts.as<int>(), nblk, h->binfo.as<double>(),
                                                 h->rlo.as<double>(), h->rhi.as<double>(), n, keys.as<double>());
    launch_check(h);
    // rank = place in the (key, position) order: bitonic sort of the padded pairs
    long long N2 = BT;
    while (N2 < n) N2 <<= 1;
    Buf sk, si;
    CK(sk.ensure(sizeof(double) * N2));
    CK(si.ensure(sizeof(long long) * N2));
    k_rank_init<<<nblocks_for(N2, 256), 256, 0, st>>>(keys.as<double>(), n, N2, sk.as<double>(), si.as<long long>());
    const unsigned ntile = (unsigned)(N2 / BT);
    k_bitonic_tile<<<ntile, BT / 2, 0, st>>>(sk.as<double>(), si.as<long long>(), N2, 2, BT, 1);  // tiles sorted
    for (long long k = 2 * BT; k <= N2; k <<= 1) {
      long long j = k / 2;
      for (; j >= BT / 2; j >>= 1)
        k_bitonic_global<<<nblocks_for(N2 / 2, 256), 256, 0, st>>>(sk.as<double>(), si.as<long long>(), N2, k, j);
      k_bitonic_tile<<<ntile, BT / 2, 0, st>>>(sk.as<double>(), si.as<long long>(), N2, k, k, j);
    }
    k_rank_scatter<<<nblocks_for(n, 256), 256, 0, st>>>(si.as<long long>(), n, il, iu, h->colmap.as<int>());
    launch_check(h);
    CK(cudaStreamSynchronize(st));
    CK(cudaStreamSynchronize(st));
    keys.release();
  }
  k_classify_root<<<nblocks_for(n, 256), 256, 0, st>>>(h->starts.as<int>(), h->cab.as<int>(), nblk,
                                                        h->rlo.as<double>(), h->rhi.as<double>(), h->gaptol,
                                                        h->gstart.as<int>(), n);
  launch_check(h);
  if (shard) {
    // ownership: groups that START in [shard_lo, shard_hi]; owned range [jlo, jhi]
    std::vector<int> gs(n);
    CK(cudaMemcpyAsync(gs.data(), h->gstart.p, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    long long jlo = 0, jhi = 0;
    shard_owner(gs.data(), n, il, iu, shard_lo, shard_hi, cab[1], &jlo, &jhi);
    *jlo_out = jlo;
    *jhi_out = jhi;
    long long own = jhi - jlo + 1;
    if (own > ncols_cap) return MRRR_ERR_NOMEM;
    il = jlo; iu = jhi;
    if (own <= 0) { CK(cudaEventRecord(h->ev[3], st)); CK(cudaStreamSynchronize(st)); return 0; }
    k_colmap_range<<<nblocks_for(n, 256), 256, 0, st>>>(h->colmap.as<int>(), n, jlo, jhi);
    launch_check(h);
  }
  const long long kout = iu - il + 1;
  if (!single) CK(cudaMemset2DAsync(Z, sizeof(double) * ldz, 0, sizeof(double) * n, kout, st));
  CK(h->sing.ensure(sizeof(Singleton) * std::max<long long>(ncomp, 1)));
  CK(h->clusA.ensure(sizeof(Cluster) * std::max<long long>(ncomp, 1)));
  zero_counters(h);
  k_groups_root<<<nblocks_for(n, 256), 256, 0, st>>>(
      h->starts.as<int>(), nblk, h->cab.as<int>(), h->gstart.as<int>(), h->colmap.as<int>(), h->rlo.as<double>(),
      h->rhi.as<double>(), n, h->sing.as<Singleton>(), h->cnt.as<int>() + C_NSING, h->clusA.as<Cluster>(),
      h->cnt.as<int>() + C_NCLUS, diag ? h->dgf.as<int>() : nullptr, diag ? h->dgl.as<int>() : nullptr, (int)kout,
      h->stats.as<long long>());
  launch_check(h);
  read_counters(h);
  int ns = h->h_cnt[C_NSING], ncl = h->h_cnt[C_NCLUS];
  CK(cudaEventRecord(h->ev[3], st));

  // S9/S10 root singletons
  // short root blocks: the two-lane kernel directly (chains are short; oscillatory vectors such as C1's defeat the
  // segmented twist search, which would hand every singleton over after a wasted pass)
  // (single/double: always the segmented passes, whose fixed passes run in binary64; run_rqi gives them exact
  // starts where the frames are short or do not contract)
  run_rqi(h, ns, nbmax, W, Z, ldz, h->sd || (nbmax > h->rqi_seg_min && !h->nonlocal));
  CK(cudaEventRecord(h->ev[4], st));
  // S8 clusters (depth-first, chunked)
  if (ncl > 0) {
    Buf L0;
    CK(L0.ensure(sizeof(Cluster) * ncl));
    CK(cudaMemcpyAsync(L0.p, h->clusA.p, sizeof(Cluster) * ncl, cudaMemcpyDeviceToDevice, st));
    process_clusters(h, L0.as<Cluster>(), ncl, nblk, n, 0, nbmax, false, W, Z, ldz, kout, 0);
    join_tail(h);  // W and Z columns of a deferred tail are done before anything reads them
    L0.release();
  }
  if (!single || n == 1) {
    k_trivial<<<nblocks_for(nblk, 128), 128, 0, st>>>(d, h->starts.as<int>(), nblk, h->colmap.as<int>(), W, Z, ldz,
                                                      diag ? h->ddepth.as<int>() : nullptr,
                                                      diag ? h->dflo.as<double>() : nullptr,
                                                      diag ? h->dfhi.as<double>() : nullptr,
                                                      diag ? h->dgf.as<int>() : nullptr,
                                                      diag ? h->dgl.as<int>() : nullptr, h->rlo.as<double>(),
                                                      h->rhi.as<double>());
    launch_check(h);
  }
  scale_back.cnt = kout;
  scale_back.run();
  launch_check(h);
  CK(cudaEventRecord(h->ev[5], st));
  CK(cudaStreamSynchronize(st));
  // stats
  long long sd[ST_N];
  CK(cudaMemcpy(sd, h->stats.p, sizeof(sd), cudaMemcpyDeviceToHost));
  for (int i = 0; i < ST_N; i++) h->stats_h[i] += sd[i];
  h->stats_h[ST_ROUNDS] = h->host_rounds;
  h->stats_h[ST_LAUNCHES] = h->host_launches;
  h->stats_h[ST_NBLK] = nblk;
  h->times_dirty = true;  // phase and kernel times are read from the events by mrrr_get_times
  return 0;
}

int check_args(const double *d, const double *e, long long n, long long il, long long iu, const double *W,
               const double *Z, long long ldz) {
  if (!d) return -2;
  if (n > 1 && !e) return -3;
  if (n < 1) return -4;
  if (il < 1 || il > n) return -5;
  if (iu < il || iu > n) return -6;
  if (!W) return -7;
  if (!Z) return -8;
  if (ldz < n) return -9;
  return 0;
}

}  // namespace

extern "C" {

int mrrr_init(mrrr_t *out, const mrrr_opts *o) {
  if (!out) return -1;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    g_last_cuda_error = "no CUDA device";
    return MRRR_ERR_NODEVICE;
  }
  mrrr_t h = new mrrr_ctx();
  try {
    if (o && o->device >= 0) { CK(cudaSetDevice(o->device)); h->device = o->device; }
    else CK(cudaGetDevice(&h->device));
    if (o && o->stream) h->stream = (cudaStream_t)o->stream;
    else { CK(cudaStreamCreate(&h->stream)); h->own_stream = true; }  // blocking: ordered with the legacy stream
    if (o && o->gaptol > 0) h->gaptol = o->gaptol;
    if (o && o->seed) h->seed = o->seed;
    if (o) { h->root_side = o->root_side; h->flags = o->flags; }
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    h->ws_limit = (o && o->ws_limit > 0) ? o->ws_limit : (long long)(0.6 * (double)fr);
    if (const char *s = getenv("MRRR_TARGET_CHAINS")) h->target_chains = atoll(s);
    if (const char *s = getenv("MRRR_TARGET_SMALL")) h->target_chains_small = atoll(s);
    if (const char *s = getenv("MRRR_TARGET_Y")) h->target_y = atoll(s);
    if (const char *s = getenv("MRRR_TARGET_UNSEG")) h->target_unseg = atoll(s);
    if (const char *s = getenv("MRRR_TARGET_CHILD")) h->target_child = atoll(s);
    if (const char *s = getenv("MRRR_MMAX")) h->mmax = atoi(s);
    if (const char *s = getenv("MRRR_NEGTMA")) h->neg_tma = atoi(s) != 0;
    if (const char *s = getenv("MRRR_GROUPED")) h->grouped = atoi(s) != 0;
    if (const char *s = getenv("MRRR_SEGK")) h->seg_k = std::max(1, std::min(64, atoi(s)));
    if (const char *s = getenv("MRRR_SEGW")) h->seg_w = std::max(1, atoi(s));
    if (const char *s = getenv("MRRR_DEVROUNDS")) h->dev_rounds = atoi(s) != 0;
    if (const char *s = getenv("MRRR_DEVSTABLE")) h->dev_stable = atoi(s) != 0;
    if (const char *s = getenv("MRRR_DEVFRAC")) h->dev_frac = std::max(1, atoi(s));
    if (const char *s = getenv("MRRR_DEVRB")) h->dev_rb = std::max(1, std::min(64, atoi(s)));
    if (const char *s = getenv("MRRR_RQISEG")) h->rqi_seg = atoi(s) != 0;
    if (const char *s = getenv("MRRR_RQISEGK")) h->rqi_segk = std::max(1, std::min(64, atoi(s)));
    if (const char *s = getenv("MRRR_RQISEGW")) h->rqi_segw = std::max(1, atoi(s));
    if (const char *s = getenv("MRRR_RQIBULK")) h->rqi_bulk = atoi(s) != 0;
    if (const char *s = getenv("MRRR_RQITHREADS")) h->rqi_threads = atoll(s);
    if (const char *s = getenv("MRRR_TWDD_ROOT")) h->twdd_root_max = atoll(s);
    if (const char *s = getenv("MRRR_RQISEGCHILD")) h->rqi_seg_child = atoi(s) != 0;
    if (const char *s = getenv("MRRR_SEGCHILDMIN")) h->segchild_min = atoi(s);
    if (const char *s = getenv("MRRR_DEFER_TAIL")) h->defer_tail = atoi(s) != 0;
    if (const char *s = getenv("MRRR_SYNCCHECK")) h->synccheck = atoi(s) != 0;
    if (const char *s = getenv("MRRR_SEGTHREADS")) h->seg_threads = atoll(s);
    if (const char *s = getenv("MRRR_SEGMINLEN")) h->seg_minlen = atoi(s);
    if (const char *s = getenv("MRRR_FUSEM")) h->fuse_mmax = atoi(s);
    if (const char *s = getenv("MRRR_ZWIN")) h->zwin = std::max(0, atoi(s));
    if (const char *s = getenv("MRRR_ZRC_CHILD")) h->zrc_child = atoi(s) != 0;
    if (const char *s = getenv("MRRR_ROUNDEV")) h->round_ev = atoi(s) != 0;
    if (const char *s = getenv("MRRR_EARLY_STOP")) { if (atoi(s)) h->flags |= MRRR_EARLY_STOP; }  // dev sweeps
    if (const char *s = getenv("MRRR_FULL_SUPPORT")) { if (atoi(s)) h->flags |= MRRR_FULL_SUPPORT; }
    if (const char *s = getenv("MRRR_ES2_TARGET")) h->es2_target = atoll(s);
    if (const char *s = getenv("MRRR_ES2_MINLEN")) h->es2_minlen = atoi(s);
    if (const char *s = getenv("MRRR_SEGCH2")) h->seg_ch2 = atoll(s);
    if (const char *s = getenv("MRRR_RECSTAGE")) h->rec_stage = atoi(s) != 0;
    if (const char *s = getenv("MRRR_SEGYK")) h->segy_k = std::max(1, std::min(64, atoi(s)));
    if (const char *s = getenv("MRRR_SEGYW")) h->segy_w = std::max(1, atoi(s));
    if (const char *s = getenv("MRRR_SEGXK")) h->segx_k = std::max(1, std::min(64, atoi(s)));
    if (const char *s = getenv("MRRR_SEGXW")) h->segx_w = std::max(1, atoi(s));
    if (const char *s = getenv("MRRR_L2PIN")) h->l2_persist = atoi(s) != 0;
    if (const char *s = getenv("MRRR_FAULT")) h->fault = atoi(s);
    if (const char *s = getenv("MRRR_BMERGE")) h->bmerge = atoi(s) != 0;
    if (const char *s = getenv("MRRR_RQISEGMIN")) h->rqi_seg_min = atoll(s);
    if (const char *s = getenv("MRRR_SEGSDK")) h->segsd_k = std::max(1, std::min(64, atoi(s)));
    {
      int dev = h->device, maxwin = 0, l2 = 0;
      cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, dev);
      cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
      h->l2_max_window = maxwin;
      // set aside up to 1/4 of L2 for persisting lines (the representation pool)
      if (h->l2_persist && maxwin > 0) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)l2 / 4);
      cudaGetLastError();
    }
    for (auto &ev : h->ev) CK(cudaEventCreate(&ev));
    CK(cudaMallocHost(&h->h_cnt, sizeof(int) * C_NCOUNTERS));
    CK(cudaMallocHost(&h->h_small, sizeof(int) * 64));
  } catch (Err &er) {
    delete h;
    return er.code;
  }
  *out = h;
  return 0;
}

int mrrr_eig(mrrr_t h, const double *d, const double *e, int64_t n, int64_t il, int64_t iu, double *W, double *Z,
             int64_t ldz) {
  if (!h) return -1;
  int a = check_args(d, e, n, il, iu, W, Z, ldz);
  if (a) return a;
  try {
    CK(cudaSetDevice(h->device));
    return solve(h, d, e, n, il, iu, W, Z, ldz, 0, 0, nullptr, nullptr, 0);
  } catch (Err &er) {
    return er.code;
  }
}

int mrrr_eig_shard(mrrr_t h, const double *d, const double *e, int64_t n, int64_t il, int64_t iu, int64_t sl,
                   int64_t su, double *W, double *Z, int64_t ldz, int64_t ncols_cap, int64_t *jlo, int64_t *jhi) {
  if (!h) return -1;
  int a = check_args(d, e, n, il, iu, W, Z, ldz);
  if (a) return (a <= -7) ? a - 2 : a;  // W, Z, ldz sit after sl, su
  if (sl < il || sl > iu) return -7;
  if (su < sl || su > iu) return -8;
  if (!jlo) return -13;
  if (!jhi) return -14;
  try {
    CK(cudaSetDevice(h->device));
    long long lo = su + 1, hi = su;
    int rc = solve(h, d, e, n, il, iu, W, Z, ldz, sl, su, &lo, &hi, ncols_cap);
    *jlo = lo;
    *jhi = hi;
    return rc;
  } catch (Err &er) {
    return er.code;
  }
}

// NCCL, opened at run time (no link dependency: the process may already hold torch's libnccl.so.2)
namespace {
struct Nccl {
  bool tried = false, ok = false;
  ncclResult_t (*get_id)(ncclUniqueId *) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char *(*err)(ncclResult_t) = nullptr;
};
Nccl &nccl() {
  static Nccl N;
  if (!N.tried) {
    N.tried = true;
    void *lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (lib) {
      N.get_id = (decltype(N.get_id))dlsym(lib, "ncclGetUniqueId");
      N.init_rank = (decltype(N.init_rank))dlsym(lib, "ncclCommInitRank");
      N.all_gather = (decltype(N.all_gather))dlsym(lib, "ncclAllGather");
      N.destroy = (decltype(N.destroy))dlsym(lib, "ncclCommDestroy");
      N.err = (decltype(N.err))dlsym(lib, "ncclGetErrorString");
      N.ok = N.get_id && N.init_rank && N.all_gather && N.destroy && N.err;
    }
    if (!N.ok) g_last_nccl_error = "libnccl.so.2 could not be loaded";
  }
  return N;
}
#define NK(x)                                                              \
  do {                                                                     \
    ncclResult_t r_ = (x);                                                 \
    if (r_ != ncclSuccess) {                                               \
      g_last_nccl_error = std::string(#x) + ": " + nccl().err(r_);         \
      throw Err{MRRR_ERR_NCCL};                                            \
    }                                                                      \
  } while (0)
}  // namespace

int mrrr_nccl_unique_id(void *id128) {
  if (!id128) return -1;
  Nccl &N = nccl();
  if (!N.ok) return MRRR_ERR_NCCL;
  try {
    ncclUniqueId id;
    NK(N.get_id(&id));
    memcpy(id128, id.internal, sizeof(id.internal));
  } catch (Err &er) {
    return er.code;
  }
  return 0;
}

int mrrr_eig_dist(mrrr_t h, const void *nccl_id, int32_t rank, int32_t world, const double *d, const double *e,
                  int64_t n, int64_t il, int64_t iu, double *W, double *Z, int64_t ldz, int64_t ncols_cap,
                  int64_t *jlo, int64_t *jhi) {
  if (!h) return -1;
  if (!nccl_id) return -2;
  if (world < 1) return -4;
  if (rank < 0 || rank >= world) return -3;
  int a = check_args(d, e, n, il, iu, W, Z, ldz);
  if (a) return a - 3;  // shift past nccl_id, rank, world
  if (!jlo) return -14;
  if (!jhi) return -15;
  Nccl &N = nccl();
  if (!N.ok) return MRRR_ERR_NCCL;
  // 1) the rank's own solve; any failure (returned code or a CUDA error) is kept local so that the rank
  //    still joins both collectives with an empty share -- no rank is left waiting in ncclAllGather
  int rc = 0;
  const long long k = iu - il + 1, per = (k + world - 1) / world;
  const long long sl = il + (long long)rank * per, su = std::min<long long>(sl + per - 1, iu);
  long long lo = su + 1, hi = su;
  try {
    CK(cudaSetDevice(h->device));
    const long long cap = std::max<long long>(ncols_cap, 1);
    CK(h->dWl.ensure(sizeof(double) * cap));
    if (sl <= su) rc = solve(h, d, e, n, il, iu, h->dWl.as<double>(), Z, ldz, sl, su, &lo, &hi, ncols_cap);
  } catch (Err &er) {
    rc = er.code;
  }
  *jlo = lo;   // on MRRR_ERR_NOMEM (owned count > ncols_cap) the needed range is still reported
  *jhi = hi;
  try {
    if (rc != 0) cudaGetLastError();  // clear a non-sticky error before the collectives
    CK(cudaSetDevice(h->device));
    // the communicator (kept while id, rank and world stay the same)
    if (!h->comm || h->comm_rank != rank || h->comm_world != world || memcmp(h->comm_id, nccl_id, 128) != 0) {
      if (h->comm) { N.destroy(h->comm); h->comm = nullptr; }
      ncclUniqueId id;
      memcpy(id.internal, nccl_id, 128);
      NK(N.init_rank(&h->comm, world, id, rank));
      memcpy(h->comm_id, nccl_id, 128);
      h->comm_rank = rank;
      h->comm_world = world;
    }
    // 2) every rank's (first owned index, count, return code); 3) the padded eigenvalue lists; 4) scatter
    //    into W.  A failed rank contributes count 0 and its code, and every rank returns an error then.
    const long long cnt = (rc == 0) ? std::max<long long>(hi - lo + 1, 0) : 0;
    long long meta_h[3] = {lo, cnt, rc};
    CK(h->dmeta.ensure(sizeof(long long) * 3));
    CK(h->dmetas.ensure(sizeof(long long) * 3 * world));
    CK(cudaMemcpyAsync(h->dmeta.p, meta_h, sizeof(meta_h), cudaMemcpyHostToDevice, h->stream));
    NK(N.all_gather(h->dmeta.p, h->dmetas.p, 3, ncclInt64, h->comm, h->stream));
    std::vector<long long> metas(3 * world);
    CK(cudaMemcpyAsync(metas.data(), h->dmetas.p, sizeof(long long) * 3 * world, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    long long mcap = 1;
    int peer_rc = 0;
    for (int r = 0; r < world; r++) {
      mcap = std::max(mcap, metas[3 * r + 1]);
      if (metas[3 * r + 2] != 0 && peer_rc == 0) peer_rc = (int)metas[3 * r + 2];
    }
    CK(h->dpad.ensure(sizeof(double) * mcap));
    CK(h->dparts.ensure(sizeof(double) * mcap * world));
    if (cnt) CK(cudaMemcpyAsync(h->dpad.p, h->dWl.p, sizeof(double) * cnt, cudaMemcpyDeviceToDevice, h->stream));
    NK(N.all_gather(h->dpad.p, h->dparts.p, (size_t)mcap, ncclDouble, h->comm, h->stream));
    for (int r = 0; r < world && peer_rc == 0; r++) {
      // owned ranges partition [il, iu] (shard_owner), so every copy stays inside W[0..k)
      const long long rl = metas[3 * r], rc_ = metas[3 * r + 1];
      if (rc_ > 0 && rl >= il && rl + rc_ - 1 <= iu)
        CK(cudaMemcpyAsync(W + (rl - il), h->dparts.as<double>() + (long long)r * mcap, sizeof(double) * rc_,
                           cudaMemcpyDeviceToDevice, h->stream));
    }
    CK(cudaStreamSynchronize(h->stream));
    if (rc == 0 && peer_rc != 0) rc = MRRR_ERR_PEER;
  } catch (Err &er) {
    return rc ? rc : er.code;
  }
  return rc;
}

int mrrr_shard_owner(const int32_t *gstart, int64_t n, int64_t il, int64_t iu, int64_t sl, int64_t su,
                     int64_t jmax, int64_t *jlo, int64_t *jhi) {
  if (!gstart) return -1;
  if (n < 1) return -2;
  if (il < 1 || il > n) return -3;
  if (iu < il || iu > n) return -4;
  if (sl < il || sl > iu) return -5;
  if (su < sl || su > iu) return -6;
  if (jmax < su || jmax > n) return -7;
  if (!jlo) return -8;
  if (!jhi) return -9;
  long long lo = 0, hi = 0;
  shard_owner(gstart, n, il, iu, sl, su, jmax, &lo, &hi);
  *jlo = lo;
  *jhi = hi;
  return 0;
}

int mrrr_eig_host(mrrr_t h, const double *d, const double *e, int64_t n, int64_t il, int64_t iu, double *W,
                  double *Z, int64_t ldz) {
  if (!h) return -1;
  int a = check_args(d, e, n, il, iu, W, Z, ldz);
  if (a) return a;
  double *dd_ = nullptr, *de = nullptr, *dW = nullptr, *dZ = nullptr;
  long long k = iu - il + 1;
  int rc = 0;
  try {
    CK(cudaSetDevice(h->device));
    // device staging buffers are cached in the handle (grown on demand)
    CK(h->hd.ensure(sizeof(double) * n));
    CK(h->he.ensure(sizeof(double) * std::max<long long>(n - 1, 1)));
    CK(h->hW.ensure(sizeof(double) * k));
    CK(h->hZ.ensure(sizeof(double) * n * k));
    dd_ = h->hd.as<double>(); de = h->he.as<double>(); dW = h->hW.as<double>(); dZ = h->hZ.as<double>();
    CK(cudaMemcpyAsync(dd_, d, sizeof(double) * n, cudaMemcpyHostToDevice, h->stream));
    if (n > 1) CK(cudaMemcpyAsync(de, e, sizeof(double) * (n - 1), cudaMemcpyHostToDevice, h->stream));
    rc = solve(h, dd_, de, n, il, iu, dW, dZ, n, 0, 0, nullptr, nullptr, 0);
    if (rc == 0) {
      CK(cudaMemcpyAsync(W, dW, sizeof(double) * k, cudaMemcpyDeviceToHost, h->stream));
      if (ldz == n) CK(cudaMemcpyAsync(Z, dZ, sizeof(double) * n * k, cudaMemcpyDeviceToHost, h->stream));
      else CK(cudaMemcpy2DAsync(Z, sizeof(double) * ldz, dZ, sizeof(double) * n, sizeof(double) * n, k,
                                cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
    }
  } catch (Err &er) {
    rc = er.code;
  }
  return rc;
}

// single/double realisation: binary32 in and out, binary64 inside, gaptol 1e-5
static int seig_device(mrrr_t h, const float *d, const float *e, long long n, long long il, long long iu, float *W,
                       float *Z, long long ldz) {
  const long long k = iu - il + 1;
  CK(h->sdin.ensure(sizeof(double) * (2 * n)));
  CK(h->sdW.ensure(sizeof(double) * k));
  CK(h->sdZ.ensure(sizeof(double) * n * k));
  double *dd_ = h->sdin.as<double>(), *de = dd_ + n;
  k_f2d<<<nblocks_for(n, 256), 256, 0, h->stream>>>(d, dd_, n);
  if (n > 1) k_f2d<<<nblocks_for(n - 1, 256), 256, 0, h->stream>>>(e, de, n - 1);
  launch_check(h);
  struct Profile {  // the handle's profile is restored on every exit path (errors throw)
    mrrr_t h;
    double g;
    ~Profile() { h->sd = false; h->gaptol = g; }
  } prof{h, h->gaptol};
  h->sd = true;
  h->gaptol = h->gaptol_sd;
  int rc = solve(h, dd_, de, n, il, iu, h->sdW.as<double>(), h->sdZ.as<double>(), n, 0, 0, nullptr, nullptr, 0);
  if (rc) return rc;
  k_w_d2f<<<nblocks_for(k, 256), 256, 0, h->stream>>>(h->sdW.as<double>(), W, k);
  for (long long c0 = 0; c0 < k; c0 += 65535) {
    const long long kc = std::min<long long>(65535, k - c0);
    k_z_d2f<<<dim3(nblocks_for(n, 256), (unsigned)kc), 256, 0, h->stream>>>(h->sdZ.as<double>() + c0 * n,
                                                                           Z + c0 * ldz, n, ldz);
  }
  launch_check(h);
  CK(cudaStreamSynchronize(h->stream));
  return 0;
}

int mrrr_seig(mrrr_t h, const float *d, const float *e, int64_t n, int64_t il, int64_t iu, float *W, float *Z,
              int64_t ldz) {
  if (!h) return -1;
  int a = check_args(reinterpret_cast<const double *>(d), reinterpret_cast<const double *>(e), n, il, iu,
                     reinterpret_cast<const double *>(W), reinterpret_cast<const double *>(Z), ldz);
  if (a) return a;
  try {
    CK(cudaSetDevice(h->device));
    return seig_device(h, d, e, n, il, iu, W, Z, ldz);
  } catch (Err &er) {
    return er.code;
  }
}

int mrrr_seig_host(mrrr_t h, const float *d, const float *e, int64_t n, int64_t il, int64_t iu, float *W, float *Z,
                   int64_t ldz) {
  if (!h) return -1;
  int a = check_args(reinterpret_cast<const double *>(d), reinterpret_cast<const double *>(e), n, il, iu,
                     reinterpret_cast<const double *>(W), reinterpret_cast<const double *>(Z), ldz);
  if (a) return a;
  const long long k = iu - il + 1;
  try {
    CK(cudaSetDevice(h->device));
    CK(h->sdhin.ensure(sizeof(float) * 2 * n));
    CK(h->sdhW.ensure(sizeof(float) * k));
    CK(h->sdhZ.ensure(sizeof(float) * n * k));
    float *df = h->sdhin.as<float>(), *ef = df + n, *dW = h->sdhW.as<float>(), *dZ = h->sdhZ.as<float>();
    CK(cudaMemcpyAsync(df, d, sizeof(float) * n, cudaMemcpyHostToDevice, h->stream));
    if (n > 1) CK(cudaMemcpyAsync(ef, e, sizeof(float) * (n - 1), cudaMemcpyHostToDevice, h->stream));
    int rc = seig_device(h, df, ef, n, il, iu, dW, dZ, n);
    if (rc) return rc;
    CK(cudaMemcpyAsync(W, dW, sizeof(float) * k, cudaMemcpyDeviceToHost, h->stream));
    if (ldz == n) CK(cudaMemcpyAsync(Z, dZ, sizeof(float) * n * k, cudaMemcpyDeviceToHost, h->stream));
    else CK(cudaMemcpy2DAsync(Z, sizeof(float) * ldz, dZ, sizeof(float) * n, sizeof(float) * n, k,
                              cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return 0;
  } catch (Err &er) {
    return er.code;
  }
}

int mrrr_get_stats(mrrr_t h, int64_t *s, int32_t ns) {
  if (!h || !s) return -1;
  for (int i = 0; i < ns && i < MRRR_NSTATS; i++) s[i] = h->stats_h[i];
  return 0;
}

int mrrr_get_times(mrrr_t h, double *ms, int32_t nt) {
  if (!h || !ms) return -1;
  if (h->times_dirty) {  // the last solve's events (complete: the solve synchronized its stream before returning)
    auto el = [&](cudaEvent_t a, cudaEvent_t b) {
      float v = 0.0f;
      cudaEventElapsedTime(&v, a, b);
      return (double)v;
    };
    h->times[0] = el(h->ev[0], h->ev[5]);
    h->times[1] = el(h->ev[0], h->ev[1]);
    h->times[2] = el(h->ev[1], h->ev[2]);
    h->times[3] = el(h->ev[2], h->ev[3]);
    h->times[4] = el(h->ev[4], h->ev[5]);
    h->times[5] = el(h->ev[3], h->ev[4]);
    h->neg_ms = 0.0;
    for (auto &p : h->tneg) h->neg_ms += el(h->tev[p.first], h->tev[p.second]);
    h->rqi_ms = 0.0;
    for (auto &p : h->trq) h->rqi_ms += el(h->tev[p.first], h->tev[p.second]);
    h->times[6] = h->rqi_launches ? h->rqi_ms / h->rqi_launches : 0.0;
    h->times[7] = (double)h->rqi_launches;
    h->times[8] = h->neg_launches ? h->neg_ms / h->neg_launches : 0.0;
    h->times[9] = (double)h->neg_launches;
    cudaGetLastError();
    h->times_dirty = false;
  }
  for (int i = 0; i < nt && i < 12; i++) ms[i] = h->times[i];
  return 0;
}

int mrrr_get_diag(mrrr_t h, mrrr_diag *g) {
  if (!h || !g) return -1;
  if (!(h->flags & MRRR_KEEP_DIAG)) return -1;
  try {
    long long n = h->last_n, k = h->last_k;
    int nblk = h->last_nblk;
    CK(cudaStreamSynchronize(h->stream));
    if (g->nblocks) g->nblocks[0] = nblk;
    if (g->block_start) for (int b = 0; b <= nblk; b++) g->block_start[b] = h->h_starts[b];
    if (g->mu || g->side) {
      std::vector<double> hb(16 * nblk);
      CK(cudaMemcpy(hb.data(), h->binfo.p, sizeof(double) * 16 * nblk, cudaMemcpyDeviceToHost));
      for (int b = 0; b < nblk; b++) {
        bool triv = h->h_starts[b + 1] - h->h_starts[b] == 1;
        if (g->mu) g->mu[b] = triv ? 0.0 : hb[16 * b];
        if (g->side) g->side[b] = triv ? 0 : (int)hb[16 * b + 6];
      }
    }
    if (g->root_lo) CK(cudaMemcpy(g->root_lo, h->rlo.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
    if (g->root_hi) CK(cudaMemcpy(g->root_hi, h->rhi.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
    if (g->root_lo && nblk > 1)
      for (int b = 0; b < nblk; b++)
        if (h->h_starts[b + 1] - h->h_starts[b] == 1) {
          // size-1 blocks: [alpha, alpha] (oracle convention); alpha comes from fin_lo via the trivial kernel
        }
    if (g->root_gstart) CK(cudaMemcpy(g->root_gstart, h->gstart.p, sizeof(int) * n, cudaMemcpyDeviceToHost));
    if (g->depth) CK(cudaMemcpy(g->depth, h->ddepth.p, sizeof(int) * k, cudaMemcpyDeviceToHost));
    if (g->grp_first) CK(cudaMemcpy(g->grp_first, h->dgf.p, sizeof(int) * MAXD * k, cudaMemcpyDeviceToHost));
    if (g->grp_last) CK(cudaMemcpy(g->grp_last, h->dgl.p, sizeof(int) * MAXD * k, cudaMemcpyDeviceToHost));
    if (g->fin_lo) CK(cudaMemcpy(g->fin_lo, h->dflo.p, sizeof(double) * k, cudaMemcpyDeviceToHost));
    if (g->fin_hi) CK(cudaMemcpy(g->fin_hi, h->dfhi.p, sizeof(double) * k, cudaMemcpyDeviceToHost));
  } catch (Err &er) {
    return er.code;
  }
  return 0;
}

int mrrr_selftest(int which, int64_t n, uint64_t seed, int64_t *bad) {
  if (!bad || n < 0) return -1;
  if (which != 1) return -1;
  try {
    unsigned long long *d = nullptr, hb = 0;
    CK(cudaMalloc(&d, sizeof(*d)));
    CK(cudaMemset(d, 0, sizeof(*d)));
    k_selftest_div<<<nblocks_for(n, 256), 256>>>(n, seed, d);
    CK(cudaGetLastError());
    CK(cudaMemcpy(&hb, d, sizeof(hb), cudaMemcpyDeviceToHost));
    cudaFree(d);
    *bad = (int64_t)hb;
  } catch (Err &er) {
    return er.code;
  }
  return 0;
}

const char *mrrr_strerror(int code) {
  switch (code) {
    case MRRR_OK: return "success";
    case MRRR_ERR_NONFINITE: return "NaN or Inf in d or e";
    case MRRR_ERR_CUDA: return g_last_cuda_error.c_str();
    case MRRR_ERR_NOMEM: return "device memory exhausted";
    case MRRR_ERR_ROOT: return "no definite root representation found";
    case MRRR_ERR_NODEVICE: return "no CUDA device";
    case MRRR_ERR_NCCL: return g_last_nccl_error.c_str();
    case MRRR_ERR_PEER: return "another rank of the multi-GPU solve failed";
    default: return code < 0 ? "invalid argument" : "unknown error";
  }
}

int mrrr_destroy(mrrr_t h) {
  if (!h) return 0;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  Buf *bufs[] = {&h->starts, &h->scal, &h->binfo, &h->bside, &h->blist, &h->cab, &h->mx, &h->my, &h->mq, &h->nodesK, &h->nodesP, &h->offsP, &h->dS, &h->dG, &h->dH, &h->repoff, &h->repcur, &h->repcta, &h->segout, &h->rnd, &h->gpart, &h->segouty, &h->segfby, &h->segoutx, &h->segoutg, &h->rqst, &h->rqrec, &h->hand, &h->lscratch,
                 &h->reps, &h->rlo, &h->rhi, &h->colmap, &h->gstart, &h->nodesA, &h->nodesB, &h->counts, &h->ex,
                 &h->excounts, &h->exmap, &h->bnA, &h->bnB, &h->sing, &h->clusA, &h->clusB, &h->ss, &h->gval,
                 &h->valid, &h->cseg, &h->bnoff, &h->ipool_lo, &h->ipool_hi, &h->yref_lo, &h->yref_hi, &h->wsA,
                 &h->wsB, &h->stats, &h->cnt, &h->ddepth, &h->dgf, &h->dgl, &h->dflo, &h->dfhi,
                 &h->hd, &h->he, &h->hW, &h->hZ, &h->zmeta, &h->hd2,
                 &h->sdin, &h->sdW, &h->sdZ, &h->sdhin, &h->sdhW, &h->sdhZ, &h->segsd};
  for (Buf *b : bufs) b->release();
  if (h->s_tail) {
    cudaStreamSynchronize(h->s_tail);
    cudaStreamDestroy(h->s_tail);
    cudaEventDestroy(h->ev_tail_in);
    cudaEventDestroy(h->ev_tail_done);
  }
  h->tail_ws.release();
  h->tail_sing.release();
  h->tail_zmeta.release();
  for (int l = 0; l < mrrr_ctx::LVL_MAX; l++) {
    h->lvl_L[l].release();
    h->lvl_NX[l].release();
    h->lvl_SG[l].release();
  }
  for (auto &ev : h->ev) cudaEventDestroy(ev);
  for (auto &ev : h->tev) cudaEventDestroy(ev);
  if (h->comm && nccl().ok) nccl().destroy(h->comm);
  h->dWl.release();
  h->dmeta.release();
  h->dmetas.release();
  h->dpad.release();
  h->dparts.release();
  if (h->h_cnt) cudaFreeHost(h->h_cnt);
  if (h->h_small) cudaFreeHost(h->h_small);
  if (h->own_stream) cudaStreamDestroy(h->stream);
  delete h;
  return 0;
}

}  // extern "C"
