/*
 * mrrr.h -- C ABI of libmrrr.so: k eigenpairs of a real symmetric tridiagonal
 * matrix T by the mixed-precision MRRR (MR^3) algorithm of arXiv 1401.4950
 * (Petschow, "MRRR-based Eigensolvers for Multi-core Processors and
 * Supercomputers"), computed on an NVIDIA B200 (sm_100a).
 *
 * Method (PAPER.md lines "P:a-b"):
 *   Alg. mrrr P:2762-2816 / Alg. mrrr2: root representation
 *   LDL^T = T - mu I, random relative perturbation, Sturm-count bisection
 *   (Alg. Bisection, Alg. negcountLDL), classification
 *   (P:3272-3292), child representations for clusters (Alg. spectrumshift
 *   P:3499-3590), and Rayleigh-quotient iteration driven by the twisted
 *   factorization (Alg. Getvec, Alg. stask) for every
 *   singleton, in the thesis's mixed precision form: fp64 input and output,
 *   double-double internal arithmetic for representations and vectors
 *   (Ch.5 P:5516-6163; double/quadruple realisation P:6270-6278).
 *   The exact step list and every reading of the paper are in DESIGN.md.
 *
 * Conventions
 *   T is given by its diagonal d[0..n-1] (alpha_1..alpha_n) and off-diagonal
 *   e[0..n-2] (beta_1..beta_{n-1}), eq:thetridiagonal P:1969-1979.
 *   Indices il..iu are 1-based and inclusive (LAPACK style); k = iu - il + 1.
 *   Outputs: W[0..k-1] ascending, W[j] = lambda_{il+j}; column j of Z
 *   (column-major, leading dimension ldz >= n) is its unit eigenvector, with
 *   the sign fixed by z(r) > 0 at the twist index r (Getvec sets z(r) = 1,
 *   P:3434).  d and e are read only.
 *
 * Return codes: 0 success; -i: argument i of the call is invalid (counting the
 * handle as 1); > 0: one of MRRR_ERR_* below.
 *
 * Threading: a handle is not re-entrant; use one handle per host thread.
 */
#ifndef MRRR_H
#define MRRR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mrrr_ctx *mrrr_t;

#define MRRR_OK 0
#define MRRR_ERR_NONFINITE 1  /* NaN or Inf in d or e */
#define MRRR_ERR_CUDA 2       /* CUDA runtime error; see mrrr_strerror(MRRR_ERR_CUDA) */
#define MRRR_ERR_NOMEM 3      /* device memory exhausted (workspace or outputs) */
#define MRRR_ERR_ROOT 4       /* no definite root shift found (S3) */
#define MRRR_ERR_NODEVICE 5   /* no CUDA device */
#define MRRR_ERR_NCCL 6       /* NCCL missing (libnccl.so.2 not loadable) or an NCCL call failed */
#define MRRR_ERR_PEER 7       /* mrrr_eig_dist: this rank succeeded but another rank failed */

#define MRRR_KEEP_DIAG 1u     /* keep integer/interval diagnostics for mrrr_get_diag */
/* Early classification stop of the root bisection (S5'): "only sufficient accuracy to classify
 * eigenvalues into well-separated and clustered is needed ... Depending on the absolute gap of the eigenvalue,
 * the refinement can be stopped earlier on" (sec. 3.2.2 remark (3); A-41).
 * Every index is bisected to rtol_c = max(rtol, 2^-(10 + ceil(log2 n))) first; index j (not the first or last
 * of its block) stops there when both of its neighbour pairs are already classification boundaries and its
 * width is at most 2^-7 of its absolute gap; the others continue to rtol = 1e-2 gaptol.  Cluster boundaries
 * are those of the default solve; stopped singletons start their RQI from the coarser interval.  Honoured by
 * mrrr_eig / mrrr_seig (and their _host forms); shards and mrrr_eig_dist apply the same rule (it depends only
 * on the indices j-1, j, j+1). */
#define MRRR_EARLY_STOP 2u
/* Numerical support of the singleton eigenvectors (S10', Getvec remark (2): "for all i < i_first
 * and for all i > i_last, z(i) can be set to zero ... easily detected and exploited"; A-42) is applied by
 * default: going outward from the twist index r (z(r) = 1), a column ends at the first edge i whose coupling
 * |dl(i)| (|z(i)| + |z(i+1)|) is at most gap * eps_x, and the rows past it are stored as exact zeros (the residual
 * changes by at most that term, so the vector moves by O(eps_x) by the gap theorem).  MRRR_FULL_SUPPORT stores
 * the whole recurrence instead (Alg. Getvec as printed).  W and every integer output are the same either way. */
#define MRRR_FULL_SUPPORT 4u

/* Options (all fields may be zero = default). */
typedef struct {
  int32_t device;     /* CUDA ordinal; < 0: the current device */
  int32_t root_side;  /* 0: auto (S3), 1: left Gershgorin end, 2: right */
  void *stream;       /* cudaStream_t used for all work; NULL: a library-owned stream */
  double gaptol;      /* classification threshold; <= 0: 1e-10 */
  uint64_t seed;      /* key of the root perturbation stream; 0: default */
  uint32_t flags;     /* MRRR_KEEP_DIAG | MRRR_EARLY_STOP | MRRR_FULL_SUPPORT */
  uint32_t reserved;
  int64_t ws_limit;   /* soft cap on workspace bytes; <= 0: 60% of free device memory */
} mrrr_opts;

/* Create a handle.  opts may be NULL.  Returns 0 or MRRR_ERR_*.
 * Ownership: the handle owns all device workspace until mrrr_destroy. */
int mrrr_init(mrrr_t *h, const mrrr_opts *opts);

/* Eigenpairs il..iu of T.  d, e, W, Z are CUDA DEVICE pointers owned by the
 * caller (e may be NULL when n == 1).  Work is issued on the handle's stream
 * after waiting for the caller's work on it; the call returns when W and Z
 * are complete.  Errors: -2 d NULL, -3 e NULL (n > 1), -4 n < 1,
 * -5 il out of [1, n], -6 iu out of [il, n], -7 W NULL, -8 Z NULL,
 * -9 ldz < n; MRRR_ERR_* otherwise. */
int mrrr_eig(mrrr_t h, const double *d, const double *e, int64_t n, int64_t il, int64_t iu, double *W,
             double *Z, int64_t ldz);

/* Same as mrrr_eig with HOST pointers (pageable or pinned): copies d, e to
 * the device, solves, copies W and Z back.  Same argument checks. */
int mrrr_eig_host(mrrr_t h, const double *d, const double *e, int64_t n, int64_t il, int64_t iu, double *W,
                  double *Z, int64_t ldz);

/* Single/double realisation: eigenpairs il..iu of T given in binary32, W and Z
 * returned in binary32, every computation in binary64 ("data conversion is only necessary when reading the
 * input and writing the output").  Parameters of that realisation:
 * gaptol fixed to 1e-5 (mrrr_opts.gaptol is ignored here), bisection to 1e-2 gaptol, epsilon_x =
 * 2^-24 in the split rule, the root perturbation and the RQI stopping test, the growth bound
 * max(64, 2^29 / sqrt(n)) spdiam (eq:newkelgbound P:6052-6056).  Accuracy target: residuals and orthogonality
 * O(n eps_s), eps_s = 2^-24.  d, e, W, Z are DEVICE pointers (float); ldz >= n.  The solve keeps binary64
 * copies of W and Z in handle workspace (8 n k bytes) before the final conversion.  Same argument checks and
 * return codes as mrrr_eig. */
int mrrr_seig(mrrr_t h, const float *d, const float *e, int64_t n, int64_t il, int64_t iu, float *W, float *Z,
              int64_t ldz);

/* mrrr_seig with HOST pointers (copies in, solve, copies out). */
int mrrr_seig_host(mrrr_t h, const float *d, const float *e, int64_t n, int64_t il, int64_t iu, float *W,
                   float *Z, int64_t ldz);

/* Index-range shard of a multi-GPU solve (one process per GPU) of the selection
 * [il, iu]: the rank's shard is the contiguous range [sl, su] (1-based, il <= sl <= su <= iu); every rank
 * builds the same root (bit-identical: the root side follows the same rule on [il, iu] as mrrr_eig), bisects
 * its shard plus guards, and computes exactly the eigenpairs of the units that START inside the shard.  A
 * unit is a root group (singleton or cluster) cut to [il, iu]: a cluster straddling a shard
 * boundary is owned by the rank holding its first index (north_star), a cluster straddling il is owned from
 * il on by the rank holding il, and no owned range reaches past iu -- so the owned ranges of all ranks
 * partition [il, iu] and every column equals the mrrr_eig(il, iu) column bit for bit.  On return
 * [*jlo, *jhi] (1-based, *jhi < *jlo if empty) is the owned range; W_local[0..] and columns of Z_local hold
 * eigenpairs *jlo..*jhi.  ncols_cap bounds the owned count (MRRR_ERR_NOMEM if exceeded, with the needed range
 * still returned).  Device pointers as in mrrr_eig.  Errors: -2 d, -3 e, -4 n, -5 il, -6 iu, -7 sl out of
 * [il, iu], -8 su out of [sl, iu], -9 W_local NULL, -10 Z_local NULL, -11 ldz < n, -13/-14 jlo/jhi NULL. */
int mrrr_eig_shard(mrrr_t h, const double *d, const double *e, int64_t n, int64_t il, int64_t iu, int64_t sl,
                   int64_t su, double *W_local, double *Z_local, int64_t ldz, int64_t ncols_cap, int64_t *jlo,
                   int64_t *jhi);

/* 128-byte NCCL unique id for mrrr_eig_dist: call on one rank, send the bytes to every rank (e.g. a
 * torch.distributed broadcast), pass them to mrrr_eig_dist everywhere.  id128: caller-owned host buffer of
 * 128 bytes.  Errors: -1 id128 NULL, MRRR_ERR_NCCL (libnccl.so.2 is opened at run time). */
int mrrr_nccl_unique_id(void *id128);

/* Multi-GPU solve, one process and one handle per GPU: rank `rank` of `world` takes the
 * contiguous shard [sl, su] of [il, iu] with ceil(k / world) indices per rank (PMRRR's static division,
 * P:4593-4599), computes the eigenpairs it owns exactly as mrrr_eig_shard does, then all-gathers the
 * eigenvalue list over NCCL so that W[0..k-1] holds all k eigenvalues on every rank;
 * Z_local (columns 0..*jhi-*jlo) holds the owned eigenvectors *jlo..*jhi (Z stays column-sharded).
 * nccl_id: the same 128 bytes on every rank (mrrr_nccl_unique_id); the communicator is created on the
 * first call and kept in the handle (recreated when the id, rank or world changes).  Every rank must
 * call (the all-gather is collective) even if its shard is empty.  A rank whose own solve fails (any
 * code, including a CUDA error) still joins both all-gathers with an empty share and returns its code;
 * the other ranks then return MRRR_ERR_PEER, so no rank waits forever.  d, e, W, Z_local are device
 * pointers as in mrrr_eig; W has k entries.  Errors: -2 nccl_id NULL, -3 rank out of [0, world),
 * -4 world < 1, -5 d NULL, -6 e NULL (n > 1), -7 n < 1, -8 il, -9 iu, -10 W NULL, -11 Z_local NULL,
 * -12 ldz < n, -14/-15 jlo/jhi NULL; MRRR_ERR_NOMEM if the owned count exceeds ncols_cap;
 * MRRR_ERR_PEER, MRRR_ERR_NCCL, MRRR_ERR_* otherwise. */
int mrrr_eig_dist(mrrr_t h, const void *nccl_id, int32_t rank, int32_t world, const double *d, const double *e,
                  int64_t n, int64_t il, int64_t iu, double *W, double *Z_local, int64_t ldz, int64_t ncols_cap,
                  int64_t *jlo, int64_t *jhi);

/* Host-only helper (no GPU needed): the ownership rule of mrrr_eig_shard (north_star
 * "a cluster straddling a shard boundary is owned by the GPU holding its first index").  gstart[j-1]
 * (host array, n entries, caller-owned) is 1 iff index j starts a root group (singleton or cluster,
 * P:3272-3292), 0 if j continues the group of j-1; only entries sl..jmax are read.  [il, iu] is the
 * selection, [sl, su] the rank's shard (1-based, il <= sl <= su <= iu), jmax >= su the last classified
 * index.  Units start at every group start in [il, iu] and at il; on return [*jlo, *jhi] is the owned range:
 * from the first unit start in [sl, su] through the end of the last unit starting there (which may extend
 * past su up to min(jmax, iu)); *jlo = su + 1, *jhi = su if no unit starts in the shard.
 * Errors: -1 gstart NULL, -2 n < 1, -3 il out of [1, n], -4 iu out of [il, n], -5 sl out of [il, iu],
 * -6 su out of [sl, iu], -7 jmax out of [su, n], -8/-9 jlo/jhi NULL. */
int mrrr_shard_owner(const int32_t *gstart, int64_t n, int64_t il, int64_t iu, int64_t sl, int64_t su,
                     int64_t jmax, int64_t *jlo, int64_t *jhi);

/* Statistics of the last call (int64 each, nstats <= MRRR_NSTATS):
 * 0 d_max, 1 #clusters processed, 2 largest cluster, 3 uncertified shifts
 * (robustness failures), 4 shift attempts, 5 RQI iterations,
 * 6 RQI bisection fallbacks, 7 bracket repairs, 8 root back-offs,
 * 9 failed clusters, 10 x-NegCount evaluations, 11 y-NegCount evaluations,
 * 12 Getvec calls, 13 bisection rounds, 14 kernel launches, 15 nblocks,
 * 16 dd qd steps in k_rqi (dstqds/dqds element steps), 17 of them with the twist quantity gamma_k,
 * 18 z-solve element steps (norm pass), 19 z-solve element steps that write Z,
 * 20 x-NegCount evaluations on the sequential bisection paths (shared-tree nodes; the algorithmic
 * count, without k-section speculation), 21 the same for y-NegCount, 22 RQI corrections rejected for an
 * inertia-inconsistent sign, 23 RQI corrections rejected for leaving the bracket (both end in the bisection
 * fallback), 24 singletons the segmented RQI handed to the two-lane kernel, 25-27 of them because the
 * x-arithmetic twist search did not resolve gamma / a segment junction failed / the RQC was rejected,
 * 28 dd rows of RQC-only (light) passes, 29 fp64 rows of the segmented twist search (both lanes),
 * 30 segmented RQI passes repeated with an 8x longer warm-up after a failed junction, 31 singletons whose
 * last two-lane Getvec ran the careful IEEE pass (zero pivots / special values), 32 segmented
 * many-representation x-NegCount chains (child bisection) whose junctions did not all verify, 33 segments those
 * chains re-ran sequentially, 34 root indices the early classification stop (MRRR_EARLY_STOP) left at the
 * stage-1 tolerance, 35 segmented root x-NegCount chains whose junctions did not all verify (re-run
 * sequentially from the failed segment), 36 singletons whose numerical support reached past the z recompute
 * window of an RQC-only acceptance (their factors came from a stored pass). */
#define MRRR_NSTATS 37
int mrrr_get_stats(mrrr_t h, int64_t *stats, int32_t nstats);

/* Diagnostics of the last call made with MRRR_KEEP_DIAG (host buffers owned
 * by the caller; any pointer may be NULL; k = #eigenpairs of the call):
 *   nblocks[1], block_start[n+1], mu[n] and side[n] per block (0 size-1 block,
 *   1 left, 2 right), root_lo/root_hi[n] per global position (NaN where not
 *   computed), root_gstart[n] (1 starts a root group, 0 member, -1 not
 *   computed), depth[k], grp_first/grp_last[MRRR_MAXD*k] (global position of
 *   the group ends containing output j at each depth, -1 if none),
 *   fin_lo/fin_hi[k] (final-node interval of output j, node frame). */
#define MRRR_MAXD 8
typedef struct {
  int32_t *nblocks, *block_start;
  double *mu;
  int32_t *side;
  double *root_lo, *root_hi;
  int32_t *root_gstart, *depth, *grp_first, *grp_last;
  double *fin_lo, *fin_hi;
} mrrr_diag;
int mrrr_get_diag(mrrr_t h, mrrr_diag *g);

/* Time of the last call in milliseconds (CUDA events on the handle's stream,
 * entry to results ready), split into phases: [0] total, [1] split+root,
 * [2] root bisection, [3] classification, [4] cluster path, [5] singleton RQI.
 * Also the average duration of the dominant kernel launches (events around each launch on the
 * handle's stream): [6] ms per singleton-RQI launch, [7] their number, [8] ms per x-NegCount
 * (root/child bisection) launch, [9] their number. */
int mrrr_get_times(mrrr_t h, double *ms, int32_t nt);

/* Built-in self tests (run on the current device).  which = 1: the NegCount division fast path
 * (csrc/kernels.cuh div_ieee, and div_fast_nocheck wherever its range test passes) against the IEEE
 * __ddiv_rn on n seeded operand pairs (random bit patterns incl. subnormals/inf/nan, near-midpoint
 * quotients, and the O(1) NegCount regime); *bad = #bitwise mismatches. */
int mrrr_selftest(int which, int64_t n, uint64_t seed, int64_t *bad);

const char *mrrr_strerror(int code);

int mrrr_destroy(mrrr_t h);

#ifdef __cplusplus
}
#endif
#endif
