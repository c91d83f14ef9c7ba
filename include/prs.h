/*
 * prs.h -- C ABI of the B200 parareal-with-splitting library (libprs.so).
 *
 * Method: arXiv 2502.08370.  The library advances the semi-discrete problem
 *     U'(t) = (A_1 + ... + A_M) U(t) + F(t),  U(0) = P u_0
 * on the unit square/cube (interior nodes only, h = 1/(n+1), Dirichlet 0, x-fastest layout)
 * with the parareal algorithm whose coarse propagator G and fine
 * propagator F are the splitting integrators FIE or DR
 * over a dimensional or domain-decomposition split.
 *
 * Conventions (all entry points):
 *   - return PRS_OK (0) or a PRS_E* code; no exception crosses the ABI; prs_last_error()
 *     returns a per-context message for the last failure.
 *   - doubles are IEEE fp64; a "state" is n^dim doubles, x fastest (index (k*n + j)*n + i).
 *   - pointers marked "device" must be device memory of the context's device; they are
 *     borrowed for the duration of the call; the caller keeps ownership.
 *   - work is enqueued on the context stream (the one passed to prs_create, or a stream
 *     the library creates when NULL); calls that return host scalars synchronise it.
 *   - a context is not thread-safe.
 */
#ifndef PRS_H
#define PRS_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PRS_OK 0
#define PRS_EINVAL 2        /* bad configuration / argument (SPEC.md:472 exit 2)      */
#define PRS_EDIVERGED 3     /* a non-finite value appeared (exit 3)      */
#define PRS_EUNSUPPORTED 4  /* valid for the method but not implemented on this path  */
#define PRS_ECUDA 5         /* CUDA runtime failure                                   */
#define PRS_ENCCL 6         /* NCCL failure (multi-GPU)                               */

#define PRS_FIE 0
#define PRS_DR 1
#define PRS_IE 2  /* unsplit implicit Euler (I - tau A) U' = U + tau F(t'): the Parareal/IE-IE
                     baseline of PAPER.md:455.  GPU path:
                     constant coefficients only (coef_kind 0; solved exactly in the sine basis,
                     ie.cuh); any other coef_kind returns PRS_EUNSUPPORTED from prs_create */

typedef struct prs_ctx prs_ctx;

/* Problem description (mirrors BASELINE.json configs; readings in DESIGN.md §3). */
typedef struct prs_problem {
    int dim;          /* 2 or 3                                                          */
    int n;            /* interior nodes per axis (>= 1)                                  */
    double c;         /* reaction coefficient, L u = div(kappa grad u) - c u */
    int coef_kind;    /* 0: kappa = 1;  1: kappa = 1 + 0.5 sin(2 pi x) sin(2 pi y) (2-D);
                         2: the full tensor of PAPER.md:523-528 (NEXT-3; 2-D DD split only) */
    int split;        /* 0: dimensional, M = dim;  1: domain decomposition, M = 2 (2-D)  */
    int dd_strips;    /* DD: number of vertical strips 2q (n % dd_strips == 0)           */
    int dd_overlap;   /* DD: overlap width in cells (even, < n/dd_strips)                */
    int dd_ramp;      /* DD: 0 linear ramp, 1 cosine ramp                                */
    int source_kind;  /* 0: F = 0;  1: F = (dim pi^2 + c - 1) e^{-t} prod_d sin(pi x_d)   */
    double T;         /* final time                                                      */
    int N;            /* coarse slices N_c, Delta T = T/N                  */
    int s;            /* fine steps per slice, delta t = Delta T / s                     */
    int G;            /* coarse scheme PRS_FIE / PRS_DR / PRS_IE                         */
    int F;            /* fine scheme   PRS_FIE / PRS_DR / PRS_IE                         */
} prs_problem;

/* Create a context.  Validates the problem before allocating (PRS_EINVAL), allocates the
 * trajectory, caches and precomputed factors of every stage matrix (I - tau A_j) for
 * tau in {Delta T, delta t}.  rank/nranks shard the N slices in contiguous
 * blocks (rank order = time order); nccl_uid is the 128-byte ncclUniqueId from
 * prs_nccl_unique_id() on rank 0, broadcast by the caller (NULL when nranks == 1).
 * cuda_stream is a cudaStream_t (NULL: the library creates a blocking stream, ordered with
 * the legacy default stream, so inputs written there are visible to the context's work). */
int prs_create(const prs_problem *prob, int rank, int nranks, const void *nccl_uid,
               void *cuda_stream, prs_ctx **out);

/* Fill a 128-byte buffer with a fresh ncclUniqueId (call on rank 0 only). */
int prs_nccl_unique_id(void *uid128);

/* In-process multi-rank world (tests of the multi-rank driver on ONE device): nranks contexts
 * of one process, created with prs_create_local(..., rank, world, ...) and driven by one host
 * thread each, exchange their slice states / bands / stop-test words through device-to-device
 * copies ordered by CUDA events and matched on the host (no kernel waits on another rank).
 * The contexts run the same driver code as NCCL ranks (the data plane is an interface with an
 * NCCL and this local implementation).  The world outlives its contexts; a
 * host-side wait that is not matched within 300 s fails with PRS_ENCCL. */
int prs_local_world_create(int nranks, void **world);
void prs_local_world_destroy(void *world);
int prs_create_local(const prs_problem *prob, int rank, void *world, void *cuda_stream, prs_ctx **out);

/* Slices [first, first+count) owned by `rank` out of nranks (host only, no GPU needed). */
int prs_partition(int N, int nranks, int rank, int *first, int *count);

/* U_0 = P u_0: n^dim doubles, host or device (u0_on_device). */
int prs_set_initial(prs_ctx *ctx, const double *u0, int u0_on_device);

/* Initial guess U^0_{n+1} = G(U^0_n); also caches G(U^0_n). */
int prs_coarse_sweep(prs_ctx *ctx);

/* F^s(U^k_n) for every local slice concurrently, then
 * Delta_n = F^s(U^k_n) - G(U^k_n) in place. */
int prs_fine_sweep(prs_ctx *ctx);

/* Sequential correction U^{k+1}_{n+1} = G(U^{k+1}_n) + Delta_n; writes the
 * global normalised update max|U^{k+1} - U^k| / ||U_0||_inf to *update_out (synchronises).
 * Returns PRS_EDIVERGED if any corrected value is non-finite. */
int prs_parareal_correct(prs_ctx *ctx, double *update_out);

/* Loop fine_sweep + parareal_correct until update <= tol or k = min(kmax, N) (finite
 * termination).  hist (kmax doubles, may be NULL) receives the updates.
 * Slices n < k are skipped at iteration k for states of >= 2^18 points (exact and bitwise
 * frozen).  With several ranks the stop test is lagged: iteration k's all-reduce
 * runs on a second stream / communicator while iteration k+1's fine sweep already runs (its
 * result is discarded on a stop), so no rank waits for the last rank's chain before
 * propagating; results are those of the unlagged loop. */
int prs_iterate(prs_ctx *ctx, int kmax, double tol, int *k_out, double *hist);

/* Copy the current iterate U^k_n (n = 0..N) to host or device memory.  Only a rank that holds
 * U_n (as slice n-1's end state, or as the start state of its first slice) may call it
 * (PRS_EINVAL elsewhere; see prs_set_ownership for cyclic ownership). */
int prs_get_slice(prs_ctx *ctx, int n, double *out, int out_on_device);

/* One FIE/DR/IE step of size tau from a device state `in` to device `out` (in != out), the
 * source sampled at t_next = t_{n+1} (SPEC.md:211 for IE).  Test hook for
 * per-step parity.  PRS_IE needs a context created with G or F = PRS_IE (its sine tables). */
int prs_step(prs_ctx *ctx, int scheme, double tau, double t_next, const double *in, double *out);

/* One step of the coarse (which = 0: tau = Delta T, source at (slice0 + b + 1) Delta T) or the
 * fine (which = 1: tau = delta t, source at ((slice0 + b) s + j + 1) delta t) propagator on B
 * consecutive device states in -> out (in != out), in the launch configuration of
 * prs_fine_sweep.  Test hook for full-size batched parity. */
int prs_step_batch(prs_ctx *ctx, int which, int slice0, int j, const double *in, double *out, int B);

/* The sequential fine solution (PAPER.md:206-208 with every slice propagated by F in turn):
 * nslices * s fine steps of size delta t from U_0 = u0 (n^dim doubles, host or device), the
 * end state U(nslices Delta T) written to out (host or device).  Runs on the calling rank
 * alone (no communication) in the fine-sweep kernels with batch 1; it is the baseline that
 * parareal's time-to-tolerance is compared against, and finite termination's reference
 * (PAPER.md:214).  Uses the fine-sweep work buffers: a fine sweep whose correction is still
 * pending is invalidated (run prs_fine_sweep again).  Synchronises. */
int prs_fine_solve(prs_ctx *ctx, const double *u0, int u0_on_device, int nslices, double *out,
                   int out_on_device);

/* Coarse-chain mode of prs_parareal_correct / prs_iterate (north star item 5).
 * mode 0 (default): owner-G -- the G step of slice n runs on the GPU that owns slice n, the
 *   chain hands U^{k+1}_n from rank to rank (ncclSend/Recv).
 * mode 1: space-parallel G -- every coarse state is cut into P bands of n/P rows and all P
 *   GPUs advance the chain together: the x stage of FIE is row-local, the y stage is a
 *   partitioned tridiagonal solve (band block tuples, all-gathered band tuples, boundary
 *   values per band); Delta_n bands are scattered from the slice owners before the chain and
 *   the U_{n+1} / G-cache bands gathered back after it.  P = nranks; with one rank, `bands`
 *   virtual bands run in the same process (tests the partitioned solve on one GPU).
 *   Supported for the 2-D dimensional split with G = FIE, P and n powers of two, n <= 4096,
 *   n % (64 P) == 0 (PRS_EUNSUPPORTED otherwise).  Results equal owner-G up to rounding. */
int prs_set_coarse_mode(prs_ctx *ctx, int mode, int bands);

/* Slice ownership across ranks ("up to N_c processors"):
 * mode 0 (default): contiguous blocks, rank order = time order (prs_partition);
 * mode 1: cyclic -- slice n on rank n mod P.  prs_iterate skips the converged slices n < k at
 *   iteration k; with contiguous blocks the ranks holding the first blocks fall
 *   idle while the last rank keeps its N/P slices every iteration, with cyclic ownership every
 *   rank keeps ceil or floor((N-k)/P) active slices (balanced without moving any state), at the
 *   price of N-1 hand-offs per coarse chain instead of P-1.  Results are bitwise those of
 *   mode 0 and of one rank.  Owner-G coarse mode, unpipelined; call before prs_coarse_sweep
 *   (reallocates the trajectory; the initial state is kept).  With cyclic ownership U_n lives on
 *   ranks n mod P (as slice n's start) and (n-1) mod P (as slice n-1's end); prs_get_slice
 *   accepts either.  One rank: a no-op. */
int prs_set_ownership(prs_ctx *ctx, int mode);

/* Pipelined parareal for prs_iterate: blocks > 0 cuts
 * the local slices into `blocks` blocks and runs each iteration as a per-block dependency
 * graph on CUDA streams: the fine sweep of block b in iteration k+1 starts as soon as the
 * coarse chain of iteration k has corrected block b (F on slice n needs only U^{k+1}_n), and
 * the chain of iteration k+1 follows the fine sweeps block by block.  The stop test of
 * iteration k is read while iteration k+1 already runs (one iteration of lookahead, on the
 * other parity of a double-buffered trajectory / G cache, drained and discarded on stop), so
 * results -- trajectory, k, update history -- are bitwise those of the unpipelined path.
 * blocks = 0 turns it off.  Supported for one rank on the on-chip sweep path (2-D dimensional
 * split, kappa = 1, n in {32, 64, 128, 256}, owner-G); PRS_EUNSUPPORTED otherwise.  Allocates
 * a second trajectory and G cache.  Only prs_iterate is pipelined. */
int prs_set_pipeline(prs_ctx *ctx, int blocks);

/* Host only (no GPU): the band exchange of space-parallel G for `rank` of nranks and N slices,
 * phase 0 (scatter of Delta bands from the slice owners), 1 (gather of U / G-cache bands back
 * to them) or 2 (seed: the bands of the current iterate U^k_1..U^k_N from their owners, issued
 * before the first band chain after set_initial / coarse_sweep / a mode switch), as the
 * point-to-point operations prs_parareal_correct issues (NCCL group).  Writes
 * up to max_ops records of 6 ints {kind: 0 send, 1 recv, 2 local copy; what: 0 Delta_slice,
 * 1 U_{slice+1}, 2 Gcache_slice; slice; band; peer rank; owner-side local state index} to ops
 * (may be NULL) and returns the number of records, or -1 on bad arguments. */
int prs_gpar_plan(int N, int nranks, int rank, int phase, int *ops, int max_ops);

/* Counters.  prs_launches: kernels this context has launched so far.  With profiling on,
 * every fine-sweep kernel launch is bracketed by CUDA events on the context stream and
 * prs_kernel_stats(kind) returns, for kind PRS_K_XPASS (contiguous-axis line solve),
 * PRS_K_LPASS (strided-axis line solve), PRS_K_DD (DD strip-block stage) or PRS_K_IE (one
 * unsplit IE step: 2 dim sine-transform launches, bracketed together), the launch
 * count, the summed device time (ms, synchronises) and the summed ALGORITHMIC work: bytes
 * (state read + state write + precomputed factors read) for the line passes,
 * fp64 flops for PRS_K_DD (two W x W transforms + the y solve per support point) and for
 * PRS_K_IE (4 dim n flops per point). */
#define PRS_K_XPASS 0
#define PRS_K_LPASS 1
#define PRS_K_DD 2
#define PRS_K_IE 3  /* unsplit IE step (sine transforms on DMMA): fp64 flops */
int prs_set_profiling(prs_ctx *ctx, int on);
long long prs_launches(const prs_ctx *ctx);
int prs_kernel_stats(prs_ctx *ctx, int kind, long long *launches, double *ms, double *bytes);

const char *prs_last_error(const prs_ctx *ctx);
void prs_destroy(prs_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif
