/*
 * igs.h -- C ABI of libigs: the B200 (sm_100a) hot path of IGS-GMRES
 * (Thomas, Carson, Rozloznik, Swirydowicz et al., arXiv 2205.07805).
 *
 * Citation keys: P:n = PAPER.md line n (the paper's LaTeX source); S:n = SPEC.md line n;
 * "Alg. 2" = Low-Synchronization Two-Reduce Iterated Gauss-Seidel GMRES;
 * "Alg. 3" = Low-Synch One-Reduce hybrid MGS-CGS GMRES;
 * R# = reading of a garbled/silent passage, listed in DESIGN.md "Readings".
 *
 * What one Arnoldi iteration does on the device (gs_iters = 2 -> Alg. 3; gs_iters = 1 ->
 * Alg. 2 Steps 1-13 + 17 with r^(3)=0, i.e. one Gauss-Seidel sweep, reading R8):
 *   z = A u                                   sparse matvec (Alg. 3 Step 4)
 *   [V_p, u]^T [u, z]  -> 2(p+1) scalars       ONE fused block dot
 *   sum of those 2(p+1) doubles over the ranks the single "Global Synchronization": fused
 *                                             into the block dot over NVLink peer memory (NCCL
 *                                             device API) by default, or one ncclAllReduce
 *   (I+L)^{-1} correction, lagged norm, Stephen's trick, Hessenberg column, Givens
 *   v_p = (u - V_p r2)/gamma ; u' = z/gamma - V_{p+1} r1   fused update
 *
 * Conventions (all entry points):
 *   - Status codes only; nothing throws or aborts across the ABI.  On a non-OK status,
 *     igs_last_error() returns a thread-local message.
 *   - All floating point is IEEE FP64.  Matrices are CSR: rowptr int64 (local offsets,
 *     rowptr[0] = 0), column indices 32- or 64-bit GLOBAL indices, strictly increasing per row.
 *   - Dense n x c blocks are column-major with leading dimension ld (elements).
 *   - The library copies the matrix at create; the caller keeps ownership of every array
 *     it passes.  The library owns its device state until igs_destroy.
 *   - Streams: all device work is enqueued on the cudaStream_t given at create (pass
 *     torch.cuda.current_stream().cuda_stream).  Calls return after their results are
 *     available to the caller (igs_solve synchronises the stream before returning).
 *   - Multi-GPU: one process per GPU; every rank calls create/solve/destroy collectively
 *     with identical (k, restart, tol, gs_iters).  Rank r owns rows
 *     [row_begin, row_begin + n_local) of A, of every n-vector and of the Krylov basis V.
 *   - There is no CPU fallback: without a CUDA device every compute call returns
 *     IGS_ERR_CUDA.
 */
#ifndef IGS_H
#define IGS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct igs_ctx igs_ctx; /* opaque; one per rank */

typedef enum {
    IGS_OK = 0,
    IGS_ERR_ARG = 1,       /* invalid argument (checked before any device work)          */
    IGS_ERR_CUDA = 2,      /* CUDA runtime error, or no CUDA device                     */
    IGS_ERR_NCCL = 3,      /* NCCL error                                                */
    IGS_ERR_OOM = 4,       /* device or host allocation failed                          */
    IGS_ERR_NONFINITE = 5, /* non-finite entry in A or b, or NaN during the solve */
    IGS_ERR_STATE = 6      /* call out of order (e.g. solve after a failed create)     */
} igs_status;

typedef enum { IGS_MEM_HOST = 0, IGS_MEM_DEVICE = 1 } igs_mem;

typedef enum {
    IGS_TERM_CONVERGED = 0, /* true relative residual <= tol                              */
    IGS_TERM_MAXITER = 1,   /* k Arnoldi iterations done                                 */
    IGS_TERM_BREAKDOWN = 2  /* (happy) breakdown: H[p,p-1] ~ 0 (reading R12) -- NOT an error */
} igs_term;

/* Algorithms of igs_solve_alg.  IGS_ALG_IGS1 and IGS_ALG_IGS2 are what igs_solve's gs_iters
 * 1 and 2 select; the other two are SURVEY §8(f) NEXT-1 / NEXT-3. */
typedef enum {
    IGS_ALG_IGS1 = 1,     /* Alg. 2 Steps 1-13 + 17, one Gauss-Seidel sweep: 1 reduction/iteration */
    IGS_ALG_IGS2 = 2,     /* Alg. 3, one-reduce hybrid MGS-CGS: 1 reduction/iteration */
    IGS_ALG_IGS2_TWO = 3, /* Alg. 2 literal, two sweeps: 2 reductions/iteration */
    IGS_ALG_MGS = 4       /* MGS-GMRES: j+2 reductions at column j */
} igs_alg;

/* Per-kernel timing classes (igs_kernel_stats). */
typedef enum {
    IGS_K_SPMV = 0,      /* z = A u (+ halo pack)                           */
    IGS_K_BLOCK_DOT = 1, /* fused [V_p,u]^T[u,z] incl. deterministic 2nd stage */
    IGS_K_ALLREDUCE = 2, /* ncclAllReduce of the 2(p+1) dots (G > 1)         */
    IGS_K_SMALL = 3,     /* replicated small step (trisolve, H, Givens)      */
    IGS_K_UPDATE = 4,    /* fused GEMV + axpy + lagged normalisation         */
    IGS_K_HALO = 5,      /* ncclSend/ncclRecv of ghost entries (G > 1)       */
    IGS_K_CYCLE = 6,     /* cycle end: y, x += V y, r = b - A x, ||r||       */
    IGS_K_PERSIST = 7,   /* persistent cycle kernel (small n, single GPU)   */
    IGS_K_COUNT = 8
} igs_kernel_kind;

/* Create a solver for this rank's row block of A.
 *   n_global    : global order n of A (square).
 *   row_begin   : first global row owned by this rank; n_local rows owned.
 *   rowptr      : int64[n_local+1], local offsets, rowptr[0] == 0, monotone.
 *   colind      : int32 or int64 [nnz_local] (colind_bits = 32 | 64), global columns in
 *                 [0, n_global), strictly increasing within each row.
 *   values      : double[nnz_local]; must be finite (else IGS_ERR_NONFINITE).
 *   where       : IGS_MEM_HOST or IGS_MEM_DEVICE for rowptr/colind/values.
 *   cuda_device : device ordinal this rank uses.
 *   nccl_unique_id : 128-byte ncclUniqueId from igs_nccl_unique_id() on rank 0, broadcast
 *                 by the caller (torch.distributed); NULL iff nranks == 1.
 *   rank, nranks: this rank and the world size; row blocks must tile [0, n_global) in rank
 *                 order (checked collectively).
 *   cuda_stream : cudaStream_t (as void*) for all device work; NULL = legacy default stream.
 * Collective over the ranks when nranks > 1.  */
igs_status igs_create(igs_ctx** out, int64_t n_global, int64_t row_begin, int64_t n_local,
                      const int64_t* rowptr, const void* colind, int colind_bits,
                      const double* values, int64_t nnz_local, igs_mem where, int cuda_device,
                      const void* nccl_unique_id, int rank, int nranks, void* cuda_stream);

/* Write a fresh ncclUniqueId (128 bytes) into out (rank 0 only). */
igs_status igs_nccl_unique_id(void* out128);

/* Device bytes a solve with this max cycle length (restart, or k if unrestarted) needs. */
size_t igs_workspace_bytes(const igs_ctx* ctx, int max_restart);

/* Optional: let the caller (torch) own the device workspace.  dev_ptr must be 256-byte
 * aligned and hold igs_workspace_bytes() bytes for every later solve's cycle length;
 * otherwise the library allocates with cudaMalloc on first use. */
igs_status igs_bind_workspace(igs_ctx* ctx, void* dev_ptr, size_t bytes);

typedef struct {
    double* x;             /* [n_local] out, caller-allocated, memory kind = vec_mem of igs_solve */
    double* H;             /* [(m+1)*m] host, col-major (ld = m+1), cycle-1 Hessenberg,
                              m = min(k, restart) (restart = 0 -> m = k); may be NULL      */
    double* res_hist;      /* [k+1] host: res_hist[0] = ||r0||/||b||, res_hist[t] = |g_t|/||b||,
                              the Givens-recurrence Arnoldi residual after iteration t
                              (reading R16); may be NULL                        */
    int want_loo;          /* in: compute ||I - V^T V||_F of the final basis         */
    double loo_frob;       /* out: NaN if !want_loo                                            */
    int iters;             /* out: total Arnoldi iterations (Hessenberg columns)              */
    int cycles;            /* out: restart cycles run                                         */
    igs_term term;         /* out                                                             */
    double true_relres;    /* out: ||b - A x|| / ||b|| recomputed at the end                  */
    int h_cols;            /* out: columns of H filled in cycle 1                             */
    int basis_cols;        /* out: normalised columns of the final basis (LOO is over these)  */
    int64_t allreduces;    /* out: NCCL allreduces issued by this solve (0 when nranks == 1)  */
    int64_t reductions;    /* out: global reductions (device block dots, each followed by one
                              allreduce when nranks > 1) executed by this solve -- the paper's
                              synchronization count.  After a convergence stop
                              the kernel-sequence path has already run the next iteration's
                              block dot (it overlaps the step that decides the stop): +1 there;
                              the persistent kernel (single GPU) counts completed iterations */
    double* lnorm_hist;    /* [k+1] host or NULL: ||L||_F of the algorithm's own correction
                              matrix L after iteration t (entries restart at each cycle;
                              lnorm_hist[0] = 0; NaN for MGS, which has no L).  gs_iters = 1
                              (Alg. 2 one sweep): L rows are a/gamma = the strictly lower part
                              of the computed basis' Gram V^T V, i.e. the paper's
                              L_k and dep^2(I+L_k) = ||L_k||_F^2.
                              gs_iters = 2 (Alg. 3): L rows are Step 9's r2/gamma, the
                              Gram of each vector BEFORE its second sweep (reading R4) -- not the
                              basis' Gram; lgram_frob below is the paper's L_k of the final
                              basis for every algorithm.                                      */
    int want_basis_diag;   /* in: compute s_norm and sigma_min of the final basis (NaN when it
                              has more than IGS_BASIS_DIAG_MAX columns)                       */
    double s_norm;         /* out: ||S||_2, S = (I + U)^{-1} U, U = strictly upper part of
                              V^T V (Paige's S; 1 when orthogonality is lost); NaN
                              if !want_basis_diag                                             */
    double sigma_min;      /* out: sigma_min(V) = sqrt(lambda_min(V^T V)) (reading R23); NaN
                              if !want_basis_diag                                             */
    double lgram_frob;     /* out: ||L_k||_F, L_k = strictly lower part of V^T V of the final
                              basis (dep^2(I+L_k)), from the same Gram as
                              loo_frob; NaN unless want_loo or want_basis_diag              */
} igs_result;

/* Solve A x = b by restarted IGS-GMRES.
 *   vec_mem  : memory kind of b, x0 and res->x (IGS_MEM_HOST: the library copies b/x0 in
 *              and x out inside the call; IGS_MEM_DEVICE: pointers into this rank's HBM).
 *   b        : [n_local] this rank's rows of the right-hand side (finite).
 *   x0       : [n_local] initial guess or NULL (= 0).
 *   k        : max total Arnoldi iterations, 1 <= k < n_global - 1.
 *   restart  : cycle length m; 0 or >= k => unrestarted.
 *   tol      : relative residual target ||b - A x|| <= tol ||b||; 0 => run exactly k
 *              iterations (unless breakdown).  Inside a cycle the Givens estimate |g_p|
 *              decides, at cycle start the true residual (SURVEY §8(c) "Driver").
 *   gs_iters : 1 (one Gauss-Seidel sweep, Alg. 2 minus Steps 14-16) or 2 (Alg. 3, one
 *              reduction per iteration; reading R7).
 * Breakdown is reported via res->term, not as an error. */
igs_status igs_solve(igs_ctx* ctx, igs_mem vec_mem, const double* b, const double* x0, int k,
                     int restart, double tol, int gs_iters, igs_result* res);

/* Same as igs_solve with an explicit algorithm (igs_alg); igs_solve(gs_iters = g) ==
 * igs_solve_alg(algorithm = g). */
igs_status igs_solve_alg(igs_ctx* ctx, igs_mem vec_mem, const double* b, const double* x0, int k,
                         int restart, double tol, int algorithm, igs_result* res);

/* Cumulative counters since create: NCCL allreduces, halo messages, Arnoldi iterations. */
igs_status igs_stats(const igs_ctx* ctx, int64_t* allreduces, int64_t* halo_msgs,
                     int64_t* iterations);

/* Per-kernel timing (CUDA events around every launch on the solver stream) -- off by
 * default; igs_set_timing(ctx, 1) enables it for later solves, and igs_kernel_stats
 * returns, for kind, the summed device milliseconds, the launch count and the summed
 * algorithmic bytes since the last reset (on = 2 resets). */
igs_status igs_set_timing(igs_ctx* ctx, int on);
igs_status igs_kernel_stats(const igs_ctx* ctx, int kind, double* ms, int64_t* launches,
                            double* bytes);

/* Facts about a context (for harnesses and tests): *value for key. */
typedef enum {
    IGS_INFO_XCHG = 0,             /* 1: reductions finish through the fused NVLink exchange
                                      (set up by the first solve), 0: ncclAllReduce / none */
    IGS_INFO_NRANKS = 1,           /* communicator size G                                   */
    IGS_INFO_NGHOST = 2,           /* ghost entries received per SpMV (halo, G > 1)         */
    IGS_INFO_NSEND = 3,            /* entries sent per SpMV                                 */
    IGS_INFO_NPEERS = 4,           /* halo peers                                            */
    IGS_INFO_NBND = 5,             /* boundary rows (multiplied after the halo)             */
    IGS_INFO_GRAPH_LAUNCHES = 6,   /* restart cycles replayed from CUDA graphs              */
    IGS_INFO_PCYCLE_LAUNCHES = 7,  /* restart cycles run by the persistent kernel           */
    IGS_INFO_SELL = 8,             /* 1: the SpMV uses the SELL-32 copy of A               */
    IGS_INFO_CSR_COMPACT = 9,      /* 1: the CSR arrays hold only the boundary rows         */
    IGS_INFO_SELL_DIAG_SLICES = 10,/* SELL slices stored as diagonal offsets (no column
                                      indices)                                */
    IGS_INFO_SELL_WALK = 11,       /* 1: every slice is diagonal and the SpMV is the kernel of
                                      resident warps walking slices          */
    IGS_INFO_SPMV_BYTES = 12,      /* bytes one SpMV launch streams in the stored format (SELL
                                      copy or CSR) incl. x and y; the byte model of the
                                      roofline keeps the CSR definition       */
    IGS_INFO_PCYCLE_ARES = 13      /* > 0: the last persistent-kernel cycle kept A in shared
                                      memory (value = CSR entries of the largest CTA share) */
} igs_info_key;
igs_status igs_info(const igs_ctx* ctx, int key, int64_t* value);

/* Failure detection.  With a communicator (nranks > 1, or the 1-rank test
 * communicators), every host wait of igs_create / igs_solve polls ncclCommGetAsyncError and
 * gives up after 2 x `seconds` without progress; the fused exchange's device barrier is
 * bounded by `seconds` (so a peer that stops arriving there is reported as a barrier
 * timeout, not as a host deadline).  Either failure aborts the communicator (ncclCommAbort) and returns
 * IGS_ERR_NCCL with the reason in igs_last_error(); later solves on the context return
 * IGS_ERR_STATE and only igs_destroy is valid.  Default 120 s (env IGS_NCCL_TIMEOUT_S at
 * create).  Test hook: env IGS_TEST_XCHG_STALL=c makes exchange number c wait for a peer
 * epoch that never arrives (exercises the device timeout on one GPU). */
igs_status igs_set_timeout(igs_ctx* ctx, double seconds);

igs_status igs_destroy(igs_ctx* ctx);
const char* igs_last_error(void);

/* ---------------------------------------------------------------------------------
 * Kernel-level entry points (device pointers, enqueue on `cuda_stream`, synchronise
 * before returning).  They run exactly the kernels igs_solve runs and exist so tests
 * can check each step against the oracle.  No context needed unless stated.
 * --------------------------------------------------------------------------------- */

/* out[0 : 2(p+1)] = [V_p^T u, u.u, V_p^T z, u.z]  (Alg. 3 Step 4), or with
 * z == NULL out[0 : p+1] = [V_p^T u, u.u].  V: n x p (ld >= n, ld even, 16-byte aligned),
 * u, z: n.  Deterministic (fixed two-stage reduction, no FP atomics). */
igs_status igs_op_block_dot(int64_t n, int p, const double* V, int64_t ld, const double* u,
                            const double* z, double* out, void* cuda_stream);

/* Measurement hook for the block dot above (same arguments and launch path): one warm-up
 * launch, then `reps` back-to-back launches timed with CUDA events on cuda_stream; *ms (host)
 * = mean milliseconds per launch.  Scratch is allocated outside the timed region.  Synchronises
 * cuda_stream.  Errors: IGS_ERR_ARG (bad sizes/alignment), IGS_ERR_CUDA / IGS_ERR_OOM. */
igs_status igs_bench_block_dot(int64_t n, int p, const double* V, int64_t ld, const double* u,
                               const double* z, double* out, int reps, float* ms, void* cuda_stream);

/* Measurement hook for the fused update below (same arguments, gamma by value): one warm-up,
 * then `reps` timed launches; *ms = mean milliseconds per launch.  Synchronises cuda_stream. */
igs_status igs_bench_update(int64_t n, int p, const double* V, int64_t ld, const double* u,
                            const double* z, const double* alpha, const double* beta, double gamma,
                            double* v_out, double* u_next, int reps, float* ms, void* cuda_stream);

/* y = A x with the context's (local, nranks == 1) matrix: x, y device [n_local]. */
igs_status igs_op_spmv(igs_ctx* ctx, const double* x, double* y);

/* Fused update:  w = u - V_p alpha (alpha == NULL -> w = u);
 *   v = w / gamma  written to v_out;  if u_next != NULL:
 *   u_next = z / gamma - (V_p beta[0:p] + v * beta[p]).
 * V: n x p (ld even), alpha: p, beta: p+1 (device). v_out may alias u. */
igs_status igs_op_update(int64_t n, int p, const double* V, int64_t ld, const double* u,
                         const double* z, const double* alpha, const double* beta, double gamma,
                         double* v_out, double* u_next, void* cuda_stream);

/* Algorithm 1 ("Inverse Compact WY Two-Reduce Gauss-Seidel Gram-Schmidt"):
 * A = Q R for a tall-skinny A (n x m, m <= n) on the solver's kernels.  All pointers device:
 * A (col-major, lda even >= n, 16-byte aligned, not modified), Q (out, n x m, ldq even >= n,
 * 16-byte aligned), R (out, m x m upper triangular, col-major, ld = m, positive diagonal).
 * sweeps = 2: two Gauss-Seidel iterations (two global reductions per column, O(eps) loss of
 * orthogonality); sweeps = 1: one (O(eps) kappa(A)).  Step 7 reading
 * R22.  *reductions (may be NULL) = block dots issued.  A (numerically) dependent
 * column -> IGS_ERR_NONFINITE.  Synchronises cuda_stream before returning. */
igs_status igs_qr(int64_t n, int m, const double* A, int64_t lda, double* Q, int64_t ldq, double* R,
                  int sweeps, int64_t* reductions, void* cuda_stream);

/* Largest basis the on-device ||S||_2 / sigma_min diagnostics accept (cyclic Jacobi on one
 * CTA is O(c^3) per sweep); igs_solve reports NaN for larger bases. */
#define IGS_BASIS_DIAG_MAX 1024

/* Basis diagnostics of a device block V (n x c, col-major, ld >= n; c <= IGS_BASIS_DIAG_MAX):
 * out3 (host) = [||I - V^T V||_F, ||S||_2, sigma_min(V)].  Same kernels
 * as igs_solve's want_loo / want_basis_diag.  Synchronises cuda_stream. */
igs_status igs_op_basis_diag(int64_t n, int c, const double* V, int64_t ld, double* out3, void* cuda_stream);

/* x = (I + L)^{-1} b by forward substitution; L strictly lower, col-major
 * order x order, ld = ldl (device); b, x device [order].  One CTA (the small-step solver). */
igs_status igs_op_trisolve(int order, const double* L, int ldl, const double* b, double* x,
                           void* cuda_stream);

/* ---------------------------------------------------------------------------------
 * Virtual ranks (test hook for the G > 1 halo path on ONE device).
 * igs_create_virtual builds out[0..nranks-1]: for each rank r the context igs_create would
 * build on GPU r for the row block [bounds[r], bounds[r+1]) of one global CSR (host
 * arrays: rowptr[n_global+1] global offsets, colind global columns, values), all on
 * cuda_device and stream cuda_stream, with the same halo plan (ghost map, send/receive
 * lists, boundary-row split) but no NCCL communicator.  igs_virtual_spmv then computes, for
 * every rank, y[r] = A_r x (b == NULL) or y[r] = b[r] - A_r x with x distributed as x[r]
 * (device, rank r's rows): it runs every rank's pack kernel into its send buffer, then each
 * rank's SpMV exactly as igs_solve does at G > 1 (interior rows while the ghosts arrive,
 * the boundary rows after them), the ghost entries copied from the owners' send buffers by
 * device copies instead of ncclSend/ncclRecv.  Virtual contexts reject igs_solve; destroy
 * each with igs_destroy.  Errors: IGS_ERR_ARG (bounds not spanning [0, n_global) in order,
 * contexts not one complete group in rank order), IGS_ERR_CUDA / IGS_ERR_OOM. */
igs_status igs_create_virtual(igs_ctx** out, int nranks, int64_t n_global, const int64_t* bounds,
                              const int64_t* rowptr, const void* colind, int colind_bits,
                              const double* values, int cuda_device, void* cuda_stream);
igs_status igs_virtual_spmv(igs_ctx* const* ctxs, int nranks, const double* const* x, double* const* y,
                            const double* const* b);
/* igs_virtual_solve runs igs_solve_alg(ctxs[r], IGS_MEM_DEVICE, b[r], NULL, k, restart, tol,
 * algorithm, &res[r]) for every member r of one virtual group at once -- one host thread and
 * one private stream per member -- i.e. the G > 1 solve of SURVEY §8(e) (row-block SpMV with
 * the halo overlapped with the interior rows, one cross-rank sum of the 2(p+1) dots per
 * iteration, replicated small state, uniform stops at the checkpoints) on a single device,
 * with the two NCCL transports emulated: the cross-rank sum stages every member's vector and
 * sums the G copies in member order (host barrier, cross-stream events, device copies; no
 * kernel ever waits on another member), the halo packs into the send buffers and copies the
 * ghosts from them.  The fused NVLink exchange, graphs and the persistent kernel are not
 * used (as at G > 1 without a symmetric window).  b[r] and res[r].x are rank r's rows
 * (device); every other igs_result field as for igs_solve.  Test hook for the one-GPU pool:
 * it checks the product's G > 1 control flow and numerics against the oracle, not NCCL.
 * Errors: as igs_solve, prefixed with the failing member; a member that fails releases the
 * others (IGS_ERR_STATE "a member failed") instead of leaving them at a barrier. */
igs_status igs_virtual_solve(igs_ctx* const* ctxs, int nranks, const double* const* b, int k, int restart,
                             double tol, int algorithm, igs_result* res);

/* ---------------------------------------------------------------------------------
 * Host-only halo planning (no device needed; used by igs_create and by CPU tests).
 * Phase 1: ghosts = sorted unique global columns of this block outside
 *   [row_begin, row_begin+n_local); ghost_owner_count[q] = ghosts owned by rank q, given
 *   the ownership boundaries bounds[0..nranks] (bounds[q] = first row of rank q).
 *   Returns the number of ghosts in *n_ghost; if ghosts != NULL it is filled (capacity
 *   must be >= *n_ghost from a first call with ghosts == NULL).
 * Phase 2: local_colind[nnz] = colind remapped to [0, n_local + n_ghost): local columns
 *   first, ghost g at n_local + g.  */
igs_status igs_plan_ghosts(int64_t row_begin, int64_t n_local, const int64_t* rowptr,
                           const void* colind, int colind_bits, int nranks,
                           const int64_t* bounds, int64_t* n_ghost, int64_t* ghosts,
                           int64_t* ghost_owner_count);
igs_status igs_plan_remap(int64_t row_begin, int64_t n_local, const int64_t* rowptr,
                          const void* colind, int colind_bits, int64_t n_ghost,
                          const int64_t* ghosts, int64_t* local_colind);

/* Host-only layout of the SELL-32 copy igs_create keeps of a short-row block (
 * the SpMV of P:1059 Step 4 reads it): slices of 32 rows; a slice whose rows use at most 8
 * distinct offsets c - r (every column local, increasing along each row) is "diagonal": its
 * ascending offset list is diag[8s..8s+7], the entry of row 32s+l with offset list[j] is
 * val[ptr[s] + 32j + l], present iff bit j of mask[32s+l]; any other slice is "explicit":
 * entry k of row 32s+l (CSR order) is val[ptr[s] + 32k + l] with column col[cptr[s] + 32k + l]
 * (cptr[s+1] == cptr[s] marks a diagonal slice).  len[r] = nonzeros of row r, 255 for the rows
 * listed in bnd_rows (ascending; G > 1 boundary rows: nothing stored).
 *   local_col: columns in the block's local space, int64; want_diag = 0 keeps every slice
 *   explicit.  Outputs (each may be NULL): ptr, cptr [ceil(n/32) + 1]; diag [8 ceil(n/32)];
 *   len, mask [32 ceil(n/32)]; val [cap_val]; col [cap_col].  *n_val, *n_col = entries the
 *   val / col arrays need (call once with val = col = NULL to size them), -1 when a row has
 *   >= 255 entries (no SELL copy is built); *n_diag = diagonal slices.  IGS_ERR_ARG on bad
 *   arguments or a capacity below the need.  No device is touched. */
igs_status igs_plan_sell(int64_t n, const int64_t* rowptr, const int64_t* local_col,
                         const double* values, int want_diag, int64_t n_bnd, const int64_t* bnd_rows,
                         int64_t* ptr, int64_t* cptr, int32_t* diag, uint8_t* len, uint8_t* mask,
                         int64_t cap_val, double* val, int64_t cap_col, int64_t* col,
                         int64_t* n_val, int64_t* n_col, int64_t* n_diag);

#ifdef __cplusplus
}
#endif
#endif /* IGS_H */
