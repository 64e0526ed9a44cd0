// igs_internal.cuh -- device-side state and kernel launchers of libigs (sm_100a).
// Nothing here is shared with oracle/ (the CPU reference); see DESIGN.md.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace igs {

// Device status word (istate[ST_STATUS]); every per-iteration kernel no-ops unless RUNNING.
enum : int { RUNNING = 0, STOP_CONVERGED = 1, STOP_BREAKDOWN = 2, STOP_END = 3, STOP_NONFINITE = 4 };
// istate slots
enum : int {
    ST_STATUS = 0,     // RUNNING / STOP_*
    ST_PDONE = 1,      // Hessenberg columns completed in this cycle
    ST_BASIS = 2,      // normalised basis columns
    ST_MODE = 3,       // update-kernel mode bits: 1 = write v_p, 2 = write u'
    ST_MODE_IT = 4,    // iteration index the mode bits belong to
    ST_CRITBD = 5,     // iteration at which the critical step saw a breakdown (else -1)
    ST_COUNT = 8
};
// scal slots (device doubles)
enum : int { SC_GAMMA = 0, SC_RHO = 1, SC_NB = 2, SC_TOL = 3, SC_ONE = 4, SC_T0 = 5, SC_LCUM = 6, SC_COUNT = 8 };

constexpr double kEps = 2.220446049250313e-16;
constexpr double kBreakdownC = 64.0;  // reading R12

// The replicated k x k state of one restart cycle (all device pointers).
struct Dev {
    int m;          // cycle capacity (columns of H)
    int ldh;        // m + 1
    int dld;        // stride between per-iteration dot vectors (>= 2(m+1))
    double* H;      // (m+1) x m, col-major, ld = ldh
    double* HP;     // (m+1) x m, Alg. 3 provisional column r^(4) (reading R1)
    double* L;      // m x m strictly lower, col-major, ld = m
    double* R;      // Givens-rotated copy of H, ld = ldh
    double* cs;     // [m] rotation cosines
    double* sn;     // [m] rotation sines
    double* g;      // [m+2] rotated rhs rho e1
    double* dots;   // [(m+1) * dld] reduced dot vector of iteration p at dots + p*dld
    double* alpha;  // [m+1] update coefficients (r^(2)) for v_p
    double* beta;   // [m+1] update coefficients (r^(1)) for u'
    double* y;      // [m+1] least-squares solution
    double* gam;    // [m+2] gamma of iteration p (written by crit, read by tail)
    double* dots2;  // [m+3] second reduction of Alg. 2 (two-reduce): V_{p+1}^T u
    double* r1h;    // [(m+1) x (m+2)] r1 of iteration p (row p): the tail of iteration p reads it
                    // while the critical step of p+1 already rewrites beta
    double* r3h;    // [(m+1) x (m+2)] r3 = (I+L_p)^{-1} r2 of iteration p, computed ahead of
                    // the tail by the persistent kernel's forward-substitution CTA (Alg. 3)
    double* cbd;    // [m+2] 1 if the critical step of iteration p saw a breakdown
    double* scal;   // [SC_COUNT]
    int* istate;    // [ST_COUNT]
    double* res_hist;  // [kmax+1]
    double* lnorm;     // [kmax+1] ||L||_F of the current cycle after iteration t
};

// ---- launchers (kernels.cu) -----------------------------------------------------------
struct SpmvArgs {
    int64_t nrows;
    const void* rowptr;  // int32 or int64 (ptr64)
    const void* col;     // int32 or int64 (idx64), local column space [0, nloc + nghost)
    const double* val;
    int ptr64, idx64, lpr;
    int64_t nloc;
    const double* ghost;  // NULL when no ghosts
    // SELL-32 copy of the same matrix (short rows; built by igs_create, IGS_SELL=0 disables):
    // slice s holds rows 32s..32s+31; entry k of row 32s+l at sell_ptr[s] + 32k + l, in the
    // CSR order of the row; rows shorter than the slice's longest are padded (never read)
    const int64_t* sell_ptr = nullptr;  // [nslices + 1]
    const uint8_t* sell_len = nullptr;  // [nrows] nonzeros of each row (<= 255)
    const double* sell_val = nullptr;
    const void* sell_col = nullptr;     // int32 or int64 (idx64), local column space
    // Diagonal slices: a slice whose rows use at most 8 distinct offsets
    // c - r (all columns local), each row's offsets strictly increasing in CSR order, keeps
    // no column indices: slice s lists its offsets in sell_diag[8s..8s+7] (ascending) and row
    // r's k-th entry has column r + sell_diag[8s + (k-th set bit of sell_mask[r])].  Other
    // slices store entry k of row 32s+l at sell_col[sell_cptr[s] + 32k + l]; a slice with
    // sell_cptr[s+1] == sell_cptr[s] stores no columns (diagonal, or no entries at all).
    const int64_t* sell_cptr = nullptr;  // [nslices + 1]
    const int32_t* sell_diag = nullptr;  // [nslices * 8]
    const uint8_t* sell_mask = nullptr;  // [nrows]
    int sell_kind = 0;                   // 0 mixed, 1 every slice diagonal, 2 none diagonal
    // every slice diagonal and nrows >= this: resident warps walking slices (spmv_sell_diag_kernel) (< 0: never)
    int64_t sell_walk_min_n = 262144;
    // G > 1: rows with a ghost column (sell_len == SELL_BOUNDARY, not in the SELL arrays),
    // multiplied by launch_spmv_rows once the halo has arrived.  With a SELL copy the CSR
    // arrays above hold only these rows (row t of the compact CSR is row bnd_rows[t])
    const int64_t* bnd_rows = nullptr;
    int64_t n_bnd = 0;
};
constexpr uint8_t SELL_BOUNDARY = 255;
// y[r] = (b[r] -) A[r,:] x for the rows in a.bnd_rows (CSR arrays, ghosts), left-to-right
void launch_spmv_rows(const SpmvArgs& a, const double* x, double* y, const double* b, bool resid,
                      const int* istate, cudaStream_t s);
// y = A x  (resid: y = b - A x).  istate may be NULL (no status check).
void launch_spmv(const SpmvArgs& a, const double* x, double* y, const double* b, bool resid,
                 const int* istate, cudaStream_t s);

// Persistent cycle kernel (kernels.cu): iterations 1..m of one Alg. 3 (gs = 2) or Alg. 2
// one-sweep (gs = 1) cycle in one cooperative launch, single GPU.  flags: 8 zeroed unsigned.
// ntri (Alg. 3): forward-substitution CTAs (1, or 2 taking alternate iterations).
cudaError_t launch_pcycle(const Dev& d, const SpmvArgs& a, double* V, int64_t ld, double* z, int64_t n,
                          int m, int gs, unsigned* flags, unsigned* counter, int grid, cudaStream_t s,
                          unsigned long long* prof = nullptr, double* part = nullptr, int xs = 0,
                          int ntri = 1, int* ares = nullptr);
// (*ares in: with xs, the most CSR entries any worker CTA owns -- pcycle_worker_ctas(grid, gs,
//  ntri) workers, warp w of CTA b taking rows w W + b, + 16 W, ... -- when A is to stay in
//  shared memory for the cycle; out: the value the launch used, 0 when it does not fit)
int pcycle_worker_ctas(int grid, int gs, int ntri);
constexpr int PCYCLE_WARPS = 16;
// (part != nullptr: row-block dots with grid x 2(m+1) partials, for larger n;
//  xs != 0: u staged in shared memory for the CSR phase A -- n <= pcycle_xs_max())
int64_t pcycle_xs_max();

// Fused block dot: out = [V_p^T u, u.u, V_p^T z, u.z] (z != NULL) or [V_p^T u, u.u].
// part: [grid * 2(p+1)] scratch, counter: one zeroed unsigned (reset by the kernel).
int bdot_grid_size(int64_t n, int num_sms);
struct XchgDev;  // xchg.cuh: fused cross-rank sum over NVLink (NCCL device API)
void launch_block_dot(int64_t n, int p, const double* V, int64_t ld, const double* u,
                      const double* z, double* out, double* part, unsigned* counter, int grid,
                      const int* istate, cudaStream_t s, const XchgDev* xc = nullptr);

// Fused update (see igs.h igs_op_update).  gamma read from *gamma_dev.
// istate/it: when istate != NULL the mode bits istate[ST_MODE] (valid iff
// istate[ST_MODE_IT] == it) select what is written; else mode = v (+ u' if u_next).
void launch_update(int64_t n, int p, const double* V, int64_t ld, const double* u,
                   const double* z, const double* alpha, const double* beta,
                   const double* gamma_dev, double* v_out, double* u_next, const int* istate,
                   int it, cudaStream_t s, const double* zdiv_dev = nullptr);

// x += V[:, :p] y with p = istate[ST_PDONE]
void launch_xupdate(int64_t n, const double* V, int64_t ld, const double* y, double* x,
                    const int* istate, int pmax, cudaStream_t s);

// Small steps (one CTA, replicated on every rank).
enum SmallStage : int { SS_PRIME_NORM = 0, SS_PRIME_H = 1, SS_CRIT = 2, SS_TAIL = 3, SS_LSQ = 4,
                        SS_CRIT2 = 5,      // Alg. 2 Steps 15, 17: r3 = (I+L)^{-1} r2, H += r3
                        SS_MGS_NORM = 6 }; // MGS: h_{j+1,j} = ||w||, Givens, status

// MGS step: h = dots[1] (v_i . z); H[i,j] = h; z -= h v_i  (one projection of modified GS)
void launch_mgs_axpy(int64_t n, const double* v, double* z, const double* hsrc, double* Hdst,
                     const int* istate, cudaStream_t s);
// Fused MGS step (kernels.cu): H[i,j] = *hsrc; z -= *hsrc v (v != NULL); *out = vn . z, or
// z . z when vn == NULL; deterministic, cross-rank sum fused when xc != NULL.  v, z, vn
// 16-byte aligned; part: >= grid + 1 doubles.
int mgs_step_grid(int64_t n, int num_sms);
void launch_mgs_step(int64_t n, const double* v, double* z, const double* vn, const double* hsrc,
                     double* Hdst, double* part, double* out, unsigned* counter, int grid,
                     const int* istate, const XchgDev* xc, cudaStream_t s);
// Alg. 2 two-reduce: first fused update + the second sweep's block dot in one pass over V_p
// (HBM) and an L2 re-read: out = [V_p^T u', v.u', u'.u']; part >= grid (p + 2) doubles.
int update_dot_grid(int64_t n, int num_sms);
int update_dot_tma_rows(int p);  // tile rows of the shared-memory variant, 0: p too large
void launch_update_dot_tma(int64_t n, int p, const double* V, int64_t ld, const double* u, const double* z,
                           const double* alpha, const double* beta, const double* gamma_dev, double* v_out,
                           double* u_next, const int* istate, int it, double* part, double* out,
                           unsigned* counter, int grid, const XchgDev* xc, cudaStream_t s);
size_t update_dot_smem(int p);
void launch_update_dot(int64_t n, int p, const double* V, int64_t ld, const double* u, const double* z,
                       const double* alpha, const double* beta, const double* gamma_dev, double* v_out,
                       double* u_next, const int* istate, int it, double* part, double* out,
                       unsigned* counter, int grid, const XchgDev* xc, cudaStream_t s);
void launch_small(const Dev& d, int stage, int gs, int p, int m, int t0, cudaStream_t s);

// Algorithm 1 (Gram-Schmidt QR) small steps; q.scal[0] = gamma, q.scal[1] = 1.
struct QrDev {
    double* R;      // m x m, col-major, ld = m
    double* L;      // m x m strictly lower, ld = m
    double* dots;   // [2 (m+1)]
    double* dots2;  // [m+1]
    double* alpha;  // [m+1]
    double* beta;   // [m+1]
    double* scal;   // [2]
};
enum QrStage : int { QR_S0 = 0, QR_S1 = 1, QR_CRIT = 2, QR_CRIT2 = 3 };
void launch_qr_small(const QrDev& q, int stage, int k, int m, cudaStream_t s);

// x = (I + L)^{-1} b (test entry point; same device routine as the small step).
void launch_trisolve(int order, const double* L, int ldl, const double* b, double* x,
                     cudaStream_t s);

// Gram matrix of V[:, :c] (local rows) into G (c x c) ; then ||I - G||_F into *out.
void launch_gram(int64_t n, int c, const double* V, int64_t ld, double* part, int splits,
                 double* G, cudaStream_t s);
void launch_loo_norm(int c, const double* G, double* out, cudaStream_t s);
// diag.cu: ||S||_2 (S = (I+U)^{-1} U, U = strictly upper part of G) and sigma_min(V) =
// sqrt(lambda_min(G)) from the Gram matrix G = V^T V (c x c); ws: basis_diag_doubles(c)
// doubles of device scratch; out (device): [||S||_2, sigma_min].
size_t basis_diag_doubles(int c);
void launch_basis_diag(int c, const double* G, double* ws, double* out, cudaStream_t s);

// halo pack: buf[i] = x[idx[i]]
void launch_pack(int64_t cnt, const int64_t* idx, const double* x, double* buf, const int* istate,
                 cudaStream_t s);

// small helpers
void launch_fill(double* p, int64_t n, double v, cudaStream_t s);
// out[i] = sum_q stage[q][i] in member order (igs_virtual_solve's emulated allreduce)
void launch_rank_sum(const double* const* stage, int G, int64_t count, double* out, cudaStream_t s);

}  // namespace igs
