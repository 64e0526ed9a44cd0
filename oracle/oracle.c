/*
 * oracle.c -- plain FP64 CPU reference for the IGS-GMRES hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_2205_07805_b200/csrc) and the
 * product path never calls it.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n (the paper, arXiv 2205.07805);
 * S:n = SPEC.md line n; R# = a reading of a garbled/silent passage, listed in
 * DESIGN.md "Readings" (= SURVEY.md §8(c)).
 *
 * What is implemented, step by step in the paper's order (0-based Hessenberg columns):
 *   OR_MGS       textbook MGS-GMRES
 *   OR_IGS1      Algorithm 2 with Steps 14-16 removed: one Gauss-Seidel
 *                sweep = inverse compact WY MGS, reading R8
 *   OR_IGS2_TWO  Algorithm 2 literal, two sweeps, two reductions
 *   OR_IGS2_ONE  Algorithm 3, one reduction with readings R1-R4
 * plus the restarted driver and the Givens least-squares update.
 *
 * Arithmetic: IEEE FP64, compiled with -ffp-contract=off.  Every row operation is a
 * left-to-right loop.  Inner products follow a "reduction order knob":
 *   dot_block == 0 : sequential left-to-right sum over all n entries;
 *   dot_block == B : sequential sums of consecutive blocks of B entries, then a
 *                    sequential sum of the block sums (used to measure the parity
 *                    noise floor, SURVEY §8(c) "Parity noise floor");
 *   dot_block == -B: the same blocks, the block sums added pairwise (reading R27; the
 *                    c5 record, 134M rows).
 * All are deterministic for any OpenMP thread count.
 *
 * Parity pins (tests/test_oracle_*.py): dense LU on tiny systems, the Arnoldi
 * relation, O(eps) orthogonality for two sweeps, eps*kappa(B_k) for one sweep and MGS,
 * beta*kappa(B_k)=O(1), scipy gmres restart counts, paper special cases (Simoncini,
 * Walker, Embree), SPEC small examples.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { OR_MGS = 0, OR_IGS1 = 1, OR_IGS2_TWO = 2, OR_IGS2_ONE = 3 };
enum { OR_TERM_CONVERGED = 0, OR_TERM_MAXITER = 1, OR_TERM_BREAKDOWN = 2 };
enum { OR_OK = 0, OR_ERR_ARG = 1, OR_ERR_OOM = 4, OR_ERR_NONFINITE = 5 };

#define EPS 2.220446049250313e-16
/* reading R12: breakdown when gamma <= 64 eps sqrt(||h_col||^2 + gamma^2) */
#define BREAKDOWN_C 64.0

static int64_t g_block = 0; /* reduction order knob, see header */

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------------------- primitives --- */

/* y = A x, each row summed left to right in CSR order ("deterministic
 * summation order (fixed left-to-right per row)"). */
void oracle_spmv(int64_t n, const int64_t* rowptr, const int64_t* colind, const double* val,
                 const double* x, double* y) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double s = 0.0;
        for (int64_t q = rowptr[i]; q < rowptr[i + 1]; q++) s += val[q] * x[colind[q]];
        y[i] = s;
    }
}

/* sum of x[0..m) as a pairwise (binary) tree: halves added recursively */
static double pairwise_sum(const double* x, int64_t m) {
    if (m <= 8) {
        double s = 0.0;
        for (int64_t i = 0; i < m; i++) s += x[i];
        return s;
    }
    const int64_t h = m / 2;
    return pairwise_sum(x, h) + pairwise_sum(x + h, m - h);
}

/* a . b with the reduction-order knob: block == 0 (or >= n) one running sum; block > 0
 * running sums over blocks of `block` entries, the block sums added in order; block < 0
 * blocks of -block entries, the block sums added pairwise (reading R27: at n = 134M the
 * running sum over 32K block sums carries ~n_blocks eps of rounding into every inner
 * product, which then dominates the basis' loss of orthogonality). */
double oracle_dot(int64_t n, const double* a, const double* b, int64_t block) {
    const int pairwise = block < 0;
    if (block < 0) block = -block;
    if (block <= 0 || block >= n) {
        double s = 0.0;
        for (int64_t i = 0; i < n; i++) s += a[i] * b[i];
        return s;
    }
    int64_t nb = (n + block - 1) / block;
    double* part = (double*)malloc((size_t)nb * sizeof(double));
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < nb; q++) {
        int64_t i0 = q * block, i1 = i0 + block < n ? i0 + block : n;
        double s = 0.0;
        for (int64_t i = i0; i < i1; i++) s += a[i] * b[i];
        part[q] = s;
    }
    double s = 0.0;
    if (pairwise) s = pairwise_sum(part, nb);
    else
        for (int64_t q = 0; q < nb; q++) s += part[q];
    free(part);
    return s;
}

static double dot(int64_t n, const double* a, const double* b) { return oracle_dot(n, a, b, g_block); }

/* x = (I + L)^{-1} b by forward substitution in natural order ("triangular
 * solves with M = I + L ... are backward stable").  L is strictly lower,
 * column-major with leading dimension ldl; only L[i][j], j < i < order, is read. */
void oracle_forward_solve_unit(int order, const double* L, int ldl, const double* b, double* x) {
    for (int i = 0; i < order; i++) {
        double s = b[i];
        for (int j = 0; j < i; j++) s -= L[i + (int64_t)j * ldl] * x[j];
        x[i] = s;
    }
}

/* t = V[:, 0:p] c  (row-wise, columns in natural order) */
static void gemv_n(int64_t n, int p, const double* V, int64_t ldv, const double* c, double* t) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double s = 0.0;
        for (int j = 0; j < p; j++) s += V[i + (int64_t)j * ldv] * c[j];
        t[i] = s;
    }
}

/* exported for the fused-update parity test: t = V[:, 0:p] c */
void oracle_gemv(int64_t n, int p, const double* V, int64_t ldv, const double* c, double* t) {
    gemv_n(n, p, V, ldv, c, t);
}

/* ------------------------------------------------------- Givens least squares --- */
/* Progressive Givens QR of H: rotate column j, update g.  R is a copy of H
 * (ld = ldh) that receives the rotated column.  Rotation: d = hypot(a,b), c = a/d,
 * s = b/d (reading: standard rotation; SURVEY §8(c) "Least squares"). */
typedef struct {
    double *R, *cs, *sn, *g;
    int ldh;
} givens_t;

static void givens_column(givens_t* G, const double* H, int j) {
    double* Rj = G->R + (int64_t)j * G->ldh;
    const double* Hj = H + (int64_t)j * G->ldh;
    for (int i = 0; i <= j + 1; i++) Rj[i] = Hj[i];
    for (int i = 0; i < j; i++) {
        double a = Rj[i], b = Rj[i + 1];
        Rj[i] = G->cs[i] * a + G->sn[i] * b;
        Rj[i + 1] = -G->sn[i] * a + G->cs[i] * b;
    }
    double a = Rj[j], b = Rj[j + 1];
    double d = hypot(a, b);
    double c = 1.0, s = 0.0;
    if (d != 0.0) { c = a / d; s = b / d; }
    G->cs[j] = c; G->sn[j] = s;
    Rj[j] = d; Rj[j + 1] = 0.0;
    G->g[j + 1] = -s * G->g[j];
    G->g[j] = c * G->g[j];
}

/* y = R[:p,:p]^{-1} g[:p] by back substitution */
static void back_substitute(const givens_t* G, int p, double* y) {
    for (int i = p - 1; i >= 0; i--) {
        double s = G->g[i];
        for (int j = i + 1; j < p; j++) s -= G->R[i + (int64_t)j * G->ldh] * y[j];
        y[i] = s / G->R[i + (int64_t)i * G->ldh];
    }
}

/* Hessenberg least squares of S:250-263 as a standalone routine for the small pins:
 * H is (p+1) x p column-major, ldh >= p+1.  Returns y (p) and the residual |g_p|. */
double oracle_hessenberg_lsq(int p, const double* H, int ldh, double rho, double* y) {
    givens_t G;
    G.ldh = ldh;
    G.R = (double*)calloc((size_t)ldh * (p > 0 ? p : 1), sizeof(double));
    G.cs = (double*)calloc((size_t)p + 1, sizeof(double));
    G.sn = (double*)calloc((size_t)p + 1, sizeof(double));
    G.g = (double*)calloc((size_t)p + 1, sizeof(double));
    G.g[0] = rho;
    for (int j = 0; j < p; j++) givens_column(&G, H, j);
    back_substitute(&G, p, y);
    double res = fabs(G.g[p]);
    free(G.R); free(G.cs); free(G.sn); free(G.g);
    return res;
}

/* ------------------------------------------------------------------ workspace --- */
typedef struct {
    int64_t n;
    const int64_t *rowptr, *colind;
    const double* val;
    int m;          /* cycle length capacity */
    int ldh;        /* m + 1 */
    double* V;      /* n x (m+1) */
    double* H;      /* (m+1) x m */
    double* HP;     /* (m+1) x m  provisional columns of Alg. 3 (r^(4)) */
    double* L;      /* m x m strictly lower (ld = m) */
    double *z, *t, *u;
    double *a, *c, *r1, *r2, *r3, *tmp;
    givens_t G;
    /* outputs of one cycle */
    int p_done;     /* Hessenberg columns completed */
    int breakdown;
    int converged;
    int basis_cols; /* normalized columns of V */
    /* ledger */
    int64_t* ledger;   /* per global iteration: reductions */
    int64_t priming_reductions;
    /* history */
    double* res_hist;
    int t_global;      /* iterations completed so far */
    double nb;         /* ||b|| */
    double tol;
} ws_t;

static void record_iteration(ws_t* W, int j, int64_t nred) {
    /* column j completed and rotated: the Arnoldi residual |g_{j+1}| (R16) */
    W->t_global++;
    if (W->res_hist) W->res_hist[W->t_global] = fabs(W->G.g[j + 1]) / W->nb;
    if (W->ledger) W->ledger[W->t_global - 1] = nred;
}

static int converged_now(ws_t* W, int j) {
    return W->tol > 0.0 && fabs(W->G.g[j + 1]) <= W->tol * W->nb;
}

static int is_breakdown(const double* hcol, int len, double gamma) {
    double s = gamma * gamma;
    for (int i = 0; i < len; i++) s += hcol[i] * hcol[i];
    return !(gamma > BREAKDOWN_C * EPS * sqrt(s));
}

#define VCOL(W, j) ((W)->V + (int64_t)(j) * (W)->n)
#define HAT(W, i, j) ((W)->H[(i) + (int64_t)(j) * (W)->ldh])
#define HPAT(W, i, j) ((W)->HP[(i) + (int64_t)(j) * (W)->ldh])
#define LAT(W, i, j) ((W)->L[(i) + (int64_t)(j) * (W)->m])

/* Priming shared by Alg. 2 and Alg. 3 (reading R2):
 * rho = ||r||; v_0 = r/rho; z = A v_0; h = v_0.z; V[:,1] = z - h v_0 (pending).
 * Returns rho. */
static double prime(ws_t* W, const double* r, double* h_out) {
    int64_t n = W->n;
    double rho = sqrt(dot(n, r, r));
    double* v0 = VCOL(W, 0);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) v0[i] = r[i] / rho;
    oracle_spmv(n, W->rowptr, W->colind, W->val, v0, W->z);
    double h = dot(n, v0, W->z);
    double* v1 = VCOL(W, 1);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) v1[i] = W->z[i] - h * v0[i];
    W->priming_reductions += 2;
    *h_out = h;
    return rho;
}

/* ---------------------------------------------------------------- MGS cycle --- */
static void cycle_mgs(ws_t* W, const double* r, int m) {
    int64_t n = W->n;
    double rho = sqrt(dot(n, r, r));
    W->priming_reductions += 1;
    W->G.g[0] = rho;
    double* v0 = VCOL(W, 0);
    for (int64_t i = 0; i < n; i++) v0[i] = r[i] / rho;
    W->basis_cols = 1;
    for (int j = 0; j < m; j++) {
        double* w = W->z;
        oracle_spmv(n, W->rowptr, W->colind, W->val, VCOL(W, j), w);
        for (int i = 0; i <= j; i++) {            /* j+1 separate reductions */
            double h = dot(n, VCOL(W, i), w);
            HAT(W, i, j) = h;
            const double* vi = VCOL(W, i);
#pragma omp parallel for schedule(static)
            for (int64_t q = 0; q < n; q++) w[q] = w[q] - h * vi[q];
        }
        double gamma = sqrt(dot(n, w, w));        /* +1 reduction */
        HAT(W, j + 1, j) = gamma;
        int bd = is_breakdown(&HAT(W, 0, j), j + 1, gamma);
        givens_column(&W->G, W->H, j);
        record_iteration(W, j, (int64_t)j + 2);
        W->p_done = j + 1;
        if (bd) { W->breakdown = 1; return; }
        double* vn = VCOL(W, j + 1);
#pragma omp parallel for schedule(static)
        for (int64_t q = 0; q < n; q++) vn[q] = w[q] / gamma;
        W->basis_cols = j + 2;
        if (converged_now(W, j)) { W->converged = 1; return; }
    }
}

/* ----------------------------------------- Algorithm 2 (one or two sweeps) cycle --- */
static void cycle_alg2(ws_t* W, const double* r, int m, int sweeps) {
    int64_t n = W->n;
    double h;
    double rho = prime(W, r, &h);                 /* Steps 1-2 */
    W->G.g[0] = rho;
    HAT(W, 0, 0) = h;
    W->basis_cols = 1;
    for (int p = 1; p <= m; p++) {
        double* w = VCOL(W, p);                   /* w_{k-1}: pending, unnormalized */
        int drain = (p == m);
        if (!drain) oracle_spmv(n, W->rowptr, W->colind, W->val, w, W->z);   /* Step 4 */
        /* Steps 5-6: ONE reduction of 2(p+1) scalars [V_p^T w, w.w, V_{p+1}^T z] */
        for (int i = 0; i < p; i++) W->a[i] = dot(n, VCOL(W, i), w);
        double s = dot(n, w, w);
        if (!drain) for (int i = 0; i <= p; i++) W->c[i] = dot(n, VCOL(W, i), W->z);
        double gamma = sqrt(s);                   /* Step 6 */
        HAT(W, p, p - 1) = gamma;                 /* gamma_{k-1} = H_{k-1,k-2} */
        int bd = is_breakdown(&HAT(W, 0, p - 1), p, gamma);
        givens_column(&W->G, W->H, p - 1);
        record_iteration(W, p - 1, (int64_t)(drain ? 1 : sweeps));
        W->p_done = p;
        if (bd) { W->breakdown = 1; return; }
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) w[i] = w[i] / gamma;   /* Step 7 */
        W->basis_cols = p + 1;
        if (converged_now(W, p - 1) || drain) { W->converged = converged_now(W, p - 1); return; }
        for (int i = 0; i <= p; i++) W->c[i] = W->c[i] / gamma;   /* Step 8 */
        W->c[p] = W->c[p] / gamma;                                /* Step 9 (R5) */
        for (int i = 0; i < p; i++) LAT(W, p, i) = W->a[i] / gamma; /* Step 10 */
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) W->z[i] = W->z[i] / gamma; /* Step 11 */
        oracle_forward_solve_unit(p + 1, W->L, W->m, W->c, W->r1);  /* Step 12 */
        gemv_n(n, p + 1, W->V, n, W->r1, W->t);                     /* Step 13 */
        double* unew = VCOL(W, p + 1);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) unew[i] = W->z[i] - W->t[i];
        if (sweeps == 2) {
            for (int i = 0; i <= p; i++) W->r2[i] = dot(n, VCOL(W, i), unew); /* Step 14 */
            oracle_forward_solve_unit(p + 1, W->L, W->m, W->r2, W->r3);     /* Step 15 */
            gemv_n(n, p + 1, W->V, n, W->r3, W->t);                           /* Step 16 */
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < n; i++) unew[i] = unew[i] - W->t[i];
            for (int i = 0; i <= p; i++) HAT(W, i, p) = W->r1[i] + W->r3[i];  /* Step 17 */
        } else {
            for (int i = 0; i <= p; i++) HAT(W, i, p) = W->r1[i];             /* Step 17, r3 = 0 */
        }
    }
}

/* ------------------------------------------------------- Algorithm 3 cycle --- */
static void cycle_alg3(ws_t* W, const double* r, int m) {
    int64_t n = W->n;
    double h;
    double rho = prime(W, r, &h);                 /* Steps 1-2, reading R2 */
    W->G.g[0] = rho;
    HPAT(W, 0, 0) = h;
    W->basis_cols = 1;
    for (int p = 1; p <= m; p++) {
        double* u = VCOL(W, p);                   /* u_{k-1}: pending */
        int drain = (p == m);
        if (!drain) oracle_spmv(n, W->rowptr, W->colind, W->val, u, W->z);   /* A u_{k-1} */
        /* Step 4: ONE reduction [V_p, u]^T [u, z] -> r2, s, c, d (2(p+1) scalars) */
        for (int i = 0; i < p; i++) W->r2[i] = dot(n, VCOL(W, i), u);
        double s = dot(n, u, u);
        double d = 0.0;
        if (!drain) {
            for (int i = 0; i < p; i++) W->c[i] = dot(n, VCOL(W, i), W->z);
            d = dot(n, u, W->z);
        }
        /* Step 5: r3 = (I + L_p)^{-1} r2 */
        oracle_forward_solve_unit(p, W->L, W->m, W->r2, W->r3);
        /* Step 6: lagged norm gamma = sqrt(||u||^2 - ||r2||^2) */
        double nr2 = 0.0;
        for (int i = 0; i < p; i++) nr2 += W->r2[i] * W->r2[i];
        double tt = s - nr2;
        double gamma = tt > 0.0 ? sqrt(tt) : 0.0;
        /* Step 14: H[:p, p-1] = hp[:p, p-1] + r3 ; H[p, p-1] = gamma (reading R3) */
        for (int i = 0; i < p; i++) HAT(W, i, p - 1) = HPAT(W, i, p - 1) + W->r3[i];
        HAT(W, p, p - 1) = gamma;
        /* breakdown: t <= 0, cancellation guard t <= 64 eps s, or R12 */
        int bd = !(tt > BREAKDOWN_C * EPS * s) || is_breakdown(&HAT(W, 0, p - 1), p, gamma);
        givens_column(&W->G, W->H, p - 1);
        record_iteration(W, p - 1, 1);
        W->p_done = p;
        if (bd) { W->breakdown = 1; return; }
        /* Steps 10-11: v_{k-1} = (u - V_p r2) / gamma  (Jacobi sweep with r2) */
        gemv_n(n, p, W->V, n, W->r2, W->t);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) u[i] = (u[i] - W->t[i]) / gamma;
        W->basis_cols = p + 1;
        if (converged_now(W, p - 1) || drain) { W->converged = converged_now(W, p - 1); return; }
        /* Steps 7-8 */
        for (int i = 0; i < p; i++) W->c[i] = W->c[i] / gamma;
        d = d / (gamma * gamma);
        /* Step 9 (reading R4): L[p, :p] = r2 / gamma */
        for (int i = 0; i < p; i++) LAT(W, p, i) = W->r2[i] / gamma;
        /* Step 12 (Stephen's trick): r1 = [c ; d - L[p,:p] . c] */
        double acc = 0.0;
        for (int i = 0; i < p; i++) acc += LAT(W, p, i) * W->c[i];
        for (int i = 0; i < p; i++) W->r1[i] = W->c[i];
        W->r1[p] = d - acc;
        /* Step 13: u' = A u / gamma - V_{p+1} r1 */
        gemv_n(n, p + 1, W->V, n, W->r1, W->t);
        double* unew = VCOL(W, p + 1);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) unew[i] = W->z[i] / gamma - W->t[i];
        /* Step 15, derived (reading R1): hp[:p+1, p] = r1 - H[:p+1, :p] (r2 / gamma) */
        for (int i = 0; i < p; i++) W->tmp[i] = W->r2[i] / gamma;
        for (int i = 0; i <= p; i++) {
            double sacc = 0.0;
            for (int j = 0; j < p; j++) sacc += HAT(W, i, j) * W->tmp[j];
            HPAT(W, i, p) = W->r1[i] - sacc;
        }
    }
}

/* ------------------------------------------- Algorithm 1: IGS Gram-Schmidt QR --- */
/* Inverse compact WY two-reduce Gauss-Seidel Gram-Schmidt (Alg. 1), 0-based:
 * A is n x m column-major (lda), Q n x m (ldq), R m x m upper (ldr = m), L m x m strictly
 * lower (may be NULL), ledger[m] reductions per column (may be NULL).  sweeps = 2 is Alg. 1;
 * sweeps = 1 drops Steps 11-13 (one Gauss-Seidel iteration).  The norm of the
 * pending w_{k-1} (Step 5) is fused into the Step-4 reduction as in Alg. 2.
 * Reading R22: Step 7 divides only the entry of r^(0) that belongs to the just-normalised
 * q_{k-1} (w_{k-1}^T a_k / gamma); the printed r^(0)_{1:k-1,k} / gamma would scale the whole
 * R column and break A = QR (the full-vector division belongs to the Arnoldi variant, where
 * the new column is A w_{k-1} itself). */
int oracle_igs_qr(int64_t n, int m, const double* A, int64_t lda, int sweeps, int64_t dot_block,
                  double* Q, int64_t ldq, double* R, double* L_out, int64_t* ledger) {
    if (n <= 0 || m <= 0 || m > n || !A || !Q || !R || (sweeps != 1 && sweeps != 2)) return OR_ERR_ARG;
    g_block = dot_block;
    double* L = (double*)calloc((size_t)m * m, sizeof(double));
    double* r0 = (double*)calloc((size_t)m + 1, sizeof(double));
    double* r1 = (double*)calloc((size_t)m + 1, sizeof(double));
    double* r2 = (double*)calloc((size_t)m + 1, sizeof(double));
    double* r3 = (double*)calloc((size_t)m + 1, sizeof(double));
    double* t = (double*)malloc((size_t)n * sizeof(double));
    if (!L || !r0 || !r1 || !r2 || !r3 || !t) return OR_ERR_OOM;
    memset(R, 0, sizeof(double) * (size_t)m * m);
#define QC(j) (Q + (int64_t)(j) * ldq)
#define AC(j) (A + (int64_t)(j) * lda)
#define RR(i, j) R[(i) + (int64_t)(j) * m]
#define LL(i, j) L[(i) + (int64_t)(j) * m]
    /* Step 1: w_1 = a_1, R_11 = ||w_1||, q_1 = w_1 / R_11 */
    double r11 = sqrt(dot(n, AC(0), AC(0)));
    if (ledger) ledger[0] = 1;
    RR(0, 0) = r11;
    for (int64_t i = 0; i < n; i++) QC(0)[i] = AC(0)[i] / r11;
    if (m > 1) {
        /* Step 2: R_12 = q_1^T a_2, w_2 = a_2 - R_12 q_1 (pending in Q's column 2) */
        const double r12 = dot(n, QC(0), AC(1));
        if (ledger) ledger[1] = 1;
        RR(0, 1) = r12;
        for (int64_t i = 0; i < n; i++) QC(1)[i] = AC(1)[i] - r12 * QC(0)[i];
    }
    for (int k = 2; k <= m; k++) {                  /* paper k = 3..m (+ the drain k = m) */
        const int drain = (k == m);
        double* w = QC(k - 1);                        /* w_{k-1}, pending */
        /* Step 4 (+5): ONE reduction: L^T = Q_{k-2}^T w, ||w||^2, r0 = Q_{k-1}^T a_k */
        for (int i = 0; i < k - 1; i++) r2[i] = dot(n, QC(i), w);
        const double s = dot(n, w, w);
        if (!drain) for (int i = 0; i < k; i++) r0[i] = dot(n, QC(i), AC(k));
        const double gamma = sqrt(s);                 /* Step 5 */
        RR(k - 1, k - 1) = gamma;                     /* gamma_{k-1} = R_{k-1,k-1} */
        for (int64_t i = 0; i < n; i++) w[i] = w[i] / gamma;   /* Step 6 */
        if (drain) break;
        r0[k - 1] = r0[k - 1] / gamma;                /* Step 7 (reading R22) */
        for (int i = 0; i < k - 1; i++) LL(k - 1, i) = r2[i] / gamma;   /* Step 8 */
        oracle_forward_solve_unit(k, L, m, r0, r1);   /* Step 9 */
        gemv_n(n, k, Q, ldq, r1, t);                  /* Step 10: u_k = a_k - Q_{k-1} r1 */
        double* u = QC(k);
        for (int64_t i = 0; i < n; i++) u[i] = AC(k)[i] - t[i];
        if (sweeps == 2) {
            for (int i = 0; i < k; i++) r2[i] = dot(n, QC(i), u);   /* Step 11 (2nd reduction) */
            oracle_forward_solve_unit(k, L, m, r2, r3);           /* Step 12 */
            gemv_n(n, k, Q, ldq, r3, t);                          /* Step 13 */
            for (int64_t i = 0; i < n; i++) u[i] = u[i] - t[i];
        }
        for (int i = 0; i < k; i++) RR(i, k) = r1[i] + (sweeps == 2 ? r3[i] : 0.0);   /* Step 14 */
        if (ledger) ledger[k] = sweeps;
    }
#undef QC
#undef AC
#undef RR
#undef LL
    if (L_out) memcpy(L_out, L, sizeof(double) * (size_t)m * m);
    free(L); free(r0); free(r1); free(r2); free(r3); free(t);
    return OR_OK;
}

/* ----------------------------------------------------------------- driver --- */
/* SURVEY §8(c) "Driver".  Arrays: colind int64 (global columns), H_out (m1+1) x m1
 * column-major (first cycle, m1 = cycle capacity), res_hist [k+1], V_out n x (m1+1)
 * (last cycle, may be NULL), L_out m1 x m1 (last cycle, may be NULL), ledger [k] (may be
 * NULL).  info[0..7] = iters, cycles, term, h_cols(first cycle), basis_cols(last cycle),
 * priming reductions, status, p_last. */
int oracle_gmres(int64_t n, const int64_t* rowptr, const int64_t* colind, const double* val,
                 const double* b, const double* x0, int k, int restart, double tol, int variant,
                 int64_t dot_block, double* x, double* H_out, double* res_hist, double* V_out,
                 double* L_out, int64_t* ledger, int64_t* info, double* true_relres) {
    if (n <= 0 || k <= 0 || !rowptr || !colind || !val || !b || !x || variant < 0 || variant > 3)
        return OR_ERR_ARG;
    for (int64_t i = 0; i < n; i++) if (!isfinite(b[i])) return OR_ERR_NONFINITE;
    for (int64_t q = 0; q < rowptr[n]; q++) if (!isfinite(val[q])) return OR_ERR_NONFINITE;
    g_block = dot_block;
    int m1 = (restart > 0 && restart < k) ? restart : k;
    ws_t W;
    memset(&W, 0, sizeof W);
    W.n = n; W.rowptr = rowptr; W.colind = colind; W.val = val;
    W.m = m1; W.ldh = m1 + 1;
    /* the basis lives in the caller's V_out when given (storage only: a 108 GB basis, c5,
       is not held twice); zeroed like the calloc'd workspace */
    if (V_out) { memset(V_out, 0, sizeof(double) * (size_t)n * (m1 + 1)); W.V = V_out; }
    else W.V = (double*)calloc((size_t)n * (m1 + 1), sizeof(double));
    W.H = (double*)calloc((size_t)(m1 + 1) * m1, sizeof(double));
    W.HP = (double*)calloc((size_t)(m1 + 1) * m1, sizeof(double));
    W.L = (double*)calloc((size_t)m1 * m1, sizeof(double));
    W.z = (double*)malloc((size_t)n * sizeof(double));
    W.t = (double*)malloc((size_t)n * sizeof(double));
    W.u = (double*)malloc((size_t)n * sizeof(double));
    W.a = (double*)calloc(m1 + 2, sizeof(double));
    W.c = (double*)calloc(m1 + 2, sizeof(double));
    W.r1 = (double*)calloc(m1 + 2, sizeof(double));
    W.r2 = (double*)calloc(m1 + 2, sizeof(double));
    W.r3 = (double*)calloc(m1 + 2, sizeof(double));
    W.tmp = (double*)calloc(m1 + 2, sizeof(double));
    W.G.ldh = m1 + 1;
    W.G.R = (double*)calloc((size_t)(m1 + 1) * m1, sizeof(double));
    W.G.cs = (double*)calloc(m1 + 1, sizeof(double));
    W.G.sn = (double*)calloc(m1 + 1, sizeof(double));
    W.G.g = (double*)calloc(m1 + 2, sizeof(double));
    double* y = (double*)calloc(m1 + 1, sizeof(double));
    if (!W.V || !W.H || !W.HP || !W.L || !W.z || !W.t || !W.u || !W.G.R || !y) return OR_ERR_OOM;
    W.ledger = ledger;
    W.res_hist = res_hist;
    W.tol = tol;

    double* r = W.u;
    if (x0) memcpy(x, x0, (size_t)n * sizeof(double)); else memset(x, 0, (size_t)n * sizeof(double));
    W.nb = sqrt(dot(n, b, b));
    int total = 0, cycles = 0, term = OR_TERM_MAXITER, h_cols = 0;
    if (W.nb == 0.0) {
        memset(x, 0, (size_t)n * sizeof(double));
        if (res_hist) res_hist[0] = 0.0;
        term = OR_TERM_CONVERGED;
        *true_relres = 0.0;
        goto done;
    }
    for (;;) {
        /* r = b - A x : the true residual at cycle start */
        oracle_spmv(n, rowptr, colind, val, x, r);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) r[i] = b[i] - r[i];
        double rn = sqrt(dot(n, r, r));
        if (total == 0 && res_hist) res_hist[0] = rn / W.nb;
        if (tol > 0.0 && rn <= tol * W.nb) { term = OR_TERM_CONVERGED; break; }
        if (total >= k) { term = OR_TERM_MAXITER; break; }
        if (rn == 0.0) { term = OR_TERM_CONVERGED; break; }
        int m = k - total < m1 ? k - total : m1;
        memset(W.H, 0, sizeof(double) * (size_t)(m1 + 1) * m1);
        memset(W.HP, 0, sizeof(double) * (size_t)(m1 + 1) * m1);
        memset(W.L, 0, sizeof(double) * (size_t)m1 * m1);
        memset(W.G.g, 0, sizeof(double) * (size_t)(m1 + 2));
        W.p_done = 0; W.breakdown = 0; W.converged = 0; W.basis_cols = 0;
        switch (variant) {
            case OR_MGS: cycle_mgs(&W, r, m); break;
            case OR_IGS1: cycle_alg2(&W, r, m, 1); break;
            case OR_IGS2_TWO: cycle_alg2(&W, r, m, 2); break;
            case OR_IGS2_ONE: cycle_alg3(&W, r, m); break;
        }
        int p = W.p_done;
        if (cycles == 0) {
            h_cols = p;
            if (H_out) memcpy(H_out, W.H, sizeof(double) * (size_t)(m1 + 1) * m1);
        }
        /* y = argmin ||rho e1 - H y||, x += V_p y */
        back_substitute(&W.G, p, y);
        gemv_n(n, p, W.V, n, y, W.t);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) x[i] = x[i] + W.t[i];
        total += p;
        cycles++;
        if (W.breakdown) {
            oracle_spmv(n, rowptr, colind, val, x, r);
            for (int64_t i = 0; i < n; i++) r[i] = b[i] - r[i];
            term = OR_TERM_BREAKDOWN;
            break;
        }
    }
    /* r holds b - A x for the final x on every exit path */
    *true_relres = sqrt(dot(n, r, r)) / W.nb;
done:
    if (L_out) memcpy(L_out, W.L, sizeof(double) * (size_t)m1 * m1);
    if (info) {
        info[0] = total; info[1] = cycles; info[2] = term; info[3] = h_cols;
        info[4] = W.basis_cols; info[5] = W.priming_reductions; info[6] = OR_OK; info[7] = W.p_done;
    }
    if (W.V != V_out) free(W.V);
    free(W.H); free(W.HP); free(W.L); free(W.z); free(W.t); free(W.u);
    free(W.a); free(W.c); free(W.r1); free(W.r2); free(W.r3); free(W.tmp);
    free(W.G.R); free(W.G.cs); free(W.G.sn); free(W.G.g); free(y);
    return OR_OK;
}
