// On-device basis diagnostics, computed from the Gram matrix
// G = V^T V of the final normalised basis (gram_kernel, the same G as the LOO):
//   ||S||_2,  S = (I + U)^{-1} U,  U = strictly upper part of G
//        (Paige's S: ||S||_2 = 1 exactly when orthogonality is lost)
//   sigma_min(V) = sqrt(lambda_min(G))  (reading R23 in DESIGN.md: the Gram route resolves
//        sigma_min to ~ c eps ||V||^2 / sigma_min absolute)
// Both eigenvalue problems are solved by a parallel cyclic Jacobi method on one CTA.
// Diagnostics only (once per solve), not on the iteration path.
#include <cuda_runtime.h>

#include <cstdint>

#include "igs_internal.cuh"

namespace igs {

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ double dsum(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(FULL, v, off);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double t = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(FULL, t, off);
        if (lane == 0) red[32] = t;
    }
    __syncthreads();
    return red[32];
}

// S = (I + U)^{-1} U, column j per CTA: s = U[:j, j], then column-oriented back substitution
// over k = j-1 .. 0 (unit diagonal): s_i -= U[i,k] s_k for i < k.  G is c x c (symmetric),
// S is written column-major (S[i + j c]); rows >= j of column j are 0.
__global__ void __launch_bounds__(128) smat_kernel(int c, const double* __restrict__ G, double* __restrict__ S) {
    extern __shared__ double sx[];
    const int j = blockIdx.x;
    for (int i = threadIdx.x; i < c; i += blockDim.x) sx[i] = i < j ? G[(int64_t)i * c + j] : 0.0;
    __syncthreads();
    for (int k = j - 1; k > 0; k--) {
        const double sk = sx[k];
        for (int i = threadIdx.x; i < k; i += blockDim.x) sx[i] = sx[i] - G[(int64_t)i * c + k] * sk;
        __syncthreads();
    }
    for (int i = threadIdx.x; i < c; i += blockDim.x) S[i + (int64_t)j * c] = sx[i];
}

// M = S^T S (c x c, column-major), 16 x 16 output tiles.
__global__ void __launch_bounds__(256) ata_kernel(int c, const double* __restrict__ S, double* __restrict__ M) {
    const int i = blockIdx.y * 16 + threadIdx.y, j = blockIdx.x * 16 + threadIdx.x;
    if (i >= c || j >= c) return;
    const double* si = S + (int64_t)i * c;
    const double* sj = S + (int64_t)j * c;
    double acc = 0.0;
    for (int k = 0; k < c; k++) acc = fma(si[k], sj[k], acc);
    M[i + (int64_t)j * c] = acc;
}

// Parallel cyclic Jacobi (round-robin pairs, Golub & Van Loan's symmetric Schur rotation) on
// a symmetric c x c matrix A (column-major, destroyed).  out[0] = lambda_min, out[1] =
// lambda_max.  Sweeps until the off-diagonal Frobenius norm is <= 1e-15 of ||A||_F.
constexpr int JT = 512;
__global__ void __launch_bounds__(JT) jacobi_eig_kernel(int c, double* A, double* out) {
    extern __shared__ double sj[];
    __shared__ double red[40];
    __shared__ int s_done;
    const int N = c + (c & 1);  // even; index c (if c odd) is a dummy
    const int np = N / 2;
    double* cs = sj;           // [np]
    double* sn = cs + np;      // [np]
    int* pp = reinterpret_cast<int*>(sn + np);  // [np]
    int* qq = pp + np;                          // [np]
    const int tid = threadIdx.x;
    double fro = 0.0;
    for (int64_t e = tid; e < (int64_t)c * c; e += JT) fro += A[e] * A[e];
    fro = dsum(fro, red);
    for (int sweep = 0; sweep < 60; sweep++) {
        double off = 0.0;
        for (int64_t e = tid; e < (int64_t)c * c; e += JT) {
            const int i = (int)(e % c), j = (int)(e / c);
            if (i != j) off += A[e] * A[e];
        }
        off = dsum(off, red);
        if (tid == 0) s_done = !(off > 1e-30 * fro);
        __syncthreads();
        if (s_done) break;
        for (int t = 0; t < N - 1; t++) {
            // pairs of this round: position 0 fixed, positions 1..N-1 rotate
            for (int k = tid; k < np; k += JT) {
                auto at = [&](int pos) { return pos == 0 ? 0 : 1 + (pos - 1 + t) % (N - 1); };
                int p = at(k), q = at(N - 1 - k);
                if (p > q) { const int tmp = p; p = q; q = tmp; }
                double cc = 1.0, ss = 0.0;
                if (q < c) {
                    const double apq = A[p + (int64_t)q * c];
                    if (apq != 0.0) {
                        const double app = A[p + (int64_t)p * c], aqq = A[q + (int64_t)q * c];
                        const double tau = (aqq - app) / (2.0 * apq);
                        const double tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        cc = 1.0 / sqrt(1.0 + tt * tt);
                        ss = tt * cc;
                    }
                } else {
                    q = -1;
                }
                pp[k] = p;
                qq[k] = q;
                cs[k] = cc;
                sn[k] = ss;
            }
            __syncthreads();
            // rows: A[p,:], A[q,:] <- J^T A
            for (int64_t w = tid; w < (int64_t)np * c; w += JT) {
                const int k = (int)(w / c), j = (int)(w % c);
                const int p = pp[k], q = qq[k];
                if (q < 0 || sn[k] == 0.0) continue;
                const double a = A[p + (int64_t)j * c], b = A[q + (int64_t)j * c];
                A[p + (int64_t)j * c] = cs[k] * a - sn[k] * b;
                A[q + (int64_t)j * c] = sn[k] * a + cs[k] * b;
            }
            __syncthreads();
            // columns: A[:,p], A[:,q] <- A J
            for (int64_t w = tid; w < (int64_t)np * c; w += JT) {
                const int k = (int)(w / c), i = (int)(w % c);
                const int p = pp[k], q = qq[k];
                if (q < 0 || sn[k] == 0.0) continue;
                const double a = A[i + (int64_t)p * c], b = A[i + (int64_t)q * c];
                A[i + (int64_t)p * c] = cs[k] * a - sn[k] * b;
                A[i + (int64_t)q * c] = sn[k] * a + cs[k] * b;
            }
            __syncthreads();
        }
    }
    if (tid == 0) {
        double lo = A[0], hi = A[0];
        for (int i = 1; i < c; i++) {
            const double d = A[i + (int64_t)i * c];
            lo = d < lo ? d : lo;
            hi = d > hi ? d : hi;
        }
        out[0] = lo;
        out[1] = hi;
    }
}

__global__ void diag_finish_kernel(const double* eigG, const double* eigM, double* out) {
    // out[0] = ||S||_2 = sqrt(lambda_max(S^T S)), out[1] = sigma_min(V) = sqrt(lambda_min(G))
    out[0] = sqrt(eigM[1] > 0.0 ? eigM[1] : 0.0);
    out[1] = sqrt(eigG[0] > 0.0 ? eigG[0] : 0.0);
}

}  // namespace

size_t basis_diag_doubles(int c) { return (size_t)3 * c * c + 8; }

// G (c x c, symmetric, unchanged); ws: basis_diag_doubles(c); out (device): [||S||_2, sigma_min]
void launch_basis_diag(int c, const double* G, double* ws, double* out, cudaStream_t s) {
    double* S = ws;
    double* M = S + (size_t)c * c;
    double* Gc = M + (size_t)c * c;
    double* eig = Gc + (size_t)c * c;  // [4]
    cudaMemcpyAsync(Gc, G, sizeof(double) * (size_t)c * c, cudaMemcpyDeviceToDevice, s);
    const size_t ssm = (size_t)c * sizeof(double);
    if (ssm > 48 * 1024) cudaFuncSetAttribute(smat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
    smat_kernel<<<c, 128, ssm, s>>>(c, G, S);
    dim3 tg((c + 15) / 16, (c + 15) / 16);
    ata_kernel<<<tg, dim3(16, 16), 0, s>>>(c, S, M);
    const int np = (c + 1) / 2;
    const size_t jsm = (size_t)np * (2 * sizeof(double) + 2 * sizeof(int));
    if (jsm > 48 * 1024) cudaFuncSetAttribute(jacobi_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)jsm);
    jacobi_eig_kernel<<<1, JT, jsm, s>>>(c, Gc, eig);
    jacobi_eig_kernel<<<1, JT, jsm, s>>>(c, M, eig + 2);
    diag_finish_kernel<<<1, 1, 0, s>>>(eig, eig + 2, out);
}

}  // namespace igs
